"""Pin the CPU oracle (oracle/specdec_oracle.c) before trusting it.

The oracle is checked against (a) the committed golden fixtures produced by
the reference itself (tests/golden/make_golden.py) and (b) the reference
library compiled in place (oracle/_ref), live, on seeded random inputs.
"""
import os
import tempfile

import numpy as np
import pytest

from conftest import golden
import pyoracle as P


def cfg_from(g):
    c = g["config"]
    return dict(num_layers=int(c[0]), num_heads=int(c[1]), head_dim=int(c[2]), vocab_size=int(c[3]),
                max_positions=int(c[4]), init_seed=int(g["seed"][0]))


def split(flat, lens):
    out, at = [], 0
    for n in lens:
        out.append([int(x) for x in flat[at: at + n]])
        at += n
    return out


def test_oracle_weights_checksum_matches_reference_fixture(oracle):
    g = golden("c1_ems_trace.npz")
    m = oracle.model_init(cfg_from(g))
    assert oracle.checksum(m) == int(g["checksum"][0])
    oracle.model_free(m)
    g2 = golden("c2_shape_l2.npz")
    m = oracle.model_init(cfg_from(g2))
    assert oracle.checksum(m) == int(g2["checksum"][0])
    oracle.model_free(m)


def test_oracle_replays_c1_trace_bit_exact(oracle):
    """Every logits row of every C1 EMS step hashes identically to the reference."""
    g = golden("c1_ems_trace.npz")
    cfg = cfg_from(g)
    V, B = cfg["vocab_size"], len(g["prompt_lens"])
    m = oracle.model_init(cfg)
    c = oracle.cache_new(0, cfg["num_layers"], B, cfg["max_positions"], cfg["num_heads"] * cfg["head_dim"])
    prompts = split(g["prompts"], g["prompt_lens"])
    oracle.forward(m, c, prompts, [(s, i) for s in range(B) for i in range(len(prompts[s]))], V)
    for s in range(B):
        oracle.commit(c, s, len(prompts[s]))
    at_tok = at_row = 0
    logits_seen = []
    for step, T in enumerate(g["step_T"]):
        counts = g["step_counts"][step]
        taus = g["step_tau"][step]
        n_s = [(1 + counts[s]) if taus[s] > 0 else 0 for s in range(B)]
        per = split(g["step_tokens"][at_tok: at_tok + T], n_s)
        slots = [(s, oracle.committed(c, s) + o) for s in range(B) for o in range(n_s[s])]
        lg, am = oracle.forward(m, c, per, slots, V)
        assert (P.fnv_rows(lg) == g["step_fnv"][at_row: at_row + T]).all(), f"step {step}"
        assert (am == g["step_argmax"][at_row: at_row + T]).all()
        logits_seen.append(lg)
        for s in range(B):
            if taus[s]:
                oracle.commit(c, s, int(taus[s]))
        assert [oracle.committed(c, s) for s in range(B)] == g["step_committed"][step].tolist()
        at_tok += T
        at_row += T
    ref_logits = g["logits"]
    ours = np.concatenate(logits_seen)[: len(ref_logits)]
    assert np.array_equal(ours.view(np.uint32), ref_logits.view(np.uint32))
    oracle.cache_free(c)
    oracle.model_free(m)


@pytest.mark.parametrize("name", ["c1_ems_decode", "c1_vanilla_decode"] +
                         [f"engine_{p}_{m}" for p in ("draft", "retrieval", "synthetic")
                          for m in ("greedy", "vanilla", "ems")])
def test_oracle_decode_matches_reference_fixture(oracle, name):
    g = golden(name + ".npz")
    cfg = cfg_from(g)
    e = g["engine"]
    ecfg = dict(mode=int(e[0]), predictor=int(e[1]), k=int(e[2]), match_len=int(e[3]), copy_len=int(e[4]),
                batch_size=int(e[5]), max_new_tokens=int(e[6]), stop_on_eos=int(e[7]), seed=int(g["engine_seed"][0]),
                synthetic_accuracy=float(g["accuracy"][0]))
    m = oracle.model_init(cfg)
    d = None
    if "draft_config" in g:
        d = oracle.model_init(cfg_from({"config": g["draft_config"], "seed": g["draft_seed"]}))
    prompts = [P.tokenize_prompt(t) for t in P.CORPUS[: ecfg["batch_size"]]]
    toks, rec, ledger = oracle.decode(ecfg, m, prompts, d)
    for s in range(ecfg["batch_size"]):
        n = int(g["gen_counts"][s])
        assert toks[s] == g["generated"][s, :n].tolist()
    if ecfg["mode"] != 0:
        assert np.array_equal(rec[:, :5], g["records"])
        assert ledger.tolist() == g["ledger"].tolist()
    oracle.model_free(m)
    if d:
        oracle.model_free(d)


def test_oracle_ragged_acceptance_batches_bit_exact(oracle):
    """acceptance.cpp check 8: 100 ragged batches (plain and split into two chunks)."""
    g = golden("ragged_acceptance8.npz")
    cfg = cfg_from(g)
    m = oracle.model_init(cfg)
    seqs_all = split(g["tokens"], g["lens"])
    at_seq = at_mid = at_row = 0
    for trial, b in enumerate(g["batch"]):
        seqs = seqs_all[at_seq: at_seq + b]
        at_seq += b
        c = oracle.cache_new(0, 2, int(b), 64, 16)
        if not g["split"][trial]:
            lg, _ = oracle.forward(m, c, seqs, [(s, i) for s in range(b) for i in range(len(seqs[s]))], 259)
        else:
            mids = g["mids"][at_mid: at_mid + b].tolist()
            heads = [q[:md] for q, md in zip(seqs, mids)]
            tails = [q[md:] for q, md in zip(seqs, mids)]
            lh, _ = oracle.forward(m, c, heads, [(s, i) for s in range(b) for i in range(len(heads[s]))], 259)
            for s in range(b):
                oracle.commit(c, s, mids[s])
            lt, _ = oracle.forward(m, c, tails, [(s, mids[s] + i) for s in range(b) for i in range(len(tails[s]))],
                                   259)
            parts, ah, at = [], 0, 0
            for s in range(b):
                parts += [lh[ah: ah + len(heads[s])], lt[at: at + len(tails[s])]]
                ah += len(heads[s])
                at += len(tails[s])
            lg = np.concatenate(parts)
        at_mid += b
        n = sum(len(q) for q in seqs)
        assert (P.fnv_rows(lg) == g["row_fnv"][at_row: at_row + n]).all(), f"trial {trial}"
        at_row += n
        oracle.cache_free(c)
    oracle.model_free(m)


def test_oracle_c2_shape_bit_exact(oracle):
    """OPT-125m-shaped layers (h=768, hd=64, V=50272), L=2: prefill + one verify step."""
    g = golden("c2_shape_l2.npz")
    cfg = cfg_from(g)
    V, B = cfg["vocab_size"], len(g["prompt_lens"])
    m = oracle.model_init(cfg)
    c = oracle.cache_new(0, 2, B, 256, 768)
    prompts = split(g["prompts"], g["prompt_lens"])
    lp, _ = oracle.forward(m, c, prompts, [(s, i) for s in range(B) for i in range(len(prompts[s]))], V)
    assert (P.fnv_rows(lp) == g["prefill_fnv"]).all()
    for s in range(B):
        oracle.commit(c, s, len(prompts[s]))
    drafts = split(g["drafts"], g["draft_counts"])
    per = [[int(g["last"][s])] + drafts[s] for s in range(B)]
    ls, am = oracle.forward(m, c, per, [(s, len(prompts[s]) + o) for s in range(B) for o in range(len(per[s]))], V)
    assert (P.fnv_rows(ls) == g["step_fnv"]).all()
    assert (am == g["step_argmax"]).all()
    oracle.cache_free(c)
    oracle.model_free(m)


# ------------------------------------------------- live reference comparisons
def test_oracle_weights_equal_reference_live(oracle, reference):
    for seed in (0xD5EED, 123, 0x10EA):
        cfg = dict(P.DEFAULT_CONFIG, init_seed=seed, num_layers=1 + seed % 3)
        mo, mr = oracle.model_init(cfg), reference.model_init(cfg)
        assert np.array_equal(oracle.weights(mo).view(np.uint32), reference.weights(mr).view(np.uint32))
        assert oracle.checksum(mo) == reference.checksum(mr)
        oracle.model_free(mo)
        reference.model_free(mr)


def test_checkpoint_interop_with_reference(oracle, reference):
    """SDCK v1 written by one side loads bit-identically on the other (model.cpp:143-221)."""
    cfg = dict(P.DEFAULT_CONFIG, init_seed=0xC0FFEE)
    with tempfile.TemporaryDirectory() as d:
        mo = oracle.model_init(cfg)
        oracle.model_save(mo, os.path.join(d, "o.bin"))
        mr = reference.model_load(os.path.join(d, "o.bin"))
        assert reference.checksum(mr) == oracle.checksum(mo)
        reference.model_save(mr, os.path.join(d, "r.bin"))
        with open(os.path.join(d, "o.bin"), "rb") as a, open(os.path.join(d, "r.bin"), "rb") as b:
            assert a.read() == b.read()
        # damaged files: truncated / trailing bytes / bad magic -> IoError (code 4)
        raw = open(os.path.join(d, "o.bin"), "rb").read()
        for bad in (raw[:-40], raw + b"extra", b"not a checkpoint at all"):
            open(os.path.join(d, "bad.bin"), "wb").write(bad)
            with pytest.raises(P.SpecdecError) as e:
                oracle.model_load(os.path.join(d, "bad.bin"))
            assert e.value.code == 4
        oracle.model_free(mo)
        reference.model_free(mr)


def test_oracle_random_ragged_forwards_match_reference_live(oracle, reference):
    rng = np.random.default_rng(0x5EED)
    cfg = dict(num_layers=2, num_heads=3, head_dim=8, vocab_size=97, max_positions=96, init_seed=99)
    mo, mr = oracle.model_init(cfg), reference.model_init(cfg)
    for trial in range(12):
        b = int(rng.integers(1, 5))
        co = oracle.cache_new(0, 2, b, 96, 24)
        cr = reference.cache_new(0, 2, b, 96, 24)
        committed = [0] * b
        for chunk in range(3):
            per = [rng.integers(0, 97, size=int(rng.integers(0, 6))).tolist() for _ in range(b)]
            if sum(map(len, per)) == 0:
                per[0] = [5]
            slots = [(s, committed[s] + o) for s in range(b) for o in range(len(per[s]))]
            lo, _ = oracle.forward(mo, co, per, slots, 97)
            lr = reference.forward(mr, cr, per, slots, 97)
            assert np.array_equal(lo.view(np.uint32), lr.view(np.uint32))
            for s in range(b):
                if per[s]:
                    tau = int(rng.integers(1, len(per[s]) + 1))
                    oracle.commit(co, s, tau)
                    reference.commit(cr, s, tau)
                    committed[s] += tau
        oracle.cache_free(co)
        reference.cache_free(cr)
    oracle.model_free(mo)
    reference.model_free(mr)


def test_oracle_restore_and_retrieval_match_reference(oracle, reference):
    rng = np.random.default_rng(0x5107)
    for _ in range(300):
        counts = rng.integers(0, 7, size=int(rng.integers(1, 12))).tolist()
        total = sum(counts)
        for flat in range(total + 1):
            try:
                a = oracle.restore_indices(counts, flat)
            except P.SpecdecError as e:
                a = ("err", e.code)
            import ctypes as C
            s, p = C.c_int32(), C.c_int32()
            rc = reference.lib.ref_restore_indices(np.asarray(counts, np.int32), len(counts), flat, C.byref(s),
                                                   C.byref(p))
            b = ("err", rc) if rc else (s.value, p.value)
            assert a == b
        ctx = rng.integers(3, 9, size=int(rng.integers(0, 40))).tolist()
        for match_len, copy_len in ((1, 3), (2, 7), (3, 4)):
            assert oracle.retrieval_predict(ctx, match_len, copy_len) == reference.retrieval_predict(ctx, match_len,
                                                                                                    copy_len)
