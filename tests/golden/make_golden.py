"""Generate the committed golden fixtures from the REFERENCE itself.

Runs only in the build container (needs oracle/_ref/libspecdec_ref.so, the
unmodified reference compiled in place by oracle/Makefile).  Every fixture is
produced through the reference's public API (Model::init/forward, verify,
UnpadArena::commit_accepted, retrieval_predict, decode_speculative) via
oracle/ref_shim.cpp.  Outputs: tests/golden/*.npz.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as P  # noqa: E402


def fnv1a(b: bytes) -> int:
    h = 14695981039346656037
    for x in b:
        h ^= x
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def fnv_rows(logits: np.ndarray) -> np.ndarray:
    return np.array([fnv1a(np.ascontiguousarray(r, dtype=np.float32).tobytes()) for r in logits], dtype=np.uint64)


def ems_trace(ref: P.Reference, cfg: dict, prompts_text: list[str], copy_len: int, budget: int,
              keep_logit_steps: int) -> dict:
    """engine.cpp:291-489 EMS branch with the retrieval predictor, driven step by
    step through the reference API so every intermediate is recorded."""
    m = ref.model_init(cfg)
    V, L, h = cfg["vocab_size"], cfg["num_layers"], cfg["num_heads"] * cfg["head_dim"]
    B = len(prompts_text)
    prompts = [P.tokenize_prompt(t) for t in prompts_text]
    c = ref.cache_new(0, L, B, cfg["max_positions"], h)
    slots = [(s, i) for s in range(B) for i in range(len(prompts[s]))]
    lg = ref.forward(m, c, prompts, slots, V)
    rows = np.cumsum([len(p) for p in prompts]) - 1
    for s in range(B):
        ref.commit(c, s, len(prompts[s]))
    toks = [list(p) + [int(np.argmax(lg[rows[s]]))] for s, p in enumerate(prompts)]
    gen = [1] * B
    rec = dict(step_tokens=[], step_T=[], step_counts=[], step_tau=[], step_argmax=[], step_committed=[],
               step_fnv=[], logits=[])
    step = 0
    while any(g < budget for g in gen):
        active = [g < budget for g in gen]
        per, counts, drafts = [], [], []
        for s in range(B):
            d = ref.retrieval_predict(toks[s], 2, copy_len) if active[s] else []
            drafts.append(d)
            per.append(([toks[s][-1]] + d) if active[s] else [])
            counts.append(len(d) if active[s] else 0)
        sl = []
        for s in range(B):
            cm = ref.committed(c, s)
            sl += [(s, cm + o) for o in range(len(per[s]))]
        lg = ref.forward(m, c, per, sl, V)
        am = lg.argmax(axis=1).astype(np.int32)
        taus = []
        at = 0
        for s in range(B):
            if not active[s]:
                taus.append(0)
                continue
            k = len(drafts[s])
            acc, tau = [], k + 1
            for j in range(k + 1):
                x = int(am[at + j])
                acc.append(x)
                if j < k and x != drafts[s][j]:
                    tau = j + 1
                    break
            tau = min(tau, budget - gen[s])
            toks[s] += acc[:tau]
            gen[s] += tau
            ref.commit(c, s, tau)
            taus.append(tau)
            at += len(per[s])
        rec["step_tokens"] += [t for p in per for t in p]
        rec["step_T"].append(len(am))
        rec["step_counts"].append(counts)
        rec["step_tau"].append(taus)
        rec["step_argmax"] += am.tolist()
        rec["step_committed"].append([ref.committed(c, s) for s in range(B)])
        rec["step_fnv"] += fnv_rows(lg).tolist()
        if step < keep_logit_steps:
            rec["logits"].append(lg)
        step += 1
    out = {k: np.array(v, dtype=np.int32) for k, v in rec.items() if k not in ("logits", "step_fnv")}
    out["step_fnv"] = np.array(rec["step_fnv"], dtype=np.uint64)
    out["logits"] = np.concatenate(rec["logits"]).astype(np.float32)
    out["generated"] = np.array([t[len(p):] for t, p in zip(toks, prompts)], dtype=np.int32)
    out["prompts"] = np.array([t for p in prompts for t in p], dtype=np.int32)
    out["prompt_lens"] = np.array([len(p) for p in prompts], dtype=np.int32)
    out["checksum"] = np.array([ref.checksum(m)], dtype=np.uint64)
    out["config"] = P.dims_of(cfg)
    out["seed"] = np.array([cfg["init_seed"]], dtype=np.uint64)
    # self-check against the reference's own decode loop
    js = ref.decode(P.engine_config(mode=2, predictor=1, copy_len=copy_len, batch_size=B, max_new_tokens=budget,
                                    stop_on_eos=0), m, prompts_text)
    for s in range(B):
        assert js["outputs"][s]["tokens"] == out["generated"][s].tolist(), "trace diverged from decode_speculative"
    ref.cache_free(c)
    ref.model_free(m)
    return out


def decode_fixture(ref: P.Reference, cfg: dict, ecfg: dict, prompts_text: list[str], draft_cfg=None) -> dict:
    m = ref.model_init(cfg)
    d = ref.model_init(draft_cfg) if draft_cfg else None
    js = ref.decode(ecfg, m, prompts_text, d)
    B = ecfg["batch_size"]
    gen = np.full((B, max(ecfg["max_new_tokens"], 1)), -1, dtype=np.int32)
    for s in range(B):
        t = js["outputs"][s]["tokens"]
        gen[s, : len(t)] = t
    recs = [(i, x["sample"], x["k"], x["tau"], int(x["clipped"])) for i, st in enumerate(js["steps"])
            for x in st["samples"]]
    out = dict(
        generated=gen,
        gen_counts=np.array([len(js["outputs"][s]["tokens"]) for s in range(B)], dtype=np.int32),
        records=np.array(recs, dtype=np.int32).reshape(-1, 5),
        ledger=np.array([js["metrics"]["useful_kv_writes"], js["metrics"]["padding_kv_writes"]], dtype=np.int64),
        avg_acceptance_length=np.array([js["metrics"]["avg_acceptance_length"]]),
        avg_padding_ratio=np.array([js["metrics"]["avg_padding_ratio"]]),
        engine=np.array([ecfg[k] for k in ("mode", "predictor", "k", "match_len", "copy_len", "batch_size",
                                           "max_new_tokens", "stop_on_eos")], dtype=np.int32),
        engine_seed=np.array([ecfg["seed"]], dtype=np.uint64),
        accuracy=np.array([ecfg["synthetic_accuracy"]]),
        config=P.dims_of(cfg),
        seed=np.array([cfg["init_seed"]], dtype=np.uint64),
    )
    if draft_cfg:
        out["draft_config"] = P.dims_of(draft_cfg)
        out["draft_seed"] = np.array([draft_cfg["init_seed"]], dtype=np.uint64)
    ref.model_free(m)
    if d:
        ref.model_free(d)
    return out


def ragged_fixture(ref: P.Reference) -> dict:
    """acceptance.cpp:364-445 (check 8): 100 random ragged batches, seed 0x8A66ED."""
    cfg = dict(num_layers=2, num_heads=2, head_dim=8, vocab_size=259, max_positions=64, init_seed=0x0A0C)
    m = ref.model_init(cfg)
    V = 259
    st = np.uint64(0x8A66ED)

    class Rng:
        def __init__(self, seed):
            self.s = seed

        def next(self):
            self.s = (self.s + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
            z = self.s
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
            return z ^ (z >> 31)

    rng = Rng(int(st))
    seqs, splits, mids, fnvs, argm = [], [], [], [], []
    for trial in range(100):
        b = 1 + rng.next() % 4
        sequences = []
        for _ in range(b):
            ln = 2 + rng.next() % 24
            sequences.append([int(rng.next() % V) for _ in range(ln)])
        split = (rng.next() & 1) != 0
        c = ref.cache_new(0, 2, b, 64, 16)
        if not split:
            slots = [(s, i) for s in range(b) for i in range(len(sequences[s]))]
            lg = ref.forward(m, c, sequences, slots, V)
            trial_mids = [0] * b
        else:
            trial_mids = [1 + int(rng.next() % (len(q) - 1)) for q in sequences]
            heads = [q[:md] for q, md in zip(sequences, trial_mids)]
            tails = [q[md:] for q, md in zip(sequences, trial_mids)]
            lh = ref.forward(m, c, heads, [(s, i) for s in range(b) for i in range(len(heads[s]))], V)
            for s in range(b):
                ref.commit(c, s, trial_mids[s])
            lt = ref.forward(m, c, tails, [(s, trial_mids[s] + i) for s in range(b) for i in range(len(tails[s]))],
                             V)
            parts, ah, at = [], 0, 0
            for s in range(b):
                parts.append(lh[ah: ah + len(heads[s])])
                ah += len(heads[s])
                parts.append(lt[at: at + len(tails[s])])
                at += len(tails[s])
            lg = np.concatenate(parts)
        # naive full-recompute oracle (naive_model.cpp) must agree within 1e-5
        at = 0
        for s in range(b):
            nv = ref.naive_forward(m, sequences[s], V)
            assert np.max(np.abs(nv - lg[at: at + len(nv)])) <= 1e-5
            at += len(nv)
        ref.cache_free(c)
        seqs.append(sequences)
        splits.append(int(split))
        mids.append(trial_mids)
        fnvs += fnv_rows(lg).tolist()
        argm += lg.argmax(axis=1).tolist()
    flat = [t for sq in seqs for q in sq for t in q]
    lens = [len(q) for sq in seqs for q in sq]
    bs = [len(sq) for sq in seqs]
    ref.model_free(m)
    return dict(tokens=np.array(flat, np.int32), lens=np.array(lens, np.int32), batch=np.array(bs, np.int32),
                split=np.array(splits, np.int32), mids=np.array([x for md in mids for x in md], np.int32),
                row_fnv=np.array(fnvs, np.uint64), argmax=np.array(argm, np.int32), config=P.dims_of(cfg),
                seed=np.array([cfg["init_seed"]], np.uint64))


def c2_fixture(ref: P.Reference) -> dict:
    """OPT-125m-shaped (h=768, 12 heads x 64, V=50272, P=2048), layer-truncated to
    L=2: ragged prefill of 8 samples then one verify step with drafts 1..8."""
    cfg = dict(num_layers=2, num_heads=12, head_dim=64, vocab_size=50272, max_positions=2048, init_seed=7)
    m = ref.model_init(cfg)
    V, B = cfg["vocab_size"], 8
    rs = np.random.default_rng(1)
    prompts = [rs.integers(3, V, size=int(rs.integers(12, 33))).astype(np.int32).tolist() for _ in range(B)]
    c = ref.cache_new(0, 2, B, 256, 768)
    lp = ref.forward(m, c, prompts, [(s, i) for s in range(B) for i in range(len(prompts[s]))], V)
    for s in range(B):
        ref.commit(c, s, len(prompts[s]))
    drafts = [rs.integers(3, V, size=1 + s % 8).astype(np.int32).tolist() for s in range(B)]
    last = [int(lp[np.cumsum([len(p) for p in prompts])[s] - 1].argmax()) for s in range(B)]
    per = [[last[s]] + drafts[s] for s in range(B)]
    ls = ref.forward(m, c, per, [(s, len(prompts[s]) + o) for s in range(B) for o in range(len(per[s]))], V)
    out = dict(prompts=np.array([t for p in prompts for t in p], np.int32),
               prompt_lens=np.array([len(p) for p in prompts], np.int32),
               drafts=np.array([t for d in drafts for t in d], np.int32),
               draft_counts=np.array([len(d) for d in drafts], np.int32), last=np.array(last, np.int32),
               prefill_argmax=lp.argmax(axis=1).astype(np.int32), prefill_fnv=fnv_rows(lp),
               step_argmax=ls.argmax(axis=1).astype(np.int32), step_fnv=fnv_rows(ls),
               step_logits_head=ls[:2].astype(np.float32), checksum=np.array([ref.checksum(m)], np.uint64),
               config=P.dims_of(cfg), seed=np.array([cfg["init_seed"]], np.uint64))
    ref.cache_free(c)
    ref.model_free(m)
    return out


def main() -> None:
    P.build()
    ref = P.Reference()
    c1 = P.DEFAULT_CONFIG
    np.savez_compressed(os.path.join(HERE, "c1_ems_trace.npz"),
                        **ems_trace(ref, c1, P.CORPUS[:4], copy_len=4, budget=128, keep_logit_steps=24))
    for name, mode in (("c1_ems", 2), ("c1_vanilla", 1)):
        e = P.engine_config(mode=mode, predictor=1, copy_len=4, batch_size=4, max_new_tokens=128, stop_on_eos=0)
        np.savez_compressed(os.path.join(HERE, f"{name}_decode.npz"), **decode_fixture(ref, c1, e, P.CORPUS[:4]))
    # test_engine.cpp:169-189 style: every predictor x layout, with EOS
    tcfg = dict(num_layers=2, num_heads=2, head_dim=8, vocab_size=259, max_positions=160, init_seed=0x10EA)
    dcfg = dict(tcfg, num_layers=1, init_seed=0x10EB)
    for pname, pred in (("draft", 0), ("retrieval", 1), ("synthetic", 2)):
        for mname, mode in (("greedy", 0), ("vanilla", 1), ("ems", 2)):
            e = P.engine_config(mode=mode, predictor=pred, k=4, batch_size=3, max_new_tokens=24, seed=17,
                                synthetic_accuracy=0.7)
            np.savez_compressed(os.path.join(HERE, f"engine_{pname}_{mname}.npz"),
                                **decode_fixture(ref, tcfg, e, P.CORPUS[:3], dcfg if pred == 0 else None))
    np.savez_compressed(os.path.join(HERE, "ragged_acceptance8.npz"), **ragged_fixture(ref))
    np.savez_compressed(os.path.join(HERE, "c2_shape_l2.npz"), **c2_fixture(ref))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
