"""fp32 CHECK mode on the B200 against the reference (golden fixtures) and the
CPU oracle: token ids, accepted counts and KV lengths bit-exact, logits
bit-exact (compared as FNV-1a hashes of each row's bytes, or bitwise)."""
import os
import tempfile

import numpy as np
import pytest

from conftest import golden
import pyoracle as P

pytestmark = pytest.mark.gpu


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


def gpu_model(sd, cfg):
    return sd.Model.init(sd.ModelConfig(**cfg), precision=sd.FP32_CHECK)


def fwd(sd, m, cache, per, slots):
    b = sd.concatenate_inputs(per)
    return m.forward(b, cache, [sd.TokenSlot(s, p) for s, p in slots])


def test_gpu_init_checksum_matches_reference(sd):
    for name in ("c1_ems_trace.npz", "c2_shape_l2.npz"):
        g = golden(name)
        m = gpu_model(sd, cfg_from(g))
        assert m.weight_checksum() == int(g["checksum"][0]), name


def test_gpu_c1_trace_bit_exact(sd):
    g = golden("c1_ems_trace.npz")
    cfg = cfg_from(g)
    B = len(g["prompt_lens"])
    m = gpu_model(sd, cfg)
    c = sd.UnpadArena(m, B, cfg["max_positions"])
    prompts = split(g["prompts"], g["prompt_lens"])
    fwd(sd, m, c, prompts, [(s, i) for s in range(B) for i in range(len(prompts[s]))])
    for s in range(B):
        c.commit_accepted(s, len(prompts[s]))
    at_tok = at_row = 0
    seen = []
    for step, T in enumerate(g["step_T"]):
        counts, taus = g["step_counts"][step], g["step_tau"][step]
        n_s = [(1 + counts[s]) if taus[s] > 0 else 0 for s in range(B)]
        per = split(g["step_tokens"][at_tok: at_tok + T], n_s)
        slots = [(s, c.committed_len(s) + o) for s in range(B) for o in range(n_s[s])]
        lg, am = fwd(sd, m, c, per, slots)
        assert (P.fnv_rows(lg) == g["step_fnv"][at_row: at_row + T]).all(), f"step {step}"
        assert (am == g["step_argmax"][at_row: at_row + T]).all()
        seen.append(lg)
        for s in range(B):
            if taus[s]:
                c.commit_accepted(s, int(taus[s]))
        assert [c.committed_len(s) for s in range(B)] == g["step_committed"][step].tolist()
        at_tok += T
        at_row += T
    ours = np.concatenate(seen)[: len(g["logits"])]
    assert np.array_equal(ours.view(np.uint32), g["logits"].view(np.uint32))


def test_gpu_fused_verify_step_c1_bit_exact(sd, oracle):
    """The device-fused step (pack -> forward -> accept/clip -> commit) walks the
    reference's C1 EMS trace: same taus, committed lengths and logits."""
    g = golden("c1_ems_trace.npz")
    cfg = cfg_from(g)
    B = len(g["prompt_lens"])
    m = gpu_model(sd, cfg)
    c = sd.UnpadArena(m, B, cfg["max_positions"])
    prompts = split(g["prompts"], g["prompt_lens"])
    lp, am = fwd(sd, m, c, prompts, [(s, i) for s in range(B) for i in range(len(prompts[s]))])
    for s in range(B):
        c.commit_accepted(s, len(prompts[s]))
    rows = np.cumsum(g["prompt_lens"]) - 1
    toks = [prompts[s] + [int(am[rows[s]])] for s in range(B)]
    gen = [1] * B
    at_row = 0
    step_taus = []
    for step, T in enumerate(g["step_T"]):
        active = [int(x < 128) for x in gen]
        drafts = [oracle.retrieval_predict(toks[s], 2, 4) if active[s] else [] for s in range(B)]
        counts = [len(d) for d in drafts]
        assert counts == g["step_counts"][step].tolist()
        tau, acc, clipped, lg = c.verify_step([t[-1] for t in toks], counts, [x for d in drafts for x in d],
                                              [128 - x for x in gen], active, False, want_logits=True)
        assert tau.tolist() == g["step_tau"][step].tolist(), f"step {step}"
        step_taus.append([int(t) for t, a in zip(tau, active) if a])
        assert (P.fnv_rows(lg) == g["step_fnv"][at_row: at_row + T]).all()
        at_row += T
        for s in range(B):
            toks[s] += acc[s, : tau[s]].tolist()
            gen[s] += int(tau[s])
        assert [c.committed_len(s) for s in range(B)] == g["step_committed"][step].tolist()
    assert [t[len(p):] for t, p in zip(toks, prompts)] == g["generated"].tolist()
    led = c.ledger()
    assert (led.useful_total(), led.padding_total()) == (int(g["step_T"].sum()) + int(g["prompt_lens"].sum()), 0)
    # one ledger step per sd_verify_step call, its taus in sample order (engine.cpp:398-487)
    assert [st.tau_list for st in led.steps()] == step_taus


@pytest.mark.parametrize("name", ["c1_ems_decode", "c1_vanilla_decode"] +
                         [f"engine_{p}_{m}" for p in ("draft", "retrieval", "synthetic")
                          for m in ("greedy", "vanilla", "ems")])
def test_gpu_decode_matches_reference(sd, name):
    """decode_greedy / decode_speculative end to end (engine.cpp:206-489) on the GPU."""
    g = golden(name + ".npz")
    cfg = cfg_from(g)
    e = g["engine"]
    modes = {0: "greedy", 1: "vanilla", 2: "ems"}
    preds = {0: "draft", 1: "retrieval", 2: "synthetic"}
    ecfg = sd.EngineConfig(mode=modes[int(e[0])], predictor=preds[int(e[1])], k=int(e[2]), match_len=int(e[3]),
                           copy_len=int(e[4]), batch_size=int(e[5]), max_new_tokens=int(e[6]),
                           stop_on_eos=bool(e[7]), seed=int(g["engine_seed"][0]),
                           synthetic_accuracy=float(g["accuracy"][0]))
    m = gpu_model(sd, cfg)
    d = gpu_model(sd, cfg_from({"config": g["draft_config"], "seed": g["draft_seed"]})) \
        if "draft_config" in g else None
    r = sd.decode(ecfg, m, P.CORPUS[: ecfg.batch_size], d)
    for s in range(ecfg.batch_size):
        assert r.generated_tokens[s] == g["generated"][s, : int(g["gen_counts"][s])].tolist()
    if ecfg.mode != "greedy":
        flat = [(i, x["sample"], x["k"], x["tau"], int(x["clipped"])) for i, st in enumerate(r.steps)
                for x in st["samples"]]
        assert np.array_equal(np.array(flat, np.int32).reshape(-1, 5), g["records"])
        assert [r.useful_kv_writes, r.padding_kv_writes] == g["ledger"].tolist()


def test_gpu_ragged_acceptance_batches_bit_exact(sd):
    g = golden("ragged_acceptance8.npz")
    m = gpu_model(sd, cfg_from(g))
    seqs_all = split(g["tokens"], g["lens"])
    at_seq = at_mid = at_row = 0
    for trial, b in enumerate(g["batch"]):
        b = int(b)
        seqs = seqs_all[at_seq: at_seq + b]
        at_seq += b
        c = sd.UnpadArena(m, b, 64)
        if not g["split"][trial]:
            lg, _ = fwd(sd, m, c, seqs, [(s, i) for s in range(b) for i in range(len(seqs[s]))])
        else:
            mids = g["mids"][at_mid: at_mid + b].tolist()
            heads = [q[:md] for q, md in zip(seqs, mids)]
            tails = [q[md:] for q, md in zip(seqs, mids)]
            lh, _ = fwd(sd, m, c, heads, [(s, i) for s in range(b) for i in range(len(heads[s]))])
            for s in range(b):
                c.commit_accepted(s, mids[s])
            lt, _ = fwd(sd, m, c, tails, [(s, mids[s] + i) for s in range(b) for i in range(len(tails[s]))])
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


def test_gpu_c2_shape_bit_exact(sd):
    """OPT-125m-shaped layers (h=768, 12x64, V=50272), L=2."""
    g = golden("c2_shape_l2.npz")
    cfg = cfg_from(g)
    B = len(g["prompt_lens"])
    m = gpu_model(sd, cfg)
    c = sd.UnpadArena(m, B, 256)
    prompts = split(g["prompts"], g["prompt_lens"])
    lp, _ = fwd(sd, m, c, prompts, [(s, i) for s in range(B) for i in range(len(prompts[s]))])
    assert (P.fnv_rows(lp) == g["prefill_fnv"]).all()
    for s in range(B):
        c.commit_accepted(s, len(prompts[s]))
    drafts = split(g["drafts"], g["draft_counts"])
    per = [[int(g["last"][s])] + drafts[s] for s in range(B)]
    ls, am = fwd(sd, m, c, per, [(s, len(prompts[s]) + o) for s in range(B) for o in range(len(per[s]))])
    assert (P.fnv_rows(ls) == g["step_fnv"]).all()
    assert (am == g["step_argmax"]).all()
    assert np.array_equal(ls[:2].view(np.uint32), g["step_logits_head"].view(np.uint32))


def tiny(seed):
    return dict(num_layers=2, num_heads=2, head_dim=8, vocab_size=259, max_positions=64, init_seed=seed)


def test_gpu_aligned_grid_with_holes_bit_identical_to_unpad(sd):
    """test_model.cpp:267-297"""
    m = gpu_model(sd, tiny(0xB17))
    a, b = sd.tokenize_prompt("hi"), sd.tokenize_prompt("longer")
    holes = len(b) - len(a)
    unpad = sd.UnpadArena(m, 2, 64)
    ref, _ = fwd(sd, m, unpad, [a, b], [(0, i) for i in range(len(a))] + [(1, i) for i in range(len(b))])
    grid = sd.PaddedGrid(m, 2, 64)
    for r in range(holes):
        grid.mark_hole(0, r)
    plans = [sd.TokenPlan(0, i, holes + i, True) for i in range(len(a))] + \
            [sd.TokenPlan(1, i, i, True) for i in range(len(b))]
    got, _ = m.forward_planned(a + b, plans, grid)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_gpu_pad_query_tokens_are_spectators(sd):
    """test_model.cpp:299-326"""
    m = gpu_model(sd, tiny(0x5150))
    prompt = sd.tokenize_prompt("spectators")
    pl = len(prompt)

    def run(with_pads):
        grid = sd.PaddedGrid(m, 1, 64)
        m.forward_planned(prompt, [sd.TokenPlan(0, i, i, True) for i in range(pl)], grid)
        grid.commit_prefill([0], [pl])
        toks = [42, 43]
        plans = [sd.TokenPlan(0, pl, pl, True), sd.TokenPlan(0, pl + 1, pl + 1, True)]
        if with_pads:
            toks.append(sd.PAD)
            plans.append(sd.TokenPlan(0, pl + 2, pl + 2, False))
        return m.forward_planned(toks, plans, grid)[0]

    bare, padded = run(False), run(True)
    assert padded.shape[0] == 3
    assert np.array_equal(bare.view(np.uint32), padded[:2].view(np.uint32))


def test_gpu_forward_validates_inputs(sd):
    """test_model.cpp:350-372"""
    m = gpu_model(sd, tiny(0x7E57))
    c = sd.UnpadArena(m, 1, 64)
    with pytest.raises(sd.ContractError):
        fwd(sd, m, c, [[sd.BOS, 9999]], [(0, 0), (0, 1)])
    with pytest.raises(sd.ContractError):
        fwd(sd, m, c, [[sd.BOS, 42]], [(0, 0), (0, 2)])
    with pytest.raises(sd.ContractError):
        fwd(sd, m, c, [[sd.BOS, 42]], [(0, 1), (0, 0)])
    small = gpu_model(sd, dict(tiny(0x7E57), max_positions=4))
    little = sd.UnpadArena(small, 1, 8)
    with pytest.raises(sd.CapacityError):
        fwd(sd, small, little, [[sd.BOS, 10, 11, 12, 13]], [(0, i) for i in range(5)])
    with pytest.raises(sd.ContractError):
        c.mark_hole(0, 0)  # unpad arena has no holes
    with pytest.raises(sd.ContractError):
        c.commit_accepted(0, 1)  # nothing written


def test_gpu_unpad_arena_contracts(sd):
    """test_kv_cache.cpp:44-85: start offsets, commit bounds, dead in-flight slots."""
    m = gpu_model(sd, dict(tiny(3), num_layers=1))
    c = sd.UnpadArena(m, 3, 16)
    assert [c.start_offset(s) for s in range(3)] == [0, 16, 32]
    with pytest.raises(sd.ContractError):
        c.start_offset(3)
    fwd(sd, m, c, [[5, 6, 7, 8, 9], [], []], [(0, i) for i in range(5)])
    c.commit_accepted(0, 4)
    assert c.committed_len(0) == 4
    with pytest.raises(sd.ContractError):
        c.commit_accepted(0, 1)  # slot 4 died
    with pytest.raises(sd.ContractError):
        c.commit_accepted(0, 0)
    k, v = c.gather_visible(0, 3, 0)
    assert k.shape == (4, 16)
    with pytest.raises(sd.ContractError):
        c.gather_visible(0, 4, 0)


def test_gpu_nonfinite_weights_raise(sd):
    """test_model.cpp:192-208: a NaN weight surfaces as Error, not garbage."""
    m = gpu_model(sd, tiny(0x7E57))
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "m.bin")
        m.save(p)
        raw = bytearray(open(p, "rb").read())
        raw[36:40] = np.array([np.nan], np.float32).tobytes()
        open(p, "wb").write(bytes(raw))
        bad = sd.Model.load(p, precision=sd.FP32_CHECK)
        c = sd.UnpadArena(bad, 1, 16)
        with pytest.raises(sd.SpecdecError):
            fwd(sd, bad, c, [[sd.BOS, 42]], [(0, 0), (0, 1)])


def test_gpu_checkpoint_roundtrip_with_oracle(sd, oracle):
    cfg = tiny(0xC0FFEE)
    m = gpu_model(sd, cfg)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "m.bin")
        m.save(p)
        mo = oracle.model_load(p)
        assert oracle.checksum(mo) == m.weight_checksum()
        oracle.model_free(mo)
        m2 = sd.Model.load(p, precision=sd.FP32_CHECK)
        assert m2.weight_checksum() == m.weight_checksum()
        open(os.path.join(d, "bad.bin"), "wb").write(b"not a checkpoint at all")
        with pytest.raises(sd.IoError):
            sd.Model.load(os.path.join(d, "bad.bin"))


@pytest.mark.parametrize("layout", [0, 1])
def test_gpu_random_verify_steps_match_oracle(sd, oracle, layout):
    """Random ragged verify steps (drafts 0..7, EOS/budget clipping) on a wider
    model (4 heads x 32): GPU fused step vs the oracle's forward + verify."""
    cfg = dict(num_layers=2, num_heads=4, head_dim=32, vocab_size=300, max_positions=256, init_seed=0x51)
    rng = np.random.default_rng(layout + 7)
    m = gpu_model(sd, cfg)
    mo = oracle.model_init(cfg)
    B = 5
    prompts = [rng.integers(3, 300, size=int(rng.integers(3, 20))).tolist() for _ in range(B)]
    ecfg = P.engine_config(mode=1 if layout else 2, predictor=1, copy_len=7, batch_size=B, max_new_tokens=40,
                           stop_on_eos=1)
    toks_o, rec_o, led_o = oracle.decode(ecfg, mo, [[0] + p for p in prompts])
    r = sd.decode(sd.EngineConfig(mode="vanilla" if layout else "ems", predictor="retrieval", copy_len=7,
                                  batch_size=B, max_new_tokens=40, stop_on_eos=True), m, [[0] + p for p in prompts])
    assert r.generated_tokens == toks_o
    flat = [(i, x["sample"], x["k"], x["tau"], int(x["clipped"])) for i, st in enumerate(r.steps)
            for x in st["samples"]]
    assert np.array_equal(np.array(flat, np.int32).reshape(-1, 5), rec_o[:, :5])
    assert [r.useful_kv_writes, r.padding_kv_writes] == led_o.tolist()
    oracle.model_free(mo)


@pytest.mark.parametrize("mode", ["greedy", "vanilla", "ems"])
def test_gpu_results_json_matches_reference(sd, mode):
    """specdec.results_json of a GPU decode (fp32 check mode) equals the
    REFERENCE's own report (results_json, engine.cpp:531-587, fixture made by
    tests/golden/make_results_json.py from oracle/_ref) key for key, minus the
    wall-clock fields: outputs and texts, RunMetrics, step records and the
    per-step write ledger."""
    import json

    fx = json.load(open(os.path.join(os.path.dirname(__file__), "golden", f"results_json_retrieval_{mode}.json")))
    e = fx["engine"]
    m = sd.Model.init(sd.ModelConfig(**fx["model"]))
    cfg = sd.EngineConfig(mode=mode, predictor="retrieval", k=e["k"], match_len=e["match_len"],
                          copy_len=e["copy_len"], batch_size=e["batch_size"], max_new_tokens=e["max_new_tokens"],
                          stop_on_eos=bool(e["stop_on_eos"]), seed=e["seed"],
                          synthetic_accuracy=e["synthetic_accuracy"])
    got = json.loads(sd.results_json(cfg, sd.decode(cfg, m, fx["prompts"])))
    for k in ("prefill_seconds", "decode_seconds", "tokens_per_second_decode", "tokens_per_second_total"):
        got["metrics"].pop(k)
    assert got == fx["results"]


def test_gpu_table1_scripted_trace_ledgers(sd):
    """acceptance.cpp:125-176 (check 2, the paper's Table 1) on the device
    arenas, through the reference's own calls: write_kv rows, commit_prefill,
    ledger steps around commit_padded / commit_accepted + note_tau.  The
    aligned grid writes 3 + 4 PAD filler rows, the unpadded arena none."""
    vec = np.full(4, 0.25, np.float32)

    def stage(arena, sample, start, count):
        for pos in range(start, start + count):
            arena.write_kv(sample, pos, 0, vec, vec)

    grid = sd.PaddedGrid.from_dims(1, 2, 32, 4)
    stage(grid, 0, 0, 1)
    stage(grid, 1, 0, 1)
    grid.commit_prefill([0, 1], [1, 1])
    grid.ledger().begin_step()
    stage(grid, 0, 1, 6)
    stage(grid, 1, 1, 3)
    grid.commit_padded([0, 1], [4, 1])
    grid.ledger().end_step()
    grid.ledger().begin_step()
    stage(grid, 0, 5, 3)
    stage(grid, 1, 5, 6)
    grid.commit_padded([0, 1], [2, 6])
    grid.ledger().end_step()
    led = grid.ledger()
    assert [st.pad_writes for st in led.steps()] == [3, 4]
    assert led.padding_by_sample() == [4, 3]
    assert [st.tau_list for st in led.steps()] == [[4, 1], [2, 6]]
    assert [grid.committed_len(s) for s in (0, 1)] == [11, 11]
    assert [grid.logical_len(s) for s in (0, 1)] == [7, 8]
    # the filler rows are real zero writes on the device, skipped by reads
    k, v = grid.gather_visible(1, 10, 0)
    assert len(k) == 8 and np.all(k == 0.25)

    arena = sd.UnpadArena.from_dims(1, 2, 32, 4)
    stage(arena, 0, 0, 1)
    stage(arena, 1, 0, 1)
    arena.commit_accepted(0, 1)
    arena.commit_accepted(1, 1)
    arena.ledger().begin_step()
    stage(arena, 0, 1, 6)
    stage(arena, 1, 1, 3)
    arena.commit_accepted(0, 4)
    arena.commit_accepted(1, 1)
    arena.ledger().note_tau(4)
    arena.ledger().note_tau(1)
    arena.ledger().end_step()
    arena.ledger().begin_step()
    stage(arena, 0, 5, 3)
    stage(arena, 1, 2, 6)
    arena.commit_accepted(0, 2)
    arena.commit_accepted(1, 6)
    arena.ledger().note_tau(2)
    arena.ledger().note_tau(6)
    arena.ledger().end_step()
    led = arena.ledger()
    assert led.padding_total() == 0 and [st.pad_writes for st in led.steps()] == [0, 0]
    assert [arena.committed_len(s) for s in (0, 1)] == [7, 8]
    assert sd.padding_ratio(grid.ledger()) == pytest.approx(sd.padding_ratio(arena.ledger()), abs=1e-15)
    with pytest.raises(sd.ContractError):  # commit_padded notes its taus: a ledger step must be open
        grid.commit_padded([0, 1], [1, 1])


def test_gpu_write_gap_is_the_padding_shortfall(sd):
    """test_engine.cpp:216-239 on the GPU engine: the vanilla run writes exactly
    the EMS run's useful KV rows plus one filler row per unit of tau_max - tau."""
    m = sd.Model.init(sd.ModelConfig(num_layers=2, num_heads=2, head_dim=8, vocab_size=259, max_positions=160,
                                     init_seed=0xACC7))
    prompts = ["The quick brown fox", "jumps over", "the lazy dog.", "Again!"]
    cfg = dict(predictor="synthetic", k=4, batch_size=4, max_new_tokens=31, seed=40, synthetic_accuracy=0.6,
               stop_on_eos=False)
    van = sd.decode(sd.EngineConfig(mode="vanilla", **cfg), m, prompts)
    ems = sd.decode(sd.EngineConfig(mode="ems", **cfg), m, prompts)
    shortfall = sum(st["tau_max"] - x["tau"] for st in van.steps for x in st["samples"])
    assert shortfall > 0
    assert van.generated_tokens == ems.generated_tokens
    assert van.useful_kv_writes == ems.useful_kv_writes
    assert ems.padding_kv_writes == 0 and van.padding_kv_writes == shortfall
    assert sum(x["kv_padding"] for st in van.steps for x in st["samples"]) == shortfall
