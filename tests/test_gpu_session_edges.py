"""Edge cases of the device-resident decode loop (sd_session_*) and of the
host-driven loop, restated from the reference's engine tests, plus the global
sample ids that make a sharded run reproduce the single-process one.

  * EOS freeze      test_engine.cpp:241-276 (a sample that ends early freezes
                    while the rest keep decoding; streams == greedy)
  * budget clip     test_engine.cpp:278-296 (clipping mid-burst)
  * zero budget     test_engine.cpp:298-305 (no-op, not an error)
  * error paths     test_engine.cpp:322-365 (config / contract / capacity)
  * global ids      engine.cpp:182-185 + SURVEY.md §8e: mix_seed(seed, step,
                    GLOBAL sample id), so shards reproduce the whole batch
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CFG = dict(num_layers=2, num_heads=4, head_dim=128, vocab_size=64, max_positions=512, init_seed=0x0E0)


def greedy(sd, m, prompts, new, eos=True):
    return sd.decode(sd.EngineConfig(mode="greedy", batch_size=len(prompts), max_new_tokens=new, stop_on_eos=eos),
                     m, prompts).generated_tokens


def session(sd, m, prompts, mode, predictor, new, eos=True, k=5, acc=0.7, base=0, traj=None):
    e = sd.EngineConfig(mode=mode, predictor=predictor, k=k, copy_len=k, batch_size=len(prompts),
                        max_new_tokens=new, stop_on_eos=eos, seed=5, synthetic_accuracy=acc, sample_id_base=base)
    s = sd.Session(m, e, 512)
    s.prefill(prompts)
    if predictor == "synthetic":
        s.set_trajectory(traj)
    return s


def trajectory(sd, m, prompts, n):
    # the synthetic predictor corrupts the target's own greedy rollout
    # (predictors.cpp:61-72); without an EOS stop it is the continuation
    return np.array(greedy(sd, m, prompts, n, eos=False), np.int32)


def test_eos_freeze_in_the_device_loop(sd):
    """One sample emits EOS early and freezes; the others keep decoding.  The
    device loop (both layouts, both device predictors) and the host-driven
    loop stop exactly where greedy decoding stops (test_engine.cpp:241-276)."""
    new = 48
    rng = np.random.default_rng(1)
    found = None
    for seed in range(0x0E0, 0x0E0 + 60):
        m = sd.Model.init(sd.ModelConfig(**dict(CFG, init_seed=seed)), precision=sd.BF16)
        prompts = [[0] + rng.integers(3, 64, size=int(rng.integers(8, 30))).tolist() for _ in range(4)]
        g = greedy(sd, m, prompts, new)
        if any(len(t) < new and t[-1] == 1 for t in g) and any(len(t) == new for t in g):
            found = (m, prompts, g)
            break
        m.close()
    assert found, "no early-stopping batch found in the seed range"
    m, prompts, g = found
    traj = trajectory(sd, m, prompts, new + 8)
    for mode in ("ems", "vanilla"):
        for pred in ("retrieval", "synthetic"):
            s = session(sd, m, prompts, mode, pred, new, traj=traj)
            steps, _ = s.run()
            toks, lk, lt = s.outputs()
            # every stream stops at its first EOS or at the budget, and a frozen
            # sample is logged inactive (k = -1) from the step after its EOS
            for j, t in enumerate(toks):
                assert len(t) == new or (t[-1] == 1 and 1 not in t[:-1]), (mode, pred, j)
                act = lk[:steps, j] >= 0
                assert not act[act.argmin():].any() if not act.all() else len(t) == new
            short = next(i for i, t in enumerate(g) if len(t) < new)
            if mode == "ems":  # the unpadded arena is bit-identical to greedy decoding
                assert toks == g, (mode, pred)
                assert (lk[:steps, short] >= 0).sum() < steps
            else:  # the padded grid shifts keys inside bf16 attention sums
                assert np.mean([a == b for a, b in zip(toks, g)]) >= 0.5, (mode, pred)
            if mode == "ems" or pred == "retrieval":
                s.reset()
                s.run_host()
                assert s.outputs()[0] == toks, (mode, pred, "host loop")
            s.close()


def test_budget_clips_mid_burst_in_the_device_loop(sd):
    """test_engine.cpp:278-296: long accepted bursts (p = 0.95, k = 6) hit a
    5-token budget; tau is clipped (logged with the 0x10000 flag) and the
    streams still equal greedy."""
    m = sd.Model.init(sd.ModelConfig(**dict(CFG, init_seed=0xC119)), precision=sd.BF16)
    rng = np.random.default_rng(2)
    prompts = [[0] + rng.integers(3, 64, size=12).tolist() for _ in range(2)]
    traj = trajectory(sd, m, prompts, 20)
    s = session(sd, m, prompts, "ems", "synthetic", 5, eos=False, k=6, acc=0.95, traj=traj)
    steps, _ = s.run()
    toks, lk, lt = s.outputs()
    assert toks == greedy(sd, m, prompts, 5, eos=False)
    assert all(len(t) <= 5 for t in toks)
    assert (lt[:steps] & 0x10000).any()


def test_zero_budget_is_a_no_op(sd):
    """test_engine.cpp:298-305: max_new_tokens = 0 returns before prefill with
    no steps, in the engine and in a device session."""
    m = sd.Model.init(sd.ModelConfig(**CFG), precision=sd.BF16)
    prompts = [[0, 5, 6, 7]]
    r = sd.decode(sd.EngineConfig(mode="ems", predictor="retrieval", k=1, copy_len=1, batch_size=1,
                                  max_new_tokens=0), m, prompts)
    assert r.generated_tokens == [[]] and r.steps == []
    s = session(sd, m, prompts, "ems", "retrieval", 0)
    steps, _ = s.run()
    toks, _, _ = s.outputs()
    assert steps == 0 and toks == [[]]
    s.reset()
    assert s.run_host()[0] == 0


def test_session_error_paths(sd):
    """test_engine.cpp:322-365 for the session entry points: configuration
    errors fail at creation, an oversized prompt fails at prefill before any
    work happens (CapacityError), and a run before prefill is a contract
    error."""
    m = sd.Model.init(sd.ModelConfig(**CFG), precision=sd.BF16)
    with pytest.raises(sd.ConfigError):  # greedy is not a speculative mode
        sd.Session(m, sd.EngineConfig(mode="greedy", predictor="retrieval", batch_size=1), 64)
    with pytest.raises(sd.ConfigError):  # draft predictor without a draft model
        sd.Session(m, sd.EngineConfig(mode="ems", predictor="draft", batch_size=1), 64)
    with pytest.raises(sd.ConfigError):  # more than one forward chunk of tokens per step
        sd.Session(m, sd.EngineConfig(mode="ems", predictor="synthetic", k=7, batch_size=40), 64)
    with pytest.raises(sd.ConfigError):
        sd.Session(m, sd.EngineConfig(mode="ems", predictor="retrieval", batch_size=1, max_new_tokens=-1), 64)
    s = sd.Session(m, sd.EngineConfig(mode="ems", predictor="retrieval", copy_len=4, batch_size=1,
                                      max_new_tokens=500), 600)
    with pytest.raises(sd.ContractError):
        s.run()
    with pytest.raises(sd.CapacityError):  # 200 + 500 + 4 > max_positions 512
        s.prefill([[0] + [5] * 199])
    fp32 = sd.Model.init(sd.ModelConfig(**CFG), precision=sd.FP32_CHECK)
    with pytest.raises(sd.ConfigError):  # the resident loop is the bf16 path
        sd.Session(fp32, sd.EngineConfig(mode="ems", predictor="retrieval", batch_size=1), 64)


@pytest.mark.parametrize("mode", ["ems", "vanilla"])
def test_global_sample_ids_reproduce_the_unsharded_run(sd, mode):
    """Samples sharded over two "ranks" (two sessions holding samples [0, 3)
    and [3, 6) with sample_id_base 0 and 3) emit the same tokens and the same
    per-sample (k, tau) records as one session over all six: the synthetic
    predictor seeds with the global sample id (engine.cpp:182-185), in the
    device loop, the host-driven loop and the engine alike."""
    m = sd.Model.init(sd.ModelConfig(**dict(CFG, vocab_size=700, init_seed=0x61D0)),
                      precision=sd.BF16)
    rng = np.random.default_rng(3)
    prompts = [[0] + rng.integers(3, 700, size=int(rng.integers(10, 40))).tolist() for _ in range(6)]
    new = 24
    traj = trajectory(sd, m, prompts, new + 8)
    whole = session(sd, m, prompts, mode, "synthetic", new, eos=False, traj=traj)
    steps, _ = whole.run()
    toks, lk, lt = whole.outputs()
    shard_toks, per_sample = [], {}
    for lo, hi in ((0, 3), (3, 6)):
        s = session(sd, m, prompts[lo:hi], mode, "synthetic", new, eos=False, base=lo, traj=traj[lo:hi])
        n, _ = s.run()
        t, k2, t2 = s.outputs()
        shard_toks += t
        for j in range(hi - lo):
            per_sample[lo + j] = (k2[:n, j][k2[:n, j] >= 0].tolist(), (t2[:n, j][k2[:n, j] >= 0] & 0xFFFF).tolist())
        s.reset()
        s.run_host()
        assert s.outputs()[0] == t
        e = sd.EngineConfig(mode=mode, predictor="synthetic", k=5, batch_size=hi - lo, max_new_tokens=new,
                            stop_on_eos=False, seed=5, synthetic_accuracy=0.7, sample_id_base=lo)
        r = sd.decode(e, m, prompts[lo:hi])
        assert r.generated_tokens == t
    if mode == "ems":
        assert shard_toks == toks
    else:  # the padded grid aligns per shard: keys move within bf16 attention chunks
        assert np.mean([a == b for a, b in zip(shard_toks, toks)]) >= 0.5
    if mode == "ems":  # tau is per sample in EMS; the padded grid aligns per shard
        for j in range(6):
            act = lk[:steps, j] >= 0
            assert per_sample[j] == (lk[:steps, j][act].tolist(), (lt[:steps, j][act] & 0xFFFF).tolist()), j
    # and a shard that forgets its base draws different drafts
    s = session(sd, m, prompts[3:], mode, "synthetic", new, eos=False, base=0, traj=traj[3:])
    n, _ = s.run()
    k0, t0 = s.outputs()[1:]
    assert [(k0[:n, j] >= 0).sum() for j in range(3)] != [(lk[:steps, 3 + j] >= 0).sum() for j in range(3)] or \
        not all(((t0[:n, j][k0[:n, j] >= 0] & 0xFFFF).tolist() == per_sample[3 + j][1]) for j in range(3))


def test_async_verify_step_on_caller_streams(sd):
    """sd_verify_step_async / _wait (stream-ordered, async
    until outputs are read): two caches' steps enqueued on two caller streams
    before either is collected give exactly the synchronous results; calls
    on a cache with a step in flight are refused (contract), and a bad step is
    rejected before anything is enqueued."""
    import torch

    cfg = dict(num_layers=2, num_heads=4, head_dim=128, vocab_size=900, max_positions=512, init_seed=0xA5)
    m = sd.Model.init(sd.ModelConfig(**cfg), precision=sd.BF16)
    rng = np.random.default_rng(3)
    B = 3
    prompts = [[0] + rng.integers(3, 900, size=int(rng.integers(20, 60))).tolist() for _ in range(B)]

    def prefilled():
        c = sd.UnpadArena(m, B, 256)
        _, am = m.forward(sd.concatenate_inputs(prompts), c,
                          [sd.TokenSlot(s, i) for s in range(B) for i in range(len(prompts[s]))], want_logits=False)
        for s in range(B):
            c.commit_accepted(s, len(prompts[s]))
        ends = np.cumsum([len(p) for p in prompts]) - 1
        return c, [int(am[e]) for e in ends]

    drafts = [rng.integers(3, 900, size=k).tolist() for k in (1, 4, 2)]
    args = lambda last: (last, [len(d) for d in drafts], [t for d in drafts for t in d], [10] * B, [1] * B, False)
    ref, last = prefilled()
    tau_r, acc_r, clip_r, _ = ref.verify_step(*args(last))
    c1, _ = prefilled()
    c2, _ = prefilled()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    c1.verify_step_async(*args(last), stream=s1.cuda_stream)
    c2.verify_step_async(*args(last), stream=s2.cuda_stream)
    with pytest.raises(sd.ContractError):
        c1.commit_accepted(0, 1)  # a step is in flight
    for c in (c2, c1):
        tau, acc, clip = c.verify_step_wait()
        assert tau.tolist() == tau_r.tolist() and acc.tolist() == acc_r.tolist() and clip.tolist() == clip_r.tolist()
        assert [c.committed_len(s) for s in range(B)] == [ref.committed_len(s) for s in range(B)]
        assert [st.tau_list for st in c.ledger().steps()] == [tau_r.tolist()]
    with pytest.raises(sd.ContractError):
        c1.verify_step_wait()  # nothing in flight any more
    bad = args(last)
    with pytest.raises(sd.ContractError):  # out-of-vocabulary draft: refused before enqueue
        c1.verify_step_async(bad[0], bad[1], [10 ** 6] * len(bad[2]), *bad[3:], stream=s1.cuda_stream)
    c1.set_stream(s1.cuda_stream)  # the synchronous step on a caller stream
    tau, acc, _, _ = c1.verify_step([int(a[t - 1]) for a, t in zip(acc_r, tau_r)], [0] * B, [], [9] * B, [1] * B,
                                    False)
    assert (tau == 1).all()
    for c in (ref, c1, c2):
        c.close()
    m.close()


def test_nccl_gather_of_session_outputs(sd):
    """The run's only collective through the library (sd_comm_*, NCCL): a
    world-1 communicator on this GPU all-gathers int32 blocks in rank order
    and sd_session_gather_outputs returns the session's own outputs.  (The
    box has one GPU; NCCL refuses two ranks on one device, so N > 1 is
    covered by the host-side sharding tests and the bench's torchrun path.)"""
    cfg = dict(num_layers=2, num_heads=4, head_dim=128, vocab_size=700, max_positions=512, init_seed=0xC0)
    m = sd.Model.init(sd.ModelConfig(**cfg), precision=sd.BF16)
    rng = np.random.default_rng(2)
    prompts = [[0] + rng.integers(3, 700, size=30).tolist() for _ in range(3)]
    e = sd.EngineConfig(mode="ems", predictor="retrieval", k=4, copy_len=4, batch_size=3, max_new_tokens=12,
                        stop_on_eos=False)
    s = sd.Session(m, e, 128)
    s.prefill(prompts)
    s.run()
    comm = sd.Comm(sd.nccl_unique_id(), 1, 0, 0)
    x = np.arange(37, dtype=np.int32)
    assert (comm.allgather_i32(x) == x[None, :]).all()
    assert s.gather_outputs(comm) == s.outputs()[0]
    comm.close()
    s.close()
    m.close()


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_verify_step_with_more_samples_than_one_pack_block(sd, precision):
    """k_pack's block scans walk the samples in chunks of 256 threads: a
    300-sample verify step (some samples inactive, draft counts 0-7) gives
    exactly the taus, accepted tokens and committed lengths of the same samples
    verified in three batches of 100 (a sample's result does not depend on the
    batch; test_engine.cpp:307-320)."""
    cfg = dict(num_layers=2, num_heads=2, head_dim=64, vocab_size=300, max_positions=128, init_seed=0x51)
    m = sd.Model.init(sd.ModelConfig(**cfg), precision=sd.FP32_CHECK if precision == "fp32" else sd.BF16)
    rng = np.random.default_rng(11)
    B = 300
    prompts = [[0] + rng.integers(3, 300, size=int(rng.integers(3, 12))).tolist() for _ in range(B)]
    active = [int(s % 7 != 3) for s in range(B)]
    counts = [int(k) * a for k, a in zip(rng.integers(0, 8, size=B), active)]  # finished samples bring no drafts
    drafts = [rng.integers(3, 300, size=k).tolist() for k in counts]

    def run(ids):
        c = sd.UnpadArena(m, len(ids), 64)
        ps = [prompts[s] for s in ids]
        _, am = m.forward(sd.concatenate_inputs(ps), c,
                          [sd.TokenSlot(i, j) for i, p in enumerate(ps) for j in range(len(p))], want_logits=False)
        for i, p in enumerate(ps):
            c.commit_accepted(i, len(p))
        ends = np.cumsum([len(p) for p in ps]) - 1
        last = [int(am[e]) for e in ends]
        tau, acc, clip, _ = c.verify_step(last, [counts[s] for s in ids], [t for s in ids for t in drafts[s]],
                                          [20] * len(ids), [active[s] for s in ids], False)
        out = [(int(tau[i]), acc[i][: tau[i]].tolist(), c.committed_len(i)) for i in range(len(ids))]
        c.close()
        return out

    whole = run(list(range(B)))
    parts = run(list(range(0, 100))) + run(list(range(100, 200))) + run(list(range(200, 300)))
    assert whole == parts
    assert all(t == 0 for (t, _, _), a in zip(whole, active) if not a)
    assert any(t > 1 for t, _, _ in whole) or precision == "bf16"
    m.close()
