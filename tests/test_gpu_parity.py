"""bf16 tcgen05 path pinned at the shapes the bench runs.

(a) The persistent attention (k_attention_tcp) against a float64 softmax of
    the same bf16 Q/K/V: extents 129-4200 keys (one chunk to 33 chunks), the
    32/64/128-key tail boxes, 1-8 draft queries and a 40-query prefill-like
    sample (5 tiles, each stopping at its own causal limit), head_dim 128 and
    64, padded-grid holes, K chunks scaled so the lazy-rescale path fires
    (model.cpp:320-349: ascending-j softmax over the visible prefix).
    Tolerance: |ctx - ref| <= 1e-2 (V entries in [-1, 1]; bf16 P and bf16
    output rounding are <= 2^-9 each), mean <= 1e-3.
(b) k_gemm against a float64 product at the exact C3 / C5 (M, K) shapes and
    T in {1, 24, 100, 192, 256} on the production grid (one CTA per SM).
    Tolerance: |err| <= 2e-3 * max|Y| + 1e-3 (fp32 accumulation order).
(c) A layer-truncated C3 forward (L = 2, h = 5120, 40 x 128 heads,
    V = 50272, ~600-token contexts, drafts 1-8) against the float64 torch
    reference (tests/torch_ref.py, pinned to the oracle by
    tests/test_torch_ref.py) on the fp32 weights of the same seed.
    Stated bf16 tolerance: max |dlogit| <= 0.15 std, mean <= 0.03 std,
    argmax agreement >= 0.9 (random-init top-1/top-2 margins are tiny).
"""
import ctypes as C
import math

import numpy as np
import pytest

from torch_ref import c3_truncated_parity

pytestmark = pytest.mark.gpu


def to_bf16_bits(x):
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def from_bf16_bits(b):
    return (b.astype(np.uint32) << 16).view(np.float32)


# ------------------------------------------------------------------ (a)
def run_attention(sd, q, kv, n_q, kv_len, ws, pad, heads, hd, cap):
    L = sd.lib()
    fn = L.sd_debug_attention
    I32 = np.ctypeslib.ndpointer(np.int32)
    fn.argtypes = [np.ctypeslib.ndpointer(np.uint16), np.ctypeslib.ndpointer(np.uint16), C.c_int, C.c_int, C.c_int,
                   C.c_int, I32, I32, I32, C.c_void_p, np.ctypeslib.ndpointer(np.uint16), C.POINTER(C.c_float)]
    T = int(np.sum(n_q))
    out = np.zeros((T, heads * hd), np.uint16)
    us = C.c_float()
    padp = pad.ctypes.data if pad is not None else None
    rc = fn(np.ascontiguousarray(q), np.ascontiguousarray(kv), len(n_q), heads, hd, cap,
            np.asarray(n_q, np.int32), np.asarray(kv_len, np.int32), np.asarray(ws, np.int32), padp, out,
            C.byref(us))
    assert rc == 0
    return out, us.value


def attention_ref(q, kv, n_q, kv_len, ws, pad, heads, hd):
    """float64 softmax(q k^T / sqrt(hd)) v over each query's visible slots
    (j <= write_slot, j < kv_len, not a hole), ascending j (model.cpp:320-349)."""
    qf = from_bf16_bits(q).astype(np.float64)
    kvf = from_bf16_bits(kv).astype(np.float64)
    out = np.zeros_like(qf)
    t = 0
    for s in range(len(n_q)):
        for i in range(n_q[s]):
            vis = np.arange(kv_len[s]) <= ws[t]
            if pad is not None:
                vis &= pad[s, : kv_len[s]] == 0
            for hh in range(heads):
                K = kvf[0, s, hh, : kv_len[s]][vis]
                V = kvf[1, s, hh, : kv_len[s]][vis]
                sc = K @ qf[t, hh * hd:(hh + 1) * hd] / math.sqrt(hd)
                p = np.exp(sc - sc.max())
                out[t, hh * hd:(hh + 1) * hd] = (p / p.sum()) @ V
            t += 1
    return out


def make_attention_case(rng, extents, nqs, heads, hd, padded=False, prefill=None):
    B = len(extents)
    cap = max(extents) + 16
    kv = rng.uniform(-1, 1, (2, B, heads, cap, hd)).astype(np.float32)
    # per-chunk key scales from {0.3, 1, 3, 6}: the chunk max jumps up (lazy
    # rescale of O^T in TMEM) and down across a sample's extent
    scales = rng.choice([0.3, 1.0, 3.0, 6.0], size=(B, heads, cap // 128 + 1))
    kv[0] *= np.repeat(scales, 128, axis=2)[:, :, :cap, None]
    kv = to_bf16_bits(kv)
    ws, n_q = [], []
    pad = np.zeros((B, cap), np.uint8) if padded else None
    for s, (e, nq) in enumerate(zip(extents, nqs)):
        if prefill is not None and s == prefill:
            nq = 40
        nq = min(nq, e)
        n_q.append(nq)
        ws += list(range(e - nq, e))  # the sample's newest slots, in order
        if padded and e > 20:  # left padding + one interior alignment hole below the queries
            pad[s, : 1 + s % 7] = 1
            pad[s, e - nq - 1] = 1
    T = sum(n_q)
    q = to_bf16_bits(rng.uniform(-1, 1, (T, heads * hd)).astype(np.float32))
    return q, kv, n_q, list(extents), ws, pad, cap


@pytest.mark.parametrize("hd,heads", [(128, 2), (64, 4)])
@pytest.mark.parametrize("padded", [False, True])
def test_attention_long_extents_vs_float64(sd, hd, heads, padded):
    rng = np.random.default_rng(hd * 7 + heads + padded)
    # 1 key past a chunk (32-box tail), 72 (128-box), 32 (32-box), 62 (64-box),
    # 9 chunks with a 76-key tail, 33 chunks, a prefill-like sample, 1028 keys,
    # an empty (finished) sample
    extents = [129, 200, 160, 190, 1100, 4200, 600, 1028, 64]
    nqs = [1, 8, 3, 5, 7, 8, 2, 6, 0]
    q, kv, n_q, kv_len, ws, pad, cap = make_attention_case(rng, extents, nqs, heads, hd, padded, prefill=6)
    out, us = run_attention(sd, q, kv, n_q, kv_len, ws, pad, heads, hd, cap)
    ref = attention_ref(q, kv, n_q, kv_len, ws, pad, heads, hd)
    got = from_bf16_bits(out).astype(np.float64)
    err = np.abs(got - ref)
    print(f"hd={hd} padded={padded}: max|err|={err.max():.2e} mean={err.mean():.2e} ({us:.1f} us)")
    assert np.isfinite(got).all()
    assert err.max() <= 1e-2 and err.mean() <= 1e-3
    out2, _ = run_attention(sd, q, kv, n_q, kv_len, ws, pad, heads, hd, cap)
    assert np.array_equal(out, out2)  # deterministic


@pytest.mark.parametrize("hd,heads", [(128, 2), (64, 4)])
def test_attention_batch_composition_invariance(sd, hd, heads):
    """A sample's context rows do not depend on the samples around it: each
    sample's keys are chunked from its slot 0 whatever the batch, so a sample
    alone gives the same bits as inside the batch (test_engine.cpp:307-320)."""
    rng = np.random.default_rng(5)
    extents, nqs = [300, 4200, 1100], [4, 8, 2]
    q, kv, n_q, kv_len, ws, pad, cap = make_attention_case(rng, extents, nqs, heads, hd)
    whole, _ = run_attention(sd, q, kv, n_q, kv_len, ws, None, heads, hd, cap)
    for s in range(3):
        r0 = sum(n_q[:s])
        alone, _ = run_attention(sd, q[r0:r0 + n_q[s]], np.ascontiguousarray(kv[:, s:s + 1]), [n_q[s]], [kv_len[s]],
                                 ws[r0:r0 + n_q[s]], None, heads, hd, cap)
        assert np.array_equal(alone, whole[r0:r0 + n_q[s]]), s


@pytest.mark.parametrize("hd,heads", [(128, 2), (64, 4)])
@pytest.mark.parametrize("padded", [False, True])
def test_prefill_attention_wide_runs_vs_float64(sd, hd, heads, padded):
    """(a') Prompt runs of >= 64 queries go to the 128-query prefill kernel
    (k_attention_wide: queries as the MMA's M, each K/V chunk streamed once per
    128 queries) in the same launch sequence as the verification kernel's
    samples: a full 128-query tile at the end of a 4200-key extent (33
    chunks, lazy rescale), a 64-query run that spans a chunk boundary, next
    to 40-, 8- and 1-query samples (verification kernel) and an empty one.  Same float64 reference
    and tolerance as (a); deterministic; a wide sample alone gives the same
    bits as inside the batch."""
    rng = np.random.default_rng(hd + 3 * heads + padded)
    extents = [4200, 700, 1100, 129, 64, 600]
    nqs = [128, 64, 8, 1, 0, 40]
    q, kv, n_q, kv_len, ws, pad, cap = make_attention_case(rng, extents, nqs, heads, hd, padded)
    out, us = run_attention(sd, q, kv, n_q, kv_len, ws, pad, heads, hd, cap)
    ref = attention_ref(q, kv, n_q, kv_len, ws, pad, heads, hd)
    got = from_bf16_bits(out).astype(np.float64)
    err = np.abs(got - ref)
    print(f"wide hd={hd} padded={padded}: max|err|={err.max():.2e} mean={err.mean():.2e} ({us:.1f} us)")
    assert np.isfinite(got).all()
    assert err.max() <= 1e-2 and err.mean() <= 1e-3
    out2, _ = run_attention(sd, q, kv, n_q, kv_len, ws, pad, heads, hd, cap)
    assert np.array_equal(out, out2)
    if not padded:
        for s in (0, 1):
            r0 = sum(n_q[:s])
            alone, _ = run_attention(sd, q[r0:r0 + n_q[s]], np.ascontiguousarray(kv[:, s:s + 1]), [n_q[s]],
                                     [kv_len[s]], ws[r0:r0 + n_q[s]], None, heads, hd, cap)
            assert np.array_equal(alone, out[r0:r0 + n_q[s]]), s


# ------------------------------------------------------------------ (b)
SHAPES = [(15360, 5120), (5120, 5120), (20480, 5120), (5120, 20480), (50432, 5120), (12288, 4096), (4096, 16384)]


@pytest.mark.parametrize("M,K", SHAPES)
def test_gemm_exact_shapes_vs_float64(sd, M, K):
    import torch

    L = sd.lib()
    fn = L.sd_debug_gemm
    fn.argtypes = [np.ctypeslib.ndpointer(np.uint16), np.ctypeslib.ndpointer(np.uint16), C.c_int, C.c_int, C.c_int,
                   C.c_int, C.c_int, np.ctypeslib.ndpointer(np.float32), C.POINTER(C.c_float)]
    g = torch.Generator(device="cuda").manual_seed(M + K)
    Wd = (torch.rand(M, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    W = Wd.view(torch.int16).cpu().numpy().view(np.uint16)
    for T in (1, 24, 100, 192, 256):
        Xd = (torch.rand(T, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
        X = Xd.view(torch.int16).cpu().numpy().view(np.uint16)
        ref = (Xd.double() @ Wd.double().T).cpu().numpy()
        Y = np.zeros((T, M), np.float32)
        us = C.c_float()
        assert fn(W, X, M, K, T, 0, 0, Y, C.byref(us)) == 0
        err = np.abs(Y - ref).max()
        print(f"M={M} K={K} T={T}: max|err|={err:.3e} max|Y|={np.abs(ref).max():.1f} {us.value:.1f} us")
        assert err <= 2e-3 * np.abs(ref).max() + 1e-3


# ------------------------------------------------------------------ (c)
def test_c3_layer_truncated_forward_vs_float64(sd):
    st = c3_truncated_parity(sd, greedy_tokens=12)
    print("C3 L=2 bf16 vs float64:", st)
    assert st["max_abs_over_std"] <= 0.15
    assert st["mean_abs_over_std"] <= 0.03
    assert st["argmax_agree"] >= 0.9
    assert st["token_agree"] >= 0.75  # greedy streams, position-wise


def test_c5_layer_truncated_forward_vs_float64(sd):
    """(c') The C5 width (OPT-6.7B shape: h = 4096, 32 heads of 128) truncated
    to L = 2, with ~4k-token prompts: prefill through the 128-query kernel in
    256-token chunks, then one ragged verify forward over ~4.1k keys per
    sample, against the float64 reference; plus greedy decoding."""
    cfg = dict(num_layers=2, num_heads=32, head_dim=128, vocab_size=50272, max_positions=4480, init_seed=0xD5EED)
    st = c3_truncated_parity(sd, cfg=cfg, B=2, seed=3, greedy_tokens=6, lo=3968, hi=4224, cap=4352)
    print("C5 L=2 bf16 vs float64:", st)
    assert st["max_abs_over_std"] <= 0.15
    assert st["mean_abs_over_std"] <= 0.03
    assert st["argmax_agree"] >= 0.9
    assert st["token_agree"] >= 0.75


# ------------------------------------------------------------------ (d)
def test_long_prompt_prefill_vs_float64(sd):
    """(d) Prefill of 600-700-token prompts (forward chunks of <= 256 tokens cut
    at multiples of 256 from each prompt's start; the 128-query prefill
    attention kernel on runs of >= 64 queries) on the unpadded arena and on
    the left-padded vanilla grid,
    at the C3 width (L = 2): the stated bf16 tolerance on sampled rows and
    argmax agreement over every prompt row."""
    from torch_ref import prefill_parity

    st = prefill_parity(sd)
    print("prefill bf16 vs float64:", st)
    for layout, s in st.items():
        assert s["max_abs_over_std"] <= 0.15, layout
        assert s["mean_abs_over_std"] <= 0.03, layout
        assert s["argmax_agree"] >= 0.9 and s["argmax_agree_all_rows"] >= 0.9, layout


def test_compact_model_long_prompt_prefill_vs_float64(sd):
    """(d') The same on a small model (C2 / C4-draft shape, L = 2): the
    cluster-GEMM layer path (two 128-token launches per 256-token chunk) and
    the 128-query prefill attention at head_dim 64, unpadded arena and the
    left-padded vanilla grid, against the float64 reference."""
    from torch_ref import prefill_parity

    cfg = dict(num_layers=2, num_heads=12, head_dim=64, vocab_size=50272, max_positions=2048, init_seed=7)
    st = prefill_parity(sd, cfg=cfg, B=3, lo=150, hi=300, seed=5, every=7)
    print("compact prefill bf16 vs float64:", st)
    for layout, s in st.items():
        assert s["max_abs_over_std"] <= 0.15, layout
        assert s["mean_abs_over_std"] <= 0.03, layout
        assert s["argmax_agree"] >= 0.9 and s["argmax_agree_all_rows"] >= 0.9, layout
