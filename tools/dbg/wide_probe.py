"""Probe the prefill attention kernel on small cases (debug helper)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
from paper_2405_07542_b200 import specdec as sd
from test_gpu_parity import make_attention_case, run_attention, attention_ref, from_bf16_bits

hd, heads = int(sys.argv[1]), int(sys.argv[2])
extents = [int(x) for x in sys.argv[3].split(",")]
nqs = [int(x) for x in sys.argv[4].split(",")]
rng = np.random.default_rng(0)
q, kv, n_q, kv_len, ws, pad, cap = make_attention_case(rng, extents, nqs, heads, hd, False)
out, us = run_attention(sd, q, kv, n_q, kv_len, ws, pad, heads, hd, cap)
ref = attention_ref(q, kv, n_q, kv_len, ws, pad, heads, hd)
got = from_bf16_bits(out).astype(np.float64)
err = np.abs(got - ref)
print("OK", sys.argv[1:], "max", err.max(), "mean", err.mean(), "finite", np.isfinite(got).all(), flush=True)
