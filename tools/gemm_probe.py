"""Time the tcgen05 GEMM in isolation on C3 shapes (sd_debug_gemm hook):
ten launches back to back, mean per launch, full GEMM and streaming kernel.

  python tools/gemm_probe.py [qkv o fc proj lm]
  python tools/gemm_probe.py --probe [shapes]   # bottleneck probes on the probe build
      (paper_2405_07542_b200/build.py --probe): the streaming kernel with its
      MMAs skipped / token loads skipped / partial stores skipped / all three
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_07542_b200 import specdec as sd  # noqa: E402

args = sys.argv[1:]
probe = "--probe" in args
if probe:
    args.remove("--probe")
    from paper_2405_07542_b200 import build as b

    sd.LIB_PATH = b.PROBE_LIB
L = sd.lib()
fn = L.sd_debug_gemm
fn.argtypes = [np.ctypeslib.ndpointer(np.uint16), np.ctypeslib.ndpointer(np.uint16), C.c_int, C.c_int, C.c_int,
               C.c_int, C.c_int, np.ctypeslib.ndpointer(np.float32), C.POINTER(C.c_float)]
rng = np.random.default_rng(0)
shapes = {"qkv": (15360, 5120), "o": (5120, 5120), "fc": (20480, 5120), "proj": (5120, 20480), "lm": (50272, 5120)}
only = args or list(shapes)
variants = ([("gemm", 0), ("stream", 8)] if not probe else
            [("stream", 8), ("noMMA", 8 | 16), ("noTok", 8 | 32), ("noPart", 8 | 64), ("W-only", 8 | 16 | 32 | 64)])
for name in only:
    M, K = shapes[name]
    W = rng.integers(0, 1 << 15, size=(M, K), dtype=np.uint16) & 0x3FFF
    for T in [int(x) for x in os.environ.get("TS", "48,112,192").split(",")]:
        X = rng.integers(0, 1 << 15, size=(T, K), dtype=np.uint16) & 0x3FFF
        Y = np.zeros((T, M), np.float32)
        res = []
        for label, flags in variants:
            us = C.c_float()
            best = 1e9
            for _ in range(3):
                assert fn(W, X, M, K, T, 0, flags | 128, Y, C.byref(us)) == 0
                best = min(best, us.value)
            res.append(f"{label}={best:6.1f}us ({M * K * 2 / best / 1e3:5.0f} GB/s)")
        print(f"{name:5s} T={T:3d} " + "  ".join(res), flush=True)
