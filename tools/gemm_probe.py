"""Time the tcgen05 GEMM in isolation on C3 shapes (sd_debug_gemm hook)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2405_07542_b200 import specdec as sd

L = sd.lib()
fn = L.sd_debug_gemm
fn.argtypes = [np.ctypeslib.ndpointer(np.uint16), np.ctypeslib.ndpointer(np.uint16), C.c_int, C.c_int, C.c_int,
               C.c_int, C.c_int, np.ctypeslib.ndpointer(np.float32), C.POINTER(C.c_float)]
rng = np.random.default_rng(0)
shapes = {"qkv": (15360, 5120), "o": (5120, 5120), "fc": (20480, 5120), "proj": (5120, 20480), "lm": (50272, 5120)}
only = sys.argv[1:] or list(shapes)
for name in only:
    M, K = shapes[name]
    W = rng.integers(0, 1 << 15, size=(M, K), dtype=np.uint16) & 0x3FFF
    for T in (48, 112, 192):
        X = rng.integers(0, 1 << 15, size=(T, K), dtype=np.uint16) & 0x3FFF
        Y = np.zeros((T, M), np.float32)
        res = []
        for grid, flags in ((0, 0), (0, 8)):
            us = C.c_float()
            best = 1e9
            for _ in range(3):
                fn(W, X, M, K, T, grid, flags, Y, C.byref(us))
                best = min(best, us.value)
            res.append(f"{'stream' if flags else 'gemm'}={best:7.1f}us ({M * K * 2 / best / 1e3:6.0f} GB/s)")
        print(f"{name:5s} T={T:3d} " + "  ".join(res), flush=True)
