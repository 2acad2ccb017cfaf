"""Streaming-kernel probe: token-ring depth (flags bits 5-7) x weight layout."""
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
modes = {}
for sb in (2, 3, 4, 6):
    modes[f"sb{sb}"] = 8 | (sb << 5)
for sb in (2, 4):
    modes[f"tiled_sb{sb}"] = 8 | 1 | (sb << 5)
modes["noMMA_sb4"] = 8 | 2 | (4 << 5)
modes["nostore_sb4"] = 8 | 4 | (4 << 5)
for name in (sys.argv[1:] or list(shapes)):
    M, K = shapes[name]
    W = rng.integers(0, 1 << 15, size=(M, K), dtype=np.uint16) & 0x3FFF
    for T in (112, 192):
        X = rng.integers(0, 1 << 15, size=(T, K), dtype=np.uint16) & 0x3FFF
        Y = np.zeros((T, M), np.float32)
        res = []
        for mname, flags in modes.items():
            us = C.c_float()
            best = 1e9
            for _ in range(5):
                fn(W, X, M, K, T, 0, flags, Y, C.byref(us))
                best = min(best, us.value)
            res.append(f"{mname}={best:5.1f}/{M * K * 2 / best / 1e3:4.0f}")
        print(f"{name:5s} T={T:3d} " + " ".join(res), flush=True)
