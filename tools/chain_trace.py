"""Phase timeline of one FC -> PROJ chain (OPT-13B shapes) via sd_debug_chain
with the in-kernel trace points, for A/B of epilogue variants (flags)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
sys.path.insert(0, "tools")
from paper_2405_07542_b200 import specdec as sd
from test_gpu_bf16 import run_chain, to_bf16_bits
from timeline import REC

L = sd.lib()
L.sd_debug_trace_begin.argtypes = [C.c_int]
L.sd_debug_trace_end.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int)]
T = int(sys.argv[1]) if len(sys.argv) > 1 else 96
K, M1, M2 = 5120, 20480, 5120
rng = np.random.default_rng(0)
X = to_bf16_bits(rng.uniform(-1, 1, (T, K)).astype(np.float32))
W1 = (rng.integers(0, 1 << 14, size=(M1, K), dtype=np.uint16) & 0x3BFF) | 0x3800
W2 = (rng.integers(0, 1 << 14, size=(M2, M1), dtype=np.uint16) & 0x3BFF) | 0x3000
b1 = np.zeros(M1, np.float32)
b2 = np.zeros(M2, np.float32)
names = {101: "A first", 102: "B dep", 103: "MMA done", 104: "drain", 105: "reduce", 106: "done", 107: "jobdata", 108: "jobdone", 109: "own-ready", 110: "others-in"}
for flags in [int(x) for x in (sys.argv[2:] or ["0"])]:
    for rep in range(2):
        run_chain(sd, X, W1, b1, W2, b2, np.zeros((T, M1), np.float32), 2, flags)
    assert L.sd_debug_trace_begin(200000) == 0
    run_chain(sd, X, W1, b1, W2, b2, np.zeros((T, M1), np.float32), 2, flags)
    buf = np.zeros(200000, REC)
    n = C.c_int()
    assert L.sd_debug_trace_end(buf.ctypes.data, 200000, C.byref(n)) == 0
    rec = buf[:n.value]
    g = rec[rec["kid"] == 1]
    t0 = g["t0"].min()
    print(f"flags={flags} T={T} kernel {(g['t1'].max() - t0) / 1e3:.1f} us")
    pts = rec[rec["kid"] >= 100]
    for gi in range(2):
        row = []
        for k in (101, 102, 103, 109, 110, 107, 108, 104, 105, 106):
            v = pts[(pts["kid"] == k) & (((pts["blk"] >> 16) & 0xff) == gi)]
            if len(v):
                d = (v["t0"].astype(np.int64) - t0) / 1e3
                row.append(f"{names[k]} {np.median(d):.1f}/{d.max():.1f}")
        print(f"  g{gi}: " + " | ".join(row))
