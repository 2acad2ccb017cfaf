"""One FC -> PROJ chain (OPT-13B shapes) through sd_debug_chain, for ncu."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_2405_07542_b200 import specdec as sd
from test_gpu_bf16 import run_chain, to_bf16_bits

T = int(sys.argv[1]) if len(sys.argv) > 1 else 112
epi = int(sys.argv[2]) if len(sys.argv) > 2 else 2
K, M1, M2 = 5120, 20480, 5120
rng = np.random.default_rng(0)
X = to_bf16_bits(rng.uniform(-1, 1, (T, K)).astype(np.float32))
W1 = (rng.integers(0, 1 << 14, size=(M1, K), dtype=np.uint16) & 0x3BFF) | 0x3800
W2 = (rng.integers(0, 1 << 14, size=(M2, M1), dtype=np.uint16) & 0x3BFF) | 0x3000
b1 = np.zeros(M1, np.float32)
b2 = np.zeros(M2, np.float32)
for _ in range(2):
    run_chain(sd, X, W1, b1, W2, b2, np.zeros((T, M1), np.float32), epi)
print("ok")
