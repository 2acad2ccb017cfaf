import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
import pyoracle as P
from paper_2405_07542_b200 import specdec as sd
from test_gpu_bf16 import bf16_vs_oracle
o = P.Oracle()
for L, H, hd in [(1, 6, 128), (1, 16, 64), (1, 8, 64), (1, 12, 64), (1, 2, 384), (1, 8, 128)]:
    cfg = dict(num_layers=L, num_heads=H, head_dim=hd, vocab_size=1000, max_positions=512, init_seed=7)
    if hd not in (64, 128):
        continue
    lg, lo, am, amo = bf16_vs_oracle(sd, o, cfg, B=2, prompt_len=6, seed=7)
    d = np.abs(lg - lo); sc = lo.std()
    print(L, H, hd, "h=", H * hd, "T=", lg.shape[0], "max", round(float((d.max(axis=1) / sc).max()), 3),
          "agree", np.mean(am == amo), flush=True)
