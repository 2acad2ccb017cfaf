"""Attribute the power-bound C3 step: the device loop at a FIXED token count
(synthetic drafts k=7 for all 24 samples: T = 192 every step) with parts of
the GEMM work switched off through SD_GEMM_DBG (bit0 skip MMAs, bit1 skip
partial stores; outputs are garbage, timing is what is measured)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_07542_b200 import specdec as sd  # noqa: E402
import bench  # noqa: E402

B = 24
K = int(os.environ.get("PROBE_K", 7))  # drafts per sample: T = B * (K + 1) every step
cfg = bench.C3
m = sd.Model.init(sd.ModelConfig(**cfg), device=0, precision=sd.BF16)
prompts = bench.prompts_for(range(B), cfg["vocab_size"], 600, 900)
cap = max(len(p) for p in prompts) + 128 + 9
e = sd.EngineConfig(mode="ems", predictor="synthetic", k=K, batch_size=B, max_new_tokens=64, stop_on_eos=False,
                    seed=1, synthetic_accuracy=0.0)
s = sd.Session(m, e, cap)
s.prefill(prompts)
rng = np.random.default_rng(0)
s.set_trajectory(rng.integers(3, cfg["vocab_size"], size=(B, 64 + 16)).astype(np.int32))
best = 1e9
for _ in range(3):
    s.reset()
    steps, ms = s.run()
    best = min(best, ms / steps)
print(f"[SD_GEMM_DBG={os.environ.get('SD_GEMM_DBG', '0')}] T={B * (K + 1)} fixed: {steps} steps, best {best:.3f} ms/step",
      flush=True)
