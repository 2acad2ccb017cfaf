"""Untraced ms per verify step of the C2 device loop (OPT-125m shape, B=8,
512-id prompts, synthetic p=0.7 drafts): same-box A/B of SD_* settings.

  python tools/c2time.py [--lib path/to/other/libspecdec_b200.so]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_07542_b200 import specdec as sd  # noqa: E402
import bench  # noqa: E402

args = sys.argv[1:]
if "--lib" in args:  # A/B against another build of the library
    i = args.index("--lib")
    sd.LIB_PATH = os.path.abspath(args[i + 1])
cfg, B = bench.C2, 8
m = sd.Model.init(sd.ModelConfig(**cfg), device=0, precision=sd.BF16)
prompts = bench.prompts_for(range(B), cfg["vocab_size"], 512, 512)
e = sd.EngineConfig(mode="ems", predictor="synthetic", k=7, batch_size=B, max_new_tokens=128, stop_on_eos=False,
                    seed=1, synthetic_accuracy=0.7)
s = sd.Session(m, e, 512 + 128 + 9)
s.prefill(prompts)
g = sd.decode(sd.EngineConfig(mode="greedy", batch_size=B, max_new_tokens=128 + 9, stop_on_eos=False), m, prompts)
s.set_trajectory(np.array(g.generated_tokens, dtype=np.int32))
best = 1e9
for _ in range(6):
    s.reset()
    steps, ms = s.run()
    best = min(best, ms / steps)
env = " ".join([f"{k}={v}" for k, v in os.environ.items() if k.startswith("SD_")] +
               ([os.path.relpath(sd.LIB_PATH, ROOT)] if "--lib" in args else []))
print(f"[{env or 'default'}] C2 B={B}: {steps} steps, best {best:.4f} ms/step", flush=True)
