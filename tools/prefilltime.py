"""Wall time of the chunked prefill (engine.cpp:330-385) through sd_session_prefill:
C5 (OPT-6.7B shape, 8 x ~4.1k-token prompts) or C3 (OPT-13B, 24 x 600-900).

  python tools/prefilltime.py [--c3] [--lib other.so]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_07542_b200 import specdec as sd  # noqa: E402
import bench  # noqa: E402

args = sys.argv[1:]
if "--lib" in args:
    i = args.index("--lib")
    sd.LIB_PATH = os.path.abspath(args[i + 1])
    del args[i:i + 2]
c3 = "--c3" in args
cfg, B, lo, hi = (bench.C3, 24, 600, 900) if c3 else (bench.C5, 8, 3968, 4224)
m = sd.Model.init(sd.ModelConfig(**cfg), device=0, precision=sd.BF16)
prompts = bench.prompts_for(range(B), cfg["vocab_size"], lo, hi)
n = sum(len(p) for p in prompts)
e = sd.EngineConfig(mode="ems", predictor="retrieval", k=7, copy_len=7, batch_size=B, max_new_tokens=16,
                    stop_on_eos=False)
s = sd.Session(m, e, max(len(p) for p in prompts) + 32)
best = 1e9
for _ in range(3):
    t0 = time.perf_counter()
    s.prefill(prompts)
    best = min(best, time.perf_counter() - t0)
lib = os.path.relpath(sd.LIB_PATH, ROOT) if "--lib" in sys.argv else "default"
print(f"[{lib}] {'C3' if c3 else 'C5'} prefill B={B}, {n} tokens: best {best * 1e3:.1f} ms "
      f"({n / best:.0f} tok/s)", flush=True)
