"""Untraced ms per verify step of the C3 device loop (A/B helper: run under
different SD_* environment settings in the same box).

  python tools/steptime.py [B] [--lib path/to/other/libspecdec_b200.so]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_07542_b200 import specdec as sd  # noqa: E402
import bench  # noqa: E402

args = sys.argv[1:]
if "--lib" in args:  # A/B against another build of the library
    i = args.index("--lib")
    sd.LIB_PATH = os.path.abspath(args[i + 1])
    del args[i:i + 2]
eager = "--eager" in args  # launch-by-launch instead of the CUDA-graph replay
if eager:
    args.remove("--eager")
c5 = "--c5" in args  # long context: OPT-6.7B shape, 4k prompts (retrieval drafts)
if c5:
    args.remove("--c5")
B = int(args[0]) if args else (8 if c5 else 24)
cfg = bench.C5 if c5 else bench.C3
m = sd.Model.init(sd.ModelConfig(**cfg), device=0, precision=sd.BF16)
prompts = bench.prompts_for(range(B), cfg["vocab_size"], *((3968, 4224) if c5 else (600, 900)))
cap = max(len(p) for p in prompts) + 128 + 9
e = sd.EngineConfig(mode="ems", predictor="retrieval", k=7, match_len=2, copy_len=7, batch_size=B, max_new_tokens=128,
                    stop_on_eos=False, seed=1)
s = sd.Session(m, e, cap)
s.prefill(prompts)
best = 1e9
for _ in range(4):
    s.reset()
    steps, ms = s.run(use_graph=not eager)
    best = min(best, ms / steps)
env = " ".join([f"{k}={v}" for k, v in os.environ.items() if k.startswith("SD_")] +
               ([os.path.relpath(sd.LIB_PATH, ROOT)] if "--lib" in sys.argv else []) + (["eager"] if eager else []))
print(f"[{env or 'default'}] {'C5' if c5 else 'C3'} B={B}: {steps} steps, best {best:.3f} ms/step", flush=True)
