"""Profile one C3 verify step: prefill outside the profiled range, then
cuProfilerStart() / N eager device steps / cuProfilerStop() so that
`ncu --profile-from-start off` captures exactly the step's kernels."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2405_07542_b200 import specdec as sd  # noqa: E402

B = int(os.environ.get("B", 24))
steps = int(os.environ.get("STEPS", 1))
cfg = bench.C3
m = sd.Model.init(sd.ModelConfig(**cfg), precision=sd.BF16)
prompts = bench.prompts_for(range(B), cfg["vocab_size"], 600, 900)
e = sd.EngineConfig(mode=os.environ.get("MODE", "ems"), predictor="retrieval", k=7, copy_len=7, batch_size=B,
                    max_new_tokens=128, stop_on_eos=False)
cap = max(map(len, prompts)) + 140 if e.mode == "ems" else 2048
s = sd.Session(m, e, cap)
s.prefill(prompts)
L = sd.lib()
L.sd_session_step.argtypes = [C.c_void_p, C.c_int]
# advance into the generation so drafts exist, then profile
assert L.sd_session_step(s._h, 20) == 0
cuda = C.CDLL("libcuda.so.1")
cuda.cuProfilerStart()
assert L.sd_session_step(s._h, steps) == 0
cuda.cuProfilerStop()
print("profiled", steps, "step(s)")
