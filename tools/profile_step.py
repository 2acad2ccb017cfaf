"""Profile one C3 verify step: prefill outside the profiled range, then
cuProfilerStart() / N eager device steps / cuProfilerStop() so that
`ncu --profile-from-start off` captures exactly the step's kernels.

META=path writes the profiled step's shape next to the launch list (token
count T and each sample's KV extent), so bench.py charges the ncu DRAM bytes
against the algorithmic bytes of the SAME step."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2405_07542_b200 import specdec as sd  # noqa: E402

import numpy as np  # noqa: E402

C2 = os.environ.get("CONFIG", "c3") == "c2"  # CONFIG=c2: OPT-125m shape, B=8, 512-id prompts, synthetic drafts
B = int(os.environ.get("B", 8 if C2 else 24))
steps = int(os.environ.get("STEPS", 1))
cfg = bench.C2 if C2 else bench.C3
m = sd.Model.init(sd.ModelConfig(**cfg), precision=sd.BF16)
prompts = bench.prompts_for(range(B), cfg["vocab_size"], *((512, 512) if C2 else (600, 900)))
e = sd.EngineConfig(mode=os.environ.get("MODE", "ems"), predictor="synthetic" if C2 else "retrieval", k=7,
                    copy_len=7, batch_size=B, max_new_tokens=128, stop_on_eos=False, seed=1,
                    synthetic_accuracy=0.7)
cap = max(map(len, prompts)) + 140 if e.mode == "ems" else 2048
s = sd.Session(m, e, cap)
s.prefill(prompts)
if C2:
    g = sd.decode(sd.EngineConfig(mode="greedy", batch_size=B, max_new_tokens=128 + 9, stop_on_eos=False), m, prompts)
    s.set_trajectory(np.array(g.generated_tokens, dtype=np.int32))
L = sd.lib()
L.sd_session_step.argtypes = [C.c_void_p, C.c_int]
# advance into the generation so drafts exist, then profile
assert L.sd_session_step(s._h, 20) == 0
toks0, _, _ = s.outputs()
committed = [len(p) + len(t) - 1 for p, t in zip(prompts, toks0)]  # ctx_len - 1 (engine.cpp:465-470)
cuda = C.CDLL("libcuda.so.1")
cuda.cuProfilerStart()
assert L.sd_session_step(s._h, steps) == 0
cuda.cuProfilerStop()
print("profiled", steps, "step(s)")
if os.environ.get("META") and steps == 1:
    _, lk, _ = s.outputs()
    k = lk[20].tolist()
    meta = {"config": "C2" if C2 else "C3", "batch": B, "mode": e.mode, "step_index": 20, "k": k,
            "T": int(sum(1 + x for x in k if x >= 0)),
            "kv_len": [c + 1 + x if x >= 0 else 0 for c, x in zip(committed, k)],
            "num_layers": cfg["num_layers"], "hidden": cfg["num_heads"] * cfg["head_dim"],
            "vocab": cfg["vocab_size"]}
    json.dump(meta, open(os.environ["META"], "w"), indent=1)
    print("meta", meta["T"], "tokens")
