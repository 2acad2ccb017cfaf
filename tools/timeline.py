"""In-graph kernel timeline of the C3 verify loop (sd_debug_trace_*).

Runs the device-resident loop (CUDA-graph replay, PDL chain) with per-CTA
globaltimer records on, then reconstructs launches (records of one kernel id
sorted by entry time, chunked by grid size) and prints, for steady-state
verify steps: step time, per-kernel-class busy time (union of its launches'
[first entry, last exit]), exposed gaps, and one layer's launch sequence.

  python tools/timeline.py [--batch 24] [--steps-traced 6] [--out gpurun_out/timeline.txt]
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys
from collections import defaultdict

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NAMES = {1: "gemm", 2: "red_store", 3: "red_gelu", 4: "red_qkv", 5: "red_resid", 6: "ln_rows", 7: "argmax",
         8: "embed_ln", 9: "attention", 10: "attn_combine", 11: "predict", 12: "pack", 13: "accept", 14: "pad_fill",
         15: "draft_pack", 16: "draft_take", 17: "draft_commit", 18: "cl_qkv", 19: "cl_gelu", 20: "cl_resid"}
from bench import TRACE_REC as REC, trace_launches as launches  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=24)
    ap.add_argument("--cap", type=int, default=6_000_000)
    ap.add_argument("--mode", default="ems")
    ap.add_argument("--draft", action="store_true", help="C4: OPT-125m-shaped draft model, k=4")
    ap.add_argument("--tail", action="store_true", help="print the step's head and tail launches instead of layer 1")
    ap.add_argument("--config", default="c3", choices=["c3", "c2", "c5"],
                    help="c2: OPT-125m shape, B=8, 512-id prompts, synthetic p=0.7 drafts (bench --config c2)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "timeline.txt"))
    a = ap.parse_args()
    import bench
    from paper_2405_07542_b200 import specdec as sd

    L = sd.lib()
    L.sd_debug_trace_begin.argtypes = [C.c_int]
    L.sd_debug_trace_end.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int)]
    cfg = {"c2": bench.C2, "c5": bench.C5}.get(a.config, bench.C3)
    if a.config in ("c2", "c5") and "--batch" not in sys.argv:
        a.batch = 8
    m = sd.Model.init(sd.ModelConfig(**cfg), device=0, precision=sd.BF16)
    lo_hi = {"c2": (512, 512), "c5": (3968, 4224)}.get(a.config, (600, 900))
    prompts = bench.prompts_for(range(a.batch), cfg["vocab_size"], *lo_hi)
    cap = max(len(p) for p in prompts) + 128 + 9 if a.mode == "ems" else cfg["max_positions"]
    if a.draft:
        d = sd.Model.init(sd.ModelConfig(**dict(bench.C2, init_seed=cfg["init_seed"] + 1)), device=0, precision=sd.BF16)
        e = sd.EngineConfig(mode=a.mode, predictor="draft", k=4, batch_size=a.batch, max_new_tokens=128,
                            stop_on_eos=False)
        s = sd.Session(m, e, cap, draft=d)
    elif a.config == "c2":
        e = sd.EngineConfig(mode=a.mode, predictor="synthetic", k=7, batch_size=a.batch, max_new_tokens=128,
                            stop_on_eos=False, seed=1, synthetic_accuracy=0.7)
        s = sd.Session(m, e, cap)
        g = sd.decode(sd.EngineConfig(mode="greedy", batch_size=a.batch, max_new_tokens=128 + 9, stop_on_eos=False),
                      m, prompts)
        s.set_trajectory(np.array(g.generated_tokens, dtype=np.int32))
    else:
        e = sd.EngineConfig(mode=a.mode, predictor="retrieval", k=7, match_len=2, copy_len=7, batch_size=a.batch,
                            max_new_tokens=128, stop_on_eos=False, seed=1)
        s = sd.Session(m, e, cap)
    s.prefill(prompts)
    for _ in range(2):
        s.reset()
        steps, ms = s.run()
    print(f"untraced: {steps} steps {ms:.1f} ms -> {ms / steps:.3f} ms/step", flush=True)
    s.reset()
    assert L.sd_debug_trace_begin(a.cap) == 0
    steps, ms = s.run()
    buf = np.zeros(a.cap, REC)
    n = C.c_int()
    assert L.sd_debug_trace_end(buf.ctypes.data, a.cap, C.byref(n)) == 0
    rec = buf[:n.value]
    print(f"traced: {steps} steps {ms:.1f} ms, {n.value} records", flush=True)
    ls = launches(rec)
    # verify steps delimited by k_predict launches; drop the last (possibly truncated) one
    starts = [l[1] for l in ls if l[0] == (17 if a.draft else 11)]
    lines = []
    tot = defaultdict(float)
    gaps_tot, n_steps, step_tot = 0.0, 0, 0.0
    for si in range(1, len(starts) - 1):
        t_a, t_b = starts[si], starts[si + 1]
        st = [l for l in ls if t_a <= l[1] < t_b]
        busy = defaultdict(float)
        # exposed gap: time where no launch is active
        ev = sorted([(l[1], 1) for l in st] + [(l[2], -1) for l in st])
        act, last, idle = 0, t_a, 0.0
        for t, d in ev:
            if act == 0 and t > last:
                idle += t - last
            act += d
            last = t
        for l in st:
            busy[NAMES[l[0]]] += (l[2] - l[1]) / 1e3
        for k, v in busy.items():
            tot[k] += v
        gaps_tot += idle / 1e3
        step_tot += (t_b - t_a) / 1e3
        n_steps += 1
        if si == 2:
            lines.append(f"--- step {si}: {len(st)} launches, {(t_b - t_a) / 1e3:.1f} us; layer 1 sequence:")
            gemm_i = [i for i, l in enumerate(st) if l[0] in (1, 18, 19, 20)]
            lo, hi = (0, min(len(st), 60)) if a.draft else (gemm_i[4], min(len(st), gemm_i[8] + 3))
            prev_end = st[lo - 1][2]
            seq = list(range(lo, hi))
            if a.tail:  # the step's first 4 and last 10 launches (embed / LM head / accept)
                seq = list(range(0, 4)) + list(range(max(4, len(st) - 10), len(st)))
                prev_end = t_a
            for l in [st[j] for j in seq]:
                lines.append(f"  {NAMES[l[0]]:13s} start {(l[1] - t_a) / 1e3:9.1f} dur {(l[2] - l[1]) / 1e3:7.1f} "
                             f"gap {(l[1] - prev_end) / 1e3:6.1f} ctas {l[3]:5d} sms {l[4]:3d} "
                             f"end-after-prev {(l[2] - prev_end) / 1e3:6.1f}")
                if l[0] in (2, 3, 4, 5, 6, 7, 9):  # per-CTA entry / exit spread (us after the predecessor's end)
                    r = rec[(rec["kid"] == l[0]) & (rec["t0"] >= l[1]) & (rec["t1"] <= l[2])]
                    if len(r):
                        en = (r["t0"].astype(np.int64) - prev_end) / 1e3
                        ex = (r["t1"].astype(np.int64) - prev_end) / 1e3
                        q = lambda v: "/".join(f"{x:.1f}" for x in np.percentile(v, [10, 50, 90, 100]))
                        lines.append(f"      ctas {len(r)}: entry p10/50/90/max {q(en)} | exit {q(ex)}")
                        if l[0] in (3, 4, 5) and len(r) > 20:  # reductions: who is slow (grid x = tile, y = group)
                            gx = {4: 60, 3: 80, 5: 20}[l[0]] if a.config == "c3" else None
                            if gx:
                                slow = r[ex >= np.percentile(ex, 90)]
                                ys = (slow["blk"] // gx).astype(int)
                                xs = (slow["blk"] % gx).astype(int)
                                lines.append(f"      slowest 10%: y {np.bincount(ys).nonzero()[0].tolist()} "
                                             f"x {sorted(set(xs.tolist()))[:40]} sms {len(set(slow['smid'].tolist()))}")
                if l[0] == 9:  # attention phases of each CTA's first item (trace points 130-133)
                    pts = rec[(rec["kid"] >= 130) & (rec["kid"] <= 133) & (rec["t0"] >= l[1]) & (rec["t0"] <= l[2])]
                    row = []
                    for k, nm in ((130, "dep"), (131, "S0 issued"), (132, "S0 ready"), (133, "item done")):
                        v = pts[pts["kid"] == k]
                        if len(v):
                            d = (v["t0"].astype(np.int64) - prev_end) / 1e3
                            row.append(f"{nm} {np.median(d):5.1f}/{d.max():5.1f}")
                    v = pts[pts["kid"] == 133]
                    if len(v):
                        row.append(f"chunks/item {np.median(v['blk'] >> 20):.0f}")
                    lines.append("      phases (median/max): " + " | ".join(row))
                if l[0] in (18, 19, 20):  # cluster GEMM phases (trace points 120-125), us after the predecessor's end
                    epi = {18: 3, 19: 2, 20: 1}[l[0]]
                    pts = rec[(rec["kid"] >= 120) & (rec["kid"] <= 127) & (rec["t0"] >= l[1]) & (rec["t0"] <= l[2])
                              & ((rec["blk"] >> 24) == epi)]
                    row = []
                    for k, nm in ((120, "dep"), (121, "ln"), (122, "mma"), (126, "tmem"), (127, "nbar"), (123, "push"),
                                  (124, "recv"), (125, "epi")):
                        v = pts[pts["kid"] == k]
                        if len(v):
                            d = (v["t0"].astype(np.int64) - prev_end) / 1e3
                            row.append(f"{nm} {np.median(d):5.1f}/{d.max():5.1f}")
                    lines.append("      phases (median/max): " + " | ".join(row))
                prev_end = max(prev_end, l[2])
    # phases inside persistent GEMM chains (trace points 101..106)
    pts = rec[rec["kid"] >= 100]
    if len(pts) and n_steps:
        names = {101: "A first load", 102: "B dep ok", 103: "MMA done", 104: "drain done", 105: "reduce done",
                 106: "LN/done"}
        t_a = starts[2]
        ch = [l for l in ls if l[0] == 1 and l[1] >= t_a][2:4]
        for c in ch:
            lines.append(f"--- chain at {(c[1] - t_a) / 1e3:.1f} us, dur {(c[2] - c[1]) / 1e3:.1f} us (phase times rel. chain start: min/med/max)")
            sel = pts[(pts["t0"] >= c[1]) & (pts["t0"] <= c[2])]
            for gi in range(4):
                row = []
                for k in range(101, 107):
                    v = sel[(sel["kid"] == k) & (((sel["blk"] >> 16) & 0xff) == gi)]
                    if len(v):
                        d = (v["t0"].astype(np.int64) - c[1]) / 1e3
                        row.append(f"{names[k]} {d.min():6.1f}/{np.median(d):6.1f}/{d.max():6.1f}")
                lines.append(f"  g{gi}: " + " | ".join(row))
                for k in (107, 108):
                    v = sel[(sel["kid"] == k) & (((sel["blk"] >> 16) & 0xff) == gi)]
                    for jn in range(6):
                        w = v[(v["blk"] >> 24) == jn]
                        if len(w):
                            d = (w["t0"].astype(np.int64) - c[1]) / 1e3
                            lines.append(f"      {'job data' if k == 107 else 'job done'} {jn}: n={len(w)} "
                                         f"{d.min():6.1f}/{np.median(d):6.1f}/{d.max():6.1f}")
    lines.append(f"=== {n_steps} steady steps, avg {step_tot / max(1, n_steps):.1f} us/step; "
                 f"no-kernel-running time {gaps_tot / max(1, n_steps):.1f} us/step")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"  {k:13s} {v / max(1, n_steps):9.1f} us/step (launch spans, overlaps double-count)")
    txt = "\n".join(lines)
    print(txt)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        f.write(txt + "\n")
    np.save(os.path.join(os.path.dirname(a.out), "timeline_rec.npy"), rec[: min(len(rec), 2_000_000)])


if __name__ == "__main__":
    main()
