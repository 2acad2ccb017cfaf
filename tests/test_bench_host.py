"""Host-side logic of bench.py (no GPU): the in-graph timeline reconstruction
behind `roofline.in_graph`, the reference-arm extrapolation and the prompt
generator the parity tests and the bench share."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def rec(kid, n, t0s, t1s, sm0=0):
    r = np.zeros(len(t0s), bench.TRACE_REC)
    r["kid"], r["n"], r["t0"], r["t1"] = kid, n, t0s, t1s
    r["smid"] = np.arange(len(t0s)) + sm0
    r["blk"] = np.arange(len(t0s))
    return r


def test_trace_launches_chunks_by_grid_and_sorts_by_start():
    # two launches of kernel 1 (grid 3), one of kernel 9 (grid 2) in between
    a = rec(1, 3, [100, 105, 101], [150, 160, 155])
    b = rec(9, 2, [170, 171], [300, 290])
    c = rec(1, 3, [310, 312, 311], [400, 420, 410])
    pts = rec(110, 0, [200], [200])  # trace points (kid >= 100) are not launches
    ls = bench.trace_launches(np.concatenate([c, pts, b, a]))
    assert [(l[0], l[1], l[2], l[3]) for l in ls] == [(1, 100, 160, 3), (9, 170, 300, 2), (1, 310, 420, 3)]
    assert all(l[4] == l[3] for l in ls)  # one SM per CTA in this synthetic trace


def test_prompts_are_deterministic_and_in_range():
    p1 = bench.prompts_for(range(4), 1000, 20, 30)
    p2 = bench.prompts_for(range(4), 1000, 20, 30)
    assert p1 == p2
    assert all(20 <= len(p) <= 30 and p[0] == 0 for p in p1)  # BOS + ids, lengths in [lo, hi]
    assert all(3 <= t < 1000 for p in p1 for t in p[1:])
    # sharding: the same global sample id gets the same prompt on any rank
    assert bench.prompts_for([2, 3], 1000, 20, 30) == p1[2:]


def test_reference_extrapolation_scales_with_layers():
    cfg = dict(bench.C3)
    one = bench.extrapolate(cfg, 1.0, 1, 14, 256)
    two = bench.extrapolate(cfg, 1.0, 2, 14, 256)
    assert one > two > 0  # timing more layers per sample means fewer extrapolated
