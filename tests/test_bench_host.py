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


def test_reference_steps_fixture_is_the_c3_trajectory():
    import json

    fx = json.load(open(bench.STEPS_FIXTURE))
    steps = fx["steps"]
    assert 50 <= len(steps) <= 130 and all(1 <= len(st) <= 24 for st in steps)
    for st in steps:
        for c, k, tau in st:
            assert 600 <= c <= 900 + 128 and 0 <= k <= 7 and 1 <= tau <= k + 1
    assert sum(tau for st in steps for _, _, tau in st) == 24 * 127  # 128 new tokens, the first from prefill


def test_run_metrics_padding_accounting():
    st = dict(steps=2, avg_tau=1.5, avg_padding_ratio=0.25, useful_kv_writes=10, kv_padding=3, input_padding=4,
              accepted=6)
    v, e = bench.run_metrics("vanilla", st, 6, 1.0), bench.run_metrics("ems", st, 6, 1.0)
    assert e["padding_kv_writes"] == 0 and v["padding_kv_writes"] == 3
    assert v["total_tokens_processed"] - e["total_tokens_processed"] == 3 + 4


def test_bench_csv_columns_extend_the_reference_schema():
    ref = ("batch_size,mode,predictor,k,total_tokens,decode_steps,avg_acceptance_length,avg_padding_ratio,"
           "total_input_padding,total_kv_padding,useful_kv_writes,padding_kv_writes,total_tokens_processed,"
           "decode_seconds,tokens_per_second_decode,tokens_per_second_total")  # tools/specdec_main.cpp:161-164
    assert bench.CSV_COLUMNS.startswith(ref + ",")
    assert bench.CSV_COLUMNS.split(",")[16:] == ["accepted_tok_s", "hbm_gbs", "roof_frac", "gpus", "cpu_cores"]


def test_gemm_algorithmic_bytes_cover_every_launch():
    b = bench.gemm_algorithmic_bytes(100, 40, 5120, 50272)
    assert len(b) == 4 * 40 + 1
    assert abs(sum(b) - (40 * 12 * 5120 ** 2 * 2 + 50272 * 5120 * 2 + 100 * 40 * (3 * 5120 + 20480) * 2
                         + 100 * 5120 * 2)) < 1


def test_reference_extrapolation_scales_with_layers():
    cfg = dict(bench.C3)
    one = bench.extrapolate(cfg, 1.0, 1, 14, 256)
    two = bench.extrapolate(cfg, 1.0, 2, 14, 256)
    assert one > two > 0  # timing more layers per sample means fewer extrapolated


def test_reference_bench_checks_follow_specdec_main():
    """The seven checks of tools/specdec_main.cpp:197-220 on hand-made runs:
    Table-1-like trajectory (taus (4, 1) then (2, 2)), identical across layouts."""
    from types import SimpleNamespace as NS

    steps = [{"samples": [{"sample": 0, "k": 3, "tau": 4, "clipped": False},
                          {"sample": 1, "k": 0, "tau": 1, "clipped": False}]},
             {"samples": [{"sample": 0, "k": 1, "tau": 2, "clipped": False},
                          {"sample": 1, "k": 1, "tau": 2, "clipped": False}]}]
    toks = [[5, 6, 7, 8, 9, 10], [5, 6, 7]]
    met = lambda useful, pad_w, in_pad, kv_pad, extra: {
        "useful_kv_writes": useful, "padding_kv_writes": pad_w, "total_input_padding": in_pad,
        "total_kv_padding": kv_pad, "total_tokens_processed": useful + extra}
    res = {"greedy": (NS(generated_tokens=toks, steps=[]), met(0, 0, 0, 0, 0)),
           "vanilla": (NS(generated_tokens=toks, steps=steps), met(8, 3, 3, 3, 6)),
           "ems": (NS(generated_tokens=toks, steps=steps), met(8, 0, 3, 3, 0))}
    chk = bench.reference_bench_checks(res)
    assert all(chk.values()), chk
    # a vanilla run that diverged fails exactly the cross-layout checks
    res["vanilla"] = (NS(generated_tokens=[toks[0], [5, 6, 4]], steps=steps[:1]), met(7, 3, 3, 3, 6))
    chk = bench.reference_bench_checks(res)
    assert not chk["aligned_output_matches_greedy"] and not chk["aligned_and_unpad_step_records_agree"]
    assert not chk["useful_writes_agree_across_layouts"]
    assert chk["unpad_output_matches_greedy"] and chk["unpad_wrote_zero_padding_slots"]


def test_in_graph_gemm_stage_classifies_and_times_each_stage():
    # one layer in program order: QKV stage, attention, O stage (+ LN), FC, PROJ (+ LN), then the LM head
    ls = [(1, 0, 100, 148, 148), (4, 90, 110, 1, 1),                     # QKV: 0 -> 110
          (9, 105, 170, 148, 148),                                        # attention ends at 170
          (1, 150, 240, 148, 148), (5, 235, 250, 1, 1), (6, 248, 260, 1, 1),  # O: 170 -> 260
          (1, 255, 400, 148, 148), (3, 395, 410, 1, 1),                   # FC: 260 -> 410
          (1, 405, 600, 148, 148), (5, 590, 615, 1, 1), (6, 612, 620, 1, 1),  # PROJ: 410 -> 620
          (1, 615, 700, 148, 148), (7, 690, 705, 1, 1),                   # LM head: 620 -> 705
          (12, 2000, 2001, 1, 1)]                                         # keeps the window open
    h, V = 64, 256
    r = bench.in_graph_gemm_stage((None, ls, (-1, 10_000)), hbm=1.0, h=h, vocab=V)
    pg = r["per_gemm"]
    assert set(pg) == {"qkv", "o", "fc", "proj", "lm"} and r["stages"] == 5
    assert pg["qkv"]["us_per_stage"] == 0.11 and pg["o"]["us_per_stage"] == 0.09
    assert pg["fc"]["us_per_stage"] == 0.15 and pg["proj"]["us_per_stage"] == 0.21
    assert pg["lm"]["us_per_stage"] == round(85 / 1e3, 2)
    assert pg["o"]["gbs"] == round(h * h * 2 / 90, 1)
