"""The reference-shaped C++ layer (include/specdec_b200.hpp):
it compiles and links against libspecdec_b200.so with the reference's type
and function names (CPU), and a program written like engine.cpp:427-485
against it reproduces the CPU oracle bit for bit on the GPU (fp32 check mode):
every logits row (FNV-1a of its bytes), every greedy pick, tau and committed
length, the ledger, and the reference's exception types."""
import os
import subprocess

import numpy as np
import pytest

import pyoracle as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2405_07542_b200", "lib")
SRC = os.path.join(ROOT, "tests", "native", "cpp_layer_test.cpp")


def build_cpp(tmp_path):
    exe = str(tmp_path / "cpp_layer_test")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                        SRC, "-L", LIBDIR, "-lspecdec_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_layer_compiles_and_links(sd, tmp_path):  # sd: the library is built and loads
    exe = build_cpp(tmp_path)
    assert os.path.getsize(exe) > 0


@pytest.mark.gpu
def test_cpp_layer_matches_oracle(sd, tmp_path, oracle):
    exe = build_cpp(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = [l.split() for l in out.stdout.splitlines()]

    # replay the same calls on the CPU oracle
    cfg = dict(num_layers=2, num_heads=2, head_dim=16, vocab_size=259, max_positions=512, init_seed=0xD5EED)
    V, B, cap = cfg["vocab_size"], 3, 64
    m = oracle.model_init(cfg)
    c = oracle.cache_new(0, cfg["num_layers"], B, cap, cfg["num_heads"] * cfg["head_dim"])
    expect = [["checksum", str(oracle.checksum(m))]]

    def fwd(tag, per_sample):
        slots = []
        for s, seq in enumerate(per_sample):
            slots += [(s, oracle.committed(c, s) + j) for j in range(len(seq))]
        logits, am = oracle.forward(m, c, per_sample, slots, V)
        h = P.fnv_rows(logits)
        for i in range(len(h)):
            expect.append(["fwd", str(tag), str(i), str(int(h[i])), str(int(np.argmax(logits[i])))])
        return logits

    prompts = [[0, 72, 101, 108, 108, 111], [0, 87, 111], [0, 33, 34, 35, 36]]
    rows = fwd(0, prompts)
    last, off = [], 0
    for s, p in enumerate(prompts):
        off += len(p)
        last.append(int(np.argmax(rows[off - 1])))
        oracle.commit(c, s, len(p))
    drafts = [[[5, 6], [], [7]], [[9], [10, 11, 12], [13, 14]]]
    for step in range(2):
        ins = [[last[s]] + drafts[step][s] for s in range(B)]
        rows = fwd(step + 1, ins)
        off = 0
        for s in range(B):
            mine = rows[off: off + len(ins[s])]
            off += len(ins[s])
            acc = []
            for j in range(len(mine)):  # engine.cpp:60-76
                acc.append(int(np.argmax(mine[j])))
                if j == len(drafts[step][s]) or acc[-1] != drafts[step][s][j]:
                    break
            oracle.commit(c, s, len(acc))
            last[s] = acc[-1]
            expect.append(["tau", str(step + 1), str(s), str(len(acc)), str(oracle.committed(c, s))])
    oracle.cache_free(c)
    oracle.model_free(m)

    got = lines[: len(expect)]
    assert got == expect
    tail = {l[0]: l[1:] for l in lines[len(expect):]}
    useful = sum(len(p) for p in prompts) + sum(1 + len(d) for st in drafts for d in st)
    assert tail["ledger"] == [str(useful), "0"]  # every written slot counted once, no padding
    assert tail["start_offset"] == [str(2 * cap)]  # kv_cache.cpp:116-120
    assert tail["contract_error_ok"] == ["prefixed"]
    committed = [e[4] for e in expect if e[0] == "tau" and e[1] == "2"]
    assert tail["lengths"] == committed + [str(s * cap) for s in range(B)]
    assert tail["batched_commit_rejected"] == ["3"] + committed  # SD_CONTRACT, nothing mutated
    assert "config_error_ok" in tail and "commit_error_ok" in tail
    # PaddedGrid through the header: filler rows 3 then 3 + 4, rows advance by tau_max, sample 1's
    # logical length by its own taus, and its first-step shortfall rows are pad rows
    assert tail["grid_padding"] == ["3", "7", "11", str(1 + 1 + 6), "1"]
