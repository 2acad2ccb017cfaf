"""C-ABI library: loads, exports every declared symbol, host-only logic works
without a GPU, and compute calls fail loudly (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "specdec_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\s*\**\s*(sd_[a-z0-9_]+)\(", src, re.M)))


def test_header_declares_the_hot_path(sd):
    syms = declared_symbols()
    for needed in ("sd_model_init", "sd_cache_create", "sd_forward", "sd_verify_step", "sd_cache_commit_accepted",
                   "sd_cache_commit_padded", "sd_restore_indices", "sd_decode", "sd_last_error"):
        assert needed in syms


def test_library_exports_every_declared_symbol(sd):
    out = subprocess.run(["nm", "-D", "--defined-only", sd.LIB_PATH], capture_output=True, text=True, check=True)
    exported = set(re.findall(r" T (sd_[a-z0-9_]+)$", out.stdout, re.M))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_library_is_sm100a(sd):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sd.LIB_PATH], capture_output=True,
                         text=True, check=True)
    assert "sm_100a" in out.stdout


def test_restore_indices_kats(sd):
    """test_ragged.cpp:29-37 known answers through the C ABI."""
    counts = [5, 2]
    assert sd.restore_indices(counts, 0) == sd.TokenSlot(0, 0)
    assert sd.restore_indices(counts, 4) == sd.TokenSlot(0, 4)
    assert sd.restore_indices(counts, 5) == sd.TokenSlot(1, 0)
    assert sd.restore_indices(counts, 6) == sd.TokenSlot(1, 1)
    with pytest.raises(sd.ContractError):
        sd.restore_indices(counts, 7)
    with pytest.raises(sd.ContractError):
        sd.restore_indices(counts, -1)
    # zero-length samples keep their count entry (test_ragged.cpp:18-24)
    b = sd.concatenate_inputs([[1], [], [2, 3]])
    assert b.concatenated_tokens == [1, 2, 3] and b.token_nums_per_sample == [1, 0, 2]
    assert sd.restore_indices(b.token_nums_per_sample, 1) == sd.TokenSlot(2, 0)
    with pytest.raises(sd.ContractError):
        sd.concatenate_inputs([])


def test_restore_indices_prefix_sum_oracle(sd):
    """test_ragged.cpp:39-60: 200 random count lists against a prefix-sum table."""
    rng = np.random.default_rng(0x5107)
    for _ in range(200):
        counts = rng.integers(0, 7, size=int(rng.integers(1, 13))).tolist()
        table = [(s, p) for s, c in enumerate(counts) for p in range(c)]
        for flat, (s, p) in enumerate(table):
            assert sd.restore_indices(counts, flat) == sd.TokenSlot(s, p)
        with pytest.raises(sd.ContractError):
            sd.restore_indices(counts, len(table))


def test_config_validation(sd):
    """test_model.cpp:96-110"""
    sd.ModelConfig().validate()
    for field, bad in (("num_layers", 0), ("num_heads", 0), ("head_dim", -1), ("vocab_size", 1),
                       ("max_positions", 0)):
        cfg = sd.ModelConfig()
        setattr(cfg, field, bad)
        with pytest.raises(sd.ConfigError):
            cfg.validate()


def test_verify_host_kats(sd):
    """test_engine.cpp:63-86 (host-side verify over logits rows)."""
    def row(i):
        r = np.zeros(259, np.float32)
        r[i] = 1.0
        return r
    rows = [row(7), row(3), row(1), row(5)]
    v = sd.verify(rows, [7, 3, 9])
    assert v.tau == 3 and v.accepted == [7, 3, 1]
    v = sd.verify(rows, [7, 3, 1])
    assert v.tau == 4 and v.accepted == [7, 3, 1, 5]
    v = sd.verify(rows, [9, 3, 1])
    assert v.tau == 1 and v.accepted == [7]
    v = sd.verify([row(6)], [])
    assert v.tau == 1 and v.accepted == [6]
    with pytest.raises(sd.ContractError):
        sd.verify(rows, [7, 3])
    assert sd.greedy_next([0.5, 0.9, 0.9, 0.2]) == 1  # ties toward the lowest id


def test_no_cpu_fallback_without_gpu(sd):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(sd.SpecdecError) as e:
        sd.Model.init(sd.ModelConfig())
    assert "no CUDA device" in str(e.value) or "sm_100a" in str(e.value)


def test_table1_scripted_trace_step_records(sd):
    """acceptance.cpp:110-188 (the paper's Table 1): predictions (5,2) with
    acceptances (4,1), then (2,5) with (2,6) -> input pads (0,3),(3,0) and KV
    pads (0,3),(4,0) in the step records."""
    rows = np.array([[0, 0, 5, 4, 0, 0], [0, 1, 2, 1, 0, 0], [1, 0, 2, 2, 0, 0], [1, 1, 5, 6, 0, 0]])
    st = sd.step_records(rows)
    assert [x["input_padding"] for x in st[0]["samples"]] == [0, 3]
    assert [x["input_padding"] for x in st[1]["samples"]] == [3, 0]
    assert [x["kv_padding"] for x in st[0]["samples"]] == [0, 3]
    assert [x["kv_padding"] for x in st[1]["samples"]] == [4, 0]


def test_nccl_bootstrap_id_without_gpu(sd):
    """sd_nccl_unique_id (libnccl.so.2 opened on first use): the 128-byte
    bootstrap id a C++ host ships from rank 0 to the other ranks."""
    a, b = sd.nccl_unique_id(), sd.nccl_unique_id()
    assert len(a) == 128 and any(a) and a != b
