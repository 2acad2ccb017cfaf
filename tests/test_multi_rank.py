"""Multi-rank host logic on CPU (gloo, world_size 2): samples sharded by
global id with no collective in the step, outputs all-gathered at the end,
must equal the single-process decode of the whole batch (batch-composition
invariance, test_engine.cpp:307-320).  The per-rank compute here is the C
oracle; on GPUs the same sharding drives libspecdec_b200 over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, strong, out_q):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as P
    from paper_2405_07542_b200 import sharding

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = P.Oracle()
    m = o.model_init(P.DEFAULT_CONFIG)
    ids = sharding.split_ids(6, world, rank) if strong else sharding.local_ids(3, rank)
    prompts = [P.tokenize_prompt(P.CORPUS[i]) for i in ids]
    e = P.engine_config(mode=2, predictor=1, copy_len=4, batch_size=len(ids), max_new_tokens=20, stop_on_eos=0)
    toks, _, _ = o.decode(e, m, prompts)
    allt = sharding.gather_outputs(toks, 20, dist)
    if rank == 0:
        out_q.put(allt)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("strong", [False, True])
def test_sharded_decode_equals_single_process(strong):
    import sys

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as P

    P.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, strong, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    o = P.Oracle()
    m = o.model_init(P.DEFAULT_CONFIG)
    prompts = [P.tokenize_prompt(P.CORPUS[i]) for i in range(6)]
    e = P.engine_config(mode=2, predictor=1, copy_len=4, batch_size=6, max_new_tokens=20, stop_on_eos=0)
    toks, _, _ = o.decode(e, m, prompts)
    assert gathered == toks


def test_split_by_prompt_length_is_contiguous_and_balanced():
    """contiguous blocks in global order, prompt-token totals
    within one prompt of the ideal share."""
    from paper_2405_07542_b200.sharding import split_ids_by_length

    rng = np.random.default_rng(5)
    for n, world in ((64, 8), (24, 4), (10, 3), (3, 4)):
        lens = rng.integers(3968, 4225, size=n).tolist() if n > 10 else rng.integers(1, 100, size=n).tolist()
        parts = [split_ids_by_length(lens, world, r) for r in range(world)]
        assert sum(parts, []) == list(range(n))  # a partition, in global order
        tot = sum(lens)
        for p in parts:
            if n >= world:
                assert p, "every rank gets a sample"
            assert abs(sum(lens[i] for i in p) - tot / world) <= max(lens) + 1
