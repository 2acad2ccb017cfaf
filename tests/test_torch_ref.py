"""Pin tests/torch_ref.py (the float64 reference the full-shape bf16 parity
tests use on the GPU) to the C oracle, which is itself pinned to the compiled
reference (tests/test_oracle.py): prefill and a ragged verify step on the
oracle's arena give the same logits as the whole-sequence torch forward to
1e-5 of the logit range, and the same greedy tokens."""
import numpy as np
import pytest

import pyoracle as P
from torch_ref import TorchRef, unflatten

CFGS = [P.DEFAULT_CONFIG,
        dict(num_layers=2, num_heads=4, head_dim=16, vocab_size=300, max_positions=160, init_seed=0x70C4),
        dict(num_layers=1, num_heads=2, head_dim=32, vocab_size=200, max_positions=300, init_seed=0x70C5)]


@pytest.mark.parametrize("cfg", CFGS, ids=["c1", "h64", "hd32"])
def test_torch_reference_matches_the_oracle(oracle, cfg):
    rng = np.random.default_rng(cfg["init_seed"] & 0xFFFF)
    V, B = cfg["vocab_size"], 3
    h = cfg["num_heads"] * cfg["head_dim"]
    mo = oracle.model_init(cfg)
    ref = TorchRef(cfg, unflatten(cfg, oracle.weights(mo).copy()))
    prompts = [[0] + rng.integers(3, V, size=int(rng.integers(5, 60))).tolist() for _ in range(B)]
    drafts = [rng.integers(3, V, size=1 + s % 4).tolist() for s in range(B)]
    co = oracle.cache_new(0, cfg["num_layers"], B, cfg["max_positions"], h)
    slots = [(s, i) for s in range(B) for i in range(len(prompts[s]))]
    lo, amo = oracle.forward(mo, co, prompts, slots, V)
    for s in range(B):
        oracle.commit(co, s, len(prompts[s]))
    per = [[int(amo[sum(len(p) for p in prompts[: s + 1]) - 1])] + drafts[s] for s in range(B)]
    slots2 = [(s, len(prompts[s]) + o) for s in range(B) for o in range(len(per[s]))]
    lo2, amo2 = oracle.forward(mo, co, per, slots2, V)
    oracle.cache_free(co)
    oracle.model_free(mo)
    ours, ours2 = [], []
    for s in range(B):
        seq = prompts[s] + per[s]
        lg = ref.logits(seq)
        ours.append(lg[: len(prompts[s])])
        ours2.append(lg[len(prompts[s]):])
    ours, ours2 = np.concatenate(ours), np.concatenate(ours2)
    for a, b, am in ((ours, lo, amo), (ours2, lo2, amo2)):
        scale = np.abs(b).max()
        assert np.abs(a - b).max() <= 1e-5 * scale, np.abs(a - b).max() / scale
        assert (a.argmax(1) == am).mean() >= 0.99  # top-1 ties within 1e-5 are possible, not expected
