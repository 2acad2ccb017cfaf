"""The draft-model path with a draft that agrees with its target: a
layer-truncated copy of the target (its first `--draft-layers` layers with the
target's own embeddings, final LayerNorm and LM head, written as an SDCK
checkpoint and loaded in bf16) -- the LayerSkip / self-speculative setting.
Random-init OPT-125m drafts agree with an unrelated target almost never
(C4: tau ~ 1); this shows what the device draft loop gains when they do.

Prints, for the same prompts and 128 new tokens per sample: the EMS device
loop with the truncated draft (k = 4), the same loop with drafts that are
always wrong (synthetic accuracy 0: one token per verify step, the greedy
rate of the same machinery), and plain greedy decoding through sd_decode.

  python tools/selfdraft.py [--config c2|c3l4] [--batch 8] [--draft-layers 2]
"""
import argparse
import os
import struct
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_07542_b200 import specdec as sd  # noqa: E402
import bench  # noqa: E402


def truncated_checkpoint(cfg, n_layers, path):
    """SDCK v1 (model.cpp:143-221) of the target's first n_layers layers."""
    m32 = sd.Model.init(sd.ModelConfig(**cfg), precision=sd.FP32_CHECK)
    c = m32.config
    with open(path, "wb") as f:
        f.write(b"SDCK")
        f.write(struct.pack("<I", 1))
        f.write(struct.pack("<5i", n_layers, c.num_heads, c.head_dim, c.vocab_size, c.max_positions))
        f.write(struct.pack("<Q", c.init_seed))
        for name in ("token_embedding", "position_embedding"):
            f.write(m32.tensor(name).astype(np.float32).tobytes())
        for l in range(n_layers):
            for name in sd.Model.LAYER_TENSORS:
                f.write(m32.tensor(name, l).astype(np.float32).tobytes())
        for name in ("final_ln_gain", "final_ln_bias", "lm_head"):
            f.write(m32.tensor(name).astype(np.float32).tobytes())
    m32.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=["c2"])
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--draft-layers", type=int, default=2)
    ap.add_argument("--new", type=int, default=128)
    a = ap.parse_args()
    cfg = bench.C2
    B, k = a.batch, 4
    path = os.path.join(tempfile.gettempdir(), "selfdraft_%d.sdck" % a.draft_layers)
    truncated_checkpoint(cfg, a.draft_layers, path)
    m = sd.Model.init(sd.ModelConfig(**cfg), precision=sd.BF16)
    d = sd.Model.load(path, precision=sd.BF16)
    prompts = bench.prompts_for(range(B), cfg["vocab_size"], 512, 512)
    cap = 512 + a.new + k + 2
    out = {}

    def timed(sess, traj=None):
        sess.prefill(prompts)
        if traj is not None:
            sess.set_trajectory(traj)
        best, steps = 1e9, 0
        for _ in range(4):
            sess.reset()
            steps, ms = sess.run()
            best = min(best, ms)
        toks, lk, lt = sess.outputs()
        acc = sum(len(t) for t in toks) - B
        return {"ms": round(best, 3), "verify_steps": steps, "tokens_per_s": round(acc / (best / 1000.0), 1),
                "avg_tau": round(acc / max(1, sum(int((np.asarray(r) >= 0).sum()) for r in lk)), 3)}, toks

    e = sd.EngineConfig(mode="ems", predictor="draft", k=k, batch_size=B, max_new_tokens=a.new, stop_on_eos=False)
    s = sd.Session(m, e, cap, draft=d)
    out["ems_truncated_draft"], toks_d = timed(s)
    s.close()
    e = sd.EngineConfig(mode="ems", predictor="synthetic", k=k, batch_size=B, max_new_tokens=a.new,
                        stop_on_eos=False, seed=1, synthetic_accuracy=0.0)
    s = sd.Session(m, e, cap)
    g = sd.decode(sd.EngineConfig(mode="greedy", batch_size=B, max_new_tokens=a.new + k + 2, stop_on_eos=False), m,
                  prompts)
    out["ems_always_wrong_drafts"], _ = timed(s, np.array(g.generated_tokens, dtype=np.int32))
    s.close()
    out["lossless"] = all(list(t) == list(gt[: len(t)]) for t, gt in zip(toks_d, g.generated_tokens))
    out["speedup_vs_one_token_per_step"] = round(out["ems_truncated_draft"]["tokens_per_s"] /
                                                 out["ems_always_wrong_drafts"]["tokens_per_s"], 3)
    out["config"] = "C2 target (12 layers, B=%d, 512-id prompts, %d new tokens) with its first %d layers as the draft, k=%d" % (
        B, a.new, a.draft_layers, k)
    import json
    print(json.dumps(out))
    os.remove(path)


if __name__ == "__main__":
    main()
