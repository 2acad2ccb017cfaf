"""Test infrastructure: a torch restatement of the reference forward
(proj/src/model.cpp:256-373) for the bf16 parity tests at full shapes, where
the scalar C oracle would take minutes.  It is pinned to the C oracle (and
through it to the compiled reference) at small shapes by
tests/test_torch_ref.py, then used on the GPU in float64 as the reference for
the tcgen05 path at the extents and widths the bench runs.

Semantics (unpadded arena; a padded grid's real tokens see exactly the same
keys because holes are skipped, kv_cache.cpp:221-235):
  h[t]   = tok_emb[id_t] + pos_emb[logical_pos_t]                 model.cpp:287-294
  per layer: x = LN1(h); q, k, v = W x + b                           :303-313
             s_j = (q . k_j) / sqrt(hd) over the sample's slots j <= t :320-341
             ctx = softmax(s) v; h += Wo ctx + bo                      :342-352
             h += W_proj gelu_tanh(W_fc LN2(h) + b_fc) + b_proj        :353-357
  logits = W_lm LN_f(h)  (no bias)                                   :361-367
LayerNorm: biased variance, eps 1e-5 (model.cpp:57-69).
"""
from __future__ import annotations

import math

import numpy as np

MODEL_TENSORS = ["token_embedding", "position_embedding", "final_ln_gain", "final_ln_bias", "lm_head"]
LAYER_TENSORS = ["ln1_gain", "ln1_bias", "wq", "bq", "wk", "bk", "wv", "bv", "wo", "bo", "ln2_gain", "ln2_bias",
                 "w_fc", "b_fc", "w_proj", "b_proj"]


def unflatten(cfg: dict, flat: np.ndarray) -> dict:
    """The declaration-order weight blob (model.cpp:166-175) as named tensors."""
    h = cfg["num_heads"] * cfg["head_dim"]
    m, V, P = 4 * h, cfg["vocab_size"], cfg["max_positions"]
    at = 0

    def take(*shape):
        nonlocal at
        n = int(np.prod(shape))
        t = flat[at: at + n].reshape(shape)
        at += n
        return t

    d = {"token_embedding": take(V, h), "position_embedding": take(P, h), "layers": []}
    for _ in range(cfg["num_layers"]):
        L = {}
        for name in LAYER_TENSORS:
            shape = {"w_fc": (m, h), "b_fc": (m,), "w_proj": (h, m)}.get(name, (h, h) if name[0] == "w" else (h,))
            L[name] = take(*shape)
        d["layers"].append(L)
    d["final_ln_gain"] = take(h)
    d["final_ln_bias"] = take(h)
    d["lm_head"] = take(V, h)
    assert at == flat.size
    return d


class TorchRef:
    """Reference forward over whole per-sample sequences.  `dtype` float64 on
    the GPU for the parity tests; float32 on the CPU when pinned to the
    oracle."""

    def __init__(self, cfg: dict, weights: dict, device="cpu", dtype=None):
        import torch

        self.torch = torch
        self.dtype = dtype or torch.float64
        self.cfg = cfg
        self.H, self.hd = cfg["num_heads"], cfg["head_dim"]
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device=device, dtype=self.dtype)
        self.w = {k: t(weights[k]) for k in MODEL_TENSORS}
        self.layers = [{k: t(L[k]) for k in LAYER_TENSORS} for L in weights["layers"]]
        self.device = device

    @staticmethod
    def _ln(x, g, b):
        mean = x.mean(-1, keepdim=True)
        var = ((x - mean) ** 2).mean(-1, keepdim=True)
        return (x - mean) / (var + 1e-5).sqrt() * g + b

    @staticmethod
    def _gelu(x):
        c = 0.7978845608028654
        return 0.5 * x * (1.0 + (c * (x + 0.044715 * x * x * x)).tanh())

    def logits(self, tokens, rows=None):
        """logits [len(rows), V] of one sample's sequence `tokens` (logical
        positions 0..n-1, causal), rows = which positions to return (all by
        default)."""
        torch = self.torch
        n = len(tokens)
        ids = torch.as_tensor(np.asarray(tokens, np.int64), device=self.device)
        h = self.w["token_embedding"][ids] + self.w["position_embedding"][:n]
        mask = torch.ones(n, n, dtype=torch.bool, device=self.device).tril()
        for L in self.layers:
            x = self._ln(h, L["ln1_gain"], L["ln1_bias"])
            q = (x @ L["wq"].T + L["bq"]).view(n, self.H, self.hd).transpose(0, 1)
            k = (x @ L["wk"].T + L["bk"]).view(n, self.H, self.hd).transpose(0, 1)
            v = (x @ L["wv"].T + L["bv"]).view(n, self.H, self.hd).transpose(0, 1)
            s = (q @ k.transpose(1, 2)) * (1.0 / math.sqrt(self.hd))
            s = s.masked_fill(~mask, float("-inf"))
            p = torch.softmax(s, dim=-1)
            ctx = (p @ v).transpose(0, 1).reshape(n, self.H * self.hd)
            h = h + ctx @ L["wo"].T + L["bo"]
            x2 = self._ln(h, L["ln2_gain"], L["ln2_bias"])
            h = h + self._gelu(x2 @ L["w_fc"].T + L["b_fc"]) @ L["w_proj"].T + L["b_proj"]
        if rows is not None:
            h = h[torch.as_tensor(np.asarray(rows, np.int64), device=self.device)]
        x = self._ln(h, self.w["final_ln_gain"], self.w["final_ln_bias"])
        return (x @ self.w["lm_head"].T).cpu().numpy()


def parity_stats(ours: np.ndarray, ref: np.ndarray) -> dict:
    """The stated bf16 tolerance metrics: max / mean |diff| over the reference
    logits' std, and argmax agreement (greedy_next, lowest id on ties)."""
    d = np.abs(ours.astype(np.float64) - ref)
    scale = float(ref.std())
    return {"max_abs_over_std": float(d.max() / scale), "mean_abs_over_std": float(d.mean() / scale),
            "argmax_agree": float(np.mean(ours.argmax(1) == ref.argmax(1))), "rows": int(ref.shape[0])}


C3_L2 = dict(num_layers=2, num_heads=40, head_dim=128, vocab_size=50272, max_positions=2048, init_seed=0xD5EED)


def c3_truncated_parity(sd, cfg=C3_L2, B=4, seed=1, greedy_tokens=0, lo=600, hi=660, cap=1024) -> dict:
    """bf16 verify-step logits of a layer-truncated C3 model (the library's
    public API: prefill + one ragged verify forward) against this float64
    reference on the fp32 weights of the same seed (an FP32_CHECK model of the
    library, itself bit-exact with the compiled reference).  Optionally also
    the greedy token agreement over `greedy_tokens` decoded tokens per sample
    (bf16 sd.decode vs float64 argmax decoding)."""
    import torch

    rng = np.random.default_rng(seed)
    V = cfg["vocab_size"]
    prompts = [[0] + rng.integers(3, V, size=int(rng.integers(lo, hi))).tolist() for _ in range(B)]
    drafts = [rng.integers(3, V, size=1 + (3 * s) % 8).tolist() for s in range(B)]
    m32 = sd.Model.init(sd.ModelConfig(**cfg), precision=sd.FP32_CHECK)
    ref = TorchRef(cfg, m32.tensors(), device="cuda", dtype=torch.float64)
    m32.close()
    m = sd.Model.init(sd.ModelConfig(**cfg), precision=sd.BF16)
    c = sd.UnpadArena(m, B, cap)
    slots = [sd.TokenSlot(s, i) for s in range(B) for i in range(len(prompts[s]))]
    _, am = m.forward(sd.concatenate_inputs(prompts), c, slots, want_logits=False)
    for s in range(B):
        c.commit_accepted(s, len(prompts[s]))
    ends = np.cumsum([len(p) for p in prompts]) - 1
    per = [[int(am[ends[s]])] + drafts[s] for s in range(B)]
    slots2 = [sd.TokenSlot(s, len(prompts[s]) + o) for s in range(B) for o in range(len(per[s]))]
    lg, am2 = m.forward(sd.concatenate_inputs(per), c, slots2)
    assert (am2 == lg.argmax(1)).all()
    rows = [ref.logits(prompts[s] + per[s], rows=range(len(prompts[s]), len(prompts[s]) + len(per[s])))
            for s in range(B)]
    c.close()
    out = parity_stats(lg, np.concatenate(rows))
    out["config"] = "h=%d shape truncated to L=%d, B=%d, %d-%d-token contexts, drafts 1-8" % (
        cfg["num_heads"] * cfg["head_dim"], cfg["num_layers"], B, lo, hi)
    if greedy_tokens:
        g = sd.decode(sd.EngineConfig(mode="greedy", batch_size=B, max_new_tokens=greedy_tokens, stop_on_eos=False),
                      m, prompts).generated_tokens
        same, prefix = 0, []
        for s in range(B):
            seq, ref_tok = list(prompts[s]), []
            for _ in range(greedy_tokens):
                ref_tok.append(int(ref.logits(seq, rows=[len(seq) - 1])[0].argmax()))
                seq.append(ref_tok[-1])
            same += sum(int(a == b) for a, b in zip(g[s], ref_tok))
            prefix.append(next((i for i, (a, b) in enumerate(zip(g[s], ref_tok)) if a != b), greedy_tokens))
        out["token_agree"] = same / (B * greedy_tokens)
        out["greedy_prefix_agree"] = float(np.mean(prefix)) / greedy_tokens
        out["greedy_tokens_per_sample"] = greedy_tokens
    m.close()
    torch.cuda.empty_cache()
    return out


def prefill_parity(sd, cfg=C3_L2, B=2, lo=600, hi=700, seed=3, every=9) -> dict:
    """Long-prompt prefill (engine.cpp:330-385) through the bf16 kernels in
    256-token chunks, on both layouts -- the unpadded arena and the vanilla
    padded grid with its left-pad holes (engine.cpp:335-357) -- against the
    float64 reference: every `every`-th prompt row's logits, and the argmax of
    every row."""
    import torch

    rng = np.random.default_rng(seed)
    V = cfg["vocab_size"]
    prompts = [[0] + rng.integers(3, V, size=int(rng.integers(lo, hi))).tolist() for _ in range(B)]
    m32 = sd.Model.init(sd.ModelConfig(**cfg), precision=sd.FP32_CHECK)
    ref = TorchRef(cfg, m32.tensors(), device="cuda", dtype=torch.float64)
    m32.close()
    want = [list(range(0, len(p), every)) + [len(p) - 1] for p in prompts]
    ref_rows = np.concatenate([ref.logits(p, rows=w) for p, w in zip(prompts, want)])
    ref_am = np.concatenate([ref.logits(p).argmax(1) for p in prompts])
    m = sd.Model.init(sd.ModelConfig(**cfg), precision=sd.BF16)
    out = {}
    for layout in ("unpad", "padded"):
        rows_needed = max(map(len, prompts))
        if layout == "unpad":
            c = sd.UnpadArena(m, B, rows_needed + 8)
            lg, am = m.forward(sd.concatenate_inputs(prompts), c,
                               [sd.TokenSlot(s, i) for s in range(B) for i in range(len(prompts[s]))])
        else:
            c = sd.PaddedGrid(m, B, rows_needed + 8)
            toks, plans = [], []
            for s, p in enumerate(prompts):
                holes = rows_needed - len(p)
                for r in range(holes):
                    c.mark_hole(s, r)
                toks += p
                plans += [sd.TokenPlan(sample=s, logical_pos=i, write_slot=holes + i, store=True) for i in range(len(p))]
            lg, am = m.forward_planned(toks, plans, c)
        c.close()
        offs = np.cumsum([0] + [len(p) for p in prompts[:-1]])
        pick = np.concatenate([o + np.asarray(w) for o, w in zip(offs, want)])
        st = parity_stats(lg[pick], ref_rows)
        st["argmax_agree_all_rows"] = float(np.mean(am == ref_am))
        st["rows_total"] = int(len(am))
        out[layout] = st
    m.close()
    torch.cuda.empty_cache()
    return out
