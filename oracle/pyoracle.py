"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the two CPU checkers.

* ``Oracle``    -> oracle/_build/libspecdec_oracle.so  (our plain-C restatement)
* ``Reference`` -> oracle/_ref/libspecdec_ref.so       (the unmodified reference
  library compiled in place, driven through oracle/ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module, and only as the checker or the timed CPU
baseline -- never as part of the product path.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libspecdec_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspecdec_ref.so")

I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")

# tokenizer.hpp:16-28 (host-only text mapping, out of the hot path)
BOS, EOS, PAD, BYTE_OFFSET = 0, 1, 2, 3

# acceptance.cpp:26-43
CORPUS = [
    "the quick brown fox jumps over the lazy dog",
    "pack my box with five dozen liquor jugs",
    "how vexingly quick daft zebras jump",
    "sphinx of black quartz judge my vow",
    "the five boxing wizards jump quickly",
    "grumpy wizards make toxic brew for the evil queen",
    "jackdaws love my big sphinx of quartz",
    "two driven jocks help fax my big quiz",
    "quick zephyrs blow vexing daft jim",
    "five quacking zephyrs jolt my wax bed",
    "crazy fredrick bought many very exquisite opal jewels",
    "we promptly judged antique ivory buckles for the next prize",
    "a mad boxer shot a quick gloved jab",
    "jinxed wizards pluck ivy from the big quilt",
    "amazingly few discotheques provide jukeboxes",
    "puzzled women bequeath jerks very exotic gifts",
]


def tokenize_prompt(text: str) -> list[int]:
    """engine.cpp:136-145: BOS + byte tokens."""
    return [BOS] + [b + BYTE_OFFSET for b in text.encode()]


def build(force: bool = False) -> None:
    """Compile oracle/ (and oracle/_ref when the reference sources exist)."""
    if force or not os.path.exists(ORACLE_SO) or (
        os.path.isdir("/root/reference/proj") and not os.path.exists(REF_SO)
    ):
        subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


class SpecdecError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class ModelConfigT(C.Structure):
    _fields_ = [
        ("num_layers", C.c_int32),
        ("num_heads", C.c_int32),
        ("head_dim", C.c_int32),
        ("vocab_size", C.c_int32),
        ("max_positions", C.c_int32),
        ("init_seed", C.c_uint64),
    ]


class EngineConfigT(C.Structure):
    _fields_ = [
        ("mode", C.c_int32),
        ("predictor", C.c_int32),
        ("k", C.c_int32),
        ("match_len", C.c_int32),
        ("copy_len", C.c_int32),
        ("batch_size", C.c_int32),
        ("max_new_tokens", C.c_int32),
        ("stop_on_eos", C.c_int32),
        ("seed", C.c_uint64),
        ("synthetic_accuracy", C.c_double),
    ]


def dims_of(cfg: dict) -> np.ndarray:
    return np.array(
        [cfg["num_layers"], cfg["num_heads"], cfg["head_dim"], cfg["vocab_size"], cfg["max_positions"]],
        dtype=np.int32,
    )


DEFAULT_CONFIG = dict(num_layers=2, num_heads=2, head_dim=16, vocab_size=259, max_positions=512,
                      init_seed=0xD5EED)  # model.hpp:14-20


class _Lib:
    prefix = ""

    def _check(self, rc: int) -> None:
        if rc != 0:
            raise SpecdecError(rc, getattr(self.lib, self.prefix + "last_error")().decode())


class Oracle(_Lib):
    """Our C restatement (oracle/specdec_oracle.c)."""

    prefix = "so_"

    def __init__(self, path: str = ORACLE_SO):
        L = C.CDLL(path)
        L.so_last_error.restype = C.c_char_p
        L.so_model_init.argtypes = [C.POINTER(ModelConfigT), C.POINTER(C.c_void_p)]
        L.so_model_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.so_model_save.argtypes = [C.c_void_p, C.c_char_p]
        L.so_model_free.argtypes = [C.c_void_p]
        L.so_model_checksum.argtypes = [C.c_void_p]
        L.so_model_checksum.restype = C.c_uint64
        L.so_model_weights.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
        L.so_model_weights.restype = C.POINTER(C.c_float)
        L.so_cache_new.argtypes = [C.c_int] * 5 + [C.POINTER(C.c_void_p)]
        L.so_cache_free.argtypes = [C.c_void_p]
        for fn in ("so_cache_committed", "so_cache_logical", "so_cache_start_offset"):
            getattr(L, fn).argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int32)]
        L.so_cache_commit.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.so_cache_commit_padded.argtypes = [C.c_void_p, I32P, I32P, C.c_int]
        L.so_cache_commit_prefill.argtypes = [C.c_void_p, I32P, I32P, C.c_int]
        L.so_cache_mark_hole.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.so_cache_write_kv.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, F32P, F32P]
        L.so_ledger_useful.argtypes = [C.c_void_p]
        L.so_ledger_useful.restype = C.c_int64
        L.so_ledger_padding.argtypes = [C.c_void_p]
        L.so_ledger_padding.restype = C.c_int64
        L.so_forward.argtypes = [C.c_void_p, C.c_void_p, I32P, I32P, C.c_int, I32P, I32P, C.c_void_p, C.c_void_p]
        L.so_forward_planned.argtypes = [C.c_void_p, C.c_void_p, I32P, C.c_int, I32P, I32P, I32P, I32P,
                                         C.c_void_p, C.c_void_p]
        L.so_restore_indices.argtypes = [I32P, C.c_int, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.so_verify.argtypes = [F32P, C.c_int, C.c_int, I32P, C.c_int, I32P, C.POINTER(C.c_int32)]
        L.so_retrieval_predict.argtypes = [I32P, C.c_int, C.c_int, C.c_int, I32P, C.POINTER(C.c_int32)]
        L.so_mix_seed.argtypes = [C.c_uint64] * 3
        L.so_mix_seed.restype = C.c_uint64
        L.so_fnv1a.argtypes = [C.c_void_p, C.c_int64]
        L.so_fnv1a.restype = C.c_uint64
        L.so_decode.argtypes = [C.POINTER(EngineConfigT), C.c_void_p, C.c_void_p, I32P, I32P, I32P, I32P,
                                I32P, C.c_int64, C.POINTER(C.c_int64), np.ctypeslib.ndpointer(np.int64)]
        self.lib = L

    # -- model
    def model_init(self, cfg: dict) -> int:
        c = ModelConfigT(**cfg)
        h = C.c_void_p()
        self._check(self.lib.so_model_init(C.byref(c), C.byref(h)))
        return h.value

    def model_load(self, path: str) -> int:
        h = C.c_void_p()
        self._check(self.lib.so_model_load(path.encode(), C.byref(h)))
        return h.value

    def model_save(self, m: int, path: str) -> None:
        self._check(self.lib.so_model_save(m, path.encode()))

    def model_free(self, m: int) -> None:
        self.lib.so_model_free(m)

    def checksum(self, m: int) -> int:
        return int(self.lib.so_model_checksum(m))

    def weights(self, m: int) -> np.ndarray:
        n = C.c_int64()
        p = self.lib.so_model_weights(m, C.byref(n))
        return np.ctypeslib.as_array(p, shape=(n.value,)).copy()

    # -- cache
    def cache_new(self, layout: int, layers: int, batch: int, cap: int, kv: int) -> int:
        h = C.c_void_p()
        self._check(self.lib.so_cache_new(layout, layers, batch, cap, kv, C.byref(h)))
        return h.value

    def cache_free(self, c: int) -> None:
        self.lib.so_cache_free(c)

    def committed(self, c: int, s: int) -> int:
        v = C.c_int32()
        self._check(self.lib.so_cache_committed(c, s, C.byref(v)))
        return v.value

    def commit(self, c: int, s: int, tau: int) -> None:
        self._check(self.lib.so_cache_commit(c, s, tau))

    def forward(self, m: int, c: int, per_sample: list[list[int]], slots: list[tuple[int, int]], vocab: int,
                want_logits: bool = True):
        tokens = np.array([t for seq in per_sample for t in seq], dtype=np.int32)
        counts = np.array([len(seq) for seq in per_sample], dtype=np.int32)
        ss = np.array([s for s, _ in slots], dtype=np.int32)
        sp = np.array([p for _, p in slots], dtype=np.int32)
        n = len(tokens)
        logits = np.zeros((n, vocab), dtype=np.float32) if want_logits else None
        am = np.zeros(n, dtype=np.int32)
        self._check(self.lib.so_forward(m, c, tokens, counts, len(per_sample), ss, sp,
                                        logits.ctypes.data if want_logits else None, am.ctypes.data))
        return logits, am

    def restore_indices(self, counts, flat):
        s, p = C.c_int32(), C.c_int32()
        self._check(self.lib.so_restore_indices(np.asarray(counts, dtype=np.int32), len(counts), flat,
                                                C.byref(s), C.byref(p)))
        return s.value, p.value

    def retrieval_predict(self, ctx, match_len, copy_len):
        ctx = np.asarray(ctx, dtype=np.int32)
        out = np.zeros(max(copy_len, 1), dtype=np.int32)
        n = C.c_int32()
        self._check(self.lib.so_retrieval_predict(ctx, len(ctx), match_len, copy_len, out, C.byref(n)))
        return out[: n.value].tolist()

    def decode(self, ecfg: dict, target: int, prompts: list[list[int]], draft: int | None = None):
        e = EngineConfigT(**ecfg)
        b = ecfg["batch_size"]
        flat = np.array([t for p in prompts for t in p], dtype=np.int32)
        lens = np.array([len(p) for p in prompts], dtype=np.int32)
        mx = max(ecfg["max_new_tokens"], 1)
        gen = np.zeros(b * mx, dtype=np.int32)
        cnt = np.zeros(b, dtype=np.int32)
        cap = b * (ecfg["max_new_tokens"] + 2) + 16
        rec = np.zeros(cap * 6, dtype=np.int32)
        nrec = C.c_int64()
        ledger = np.zeros(2, dtype=np.int64)
        self._check(self.lib.so_decode(C.byref(e), target, draft, flat, lens, gen, cnt, rec, cap,
                                       C.byref(nrec), ledger))
        tokens = [gen[s * mx: s * mx + cnt[s]].tolist() for s in range(b)]
        return tokens, rec[: nrec.value * 6].reshape(-1, 6), ledger


def fnv_rows(logits) -> np.ndarray:
    """FNV-1a of each fp32 row's bytes (fast path through the C oracle)."""
    lib = _fnv_lib()
    a = np.ascontiguousarray(logits, dtype=np.float32)
    a = a.reshape(a.shape[0], -1) if a.ndim > 1 else a.reshape(1, -1)
    return np.array([lib.so_fnv1a(r.ctypes.data, r.nbytes) for r in a], dtype=np.uint64)


_FNV = None


def _fnv_lib():
    global _FNV
    if _FNV is None:
        _FNV = Oracle().lib
    return _FNV


class Reference(_Lib):
    """The unmodified reference library (oracle/_ref/libspecdec_ref.so)."""

    prefix = "ref_"

    def __init__(self, path: str = REF_SO):
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_model_init.argtypes = [I32P, C.c_uint64, C.POINTER(C.c_void_p)]
        L.ref_model_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_model_save.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_model_free.argtypes = [C.c_void_p]
        L.ref_model_checksum.argtypes = [C.c_void_p]
        L.ref_model_checksum.restype = C.c_uint64
        L.ref_model_tensor_count.argtypes = [C.c_void_p]
        L.ref_model_tensor.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.POINTER(C.c_float)), C.POINTER(C.c_int64)]
        L.ref_cache_new.argtypes = [C.c_int] * 5 + [C.POINTER(C.c_void_p)]
        L.ref_cache_free.argtypes = [C.c_void_p]
        for fn in ("ref_cache_committed", "ref_cache_logical", "ref_cache_start_offset"):
            getattr(L, fn).argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int32)]
        L.ref_cache_commit.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_cache_commit_padded.argtypes = [C.c_void_p, I32P, I32P, C.c_int]
        L.ref_cache_commit_prefill.argtypes = [C.c_void_p, I32P, I32P, C.c_int]
        L.ref_cache_mark_hole.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_cache_write_kv.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, F32P, F32P]
        L.ref_ledger_useful.argtypes = [C.c_void_p]
        L.ref_ledger_useful.restype = C.c_int64
        L.ref_ledger_padding.argtypes = [C.c_void_p]
        L.ref_ledger_padding.restype = C.c_int64
        L.ref_forward.argtypes = [C.c_void_p, C.c_void_p, I32P, I32P, C.c_int, I32P, I32P, C.c_void_p]
        L.ref_forward_planned.argtypes = [C.c_void_p, C.c_void_p, I32P, C.c_int, I32P, I32P, I32P, I32P,
                                          C.c_void_p]
        L.ref_naive_forward.argtypes = [C.c_void_p, I32P, C.c_int, F32P]
        L.ref_restore_indices.argtypes = [I32P, C.c_int, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.ref_verify.argtypes = [F32P, C.c_int, C.c_int, I32P, C.c_int, I32P, C.POINTER(C.c_int32)]
        L.ref_retrieval_predict.argtypes = [I32P, C.c_int, C.c_int, C.c_int, I32P, C.POINTER(C.c_int32)]
        L.ref_mix_seed.argtypes = [C.c_uint64] * 3
        L.ref_mix_seed.restype = C.c_uint64
        L.ref_decode.argtypes = [C.c_int] * 8 + [C.c_uint64, C.c_double, C.c_void_p, C.c_void_p,
                                                 C.POINTER(C.c_char_p), C.c_char_p, C.c_int64,
                                                 C.POINTER(C.c_int64)]
        self.lib = L

    def model_init(self, cfg: dict) -> int:
        h = C.c_void_p()
        self._check(self.lib.ref_model_init(dims_of(cfg), cfg["init_seed"], C.byref(h)))
        return h.value

    def model_load(self, path: str) -> int:
        h = C.c_void_p()
        self._check(self.lib.ref_model_load(path.encode(), C.byref(h)))
        return h.value

    def model_save(self, m: int, path: str) -> None:
        self._check(self.lib.ref_model_save(m, path.encode()))

    def model_free(self, m: int) -> None:
        self.lib.ref_model_free(m)

    def checksum(self, m: int) -> int:
        return int(self.lib.ref_model_checksum(m))

    def weights(self, m: int) -> np.ndarray:
        out = []
        for i in range(self.lib.ref_model_tensor_count(m)):
            p, n = C.POINTER(C.c_float)(), C.c_int64()
            self._check(self.lib.ref_model_tensor(m, i, C.byref(p), C.byref(n)))
            out.append(np.ctypeslib.as_array(p, shape=(n.value,)).copy())
        return np.concatenate(out)

    def cache_new(self, layout, layers, batch, cap, kv) -> int:
        h = C.c_void_p()
        self._check(self.lib.ref_cache_new(layout, layers, batch, cap, kv, C.byref(h)))
        return h.value

    def cache_free(self, c: int) -> None:
        self.lib.ref_cache_free(c)

    def committed(self, c: int, s: int) -> int:
        v = C.c_int32()
        self._check(self.lib.ref_cache_committed(c, s, C.byref(v)))
        return v.value

    def commit(self, c: int, s: int, tau: int) -> None:
        self._check(self.lib.ref_cache_commit(c, s, tau))

    def write_kv(self, c, s, pos, layer, k, v) -> None:
        self._check(self.lib.ref_cache_write_kv(c, s, pos, layer, np.ascontiguousarray(k, np.float32),
                                                np.ascontiguousarray(v, np.float32)))

    def forward(self, m, c, per_sample, slots, vocab):
        tokens = np.array([t for seq in per_sample for t in seq], dtype=np.int32)
        counts = np.array([len(seq) for seq in per_sample], dtype=np.int32)
        ss = np.array([s for s, _ in slots], dtype=np.int32)
        sp = np.array([p for _, p in slots], dtype=np.int32)
        logits = np.zeros((len(tokens), vocab), dtype=np.float32)
        self._check(self.lib.ref_forward(m, c, tokens, counts, len(per_sample), ss, sp, logits.ctypes.data))
        return logits

    def forward_planned(self, m, c, tokens, sample, logical, slot, store, vocab):
        n = len(tokens)
        logits = np.zeros((n, vocab), dtype=np.float32)
        a = lambda x: np.asarray(x, dtype=np.int32)
        self._check(self.lib.ref_forward_planned(m, c, a(tokens), n, a(sample), a(logical), a(slot), a(store),
                                                 logits.ctypes.data))
        return logits

    def naive_forward(self, m, tokens, vocab):
        t = np.asarray(tokens, dtype=np.int32)
        logits = np.zeros((len(t), vocab), dtype=np.float32)
        self._check(self.lib.ref_naive_forward(m, t, len(t), logits))
        return logits

    def retrieval_predict(self, ctx, match_len, copy_len):
        ctx = np.asarray(ctx, dtype=np.int32)
        out = np.zeros(max(copy_len, 1), dtype=np.int32)
        n = C.c_int32()
        self._check(self.lib.ref_retrieval_predict(ctx, len(ctx), match_len, copy_len, out, C.byref(n)))
        return out[: n.value].tolist()

    def decode(self, ecfg: dict, target: int, prompts_text: list[str], draft: int | None = None) -> dict:
        arr = (C.c_char_p * len(prompts_text))(*[p.encode() for p in prompts_text])
        n = C.c_int64()
        self._check(self.lib.ref_decode(ecfg["mode"], ecfg["predictor"], ecfg["k"], ecfg["match_len"],
                                        ecfg["copy_len"], ecfg["batch_size"], ecfg["max_new_tokens"],
                                        ecfg["stop_on_eos"], ecfg["seed"], ecfg["synthetic_accuracy"], target,
                                        draft, arr, None, 0, C.byref(n)))
        buf = C.create_string_buffer(2 * n.value + 4096)  # timings vary in length
        self._check(self.lib.ref_decode(ecfg["mode"], ecfg["predictor"], ecfg["k"], ecfg["match_len"],
                                        ecfg["copy_len"], ecfg["batch_size"], ecfg["max_new_tokens"],
                                        ecfg["stop_on_eos"], ecfg["seed"], ecfg["synthetic_accuracy"], target,
                                        draft, arr, buf, 2 * n.value + 4096, C.byref(n)))
        return json.loads(buf.value.decode())


def engine_config(**kw) -> dict:
    """EngineConfig defaults (engine.hpp:21-34)."""
    base = dict(mode=2, predictor=0, k=4, match_len=2, copy_len=7, batch_size=1, max_new_tokens=64,
                stop_on_eos=1, seed=1, synthetic_accuracy=0.8)
    base.update(kw)
    return base


def step_records(rec: np.ndarray) -> list[dict]:
    """make_step_record (engine.cpp:78-105) rebuilt from flat oracle rows."""
    out = []
    for step in sorted(set(rec[:, 0].tolist())):
        rows = rec[rec[:, 0] == step]
        ks, taus = rows[:, 2].tolist(), rows[:, 3].tolist()
        kmax, tmax = max(ks), max(taus)
        out.append(dict(
            samples=[dict(sample=int(r[1]), k=int(r[2]), input_padding=kmax - int(r[2]), tau=int(r[3]),
                          kv_padding=tmax - int(r[3]), clipped=bool(r[4])) for r in rows],
            tau_max=tmax,
        ))
    return out
