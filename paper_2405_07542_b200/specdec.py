"""Python mirror of the reference `specdec` hot-path API over the C ABI.

Names, argument meaning and error behaviour follow the reference C++ library
(/root/reference/proj/include/specdec/*.hpp) so tests read like its own
tests.  Everything computes through libspecdec_b200.so (CUDA, sm_100a); there
is no CPU fallback -- importing works anywhere, but creating a Model without a
B200 raises SpecdecError (SD_INTERNAL).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = _DEFAULT_LIB = os.path.join(_PKG, "lib", "libspecdec_b200.so")

I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
I64P = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")

# tokenizer.hpp:16-28
BOS, EOS, PAD, BYTE_OFFSET, VOCAB_SIZE = 0, 1, 2, 3, 259

FP32_CHECK, BF16 = 0, 1
UNPAD, PADDED = 0, 1


# ---------------------------------------------------------------- errors
class SpecdecError(RuntimeError):
    """specdec::Error (common.hpp:13-15)."""

    code = 5


class ConfigError(SpecdecError):
    code = 1


class CapacityError(SpecdecError):
    code = 2


class ContractError(SpecdecError):
    code = 3


class IoError(SpecdecError):
    code = 4


_ERRORS = {1: ConfigError, 2: CapacityError, 3: ContractError, 4: IoError, 5: SpecdecError}


class _ModelConfigT(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_heads", C.c_int32), ("head_dim", C.c_int32),
                ("vocab_size", C.c_int32), ("max_positions", C.c_int32), ("init_seed", C.c_uint64)]


class _EngineConfigT(C.Structure):
    _fields_ = [("mode", C.c_int32), ("predictor", C.c_int32), ("k", C.c_int32), ("match_len", C.c_int32),
                ("copy_len", C.c_int32), ("batch_size", C.c_int32), ("max_new_tokens", C.c_int32),
                ("stop_on_eos", C.c_int32), ("seed", C.c_uint64), ("synthetic_accuracy", C.c_double),
                ("sample_id_base", C.c_int32)]


_lib = None


def lib() -> C.CDLL:
    """Load libspecdec_b200.so (fails loudly when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python __graft_entry__.py build` (no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, pp = C.c_void_p, C.POINTER(C.c_void_p)
    sig = {
        "sd_last_error": ([], C.c_char_p),
        "sd_kernel_launches": ([], C.c_int64),
        "sd_config_validate": ([C.POINTER(_ModelConfigT)], C.c_int),
        "sd_model_init": ([C.POINTER(_ModelConfigT), C.c_int, C.c_int, pp], C.c_int),
        "sd_model_load": ([C.c_char_p, C.c_int, C.c_int, pp], C.c_int),
        "sd_model_save": ([vp, C.c_char_p], C.c_int),
        "sd_model_checksum": ([vp, C.POINTER(C.c_uint64)], C.c_int),
        "sd_model_get_config": ([vp, C.POINTER(_ModelConfigT)], C.c_int),
        "sd_model_weight_bytes": ([vp], C.c_int64),
        "sd_model_get_tensor": ([vp, C.c_int, C.c_int, np.ctypeslib.ndpointer(np.float32), C.c_int64], C.c_int),
        "sd_model_destroy": ([vp], None),
        "sd_cache_create": ([vp, C.c_int, C.c_int, C.c_int, pp], C.c_int),
        "sd_cache_committed_len": ([vp, C.c_int, C.POINTER(C.c_int32)], C.c_int),
        "sd_cache_logical_len": ([vp, C.c_int, C.POINTER(C.c_int32)], C.c_int),
        "sd_cache_start_offset": ([vp, C.c_int, C.POINTER(C.c_int32)], C.c_int),
        "sd_cache_commit_accepted": ([vp, C.c_int, C.c_int], C.c_int),
        "sd_cache_commit_padded": ([vp, I32P, I32P, C.c_int], C.c_int),
        "sd_cache_commit_prefill": ([vp, I32P, I32P, C.c_int], C.c_int),
        "sd_cache_mark_hole": ([vp, C.c_int, C.c_int], C.c_int),
        "sd_cache_is_pad": ([vp, C.c_int, C.c_int, C.POINTER(C.c_int32)], C.c_int),
        "sd_cache_ledger": ([vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
        "sd_cache_gather_visible": ([vp, C.c_int, C.c_int, C.c_int, F32P, F32P, C.POINTER(C.c_int32)], C.c_int),
        "sd_cache_destroy": ([vp], None),
        "sd_cache_create_dims": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, pp], C.c_int),
        "sd_cache_write_kv": ([vp, C.c_int, C.c_int, C.c_int, F32P, F32P], C.c_int),
        "sd_ledger_create": ([C.c_int, pp], C.c_int),
        "sd_ledger_destroy": ([vp], None),
        "sd_cache_ledger_handle": ([vp, pp], C.c_int),
        "sd_ledger_note_useful": ([vp, C.c_int], C.c_int),
        "sd_ledger_note_padding": ([vp, C.c_int], C.c_int),
        "sd_ledger_begin_step": ([vp], C.c_int),
        "sd_ledger_note_tau": ([vp, C.c_int], C.c_int),
        "sd_ledger_end_step": ([vp], C.c_int),
        "sd_ledger_batch": ([vp, C.POINTER(C.c_int32)], C.c_int),
        "sd_ledger_totals": ([vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
        "sd_ledger_by_sample": ([vp, I64P, I64P], C.c_int),
        "sd_ledger_num_steps": ([vp, C.POINTER(C.c_int64)], C.c_int),
        "sd_ledger_step": ([vp, C.c_int64, I32P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                            C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
        "sd_ledger_dump_json": ([vp, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)], C.c_int),
        "sd_ledger_padding_ratio": ([vp, C.POINTER(C.c_double)], C.c_int),
        "sd_restore_indices": ([I32P, C.c_int, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32)], C.c_int),
        "sd_forward": ([vp, vp, I32P, I32P, C.c_int, I32P, I32P, vp, vp], C.c_int),
        "sd_forward_planned": ([vp, vp, I32P, C.c_int, I32P, I32P, I32P, I32P, vp, vp], C.c_int),
        "sd_verify_step": ([vp, vp, I32P, I32P, I32P, I32P, I32P, C.c_int, I32P, I32P, I32P, vp], C.c_int),
        "sd_decode": ([C.POINTER(_EngineConfigT), vp, vp, I32P, I32P, I32P, I32P, I32P, C.c_int64,
                       C.POINTER(C.c_int64), I64P, np.ctypeslib.ndpointer(np.float64)], C.c_int),
        "sd_profile_enable": ([C.c_int], C.c_int),
        "sd_profile_read": ([np.ctypeslib.ndpointer(np.float64), C.c_int], C.c_int),
        "sd_session_last_error": ([], C.c_char_p),
        "sd_session_create": ([vp, C.POINTER(_EngineConfigT), C.c_int, pp], C.c_int),
        "sd_session_create_draft": ([vp, vp, C.POINTER(_EngineConfigT), C.c_int, pp], C.c_int),
        "sd_session_prefill": ([vp, I32P, I32P], C.c_int),
        "sd_session_set_trajectory": ([vp, I32P, C.c_int], C.c_int),
        "sd_session_reset": ([vp], C.c_int),
        "sd_session_run": ([vp, C.c_int, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_float)], C.c_int),
        "sd_session_run_host": ([vp, C.POINTER(C.c_int32), C.POINTER(C.c_float), C.POINTER(C.c_int64),
                                 C.POINTER(C.c_int64)], C.c_int),
        "sd_session_outputs": ([vp, I32P, I32P, vp, vp, C.c_int], C.c_int),
        "sd_session_destroy": ([vp], None),
        "sd_session_draft_log": ([vp, I32P, C.c_int], C.c_int),
        "sd_verify_step_async": ([vp, vp, I32P, I32P, I32P, I32P, I32P, C.c_int, vp], C.c_int),
        "sd_verify_step_wait": ([vp, I32P, I32P, I32P], C.c_int),
        "sd_cache_set_stream": ([vp, vp], C.c_int),
        "sd_comm_last_error": ([], C.c_char_p),
        "sd_nccl_unique_id": ([np.ctypeslib.ndpointer(np.uint8)], C.c_int),
        "sd_comm_init": ([np.ctypeslib.ndpointer(np.uint8), C.c_int, C.c_int, C.c_int, pp], C.c_int),
        "sd_comm_size": ([vp, C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
        "sd_comm_destroy": ([vp], None),
        "sd_comm_allgather_i32": ([vp, I32P, C.c_int64, I32P], C.c_int),
        "sd_session_gather_outputs": ([vp, vp, I32P, I32P], C.c_int),
    }
    for name, (args, res) in sig.items():
        if LIB_PATH != _DEFAULT_LIB and not hasattr(L, name):
            continue  # an older build loaded for an A/B timing (tools/steptime.py --lib)
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc != 0:
        raise _ERRORS.get(rc, SpecdecError)(lib().sd_last_error().decode())


def kernel_launches() -> int:
    return int(lib().sd_kernel_launches())


def _i32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32).reshape(-1))


# ---------------------------------------------------------------- model
@dataclass
class ModelConfig:
    """model.hpp:14-25"""

    num_layers: int = 2
    num_heads: int = 2
    head_dim: int = 16
    vocab_size: int = VOCAB_SIZE
    max_positions: int = 512
    init_seed: int = 0xD5EED

    def hidden(self) -> int:
        return self.num_heads * self.head_dim

    def mlp_hidden(self) -> int:
        return 4 * self.hidden()

    def _c(self) -> _ModelConfigT:
        return _ModelConfigT(self.num_layers, self.num_heads, self.head_dim, self.vocab_size, self.max_positions,
                             self.init_seed)

    def validate(self) -> None:
        _check(lib().sd_config_validate(C.byref(self._c())))


@dataclass
class TokenSlot:
    """ragged.hpp:23-28"""

    original_batch_index: int = 0
    original_sequence_position: int = 0


@dataclass
class TokenPlan:
    """model.hpp:41-46"""

    sample: int = 0
    logical_pos: int = 0
    write_slot: int = 0
    store: bool = True


@dataclass
class RaggedBatch:
    """ragged.hpp:13-19"""

    concatenated_tokens: list = field(default_factory=list)
    token_nums_per_sample: list = field(default_factory=list)
    total_input_token_nums: int = 0

    def batch_size(self) -> int:
        return len(self.token_nums_per_sample)


def concatenate_inputs(per_sample) -> RaggedBatch:
    """Algorithm 1 (ragged.cpp:6-17)."""
    if len(per_sample) == 0:
        raise ContractError("contract: batch must have at least one sample")
    out = RaggedBatch()
    for seq in per_sample:
        out.concatenated_tokens.extend(int(t) for t in seq)
        out.token_nums_per_sample.append(len(seq))
        out.total_input_token_nums += len(seq)
    return out


def restore_indices(counts, flat_index: int) -> TokenSlot:
    """Algorithm 2 (ragged.cpp:19-36), through the C ABI."""
    s, p = C.c_int32(), C.c_int32()
    _check(lib().sd_restore_indices(_i32(counts), len(counts), int(flat_index), C.byref(s), C.byref(p)))
    return TokenSlot(s.value, p.value)


def attention_extent(slot: TokenSlot, cache_committed_len: int) -> int:
    """ragged.hpp:41-43"""
    return cache_committed_len + slot.original_sequence_position + 1


def greedy_next(row) -> int:
    """model.cpp:34-41: argmax, ties toward the lowest id (np.argmax keeps the first)."""
    row = np.asarray(row)
    if row.size == 0:
        raise ContractError("contract: argmax over an empty row")
    return int(np.argmax(row))


@dataclass
class VerifyResult:
    accepted: list
    tau: int


def verify(rows, drafts) -> VerifyResult:
    """engine.cpp:60-76 over host logits rows (the device path fuses this into k_accept)."""
    if len(rows) != len(drafts) + 1:
        raise ContractError("contract: verification needs one logits row per draft plus the bonus row")
    acc = []
    k = len(drafts)
    for j in range(k + 1):
        x = greedy_next(rows[j])
        acc.append(x)
        if j == k:
            return VerifyResult(acc, k + 1)
        if x != drafts[j]:
            return VerifyResult(acc, j + 1)
    raise AssertionError("unreachable")


class Model:
    """specdec::Model (model.hpp:54-103) resident on one B200."""

    def __init__(self, handle: int, precision: int):
        self._h = handle
        self.precision = precision

    @staticmethod
    def init(config: ModelConfig, device: int = 0, precision: int = FP32_CHECK) -> "Model":
        h = C.c_void_p()
        _check(lib().sd_model_init(C.byref(config._c()), device, precision, C.byref(h)))
        return Model(h.value, precision)

    @staticmethod
    def load(path: str, device: int = 0, precision: int = FP32_CHECK) -> "Model":
        h = C.c_void_p()
        _check(lib().sd_model_load(path.encode(), device, precision, C.byref(h)))
        return Model(h.value, precision)

    def save(self, path: str) -> None:
        _check(lib().sd_model_save(self._h, path.encode()))

    def close(self) -> None:
        if self._h:
            lib().sd_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def config(self) -> ModelConfig:
        c = _ModelConfigT()
        _check(lib().sd_model_get_config(self._h, C.byref(c)))
        return ModelConfig(c.num_layers, c.num_heads, c.head_dim, c.vocab_size, c.max_positions, c.init_seed)

    def weight_checksum(self) -> int:
        v = C.c_uint64()
        _check(lib().sd_model_checksum(self._h, C.byref(v)))
        return int(v.value)

    def weight_bytes(self) -> int:
        return int(lib().sd_model_weight_bytes(self._h))

    # weight access for independent reimplementations (model.hpp:81-87)
    MODEL_TENSORS = ["token_embedding", "position_embedding", "final_ln_gain", "final_ln_bias", "lm_head"]
    LAYER_TENSORS = ["ln1_gain", "ln1_bias", "wq", "bq", "wk", "bk", "wv", "bv", "wo", "bo", "ln2_gain", "ln2_bias",
                     "w_fc", "b_fc", "w_proj", "b_proj"]

    def tensor(self, name: str, layer: int = -1) -> np.ndarray:
        c = self.config
        h, m, V, P = c.hidden(), c.mlp_hidden(), c.vocab_size, c.max_positions
        if layer < 0:
            idx = self.MODEL_TENSORS.index(name)
            shape = [(V, h), (P, h), (h,), (h,), (V, h)][idx]
        else:
            idx = self.LAYER_TENSORS.index(name)
            shape = {"w_fc": (m, h), "b_fc": (m,), "w_proj": (h, m)}.get(name, (h, h) if name[0] == "w" else (h,))
        out = np.empty(int(np.prod(shape)), np.float32)
        _check(lib().sd_model_get_tensor(self._h, layer, idx, out, out.size))
        return out.reshape(shape)

    def tensors(self) -> dict:
        """Every weight as fp32: {"token_embedding": ..., "layers": [{...}, ...], ...}."""
        d = {n: self.tensor(n) for n in self.MODEL_TENSORS}
        d["layers"] = [{n: self.tensor(n, l) for n in self.LAYER_TENSORS} for l in range(self.config.num_layers)]
        return d

    def forward(self, batch: RaggedBatch, cache: "CacheArena", slots, want_logits: bool = True):
        """Model::forward (model.cpp:235-254). Returns (logits [T,V] or None, argmax [T])."""
        T = batch.total_input_token_nums
        V = self.config.vocab_size
        logits = np.zeros((T, V), dtype=np.float32) if want_logits else None
        am = np.zeros(max(T, 1), dtype=np.int32)
        ss = _i32([s.original_batch_index for s in slots])
        sp = _i32([s.original_sequence_position for s in slots])
        if len(slots) != T:
            raise ContractError("contract: slot list does not cover the batch")
        _check(lib().sd_forward(self._h, cache._h, _i32(batch.concatenated_tokens),
                                _i32(batch.token_nums_per_sample), batch.batch_size(), ss, sp,
                                logits.ctypes.data if want_logits else None, am.ctypes.data))
        return logits, am[:T]

    def forward_planned(self, tokens, plans, cache: "CacheArena", want_logits: bool = True):
        """Model::forward_planned (model.cpp:256-373)."""
        n = len(tokens)
        if len(plans) != n:
            raise ContractError("contract: token and plan lists differ in length")
        V = self.config.vocab_size
        logits = np.zeros((n, V), dtype=np.float32) if want_logits else None
        am = np.zeros(max(n, 1), dtype=np.int32)
        _check(lib().sd_forward_planned(self._h, cache._h, _i32(tokens), n, _i32([p.sample for p in plans]),
                                        _i32([p.logical_pos for p in plans]), _i32([p.write_slot for p in plans]),
                                        _i32([1 if p.store else 0 for p in plans]),
                                        logits.ctypes.data if want_logits else None, am.ctypes.data))
        return logits, am[:n]


# ---------------------------------------------------------------- caches
@dataclass
class LedgerStep:
    """kv_cache.hpp:13-18"""

    tau_list: list
    tau_max: int
    pad_writes: int
    useful_writes: int


class WriteLedger:
    """WriteLedger (kv_cache.hpp:21-57): a standalone ledger (WriteLedger(batch))
    or, from CacheArena.ledger(), the view of a cache's own ledger."""

    def __init__(self, batch_size: int = 0, _cache=None):
        h = C.c_void_p()
        if _cache is None:
            _check(lib().sd_ledger_create(batch_size, C.byref(h)))
        else:
            _check(lib().sd_cache_ledger_handle(_cache._h, C.byref(h)))
        self._h, self._cache = h.value, _cache  # a view keeps its cache alive

    def __del__(self):
        try:
            if self._h and self._cache is None:
                lib().sd_ledger_destroy(self._h)
        except Exception:
            pass

    def note_useful(self, sample: int) -> None:
        _check(lib().sd_ledger_note_useful(self._h, sample))

    def note_padding(self, sample: int) -> None:
        _check(lib().sd_ledger_note_padding(self._h, sample))

    def begin_step(self) -> None:
        _check(lib().sd_ledger_begin_step(self._h))

    def note_tau(self, tau: int) -> None:
        _check(lib().sd_ledger_note_tau(self._h, tau))

    def end_step(self) -> None:
        _check(lib().sd_ledger_end_step(self._h))

    def _totals(self):
        u, p = C.c_int64(), C.c_int64()
        _check(lib().sd_ledger_totals(self._h, C.byref(u), C.byref(p)))
        return u.value, p.value

    def useful_total(self) -> int:
        return self._totals()[0]

    def padding_total(self) -> int:
        return self._totals()[1]

    def total(self) -> int:
        return sum(self._totals())

    def _by_sample(self):
        b = C.c_int32()
        _check(lib().sd_ledger_batch(self._h, C.byref(b)))
        u = np.zeros(max(1, b.value), np.int64)
        p = np.zeros_like(u)
        _check(lib().sd_ledger_by_sample(self._h, u, p))
        return u[: b.value].tolist(), p[: b.value].tolist()

    def useful_by_sample(self) -> list:
        return self._by_sample()[0]

    def padding_by_sample(self) -> list:
        return self._by_sample()[1]

    def steps(self) -> list:
        n = C.c_int64()
        _check(lib().sd_ledger_num_steps(self._h, C.byref(n)))
        out = []
        for i in range(n.value):
            buf = np.zeros(1024, np.int32)
            nt, tm, pw, uw = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64()
            _check(lib().sd_ledger_step(self._h, i, buf, len(buf), C.byref(nt), C.byref(tm), C.byref(pw),
                                        C.byref(uw)))
            if nt.value > len(buf):
                buf = np.zeros(nt.value, np.int32)
                _check(lib().sd_ledger_step(self._h, i, buf, len(buf), C.byref(nt), C.byref(tm), C.byref(pw),
                                            C.byref(uw)))
            out.append(LedgerStep(buf[: nt.value].tolist(), tm.value, pw.value, uw.value))
        return out

    def dump_json(self) -> str:
        n = C.c_int64()
        _check(lib().sd_ledger_dump_json(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib().sd_ledger_dump_json(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()


def padding_ratio(ledger: WriteLedger) -> float:
    """padding_ratio (kv_cache.cpp:64-76)"""
    v = C.c_double()
    _check(lib().sd_ledger_padding_ratio(ledger._h, C.byref(v)))
    return v.value


class CacheArena:
    """CacheArena read contract (kv_cache.hpp:65-100) over the device arena.

    CacheArena(model, batch, capacity) builds the arena for a model;
    CacheArena.from_dims(num_layers, batch, capacity, kv_dim) is the
    reference's model-less constructor (kv_cache.cpp:78-88): rows can be stored
    with write_kv, and the first forward binds a model of that depth and width."""

    layout = UNPAD

    def __init__(self, model: Model, batch_size: int, capacity: int):
        h = C.c_void_p()
        _check(lib().sd_cache_create(model._h, batch_size, capacity, self.layout, C.byref(h)))
        self._h = h.value
        self.model = model
        self._batch = batch_size
        self._capacity = capacity

    @classmethod
    def from_dims(cls, num_layers: int, batch_size: int, capacity: int, kv_dim: int, precision: int = 0,
                  device: int = 0):
        self = cls.__new__(cls)
        h = C.c_void_p()
        _check(lib().sd_cache_create_dims(num_layers, batch_size, capacity, kv_dim, cls.layout, device, precision,
                                          C.byref(h)))
        self._h, self.model, self._batch, self._capacity = h.value, None, batch_size, capacity
        self._kv_dim = kv_dim
        return self

    def write_kv(self, sample: int, position: int, layer: int, k_vec, v_vec) -> None:
        """CacheArena::write_kv (kv_cache.cpp:128-138, 203-213)"""
        k = np.ascontiguousarray(k_vec, dtype=np.float32)
        v = np.ascontiguousarray(v_vec, dtype=np.float32)
        _check(lib().sd_cache_write_kv(self._h, sample, position, layer, k, v))

    def batch_size(self) -> int:
        return self._batch

    def capacity(self) -> int:
        return self._capacity

    def close(self) -> None:
        if self._h:
            lib().sd_cache_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def committed_len(self, sample: int) -> int:
        v = C.c_int32()
        _check(lib().sd_cache_committed_len(self._h, sample, C.byref(v)))
        return v.value

    def logical_len(self, sample: int) -> int:
        v = C.c_int32()
        _check(lib().sd_cache_logical_len(self._h, sample, C.byref(v)))
        return v.value

    def mark_hole(self, sample: int, position: int) -> None:
        _check(lib().sd_cache_mark_hole(self._h, sample, position))

    def ledger(self) -> WriteLedger:
        """The cache's own WriteLedger (kv_cache.hpp:95-96)."""
        return WriteLedger(_cache=self)

    def gather_visible(self, sample: int, upto: int, layer: int):
        hidden = self.model.config.hidden() if self.model is not None else self._kv_dim
        k = np.zeros((upto + 1) * hidden, dtype=np.float32)
        v = np.zeros_like(k)
        n = C.c_int32()
        _check(lib().sd_cache_gather_visible(self._h, sample, upto, layer, k, v, C.byref(n)))
        return k.reshape(-1, hidden)[: n.value], v.reshape(-1, hidden)[: n.value]

    def verify_step(self, last_tokens, draft_counts, drafts, budget_left, active, stop_on_eos: bool,
                    want_logits: bool = False):
        """One fused device verify step (sd_verify_step)."""
        B = self._batch
        counts = _i32(draft_counts)
        kmax = int(max([c for c, a in zip(counts, active) if a] or [0]))
        tau = np.zeros(B, dtype=np.int32)
        clipped = np.zeros(B, dtype=np.int32)
        acc = np.full(B * (kmax + 1), -1, dtype=np.int32)
        T = sum((1 + (kmax if self.layout == PADDED else c)) for c, a in zip(counts, active) if a)
        logits = np.zeros((max(T, 1), self.model.config.vocab_size), dtype=np.float32) if want_logits else None
        _check(lib().sd_verify_step(self.model._h, self._h, _i32(last_tokens), counts,
                                    _i32(drafts) if len(drafts) else np.zeros(1, np.int32), _i32(budget_left),
                                    _i32(active), int(stop_on_eos), tau, acc, clipped,
                                    logits.ctypes.data if want_logits else None))
        return tau, acc.reshape(B, kmax + 1), clipped.astype(bool), (logits[:T] if want_logits else None)


    def verify_step_async(self, last_tokens, draft_counts, drafts, budget_left, active, stop_on_eos: bool,
                          stream: int | None = None) -> None:
        """sd_verify_step_async: enqueue one verify step on `stream` (a raw
        cudaStream_t, e.g. torch.cuda.Stream().cuda_stream; None = the cache's
        stream) and return; collect it with verify_step_wait."""
        counts = _i32(draft_counts)
        self._inflight_kmax = int(max([c for c, a in zip(counts, active) if a] or [0]))
        _check(lib().sd_verify_step_async(self.model._h, self._h, _i32(last_tokens), counts,
                                          _i32(drafts) if len(drafts) else np.zeros(1, np.int32),
                                          _i32(budget_left), _i32(active), int(stop_on_eos), stream))

    def verify_step_wait(self):
        """sd_verify_step_wait -> (tau, accepted [B][k_max+1], clipped)"""
        B, kmax = self._batch, self._inflight_kmax
        tau = np.zeros(B, dtype=np.int32)
        clipped = np.zeros(B, dtype=np.int32)
        acc = np.full(B * (kmax + 1), -1, dtype=np.int32)
        _check(lib().sd_verify_step_wait(self._h, tau, acc, clipped))
        return tau, acc.reshape(B, kmax + 1), clipped.astype(bool)

    def set_stream(self, stream: int | None) -> None:
        """sd_cache_set_stream: order this cache's device work on `stream`."""
        _check(lib().sd_cache_set_stream(self._h, stream))


class UnpadArena(CacheArena):
    """kv_cache.hpp:105-128"""

    layout = UNPAD

    def start_offset(self, sample: int) -> int:
        v = C.c_int32()
        _check(lib().sd_cache_start_offset(self._h, sample, C.byref(v)))
        return v.value

    def commit_accepted(self, sample: int, tau: int) -> None:
        _check(lib().sd_cache_commit_accepted(self._h, sample, tau))


class PaddedGrid(CacheArena):
    """kv_cache.hpp:133-168"""

    layout = PADDED

    def is_pad(self, sample: int, row: int) -> bool:
        v = C.c_int32()
        _check(lib().sd_cache_is_pad(self._h, sample, row, C.byref(v)))
        return bool(v.value)

    def commit_prefill(self, samples, prompt_lens) -> None:
        _check(lib().sd_cache_commit_prefill(self._h, _i32(samples), _i32(prompt_lens), len(samples)))

    def commit_padded(self, samples, taus) -> None:
        _check(lib().sd_cache_commit_padded(self._h, _i32(samples), _i32(taus), len(samples)))


# ---------------------------------------------------------------- engine
# modes 3 / 4: the paper's 2x2 ablation, device-resident
# sessions only -- "unpad_input": unpadded input tokens over the padded KV
# grid; "unpad_kv": padded input (PAD spectators) over the unpadded KV arena
MODES = {"greedy": 0, "vanilla": 1, "ems": 2, "unpad_input": 3, "unpad_kv": 4}
PREDICTORS = {"draft": 0, "retrieval": 1, "synthetic": 2}


@dataclass
class EngineConfig:
    """engine.hpp:21-34"""

    mode: str = "ems"
    predictor: str = "draft"
    k: int = 4
    match_len: int = 2
    copy_len: int = 7
    batch_size: int = 1
    max_new_tokens: int = 64
    stop_on_eos: bool = True
    seed: int = 1
    synthetic_accuracy: float = 0.8
    sample_id_base: int = 0  # global id of local sample 0 (sharded runs, engine.cpp:182-185)

    def _c(self) -> _EngineConfigT:
        if self.mode not in MODES:
            raise ConfigError(f"config: unknown mode: {self.mode}")
        if self.predictor not in PREDICTORS:
            raise ConfigError(f"config: unknown predictor: {self.predictor}")
        return _EngineConfigT(MODES[self.mode], PREDICTORS[self.predictor], self.k, self.match_len, self.copy_len,
                              self.batch_size, self.max_new_tokens, int(self.stop_on_eos), self.seed,
                              self.synthetic_accuracy, self.sample_id_base)


@dataclass
class DecodeResult:
    generated_tokens: list
    steps: list
    useful_kv_writes: int
    padding_kv_writes: int
    prefill_seconds: float
    decode_seconds: float
    prompt_lens: list = None


def tokenize_prompt(text: str) -> list[int]:
    """engine.cpp:136-145: BOS + byte tokens."""
    return [BOS] + [b + BYTE_OFFSET for b in text.encode()]


def decode(config: EngineConfig, target: Model, prompts, draft: Model | None = None) -> DecodeResult:
    """decode_greedy / decode_speculative (engine.cpp:206-489) through sd_decode.
    prompts: list of token-id lists (BOS included) or of strings."""
    toks = [tokenize_prompt(p) if isinstance(p, str) else list(p) for p in prompts]
    if len(toks) != config.batch_size:
        raise ContractError("contract: prompt count does not match batch_size")
    b = config.batch_size
    mx = max(config.max_new_tokens, 1)
    gen = np.zeros(b * mx, dtype=np.int32)
    cnt = np.zeros(b, dtype=np.int32)
    cap = b * (config.max_new_tokens + 2) + 16
    rec = np.zeros(cap * 6, dtype=np.int32)
    nrec = C.c_int64()
    ledger = np.zeros(2, dtype=np.int64)
    timing = np.zeros(2, dtype=np.float64)
    flat = _i32([t for p in toks for t in p])
    lens = _i32([len(p) for p in toks])
    _check(lib().sd_decode(C.byref(config._c()), target._h, draft._h if draft else None, flat, lens, gen, cnt, rec,
                           cap, C.byref(nrec), ledger, timing))
    tokens = [gen[s * mx: s * mx + cnt[s]].tolist() for s in range(b)]
    rows = rec[: nrec.value * 6].reshape(-1, 6)
    return DecodeResult(tokens, step_records(rows), int(ledger[0]), int(ledger[1]), float(timing[0]),
                        float(timing[1]), [len(p) for p in toks])


def step_records(rows: np.ndarray) -> list[dict]:
    """make_step_record (engine.cpp:78-105) from flat {step, sample, k, tau, clipped} rows."""
    out = []
    for step in sorted(set(rows[:, 0].tolist())):
        r = rows[rows[:, 0] == step]
        ks, taus = r[:, 2].tolist(), r[:, 3].tolist()
        kmax, tmax = max(ks), max(taus)
        delta_bar = tmax - sum(taus) / len(taus)
        out.append(dict(
            samples=[dict(sample=int(x[1]), k=int(x[2]), input_padding=kmax - int(x[2]), tau=int(x[3]),
                          kv_padding=tmax - int(x[3]), clipped=bool(x[4])) for x in r],
            tau_max=tmax,
            delta_bar=delta_bar,
            r_bar=delta_bar / tmax,
        ))
    return out


def detokenize_text(tokens) -> str:
    """text_without_specials + tok::detokenize (engine.cpp:148-155): byte
    tokens to bytes, specials dropped; ids outside the byte vocabulary (large
    synthetic vocabularies) and invalid UTF-8 become U+FFFD, as the
    reference's JSON dump does with error_handler_t::replace."""
    out = bytearray()
    for t in tokens:
        if t in (BOS, EOS, PAD):
            continue
        out += bytes([t - BYTE_OFFSET]) if BYTE_OFFSET <= t < VOCAB_SIZE else "\ufffd".encode()
    return out.decode("utf-8", errors="replace")


def results_json(config: EngineConfig, result: DecodeResult) -> str:
    """The reference's report (results_json, engine.cpp:531-587): config,
    outputs (tokens + text), RunMetrics (engine.cpp:107-126, 255-287,
    486-527), per-step records and the per-step write ledger
    (WriteLedger::dump_json, kv_cache.cpp:53-62), same keys and meaning."""
    import json

    b = config.batch_size
    gen = [len(t) for t in result.generated_tokens]
    plens = result.prompt_lens or [0] * b
    steps = result.steps
    total_gen = sum(gen)
    if config.max_new_tokens == 0:  # engine.cpp:223-226, 314-317: default RunMetrics, no prefill
        decode_steps, avg_tau, avg_r, in_pad, kv_pad, real, pad_proc, ledger = 0, 0.0, 0.0, 0, 0, 0, 0, []
        steps = []
    elif config.mode == "greedy":
        decode_steps = max(gen) - 1 if gen else 0
        avg_tau, avg_r, in_pad, kv_pad = 1.0, 0.0, 0, 0
        real = sum(p + g - 1 for p, g in zip(plens, gen))
        pad_proc = 0
        ledger = []
    else:
        decode_steps = len(steps)
        taus = [x["tau"] for st in steps for x in st["samples"]]
        avg_tau = sum(taus) / len(taus) if taus else 0.0
        avg_r = sum(st["r_bar"] for st in steps) / len(steps) if steps else 0.0
        in_pad = sum(x["input_padding"] for st in steps for x in st["samples"])
        kv_pad = sum(x["kv_padding"] for st in steps for x in st["samples"])
        real = sum(plens) + sum(1 + x["k"] for st in steps for x in st["samples"])
        pad_proc = in_pad + kv_pad if config.mode == "vanilla" else 0
        ledger = [dict(tau_list=[x["tau"] for x in st["samples"]], tau_max=st["tau_max"],
                       pad_writes=sum(x["kv_padding"] for x in st["samples"]) if config.mode == "vanilla" else 0,
                       useful_writes=sum(1 + x["k"] for x in st["samples"])) for st in steps]
    wall = result.prefill_seconds + result.decode_seconds
    out = {
        "config": {"mode": config.mode, "predictor": config.predictor, "k": config.k, "match_len": config.match_len,
                   "copy_len": config.copy_len, "batch_size": b, "max_new_tokens": config.max_new_tokens,
                   "stop_on_eos": bool(config.stop_on_eos), "seed": config.seed,
                   "synthetic_accuracy": config.synthetic_accuracy},
        "outputs": [{"tokens": list(map(int, t)), "text": detokenize_text(t)} for t in result.generated_tokens],
        "metrics": {"decode_steps": decode_steps, "tokens_generated": gen, "total_tokens_generated": total_gen,
                    "avg_acceptance_length": avg_tau, "avg_padding_ratio": avg_r,
                    "total_input_padding": in_pad, "total_kv_padding": kv_pad,
                    "useful_kv_writes": result.useful_kv_writes, "padding_kv_writes": result.padding_kv_writes,
                    "real_tokens_processed": real, "pad_tokens_processed": pad_proc,
                    "total_tokens_processed": real + pad_proc,
                    "prefill_seconds": result.prefill_seconds, "decode_seconds": result.decode_seconds,
                    "tokens_per_second_decode": total_gen / result.decode_seconds if result.decode_seconds > 0 else 0.0,
                    "tokens_per_second_total": total_gen / wall if wall > 0 else 0.0},
        "steps": [{"samples": st["samples"], "tau_max": st["tau_max"], "delta_bar": st["delta_bar"],
                   "r_bar": st["r_bar"]} for st in steps],
        "ledger": ledger,
    }
    return json.dumps(out, indent=2, ensure_ascii=False)


# ---------------------------------------------------------------- sessions
PROFILE_KINDS = ["gemm_qkv", "gemm_o", "gemm_fc", "gemm_proj", "gemm_lm", "attention", "layernorm", "misc",
                 "gemm_stream"]


def profile_enable(on: bool) -> None:
    _check(lib().sd_profile_enable(int(on)))


def profile_read() -> dict:
    out = np.zeros(len(PROFILE_KINDS) * 3, dtype=np.float64)
    _check(lib().sd_profile_read(out, len(PROFILE_KINDS)))
    out = out.reshape(-1, 3)
    return {k: dict(launches=int(r[0]), ms=float(r[1]), bytes=float(r[2])) for k, r in zip(PROFILE_KINDS, out)}


def _scheck(rc: int) -> None:
    if rc != 0:
        raise _ERRORS.get(rc, SpecdecError)(lib().sd_session_last_error().decode())


def _ccheck(rc: int) -> None:
    if rc != 0:
        raise _ERRORS.get(rc, SpecdecError)(lib().sd_comm_last_error().decode())


def nccl_unique_id() -> bytes:
    """sd_nccl_unique_id: the 128-byte NCCL bootstrap id rank 0 ships to the others."""
    out = np.zeros(128, np.uint8)
    _ccheck(lib().sd_nccl_unique_id(out))
    return out.tobytes()


class Comm:
    """sd_comm: one rank's NCCL communicator for the end-of-run gather."""

    def __init__(self, uid: bytes, world: int, rank: int, device: int = 0):
        h = C.c_void_p()
        _ccheck(lib().sd_comm_init(np.frombuffer(uid, np.uint8).copy(), world, rank, device, C.byref(h)))
        self._h, self.world, self.rank = h.value, world, rank

    def allgather_i32(self, local) -> np.ndarray:
        x = np.ascontiguousarray(local, dtype=np.int32).ravel()
        out = np.zeros(x.size * self.world, np.int32)
        _ccheck(lib().sd_comm_allgather_i32(self._h, x, x.size, out))
        return out.reshape(self.world, -1)

    def close(self) -> None:
        if self._h:
            lib().sd_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Session:
    """A prefilled batch whose decode loop (engine.cpp:391-489) runs on the GPU."""

    def __init__(self, model: Model, config: EngineConfig, capacity: int, draft: Model | None = None):
        h = C.c_void_p()
        if config.predictor == "draft":
            if draft is None:
                raise ConfigError("draft predictor needs a draft model")
            _scheck(lib().sd_session_create_draft(model._h, draft._h, C.byref(config._c()), capacity, C.byref(h)))
        else:
            _scheck(lib().sd_session_create(model._h, C.byref(config._c()), capacity, C.byref(h)))
        self._h = h.value
        self.model = model
        self.draft = draft  # keeps the draft model alive with the session
        self.config = config

    def close(self):
        if self._h:
            lib().sd_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prefill(self, prompts) -> None:
        flat = _i32([t for p in prompts for t in p])
        _scheck(lib().sd_session_prefill(self._h, flat, _i32([len(p) for p in prompts])))

    def set_trajectory(self, traj: np.ndarray) -> None:
        traj = np.ascontiguousarray(traj, dtype=np.int32)
        _scheck(lib().sd_session_set_trajectory(self._h, traj.reshape(-1), traj.shape[1]))

    def reset(self) -> None:
        _scheck(lib().sd_session_reset(self._h))

    def run(self, use_graph: bool = True, graph_steps: int = 8):
        steps, ms = C.c_int32(), C.c_float()
        _scheck(lib().sd_session_run(self._h, int(use_graph), graph_steps, C.byref(steps), C.byref(ms)))
        return steps.value, ms.value

    def run_host(self):
        steps, ms, h2d, d2h = C.c_int32(), C.c_float(), C.c_int64(), C.c_int64()
        _scheck(lib().sd_session_run_host(self._h, C.byref(steps), C.byref(ms), C.byref(h2d), C.byref(d2h)))
        return steps.value, ms.value, h2d.value, d2h.value

    def outputs(self):
        B, mx = self.config.batch_size, self.config.max_new_tokens
        gen = np.zeros(B * mx, dtype=np.int32)
        cnt = np.zeros(B, dtype=np.int32)
        steps = mx + 2
        lk = np.zeros(steps * B, dtype=np.int32)
        lt = np.zeros(steps * B, dtype=np.int32)
        _scheck(lib().sd_session_outputs(self._h, gen, cnt, lk.ctypes.data, lt.ctypes.data, steps))
        tokens = [gen[s * mx: s * mx + min(cnt[s], mx)].tolist() for s in range(B)]
        return tokens, lk.reshape(steps, B), lt.reshape(steps, B)

    def gather_outputs(self, comm: "Comm"):
        """sd_session_gather_outputs: every rank's generated tokens, global sample order."""
        B, mx = self.config.batch_size, self.config.max_new_tokens
        gen = np.zeros(comm.world * B * mx, np.int32)
        cnt = np.zeros(comm.world * B, np.int32)
        _scheck(lib().sd_session_gather_outputs(self._h, comm._h, gen, cnt))
        return [gen[i * mx: i * mx + min(cnt[i], mx)].tolist() for i in range(comm.world * B)]

    def draft_log(self) -> np.ndarray:
        """[steps][B][kcap] drafts each verify step checked (valid below log_k)."""
        B = self.config.batch_size
        kcap = max(1, self.config.copy_len if self.config.predictor == "retrieval" else self.config.k)
        steps = self.config.max_new_tokens + 2
        out = np.zeros(steps * B * kcap, dtype=np.int32)
        _scheck(lib().sd_session_draft_log(self._h, out, steps))
        return out.reshape(steps, B, kcap)
