"""ctypes binding of ``libamusd.so`` (the C-ABI declared in include/amusd.h).

There is no CPU fallback: if the CUDA library is missing this module raises
at import of any device object, loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import (
    InvalidInputError,
    InvalidRollbackError,
    ProtocolViolationError,
    SpecDecError,
)

LIB_PATH = Path(__file__).resolve().parent / "libamusd.so"
KMAX = 16
MAX_LAYERS = 128

F32, BF16 = 0, 1
ENGINE_AR, ENGINE_SYNC, ENGINE_ASYNC, ENGINE_ASYNC_DRAFT, ENGINE_ASYNC_VERIFY = range(5)
COIN_NONE, COIN_SELF, COIN_CANON = range(3)


class TfConfig(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("vocab", "d_model", "n_layers", "n_heads", "n_kv_heads", "head_dim",
                                         "ffn", "max_seq", "dtype", "eos_token", "exclude_eos")] + [
        ("norm_eps", C.c_float), ("use_tensor_cores", C.c_int)]


class TfWeights(C.Structure):
    _fields_ = [("embed", C.c_void_p), ("lm_head", C.c_void_p), ("final_norm", C.c_void_p),
                ("rope_cos", C.c_void_p), ("rope_sin", C.c_void_p)] + [
        (n, C.c_void_p * MAX_LAYERS) for n in ("attn_norm", "wqkv", "wo", "mlp_norm", "wgate", "wup", "wdown")]


PATH_PERSISTENT, PATH_KERNELS, PATH_SIMT, PATH_DECODE, PATH_CLUSTER = 0, 1, 2, 3, 4  # amusd_model_set_path


class SessionDesc(C.Structure):
    _fields_ = [("prompt_len", C.c_int), ("max_new_tokens", C.c_int), ("draft_window_k", C.c_int),
                ("max_draft_lead", C.c_int), ("max_window", C.c_int), ("coin_mode", C.c_int),
                ("rho", C.c_double), ("coin_seed", C.c_uint64), ("canon", C.c_void_p), ("canon_len", C.c_int),
                ("trace_cap", C.c_int), ("jitter_ns", C.c_int), ("jitter_seed", C.c_uint64)]


class RunInfo(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("p_v", "p_d", "complete", "error", "verify_steps", "rollbacks",
                                         "drafted", "acks", "n_draft_events", "n_verify_events",
                                         "draft_iters", "verify_iters", "draft_cuts")]


class TpShard(C.Structure):  # amusd_tp_shard
    _fields_ = [(n, C.c_int) for n in ("tp_rank", "tp_size", "n_heads_full", "n_kv_heads_full", "ffn_full",
                                         "vocab_offset", "vocab_total")]


class TpPeer(C.Structure):  # amusd_tp_peer
    _fields_ = [("ws", C.c_void_p), ("tile_cnt", C.c_void_p), ("best", C.c_void_p), ("sched", C.c_void_p),
                ("lm_items", C.c_int), ("pad", C.c_int)]


class TraceEvent(C.Structure):
    _fields_ = [("t_ns", C.c_int64), ("busy_ns", C.c_int64), ("kind", C.c_int32), ("pos_lo", C.c_int32),
                ("pos_hi", C.c_int32), ("draft_accepted", C.c_int32)]


# (name, restype, argtypes) -- every entry point of include/amusd.h
_P, _I, _SZ, _VP = C.POINTER, C.c_int, C.c_size_t, C.c_void_p
SIGNATURES = [
    ("amusd_abi_version", _I, []),
    ("amusd_last_error", C.c_char_p, []),
    ("amusd_tf_state_bytes", _SZ, [_P(TfConfig)]),
    ("amusd_tf_create", _I, [_P(_VP), _P(TfConfig), _P(TfWeights), _VP, _SZ]),
    ("amusd_hash_state_bytes", _SZ, [_I]),
    ("amusd_hash_create", _I, [_P(_VP), C.c_uint64, _I, _I, _I, C.c_double, _I, _VP, _SZ]),
    ("amusd_scripted_state_bytes", _SZ, [_I, _I]),
    ("amusd_scripted_create", _I, [_P(_VP), _P(C.c_int32), _I, _I, _I, _I, _I, _VP, _SZ, _VP]),
    ("amusd_model_destroy", _I, [_VP]),
    ("amusd_tf_shard_state_bytes", _SZ, [_P(TfConfig), _P(TpShard)]),
    ("amusd_tf_create_shard", _I, [_P(_VP), _P(TfConfig), _P(TpShard), _P(TfWeights), _VP, _SZ]),
    ("amusd_tp_export", _I, [_VP, _P(TpPeer)]),
    ("amusd_tp_connect", _I, [_VP, _P(TpPeer), _I]),
    ("amusd_model_set_max_grid", _I, [_VP, _I]),
    ("amusd_peer_enable", _I, [_I, _I]),
    ("amusd_prefill_bytes", _SZ, [_VP, _I]),
    ("amusd_decode_bytes", _SZ, [_VP]),
    ("amusd_cluster_bytes", _SZ, [_VP]),
    ("amusd_model_set_cluster", _I, [_VP, _VP, _SZ]),
    ("amusd_model_set_decode", _I, [_VP, _VP, _SZ]),
    ("amusd_model_set_prefill", _I, [_VP, _VP, _SZ, _I]),
    ("amusd_session_tp_inbox", _I, [_VP, _P(_VP)]),
    ("amusd_session_set_tp", _I, [_VP, _I, _P(_VP), _I]),
    ("amusd_model_set_path", _I, [_VP, _I]),
    ("amusd_model_set_grid", _I, [_VP, _I]),
    ("amusd_model_release_row_major", _I, [_VP]),
    ("amusd_model_set_timeline", _I, [_VP, _VP, _SZ]),
    ("amusd_init_state", _I, [_VP, _P(C.c_int32), _I, _VP]),
    ("amusd_next_token", _I, [_VP, _P(C.c_int32), _VP]),
    ("amusd_advance", _I, [_VP, _P(C.c_int32), _I, _VP]),
    ("amusd_rollback", _I, [_VP, _I, _VP]),
    ("amusd_verify_tokens", _I, [_VP, _P(C.c_int32), _I, _P(C.c_int32), _VP]),
    ("amusd_prefix_length", _I, [_VP, _P(_I)]),
    ("amusd_last_logits", _I, [_VP, _P(C.c_float), _I, _VP]),
    ("amusd_mailbox_capacity", _I, [_P(SessionDesc)]),
    ("amusd_mailbox_bytes", _SZ, [_I]),
    ("amusd_session_bytes", _SZ, [_P(SessionDesc)]),
    ("amusd_session_create", _I, [_P(_VP), _VP, _VP, _P(SessionDesc), _VP, _SZ, _VP, _VP]),
    ("amusd_session_destroy", _I, [_VP]),
    ("amusd_session_reset", _I, [_VP, _P(C.c_int32), _I, _VP]),
    ("amusd_session_launch", _I, [_VP, _I, _VP, _VP]),
    ("amusd_session_build", _I, [_VP, _I]),
    ("amusd_session_info", _I, [_VP, _P(RunInfo), _P(C.c_int32), _I, _VP]),
    ("amusd_session_trace", _I, [_VP, _I, _P(TraceEvent), _I, _P(_I), _VP]),
    ("amusd_time_forward", _I, [_VP, _I, _I, _I, _I, _P(C.c_float), _VP]),
    ("amusd_session_kernels_per_step", _I, [_VP, _I, _P(_I), _P(_I)]),
    ("amusd_fill_uniform", _I, [_VP, _I, _SZ, C.c_uint64, C.c_float, _VP]),
    ("amusd_ipc_export", _I, [_VP, _P(C.c_uint8), _P(_SZ)]),
    ("amusd_ipc_import", _I, [_P(C.c_uint8), _SZ, _P(_VP), _P(_VP)]),
    ("amusd_ipc_close", _I, [_VP]),
    ("amusd_device_clock", _I, [_P(C.c_int64), _VP, _VP]),
]

_lib = None


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the CUDA library; raise loudly if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise SpecDecError(
            f"CUDA extension {p} is missing: build it with `python -m paper_2410_17375_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.amusd_abi_version() != 1:
        raise SpecDecError("libamusd ABI version mismatch")
    _lib = lib
    return lib


_STATUS = {
    1: InvalidInputError,
    2: InvalidRollbackError,
    3: ProtocolViolationError,
    4: SpecDecError,
    5: SpecDecError,
}


def check(status: int) -> None:
    """Map an amusd_status onto the reference exception hierarchy (errors.py:4-29)."""
    if status == 0:
        return
    msg = load().amusd_last_error().decode(errors="replace")
    raise _STATUS.get(status, SpecDecError)(msg)


def int_array(values):
    arr = (C.c_int32 * max(1, len(values)))(*values)
    return arr
