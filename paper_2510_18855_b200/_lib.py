"""ctypes binding of ``libicepop_b200.so`` (declared in ``include/icepop.h``).

This is the only place Python touches the native library. There is no fallback:
if the shared object is missing or the device is not sm_100, every entry point
raises instead of silently computing on the CPU.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import NumericError

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("ICEPOP_B200_LIB", _HERE / "libicepop_b200.so"))

OK, EINVAL, ENUMERIC, ECUDA, EARCH = 0, 1, 2, 3, 4
ALGO_ICEPOP, ALGO_GRPO, ALGO_TIS = 0, 1, 2
W_DV, W_VD = 0, 1
NSTATS = 8
ABI_VERSION = 4
PROBS_SLAB = 64  # ICEPOP_PROBS_SLAB: vocab columns per tile_max entry


def tile_max_ld(vocab: int) -> int:
    """ICEPOP_TILE_MAX_LD: row length of tile_max (one float4 per 256-column K1 tile)."""
    return 4 * ((vocab + 255) // 256)
STAT_OBJECTIVE, STAT_N_POPPED, STAT_TOKENS, STAT_SUM_ENTROPY = 0, 1, 2, 3
STAT_SUM_ENTROPY_POPPED, STAT_SUM_LOGP, STAT_SUM_KL, STAT_ERRORS = 4, 5, 6, 7

_c_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_f64 = ctypes.c_double
_sz = ctypes.c_size_t


class Config(ctypes.Structure):
    _fields_ = [
        ("alpha", _f64),
        ("beta", _f64),
        ("clip_eps", _f64),
        ("tis_cap", _f64),
        ("temperature", _f64),
        ("kl_coeff", _f64),
        ("algo", _i32),
        ("_pad", _i32),
    ]


class Shape(ctypes.Structure):
    _fields_ = [
        ("n_tokens", _i64),
        ("token_offset", _i64),
        ("hidden", _i64),
        ("vocab", _i64),
        ("n_seqs", _i32),
        ("n_groups", _i32),
        ("weight_layout", _i32),
        ("_pad", _i32),
    ]


class Batch(ctypes.Structure):
    _fields_ = [
        ("tokens", _c_p),
        ("lp_train_old", _c_p),
        ("lp_infer_old", _c_p),
        ("cu_seqlens", _c_p),
        ("group_offsets", _c_p),
        ("advantages", _c_p),
        ("rewards", _c_p),
        ("calib", _c_p),
    ]


class FwdOut(ctypes.Structure):
    _fields_ = [
        ("lse", _c_p),
        ("lp_cur", _c_p),
        ("entropy", _c_p),
        ("kept", _c_p),
        ("calib", _c_p),
        ("surrogate", _c_p),
        ("coeff", _c_p),
        ("stats", _c_p),
        ("kl", _c_p),
        ("lse_ref", _c_p),
        ("kl_w", _c_p),
        ("probs", _c_p),
        ("tile_max", _c_p),
    ]


class Saved(ctypes.Structure):
    _fields_ = [
        ("tokens", _c_p),
        ("lse", _c_p),
        ("coeff", _c_p),
        ("lse_ref", _c_p),
        ("kl", _c_p),
        ("kl_w", _c_p),
        ("probs", _c_p),
        ("tile_max", _c_p),
        ("lp_cur", _c_p),
    ]


class F64Out(ctypes.Structure):
    _fields_ = [
        ("lse", _c_p),
        ("lp_cur", _c_p),
        ("entropy", _c_p),
        ("kl", _c_p),
        ("lse_ref", _c_p),
        ("kept", _c_p),
        ("calib", _c_p),
        ("surrogate", _c_p),
        ("coeff", _c_p),
        ("stats", _c_p),
    ]


class RsTarget(ctypes.Structure):
    _fields_ = [
        ("world", _i32),
        ("rank", _i32),
        ("shard_rows", _i64),
        ("slots", _c_p * 8),
    ]


_P = ctypes.POINTER
# name -> (restype, argtypes); every symbol include/icepop.h declares.
SIGNATURES: dict[str, tuple] = {
    "icepop_abi_version": (ctypes.c_int, []),
    "icepop_last_error": (ctypes.c_char_p, []),
    "icepop_device_check": (ctypes.c_int, [ctypes.c_int]),
    "icepop_group_advantages": (ctypes.c_int, [_c_p, _c_p, _i32, _i32, _c_p, _c_p]),
    "icepop_workspace_bytes": (ctypes.c_int, [_P(Shape), _i64, _i32, _P(_sz), _P(_sz)]),
    "icepop_fwd_bf16": (
        ctypes.c_int,
        [_P(Shape), _P(Config), _c_p, _c_p, _c_p, _P(Batch), _P(FwdOut), _c_p, _sz, _c_p],
    ),
    "icepop_fwd_epilogue_bf16": (
        ctypes.c_int,
        [_P(Shape), _P(Config), _P(Batch), _i32, _P(FwdOut), _c_p, _sz, _c_p],
    ),
    "icepop_fwd_onpolicy": (
        ctypes.c_int,
        [_P(Shape), _P(Config), _P(Batch), _c_p, _c_p, _P(FwdOut), _c_p, _sz, _c_p],
    ),
    "icepop_logprob_bf16": (
        ctypes.c_int,
        [_P(Shape), _f64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _sz, _c_p],
    ),
    "icepop_bwd_bf16": (
        ctypes.c_int,
        [_P(Shape), _P(Config), _c_p, _c_p, _c_p, _P(Saved), _f64, _c_p, _i32, _c_p, _i32, _c_p, _sz, _c_p],
    ),
    "icepop_bwd_bf16_rs": (
        ctypes.c_int,
        [_P(Shape), _P(Config), _c_p, _c_p, _c_p, _P(Saved), _f64, _c_p, _i32, _P(RsTarget), _c_p, _c_p, _sz, _c_p],
    ),
    "icepop_rs_fold": (ctypes.c_int, [_c_p, _i32, _i64, _c_p, _c_p]),
    "icepop_peer_alloc": (ctypes.c_int, [_sz, _P(_c_p)]),
    "icepop_peer_free": (ctypes.c_int, [_c_p]),
    "icepop_peer_export": (ctypes.c_int, [_c_p, _c_p]),
    "icepop_peer_import": (ctypes.c_int, [_c_p, _P(_c_p)]),
    "icepop_peer_close": (ctypes.c_int, [_c_p]),
    "icepop_dz_bf16": (ctypes.c_int, [_P(Shape), _f64, _c_p, _c_p, _c_p, _P(Saved), _f64, _c_p, _i64, _c_p]),
    "icepop_kl_bf16": (ctypes.c_int, [_P(Shape), _f64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "icepop_delta_gap_workspace_bytes": (ctypes.c_int, [_P(Shape), _i32, _P(_sz)]),
    "icepop_delta_gap_bf16": (ctypes.c_int, [_P(Shape), _f64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _sz,
                                             _c_p]),
    "icepop_delta_gap_f64": (ctypes.c_int, [_P(Shape), _f64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _sz,
                                            _c_p]),
    "icepop_sgd_update_f32": (ctypes.c_int, [_c_p, _c_p, _c_p, _c_p, _i64, _f64, _f64, _c_p, _c_p]),
    "icepop_sgd_update_f64": (ctypes.c_int, [_c_p, _c_p, _c_p, _c_p, _c_p, _i64, _f64, _f64, _c_p, _c_p]),
    "icepop_workspace_bytes_f64": (ctypes.c_int, [_P(Shape), _i32, _P(_sz)]),
    "icepop_fwd_f64": (
        ctypes.c_int,
        [_P(Shape), _P(Config), _c_p, _c_p, _c_p, _P(Batch), _P(F64Out), _c_p, _sz, _c_p],
    ),
    "icepop_bwd_f64": (
        ctypes.c_int,
        [_P(Shape), _P(Config), _c_p, _c_p, _c_p, _P(Batch), _P(F64Out), _f64, _c_p, _c_p, _i32, _c_p, _sz, _c_p],
    ),
    "icepop_finish": (ctypes.c_int, [_c_p, _c_p]),
    "icepop_gemm_bf16": (ctypes.c_int, [_c_p, _c_p, _c_p, _i64, _i64, _i64, _i32, _i32, _i32, _i32, _c_p]),
    "icepop_wave_barrier_abandons": (ctypes.c_int, [_P(_i64)]),
    "icepop_set_cta_group": (ctypes.c_int, [_i32]),
    "icepop_set_wide_tiles": (ctypes.c_int, [_i32]),
    "icepop_set_k1_wide": (ctypes.c_int, [_i32]),
    "icepop_set_skip_inactive": (ctypes.c_int, [_i32]),
    "icepop_set_k1_run": (ctypes.c_int, [_i32]),
}

_lib: ctypes.CDLL | None = None
_device_ok: set[int] = set()


def load() -> ctypes.CDLL:
    """Load the shared library (no device needed) and bind every declared symbol."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"libicepop_b200.so not found at {LIB_PATH}; build it with `make -C {_HERE.parent}` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.icepop_abi_version() != ABI_VERSION:
        raise RuntimeError("libicepop_b200.so ABI version mismatch")
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().icepop_last_error()
    return msg.decode() if msg else ""


def check(code: int) -> None:
    """Map a return code to the reference's exception types (include/icepop.h)."""
    if code == OK:
        return
    msg = last_error()
    if code == EINVAL:
        raise ValueError(msg)
    if code == ENUMERIC:
        raise NumericError(msg)
    raise RuntimeError(f"libicepop_b200 error {code}: {msg}")


def ensure_device(device_index: int) -> ctypes.CDLL:
    lib = load()
    if device_index not in _device_ok:
        check(lib.icepop_device_check(device_index))
        _device_ok.add(device_index)
    return lib


def wave_barrier_abandons(device_index: int = 0) -> int:
    """Long-K GEMM launches on this device whose wave barriers timed out (include/icepop.h)."""
    lib = ensure_device(device_index)
    n = _i64(0)
    check(lib.icepop_wave_barrier_abandons(ctypes.byref(n)))
    return int(n.value)


def ptr(t) -> int | None:
    """Device pointer of a tensor (or None)."""
    return None if t is None else t.data_ptr()
