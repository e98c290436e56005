"""ctypes binding of libsvb.so (include/svb.h).

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``)
and loaded from this package directory.  There is no fallback: if the library
is missing every entry point raises, so a GPU run can never silently fall
back to CPU arithmetic.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint64, c_void_p  # noqa: F401

import numpy as np

from .result import BackendError, QubitCapError

LIB_PATH = os.environ.get("SVB_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsvb.so")

SVB_OK, SVB_E_ARG, SVB_E_CAP, SVB_E_OOM, SVB_E_CUDA, SVB_E_NCCL, SVB_E_SAMPLING = range(7)
SVB_C64, SVB_C128 = 0, 1
SAMPLER_ALIAS, SAMPLER_CDF = 0, 1
OPT_FUSION, OPT_MAX_HIGH, OPT_JIT_MIN_N, OPT_TC_MIN_K = 0, 1, 2, 3
ENGINE_AUTO, ENGINE_TENSOR, ENGINE_FMA = 0, 1, 2

try:  # the reference's error type when installed (sampling.py:17-18)
    from polysim.sampling import SamplingError  # type: ignore
except ImportError:

    class SamplingError(ValueError):
        pass


class SvbGate(ctypes.Structure):
    _fields_ = [("k", c_int32), ("qubits", c_int32 * 2), ("reserved", c_int32), ("mat", c_double * 32)]


GATE_DTYPE = np.dtype([("k", "<i4"), ("q", "<i4", (2,)), ("r", "<i4"), ("mat", "<f8", (32,))])
assert GATE_DTYPE.itemsize == ctypes.sizeof(SvbGate) == 272
# svb_gate_op: compact batch record (kind, q0, q1, reserved, params[3])
GATE_OP_DTYPE = np.dtype([("kind", "<i4"), ("q0", "<i4"), ("q1", "<i4"), ("r", "<i4"), ("p", "<f8", (3,))])
assert GATE_OP_DTYPE.itemsize == 40

_h = c_void_p
_dp = POINTER(c_double)
_u64p = POINTER(c_uint64)
_i32p = POINTER(c_int32)
_i64p = POINTER(c_int64)

_SIGS = {
    "svb_last_error": (ctypes.c_char_p, []),
    "svb_version": (c_int, []),
    "svb_max_qubits": (c_int, [c_int, c_int, POINTER(c_int)]),
    "svb_host_alloc": (c_int, [c_uint64, POINTER(c_void_p)]),
    "svb_host_free": (c_int, [c_void_p]),
    "svb_set_option": (c_int, [_h, c_int, c_int]),
    "svb_last_stats": (c_int, [_h, _i64p, _i64p, _i64p]),
    "svb_sync": (c_int, [_h]),
    "svb_timer_start": (c_int, [_h]),
    "svb_timer_stop": (c_int, [_h, _dp]),
    "svb_profile": (c_int, [_h, c_int]),
    "svb_profile_read": (c_int, [_h, _dp]),
    "svb_profile_passes": (c_int, [_h, _dp, c_int, _i32p]),
    "svb_create": (c_int, [c_int, c_int, c_int, POINTER(c_void_p)]),
    "svb_destroy": (c_int, [_h]),
    "svb_managed_alloc": (c_int, [c_uint64, c_int, POINTER(c_void_p)]),
    "svb_managed_free": (c_int, [c_void_p]),
    "svb_create_view": (c_int, [c_int, c_int, c_void_p, POINTER(c_void_p)]),
    "svb_set_zero": (c_int, [_h]),
    "svb_copy_state": (c_int, [_h, _h]),
    "svb_n_qubits": (c_int, [_h]),
    "svb_set_amplitudes": (c_int, [_h, c_void_p, c_uint64, c_uint64]),
    "svb_get_amplitudes": (c_int, [_h, c_void_p, c_uint64, c_uint64]),
    "svb_apply": (c_int, [_h, c_void_p, c_int]),
    "svb_apply_z": (c_int, [_h, c_void_p, c_int, _i32p, c_int, _dp]),
    "svb_marginal_probs": (c_int, [_h, _i32p, c_int, _dp]),
    "svb_expect_z": (c_int, [_h, _u64p, c_int, _dp]),
    "svb_compare": (c_int, [_h, _h, _dp]),
    "svb_apply_matrix": (c_int, [_h, _i32p, c_int, _dp, c_int]),
    "svb_last_engine": (c_int, [_h]),
    "svb_sample": (c_int, [_h, _i32p, c_int, _i32p, c_int, c_uint64, _u64p, c_int, _u64p, _u64p, _u64p]),
    "svb_alias_table": (c_int, [c_int, _dp, c_uint64, _dp, _i64p]),
    "svb_rng_seed": (c_int, [_h, _u64p]),
    "svb_batch_small": (c_int, [c_int, c_int, c_int, _i32p, _i32p, _i32p, c_void_p, c_int, _u64p, _i32p,
                                POINTER(ctypes.c_int8), c_uint64, _u64p]),
    "svb_batch_run": (c_int, [c_int, c_int, c_int, _i32p, _i32p, _i32p, c_void_p, c_void_p, c_int, c_int, _u64p,
                              _i32p, POINTER(ctypes.c_int8), c_uint64, c_int, c_int, _u64p, _i32p]),
    "svb_expand_gates": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "svb_device_ptr": (c_int, [_h, POINTER(c_void_p), _u64p, _i64p]),
    "svb_half_copy": (c_int, [_h, c_int, c_int, c_void_p, c_int]),
    "svb_clear": (c_int, [_h]),
    "svb_block_copy": (c_int, [_h, _i32p, c_int, c_uint64, c_uint64, c_uint64, c_void_p, c_int, c_int]),
    "svb_outer": (c_int, [_h, _h, _h]),
    "svb_permute_qubits": (c_int, [_h, POINTER(c_int32)]),
    "svb_select_half": (c_int, [_h, _h, c_int, c_int]),
    "svb_alias_sample": (c_int, [c_int, _dp, _i64p, c_uint64, c_uint64, _u64p, _u64p]),
    "svb_alias_upload": (c_int, [c_int, _dp, _i64p, c_uint64, ctypes.POINTER(c_void_p)]),
    "svb_alias_sample_table": (c_int, [c_void_p, c_uint64, _u64p, _u64p]),
    "svb_alias_release": (c_int, [c_void_p]),
    "svb_alias_draw": (c_int, [c_int, _dp, c_uint64, c_uint64, POINTER(c_uint64), POINTER(c_uint64)]),
    "svb_sample_slice": (c_int, [_h, c_uint64, _u64p, c_double, c_double, c_double, _i32p, c_int, c_uint64, _u64p,
                                 _u64p, _u64p]),
    "svb_measure": (c_int, [_h, c_int, _i32p]),
    "svb_reset": (c_int, [_h, c_int]),
    "svb_replay": (c_int, [_h, _h, _i32p, c_int, c_void_p, _i32p, c_uint64, _u64p, _u64p]),
    "svb_replay_small": (c_int, [c_int, c_int, c_int, c_void_p, _i32p, c_int, c_void_p, c_int, c_uint64, _u64p,
                                 _u64p]),
    "svb_plan": (c_int, [c_int, c_int, c_void_p, c_int, _i64p, _i64p, _i64p, _i32p]),
    "svb_emulate_apply": (c_int, [c_int, c_int, c_void_p, c_int, c_void_p, c_int]),
    "svb_jit_check": (c_int, [c_int, c_int, c_void_p, c_int, _i64p, ctypes.c_char_p, c_int]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """The loaded library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BackendError(
                f"libsvb.so not found at {LIB_PATH}; build it with `make` or __graft_entry__.build()"
            )
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == SVB_OK:
        return
    msg = lib().svb_last_error().decode(errors="replace")
    if rc == SVB_E_ARG:
        raise ValueError(msg)
    if rc == SVB_E_CAP:
        raise QubitCapError(msg)
    if rc == SVB_E_SAMPLING:
        raise SamplingError(msg)
    raise BackendError(f"libsvb error {rc}: {msg}")


def ptr(a: np.ndarray, ctype=None):
    p = a.ctypes.data_as(c_void_p)
    return ctypes.cast(p, POINTER(ctype)) if ctype is not None else p
