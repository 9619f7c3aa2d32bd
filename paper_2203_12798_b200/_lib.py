"""ctypes binding of libdpar2_b200.so (include/dpar2_b200.h).

The library is REQUIRED: there is no CPU fallback.  ``lib()`` raises if the
shared object is missing or fails to load, and every device call checks the
returned dp2_status.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libdpar2_b200.so"
_lib = None

c_i32, c_i64, c_sz, c_f32, c_f64, c_vp = C.c_int32, C.c_int64, C.c_size_t, C.c_float, C.c_double, C.c_void_p
P = C.POINTER

DP2_OK, DP2_ERR_NONFINITE, DP2_ERR_NOCONV, DP2_ERR_SHAPE, DP2_ERR_CUDA, DP2_ERR_ARG = range(6)
DP2_F64, DP2_F32 = 0, 1
STATUS_WORDS = 8
INT64_MAX = (1 << 63) - 1


class Store(C.Structure):
    """Mirror of ``dp2_store`` (include/dpar2_b200.h)."""

    _fields_ = [
        ("X", c_vp), ("dtype", c_i32), ("nseg", c_i32), ("ldx", c_i64), ("J", c_i64), ("K", c_i64),
        ("total_rows", c_i64), ("npieces", c_i64), ("row_off", c_vp), ("piece_slice", c_vp),
        ("piece_row0", c_vp), ("piece_rows", c_vp), ("seg_begin", c_vp), ("slice_piece", c_vp),
    ]


# name -> (restype, argtypes)
_SIGS = {
    "dp2_abi_version": (c_i32, []),
    "dp2_status_string": (C.c_char_p, [c_i32]),
    "dp2_last_error": (C.c_char_p, []),
    "dp2_device_sm_count": (c_i32, []),
    "dp2_launch_count": (c_i64, [c_i32]),
    "dp2_status_init": (c_i32, [c_vp, c_vp]),
    "dp2_stream_segments": (c_i32, [c_i32, c_i64, c_i32]),
    "dp2_set_sketch_engine": (c_i32, [c_i32]),
    "dp2_sketch_kind": (c_i32, [P(Store), c_i32, c_i32, c_i32]),
    "dp2_greedy_partition": (c_i32, [P(c_i64), c_i64, c_i32, P(c_i64), P(c_i32), P(c_i64)]),
    "dp2_piece_capacity": (c_i64, [c_i64, c_i32]),
    "dp2_plan_pieces": (c_i32, [P(c_i64), c_i64, c_i32, P(c_i32), P(c_i64), P(c_i32), P(c_i32), P(c_i32),
                                P(c_i64)]),
    "dp2_derived_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "dp2_omega_generate_stream": (c_i32, [C.c_uint64, c_i64, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "dp2_d2h_staged": (c_i32, [c_vp, c_vp, c_sz, c_vp]),
    "dp2_omega_generate": (c_i32, [C.c_uint64, c_i64, c_i32, c_vp, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp,
                                   c_vp]),
    "dp2_omega_replay": (c_i32, [c_vp, c_i64, P(c_f64), P(c_i32)]),
    "dp2_omega_patch": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_i32, c_vp, c_vp, P(c_i32), c_vp]),
    "dp2_slice_stats": (c_i32, [P(Store), c_vp, c_vp, c_vp]),
    "dp2_copy_h2d_small": (c_i32, [c_vp, c_vp, c_sz, c_vp]),
    "dp2_sketch_uses_tc": (c_i32, [P(Store), c_i32]),
    "dp2_host_first_nonfinite": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_i32, P(c_i64)]),
    "dp2_stream_pass": (c_i32, [P(Store), c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dp2_stage1_workspace": (c_sz, [P(Store), c_i32, c_i32]),
    "dp2_stage1": (c_i32, [P(Store), c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp,
                           P(c_f32), c_vp]),
    "dp2_stage1_signs": (c_i32, [P(Store), c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp,
                                 P(c_f32), c_vp]),
    "dp2_stage1_power": (c_i32, [P(Store), c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz,
                                 c_vp, P(c_f32), c_vp]),
    "dp2_stage2_workspace": (c_sz, [c_i64, c_i64, c_i32, c_i32]),
    "dp2_stage2_power": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp,
                                 c_vp]),
    "dp2_stage2": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp, c_vp]),
    "dp2_als_workspace": (c_sz, [c_i64, c_i64, c_i32]),
    "dp2_als_stamp_offset": (c_sz, [c_i64, c_i64, c_i32]),
    "dp2_als_run": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_f64, c_i32,
                            c_vp, c_vp, c_vp, c_i32, c_vp, c_sz, c_vp, c_vp]),
    "dp2_als_phase": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_f64,
                              c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp, c_vp]),
    "dp2_update_rotations": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                     c_sz, c_vp, c_vp]),
    "dp2_mttkrp": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz,
                           c_vp]),
    "dp2_update_factors": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_sz,
                                   c_vp, c_vp]),
    "dp2_convergence_metric": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp,
                                       c_sz, c_vp]),
    "dp2_assemble_q": (c_i32, [P(Store), c_vp, c_i32, c_vp, c_vp, c_vp]),
    "dp2_assemble_q_signed": (c_i32, [P(Store), c_vp, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "dp2_fitness_workspace": (c_sz, [P(Store)]),
    "dp2_fitness": (c_i32, [P(Store), c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "dp2_gemm_tn": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_i32, c_vp, c_vp]),
    "dp2_zero_pass_workspace": (c_sz, [c_i64, c_i32]),
    "dp2_fitness_zero_pass": (c_i32, [c_vp, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz,
                                      c_vp]),
}

EXPORTS = tuple(_SIGS)


def lib():
    """Load (once) and return the native library; raise loudly if absent."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise RuntimeError(
                f"{_LIB_PATH} is missing: build it with `python -m paper_2203_12798_b200.build` "
                "(there is no CPU fallback)")
        handle = C.CDLL(str(_LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.dp2_abi_version() != 1:
            raise RuntimeError("libdpar2_b200.so ABI version mismatch")
        _lib = handle
    return _lib


def check(status, what):
    """Raise for a non-OK dp2_status returned by a call."""
    if status != DP2_OK:
        msg = lib().dp2_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed ({lib().dp2_status_string(status).decode()}): {msg}")


def lib_path():
    return _LIB_PATH
