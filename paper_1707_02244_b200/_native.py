"""ctypes binding of the C-ABI in include/circlasso_b200.h.

The shared library is built in-tree (paper_1707_02244_b200/_lib/) by
``make -C paper_1707_02244_b200`` or ``__graft_entry__.build()``.  There is
no fallback: if the library is missing, importing the package fails.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libcirclasso_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"circlasso_b200 native library not built: {LIB_PATH} is missing "
        "(run `make -C paper_1707_02244_b200` or __graft_entry__.build())")

lib = C.CDLL(LIB_PATH)

_d = C.POINTER(C.c_double)
_i64 = C.POINTER(C.c_int64)
_vp = C.c_void_p


class cl_config(C.Structure):
    _fields_ = [("alpha", C.c_double), ("tau", C.c_double), ("rho", C.c_double), ("sigma", C.c_double),
                ("tau1", C.c_double), ("tau2", C.c_double), ("max_iter", C.c_int64), ("target_mse", C.c_double),
                ("check_every", C.c_int32), ("pairing", C.c_int32), ("engine", C.c_int32),
                ("dense_cap", C.c_int64)]


class cl_bench_row(C.Structure):
    _fields_ = [("algorithm", C.c_char_p), ("n", C.c_int64), ("m", C.c_int64), ("k", C.c_int64),
                ("seed", C.c_uint64), ("iterations", C.c_int64), ("setup_seconds", C.c_double),
                ("total_seconds", C.c_double), ("final_mse", C.c_double), ("footprint_bytes", C.c_uint64),
                ("status", C.c_char_p)]


class cl_report(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("setup_seconds", C.c_double), ("total_seconds", C.c_double),
                ("footprint_bytes", C.c_uint64), ("metric", C.c_int32), ("reached_target", C.c_int32),
                ("final_metric", C.c_double), ("trace_len", C.c_int64)]


_SIGS = {
    "cl_abi_version": (C.c_int, []),
    "cl_last_error": (C.c_char_p, []),
    "cl_config_default": (None, [C.POINTER(cl_config)]),
    "cl_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "cl_make_problem": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_uint64, _d, _i64, _d, _i64, _d]),
    "cl_gen_sparse_signal": (C.c_int, [C.c_int64, C.c_int64, C.c_uint64, _d, _i64]),
    "cl_gen_circulant_sensing": (C.c_int, [C.c_int64, C.c_int64, C.c_uint64, _d, _i64]),
    "cl_measure": (C.c_int, [C.c_int64, C.c_int64, _d, _i64, _d, _d]),
    "cl_gen_star_field": (C.c_int, [C.c_int64, C.c_int64, C.c_double, C.c_uint64, _d]),
    "cl_blur_row": (C.c_int, [C.c_int64, C.c_int64, _d]),
    "cl_compose_rows": (C.c_int, [C.c_int64, _d, _d, _d]),
    "cl_spectral_norm": (C.c_int, [C.c_int64, _d, _d]),
    "cl_regularized_gram_inverse": (C.c_int, [C.c_int64, _d, C.c_double, C.c_double, _d]),
    "cl_mask_gram_inverse": (C.c_int, [C.c_int64, C.c_int64, _i64, C.c_double, _d]),
    "cl_circ_matvec": (C.c_int, [C.c_int, C.c_int64, _d, _d, C.c_int, _d]),
    "cl_partial_matvec": (C.c_int, [C.c_int, C.c_int64, C.c_int64, _d, _i64, _d, _d]),
    "cl_partial_transpose_matvec": (C.c_int, [C.c_int, C.c_int64, C.c_int64, _d, _i64, _d, _d]),
    "cl_solver_create": (C.c_int, [C.c_int, C.c_int64, C.c_int64, _d, _i64, _d, C.POINTER(cl_config), C.c_int,
                                   C.POINTER(_vp)]),
    "cl_solver_destroy": (None, [_vp]),
    "cl_solver_set_truth": (C.c_int, [_vp, _d]),
    "cl_solver_step": (C.c_int, [_vp, C.c_int64]),
    "cl_solver_step_checked": (C.c_int, [_vp, _d, C.POINTER(C.c_int)]),
    "cl_solver_run": (C.c_int, [_vp, C.POINTER(cl_report), _d, _i64, _d, _d, C.c_int64]),
    "cl_solver_get": (C.c_int, [_vp, C.c_char_p, _d]),
    "cl_solver_set": (C.c_int, [_vp, C.c_char_p, _d]),
    "cl_solver_info": (C.c_int, [_vp, _i64, _i64, _i64, _d, _d]),
    "cl_solver_synchronize": (C.c_int, [_vp]),
    "cl_solver_last_step_ms": (C.c_int, [_vp, _d]),
    "cl_solver_phase_ms": (C.c_int, [_vp, _d, C.POINTER(C.c_int)]),
    "cl_solver_phase_history": (C.c_int, [_vp, _d, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
    "cl_solver_profile": (C.c_int, [_vp, C.c_int]),
    "cl_solver_shard": (C.c_int, [_vp, C.c_int, C.c_int]),
    "cl_solver_stream": (C.c_int, [_vp, C.POINTER(_vp)]),
    "cl_solver_run_phase": (C.c_int, [_vp, C.c_int]),
    "cl_solver_phase_output": (C.c_int, [_vp, C.c_int, C.POINTER(_vp), _i64, _i64, _i64]),
    "cl_shard_ranges": (C.c_int, [C.c_int, C.c_int64, C.c_int64, _i64, C.c_int, C.c_int, _i64, _i64, _i64, _i64]),
    "cl_ffma_peak": (C.c_int, [C.c_int, _d]),
    "cl_comm_unique_id": (C.c_int, [C.c_char_p]),
    "cl_comm_init_rank": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]),
    "cl_comm_destroy": (None, [_vp]),
    "cl_solver_attach_comm": (C.c_int, [_vp, _vp]),
    "cl_solver_peer_export": (C.c_int, [_vp, C.c_int, C.c_int, C.c_char_p]),
    "cl_solver_peer_attach": (C.c_int, [_vp, C.c_char_p]),
    "cl_group_create": (C.c_int, [C.c_int, C.c_int64, C.c_int64, _d, _i64, _d, C.POINTER(cl_config),
                                  C.POINTER(C.c_int), C.c_int, C.c_int, C.POINTER(_vp)]),
    "cl_group_destroy": (None, [_vp]),
    "cl_group_set_truth": (C.c_int, [_vp, _d]),
    "cl_group_step": (C.c_int, [_vp, C.c_int64]),
    "cl_group_run": (C.c_int, [_vp, C.POINTER(cl_report), _d, _i64, _d, _d, C.c_int64]),
    "cl_group_get": (C.c_int, [_vp, C.c_char_p, _d]),
    "cl_group_synchronize": (C.c_int, [_vp]),
    "cl_group_info": (C.c_int, [_vp, C.POINTER(C.c_int), _i64, C.POINTER(C.c_int)]),
    "cl_write_vector": (C.c_int, [C.c_char_p, _d, C.c_int64]),
    "cl_read_vector": (C.c_int, [C.c_char_p, _d, C.c_int64, _i64]),
    "cl_write_operator": (C.c_int, [C.c_char_p, C.c_int64, C.c_int64, _d, _i64]),
    "cl_read_operator": (C.c_int, [C.c_char_p, _d, C.c_int64, _i64, C.c_int64, _i64, _i64]),
    "cl_write_pgm": (C.c_int, [C.c_char_p, C.c_int64, C.c_int64, _d]),
    "cl_read_pgm": (C.c_int, [C.c_char_p, _d, C.c_int64, _i64, _i64]),
    "cl_bench_iters_per_second": (C.c_double, [C.POINTER(cl_bench_row)]),
    "cl_bench_csv_header": (C.c_int, [C.c_char_p, C.c_int64, _i64]),
    "cl_bench_csv_row": (C.c_int, [C.POINTER(cl_bench_row), C.c_char_p, C.c_int64, _i64]),
    "cl_matvec_scheme_bench": (C.c_int, [C.c_int, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_int64, _d, _d,
                                         C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), _d]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)

if lib.cl_abi_version() != 3:
    raise ImportError("circlasso_b200: C-ABI version mismatch")
