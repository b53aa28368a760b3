"""ctypes declarations for include/sdr_b200.h (libsdr_b200.so).

The shared library is built in-tree (``make`` / ``__graft_entry__.build()``)
into ``paper_2311_14206_b200/_lib/``. There is no fallback: if the library is
missing or fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SDR_LIB_PATH") or os.path.join(_HERE, "_lib", "libsdr_b200.so")  # override: A/B builds
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "sdr_b200.h")

vp, i32, i64, u64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
P = C.POINTER
cint = C.c_int


class sdr_config(C.Structure):
    _fields_ = [("m", i64), ("t", i64), ("k", i64), ("s", i64), ("tol", f64), ("safety_init", f64),
                ("max_restarts", i32), ("variant", i32), ("sketch_seed", u64), ("rank_tol", f64),
                ("breakdown_tol", f64)]


class sdr_baseline_config(C.Structure):
    _fields_ = [("m", i64), ("tol", f64), ("max_restarts", i32), ("breakdown_tol", f64)]


class sdr_iteration_event(C.Structure):
    _fields_ = [("cycle", i32), ("step", i64), ("iteration", i64), ("sres", f64), ("new_basis_sketch_norm", f64),
                ("y", P(f64)), ("y_len", i64), ("space_dim", i64)]


class sdr_residual_event(C.Structure):
    _fields_ = [("cycle", i32), ("iteration", i64), ("sres", f64), ("true_residual", f64)]


ITER_CB = C.CFUNCTYPE(None, P(sdr_iteration_event), vp)
RES_CB = C.CFUNCTYPE(None, P(sdr_residual_event), vp)


class sdr_callbacks(C.Structure):
    _fields_ = [("on_iteration", ITER_CB), ("on_residual_check", RES_CB), ("user", vp)]


HC_ALLREDUCE = C.CFUNCTYPE(cint, P(f64), i64, vp)
HC_ALLGATHER = C.CFUNCTYPE(cint, P(i64), i64, P(i64), vp)
HC_EXCHANGE = C.CFUNCTYPE(cint, cint, P(f64), i64, P(f64), i64, vp)


class sdr_host_comm(C.Structure):
    _fields_ = [("allreduce_sum", HC_ALLREDUCE), ("allgather_i64", HC_ALLGATHER), ("exchange", HC_EXCHANGE),
                ("user", vp)]


APPLY_FN = C.CFUNCTYPE(cint, vp, vp, vp, vp)

SIGNATURES = {
    "sdr_last_error": (C.c_char_p, []),
    "sdr_version": (cint, [P(cint), P(cint), P(cint)]),
    "sdr_ctx_create": (cint, [cint, P(vp)]),
    "sdr_nccl_unique_id": (cint, [vp]),
    "sdr_ctx_create_dist": (cint, [cint, cint, cint, vp, P(vp)]),
    "sdr_ctx_create_hostcomm": (cint, [cint, cint, cint, P(sdr_host_comm), P(vp)]),
    "sdr_operator_create_callback": (cint, [vp, i64, i64, APPLY_FN, vp, P(vp)]),
    "sdr_ctx_destroy": (cint, [vp]),
    "sdr_ctx_info": (cint, [vp, P(cint), P(cint), P(cint), P(cint)]),
    "sdr_ctx_stream": (cint, [vp, P(vp)]),
    "sdr_ctx_synchronize": (cint, [vp]),
    "sdr_ctx_set_timing": (cint, [vp, cint]),
    "sdr_ctx_timing_reset": (cint, [vp]),
    "sdr_ctx_timing_get": (cint, [vp, C.c_char_p, P(i64), P(f64)]),
    "sdr_ctx_launch_count": (cint, [vp, P(i64)]),
    "sdr_csr_create": (cint, [vp, i64, i64, vp, vp, vp, P(vp)]),
    "sdr_csr_create_local": (cint, [vp, i64, i64, i64, i64, vp, vp, vp, P(vp)]),
    "sdr_csr_destroy": (cint, [vp]),
    "sdr_csr_info": (cint, [vp, P(i64), P(i64), P(i64), P(i64), P(i64), P(i64), P(i64)]),
    "sdr_csr_storage": (cint, [vp, P(i32), P(i32), P(i64), P(i64)]),
    "sdr_debug_trace": (cint, [vp, vp, i64, P(i64)]),
    "sdr_debug_timeline": (cint, [vp, C.c_char_p]),
    "sdr_debug_stamps": (cint, [vp, C.c_char_p]),
    "sdr_spmv": (cint, [vp, vp, vp, i64, vp]),
    "sdr_sketch_create_srdct": (cint, [vp, i64, i64, u64, P(vp)]),
    "sdr_sketch_create_identity": (cint, [vp, i64, P(vp)]),
    "sdr_sketch_create_sparse_sign": (cint, [vp, i64, i64, u64, i64, P(vp)]),
    "sdr_sketch_destroy": (cint, [vp]),
    "sdr_sketch_info": (cint, [vp, P(cint), P(i64), P(i64), P(u64), P(i64)]),
    "sdr_sketch_rows": (cint, [vp, vp]),
    "sdr_sketch_signs": (cint, [vp, vp]),
    "sdr_sketch_apply": (cint, [vp, vp, vp, i64, vp]),
    "sdr_gaussian_vector": (cint, [i64, u64, vp]),
    "sdr_uniform_stream": (cint, [i64, u64, vp]),
    "sdr_srdct_indices": (cint, [i64, i64, u64, vp, vp]),
    "sdr_sparse_sign_entries": (cint, [i64, u64, i64, i64, i64, vp, vp]),
    "sdr_qr_create": (cint, [i64, i64, f64, P(vp)]),
    "sdr_qr_destroy": (cint, [vp]),
    "sdr_qr_append": (cint, [vp, vp, i64, P(i64), P(cint)]),
    "sdr_qr_exclude": (cint, [vp, i64]),
    "sdr_qr_cols": (cint, [vp, P(i64)]),
    "sdr_qr_solve": (cint, [vp, vp, i64, vp, P(f64)]),
    "sdr_qr_factors": (cint, [vp, vp, vp]),
    "sdr_harmonic": (cint, [vp, vp, i64, i64, i64, f64, P(i64), P(i64), P(cint), P(cint), vp, vp, vp]),
    "sdr_harmonic_qr": (cint, [vp, vp, i64, i64, i64, f64, i32, P(i64), P(i64), P(cint), P(cint), vp, vp, vp]),
    "sdr_partition_halo": (cint, [cint, cint, vp, vp, vp, vp, vp, vp, vp, vp]),
    "sdr_partition_rows": (cint, [i64, cint, i64, vp, vp]),
    "sdr_gen_neumann": (cint, [i64, f64, P(i64), vp, vp, vp]),
    "sdr_gen_convdiff2d": (cint, [i64, f64, f64, f64, vp, P(i64), vp, vp, vp]),
    "sdr_gen_convdiff3d": (cint, [i64, f64, f64, f64, i64, i64, P(i64), vp, vp, vp]),
    "sdr_csr_create_convdiff3d": (cint, [vp, i64, i64, i64, f64, f64, f64, i64, i64, P(vp)]),
    "sdr_config_default": (cint, [P(sdr_config)]),
    "sdr_config_validate": (cint, [P(sdr_config)]),
    "sdr_recycle_create": (cint, [vp, P(vp)]),
    "sdr_recycle_destroy": (cint, [vp]),
    "sdr_recycle_info": (cint, [vp, P(i64), P(i64), P(i64), P(cint)]),
    "sdr_recycle_get": (cint, [vp, vp, vp, vp, vp]),
    "sdr_recycle_set": (cint, [vp, vp, i64, i64, i64, vp, vp, vp, cint]),
    "sdr_recycle_drop_columns": (cint, [vp, vp, i64]),
    "sdr_recycle_refresh": (cint, [vp, vp, vp, vp, cint, vp]),
    "sdr_krylov_run": (cint, [vp, vp, vp, vp, i64, i64, i64, f64, vp, vp, vp, vp, P(i64), P(cint), P(f64), vp]),
    "sdr_solve": (cint, [vp, vp, vp, vp, P(sdr_config), vp, vp, P(sdr_callbacks), vp, P(vp)]),
    "sdr_mm_read_file": (cint, [C.c_char_p, P(vp)]),
    "sdr_mm_read_string": (cint, [C.c_char_p, i64, P(vp)]),
    "sdr_host_csr_info": (cint, [vp, P(i64), P(i64), P(i64)]),
    "sdr_host_csr_arrays": (cint, [vp, P(P(i64)), P(P(i64)), P(P(f64))]),
    "sdr_host_csr_destroy": (cint, [vp]),
    "sdr_mm_write_file": (cint, [C.c_char_p, i64, i64, vp, vp, vp]),
    "sdr_mm_write_string": (cint, [i64, i64, vp, vp, vp, C.c_char_p, P(i64)]),
    "sdr_csr_read_matrix_market": (cint, [vp, C.c_char_p, P(vp)]),
    "sdr_space_file_read": (cint, [C.c_char_p, P(vp)]),
    "sdr_space_file_read_bytes": (cint, [C.c_char_p, i64, P(vp)]),
    "sdr_space_file_info": (cint, [vp, P(i64), P(i64), P(i64), P(cint)]),
    "sdr_space_file_arrays": (cint, [vp, P(P(f64)), P(P(f64)), P(P(f64))]),
    "sdr_space_file_destroy": (cint, [vp]),
    "sdr_space_file_write": (cint, [C.c_char_p, i64, i64, i64, cint, vp, vp, vp]),
    "sdr_space_file_write_bytes": (cint, [i64, i64, i64, cint, vp, vp, vp, C.c_char_p, P(i64)]),
    "sdr_recycle_save_file": (cint, [vp, vp, C.c_char_p]),
    "sdr_recycle_load_file": (cint, [vp, vp, C.c_char_p]),
    "sdr_debug_block_product": (cint, [vp, i32, i64, vp, i64, i32, vp, i64, i32, vp, i32, vp, i64, vp]),
    "sdr_debug_peer_emulate": (cint, [i32, i32, i32, vp, vp]),
    "sdr_ctx_set_stamps": (cint, [vp, cint]),
    "sdr_debug_time_step": (cint, [vp, vp, vp, vp, i64, i64, i64, i32, P(f64), P(f64)]),
    "sdr_csr_create_complex": (cint, [vp, i64, i64, vp, vp, vp, P(vp)]),
    "sdr_spmm": (cint, [vp, vp, i64, vp, i64, vp, i64]),
    "sdr_baseline_config_default": (cint, [P(sdr_baseline_config)]),
    "sdr_baseline_gmres": (cint, [vp, vp, vp, vp, P(sdr_baseline_config), vp, P(vp)]),
    "sdr_solve_sequence": (cint, [vp, i32, vp, vp, vp, vp, i32, P(sdr_config), vp, vp, vp, vp]),
    "sdr_report_destroy": (cint, [vp]),
    "sdr_report_summary": (cint, [vp, P(cint), P(i64), P(i32), P(f64), P(f64), P(f64)]),
    "sdr_report_counters": (cint, [vp, P(i64), P(i64), P(i64)]),
    "sdr_report_samples": (cint, [vp, cint, P(i64), vp, vp]),
    "sdr_report_cycles": (cint, [vp, P(i64), vp]),
    "sdr_report_notes": (cint, [vp, P(i64)]),
    "sdr_report_note": (C.c_char_p, [vp, i64]),
    "sdr_report_error": (C.c_char_p, [vp]),
    "sdr_report_phase": (cint, [vp, C.c_char_p, P(f64)]),
    "sdr_report_timing": (cint, [vp, P(f64), P(f64), P(f64)]),
}

_lib = None


def header_symbols():
    """Every function the public header declares (for the export test)."""
    with open(HEADER_PATH) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"SDR_API\s+[^;(]*?\b(sdr_\w+)\s*\(", text)))


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libsdr_b200.so not built at {LIB_PATH}; run `make` or __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L
