"""ctypes binding of the C ABI in include/hz_b200.h (libhz_b200.so, in-tree).

The library is the product: there is no Python or CPU fallback. Importing
this module without the built library raises immediately; calling a compute
entry point without a CUDA device raises CudaError (status HZ_CUDA).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# HZ_LIB_PATH: an alternative build of the same library (A/B timing of
# compile-time variants, scripts/build_variant.py); default the in-tree one
LIB_PATH = os.environ.get("HZ_LIB_PATH") or os.path.join(_HERE, "libhz_b200.so")

# C-ABI symbols (include/hz_b200.h); tests check the library exports each one.
EXPORTS = (
    "hz_abi_version", "hz_last_error_message", "hz_device_count", "hz_options_default",
    "hz_problem_create", "hz_problem_destroy", "hz_problem_ppw", "hz_problem_num_nodes",
    "hz_apply_block", "hz_apply_block_device", "hz_solver_create", "hz_solver_destroy",
    "hz_solver_set_tolerance", "hz_solve_block", "hz_solve_block_device", "hz_solve_block_device_stream",
    "hz_solve_helmholtz", "hz_cycle", "hz_cycle_device", "hz_cycle_device_stream", "hz_coarse_solve", "hz_hierarchy_num_levels",
    "hz_hierarchy_level_dims", "hz_hierarchy_level_coefficients", "hz_sensitivity_accumulate",
    "hz_sensitivity_accumulate_device", "hz_kernel_launch_count", "hz_profile_begin",
    "hz_profile_end", "hz_profile_report", "hz_measure_fp64_peak", "hz_solve_blocks_multi", "hz_solve_blocks_multi_device", "hz_solver_set_slabs", "hz_solver_slab_info",
    "hz_sampling_create", "hz_sampling_destroy", "hz_sampling_num_receivers", "hz_sampling_receiver",
    "hz_sample_device", "hz_sample", "hz_sample_adjoint_device", "hz_sample_adjoint",
    "hz_fwi_sensitivity_rhs_device", "hz_fwi_jacobian_vec", "hz_fwi_jacobian_vec_device",
    "hz_fwi_jacobian_transpose_vec", "hz_fwi_jacobian_transpose_vec_device", "hz_compact16_device",
    "hz_solve_helmholtz_compact16", "hz_compact16", "hz_block_gram_device", "hz_block_add_scaled_device", "hz_profile_trace",
    "hz_problem_mass", "hz_problem_gamma_factor", "hz_problem_nearest_node", "hz_problem_point_source",
    "hz_point_sources_device", "hz_problem_to_csr", "hz_fwi_sensitivity_rhs", "hz_hierarchy_cycle",
    "hz_block_krylov", "hz_slab_vmm_chunks", "hz_problem_create_ex",
)


class hz_cycle_spec(C.Structure):
    _fields_ = [("kind", C.c_int), ("pre", C.c_int), ("post", C.c_int), ("jacobi_weight", C.c_double),
                ("k_inner", C.c_int)]


class hz_options(C.Structure):
    _fields_ = [("method", C.c_int), ("tol", C.c_double), ("max_cycles", C.c_int),
                ("nlevels", C.c_int), ("shift_factor", C.c_double), ("cycle_kind", C.c_int),
                ("pre", C.c_int), ("post", C.c_int), ("jacobi_weight", C.c_double),
                ("k_inner", C.c_int), ("fgmres_restart", C.c_int),
                ("dense_threshold", C.c_int64), ("precond_precision", C.c_int),
                ("rhs_block", C.c_int)]


class hz_report(C.Structure):
    _fields_ = [("cycles", C.c_int), ("qr_factorizations", C.c_int),
                ("block_gram_products", C.c_int64), ("wall_s", C.c_double),
                ("history_len", C.c_int), ("col_cycles", C.POINTER(C.c_int)),
                ("rel_residual", C.POINTER(C.c_double)), ("converged", C.POINTER(C.c_int)),
                ("history", C.POINTER(C.c_double)), ("history_cap", C.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `python paper_1607_00968_b200/build_ext.py` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.hz_last_error_message.restype = C.c_char_p
        L.hz_problem_num_nodes.restype = C.c_int64
        L.hz_kernel_launch_count.restype = C.c_int64
        L.hz_slab_vmm_chunks.restype = C.c_int64
        L.hz_profile_report.restype = C.c_int64
        L.hz_profile_report.argtypes = [C.c_char_p, C.c_int64]
        L.hz_profile_trace.restype = C.c_int64
        L.hz_profile_trace.argtypes = [C.c_char_p, C.c_int64]
        vp, i64, dbl, i32 = C.c_void_p, C.c_int64, C.c_double, C.c_int
        L.hz_problem_create.argtypes = [i32, vp, vp, vp, dbl, dbl, vp, i32, i32, C.POINTER(vp)]
        L.hz_problem_create_ex.argtypes = [i32, vp, vp, vp, dbl, dbl, vp, i32, i32, i32, C.POINTER(vp)]
        L.hz_problem_destroy.argtypes = [vp]
        L.hz_problem_ppw.argtypes = [vp, C.POINTER(dbl)]
        L.hz_problem_num_nodes.argtypes = [vp]
        L.hz_apply_block.argtypes = [vp, i64, i32, vp, vp]
        L.hz_apply_block_device.argtypes = [vp, i64, i32, vp, vp, vp]
        L.hz_solver_create.argtypes = [vp, C.POINTER(hz_options), C.POINTER(vp)]
        L.hz_solver_destroy.argtypes = [vp]
        L.hz_solver_set_tolerance.argtypes = [vp, dbl]
        L.hz_solve_block.argtypes = [vp, i64, i32, vp, vp, C.POINTER(hz_report)]
        L.hz_solve_block_device.argtypes = [vp, i64, i32, vp, vp, C.POINTER(hz_report)]
        L.hz_solve_helmholtz.argtypes = [vp, i64, i32, vp, vp, C.POINTER(hz_report)]
        L.hz_cycle.argtypes = [vp, i64, i32, vp, vp]
        L.hz_block_gram_device.argtypes = [i64, i32, i32, vp, vp, vp]
        L.hz_block_add_scaled_device.argtypes = [i64, i32, i32, vp, vp, vp]
        L.hz_cycle_device.argtypes = [vp, i64, i32, vp, vp]
        L.hz_cycle_device_stream.argtypes = [vp, i64, i32, vp, vp, vp]
        L.hz_problem_mass.argtypes = [vp, vp]
        L.hz_problem_gamma_factor.argtypes = [vp, vp]
        L.hz_problem_nearest_node.argtypes = [vp, vp, vp, C.POINTER(i64)]
        L.hz_problem_point_source.argtypes = [vp, vp, vp, dbl, dbl, vp]
        L.hz_point_sources_device.argtypes = [vp, vp, i32, vp, vp, vp, vp]
        L.hz_problem_to_csr.argtypes = [vp, dbl, vp, vp, vp, i64, C.POINTER(i64)]
        L.hz_fwi_sensitivity_rhs.argtypes = [vp, i64, i32, vp, vp, vp]
        L.hz_hierarchy_cycle.argtypes = [vp, C.POINTER(hz_cycle_spec), i64, i32, vp, vp, i32]
        L.hz_block_krylov.argtypes = [vp, i32, C.POINTER(hz_cycle_spec), i32, dbl, i32, i64, i32, vp, vp,
                                      C.POINTER(hz_report)]
        L.hz_solve_block_device_stream.argtypes = [vp, i64, i32, vp, vp, C.POINTER(hz_report), vp]
        L.hz_coarse_solve.argtypes = [vp, i64, i32, vp, vp]
        L.hz_hierarchy_num_levels.argtypes = [vp, C.POINTER(i32)]
        L.hz_hierarchy_level_dims.argtypes = [vp, i32, vp]
        L.hz_hierarchy_level_coefficients.argtypes = [vp, i32, vp, i64]
        L.hz_sensitivity_accumulate.argtypes = [vp, i64, i32, vp, vp, vp, i32]
        L.hz_sensitivity_accumulate_device.argtypes = [vp, i64, i32, vp, vp, vp, i32, vp]
        L.hz_options_default.argtypes = [C.POINTER(hz_options)]
        L.hz_solver_set_slabs.argtypes = [vp, i32, vp]
        L.hz_solver_slab_info.argtypes = [vp, C.POINTER(i32), C.POINTER(i32), vp, i32]
        L.hz_sampling_create.argtypes = [vp, vp, i64, vp, C.POINTER(vp)]
        L.hz_sampling_destroy.argtypes = [vp]
        L.hz_sampling_num_receivers.restype = i64
        L.hz_sampling_num_receivers.argtypes = [vp]
        L.hz_sampling_receiver.argtypes = [vp, i64, vp, vp, C.POINTER(i32)]
        L.hz_sample_device.argtypes = [vp, i32, vp, vp, vp]
        L.hz_sample.argtypes = [vp, i32, vp, vp]
        L.hz_sample_adjoint_device.argtypes = [vp, i32, vp, vp, i32, vp]
        L.hz_sample_adjoint.argtypes = [vp, i32, vp, vp, i32]
        L.hz_fwi_sensitivity_rhs_device.argtypes = [vp, i64, i32, vp, vp, vp, vp]
        L.hz_fwi_jacobian_vec.argtypes = [vp, vp, i64, i32, vp, vp, vp, C.POINTER(hz_report)]
        L.hz_fwi_jacobian_vec_device.argtypes = [vp, vp, i64, i32, vp, vp, vp, C.POINTER(hz_report)]
        L.hz_fwi_jacobian_transpose_vec.argtypes = [vp, vp, i64, i32, vp, vp, vp, i32, C.POINTER(hz_report)]
        L.hz_fwi_jacobian_transpose_vec_device.argtypes = [vp, vp, i64, i32, vp, vp, vp, i32,
                                                           C.POINTER(hz_report)]
        L.hz_compact16_device.argtypes = [i64, i32, vp, vp, vp, vp]
        L.hz_compact16.argtypes = [i64, i32, vp, vp, vp]
        L.hz_solve_helmholtz_compact16.argtypes = [vp, i64, i32, vp, vp, vp, C.POINTER(hz_report)]
        _lib = L
    return _lib


def loaded_path() -> str:
    lib()
    return LIB_PATH
