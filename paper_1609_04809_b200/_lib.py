"""ctypes binding of the product library ``libpf_gpu.so`` (include/pf_gpu.h, include/pf_setup.h).

The library is built in-tree by ``make -C paper_1609_04809_b200/csrc`` (or
``__graft_entry__.build()``).  There is no fallback: if the shared object is missing
or a call fails, a Python exception mirroring the reference's C++ exception type is
raised.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PF_LIB_PATH") or os.path.join(HERE, "libpf_gpu.so")  # override: experiments only

# pf_status
PF_OK = 0
PF_ERR_INVALID_ARGUMENT = 1
PF_ERR_SINGULAR_DIAGONAL = 2
PF_ERR_NO_CONVERGENCE = 3
PF_ERR_TRANSPORT = 4
PF_ERR_CUDA = 5
PF_ERR_STATE = 6

PF_CH_MASTER_SLAVE, PF_CH_HALO1, PF_CH_HALO2 = 0, 1, 2
PF_UPDATE_SCATTER, PF_UPDATE_ACCUMULATE_THEN_SCATTER = 0, 1
PF_SMOOTHER_JACOBI, PF_SMOOTHER_GAUSS_SEIDEL, PF_SMOOTHER_MULTICOLOR_SOR = 0, 1, 2
PF_PROBLEM_BASELINE, PF_PROBLEM_REFERENCE_POISSON, PF_PROBLEM_UNIT_SOURCE, PF_PROBLEM_HEAT = 0, 1, 2, 3
PF_PROBLEM_LOGNORMAL = 4
PF_FE_Q2, PF_FE_ROTATED_Q1 = 2, 3
PF_COEF_CONSTANT, PF_COEF_LOGNORMAL = 0, 1


class PfError(RuntimeError):
    """parfem::Error (errors.hpp:9-12)."""


class SingularDiagonalError(PfError):
    """parfem::SingularDiagonalError (errors.hpp:26-29)."""


class NoConvergenceError(PfError):
    """parfem::NoConvergenceError (errors.hpp:31-34)."""


class TransportError(PfError):
    """parfem::TransportError (errors.hpp:14-17)."""


class CudaError(PfError):
    """Device or driver failure."""


class InvalidArgument(PfError, ValueError):
    """std::invalid_argument."""


_ERRORS = {
    PF_ERR_INVALID_ARGUMENT: InvalidArgument,
    PF_ERR_SINGULAR_DIAGONAL: SingularDiagonalError,
    PF_ERR_NO_CONVERGENCE: NoConvergenceError,
    PF_ERR_TRANSPORT: TransportError,
    PF_ERR_CUDA: CudaError,
    PF_ERR_STATE: PfError,
}


class ChannelDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("peer", C.c_int32), ("n_send", C.c_int32),
                ("n_recv", C.c_int32), ("send_dofs", C.c_void_p), ("recv_dofs", C.c_void_p)]


class LevelDesc(C.Structure):
    _fields_ = [("n_dofs", C.c_int32), ("n_own_dofs", C.c_int32),
                ("row_offsets", C.c_void_p), ("col_indices", C.c_void_p), ("values", C.c_void_p),
                ("owns_row", C.c_void_p), ("is_dirichlet", C.c_void_p), ("color", C.c_void_p),
                ("n_channels", C.c_int32), ("channels", C.POINTER(ChannelDesc)),
                ("p_offsets", C.c_void_p), ("p_cols", C.c_void_p), ("p_weights", C.c_void_p),
                ("row_order", C.c_void_p)]


class LoadDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n_cells", C.c_int32), ("n_dofs", C.c_int32),
                ("lattice", C.c_void_p), ("cells", C.c_void_p), ("factor", C.c_void_p),
                ("extent", C.c_void_p), ("phi", C.c_void_p), ("qweight", C.c_double),
                ("boundary", C.c_void_p), ("is_dirichlet", C.c_void_p)]


class AssemblyDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n_cells", C.c_int32), ("n_dofs", C.c_int32), ("n_coarse", C.c_int32),
                ("level", C.c_int32), ("lattice", C.c_void_p), ("cell_mask", C.c_void_p),
                ("is_dirichlet", C.c_void_p), ("kappa", C.c_void_p), ("elem", C.c_void_p),
                ("elem_class", C.c_void_p), ("n_classes", C.c_int32)]


class FeAssemblyDesc(C.Structure):
    _fields_ = [("family", C.c_int32), ("n_cells", C.c_int32), ("n_dofs", C.c_int32), ("keys4", C.c_void_p),
                ("is_dirichlet", C.c_void_p), ("elem", C.c_void_p), ("kappa", C.c_void_p)]


class SetupOptions(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n_coarse", C.c_int32), ("n_levels", C.c_int32), ("n_ranks", C.c_int32),
                ("rank", C.c_int32), ("problem", C.c_int32), ("dt", C.c_double), ("seed", C.c_uint64),
                ("direct_halos", C.c_int32)]


class SmootherConfig(C.Structure):
    _fields_ = [("kind", C.c_int32), ("sweeps", C.c_int32), ("local_sweeps", C.c_int32),
                ("damping", C.c_double)]


class MultigridConfig(C.Structure):
    _fields_ = [("cycles", C.c_int32), ("smoother", SmootherConfig), ("pre_smooth", C.c_int32),
                ("post_smooth", C.c_int32), ("coarse_tol", C.c_double),
                ("coarse_max_iter", C.c_int32), ("outer_tol", C.c_double),
                ("outer_max_cycles", C.c_int32)]


class SolveStats(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32),
                ("initial_residual", C.c_double), ("final_residual", C.c_double),
                ("solve_seconds", C.c_double), ("comm_seconds", C.c_double)]


# Every symbol include/pf_gpu.h and include/pf_setup.h declare (checked by the CPU tests).
EXPORTS = [
    "pf_last_error", "pf_version", "pf_device_count", "pf_set_host_threads", "pf_default_smoother_config", "pf_default_multigrid_config",
    "pf_hierarchy_create", "pf_hierarchy_set_level", "pf_hierarchy_finalize", "pf_nccl_unique_id",
    "pf_hierarchy_init_nccl", "pf_nccl_selftest", "pf_hierarchy_set_fused_exchanges", "pf_hierarchy_set_colorwise_exchange", "pf_hierarchy_set_coarse_direct", "pf_hierarchy_set_option", "pf_hierarchy_get_option", "pf_option_names", "pf_debug_guard_failures", "pf_debug_guard_selftest", "pf_hierarchy_set_coarse_replica", "pf_hierarchy_set_replica_level",
    "pf_hierarchy_destroy",
    "pf_loopback_create", "pf_loopback_destroy", "pf_hierarchy_init_loopback", "pf_hierarchy_device_bytes",
    "pf_hierarchy_peer_export", "pf_hierarchy_init_peer", "pf_hierarchy_graph_count",
    "pf_hierarchy_drop_transport",
    "pf_vector_create", "pf_vector_destroy", "pf_vector_upload", "pf_vector_download",
    "pf_vector_fill", "pf_vector_copy", "pf_host_alloc", "pf_host_free", "pf_spmv", "pf_residual_norm", "pf_smooth",
    "pf_coarse_solve", "pf_prolongate", "pf_restrict_residual", "pf_update_master_slave",
    "pf_update_halo1", "pf_update_halo2", "pf_allreduce_sum", "pf_v_cycle", "pf_solve_outer",
    "pf_solve_outer_host", "pf_launch_count", "pf_reset_launch_count", "pf_time_sweep",
    "pf_time_vcycle", "pf_hierarchy_stream", "pf_level_info",
    "pf_operator_create", "pf_operator_set_values", "pf_operator_apply", "pf_operator_destroy",
    "pf_load_create", "pf_load_set", "pf_load_assemble", "pf_load_apply_dirichlet", "pf_load_destroy",
    "pf_cn_rhs", "pf_heat_run", "pf_assembly_create", "pf_assembly_set", "pf_assemble_operator",
    "pf_assembly_destroy", "pf_operator_get_values",
    "pf_setup_create", "pf_setup_create_heat", "pf_setup_destroy", "pf_setup_level", "pf_setup_level_keys",
    "pf_setup_rhs", "pf_setup_counts", "pf_setup_seconds", "pf_setup_rhs_operator", "pf_setup_load_at",
    "pf_setup_load_desc", "pf_setup_scales", "pf_setup_export_matrixmarket", "pf_setup_create_lognormal",
    "pf_setup_kappa", "pf_setup_assembly_desc", "pf_setup_create_opts", "pf_setup_release_matrices",
    "pf_hierarchy_set_level_from_setup",
    "pf_fe_setup_create", "pf_fe_setup_create_part", "pf_fe_setup_destroy", "pf_fe_setup_level", "pf_fe_setup_level_keys",
    "pf_fe_setup_rhs", "pf_fe_setup_kappa", "pf_fe_setup_seconds", "pf_fe_setup_assembly_desc",
    "pf_fe_assembly_set",
]

_lib = None


def lib():
    """Load libpf_gpu.so once; raise if it was not built (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: build it with `make -C {os.path.join(HERE, 'csrc')}`")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    PP = C.POINTER(C.c_void_p)
    i64p = C.POINTER(C.c_int64)
    dp = C.POINTER(C.c_double)
    L.pf_last_error.restype = C.c_char_p
    L.pf_version.restype = C.c_char_p
    L.pf_setup_last_error.restype = C.c_char_p
    L.pf_fe_last_error.restype = C.c_char_p
    L.pf_default_smoother_config.argtypes = [C.POINTER(SmootherConfig)]
    L.pf_default_multigrid_config.argtypes = [C.POINTER(MultigridConfig)]
    sigs = {
        "pf_device_count": [C.POINTER(C.c_int)],
        "pf_hierarchy_create": [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, PP],
        "pf_hierarchy_set_level": [P, C.c_int, C.c_int, C.POINTER(LevelDesc)],
        "pf_hierarchy_finalize": [P],
        "pf_nccl_unique_id": [P, C.c_int],
        "pf_hierarchy_init_nccl": [P, P, C.c_int],
        "pf_nccl_selftest": [C.c_int, C.POINTER(C.c_int)],
        "pf_hierarchy_set_fused_exchanges": [P, C.c_int],
        "pf_hierarchy_set_colorwise_exchange": [P, C.c_int],
        "pf_hierarchy_set_coarse_direct": [P, C.c_int],
        "pf_hierarchy_set_option": [P, C.c_char_p, C.c_int64],
        "pf_hierarchy_get_option": [P, C.c_char_p, C.POINTER(C.c_int64)],
        "pf_set_host_threads": [C.c_int, C.POINTER(C.c_int)],
        "pf_option_names": [C.c_char_p, C.c_int64],
        "pf_debug_guard_failures": [C.POINTER(C.c_int64)],
        "pf_debug_guard_selftest": [C.c_int, C.POINTER(C.c_int)],
        "pf_setup_create_opts": [C.POINTER(SetupOptions), PP],
        "pf_setup_release_matrices": [P],
        "pf_hierarchy_set_level_from_setup": [P, C.c_int, C.c_int, P],
        "pf_hierarchy_set_coarse_replica": [P, C.c_int, C.POINTER(LevelDesc)],
        "pf_hierarchy_set_replica_level": [P, C.c_int, C.c_int, C.POINTER(LevelDesc)],
        "pf_loopback_create": [C.c_int, PP],
        "pf_loopback_destroy": [P],
        "pf_hierarchy_init_loopback": [P, P],
        "pf_hierarchy_peer_export": [P, P, C.c_int64, i64p],
        "pf_hierarchy_init_peer": [P, P, C.c_int64],
        "pf_hierarchy_graph_count": [P, i64p],
        "pf_hierarchy_drop_transport": [P],
        "pf_hierarchy_destroy": [P],
        "pf_hierarchy_device_bytes": [P, i64p],
        "pf_vector_create": [P, C.c_int, PP],
        "pf_vector_destroy": [P],
        "pf_vector_upload": [P, C.c_int, P, C.c_int64],
        "pf_vector_download": [P, C.c_int, P, C.c_int64],
        "pf_vector_fill": [P, C.c_double],
        "pf_vector_copy": [P, P],
        "pf_host_alloc": [PP, C.c_int64],
        "pf_host_free": [P],
        "pf_spmv": [P, C.c_int, P, P],
        "pf_residual_norm": [P, C.c_int, P, P, dp],
        "pf_smooth": [P, C.c_int, P, P, C.POINTER(SmootherConfig)],
        "pf_coarse_solve": [P, C.c_int, P, P, C.c_double, C.c_int, C.POINTER(SolveStats)],
        "pf_prolongate": [P, C.c_int, P, P],
        "pf_restrict_residual": [P, C.c_int, P, P],
        "pf_update_master_slave": [P, C.c_int, P, C.c_int],
        "pf_update_halo1": [P, C.c_int, P],
        "pf_update_halo2": [P, C.c_int, P],
        "pf_allreduce_sum": [P, dp, dp],
        "pf_v_cycle": [P, P, P, C.POINTER(MultigridConfig), C.POINTER(SolveStats)],
        "pf_solve_outer": [P, P, P, C.POINTER(MultigridConfig), C.POINTER(SolveStats), dp, C.c_int],
        "pf_solve_outer_host": [P, PP, PP, C.POINTER(MultigridConfig), C.POINTER(SolveStats), dp,
                                C.c_int],
        "pf_launch_count": [P, i64p],
        "pf_reset_launch_count": [P],
        "pf_time_sweep": [P, C.c_int, C.c_int, C.c_int, dp, dp],
        "pf_time_vcycle": [P, P, P, C.POINTER(MultigridConfig), C.c_int, dp],
        "pf_level_info": [P, C.c_int, C.c_int, i64p, i64p, i64p, i64p],
        "pf_hierarchy_stream": [P, PP],
        "pf_operator_create": [P, C.c_int, PP],
        "pf_operator_set_values": [P, C.c_int, P, C.c_int64],
        "pf_operator_apply": [P, P, P],
        "pf_operator_destroy": [P],
        "pf_load_create": [P, C.c_int, PP],
        "pf_load_set": [P, C.c_int, C.POINTER(LoadDesc)],
        "pf_load_assemble": [P, C.c_double, P],
        "pf_load_apply_dirichlet": [P, C.c_int, C.c_double, P, P],
        "pf_load_destroy": [P],
        "pf_cn_rhs": [P, P, P, P, P, C.c_double, C.c_int, C.c_double, P, P],
        "pf_assembly_create": [P, C.c_int, PP],
        "pf_assembly_set": [P, C.c_int, C.POINTER(AssemblyDesc)],
        "pf_assemble_operator": [P, P],
        "pf_assembly_destroy": [P],
        "pf_operator_get_values": [P, C.c_int, P, C.c_int64],
        "pf_setup_assembly_desc": [P, C.POINTER(AssemblyDesc)],
        "pf_heat_run": [P, P, P, P, P, C.c_int, C.c_int, C.c_double, dp, C.c_int, dp,
                        C.POINTER(MultigridConfig), C.POINTER(SolveStats), dp, C.c_int,
                        C.POINTER(C.c_int)],
        "pf_setup_create": [C.c_int] * 6 + [PP],
        "pf_setup_create_heat": [C.c_int] * 5 + [C.c_double, PP],
        "pf_setup_create_lognormal": [C.c_int] * 5 + [C.c_uint64, PP],
        "pf_setup_kappa": [P, PP, i64p],
        "pf_setup_rhs_operator": [P, PP, i64p],
        "pf_setup_load_at": [P, C.c_double, P, C.c_int64],
        "pf_setup_load_desc": [P, C.POINTER(LoadDesc)],
        "pf_setup_scales": [P, C.c_double, dp, C.POINTER(C.c_int32), dp],
        "pf_setup_export_matrixmarket": [P, C.c_int, C.c_char_p, C.c_char_p, i64p, i64p],
        "pf_setup_destroy": [P],
        "pf_setup_level": [P, C.c_int, C.POINTER(LevelDesc)],
        "pf_setup_level_keys": [P, C.c_int, PP, PP],
        "pf_setup_rhs": [P, PP, PP, i64p],
        "pf_setup_counts": [P, C.c_int, i64p, i64p, i64p, i64p],
        "pf_setup_seconds": [P, dp],
        "pf_fe_setup_create": [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, PP],
        "pf_fe_setup_create_part": [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, PP],
        "pf_fe_setup_destroy": [P],
        "pf_fe_setup_level": [P, C.c_int, C.POINTER(LevelDesc)],
        "pf_fe_setup_level_keys": [P, C.c_int, PP, PP],
        "pf_fe_setup_rhs": [P, PP, PP, PP, i64p],
        "pf_fe_setup_kappa": [P, PP, i64p],
        "pf_fe_setup_seconds": [P, dp],
        "pf_fe_setup_assembly_desc": [P, C.c_int, C.POINTER(FeAssemblyDesc)],
        "pf_fe_assembly_set": [P, C.c_int, C.POINTER(FeAssemblyDesc)],
    }
    for name, args in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    _lib = L
    return L


def check(rc: int, setup: bool | str = False) -> None:
    if rc == PF_OK:
        return
    L = lib()
    msg = (L.pf_fe_last_error() if setup == "fe" else L.pf_setup_last_error() if setup
           else L.pf_last_error()).decode()
    raise _ERRORS.get(rc, PfError)(msg)
