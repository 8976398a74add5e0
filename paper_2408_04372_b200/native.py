"""ctypes binding of the C ABI in include/stmg_b200.h (libstmg_b200.so, built
in-tree by paper_2408_04372_b200/csrc/Makefile). Loading fails loudly when the
extension is missing: there is no CPU fallback on the product path."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libstmg_b200.so")

c_double_p = C.POINTER(C.c_double)
c_int_p = C.POINTER(C.c_int)
c_ll_p = C.POINTER(C.c_longlong)


class MgOptions(C.Structure):
    _fields_ = [("n_smooth", C.c_int), ("direct_coarse_max", C.c_longlong), ("coarse_rel_tol", C.c_double),
                ("coarse_max_iters", C.c_int), ("eig_iters", C.c_int), ("seed", C.c_ulonglong)]


class GmresOptions(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("restart", C.c_int), ("rel_tol", C.c_double), ("abs_tol", C.c_double)]


class GmresResult(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("initial_residual", C.c_double),
                ("final_residual", C.c_double), ("history_len", C.c_int)]


class Problem(C.Structure):
    """stmg_problem: the resolved ProblemSpec (include/stmg/driver.hpp:14-48)."""
    _fields_ = [("equation", C.c_int), ("scheme", C.c_int), ("problem", C.c_int), ("k", C.c_int), ("p", C.c_int),
                ("dim", C.c_int), ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("t_final", C.c_double),
                ("refinements", C.c_int), ("base_cells", C.c_int), ("base_time_intervals", C.c_int),
                ("batch", C.c_int), ("frequency", C.c_double), ("shm_s", C.c_double), ("perturb", C.c_double),
                ("seed", C.c_ulonglong), ("rho_random_lo", C.c_double), ("rho_random_hi", C.c_double),
                ("abs_tol", C.c_double), ("rel_tol", C.c_double), ("max_iters", C.c_int), ("restart", C.c_int),
                ("n_smooth", C.c_int), ("precondition", C.c_int), ("probe_samples_per_step", C.c_int),
                ("n_strategy", C.c_int), ("strategy", C.c_int * 32), ("timers", C.c_int)]


class RunReport(C.Structure):
    """stmg_run_report (include/stmg/driver.hpp:54-91)."""
    _fields_ = [("converged", C.c_int), ("n_space_dofs", C.c_longlong), ("n_steps_total", C.c_int),
                ("n_batches", C.c_int), ("dofs_global", C.c_longlong), ("n_batches_run", C.c_int),
                ("mean_iterations", C.c_double), ("work", C.c_double), ("has_error_u", C.c_int),
                ("has_error_v", C.c_int), ("error_u", C.c_double * 3), ("error_v", C.c_double * 3),
                ("n_levels", C.c_int), ("sections", C.c_double * 5), ("n_probe_samples", C.c_longlong)]


LINEAR_MAP = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)
HOST_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, c_double_p, C.c_longlong)
HOST_SENDRECV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, c_double_p, c_double_p, C.c_longlong)


class HostTransport(C.Structure):
    """stmg_host_transport: callbacks of the host-staged communicator."""
    _fields_ = [("ctx", C.c_void_p), ("allreduce_sum", HOST_ALLREDUCE), ("sendrecv", HOST_SENDRECV)]

# (name, restype, argtypes): every symbol declared in include/stmg_b200.h
SIGNATURES = [
    ("stmg_last_error", C.c_char_p, []),
    ("stmg_version", C.c_char_p, []),
    ("stmg_kernel_launches", C.c_longlong, []),
    ("stmg_quadrature", C.c_int, [C.c_int, C.c_int, c_double_p, c_double_p]),
    ("stmg_temporal_weights", C.c_int, [C.c_int, C.c_int, c_double_p, c_double_p, c_double_p, c_double_p, c_double_p]),
    ("stmg_block_coefficients", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, c_double_p, c_double_p]),
    ("stmg_mesh_create_box", C.c_int, [C.c_int, c_double_p, c_double_p, c_ll_p, C.c_int, c_double_p,
                                       C.c_void_p]),
    ("stmg_mesh_create", C.c_int, [C.c_int, c_double_p, c_double_p, C.c_longlong, C.c_int, c_double_p,
                                   C.c_void_p]),
    ("stmg_mesh_destroy", None, [C.c_void_p]),
    ("stmg_st_operator_create", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                          C.c_int, c_double_p, C.c_void_p]),
    ("stmg_st_operator_destroy", None, [C.c_void_p]),
    ("stmg_st_operator_n_dofs", C.c_longlong, [C.c_void_p]),
    ("stmg_st_operator_n_space", C.c_longlong, [C.c_void_p]),
    ("stmg_st_operator_n_t", C.c_int, [C.c_void_p]),
    ("stmg_st_operator_apply", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_st_operator_apply_host", C.c_int, [C.c_void_p, c_double_p, c_double_p]),
    ("stmg_spatial_apply", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_st_operator_residual", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_st_operator_interpolate", C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_double, c_double_p, C.c_double,
                                               C.c_int, C.c_void_p, C.c_void_p]),
    ("stmg_st_operator_assemble_rhs", C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_void_p,
                                                C.c_void_p, C.c_void_p]),
    ("stmg_st_operator_extract_final", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                 C.c_void_p, C.c_void_p]),
    ("stmg_asm_create", C.c_int, [C.c_void_p, C.c_void_p]),
    ("stmg_asm_destroy", None, [C.c_void_p]),
    ("stmg_asm_add_correction", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_transfer_create", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_transfer_destroy", None, [C.c_void_p]),
    ("stmg_transfer_prolong", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_transfer_restrict", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_mg_options_default", None, [C.POINTER(MgOptions)]),
    ("stmg_multigrid_create", C.c_int, [C.c_int, C.c_int, C.c_void_p, c_double_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_double, C.c_int, c_int_p, C.POINTER(MgOptions), C.c_void_p]),
    ("stmg_multigrid_destroy", None, [C.c_void_p]),
    ("stmg_multigrid_n_levels", C.c_int, [C.c_void_p]),
    ("stmg_multigrid_level_info", C.c_int, [C.c_void_p, C.c_int, c_int_p, c_ll_p, c_double_p]),
    ("stmg_multigrid_set_omega", C.c_int, [C.c_void_p, C.c_int, C.c_double]),
    ("stmg_multigrid_smoother_kind", C.c_int, [C.c_void_p, C.c_int]),
    ("stmg_multigrid_smoother_bytes", C.c_longlong, [C.c_void_p, C.c_int]),
    ("stmg_multigrid_operator_at", C.c_void_p, [C.c_void_p, C.c_int]),
    ("stmg_multigrid_apply", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_multigrid_apply_host", C.c_int, [C.c_void_p, c_double_p, c_double_p]),
    ("stmg_multigrid_smooth", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_multigrid_asm_add_correction", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_multigrid_prolong", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_multigrid_restrict", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_multigrid_device_bytes", C.c_longlong, [C.c_void_p]),
    ("stmg_gmres_options_default", None, [C.POINTER(GmresOptions)]),
    ("stmg_gmres", C.c_int, [C.c_longlong, LINEAR_MAP, C.c_void_p, LINEAR_MAP, C.c_void_p, C.c_void_p, C.c_void_p,
                             C.POINTER(GmresOptions), C.POINTER(GmresResult), c_double_p, C.c_int, C.c_void_p]),
    ("stmg_solve", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(GmresOptions),
                             C.POINTER(GmresResult), c_double_p, C.c_int, C.c_void_p]),
    ("stmg_solve_host", C.c_int, [C.c_void_p, C.c_int, c_double_p, c_double_p, C.POINTER(GmresOptions),
                                  C.POINTER(GmresResult), c_double_p, C.c_int]),
    ("stmg_st_operator_error_norms", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                               c_double_p]),
    ("stmg_march", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_void_p,
                             C.POINTER(GmresOptions), c_int_p, c_double_p, C.c_void_p]),
    ("stmg_march_probes", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_void_p,
                                    C.POINTER(GmresOptions), c_int_p, c_double_p, C.c_int, c_double_p, C.c_int,
                                    c_double_p, c_double_p, C.c_void_p]),
    # z-slab partitioned solve
    ("stmg_nccl_unique_id", C.c_int, [C.c_char_p]),
    ("stmg_problem_sizes", C.c_int, [C.POINTER(Problem), c_int_p, c_int_p, c_ll_p]),
    ("stmg_run", C.c_int, [C.POINTER(Problem), C.c_int, c_double_p, C.POINTER(RunReport), C.c_int, c_int_p,
                           c_double_p, c_int_p, C.c_int, c_int_p, c_ll_p, c_double_p, C.c_longlong, c_double_p,
                           c_double_p]),
    ("stmg_level_plan", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, c_int_p, C.c_int,
                                  c_int_p, c_int_p, c_double_p]),
    ("stmg_perturbed_vertices", C.c_int, [C.c_int, c_double_p, c_double_p, C.c_int, C.c_int, C.c_double,
                                          C.c_ulonglong, c_double_p]),
    ("stmg_comm_create", C.c_int, [C.c_int, C.c_int, C.c_char_p, C.c_void_p]),
    ("stmg_comm_destroy", None, [C.c_void_p]),
    ("stmg_comm_create_host", C.c_int, [C.c_int, C.c_int, C.POINTER(HostTransport), C.c_void_p]),
    ("stmg_slab_plan", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_longlong, C.c_int, c_int_p,
                                 c_int_p]),
    ("stmg_slab_multigrid_create", C.c_int, [C.c_int, C.c_int, C.c_void_p, c_double_p, C.c_int, C.c_int, C.c_int,
                                             C.c_int, C.c_double, C.c_int, c_int_p, C.c_void_p, C.c_int, C.c_int,
                                             C.c_int, C.c_void_p, C.c_void_p]),
    ("stmg_slab_multigrid_destroy", None, [C.c_void_p]),
    ("stmg_slab_multigrid_local_dofs", C.c_longlong, [C.c_void_p]),
    ("stmg_slab_multigrid_info", C.c_int, [C.c_void_p, c_int_p]),
    ("stmg_slab_multigrid_part", C.c_int, [C.c_void_p, C.c_int, c_ll_p, c_ll_p, c_ll_p]),
    ("stmg_slab_multigrid_omega", C.c_double, [C.c_void_p, C.c_int]),
    ("stmg_slab_multigrid_set_omega", C.c_int, [C.c_void_p, C.c_int, C.c_double]),
    ("stmg_slab_multigrid_apply", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_slab_multigrid_vcycle", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_slab_multigrid_asm_add_correction", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_slab_multigrid_solve", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(GmresOptions),
                                            C.POINTER(GmresResult), C.c_void_p]),
    ("stmg_slab_multigrid_dot", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, c_double_p]),
    ("stmg_slab_multigrid_scatter", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stmg_slab_multigrid_gather", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
]

_lib = None


def load() -> C.CDLL:
    """Load the sm_100a extension; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"stmg-b200: CUDA extension missing at {LIB_PATH}; run __graft_entry__.build()")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class StmgError(RuntimeError):
    pass


class StmgInvalidArgument(StmgError, ValueError):
    pass


def check(rc: int) -> None:
    """Rethrow a C-ABI status as the reference's exception kind
    (invalid_argument -> ValueError subclass, runtime_error -> RuntimeError)."""
    if rc == 0:
        return
    msg = load().stmg_last_error().decode()
    if rc == -1:
        raise StmgInvalidArgument(msg)
    raise StmgError(msg)
