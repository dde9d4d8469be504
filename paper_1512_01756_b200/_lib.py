"""ctypes binding of the in-tree C-ABI library ``lib/libsmpm_b200.so``.

The product path has no CPU fallback: if the library or a usable sm_100
device is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SMPM_LIB: an alternative in-tree build of the same library (kernel variants for experiments)
LIB_PATH = os.environ.get("SMPM_LIB") or os.path.join(HERE, "lib", "libsmpm_b200.so")

SMPM_SCHUR, SMPM_BJ, SMPM_DBJ, SMPM_2LAS = 0, 1, 2, 3
METHODS = {"schur": SMPM_SCHUR, "bj": SMPM_BJ, "dbj": SMPM_DBJ, "2las": SMPM_2LAS}
ORTH = {"cgs2": 0, "mgs": 1}
STATUS = {0: "OK", 1: "EINVAL", 2: "ERUNTIME", 3: "ENONFINITE", 4: "ESINGULAR", 5: "ECUDA", 6: "ENCCL"}

# every symbol include/smpm_b200.h declares
EXPORTS = [
    "smpm_last_error", "smpm_version", "smpm_ctx_create", "smpm_ctx_destroy", "smpm_ctx_stream",
    "smpm_batch_create", "smpm_batch_destroy", "smpm_batch_dims", "smpm_batch_set_couplings",
    "smpm_batch_set_interface_blocks", "smpm_batch_set_nullspace", "smpm_batch_set_spectral", "smpm_batch_finalize",
    "smpm_batch_coarse_info", "smpm_apply_S", "smpm_apply_St", "smpm_apply_block_jacobi_inv", "smpm_apply_Z",
    "smpm_apply_Zt", "smpm_coarse_solve", "smpm_apply_P", "smpm_apply_Q", "smpm_project_out", "smpm_solve",
    "smpm_deflated_solve", "smpm_two_level_schwarz_solve", "smpm_solve_host", "smpm_prefetch_rhs", "smpm_batch_launch_count",
    "smpm_batch_profile", "smpm_fp64_peak", "smpm_batch_set_strip_factors", "smpm_batch_set_fdm", "smpm_schur_rhs",
    "smpm_recover_solution", "smpm_solve_stacked", "smpm_fourier_y", "smpm_inverse_fourier_y",
    "smpm_batch_load_schur_blocks", "smpm_batch_set_tuning", "smpm_batch_query", "smpm_batch_set_trace", "smpm_batch_set_allreduce",
]
# smpm_batch_set_tuning keys (include/smpm_b200.h)
TUNING_KEYS = ["segb", "spec_v2", "xform", "xform_parity", "xform_ws", "xform_ares", "sp_stage", "spectral", "spec_2las", "p2fuse", "cgs_defer", "cgs_lanes", "gt_vblock", "grid_per_sm", "gt_ctas", "coarse_fork",
               "grid_nocoop", "pdl", "pythag", "grid", "grid_max", "tail_rows", "post_fuse", "early"]
PROFILE_CLASSES = ["schur_gemm", "bj_gemm", "deflation", "orthogonalization", "other", "reserved5", "grid_tail",
                   "spectral_op", "transform", "reserved"]


# smpm_allreduce_fn: int fn(void* user, double* device_buf, int count, void* stream)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p)


class SmpmError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"smpm_b200 {STATUS.get(code, code)}: {msg}")
        self.code = code


class Report(C.Structure):
    """smpm_report (KrylovReport + krylov_s_applies)."""
    _fields_ = [
        ("iterations", C.c_int),
        ("converged", C.c_int),
        ("mismatch_warning", C.c_int),
        ("history_len", C.c_int),
        ("operator_applies", C.c_longlong),
        ("krylov_s_applies", C.c_longlong),
        ("final_rel_residual", C.c_double),
        ("wall_time_s", C.c_double),
    ]


class SolveOptions(C.Structure):
    _fields_ = [
        ("tol", C.c_double),
        ("max_iter", C.c_int),
        ("restart", C.c_int),
        ("orth", C.c_int),
        ("fuse_deflation", C.c_int),
        ("final_residual_check", C.c_int),
    ]


class StripFactors(C.Structure):
    """smpm_strip_factors (fast-diagonalisation factors of the strip operator)."""
    _fields_ = [
        ("Vx", C.c_void_p * 3),
        ("Vx_inv", C.c_void_p * 3),
        ("lx", C.c_void_p * 3),
        ("lz", C.c_void_p),
        ("tW", C.c_void_p),
        ("tE", C.c_void_p),
        ("tau", C.c_double),
        ("mu", C.c_void_p),
    ]


_lib = None


def lib():
    """Load the library (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SmpmError(5, f"{LIB_PATH} is missing; run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    vp, dp, ip, llp = C.c_void_p, C.c_void_p, C.c_int, C.c_longlong
    L.smpm_last_error.restype = C.c_char_p
    L.smpm_version.restype = C.c_char_p
    L.smpm_ctx_create.argtypes = [ip, C.POINTER(vp)]
    L.smpm_ctx_destroy.argtypes = [vp]
    L.smpm_ctx_stream.restype = vp
    L.smpm_ctx_stream.argtypes = [vp]
    L.smpm_batch_create.argtypes = [vp, ip, ip, ip, ip, C.POINTER(vp)]
    L.smpm_batch_destroy.argtypes = [vp]
    L.smpm_batch_dims.argtypes = [vp, C.POINTER(llp), C.POINTER(ip), C.POINTER(ip)]
    L.smpm_batch_set_couplings.argtypes = [vp, ip, dp, dp, dp]
    L.smpm_batch_set_interface_blocks.argtypes = [vp, ip, C.POINTER(dp), C.POINTER(llp), C.POINTER(C.c_void_p),
                                                  C.POINTER(C.c_void_p), C.POINTER(ip)]
    L.smpm_batch_set_nullspace.argtypes = [vp, ip, dp]
    L.smpm_batch_load_schur_blocks.argtypes = [vp, ip, C.c_char_p]
    L.smpm_batch_set_spectral.argtypes = [vp, ip, dp, dp, dp]
    L.smpm_batch_finalize.argtypes = [vp]
    L.smpm_batch_coarse_info.argtypes = [vp, dp, C.POINTER(ip), C.POINTER(ip)]
    for f in ("smpm_apply_S", "smpm_apply_St", "smpm_apply_block_jacobi_inv", "smpm_apply_Z", "smpm_apply_Zt",
              "smpm_coarse_solve", "smpm_apply_Q"):
        getattr(L, f).argtypes = [vp, dp, dp, vp]
    L.smpm_apply_P.argtypes = [vp, dp, dp, ip, vp]
    L.smpm_project_out.argtypes = [vp, llp, dp, dp, dp, vp]
    L.smpm_solve.argtypes = [vp, ip, dp, dp, C.POINTER(SolveOptions), C.POINTER(Report), dp, vp]
    L.smpm_deflated_solve.argtypes = [vp, dp, dp, C.POINTER(SolveOptions), C.POINTER(Report), dp, vp]
    L.smpm_two_level_schwarz_solve.argtypes = [vp, dp, dp, C.POINTER(SolveOptions), C.POINTER(Report), dp, vp]
    L.smpm_solve_host.argtypes = [vp, ip, dp, dp, C.POINTER(SolveOptions), C.POINTER(Report), dp]
    L.smpm_prefetch_rhs.argtypes = [vp, dp]
    L.smpm_solve_stacked.argtypes = [vp, ip, dp, dp, C.POINTER(SolveOptions), C.POINTER(Report), dp, vp]
    L.smpm_batch_launch_count.restype = llp
    L.smpm_batch_launch_count.argtypes = [vp]
    L.smpm_batch_profile.argtypes = [vp, ip, C.POINTER(C.c_double), C.POINTER(C.c_longlong), ip]
    L.smpm_fp64_peak.argtypes = [ip, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.smpm_batch_set_strip_factors.argtypes = [vp, C.POINTER(StripFactors)]
    L.smpm_batch_set_fdm.argtypes = [vp, ip, dp, dp, C.POINTER(StripFactors)]
    L.smpm_schur_rhs.argtypes = [vp, dp, dp, vp]
    L.smpm_fourier_y.argtypes = [llp, ip, dp, dp, vp]
    L.smpm_inverse_fourier_y.argtypes = [llp, ip, dp, dp, vp]
    L.smpm_recover_solution.argtypes = [vp, dp, dp, dp, vp]
    L.smpm_batch_set_tuning.argtypes = [vp, C.c_char_p, llp]
    L.smpm_batch_set_allreduce.argtypes = [vp, ALLREDUCE_FN, vp]
    L.smpm_batch_query.argtypes = [vp, C.c_char_p, C.POINTER(C.c_longlong)]
    L.smpm_batch_set_trace.argtypes = [vp, ip, C.c_char_p]
    _lib = L
    return L


def check(rc):
    if rc != 0:
        raise SmpmError(rc, lib().smpm_last_error().decode())
