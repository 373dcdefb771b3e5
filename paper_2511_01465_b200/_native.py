"""ctypes binding of libodescan_b200.so (the C ABI in include/odescan_b200.h).

This module is the only place the product touches the native library.  There
is no fallback: if the library is missing, or a GPU call fails, the error is
raised (NativeError / RuntimeError) instead of silently computing on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libodescan_b200.so"

ODX_OK, ODX_EINVAL, ODX_EUNSUPPORTED, ODX_ECUDA, ODX_EWORKSPACE = 0, -1, -2, -3, -4
ST_MAXITER, ST_CONVERGED, ST_NONFINITE, ST_SINGULAR = 0, 1, 2, 3
STEP_EXPLICIT_RK, STEP_IMPLICIT_WEIGHTED = 0, 1
MAX_PARAMS = 64
MAX_STAGES = 4

# problem ids (ODX_PROB_* in include/odescan_b200.h)
PROB_LOGISTIC, PROB_VDP, PROB_CARTPOLE, PROB_CARTPOLE_SQ, PROB_DAHLQUIST = 0, 1, 2, 3, 4
PROB_ROBERTSON, PROB_LORENZ63, PROB_ALLEN_CAHN, PROB_EXP_GROWTH, PROB_SQUARE = 5, 6, 7, 8, 9
PROB_LINEAR = 10

# every symbol the header declares (checked by tests/test_abi.py)
EXPORTS = (
    "odx_abi_version", "odx_last_error", "odx_supported", "odx_launch_count", "odx_last_route",
    "odx_solve_workspace_bytes",
    "odx_solve", "odx_solve_host", "odx_host_threads_max", "odx_set_host_threads",
    "odx_initial_guess", "odx_seq_march", "odx_parareal_coarse", "odx_build_explicit", "odx_build_implicit",
    "odx_scan_affine_workspace_bytes", "odx_scan_affine", "odx_max_abs", "odx_add_inplace",
    "odx_shard_workspace_bytes", "odx_shard_local", "odx_shard_fixup", "odx_shard_step",
    "odx_shard_decide_step", "odx_nccl_available", "odx_nccl_unique_id", "odx_nccl_comm_init",
    "odx_nccl_comm_destroy", "odx_solve_sharded_workspace_bytes", "odx_solve_sharded",
)


class OdxProblem(C.Structure):
    _fields_ = [("problem_id", C.c_int32), ("dim", C.c_int32), ("n_params", C.c_int32),
                ("reserved", C.c_int32), ("params", C.c_double * MAX_PARAMS)]


class OdxStepper(C.Structure):
    _fields_ = [("kind", C.c_int32), ("stages", C.c_int32),
                ("a", C.c_double * (MAX_STAGES * MAX_STAGES)), ("b", C.c_double * MAX_STAGES),
                ("w_prev", C.c_double), ("w_next", C.c_double)]


class OdxNewtonCfg(C.Structure):
    _fields_ = [("max_iters", C.c_int32), ("abort_nonfinite", C.c_int32),
                ("residual_tol", C.c_double), ("step_tol", C.c_double)]


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        super().__init__(f"libodescan_b200 error {code}: {msg}")


_lib = None


def lib():
    """Load the native library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2511_01465_b200.build` "
            f"(there is no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    vp, i64, i32, dbl, sz = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_size_t
    P_, S_, CFG = C.POINTER(OdxProblem), C.POINTER(OdxStepper), C.POINTER(OdxNewtonCfg)
    L.odx_abi_version.restype = C.c_int
    L.odx_last_error.restype = C.c_char_p
    L.odx_launch_count.restype = C.c_int64
    L.odx_last_route.restype = C.c_char_p
    L.odx_last_route.argtypes = []
    L.odx_supported.restype = C.c_int
    L.odx_host_threads_max.restype = C.c_int
    L.odx_host_threads_max.argtypes = []
    L.odx_set_host_threads.restype = C.c_int
    L.odx_set_host_threads.argtypes = [C.c_int]
    L.odx_supported.argtypes = [P_, S_]
    L.odx_solve_workspace_bytes.restype = sz
    L.odx_solve_workspace_bytes.argtypes = [P_, S_, i64, i64, CFG]
    L.odx_solve.restype = C.c_int
    L.odx_solve.argtypes = [P_, S_, vp, vp, i64, i64, dbl, CFG, vp, vp, vp, vp, vp, vp, sz, vp]
    L.odx_solve_host.restype = C.c_int
    L.odx_solve_host.argtypes = [P_, S_, vp, vp, vp, i64, i64, dbl, CFG, vp, vp, vp, vp, vp, vp]
    L.odx_initial_guess.restype = C.c_int
    L.odx_initial_guess.argtypes = [P_, i32, vp, vp, i64, i64, dbl, vp]
    L.odx_seq_march.restype = C.c_int
    L.odx_seq_march.argtypes = [P_, S_, vp, vp, i64, i64, dbl, dbl, i32, vp, vp]
    L.odx_parareal_coarse.restype = C.c_int
    L.odx_parareal_coarse.argtypes = [P_, S_, vp, vp, vp, vp, i32, i64, dbl, i32, vp]
    L.odx_build_explicit.restype = C.c_int
    L.odx_build_explicit.argtypes = [P_, S_, vp, vp, i64, dbl, vp, vp, vp, vp]
    L.odx_build_implicit.restype = C.c_int
    L.odx_build_implicit.argtypes = [P_, S_, vp, vp, i64, dbl, vp, vp, vp, vp, vp]
    L.odx_scan_affine_workspace_bytes.restype = sz
    L.odx_scan_affine_workspace_bytes.argtypes = [i64, i32]
    L.odx_scan_affine.restype = C.c_int
    L.odx_scan_affine.argtypes = [vp, vp, i64, i32, vp, vp, vp, sz, vp]
    L.odx_max_abs.restype = C.c_int
    L.odx_max_abs.argtypes = [vp, i64, i32, vp, vp]
    L.odx_add_inplace.restype = C.c_int
    L.odx_add_inplace.argtypes = [vp, vp, i64, i32, vp]
    L.odx_shard_workspace_bytes.restype = sz
    L.odx_shard_workspace_bytes.argtypes = [P_, S_, i64]
    L.odx_shard_local.restype = C.c_int
    L.odx_shard_local.argtypes = [P_, S_, vp, vp, i64, i64, dbl, vp, vp, sz, vp]
    L.odx_shard_fixup.restype = C.c_int
    L.odx_shard_fixup.argtypes = [P_, vp, i32, i32, vp, i64, vp, vp, vp, sz, vp]
    L.odx_shard_step.restype = C.c_int
    L.odx_shard_step.argtypes = [P_, S_, vp, i32, i32, vp, vp, i64, i64, dbl, vp, vp, sz, vp]
    L.odx_nccl_available.restype = C.c_int
    L.odx_nccl_available.argtypes = []
    L.odx_nccl_unique_id.restype = C.c_int
    L.odx_nccl_unique_id.argtypes = [vp]
    L.odx_nccl_comm_init.restype = C.c_int
    L.odx_nccl_comm_init.argtypes = [C.POINTER(C.c_void_p), i32, vp, i32]
    L.odx_nccl_comm_destroy.restype = C.c_int
    L.odx_nccl_comm_destroy.argtypes = [vp]
    L.odx_solve_sharded_workspace_bytes.restype = sz
    L.odx_solve_sharded_workspace_bytes.argtypes = [P_, S_, i64, i32]
    L.odx_solve_sharded.restype = C.c_int
    L.odx_solve_sharded.argtypes = [P_, S_, CFG, vp, i32, i32, vp, vp, i64, i64, dbl, vp, vp, vp,
                                    i32, vp, sz, vp]
    L.odx_shard_decide_step.restype = C.c_int
    L.odx_shard_decide_step.argtypes = [P_, S_, CFG, vp, i32, i32, i32, vp, vp,
                                        i64, i64, dbl, vp, vp, vp, vp, vp, sz, vp]
    if L.odx_abi_version() != 1:
        raise RuntimeError("libodescan_b200 ABI version mismatch")
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != ODX_OK:
        msg = lib().odx_last_error().decode(errors="replace")
        if rc == ODX_EINVAL:
            raise ValueError(msg)
        raise NativeError(rc, msg)


def make_problem(problem_id: int, dim: int, params) -> OdxProblem:
    p = OdxProblem()
    p.problem_id = int(problem_id)
    p.dim = int(dim)
    vals = [float(v) for v in params]
    if len(vals) > MAX_PARAMS:
        raise ValueError("too many problem parameters")
    p.n_params = len(vals)
    for i, v in enumerate(vals):
        p.params[i] = v
    return p


def make_explicit(a, b) -> OdxStepper:
    import numpy as np
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    s = b.shape[0]
    if s < 1 or s > MAX_STAGES:
        raise ValueError(f"explicit tableaus with 1..{MAX_STAGES} stages have a device path")
    st = OdxStepper()
    st.kind = STEP_EXPLICIT_RK
    st.stages = s
    for i in range(s):
        st.b[i] = float(b[i])
        for j in range(s):
            st.a[i * s + j] = float(a[i, j])
    return st


def make_implicit(w_prev: float, w_next: float) -> OdxStepper:
    st = OdxStepper()
    st.kind = STEP_IMPLICIT_WEIGHTED
    st.stages = 1
    st.w_prev = float(w_prev)
    st.w_next = float(w_next)
    return st


def make_cfg(max_iters: int, residual_tol: float, step_tol: float,
             abort_nonfinite: bool) -> OdxNewtonCfg:
    return OdxNewtonCfg(int(max_iters), int(bool(abort_nonfinite)), float(residual_tol),
                        float(step_tol))


def ptr(t) -> int:
    """Device pointer of a torch tensor (0 for None)."""
    return 0 if t is None else int(t.data_ptr())


def stream_handle(device=None) -> int:
    import torch
    return int(torch.cuda.current_stream(device).cuda_stream)


def exported_symbols():
    L = lib()
    return {name: hasattr(L, name) for name in EXPORTS}


if os.environ.get("ODESCAN_B200_EAGER_LOAD"):
    lib()
