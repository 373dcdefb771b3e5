"""CPU ORACLE (test infrastructure only) — ctypes front end of odescan_oracle.c.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module, and only as the checker / the timed CPU reference.  The product
package paper_2511_01465_b200 never imports it.

Each function restates one compiled loop of the reference package
/root/reference/pkg/src/odescan/_kernels.py (file:line in the docstrings); the C
implementation is bit-identical to the numba reference (pinned by
tests/test_oracle_golden.py against tests/golden/*.npz, which the reference
itself produced via tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libodescan_oracle.so"

# Problem ids: same numbering as include/odescan_b200.h (ODX_PROB_*).
PROB = {
    "logistic": 0, "vdp": 1, "cartpole": 2, "cartpole_sq": 3, "dahlquist": 4,
    "robertson": 5, "lorenz63": 6, "allen_cahn": 7, "exp_growth": 8,
    "square": 9, "linear": 10,
}

ST_MAXITER, ST_CONVERGED, ST_NONFINITE, ST_SINGULAR = 0, 1, 2, 3
EXPLICIT, IMPLICIT = 0, 1


class Stepper(C.Structure):
    """Mirror of odx_stepper."""
    _fields_ = [("kind", C.c_int32), ("stages", C.c_int32),
                ("a", C.c_double * 16), ("b", C.c_double * 4),
                ("w_prev", C.c_double), ("w_next", C.c_double)]


class NewtonCfg(C.Structure):
    """Mirror of odx_newton_cfg."""
    _fields_ = [("max_iters", C.c_int32), ("abort_nonfinite", C.c_int32),
                ("residual_tol", C.c_double), ("step_tol", C.c_double)]


RK4_A = np.array([[0.0, 0.0, 0.0, 0.0], [0.5, 0.0, 0.0, 0.0],
                  [0.0, 0.5, 0.0, 0.0], [0.0, 0.0, 1.0, 0.0]])
RK4_B = np.array([1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0])
EULER_A = np.zeros((1, 1))
EULER_B = np.ones(1)


def explicit_stepper(a, b) -> Stepper:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    s = b.shape[0]
    st = Stepper()
    st.kind = EXPLICIT
    st.stages = s
    for i in range(s):
        st.b[i] = b[i]
        for j in range(s):
            st.a[i * s + j] = a[i, j]
    return st


def implicit_stepper(w_prev, w_next) -> Stepper:
    st = Stepper()
    st.kind = IMPLICIT
    st.w_prev = float(w_prev)
    st.w_next = float(w_next)
    return st


def stepper_by_name(name: str) -> Stepper:
    if name == "rk4":
        return explicit_stepper(RK4_A, RK4_B)
    if name == "euler":
        return explicit_stepper(EULER_A, EULER_B)
    if name == "backward_euler":
        return implicit_stepper(0.0, 1.0)
    if name == "trapezoidal":
        return implicit_stepper(0.5, 0.5)
    raise ValueError(name)


_lib = None

_dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build_library(force: bool = False) -> Path:
    """Compile the oracle with its Makefile (gcc + OpenMP)."""
    if force or not _LIB_PATH.exists() or (
            _LIB_PATH.stat().st_mtime < (_HERE / "odescan_oracle.c").stat().st_mtime):
        subprocess.run(["make", "-C", str(_HERE), "-B" if force else "all"],
                       check=True, capture_output=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build_library()
        L = C.CDLL(str(_LIB_PATH))
        i64, i32, dbl = C.c_int64, C.c_int32, C.c_double
        L.orc_max_abs.restype = dbl
        L.orc_max_abs.argtypes = [_dp, i64, C.c_int]
        L.orc_add_inplace.argtypes = [_dp, _dp, i64, C.c_int]
        L.orc_scan_affine.restype = C.c_int
        L.orc_scan_affine.argtypes = [_dp, _dp, i64, C.c_int, C.c_void_p, _dp]
        L.orc_scan_sequential.argtypes = [_dp, _dp, i64, C.c_int, _dp]
        L.orc_build_explicit.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, C.c_int, _dp, _dp,
                                         i64, dbl, _dp, _dp, _dp]
        L.orc_build_implicit.restype = i64
        L.orc_build_implicit.argtypes = [C.c_int, C.c_int, _dp, dbl, dbl, _dp, _dp, i64, dbl,
                                         _dp, _dp, _dp]
        L.orc_build_explicit_range.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, C.c_int, _dp,
                                               _dp, i64, dbl, _dp, _dp, _dp, i64]
        L.orc_build_implicit_range.restype = i64
        L.orc_build_implicit_range.argtypes = [C.c_int, C.c_int, _dp, dbl, dbl, _dp, _dp, i64,
                                               dbl, _dp, _dp, _dp, i64]
        L.orc_seq_explicit.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, C.c_int, _dp, dbl, i64,
                                       _dp]
        L.orc_seq_implicit.restype = i64
        L.orc_seq_implicit.argtypes = [C.c_int, C.c_int, _dp, dbl, dbl, _dp, dbl, i64, dbl,
                                       C.c_int, _dp]
        L.orc_solve.restype = C.c_int
        L.orc_solve.argtypes = [C.c_int, C.c_int, _dp, C.POINTER(Stepper), _dp, _dp, i64, dbl,
                                C.POINTER(NewtonCfg), _dp, _dp, C.POINTER(C.c_int32),
                                C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.c_void_p]
        L.orc_lu_factor.restype = C.c_int
        L.orc_lu_factor.argtypes = [_dp, np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS"),
                                    C.c_int]
        L.orc_lu_solve.argtypes = [_dp, np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS"),
                                   _dp, C.c_int]
        _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _params(params):
    p = np.zeros(64)
    if params is not None:
        q = np.asarray(params, np.float64).ravel()
        p[: q.size] = q
    return p


def max_abs(A) -> float:
    """_kernels.max_abs  _kernels.py:84-95 (NaN-ignoring)."""
    A = _f64(A)
    A2 = A.reshape(A.shape[0], -1) if A.ndim > 1 else A.reshape(-1, 1)
    return float(lib().orc_max_abs(A2, A2.shape[0], A2.shape[1]))


def add_inplace(X, U) -> None:
    """_kernels.add_inplace  _kernels.py:98-103."""
    assert X.flags.c_contiguous and X.dtype == np.float64
    U = _f64(U)
    lib().orc_add_inplace(X, U, X.shape[0], X.shape[1])


def scan_affine(F, c, want_F: bool = True):
    """_kernels.scan_affine  _kernels.py:116-233 (Blelloch, bit-identical)."""
    F = _f64(F)
    c = _f64(c)
    n, d = c.shape
    cp = np.empty((n, d))
    Fp = np.empty((n, d, d)) if want_F else None
    ptr = Fp.ctypes.data if want_F else None
    rc = lib().orc_scan_affine(F, c, n, d, ptr, cp)
    if rc != 0:
        raise MemoryError("oracle scan_affine allocation failed")
    return Fp, cp


def scan_sequential(F, c):
    """Offsets of affine_scan.scan_sequential (affine_scan.py:106-113): the
    left-to-right recursion cp_k = F_k cp_{k-1} + c_k (element 0's F ignored)."""
    F = _f64(F)
    c = _f64(c)
    n, d = c.shape
    cp = np.empty((n, d))
    lib().orc_scan_sequential(F, c, n, d, cp)
    return cp


def build_explicit(pid, params, a, b, x0, X, dt):
    """_kernels.build_explicit  _kernels.py:299-342."""
    X = _f64(X)
    n, d = X.shape
    a = _f64(a)
    b = _f64(b)
    Fe = np.empty((n, d, d))
    ce = np.empty((n, d))
    h = np.empty((n, d))
    lib().orc_build_explicit(pid, d, _params(params), a, b, b.shape[0], _f64(x0), X, n,
                             float(dt), Fe, ce, h)
    return Fe, ce, h


def build_implicit(pid, params, w_prev, w_next, x0, X, dt):
    """_kernels.build_implicit  _kernels.py:393-464; returns (Fe, ce, h, first_bad)."""
    X = _f64(X)
    n, d = X.shape
    Fe = np.empty((n, d, d))
    ce = np.empty((n, d))
    h = np.empty((n, d))
    bad = lib().orc_build_implicit(pid, d, _params(params), float(w_prev), float(w_next),
                                   _f64(x0), X, n, float(dt), Fe, ce, h)
    return Fe, ce, h, int(bad)


def build_range(pid, params, stepper: Stepper, halo, X, dt, offset):
    """Elements of steps offset.. of a trajectory (sharding tests): prev of the
    first local step is `halo`; F is zeroed only at the global step 0."""
    X = _f64(X)
    n, d = X.shape
    Fe = np.empty((n, d, d))
    ce = np.empty((n, d))
    h = np.empty((n, d))
    if stepper.kind == EXPLICIT:
        s = stepper.stages
        a = np.array([stepper.a[i] for i in range(s * s)]).reshape(s, s)
        b = np.array([stepper.b[i] for i in range(s)])
        lib().orc_build_explicit_range(pid, d, _params(params), a, b, s, _f64(halo), X, n,
                                       float(dt), Fe, ce, h, int(offset))
        bad = -1
    else:
        bad = lib().orc_build_implicit_range(pid, d, _params(params), stepper.w_prev,
                                             stepper.w_next, _f64(halo), X, n, float(dt), Fe, ce,
                                             h, int(offset))
    return Fe, ce, h, int(bad)


def seq_explicit(pid, params, a, b, x0, dt, n):
    """_kernels.seq_explicit  _kernels.py:345-360."""
    x0 = _f64(x0)
    X = np.empty((n, x0.shape[0]))
    b = _f64(b)
    lib().orc_seq_explicit(pid, x0.shape[0], _params(params), _f64(a), b, b.shape[0], x0,
                           float(dt), n, X)
    return X


def seq_implicit(pid, params, w_prev, w_next, x0, dt, n, tol=1e-12, max_inner=50):
    """_kernels.seq_implicit  _kernels.py:467-526; returns (X, code)."""
    x0 = _f64(x0)
    X = np.empty((n, x0.shape[0]))
    code = lib().orc_seq_implicit(pid, x0.shape[0], _params(params), float(w_prev),
                                  float(w_next), x0, float(dt), n, float(tol), int(max_inner), X)
    return X, int(code)


def solve(pid, params, stepper: Stepper, x0, guess, dt, max_iters, residual_tol=0.0,
          step_tol=0.0, abort_nonfinite=True, trace=False):
    """solve() control flow, newton_pint.py:326-406, plus the BASELINE step rule.

    Returns a dict with X (final iterate), hist, shist (length max_iters+1, NaN
    where not reached), iters, status (ST_*), status_index and, with
    trace=True, the (max_iters+1, N, d) stack of iterates (NaN past the end).
    """
    X = np.array(guess, dtype=np.float64, copy=True, order="C")
    n, d = X.shape
    hist = np.full(max_iters + 1, np.nan)
    shist = np.full(max_iters + 1, np.nan)
    iters = C.c_int32(0)
    status = C.c_int32(-1)
    sidx = C.c_int64(-1)
    cfg = NewtonCfg(int(max_iters), int(bool(abort_nonfinite)), float(residual_tol),
                    float(step_tol))
    tr = np.full((max_iters + 1, n, d), np.nan) if trace else None
    rc = lib().orc_solve(pid, d, _params(params), C.byref(stepper), _f64(x0), X, n, float(dt),
                         C.byref(cfg), hist, shist, C.byref(iters), C.byref(status),
                         C.byref(sidx), tr.ctypes.data if trace else None)
    if rc != 0:
        raise MemoryError("oracle solve allocation failed")
    out = dict(X=X, hist=hist, shist=shist, iters=iters.value, status=status.value,
               status_index=sidx.value)
    if trace:
        out["trace"] = tr
    return out


def set_threads(n: int) -> None:
    """OpenMP thread count for subsequent oracle calls (CPU-baseline timing)."""
    os.environ["OMP_NUM_THREADS"] = str(int(n))
    try:
        gomp = C.CDLL("libgomp.so.1")
        gomp.omp_set_num_threads(int(n))
    except OSError:
        pass
