"""Device ops mirroring the reference's compiled loops one to one.

odescan._kernels (/root/reference/pkg/src/odescan/_kernels.py) exposes
build_explicit (:299-342), build_implicit (:393-464), scan_affine (:116-233),
max_abs (:84-95) and add_inplace (:98-103) over numpy arrays.  These are the
same operations on CUDA torch tensors (fp64, C-contiguous), each one call into
libodescan_b200.so.  solve() does not use them — it runs the fused solve
kernels (one launch per solve for resident / one-wave trajectories, one launch
per Newton iteration for long ones) — they exist for parity bisection and for
callers that drive their own Newton loop.
"""

from __future__ import annotations

import torch

from . import _native as N

__all__ = ["build_explicit", "build_implicit", "scan_affine", "max_abs", "add_inplace"]


def _chk(*ts):
    for t in ts:
        if t is None:
            continue
        if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise ValueError("device ops take contiguous float64 CUDA tensors")


def build_explicit(problem, stepper, x0, X, dt):
    """(Fe, ce, h) for an explicit stepper; _kernels.build_explicit."""
    _chk(x0, X)
    n, d = X.shape
    Fe = torch.empty((n, d, d), dtype=torch.float64, device=X.device)
    ce = torch.empty((n, d), dtype=torch.float64, device=X.device)
    h = torch.empty((n, d), dtype=torch.float64, device=X.device)
    N.check(N.lib().odx_build_explicit(problem.native(), stepper.native(), N.ptr(x0), N.ptr(X),
                                       n, float(dt), N.ptr(Fe), N.ptr(ce), N.ptr(h),
                                       N.stream_handle(X.device)))
    return Fe, ce, h


def build_implicit(problem, stepper, x0, X, dt):
    """(Fe, ce, h, first_bad) for an implicit stepper; _kernels.build_implicit."""
    _chk(x0, X)
    n, d = X.shape
    Fe = torch.empty((n, d, d), dtype=torch.float64, device=X.device)
    ce = torch.empty((n, d), dtype=torch.float64, device=X.device)
    h = torch.empty((n, d), dtype=torch.float64, device=X.device)
    bad = torch.empty(1, dtype=torch.int64, device=X.device)
    N.check(N.lib().odx_build_implicit(problem.native(), stepper.native(), N.ptr(x0), N.ptr(X),
                                       n, float(dt), N.ptr(Fe), N.ptr(ce), N.ptr(h), N.ptr(bad),
                                       N.stream_handle(X.device)))
    return Fe, ce, h, int(bad.item())


def scan_affine(F, c, want_F: bool = True):
    """Inclusive affine scan (Fp, cp); _kernels.scan_affine."""
    _chk(F, c)
    n, d = c.shape
    L = N.lib()
    ws_bytes = L.odx_scan_affine_workspace_bytes(n, d)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=c.device)
    Fp = torch.empty_like(F) if want_F else None
    cp = torch.empty_like(c)
    N.check(L.odx_scan_affine(N.ptr(F), N.ptr(c), n, d, N.ptr(Fp), N.ptr(cp), N.ptr(ws),
                              ws_bytes, N.stream_handle(c.device)))
    return Fp, cp


def max_abs(A) -> float:
    """NaN-ignoring max |A| (_kernels.max_abs semantics)."""
    _chk(A)
    A2 = A.reshape(A.shape[0], -1)
    out = torch.empty(1, dtype=torch.float64, device=A.device)
    N.check(N.lib().odx_max_abs(N.ptr(A2), A2.shape[0], A2.shape[1], N.ptr(out),
                                N.stream_handle(A.device)))
    return float(out.item())


def add_inplace(X, U) -> None:
    """X += U; _kernels.add_inplace."""
    _chk(X, U)
    n, d = X.shape
    N.check(N.lib().odx_add_inplace(N.ptr(X), N.ptr(U), n, d, N.stream_handle(X.device)))
