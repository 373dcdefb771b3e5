"""ODE problems: the reference's plug-in type and its benchmark IVPs.

Mirrors odescan.problems (/root/reference/pkg/src/odescan/problems.py): the
frozen dataclass OdeProblem (:36-65) with the same fields and validation, the
five benchmark factories and get_problem/PROBLEM_NAMES (:331-350).

What changes is what the solver runs.  The reference's solver specialises its
numba kernels on the problem's compiled f_into/jac_into (_kernels.py:7-9); a
numba dispatcher cannot run on the GPU, so here every problem also carries a
`device` spec (problem id, parameters) selecting a compiled CUDA functor
(include/odescan_b200.h ODX_PROB_*).  solve() requires it and raises for a
problem without one — there is no CPU fallback.  f / jac_f / f_into /
jac_into remain as host numpy callables for guesses and checks.

The BASELINE problems (Lorenz-63, van der Pol with mu and x0 as parameters,
periodic Allen-Cahn method of lines) are added as further factories.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _native as N

__all__ = [
    "OdeProblem", "logistic", "van_der_pol", "cart_pole", "dahlquist", "robertson",
    "lorenz63", "allen_cahn", "exp_growth", "square", "linear", "get_problem",
    "PROBLEM_NAMES", "EXTRA_PROBLEM_NAMES",
]


@dataclass(frozen=True)
class OdeProblem:
    """An autonomous IVP dx/dt = f(x), x(t0) = x0 on [t0, tf].

    Same fields and validation as the reference (problems.py:36-65), plus
    `device` = (problem_id, params) naming the CUDA functor the solver runs.
    """

    name: str
    dim: int
    f: Callable
    jac_f: Callable
    x0: np.ndarray
    t0: float
    tf: float
    stiff: bool = False
    f_into: Optional[Callable] = field(default=None, repr=False)
    jac_into: Optional[Callable] = field(default=None, repr=False)
    device: Optional[tuple] = field(default=None, repr=False)

    def __post_init__(self):
        if not self.tf > self.t0:
            raise ValueError(f"need tf > t0, got [{self.t0}, {self.tf}]")
        x0 = np.asarray(self.x0, dtype=np.float64)
        if x0.shape != (self.dim,):
            raise ValueError(f"x0 has shape {x0.shape}, expected ({self.dim},)")
        object.__setattr__(self, "x0", x0)

    def native(self) -> "N.OdxProblem":
        """The ABI descriptor (raises ValueError without a device functor)."""
        if self.device is None:
            raise ValueError(
                f"problem {self.name!r} has no device functor; the B200 solver needs one "
                f"(OdeProblem(..., device=(problem_id, params)))")
        pid, params = self.device
        return N.make_problem(pid, self.dim, params)


def _make(name, dim, f_into, jac_into, x0, t0, tf, device, stiff=False) -> OdeProblem:
    def f(x):
        out = np.empty(dim)
        f_into(np.asarray(x, dtype=np.float64), out)
        return out

    def jac_f(x):
        out = np.empty((dim, dim))
        jac_into(np.asarray(x, dtype=np.float64), out)
        return out

    return OdeProblem(name=name, dim=dim, f=f, jac_f=jac_f, x0=np.asarray(x0, np.float64),
                      t0=float(t0), tf=float(tf), stiff=stiff, f_into=f_into,
                      jac_into=jac_into, device=device)


# --- logistic: dP/dt = r P (1 - P/K), problems.py:85-114 --------------------

def logistic(r: float = 1.0, K: float = 1.0, x0=(0.1,), t0=0.0, tf=10.0) -> OdeProblem:
    """Logistic growth, P(0) = 0.1 on [0, 10] by default."""
    def f_into(x, out):
        out[0] = r * x[0] * (1.0 - x[0] / K)

    def jac_into(x, out):
        out[0, 0] = r * (1.0 - 2.0 * x[0] / K)
    return _make("logistic", 1, f_into, jac_into, x0, t0, tf, (N.PROB_LOGISTIC, (r, K)))


# --- van der Pol, problems.py:117-147 ----------------------------------------

def van_der_pol(mu: float = 1.0, x0=(0.0, 1.0), t0=0.0, tf=10.0) -> OdeProblem:
    """van der Pol oscillator, state (x, dx/dt); defaults are the reference's."""
    def f_into(x, out):
        out[0] = x[1]
        out[1] = mu * (1.0 - x[0] * x[0]) * x[1] - x[0]

    def jac_into(x, out):
        out[0, 0] = 0.0
        out[0, 1] = 1.0
        out[1, 0] = -2.0 * mu * x[0] * x[1] - 1.0
        out[1, 1] = mu * (1.0 - x[0] * x[0])
    return _make("vdp", 2, f_into, jac_into, x0, t0, tf, (N.PROB_VDP, (mu,)),
                 stiff=mu >= 10.0)


# --- cart-pole, problems.py:150-242 ------------------------------------------

_CP = (9.81, 0.5, 10.0, 1.0)  # g, l, m_c, m_p


def cart_pole(centripetal_term: bool = False) -> OdeProblem:
    """Unactuated cart-pole released horizontally, t in [0, 4]."""
    G, L, MC, MP = _CP

    def f_into(x, out):
        s, c, w = math.sin(x[2]), math.cos(x[2]), x[3]
        den = MC + MP * s * s
        out[0] = x[1]
        if centripetal_term:
            out[1] = MP * s * (L * w * w + G * c) / den
        else:
            out[1] = MP * s * (L * w + G * c) / den
        out[2] = w
        out[3] = (-MP * L * w * w * c * s - (MC + MP) * G * s) / (L * den)

    def jac_into(x, out):
        s, c, w = math.sin(x[2]), math.cos(x[2]), x[3]
        den = MC + MP * s * s
        dden = 2.0 * MP * s * c
        out[:, :] = 0.0
        out[0, 1] = 1.0
        out[2, 3] = 1.0
        if centripetal_term:
            num1 = MP * s * (L * w * w + G * c)
            dnum1 = MP * c * (L * w * w + G * c) + MP * s * (-G * s)
            out[1, 3] = 2.0 * MP * s * L * w / den
        else:
            num1 = MP * s * (L * w + G * c)
            dnum1 = MP * c * (L * w + G * c) + MP * s * (-G * s)
            out[1, 3] = MP * s * L / den
        out[1, 2] = dnum1 / den - num1 * dden / (den * den)
        num3 = -MP * L * w * w * c * s - (MC + MP) * G * s
        dnum3 = -MP * L * w * w * (c * c - s * s) - (MC + MP) * G * c
        out[3, 2] = dnum3 / (L * den) - num3 * dden / (L * den * den)
        out[3, 3] = -2.0 * MP * L * w * c * s / (L * den)
    pid = N.PROB_CARTPOLE_SQ if centripetal_term else N.PROB_CARTPOLE
    return _make("cartpole", 4, f_into, jac_into, (0.0, 0.0, math.pi / 2.0, 0.0), 0.0, 4.0,
                 (pid, _CP))


# --- Dahlquist, problems.py:245-272 -------------------------------------------

def dahlquist(lam: float = -1000.0) -> OdeProblem:
    """Stiff scalar test equation, y(0) = 1 on [0, 4]."""
    def f_into(x, out):
        out[0] = lam * x[0]

    def jac_into(x, out):
        out[0, 0] = lam
    return _make("dahlquist", 1, f_into, jac_into, (1.0,), 0.0, 4.0,
                 (N.PROB_DAHLQUIST, (lam,)), stiff=True)


# --- Robertson, problems.py:275-318 -------------------------------------------

_ROB = (0.04, 3.0e7, 1.0e4)


def robertson() -> OdeProblem:
    """Robertson's three-species reaction, y(0) = (1, 0, 0) on [0, 500]."""
    k1, k2, k3 = _ROB

    def f_into(x, out):
        out[0] = -k1 * x[0] + k3 * x[1] * x[2]
        out[1] = k1 * x[0] - k2 * x[1] * x[1] - k3 * x[1] * x[2]
        out[2] = k2 * x[1] * x[1]

    def jac_into(x, out):
        out[0, 0] = -k1
        out[0, 1] = k3 * x[2]
        out[0, 2] = k3 * x[1]
        out[1, 0] = k1
        out[1, 1] = -2.0 * k2 * x[1] - k3 * x[2]
        out[1, 2] = -k3 * x[1]
        out[2, 0] = 0.0
        out[2, 1] = 2.0 * k2 * x[1]
        out[2, 2] = 0.0
    return _make("robertson", 3, f_into, jac_into, (1.0, 0.0, 0.0), 0.0, 500.0,
                 (N.PROB_ROBERTSON, _ROB), stiff=True)


# --- BASELINE problems ---------------------------------------------------------

def lorenz63(sigma: float = 10.0, rho: float = 28.0, beta: float = 8.0 / 3.0,
             x0=(1.0, 1.0, 1.0), t0=0.0, tf=10.24) -> OdeProblem:
    """Lorenz-63 (BASELINE cfg 1/3)."""
    def f_into(x, out):
        out[0] = sigma * (x[1] - x[0])
        out[1] = x[0] * (rho - x[2]) - x[1]
        out[2] = x[0] * x[1] - beta * x[2]

    def jac_into(x, out):
        out[0, 0] = -sigma
        out[0, 1] = sigma
        out[0, 2] = 0.0
        out[1, 0] = rho - x[2]
        out[1, 1] = -1.0
        out[1, 2] = -x[0]
        out[2, 0] = x[1]
        out[2, 1] = x[0]
        out[2, 2] = -beta
    return _make("lorenz63", 3, f_into, jac_into, x0, t0, tf,
                 (N.PROB_LORENZ63, (sigma, rho, beta)))


def allen_cahn(n: int = 64, eps: float = 0.01, dx: float | None = None, u0=None, t0=0.0,
               tf=65.536) -> OdeProblem:
    """Allen-Cahn u_t = eps u_xx + u - u^3 on n periodic points (BASELINE cfg 4)."""
    dx = 1.0 / n if dx is None else float(dx)
    if u0 is None:
        u0 = 0.1 * np.sin(2.0 * math.pi * np.arange(n) / n)

    def f_into(x, out):
        cdiff = eps / (dx * dx)
        um = np.roll(x, 1)
        up = np.roll(x, -1)
        out[:] = cdiff * ((um - 2.0 * x) + up) + (x - x * x * x)

    def jac_into(x, out):
        cdiff = eps / (dx * dx)
        out[:, :] = 0.0
        for i in range(n):
            out[i, i] = -2.0 * cdiff + (1.0 - 3.0 * (x[i] * x[i]))
            out[i, (i + n - 1) % n] += cdiff
            out[i, (i + 1) % n] += cdiff
    return _make("allen_cahn", n, f_into, jac_into, u0, t0, tf,
                 (N.PROB_ALLEN_CAHN, (eps, dx)), stiff=True)


# --- problems the reference's tests define (tests/test_newton_pint.py:28-68) ---

def exp_growth(x0=(0.0,), t0=0.0, tf=1.0) -> OdeProblem:
    """dy/dt = exp(y): overflows fast (divergence-path checks)."""
    def f_into(x, out):
        out[0] = math.exp(x[0]) if x[0] < 709.0 else math.inf

    def jac_into(x, out):
        out[0, 0] = math.exp(x[0]) if x[0] < 709.0 else math.inf
    return _make("exp_growth", 1, f_into, jac_into, x0, t0, tf, (N.PROB_EXP_GROWTH, ()))


def square(x0=(1.0,), t0=0.0, tf=1.0) -> OdeProblem:
    """dy/dt = y^2 (singular backward-Euler block at y = 1/(2 dt))."""
    def f_into(x, out):
        out[0] = x[0] * x[0]

    def jac_into(x, out):
        out[0, 0] = 2.0 * x[0]
    return _make("square", 1, f_into, jac_into, x0, t0, tf, (N.PROB_SQUARE, ()))


def linear(A, x0, t0=0.0, tf=1.0) -> OdeProblem:
    """dx/dt = A x (dim <= 4 on the device)."""
    A = np.asarray(A, np.float64)
    d = A.shape[0]

    def f_into(x, out):
        out[:] = A @ x

    def jac_into(x, out):
        out[:, :] = A
    return _make("linear", d, f_into, jac_into, x0, t0, tf, (N.PROB_LINEAR, tuple(A.ravel())))


_FACTORIES = {
    "logistic": logistic,
    "vdp": van_der_pol,
    "cartpole": cart_pole,
    "dahlquist": dahlquist,
    "robertson": robertson,
}
_EXTRA = {"lorenz63": lorenz63, "allen_cahn": allen_cahn}

PROBLEM_NAMES = tuple(sorted(_FACTORIES))
EXTRA_PROBLEM_NAMES = tuple(sorted(_EXTRA))


def get_problem(name: str) -> OdeProblem:
    """Look a benchmark problem up by its CLI name (problems.py:342-350)."""
    factory = _FACTORIES.get(name) or _EXTRA.get(name)
    if factory is None:
        raise ValueError(
            f"unknown problem {name!r}; available: {', '.join(PROBLEM_NAMES)}")
    return factory()
