"""The five BASELINE.json workloads, with seeded synthetic inputs.

BASELINE.json fixes the problems, step maps, sizes and stop rules; it leaves
the seeds open, so every config draws from a fresh numpy default_rng(0) in the
order written in SURVEY.md §8(d).  None of these ODEs ships with the reference
(SURVEY F4); they are added through its plug-in type (OdeProblem) exactly the
way its tests add custom problems (tests/test_newton_pint.py:28-68).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class BaselineConfig:
    cid: int
    name: str
    problem: str          # registry name in problems.py
    params: tuple         # problem parameters (device functor arguments)
    dim: int
    stepper: str          # steppers.py registry name
    dt: float
    n_steps: int
    batch: int = 1
    max_iters: int = 100
    step_tol: float = 1e-10
    abort_nonfinite: bool = True
    oracle_n_steps: int | None = None   # CPU-oracle size when full N is too big
    notes: str = ""

    def x0s(self) -> np.ndarray:
        """(batch, dim) initial conditions, seeded per SURVEY §8(d)."""
        rng = np.random.default_rng(0)
        if self.cid == 1:
            return np.array([[1.0, 1.0, 1.0]])
        if self.cid == 2:
            return np.array([[2.0, 0.0]])
        if self.cid == 3:
            return np.array([1.0, 1.0, 1.0]) + rng.normal(0.0, 0.5, size=(self.batch, 3))
        if self.cid == 4:
            i = np.arange(self.dim)
            u0 = 0.1 * np.sin(2.0 * math.pi * i / self.dim) + rng.normal(0.0, 0.01, self.dim)
            return u0[None, :]
        if self.cid == 5:
            return np.array([[2.0, 0.0]])
        raise ValueError(self.cid)

    def guess(self, n_steps: int | None = None, batch: int | None = None) -> np.ndarray:
        """Constant-x0 initial guess (replicate_x0, newton_pint.py:189-190): (B, N, d)."""
        n = self.n_steps if n_steps is None else n_steps
        x0 = self.x0s()
        if batch is not None:
            x0 = x0[:batch]
        return np.ascontiguousarray(np.repeat(x0[:, None, :], n, axis=1))


LORENZ = (10.0, 28.0, 8.0 / 3.0)

CONFIGS = {
    1: BaselineConfig(1, "cfg1_lorenz63_rk4", "lorenz63", LORENZ, 3, "rk4", 0.01, 1024,
                      notes="single trajectory, the reference's CPU-runnable case"),
    2: BaselineConfig(2, "cfg2_vdp_mu10_backward_euler", "vdp", (10.0,), 2, "backward_euler",
                      1e-3, 65536),
    3: BaselineConfig(3, "cfg3_lorenz63_batch4096_rk4", "lorenz63", LORENZ, 3, "rk4", 0.01,
                      2048, batch=4096),
    4: BaselineConfig(4, "cfg4_allen_cahn64_backward_euler", "allen_cahn", (0.01, 1.0 / 64.0),
                      64, "backward_euler", 1e-3, 65536, oracle_n_steps=4096),
    5: BaselineConfig(5, "cfg5_vdp_mu1_rk4_fixed10", "vdp", (1.0,), 2, "rk4", 1e-3, 2 ** 26,
                      max_iters=10, step_tol=0.0, abort_nonfinite=False,
                      oracle_n_steps=2 ** 22),
}


def get_config(cid: int) -> BaselineConfig:
    return CONFIGS[int(cid)]
