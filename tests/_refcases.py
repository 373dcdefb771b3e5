"""Reference problem constants used by the parity tests.

Values restate /root/reference/pkg/src/odescan/problems.py (constants at
:85-86, :117, :155-158, :245, :275-277 and the factories' x0 / [t0, tf]).
"""

import math

import numpy as np

# name -> (problem id (ODX_PROB_*), dim, params, x0, t0, tf)
REF_PROBLEMS = {
    "logistic": (0, 1, (1.0, 1.0), np.array([0.1]), 0.0, 10.0),
    "vdp": (1, 2, (1.0,), np.array([0.0, 1.0]), 0.0, 10.0),
    "cartpole": (2, 4, (9.81, 0.5, 10.0, 1.0), np.array([0.0, 0.0, math.pi / 2.0, 0.0]), 0.0, 4.0),
    "cartpole_sq": (3, 4, (9.81, 0.5, 10.0, 1.0), np.array([0.0, 0.0, math.pi / 2.0, 0.0]), 0.0, 4.0),
    "dahlquist": (4, 1, (-1000.0,), np.array([1.0]), 0.0, 4.0),
    "robertson": (5, 3, (0.04, 3.0e7, 1.0e4), np.array([1.0, 0.0, 0.0]), 0.0, 500.0),
}

# golden build specs (tests/golden/make_golden.py kernels_golden order)
BUILD_SPECS = {
    "logistic": (0, 1, (1.0, 1.0)),
    "vdp": (1, 2, (1.0,)),
    "cartpole": (2, 4, (9.81, 0.5, 10.0, 1.0)),
    "dahlquist": (4, 1, (-1000.0,)),
    "robertson": (5, 3, (0.04, 3.0e7, 1.0e4)),
    "cartpole_sq": (3, 4, (9.81, 0.5, 10.0, 1.0)),
    "lorenz63": (6, 3, (10.0, 28.0, 8.0 / 3.0)),
    "vdp10": (1, 2, (10.0,)),
    "allen_cahn": (7, 64, (0.01, 1.0 / 64.0)),
}


def n_steps(t0, tf, dt):
    return int(round((tf - t0) / dt))


def guess_array(policy, x0, n):
    d = x0.shape[0]
    if policy == "ones":
        return np.ones((n, d))
    if policy == "zeros":
        return np.zeros((n, d))
    if policy == "replicate_x0":
        return np.tile(x0, (n, 1))
    raise ValueError(policy)
