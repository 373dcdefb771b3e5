"""Host-side API of the drop-in package (no GPU): types, validation and
conventions mirrored from /root/reference/pkg/src/odescan (newton_pint.py,
problems.py, steppers.py, affine_scan.py) — the reference's own unit tests
for these, restated."""

import math

import numpy as np
import pytest

import paper_2511_01465_b200 as od
from conftest import central_diff_jacobian


def test_public_names():
    for name in ("solve", "NewtonConfig", "SolveReport", "Trajectory", "NonFiniteError",
                 "SingularDiagonalBlockError", "get_problem", "get_stepper", "OdeProblem",
                 "initial_guess", "n_steps_for", "GUESS_POLICIES", "RK4_TABLEAU",
                 "AffineElement", "combine", "scan_parallel", "scan_sequential"):
        assert hasattr(od, name)
    assert od.PROBLEM_NAMES == ("cartpole", "dahlquist", "logistic", "robertson", "vdp")
    assert od.STEPPER_NAMES == ("backward_euler", "euler", "rk4", "trapezoidal")
    assert od.GUESS_POLICIES == ("ones", "zeros", "replicate_x0", "coarse_euler")


def test_n_steps_for():
    assert od.n_steps_for(od.get_problem("logistic"), 1e-2) == 1000
    assert od.n_steps_for(od.get_problem("dahlquist"), 0.1) == 40
    with pytest.raises(ValueError):
        od.n_steps_for(od.get_problem("logistic"), 0.3)
    with pytest.raises(ValueError):
        od.n_steps_for(od.get_problem("logistic"), 0.0)


def test_trajectory_and_config_validation():
    t = od.Trajectory(np.array([1.0]), np.array([[2.0], [3.0]]), 0.5, 2)
    np.testing.assert_array_equal(t.full_states()[:, 0], [1.0, 2.0, 3.0])
    with pytest.raises(ValueError):
        od.Trajectory(np.array([1.0]), np.ones((2, 2)), 0.5, 2)
    with pytest.raises(ValueError):
        od.Trajectory(np.array([1.0]), np.ones((2, 1)), 0.5, 3)
    with pytest.raises(ValueError):
        od.NewtonConfig(max_iters=0)
    with pytest.raises(ValueError):
        od.NewtonConfig(max_iters=1, residual_tol=-1.0)
    with pytest.raises(ValueError):
        od.NewtonConfig(max_iters=1, step_tol=-1.0)


def test_initial_guess_policies():
    p = od.get_problem("vdp")
    np.testing.assert_array_equal(od.initial_guess("ones", p, 4).states, np.ones((4, 2)))
    np.testing.assert_array_equal(od.initial_guess("replicate_x0", p, 3).states,
                                  np.tile(p.x0, (3, 1)))
    q = od.get_problem("logistic")
    g = od.initial_guess("coarse_euler", q, 250)  # stride 2
    v = q.x0.copy()
    for k in range(0, 250, 2):
        v = v + 2 * (10.0 / 250) * q.f(v)
        np.testing.assert_allclose(g.states[k], v, rtol=1e-14)
    with pytest.raises(ValueError):
        od.initial_guess("interpolate", q, 10)


@pytest.mark.parametrize("name", ["logistic", "vdp", "cartpole", "dahlquist", "robertson",
                                  "lorenz63", "allen_cahn"])
def test_host_jacobians_match_central_differences(name):
    p = od.get_problem(name)
    rng = np.random.default_rng(3)
    x = p.x0 + 0.1 * rng.standard_normal(p.dim)
    J = p.jac_f(x)
    np.testing.assert_allclose(J, central_diff_jacobian(p.f, x), rtol=1e-5,
                               atol=1e-6 * max(1.0, np.abs(J).max()))


def test_solve_validation_before_any_gpu_work():
    p1, p2 = od.get_problem("logistic"), od.get_problem("vdp")
    with pytest.raises(ValueError):
        od.solve(p1, od.get_stepper("rk4", p2), 0.1, "ones", od.NewtonConfig(max_iters=1))
    nodev = od.OdeProblem(name="custom", dim=1, f=lambda x: x, jac_f=lambda x: np.ones((1, 1)),
                          x0=np.array([1.0]), t0=0.0, tf=1.0)
    with pytest.raises(ValueError, match="device functor"):
        od.solve(nodev, od.get_stepper("euler", nodev), 0.1)


def test_affine_scan_algebra():
    rng = np.random.default_rng(17)
    els = [od.AffineElement(rng.standard_normal((3, 3)), rng.standard_normal(3)) for _ in range(9)]
    seq = od.scan_sequential(els)
    par = od.scan_parallel(els)
    for a, b in zip(seq, par):
        np.testing.assert_allclose(a.F, b.F, rtol=1e-10, atol=1e-10)
        np.testing.assert_allclose(a.c, b.c, rtol=1e-10, atol=1e-10)
    e1, e2 = els[0], els[1]
    z = rng.standard_normal(3)
    c = od.combine(e1, e2)
    np.testing.assert_allclose(c.F @ z + c.c, e2.F @ (e1.F @ z + e1.c) + e2.c, rtol=1e-13)
    with pytest.raises(ValueError):
        od.scan_parallel([])


def test_baseline_configs_inputs():
    from paper_2511_01465_b200.configs import CONFIGS
    assert [CONFIGS[i].n_steps for i in range(1, 6)] == [1024, 65536, 2048, 65536, 2 ** 26]
    x3 = CONFIGS[3].x0s()
    assert x3.shape == (4096, 3)
    rng = np.random.default_rng(0)
    np.testing.assert_array_equal(x3, 1.0 + rng.normal(0.0, 0.5, size=(4096, 3)))
    u0 = CONFIGS[4].x0s()[0]
    assert u0.shape == (64,) and abs(u0[16] - 0.1) < 0.05
    assert math.isclose(CONFIGS[1].params[2], 8.0 / 3.0)


def test_sequential_baselines_validate_without_gpu():
    """baselines.solve_sequential_* reject what the reference rejects
    (baselines.py:64-125) before touching the device."""
    import paper_2511_01465_b200 as pkg
    p = pkg.van_der_pol()
    rk4 = pkg.get_stepper("rk4", p)
    be = pkg.get_stepper("backward_euler", p)
    with pytest.raises(ValueError):
        pkg.solve_sequential_explicit(p, be, 1e-3)
    with pytest.raises(ValueError):
        pkg.solve_sequential_implicit(p, rk4, 1e-3)
    with pytest.raises(ValueError):
        pkg.solve_sequential_implicit(p, be, 1e-3, inner_newton_tol=-1.0)
    with pytest.raises(ValueError):
        pkg.solve_sequential_implicit(p, be, 1e-3, inner_max_iters=0)
    with pytest.raises(ValueError):
        pkg.solve_sequential_explicit(p, rk4, 1e-3, n_steps=-1)
    other = pkg.van_der_pol()
    with pytest.raises(ValueError):
        pkg.solve_sequential_explicit(other, rk4, 1e-3)
    t = pkg.solve_sequential_explicit(p, rk4, 1e-3, n_steps=0)
    assert t.states.shape == (0, 2)
