"""CPU tests of the host-side drop-in surface the reference exports beside solve():
linalg_small (linalg_small.py:29-118), threads (threads.py:17-32), the
list-based Newton-step / dense-Jacobian functions (newton_pint.py:214-312,
tests/test_newton_pint.py:197-236 pattern) and the export list itself
(pkg/src/odescan/__init__.py:68-118)."""

import numpy as np
import pytest

from conftest import assert_bitwise

# the reference's public names (pkg/src/odescan/__init__.py:68-118)
REFERENCE_ALL = [
    "AffineElement", "combine", "identity", "init_elements", "scan_parallel", "scan_sequential",
    "extract_states", "InnerNewtonFailedError", "PararealConfig", "PararealResult",
    "solve_parareal", "solve_sequential_explicit", "solve_sequential_implicit",
    "SingularMatrixError", "inf_norm", "lu_solve", "mat_mul", "mat_vec", "GUESS_POLICIES",
    "NewtonConfig", "NonFiniteError", "SingularDiagonalBlockError", "SolveReport", "Trajectory",
    "initial_guess", "n_steps_for", "solve", "PROBLEM_NAMES", "OdeProblem", "cart_pole",
    "dahlquist", "get_problem", "logistic", "robertson", "van_der_pol", "EULER_TABLEAU",
    "RK4_TABLEAU", "STEPPER_NAMES", "ButcherTableau", "StepperIncrement", "explicit_euler",
    "explicit_rk", "get_stepper", "implicit_euler", "trapezoidal", "hardware_threads",
    "max_threads", "set_threads", "__version__",
]


def test_every_reference_export_present():
    import paper_2511_01465_b200 as od
    missing = [n for n in REFERENCE_ALL if not hasattr(od, n)]
    assert not missing, missing
    assert set(REFERENCE_ALL) <= set(od.__all__)


def test_lu_bit_identical_to_reference_goldens(golden_kernels):
    from paper_2511_01465_b200.linalg_small import _lu_solve_vec, lu_factor
    g = golden_kernels
    for i in range(6):
        lu, piv, st = lu_factor(g[f"lu{i}_A"])
        assert st == int(g[f"lu{i}_status"])
        if st < 0:
            assert_bitwise(lu, g[f"lu{i}_LU"], f"LU {i}")
            assert np.array_equal(piv, g[f"lu{i}_piv"])
            assert_bitwise(_lu_solve_vec(lu, piv, g[f"lu{i}_b"].copy()), g[f"lu{i}_x"], f"x {i}")


def test_lu_solve_api():
    import paper_2511_01465_b200 as od
    rng = np.random.default_rng(3)
    A = rng.standard_normal((5, 5)) + 5 * np.eye(5)
    b = rng.standard_normal(5)
    B = rng.standard_normal((5, 3))
    np.testing.assert_allclose(od.lu_solve(A, b), np.linalg.solve(A, b), rtol=1e-12)
    X = od.lu_solve(A, B)
    assert X.shape == B.shape
    np.testing.assert_allclose(X, np.linalg.solve(A, B), rtol=1e-12)
    S = np.array([[1.0, 2.0], [2.0, 4.0]])
    with pytest.raises(od.SingularMatrixError) as ei:
        od.lu_solve(S, np.ones(2))
    assert ei.value.pivot_index == 1
    with pytest.raises(od.SingularMatrixError) as ei:
        od.lu_solve(np.zeros((3, 3)), np.ones(3))
    assert ei.value.pivot_index == 0
    for bad in (np.ones((2, 3)), np.ones(3), np.zeros((0, 0))):
        with pytest.raises(ValueError):
            od.lu_solve(bad, np.ones(2))
    with pytest.raises(ValueError):
        od.lu_solve(np.eye(2), np.ones(3))
    with pytest.raises(ValueError):
        od.mat_mul(np.ones((2, 3)), np.ones((2, 3)))
    with pytest.raises(ValueError):
        od.mat_vec(np.ones((2, 3)), np.ones(2))
    np.testing.assert_array_equal(od.mat_vec(np.eye(2), [1.0, 2.0]), [1.0, 2.0])
    assert od.inf_norm([[1.0, -3.0], [2.0, 0.5]]) == 3.0
    with pytest.raises(ValueError):
        od.inf_norm([])


def test_threads_contract():
    import paper_2511_01465_b200 as od
    m = od.max_threads()
    assert m >= 1
    assert od.hardware_threads() >= 1
    assert od.set_threads(0) == 1
    assert od.set_threads(10 ** 6) == m
    assert od.set_threads(1) == 1
    od.set_threads(m)


@pytest.mark.parametrize("n", [2, 5, 50])
def test_newton_step_explicit_vs_dense(n):
    """tests/test_newton_pint.py:199-211 (criterion 2): scan step == -H^-1 h."""
    import paper_2511_01465_b200 as od
    p = od.get_problem("logistic")
    st = od.get_stepper("rk4", p)
    rng = np.random.default_rng(n)
    traj = od.Trajectory(p.x0.copy(), 0.5 + 0.2 * rng.standard_normal((n, 1)),
                         (p.tf - p.t0) / n, n)
    h = od.residual_explicit(traj, st)
    u_scan = np.concatenate(od.newton_step_explicit(traj, h, st))
    H = od.dense_jacobian_explicit(traj, st)
    u_dense = np.linalg.solve(H, -np.concatenate(h))
    np.testing.assert_allclose(u_scan, u_dense, rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("n", [2, 5, 50])
def test_newton_step_implicit_vs_dense(n):
    import paper_2511_01465_b200 as od
    p = od.get_problem("dahlquist")
    st = od.get_stepper("backward_euler", p)
    rng = np.random.default_rng(100 + n)
    traj = od.Trajectory(p.x0.copy(), rng.standard_normal((n, 1)), (p.tf - p.t0) / n, n)
    h = od.residual_implicit(traj, st)
    u_scan = np.concatenate(od.newton_step_implicit(traj, h, st))
    H = od.dense_jacobian_implicit(traj, st)
    np.testing.assert_allclose(u_scan, np.linalg.solve(H, -np.concatenate(h)), rtol=1e-9,
                               atol=1e-9)


def test_newton_step_errors():
    import paper_2511_01465_b200 as od
    p = od.get_problem("logistic")
    traj = od.initial_guess("ones", p, 4)
    with pytest.raises(ValueError):
        od.residual_explicit(traj, od.get_stepper("backward_euler", p))
    with pytest.raises(ValueError):
        od.residual_implicit(traj, od.get_stepper("rk4", p))
    sq = od.problems.square()
    st = od.get_stepper("backward_euler", sq)
    traj = od.Trajectory(sq.x0.copy(), np.full((10, 1), 5.0), 0.1, 10)
    with pytest.raises(od.SingularDiagonalBlockError) as ei:
        od.newton_step_implicit(traj, od.residual_implicit(traj, st), st)
    assert ei.value.block_index == 0
