"""Pin the CPU oracle (oracle/odescan_oracle.c) to the reference itself.

Every fixture in tests/golden/*.npz was produced by the reference package's
own numba kernels and solve() (tests/golden/make_golden.py).  The oracle must
reproduce them BIT FOR BIT — including NaN placement and signed zeros — which
is what licenses it as the parity checker for the CUDA path.
"""

import numpy as np
import pytest

from conftest import assert_bitwise
from _refcases import BUILD_SPECS, REF_PROBLEMS, guess_array, n_steps


def test_scan_affine_reference_sizes(oracle, golden_kernels):
    g = golden_kernels
    for n in (1, 2, 5, 33, 256):
        Fp, cp = oracle.scan_affine(g[f"scan_n{n}_F"], g[f"scan_n{n}_c"])
        assert_bitwise(Fp, g[f"scan_n{n}_Fp"], f"Fp n={n}")
        assert_bitwise(cp, g[f"scan_n{n}_cp"], f"cp n={n}")


@pytest.mark.parametrize("d", [1, 2, 4])
def test_scan_affine_dims(oracle, golden_kernels, d):
    g = golden_kernels
    Fp, cp = oracle.scan_affine(g[f"scand{d}_F"], g[f"scand{d}_c"])
    assert_bitwise(Fp, g[f"scand{d}_Fp"], "Fp")
    assert_bitwise(cp, g[f"scand{d}_cp"], "cp")


def test_scan_affine_nonfinite(oracle, golden_kernels):
    g = golden_kernels
    Fp, cp = oracle.scan_affine(g["scannf_F"], g["scannf_c"])
    assert_bitwise(Fp, g["scannf_Fp"], "Fp")
    assert_bitwise(cp, g["scannf_cp"], "cp")


def test_max_abs_nan_semantics(oracle, golden_kernels):
    g = golden_kernels
    i = 0
    while f"maxabs{i}_A" in g:
        assert_bitwise(oracle.max_abs(g[f"maxabs{i}_A"]), g[f"maxabs{i}_out"], f"case {i}")
        i += 1
    assert i >= 8


def test_max_abs_thread_independent(oracle, golden_kernels):
    A = golden_kernels["maxabs6_A"]
    ref = golden_kernels["maxabs6_out"]
    for t in (1, 3, 8):
        oracle.set_threads(t)
        assert_bitwise(oracle.max_abs(A), ref, f"threads={t}")
    oracle.set_threads(8)


def test_lu(oracle, golden_kernels):
    g = golden_kernels
    for i in range(6):
        A = g[f"lu{i}_A"].copy()
        d = A.shape[0]
        piv = np.zeros(d, np.int64)
        st = oracle.lib().orc_lu_factor(A, piv, d)
        assert st == int(g[f"lu{i}_status"])
        if st < 0:
            assert_bitwise(A, g[f"lu{i}_LU"], f"LU {i}")
            assert np.array_equal(piv, g[f"lu{i}_piv"])
            x = g[f"lu{i}_b"].copy()
            oracle.lib().orc_lu_solve(A, piv, x, d)
            assert_bitwise(x, g[f"lu{i}_x"], f"x {i}")


@pytest.mark.parametrize("name", list(BUILD_SPECS))
def test_build_explicit(oracle, golden_kernels, name):
    g = golden_kernels
    pid, d, params = BUILD_SPECS[name]
    for sname, (a, b) in (("rk4", (oracle.RK4_A, oracle.RK4_B)),
                          ("euler", (oracle.EULER_A, oracle.EULER_B))):
        key = f"bx_{name}_{sname}"
        Fe, ce, h = oracle.build_explicit(pid, params, a, b, g[key + "_x0"], g[key + "_X"],
                                          float(g[key + "_dt"]))
        assert_bitwise(h, g[key + "_h"], key + " h")
        assert_bitwise(ce, g[key + "_ce"], key + " ce")
        assert_bitwise(Fe, g[key + "_Fe"], key + " Fe")


@pytest.mark.parametrize("name", list(BUILD_SPECS))
def test_build_implicit(oracle, golden_kernels, name):
    g = golden_kernels
    pid, d, params = BUILD_SPECS[name]
    for sname, (wp, wn) in (("be", (0.0, 1.0)), ("trap", (0.5, 0.5))):
        key = f"bi_{name}_{sname}"
        Fe, ce, h, bad = oracle.build_implicit(pid, params, wp, wn, g[key + "_x0"],
                                               g[key + "_X"], float(g[key + "_dt"]))
        assert bad == int(g[key + "_bad"])
        assert_bitwise(h, g[key + "_h"], key + " h")
        assert_bitwise(ce, g[key + "_ce"], key + " ce")
        assert_bitwise(Fe, g[key + "_Fe"], key + " Fe")


def test_build_implicit_zero_weight_nan_leak(oracle, golden_kernels):
    """backward Euler still evaluates f/J at prev; inf*0 leaks NaN."""
    g = golden_kernels
    Fe, ce, h, bad = oracle.build_implicit(1, (10.0,), 0.0, 1.0, np.array([2.0, 0.0]),
                                           g["bi_leak_X"], 1e-3)
    assert bad == int(g["bi_leak_bad"])
    assert_bitwise(h, g["bi_leak_h"], "h")
    assert_bitwise(ce, g["bi_leak_ce"], "ce")
    assert_bitwise(Fe, g["bi_leak_Fe"], "Fe")
    assert np.isnan(Fe).any()


def test_build_implicit_singular_block(oracle, golden_kernels):
    g = golden_kernels
    Fe, ce, h, bad = oracle.build_implicit(9, (), 0.0, 1.0, np.array([1.0]), g["bi_sing_X"], 0.1)
    assert bad == int(g["bi_sing_bad"]) == 0
    assert_bitwise(Fe, g["bi_sing_Fe"], "Fe")
    assert_bitwise(ce, g["bi_sing_ce"], "ce")


def test_solve_matches_reference_solve(oracle, golden_solves):
    """The oracle driver with residual_tol=0 is exactly odescan.solve()."""
    g = golden_solves
    i = 0
    while f"solve{i}_meta" in g:
        name, sname, policy = [str(s) for s in g[f"solve{i}_meta"]]
        pid, d, params, x0, t0, tf = REF_PROBLEMS[name]
        dt = float(g[f"solve{i}_dt"])
        n = n_steps(t0, tf, dt)
        r = oracle.solve(pid, params, oracle.stepper_by_name(sname), x0,
                         guess_array(policy, x0, n), dt, int(g[f"solve{i}_iters"]))
        assert r["status"] == oracle.ST_MAXITER
        assert_bitwise(r["hist"], g[f"solve{i}_hist"], f"{name}/{sname} hist")
        assert_bitwise(r["shist"], g[f"solve{i}_shist"], f"{name}/{sname} shist")
        assert_bitwise(r["X"], g[f"solve{i}_X"], f"{name}/{sname} X")
        i += 1
    assert i == 8


def test_solve_residual_rule(oracle, golden_solves):
    g = golden_solves
    pid, d, params, x0, t0, tf = REF_PROBLEMS["logistic"]
    n = n_steps(t0, tf, 0.1)
    r = oracle.solve(pid, params, oracle.stepper_by_name("rk4"), x0, np.ones((n, 1)), 0.1, 20,
                     residual_tol=1e-6)
    assert r["status"] == oracle.ST_CONVERGED
    assert r["iters"] == int(g["rtol_iters"])
    assert_bitwise(r["hist"][: r["iters"] + 1], g["rtol_hist"], "hist")
    assert_bitwise(r["X"], g["rtol_X"], "X")


def test_solve_nonfinite_iteration_zero(oracle):
    """tests/test_newton_pint.py:387-394: exp problem from a guess of 800."""
    r = oracle.solve(8, (), oracle.stepper_by_name("euler"), np.array([0.0]),
                     np.full((4, 1), 800.0), 0.25, 3)
    assert r["status"] == oracle.ST_NONFINITE and r["status_index"] == 0


def test_solve_singular(oracle):
    """tests/test_newton_pint.py:396-404: square problem, BE block 1-2*0.1*5 = 0."""
    r = oracle.solve(9, (), oracle.stepper_by_name("backward_euler"), np.array([1.0]),
                     np.full((10, 1), 5.0), 0.1, 2)
    assert r["status"] == oracle.ST_SINGULAR and r["status_index"] == 0


# ---- BASELINE configs (reference kernels under the BASELINE driver) --------

def _cfg_run(oracle, cfg, n=None, max_iters=None, step_tol=None, abort=None, trace=False,
             batch_index=0):
    from paper_2511_01465_b200.configs import CONFIGS  # noqa: F401  (pure numpy)
    pid = oracle.PROB[cfg.problem]
    x0 = cfg.x0s()[batch_index]
    n = cfg.n_steps if n is None else n
    guess = np.tile(x0, (n, 1))
    return oracle.solve(pid, cfg.params, oracle.stepper_by_name(cfg.stepper), x0, guess, cfg.dt,
                        cfg.max_iters if max_iters is None else max_iters,
                        step_tol=cfg.step_tol if step_tol is None else step_tol,
                        abort_nonfinite=cfg.abort_nonfinite if abort is None else abort,
                        trace=trace)


def test_cfg1(oracle, golden_baseline):
    from paper_2511_01465_b200.configs import CONFIGS
    g = golden_baseline
    r = _cfg_run(oracle, CONFIGS[1], trace=True)
    assert r["status"] == int(g["cfg1_status"]) == oracle.ST_NONFINITE
    assert r["status_index"] == int(g["cfg1_index"]) == 1
    assert_bitwise(r["hist"], g["cfg1_hist"], "hist")
    assert_bitwise(r["trace"][1], g["cfg1_X1"], "iterate 1")
    r = _cfg_run(oracle, CONFIGS[1], max_iters=3, step_tol=0.0, abort=False, trace=True)
    assert_bitwise(r["hist"], g["cfg1_fixed3_hist"], "fixed3 hist")
    assert_bitwise(r["X"], g["cfg1_fixed3_X"], "fixed3 X")
    assert_bitwise(r["trace"][2], g["cfg1_fixed3_X2"], "fixed3 X2")


def test_cfg2(oracle, golden_baseline):
    from paper_2511_01465_b200.configs import CONFIGS
    g = golden_baseline
    r = _cfg_run(oracle, CONFIGS[2], trace=True)
    assert r["status"] == int(g["cfg2_status"]) == oracle.ST_NONFINITE
    assert r["status_index"] == int(g["cfg2_index"]) == 2
    assert_bitwise(r["hist"], g["cfg2_hist"], "hist")
    assert_bitwise(r["shist"], g["cfg2_shist"], "shist")
    assert_bitwise(r["trace"][1][::16], g["cfg2_X1_sub"], "X1")
    assert_bitwise(r["trace"][2][::16], g["cfg2_X2_sub"], "X2")
    r = _cfg_run(oracle, CONFIGS[2], n=4096, max_iters=4, step_tol=0.0, abort=False, trace=True)
    assert_bitwise(r["hist"], g["cfg2s_hist"], "small hist")
    assert_bitwise(r["X"], g["cfg2s_X"], "small X")


def test_cfg3_statuses_subset(oracle, golden_baseline):
    from paper_2511_01465_b200.configs import CONFIGS
    g = golden_baseline
    cfg = CONFIGS[3]
    for b in list(range(4)) + [1000, 4095]:
        r = _cfg_run(oracle, cfg, trace=b < 4, batch_index=b)
        assert r["status"] == int(g["cfg3_status"][b])
        assert r["status_index"] == int(g["cfg3_index"][b])
        assert r["iters"] == int(g["cfg3_iters"][b])
        if b < 4:
            assert_bitwise(r["trace"][1], g[f"cfg3_b{b}_X1"], f"b{b} X1")
            assert_bitwise(r["hist"], g[f"cfg3_b{b}_hist"], f"b{b} hist")
    assert (g["cfg3_status"] == oracle.ST_NONFINITE).all()


def test_cfg4_small(oracle, golden_baseline):
    from paper_2511_01465_b200.configs import CONFIGS
    g = golden_baseline
    r = _cfg_run(oracle, CONFIGS[4], n=512, max_iters=3, step_tol=0.0, abort=False, trace=True)
    assert_bitwise(r["hist"], g["cfg4t_hist"], "hist")
    assert_bitwise(r["trace"][1], g["cfg4t_X1"], "X1")
    assert_bitwise(r["X"], g["cfg4t_X"], "X")


@pytest.mark.slow
def test_cfg4_converges_at_4096(oracle, golden_baseline):
    from paper_2511_01465_b200.configs import CONFIGS
    g = golden_baseline
    r = _cfg_run(oracle, CONFIGS[4], n=4096, trace=False)
    assert r["status"] == int(g["cfg4s_status"]) == oracle.ST_CONVERGED
    assert r["iters"] == int(g["cfg4s_iters"])
    assert_bitwise(r["hist"], g["cfg4s_hist"], "hist")
    assert_bitwise(r["X"][::32], g["cfg4s_X_sub"], "X")


def test_cfg5_small(oracle, golden_baseline):
    from paper_2511_01465_b200.configs import CONFIGS
    g = golden_baseline
    r = _cfg_run(oracle, CONFIGS[5], n=65536, max_iters=10, trace=False)
    assert_bitwise(r["hist"], g["cfg5s_hist"], "hist")
    fin = np.isfinite(r["X"]).all(axis=1)
    assert fin.sum() == int(g["cfg5s_finite_rows"])
    assert_bitwise(r["X"][::64], g["cfg5s_X_sub"], "X")
