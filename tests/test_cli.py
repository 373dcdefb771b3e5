"""The odescan-compatible CLI: usage errors on the CPU,
solve / residuals / bench CSVs on the GPU (reference: cli_bench.py and its
tests, tests/test_cli_bench.py)."""

import numpy as np
import pytest


def _main(argv):
    from paper_2511_01465_b200.cli_bench import main
    return main(argv)


@pytest.mark.parametrize("argv", [
    ["solve", "--problem", "nope", "--stepper", "rk4", "--dt", "0.01", "--out", "x.csv"],
    ["solve", "--problem", "vdp", "--stepper", "nope", "--dt", "0.01", "--out", "x.csv"],
    ["solve", "--problem", "vdp", "--method", "nope", "--stepper", "rk4", "--dt", "0.01",
     "--out", "x.csv"],
    ["bench", "--problem", "vdp", "--stepper", "rk4", "--dt", "0.01,abc", "--out", "x.csv"],
    ["solve", "--problem", "vdp", "--stepper", "rk4", "--dt", "0.01", "--guess", "no_such_file",
     "--out", "x.csv"],
    ["solve", "--problem", "vdp", "--stepper", "rk4", "--dt", "0.01", "--threads", "0",
     "--out", "x.csv"],
    ["solve", "--problem", "robertson", "--method", "parareal", "--stepper", "rk4", "--dt",
     "0.001", "--out", "x.csv"],
    ["solve", "--problem", "vdp"],
])
def test_usage_errors_exit_2(argv, tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    assert _main(argv) == 2


@pytest.mark.gpu
def test_cli_solve_residuals_bench(tmp_path):
    import paper_2511_01465_b200 as pkg
    out = tmp_path / "traj.csv"
    argv = ["solve", "--problem", "vdp", "--stepper", "rk4", "--dt", "0.01", "--iters", "5",
            "--out", str(out)]
    assert _main(argv) == 0
    text = out.read_text()
    lines = text.splitlines()
    p = pkg.get_problem("vdp")
    n = pkg.n_steps_for(p, 0.01)
    assert lines[0] == "t,x_0,x_1" and len(lines) == n + 2
    data = np.genfromtxt(str(out), delimiter=",", skip_header=1)
    rep = pkg.solve(p, pkg.get_stepper("rk4", p), 0.01, "ones", pkg.NewtonConfig(max_iters=5))
    assert np.array_equal(data[1:, 1:], np.asarray(rep.trajectory.states))
    out2 = tmp_path / "traj2.csv"
    assert _main(argv[:-1] + [str(out2)]) == 0
    assert out2.read_text() == text  # byte-for-byte reproducible
    res = tmp_path / "res.csv"
    assert _main(["residuals", "--problem", "vdp", "--stepper", "rk4", "--dt", "0.01",
                  "--iters", "5", "--out", str(res)]) == 0
    r = res.read_text().splitlines()
    assert r[0] == "iteration,residual_inf_norm" and len(r) == 1 + 6
    assert float(r[1].split(",")[1]) == rep.residual_history[0]
    bench = tmp_path / "bench.csv"
    assert _main(["bench", "--problem", "logistic", "--method", "parallel_newton,sequential,parareal",
                  "--stepper", "rk4", "--dt", "0.01,0.005", "--reps", "2", "--warmup", "1",
                  "--out", str(bench)]) == 0
    rows = bench.read_text().splitlines()
    assert len(rows) == 1 + 3 * 2
    assert rows[0].startswith("problem,method,stepper,dt,n_states")
    for row in rows[1:]:
        f = row.split(",")
        assert float(f[7]) < 1e-6 or f[1] == "parareal"  # converged residuals


@pytest.mark.gpu
def test_cli_guess_file_and_solver_error(tmp_path):
    out = tmp_path / "g.csv"
    assert _main(["solve", "--problem", "logistic", "--stepper", "rk4", "--dt", "0.01",
                  "--iters", "8", "--out", str(out)]) == 0
    out2 = tmp_path / "g2.csv"
    assert _main(["solve", "--problem", "logistic", "--stepper", "rk4", "--dt", "0.01",
                  "--iters", "2", "--guess", str(out), "--out", str(out2)]) == 0
    # cart-pole from the constant guess diverges: NonFiniteError -> exit 1
    assert _main(["solve", "--problem", "cartpole", "--stepper", "rk4", "--dt", "0.001",
                  "--iters", "11", "--out", str(tmp_path / "c.csv")]) in (0, 1)
