"""Golden vectors for the §8(f) rows, produced by the reference itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden_f.py        # writes tests/golden/f_rows.npz

Like make_golden.py it imports a temp copy of the reference package and
records, from the reference's OWN code:
  * scanseq_*  — affine_scan.init_elements / scan_sequential / extract_states
                 (affine_scan.py:84-160) on seeded elements, incl. inf/NaN
  * seqx_*     — baselines.solve_sequential_explicit (baselines.py:63-82)
  * seqi_*     — baselines.solve_sequential_implicit (baselines.py:85-118)
  * par_*      — baselines.solve_parareal (baselines.py:164-227): final
                 nodes, every round's nodes, the fine trajectory
  * cli_*      — the bytes of the reference CLI's output files
                 (cli_bench.py main(): `solve` with methods sequential /
                 parallel_newton / parareal and `residuals`)
Problems are the reference's registry problems (get_problem) plus Lorenz-63
plugged in through OdeProblem like its tests add problems.
"""

from __future__ import annotations

import os
import shutil
import sys
import tempfile
from pathlib import Path

OUT = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")

_tmp = Path(tempfile.mkdtemp(prefix="odescan_ref_f_"))
shutil.copytree(REF_SRC, _tmp / "src")
os.environ.setdefault("NUMBA_CACHE_DIR", str(_tmp / "numba_cache"))
sys.dont_write_bytecode = True
sys.path.insert(0, str(_tmp / "src"))

import numba  # noqa: E402
import numpy as np  # noqa: E402
from numba import njit  # noqa: E402

from odescan import affine_scan as AS  # noqa: E402
from odescan import baselines as BL  # noqa: E402
from odescan import cli_bench  # noqa: E402
from odescan.problems import OdeProblem, get_problem  # noqa: E402
from odescan.steppers import get_stepper  # noqa: E402

VERSIONS = np.array([f"numba={numba.__version__}", f"numpy={np.__version__}",
                     f"python={sys.version.split()[0]}"])


def lorenz_problem():
    sigma, rho, beta = 10.0, 28.0, 8.0 / 3.0

    @njit(cache=False)
    def f_into(x, out):
        out[0] = sigma * (x[1] - x[0])
        out[1] = x[0] * (rho - x[2]) - x[1]
        out[2] = x[0] * x[1] - beta * x[2]

    @njit(cache=False)
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

    def f(x):
        o = np.empty(3)
        f_into(np.asarray(x, np.float64), o)
        return o

    def jac_f(x):
        o = np.empty((3, 3))
        jac_into(np.asarray(x, np.float64), o)
        return o
    return OdeProblem(name="lorenz63", dim=3, x0=np.array([1.0, 1.0, 1.0]), t0=0.0, tf=2.0,
                      f=f, jac_f=jac_f, stiff=False, f_into=f_into, jac_into=jac_into)


def scanseq_golden(g):
    rng = np.random.default_rng(7)
    for d, n in ((1, 257), (2, 1000), (3, 64)):
        F = rng.normal(0.0, 0.6, size=(n, d, d))
        c = rng.normal(size=(n, d))
        if d == 2:  # non-finite entries: NaN / inf must propagate as the fold does
            F[500, 0, 1] = np.inf
            c[700, 1] = np.nan
        z0 = rng.normal(size=d)
        els = AS.init_elements(list(F), list(c), z0)
        states = np.array(AS.extract_states(AS.scan_sequential(els)))
        g[f"scanseq_d{d}_F"], g[f"scanseq_d{d}_c"], g[f"scanseq_d{d}_z0"] = F, c, z0
        g[f"scanseq_d{d}_states"] = states


def sequential_golden(g):
    cases_x = [("logistic", "rk4", 0.01), ("logistic", "euler", 0.05), ("vdp", "rk4", 0.01),
               ("dahlquist", "euler", 0.001), ("cartpole", "rk4", 0.01)]
    for name, sname, dt in cases_x:
        p = get_problem(name)
        st = get_stepper(sname, p)
        tr = BL.solve_sequential_explicit(p, st, dt)
        g[f"seqx_{name}_{sname}"] = tr.states
        g[f"seqx_{name}_{sname}_dt"] = dt
    p = lorenz_problem()
    g["seqx_lorenz63_rk4"] = BL.solve_sequential_explicit(p, get_stepper("rk4", p), 0.01).states
    g["seqx_lorenz63_rk4_dt"] = 0.01
    for name, dt in (("dahlquist", 0.01), ("vdp", 0.01), ("robertson", 0.5)):
        p = get_problem(name)
        tr = BL.solve_sequential_implicit(p, get_stepper("backward_euler", p), dt)
        g[f"seqi_{name}_backward_euler"] = tr.states
        g[f"seqi_{name}_backward_euler_dt"] = dt


def parareal_golden(g):
    for name, m, sub, its in (("logistic", 10, 100, 4), ("vdp", 20, 50, 3)):
        p = get_problem(name)
        st = get_stepper("rk4", p)
        res = BL.solve_parareal(p, st, st, BL.PararealConfig(n_coarse=m, n_iterations=its,
                                                             fine_substeps=sub))
        g[f"par_{name}_nodes"] = res.coarse_nodes
        g[f"par_{name}_history"] = np.stack(res.node_history)
        g[f"par_{name}_states"] = res.trajectory.states
        g[f"par_{name}_cfg"] = np.array([m, sub, its])


CLI_RUNS = {
    "solve_seq_logistic": ["solve", "--problem", "logistic", "--method", "sequential",
                           "--stepper", "rk4", "--dt", "0.01"],
    "solve_seq_vdp_be": ["solve", "--problem", "vdp", "--method", "sequential",
                         "--stepper", "backward_euler", "--dt", "0.01"],
    "solve_newton_logistic": ["solve", "--problem", "logistic", "--method", "parallel_newton",
                              "--stepper", "rk4", "--dt", "0.01", "--iters", "11"],
    "solve_parareal_logistic": ["solve", "--problem", "logistic", "--method", "parareal",
                                "--stepper", "rk4", "--dt", "0.01", "--iters", "4"],
    "residuals_vdp": ["residuals", "--problem", "vdp", "--stepper", "rk4", "--dt", "0.01",
                      "--iters", "11"],
}


def cli_golden(g):
    for key, args in CLI_RUNS.items():
        out = _tmp / f"{key}.csv"
        rc = cli_bench.main([*args, "--out", str(out)])
        assert rc == 0, (key, rc)
        g[f"cli_{key}"] = np.frombuffer(out.read_bytes(), dtype=np.uint8)
        g[f"cli_{key}_args"] = np.array(args)


def main():
    g = {}
    scanseq_golden(g)
    sequential_golden(g)
    parareal_golden(g)
    cli_golden(g)
    np.savez_compressed(OUT / "f_rows.npz", versions=VERSIONS, **g)
    print("wrote", OUT / "f_rows.npz", len(g), "arrays")


if __name__ == "__main__":
    main()
