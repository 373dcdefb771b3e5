"""§8(f) rows pinned to vectors produced by the reference itself
(tests/golden/make_golden_f.py -> tests/golden/f_rows.npz).

CPU: the oracle's restatement of affine_scan.scan_sequential.
GPU: the sequential marchers (baselines.solve_sequential_explicit / _implicit,
baselines.py:63-118), Parareal (solve_parareal, baselines.py:164-227) and the
CLI's output files (cli_bench.py) against the reference's own outputs.

The sequential explicit marcher and Parareal's coarse sweep are compiled
without FMA contraction (build.py SEQ_FLAGS) and follow the reference's
operation order, so on polynomial right-hand sides they are bit-identical to
the reference; the CLI's sequential CSV is then byte-identical.  Cart-pole
(sin / cos: CUDA's libm is not glibc's) and the implicit marcher (pivot
reciprocals) are compared at 1e-12.
"""

from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden" / "f_rows.npz"


@pytest.fixture(scope="module")
def g():
    return np.load(GOLD)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_oracle_scan_sequential_vs_reference(g, d):
    from oracle import oracle as O
    F, c, z0 = g[f"scanseq_d{d}_F"], g[f"scanseq_d{d}_c"], g[f"scanseq_d{d}_z0"]
    c2 = c.copy()
    c2[0] = F[0] @ z0 + c[0]  # init_elements' element 0 (affine_scan.py:100)
    got = O.scan_sequential(F, c2)
    ref = g[f"scanseq_d{d}_states"]
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    fin = np.isfinite(ref)
    np.testing.assert_allclose(got[fin], ref[fin], rtol=1e-13, atol=1e-13)


def _pkg():
    import paper_2511_01465_b200 as P
    return P


def _problem(P, name):
    if name == "lorenz63":
        return P.lorenz63(x0=(1.0, 1.0, 1.0), tf=2.0)
    return P.get_problem(name)


SEQX = ["logistic_rk4", "logistic_euler", "vdp_rk4", "dahlquist_euler", "lorenz63_rk4",
        "cartpole_rk4"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", SEQX)
def test_sequential_explicit_vs_reference(g, case):
    P = _pkg()
    from paper_2511_01465_b200.baselines import solve_sequential_explicit
    name, sname = case.rsplit("_", 1)
    prob = _problem(P, name)
    tr = solve_sequential_explicit(prob, P.get_stepper(sname, prob), float(g[f"seqx_{case}_dt"]))
    ref = g[f"seqx_{case}"]
    got = np.asarray(tr.states)
    assert got.shape == ref.shape
    if name == "cartpole":
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
    else:
        assert np.array_equal(got, ref), float(np.max(np.abs(got - ref)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["dahlquist", "vdp", "robertson"])
def test_sequential_implicit_vs_reference(g, name):
    P = _pkg()
    from paper_2511_01465_b200.baselines import solve_sequential_implicit
    prob = P.get_problem(name)
    tr = solve_sequential_implicit(prob, P.get_stepper("backward_euler", prob),
                                   float(g[f"seqi_{name}_backward_euler_dt"]))
    ref = g[f"seqi_{name}_backward_euler"]
    got = np.asarray(tr.states)
    assert got.shape == ref.shape
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["logistic", "vdp"])
def test_parareal_vs_reference(g, name):
    P = _pkg()
    from paper_2511_01465_b200.baselines import PararealConfig, solve_parareal
    m, sub, its = (int(v) for v in g[f"par_{name}_cfg"])
    prob = P.get_problem(name)
    st = P.get_stepper("rk4", prob)
    res = solve_parareal(prob, st, st, PararealConfig(n_coarse=m, n_iterations=its,
                                                      fine_substeps=sub))
    for key, got in (("nodes", res.coarse_nodes), ("history", np.stack(res.node_history)),
                     ("states", res.trajectory.states)):
        ref = g[f"par_{name}_{key}"]
        got = np.asarray(got)
        assert got.shape == ref.shape, key
        assert np.array_equal(got, ref), (key, float(np.max(np.abs(got - ref))))


def _cli(argv, out):
    from paper_2511_01465_b200.cli_bench import main
    return main([*argv, "--out", str(out)])


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["solve_seq_logistic", "solve_seq_vdp_be",
                                 "solve_newton_logistic", "solve_parareal_logistic",
                                 "residuals_vdp"])
def test_cli_output_vs_reference_cli(g, key, tmp_path):
    """The CLI's output file against the reference CLI's, run with the same
    arguments: byte-identical where the computation is (sequential explicit,
    Parareal); otherwise the same header, row count and t column bytes, and
    values at 1e-9 scaled (parallel Newton: FMA / scan association)."""
    args = [str(a) for a in g[f"cli_{key}_args"]]
    out = tmp_path / "out.csv"
    assert _cli(args, out) == 0
    mine = out.read_bytes()
    ref = g[f"cli_{key}"].tobytes()
    if key in ("solve_seq_logistic", "solve_parareal_logistic"):
        assert mine == ref
        return
    a, b = mine.decode().splitlines(), ref.decode().splitlines()
    assert a[0] == b[0] and len(a) == len(b)
    if key.startswith("solve"):  # identical time column
        assert [r.split(",")[0] for r in a] == [r.split(",")[0] for r in b]
    x = np.array([[float(v) for v in r.split(",")] for r in a[1:]])
    y = np.array([[float(v) for v in r.split(",")] for r in b[1:]])
    if key.startswith("residuals"):
        assert np.array_equal(x[:, 0], y[:, 0])
        np.testing.assert_allclose(x[:, 1], y[:, 1], rtol=1e-7, atol=1e-15)
    else:
        scale = max(1.0, float(np.abs(y).max()))
        assert float(np.abs(x - y).max()) <= 1e-9 * scale
