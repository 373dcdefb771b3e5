"""Every long-trajectory route of the single-GPU solve against the oracle.

The route is chosen once per process from the environment
(solve_small_launch.cuh), so each case runs in a subprocess:
  default              single-pass chained kernel (solve_chain2.cuh: independent warp groups
                       per CTA), d <= 3
  ODX_CHAIN=0          fused tiled passes (shard_tiled.cuh: fused_tiled_solve)
  + ODX_FUSED_TILED=0  streaming warp-specialised kernel (solve_ws.cuh)
  + ODX_TILED=1        two-pass tiled kernels (solve_tiled.cuh)
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
REPO = Path(__file__).resolve().parents[1]

SCRIPT = r'''
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2511_01465_b200 as pkg
from oracle import oracle as O
name, n, dt, iters = sys.argv[2], int(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
if name == "vdp_rk4":
    prob, sname = pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * dt), "rk4"
elif name == "vdp_be":
    prob, sname = pkg.van_der_pol(mu=10.0, x0=(2.0, 0.0), tf=n * dt), "backward_euler"
elif name == "vdp_euler":
    prob, sname = pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * dt), "euler"
elif name == "logistic_rk4":
    prob, sname = pkg.logistic(x0=(0.1,), tf=n * dt), "rk4"
else:
    prob, sname = pkg.lorenz63(x0=(1.0, 1.0, 1.0), tf=n * dt), "rk4"
nat = prob.native()
pid, params = nat.problem_id, tuple(nat.params[:nat.n_params])
ost = O.stepper_by_name(sname)
if sname == "rk4":
    seq = O.seq_explicit(pid, params, O.RK4_A, O.RK4_B, prob.x0, dt, n)
elif sname == "euler":
    seq = O.seq_explicit(pid, params, O.EULER_A, O.EULER_B, prob.x0, dt, n)
else:
    seq, _ = O.seq_implicit(pid, params, ost.w_prev, ost.w_next, prob.x0, dt, n)
guess = seq * (1.0 + 1e-3 * np.random.default_rng(3).standard_normal(seq.shape))
conf = pkg.NewtonConfig(max_iters=iters, abort_on_nonfinite=False)
rep = pkg.solve(prob, pkg.get_stepper(sname, prob), dt,
                guess=pkg.Trajectory(prob.x0.copy(), guess, dt, n), config=conf)
ref = O.solve(pid, params, ost, prob.x0, guess, dt, iters, abort_nonfinite=False)
X = np.asarray(rep.trajectory.states)
fin = np.isfinite(ref["X"]).all(axis=1)
scale = max(1.0, float(np.abs(ref["X"][fin]).max()))
err = float(np.abs(X[fin] - ref["X"][fin]).max()) / scale
h = np.asarray(rep.residual_history, dtype=float)
hr = ref["hist"][:len(h)]
# relative to each entry, with a floor at round-off of the initial residual
# (late entries ~1e-11 are differences of nearly equal O(1) numbers)
hrel = float(np.max(np.abs(h - hr) / (hr + 1e-6 * hr[0]))) if len(h) else 0.0
print(json.dumps(dict(err=err, hrel=hrel, iters=rep.iterations_run, ref_iters=ref["iters"],
                      fin_equal=bool(np.array_equal(fin, np.isfinite(X).all(axis=1))))))
'''


@pytest.mark.parametrize("route", ["chain", "fused_tiled", "ws", "tiled"])
@pytest.mark.parametrize("case", [("vdp_rk4", 1 << 21, 1e-3, 5), ("vdp_be", 600000, 1e-4, 4),
                                  ("lorenz_rk4", 500001, 1e-5, 4)])
def test_long_trajectory_routes(case, route):
    env = dict(os.environ)
    env.pop("ODX_FUSED_TILED", None)
    env.pop("ODX_TILED", None)
    env.pop("ODX_CHAIN", None)
    if route != "chain":
        env["ODX_CHAIN"] = "0"
    if route not in ("chain", "fused_tiled"):
        env["ODX_FUSED_TILED"] = "0"
    if route == "tiled":
        env["ODX_TILED"] = "1"
    name, n, dt, iters = case
    out = subprocess.run([sys.executable, "-c", SCRIPT, str(REPO), name, str(n), str(dt),
                          str(iters)], env=env, capture_output=True, text=True, timeout=600,
                         cwd=str(REPO))
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["fin_equal"]
    assert r["err"] <= 1e-9, r
    assert r["hrel"] <= 1e-7, r
    assert abs(r["iters"] - r["ref_iters"]) <= 1


# Cheap builds (explicit Euler, d = 1) run the chain kernel at the scanner's rate — the
# regime in which the kernel's first cut (control-warp hand-off) could deadlock.
@pytest.mark.parametrize("case", [("vdp_euler", 3000001, 1e-4, 4), ("logistic_rk4", 3000001, 1e-4, 4)])
def test_chain_cheap_builds(case):
    env = dict(os.environ)
    for k in ("ODX_FUSED_TILED", "ODX_TILED", "ODX_CHAIN"):
        env.pop(k, None)
    name, n, dt, iters = case
    out = subprocess.run([sys.executable, "-c", SCRIPT, str(REPO), name, str(n), str(dt),
                          str(iters)], env=env, capture_output=True, text=True, timeout=600,
                         cwd=str(REPO))
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["fin_equal"]
    assert r["err"] <= 1e-9, r
    assert r["hrel"] <= 1e-7, r
    assert abs(r["iters"] - r["ref_iters"]) <= 1


@pytest.mark.parametrize("stepper", ["rk4", "euler"])
def test_chain_deterministic(stepper):
    """The default long-trajectory route (single-pass chained kernel) repeated on
    the same input: bit-identical iterates and histories, run after run.  Tiles
    are claimed dynamically and the groups of a CTA drift against each other,
    but every composition has a fixed shape (thread, warp, group tile, scanner
    window), so no value depends on which group built a tile or when its carry
    arrived.  (compute-sanitizer is closed on this pool; this is the race
    check that can run: a torn record or a stale carry would show up as a
    differing bit.)  `euler` is the cheap-build regime, where the scanner and
    the carry polls are under the most pressure."""
    import numpy as np
    import paper_2511_01465_b200 as pkg
    from paper_2511_01465_b200.newton_pint import solve_batch
    n, dt = 1 << 22, 1e-3
    prob = pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * dt)
    st = pkg.get_stepper(stepper, prob)
    conf = pkg.NewtonConfig(max_iters=4, abort_on_nonfinite=False)
    guess = np.tile(prob.x0, (1, n, 1)) + 1e-3
    a = solve_batch(prob, st, dt, prob.x0[None], guess, conf)
    for _ in range(5):
        b = solve_batch(prob, st, dt, prob.x0[None], guess, conf)
        assert np.array_equal(a.states, b.states, equal_nan=True)
        assert np.array_equal(a.residual_history, b.residual_history, equal_nan=True)


def test_grid_resident_deterministic():
    """cfg2's grid-resident solve (halo rows handed over as tagged 16-byte
    chunks, aggregates double-buffered by iteration parity) repeated: every
    run bit-identical."""
    import torch
    import paper_2511_01465_b200 as pkg
    from paper_2511_01465_b200.newton_pint import solve_device
    n = 65536
    prob = pkg.van_der_pol(mu=10.0, x0=(2.0, 0.0), tf=n * 1e-3)
    st = pkg.get_stepper("backward_euler", prob)
    P, S = prob.native(), st.native()
    x0 = torch.tensor([[2.0, 0.0]], dtype=torch.float64, device="cuda")
    X0 = x0[:, None, :].expand(1, n, 2).contiguous()
    conf = pkg.NewtonConfig(max_iters=10, abort_on_nonfinite=False)
    ref = None
    for _ in range(60):
        X = X0.clone()
        solve_device(P, S, x0, X, 1e-3, conf)
        if ref is None:
            ref = X
        else:
            assert torch.equal(torch.nan_to_num(X, nan=7.0), torch.nan_to_num(ref, nan=7.0))
