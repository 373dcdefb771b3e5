"""Small solves on every device route, for compute-sanitizer runs
(racecheck / synccheck / memcheck), one route per process:

    ODX_CHAIN=0 compute-sanitizer --tool racecheck python tools/sanitize_cases.py fused
Routes: resident, grid, chain (ODX_GRID_RESIDENT=0), fused (+ ODX_CHAIN=0),
ws (+ ODX_FUSED_TILED=0), dense (Allen-Cahn d=64) — tools/sanitize_all.sh sets
the switches.  Each result is checked against
the oracle so a sanitizer run also shows the route computed the right thing.
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2511_01465_b200 as pkg  # noqa: E402
from oracle import oracle as O  # noqa: E402

route = sys.argv[1]
iters = 2
if route == "resident":
    prob, sname, n, dt, pid = pkg.lorenz63(tf=10.24), "rk4", 1024, 0.01, O.PROB["lorenz63"]
elif route == "grid":
    prob, sname, n, dt, pid = pkg.van_der_pol(mu=10.0, x0=(2.0, 0.0), tf=4.096), "backward_euler", 4096, 1e-3, O.PROB["vdp"]
elif route == "dense":
    prob = pkg.allen_cahn(n=64, eps=0.01, dx=1.0 / 64, tf=0.256)
    sname, n, dt, pid = "backward_euler", 256, 1e-3, O.PROB["allen_cahn"]
else:  # chain / fused / ws: long-trajectory routes (N above the one-wave limit)
    n = 160000
    prob, sname, dt, pid = pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * 1e-3), "rk4", 1e-3, O.PROB["vdp"]
st = pkg.get_stepper(sname, prob)
conf = pkg.NewtonConfig(max_iters=iters, abort_on_nonfinite=False)
rep = pkg.solve(prob, st, dt, guess="replicate_x0", config=conf)
nat = prob.native()
params = tuple(nat.params[:nat.n_params])
ref = O.solve(pid, params, O.stepper_by_name(sname), prob.x0, np.tile(prob.x0, (n, 1)), dt, iters,
              abort_nonfinite=False)
X = np.asarray(rep.trajectory.states)
fin = np.isfinite(ref["X"])
scale = max(1.0, float(np.abs(ref["X"][fin]).max()))
err = float(np.abs(X[fin] - ref["X"][fin]).max()) / scale
from paper_2511_01465_b200 import _native as N  # noqa: E402
print(f"route {route}: {N.lib().odx_last_route().decode()}; scaled err {err:.2e}")
assert err <= 1e-9
