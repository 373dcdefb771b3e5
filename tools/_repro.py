import sys, numpy as np
sys.path.insert(0, '.')
import paper_2511_01465_b200 as pkg
from paper_2511_01465_b200.newton_pint import solve_batch
from paper_2511_01465_b200.configs import CONFIGS
import oracle.oracle as O
def tiled(n):
    dt = 1e-3
    prob = pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * dt)
    st = pkg.get_stepper("rk4", prob)
    x0 = np.array([2.0, 0.0])
    conf = pkg.NewtonConfig(max_iters=3, abort_on_nonfinite=False)
    r = solve_batch(prob, st, dt, x0[None], None, conf)
    return r
n = 200003
ref = O.solve(1, (1.0,), O.stepper_by_name("rk4"), np.array([2.0, 0.0]), np.tile([2.0, 0.0], (n, 1)), 1e-3, 3, abort_nonfinite=False)
def relerr(r):
    X = np.asarray(r.states[0]); R = ref["X"]
    fin = np.isfinite(R)
    scale = max(1.0, np.max(np.abs(R[fin])))
    mask_ok = np.array_equal(np.isfinite(R).all(1), np.isfinite(X).all(1))
    return np.max(np.abs(X[fin] - R[fin])) / scale, mask_ok, np.max(np.abs(r.residual_history[0][:2] - ref["hist"][:2]))
r0 = tiled(n)
print("before dense", relerr(r0))
cfg = CONFIGS[4]
prob = pkg.allen_cahn(n=64, eps=cfg.params[0], dx=cfg.params[1], u0=cfg.x0s()[0], tf=65536 * cfg.dt)
st = pkg.get_stepper("backward_euler", prob)
solve_batch(prob, st, cfg.dt, cfg.x0s(), None, pkg.NewtonConfig(max_iters=3, step_tol=0.0, abort_on_nonfinite=False))
for rep in range(3):
    r1 = tiled(n)
    X = np.asarray(r1.states[0]); R = ref["X"]
    diff = ~((X == R) | (np.isnan(X) & np.isnan(R)))
    rows = np.where(diff.any(axis=1))[0]
    print("after dense rep", rep, relerr(r1), r1.residual_history[0])
