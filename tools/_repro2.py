import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2511_01465_b200 as pkg
from paper_2511_01465_b200 import newton_pint as NP
from paper_2511_01465_b200.newton_pint import solve_batch
import oracle.oracle as O
def tiled(n):
    dt = 1e-3
    prob = pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * dt)
    st = pkg.get_stepper("rk4", prob)
    x0 = np.array([2.0, 0.0])
    conf = pkg.NewtonConfig(max_iters=3, abort_on_nonfinite=False)
    return solve_batch(prob, st, dt, x0[None], None, conf)
n = 200003
print("fresh", tiled(n).residual_history[0])
# poison the cached workspace with large values
ws = next(iter(NP._BUF.ws.values()))
print("ws bytes", ws.numel())
ws.view(torch.float64)[: ws.numel() // 8] = 1e10
torch.cuda.synchronize()
print("poisoned", tiled(n).residual_history[0])
