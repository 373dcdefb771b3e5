import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2511_01465_b200 as pkg
from paper_2511_01465_b200 import newton_pint as NP
from paper_2511_01465_b200.newton_pint import solve_batch
def gr(n):
    dt = 1e-3
    prob = pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * dt)
    st = pkg.get_stepper("rk4", prob)
    x0 = np.array([2.0, 0.0])
    conf = pkg.NewtonConfig(max_iters=3, abort_on_nonfinite=False)
    return solve_batch(prob, st, dt, x0[None], None, conf)
n = 200003
dev = torch.device("cuda", 0)
gr(n)
big = NP._BUF.workspace(dev, 3 << 30)
f = big.view(torch.float64)
for lo, val in ((0, 0.0), (0, 1e10), (2048, 1e10), (1 << 16, 1e10), (1 << 20, 1e10), (1 << 24, 1e10)):
    f.fill_(0.0)
    f[lo:].fill_(val)
    torch.cuda.synchronize()
    hs = [gr(n).residual_history[0][1] for _ in range(3)]
    print("poison from double", lo, "val", val, "hist1", hs)
