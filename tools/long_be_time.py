"""Fused tiled route, implicit (VdP mu=10, backward Euler) at N = 2^22, 10 fixed iterations."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_01465_b200 as pkg  # noqa: E402
from paper_2511_01465_b200.newton_pint import solve_device  # noqa: E402

n = 1 << 22
prob = pkg.van_der_pol(mu=10.0, x0=(2.0, 0.0), tf=n * 1e-3)
st = pkg.get_stepper("backward_euler", prob)
P, S = prob.native(), st.native()
x0 = torch.tensor([[2.0, 0.0]], dtype=torch.float64, device="cuda")
X0 = x0[:, None, :].expand(1, n, 2).contiguous()
conf = pkg.NewtonConfig(max_iters=10, abort_on_nonfinite=False)
ts = []
for r in range(6):
    X = X0.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); solve_device(P, S, x0, X, 1e-3, conf); e1.record()
    torch.cuda.synchronize()
    if r:
        ts.append(e0.elapsed_time(e1))
print("vdp BE N=2^22 10 it:", round(float(np.median(ts)), 4), "ms")
