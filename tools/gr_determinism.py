"""Repeat the cfg2 grid-resident solve and require bit-identical iterates
(a torn halo read or an ordering race would show up as a difference).
    python tools/gr_determinism.py [repeats]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2511_01465_b200 as pkg  # noqa: E402
from paper_2511_01465_b200.newton_pint import solve_device  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
bad = 0
for mu, sname, n in ((10.0, "backward_euler", 65536), (1.0, "rk4", 65536), (1.0, "rk4", 40000)):
    prob = pkg.van_der_pol(mu=mu, x0=(2.0, 0.0), tf=n * 1e-3)
    st = pkg.get_stepper(sname, prob)
    P, S = prob.native(), st.native()
    x0 = torch.tensor([[2.0, 0.0]], dtype=torch.float64, device="cuda")
    X0 = x0[:, None, :].expand(1, n, 2).contiguous()
    conf = pkg.NewtonConfig(max_iters=10, abort_on_nonfinite=False)
    ref = None
    for r in range(reps):
        X = X0.clone()
        solve_device(P, S, x0, X, 1e-3, conf)
        if ref is None:
            ref = X
        elif not torch.equal(torch.nan_to_num(X, nan=7.0), torch.nan_to_num(ref, nan=7.0)):
            bad += 1
    torch.cuda.synchronize()
    print(f"{sname} mu={mu} n={n}: {reps} solves, mismatches so far {bad}")
sys.exit(1 if bad else 0)
