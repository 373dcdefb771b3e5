import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2511_01465_b200 as pkg
from paper_2511_01465_b200.newton_pint import solve_batch
from bench import Workload, cfg_id
w = Workload(cfg_id("cfg2"), 10)
conf = pkg.NewtonConfig(max_iters=10, abort_on_nonfinite=False)
x0 = w.x0.cpu().numpy()
g = np.ascontiguousarray(np.broadcast_to(w.host_guess, (w.B, w.n, w.d)))
gp = torch.empty((w.B, w.n, w.d), dtype=torch.float64, pin_memory=True).numpy()
np.copyto(gp, g)
for name, gg in (("pageable", g), ("pinned", gp)):
    for i in range(8):
        t = time.perf_counter()
        rep = solve_batch(w.prob, w.stepper, w.cfg.dt, x0, gg, conf)
        if i >= 6: print(name, "total us", round((time.perf_counter() - t) * 1e6, 1), file=sys.stderr)
