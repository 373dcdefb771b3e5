"""Python-side overhead of solve_batch's host path (cfg2)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_01465_b200 as pkg  # noqa: E402
from paper_2511_01465_b200 import newton_pint as NP  # noqa: E402
from paper_2511_01465_b200 import _native as N  # noqa: E402
from bench import Workload, cfg_id  # noqa: E402

w = Workload(cfg_id("cfg2"), 10)
config = pkg.NewtonConfig(max_iters=10, abort_on_nonfinite=False)
x0s = w.x0.cpu().numpy()
X = np.ascontiguousarray(np.broadcast_to(w.host_guess, (w.B, w.n, w.d)))
dev = torch.device("cuda")
for _ in range(5):
    NP.solve_batch(w.prob, w.stepper, w.cfg.dt, x0s, X, config)
def t(f, n=200):
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    return (time.perf_counter() - t0) / n * 1e6
print("validate", t(lambda: NP._validate(w.prob, w.stepper)))
print("n_steps_for", t(lambda: NP.n_steps_for(w.prob, w.cfg.dt)))
print("_device", t(lambda: NP._device(None)))
print("pinned empty", t(lambda: torch.empty((1, w.n, 2), dtype=torch.float64, pin_memory=True).numpy()))
print("np.empty x5", t(lambda: [np.empty(11) for _ in range(5)]))
print("make_cfg", t(lambda: N.make_cfg(10, 0.0, 0.0, False)))
print("cuda.device ctx", t(lambda: torch.cuda.device(dev).__enter__()))
print("current_stream", t(lambda: torch.cuda.current_stream(dev).cuda_stream))
print("ascontig", t(lambda: np.ascontiguousarray(X, dtype=np.float64)))
print("solve_batch", t(lambda: NP.solve_batch(w.prob, w.stepper, w.cfg.dt, x0s, X, config), 50))
P, S = NP._validate(w.prob, w.stepper)
print("_solve_host", t(lambda: NP._solve_host(P, S, x0s, X, w.cfg.dt, config, dev), 50))
