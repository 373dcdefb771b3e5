"""Break the end-to-end cfg2 call (solve_batch with host numpy) into parts."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_01465_b200 as pkg  # noqa: E402
from paper_2511_01465_b200 import newton_pint as NP  # noqa: E402
from bench import Workload, cfg_id  # noqa: E402

w = Workload(cfg_id("cfg2"), 10)
conf = pkg.NewtonConfig(max_iters=10, abort_on_nonfinite=False)
x0_host = w.x0.cpu().numpy()
guess_host = np.ascontiguousarray(np.broadcast_to(w.host_guess, (w.B, w.n, w.d)))
for _ in range(5):
    NP.solve_batch(w.prob, w.stepper, w.cfg.dt, x0_host, guess_host, conf)
torch.cuda.synchronize()
T = {}
def tic(k, t0):
    T.setdefault(k, []).append((time.perf_counter() - t0) * 1e6)
for _ in range(30):
    t = time.perf_counter()
    NP.solve_batch(w.prob, w.stepper, w.cfg.dt, x0_host, guess_host, conf)
    tic("total solve_batch", t)
    dev = torch.device("cuda")
    t = time.perf_counter(); x0t = NP._to_device(x0_host, dev, ("x0", dev)); torch.cuda.synchronize(); tic("x0 h2d", t)
    t = time.perf_counter(); X = NP._to_device(guess_host, dev, ("X", dev)); torch.cuda.synchronize(); tic("X h2d (copyto+dma)", t)
    t = time.perf_counter(); P, S = NP._validate(w.prob, w.stepper); tic("validate", t)
    t = time.perf_counter(); out = NP.solve_device(P, S, x0t, X, w.cfg.dt, conf); tic("solve_device enqueue", t)
    torch.cuda.synchronize(); tic("solve_device+sync", t)
    t = time.perf_counter(); oh = NP._fetch(out, ("out", dev)); torch.cuda.synchronize(); tic("fetch out", t)
    t = time.perf_counter(); sh = NP._fetch(X, ("Xo", dev)); torch.cuda.synchronize(); tic("fetch X", t)
    t = time.perf_counter(); NP._unpack_outcome(oh.numpy(), 1, 11); tic("unpack", t)
    t = time.perf_counter(); sh.numpy().copy(); tic("states copy", t)
for k, v in T.items():
    print(f"{k:28s} median {np.median(v):8.1f} us")
