"""Python-side overhead of solve_batch(numpy) for cfg2, part by part."""
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
conf = pkg.NewtonConfig(max_iters=10, abort_on_nonfinite=False)
x0 = w.x0.cpu().numpy()
g = np.ascontiguousarray(np.broadcast_to(w.host_guess, (w.B, w.n, w.d)))
dev = torch.device("cuda")
for _ in range(10):
    NP.solve_batch(w.prob, w.stepper, w.cfg.dt, x0, g, conf)
acc = {}
for it in range(50):
    t = [time.perf_counter()]
    P, S = NP._validate(w.prob, w.stepper); t.append(time.perf_counter())
    n = NP.n_steps_for(w.prob, w.cfg.dt); dv = NP._device(None); t.append(time.perf_counter())
    states = torch.empty((w.B, n, w.d), dtype=torch.float64, pin_memory=True).numpy(); t.append(time.perf_counter())
    H = 11
    hist = np.empty((w.B, H)); shist = np.empty((w.B, H)); iters = np.empty(w.B, np.int32)
    status = np.empty(w.B, np.int32); sidx = np.empty(w.B, np.int64); t.append(time.perf_counter())
    cfg = N.make_cfg(10, 0.0, 0.0, False); t.append(time.perf_counter())
    with torch.cuda.device(dv):
        s = torch.cuda.current_stream(dv).cuda_stream
        t.append(time.perf_counter())
        N.check(N.lib().odx_solve_host(P, S, x0.ctypes.data, g.ctypes.data, states.ctypes.data,
                                       w.B, n, float(w.cfg.dt), cfg, hist.ctypes.data,
                                       shist.ctypes.data, iters.ctypes.data, status.ctypes.data,
                                       sidx.ctypes.data, s))
    t.append(time.perf_counter())
    t0 = time.perf_counter(); NP.solve_batch(w.prob, w.stepper, w.cfg.dt, x0, g, conf); t.append(time.perf_counter() - t0 + t[-1])
    if it >= 10:
        for i, name in enumerate(["validate", "n+device", "pinned states", "np arrays", "cfg",
                                  "ctx+stream", "odx_solve_host", "solve_batch total"]):
            acc.setdefault(name, []).append((t[i + 1] - t[i]) * 1e6)
for k, v in acc.items():
    print(f"{k:20s} {np.median(v):8.1f} us")
