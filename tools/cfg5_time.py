"""Time cfg5 (VdP mu=1 RK4, N=2^26, fixed 10 Newton iterations) on the current
route (ODX_CHAIN / ODX_FUSED_TILED select it) and check a small case against
the oracle first.

    python tools/cfg5_time.py [--n N] [--reps R] [--check-n N]
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import Workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 26)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--check-n", type=int, default=1 << 20)
a = ap.parse_args()

if a.check_n:
    from oracle import oracle as O
    w = Workload(5, 3, n_override=a.check_n)
    w.reset()
    w.launch()
    torch.cuda.synchronize()
    X = w.X[0].cpu().numpy()
    cfg = w.cfg
    x0 = cfg.x0s()[0]
    O.set_threads(os.cpu_count())
    ref = O.solve(1, cfg.params, O.stepper_by_name("rk4"), x0, np.tile(x0, (a.check_n, 1)), cfg.dt,
                  3, abort_nonfinite=False)
    R = ref["X"]
    fr, fx = np.isfinite(R).all(1), np.isfinite(X).all(1)
    both = fr & fx
    scale = max(1.0, np.abs(R[both]).max())
    err = np.abs(X[both] - R[both]).max() / scale
    print(f"check N={a.check_n} 3 it: mask mismatches {(fr != fx).sum()}, scaled err {err:.3e}, "
          f"hist gpu {w.hist[0].cpu().numpy()} ref {ref['hist']}", flush=True)
    del w

w = Workload(5, a.iters, n_override=a.n)
ts = []
for r in range(a.reps + 1):
    w.reset()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    w.launch()
    e1.record()
    torch.cuda.synchronize()
    if r:
        ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
print(f"cfg5 N={a.n} {a.iters} it: {ms:.3f} ms per solve ({ms / a.iters:.3f} ms/it), "
      f"{a.n * a.iters / ms / 1e6:.2f} G steps/s; all {['%.3f' % t for t in ts]}", flush=True)
