"""Locate wrong rows of the chained pass: one Newton update on cfg5's problem,
GPU vs oracle, rows mapped to (tile, warp, lane, item)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from bench import Workload
from oracle import oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
T, ITEMS = int(os.environ.get("CHAIN_T", 896)), 4
w = Workload(5, 1, n_override=n)
w.reset(); w.launch(); torch.cuda.synchronize()
X = w.X[0].cpu().numpy()
cfg = w.cfg; x0 = cfg.x0s()[0]
O.set_threads(os.cpu_count())
R = O.solve(1, cfg.params, O.stepper_by_name("rk4"), x0, np.tile(x0, (n, 1)), cfg.dt, 1, abort_nonfinite=False)["X"]
err = np.abs(X - R).max(1) / np.maximum(1, np.abs(R).max(1))
bad = np.nonzero(err > 1e-9)[0]
print("bad rows", bad.size, "of", n)
if bad.size:
    k = bad[:10]
    for r in k:
        t, o = divmod(int(r), T); thr, it = divmod(o, ITEMS)
        print(f"row {r}: tile {t} thread {thr} (warp {thr // 32} lane {thr % 32}) item {it} err {err[r]:.3e}")
    tiles = np.unique(bad // T)
    print("bad tiles", tiles.size, tiles[:20])
    # within the first bad tile: which offsets
    t0 = tiles[0]
    offs = bad[(bad // T) == t0] % T
    print("first bad tile offsets: min", offs.min(), "max", offs.max(), "count", offs.size)
