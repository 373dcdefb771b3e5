"""Diagnose non-finite row-mask differences of cfg5 iterates (GPU vs oracle)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import paper_2511_01465_b200 as pkg
from oracle import oracle as O
from test_gpu_parity import _gpu_cfg_solve
from paper_2511_01465_b200.configs import CONFIGS
np.set_printoptions(precision=17, linewidth=200)
cfg = CONFIGS[5]
n = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.oracle_n_steps
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3
x0 = cfg.x0s()[0]
O.set_threads(os.cpu_count())
ref = O.solve(1, cfg.params, O.stepper_by_name("rk4"), x0, np.tile(x0, (n, 1)), cfg.dt, K, abort_nonfinite=False, trace=True)
for k in range(1, K + 1):
    X = _gpu_cfg_solve(pkg, cfg, n=n, max_iters=k).states[0]
    R = ref["trace"][k]
    fr, fx = np.isfinite(R).all(1), np.isfinite(X).all(1)
    bad = np.nonzero(fr != fx)[0]
    both = fr & fx
    rel = np.abs(X[both] - R[both]) / np.maximum(1.0, np.abs(R[both]))
    print(f"iterate {k}: finite ref {fr.sum()} gpu {fx.sum()} mismatched rows {bad.size}; "
          f"max rel err on common finite rows {rel.max() if rel.size else 0:.3e}; max|R| {np.abs(R[fr]).max():.3e}")
    if bad.size:
        print("  first rows:", bad[:20])
        for r in bad[:6]:
            print(f"  row {r}: ref {R[r]} gpu {X[r]}; ref prev-iterate {ref['trace'][k-1][r]} rows r-1 {ref['trace'][k-1][r-1]}")
        # runs of finiteness around
        r = bad[0]
        print("  ref finite pattern around:", fr[r-5:r+6].astype(int), " gpu:", fx[r-5:r+6].astype(int))
