"""Run one BASELINE workload solve a few times (for ncu / nsight captures).

    python tools/profile_one.py --workload cfg5 --iters 2 --reps 2
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import Workload, cfg_id  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--stop-rule", action="store_true")
a = ap.parse_args()
w = Workload(cfg_id(a.workload), a.iters, n_override=a.n)
if a.stop_rule:
    w.set_mode(fixed=False)
for _ in range(a.reps):
    w.reset()
    w.launch()
torch.cuda.synchronize()
it, st, ix = w.outcome()
print("done", a.workload, "iters", it[:4], "status", st[:4])
