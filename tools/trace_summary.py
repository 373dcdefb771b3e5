"""Summarise a tools/trace_ws timeline (8 u64 stamps per tile)."""
import sys

import numpy as np

for f in sys.argv[1:]:
    a = np.fromfile(f, dtype=np.uint64).reshape(-1, 16).astype(np.float64)
    a = a[a[:, 0] > 0]
    t0 = a[:, 6].min()
    cols = [c for c in range(11) if c != 7]
    a[:, cols] -= t0
    parts = (("claim->build", a[:, 0] - a[:, 6]), ("build", a[:, 1] - a[:, 0]),
             ("  items", a[:, 8] - a[:, 0]), ("  warp scan", a[:, 9] - a[:, 8]),
             ("  tile barrier", a[:, 10] - a[:, 9]), ("  agg publish", a[:, 1] - a[:, 10]),
             ("agg->lookback", a[:, 2] - a[:, 1]), ("lookback", a[:, 3] - a[:, 2]),
             ("pref->apply", a[:, 4] - a[:, 3]), ("apply", a[:, 5] - a[:, 4]))
    print(f, "tiles", len(a), "iteration span us", round(a[:, 5].max() / 1e3, 1))
    parts = tuple(x for x in parts if not x[0].startswith("  ") or a[:, 8].max() > 0)
    for name, c in (("lb rounds", 11), ("lb tma ns", 12), ("lb distance", 13), ("lb copy ns", 14), ("lb reduce ns", 15)):
        v = a[:, c]
        print(f"  {name:14s} mean {v.mean():8.2f}     p50 {np.median(v):8.2f}  "
              f"p90 {np.percentile(v, 90):8.2f}  max {v.max():8.2f}")
    for name, v in parts:
        print(f"  {name:14s} mean {v.mean()/1e3:8.2f} us  p50 {np.median(v)/1e3:8.2f}  "
              f"p90 {np.percentile(v, 90)/1e3:8.2f}  max {v.max()/1e3:8.2f}")
