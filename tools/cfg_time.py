"""Device time of one BASELINE config's fixed-iteration solve (median of reps).

    python tools/cfg_time.py cfg3 [cfg1 ...]
"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import Workload, cfg_id  # noqa: E402

for name in sys.argv[1:] or ["cfg3"]:
    w = Workload(cfg_id(name), 10)
    ts = []
    for r in range(12):
        w.reset()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        w.launch()
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    print(f"{name}: {statistics.median(ts):.4f} ms (min {min(ts):.4f})", flush=True)
    del w
    torch.cuda.empty_cache()
