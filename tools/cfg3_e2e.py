"""cfg3 (4096 x 2048 Lorenz RK4) end to end through solve_batch with host numpy buffers
(the bench's e2e leg alone): ODX_HOST_THREADS / ODX_HOST_PIPELINE A/B.

    python tools/cfg3_e2e.py
"""
import sys, statistics
sys.path.insert(0, ".")
from bench import Workload, e2e_steps
w = Workload(3, 10)
d, h2d, d2h, note = e2e_steps(w, 8, 3)
print("cfg3 e2e ms:", round(statistics.median(d), 3))
