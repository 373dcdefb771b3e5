"""Per-rank cost of one time-sharded Newton iteration (cfg5 shape at N/R steps),
measured on one GPU: the projected per-iteration time of an R-GPU run, minus
the all-gather.  python tools/shard_rank_time.py [R]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_01465_b200 as pkg  # noqa: E402
from paper_2511_01465_b200.sharded import DeviceShard, rec_len  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = (1 << 26) // R
dt = 1e-3
prob = pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * dt)
st = pkg.get_stepper("rk4", prob)
X = torch.tensor([2.0, 0.0], dtype=torch.float64, device="cuda").repeat(n, 1).contiguous()
halo = torch.tensor([2.0, 0.0], dtype=torch.float64, device="cuda")
sh = DeviceShard(prob, st, dt, X, halo, offset=n * (R // 2), rank=R // 2, nranks=R)
recs = np.zeros((R, rec_len(2)))
recs[:, :4] = np.eye(2).ravel()
recs[:, -4] = 1.0   # rn
recs[:, -1] = -1.0  # no singular step
for it in range(3):
    sh.local(it)
    sh.fixup(recs)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
t_loc, t_fix = [], []
for it in range(10):
    e[0].record(); sh.local(it); e[1].record(); sh.fixup(recs); e[2].record()
    torch.cuda.synchronize()
    t_loc.append(e[0].elapsed_time(e[1])); t_fix.append(e[1].elapsed_time(e[2]))
print(f"R={R} n_local={n}: local {np.median(t_loc):.3f} ms, fixup {np.median(t_fix):.3f} ms, "
      f"total {np.median(t_loc) + np.median(t_fix):.3f} ms per iteration (two-pass)")
t_step = []
for it in range(13):
    e[0].record(); sh.advance(recs); e[1].record()
    torch.cuda.synchronize()
    if it >= 3:
        t_step.append(e[0].elapsed_time(e[1]))
print(f"R={R} n_local={n}: fused step {np.median(t_step):.3f} ms per iteration")

from paper_2511_01465_b200 import _native as N  # noqa: E402
cfg = N.make_cfg(1000, 0.0, 0.0, False)
hist = torch.full((1001,), float("nan"), dtype=torch.float64, device="cuda")
shist = hist.clone()
state = torch.zeros(4, dtype=torch.int64, device="cuda")
sh.recs_dev.copy_(torch.from_numpy(recs))
t_dec = []
for it in range(1, 14):
    e[0].record(); sh.decide_step(it, cfg, hist, shist, state); e[1].record()
    torch.cuda.synchronize()
    if it > 3:
        t_dec.append(e[0].elapsed_time(e[1]))
# back-to-back, as the device-decided protocol enqueues them (no host sync)
e[0].record()
for it in range(14, 34):
    sh.decide_step(it, cfg, hist, shist, state)
e[1].record()
torch.cuda.synchronize()
print(f"R={R} n_local={n}: decide+step {np.median(t_dec):.3f} ms per iteration, "
      f"{e[0].elapsed_time(e[1]) / 20:.3f} ms back-to-back")
