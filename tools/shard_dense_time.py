"""Per-rank cost of one time-sharded d = 64 iteration (cfg4 at N/R steps),
measured on one GPU, all-gather excluded.  python tools/shard_dense_time.py [R]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_01465_b200 as pkg  # noqa: E402
from paper_2511_01465_b200.configs import CONFIGS  # noqa: E402
from paper_2511_01465_b200.sharded import DeviceShard, rec_len  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = CONFIGS[4]
n = cfg.n_steps // R
prob = pkg.allen_cahn(n=cfg.dim, eps=cfg.params[0], dx=cfg.params[1], u0=cfg.x0s()[0],
                      tf=n * cfg.dt)
st = pkg.get_stepper(cfg.stepper, prob)
x0 = torch.as_tensor(prob.x0, device="cuda")
X = x0.repeat(n, 1).contiguous()
sh = DeviceShard(prob, st, cfg.dt, X, x0, offset=n * (R // 2), rank=R // 2, nranks=R, fused=False)
recs = np.zeros((R, rec_len(64)))
recs[:, :4096] = np.eye(64).ravel()
recs[:, -1] = -1.0
for it in range(2):
    sh.local(it)
    sh.fixup(recs)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
tl, tf = [], []
for it in range(5):
    e[0].record(); sh.local(it); e[1].record(); sh.fixup(recs); e[2].record()
    torch.cuda.synchronize()
    tl.append(e[0].elapsed_time(e[1])); tf.append(e[1].elapsed_time(e[2]))
print(f"d=64 R={R} n_local={n}: local {np.median(tl):.3f} ms, fixup {np.median(tf):.3f} ms, "
      f"total {np.median(tl) + np.median(tf):.3f} ms per iteration")

# device-decided step (decision + fix-up + next local), back to back
from paper_2511_01465_b200 import _native as N  # noqa: E402
cfgc = N.make_cfg(1000, 0.0, 0.0, False)
hist = torch.full((1001,), float("nan"), dtype=torch.float64, device="cuda")
state = torch.zeros(4, dtype=torch.int64, device="cuda")
sh.recs_dev.copy_(torch.from_numpy(recs))
sh.decide_step(1, cfgc, hist, hist.clone(), state)
torch.cuda.synchronize()
e[0].record()
for it in range(2, 12):
    sh.decide_step(it, cfgc, hist, hist.clone(), state)
e[1].record()
torch.cuda.synchronize()
print(f"d=64 R={R} n_local={n}: device-decided step {e[0].elapsed_time(e[1]) / 10:.3f} ms "
      f"per iteration (back to back), stopped={int(state[0].item())}")
