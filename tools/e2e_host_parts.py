"""Time the steps of newton_pint._solve_host for cfg2 (host numpy in/out)."""
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
config = pkg.NewtonConfig(max_iters=10, abort_on_nonfinite=False)
x0s = w.x0.cpu().numpy()
X = np.ascontiguousarray(np.broadcast_to(w.host_guess, (w.B, w.n, w.d)))
dev = torch.device("cuda")
P, S = NP._validate(w.prob, w.stepper)
for _ in range(5):
    NP._solve_host(P, S, x0s, X, w.cfg.dt, config, dev)
T = {}
for _ in range(40):
    t0 = time.perf_counter()
    marks = []
    def m(name):
        marks.append((name, time.perf_counter()))
    B, n, d = X.shape
    H = config.max_iters + 1
    o_sh, o_sidx, o_it, o_st, out_bytes = NP._outcome_layout(B, H)
    nx0, nX = B * d * 8, B * n * d * 8
    o_X = (nx0 + 255) // 256 * 256
    o_out = o_X + (nX + 255) // 256 * 256
    region = NP._BUF.device_region(dev, o_out + out_bytes)
    stage_t = NP._BUF.host(("in", dev), o_X + nX)
    stage = stage_t.numpy()
    m("setup")
    stage[:nx0].view(np.float64)[:] = x0s.reshape(-1)
    np.copyto(stage[o_X:o_X + nX].view(np.float64).reshape(B, n, d), X)
    m("host memcpy")
    region[: o_X + nX].copy_(stage_t[: o_X + nX], non_blocking=True)
    m("h2d enqueue")
    cfg = N.make_cfg(config.max_iters, config.residual_tol, config.step_tol, config.abort_on_nonfinite)
    ws = NP._BUF.workspace(dev, NP._BUF.ws_bytes(P, S, B, n, cfg))
    base = region.data_ptr(); ob = base + o_out
    m("cfg+ws")
    N.check(N.lib().odx_solve(P, S, base, base + o_X, B, n, float(w.cfg.dt), cfg, ob, ob + o_sh, ob + o_it,
                        ob + o_st, ob + o_sidx, ws.data_ptr(), ws.numel(),
                        torch.cuda.current_stream(dev).cuda_stream))
    m("odx_solve call")
    back = torch.empty(o_out - o_X + out_bytes, dtype=torch.uint8, pin_memory=True)
    m("pinned alloc")
    back.copy_(region[o_X: o_out + out_bytes], non_blocking=True)
    m("d2h enqueue")
    torch.cuda.current_stream(dev).synchronize()
    m("sync (gpu: h2d+solve+d2h)")
    raw = back.numpy()
    states = raw[:nX].view(np.float64).reshape(B, n, d)
    res = NP._unpack_outcome(raw[o_out - o_X:], B, H)
    m("unpack")
    prev = t0
    for k, t in marks:
        T.setdefault(k, []).append((t - prev) * 1e6)
        prev = t
    T.setdefault("TOTAL", []).append((prev - t0) * 1e6)
for k, v in T.items():
    print(f"{k:28s} median {np.median(v):8.1f} us")
