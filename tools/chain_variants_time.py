"""Time long single trajectories of several (problem, stepper) pairs on the current
chain route (solve_chain2.cuh), device-resident, 5 fixed iterations.

    python tools/chain_variants_time.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_01465_b200 as pkg  # noqa: E402
from paper_2511_01465_b200 import _native as N  # noqa: E402

CASES = [
    ("vdp rk4", lambda n, dt: pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * dt), "rk4", 1 << 25, 1e-3),
    ("vdp euler", lambda n, dt: pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * dt), "euler", 1 << 25, 1e-4),
    ("vdp backward_euler", lambda n, dt: pkg.van_der_pol(mu=10.0, x0=(2.0, 0.0), tf=n * dt), "backward_euler", 1 << 25, 1e-4),
    ("logistic rk4", lambda n, dt: pkg.logistic(x0=(0.1,), tf=n * dt), "rk4", 1 << 25, 1e-4),
    ("lorenz rk4", lambda n, dt: pkg.lorenz63(x0=(1.0, 1.0, 1.0), tf=n * dt), "rk4", 1 << 24, 1e-5),
]
iters = 5
if len(sys.argv) > 1:
    CASES = [CASES[int(a)] for a in sys.argv[1:]]
L = N.lib()
dev = torch.device("cuda", 0)
for name, mk, stn, n, dt in CASES:
    prob = mk(n, dt)
    st = pkg.get_stepper(stn, prob)
    P, S = prob.native(), st.native()
    d = prob.dim
    x0 = torch.from_numpy(np.asarray(prob.x0, dtype=np.float64)[None]).to(dev)
    guess = x0[:, None, :].expand(1, n, d).contiguous()
    X = torch.empty_like(guess)
    cfg = N.make_cfg(iters, 0.0, 0.0, False)
    hist = torch.empty((1, iters + 1), dtype=torch.float64, device=dev)
    sh = torch.empty_like(hist)
    it_t = torch.empty(1, dtype=torch.int32, device=dev)
    stt = torch.empty(1, dtype=torch.int32, device=dev)
    six = torch.empty(1, dtype=torch.int64, device=dev)
    wsb = L.odx_solve_workspace_bytes(P, S, 1, n, cfg)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    ts = []
    for r in range(4):
        X.copy_(guess)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        N.check(L.odx_solve(P, S, N.ptr(x0), N.ptr(X), 1, n, float(dt), cfg, N.ptr(hist), N.ptr(sh),
                            N.ptr(it_t), N.ptr(stt), N.ptr(six), N.ptr(ws), wsb, N.stream_handle(dev)))
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    route = L.odx_last_route().decode()[:24]
    print(f"{name:22s} N=2^{int(np.log2(n))} {iters} it: {ms:8.3f} ms  ({n * iters / ms / 1e6:7.2f} G steps/s)  [{route}]", flush=True)
    del X, guess, ws
    torch.cuda.empty_cache()
