"""Out-of-bounds write canaries for every device route (compute-sanitizer is
closed on this pool, so the check is our own): the iterate X, the histories,
the outcome vectors and the workspace each sit inside a larger allocation
whose guard bands hold a NaN bit pattern; after a solve through the C ABI
(odx_solve) every guard byte must be untouched and the result must match the
oracle.  Routes are chosen per process from the environment, so each case
runs in a subprocess (as tests/test_gpu_paths.py)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
REPO = Path(__file__).resolve().parents[1]

SCRIPT = r'''
import json, sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
import paper_2511_01465_b200 as pkg
from paper_2511_01465_b200 import _native as N
from oracle import oracle as O
case, n, B = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
if case == "lorenz":
    prob, sname, dt, pid = pkg.lorenz63(tf=n * 0.01), "rk4", 0.01, O.PROB["lorenz63"]
elif case == "vdp_be":
    prob, sname, dt, pid = pkg.van_der_pol(mu=10.0, x0=(2.0, 0.0), tf=n * 1e-3), "backward_euler", 1e-3, O.PROB["vdp"]
elif case == "ac":
    prob, sname, dt, pid = pkg.allen_cahn(n=64, eps=0.01, dx=1 / 64, tf=n * 1e-3), "backward_euler", 1e-3, O.PROB["allen_cahn"]
else:
    prob, sname, dt, pid = pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * 1e-3), "rk4", 1e-3, O.PROB["vdp"]
st = pkg.get_stepper(sname, prob)
P, S = prob.native(), st.native()
d = prob.dim
iters = 3
cfg = N.make_cfg(iters, 0.0, 0.0, False)
dev = torch.device("cuda")
G = 4096  # guard doubles on each side
PAT = np.frombuffer(np.uint64(0x7ff8dead5a5a5a5a).tobytes(), dtype=np.float64)[0]

def guarded(count, dtype=torch.float64):
    nbytes = count * torch.tensor([], dtype=dtype).element_size()
    n8 = (nbytes + 7) // 8
    buf = torch.full((n8 + 2 * G,), PAT, dtype=torch.float64, device=dev)
    return buf, buf[G:G + n8]

rng = np.random.default_rng(0)
x0s = np.tile(prob.x0, (B, 1)) + (0.01 * rng.standard_normal((B, d)) if B > 1 else 0.0)
guess = np.ascontiguousarray(np.repeat(x0s[:, None, :], n, axis=1))
bx, X = guarded(B * n * d)
X.copy_(torch.from_numpy(guess.ravel()))
bh, hist = guarded(B * (iters + 1))
bs, shist = guarded(B * (iters + 1))
bo, outv = guarded(B * 4)  # iters (i32) + status (i32) + sidx (i64) packed in 16 B per trajectory
x0t = torch.from_numpy(x0s.ravel()).to(dev)
ws_bytes = N.lib().odx_solve_workspace_bytes(P, S, B, n, cfg)
bw, ws = guarded((ws_bytes + 7) // 8)
before = [b.clone() for b in (bx, bh, bs, bo, bw)]
it_p = outv.data_ptr()
stat_p = it_p + 4 * B
sidx_p = it_p + 8 * B
N.check(N.lib().odx_solve(P, S, N.ptr(x0t), N.ptr(X), B, n, float(dt), cfg, N.ptr(hist),
                          N.ptr(shist), it_p, stat_p, sidx_p, N.ptr(ws), ws_bytes,
                          N.stream_handle(dev)))
torch.cuda.synchronize()
bad = []
for name, b0, b1 in zip(("X", "hist", "shist", "outcome", "workspace"), before, (bx, bh, bs, bo, bw)):
    for lo, hi in ((0, G), (b1.numel() - G, b1.numel())):
        if not torch.equal(b0[lo:hi].view(torch.int64), b1[lo:hi].view(torch.int64)):
            bad.append(name)
Xh = X.cpu().numpy().reshape(B, n, d)
errs = []
for b in range(B):
    ref = O.solve(pid, tuple(P.params[:P.n_params]), O.stepper_by_name(sname), x0s[b],
                  guess[b], dt, iters, abort_nonfinite=False)
    fin = np.isfinite(ref["X"])
    scale = max(1.0, float(np.abs(ref["X"][fin]).max()))
    errs.append(float(np.abs(Xh[b][fin] - ref["X"][fin]).max()) / scale)
print(json.dumps(dict(bad=bad, err=max(errs), route=N.lib().odx_last_route().decode())))
'''

CASES = [
    ("resident", "lorenz", 1000, 3, {}),
    ("resident_batch", "lorenz", 2048, 37, {}),
    ("grid", "vdp_be", 65536 - 77, 1, {}),
    ("chain", "vdp_rk4", 300007, 1, {"ODX_GRID_RESIDENT": "0"}),
    ("chain_d3", "lorenz", 200001, 1, {"ODX_GRID_RESIDENT": "0"}),
    ("fused", "vdp_rk4", 300007, 1, {"ODX_GRID_RESIDENT": "0", "ODX_CHAIN": "0"}),
    ("ws", "vdp_rk4", 300007, 1, {"ODX_GRID_RESIDENT": "0", "ODX_CHAIN": "0",
                                  "ODX_FUSED_TILED": "0"}),
    ("tiled", "vdp_rk4", 300007, 1, {"ODX_GRID_RESIDENT": "0", "ODX_CHAIN": "0",
                                     "ODX_FUSED_TILED": "0", "ODX_TILED": "1"}),
    ("dense", "ac", 4099, 1, {}),
]


@pytest.mark.parametrize("label,case,n,B,env", CASES, ids=[c[0] for c in CASES])
def test_no_write_outside_buffers(label, case, n, B, env):
    e = dict(os.environ)
    for k in ("ODX_GRID_RESIDENT", "ODX_CHAIN", "ODX_FUSED_TILED", "ODX_TILED"):
        e.pop(k, None)
    e.update(env)
    out = subprocess.run([sys.executable, "-c", SCRIPT, str(REPO), case, str(n), str(B)], env=e,
                         capture_output=True, text=True, timeout=600, cwd=str(REPO))
    assert out.returncode == 0, out.stderr[-3000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["bad"] == [], r
    assert r["err"] <= 1e-9, r
    expect = {"resident": "resident_solve", "resident_batch": "resident_solve",
              "grid": "grid_resident", "chain": "chain2_pass", "chain_d3": "chain2_pass",
              "fused": "shard_fused", "ws": "persistent_ws", "tiled": "tiled_build",
              "dense": "dense d=64"}[label]
    assert expect in r["route"], r
