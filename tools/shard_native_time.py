"""Per-iteration cost of the native time-sharded loop (odx_solve_sharded) on
ONE rank at cfg5's per-rank size for R ranks, with a real NCCL communicator
(world size 1: the all-gather runs but moves nothing across GPUs).
    python tools/shard_native_time.py [R]"""
import os
import socket
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2511_01465_b200 as pkg  # noqa: E402
from paper_2511_01465_b200.sharded import nccl_comm, run_native  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
n = (1 << 26) // R
dt = 1e-3
prob = pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * dt)
st = pkg.get_stepper("rk4", prob)
halo = torch.tensor([2.0, 0.0], dtype=torch.float64, device="cuda")
comm = nccl_comm()
res = {}
for iters in (2, 12):
    conf = pkg.NewtonConfig(max_iters=iters, abort_on_nonfinite=False)
    ts = []
    for rep in range(4):
        X = halo.repeat(n, 1).contiguous()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = run_native(prob, st, dt, X, halo, 0, 0, 1, comm, conf, poll=0)
        e1.record()
        torch.cuda.synchronize()
        if rep:
            ts.append(e0.elapsed_time(e1))
    res[iters] = float(np.median(ts))
per_it = (res[12] - res[2]) / 10
print(f"R={R} n_local={n}: native loop {res[12]:.3f} ms for 12 iterations, "
      f"{per_it:.3f} ms per iteration (incl. NCCL all-gather + decision)")
dist.destroy_process_group()
