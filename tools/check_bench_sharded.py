"""Exercise bench.py's N > 1 time-sharded cfg5 entry at world size 1 (the
code path the driver's scaling run takes, with a real NCCL process group).

The whole main() of the N > 1 run (headline line, sharded e2e, the
configs["cfg4_time_sharded"] entry) can be exercised the same way:
    ODX_BENCH_FORCE_SHARDED=1 python bench.py --steps 5 --warmup 3 --no-cpu
(profiles/r2/bench_forced_sharded_w1_r2h.json)."""
import os
import socket
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402

with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
buf = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
for cid in (5, 4):
    tw = bench.TimeShardedWorkload(cid, 10, 0, 1)
    td, tl = bench.time_steps(tw, 3, 2, lambda: bench.flush_l2(buf))
    it, st, ix = tw.outcome()
    print(f"cfg{cid} time-sharded x1: {sum(td) / len(td):.3f} ms per solve, launches {tl}, "
          f"iters {it[0]} status {st[0]}")
    del tw
    torch.cuda.empty_cache()
dist.destroy_process_group()
