"""Multi-GPU partitioning of the Newton solve.

Two partitionings, one rank per GPU, torch.distributed for the plumbing:

* batch sharding (BASELINE cfg 3): B independent trajectories split into
  contiguous slices; each rank runs solve_batch on its slice.  No data-path
  collective; one all_gather of the per-trajectory outcomes at the end.

* time sharding (cfg 5, and any d <= 4 trajectory): rank r owns the contiguous
  steps [offset_r, offset_r + n_r).  Per Newton iteration of the reference
  loop (newton_pint.py:366-396) every rank
    1. builds and scans its steps locally  -> record (odx_shard_local)
    2. all-gathers the records             -> ONE collective per iteration
    3. takes solve()'s decision from the gathered residual norms / singular
       indices / previous step norms (identical on every rank)
    4. folds the carries of ranks < r and fixes up its steps, moving its halo
       by its carry (odx_shard_fixup) — no second exchange.

The protocol (ShardedNewton) is backend-agnostic: DeviceShard drives the
CUDA kernels through the C ABI; the CPU tests plug in an oracle backend and
run it over gloo.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as N

__all__ = ["chunk_bounds", "rec_len", "decide", "ShardedNewton", "DeviceShard",
           "solve_time_sharded", "solve_batch_sharded", "TimeShardedReport"]


def chunk_bounds(n_total: int, nranks: int, rank: int) -> tuple[int, int]:
    """(offset, n_local) of rank's contiguous chunk; sizes differ by at most 1."""
    base, rem = divmod(n_total, nranks)
    off = rank * base + min(rank, rem)
    return off, base + (1 if rank < rem else 0)


def rec_len(d: int) -> int:
    """ODX_SHARD_REC(d): [F_agg | c_agg | x_last | rn | sc | step_prev | bad]."""
    return d * d + 2 * d + 4


def _nan_max(values) -> float:
    out = 0.0
    for v in values:
        v = float(v)
        if v > out:
            out = v
    return out


def decide(it: int, max_iters: int, residual_tol: float, step_tol: float, abort: bool,
           rn: float, bad: int, step_prev: float):
    """solve()'s decision sequence (newton_pint.py:373-394) + the step rule.

    Same order as the device kernels and oracle/odescan_oracle.c:orc_solve.
    Returns (stop, status, status_index, iterations_run).
    """
    if bad >= 0:
        return True, N.ST_SINGULAR, bad, it
    if math.isinf(rn) and abort:
        return True, N.ST_NONFINITE, it, it
    conv = (residual_tol > 0 and rn <= residual_tol) or (
        step_tol > 0 and it > 0 and step_prev < step_tol)
    if it >= max_iters:
        return True, (N.ST_CONVERGED if conv else N.ST_MAXITER), -1, max_iters
    if conv:
        return True, N.ST_CONVERGED, -1, it
    return False, -1, -1, it


@dataclass
class TimeShardedReport:
    X_local: object
    offset: int
    residual_history: list
    scaled_residual_history: list
    iterations_run: int
    status: int
    status_index: int


class ShardedNewton:
    """The per-iteration protocol of the time-sharded solve.

    backend: .local(it) -> record (1-D array-like, rec_len(d));
             .fixup(records (R, REC) host numpy) -> None;
             .step() -> float, max|dx| of the last fix-up on this rank;
             or, with backend.fused true, .advance(records) -> record: the
             fix-up of this iteration and the local pass of the next in one
             call, the record's step_prev slot filled by the backend.
    gather:  (record, step_local or None) -> (R, REC) numpy (the all-gather;
             step_local, when not None, goes into the step_prev slot).
    """

    def __init__(self, backend, gather, d: int, max_iters: int, residual_tol: float = 0.0,
                 step_tol: float = 0.0, abort_nonfinite: bool = True):
        self.backend, self.gather, self.d = backend, gather, d
        self.max_iters, self.rtol, self.stol = max_iters, residual_tol, step_tol
        self.abort = abort_nonfinite

    def run(self) -> dict:
        d = self.d
        i_rn, i_sc, i_step, i_bad = d * d + 2 * d, d * d + 2 * d + 1, d * d + 2 * d + 2, d * d + 2 * d + 3
        fused = bool(getattr(self.backend, "fused", False))
        hist, shist = [], []
        step_local = math.nan
        status = idx = -1
        iters = 0
        rec = None
        for it in range(self.max_iters + 1):
            if it == 0 or not fused:
                rec = self.backend.local(it)
            recs = np.asarray(self.gather(rec, None if fused else step_local), dtype=np.float64)
            rn = _nan_max(recs[:, i_rn])
            sc = _nan_max(recs[:, i_sc])
            bads = [int(b) for b in recs[:, i_bad] if b >= 0]
            bad = min(bads) if bads else -1
            steps = recs[:, i_step]
            step_prev = math.nan if it == 0 else _nan_max(steps)
            stop, status, idx, iters = decide(it, self.max_iters, self.rtol, self.stol,
                                              self.abort, rn, bad, step_prev)
            if status != N.ST_SINGULAR:
                hist.append(rn)
                shist.append(sc)
            if stop:
                break
            if fused:
                rec = self.backend.advance(recs)
            else:
                self.backend.fixup(recs)
                step_local = self.backend.step()
        return dict(hist=hist, shist=shist, iters=iters, status=status, status_index=idx)


class DeviceShard:
    """One rank's chunk on its GPU, driven through odx_shard_local and either
    odx_shard_fixup (two passes per iteration) or, with fused=True (the
    default), odx_shard_step (one pass: update + next build)."""

    def __init__(self, problem, stepper, dt: float, X_local, halo, offset: int, rank: int,
                 nranks: int, fused: bool = True):
        import torch
        self.torch = torch
        self.P, self.S = problem.native(), stepper.native()
        self.dt = float(dt)
        self.X = X_local          # (n, d) fp64 CUDA, updated in place
        self.halo = halo.clone()  # (d,) fp64 CUDA
        self.offset, self.rank, self.nranks = int(offset), int(rank), int(nranks)
        n, d = X_local.shape
        self.n, self.d = n, d
        L = N.lib()
        self.ws_bytes = L.odx_shard_workspace_bytes(self.P, self.S, n)
        if self.ws_bytes == 0:
            raise ValueError("time sharding supports small state dims (d <= 4)")
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=X_local.device)
        self.rec = torch.empty(rec_len(d), dtype=torch.float64, device=X_local.device)
        self.step_t = torch.zeros(1, dtype=torch.float64, device=X_local.device)
        self.recs_dev = torch.empty((nranks, rec_len(d)), dtype=torch.float64,
                                    device=X_local.device)
        self.fused = bool(fused)

    def local(self, it):
        N.check(N.lib().odx_shard_local(self.P, self.S, N.ptr(self.halo), N.ptr(self.X), self.n,
                                        self.offset, self.dt, N.ptr(self.rec), N.ptr(self.ws),
                                        self.ws_bytes, N.stream_handle(self.X.device)))
        return self.rec

    def fixup(self, recs_host):
        self.recs_dev.copy_(self.torch.from_numpy(np.ascontiguousarray(recs_host)))
        N.check(N.lib().odx_shard_fixup(self.P, N.ptr(self.recs_dev), self.rank, self.nranks,
                                        N.ptr(self.X), self.n, N.ptr(self.halo),
                                        N.ptr(self.step_t), N.ptr(self.ws), self.ws_bytes,
                                        N.stream_handle(self.X.device)))

    def step(self) -> float:
        return float(self.step_t.item())

    def decide_step(self, it, cfg, hist, shist, state):
        """odx_shard_decide_step: decision of iteration `it` on the device from
        self.recs_dev (already gathered), then the fused step if continuing."""
        N.check(N.lib().odx_shard_decide_step(
            self.P, self.S, cfg, N.ptr(self.recs_dev), self.rank, self.nranks, int(it),
            N.ptr(self.halo), N.ptr(self.X), self.n, self.offset, self.dt, N.ptr(self.rec),
            N.ptr(hist), N.ptr(shist), N.ptr(state), N.ptr(self.ws), self.ws_bytes,
            N.stream_handle(self.X.device)))
        return self.rec

    def advance(self, recs_host):
        self.recs_dev.copy_(self.torch.from_numpy(np.ascontiguousarray(recs_host)))
        N.check(N.lib().odx_shard_step(self.P, self.S, N.ptr(self.recs_dev), self.rank,
                                       self.nranks, N.ptr(self.halo), N.ptr(self.X), self.n,
                                       self.offset, self.dt, N.ptr(self.rec), N.ptr(self.ws),
                                       self.ws_bytes, N.stream_handle(self.X.device)))
        return self.rec


def run_device_decided(shards, gather_into, config, poll: int = 8) -> dict:
    """The time-sharded protocol with the decision taken on the device.

    shards: the DeviceShard(s) driven by this process (one per rank; several
    only when emulating ranks on one GPU).  gather_into(): all-gathers every
    shard's .rec into its .recs_dev on the device (NCCL, no host sync).
    Per iteration the host only enqueues: all-gather, decide_step.  It reads
    the stop flag every `poll` iterations; iterations enqueued after the stop
    are no-ops on the device.  Returns ShardedNewton.run()'s dict.
    """
    import torch
    sh0 = shards[0]
    dev = sh0.X.device
    m = int(config.max_iters)
    cfg = N.make_cfg(m, config.residual_tol, config.step_tol, config.abort_on_nonfinite)
    bufs = []
    for _ in shards:
        bufs.append((torch.full((m + 1,), math.nan, dtype=torch.float64, device=dev),
                     torch.full((m + 1,), math.nan, dtype=torch.float64, device=dev),
                     torch.zeros(4, dtype=torch.int64, device=dev)))
    for s in shards:
        s.local(0)
    for it in range(m + 1):
        gather_into()
        for s, (h, sh, st) in zip(shards, bufs):
            s.decide_step(it, cfg, h, sh, st)
        if it < m and (it + 1) % poll == 0 and int(bufs[0][2][0].item()):
            break
    return _decided_outcome(*bufs[0])


def _decided_outcome(hist, shist, state) -> dict:
    """ShardedNewton.run()'s dict from the device-side decision buffers."""
    h, sh, st = (b.cpu().numpy() for b in (hist, shist, state))
    stopped, status, iters, idx = (int(v) for v in st)
    if not stopped:
        raise RuntimeError("device-decided protocol did not reach a decision")
    n_hist = iters + 1 - (1 if status == N.ST_SINGULAR else 0)
    return dict(hist=[float(v) for v in h[:n_hist]], shist=[float(v) for v in sh[:n_hist]],
                iters=iters, status=status, status_index=idx)


_COMMS: dict = {}


def nccl_comm(group=None) -> int:
    """An ncclComm_t of this process's libnccl.so.2 over the ranks of `group`
    (made once per group and device; rank 0's unique id is broadcast through
    torch.distributed).  Used by the native loop, odx_solve_sharded."""
    import ctypes as C
    import torch
    import torch.distributed as dist
    key = (id(group), torch.cuda.current_device())
    if key in _COMMS:
        return _COMMS[key]
    L = N.lib()
    if not L.odx_nccl_available():
        raise RuntimeError("libnccl.so.2 is not loadable: use protocol='device'")
    R, r = dist.get_world_size(group), dist.get_rank(group)
    uid = C.create_string_buffer(128)
    if r == 0:
        N.check(L.odx_nccl_unique_id(uid))
    obj = [uid.raw]
    src = 0 if group is None else dist.get_global_rank(group, 0)
    dist.broadcast_object_list(obj, src=src, group=group)
    uid = C.create_string_buffer(obj[0], 128)
    comm = C.c_void_p()
    N.check(L.odx_nccl_comm_init(C.byref(comm), R, uid, r))
    _COMMS[key] = comm.value
    return comm.value


def run_native(problem, stepper, dt, X_local, halo, offset, rank, nranks, comm, config,
               poll: int = 8) -> dict:
    """The whole per-rank loop in one library call (odx_solve_sharded): local
    pass, then per iteration ncclAllGather + device-decided fused step, all on
    the current stream."""
    import torch
    L = N.lib()
    P, S = problem.native(), stepper.native()
    dev = X_local.device
    n = X_local.shape[0]
    m = int(config.max_iters)
    cfg = N.make_cfg(m, config.residual_tol, config.step_tol, config.abort_on_nonfinite)
    wsb = L.odx_solve_sharded_workspace_bytes(P, S, n, nranks)
    if wsb == 0:
        raise ValueError("time sharding supports small state dims (d <= 4)")
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    hist = torch.full((m + 1,), math.nan, dtype=torch.float64, device=dev)
    shist = torch.full((m + 1,), math.nan, dtype=torch.float64, device=dev)
    state = torch.zeros(4, dtype=torch.int64, device=dev)
    N.check(L.odx_solve_sharded(P, S, cfg, comm, rank, nranks, N.ptr(halo), N.ptr(X_local), n,
                                int(offset), float(dt), N.ptr(hist), N.ptr(shist), N.ptr(state),
                                int(poll), N.ptr(ws), wsb, N.stream_handle(dev)))
    return _decided_outcome(hist, shist, state)


def _torch_gather(group, d, device):
    import torch
    import torch.distributed as dist
    R = dist.get_world_size(group)

    def gather(rec, step_local):
        r = rec.clone() if hasattr(rec, "clone") else torch.as_tensor(rec, dtype=torch.float64)
        r = r.to(device)
        if step_local is not None:
            r[d * d + 2 * d + 2] = step_local
        out = torch.empty((R, r.numel()), dtype=torch.float64, device=device)
        dist.all_gather_into_tensor(out, r, group=group)
        return out.cpu().numpy()
    return gather


def solve_time_sharded(problem, stepper, dt: float, X_local, offset: int, config, group=None,
                       protocol: str = "device"):
    """Time-sharded solve of one trajectory across the ranks of `group`.

    protocol: "device" (default) — fused passes, decision on the device, no
    host round trip per iteration, the loop and torch's NCCL all-gather
    driven from Python; "native" — the same loop inside the library
    (odx_solve_sharded, its own NCCL communicator); "host" — fused passes,
    decision on the host (ShardedNewton); "two_pass" — separate local /
    fix-up passes.

    X_local: this rank's (n_local, d) CUDA tensor of the initial guess (updated
    in place to the final iterate).  Chunks must be contiguous and ordered by
    rank (chunk_bounds).  Returns a TimeShardedReport; errors are reported as
    statuses, like solve_batch.
    """
    import torch
    import torch.distributed as dist
    if protocol not in ("device", "native", "host", "two_pass"):
        raise ValueError(f"unknown protocol {protocol!r}")
    if problem.dim > 4 and protocol == "host":
        protocol = "device"  # the d = 64 shard has no host-decided fused step
    R = dist.get_world_size(group)
    r = dist.get_rank(group)
    d = problem.dim
    dev = X_local.device
    # initial halos: the last guess row of rank r-1 (x0 on rank 0)
    last = X_local[-1].clone().contiguous()
    lasts = torch.empty((R, d), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(lasts, last, group=group)
    x0 = torch.as_tensor(problem.x0, dtype=torch.float64, device=dev)
    halo = x0 if r == 0 else lasts[r - 1].clone()
    if protocol == "native":
        out = run_native(problem, stepper, dt, X_local, halo.contiguous(), offset, r, R,
                         nccl_comm(group), config)
    elif protocol == "device":
        shard = DeviceShard(problem, stepper, dt, X_local, halo, offset, r, R, fused=True)

        def gather_into():
            dist.all_gather_into_tensor(shard.recs_dev, shard.rec, group=group)
        out = run_device_decided([shard], gather_into, config)
    else:
        shard = DeviceShard(problem, stepper, dt, X_local, halo, offset, r, R,
                            fused=(protocol == "host"))
        proto = ShardedNewton(shard, _torch_gather(group, d, dev), d, config.max_iters,
                              config.residual_tol, config.step_tol, config.abort_on_nonfinite)
        out = proto.run()
    return TimeShardedReport(X_local=X_local, offset=offset, residual_history=out["hist"],
                             scaled_residual_history=out["shist"], iterations_run=out["iters"],
                             status=out["status"], status_index=out["status_index"])


def solve_batch_sharded(problem, stepper, dt: float, x0s, config, group=None, solve_fn=None):
    """Batch sharding: contiguous slices of the B trajectories per rank.

    Runs solve_batch on this rank's slice (no collective on the data path) and
    all-gathers the per-trajectory statuses / iteration counts.  Returns
    (local BatchSolveReport, offset, gathered dict).  solve_fn(x0_slice) may
    replace the device solve (the gloo tests run the CPU oracle there); the
    status exchange then uses host tensors when the group is not NCCL.
    """
    import torch
    import torch.distributed as dist
    from .newton_pint import solve_batch
    R = dist.get_world_size(group)
    r = dist.get_rank(group)
    x0s = np.asarray(x0s)
    B = int(x0s.shape[0])
    off, nb = chunk_bounds(B, R, r)
    if solve_fn is None:
        def solve_fn(xs):
            return solve_batch(problem, stepper, dt, xs, None, config)
    rep = solve_fn(x0s[off:off + nb])
    dev = (torch.device("cuda", torch.cuda.current_device())
           if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    per = (B + R - 1) // R
    st = torch.full((per,), -9, dtype=torch.int64, device=dev)
    st[:nb] = torch.as_tensor(np.asarray(rep.status), dtype=torch.int64)
    its = torch.full((per,), -9, dtype=torch.int64, device=dev)
    its[:nb] = torch.as_tensor(np.asarray(rep.iterations_run), dtype=torch.int64)
    all_st = torch.empty((R * per,), dtype=torch.int64, device=dev)  # flat: gloo needs it
    all_it = torch.empty((R * per,), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(all_st, st, group=group)
    dist.all_gather_into_tensor(all_it, its, group=group)
    sts = all_st.cpu().numpy().ravel()
    itv = all_it.cpu().numpy().ravel()
    keep = sts != -9
    return rep, off, dict(status=sts[keep], iterations_run=itv[keep])
