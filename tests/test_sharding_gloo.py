"""Multi-rank paths on the CPU: world_size-2 gloo runs of the sharding protocol.

The time-sharded protocol (paper_2511_01465_b200/sharded.py: local build+scan,
one all-gather of records per Newton iteration, identical decisions, carry
fix-up, halo += carry) runs with the oracle backend on two gloo ranks and must
reproduce the unsharded oracle solve (newton_pint.py:366-396 semantics):
statuses and iteration counts exactly, iterates to 1e-9 scaled.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = {
    # name: (pid, params, stepper, x0, N, dt, max_iters, step_tol, abort)
    "vdp1_rk4_fixed": (1, (1.0,), "rk4", [2.0, 0.0], 1001, 1e-3, 5, 0.0, False),
    "vdp10_be_stop": (1, (10.0,), "backward_euler", [2.0, 0.0], 4096, 1e-3, 100, 1e-10, True),
    "lorenz_cfg1": (6, (10.0, 28.0, 8.0 / 3.0), "rk4", [1.0, 1.0, 1.0], 1024, 0.01, 100, 1e-10,
                    True),
    "logistic_converge": (0, (1.0, 1.0), "rk4", [0.1], 1000, 1e-2, 11, 1e-10, True),
    # the d = 64 record (64 x 64 rank aggregate): cfg4's Allen-Cahn problem and
    # x0, N = 256, until converged
    "allen_cahn_cfg4": (7, (0.01, 0.015625), "backward_euler", "cfg4_x0", 256, 1e-3, 20, 1e-10,
                        True),
}
# initial guess per case (default: replicate x0); the logistic case uses the
# reference's own convergent "ones" guess (tests/test_acceptance.py crit 3)
GUESS_ONES = {"logistic_converge"}


def _x0(x0):
    if isinstance(x0, str):  # a golden fixture entry
        from pathlib import Path
        return np.load(Path(__file__).resolve().parent / "golden" / "baseline.npz")[x0]
    return np.asarray(x0, np.float64)


def _worker(rank, world, port, case, q, fused=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from _oracle_shard import OracleShard
        from oracle import oracle as O
        from paper_2511_01465_b200.sharded import ShardedNewton, chunk_bounds
        pid, params, sname, x0, n, dt, max_iters, step_tol, abort = CASES[case]
        x0 = _x0(x0)
        off, nl = chunk_bounds(n, world, rank)
        guess = np.ones((n, x0.shape[0])) if case in GUESS_ONES else np.tile(x0, (n, 1))
        halo = x0 if rank == 0 else guess[off - 1]
        be = OracleShard(pid, params, O.stepper_by_name(sname), dt, guess[off:off + nl], halo,
                         off, rank, world, fused=fused)
        d = x0.shape[0]

        def gather(rec, step_local):
            r = torch.as_tensor(np.asarray(rec, np.float64).copy())
            if step_local is not None:
                r[d * d + 2 * d + 2] = step_local
            out = [torch.empty_like(r) for _ in range(world)]
            dist.all_gather(out, r)
            return torch.stack(out).numpy()

        out = ShardedNewton(be, gather, d, max_iters, 0.0, step_tol, abort).run()
        q.put((rank, off, be.X, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fused", [False, True], ids=["two_pass", "fused"])
@pytest.mark.parametrize("case", list(CASES))
def test_time_sharded_protocol_gloo(oracle, case, fused):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q, fused)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    X = np.concatenate([r[2] for r in res])
    outs = [r[3] for r in res]
    assert outs[0]["status"] == outs[1]["status"] and outs[0]["iters"] == outs[1]["iters"]
    pid, params, sname, x0, n, dt, max_iters, step_tol, abort = CASES[case]
    x0 = _x0(x0)
    guess = np.ones((n, x0.shape[0])) if case in GUESS_ONES else np.tile(x0, (n, 1))
    ref = oracle.solve(pid, params, oracle.stepper_by_name(sname), x0, guess, dt,
                       max_iters, step_tol=step_tol, abort_nonfinite=abort)
    assert outs[0]["status"] == ref["status"]
    assert outs[0]["iters"] == ref["iters"]
    hist = np.array(outs[0]["hist"])
    np.testing.assert_allclose(hist, ref["hist"][: len(hist)], rtol=1e-7, atol=0)
    if ref["status"] != oracle.ST_NONFINITE:
        fin = np.isfinite(ref["X"])
        scale = max(1.0, float(np.abs(ref["X"][fin]).max()))
        assert np.abs(X[fin] - ref["X"][fin]).max() <= 1e-9 * scale


def test_chunk_bounds_partition():
    from paper_2511_01465_b200.sharded import chunk_bounds
    for n in (1, 7, 64, 1001):
        for R in (1, 2, 3, 8):
            if R > n:
                continue
            spans = [chunk_bounds(n, R, r) for r in range(R)]
            assert spans[0][0] == 0
            for (o1, n1), (o2, _) in zip(spans, spans[1:]):
                assert o1 + n1 == o2
            assert sum(s[1] for s in spans) == n
            assert max(s[1] for s in spans) - min(s[1] for s in spans) <= 1


def test_decide_matches_oracle_semantics():
    from paper_2511_01465_b200 import _native as N
    from paper_2511_01465_b200.sharded import decide
    nan = float("nan")
    assert decide(0, 5, 0.0, 0.0, True, 1.0, 3, nan) == (True, N.ST_SINGULAR, 3, 0)
    assert decide(2, 5, 0.0, 0.0, True, float("inf"), -1, 1.0) == (True, N.ST_NONFINITE, 2, 2)
    assert decide(2, 5, 0.0, 0.0, False, float("inf"), -1, 1.0)[0] is False
    assert decide(5, 5, 0.0, 0.0, True, 1.0, -1, 1.0) == (True, N.ST_MAXITER, -1, 5)
    assert decide(3, 5, 1e-6, 0.0, True, 1e-7, -1, 1.0) == (True, N.ST_CONVERGED, -1, 3)
    assert decide(3, 5, 0.0, 1e-10, True, 1.0, -1, 1e-11) == (True, N.ST_CONVERGED, -1, 3)
    assert decide(0, 5, 0.0, 1e-10, True, 1.0, -1, nan)[0] is False


def _batch_oracle_solve(x0s, n, dt, max_iters, step_tol):
    """Per-trajectory oracle solves (the CPU stand-in for solve_batch)."""
    from types import SimpleNamespace
    from oracle import oracle as O
    st, its = [], []
    for x0 in x0s:
        r = O.solve(6, (10.0, 28.0, 8.0 / 3.0), O.stepper_by_name("rk4"), x0, np.tile(x0, (n, 1)),
                    dt, max_iters, step_tol=step_tol, abort_nonfinite=True)
        st.append(r["status"])
        its.append(r["iters"])
    return SimpleNamespace(status=np.array(st), iterations_run=np.array(its))


BATCH = dict(B=37, n=256, dt=0.01, max_iters=100, step_tol=1e-10)


def _batch_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_01465_b200.configs import CONFIGS
        from paper_2511_01465_b200.sharded import solve_batch_sharded
        x0s = CONFIGS[3].x0s()[:BATCH["B"]]
        rep, off, gathered = solve_batch_sharded(
            None, None, BATCH["dt"], x0s, None,
            solve_fn=lambda xs: _batch_oracle_solve(xs, BATCH["n"], BATCH["dt"],
                                                    BATCH["max_iters"], BATCH["step_tol"]))
        q.put((rank, off, len(rep.status), gathered["status"].tolist(),
               gathered["iterations_run"].tolist()))
    finally:
        dist.destroy_process_group()


def test_batch_sharded_two_ranks_gloo():
    """solve_batch_sharded (sharded.py) on two gloo ranks: contiguous uneven
    slices (19 + 18 of cfg3's first 37 trajectories), no data-path collective,
    the statuses / iteration counts all-gathered in trajectory order — equal on
    both ranks and to the unsharded per-trajectory solves (BASELINE stop rule)."""
    from paper_2511_01465_b200.configs import CONFIGS
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [(r[1], r[2]) for r in res] == [(0, 19), (19, 18)]
    assert res[0][3] == res[1][3] and res[0][4] == res[1][4]
    ref = _batch_oracle_solve(CONFIGS[3].x0s()[:BATCH["B"]], BATCH["n"], BATCH["dt"],
                              BATCH["max_iters"], BATCH["step_tol"])
    assert res[0][3] == ref.status.tolist()
    assert res[0][4] == ref.iterations_run.tolist()
