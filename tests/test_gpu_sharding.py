"""GPU checks of the multi-GPU paths on ONE device.

* emulated ranks: R DeviceShard objects (odx_shard_local / odx_shard_fixup)
  on one GPU, records concatenated in place of the all-gather; the protocol is
  bulk-synchronous, so no kernel waits on another rank's kernel
* the real torch.distributed/NCCL drivers at world size 1
Both must reproduce the single-GPU solve and the oracle.
"""

import os
import socket
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _emulate(pkg, prob, st, dt, guess, R, max_iters, step_tol=0.0, abort=False, mode="two_pass"):
    from paper_2511_01465_b200.sharded import (DeviceShard, ShardedNewton, chunk_bounds,
                                               run_device_decided)
    fused = mode != "two_pass"
    n, d = guess.shape
    shards = []
    for r in range(R):
        off, nl = chunk_bounds(n, R, r)
        X = torch.from_numpy(np.ascontiguousarray(guess[off:off + nl])).cuda()
        halo = torch.from_numpy(prob.x0 if r == 0 else guess[off - 1]).cuda()
        shards.append(DeviceShard(prob, st, dt, X, halo, off, r, R, fused=fused))

    class Lockstep:
        """All R ranks behind one backend: local() of every rank, then fixups."""
        def __init__(self):
            self.steps = [float("nan")] * R

        def local(self, it):
            return [s.local(it).clone() for s in shards]

        def fixup(self, recs):
            for s in shards:
                s.fixup(recs)
            self.steps = [s.step() for s in shards]

        def step(self):
            return self.steps

        def advance(self, recs):
            return [s.advance(recs).clone() for s in shards]

    if mode == "device":
        def gather_into():
            allrec = torch.stack([s.rec for s in shards])
            for s in shards:
                s.recs_dev.copy_(allrec)
        conf = pkg.NewtonConfig(max_iters=max_iters, step_tol=step_tol, abort_on_nonfinite=abort)
        res = run_device_decided(shards, gather_into, conf, poll=3)
        X = np.concatenate([s.X.cpu().numpy() for s in shards])
        return X, res

    be = Lockstep()
    be.fused = fused

    def gather(recs, step_locals):
        out = torch.stack(recs).cpu().numpy()
        if isinstance(step_locals, list):
            out[:, d * d + 2 * d + 2] = step_locals
        return out

    res = ShardedNewton(be, gather, d, max_iters, 0.0, step_tol, abort).run()
    X = np.concatenate([s.X.cpu().numpy() for s in shards])
    return X, res


@pytest.mark.parametrize("case", [
    ("vdp1_rk4", 1.0, "rk4", 1e-3, 20000, 10, 0.0, False),
    ("vdp10_be", 10.0, "backward_euler", 1e-3, 65536, 100, 1e-10, True),
])
@pytest.mark.parametrize("mode", ["two_pass", "host", "device"])
@pytest.mark.parametrize("R", [2, 3, 8])
def test_emulated_time_sharding(oracle, case, R, mode):
    import paper_2511_01465_b200 as pkg
    name, mu, sname, dt, n, iters, stol, abort = case
    prob = pkg.van_der_pol(mu=mu, x0=(2.0, 0.0), tf=n * dt)
    st = pkg.get_stepper(sname, prob)
    guess = np.tile(prob.x0, (n, 1))
    X, res = _emulate(pkg, prob, st, dt, guess, R, iters, stol, abort, mode)
    ref = oracle.solve(1, (mu,), oracle.stepper_by_name(sname), prob.x0, guess, dt, iters,
                       step_tol=stol, abort_nonfinite=abort)
    assert res["status"] == ref["status"]
    assert abs(res["iters"] - ref["iters"]) <= 1
    h = np.array(res["hist"])
    np.testing.assert_allclose(h[:2], ref["hist"][:2], rtol=1e-7)
    if ref["status"] != oracle.ST_NONFINITE:
        fin = np.isfinite(ref["X"]).all(axis=1)
        assert np.array_equal(fin, np.isfinite(X).all(axis=1))
        scale = max(1.0, float(np.abs(ref["X"][fin]).max()))
        assert np.abs(X[fin] - ref["X"][fin]).max() <= 1e-9 * scale


def test_nccl_drivers_world_size_one(oracle):
    import torch.distributed as dist
    import paper_2511_01465_b200 as pkg
    from paper_2511_01465_b200.configs import CONFIGS
    from paper_2511_01465_b200.sharded import solve_batch_sharded, solve_time_sharded
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n, dt = 200000, 1e-3
        prob = pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * dt)
        st = pkg.get_stepper("rk4", prob)
        seq = oracle.seq_explicit(1, (1.0,), oracle.RK4_A, oracle.RK4_B, prob.x0, dt, n)
        guess = seq * (1.0 + 1e-3 * np.random.default_rng(5).standard_normal(seq.shape))
        ref = oracle.solve(1, (1.0,), oracle.stepper_by_name("rk4"), prob.x0, guess, dt, 12,
                           step_tol=1e-10, abort_nonfinite=False)
        assert ref["status"] == oracle.ST_CONVERGED and ref["iters"] < 12
        scale = max(1.0, float(np.abs(ref["X"]).max()))
        for protocol in ("native", "device", "host", "two_pass"):
            X = torch.from_numpy(guess.copy()).cuda()
            conf = pkg.NewtonConfig(max_iters=12, step_tol=1e-10, abort_on_nonfinite=False)
            rep = solve_time_sharded(prob, st, dt, X, 0, conf, protocol=protocol)
            assert rep.status == ref["status"], protocol
            assert abs(rep.iterations_run - ref["iters"]) <= 1, protocol
            assert np.abs(X.cpu().numpy() - ref["X"]).max() <= 1e-9 * scale, protocol
            h = np.array(rep.residual_history)
            hr = ref["hist"][:len(h)]
            assert (np.abs(h - hr) <= 1e-7 * hr + 1e-9 * hr[0]).all(), protocol
        # the d = 64 path (two-pass protocol) through the same driver
        c4 = CONFIGS[4]
        ac = pkg.allen_cahn(n=c4.dim, eps=c4.params[0], dx=c4.params[1], u0=c4.x0s()[0],
                            tf=4096 * c4.dt)
        import numpy as _np
        g = _np.load(Path(__file__).resolve().parent / "golden" / "baseline.npz")
        ref = g["cfg4s_X_sub"]
        for protocol in ("device", "native", "two_pass"):
            Xa = torch.from_numpy(np.tile(ac.x0, (4096, 1))).cuda()
            rep = solve_time_sharded(ac, pkg.get_stepper(c4.stepper, ac), c4.dt, Xa, 0,
                                     pkg.NewtonConfig(max_iters=c4.max_iters,
                                                      step_tol=c4.step_tol), protocol=protocol)
            assert rep.status == int(g["cfg4s_status"]), protocol
            assert abs(rep.iterations_run - int(g["cfg4s_iters"])) <= 1, protocol
            err = _np.abs(Xa.cpu().numpy()[::32] - ref).max()
            assert err <= 1e-9 * max(1.0, float(_np.abs(ref).max())), protocol
        cfg = CONFIGS[3]
        lor = pkg.lorenz63(x0=(1.0, 1.0, 1.0), tf=cfg.n_steps * cfg.dt)
        local, off, gathered = solve_batch_sharded(lor, pkg.get_stepper("rk4", lor), cfg.dt,
                                                   cfg.x0s()[:64],
                                                   pkg.NewtonConfig(max_iters=100,
                                                                    step_tol=1e-10))
        assert off == 0 and gathered["status"].shape == (64,)
        assert (gathered["status"] == 2).all()  # NONFINITE(1), SURVEY A.1
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["two_pass", "host", "device"])
@pytest.mark.parametrize("case", [
    # multi-tile chunks (n_local > chunks x tile): the chunk-boundary rows
    ("vdp_long", "rk4", 1 << 20, 1e-3, 2, 4),
    ("lorenz_be", "backward_euler", 300000, 1e-5, 3, 5),
    ("linear4_rk4", "rk4", 700001, 1e-4, 3, 3),
    ("logistic_be", "backward_euler", 500003, 1e-5, 4, 4),
])
def test_emulated_time_sharding_long(oracle, case, mode):
    import paper_2511_01465_b200 as pkg
    name, sname, n, dt, R, iters = case
    if name == "vdp_long":
        prob = pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * dt)
    elif name == "lorenz_be":
        prob = pkg.lorenz63(x0=(1.0, 1.0, 1.0), tf=n * dt)
    elif name == "logistic_be":
        prob = pkg.problems.logistic(tf=n * dt)
    else:
        A = np.array([[-1.0, 0.5, 0.0, 0.1], [0.0, -2.0, 0.3, 0.0],
                      [0.2, 0.0, -0.5, 0.4], [0.0, -0.1, 0.0, -1.5]])
        from paper_2511_01465_b200.problems import linear
        prob = linear(A, x0=(1.0, -1.0, 0.5, 2.0), tf=n * dt)
    nat = prob.native()
    pid, params = nat.problem_id, tuple(nat.params[:nat.n_params])
    st = pkg.get_stepper(sname, prob)
    # guess: the sequential trajectory, perturbed (a constant guess over a long
    # chaotic / oscillating horizon drives late rows to ~1e270, where 1-ulp
    # differences are amplified past any fixed tolerance)
    ostep = oracle.stepper_by_name(sname)
    if sname == "rk4":
        seq = oracle.seq_explicit(pid, params, oracle.RK4_A, oracle.RK4_B, prob.x0, dt, n)
    else:
        seq, _ = oracle.seq_implicit(pid, params, ostep.w_prev, ostep.w_next, prob.x0, dt, n)
    rng = np.random.default_rng(7)
    guess = seq * (1.0 + 1e-3 * rng.standard_normal(seq.shape))
    X, res = _emulate(pkg, prob, st, dt, guess, R, iters, 0.0, False, mode)
    ref = oracle.solve(pid, params, oracle.stepper_by_name(sname), prob.x0, guess, dt, iters,
                       abort_nonfinite=False)
    assert res["status"] == ref["status"] and res["iters"] == ref["iters"]
    h, hr = np.array(res["hist"]), ref["hist"][:len(res["hist"])]
    big = hr > 1e-12  # below that the history is round-off
    np.testing.assert_allclose(h[big], hr[big], rtol=1e-7)
    assert (h[~big] <= 1e-12).all()
    fin = np.isfinite(ref["X"]).all(axis=1)
    assert np.array_equal(fin, np.isfinite(X).all(axis=1))
    scale = max(1.0, float(np.abs(ref["X"][fin]).max()))
    assert np.abs(X[fin] - ref["X"][fin]).max() <= 1e-9 * scale


@pytest.mark.parametrize("mode", ["two_pass", "device"])
@pytest.mark.parametrize("R", [2, 3])
def test_emulated_time_sharding_dense(golden_baseline, R, mode):
    """cfg4's d = 64 Allen-Cahn path split along time (two-pass protocol,
    rank aggregate M_r = F_last ... F_first from the chunk aggregates): the
    N = 4096 run converges like the unsharded oracle (golden cfg4s_*)."""
    import paper_2511_01465_b200 as pkg
    from paper_2511_01465_b200.configs import CONFIGS
    cfg = CONFIGS[4]
    n = 4096
    prob = pkg.allen_cahn(n=cfg.dim, eps=cfg.params[0], dx=cfg.params[1], u0=cfg.x0s()[0],
                          tf=n * cfg.dt)
    st = pkg.get_stepper(cfg.stepper, prob)
    guess = np.tile(prob.x0, (n, 1))
    X, res = _emulate(pkg, prob, st, cfg.dt, guess, R, cfg.max_iters, cfg.step_tol,
                      cfg.abort_nonfinite, mode)
    g = golden_baseline
    assert res["status"] == int(g["cfg4s_status"])
    assert abs(res["iters"] - int(g["cfg4s_iters"])) <= 1
    ref = g["cfg4s_X_sub"]
    scale = max(1.0, float(np.abs(ref).max()))
    assert np.abs(X[::32] - ref).max() <= 1e-9 * scale
    h = np.array(res["hist"])
    hr = g["cfg4s_hist"][:len(h)]
    assert (np.abs(h - hr) <= 1e-7 * hr + 1e-9 * hr[0]).all()


@pytest.mark.parametrize("mode", ["two_pass", "device"])
def test_emulated_time_sharding_dense_full_size(mode):
    """cfg4 at its full N = 65536 over 8 emulated ranks, 3 fixed iterations
    (diverging iterates up to ~1e19): against the unsharded GPU solve, which
    tests/test_gpu_parity.py pins to the oracle."""
    import paper_2511_01465_b200 as pkg
    from paper_2511_01465_b200.configs import CONFIGS
    from paper_2511_01465_b200.newton_pint import solve_batch
    cfg = CONFIGS[4]
    n = cfg.n_steps
    prob = pkg.allen_cahn(n=cfg.dim, eps=cfg.params[0], dx=cfg.params[1], u0=cfg.x0s()[0],
                          tf=n * cfg.dt)
    st = pkg.get_stepper(cfg.stepper, prob)
    guess = np.tile(prob.x0, (n, 1))
    X, res = _emulate(pkg, prob, st, cfg.dt, guess, 8, 3, 0.0, False, mode)
    conf = pkg.NewtonConfig(max_iters=3, abort_on_nonfinite=False)
    ref = solve_batch(prob, st, cfg.dt, prob.x0[None], None, conf)
    R = ref.states[0]
    fin = np.isfinite(R).all(axis=1)
    assert np.array_equal(fin, np.isfinite(X).all(axis=1))
    scale = max(1.0, float(np.abs(R[fin]).max()))
    assert np.abs(X[fin] - R[fin]).max() <= 1e-9 * scale
    assert res["iters"] == int(ref.iterations_run[0]) and res["status"] == int(ref.status[0])


@pytest.mark.parametrize("mode", ["two_pass", "host", "device"])
@pytest.mark.parametrize("n,R", [(5, 5), (7, 3), (2, 2), (1000, 7)])
def test_emulated_time_sharding_tiny_ranks(oracle, n, R, mode):
    """Ranks with one or a few steps (a single partial tile and chunk)."""
    import paper_2511_01465_b200 as pkg
    dt = 1e-2
    prob = pkg.van_der_pol(mu=1.0, x0=(2.0, 0.0), tf=n * dt)
    st = pkg.get_stepper("rk4", prob)
    guess = np.tile(prob.x0, (n, 1))
    X, res = _emulate(pkg, prob, st, dt, guess, R, 4, 0.0, False, mode)
    ref = oracle.solve(1, (1.0,), oracle.stepper_by_name("rk4"), prob.x0, guess, dt, 4,
                       abort_nonfinite=False)
    assert res["status"] == ref["status"] and res["iters"] == ref["iters"]
    fin = np.isfinite(ref["X"]).all(axis=1)
    assert np.array_equal(fin, np.isfinite(X).all(axis=1))
    scale = max(1.0, float(np.abs(ref["X"][fin]).max()))
    assert np.abs(X[fin] - ref["X"][fin]).max() <= 1e-9 * scale


@pytest.mark.parametrize("mode", ["two_pass", "device"])
def test_emulated_time_sharding_dense_tiny_ranks(golden_baseline, mode):
    """d = 64 ranks of 2 steps (one chunk, a one-level tree)."""
    import paper_2511_01465_b200 as pkg
    from paper_2511_01465_b200.configs import CONFIGS
    from paper_2511_01465_b200.newton_pint import solve_batch
    cfg = CONFIGS[4]
    n = 8
    prob = pkg.allen_cahn(n=cfg.dim, eps=cfg.params[0], dx=cfg.params[1], u0=cfg.x0s()[0],
                          tf=n * cfg.dt)
    st = pkg.get_stepper(cfg.stepper, prob)
    X, res = _emulate(pkg, prob, st, cfg.dt, np.tile(prob.x0, (n, 1)), 4, 3, 0.0, False, mode)
    ref = solve_batch(prob, st, cfg.dt, prob.x0[None], None,
                      pkg.NewtonConfig(max_iters=3, abort_on_nonfinite=False))
    R = ref.states[0]
    assert np.abs(X - R).max() <= 1e-9 * max(1.0, float(np.abs(R).max()))
