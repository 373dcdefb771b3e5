"""Oracle backend for the time-sharding protocol (CPU tests over gloo).

Each rank builds its steps with the oracle's range build (the reference's
_kernels.build_* over a sub-range), scans them with the oracle Blelloch scan
and fixes up with numpy — the same record layout and protocol
(paper_2511_01465_b200.sharded.ShardedNewton) the CUDA backend uses.
"""

import numpy as np

from oracle import oracle as O


class OracleShard:
    def __init__(self, pid, params, stepper, dt, X_local, halo, offset, rank, nranks,
                 fused=False):
        self.fused = bool(fused)
        self.pid, self.params, self.stepper, self.dt = pid, params, stepper, float(dt)
        self.X = np.array(X_local, np.float64, copy=True)
        self.halo = np.array(halo, np.float64, copy=True)
        self.offset, self.rank, self.nranks = int(offset), int(rank), int(nranks)
        self.d = self.X.shape[1]
        self._step = float("nan")

    def local(self, it):
        d = self.d
        Fe, ce, h, bad = O.build_range(self.pid, self.params, self.stepper, self.halo, self.X,
                                       self.dt, self.offset)
        self.Fp, self.cp = O.scan_affine(Fe, ce)
        rn = O.max_abs(h)
        sc = rn if self.stepper.kind == O.EXPLICIT else O.max_abs(ce)
        rec = np.concatenate([self.Fp[-1].ravel(), self.cp[-1], self.X[-1],
                              [rn, sc, np.nan, float(bad)]])
        assert rec.shape[0] == d * d + 2 * d + 4
        return rec

    def fixup(self, recs):
        d = self.d
        z = np.zeros(d)
        for q in range(self.rank):
            F = recs[q, : d * d].reshape(d, d)
            c = recs[q, d * d: d * d + d]
            z = F @ z + c
        dx = np.einsum("kij,j->ki", self.Fp, z) + self.cp
        self.X += dx
        self._step = O.max_abs(dx)
        if self.rank > 0:
            self.halo = self.halo + z

    def step(self):
        return self._step

    def advance(self, recs):
        """fused protocol: fix-up, then the next local pass with step_prev set"""
        self.fixup(recs)
        rec = self.local(None)
        rec[self.d * self.d + 2 * self.d + 2] = self._step
        return rec
