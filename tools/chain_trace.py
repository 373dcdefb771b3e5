"""Summarise an ODX_CHAIN_TRACE dump (solve_chain.cuh): per-tile stamps of pass 1
   0 claimed  1 build start  2 A published  3 P published (scanner)
   4 carry obtained (control)  5 applied  6 CTA  7 scanner ready-run length

    ODX_CHAIN_TRACE=/tmp/tr.bin python tools/cfg5_time.py ... ; python tools/chain_trace.py /tmp/tr.bin
"""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 8).astype(np.int64)
n = a.shape[0]
t0 = a[:, 0][a[:, 0] > 0].min()
s = a.copy()
for k in range(6):
    s[:, k] = np.where(a[:, k] > 0, a[:, k] - t0, -1)
ok = (s[:, :6] >= 0).all(1)
print(f"tiles {n}, complete {ok.sum()}; span {s[:, 5].max() / 1e3:.1f} us")
v = s[ok]
def q(x):
    return " ".join(f"{np.percentile(x, p):8.2f}" for p in (5, 50, 95, 99))
print("percentiles (us)             p5      p50      p95      p99")
print("claim -> build start  ", q((v[:, 1] - v[:, 0]) / 1e3))
print("build -> A published  ", q((v[:, 2] - v[:, 1]) / 1e3))
print("A -> P (scanner)      ", q((v[:, 3] - v[:, 2]) / 1e3))
pprev = np.concatenate([[0], s[:-1, 3]])
okp = ok & (pprev >= 0)
okp[0] = False
print("P(t-1) -> carry(t)    ", q((s[okp, 4] - pprev[okp]) / 1e3))
print("A(t) -> carry(t)      ", q((v[:, 4] - v[:, 2]) / 1e3))
print("carry -> applied      ", q((v[:, 5] - v[:, 4]) / 1e3))
print("build start -> applied", q((v[:, 5] - v[:, 1]) / 1e3))
# per-CTA tile period
cta = a[:, 6]
per = []
for c in np.unique(cta[ok]):
    bs = np.sort(s[ok & (cta == c), 1])
    if bs.size > 2:
        per.append(np.diff(bs))
per = np.concatenate(per)
print("tile period per CTA   ", q(per / 1e3))
# scanner: P publication rate over time, and the A frontier vs P frontier
P = np.sort(s[s[:, 3] >= 0, 3])
print(f"scanner: {P.size} prefixes in {(P[-1] - P[0]) / 1e3:.1f} us = {P.size / ((P[-1] - P[0]) / 1e3):.1f} tiles/us;"
      f" mean run {a[:, 7][a[:, 7] > 0].mean():.1f}")
A = np.sort(s[s[:, 2] >= 0, 2])
print(f"A publication: {A.size} in {(A[-1] - A[0]) / 1e3:.1f} us = {A.size / ((A[-1] - A[0]) / 1e3):.1f} tiles/us")
mid = n // 2
print("tiles around the middle:")
for t in range(mid, mid + 6):
    print(t, (s[t, :6] / 1e3).round(2), "cta", a[t, 6], "run", a[t, 7])
# scanner rounds: tiles published together share (almost) one timestamp
order = np.argsort(s[:, 3])
Pt = s[order, 3]
Pt = Pt[Pt >= 0]
gaps = np.diff(Pt)
starts = np.concatenate([[0], np.nonzero(gaps > 300)[0] + 1])  # >0.3 us apart: new round
rt = Pt[starts]
sizes = np.diff(np.concatenate([starts, [Pt.size]]))
print(f"scanner rounds: {starts.size}; round period (us) p50 {np.median(np.diff(rt)) / 1e3:.2f} "
      f"p95 {np.percentile(np.diff(rt), 95) / 1e3:.2f}; tiles/round p50 {np.median(sizes):.0f} mean {sizes.mean():.1f}")
# A frontier vs P frontier at the middle of the pass
tm = np.median(Pt)
a_front = int((s[:, 2] >= 0)[(s[:, 2] <= tm)].sum()) if False else int(((s[:, 2] >= 0) & (s[:, 2] <= tm)).sum())
p_front = int(((s[:, 3] >= 0) & (s[:, 3] <= tm)).sum())
print(f"at t={tm / 1e3:.0f} us: {a_front} aggregates published, {p_front} prefixes published")
