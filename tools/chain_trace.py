"""Summarise an ODX_CHAIN_TRACE dump (solve_chain.cuh): per-tile stamps of pass 1
   0 claimed  1 build start  2 A published  3 P published (scanner)
   4 carry obtained (control)  5 applied  6 CTA  7 scanner warp
   8 iteration top (after the hand-off barrier)  9 build loop done  10 warp scan done
   11 iteration end (after the apply)  12 / 13 = 9 / 11 on warp 3 (shares its scheduler
   with the control warp)

    ODX_CHAIN_TRACE=/tmp/tr.bin python tools/cfg5_time.py ... ; python tools/chain_trace.py /tmp/tr.bin
"""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 16).astype(np.int64)
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

# compute-side phases of the iteration that builds tile t (thread 0 unless noted)
okc = ok & (a[:, 8] > 0) & (a[:, 9] > 0) & (a[:, 10] > 0) & (a[:, 11] > 0)
c = a[okc]
print("top -> build start (loads issued)", q((c[:, 1] - c[:, 8]) / 1e3))
print("build loop                       ", q((c[:, 9] - c[:, 1]) / 1e3))
print("warp scan                        ", q((c[:, 10] - c[:, 9]) / 1e3))
print("apply                            ", q((c[:, 11] - c[:, 10]) / 1e3))
print("iteration busy (top -> end)      ", q((c[:, 11] - c[:, 8]) / 1e3))
okw = okc & (a[:, 12] > 0) & (a[:, 13] > 0)
c3 = a[okw]
if c3.shape[0]:  # (solve_chain.cuh's 7 + 1 warp kernel only)
    print("warp 3: build loop (from w0 start)", q((c3[:, 12] - c3[:, 1]) / 1e3))
    print("warp 3: iteration end vs warp 0   ", q((c3[:, 13] - c3[:, 11]) / 1e3))
# barrier wait: next tile's top on the same CTA minus this iteration's end
waits = []
for cc in np.unique(cta[okc]):
    m = okc & (cta == cc)
    idx = np.argsort(a[m, 8])
    tops = a[m, 8][idx]
    ends = a[m, 11][idx]
    if tops.size > 2:
        waits.append(tops[1:] - ends[:-1])
waits = np.concatenate(waits)
print("end -> next top (barrier wait)   ", q(waits / 1e3))

# scanner windows (solve_chain2.cuh): lane 0's stamps on the window's first tile
win = (a[:, 12] > 0) & (a[:, 13] > 0) & (a[:, 14] > 0) & (a[:, 3] > 0)
if win.sum() > 8:
    ws = a[win]
    idx = np.nonzero(win)[0]
    wl = int(np.median(np.diff(idx)))
    print(f"scanner windows: {win.sum()} of {wl} tiles")
    lastA = np.array([a[i:i + wl, 2].max() for i in idx])
    print("window start -> complete (poll)  ", q((ws[:, 13] - ws[:, 12]) / 1e3))
    print("last A of window -> complete     ", q((ws[:, 13] - lastA) / 1e3))
    print("complete -> state obtained       ", q((ws[:, 14] - ws[:, 13]) / 1e3))
    print("state obtained -> P published    ", q((ws[:, 3] - ws[:, 14]) / 1e3))
    print("polls per window                 ", q(ws[:, 7].astype(float)))
    st = np.sort(ws[:, 14])
    print("state hand-off interval          ", q(np.diff(st) / 1e3))
