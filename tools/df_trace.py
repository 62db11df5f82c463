"""Analyse a coarse dataflow factorization trace (BDDC_COOP_TRACE=<file>, coarse_coop.cu).

Prints the span, per-type run/wait totals, CTA idle share and the critical path: starting
from the last task to finish, each step goes to whatever released the task (the producer of
its last-satisfied dependency, or the CTA's previous task when it did not wait).
Diagnostics only.
"""

from __future__ import annotations

import sys
from collections import defaultdict

import numpy as np

NAMES = ["EA", "PT", "TS", "X1", "SY", "X2", "W", "CB", "SP", "SB", "SCP", "SC", "SM", "LT"]


def load(path):
    raw = open(path, "rb").read()
    n, tsz, ndep, nsig = np.frombuffer(raw[:16], dtype=np.int32)
    nint = tsz // 4
    tasks = np.frombuffer(raw[16:16 + n * tsz], dtype=np.int32).reshape(n, nint)
    tr = np.frombuffer(raw[16 + n * tsz:], dtype=np.uint64).reshape(n, 4).astype(np.int64)
    typ, node, a, b, arg = (tasks[:, i] for i in range(5))
    dep = tasks[:, 5:5 + ndep]
    tgt = tasks[:, 5 + ndep:5 + 2 * ndep]
    sig = tasks[:, 5 + 2 * ndep:5 + 2 * ndep + nsig]
    return dict(n=n, typ=typ, node=node, a=a, b=b, arg=arg, dep=dep, tgt=tgt, sig=sig, tr=tr)


def main(path):
    d = load(path)
    tr = d["tr"]
    t0 = tr[:, 0].min()
    deq, rdy, end, cta = tr[:, 0] - t0, tr[:, 1] - t0, tr[:, 2] - t0, tr[:, 3]
    span = end.max()
    ncta = int(cta.max()) + 1
    run = end - rdy
    wait = rdy - deq
    print(f"tasks {d['n']}  CTAs {ncta}  span {span / 1e3:.1f} us")
    print(f"busy share {run.sum() / (span * ncta):.3f}  wait share {wait.sum() / (span * ncta):.3f}")
    for k, nm in enumerate(NAMES):
        m = d["typ"] == k
        if m.any():
            print(f"  {nm:3s} n={m.sum():7d} run {run[m].sum() / 1e3 / ncta:8.1f} us/CTA "
                  f"(avg {run[m].mean() / 1e3:6.2f}, p90 {np.percentile(run[m], 90) / 1e3:6.2f})  "
                  f"wait {wait[m].sum() / 1e3 / ncta:8.1f} us/CTA")
    # producers per counter
    prod = defaultdict(list)
    for i in range(d["n"]):
        for c in d["sig"][i]:
            if c >= 0:
                prod[int(c)].append(i)
    # per-CTA previous task
    order = np.lexsort((deq, cta))
    prev = np.full(d["n"], -1)
    for j in range(1, len(order)):
        if cta[order[j]] == cta[order[j - 1]]:
            prev[order[j]] = order[j - 1]
    cur = int(np.argmax(end))
    path = []
    while cur >= 0:
        path.append(cur)
        best, bt = -1, -1
        if wait[cur] > 2000:  # waited > 2 us: released by a producer
            for c, tg in zip(d["dep"][cur], d["tgt"][cur]):
                if c < 0:
                    continue
                ends = sorted((end[p], p) for p in prod[int(c)])
                if len(ends) >= tg:
                    e, p = ends[tg - 1]
                    if e <= rdy[cur] + 1000 and e > bt:
                        best, bt = p, e
        if best < 0:
            best = int(prev[cur])
        cur = best
    path.reverse()
    by = defaultdict(float)
    gaps = 0.0
    for i, p in enumerate(path):
        by[NAMES[d["typ"][p]]] += run[p]
        if i:
            gaps += max(0, rdy[p] - end[path[i - 1]])
    print(f"critical path: {len(path)} tasks, run {sum(by.values()) / 1e3:.1f} us, gaps {gaps / 1e3:.1f} us")
    for k, v in sorted(by.items(), key=lambda kv: -kv[1]):
        print(f"  {k:3s} {v / 1e3:8.1f} us")
    if len(sys.argv) > 2:
        for p in path:
            print(f"    {NAMES[d['typ'][p]]:3s} node {d['node'][p]:6d} a {d['a'][p]:4d} b {d['b'][p]:4d} "
                  f"arg {d['arg'][p]:3d}  deq {deq[p] / 1e3:8.1f} rdy {rdy[p] / 1e3:8.1f} end {end[p] / 1e3:8.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
