"""Analyse a dataflow coarse-solve trace (BDDC_SOLVE_TRACE=<file>, coarse_coop.cu).

Span, busy/wait shares and the critical path (the producer that released each task, or the
CTA's previous task), with per-task rows/columns. Diagnostics only.
"""

from __future__ import annotations

import sys
from collections import defaultdict

import numpy as np


def main(path, verbose=False):
    raw = open(path, "rb").read()
    n, tsz = np.frombuffer(raw[:8], dtype=np.int32)
    w = np.frombuffer(raw[8:8 + n * tsz], dtype=np.int32).reshape(n, tsz // 4)
    tr = np.frombuffer(raw[8 + n * tsz:], dtype=np.uint64).reshape(n, 4).astype(np.int64)
    node, r0, c0, s, f = w[:, 8], w[:, 9], w[:, 10], w[:, 11], w[:, 12]
    np_, mode = w[:, 17], w[:, 18]
    cw = ((tsz - 20) // 8 * 8) // 4  # CsTask words (8-byte aligned) precede the SdTask fields
    dirn, dep, tgt, sig0, sig1 = (w[:, cw + k] for k in range(5))
    t0 = tr[:, 0].min()
    deq, rdy, end, cta = tr[:, 0] - t0, tr[:, 1] - t0, tr[:, 2] - t0, tr[:, 3]
    span = end.max()
    ncta = int(cta.max()) + 1
    run, wait = end - rdy, rdy - deq
    print(f"tasks {n} CTAs {ncta} span {span / 1e3:.1f} us  busy {run.sum() / span / ncta:.3f} "
          f"wait {wait.sum() / span / ncta:.3f}")
    for d in (0, 1):
        m = dirn == d
        print(f"  {'fwd' if d == 0 else 'bwd'} n={m.sum():6d} run avg {run[m].mean() / 1e3:.2f} us "
              f"first {deq[m].min() / 1e3:.1f} last end {end[m].max() / 1e3:.1f} us")
    prod = defaultdict(list)
    for i in range(n):
        for c in (sig0[i], sig1[i]):
            if c >= 0:
                prod[int(c)].append(i)
    cur = int(np.argmax(end))
    path = []
    order = np.lexsort((deq, cta))
    prev = np.full(n, -1)
    for j in range(1, n):
        if cta[order[j]] == cta[order[j - 1]]:
            prev[order[j]] = order[j - 1]
    while cur >= 0:
        path.append(cur)
        nxt = -1
        if dep[cur] >= 0 and wait[cur] > 500:
            ends = sorted(end[p] for p in prod[int(dep[cur])])
            cands = [p for p in prod[int(dep[cur])] if end[p] <= rdy[cur] + 500]
            if cands:
                nxt = max(cands, key=lambda p: end[p])
        if nxt < 0:
            nxt = int(prev[cur])
        cur = nxt
    path.reverse()
    print(f"critical path: {len(path)} tasks")
    for p in path:
        print(f"  {'F' if dirn[p] == 0 else 'B'} node {node[p]:5d} s {s[p]:4d} f {f[p]:4d} r0 {r0[p]:4d} "
              f"c0 {c0[p]:4d} np {np_[p]} mode {mode[p]}  deq {deq[p] / 1e3:7.1f} rdy {rdy[p] / 1e3:7.1f} "
              f"end {end[p] / 1e3:7.1f}")


if __name__ == "__main__":
    main(sys.argv[1], len(sys.argv) > 2)
