"""Host check of the coarse dataflow program (coarse_coop.cu coop_build) for ONE front:
rebuilds the task DAG with the same rules, executes the tasks with numpy in random
topological orders (any order the dependencies allow), and compares [X; W21] and the
update block with a dense reference. A missing dependency shows up as an order-dependent
result. Usage: python tools/df_program_check.py s b [trials]"""
import sys
import numpy as np

T = 64
G = 4


def build(s, f):
    np_ = -(-s // T)
    Tt = -(-f // T)
    tasks = []  # dict(type, a, b, arg, deps=[(ctr, tgt)], sigs=[(ctr, w)])
    ctr = {}

    def c(name):
        if name not in ctr:
            ctr[name] = 0
        return name

    def upd(I, J):
        return c(("upd", I, J))

    def tiles_of(r0, r1):
        return r0 // T, (min(r1, f) - 1) // T

    def dep_tile(deps, r0, c0, p):
        if p <= 0:
            return
        ri, ci = tiles_of(r0, r0 + T), tiles_of(c0, c0 + T)
        for I in range(ri[0], ri[1] + 1):
            for J in range(ci[0], ci[1] + 1):
                if I >= J:
                    deps.append((upd(I, J), p))

    tot = dict(sy=0, ts=0)
    tasks.append(dict(type="PT", a=0, b=0, arg=0, deps=[], sigs=[(c(("pt", 0)), 1)]))
    ng = -(-s // (G * T))
    for g in range(ng):
        k0, k1 = g * G * T, min(s, (g + 1) * G * T)
        p0, p1 = k0 // T, -(-k1 // T)
        gts = 0
        for p in range(p0, p1):
            k = p * T
            nb = min(T, s - k)
            rest = f - k - nb
            nt = -(-rest // T)
            for a in range(nt):
                d = [(c(("pt", p)), 1)]
                dep_tile(d, k + nb + a * T, k, p)
                tasks.append(dict(type="TS", a=a, b=0, arg=p, deps=d,
                                  sigs=[(c(("tsr", p, a)), 1), (c("tsall"), 1), (c(("gts", g)), 1)]))
                tot["ts"] += 1
                gts += 1
            ncol = -(-(k1 - k - nb) // T)
            for a in range(nt):
                for bb in range(0, min(a, ncol - 1) + 1) if ncol > 0 else []:
                    d = [(c(("tsr", p, a)), 1)]
                    if bb != a:
                        d.append((c(("tsr", p, bb)), 1))
                    dep_tile(d, k + nb + a * T, k + nb + bb * T, p)
                    sg = []
                    if nb == T:
                        sg.append((upd(p + 1 + a, p + 1 + bb), 1))
                    sg.append((c("syall"), 1))
                    if a == 0 and bb == 0 and k + nb < s:
                        sg.append((c(("pt", p + 1)), 1))
                    tasks.append(dict(type="SY", a=a, b=bb, arg=p, deps=d, sigs=sg))
                    tot["sy"] += 1
        ntg = -(-(f - k1) // T)
        for a in range(ntg):
            for bb in range(a + 1):
                d = [(c(("gts", g)), gts)] if gts else []
                dep_tile(d, k1 + a * T, k1 + bb * T, p0)
                sg = []
                if k1 < s:
                    sg.append((upd(p1 + a, p1 + bb), p1 - p0))
                sg.append((c("syall"), 1))
                if a == 0 and bb == 0 and k1 < s:
                    sg.append((c(("pt", p1)), 1))
                tasks.append(dict(type="SYG", a=a, b=bb, arg=g, deps=d, sigs=sg))
                tot["sy"] += 1
    for p in range(np_):
        for cc in range(p):
            for qq in range(p - cc):
                m = cc + qq
                d = [(c(("tsr", m, p - m - 1)), 1), (c(("x2", m, cc)), 1)]
                if p >= 2:
                    d.append((c(("x2row", p - 2)), p - 1))
                tasks.append(dict(type="X1", a=cc, b=qq, arg=p, deps=d, sigs=[(c(("x1", p)), 1)]))
        for cc in range(p + 1):
            d = [(c(("pt", p)), 1), (c("syall"), tot["sy"])]
            if cc < p:
                d.append((c(("x1", p)), p * (p + 1) // 2))
            tasks.append(dict(type="X2", a=cc, b=0, arg=p, deps=d,
                              sigs=[(c(("x2", p, cc)), 1), (c(("x2row", p)), 1), (c(("x2col", cc)), 1)]))
    b = f - s
    for a in range(-(-b // T)) if b > 0 else []:
        for cc in range(np_):
            tasks.append(dict(type="W", a=a, b=cc, arg=0,
                              deps=[(c("tsall"), tot["ts"]), (c(("x2col", cc)), np_ - cc)], sigs=[]))
    return tasks


def run(s, b, order_seed):
    f = s + b
    rng = np.random.default_rng(0)
    M = rng.standard_normal((f, f))
    A = M @ M.T + f * np.eye(f)
    F = np.tril(A).copy()  # lower triangle holds the front
    tasks = build(s, f)
    inv = {}
    Y = {}
    W = np.zeros((b, s))
    ctr = {}
    done = [False] * len(tasks)
    rs = np.random.default_rng(order_seed)

    def ready(t):
        return all(ctr.get(cx, 0) >= tg for cx, tg in t["deps"])

    def potrf_inv(k):
        nb = min(T, s - k)
        D = F[k:k + nb, k:k + nb]
        L = np.linalg.cholesky(np.tril(D) + np.tril(D, -1).T)
        F[k:k + nb, k:k + nb] = L
        inv[k // T] = np.linalg.inv(L)

    X = None
    remaining = list(range(len(tasks)))
    while remaining:
        cand = [i for i in remaining if ready(tasks[i])]
        assert cand, "deadlock"
        i = cand[rs.integers(len(cand))] if order_seed else cand[0]
        remaining.remove(i)
        t = tasks[i]
        ty, a, bb, arg = t["type"], t["a"], t["b"], t["arg"]
        if ty == "PT":
            potrf_inv(0)
        elif ty == "TS":
            k = arg * T
            nb = min(T, s - k)
            r0 = k + nb + a * T
            r1 = min(f, r0 + T)
            F[r0:r1, k:k + nb] = F[r0:r1, k:k + nb] @ inv[arg].T
        elif ty in ("SY", "SYG"):
            if ty == "SY":
                k = arg * T
                nb = min(T, s - k)
                base, kk0, kk1 = k + nb, k, k + nb
            else:
                kk0, kk1 = arg * G * T, min(s, (arg + 1) * G * T)
                base = kk1
            r0, c0 = base + a * T, base + bb * T
            r1, c1 = min(f, r0 + T), min(f, c0 + T)
            if ty == "SY":  # inside the group's block column only
                c1 = min(c1, min(s, (arg // G + 1) * G * T))
            upd_ = F[r0:r1, kk0:kk1] @ F[c0:c1, kk0:kk1].T
            blk = F[r0:r1, c0:c1] - upd_
            if a == bb:
                blk = np.tril(blk)
                F[r0:r1, c0:c1] = blk + np.triu(F[r0:r1, c0:c1], 1)
            else:
                F[r0:r1, c0:c1] = blk
            if a == 0 and bb == 0 and base < s:
                potrf_inv(base)
        elif ty == "X1":
            p, cc, qq = arg, a, bb
            k = p * T
            nb = min(T, s - k)
            c = cc * T
            kq0 = c + qq * T
            kq1 = min(k, kq0 + T)
            Y[(p, cc, qq)] = F[k:k + nb, kq0:kq1] @ F[kq0:kq1, c:c + min(T, k - c)]
        elif ty == "X2":
            p, cc = arg, a
            k = p * T
            nb = min(T, s - k)
            c = cc * T
            if c < k:
                nq = -(-(k - c) // T)
                Ysum = sum(Y[(p, cc, q)] for q in range(nq))
                F[k:k + nb, c:c + T] = -inv[p] @ Ysum
            else:
                F[k:k + nb, k:k + nb] = inv[p]
        elif ty == "W":
            c = bb * T
            r0 = s + a * T
            r1 = min(f, r0 + T)
            W[r0 - s:r1 - s, c:c + min(T, s - c)] = F[r0:r1, c:s] @ F[c:s, c:c + min(T, s - c)]
        for cx, w in t["sigs"]:
            ctr[cx] = ctr.get(cx, 0) + w
    # reference
    L = np.linalg.cholesky(A)
    L11, L21 = L[:s, :s], L[s:, :s]
    Xr = np.linalg.inv(L11)
    Wr = L21 @ Xr
    U = A[s:, s:] - L21 @ L21.T
    eX = np.abs(np.tril(F[:s, :s]) - Xr).max() / np.abs(Xr).max()
    eW = np.abs(W - Wr).max() / max(np.abs(Wr).max(), 1e-300) if b else 0.0
    eU = np.abs(np.tril(F[s:, s:]) - np.tril(U)).max() / np.abs(U).max() if b else 0.0
    return eX, eW, eU, len(tasks)


if __name__ == "__main__":
    s, b = int(sys.argv[1]), int(sys.argv[2])
    trials = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    for seed in range(trials):
        print(seed, "errors X %.2e W %.2e U %.2e (%d tasks)" % run(s, b, seed))
