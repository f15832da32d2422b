"""Independent second implementation of the analysis for small integer instances (test pin).

Written separately from oracle/analysis.cpp, in a different style, and -- the point of it -- it never
iterates a recurrence: every least fixed point is found by the closed characterisation
    lfp(F) = min{ t >= 0 : F(t) <= t }     (F monotone non-decreasing)
by a linear scan over integer t up to the cutoff.  Agreement with the oracle on thousands of random
small sets pins the oracle's iteration (start values, convergence test, cutoff handling, dependency
order) and catches index/sign slips that a single implementation could hide.
"""
import math
import random

from gen.inputs import ACCEL, BEST_EFFORT, CPU, CRITICAL, SPIN, SUSPEND, System, cb, flatten, Seg

INF = None  # UNB / UNSCHED


def ceil_div(a, b):
    return -(-a // b)


def mu(t, T):  # Eq.2
    return ceil_div(t, T) + 1


def lfp_scan(F, cutoff):
    for t in range(0, cutoff + 1):
        if F(t) <= t:
            return t
    return INF


def analyse(s: System, comm: int, sound: bool = False):
    chains = s.chains
    # sub-chains
    subs = []  # (chain index, exec, [callback indices])
    for ci, ch in enumerate(chains):
        for j, c in enumerate(ch.cbs):
            if j == 0 or c.exec != ch.cbs[j - 1].exec:
                subs.append([ci, c.exec, []])
            subs[-1][2].append(j)
    prio = {ci: ch.prio for ci, ch in enumerate(chains)}
    period = {ci: ch.T for ci, ch in enumerate(chains)}
    cut = {ci: min(ch.D, ch.T) for ci, ch in enumerate(chains)}
    # accelerator segments: dict id -> info
    segs = []
    for si, (ci, ex, cbs) in enumerate(subs):
        for j in cbs:
            for g in chains[ci].cbs[j].segs:
                if g.kind == ACCEL:
                    n, units, sc, eps, kap = s.accels[g.accel]
                    segs.append(dict(chain=ci, sub=si, cb=j, a=g.accel, u=g.unit,
                                     Astar=g.wcet + (2 * kap if n > 1 else 0), eps=eps))
    # buckets
    bucket = {}
    for a, (n, units, sc, eps, kap) in enumerate(s.accels):
        users = sorted({q["chain"] for q in segs if q["a"] == a}, key=lambda c: -prio[c])
        if users:
            size = math.ceil(len(users) / n)
            for r, c in enumerate(users):
                bucket[(c, a)] = (n - 1) - (r // size)
    same_unit = lambda p, q: p["a"] == q["a"] and p["u"] == q["u"]
    lpb = [max([q["Astar"] for q in segs if same_unit(p, q) and prio[q["chain"]] < prio[p["chain"]]
                and bucket[(q["chain"], q["a"])] == bucket[(p["chain"], p["a"])]] + [0]) for p in segs]
    hps = [[q for q in segs if same_unit(p, q) and prio[q["chain"]] > prio[p["chain"]]] for p in segs]

    H = []
    for i, p in enumerate(segs):
        G = lambda h, i=i, p=p: p["Astar"] + lpb[i] + sum(mu(h, period[q["chain"]]) * q["Astar"] for q in hps[i])
        H.append(lfp_scan(G, cut[p["chain"]]))

    mine = lambda si: [i for i, p in enumerate(segs) if p["sub"] == si]
    E_cb = lambda ci, j: sum(g.wcet for g in chains[ci].cbs[j].segs if g.kind == CPU)
    E = [sum(E_cb(ci, j) for j in cbs) for (ci, ex, cbs) in subs]
    eps_sum = [sum(segs[i]["eps"] for i in mine(si)) for si in range(len(subs))]

    def S(si):
        vals = [H[i] for i in mine(si)]
        return INF if any(v is INF for v in vals) else sum(vals)

    def C(si, R):
        own = mine(si)
        union = {id(q): q for i in own for q in hps[i]}
        return sum(segs[i]["Astar"] + lpb[i] for i in own) + sum(mu(R, period[q["chain"]]) * q["Astar"] for q in union.values())

    def Hstar(si, R):
        s_ = S(si)
        c_ = C(si, R)
        return (c_ if s_ is INF else min(s_, c_)) + eps_sum[si]

    core = lambda si: s.execs[subs[si][1]][0]
    pp = lambda si: s.execs[subs[si][1]][1]
    spins = lambda si: s.execs[subs[si][1]][2] == SPIN
    hp = lambda c: [h for h in range(len(subs)) if h != c and subs[h][1] == subs[c][1] and prio[subs[h][0]] > prio[subs[c][0]]]
    lp = lambda c: [h for h in range(len(subs)) if h != c and subs[h][1] == subs[c][1] and prio[subs[h][0]] < prio[subs[c][0]]]
    hpp = lambda c: [h for h in range(len(subs)) if subs[h][1] != subs[c][1] and core(h) == core(c) and pp(h) > pp(c)]

    R, Hs = {}, {}

    def solve(c):
        if c in R:
            return
        deps = hp(c) + [h for h in hpp(c) if spins(h)]
        for h in deps:
            solve(h)
        if any(R[h] is INF for h in deps):
            R[c] = INF
            return
        B = 0
        for l in lp(c):
            li = subs[l][0]
            for j in subs[l][2]:
                v = E_cb(li, j)
                if sound:
                    for i in mine(l):
                        if segs[i]["cb"] == j:
                            if H[i] is INF:
                                R[c] = INF
                                return
                            v += H[i] + segs[i]["eps"]
                B = max(B, v)

        def F(t):
            v = B + E[c] + Hstar(c, t)
            v += sum(mu(t, period[subs[h][0]]) * (E[h] + Hs[h]) for h in hp(c))
            v += sum(mu(t, period[subs[h][0]]) * (E[h] + (Hs[h] if spins(h) else eps_sum[h])) for h in hpp(c))
            return v

        R[c] = lfp_scan(F, cut[subs[c][0]])
        if R[c] is not INF:
            Hs[c] = Hstar(c, R[c])

    for c in range(len(subs)):
        solve(c)
    out = []
    for ci in range(len(chains)):
        mysubs = [si for si in range(len(subs)) if subs[si][0] == ci]
        if any(R[si] is INF for si in mysubs):
            out.append(INF)
        else:
            out.append(sum(R[si] for si in mysubs) + comm * (len(mysubs) - 1))
    return out


def random_small_system(rng: random.Random, max_chains=4, tmax=60) -> System:
    """Random valid small set with integer times (unit 1), every structural feature exercised."""
    s = System()
    n_acc = rng.randint(1, 2)
    n_cores = rng.randint(1, 2)
    for a in range(n_acc):
        s.accel(buckets=rng.choice([1, 1, 2, 3]), units=rng.choice([1, 1, 2]), server_core=10 + a,
                eps=rng.choice([0, 0, 1]), kappa=rng.choice([0, 1]))
    n_exec = rng.randint(1, 3)
    used = set()
    for x in range(n_exec):
        core = rng.randrange(n_cores)
        while True:
            p = rng.randint(1, 5)
            if (core, p) not in used:
                used.add((core, p))
                break
        s.executor(core=core, prio=p, wait=rng.choice([SUSPEND, SPIN]))
    m = rng.randint(1, max_chains)
    prios = rng.sample(range(1, 20), m)
    for c in range(m):
        T = rng.randint(8, tmax)
        cls = rng.choice([CRITICAL, CRITICAL, BEST_EFFORT])
        D = rng.randint(max(1, T // 2), T) if cls == CRITICAL else rng.randint(max(1, T // 2), T + T // 2)
        ncb = rng.randint(1, 3)
        ex_seq = []
        for j in range(ncb):  # contiguous executor runs
            if j == 0 or rng.random() < 0.3:
                choices = [x for x in range(n_exec) if x not in ex_seq] or [ex_seq[-1]]
                ex_seq.append(rng.choice(choices))
            else:
                ex_seq.append(ex_seq[-1])
        cbs = []
        for j in range(ncb):
            pattern = rng.choice(["C", "CA", "AC", "CAC", "A", "ACA"])
            segs = []
            for k in pattern:
                if k == "C":
                    segs.append(Seg(CPU, rng.randint(1, 3)))
                else:
                    a = rng.randrange(n_acc)
                    segs.append(Seg(ACCEL, rng.randint(1, 4), a, rng.randrange(s.accels[a][1])))
            cbs.append(cb(ex_seq[j], *segs))
        s.chain(T=T, D=D, prio=prios[c], cls=cls, cbs=cbs)
    return s
