"""Naive tick-by-tick simulator of DESIGN.md App. A (D1-D17) for tiny integer instances (test pin).

An independent second implementation of the simulation semantics: Python, no event queue, time
advances one integer unit per tick and every piece of remaining work is decremented by one when it
progresses.  Agreement with oracle/des.cpp (event-driven, jumps to the next event) on random tiny
sets pins the oracle's time-advance, timers, preemption and tie-breaking code.
"""
import math


def buckets_of(s):
    out = {}
    for a, (n, units, sc, eps, kap) in enumerate(s.accels):
        users = sorted({ci for ci, ch in enumerate(s.chains) for c in ch.cbs for g in c.segs
                        if g.kind == 1 and g.accel == a}, key=lambda ci: -s.chains[ci].prio)
        if users:
            g = math.ceil(len(users) / n)
            for r, ci in enumerate(users):
                out[(ci, a)] = n - 1 - r // g
    return out


def simulate(s, horizon, phases, comm):
    B = buckets_of(s)
    ubase, u = [], 0
    for (n, units, sc, eps, kap) in s.accels:
        ubase.append(u)
        u += units
    unit_acc = [a for a, (n, units, *_r) in enumerate(s.accels) for _ in range(units)]
    m = len(s.chains)
    nxt = [0] * m
    insts = {c: [] for c in range(m)}  # live instances: dict(release,k,cb,state,ready_at)
    ex = [dict(job=None, seg=0, phase="none", rem=0, timer=0) for _ in s.execs]
    units = [dict(q=[], state="idle", cur=None, end=0) for _ in unit_acc]
    owner = {}
    seq = [0]
    stats = [dict(mx=0, n=0, miss=0, drop=0, peak=0) for _ in range(m)]

    def exec_of(c, j):
        return s.chains[c].cbs[j].exec

    def ready_at_exec(x):
        return [(c, I) for c in range(m) for I in insts[c] if I["state"] == "ready" and exec_of(c, I["cb"]) == x]

    def begin(x, t):
        e = ex[x]
        c, I = e["job"]
        g = s.chains[c].cbs[I["cb"]].segs[e["seg"]]
        if g.kind == 0:
            e["phase"], e["rem"] = "cpu", g.wcet
        else:
            eps = s.accels[g.accel][3]
            if s.execs[x][2] == 1:
                e["phase"], e["rem"] = "eps_spin", eps
            else:
                e["phase"], e["timer"] = "eps_susp", t + eps

    def seg_done(x, t):
        e = ex[x]
        c, I = e["job"]
        e["seg"] += 1
        if e["seg"] < len(s.chains[c].cbs[I["cb"]].segs):
            begin(x, t)
            return
        if I["cb"] + 1 < len(s.chains[c].cbs):
            nx = exec_of(c, I["cb"] + 1)
            I["cb"] += 1
            if nx == x:
                I["state"] = "ready"
            else:
                I["state"], I["ready_at"] = "transit", t + comm
        else:
            r = t - I["release"]
            stats[c]["mx"] = max(stats[c]["mx"], r)
            stats[c]["n"] += 1
            stats[c]["miss"] += r > s.chains[c].D
            insts[c].remove(I)
        e["job"], e["phase"] = None, "none"

    def runnable(x):
        e = ex[x]
        if e["phase"] == "none":
            return bool(ready_at_exec(x))
        if e["phase"] in ("cpu", "eps_spin"):
            return True
        if e["phase"] == "wait":
            return s.execs[x][2] == 1
        return False

    def pick(uq, exclude=None):
        cands = [r for r in uq if r is not exclude]
        if not cands:
            return None
        return max(cands, key=lambda r: (r["bucket"], r["started"], r["prio"], -r["seq"]))

    for t in range(0, 10 ** 9):
        while True:  # D15
            any_a = False
            while True:
                ch = False
                for ui, U in enumerate(units):
                    if U["state"] in ("swout", "swin") and U["end"] == t:
                        if U["state"] == "swout":
                            U["state"], U["cur"] = "idle", None
                        else:
                            U["state"] = "run"
                        ch = True
                    if U["state"] == "run" and U["cur"]["rem"] == 0:
                        r = U["cur"]
                        U["q"].remove(r)
                        U["state"], U["cur"] = "idle", None
                        seg_done(r["exec"], t)
                        ch = True
                enq = []
                for x, e in enumerate(ex):
                    if e["phase"] == "cpu" and e["rem"] == 0:
                        seg_done(x, t)
                        ch = True
                    elif (e["phase"] == "eps_spin" and e["rem"] == 0) or (e["phase"] == "eps_susp" and e["timer"] == t):
                        e["phase"] = "wait"
                        enq.append(x)
                        ch = True
                enq.sort(key=lambda x: (ex[x]["job"][0], ex[x]["job"][1]["k"]))
                for x in enq:
                    c, I = ex[x]["job"]
                    g = s.chains[c].cbs[I["cb"]].segs[ex[x]["seg"]]
                    units[ubase[g.accel] + g.unit]["q"].append(dict(exec=x, bucket=B[(c, g.accel)], prio=s.chains[c].prio,
                                                                    seq=seq[0], rem=g.wcet, started=False))
                    seq[0] += 1
                for c in range(m):
                    for I in insts[c]:
                        if I["state"] == "transit" and I["ready_at"] == t:
                            I["state"] = "ready"
                            ch = True
                for c in range(m):
                    r = phases[c] + nxt[c] * s.chains[c].T
                    if r != t or r >= horizon:
                        continue
                    if s.chains[c].cls == 1:
                        kept = [I for I in insts[c] if not (I["state"] == "ready" and I["cb"] == 0)]
                        stats[c]["drop"] += len(insts[c]) - len(kept)
                        insts[c] = kept
                    insts[c].append(dict(release=t, k=nxt[c], cb=0, state="ready", ready_at=0))  # D14: queue
                    stats[c]["peak"] = max(stats[c]["peak"], len(insts[c]))
                    nxt[c] += 1
                    ch = True
                if not ch:
                    break
                any_a = True
            chb = False
            for x, e in enumerate(ex):
                if e["phase"] == "none" and owner.get(s.execs[x][0]) == x and ready_at_exec(x):
                    c, I = max(ready_at_exec(x), key=lambda ci: (s.chains[ci[0]].prio, -ci[1]["release"], -ci[1]["cb"]))
                    I["state"] = "running"
                    e["job"], e["seg"] = (c, I), 0
                    begin(x, t)
                    chb = True
            for core in sorted({xc for (xc, _p, _w) in s.execs}):
                cand = [x for x in range(len(ex)) if s.execs[x][0] == core and runnable(x)]
                best = max(cand, key=lambda x: s.execs[x][1]) if cand else None
                if owner.get(core) != best:
                    owner[core] = best
                    chb = True
            for ui, U in enumerate(units):
                n, _u, _sc, _e, kap = s.accels[unit_acc[ui]]
                kap = kap if n > 1 else 0
                if U["state"] == "idle":
                    r = pick(U["q"])
                    if r is not None:
                        U["cur"] = r
                        if r["started"]:
                            U["state"], U["end"] = "swin", t + kap
                        else:
                            r["started"], U["state"] = True, "run"
                        chb = True
                elif U["state"] == "run" and n > 1:
                    r = pick(U["q"], exclude=U["cur"])
                    if r is not None and r["bucket"] > U["cur"]["bucket"]:
                        U["state"], U["end"] = "swout", t + kap
                        chb = True
            if not any_a and not chb:
                break
        # anything left?
        busy = any(insts[c] for c in range(m)) or any(phases[c] + nxt[c] * s.chains[c].T < horizon for c in range(m))
        if not busy and all(U["state"] == "idle" and not U["q"] for U in units):
            break
        # one tick of progress
        for x, e in enumerate(ex):
            if e["phase"] in ("cpu", "eps_spin") and owner.get(s.execs[x][0]) == x:
                e["rem"] -= 1
        for U in units:
            if U["state"] == "run":
                U["cur"]["rem"] -= 1
    return {k: [st[k] for st in stats] for k in ("mx", "n", "miss", "drop", "peak")}
