"""Independent pure-Python pins for the oracle (small inputs only).

Nothing here imports ``oracle/`` or the CUDA package: these are second,
deliberately different formulations of the same definitions, used to pin the
oracle before it is trusted:

* ``enumerate_paths`` -- brute force over every path of the alive induced
  subgraph (Table 2's tl / bl / CP definitions, read
  literally: the costliest path, not a DP);
* ``hop_levels`` -- level[v] = 1 + max level[pred] by memoised recursion over
  predecessors (no queue);
* ``naive_memory`` -- Eq. 3 as explicit intervals per PE and
  a stabbing sum per visit position, instead of the oracle's running tracker.
"""
from __future__ import annotations

import functools
import sys

REMOVED, UNASSIGNED = -1, -2


def comm_prime(part, u, v, w):
    if part is None:
        return w
    if part[u] == UNASSIGNED or part[v] == UNASSIGNED:
        return w
    return 0 if part[u] == part[v] else w


def enumerate_paths(V, src, dst, c, w, part=None):
    """Return (tl, bl, L, cp) by enumerating every path of the alive subgraph.

    tl(n): max over paths ending at n of the path length minus comp(n);
    bl(n): max over paths starting at n of the path length;
    cp: the lexicographically smallest (by node-id sequence) among the
    maximum-length paths that start at an entry node and end at an exit node
    of the alive subgraph.
    """
    alive = [part is None or part[v] != REMOVED for v in range(V)]
    succ = [[] for _ in range(V)]
    pred = [[] for _ in range(V)]
    for k in range(len(src)):
        u, v = int(src[k]), int(dst[k])
        if alive[u] and alive[v]:
            succ[u].append((v, int(w[k])))
            pred[v].append(u)
    tl = [-1] * V
    bl = [-1] * V
    best = [-1, None]

    sys.setrecursionlimit(10000)

    def dfs(path, length):
        n = path[-1]
        tl[n] = max(tl[n], length - int(c[n]))
        # a path starting at path[0] of this length
        s = path[0]
        bl[s] = max(bl[s], length)
        if not pred[s] and not succ[n]:
            if length > best[0] or (length == best[0] and list(path) < best[1]):
                best[0], best[1] = length, list(path)
        for v, wv in succ[n]:
            path.append(v)
            dfs(path, length + comm_prime(part, n, v, wv) + int(c[v]))
            path.pop()

    for v in range(V):
        if alive[v]:
            dfs([v], int(c[v]))
    L = best[0] if best[1] is not None else 0
    cp = best[1] if best[1] is not None else []
    return tl, bl, L, cp


def hop_levels(V, src, dst):
    pred = [[] for _ in range(V)]
    for u, v in zip(src, dst):
        pred[int(v)].append(int(u))

    @functools.lru_cache(maxsize=None)
    def lev(v):
        return 0 if not pred[v] else 1 + max(lev(p) for p in pred[v])

    sys.setrecursionlimit(100000)
    return [lev(v) for v in range(V)]


def naive_memory(V, src, dst, part, P, mem, kind, st, cap_eff):
    """Eq. 3 as intervals on visit positions (reading R8-R12 in DESIGN.md)."""
    level = hop_levels(V, src, dst)
    order = sorted(range(V), key=lambda n: (int(st[n]), level[n], n))
    pos = [0] * V
    for i, n in enumerate(order):
        pos[n] = i
    eff = [0 if int(kind[n]) == 2 else int(mem[n]) for n in range(V)]
    succ = [[] for _ in range(V)]
    pred = [[] for _ in range(V)]
    for u, v in zip(src, dst):
        succ[int(u)].append(int(v))
        pred[int(v)].append(int(u))
    intervals = []  # (owner, pe, start, end, amount, type)
    for n in range(V):
        h = int(part[n])
        lastq = {}
        for u in succ[n]:
            q = int(part[u])
            lastq[q] = max(lastq.get(q, -1), pos[u])
        if int(kind[n]) == 1:  # residual: term 1, whole pass on its PE
            intervals.append((n, h, 0, V - 1, eff[n], "res_home"))
        elif int(kind[n]) == 0:  # normal: terms 2+3 on its own PE
            intervals.append((n, h, pos[n], max(pos[n], lastq.get(h, -1)), eff[n], "home"))
        for q, last in lastq.items():  # term 3 on consumer PEs
            if q != h:
                intervals.append((n, q, pos[n], last, eff[n], "remote"))
    mcons = [[0] * V for _ in range(P)]
    for (_, q, s, e, a, _) in intervals:
        for i in range(s, e + 1):
            mcons[q][i] += a
    peak, ppos, fo, ob = [], [], [], []
    for q in range(P):
        row = mcons[q]
        if V:
            m = max(row)
            peak.append(m)
            ppos.append(row.index(m))
        else:
            peak.append(0)
            ppos.append(-1)
        f = next((i for i in range(V) if row[i] > int(cap_eff[q])), -1)
        fo.append(f)
        ob.append(row[f] - int(cap_eff[q]) if f >= 0 else 0)
    mpot = []
    for n in range(V):
        h = int(part[n])
        tot = eff[n]
        for (o, q, s, e, a, t) in intervals:
            if o != n and q == h and e == pos[n] and t != "res_home":
                tot += a
        mpot.append(tot)
    return dict(mcons=mcons, peak=peak, peak_pos=ppos, first_over=fo, over_bytes=ob, mpot=mpot,
                order=order)


def naive_emulate(V, src, dst, c, w, part, P, level):
    """The TF FIFO scheduler (reading R17) as a TIME-STEPPED
    simulation with per-PE state, integer time t = 0, 1, 2, ... (small costs):
    at each instant, node outputs that arrive at t are counted (an input from
    another PE arrives comm(e) after its producer finishes), a node whose
    inputs have all arrived enters its PE's FIFO queue, and idle PEs start
    queued nodes -- within one instant the entries are started in (entry time,
    level, id) order, and a zero-duration node finishes in the same instant.
    Returns (st, ft, makespan).  Deliberately unlike the oracle's global
    priority queue: no heap, no precomputed ready times."""
    preds = [[] for _ in range(V)]
    succs = [[] for _ in range(V)]
    for k, (a, b) in enumerate(zip(src, dst)):
        preds[b].append(a)
        succs[a].append((b, w[k]))
    arrived = [0] * V
    arrivals = {}                      # time -> list of nodes receiving one input
    queue = [[] for _ in range(P)]     # entries (entry time, level, id)
    running = [None] * P               # (node, end time)
    st, ft = [None] * V, [None] * V
    for v in range(V):
        if not preds[v]:
            queue[part[v]].append((0, level[v], v))
    done, t = 0, 0
    horizon = sum(c) + sum(w) + 1
    while done < V:
        assert t <= horizon, "emulation did not terminate"
        while True:
            # every event of instant t is applied before a PE commits to a node:
            # the inputs arriving at t, then the nodes finishing at t
            if t in arrivals:
                for v in arrivals.pop(t):
                    arrived[v] += 1
                    if arrived[v] == len(preds[v]):
                        queue[part[v]].append((t, level[v], v))
                continue
            fin = [q for q in range(P) if running[q] is not None and running[q][1] == t]
            if fin:
                for q in fin:
                    v = running[q][0]
                    running[q] = None
                    done += 1
                    for s, ws in succs[v]:
                        at = t + (0 if part[s] == part[v] else ws)
                        arrivals.setdefault(at, []).append(s)
                continue
            # then the smallest queued entry of any idle PE starts (one at a time:
            # a zero-duration node finishes within the instant)
            cand = [min(queue[q]) + (q,) for q in range(P) if running[q] is None and queue[q]]
            if not cand:
                break
            _, _, v, q = min(cand)
            queue[q].remove(min(queue[q]))
            st[v], ft[v] = t, t + c[v]
            running[q] = (v, ft[v])
        t += 1
    return st, ft, (max(ft) if V else 0)


def naive_mpot_at(V, src, dst, part, mem, kind, pos, q, i):
    """Table 2's M_pot(n, t) at visit position i on PE q, read
    literally per node n on q (reading R20): the outputs of n's direct
    ancestors executed before t (pos <= i) for which n is the last direct
    descendant on its pe and which still occupy q at t (pos(n) >= i), not
    residual on q, plus n's own memory while it executes (pos(n) == i)."""
    RES, REF = 1, 2
    succ = [[] for _ in range(V)]
    pred = [[] for _ in range(V)]
    for a, b in zip(src, dst):
        succ[a].append(b)
        pred[b].append(a)
    out = [0] * V
    for n in range(V):
        if part[n] != q:
            continue
        tot = mem[n] if (pos[n] == i and kind[n] != REF) else 0
        if pos[n] >= i:
            for p in pred[n]:
                if pos[p] > i or kind[p] == REF or (kind[p] == RES and part[p] == q):
                    continue
                on_q = [s for s in succ[p] if part[s] == q]
                if max(on_q, key=lambda s: pos[s]) == n:
                    tot += mem[p]
        out[n] = tot
    return out
