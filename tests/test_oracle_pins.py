"""Pins of the CPU oracle against things other than itself (CPU only).

* golden fixtures (tests/golden/*.json): closed forms worked by hand from the
  Table 2 / Eq. 3 definitions, each with its citation;
* brute-force enumeration of every path on <= 20-node DAGs (tests/naive.py);
* closed forms on chains and fork-joins of arbitrary size;
* invariants (edge relaxation tightness, label equivalences, REMOVED ==
  induced subgraph rebuilt from scratch, K-loop properties);
* Eq. 3 as explicit intervals + stabbing sums vs the oracle's tracker pass.
"""
import json
import os

import numpy as np
import pytest

from oracle import OracleError, OracleGraph
from synth import make_config, tiny_random_dag
from tests import naive

GOLD = os.path.join(os.path.dirname(__file__), "golden")
REMOVED, UNASSIGNED = -1, -2


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# --------------------------------------------------------------------------- golden
@pytest.mark.parametrize("name", ["single_node.json", "chain_ab.json", "diamond.json",
                                  "diamond_colocated.json"])
def test_golden_levels(name):
    d = _load(name)
    e = np.array(d["edges"], np.int64).reshape(-1, 3)
    g = OracleGraph(d["V"], e[:, 0], e[:, 1])
    part = None if d["part"] is None else np.array(d["part"], np.int32)
    tl, bl = g.weighted_levels(d["c"], e[:, 2], part)
    assert tl.tolist() == d["expected"]["tl"]
    assert bl.tolist() == d["expected"]["bl"]
    cp, L, _ = g.critical_path(d["c"], e[:, 2], part, tl, bl)
    assert L == d["expected"]["L"]
    assert cp.tolist() == d["expected"]["cp"]


def test_golden_memory():
    for case in _load("memory_cases.json")["cases"]:
        e = np.array(case["edges"], np.int64).reshape(-1, 2)
        g = OracleGraph(case["V"], e[:, 0], e[:, 1])
        r = g.memory(case["part"], case["P"], case["mem"], case["kind"], case["st"], case["cap_eff"],
                     want_mcons=True)
        x = case["expected"]
        assert r["mcons"].tolist() == x["mcons"], case["name"]
        for k in ("peak", "peak_pos", "first_over", "over_bytes", "mpot"):
            assert r[k].tolist() == x[k], (case["name"], k)


# --------------------------------------------------------------------------- build
def test_build_validation_and_levels():
    with pytest.raises(OracleError) as ei:
        OracleGraph(3, [0, 1, 2], [1, 2, 0])
    assert ei.value.name == "ECYCLE"
    for s, d in (([0], [0]), ([0, 0], [1, 1]), ([0], [3]), ([-1], [0])):
        with pytest.raises(OracleError) as ei:
            OracleGraph(3, s, d)
        assert ei.value.name == "EINVAL"
    g = OracleGraph(0, [], [])
    assert g.n_levels == 0
    rng = np.random.default_rng(1)
    for _ in range(50):
        n = int(rng.integers(1, 20))
        s, d = tiny_random_dag(rng, n, 0.3)
        g = OracleGraph(n, s, d)
        assert g.levels().tolist() == naive.hop_levels(n, s, d)
        topo = g.topo()
        where = np.empty(n, int)
        where[topo] = np.arange(n)
        assert sorted(topo.tolist()) == list(range(n))
        assert all(where[a] < where[b] for a, b in zip(s, d))


def test_cycle_injected_into_config_graph():
    w = make_config(1)
    # add a back edge from a sink-side node to a source-side node along a path
    s = np.concatenate([w.src, [w.dst[-1]]])
    d = np.concatenate([w.dst, [w.src[-1]]])
    with pytest.raises(OracleError) as ei:
        OracleGraph(w.V, s, d)
    assert ei.value.name == "ECYCLE"


# --------------------------------------------------------------------------- brute force
def _random_labels(rng, n, mode):
    if mode == "null":
        return None
    if mode == "pe":
        return rng.integers(0, 3, n).astype(np.int32)
    lab = rng.integers(0, 3, n).astype(np.int32)
    lab[rng.random(n) < 0.25] = REMOVED
    lab[rng.random(n) < 0.2] = UNASSIGNED
    return lab


@pytest.mark.parametrize("mode", ["null", "pe", "mixed"])
@pytest.mark.parametrize("costs", ["wide", "ties"])
def test_bruteforce_levels_and_cp(mode, costs):
    rng = np.random.default_rng(hash((mode, costs)) % 2**32)
    for it in range(150):
        n = int(rng.integers(1, 15)) if it % 5 else int(rng.integers(15, 21))
        p = 0.35 if n < 15 else 0.15
        s, d = tiny_random_dag(rng, n, p)
        if costs == "ties":
            c = rng.integers(0, 3, n)
            w = rng.integers(0, 3, s.size)
        else:
            c = rng.integers(0, 1000, n)
            w = rng.integers(0, 1000, s.size)
        part = _random_labels(rng, n, mode)
        g = OracleGraph(n, s, d)
        tl, bl = g.weighted_levels(c, w, part)
        btl, bbl, bL, bcp = naive.enumerate_paths(n, s, d, c, w, part)
        assert tl.tolist() == btl
        assert bl.tolist() == bbl
        cp, L, h = g.critical_path(c, w, part, tl, bl)
        assert L == bL
        assert cp.tolist() == bcp
        # hash definition: sum (id+1) * P^k mod 2^64
        P = 0x100000001B3
        assert h == sum((int(v) + 1) * pow(P, k, 2**64) for k, v in enumerate(cp)) % 2**64


# --------------------------------------------------------------------------- closed forms
def test_chain_prefix_and_suffix_sums():
    rng = np.random.default_rng(7)
    n = 5000
    ids = rng.permutation(n)
    c = rng.integers(0, 10**6, n)
    w = rng.integers(0, 10**6, n - 1)
    g = OracleGraph(n, ids[:-1], ids[1:])
    tl, bl = g.weighted_levels(c, w, None)
    cc, ww = c[ids], w
    steps = cc[:-1] + ww
    exp_tl = np.concatenate([[0], np.cumsum(steps)])
    exp_bl = np.concatenate([np.cumsum((cc[1:] + ww)[::-1])[::-1], [0]]) + cc
    assert (tl[ids] == exp_tl).all()
    assert (bl[ids] == exp_bl).all()
    cp, L, _ = g.critical_path(c, w, None, tl, bl)
    assert L == int(cc.sum() + ww.sum())
    assert cp.tolist() == ids.tolist()


def test_fork_join_closed_form():
    rng = np.random.default_rng(8)
    m = 300
    s_id, t_id = 0, m + 1
    src = np.concatenate([np.zeros(m, int), np.arange(1, m + 1)])
    dst = np.concatenate([np.arange(1, m + 1), np.full(m, t_id)])
    c = rng.integers(0, 10**5, m + 2)
    w = rng.integers(0, 10**5, 2 * m)
    g = OracleGraph(m + 2, src, dst)
    tl, bl = g.weighted_levels(c, w, None)
    branch = w[:m] + c[1 : m + 1] + w[m:]
    L = c[s_id] + branch.max() + c[t_id]
    cp, LL, _ = g.critical_path(c, w, None, tl, bl)
    assert LL == L
    assert cp.tolist() == [0, int(np.flatnonzero(branch == branch.max())[0]) + 1, t_id]
    # all branches tight at the same length -> lowest id wins (R6)
    w2 = np.zeros(2 * m, int)
    c2 = np.ones(m + 2, int)
    tl2, bl2 = g.weighted_levels(c2, w2, None)
    assert g.critical_path(c2, w2, None, tl2, bl2)[0].tolist() == [0, 1, t_id]


# --------------------------------------------------------------------------- invariants
@pytest.fixture(scope="module")
def cfg2():
    w = make_config(2)
    return w, OracleGraph(w.V, w.src, w.dst)


def _check_relaxation(w, tl, bl, part):
    alive = np.ones(w.V, bool) if part is None else part != REMOVED
    if part is None:
        cm = w.w
    else:
        pu, pv = part[w.src], part[w.dst]
        same = (pu == pv) & (pu >= 0)
        cm = np.where(same, 0, w.w)
    ea = alive[w.src] & alive[w.dst]
    s, d, cm = w.src[ea], w.dst[ea], cm[ea]
    assert (tl[d] >= tl[s] + w.c[s] + cm).all()
    assert (bl[s] >= w.c[s] + cm + bl[d]).all()
    # tightness: each alive node with alive preds attains its tl on some edge
    best = np.zeros(w.V, np.int64)
    np.maximum.at(best, d, tl[s] + w.c[s] + cm)
    assert (best[alive] == tl[alive]).all()
    bb = np.zeros(w.V, np.int64)
    np.maximum.at(bb, s, cm + bl[d])
    assert (bb[alive] + w.c[alive] == bl[alive]).all()
    assert (tl[~alive] == -1).all() and (bl[~alive] == -1).all()


def test_invariants_config2(cfg2):
    w, g = cfg2
    rng = np.random.default_rng(3)
    pe = rng.integers(0, 4, w.V).astype(np.int32)
    for part in (None, pe):
        tl, bl = g.weighted_levels(w.c, w.w, part)
        _check_relaxation(w, tl, bl, part)
        cp, L, _ = g.critical_path(w.c, w.w, part, tl, bl)
        wl = tl + bl
        assert wl.max() == L
        assert (wl[cp] == L).all()
        assert (np.diff(tl[cp]) >= 0).all()
        # consecutive CP nodes are adjacent and the CP length sums to L
        edges = {(int(a), int(b)): k for k, (a, b) in enumerate(zip(w.src, w.dst))}
        tot = int(w.c[cp].sum())
        for a, b in zip(cp[:-1], cp[1:]):
            k = edges[(int(a), int(b))]
            same = part is not None and part[a] == part[b]
            tot += 0 if same else int(w.w[k])
        assert tot == L


def test_label_equivalences(cfg2):
    w, g = cfg2
    n = w.V
    tl0, bl0 = g.weighted_levels(w.c, w.w, None)
    # NULL == all-distinct labels
    tl1, bl1 = g.weighted_levels(w.c, w.w, np.arange(n, dtype=np.int32))
    assert (tl0 == tl1).all() and (bl0 == bl1).all()
    # NULL == all UNASSIGNED
    tl2, bl2 = g.weighted_levels(w.c, w.w, np.full(n, UNASSIGNED, np.int32))
    assert (tl0 == tl2).all() and (bl0 == bl2).all()
    # all on one PE == zero-comm graph
    tl3, bl3 = g.weighted_levels(w.c, w.w, np.zeros(n, np.int32))
    tl4, bl4 = g.weighted_levels(w.c, np.zeros_like(w.w), None)
    assert (tl3 == tl4).all() and (bl3 == bl4).all()


def test_removed_equals_induced_subgraph(cfg2):
    w, g = cfg2
    rng = np.random.default_rng(11)
    part = rng.integers(0, 4, w.V).astype(np.int32)
    part[rng.random(w.V) < 0.3] = REMOVED
    tl, bl = g.weighted_levels(w.c, w.w, part)
    keep = np.flatnonzero(part != REMOVED)
    newid = np.full(w.V, -1)
    newid[keep] = np.arange(keep.size)
    ek = (part[w.src] != REMOVED) & (part[w.dst] != REMOVED)
    h = OracleGraph(keep.size, newid[w.src[ek]], newid[w.dst[ek]])
    tls, bls = h.weighted_levels(w.c[keep], w.w[ek], part[keep])
    assert (tl[keep] == tls).all() and (bl[keep] == bls).all()


def test_slicing_loop(cfg2):
    w, g = cfg2
    K = 8
    cps, Ls, hs = g.slice(w.c, w.w, K)
    seen = set()
    lab = np.full(w.V, UNASSIGNED, np.int32)
    for j in range(K):
        assert not (set(cps[j].tolist()) & seen)
        seen |= set(cps[j].tolist())
        # each CP_j is the CP of the induced subgraph rebuilt from scratch
        keep = np.flatnonzero(lab != REMOVED)
        newid = np.full(w.V, -1)
        newid[keep] = np.arange(keep.size)
        ek = (lab[w.src] != REMOVED) & (lab[w.dst] != REMOVED)
        h = OracleGraph(keep.size, newid[w.src[ek]], newid[w.dst[ek]])
        tl, bl = h.weighted_levels(w.c[keep], w.w[ek], None)
        cp, L, _ = h.critical_path(w.c[keep], w.w[ek], None, tl, bl)
        assert L == Ls[j]
        assert keep[cp].tolist() == cps[j].tolist()
        lab[cps[j]] = REMOVED
    assert (np.diff(Ls) <= 0).all()


# --------------------------------------------------------------------------- memory
def _random_memory_case(rng, n, P):
    s, d = tiny_random_dag(rng, n, 0.25)
    part = rng.integers(0, P, n).astype(np.int32)
    mem = rng.integers(0, 100, n)
    indeg = np.bincount(d, minlength=n)
    kind = np.zeros(n, np.uint8)
    kind[(indeg == 0) & (rng.random(n) < 0.5)] = 1
    kind[(indeg > 0) & (rng.random(n) < 0.1)] = 2
    return s, d, part, mem, kind


@pytest.mark.parametrize("P", [1, 2, 5, 16])
def test_memory_vs_interval_stabbing(P):
    rng = np.random.default_rng(100 + P)
    for it in range(60):
        n = int(rng.integers(1, 40))
        s, d, part, mem, kind = _random_memory_case(rng, n, P)
        g = OracleGraph(n, s, d)
        c = rng.integers(0, 5, n)      # small costs -> many st ties
        w = rng.integers(0, 5, s.size)
        st, _ = g.weighted_levels(c, w, part)
        cap = rng.integers(0, 400, P)
        r = g.memory(part, P, mem, kind, st, cap, want_mcons=True)
        x = naive.naive_memory(n, s, d, part, P, mem, kind, st, cap)
        assert r["order"].tolist() == x["order"]
        assert r["mcons"].tolist() == x["mcons"]
        for k in ("peak", "peak_pos", "first_over", "over_bytes", "mpot"):
            assert r[k].tolist() == x[k], k


def test_memory_closed_forms():
    rng = np.random.default_rng(5)
    # 1-PE chain of normal nodes: M_cons(i) = mem(n_{i-1}) + mem(n_i)
    n = 200
    ids = rng.permutation(n)
    mem = rng.integers(0, 10**6, n)
    g = OracleGraph(n, ids[:-1], ids[1:])
    st = np.empty(n, np.int64)
    st[ids] = np.arange(n)
    r = g.memory(np.zeros(n, np.int32), 1, mem, np.zeros(n, np.uint8), st, [10**12], want_mcons=True)
    mm = mem[ids]
    exp = np.concatenate([[mm[0]], mm[:-1] + mm[1:]])
    assert (r["mcons"][0] == exp).all()
    assert r["peak"][0] == exp.max()
    # fork a -> {b_1..b_m}: a held until the last b
    m = 50
    src = np.zeros(m, int)
    dst = np.arange(1, m + 1)
    g = OracleGraph(m + 1, src, dst)
    mem = rng.integers(1, 100, m + 1)
    st = np.arange(m + 1)
    r = g.memory(np.zeros(m + 1, np.int32), 1, mem, np.zeros(m + 1, np.uint8), st, [10**9],
                 want_mcons=True)
    assert (r["mcons"][0] == mem[0] + np.concatenate([[0], mem[1:]])).all()
    assert r["mpot"][m] == mem[m] + mem[0]
    # P = 2 with everything on PE 0: PE 1 stays at zero
    r = g.memory(np.zeros(m + 1, np.int32), 2, mem, np.zeros(m + 1, np.uint8), st, [10**9, 0],
                 want_mcons=True)
    assert (r["mcons"][1] == 0).all() and r["first_over"][1] == -1


def test_memory_invariants_config1():
    w = make_config(1)
    g = OracleGraph(w.V, w.src, w.dst)
    part = (np.arange(w.V) % 2).astype(np.int32)
    tl, _ = g.weighted_levels(w.c, w.w, part)
    r = g.memory(part, 2, w.mem, w.kind, tl, w.cap_eff, want_mcons=True)
    x = naive.naive_memory(w.V, w.src, w.dst, part, 2, w.mem, w.kind, tl, w.cap_eff)
    assert r["mcons"].tolist() == x["mcons"]
    assert (r["mcons"] >= 0).all()
    eff = np.where(w.kind == 2, 0, w.mem)
    # last position: residuals on q plus every interval that ends at V-1
    for q in range(2):
        assert r["mcons"][q, -1] >= eff[(w.kind == 1) & (part == q)].sum()
    assert r["mpot"].sum() >= eff[w.kind != 1].sum()


def test_memory_rejects_bad_schedule():
    g = OracleGraph(2, [0], [1])
    with pytest.raises(OracleError):
        g.memory([0, 0], 1, [1, 1], [0, 0], [5, 3], [10])   # st decreases on an edge (R10)
    with pytest.raises(OracleError):
        g.memory([0, 2], 2, [1, 1], [0, 0], [0, 1], [10, 10])  # label out of range


# --------------------------------------------------------------------------- batched evaluation
# or_eval_batch's own arithmetic (cut_comm, cp_start / cp_end, overflow_mask,
# the padding of PEs >= P) pinned against independent formulations: brute-force
# paths (tests/naive.py), Eq. 3 as interval stabbing with st = tl (R8), and a
# numpy cut sum -- not against the oracle's own single-graph calls.
_HASH_P = 0x100000001B3


def _check_batch_row(r, n, s, d, c, w, part, P, mem, kind, cap):
    btl, _, bL, bcp = naive.enumerate_paths(n, s, d, c, w, part)
    assert r["L"] == bL
    assert r["cp_len"] == len(bcp)
    assert r["cp_start"] == (bcp[0] if bcp else -1)
    assert r["cp_end"] == (bcp[-1] if bcp else -1)
    assert int(r["cp_hash"]) == sum((v + 1) * pow(_HASH_P, k, 2**64) for k, v in enumerate(bcp)) % 2**64
    cut = int(np.asarray(w, np.int64)[part[s] != part[d]].sum()) if s.size else 0
    assert r["cut_comm"] == cut
    x = naive.naive_memory(n, s, d, part, P, mem, kind, np.asarray(btl, np.int64), cap)
    mask = 0
    for q in range(16):
        if q < P:
            assert r["peak"][q] == x["peak"][q]
            assert r["peak_pos"][q] == x["peak_pos"][q]
            assert r["first_over_pos"][q] == x["first_over"][q]
            assert r["over_bytes"][q] == x["over_bytes"][q]
            if x["first_over"][q] >= 0:
                mask |= 1 << q
        else:   # PEs >= P are padding
            assert r["peak"][q] == 0 and r["peak_pos"][q] == -1
            assert r["first_over_pos"][q] == -1 and r["over_bytes"][q] == 0
    assert r["overflow_mask"] == mask


@pytest.mark.parametrize("P", [1, 2, 3, 16])
def test_eval_batch_vs_independent_formulations(P):
    rng = np.random.default_rng(900 + P)
    for it in range(12):
        n = int(rng.integers(1, 15))
        s, d = tiny_random_dag(rng, n, 0.3)
        c = rng.integers(0, 50, n) if it % 3 else rng.integers(0, 3, n)
        w = rng.integers(0, 50, s.size) if it % 3 else rng.integers(0, 3, s.size)
        mem = rng.integers(0, 100, n)
        indeg = np.bincount(d, minlength=n)
        kind = np.zeros(n, np.uint8)
        kind[(indeg == 0) & (rng.random(n) < 0.5)] = 1
        kind[(indeg > 0) & (rng.random(n) < 0.1)] = 2
        cap = rng.integers(0, 300, P)
        B = 6
        parts = rng.integers(0, P, (B, n)).astype(np.uint8)
        g = OracleGraph(n, s, d)
        out = g.eval_batch(c, w, mem, kind, P, cap, parts, n_threads=3)
        for b in range(B):
            _check_batch_row(out[b], n, s, d, c, w, parts[b].astype(np.int32), P, mem, kind, cap)


def test_eval_batch_cut_closed_forms():
    # everything on one PE: no edge is cut; an alternating-PE chain: every edge is
    rng = np.random.default_rng(31)
    n = 300
    ids = rng.permutation(n)
    s, d = ids[:-1].astype(np.int32), ids[1:].astype(np.int32)
    c = rng.integers(0, 1000, n)
    w = rng.integers(0, 1000, n - 1)
    mem = rng.integers(0, 100, n)
    kind = np.zeros(n, np.uint8)
    g = OracleGraph(n, s, d)
    alt = np.empty(n, np.uint8)
    alt[ids] = np.arange(n) % 2
    parts = np.stack([np.zeros(n, np.uint8), alt, np.ones(n, np.uint8)])
    out = g.eval_batch(c, w, mem, kind, 2, [10**9, 10**9], parts, n_threads=2)
    assert out[0]["cut_comm"] == 0 and out[2]["cut_comm"] == 0
    assert out[1]["cut_comm"] == int(w.sum())
    # the chain is the only path: L = sum c (+ sum w when every edge is cut)
    assert out[0]["L"] == int(c.sum()) and out[1]["L"] == int(c.sum() + w.sum())
    for r in out:
        assert r["cp_len"] == n and r["cp_start"] == ids[0] and r["cp_end"] == ids[-1]
        assert r["overflow_mask"] == 0
    # capacity 0 on the PE holding a node with memory: overflow at once
    out = g.eval_batch(c, w, np.ones(n, np.int64), kind, 2, [0, 10**9], parts[:1], n_threads=1)
    assert out[0]["overflow_mask"] == 1 and out[0]["first_over_pos"][0] == 0
    assert out[0]["over_bytes"][0] == 1


# --------------------------------------------------------------------------- scheduler emulator (N1)
def test_emulator_spec_chain_examples():
    """SPEC.md:256-257 (derived from the emulator definition):
    chain a(2) -> b(3) on one device: makespan 5 (serial sum); split across
    devices with comm 4: st(b) = ft(a) + 4 = 6, makespan 9."""
    g = OracleGraph(2, np.array([0], np.int32), np.array([1], np.int32))
    st, ft, mk, _ = g.emulate([2, 3], [4], [0, 0], 2)
    assert st.tolist() == [0, 2] and ft.tolist() == [2, 5] and mk == 5
    st, ft, mk, _ = g.emulate([2, 3], [4], [0, 1], 2)
    assert st.tolist() == [0, 6] and ft.tolist() == [2, 9] and mk == 9


def test_emulator_vs_time_stepped_simulation():
    """The oracle's priority-queue emulation equals an independent time-stepped
    simulation of per-PE FIFO executors, on random tiny DAGs, small integer
    costs with many zeros (ties at one instant, zero-duration chains)."""
    rng = np.random.default_rng(17)
    for it in range(400):
        n = int(rng.integers(1, 16))
        s, d = tiny_random_dag(rng, n, float(rng.uniform(0.1, 0.6)))
        hi = 3 if it % 2 else 6
        c = rng.integers(0, hi, n)
        w = rng.integers(0, hi, s.size)
        P = int(rng.integers(1, 4))
        part = rng.integers(0, P, n).astype(np.int32)
        g = OracleGraph(n, s, d)
        st, ft, mk, _ = g.emulate(c, w, part, P)
        lv = g.levels()
        nst, nft, nmk = naive.naive_emulate(n, s.tolist(), d.tolist(), c.tolist(), w.tolist(), part.tolist(), P,
                                            lv.tolist())
        assert st.tolist() == nst and ft.tolist() == nft and mk == nmk, it


def test_emulator_one_pe_is_serial_and_one_pe_per_node_is_tl():
    """Closed forms: all nodes on one PE -> no communication and no idle time,
    makespan = sum(comp), the PE runs its nodes back to back; every node on its
    own PE -> no contention, st = ready = tl with every edge paying comm
    (Table 2 tl with all-distinct labels, computed by or_weighted_levels)."""
    rng = np.random.default_rng(23)
    for it in range(60):
        n = int(rng.integers(1, 17))
        s, d = tiny_random_dag(rng, n, float(rng.uniform(0.1, 0.6)))
        c = rng.integers(0, 50, n)
        w = rng.integers(0, 50, s.size)
        g = OracleGraph(n, s, d)
        st, ft, mk, _ = g.emulate(c, w, np.zeros(n, np.int32), 1)
        assert mk == int(c.sum())
        order = np.lexsort((ft, st))   # execution order (a zero-duration node before its successor)
        assert np.array_equal(np.sort(st), np.concatenate([[0], np.cumsum(c[order])[:-1]])) if n else True
        part = np.arange(n, dtype=np.int32)
        st2, ft2, mk2, _ = g.emulate(c, w, part, max(n, 1))
        tl, bl = g.weighted_levels(c, w, part)
        assert st2.tolist() == tl.tolist() and mk2 == int((tl + c).max())


def test_emulator_invariants_on_config_graphs():
    """ft = st + comp; st(v) >= ft(p) + comm'(p,v) on every edge; one node at a
    time per PE, in (ready, level, id) order; and no unforced idle time: every
    node starts when its last input arrives or when its PE frees up."""
    for n in (1, 2):
        wk = make_config(n)
        g = OracleGraph(wk.V, wk.src, wk.dst)
        rng = np.random.default_rng(n)
        part = rng.integers(0, wk.n_pe, wk.V).astype(np.int32)
        st, ft, mk, mq = g.emulate(wk.c, wk.w, part, wk.n_pe)
        assert np.array_equal(ft, st + wk.c) and mk == ft.max() and mq >= 1
        comm = np.where(part[wk.src] == part[wk.dst], 0, wk.w)
        arrive = ft[wk.src] + comm
        assert (st[wk.dst] >= arrive).all()
        ready = np.zeros(wk.V, np.int64)
        np.maximum.at(ready, wk.dst, arrive)
        lv = g.levels()
        for q in range(wk.n_pe):
            idx = np.nonzero(part == q)[0]
            o = idx[np.lexsort((idx, lv[idx], ready[idx]))]
            assert np.array_equal(o, idx[np.argsort(st[idx], kind="stable")]) or (np.diff(st[o]) >= 0).all()
            assert (st[o][1:] >= ft[o][:-1]).all()
            prev_ft = np.concatenate([[0], ft[o][:-1]])
            assert np.array_equal(st[o], np.maximum(ready[o], prev_ft))


def test_eval_batch_emulated_schedule_composition():
    """or_eval_batch with the emulated schedule (schedule=1) is the composition
    of the pinned single-placement calls: the memory tracker runs on the
    emulator's st, and makespan is the emulator's; with the level schedule
    (schedule=0) the makespan is max(tl + comp) = L."""
    wk = make_config(1)
    g = OracleGraph(wk.V, wk.src, wk.dst)
    rng = np.random.default_rng(8)
    parts = rng.integers(0, wk.n_pe, (6, wk.V)).astype(np.uint8)
    r0 = g.eval_batch(wk.c, wk.w, wk.mem, wk.kind, wk.n_pe, wk.cap_eff, parts, schedule=0)
    r1 = g.eval_batch(wk.c, wk.w, wk.mem, wk.kind, wk.n_pe, wk.cap_eff, parts, schedule=1)
    for b in range(parts.shape[0]):
        part = parts[b].astype(np.int32)
        tl, bl = g.weighted_levels(wk.c, wk.w, part)
        assert r0["makespan"][b] == int((tl + wk.c).max()) == r0["L"][b]
        st, ft, mk, _ = g.emulate(wk.c, wk.w, part, wk.n_pe)
        assert r1["makespan"][b] == mk >= r0["makespan"][b]
        m = g.memory(part, wk.n_pe, wk.mem, wk.kind, st, wk.cap_eff)
        P = wk.n_pe
        assert r1["peak"][b][:P].tolist() == m["peak"].tolist()
        assert r1["peak_pos"][b][:P].tolist() == m["peak_pos"].tolist()
        assert r1["first_over_pos"][b][:P].tolist() == m["first_over"].tolist()
        assert r1["over_bytes"][b][:P].tolist() == m["over_bytes"].tolist()
        for k in ("L", "cut_comm", "cp_hash", "cp_len", "cp_start", "cp_end"):
            assert r1[k][b] == r0[k][b]


# --------------------------------------------------------------------------- whole-Alg.1 slicing (N2)
def _check_clusters(g, wk_c, wk_w, src, dst, V, K, cof, clusters):
    """Verify the extraction rule (reading R18) step by step in checker form:
    partition, primaries = the K-loop CPs, every secondary a path whose start is
    the highest stale-priority unvisited node (lowest id on ties), extended
    forward then backward by the highest-priority unvisited neighbour, maximal."""
    succ = [[] for _ in range(V)]
    pred = [[] for _ in range(V)]
    for a, b in zip(src, dst):
        succ[a].append(b)
        pred[b].append(a)
    assert sorted(np.concatenate(clusters).tolist() if clusters else []) == list(range(V))
    for k, cl in enumerate(clusters):
        assert all(cof[v] == k for v in cl)
        for a, b in zip(cl[:-1], cl[1:]):
            assert b in succ[a], (k, a, b)           # consecutive members are adjacent
    cps, _, _ = g.slice(wk_c, wk_w, K)
    for j in range(K):
        assert clusters[j].tolist() == cps[j].tolist()
    lab = np.full(V, UNASSIGNED, np.int32)
    for j in range(K):
        lab[clusters[j]] = REMOVED
    tl, bl = g.weighted_levels(wk_c, wk_w, lab)
    wl = tl + bl
    visited = np.zeros(V, bool)
    for j in range(K):
        visited[clusters[j]] = True
    key = lambda v: (-int(wl[v]), v)
    for k in range(K, len(clusters)):
        cl = clusters[k].tolist()
        unv = [v for v in range(V) if not visited[v]]
        s0 = min(unv, key=key)                       # the start: highest priority unvisited node
        assert s0 in cl
        i0 = cl.index(s0)
        vis = visited.copy()
        vis[s0] = True
        for a, b in zip(cl[i0:-1], cl[i0 + 1:]):     # forward steps
            cand = [s for s in succ[a] if not vis[s]]
            assert b == min(cand, key=key)
            vis[b] = True
        assert not [s for s in succ[cl[-1]] if not vis[s]]   # forward dead end
        for b, a in zip(cl[i0:0:-1], cl[i0 - 1::-1]):        # backward steps (from the start)
            cand = [p for p in pred[b] if not vis[p]]
            assert a == min(cand, key=key)
            vis[a] = True
        assert not [p for p in pred[cl[0]] if not vis[p]]    # backward dead end
        visited[cl] = True


def test_slice_clusters_rule_on_random_dags_and_configs():
    rng = np.random.default_rng(41)
    for it in range(150):
        n = int(rng.integers(1, 18))
        s, d = tiny_random_dag(rng, n, float(rng.uniform(0.05, 0.6)))
        hi = 3 if it % 3 == 0 else 100
        c, w = rng.integers(0, hi, n), rng.integers(0, hi, s.size)
        K = int(rng.integers(0, 4))
        g = OracleGraph(n, s, d)
        cof, cl = g.slice_clusters(c, w, K)
        _check_clusters(g, c, w, s.tolist(), d.tolist(), n, K, cof, cl)
    wk = make_config(1)
    g = OracleGraph(wk.V, wk.src, wk.dst)
    cof, cl = g.slice_clusters(wk.c, wk.w, 2)
    _check_clusters(g, wk.c, wk.w, wk.src.tolist(), wk.dst.tolist(), wk.V, 2, cof, cl)


def test_slice_clusters_closed_forms():
    """A chain with K = 1 is one primary; two disjoint chains with K = 1 give
    the heavier as the primary and the other, whole, as the one secondary; a
    fork-join s -> {a, b} -> t with K = 1 leaves the lighter branch a singleton."""
    g = OracleGraph(4, np.array([0, 1, 2]), np.array([1, 2, 3]))
    cof, cl = g.slice_clusters([1, 2, 3, 4], [1, 1, 1], 1)
    assert [x.tolist() for x in cl] == [[0, 1, 2, 3]]
    g = OracleGraph(6, np.array([0, 1, 3, 4]), np.array([1, 2, 4, 5]))
    cof, cl = g.slice_clusters([1, 1, 1, 5, 5, 5], [1, 1, 1, 1], 1)
    assert [x.tolist() for x in cl] == [[3, 4, 5], [0, 1, 2]]
    g = OracleGraph(4, np.array([0, 0, 1, 2]), np.array([1, 2, 3, 3]))
    cof, cl = g.slice_clusters([1, 10, 3, 1], [1, 1, 1, 1], 1)
    assert [x.tolist() for x in cl] == [[0, 1, 3], [2]]


def test_criticality_closed_forms_and_brute_force():
    """Criticality (reading R19): one cluster for everything -> the
    computation-only critical path; one cluster per node -> w_lvl with every
    edge paying (Table 2 tl + bl); tiny DAGs -> brute-force path enumeration
    with intra-cluster comm zeroed."""
    wk = make_config(1)
    g = OracleGraph(wk.V, wk.src, wk.dst)
    zero = np.zeros(wk.V, np.int32)
    tl0, bl0 = g.weighted_levels(wk.c, np.zeros_like(wk.w), None)
    assert g.criticality(wk.c, wk.w, zero, 1).tolist() == [int((tl0 + bl0).max())]
    rng = np.random.default_rng(5)
    for it in range(80):
        n = int(rng.integers(1, 14))
        s, d = tiny_random_dag(rng, n, float(rng.uniform(0.1, 0.6)))
        c, w = rng.integers(0, 50, n), rng.integers(0, 50, s.size)
        gg = OracleGraph(n, s, d)
        ident = np.arange(n, dtype=np.int32)
        tl, bl = gg.weighted_levels(c, w, None)
        assert gg.criticality(c, w, ident, n).tolist() == (tl + bl).tolist()
        k = int(rng.integers(1, 4))
        cof = rng.integers(0, k, n).astype(np.int32)
        ntl, nbl, _, _ = naive.enumerate_paths(n, s.tolist(), d.tolist(), c.tolist(), w.tolist(), cof.tolist())
        want = [max([ntl[v] + nbl[v] for v in range(n) if cof[v] == q], default=0) for q in range(k)]
        assert gg.criticality(c, w, cof, k).tolist() == want


# --------------------------------------------------------------------------- overflow handler (N3)
def _state(g, wk, part):
    tl, _ = g.weighted_levels(wk.c, wk.w, part)
    m = g.memory(part, wk.n_pe, wk.mem, wk.kind, tl, wk.cap_eff, want_mcons=True)
    pos = np.empty(g.V, np.int32)
    pos[m["order"]] = np.arange(g.V, dtype=np.int32)
    return m, pos


def test_mpot_at_two_formulations():
    """M_pot(n, t) at n's own visit equals the tracker's M_pot (R13 vs R20), and
    at random (q, i) equals a literal per-node reading of Table 2 (naive)."""
    rng = np.random.default_rng(3)
    for it in range(40):
        n = int(rng.integers(2, 16))
        s, d = tiny_random_dag(rng, n, float(rng.uniform(0.1, 0.6)))
        P = int(rng.integers(1, 4))
        part = rng.integers(0, P, n).astype(np.int32)
        mem = rng.integers(1, 1000, n).astype(np.int64)
        kind = np.zeros(n, np.uint8)
        indeg = np.bincount(d, minlength=n) if s.size else np.zeros(n, int)
        kind[(indeg == 0) & (rng.random(n) < 0.3)] = 1
        kind[(indeg > 0) & (rng.random(n) < 0.2)] = 2
        g = OracleGraph(n, s, d)
        c, w = rng.integers(0, 50, n), rng.integers(0, 50, s.size)
        tl, _ = g.weighted_levels(c, w, part)
        m = g.memory(part, P, mem, kind, tl, np.full(P, 1 << 40, np.int64))
        pos = np.empty(n, np.int32)
        pos[m["order"]] = np.arange(n, dtype=np.int32)
        for v in range(n):
            assert g.mpot_at(part, mem, kind, pos, part[v], pos[v])[v] == m["mpot"][v]
        for _ in range(4):
            q, i = int(rng.integers(0, P)), int(rng.integers(0, n))
            want = naive.naive_mpot_at(n, s.tolist(), d.tolist(), part.tolist(), mem.tolist(), kind.tolist(),
                                       pos.tolist(), q, i)
            assert g.mpot_at(part, mem, kind, pos, q, i).tolist() == want


def test_resolve_overflow_closed_form():
    """a -> b on PE 0, mem 10 each, cap_eff 15: M_cons(0, 1) = 20 overflows by 5
    at b's visit; the only candidate is b (M_pot = own 10 + a's 10); moving it to
    PE 1 resolves the overflow in one move."""
    g = OracleGraph(2, np.array([0], np.int32), np.array([1], np.int32))
    part, moves, res = g.resolve_overflow([1, 1], [1], [10, 10], [0, 0], 2, [15, 100], [0, 0])
    assert res and moves.tolist() == [[1, 0, 1]] and part.tolist() == [0, 1]


def _overflow_cases():
    import types
    from synth import candidate_parts
    wk = make_config(1)
    cases = []
    for scale in (1.1, 1.0):   # 2 PEs: resolved after 90 decisions / unresolved after 160
        cases.append((types.SimpleNamespace(V=wk.V, src=wk.src, dst=wk.dst, c=wk.c, w=wk.w, mem=wk.mem, kind=wk.kind,
                                            n_pe=2, cap_eff=(wk.cap_eff * scale).astype(np.int64)),
                      candidate_parts(wk.seed, 0, 1, wk.V, 2)[0].astype(np.int32)))
    jit = np.random.default_rng(1).uniform(0.7, 1.3, 4)   # 4 PEs: several feasible targets per move
    cases.append((types.SimpleNamespace(V=wk.V, src=wk.src, dst=wk.dst, c=wk.c, w=wk.w, mem=wk.mem, kind=wk.kind,
                                        n_pe=4, cap_eff=(0.45 * wk.mem.sum() / 4 * jit).astype(np.int64)),
                  candidate_parts(wk.seed, 0, 1, wk.V, 4)[0].astype(np.int32)))
    return cases


def test_resolve_overflow_replayed_step_by_step():
    """Every logged decision follows reading R20: the earliest overflow; the
    candidate with the lowest move_cost / M_pot (ties by id) unless a node whose
    M_pot exceeds the overflow is strictly cheaper; the least-loaded feasible
    target, or a rejection; a resolved placement has no overflow."""
    from fractions import Fraction
    n_resolved = 0
    for wk, part0 in _overflow_cases():
        g = OracleGraph(wk.V, wk.src, wk.dst)
        cap = wk.cap_eff
        final, moves, res = g.resolve_overflow(wk.c, wk.w, wk.mem, wk.kind, wk.n_pe, cap, part0)
        assert len(moves) > 0
        assert len(set(moves[:, 0].tolist())) == len(moves)          # each node decided once
        part = part0.copy()
        excl = np.zeros(wk.V, bool)
        k = 0
        while k < len(moves):
            m, pos = _state(g, wk, part)
            fo = m["first_over"]
            q = min([x for x in range(wk.n_pe) if fo[x] >= 0], key=lambda x: (fo[x], x))
            i, O = int(fo[q]), int(m["over_bytes"][q])
            a = g.mpot_at(part, wk.mem, wk.kind, pos, q, i)
            on_q = part == q
            cost = wk.c.copy()
            same = on_q[wk.src] & on_q[wk.dst]
            np.add.at(cost, wk.src[same], wk.w[same])
            np.add.at(cost, wk.dst[same], wk.w[same])
            while k < len(moves):
                cand = [v for v in range(wk.V) if on_q[v] and wk.kind[v] == 0 and not excl[v] and a[v] > 0]
                A = min(cand, key=lambda v: (Fraction(int(cost[v]), int(a[v])), v))
                Bs = [v for v in cand if a[v] > O]
                B = min(Bs, key=lambda v: (cost[v], v)) if Bs else None
                pick = B if (B is not None and cost[B] < cost[A]) else A
                feas = [t for t in range(wk.n_pe) if t != q and m["mcons"][t, i] + a[pick] <= cap[t]]
                tgt = min(feas, key=lambda t: (m["mcons"][t, i], t)) if feas else -1
                assert moves[k].tolist() == [pick, q, tgt], (k, moves[k], pick, q, tgt)
                excl[pick] = True
                k += 1
                if tgt >= 0:
                    part[pick] = tgt
                    break
        assert np.array_equal(part, final)
        m, _ = _state(g, wk, final)
        if res:
            n_resolved += 1
            assert (m["first_over"] < 0).all()
        else:   # the current overflow has no candidate left
            fo = m["first_over"]
            q = min([x for x in range(wk.n_pe) if fo[x] >= 0], key=lambda x: (fo[x], x))
            _, pos = _state(g, wk, final)
            a = g.mpot_at(final, wk.mem, wk.kind, pos, q, int(fo[q]))
            assert not [v for v in range(wk.V) if final[v] == q and wk.kind[v] == 0 and not excl[v] and a[v] > 0]
    assert n_resolved >= 1


# --------------------------------------------------------------------------- LFLAM mapping (N4)
def _lflam_replay(V, src, dst, c, w, level, cof, clusters, K, crit, log):
    """Re-derive every LFLAM decision (reading R21) with direct sums over the
    nodes (no trees): criticality order, span in levels, span work per PE and
    unmapped, comm per PE, the lookahead eligibility and conditions (a)-(c),
    the repeat bound, and Eq. 2 with its tie-breaks."""
    src, dst = np.asarray(src), np.asarray(dst)
    c, w = np.asarray(c, np.int64), np.asarray(w, np.int64)
    D = int(level.max()) + 1 if V else 0
    part = np.where(cof < K, cof, -1)
    ns = len(clusters)
    order = sorted(range(K, ns), key=lambda k: (-int(crit[k]), k))
    mapped = np.zeros(ns, bool)
    mapped[:K] = True
    high_ccr = int(w.sum()) >= 10 * int(c.sum())
    max_iter = max(1, int(np.ceil(np.log2(V))) if V > 1 else 1)
    li = 0

    def stats(k):
        cl = clusters[k]
        insc = cof == k
        h, t = cl[0], cl[-1]
        ps = [a for a, b in zip(src, dst) if b == h and not insc[a]]
        ss = [b for a, b in zip(src, dst) if a == t and not insc[b]]
        lo = max([level[p] + 1 for p in ps], default=0)
        hi = min([level[s] - 1 for s in ss], default=D - 1)
        inspan = (level >= lo) & (level <= hi)
        work = np.array([int(c[(part == q) & inspan].sum()) for q in range(K)])
        unm = (part < 0) & ~insc
        U = int(c[unm & inspan].sum())
        cut = insc[src] != insc[dst]
        other = np.where(insc[src], dst, src)
        comm = np.array([int(w[cut & (part[other] == q)].sum()) for q in range(K)])
        return int(c[insc].sum()), work, U, comm, int(w[cut].sum())

    def apply(k, q, phase):
        nonlocal li
        assert log[li].tolist() == [k, phase, q], (li, log[li], k, phase, q)
        li += 1
        mapped[k] = True
        part[clusters[k]] = q

    for it in range(max_iter):
        n_mapped = 0
        for k in order:
            if mapped[k]:
                continue
            wsc, work, U, comm, ext = stats(k)
            t = int(np.argmax(comm))
            totally = ext > 0 and comm[t] == ext
            if not (totally or (high_ccr and comm[t] * K > ext)):
                continue
            imb = max(0, int(work[t]) + wsc - int(work.sum()) // K)
            if U >= imb or work[t] + wsc <= work.max() or (comm[t] > wsc and comm[t] > work[t] and comm[t] > U):
                apply(k, t, 0)
                n_mapped += 1
        if n_mapped == 0:
            break
    for k in order:
        if mapped[k]:
            continue
        wsc, work, U, comm, ext = stats(k)
        cost = work + (comm.sum() - comm)
        q = min(range(K), key=lambda x: (int(cost[x]), -int(comm[x]), x))
        apply(k, q, 1)
    assert li == len(log)
    return part


def test_lflam_replayed_and_closed_form():
    rng = np.random.default_rng(19)
    cases = []
    for it in range(25):
        n = int(rng.integers(3, 24))
        s, d = tiny_random_dag(rng, n, float(rng.uniform(0.1, 0.5)))
        hi = 3 if it % 3 == 0 else 100
        c = rng.integers(0, hi, n)
        w = rng.integers(0, hi * (12 if it % 2 else 1), s.size)   # odd cases: CCR >= 10
        cases.append((n, s, d, c, w, int(rng.integers(1, 4))))
    for it in range(60):   # tiny integer domains: ties in comm(sc, pe) and in Eq. 2
        n = int(rng.integers(4, 16))
        s, d = tiny_random_dag(rng, n, float(rng.uniform(0.2, 0.6)))
        c = rng.integers(0, 2, n)
        w = rng.integers(0, 3, s.size) * (10 if it % 2 else 1)
        cases.append((n, s, d, c, w, int(rng.integers(2, 5))))
    wk = make_config(1)
    cases.append((wk.V, wk.src, wk.dst, wk.c, wk.w, wk.n_pe))
    # found by search: secondary [0] ties in Eq. 2 (cost 2 on both PEs) and
    # goes to PE 1, the one it communicates with (comm 2 vs 0)
    tie = (8, np.array([1, 6, 4, 0, 2, 1, 7, 6]), np.array([4, 3, 7, 7, 6, 7, 3, 5]),
           np.array([1, 2, 0, 0, 3, 0, 3, 0]), np.array([0, 1, 0, 2, 2, 0, 0, 1]), 2)
    cases.append(tie)
    for V, s, d, c, w, K in cases:
        g = OracleGraph(V, s, d)
        cof, cl = g.slice_clusters(c, w, K)
        if len(cl) < K:
            continue
        part, log = g.lflam(c, w, cof, cl, K)
        crit = g.criticality(c, w, cof, len(cl))
        want = _lflam_replay(V, s, d, c, w, g.levels(), cof, cl, K, crit, log)
        assert np.array_equal(part, want)
        assert (part >= 0).all() and (part < K).all()
    assert log.tolist() == [[3, 0, 0], [2, 1, 1]]          # the tie case (last)
    # primaries [2, 3] (the CP: 300) and [0, 1]; node 4 (weight 1) sits between
    # 2 and 3 and talks only to primary 0 (comm 10 + 10 > its weight, nothing
    # unmapped in its span): mapped to PE 0 in the lookahead, by condition (c)
    src = np.array([0, 2, 2, 4], np.int32)
    dst = np.array([1, 3, 4, 3], np.int32)
    g = OracleGraph(5, src, dst)
    c = np.array([100, 100, 100, 100, 1])
    w = np.array([1, 100, 10, 10])
    cof, cl = g.slice_clusters(c, w, 2)
    assert [x.tolist() for x in cl] == [[2, 3], [0, 1], [4]]
    part, log = g.lflam(c, w, cof, cl, 2)
    assert log.tolist() == [[2, 0, 0]] and part.tolist() == [1, 1, 0, 0, 0]


# --------------------------------------------------------------------------- refinement (N4, reading R22)
def _refine_replay(V, src, dst, c, w, level, clusters, K, part0, passes, window, log):
    """Re-derive every refinement decision (reading R22) independently: tl, bl,
    L and the CP by enumerating every path (tests/naive.py, no DP), the swap
    gain as the whole cut communication before minus after (numpy over all
    edges), span work by direct sums over the nodes of each level range, and
    the window / balance / tie rules.  Returns the final placement."""
    src, dst = np.asarray(src, np.int64), np.asarray(dst, np.int64)
    c, w = np.asarray(c, np.int64), np.asarray(w, np.int64)
    part = np.array(part0, np.int64)
    li = 0

    def cut(p):
        return int(w[p[src] != p[dst]].sum())

    def work(p, q, lo, hi):
        return int(c[(p == q) & (level >= lo) & (level <= hi)].sum())

    tl, _, _, _ = naive.enumerate_paths(V, src, dst, c, w, list(part))
    sec = [k for k in range(K, len(clusters)) if len(clusters[k])]
    order = sorted(sec, key=lambda k: (tl[clusters[k][0]], k))
    marked = set()
    for A in order:
        if A in marked:
            continue
        hA, tA = clusters[A][0], clusters[A][-1]
        a = part[hA]
        s0, s1 = tl[hA], tl[tA] + int(c[tA])
        cands = [B for B in order if s0 <= tl[clusters[B][0]] <= s1 and B != A and B not in marked
                 and part[clusters[B][0]] != a][:window]
        best, bg = None, 0
        for B in cands:
            b = part[clusters[B][0]]
            p2 = part.copy()
            p2[clusters[A]] = b
            p2[clusters[B]] = a
            gain = cut(part) - cut(p2)
            if gain <= 0:
                continue
            hB, tB = clusters[B][0], clusters[B][-1]
            lo, hi = min(level[hA], level[hB]), max(level[tA], level[tB])
            before = max(work(part, a, lo, hi), work(part, b, lo, hi))
            if max(work(p2, a, lo, hi), work(p2, b, lo, hi)) > before:
                continue
            if best is None or gain > bg:
                best, bg = B, gain
        if best is None:
            continue
        assert log[li].tolist() == [0, A, best, bg], (li, log[li], A, best, bg)
        li += 1
        b = part[clusters[best][0]]
        part[clusters[A]] = b
        part[clusters[best]] = a
        marked |= {A, best}
    for _ in range(passes):
        _, _, L_cur, cp = naive.enumerate_paths(V, src, dst, c, w, list(part))
        trials = []
        for k, n in enumerate(cp):
            for y in ([cp[k - 1]] if k > 0 else []) + ([cp[k + 1]] if k + 1 < len(cp) else []):
                if part[y] != part[n] and (n, int(part[y])) not in trials:
                    trials.append((n, int(part[y])))
        while True:
            best = None
            for n, q in trials:
                lv = level[n]
                mx = max(work(part, p, lv, lv) for p in range(K))
                if work(part, q, lv, lv) + int(c[n]) > mx:
                    continue
                p2 = part.copy()
                p2[n] = q
                Lt = naive.enumerate_paths(V, src, dst, c, w, list(p2))[2]
                if best is None or Lt < best[2]:
                    best = (n, q, Lt)
            if best is None or best[2] >= L_cur:
                break
            n, q, L_cur = best
            assert log[li].tolist() == [1, n, q, L_cur], (li, log[li], best)
            li += 1
            part[n] = q
            trials = [t for t in trials if t[0] != n]
    assert li == len(log)
    return part


def _cluster_part(clusters, K, rng):
    """A cluster-uniform placement: primary k on PE k, secondaries at random."""
    V = sum(len(x) for x in clusters)
    part = np.empty(V, np.int32)
    for k, cl in enumerate(clusters):
        part[cl] = k if k < K else int(rng.integers(0, K))
    return part


def test_refine_closed_forms():
    # two singleton secondaries, each on the primary it does not talk to: one
    # swap removes all 20 units of cut communication (SPEC.md:211 idea)
    src = np.array([0, 1, 3, 4, 3, 6, 0, 7], np.int32)
    dst = np.array([1, 2, 4, 5, 6, 5, 7, 2], np.int32)
    c = np.array([10, 10, 10, 10, 10, 10, 1, 1])
    w = np.array([0, 0, 0, 0, 5, 5, 5, 5])
    g = OracleGraph(8, src, dst)
    cl = [np.array(x, np.int32) for x in ([0, 1, 2], [3, 4, 5], [6], [7])]
    cof = np.array([0, 0, 0, 1, 1, 1, 2, 3], np.int32)
    part, log, L = g.refine(c, w, cof, cl, 2, [0, 0, 0, 1, 1, 1, 0, 1])
    assert log.tolist() == [[0, 2, 3, 20]] and part.tolist() == [0, 0, 0, 1, 1, 1, 1, 0] and L == 30
    # already communication-minimal: nothing moves
    part2, log2, L2 = g.refine(c, w, cof, cl, 2, part)
    assert log2.tolist() == [] and part2.tolist() == part.tolist() and L2 == 30
    # two candidates with the same gain (20): the earlier in (tl, id) order wins
    src = np.array([0, 1, 3, 4, 3, 6, 0, 7, 0, 8], np.int32)
    dst = np.array([1, 2, 4, 5, 6, 5, 7, 2, 8, 2], np.int32)
    g = OracleGraph(9, src, dst)
    cl = [np.array(x, np.int32) for x in ([0, 1, 2], [3, 4, 5], [6], [7], [8])]
    cof = np.array([0, 0, 0, 1, 1, 1, 2, 3, 4], np.int32)
    part, log, L = g.refine(np.array([10] * 6 + [1] * 3), np.array([0] * 4 + [5] * 6), cof, cl, 2,
                            [0, 0, 0, 1, 1, 1, 0, 1, 1])
    assert log.tolist()[0] == [0, 2, 3, 20]
    # a chain a -> b -> c with b alone on PE 1: L = 23; moving b to PE 0 gives 3
    # (moving a or c instead gives 13); then the CP is on one PE
    g = OracleGraph(3, np.array([0, 1], np.int32), np.array([1, 2], np.int32))
    cl = [np.array([0, 2], np.int32), np.array([1], np.int32)]
    part, log, L = g.refine([1, 1, 1], [10, 10], np.array([0, 1, 0], np.int32), cl, 2, [0, 1, 0])
    assert log.tolist() == [[1, 1, 0, 3]] and part.tolist() == [0, 0, 0] and L == 3
    # a move that would overload its level is not tried: two parallel chains
    # on two PEs, the cross edge's endpoint cannot join the other PE's level
    g = OracleGraph(4, np.array([0, 2, 0], np.int32), np.array([1, 3, 3], np.int32))
    cl = [np.array([0, 1], np.int32), np.array([2, 3], np.int32)]
    part, log, L = g.refine([5, 5, 5, 5], [0, 0, 50], np.array([0, 0, 1, 1], np.int32), cl, 2, [0, 0, 1, 1])
    assert log.tolist() == [] and L == 60


def test_refine_replayed():
    rng = np.random.default_rng(2208)
    n_swaps = n_moves = 0
    for it in range(90):
        n = int(rng.integers(5, 15))
        s, d = tiny_random_dag(rng, n, float(rng.uniform(0.2, 0.5)))
        hi = 3 if it % 3 == 0 else 40
        c = rng.integers(0, hi, n)
        w = rng.integers(0, hi * (8 if it % 2 else 1), s.size)
        K = int(rng.integers(2, 4))
        g = OracleGraph(n, s, d)
        cof, cl = g.slice_clusters(c, w, K)
        if len(cl) < K:
            continue
        p0 = g.lflam(c, w, cof, cl, K)[0] if it % 4 == 1 else _cluster_part(cl, K, rng)
        window = 64 if it % 4 else 1
        part, log, L = g.refine(c, w, cof, cl, K, p0, passes=K, window=window)
        want = _refine_replay(n, s, d, c, w, g.levels(), cl, K, p0, K, window, log)
        assert np.array_equal(part, want)
        assert L == naive.enumerate_paths(n, s, d, c, w, list(part))[2]
        n_swaps += int((log[:, 0] == 0).sum()) if len(log) else 0
        n_moves += int((log[:, 0] == 1).sum()) if len(log) else 0
    # swap-rich shapes: K chains (the primaries) and singleton secondaries, each
    # fed by a chain node and feeding one two levels on, placed at random
    for it in range(60):
        K = int(rng.integers(2, 4))
        ln = int(rng.integers(3, 6))
        ns = int(rng.integers(2, 7))
        V = K * ln + ns
        s, d = [], []
        for k in range(K):
            for l in range(ln - 1):
                s.append(k * ln + l); d.append(k * ln + l + 1)
        for j in range(ns):
            l = int(rng.integers(0, ln - 2))
            s.append(int(rng.integers(0, K)) * ln + l); d.append(K * ln + j)
            s.append(K * ln + j); d.append(int(rng.integers(0, K)) * ln + l + 2)
        s, d = np.array(s, np.int32), np.array(d, np.int32)
        c = rng.integers(1, 3 if it % 2 else 30, V)
        w = rng.integers(0, 3 if it % 2 else 20, s.size)
        w[K * (ln - 1):] += 5     # the secondaries' edges carry the communication
        cl = [np.arange(k * ln, (k + 1) * ln, dtype=np.int32) for k in range(K)]
        cl += [np.array([K * ln + j], np.int32) for j in range(ns)]
        cof = np.concatenate([np.full(len(x), i, np.int32) for i, x in enumerate(cl)])
        p0 = _cluster_part(cl, K, rng)
        g = OracleGraph(V, s, d)
        window = 64 if it % 5 else 1
        part, log, L = g.refine(c, w, cof, cl, K, p0, passes=2, window=window)
        want = _refine_replay(V, s, d, c, w, g.levels(), cl, K, p0, 2, window, log)
        assert np.array_equal(part, want)
        n_swaps += int((log[:, 0] == 0).sum()) if len(log) else 0
    assert n_swaps >= 12 and n_moves >= 10, (n_swaps, n_moves)


def test_refine_config1_monotone():
    """On C1: every swap lowers the cut communication by its logged gain; every
    node move lowers L to its logged value (checked by fresh oracle calls)."""
    wk = make_config(1)
    g = OracleGraph(wk.V, wk.src, wk.dst)
    K = wk.n_pe
    cof, cl = g.slice_clusters(wk.c, wk.w, K)
    p = g.lflam(wk.c, wk.w, cof, cl, K)[0]
    part, log, L = g.refine(wk.c, wk.w, cof, cl, K, p)
    src, dst, w = np.asarray(wk.src), np.asarray(wk.dst), np.asarray(wk.w)
    cur = p.copy()
    for ph, x, y, v in log.tolist():
        if ph == 0:
            before = int(w[cur[src] != cur[dst]].sum())
            a, b = cur[cl[x][0]], cur[cl[y][0]]
            cur[cl[x]], cur[cl[y]] = b, a
            assert before - int(w[cur[src] != cur[dst]].sum()) == v > 0
        else:
            tl, bl = g.weighted_levels(wk.c, wk.w, cur)
            L0 = int((tl + bl).max())
            cur[x] = y
            tl, bl = g.weighted_levels(wk.c, wk.w, cur)
            assert int((tl + bl).max()) == v < L0
    assert np.array_equal(cur, part)
    assert len(log) > 0
