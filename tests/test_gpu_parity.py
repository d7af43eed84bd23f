"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element, bit-exact (all values are integers).

Covers configs 1-4 of BASELINE.json at full size (the C oracle finishes them
in about a second), the batched evaluation on configs 1-3, and the adversarial
suite: ties, empty / single-node / edgeless / disconnected graphs, a 1e5 chain,
1e5-leaf stars in both directions, costs at the 2^62 bound, P = 1 and P = 16,
validation errors, and determinism across repeated calls.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import OracleGraph  # noqa: E402
from synth import candidate_parts, make_config, tiny_random_dag  # noqa: E402

pytestmark = pytest.mark.gpu

REMOVED, UNASSIGNED = -1, -2


@pytest.fixture(scope="session", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2008_08636_b200 import build

    build.build()


def _G(V, src, dst, c=None, w=None):
    from paper_2008_08636_b200 import Graph

    G = Graph(V, np.asarray(src, np.int32), np.asarray(dst, np.int32))
    if c is not None:
        G.set_costs(np.asarray(c, np.int64), np.asarray(w, np.int64))
    return G


_CACHE = {}


def _cfg(n):
    if n not in _CACHE:
        w = make_config(n)
        _CACHE[n] = (w, OracleGraph(w.V, w.src, w.dst), _G(w.V, w.src, w.dst, w.c, w.w))
    return _CACHE[n]


def _labels(w, mode, seed=0):
    rng = np.random.default_rng(seed)
    if mode == "null":
        return None
    lab = rng.integers(0, w.n_pe, w.V).astype(np.int32)
    if mode == "mixed":
        lab[rng.random(w.V) < 0.2] = REMOVED
        lab[rng.random(w.V) < 0.1] = UNASSIGNED
    return lab


def _gpu_levels(G, part):
    tl, bl = G.weighted_levels(part)
    return tl.cpu().numpy(), bl.cpu().numpy()


def _gpu_cp(G, tl, bl, part):
    cp, scal = G.critical_path(torch.as_tensor(tl).cuda(), torch.as_tensor(bl).cuda(), part)
    return G.unpack_cp(cp, scal)


# ------------------------------------------------------------------- configs
@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_levels_and_canonical_order(n):
    w, og, G = _cfg(n)
    assert G.n_levels == og.n_levels
    assert (G.levels().cpu().numpy() == og.levels()).all()
    perm = G.perm.cpu().numpy()
    assert np.array_equal(np.sort(perm), np.arange(w.E))
    key = w.src[perm].astype(np.int64) * w.V + w.dst[perm]
    assert (np.diff(key) > 0).all()
    indeg = np.bincount(w.dst, minlength=w.V)
    outdeg = np.bincount(w.src, minlength=w.V)
    assert G.max_in == indeg.max() and G.max_out == outdeg.max()


@pytest.mark.parametrize("n", [1, 2, 3, 4])
@pytest.mark.parametrize("mode", ["null", "pe", "mixed"])
def test_weighted_levels_and_cp(n, mode):
    w, og, G = _cfg(n)
    part = _labels(w, mode, seed=n)
    tl_o, bl_o = og.weighted_levels(w.c, w.w, part)
    tl, bl = _gpu_levels(G, part)
    assert np.array_equal(tl, tl_o)
    assert np.array_equal(bl, bl_o)
    cp_o, L_o, h_o = og.critical_path(w.c, w.w, part, tl_o, bl_o)
    cp, L, h = _gpu_cp(G, tl, bl, part)
    assert L == L_o
    assert np.array_equal(cp, cp_o)
    assert h == h_o


def test_per_call_costs_equal_bound_costs():
    w, og, G = _cfg(2)
    perm = G.perm.cpu().numpy()
    part = _labels(w, "pe", 5)
    tl1, bl1 = G.weighted_levels(part)
    tl2, bl2 = G.weighted_levels(part, node_cost=w.c, edge_cost=w.w[perm])   # canonical order
    assert torch.equal(tl1, tl2) and torch.equal(bl1, bl2)
    cp1, s1 = G.critical_path(tl1, bl1, part)
    cp2, s2 = G.critical_path(tl2, bl2, part, node_cost=w.c, edge_cost=w.w[perm])
    assert G.unpack_cp(cp1, s1)[1:] == G.unpack_cp(cp2, s2)[1:]


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_slicing_loop(n):
    w, og, G = _cfg(n)
    K = max(w.K, 2)
    cps_o, Ls_o, hs_o = og.slice(w.c, w.w, K)
    cps, lens, Ls, hs = G.slice(K)
    lens, Ls, hs = lens.cpu().numpy(), Ls.cpu().numpy(), hs.cpu().numpy().view(np.uint64)
    cps = cps.cpu().numpy()
    for j in range(K):
        assert lens[j] == len(cps_o[j])
        assert np.array_equal(cps[j, : lens[j]], cps_o[j])
    assert np.array_equal(Ls, Ls_o)
    assert np.array_equal(hs, hs_o)


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_memory_potential(n):
    w, og, G = _cfg(n)
    part = candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)
    tl_o, _ = og.weighted_levels(w.c, w.w, part)
    want = og.memory(part, w.n_pe, w.mem, w.kind, tl_o, w.cap_eff, want_mcons=(n <= 3))
    tl, _ = G.weighted_levels(part)
    got = G.memory_potential(part, w.n_pe, w.mem, w.kind, tl, w.cap_eff, want_mcons=(n <= 3))
    for k in ("mpot", "peak", "peak_pos", "first_over", "over_bytes"):
        assert np.array_equal(got[k].cpu().numpy(), want[k]), k
    if n <= 3:
        assert np.array_equal(got["mcons"].cpu().numpy(), want["mcons"])


@pytest.mark.parametrize("P", [1, 3, 16])
def test_memory_pe_counts(P):
    w, og, G = _cfg(1)
    part = candidate_parts(11, 0, 1, w.V, P)[0].astype(np.int32)
    st, _ = og.weighted_levels(w.c, w.w, part)
    cap = np.full(P, int(w.cap_eff[0]) // P, np.int64)
    want = og.memory(part, P, w.mem, w.kind, st, cap, want_mcons=True)
    got = G.memory_potential(part, P, w.mem, w.kind, st, cap, want_mcons=True)
    for k in ("mpot", "peak", "peak_pos", "first_over", "over_bytes", "mcons"):
        assert np.array_equal(got[k].cpu().numpy(), want[k]), k


def _compare_results(got, want):
    for f in want.dtype.names:
        assert np.array_equal(got[f], want[f]), f


@pytest.mark.parametrize("n,B", [(1, 70), (2, 6), (3, 40)])
def test_eval_batch(n, B):
    from paper_2008_08636_b200 import Graph

    w, og, G = _cfg(n)
    for mode in ("uniform", "refine"):
        parts = candidate_parts(w.seed, 0, B, w.V, w.n_pe, mode)
        want = og.eval_batch(w.c, w.w, w.mem, w.kind, w.n_pe, w.cap_eff, parts)
        got = Graph.results_to_numpy(G.eval_batch(parts, w.n_pe, w.mem, w.kind, w.cap_eff))
        _compare_results(got, want)


def _batch_check(V, src, dst, c, w, P, B, seed=0, mode="uniform"):
    """pdnn_eval_batch vs the oracle's per-candidate evaluation on random
    placements (uint8 labels in [0, P)), synthetic mem / kinds / capacities."""
    from paper_2008_08636_b200 import Graph

    rng = np.random.default_rng(seed)
    og = OracleGraph(V, src, dst)
    G = _G(V, src, dst, c, w)
    parts = rng.integers(0, P, (B, V)).astype(np.uint8)
    if mode == "refine" and V:
        parts[:] = parts[0]
        flip = rng.random((B, V)) < 0.02
        parts[flip] = rng.integers(0, P, int(flip.sum())).astype(np.uint8)
    mem = rng.integers(0, 1 << 24, V).astype(np.int64)
    kind = np.zeros(V, np.uint8)
    indeg = np.bincount(np.asarray(dst, np.int64), minlength=V) if len(dst) else np.zeros(V, int)
    kind[(indeg == 0) & (rng.random(V) < 0.3)] = 1
    kind[(indeg > 0) & (rng.random(V) < 0.05)] = 2
    cap = rng.integers(1 << 20, 1 << 26, P).astype(np.int64)
    want = og.eval_batch(np.asarray(c, np.int64), np.asarray(w, np.int64), mem, kind, P, cap, parts)
    got = Graph.results_to_numpy(G.eval_batch(parts, P, mem, kind, cap))
    _compare_results(got, want)


@pytest.mark.parametrize("P", [1, 2, 16])
def test_eval_batch_pe_counts(P):
    w = make_config(1)
    _batch_check(w.V, w.src, w.dst, w.c, w.w, P, 37, seed=P)


def test_eval_batch_random_small_dags_and_ties():
    rng = np.random.default_rng(7)
    for it in range(12):
        n = int(rng.integers(1, 21))
        s, d = tiny_random_dag(rng, n, float(rng.uniform(0.05, 0.5)))
        if it % 2:
            c, w = rng.integers(0, 3, n), rng.integers(0, 3, s.size)   # massive ties
        else:
            c, w = rng.integers(0, 1000, n), rng.integers(0, 1000, s.size)
        _batch_check(n, s, d, c, w, int(rng.integers(1, 5)), int(rng.integers(1, 70)), seed=it)
    w1 = make_config(1, mode="ties")
    _batch_check(w1.V, w1.src, w1.dst, w1.c, w1.w, 4, 33, seed=5, mode="refine")


def test_eval_batch_degenerate():
    _batch_check(1, np.zeros(0, np.int32), np.zeros(0, np.int32), [7], [], 2, 5)
    _batch_check(40, np.zeros(0, np.int32), np.zeros(0, np.int32), np.arange(40), [], 3, 33)


@pytest.mark.parametrize("direction", ["out", "in"])
def test_eval_batch_hub_stars(direction):
    n = 20_001   # hubs split into many parts in both sweep directions
    rng = np.random.default_rng(3)
    hub = np.zeros(n - 1, np.int32)
    leaves = np.arange(1, n, dtype=np.int32)
    src, dst = (hub, leaves) if direction == "out" else (leaves, hub)
    _batch_check(n, src, dst, rng.integers(0, 10**6, n), rng.integers(0, 10**6, n - 1), 8, 40, seed=1)
    _batch_check(n, src, dst, np.ones(n, np.int64), np.ones(n - 1, np.int64), 8, 33, seed=2)   # all ties


def test_eval_batch_costs_at_the_bound():
    """st spans ~62 bits: the segmented sort cannot pack (st, rank) into 64 bits
    and moves (key, value) pairs instead."""
    n = 64
    src, dst = np.arange(n - 1, dtype=np.int32), np.arange(1, n, dtype=np.int32)
    lim = (1 << 62) - 1
    c = np.full(n, lim // (2 * n - 1), np.int64)
    w = np.full(n - 1, lim // (2 * n - 1), np.int64)
    c[0] += lim - int(c.sum() + w.sum())
    _batch_check(n, src, dst, c, w, 2, 33, seed=4)
    rng = np.random.default_rng(6)   # plus a fan-out / fan-in so st has ties and branches
    s2 = np.concatenate([src, np.zeros(10, np.int32)]); d2 = np.concatenate([dst, np.arange(64, 74, dtype=np.int32)])
    c2 = np.concatenate([c, rng.integers(0, 1 << 50, 10)]); w2 = np.concatenate([w, rng.integers(0, 1 << 50, 10)])
    c2[0] -= int(c2[64:].sum() + w2[63:].sum())
    _batch_check(74, s2, d2, c2, w2, 3, 40, seed=5)


def test_eval_batch_multi_group_subprocess():
    """B > candidates per group: groups run back to back on one workspace.  The
    group cap is a debug knob, so the subprocess loads the debug-knob build."""
    import os
    import subprocess
    import sys

    code = ("import numpy as np, sys; sys.path.insert(0, '.');"
            "from paper_2008_08636_b200 import _binding, build;"
            "_binding.load_library(build.build(debug_knobs=True));"
            "from tests.test_gpu_parity import _batch_check; from synth import make_config;"
            "w = make_config(1); _batch_check(w.V, w.src, w.dst, w.c, w.w, 4, 100, seed=9);"
            "w = make_config(2); _batch_check(w.V, w.src, w.dst, w.c, w.w, 4, 70, seed=3); print('ok')")
    env = dict(os.environ, PDNN_BATCH_GROUP="32")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def _hub_graph(n=2001, seed=11):
    """A layered graph with out- and in-hubs (split into several batched parts)."""
    rng = np.random.default_rng(seed)
    src = [np.zeros(n - 2, np.int32), np.arange(1, n - 1, dtype=np.int32)]
    dst = [np.arange(1, n - 1, dtype=np.int32), np.full(n - 2, n - 1, np.int32)]
    a = rng.integers(1, n - 2, 3 * n); b = rng.integers(1, n - 2, 3 * n)
    keep = a < b
    pairs = np.unique(np.stack([a[keep], b[keep]], 1), axis=0)
    src.append(pairs[:, 0].astype(np.int32)); dst.append(pairs[:, 1].astype(np.int32))
    s, d = np.concatenate(src), np.concatenate(dst)
    return n, s, d, rng.integers(0, 10**6, n), rng.integers(0, 10**6, s.size)


def test_eval_batch_workspace_reuse_shrinking_batches():
    """ADVICE (round 1): one Graph, one workspace, batch sizes that shrink and
    grow again (the batched region's layout changes with the batch size; the
    workspace guard must reset its persistent state), on a graph with hubs."""
    from paper_2008_08636_b200 import Graph

    n, s, d, c, w = _hub_graph()
    og = OracleGraph(n, s, d)
    G = _G(n, s, d, c, w)
    rng = np.random.default_rng(5)
    P = 4
    mem = rng.integers(0, 1 << 24, n).astype(np.int64)
    kind = np.zeros(n, np.uint8)
    cap = rng.integers(1 << 20, 1 << 26, P).astype(np.int64)
    ws0 = None
    for B in (4096, 2048, 1024, 4096, 96, 4096, 33):
        parts = rng.integers(0, P, (B, n)).astype(np.uint8)
        got = Graph.results_to_numpy(G.eval_batch(parts, P, mem, kind, cap))
        if ws0 is None:
            ws0 = G._ws.data_ptr()
        assert G._ws.data_ptr() == ws0   # the same workspace all along
        want = og.eval_batch(np.asarray(c, np.int64), np.asarray(w, np.int64), mem, kind, P, cap, parts)
        _compare_results(got, want)


def test_eval_batch_odd_chunk_counts():
    """Chunk counts (x 32 candidates) with large odd factors: the launch pads
    the chunk count instead of shrinking the grid or failing."""
    w = make_config(1)
    for B in (139 * 32, 601 * 32 - 5, 307 * 32 + 1):
        _batch_check(w.V, w.src, w.dst, w.c, w.w, 2, B, seed=B)


def test_eval_batch_two_threads_two_streams():
    """Two host threads, each with its own stream and workspace, evaluate
    batches of one graph concurrently; every result equals the oracle's (the
    CP walk's side stream and its fork / join events are per call)."""
    import threading
    from paper_2008_08636_b200 import Graph

    w, og, G0 = _cfg(2)
    Gs = [_G(w.V, w.src, w.dst, w.c, w.w) for _ in range(2)]
    B = 64
    parts = [candidate_parts(w.seed, 1000 * t, 1000 * t + B, w.V, w.n_pe, "uniform") for t in range(2)]
    want = [og.eval_batch(w.c, w.w, w.mem, w.kind, w.n_pe, w.cap_eff, p) for p in parts]
    errors = []

    def run(t):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                pt = torch.as_tensor(parts[t]).cuda()
                for _ in range(6):
                    out = Gs[t].eval_batch(pt, w.n_pe, w.mem, w.kind, w.cap_eff, stream=st)
                    st.synchronize()
                    _compare_results(Graph.results_to_numpy(out), want[t])
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=run, args=(t,)) for t in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors


def test_workspace_shared_by_two_graphs():
    """One caller workspace used alternately by two different graphs (the C ABI
    allows it): the layout guard resets the persistent state on every switch."""
    wa, oa, Ga = _cfg(1)
    wb, ob, Gb = _cfg(2)
    ws = torch.zeros(max(Ga.workspace().numel(), Gb.workspace().numel()), dtype=torch.uint8, device="cuda")
    Ga._ws, Gb._ws = ws, ws
    Ga._ws_bytes = Gb._ws_bytes = ws.numel()
    for G, wk, og in ((Ga, wa, oa), (Gb, wb, ob), (Ga, wa, oa), (Gb, wb, ob)):
        part = _labels(wk, "pe", seed=3)
        tl, bl = _gpu_levels(G, part)
        tl_o, bl_o = og.weighted_levels(wk.c, wk.w, part)
        assert np.array_equal(tl, tl_o) and np.array_equal(bl, bl_o)
        m = G.memory_potential(part, wk.n_pe, wk.mem, wk.kind, torch.as_tensor(tl).cuda(), wk.cap_eff)
        m_o = og.memory(part, wk.n_pe, wk.mem, wk.kind, tl_o, wk.cap_eff)
        for k in ("mpot", "peak", "peak_pos", "first_over", "over_bytes"):
            assert np.array_equal(m[k].cpu().numpy(), m_o[k]), k


def test_determinism_repeated_calls():
    w, og, G = _cfg(3)
    part = _labels(w, "pe", 9)
    ref = None
    for _ in range(7):   # > 3 epochs: the tag cycle wraps
        tl, bl = G.weighted_levels(part)
        cp, s = G.critical_path(tl, bl, part)
        cur = (tl.cpu().numpy(), bl.cpu().numpy(), G.unpack_cp(cp, s))
        if ref is None:
            ref = cur
        else:
            assert np.array_equal(cur[0], ref[0]) and np.array_equal(cur[1], ref[1])
            assert np.array_equal(cur[2][0], ref[2][0]) and cur[2][1:] == ref[2][1:]
        tl, bl = G.weighted_levels(None)  # interleave another label mode
    # a fresh workspace gives the same answer
    G._ws = None
    tl2, _ = G.weighted_levels(part)
    assert np.array_equal(tl2.cpu().numpy(), ref[0])


# ------------------------------------------------------------------- adversarial
def _full_check(V, src, dst, c, w, parts=(None,), K=2, P=2):
    og = OracleGraph(V, src, dst)
    G = _G(V, src, dst, c, w)
    assert G.n_levels == og.n_levels
    for part in parts:
        tl_o, bl_o = og.weighted_levels(c, w, part)
        tl, bl = _gpu_levels(G, part)
        assert np.array_equal(tl, tl_o) and np.array_equal(bl, bl_o)
        cp_o, L_o, h_o = og.critical_path(c, w, part, tl_o, bl_o)
        cp, L, h = _gpu_cp(G, tl, bl, part)
        assert (L, h) == (L_o, h_o) and np.array_equal(cp, cp_o)
    if V:
        cps_o, Ls_o, _ = og.slice(c, w, K)
        cps, lens, Ls, _ = G.slice(K)
        assert np.array_equal(Ls.cpu().numpy(), Ls_o)
        for j in range(K):
            assert np.array_equal(cps[j, : int(lens[j])].cpu().numpy(), cps_o[j])
        rng = np.random.default_rng(V)
        lab = rng.integers(0, P, V).astype(np.int32)
        mem = rng.integers(0, 1 << 20, V).astype(np.int64)
        kind = np.zeros(V, np.uint8)
        indeg = np.bincount(dst, minlength=V) if len(dst) else np.zeros(V, int)
        kind[(indeg == 0) & (rng.random(V) < 0.3)] = 1
        kind[(indeg > 0) & (rng.random(V) < 0.1)] = 2
        st, _ = og.weighted_levels(c, w, lab)
        cap = rng.integers(0, 1 << 22, P).astype(np.int64)
        want = og.memory(lab, P, mem, kind, st, cap, want_mcons=V <= 200_000)
        got = G.memory_potential(lab, P, mem, kind, st, cap, want_mcons=V <= 200_000)
        for k in ("mpot", "peak", "peak_pos", "first_over", "over_bytes") + (("mcons",) if V <= 200_000 else ()):
            assert np.array_equal(got[k].cpu().numpy(), want[k]), k


def test_random_small_dags():
    rng = np.random.default_rng(42)
    for it in range(60):
        n = int(rng.integers(1, 21))
        s, d = tiny_random_dag(rng, n, float(rng.uniform(0.05, 0.5)))
        if it % 3 == 0:
            c, w = rng.integers(0, 3, n), rng.integers(0, 3, s.size)
        else:
            c, w = rng.integers(0, 1000, n), rng.integers(0, 1000, s.size)
        lab = rng.integers(0, 3, n).astype(np.int32)
        mix = lab.copy()
        mix[rng.random(n) < 0.3] = REMOVED
        mix[rng.random(n) < 0.2] = UNASSIGNED
        _full_check(n, s, d, c, w, parts=(None, lab, mix), K=3, P=int(rng.integers(1, 5)))


def test_all_zero_costs_maximal_ties():
    w = make_config(1)
    z = np.zeros(w.V, np.int64)
    _full_check(w.V, w.src, w.dst, z, np.zeros(w.E, np.int64),
                parts=(None, _labels(w, "pe", 1), _labels(w, "mixed", 2)))
    w1 = make_config(1, mode="ties")
    _full_check(w1.V, w1.src, w1.dst, w1.c, w1.w, parts=(None, _labels(w1, "pe", 3)))


def test_tiny_and_degenerate_graphs():
    _full_check(1, [], [], [5], [])
    _full_check(50, [], [], np.arange(50), [], parts=(None, np.arange(50, dtype=np.int32) % 3))
    a = make_config(1)
    V2 = 2 * a.V
    src = np.concatenate([a.src, a.src + a.V])
    dst = np.concatenate([a.dst, a.dst + a.V])
    _full_check(V2, src, dst, np.concatenate([a.c, a.c[::-1]]), np.concatenate([a.w, a.w]))


def test_empty_graph_and_all_removed():
    from paper_2008_08636_b200 import Graph

    G = Graph(0, np.zeros(0, np.int32), np.zeros(0, np.int32))
    G.set_costs(np.zeros(0, np.int64), np.zeros(0, np.int64))
    assert G.n_levels == 0
    cps, lens, Ls, hs = G.slice(2)
    assert lens.cpu().tolist() == [0, 0]
    w, og, G = _cfg(1)
    tl, bl = G.weighted_levels(np.full(w.V, REMOVED, np.int32))
    assert (tl == -1).all() and (bl == -1).all()
    cp, s = G.critical_path(tl, bl, np.full(w.V, REMOVED, np.int32))
    assert G.unpack_cp(cp, s)[1:] == (0, 0)


def test_long_chain():
    n = 100_000
    rng = np.random.default_rng(1)
    ids = rng.permutation(n).astype(np.int32)
    c = rng.integers(0, 10**6, n)
    w = rng.integers(0, 10**6, n - 1)
    _full_check(n, ids[:-1], ids[1:], c, w, parts=(None, rng.integers(0, 4, n).astype(np.int32)), K=2)


@pytest.mark.parametrize("direction", ["out", "in"])
def test_hub_stars(direction):
    n = 100_001
    rng = np.random.default_rng(2)
    hub = np.zeros(n - 1, np.int32)
    leaves = np.arange(1, n, dtype=np.int32)
    src, dst = (hub, leaves) if direction == "out" else (leaves, hub)
    c = rng.integers(0, 10**6, n)
    w = rng.integers(0, 10**6, n - 1)
    lab = rng.integers(0, 8, n).astype(np.int32)
    mix = lab.copy()
    mix[rng.random(n) < 0.3] = REMOVED
    _full_check(n, src, dst, c, w, parts=(None, lab, mix), K=3, P=8)
    # equal-length branches: the lowest id wins every tie
    _full_check(n, src, dst, np.ones(n, np.int64), np.ones(n - 1, np.int64), parts=(None,), K=2)


def test_costs_at_the_overflow_bound():
    from paper_2008_08636_b200 import Graph, PdnnError

    n = 64
    src, dst = np.arange(n - 1, dtype=np.int32), np.arange(1, n, dtype=np.int32)
    lim = (1 << 62) - 1
    c = np.full(n, lim // (2 * n - 1), np.int64)
    w = np.full(n - 1, lim // (2 * n - 1), np.int64)
    c[0] += lim - int(c.sum() + w.sum())        # total == 2^62 - 1: accepted
    _full_check(n, src, dst, c, w)
    G = Graph(n, src, dst)
    c2 = c.copy()
    c2[0] += 1                                   # total == 2^62: rejected
    with pytest.raises(PdnnError) as ei:
        G.set_costs(c2, w)
    assert ei.value.name == "PDNN_EOVERFLOW"
    c3 = c.copy()
    c3[5] = -1
    with pytest.raises(PdnnError) as ei:
        G.set_costs(c3, w)
    assert ei.value.name == "PDNN_EOVERFLOW"


def test_build_errors():
    from paper_2008_08636_b200 import Graph, PdnnError

    cases = [((3, [0, 1, 2], [1, 2, 0]), "PDNN_ECYCLE"), ((3, [0], [0]), "PDNN_EINVAL"),
             ((3, [0, 0], [1, 1]), "PDNN_EINVAL"), ((3, [0], [3]), "PDNN_EINVAL"),
             ((3, [-1], [0]), "PDNN_EINVAL")]
    for args, name in cases:
        with pytest.raises(PdnnError) as ei:
            Graph(args[0], np.array(args[1], np.int32), np.array(args[2], np.int32))
        assert ei.value.name == name
    w = make_config(2)
    with pytest.raises(PdnnError) as ei:
        Graph(w.V, np.concatenate([w.src, [w.dst[0]]]), np.concatenate([w.dst, [w.src[0]]]))
    assert ei.value.name == "PDNN_ECYCLE"


def test_native_library_is_loaded():
    import paper_2008_08636_b200 as P

    before = P.launch_count()
    w, og, G = _cfg(1)
    G.weighted_levels(None)
    torch.cuda.synchronize()
    assert P.launch_count() > before
    maps = open("/proc/self/maps").read()
    assert "libpdnn.so" in maps


@pytest.mark.parametrize("mode", ["uniform", "refine"])
def test_eval_batch_full_size_c5_all(mode):
    """Config 5 at BASELINE.json's full size, in bench.py's launch configuration
    (all 4,096 candidates of the TRN-shaped graph in one pdnn_eval_batch call),
    EVERY candidate compared with the oracle (run on all host cores), in both
    candidate distributions (uniform iid and refinement trials)."""
    from paper_2008_08636_b200 import Graph

    w = make_config(5)
    B = 4096
    parts_h = np.empty((B, w.V), np.uint8)
    for b0 in range(0, B, 256):   # host generation in chunks (the generator's temporaries are 8 B per label)
        parts_h[b0:b0 + 256] = candidate_parts(w.seed, b0, b0 + 256, w.V, w.n_pe, mode)
    parts = torch.as_tensor(parts_h).cuda()
    G = _G(w.V, w.src, w.dst, w.c, w.w)
    got = Graph.results_to_numpy(G.eval_batch(parts, w.n_pe, w.mem, w.kind, w.cap_eff))
    assert got.shape[0] == B
    del parts
    og = OracleGraph(w.V, w.src, w.dst)
    want = og.eval_batch(w.c, w.w, w.mem, w.kind, w.n_pe, w.cap_eff, parts_h)
    _compare_results(got, want)


def test_memory_pe16_many_tiles():
    """P = 16 (the widest per-PE scan) over ~120 scan tiles of the TRN graph."""
    w, og, G = _cfg(3)
    P = 16
    part = candidate_parts(17, 0, 1, w.V, P)[0].astype(np.int32)
    st, _ = og.weighted_levels(w.c, w.w, part)
    cap = np.full(P, int(w.mem.sum()) // (4 * P), np.int64)
    want = og.memory(part, P, w.mem, w.kind, st, cap)
    got = G.memory_potential(part, P, w.mem, w.kind, st, cap)
    for k in ("mpot", "peak", "peak_pos", "first_over", "over_bytes"):
        assert np.array_equal(got[k].cpu().numpy(), want[k]), k


def test_memory_at_the_bounds():
    """Single placement with st near 2^62 (the chunked sort cannot pack
    (st, rank) into 64 bits and moves key / value pairs) and sum(mem) just
    under 2^61 (large positive and negative scan-tile aggregates in the
    look-back words), on the Word-RNN graph (30 scan tiles)."""
    w = make_config(2)
    rng = np.random.default_rng(61)
    E = w.src.size
    cap_each = ((1 << 62) - 1) // (w.V + E)
    c = rng.integers(0, cap_each, w.V).astype(np.int64)
    wc = rng.integers(0, cap_each, E).astype(np.int64)
    og = OracleGraph(w.V, w.src, w.dst)
    G = _G(w.V, w.src, w.dst, c, wc)
    P = 4
    part = rng.integers(0, P, w.V).astype(np.int32)
    st, _ = og.weighted_levels(c, wc, part)
    assert int(st.max()).bit_length() + int(w.V - 1).bit_length() > 64
    mem = rng.integers(0, ((1 << 61) - 1) // w.V, w.V).astype(np.int64)
    assert int(mem.sum()) < (1 << 61)
    cap = np.full(P, int(mem.sum()) // (2 * P), np.int64)
    want = og.memory(part, P, mem, w.kind, st, cap, want_mcons=True)
    got = G.memory_potential(part, P, mem, w.kind, st, cap, want_mcons=True)
    for k in ("mpot", "peak", "peak_pos", "first_over", "over_bytes", "mcons"):
        assert np.array_equal(got[k].cpu().numpy(), want[k]), k


@pytest.mark.parametrize("n", [1, 2])
def test_cuda_graph_replay(n):
    """The whole single-graph step (K slicing sweeps + CP, placement sweep, CP,
    memory tracker) captured once in a CUDA graph (cooperative launches,
    memsets and all) and replayed with new placements written into the
    captured input: every replay equals the oracle (the library keeps its
    per-call state -- sweep epochs, tickets, look-back words -- on the device)."""
    w, og, G = _cfg(n)
    K = w.K
    part_d = torch.empty(w.V, dtype=torch.int32, device="cuda")
    part_d.copy_(torch.as_tensor(candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)))
    mem = torch.as_tensor(w.mem).cuda()
    kind = torch.as_tensor(w.kind).cuda()
    cap = torch.as_tensor(w.cap_eff).cuda()
    G.workspace()
    outs = {}

    def step():
        outs["slice"] = G.slice(K)
        tl, bl = G.weighted_levels(part_d)
        outs["lv"] = (tl, bl)
        outs["cp"] = G.critical_path(tl, bl, part_d)
        outs["mem"] = G.memory_potential(part_d, w.n_pe, mem, kind, tl, cap)

    step()   # warm-up outside the capture (first-call attribute setup)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    cps_o, L_o, h_o = og.slice(w.c, w.w, K)
    for rep in range(3):
        part = candidate_parts(w.seed, rep + 1, rep + 2, w.V, w.n_pe, "uniform")[0].astype(np.int32)
        part_d.copy_(torch.as_tensor(part))
        g.replay()
        torch.cuda.synchronize()
        cps, lens, Ls, hs = outs["slice"]
        for j in range(K):
            assert np.array_equal(cps[j, : int(lens[j])].cpu().numpy(), cps_o[j])
        assert np.array_equal(Ls.cpu().numpy(), L_o)
        tl_o, bl_o = og.weighted_levels(w.c, w.w, part)
        assert np.array_equal(outs["lv"][0].cpu().numpy(), tl_o) and np.array_equal(outs["lv"][1].cpu().numpy(), bl_o)
        cp_g, L, h = G.unpack_cp(*outs["cp"])
        cp_o, Lc_o, hc_o = og.critical_path(w.c, w.w, part, tl_o, bl_o)
        assert np.array_equal(cp_g, cp_o) and L == Lc_o and h == hc_o
        m_o = og.memory(part, w.n_pe, w.mem, w.kind, tl_o, w.cap_eff)
        for k in ("mpot", "peak", "peak_pos", "first_over", "over_bytes"):
            assert np.array_equal(outs["mem"][k].cpu().numpy(), m_o[k]), k


# ------------------------------------------------------------------- scheduler emulator (N1)
@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_emulate_vs_oracle(n):
    """pdnn_emulate (one warp per placement) equals the oracle's emulation:
    st, ft of every node and the makespan, for two placements per config
    (C3's ready queue peaks at ~22.7k entries -- the heap spills from shared
    to global memory; C4 starts with 318,750 queued entries)."""
    w, og, G = _cfg(n)
    for mode in ("uniform", "refine"):
        part = candidate_parts(w.seed, 0, 1, w.V, w.n_pe, mode)[0].astype(np.int32)
        st, ft, mk = G.emulate(part, w.n_pe)
        st_o, ft_o, mk_o, _ = og.emulate(w.c, w.w, part, w.n_pe)
        assert np.array_equal(st.cpu().numpy(), st_o) and np.array_equal(ft.cpu().numpy(), ft_o)
        assert int(mk.item()) == mk_o


def test_emulate_random_small_dags_and_ties():
    rng = np.random.default_rng(31)
    for it in range(40):
        n = int(rng.integers(1, 30))
        s, d = tiny_random_dag(rng, n, float(rng.uniform(0.05, 0.5)))
        hi = 3 if it % 2 else 1000
        c, w = rng.integers(0, hi, n), rng.integers(0, hi, s.size)
        P = int(rng.integers(1, 5))
        part = rng.integers(0, P, n).astype(np.int32)
        og = OracleGraph(n, s, d)
        G = _G(n, s, d, c, w)
        st, ft, mk = G.emulate(part, P)
        st_o, ft_o, mk_o, _ = og.emulate(c, w, part, P)
        assert np.array_equal(st.cpu().numpy(), st_o) and np.array_equal(ft.cpu().numpy(), ft_o), it
        assert int(mk.item()) == mk_o


@pytest.mark.parametrize("direction", ["out", "in"])
def test_emulate_hub_stars(direction):
    n = 20_001   # 20k nodes released at once (out-hub): the heap spills to global memory
    rng = np.random.default_rng(4)
    hub = np.zeros(n - 1, np.int32)
    leaves = np.arange(1, n, dtype=np.int32)
    src, dst = (hub, leaves) if direction == "out" else (leaves, hub)
    c, w = rng.integers(0, 10**6, n), rng.integers(0, 10**6, n - 1)
    part = rng.integers(0, 8, n).astype(np.int32)
    st, ft, mk = _G(n, src, dst, c, w).emulate(part, 8)
    st_o, ft_o, mk_o, _ = OracleGraph(n, src, dst).emulate(c, w, part, 8)
    assert np.array_equal(st.cpu().numpy(), st_o) and int(mk.item()) == mk_o


@pytest.mark.parametrize("n,B", [(1, 70), (2, 6), (3, 8)])
def test_eval_batch_emulated_schedule(n, B):
    """pdnn_eval_batch on the emulated FIFO schedule: the memory tracker visits
    nodes in emulated-st order; every field (makespan included) equals the
    oracle's evaluation with schedule=1."""
    from paper_2008_08636_b200 import Graph

    w, og, G = _cfg(n)
    for mode in ("uniform", "refine"):
        parts = candidate_parts(w.seed, 0, B, w.V, w.n_pe, mode)
        want = og.eval_batch(w.c, w.w, w.mem, w.kind, w.n_pe, w.cap_eff, parts, schedule=1)
        got = Graph.results_to_numpy(G.eval_batch(parts, w.n_pe, w.mem, w.kind, w.cap_eff, schedule=1))
        _compare_results(got, want)


def test_memory_potential_default_st_is_tl():
    """st = NULL: the tracker runs on the level schedule st = tl under the
    placement (reading R8), computed inside the call from the bound costs."""
    w, og, G = _cfg(2)
    part = candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)
    m = G.memory_potential(part, w.n_pe, w.mem, w.kind, None, w.cap_eff)
    tl_o, _ = og.weighted_levels(w.c, w.w, part)
    m_o = og.memory(part, w.n_pe, w.mem, w.kind, tl_o, w.cap_eff)
    for k in ("mpot", "peak", "peak_pos", "first_over", "over_bytes"):
        assert np.array_equal(m[k].cpu().numpy(), m_o[k]), k


def test_validate():
    from paper_2008_08636_b200 import PdnnError

    w, og, G = _cfg(1)
    part = candidate_parts(w.seed, 0, 1, w.V, w.n_pe)[0].astype(np.int32)
    tl, _ = og.weighted_levels(w.c, w.w, part)
    st, _, _, _ = og.emulate(w.c, w.w, part, w.n_pe)
    perm = G.perm.cpu().numpy()
    wc = w.w[perm]                                   # canonical edge order
    G.validate(w.c, wc, part, w.n_pe, w.mem, w.kind, tl)
    G.validate(part=part, n_pe=w.n_pe, st=st)        # the emulated schedule is a valid visit order
    G.validate(part=np.where(part == 0, -1, part).astype(np.int32), n_pe=0)   # REMOVED labels for the sweep

    def bad(status, **kw):
        with pytest.raises(PdnnError) as ei:
            G.validate(**kw)
        assert ei.value.name == status, (status, kw.keys())

    c2 = w.c.copy(); c2[5] = -1
    bad("PDNN_EOVERFLOW", node_cost=c2, edge_cost=wc)
    c3 = w.c.copy(); c3[7] = (1 << 62) - int(w.c.sum() + wc.sum()) + int(w.c[7])
    bad("PDNN_EOVERFLOW", node_cost=c3, edge_cost=wc)
    p2 = part.copy(); p2[3] = w.n_pe
    bad("PDNN_EINVAL", part=p2, n_pe=w.n_pe)
    k2 = w.kind.copy(); k2[9] = 3
    bad("PDNN_EINVAL", kind=k2)
    m2 = w.mem.copy(); m2[0] = 1 << 61
    bad("PDNN_EOVERFLOW", mem=m2)
    s2 = tl.copy(); e0 = int(np.nonzero(tl[w.dst] > 0)[0][0]); s2[w.dst[e0]] = tl[w.src[e0]] - 1
    bad("PDNN_EINVAL", st=s2)


# ------------------------------------------------------------------- whole-Alg.1 slicing and criticality (N2)
def _gpu_clusters(G, K, c=None, w=None):
    cof, mem, off, nc = G.slice_clusters(K, c, w)
    n = int(nc.item())
    off = off.cpu().numpy()[: n + 1]
    mem = mem.cpu().numpy()
    return cof.cpu().numpy(), [mem[off[i]:off[i + 1]] for i in range(n)]


@pytest.mark.parametrize("n", [1, 2, 3])
def test_slice_clusters_vs_oracle(n):
    """Primaries, stale-priority secondaries (reading R18) and the criticality
    of every cluster (R19) equal the oracle's, node for node."""
    w, og, G = _cfg(n)
    cof, cl = _gpu_clusters(G, w.K)
    cof_o, cl_o = og.slice_clusters(w.c, w.w, w.K)
    assert np.array_equal(cof, cof_o)
    assert len(cl) == len(cl_o) and all(np.array_equal(a, b) for a, b in zip(cl, cl_o))
    crit = G.criticality(cof, len(cl)).cpu().numpy()
    assert np.array_equal(crit, og.criticality(w.c, w.w, cof_o, len(cl_o)))


def test_slice_clusters_random_small_dags_and_ties():
    rng = np.random.default_rng(12)
    for it in range(30):
        n = int(rng.integers(1, 30))
        s, d = tiny_random_dag(rng, n, float(rng.uniform(0.05, 0.5)))
        hi = 3 if it % 2 else 1000
        c, w = rng.integers(0, hi, n), rng.integers(0, hi, s.size)
        K = int(rng.integers(0, 4))
        og = OracleGraph(n, s, d)
        G = _G(n, s, d, c, w)
        cof, cl = _gpu_clusters(G, K)
        cof_o, cl_o = og.slice_clusters(c, w, K)
        assert np.array_equal(cof, cof_o), it
        assert len(cl) == len(cl_o) and all(np.array_equal(a, b) for a, b in zip(cl, cl_o)), it
        crit = G.criticality(cof, len(cl)).cpu().numpy()
        assert np.array_equal(crit, og.criticality(c, w, cof_o, len(cl_o))), it


# ------------------------------------------------------------------- overflow handler (N3)
def test_resolve_overflow_vs_oracle():
    """pdnn_resolve_overflow takes exactly the oracle's decisions (reading R20):
    the same move / rejection log, final placement and outcome, on 2-PE cases
    that resolve (90 decisions) and run out of candidates (160), and on a 4-PE
    case with several feasible targets per move."""
    from tests.test_oracle_pins import _overflow_cases

    for wk, part0 in _overflow_cases():
        og = OracleGraph(wk.V, wk.src, wk.dst)
        want_part, want_moves, want_res = og.resolve_overflow(wk.c, wk.w, wk.mem, wk.kind, wk.n_pe, wk.cap_eff, part0)
        G = _G(wk.V, wk.src, wk.dst, wk.c, wk.w)
        part, moves, res = G.resolve_overflow(part0, wk.n_pe, wk.mem, wk.kind, wk.cap_eff)
        assert res == want_res
        assert np.array_equal(moves, want_moves)
        assert np.array_equal(part.cpu().numpy(), want_part)


@pytest.mark.parametrize("n,scale", [(2, 1.0), (3, 1.6)])
def test_resolve_overflow_config_graphs(n, scale):
    w, og, G = _cfg(n)
    part0 = candidate_parts(w.seed, 0, 1, w.V, w.n_pe, "refine")[0].astype(np.int32)
    cap = (w.cap_eff * scale).astype(np.int64)
    want_part, want_moves, want_res = og.resolve_overflow(w.c, w.w, w.mem, w.kind, w.n_pe, cap, part0, max_moves=40)
    part, moves, res = G.resolve_overflow(part0, w.n_pe, w.mem, w.kind, cap, max_moves=40)
    assert res == want_res and np.array_equal(moves, want_moves)
    assert np.array_equal(part.cpu().numpy(), want_part)


# ------------------------------------------------------------------- LFLAM mapping (N4)
def _flat_clusters(cl):
    members = np.concatenate(cl).astype(np.int32) if len(cl) else np.zeros(0, np.int32)
    off = np.zeros(len(cl) + 1, np.int32)
    off[1:] = np.cumsum([len(x) for x in cl])
    return members, off


def _lflam_check(G, og, c, w, K, bound=True):
    cof_o, cl_o = og.slice_clusters(c, w, K)
    if len(cl_o) < K:
        return None
    want_part, want_log = og.lflam(c, w, cof_o, cl_o, K)
    members, off = _flat_clusters(cl_o)
    per_call = () if bound else (c, np.asarray(w)[G.perm.cpu().numpy()])     # canonical edge order
    part, log = G.lflam(cof_o, members, off, len(cl_o), K, *per_call)
    assert np.array_equal(log.cpu().numpy(), want_log)
    assert np.array_equal(part.cpu().numpy(), want_part)
    return want_log


@pytest.mark.parametrize("n", [1, 2, 6, 3, 7, 4])
def test_lflam_vs_oracle(n):
    """pdnn_lflam takes exactly the oracle's decisions (reading R21) -- the
    same (cluster, phase, PE) log and placement -- on the config graphs
    (C1/C2/C6: placement and trees in shared memory; C3 (D = 4,111) and C7
    (D = 90,902): both in global memory; C4 (1.5M nodes, D = 64): trees in
    shared, placement in global memory), and chained after pdnn_slice_clusters."""
    w, og, G = _cfg(n)
    log = _lflam_check(G, og, w.c, w.w, w.K)
    assert (log[:, 1] == 0).any() and (log[:, 1] == 1).any()      # both phases decide
    cof, mem, off, nc = G.slice_clusters(w.K)
    part, log2 = G.lflam(cof, mem, off, int(nc.item()), w.K)
    assert np.array_equal(log2.cpu().numpy(), log)


def test_lflam_random_small_dags_and_ties():
    """Tiny integer domains (ties in comm and in Eq. 2), high-CCR cases, K up to
    4, costs bound and per call."""
    rng = np.random.default_rng(21)
    done = 0
    for it in range(60):
        n = int(rng.integers(3, 40))
        s, d = tiny_random_dag(rng, n, float(rng.uniform(0.1, 0.6)))
        if it % 3 == 0:
            c, w = rng.integers(0, 2, n), rng.integers(0, 3, s.size) * (10 if it % 2 else 1)
        else:
            c, w = rng.integers(0, 100, n), rng.integers(0, 100 * (12 if it % 2 else 1), s.size)
        K = int(rng.integers(1, 5))
        og = OracleGraph(n, s, d)
        G = _G(n, s, d, c, w) if it % 2 else _G(n, s, d)
        done += _lflam_check(G, og, c, w, K, bound=bool(it % 2)) is not None
    assert done > 40


def test_lflam_global_state_subprocess():
    """The global-memory state path (forced by a debug knob) on C2 and on tie
    cases gives the same decisions."""
    import os
    import subprocess
    import sys

    code = ("import numpy as np, sys; sys.path.insert(0, '.');"
            "from paper_2008_08636_b200 import _binding, build;"
            "_binding.load_library(build.build(debug_knobs=True));"
            "from tests.test_gpu_parity import _lflam_check, _cfg, test_lflam_random_small_dags_and_ties;"
            "w, og, G = _cfg(2); _lflam_check(G, og, w.c, w.w, w.K);"
            "test_lflam_random_small_dags_and_ties(); print('ok')")
    env = dict(os.environ, PDNN_LFLAM_GLOBAL="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


# ------------------------------------------------------------------- refinement (N4, reading R22)
def _refine_check(G, og, c, w, cof, cl, K, part0, passes=None, window=64, bound=True):
    want_part, want_log, want_L = og.refine(c, w, cof, cl, K, part0, passes=passes, window=window)
    members, off = _flat_clusters(cl)
    per_call = {} if bound else dict(node_cost=c, edge_cost=np.asarray(w)[G.perm.cpu().numpy()])
    part, log, L = G.refine(cof, members, off, len(cl), K, part0, passes=passes, window=window, **per_call)
    assert log.tolist() == want_log.tolist()
    assert np.array_equal(part.cpu().numpy(), want_part)
    assert L == want_L
    return want_log


@pytest.mark.parametrize("n", [1, 6, 2])
def test_refine_vs_oracle(n):
    """pdnn_refine takes exactly the oracle's decisions (reading R22) -- the
    same swap / move log, placement and final L -- after LFLAM on the config
    graphs, and from a random cluster-uniform placement (more swaps)."""
    w, og, G = _cfg(n)
    cof, cl = og.slice_clusters(w.c, w.w, w.K)
    p_lflam = og.lflam(w.c, w.w, cof, cl, w.K)[0]
    passes = 1 if n == 2 else None          # the oracle's C2 pass takes ~8 s
    log = _refine_check(G, og, w.c, w.w, cof, cl, w.K, p_lflam, passes=passes)
    assert (log[:, 0] == 0).sum() > 0 and (log[:, 0] == 1).sum() > 0
    if n == 2:
        return
    rng = np.random.default_rng(n)
    p_rand = np.empty(w.V, np.int32)
    for k, x in enumerate(cl):
        p_rand[x] = k if k < w.K else int(rng.integers(0, w.K))
    log2 = _refine_check(G, og, w.c, w.w, cof, cl, w.K, p_rand, passes=1)
    assert (log2[:, 0] == 0).sum() > 0


def test_refine_random_small_dags():
    """Tiny DAGs with tie-heavy costs, window 1 and 64, K up to 4, costs bound
    and per call, and swap-rich chain + singleton shapes."""
    rng = np.random.default_rng(23)
    n_swaps = n_moves = 0
    for it in range(60):
        n = int(rng.integers(4, 40))
        s, d = tiny_random_dag(rng, n, float(rng.uniform(0.1, 0.5)))
        if it % 3 == 0:
            c, w = rng.integers(0, 3, n), rng.integers(0, 4, s.size)
        else:
            c, w = rng.integers(0, 50, n), rng.integers(0, 50 * (8 if it % 2 else 1), s.size)
        K = int(rng.integers(2, 5))
        og = OracleGraph(n, s, d)
        cof, cl = og.slice_clusters(c, w, K)
        if len(cl) < K:
            continue
        p0 = np.empty(n, np.int32)
        for k, x in enumerate(cl):
            p0[x] = k if k < K else int(rng.integers(0, K))
        G = _G(n, s, d, c, w) if it % 2 else _G(n, s, d)
        log = _refine_check(G, og, c, w, cof, cl, K, p0, window=1 if it % 5 == 0 else 64, bound=bool(it % 2))
        n_swaps += int((log[:, 0] == 0).sum()) if len(log) else 0
        n_moves += int((log[:, 0] == 1).sum()) if len(log) else 0
    assert n_swaps > 10 and n_moves > 10, (n_swaps, n_moves)


def test_refine_rejects_split_clusters():
    from paper_2008_08636_b200 import PdnnError

    w, og, G = _cfg(1)
    cof, cl = og.slice_clusters(w.c, w.w, w.K)
    members, off = _flat_clusters(cl)
    part = np.zeros(w.V, np.int32)
    part[cl[0][0]] = 1                     # primary 0 now spans two PEs
    with pytest.raises(PdnnError):
        G.refine(cof, members, off, len(cl), w.K, part)
    with pytest.raises(PdnnError):
        G.refine(cof, members, off, len(cl), w.K, np.full(w.V, w.K, np.int32))   # label out of range


# ------------------------------------------------------------------- sweep schedule invariant
def _schedule_ok(G, V, src, dst, which):
    """Every item of the dataflow sweep depends only on items dealt before it
    (the deadlock-freedom invariant of sweep.cu) in the given item order."""
    import ctypes as C

    from paper_2008_08636_b200 import load_library

    lib = load_library()
    fn = getattr(lib, which)
    fn.argtypes = [C.c_void_p, C.c_void_p]
    n = fn(G.handle, None)
    it = np.zeros((max(n, 1), 4), np.int32)
    assert fn(G.handle, it.ctypes.data) == 0
    it = it[:n]
    lvl = G.levels().cpu().numpy()
    orig = np.lexsort((np.arange(V), lvl))               # rank -> node id: stable (level, id)
    rank = np.empty(V, np.int64)
    rank[orig] = np.arange(V)
    fi = lib.pdnn_debug_sweep_inodes
    fi.argtypes = [C.c_void_p, C.c_void_p]
    ni = fi(G.handle, None)
    inodes = np.zeros(max(ni, 1), np.int32)
    assert fi(G.handle, inodes.ctypes.data) == 0
    fwd = it[:, 0] >= 0
    r0 = np.where(fwd, it[:, 0], ~it[:, 0])
    cnt = np.where(it[:, 1] > 0, it[:, 1], 1)
    idx = np.repeat(np.arange(n), cnt)
    offs = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    nodes = np.repeat(r0, cnt) + offs
    ixd = np.repeat(((it[:, 3] & (1 << 30)) != 0) & (it[:, 1] > 0), cnt)   # indexed items: ranks listed in inodes
    nodes[ixd] = inodes[nodes[ixd]]
    assert not (ixd & np.repeat(fwd, cnt)).any()                      # only bl items are indexed
    dirn = np.repeat(fwd, cnt)
    big = np.iinfo(np.int64).max
    first = {d: np.full(V, big) for d in (True, False)}
    last = {d: np.full(V, -1) for d in (True, False)}
    for d in (True, False):
        m = dirn == d
        np.minimum.at(first[d], nodes[m], idx[m])
        np.maximum.at(last[d], nodes[m], idx[m])
    u, v = rank[np.asarray(src)], rank[np.asarray(dst)]
    lv = np.sort(lvl)                                      # level by rank
    tl_dep = lv[u] >= 1                                    # level 0: published by the prologue
    assert (last[True][u[tl_dep]] < first[True][v[tl_dep]]).all()
    assert (last[False][v] < first[False][u]).all()
    # every node of level >= 1 has tl items, every node bl items
    assert (first[True][lv >= 1] < big).all() and (first[False] < big).all()


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_sweep_schedule_is_topological(n):
    """Both item orders of the dataflow sweep (by wave for whole-graph sweeps,
    proportional for the K-loop's sweeps with REMOVED nodes) deal every item
    after every item it waits for."""
    w, og, G = _cfg(n)
    _schedule_ok(G, w.V, w.src, w.dst, "pdnn_debug_sweep_items")
    _schedule_ok(G, w.V, w.src, w.dst, "pdnn_debug_sweep_items_rm")


def test_sweep_schedule_is_topological_hubs_and_random():
    rng = np.random.default_rng(31)
    cases = []
    n = 3000                                   # a fan-out hub and a fan-in hub (split parts in both sweeps)
    cases.append((n, np.concatenate([np.zeros(n - 2, np.int32), np.arange(1, n - 1, dtype=np.int32)]),
                  np.concatenate([np.arange(1, n - 1, dtype=np.int32), np.full(n - 2, n - 1, np.int32)])))
    for it in range(6):
        m = int(rng.integers(50, 400))
        s, d = tiny_random_dag(rng, m, float(rng.uniform(0.02, 0.2)))
        cases.append((m, s, d))
    for V, s, d in cases:
        G = _G(V, s, d)
        _schedule_ok(G, V, s, d, "pdnn_debug_sweep_items")
        _schedule_ok(G, V, s, d, "pdnn_debug_sweep_items_rm")


@pytest.mark.parametrize("n", [1, 2, 6])
def test_eval_batch_wide_schedule(n):
    """1,024+ candidates switch the batched sweep to its wide schedule (two
    nodes per item); every candidate vs the oracle on the other graph shapes."""
    from paper_2008_08636_b200 import Graph

    w, og, G = _cfg(n)
    B = 1056
    parts_h = candidate_parts(w.seed, 0, B, w.V, w.n_pe, "uniform" if n != 2 else "refine")
    got = Graph.results_to_numpy(G.eval_batch(parts_h, w.n_pe, w.mem, w.kind, w.cap_eff))
    want = og.eval_batch(w.c, w.w, w.mem, w.kind, w.n_pe, w.cap_eff, parts_h)
    _compare_results(got, want)


@pytest.mark.parametrize("B", [256, 700, 1024])
def test_eval_batch_single_node_moves(B):
    """Refinement-trial batches: one placement with a single node moved per
    candidate (the node-level passes' trials), in the narrow and the wide
    batched schedule, vs the oracle."""
    from paper_2008_08636_b200 import Graph

    w, og, G = _cfg(2)
    rng = np.random.default_rng(B)
    base = rng.integers(0, w.n_pe, w.V).astype(np.uint8)
    parts_h = np.repeat(base[None, :], B, axis=0)
    nodes = rng.integers(0, w.V, B)
    parts_h[np.arange(B), nodes] = (base[nodes] + 1 + rng.integers(0, w.n_pe - 1, B)) % w.n_pe
    got = Graph.results_to_numpy(G.eval_batch(parts_h, w.n_pe, w.mem, w.kind, w.cap_eff))
    want = og.eval_batch(w.c, w.w, w.mem, w.kind, w.n_pe, w.cap_eff, parts_h)
    _compare_results(got, want)


def test_refine_c2_all_passes():
    """C2 after LFLAM with all K node-level passes (the late rounds score a few
    trials each: the batched sweep's launches stay full groups, so its epoch
    tags never meet a chunk idle for two launches) -- identical to the oracle."""
    w, og, G = _cfg(2)
    cof, cl = og.slice_clusters(w.c, w.w, w.K)
    p_lflam = og.lflam(w.c, w.w, cof, cl, w.K)[0]
    log = _refine_check(G, og, w.c, w.w, cof, cl, w.K, p_lflam)
    assert (log[:, 0] == 1).sum() > 20
