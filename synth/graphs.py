"""Seeded DAG generators shaped like the paper's workloads.

No method arithmetic lives here: the generators draw node/edge structure,
integer costs (ns), memory sizes (bytes), node kinds, capacities and candidate
placements.  Node ids are handed out in construction order (forward pass, then
backward pass, then optimizer ops), as a TensorFlow graph would number them.

Shapes (Table 3 node counts; Table 5 DoP/CCR,
PAPER.md:1181-1185):
  C1 layered random DAG, 2,000 nodes / ~5k edges, 2 PEs, K=2
  C2 Word-RNN grid (48 layers x 28 steps of LSTM-cell templates), ~60k / ~150k
  C3 Transformer (64 layers: 16-head fork-join + FFN, Adam chains, hub
     constants with out-degree up to ~2.3e4, gradient AddN fan-in ~1e3), ~250k / ~700k
  C4 E3D-shaped wide DAG, 64 levels, ~1.5M nodes / ~4.5M edges
  C5 C3's graph with 4,096 candidate placements
  C6 Char-CRN (character CNN + highway + LSTM), ~25k nodes, 4 PEs, K=8
  C7 WRN (a chain of 101 residual units + optimizer chains), ~136k nodes, 8 PEs
  C8 / C9 C4's 1.5M nodes at D = 256 and at E3D's degree of parallelism (D = 20k)
"""
from __future__ import annotations

import dataclasses

import numpy as np

CONFIG_NAMES = {
    1: "c1_layered_2k",
    2: "c2_word_rnn_60k",
    3: "c3_trn_250k",
    4: "c4_e3d_wide_1p5m",
    5: "c5_batch_trn_4096",
    # the other shapes north_star names (Table 3 / Table 5), reported beside C2-C4
    6: "c6_char_crn_25k",
    7: "c7_wrn_136k",
    8: "c8_e3d_1p5m_d256",
    9: "c9_e3d_1p5m_dop_faithful",
}

KIND_NORMAL, KIND_RESIDUAL, KIND_REFERENCE = 0, 1, 2
_LOG_C = (np.log(1e2), np.log(1e7))          # comp(n): log-uniform ns
_LOG_MEM = (np.log(2.0**8), np.log(2.0**28))  # mem(n): log-uniform bytes


@dataclasses.dataclass
class Workload:
    name: str
    V: int
    src: np.ndarray   # int32[E], construction order (not sorted)
    dst: np.ndarray   # int32[E]
    c: np.ndarray     # int64[V] comp(n), ns
    w: np.ndarray     # int64[E] comm(e), ns, aligned with src/dst
    mem: np.ndarray   # int64[V] bytes
    kind: np.ndarray  # uint8[V] 0 normal / 1 residual / 2 reference
    n_pe: int
    K: int
    cap_eff: np.ndarray  # int64[n_pe]
    seed: int
    ccr_target: float

    @property
    def E(self) -> int:
        return int(self.src.shape[0])


# ----------------------------------------------------------------------------
# building blocks
# ----------------------------------------------------------------------------
class _Builder:
    def __init__(self):
        self.n = 0
        self.src: list[np.ndarray] = []
        self.dst: list[np.ndarray] = []
        self.kind_ranges: list[tuple[int, int, int]] = []

    def nodes(self, k: int, kind: int = KIND_NORMAL) -> int:
        s = self.n
        self.n += int(k)
        if kind != KIND_NORMAL and k > 0:
            self.kind_ranges.append((s, int(k), kind))
        return s

    def edges(self, s, d):
        s = np.asarray(s, np.int64).ravel()
        d = np.asarray(d, np.int64).ravel()
        assert s.shape == d.shape
        if s.size:
            self.src.append(s)
            self.dst.append(d)

    def finish(self, rng: np.random.Generator):
        src = np.concatenate(self.src) if self.src else np.zeros(0, np.int64)
        dst = np.concatenate(self.dst) if self.dst else np.zeros(0, np.int64)
        key = src * self.n + dst
        _, first = np.unique(key, return_index=True)   # drop duplicate pairs
        first.sort()                                    # keep construction order
        src, dst = src[first], dst[first]
        kind = np.zeros(self.n, np.uint8)
        for s, k, kd in self.kind_ranges:
            kind[s : s + k] = kd
        return self.n, src.astype(np.int32), dst.astype(np.int32), kind


def _template(rng: np.random.Generator, n_ops: int, depth: int, extra: float, back: int = 3):
    """A random op-level DAG with ops 0..n_ops-1 in `depth` sub-levels; op 0 is
    the only op of sub-level 0 (the cell input) and op n_ops-1 the only op of
    the last sub-level (the cell output).  Every op of sub-level k>=1 has one
    predecessor in sub-level k-1 plus Poisson(extra) more from k-back..k-1."""
    assert n_ops >= depth >= 3
    counts = np.ones(depth, np.int64)
    rest = n_ops - depth
    if rest:
        counts[1:-1] += np.bincount(rng.integers(1, depth - 1, rest), minlength=depth)[1:-1]
    starts = np.concatenate([[0], np.cumsum(counts)])
    src, dst, lvl = [], [], np.repeat(np.arange(depth), counts)
    for k in range(1, depth):
        ids = np.arange(starts[k], starts[k + 1])
        ps, pe = starts[k - 1], starts[k]
        src.append(rng.integers(ps, pe, ids.size))
        dst.append(ids)
        ne = rng.poisson(extra, ids.size)
        lo = starts[max(0, k - back)]
        tot = int(ne.sum())
        if tot:
            src.append(rng.integers(lo, pe, tot))
            dst.append(np.repeat(ids, ne))
    # every op except the output must feed something later, so the output
    # collects the cell (keeps cells fork-join shaped)
    src = np.concatenate(src)
    dst = np.concatenate(dst)
    has_out = np.zeros(n_ops, bool)
    has_out[src] = True
    dangling = np.nonzero(~has_out[:-1])[0]
    # connect dangling ops to a random op of a later sub-level (the output at least)
    tgt = np.empty(dangling.size, np.int64)
    for i, o in enumerate(dangling):
        k = lvl[o]
        tgt[i] = rng.integers(starts[k + 1], n_ops)
    src = np.concatenate([src, dangling])
    dst = np.concatenate([dst, tgt])
    return src.astype(np.int64), dst.astype(np.int64), lvl


def _tile(b: _Builder, tmpl, n_cells: int) -> int:
    """Place n_cells copies of template `tmpl` (contiguous ids); returns base."""
    tsrc, tdst, tl = tmpl
    n_ops = tl.size
    base = b.nodes(n_cells * n_ops)
    offs = base + np.arange(n_cells, dtype=np.int64)[:, None] * n_ops
    b.edges(tsrc[None, :] + offs, tdst[None, :] + offs)
    return base


# ----------------------------------------------------------------------------
# generators
# ----------------------------------------------------------------------------
def layered_dag(seed: int, n_levels: int, width: int, lam: float, max_indeg: int, back: int,
                n_params: int = 0, param_fanout: float = 1.5):
    """Layered random DAG: level l >= 1 nodes take one predecessor from level
    l-1 and Poisson(lam) more (capped at max_indeg total) from levels
    l-back..l-1.  n_params extra in-degree-0 parameter nodes (residual) each
    feed 1+Poisson(param_fanout-1) compute nodes at random levels >= 1."""
    rng = np.random.Generator(np.random.PCG64(seed))
    b = _Builder()
    pbase = b.nodes(n_params, KIND_RESIDUAL)
    cbase = b.nodes(n_levels * width)
    for l in range(1, n_levels):
        ids = cbase + l * width + np.arange(width)
        b.edges(cbase + (l - 1) * width + rng.integers(0, width, width), ids)
        ne = np.minimum(rng.poisson(lam, width), max_indeg - 1)
        tot = int(ne.sum())
        if tot:
            lo = cbase + max(0, l - back) * width
            hi = cbase + l * width
            b.edges(rng.integers(lo, hi, tot), np.repeat(ids, ne))
    if n_params:
        fo = 1 + rng.poisson(max(param_fanout - 1.0, 0.0), n_params)
        tgt = cbase + width + rng.integers(0, (n_levels - 1) * width, int(fo.sum()))
        b.edges(np.repeat(pbase + np.arange(n_params), fo), tgt)
    return b.finish(rng)


def word_rnn_dag(seed: int, layers: int = 48, steps: int = 28):
    """Word-RNN-shaped unrolled graph: a layers x steps grid
    of LSTM-cell templates (forward 15 ops / depth 8), the mirrored backward
    grid (30 ops / depth 12) with activation edges from the forward cells, a
    loss node, per-layer weights (residual) fanning out to all steps, per-layer
    gradient AddN (fan-in = steps) and an apply op (reference) per weight."""
    rng = np.random.Generator(np.random.PCG64(seed))
    b = _Builder()
    fw = _template(rng, 15, 8, 1.9)
    bw = _template(rng, 30, 12, 1.9)
    nf, nb = fw[2].size, bw[2].size
    W = b.nodes(layers, KIND_RESIDUAL)
    X = b.nodes(steps, KIND_RESIDUAL)          # embedded inputs (persist across the step)
    F = _tile(b, fw, layers * steps)
    loss = b.nodes(1)
    Bk = _tile(b, bw, layers * steps)
    G = b.nodes(layers)
    A = b.nodes(layers, KIND_REFERENCE)
    l, t = np.meshgrid(np.arange(layers), np.arange(steps), indexing="ij")
    cell = (l * steps + t).ravel()
    l, t = l.ravel(), t.ravel()
    fin = F + cell * nf
    fout = fin + nf - 1
    # forward recurrences
    m = l > 0
    b.edges(fout[m] - nf * steps, fin[m])          # from (l-1, t)
    m = t > 0
    b.edges(fout[m] - nf, fin[m])                  # from (l, t-1)
    b.edges(X + t[l == 0], fin[l == 0])
    b.edges(W + l, fin + 1)                        # weight -> matmul op
    b.edges(fout[l == layers - 1], np.full(steps, loss))
    # backward grid
    bin_ = Bk + cell * nb
    bout = bin_ + nb - 1
    m = l < layers - 1
    b.edges(bout[m] + nb * steps, bin_[m])         # from (l+1, t)
    m = t < steps - 1
    b.edges(bout[m] + nb, bin_[m])                 # from (l, t+1)
    b.edges(np.full(int((l == layers - 1).sum()), loss), bin_[l == layers - 1])
    for k in range(3):                             # saved activations
        fo = fin + rng.integers(1, nf - 1, cell.size)
        bo = bin_ + rng.integers(1, nb - 1, cell.size)
        b.edges(fo, bo)
    b.edges(W + l, bin_ + 2)
    b.edges(bout, G + l)                           # gradient AddN, fan-in = steps
    b.edges(G + np.arange(layers), A + np.arange(layers))
    b.edges(W + np.arange(layers), A + np.arange(layers))
    return b.finish(rng)


def transformer_dag(seed: int, layers: int = 64, heads: int = 16, params_per_layer: int = 118,
                    adam_ops: int = 22):
    """Transformer-shaped training graph: per layer a
    16-head fork-join (12-op / depth-10 head templates) followed by an FFN
    template (40 ops / depth 15); the mirrored backward pass (24-op heads, 80-op
    FFN); per parameter tensor a residual param node plus m/v slots, a gradient
    AddN, an Adam chain and an assign (reference).  Hubs: a global-step, a
    learning-rate and an epsilon constant feed every Adam chain (out-degree
    ~7e3 .. 2.1e4), and the shared-embedding gradient AddN has fan-in ~1e3."""
    rng = np.random.Generator(np.random.PCG64(seed))
    b = _Builder()
    hf = _template(rng, 12, 10, 1.6)
    ff = _template(rng, 40, 15, 1.6)
    hb = _template(rng, 24, 15, 1.6)
    fb = _template(rng, 80, 20, 1.6)
    ad = _template(rng, adam_ops, adam_ops // 2, 1.6)
    n_hf, n_ff, n_hb, n_fb, n_ad = hf[2].size, ff[2].size, hb[2].size, fb[2].size, ad[2].size
    hubs = b.nodes(3)                                  # global step, lr, epsilon
    emb = b.nodes(1, KIND_RESIDUAL)
    tok = b.nodes(1, KIND_RESIDUAL)
    Pn = layers * params_per_layer
    par = b.nodes(Pn, KIND_RESIDUAL)
    slots = b.nodes(2 * Pn, KIND_RESIDUAL)
    x = b.nodes(1)
    b.edges([emb, tok], [x, x])
    prev = x
    fwd_layer = []
    for L in range(layers):
        split = b.nodes(1)
        b.edges([prev], [split])
        H = _tile(b, hf, heads)
        hin = H + np.arange(heads) * n_hf
        b.edges(np.full(heads, split), hin)
        cat = b.nodes(1)
        b.edges(hin + n_hf - 1, np.full(heads, cat))
        FF = _tile(b, ff, 1)
        b.edges([cat], [FF])
        pl = par + L * params_per_layer
        # weights feed the head matmuls and FFN ops
        k = params_per_layer
        tgt = np.concatenate([hin + 1, FF + rng.integers(1, n_ff - 1, k - heads)])
        b.edges(pl + np.arange(k), tgt)
        prev = FF + n_ff - 1
        fwd_layer.append((hin, FF))
    loss = b.nodes(1)
    b.edges([prev], [loss])
    prev = loss
    grad_src = [[] for _ in range(layers)]
    emb_grads = []
    for L in reversed(range(layers)):
        hin_f, FF_f = fwd_layer[L]
        FB = _tile(b, fb, 1)
        b.edges([prev], [FB])
        for k in range(4):
            b.edges([FF_f + int(rng.integers(1, n_ff - 1))], [FB + int(rng.integers(1, n_fb - 1))])
        split = b.nodes(1)
        b.edges([FB + n_fb - 1], [split])
        H = _tile(b, hb, heads)
        hin = H + np.arange(heads) * n_hb
        b.edges(np.full(heads, split), hin)
        b.edges(hin_f + rng.integers(1, n_hf - 1, heads), hin + rng.integers(1, n_hb - 1, heads))
        cat = b.nodes(1)
        b.edges(hin + n_hb - 1, np.full(heads, cat))
        prev = cat
        # gradient producers for this layer's params: random backward ops
        cand = np.concatenate([FB + np.arange(1, n_fb), (hin[:, None] + np.arange(1, n_hb)).ravel()])
        grad_src[L] = cand
        emb_grads.append(rng.choice(cand, 16, replace=False))
    # shared-embedding gradient AddN, fan-in ~1e3
    eg = b.nodes(1)
    b.edges(np.concatenate(emb_grads), np.full(16 * layers, eg))
    b.edges([prev], [eg])
    ea = b.nodes(1, KIND_REFERENCE)
    b.edges([eg, emb], [ea, ea])
    # optimizer: per param AddN + Adam chain + assign
    G = b.nodes(Pn)
    fan = 1 + rng.poisson(2.0, Pn)
    srcs = np.concatenate([rng.choice(grad_src[i // params_per_layer], f) for i, f in enumerate(fan)])
    b.edges(srcs, np.repeat(G + np.arange(Pn), fan))
    AD = _tile(b, ad, Pn)
    ain = AD + np.arange(Pn) * n_ad
    b.edges(G + np.arange(Pn), ain)
    b.edges(slots + 2 * np.arange(Pn), ain + 1)
    b.edges(slots + 2 * np.arange(Pn) + 1, ain + 2)
    b.edges(np.full(Pn, hubs + 0), ain + 3)                  # global step (hub)
    b.edges(np.full(Pn, hubs + 1), ain + n_ad - 3)           # learning rate (hub)
    for k in (4, 5, 6):                                       # epsilon / betas (hub)
        b.edges(np.full(Pn, hubs + 2), ain + k)
    asg = b.nodes(Pn, KIND_REFERENCE)
    b.edges(ain + n_ad - 1, asg + np.arange(Pn))
    b.edges(par + np.arange(Pn), asg + np.arange(Pn))
    return b.finish(rng)


def e3d_wide_dag(seed: int, n_levels: int = 64, width: int = 18_750, n_params: int = 300_000):
    """E3D-LSTM-shaped wide DAG: 64 compute levels of
    18,750 ops; each op reads the previous level plus a Poisson "recall"
    fan-in from the previous 5 levels (<= 5 total), and 300k parameter nodes
    (residual) feed 1-3 compute ops each."""
    return layered_dag(seed, n_levels, width, lam=2.75, max_indeg=5, back=5,
                       n_params=n_params, param_fanout=1.5)


def char_crn_dag(seed: int, layers: int = 8, steps: int = 35, filters: int = 16, highway: int = 2):
    """Char-CRN-shaped graph (character-aware CNN + highway + LSTM language
    model: 8 layers, 22,748 nodes; Table 5 DoP 49, CCR 57,
    PAPER.md:1182): per time step a character-CNN of `filters` parallel
    conv branches (6-op / depth-5 templates) joined by a concat, `highway`
    highway blocks (8 ops / depth 6) feeding a layers x steps grid of LSTM
    cells (18 ops / depth 8); the mirrored backward pass; residual parameters
    (filters, highway, per-layer LSTM weights) fanning out to every step,
    per-parameter gradient AddN (fan-in = steps) and an apply op (reference).
    The per-step CNN stacks are independent across steps (the wide part)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    b = _Builder()
    cf, hf, lf = _template(rng, 6, 5, 1.0), _template(rng, 8, 6, 1.2), _template(rng, 18, 8, 1.9)
    cb, hb, lb = _template(rng, 10, 7, 1.0), _template(rng, 14, 9, 1.2), _template(rng, 34, 12, 1.9)
    ncf, nhf, nlf = cf[2].size, hf[2].size, lf[2].size
    ncb, nhb, nlb = cb[2].size, hb[2].size, lb[2].size
    Wc = b.nodes(filters, KIND_RESIDUAL)
    Wh = b.nodes(highway, KIND_RESIDUAL)
    Wl = b.nodes(layers, KIND_RESIDUAL)
    X = b.nodes(steps, KIND_RESIDUAL)                 # character ids of each word
    emb = b.nodes(steps)                              # char embedding lookups
    b.edges(X + np.arange(steps), emb + np.arange(steps))
    C = _tile(b, cf, steps * filters)                 # [step][filter] conv branches
    cin = C + np.arange(steps * filters) * ncf
    b.edges(np.repeat(emb + np.arange(steps), filters), cin)
    b.edges(np.tile(Wc + np.arange(filters), steps), cin + 1)
    cat = b.nodes(steps)
    b.edges(cin + ncf - 1, np.repeat(cat + np.arange(steps), filters))
    H = _tile(b, hf, steps * highway)                 # [step][block]
    hin = H + np.arange(steps * highway) * nhf
    st_, hk = np.repeat(np.arange(steps), highway), np.tile(np.arange(highway), steps)
    first = hk == 0
    b.edges(cat + st_[first], hin[first])
    b.edges(hin[~first] - 1, hin[~first])             # block k-1's output (its last op) feeds block k
    b.edges(Wh + hk, hin + 1)
    hout = hin[hk == highway - 1] + nhf - 1           # per step
    Lf = _tile(b, lf, layers * steps)
    l, t = np.meshgrid(np.arange(layers), np.arange(steps), indexing="ij")
    cell = (l * steps + t).ravel()
    l, t = l.ravel(), t.ravel()
    fin = Lf + cell * nlf
    fout = fin + nlf - 1
    m = l > 0
    b.edges(fout[m] - nlf * steps, fin[m])
    m = t > 0
    b.edges(fout[m] - nlf, fin[m])
    b.edges(hout[t[l == 0]], fin[l == 0])
    b.edges(Wl + l, fin + 1)
    loss = b.nodes(1)
    b.edges(fout[l == layers - 1], np.full(steps, loss))
    # backward
    Lb = _tile(b, lb, layers * steps)
    bin_ = Lb + cell * nlb
    bout = bin_ + nlb - 1
    m = l < layers - 1
    b.edges(bout[m] + nlb * steps, bin_[m])
    m = t < steps - 1
    b.edges(bout[m] + nlb, bin_[m])
    b.edges(np.full(int((l == layers - 1).sum()), loss), bin_[l == layers - 1])
    b.edges(fin + rng.integers(1, nlf - 1, cell.size), bin_ + rng.integers(1, nlb - 1, cell.size))
    HB = _tile(b, hb, steps * highway)
    hbin = HB + np.arange(steps * highway) * nhb
    last = hk == highway - 1
    b.edges(bout[l == 0][st_[last]], hbin[last])      # LSTM layer-0 grads enter the top highway block
    b.edges(hbin[~last] + nhb + nhb - 1, hbin[~last])  # block k+1's output feeds block k (same step)
    b.edges(hin + rng.integers(1, nhf - 1, hin.size), hbin + rng.integers(1, nhb - 1, hin.size))
    CB = _tile(b, cb, steps * filters)
    cbin = CB + np.arange(steps * filters) * ncb
    b.edges(np.repeat(hbin[first] + nhb - 1, filters), cbin)
    b.edges(cin + rng.integers(1, ncf - 1, cin.size), cbin + rng.integers(1, ncb - 1, cin.size))
    # gradients: AddN over the steps, apply ops (reference)
    G = b.nodes(filters + highway + layers)
    b.edges(cbin + ncb - 1, G + np.tile(np.arange(filters), steps))
    b.edges(hbin + nhb - 1, G + filters + hk)
    b.edges(bout, G + filters + highway + l)
    A = b.nodes(filters + highway + layers, KIND_REFERENCE)
    nP = filters + highway + layers
    b.edges(G + np.arange(nP), A + np.arange(nP))
    b.edges(np.concatenate([Wc + np.arange(filters), Wh + np.arange(highway), Wl + np.arange(layers)]),
            A + np.arange(nP))
    return b.finish(rng)


def wrn_dag(seed: int, units: int = 101, params_per_unit: int = 6, opt_ops: int = 22):
    """WRN-shaped graph (wide residual network: 101 residual
    units, 187,742 nodes; Table 5 DoP 1.16, CCR 13.02): a chain
    of residual units, each a forward template (BN-ReLU-conv x 2 + shortcut
    add: 400 ops / depth 300) and, mirrored, a backward template (800 ops /
    depth 600); per unit `params_per_unit` residual weights feeding its
    forward and backward ops, a gradient AddN and a momentum-update chain
    (`opt_ops` ops) ending in an assign (reference) per weight.  Deep and
    narrow: almost every op is on the forward-backward chain."""
    rng = np.random.Generator(np.random.PCG64(seed))
    b = _Builder()
    uf, ub, op = _template(rng, 400, 300, 0.6, back=2), _template(rng, 800, 600, 0.6, back=2), \
        _template(rng, opt_ops, opt_ops // 2, 1.2)
    nuf, nub, nop = uf[2].size, ub[2].size, op[2].size
    Pn = units * params_per_unit
    par = b.nodes(Pn, KIND_RESIDUAL)
    x = b.nodes(1, KIND_RESIDUAL)
    F = _tile(b, uf, units)
    fin = F + np.arange(units) * nuf
    b.edges([x], [fin[0]])
    b.edges(fin[:-1] + nuf - 1, fin[1:])              # unit chain
    b.edges(fin[:-1], fin[1:] + nuf - 2)              # shortcut into the next unit's add
    pu = np.repeat(np.arange(units), params_per_unit)
    b.edges(par + np.arange(Pn), fin[pu] + rng.integers(1, nuf - 1, Pn))
    loss = b.nodes(1)
    b.edges([fin[-1] + nuf - 1], [loss])
    B = _tile(b, ub, units)                           # unit u's backward at B + (units-1-u) * nub
    bin_ = B + (units - 1 - np.arange(units)) * nub
    b.edges([loss], [bin_[-1]])
    b.edges(bin_[1:] + nub - 1, bin_[:-1])
    for k in range(4):                                # saved activations
        b.edges(fin + rng.integers(1, nuf - 1, units), bin_ + rng.integers(1, nub - 1, units))
    b.edges(par + np.arange(Pn), bin_[pu] + rng.integers(1, nub - 1, Pn))
    G = b.nodes(Pn)
    b.edges(bin_[pu] + rng.integers(1, nub - 1, Pn), G + np.arange(Pn))
    b.edges(bin_[pu] + rng.integers(1, nub - 1, Pn), G + np.arange(Pn))
    O = _tile(b, op, Pn)
    oin = O + np.arange(Pn) * nop
    b.edges(G + np.arange(Pn), oin)
    asg = b.nodes(Pn, KIND_REFERENCE)
    b.edges(oin + nop - 1, asg + np.arange(Pn))
    b.edges(par + np.arange(Pn), asg + np.arange(Pn))
    return b.finish(rng)


def tiny_random_dag(rng: np.random.Generator, n: int, p: float):
    """Random DAG on n <= 20 nodes with shuffled ids (ids not topological)."""
    order = rng.permutation(n)
    src, dst = [], []
    for i in range(n):
        for j in range(i + 1, n):
            if rng.random() < p:
                src.append(order[i])
                dst.append(order[j])
    perm = rng.permutation(len(src))
    return (np.asarray(src, np.int32)[perm] if src else np.zeros(0, np.int32),
            np.asarray(dst, np.int32)[perm] if dst else np.zeros(0, np.int32))


# ----------------------------------------------------------------------------
# costs, memory, kinds, capacities
# ----------------------------------------------------------------------------
def attach_costs(rng: np.random.Generator, V: int, E: int, ccr: float, mode: str = "loguniform",
                 zero_frac: float = 0.05):
    """comp(n) log-uniform over [1e2, 1e7] ns with zero_frac exact zeros (TF
    plumbing ops); comm(e) log-uniform then integer-scaled so that
    sum(comm)/sum(comp) ~= ccr; mem(n) log-uniform over [2^8, 2^28] bytes.
    mode == "ties": comp, comm in {0,1,2} (maximal ties)."""
    if mode == "ties":
        c = rng.integers(0, 3, V).astype(np.int64)
        w = rng.integers(0, 3, E).astype(np.int64)
    else:
        c = np.exp(rng.uniform(*_LOG_C, V)).astype(np.int64)
        c[rng.random(V) < zero_frac] = 0
        wr = np.exp(rng.uniform(*_LOG_C, E))
        if E and ccr > 0:
            scale = ccr * float(c.sum()) / float(wr.sum())
            w = np.floor(wr * scale).astype(np.int64)
        else:
            w = np.zeros(E, np.int64)
    mem = np.exp(rng.uniform(*_LOG_MEM, V)).astype(np.int64)
    return c, w, mem


def _finish_kinds(rng, V, src, dst, kind):
    """Residual nodes must have in-degree 0 (parameters); a reference node is
    a direct consumer of a residual.  Add reference marks to ~5% of nodes by
    picking consumers of residual nodes when the generator did not."""
    indeg = np.bincount(dst, minlength=V)
    kind = kind.copy()
    kind[(kind == KIND_RESIDUAL) & (indeg > 0)] = KIND_NORMAL
    if (kind == KIND_REFERENCE).mean() < 0.01:
        cons = np.unique(dst[kind[src] == KIND_RESIDUAL])
        cons = cons[kind[cons] == KIND_NORMAL]
        k = min(cons.size, int(0.05 * V))
        if k:
            kind[rng.choice(cons, k, replace=False)] = KIND_REFERENCE
    return kind


def _cap(rng, mem, n_pe, frac):
    """cap_eff = cap - cap // 10 (the 10% reserve) with
    cap = frac * sum(mem) / n_pe, jittered +-10% per PE."""
    tot = float(mem.sum())
    cap = (frac * tot / n_pe * rng.uniform(0.9, 1.1, n_pe)).astype(np.int64)
    return cap - cap // 10


def make_config(n: int, seed: int | None = None, mode: str = "loguniform") -> Workload:
    """Configs 1-5 of BASELINE.json, and the extra shapes 6-9 (Char-CRN, WRN,
    C4 at D=256 and at E3D's DoP); seed defaults to 2008086 + n."""
    if seed is None:
        seed = 2008086 + n
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    if n == 1:
        V, src, dst, kind = layered_dag(seed, 50, 32, lam=1.2, max_indeg=6, back=3,
                                        n_params=400, param_fanout=2.5)
        n_pe, K, ccr = 2, 2, 1.0
    elif n == 2:
        V, src, dst, kind = word_rnn_dag(seed)
        n_pe, K, ccr = 4, 8, 14.5
    elif n in (3, 5):
        V, src, dst, kind = transformer_dag(seed if n == 3 else 2008086 + 3)
        n_pe, K, ccr = 8, 8, 13.7
    elif n == 4:
        V, src, dst, kind = e3d_wide_dag(seed)
        n_pe, K, ccr = 8, 1, 1.12
    elif n == 6:
        V, src, dst, kind = char_crn_dag(seed)
        n_pe, K, ccr = 4, 8, 57.0
    elif n == 7:
        V, src, dst, kind = wrn_dag(seed)
        n_pe, K, ccr = 8, 8, 13.02
    elif n == 8:   # C4 with 256 levels (the same 1.5M nodes, 4x narrower)
        V, src, dst, kind = layered_dag(seed, 256, 4_688, lam=2.75, max_indeg=5, back=5, n_params=300_000,
                                        param_fanout=1.5)
        n_pe, K, ccr = 8, 1, 1.12
    elif n == 9:   # C4 at E3D's degree of parallelism (DoP 3.3, Table 5): 20,000 levels of 60 ops
        V, src, dst, kind = layered_dag(seed, 20_000, 60, lam=2.75, max_indeg=5, back=5, n_params=300_000,
                                        param_fanout=1.5)
        n_pe, K, ccr = 8, 1, 1.12
    else:
        raise ValueError(n)
    kind = _finish_kinds(rng, V, src, dst, kind)
    c, w, mem = attach_costs(rng, V, src.size, ccr, mode=mode)
    cap_eff = _cap(rng, mem, n_pe, {1: 0.5, 2: 0.06}.get(n, 0.12))
    return Workload(CONFIG_NAMES[n], V, src, dst, c, w, mem, kind, n_pe, K, cap_eff, seed, ccr)


# ----------------------------------------------------------------------------
# candidate placements (batched evaluation, config 5)
# ----------------------------------------------------------------------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """The splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def candidate_parts(seed: int, b0: int, b1: int, V: int, n_pe: int, mode: str = "uniform") -> np.ndarray:
    """Candidates b0..b1-1 as uint8[b1-b0][V].
    uniform: label = splitmix64(seed, cand, node) mod n_pe (iid).
    refine:  a block placement by node id (id * n_pe // V) with ~1% of the
             nodes re-labelled per candidate (refinement-trial-like)."""
    cand = np.arange(b0, b1, dtype=np.uint64)[:, None]
    node = np.arange(V, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        key = (np.uint64(seed) * np.uint64(0xD1B54A32D192ED03) + cand * np.uint64(0x9E3779B97F4A7C15)
               + node * np.uint64(0xC2B2AE3D27D4EB4F)) & _M64
    h = splitmix64(key)
    if mode == "uniform":
        return (h % np.uint64(n_pe)).astype(np.uint8)
    base = (np.arange(V, dtype=np.int64) * n_pe // max(V, 1)).astype(np.uint8)[None, :]
    flip = (h >> np.uint64(32)) % np.uint64(100) == 0
    return np.where(flip, (h % np.uint64(n_pe)).astype(np.uint8), base).astype(np.uint8)
