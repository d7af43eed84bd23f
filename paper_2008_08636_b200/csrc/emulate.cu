// emulate.cu -- the TF FIFO scheduler emulator (§8(f) NEXT row N1).
//
// "TensorFlow scheduler maintains a ready queue that is initially filled with
// nodes with no ancestors.  Each node in the graph has an in-degree ...  The
// nodes are executed in FIFO order.  Once a node is executed, the in-degrees
// of its children are decremented by one.  Any node having an in-degree of
// zero will be pushed to the queue." (Memory Heuristic I)
// In reading R17: each PE runs one node at a time; a node enters
// the queue when its last input arrives,
//     ready(v) = max(0, max over preds p of ft(p) + comm'(p, v)),
// the queue is FIFO by entry time with ties by (level, id), and
//     st(v) = max(ready(v), ft(previous node on pe(v))),  ft = st + comp.
//
// B200 design: the emulation is a sequential
// discrete-event simulation per placement (a pop depends on every earlier
// pop), so it runs as ONE warp per placement -- a single placement on one
// CTA, a batch of candidates on one CTA each.  The warp pops in (ready, rank)
// order (rank = the graph's stable (level, id) order, so the key is exactly
// R17's), relaxes the popped node's out-edges with its 32 lanes in parallel
// (arrival times, in-degree countdown) and pushes the released successors.
// The queue is a binary heap whose first `cap` entries live in shared memory
// (16,384 for a single placement, 3,072 per candidate of a batch) and the
// rest in a per-placement global spill area; the initial
// entries (every level-0 node, all with ready 0) are not pushed at all: they
// are exactly ranks [0, n_entry) in key order, consumed by a cursor.
#include "internal.cuh"

namespace pdnn {

constexpr int kEmuSmemCap = 3072;          // heap entries in shared memory per candidate (12 B each)
constexpr int kEmuSmemCapSingle = 16384;   // a single placement: one CTA, most of the SM's shared memory

struct EmuArgs {
    int32_t V, n_entry, P;
    const int32_t* in_off;
    const int32_t* out_off;
    const int32_t* out_dst;
    const int64_t* c;          // rank space
    const int64_t* out_cost;   // forward-CSR order
    const int32_t* orig;
    const int32_t* lab32;      // rank-space labels (single placement), or
    const uint8_t* lab8;       // candidate-major rank-space labels [cand][V]
    int64_t* ready;            // [cand][V] scratch
    int32_t* indeg;            // [cand][V] scratch
    int64_t* hk;               // [cand][V] heap spill keys (ready)
    int32_t* hr;               // [cand][V] heap spill ranks
    int64_t* st_orig;          // single placement: st / ft in node-id order (nullable)
    int64_t* ft_orig;
    int64_t* st_rank;          // batched: st in rank order [cand][V] (the tracker's sort keys), nullable
    int64_t* makespan;         // single placement: device scalar (nullable)
    pdnn_eval_result* out;     // batched: results (makespan field), nullable
    int32_t n_cand;
    int32_t cap;               // heap entries in (dynamic) shared memory
};

struct EmuHeap {
    int64_t* sk;   // shared
    int32_t* sr;
    int64_t* gk;   // global spill (index >= cap)
    int32_t* gr;
    int32_t cap;
    __device__ __forceinline__ void get(int32_t i, int64_t& k, int32_t& r) const {
        if (i < cap) { k = sk[i]; r = sr[i]; }
        else { k = gk[i - cap]; r = gr[i - cap]; }
    }
    __device__ __forceinline__ void set(int32_t i, int64_t k, int32_t r) const {
        if (i < cap) { sk[i] = k; sr[i] = r; }
        else { gk[i - cap] = k; gr[i - cap] = r; }
    }
};
__device__ __forceinline__ bool key_less(int64_t ka, int32_t ra, int64_t kb, int32_t rb) {
    return ka < kb || (ka == kb && ra < rb);
}
__device__ void heap_push(const EmuHeap& h, int32_t& n, int64_t k, int32_t r) {
    int32_t i = n++;
    while (i > 0) {
        const int32_t p = (i - 1) >> 1;
        int64_t pk;
        int32_t pr;
        h.get(p, pk, pr);
        if (!key_less(k, r, pk, pr)) break;
        h.set(i, pk, pr);
        i = p;
    }
    h.set(i, k, r);
}
__device__ void heap_pop(const EmuHeap& h, int32_t& n) {   // removes the top
    int64_t xk;
    int32_t xr;
    h.get(--n, xk, xr);
    int32_t i = 0;
    for (;;) {
        int32_t c = 2 * i + 1;
        if (c >= n) break;
        int64_t ck, dk;
        int32_t cr, dr;
        h.get(c, ck, cr);
        if (c + 1 < n) {
            h.get(c + 1, dk, dr);
            if (key_less(dk, dr, ck, cr)) { ++c; ck = dk; cr = dr; }
        }
        if (!key_less(ck, cr, xk, xr)) break;
        h.set(i, ck, cr);
        i = c;
    }
    if (n > 0) h.set(i, xk, xr);
}

template <bool U8>
__global__ void __launch_bounds__(32) k_emulate(EmuArgs a) {
    extern __shared__ __align__(16) unsigned char emu_smem[];
    int64_t* s_k = reinterpret_cast<int64_t*>(emu_smem);              // [cap]
    int32_t* s_r = reinterpret_cast<int32_t*>(emu_smem + 8 * (size_t)a.cap);
    __shared__ int64_t s_free[PDNN_MAX_PE];
    const int lane = threadIdx.x;
    const int32_t b = blockIdx.x;   // placement (candidate) of this warp
    if (b >= a.n_cand) return;
    const int32_t V = a.V;
    const size_t o = (size_t)b * V;
    int64_t* ready = a.ready + o;
    int32_t* indeg = a.indeg + o;
    const EmuHeap h{s_k, s_r, a.hk + o, a.hr + o, a.cap};
    auto label = [&](int32_t r) -> int32_t { return U8 ? (int32_t)a.lab8[o + r] : a.lab32[r]; };
    // every node starts with its full in-degree and no input arrived
    for (int32_t r = lane; r < V; r += 32) {
        indeg[r] = a.in_off[r + 1] - a.in_off[r];
        ready[r] = 0;
    }
    if (lane < PDNN_MAX_PE) s_free[lane] = 0;
    __syncwarp();
    int32_t n = 0;          // heap size (lane 0's copy is authoritative; kept warp-uniform)
    int32_t cur = 0;        // cursor over the initial entries (ranks [0, n_entry), ready 0)
    int64_t span = 0;
    for (int32_t done = 0; done < V; ++done) {
        // pop the smallest (ready, rank): the initial run vs the heap top
        int64_t rdy = 0;
        int32_t v = 0;
        if (lane == 0) {
            int64_t tk = 0;
            int32_t tr = 0;
            if (n > 0) h.get(0, tk, tr);
            if (cur < a.n_entry && (n == 0 || key_less(0, cur, tk, tr))) {
                v = cur++;
                rdy = 0;
            } else {
                v = tr;
                rdy = tk;
                heap_pop(h, n);
            }
        }
        v = __shfl_sync(0xffffffffu, v, 0);
        rdy = __shfl_sync(0xffffffffu, rdy, 0);
        const int32_t q = label(v) & (PDNN_MAX_PE - 1);   // labels in [0, n_pe) (precondition)
        const int64_t st = rdy > s_free[q] ? rdy : s_free[q];
        const int64_t ft = st + a.c[v];
        __syncwarp();
        if (lane == 0) {
            s_free[q] = ft;
            span = ft > span ? ft : span;
            const int32_t ov = a.orig[v];
            if (a.st_orig) { a.st_orig[ov] = st; a.ft_orig[ov] = ft; }
            if (a.st_rank) a.st_rank[o + v] = st;
        }
        // once a node is executed, the in-degrees of its children drop by one
        const int32_t e0 = a.out_off[v], e1 = a.out_off[v + 1];
        for (int32_t eb = e0; eb < e1; eb += 32) {
            const int32_t e = eb + lane;
            bool rel = false;
            int64_t rs = 0;
            int32_t s = 0;
            if (e < e1) {
                s = a.out_dst[e];
                const int64_t arrive = ft + ((label(s) & (PDNN_MAX_PE - 1)) == q ? 0 : a.out_cost[e]);
                const int64_t r0 = ready[s];
                rs = arrive > r0 ? arrive : r0;
                ready[s] = rs;
                const int32_t d = indeg[s] - 1;
                indeg[s] = d;
                rel = d == 0;
            }
            // released successors enter the queue (lane 0 pushes them in lane order)
            unsigned m = __ballot_sync(0xffffffffu, rel);
            while (m) {
                const int src = __ffs(m) - 1;
                m &= m - 1;
                const int64_t k = __shfl_sync(0xffffffffu, rs, src);
                const int32_t r = __shfl_sync(0xffffffffu, s, src);
                if (lane == 0) heap_push(h, n, k, r);
            }
        }
        __syncwarp();
    }
    if (lane == 0) {
        if (a.makespan) *a.makespan = span;
        if (a.out) a.out[b].makespan = span;
    }
}

size_t emulate_ws_bytes(const pdnn_graph* g, int32_t n_cand) {
    return (size_t)std::max(n_cand, 1) * (size_t)std::max(g->V, 1) * (8 + 4 + 8 + 4);
}

pdnn_status launch_emulate(const pdnn_graph* g, const Costs& C, const int32_t* lab32, const uint8_t* lab8,
                           int32_t P, int32_t n_cand, void* scratch, int64_t* st_orig, int64_t* ft_orig,
                           int64_t* st_rank, int64_t* makespan, pdnn_eval_result* out, cudaStream_t s) {
    if (n_cand <= 0) return PDNN_OK;
    EmuArgs a;
    a.V = g->V;
    a.n_entry = g->n_entry;
    a.P = P;
    a.in_off = g->in_off;
    a.out_off = g->out_off;
    a.out_dst = g->out_dst;
    a.c = C.c;
    a.out_cost = C.out_cost;
    a.orig = g->orig;
    a.lab32 = lab32;
    a.lab8 = lab8;
    const size_t nv = (size_t)n_cand * (size_t)std::max(g->V, 1);
    char* p = static_cast<char*>(scratch);
    a.ready = reinterpret_cast<int64_t*>(p);
    a.hk = reinterpret_cast<int64_t*>(p + 8 * nv);
    a.indeg = reinterpret_cast<int32_t*>(p + 16 * nv);
    a.hr = reinterpret_cast<int32_t*>(p + 20 * nv);
    a.st_orig = st_orig;
    a.ft_orig = ft_orig;
    a.st_rank = st_rank;
    a.makespan = makespan;
    a.out = out;
    a.n_cand = n_cand;
    if (g->V == 0) {
        if (makespan) PDNN_CUDA_TRY(cudaMemsetAsync(makespan, 0, 8, s));
        return PDNN_OK;
    }
    // the heap's first `cap` entries in shared memory: a single placement takes
    // most of the SM (C4's queue holds ~20k entries: its deep levels were
    // global-memory round trips on every pop and push); a batch keeps several
    // candidates per SM
    a.cap = n_cand == 1 ? kEmuSmemCapSingle : kEmuSmemCap;
    const int smem = 12 * a.cap;
    const void* fn = lab8 ? (const void*)k_emulate<true> : (const void*)k_emulate<false>;
    PDNN_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (lab8) k_emulate<true><<<n_cand, 32, smem, s>>>(a);
    else k_emulate<false><<<n_cand, 32, smem, s>>>(a);
    count_launch();
    PDNN_LAUNCH_CHECK();
    return PDNN_OK;
}

}  // namespace pdnn

using namespace pdnn;

extern "C" pdnn_status pdnn_emulate(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                                    const int32_t* part, int32_t n_pe, int64_t* st, int64_t* ft,
                                    int64_t* makespan, void* ws, size_t ws_bytes, void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (n_pe < 1 || n_pe > PDNN_MAX_PE) { set_error("n_pe must be in [1, 16]"); return PDNN_EINVAL; }
    if (!makespan || (g->V > 0 && (!part || !st || !ft))) { set_error("null argument"); return PDNN_EINVAL; }
    const WsLayout L = ws_layout(g, PDNN_OP_EMULATE, 0);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    pdnn_status rc = ws_guard(ws, 0, 0, L.single_end, L.sig_single, s);
    if (rc) return rc;
    Costs C;
    if ((rc = resolve_costs(g, node_cost, edge_cost, ws, L, s, &C))) return rc;
    int32_t* pr = ws_ptr<int32_t>(ws, L.part_rank);
    if ((rc = launch_labels(g, part, nullptr, 0, nullptr, pr, s))) return rc;
    return launch_emulate(g, C, pr, nullptr, n_pe, 1, ws_ptr<void>(ws, L.emu), st, ft, nullptr, makespan, nullptr, s);
}
