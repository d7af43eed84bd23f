// cp.cu -- critical-path extraction (§8(a) row a5) and the K-sweep slicing
// loop (row a6).
//
// CP (Table 2 "CP"; find_heaviest_path with fresh weighted
// levels), reading R5/R6 of DESIGN.md:
//   L     = max over alive n of tl(n) + bl(n)
//   start = lowest-id alive node with no alive predecessor and bl == L
//   next  = lowest-id alive successor s with comm'(u,s) + bl(s) == bl(u) - comp(u)
// Every node of that walk is critical (tl + bl == L), so one launch:
//   1. each CTA reduces max(tl+bl) over a contiguous id range and keeps, in id
//      order, the nodes attaining its local maximum;
//   2. the last CTA to finish (atomic ticket) takes L = max of the CTA maxima,
//      gathers the candidates of the CTAs whose maximum is L (= all critical
//      nodes, ascending id), computes each one's tight successor and entry
//      flag with a warp per node, and walks the path in shared memory.
// If the critical set does not fit (massive ties), the last CTA falls back
// to a slow but general scan over all nodes and a walk through global memory.
#include <cooperative_groups.h>

#include "internal.cuh"

namespace pdnn {

struct CpArgs {
    int32_t V;
    const int64_t* tl;
    const int64_t* bl;
    const int32_t* part;  // node-id order, nullable
    const int64_t* c_rank;
    const int32_t* rank_of;
    const int32_t* orig;
    const int32_t* in_off;
    const int32_t* in_src;
    const int32_t* out_off;
    const int32_t* out_dst;
    const int64_t* out_cost;
    long long* M;          // [grid] per-CTA max of tl + bl
    int32_t* ctl;          // [0] critical count m, [1] start id, [2] walk/doubling flag
    unsigned long long* hacc;   // hash accumulator
    int32_t* list;         // [V] critical nodes (ids), compaction order
    int32_t* pos;          // [V] by id: index in list (valid for critical nodes only)
    int32_t* A0;           // [V] pointer doubling: 2^r-th successor index (-1: past the end)
    int32_t* A1;
    int32_t* d0;           // [V] distance to the end of the successor chain
    int32_t* d1;
    uint8_t* mark;         // [V] on the path from start
    int32_t* cp_nodes;
    int32_t* cp_len;
    int64_t* Lout;
    uint64_t* hash;
    int32_t* mark_orig;
    int32_t* mark_rank;
};

constexpr uint64_t kHashP = 0x100000001B3ull;
constexpr int kCpWalkMax = 4096;   // critical sets up to this size are walked in shared memory

// G <- G - {path}: the removed label goes to both copies of the labels
__device__ __forceinline__ void mark_removed(const CpArgs& a, int32_t u) {
    a.mark_orig[u] = PDNN_REMOVED;
    a.mark_rank[a.rank_of[u]] = PDNN_REMOVED;
}

__device__ __forceinline__ bool is_alive(const CpArgs& a, int32_t v) {
    return a.part == nullptr || a.part[v] != PDNN_REMOVED;
}
__device__ __forceinline__ int64_t commp(const CpArgs& a, int32_t u, int32_t v, int64_t w) {
    if (!a.part) return w;
    const int32_t pu = a.part[u], pv = a.part[v];
    return (pu == pv && pu >= 0) ? 0 : w;
}

// tight successor (lowest id) and "has alive successor" of node u, computed by
// one warp.  Returns next id or -1; *any = has an alive successor.
__device__ int32_t warp_next(const CpArgs& a, int32_t u, int lane, bool* any) {
    const int32_t r = a.rank_of[u];
    const int64_t target = a.bl[u] - a.c_rank[r];
    int32_t best = 0x7fffffff;
    bool has = false;
    for (int32_t e = a.out_off[r] + lane; e < a.out_off[r + 1]; e += 32) {
        const int32_t s = a.orig[a.out_dst[e]];
        if (!is_alive(a, s)) continue;
        has = true;
        if (commp(a, u, s, a.out_cost[e]) + a.bl[s] == target && s < best) best = s;
    }
    *any = __any_sync(0xffffffffu, has);
    best = __reduce_min_sync(0xffffffffu, best);
    return best == 0x7fffffff ? -1 : best;
}

__device__ bool warp_has_alive_pred(const CpArgs& a, int32_t u, int lane) {
    const int32_t r = a.rank_of[u];
    bool has = false;
    for (int32_t e = a.in_off[r] + lane; e < a.in_off[r + 1]; e += 32)
        if (is_alive(a, a.orig[a.in_src[e]])) has = true;
    return __any_sync(0xffffffffu, has);
}

__device__ __forceinline__ uint64_t pow_p(uint32_t k) {   // kHashP^k mod 2^64
    uint64_t r = 1, b = kHashP;
    while (k) {
        if (k & 1) r *= b;
        b *= b;
        k >>= 1;
    }
    return r;
}

// One cooperative launch:
//   1. L = max over alive n of tl + bl (per-CTA maxima, then every CTA reduces them);
//   2. the critical nodes (tl + bl == L: every node of every longest path) are
//      compacted into a list; pos[id] = their index;
//   3. a warp per critical node computes its tight successor (lowest id, R5) --
//      itself critical -- and whether it is an alive entry node; start = the
//      lowest-id critical entry node;
//   4. the path start -> next -> ... is either walked by one CTA in shared
//      memory (m <= kCpWalkMax) or found by pointer doubling over the list:
//      round r marks the 2^r-th successors of the marked nodes and doubles the
//      jump pointers / distances-to-end, so after ceil(log2 m) rounds every
//      node of the path is marked and sits at position dist(start) - dist(node).
__global__ void __launch_bounds__(kCpThreads) k_cp(CpArgs a) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ int32_t s_nidx[];   // [2][kCpWalkMax] successor indices + ids (CTA 0's walk)
    int32_t* s_list = s_nidx + kCpWalkMax;
    __shared__ long long s_red[kCpThreads / 32];
    __shared__ long long s_L;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t nth = (int64_t)gridDim.x * kCpThreads;
    const int64_t gtid = (int64_t)blockIdx.x * kCpThreads + tid;
    const int gwarp = (int)(gtid >> 5), nwarps = (int)(nth >> 5);

    // ---- 1. per-CTA max of tl + bl over alive nodes (kCpU loads in flight per thread)
    long long m = -1;
    for (int64_t v0 = gtid; v0 < a.V; v0 += kCpU * nth) {
        int64_t t[kCpU], b[kCpU];
#pragma unroll
        for (int u = 0; u < kCpU; ++u) {
            const int64_t v = v0 + u * nth;
            t[u] = v < a.V ? __ldcg(&a.tl[v]) : -1;
            b[u] = v < a.V ? __ldcg(&a.bl[v]) : 0;
        }
#pragma unroll
        for (int u = 0; u < kCpU; ++u)
            if (t[u] >= 0) m = t[u] + b[u] > m ? t[u] + b[u] : m;
    }
    m = warp_max_i64(m);
    if (lane == 0) s_red[warp] = m;
    __syncthreads();
    if (tid == 0) {
        long long x = -1;
        for (int w = 0; w < kCpThreads / 32; ++w) x = s_red[w] > x ? s_red[w] : x;
        a.M[blockIdx.x] = x;
        if (blockIdx.x == 0) { a.ctl[0] = 0; a.ctl[1] = 0x7fffffff; *a.hacc = 0ull; }
    }
    grid.sync();

    // ---- 2. L, and the critical nodes compacted into the list
    {
        long long x = -1;
        for (int i = tid; i < (int)gridDim.x; i += kCpThreads) x = a.M[i] > x ? a.M[i] : x;
        x = warp_max_i64(x);
        if (lane == 0) s_red[warp] = x;
        __syncthreads();
        if (tid == 0) {
            long long y = -1;
            for (int w = 0; w < kCpThreads / 32; ++w) y = s_red[w] > y ? s_red[w] : y;
            s_L = y;
        }
        __syncthreads();
    }
    const long long L = s_L;
    if (L < 0) {   // no alive node
        if (gtid == 0) { *a.cp_len = 0; *a.Lout = 0; *a.hash = 0; }
        return;
    }
    for (int64_t v0 = (int64_t)blockIdx.x * kCpThreads + warp * 32; v0 < a.V; v0 += nth) {
        const int64_t v = v0 + lane;
        bool crit = false;
        if (v < a.V) {
            const int64_t t = __ldcg(&a.tl[v]);
            crit = t >= 0 && t + __ldcg(&a.bl[v]) == L;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, crit);
        if (bal) {
            int32_t base = 0;
            if (lane == 0) base = atomicAdd(&a.ctl[0], __popc(bal));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (crit) {
                const int32_t i = base + __popc(bal & ((1u << lane) - 1u));
                a.list[i] = (int32_t)v;
                a.pos[v] = i;
            }
        }
    }
    grid.sync();

    // ---- 3. tight successor and entry flag of every critical node
    const int32_t mc = *(volatile int32_t*)&a.ctl[0];
    for (int32_t i = gwarp; i < mc; i += nwarps) {
        const int32_t u = a.list[i];
        bool any;
        const int32_t nx = warp_next(a, u, lane, &any);
        bool entry = false;
        if (a.tl[u] == 0) entry = !warp_has_alive_pred(a, u, lane);
        if (lane == 0) {
            const int32_t ni = (any && nx >= 0) ? a.pos[nx] : -1;
            a.A0[i] = ni;
            a.d0[i] = ni >= 0 ? 1 : 0;
            a.mark[i] = 0;
            if (entry) atomicMin(&a.ctl[1], u);
        }
    }
    grid.sync();
    const int32_t start = *(volatile int32_t*)&a.ctl[1];
    const int32_t s0 = a.pos[start];

    // ---- 4a. short critical sets: one CTA walks the successor indices in shared memory
    if (mc <= kCpWalkMax) {
        if (blockIdx.x != 0) return;
        for (int32_t i = tid; i < mc; i += kCpThreads) {
            s_nidx[i] = a.A0[i];
            s_list[i] = a.list[i];
        }
        __syncthreads();
        if (tid == 0) {
            int32_t i = s0, k = 0;
            uint64_t h = 0, pw = 1;
            while (i >= 0) {
                const int32_t u = s_list[i];
                a.cp_nodes[k++] = u;
                h += (uint64_t)(u + 1) * pw;
                pw *= kHashP;
                if (a.mark_orig) mark_removed(a, u);
                i = s_nidx[i];
            }
            *a.cp_len = k;
            *a.Lout = L;
            *a.hash = h;
        }
        return;
    }
    // ---- 4b. long critical sets: pointer doubling over the list
    if (gtid == 0) a.mark[s0] = 1;
    grid.sync();
    int32_t *A = a.A0, *An = a.A1, *d = a.d0, *dn = a.d1;
    for (int32_t span = 1; span < mc; span <<= 1) {
        for (int32_t i = (int32_t)gtid; i < mc; i += (int32_t)nth)   // marked nodes mark their 2^r-th successor
            if (a.mark[i] && A[i] >= 0) a.mark[A[i]] = 1;
        for (int32_t i = (int32_t)gtid; i < mc; i += (int32_t)nth) {   // then the jumps double
            const int32_t j = A[i];
            An[i] = j >= 0 ? A[j] : -1;
            dn[i] = d[i] + (j >= 0 ? d[j] : 0);
        }
        grid.sync();
        int32_t* t = A; A = An; An = t;
        t = d; d = dn; dn = t;
    }
    const int32_t len = d[s0] + 1;
    for (int32_t i = (int32_t)gtid; i < mc; i += (int32_t)nth)
        if (a.mark[i]) {
            const int32_t k = d[s0] - d[i];
            const int32_t u = a.list[i];
            a.cp_nodes[k] = u;
            atomicAdd(a.hacc, (unsigned long long)((uint64_t)(u + 1) * pow_p((uint32_t)k)));
            if (a.mark_orig) mark_removed(a, u);
        }
    grid.sync();
    if (gtid == 0) {
        *a.cp_len = len;
        *a.Lout = L;
        *a.hash = *(volatile unsigned long long*)a.hacc;
    }
}

int cp_grid_size(const pdnn_graph* g) {
    const int bpsm = kernel_occupancy((const void*)k_cp, kCpThreads, kCpWalkMax * 8);
    const int need = std::max(1, ceil_div(g->V, kCpThreads * 4));   // >= 4 nodes per thread
    return std::max(1, std::min(std::min(bpsm, 2) * g->num_sms, need));
}

pdnn_status launch_cp(const pdnn_graph* g, const Costs& C, const int32_t* part_orig,
                      const int64_t* tl, const int64_t* bl, int32_t* cp_nodes, int32_t* cp_len,
                      int64_t* Lout, uint64_t* hash, int32_t* mark_orig, int32_t* mark_rank,
                      void* ws, const WsLayout& L, cudaStream_t s) {
    if (g->V == 0) {
        PDNN_CUDA_TRY(cudaMemsetAsync(cp_len, 0, 4, s));
        PDNN_CUDA_TRY(cudaMemsetAsync(Lout, 0, 8, s));
        PDNN_CUDA_TRY(cudaMemsetAsync(hash, 0, 8, s));
        return PDNN_OK;
    }
    CpArgs a;
    a.V = g->V;
    a.tl = tl;
    a.bl = bl;
    a.part = part_orig;
    a.c_rank = C.c;
    a.rank_of = g->rank_of;
    a.orig = g->orig;
    a.in_off = g->in_off;
    a.in_src = g->in_src;
    a.out_off = g->out_off;
    a.out_dst = g->out_dst;
    a.out_cost = C.out_cost;
    a.M = ws_ptr<long long>(ws, L.cp_M);
    a.ctl = ws_ptr<int32_t>(ws, L.cp_ctl);
    a.hacc = ws_ptr<unsigned long long>(ws, L.cp_ctl + 16);
    a.list = ws_ptr<int32_t>(ws, L.cp_list);
    a.pos = ws_ptr<int32_t>(ws, L.cp_pos);
    a.A0 = ws_ptr<int32_t>(ws, L.cp_A);
    a.A1 = a.A0 + g->V;
    a.d0 = ws_ptr<int32_t>(ws, L.cp_d);
    a.d1 = a.d0 + g->V;
    a.mark = ws_ptr<uint8_t>(ws, L.cp_mark);
    a.cp_nodes = cp_nodes;
    a.cp_len = cp_len;
    a.Lout = Lout;
    a.hash = hash;
    a.mark_orig = mark_orig;
    a.mark_rank = mark_rank;
    const int grid = std::min(cp_grid_size(g), L.cp_grid);
    void* args[] = {(void*)&a};
    PDNN_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_cp, dim3(grid), dim3(kCpThreads), args,
                                              kCpWalkMax * 8, s));
    count_launch();
    return PDNN_OK;
}

}  // namespace pdnn

using namespace pdnn;

extern "C" pdnn_status pdnn_critical_path(const pdnn_graph* g, const int64_t* node_cost,
                                          const int64_t* edge_cost, const int32_t* part,
                                          const int64_t* tl, const int64_t* bl, int32_t* cp_nodes,
                                          int32_t* cp_len, int64_t* Lout, uint64_t* cp_hash, void* ws,
                                          size_t ws_bytes, void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (!cp_len || !Lout || !cp_hash || (g->V > 0 && (!tl || !bl || !cp_nodes))) {
        set_error("null argument");
        return PDNN_EINVAL;
    }
    const WsLayout L = ws_layout(g, PDNN_OP_CRITICAL_PATH, 0);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    pdnn_status st = ws_guard(ws, 0, 0, L.single_end, L.sig_single, s);
    if (st) return st;
    Costs C;
    if ((st = resolve_costs(g, node_cost, edge_cost, ws, L, s, &C))) return st;
    return launch_cp(g, C, part, tl, bl, cp_nodes, cp_len, Lout, cp_hash, nullptr, nullptr, ws, L, s);
}

extern "C" pdnn_status pdnn_slice(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                                  int32_t K, int32_t cap, int32_t* cps, int32_t* cp_lens, int64_t* Ls,
                                  uint64_t* hashes, void* ws, size_t ws_bytes, void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (K < 0 || cap < g->n_levels || (K > 0 && (!cps || !cp_lens || !Ls || !hashes))) {
        set_error("bad K / cap or null output");
        return PDNN_EINVAL;
    }
    const WsLayout L = ws_layout(g, PDNN_OP_SLICE, 0);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    pdnn_status st = ws_guard(ws, 0, 0, L.single_end, L.sig_single, s);
    if (st) return st;
    Costs C;
    if ((st = resolve_costs(g, node_cost, edge_cost, ws, L, s, &C, /*need_blob=*/true))) return st;
    int32_t* po = ws_ptr<int32_t>(ws, L.part_o);
    int32_t* pr = ws_ptr<int32_t>(ws, L.part_rank);
    int64_t* tl = ws_ptr<int64_t>(ws, L.tl_o);
    int64_t* bl = ws_ptr<int64_t>(ws, L.bl_o);
    // the first sweep runs on the whole graph with every node UNASSIGNED, which
    // is exactly the label-free sweep (every edge pays, reading R2/R3); the labels
    // are needed only to remove the paths found before the next sweeps
    const bool marks = K > 1;
    if (marks && (st = launch_labels(g, nullptr, nullptr, PDNN_UNASSIGNED, po, pr, s))) return st;
    for (int32_t j = 0; j < K; ++j) {
        // G <- G - {heaviest_path}: recompute the weighted levels on the rest (R4)
        if ((st = launch_sweep(g, C, j == 0 ? nullptr : pr, tl, bl, ws, L, s, /*removal=*/j > 0))) return st;
        if ((st = launch_cp(g, C, marks ? po : nullptr, tl, bl, cps + (size_t)j * cap, cp_lens + j, Ls + j,
                            hashes + j, marks ? po : nullptr, marks ? pr : nullptr, ws, L, s)))
            return st;
    }
    return PDNN_OK;
}
