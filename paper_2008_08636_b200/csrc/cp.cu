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
#include "internal.cuh"

namespace pdnn {

struct CpArgs {
    int32_t V;
    int32_t chunk;
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
    long long* M;
    int32_t* cnt;
    int32_t* list;
    int32_t* lnext;      // [grid][kCpCap] tight successor of each local candidate (-1: exit)
    uint8_t* lentry;     // [grid][kCpCap] candidate is an alive entry node
    int32_t* next_scr;
    WsHeader* hdr;
    int32_t* cp_nodes;
    int32_t* cp_len;
    int64_t* Lout;
    uint64_t* hash;
    int32_t* mark_orig;
    int32_t* mark_rank;
};

constexpr uint64_t kHashP = 0x100000001B3ull;

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

__global__ void __launch_bounds__(kCpThreads) k_cp(CpArgs a) {
    __shared__ long long s_red[kCpThreads / 32];
    __shared__ int32_t s_wcnt[kCpThreads / 32];
    __shared__ int32_t s_list[kCpListCap];
    __shared__ int32_t s_next[kCpListCap];
    __shared__ int32_t s_nidx[kCpListCap];
    __shared__ uint8_t s_entry[kCpListCap];
    __shared__ int32_t s_cand[kCpCap];
    __shared__ long long s_L;
    __shared__ int32_t s_total, s_fast, s_start, s_last;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarp = kCpThreads / 32;
    const int32_t lo = blockIdx.x * a.chunk;
    const int32_t hi = min(a.V, lo + a.chunk);

    // ---- phase 1: local max of tl + bl over alive nodes
    long long m = -1;
    // kCpU nodes per thread per round, both loads of each issued before any use
    for (int32_t v0 = lo + tid; v0 < hi; v0 += kCpU * kCpThreads) {
        int64_t t[kCpU], b[kCpU];
#pragma unroll
        for (int u = 0; u < kCpU; ++u) {
            const int32_t v = v0 + u * kCpThreads;
            t[u] = v < hi ? __ldcg(&a.tl[v]) : -1;
            b[u] = v < hi ? __ldcg(&a.bl[v]) : 0;
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
        for (int w = 0; w < nwarp; ++w) x = s_red[w] > x ? s_red[w] : x;
        s_L = x;
        s_total = 0;
    }
    __syncthreads();
    const long long Mb = s_L;
    // ---- the nodes attaining Mb, in id order (capacity kCpCap).  They are few:
    // collect them unordered with a shared-memory counter, then rank each by
    // id (n <= kCpCap, O(n^2) comparisons spread over the CTA).  A CTA with
    // more than kCpCap of them only reports the count (the last CTA then takes
    // the general path, which does not read the lists).
    if (Mb >= 0) {
        for (int32_t v = lo + tid; v < hi; v += kCpThreads) {
            const int64_t t = a.tl[v];
            if (t >= 0 && t + a.bl[v] == Mb) {
                const int32_t p = atomicAdd(&s_total, 1);
                if (p < kCpCap) s_next[p] = v;   // s_next: scratch until the walk
            }
        }
        __syncthreads();
        const int32_t nc = s_total < kCpCap ? s_total : kCpCap;
        if (s_total <= kCpCap && tid < nc) {
            const int32_t v = s_next[tid];
            int32_t r = 0;
            for (int32_t j = 0; j < nc; ++j) r += s_next[j] < v;
            s_cand[r] = v;
            a.list[(size_t)blockIdx.x * kCpCap + r] = v;
        }
        __syncthreads();
    }
    // tight successor and entry flag of every local candidate, computed here in
    // parallel by all CTAs (only the candidates of CTAs whose maximum is the
    // global L are used), so the last CTA only concatenates and walks
    if (Mb >= 0) {
        const int32_t nc = s_total <= kCpCap ? s_total : 0;   // an overflowing CTA's list is never read
        for (int32_t i = warp; i < nc; i += nwarp) {
            const int32_t u = s_cand[i];
            bool any;
            const int32_t nx = warp_next(a, u, lane, &any);
            bool entry = false;
            if (a.tl[u] == 0) entry = !warp_has_alive_pred(a, u, lane);
            if (lane == 0) {
                a.lnext[(size_t)blockIdx.x * kCpCap + i] = any ? nx : -1;
                a.lentry[(size_t)blockIdx.x * kCpCap + i] = entry;
            }
        }
    }
    __threadfence();  // publish this CTA's list entries before the ticket
    __syncthreads();
    if (tid == 0) {
        a.M[blockIdx.x] = Mb;
        a.cnt[blockIdx.x] = s_total;
        __threadfence();
        const uint32_t t = atomicAdd(&a.hdr->cp_ticket, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    // ---- last CTA: global L and the critical set (one entry per thread:
    // gridDim.x <= kCpThreads)
    const int b = tid;
    const bool inb = b < (int)gridDim.x;
    const long long Mb2 = inb ? *(volatile long long*)&a.M[b] : -1;
    long long L = warp_max_i64(Mb2);
    if (lane == 0) s_red[warp] = L;
    __syncthreads();
    if (tid == 0) {
        long long x = -1;
        for (int w = 0; w < nwarp; ++w) x = s_red[w] > x ? s_red[w] : x;
        s_L = x;
        s_start = 0x7fffffff;
        a.hdr->cp_ticket = 0;  // self-reset for the next call
    }
    __syncthreads();
    L = s_L;
    // candidates of the CTAs whose maximum is L, concatenated in CTA order
    const int32_t cb = (inb && Mb2 == L && L >= 0) ? *(volatile int32_t*)&a.cnt[b] : 0;
    const bool ovf = cb > kCpCap;
    // block exclusive scan of cb
    int32_t incl = cb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_wcnt[warp] = incl;
    const int any_ovf = __syncthreads_or(ovf);
    int32_t wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += s_wcnt[w];
    const int32_t excl = wbase + incl - cb;
    if (tid == kCpThreads - 1) {
        s_total = excl + cb;
        s_fast = !any_ovf && (excl + cb) <= kCpListCap;
    }
    __syncthreads();
    if (s_fast)
        for (int32_t k = 0; k < cb; ++k) {
            const size_t src = (size_t)b * kCpCap + k;
            s_list[excl + k] = *(volatile int32_t*)&a.list[src];
            s_next[excl + k] = *(volatile int32_t*)&a.lnext[src];
            s_entry[excl + k] = *(volatile uint8_t*)&a.lentry[src];
        }
    __syncthreads();
    if (L < 0) {  // no alive node
        if (tid == 0) { *a.cp_len = 0; *a.Lout = 0; *a.hash = 0; }
        return;
    }
    if (s_fast) {
        const int32_t n = s_total;
        for (int32_t i = tid; i < n; i += kCpThreads)
            if (s_entry[i]) atomicMin(&s_start, i);
        __syncthreads();
        for (int32_t i = tid; i < n; i += kCpThreads) {  // index of next in the sorted list
            const int32_t x = s_next[i];
            int32_t j = -1;
            if (x >= 0) {
                int32_t l = 0, h = n - 1;
                while (l <= h) {
                    const int32_t md = (l + h) >> 1;
                    const int32_t y = s_list[md];
                    if (y == x) { j = md; break; }
                    if (y < x) l = md + 1; else h = md - 1;
                }
            }
            s_nidx[i] = j;
        }
        __syncthreads();
        if (tid == 0) {
            int32_t i = s_start, k = 0;
            uint64_t h = 0, pw = 1;
            while (i >= 0 && i < n) {
                const int32_t u = s_list[i];
                a.cp_nodes[k++] = u;
                h += (uint64_t)(u + 1) * pw;
                pw *= kHashP;
                if (a.mark_orig) mark_removed(a, u);
                if (s_next[i] < 0) break;
                i = s_nidx[i];
            }
            *a.cp_len = k;
            *a.Lout = L;
            *a.hash = h;
        }
        return;
    }
    // ---- slow path: all nodes, next pointers in global memory
    for (int32_t v0 = warp; v0 < a.V; v0 += nwarp) {
        const int64_t t = a.tl[v0];
        if (t < 0 || t + a.bl[v0] != L) continue;
        bool any;
        const int32_t nx = warp_next(a, v0, lane, &any);
        bool entry = false;
        if (t == 0) entry = !warp_has_alive_pred(a, v0, lane);
        if (lane == 0) {
            a.next_scr[v0] = any ? nx : -1;
            if (entry) atomicMin(&s_start, v0);
        }
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence_block();
        int32_t u = s_start, k = 0;
        uint64_t h = 0, pw = 1;
        while (u >= 0 && u < a.V) {
            a.cp_nodes[k++] = u;
            h += (uint64_t)(u + 1) * pw;
            pw *= kHashP;
            if (a.mark_orig) mark_removed(a, u);
            u = *(volatile int32_t*)&a.next_scr[u];
        }
        *a.cp_len = k;
        *a.Lout = L;
        *a.hash = h;
    }
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
    a.chunk = ceil_div(g->V, L.cp_grid);
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
    a.cnt = ws_ptr<int32_t>(ws, L.cp_cnt);
    a.list = ws_ptr<int32_t>(ws, L.cp_list);
    a.lnext = ws_ptr<int32_t>(ws, L.cp_lnext);
    a.lentry = ws_ptr<uint8_t>(ws, L.cp_lentry);
    a.next_scr = ws_ptr<int32_t>(ws, L.cp_next);
    a.hdr = ws_ptr<WsHeader>(ws, L.hdr);
    a.cp_nodes = cp_nodes;
    a.cp_len = cp_len;
    a.Lout = Lout;
    a.hash = hash;
    a.mark_orig = mark_orig;
    a.mark_rank = mark_rank;
    const int grid = ceil_div(g->V, a.chunk);
    k_cp<<<grid, kCpThreads, 0, s>>>(a);
    count_launch();
    PDNN_LAUNCH_CHECK();
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
        if ((st = launch_sweep(g, C, j == 0 ? nullptr : pr, tl, bl, ws, L, s))) return st;
        if ((st = launch_cp(g, C, marks ? po : nullptr, tl, bl, cps + (size_t)j * cap, cp_lens + j, Ls + j,
                            hashes + j, marks ? po : nullptr, marks ? pr : nullptr, ws, L, s)))
            return st;
    }
    return PDNN_OK;
}
