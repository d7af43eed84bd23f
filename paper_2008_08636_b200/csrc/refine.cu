// refine.cu -- the refinement step of ParDNN's Step 1 (appendix "Complexity
// of Refinement"): §8(f) NEXT row N4 (second half), in
// reading R22.
//
//   phase 1  cluster swaps: tl under the placement once; the secondaries
//            sorted by (tl of their first node, id); for every unmarked A in
//            that order the candidates are the first `window` unmarked B
//            (sorted order) on another PE with tl(h_B) in span_t(A) =
//            [tl(h_A), tl(t_A) + comp(t_A)] (a binary search gives the start);
//            the B with the largest cut-communication gain > 0 whose swap
//            does not raise max(work(a, R), work(b, R)) over the levels R
//            both clusters cover (level-indexed Fenwick trees) is swapped and
//            both are marked;
//   phase 2  `passes` node-level passes: tl, bl and the CP under the
//            placement; trials (n, q) = a CP node and the PE of its CP
//            predecessor / successor when it differs; rounds: every trial
//            still alive whose move keeps work(q, level n) + comp(n) <= the
//            level's max work is scored by the candidate-parallel batched
//            sweep (lane = trial, L only); the least L (earliest trial on
//            ties) is applied if it is below the current L.
//
// B200 design.  Everything a decision reads that no
// decision changes is computed up front in parallel: the sort of the
// secondaries (one CUB radix sort), per secondary its window start, span,
// weight and its flattened external edges (other end, its cluster, comm).
// The swap decisions form a chain (a swap changes the placement the next
// decision reads), so they run on ONE CTA: the threads collect the window's
// candidates with an ordered block compaction, each warp scores candidates
// (lanes stride over the flattened edges of A and B; Fenwick range sums on
// lanes 0-3), and the block applies the best swap.  Phase 2's trial scores
// are the data-parallel part: up to kRefineGroup trial placements per
// launch of the batched sweep (bsweep.cu), one 32-trial chunk per warp.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <chrono>
#include <cstdio>

#include "internal.cuh"

namespace pdnn {

#ifndef PDNN_RF_THREADS
#define PDNN_RF_THREADS 512   // (256 / 512 / 1024 measured on C3: swaps 4.30 / 3.51 / 3.44 s)
#endif
constexpr int kRfThreads = PDNN_RF_THREADS;   // the swap-decision CTA
constexpr int kRfMaxWindow = 1024;

struct __align__(16) RfSec {     // a secondary's static record, by sorted position
    long long s0, s1;            // span_t: tl(h), tl(t) + comp(t); s0 = LLONG_MAX for an empty cluster
    long long w;                 // comp of its members
    int32_t k, h;                // cluster id, first member (node id; -1 if empty)
    int32_t lvl_lo, lvl_hi;      // level(h), level(t)
    int32_t lb;                  // first sorted position with s0 >= this s0
    int32_t e0, e1;              // its external edges in ey / ew
    int32_t pad;
};

static_assert(sizeof(RfSec) <= 64, "the workspace reserves 64 bytes per secondary");

static int rf_grid(int64_t n, int threads = 256) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 16));
}

// every cluster's members on one PE, every label in [0, K)
__global__ void k_rf_check(int32_t nc, int32_t K, const int32_t* __restrict__ members,
                           const int32_t* __restrict__ cl_off, const int32_t* __restrict__ part,
                           int32_t* __restrict__ bad) {
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nc; k += gridDim.x * blockDim.x) {
        const int32_t m0 = cl_off[k], m1 = cl_off[k + 1];
        if (m1 <= m0) continue;
        const int32_t p = part[members[m0]];
        bool ok = p >= 0 && p < K;
        for (int32_t m = m0 + 1; m < m1 && ok; ++m) ok = part[members[m]] == p;
        if (!ok) atomicExch(bad, 1);
    }
}

// per-(PE, level) comp sums of the placement
__global__ void k_rf_lvl(int32_t V, int32_t D, const int32_t* __restrict__ rank_of, const int32_t* __restrict__ level,
                         const int64_t* __restrict__ c_rank, const int32_t* __restrict__ part,
                         unsigned long long* __restrict__ lvl) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
        atomicAdd(&lvl[(size_t)part[v] * D + level[v]], (unsigned long long)c_rank[rank_of[v]]);
}

// sort keys of the secondaries: tl of the first member (empty clusters last)
__global__ void k_rf_keys(int32_t K, int32_t ns, const int32_t* __restrict__ members, const int32_t* __restrict__ cl_off,
                          const int64_t* __restrict__ tl, uint64_t* __restrict__ keys, int32_t* __restrict__ ids) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x) {
        const int32_t k = K + i;
        keys[i] = cl_off[k + 1] > cl_off[k] ? (uint64_t)tl[members[cl_off[k]]] : ~0ull;
        ids[i] = k;
    }
}

// one warp per sorted position: span, weight, level range, window start and
// the number of external edges
__global__ void k_rf_rec(int32_t ns, int32_t D, const int32_t* __restrict__ order, const uint64_t* __restrict__ skeys,
                         const int32_t* __restrict__ members, const int32_t* __restrict__ cl_off,
                         const int32_t* __restrict__ cluster_of, const int32_t* __restrict__ rank_of,
                         const int32_t* __restrict__ orig, const int32_t* __restrict__ level,
                         const int64_t* __restrict__ c_rank, const int64_t* __restrict__ tl,
                         const int32_t* __restrict__ in_off, const int32_t* __restrict__ in_src,
                         const int32_t* __restrict__ out_off, const int32_t* __restrict__ out_dst,
                         RfSec* __restrict__ R, int32_t* __restrict__ ecount) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; p < ns; p += nw) {
        const int32_t k = order[p], m0 = cl_off[k], m1 = cl_off[k + 1];
        long long w = 0;
        int32_t ne = 0;
        for (int32_t m = m0 + lane; m < m1; m += 32) {
            const int32_t u = members[m], r = rank_of[u];
            w += c_rank[r];
            for (int32_t e = in_off[r]; e < in_off[r + 1]; ++e) ne += cluster_of[orig[in_src[e]]] != k;
            for (int32_t e = out_off[r]; e < out_off[r + 1]; ++e) ne += cluster_of[orig[out_dst[e]]] != k;
        }
        w = warp_sum_i64(w);
        ne = (int32_t)warp_sum_i64(ne);
        if (lane == 0) {
            RfSec x;
            x.k = k;
            x.w = w;
            x.pad = 0;
            x.e0 = x.e1 = 0;
            if (m1 > m0) {
                const int32_t h = members[m0], t = members[m1 - 1];
                x.h = h;
                x.s0 = tl[h];
                x.s1 = tl[t] + c_rank[rank_of[t]];
                x.lvl_lo = level[h];
                x.lvl_hi = level[t];
                // first sorted position whose key is >= s0 (the keys are sorted)
                int32_t lo = 0, hi = ns;
                while (lo < hi) {
                    const int32_t mid = (lo + hi) >> 1;
                    if (skeys[mid] < (uint64_t)x.s0) lo = mid + 1; else hi = mid;
                }
                x.lb = lo;
            } else {
                x.h = -1;
                x.s0 = x.s1 = LLONG_MAX;
                x.lvl_lo = 0;
                x.lvl_hi = -1;
                x.lb = ns;
            }
            R[p] = x;
            ecount[p] = ne;
        }
    }
}

// flattened external edges of each sorted position: (other end, its cluster), comm
__global__ void k_rf_fill(int32_t ns, const int32_t* __restrict__ members, const int32_t* __restrict__ cl_off,
                          const int32_t* __restrict__ cluster_of, const int32_t* __restrict__ rank_of,
                          const int32_t* __restrict__ orig, const int32_t* __restrict__ in_off,
                          const int32_t* __restrict__ in_src, const int64_t* __restrict__ in_cost,
                          const int32_t* __restrict__ out_off, const int32_t* __restrict__ out_dst,
                          const int64_t* __restrict__ out_cost, const int32_t* __restrict__ eoff,
                          RfSec* __restrict__ R, int2* __restrict__ ey, long long* __restrict__ ew) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; p < ns; p += nw) {
        const int32_t k = R[p].k, m0 = cl_off[k], m1 = cl_off[k + 1];
        const int32_t base = eoff[p];
        int32_t at = base;
        // lane-ordered appends: a lane's count, then a warp prefix per member batch
        for (int32_t mb = m0; mb < m1; mb += 32) {
            const int32_t m = mb + lane;
            int32_t cnt = 0, r = -1;
            if (m < m1) {
                r = rank_of[members[m]];
                for (int32_t e = in_off[r]; e < in_off[r + 1]; ++e) cnt += cluster_of[orig[in_src[e]]] != k;
                for (int32_t e = out_off[r]; e < out_off[r + 1]; ++e) cnt += cluster_of[orig[out_dst[e]]] != k;
            }
            int32_t pre = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, pre, o);
                if (lane >= o) pre += y;
            }
            int32_t j = at + pre - cnt;
            if (m < m1) {
                for (int32_t e = in_off[r]; e < in_off[r + 1]; ++e) {
                    const int32_t y = orig[in_src[e]], cy = cluster_of[y];
                    if (cy == k) continue;
                    ey[j] = make_int2(y, cy);
                    ew[j] = in_cost[e];
                    ++j;
                }
                for (int32_t e = out_off[r]; e < out_off[r + 1]; ++e) {
                    const int32_t y = orig[out_dst[e]], cy = cluster_of[y];
                    if (cy == k) continue;
                    ey[j] = make_int2(y, cy);
                    ew[j] = out_cost[e];
                    ++j;
                }
            }
            at += __shfl_sync(0xffffffffu, pre, 31);
        }
        if (lane == 0) {
            R[p].e0 = base;
            R[p].e1 = at;
        }
    }
}

__device__ __forceinline__ long long rf_prefix(const long long* t, int32_t i) {   // levels [0, i)
    long long s = 0;
    for (; i > 0; i -= i & -i) s += __ldcg(t + i);
    return s;
}
__device__ __forceinline__ long long rf_range(const long long* t, int32_t lo, int32_t hi) {
    return hi < lo ? 0 : rf_prefix(t, hi + 1) - rf_prefix(t, lo);
}
__device__ __forceinline__ void rf_add(long long* t, int32_t D, int32_t l, long long c) {
    for (int32_t i = l + 1; i <= D; i += i & -i)
        atomicAdd(reinterpret_cast<unsigned long long*>(t + i), (unsigned long long)c);
}

struct RfArgs {
    int32_t ns, K, D, window;
    const RfSec* R;
    const int2* ey;
    const long long* ew;
    const int32_t* members;
    const int32_t* cl_off;
    const int32_t* level;
    const int32_t* rank_of;
    const int64_t* c_rank;
    int32_t* part;
    long long* tree;          // [K][D + 1]
    uint8_t* marked;          // by sorted position
    long long* log;           // [.][4]
    int32_t* n_log;
};

// phase 1: the swap decisions, in sorted order, on one CTA
__global__ void __launch_bounds__(kRfThreads) k_rf_swap(RfArgs a) {
    __shared__ int32_t s_cand[kRfMaxWindow];
    __shared__ long long s_gain[kRfMaxWindow];
    __shared__ int32_t s_wcnt[kRfThreads / 32];
    __shared__ int32_t s_best, s_nl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kRfThreads / 32;
    const int32_t K = a.K, D = a.D;
    if (tid == 0) s_nl = 0;
    __syncthreads();
    for (int32_t i = 0; i < a.ns; ++i) {
        const RfSec A = a.R[i];
        if (A.h < 0) break;                                // empty clusters sort last
        if (__ldcg(a.marked + i)) continue;
        const int32_t pa = __ldcg(a.part + A.h);
        // the first `window` qualifying B in sorted order with s0(B) in [s0(A), s1(A)]
        int32_t count = 0;
        for (int32_t base = A.lb; base < a.ns && count < a.window; base += kRfThreads) {
            const int32_t j = base + tid;
            bool inwin = false, q = false;
            if (j < a.ns) {
                const long long s0 = a.R[j].s0;
                inwin = s0 <= A.s1;
                if (inwin && j != i && !__ldcg(a.marked + j)) q = __ldcg(a.part + a.R[j].h) != pa;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, q);
            if (lane == 0) s_wcnt[warp] = __popc(bal);
            const int out = __syncthreads_or(j >= a.ns || !inwin);
            int32_t pre = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const int32_t x = s_wcnt[w];
                pre += w < warp ? x : 0;
                tot += x;
            }
            const int32_t r = count + pre + __popc(bal & ((1u << lane) - 1));
            if (q && r < a.window) s_cand[r] = j;
            count += tot;
            __syncthreads();
            if (out) break;
        }
        const int32_t nc = min(count, a.window);
        if (nc == 0) continue;
        // score the candidates: a warp per candidate
        for (int32_t ci = warp; ci < nc; ci += NW) {
            const int32_t j = s_cand[ci];
            const RfSec B = a.R[j];
            const int32_t pb = __ldcg(a.part + B.h);
            long long before = 0, after = 0;
            for (int32_t e = A.e0 + lane; e < A.e1; e += 32) {
                const int2 y = a.ey[e];
                const long long w = a.ew[e];
                const int32_t py = __ldcg(a.part + y.x);
                const int32_t ny = y.y == B.k ? pa : py;
                before += pa != py ? w : 0;
                after += pb != ny ? w : 0;
            }
            for (int32_t e = B.e0 + lane; e < B.e1; e += 32) {
                const int2 y = a.ey[e];
                if (y.y == A.k) continue;                       // counted with A
                const long long w = a.ew[e];
                const int32_t py = __ldcg(a.part + y.x);
                before += pb != py ? w : 0;
                after += pa != py ? w : 0;
            }
            const long long gain = warp_sum_i64(before) - warp_sum_i64(after);
            long long ok = 0;
            if (gain > 0) {
                const int32_t rl = min(A.lvl_lo, B.lvl_lo), rh = max(A.lvl_hi, B.lvl_hi);
                // lanes 0-3: the four prefix sums of work(a, R), work(b, R)
                long long x = 0;
                if (lane < 4) x = rf_prefix(a.tree + (size_t)(lane < 2 ? pa : pb) * (D + 1), (lane & 1) ? rl : rh + 1);
                const long long x1 = __shfl_sync(0xffffffffu, x, 1), x2 = __shfl_sync(0xffffffffu, x, 2);
                const long long x3 = __shfl_sync(0xffffffffu, x, 3);
                x = __shfl_sync(0xffffffffu, x, 0);
                const long long wa = x - x1, wb = x2 - x3;
                const long long na = wa - A.w + B.w, nb = wb - B.w + A.w;
                if (max(na, nb) <= max(wa, wb)) ok = gain;
            }
            if (lane == 0) s_gain[ci] = ok;
        }
        __syncthreads();
        if (tid == 0) {
            int32_t best = -1;
            long long bg = 0;
            for (int32_t ci = 0; ci < nc; ++ci)
                if (s_gain[ci] > bg) { bg = s_gain[ci]; best = ci; }
            s_best = best;
            if (best >= 0) {
                const int32_t j = s_cand[best];
                const int32_t nl = s_nl;
                a.log[4 * (size_t)nl] = 0;
                a.log[4 * (size_t)nl + 1] = A.k;
                a.log[4 * (size_t)nl + 2] = a.R[j].k;
                a.log[4 * (size_t)nl + 3] = bg;
                s_nl = nl + 1;
                a.marked[i] = 1;
                a.marked[j] = 1;
            }
        }
        __syncthreads();
        if (s_best >= 0) {
            const RfSec B = a.R[s_cand[s_best]];
            const int32_t pb = __ldcg(a.part + B.h);
            __syncthreads();                                   // every thread has read pb before the writes
            for (int side = 0; side < 2; ++side) {
                const int32_t k = side ? B.k : A.k;
                const int32_t from = side ? pb : pa, to = side ? pa : pb;
                for (int32_t m = a.cl_off[k] + tid; m < a.cl_off[k + 1]; m += kRfThreads) {
                    const int32_t u = a.members[m];
                    const int32_t l = a.level[u];
                    const long long c = a.c_rank[a.rank_of[u]];
                    rf_add(a.tree + (size_t)from * (D + 1), D, l, -c);
                    rf_add(a.tree + (size_t)to * (D + 1), D, l, c);
                    a.part[u] = to;
                }
            }
        }
        __syncthreads();
    }
    if (tid == 0) *a.n_log = s_nl;
}

// phase 2: the trials of a pass from its CP, in (CP index, predecessor's PE
// first) order, without a duplicate (n, q)
__global__ void __launch_bounds__(1024) k_rf_trials(const int32_t* __restrict__ cp, const int32_t* __restrict__ cp_len,
                                                    const int32_t* __restrict__ part, int32_t* __restrict__ tn,
                                                    int32_t* __restrict__ tq, uint8_t* __restrict__ tdead,
                                                    int32_t* __restrict__ n_trials) {
    __shared__ int32_t s_w[32];
    __shared__ int32_t s_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t n = *cp_len;
    if (tid == 0) s_base = 0;
    __syncthreads();
    for (int32_t k0 = 0; k0 < n; k0 += 1024) {
        const int32_t k = k0 + tid;
        int32_t node = -1, q0 = -1, q1 = -1;
        if (k < n) {
            node = cp[k];
            const int32_t p = part[node];
            if (k > 0 && part[cp[k - 1]] != p) q0 = part[cp[k - 1]];
            if (k + 1 < n && part[cp[k + 1]] != p) q1 = part[cp[k + 1]];
            if (q1 == q0) q1 = -1;
        }
        const int32_t cnt = (q0 >= 0) + (q1 >= 0);
        int32_t pre = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= o) pre += y;
        }
        if (lane == 31) s_w[warp] = pre;
        __syncthreads();
        int32_t wpre = 0, tot = 0;
        for (int w = 0; w < 32; ++w) {
            wpre += w < warp ? s_w[w] : 0;
            tot += s_w[w];
        }
        int32_t at = s_base + wpre + pre - cnt;
        if (q0 >= 0) { tn[at] = node; tq[at] = q0; tdead[at] = 0; ++at; }
        if (q1 >= 0) { tn[at] = node; tq[at] = q1; tdead[at] = 0; }
        __syncthreads();
        if (tid == 0) s_base += tot;
        __syncthreads();
    }
    if (tid == 0) *n_trials = s_base;
}

// the trials to score this round: alive, and the move keeps work(q, level n)
// + comp(n) <= the level's max work; in trial order
__global__ void __launch_bounds__(1024) k_rf_elig(int32_t K, int32_t D, const int32_t* __restrict__ n_trials,
                                                  const int32_t* __restrict__ tn, const int32_t* __restrict__ tq,
                                                  const uint8_t* __restrict__ tdead, const int32_t* __restrict__ level,
                                                  const int32_t* __restrict__ rank_of,
                                                  const int64_t* __restrict__ c_rank, const long long* __restrict__ tree,
                                                  int32_t* __restrict__ elig, int32_t* __restrict__ n_elig) {
    __shared__ int32_t s_w[32];
    __shared__ int32_t s_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t nt = *n_trials;
    if (tid == 0) s_base = 0;
    __syncthreads();
    for (int32_t t0 = 0; t0 < nt; t0 += 1024) {
        const int32_t t = t0 + tid;
        bool ok = false;
        if (t < nt && !tdead[t]) {
            const int32_t n = tn[t], q = tq[t], l = level[n];
            long long mx = 0, wq = 0;
            for (int32_t p = 0; p < K; ++p) {
                const long long x = rf_range(tree + (size_t)p * (D + 1), l, l);
                mx = max(mx, x);
                if (p == q) wq = x;
            }
            ok = wq + c_rank[rank_of[n]] <= mx;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (lane == 0) s_w[warp] = __popc(bal);
        __syncthreads();
        int32_t wpre = 0, tot = 0;
        for (int w = 0; w < 32; ++w) {
            wpre += w < warp ? s_w[w] : 0;
            tot += s_w[w];
        }
        if (ok) elig[s_base + wpre + __popc(bal & ((1u << lane) - 1))] = t;
        __syncthreads();
        if (tid == 0) s_base += tot;
        __syncthreads();
    }
    if (tid == 0) *n_elig = s_base;
}

// trial placements [ng][V] (uint8): the current placement with one node moved
// (rows nb.. of a partial group: the current placement itself)
__global__ void k_rf_rows(int32_t V, int32_t ng, int32_t nb, int32_t e0, const int32_t* __restrict__ elig,
                          const int32_t* __restrict__ tn, const int32_t* __restrict__ tq,
                          const int32_t* __restrict__ part, uint8_t* __restrict__ rows) {
    const int64_t n = (int64_t)ng * V;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = (int32_t)(x / V), v = (int32_t)(x % V);
        const int32_t t = j < nb ? elig[e0 + j] : -1;
        rows[x] = (uint8_t)(t >= 0 && v == tn[t] ? tq[t] : part[v]);
    }
}

// the least L (earliest eligible trial on ties); applied if below the current L
__global__ void __launch_bounds__(1024) k_rf_pick(int32_t D, const int32_t* __restrict__ n_elig,
                                                  const int32_t* __restrict__ elig, const pdnn_eval_result* __restrict__ res,
                                                  const int32_t* __restrict__ n_trials, const int32_t* __restrict__ tn,
                                                  const int32_t* __restrict__ tq, uint8_t* __restrict__ tdead,
                                                  const int32_t* __restrict__ level, const int32_t* __restrict__ rank_of,
                                                  const int64_t* __restrict__ c_rank, int32_t* __restrict__ part,
                                                  long long* __restrict__ tree, long long* __restrict__ L_cur,
                                                  long long* __restrict__ log, int32_t* __restrict__ n_log,
                                                  int32_t* __restrict__ moved) {
    __shared__ long long s_L[32];
    __shared__ int32_t s_i[32];
    __shared__ int32_t s_pick;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t ne = *n_elig;
    long long bL = LLONG_MAX;
    int32_t bi = INT_MAX;
    for (int32_t i = tid; i < ne; i += 1024) {
        const long long x = res[i].L;
        if (x < bL) { bL = x; bi = i; }     // ascending i per thread: the first minimum
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long oL = __shfl_xor_sync(0xffffffffu, bL, o);
        const int32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oL < bL || (oL == bL && oi < bi)) { bL = oL; bi = oi; }
    }
    if (lane == 0) { s_L[warp] = bL; s_i[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < 32; ++w)
            if (s_L[w] < bL || (s_L[w] == bL && s_i[w] < bi)) { bL = s_L[w]; bi = s_i[w]; }
        s_pick = -1;
        if (ne > 0 && bL < *L_cur) {
            const int32_t t = elig[bi], n = tn[t], q = tq[t];
            const int32_t l = level[n];
            const long long c = c_rank[rank_of[n]];
            rf_add(tree + (size_t)part[n] * (D + 1), D, l, -c);
            rf_add(tree + (size_t)q * (D + 1), D, l, c);
            part[n] = q;
            *L_cur = bL;
            const int32_t nl = *n_log;
            log[4 * (size_t)nl] = 1;
            log[4 * (size_t)nl + 1] = n;
            log[4 * (size_t)nl + 2] = q;
            log[4 * (size_t)nl + 3] = bL;
            *n_log = nl + 1;
            s_pick = n;
        }
        *moved = s_pick >= 0;
    }
    __syncthreads();
    const int32_t n = s_pick;
    if (n >= 0) {
        const int32_t nt = *n_trials;
        for (int32_t t = tid; t < nt; t += 1024)
            if (tn[t] == n) tdead[t] = 1;
    }
}

__global__ void k_rf_copy_L(const int64_t* __restrict__ L, long long* __restrict__ L_cur) { *L_cur = *L; }

size_t refine_temp_bytes(int32_t n) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, std::max(n, 1));
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const int32_t*)nullptr, (int32_t*)nullptr, std::max(n, 1) + 1);
    return std::max(a, b);
}

// sweep + CP under `part`: cp nodes, cp_len, L in the CP scratch
static pdnn_status rf_sweep_cp(const pdnn_graph* g, const Costs& C, int32_t* part, void* ws, const WsLayout& L,
                               int32_t* cp, int32_t* cp_len, int64_t* Ld, uint64_t* hash, cudaStream_t s) {
    pdnn_status st;
    int32_t* pr = ws_ptr<int32_t>(ws, L.part_rank);
    int64_t* tl = ws_ptr<int64_t>(ws, L.tl_o);
    int64_t* bl = ws_ptr<int64_t>(ws, L.bl_o);
    if ((st = launch_labels(g, part, nullptr, 0, nullptr, pr, s))) return st;
    if ((st = launch_sweep(g, C, pr, tl, bl, ws, L, s))) return st;
    return launch_cp(g, C, part, tl, bl, cp, cp_len, Ld, hash, nullptr, nullptr, ws, L, s);
}

}  // namespace pdnn

using namespace pdnn;

extern "C" pdnn_status pdnn_refine(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                                   const int32_t* cluster_of, const int32_t* members, const int32_t* cl_off,
                                   int32_t n_clusters, int32_t K, int32_t passes, int32_t window, int32_t* part,
                                   int64_t* log_host, int32_t log_cap, int32_t* n_log, int64_t* L_host, void* ws,
                                   size_t ws_bytes, void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (K < 1 || K > PDNN_MAX_PE || n_clusters < K || n_clusters > g->V + K || passes < 0 || window < 1 ||
        window > kRfMaxWindow || log_cap < 0 || !cl_off || !n_log || !L_host || (log_cap > 0 && !log_host) ||
        (g->V > 0 && (!cluster_of || !members || !part))) {
        set_error("bad K / n_clusters / passes / window or null argument");
        return PDNN_EINVAL;
    }
    const WsLayout L = ws_layout(g, PDNN_OP_REFINE, 0);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    pdnn_status st = ws_guard(ws, 0, 0, L.single_end, L.sig_single, s);
    if (st) return st;
    if ((st = ws_guard(ws, 1, L.single_end, L.total, L.sig_batch, s))) return st;
    *n_log = 0;
    *L_host = 0;
    const int32_t V = g->V, D = std::max(g->n_levels, 1), nc = n_clusters, ns = nc - K;
    if (V == 0) return PDNN_OK;
    Costs C;
    if ((st = resolve_costs(g, node_cost, edge_cost, ws, L, s, &C, /*need_blob=*/true))) return st;
    int32_t* ctl = ws_ptr<int32_t>(ws, L.rf_ctl);   // [0] bad [1] n_log [2] n_trials [3] n_elig [4] moved [5] cp_len
    long long* L_cur = ws_ptr<long long>(ws, L.rf_ctl + 64);
    int64_t* Ld = ws_ptr<int64_t>(ws, L.rf_ctl + 72);
    uint64_t* hash = ws_ptr<uint64_t>(ws, L.rf_ctl + 80);
    long long* logd = ws_ptr<long long>(ws, L.rf_log);
    long long* tree = ws_ptr<long long>(ws, L.rf_tree);
    unsigned long long* lvl = ws_ptr<unsigned long long>(ws, L.rf_lvl);
    PDNN_CUDA_TRY(cudaMemsetAsync(ctl, 0, 64, s));
    k_rf_check<<<rf_grid(nc), 256, 0, s>>>(nc, K, members, cl_off, part, ctl);
    count_launch();
    PDNN_LAUNCH_CHECK();
    int32_t bad = 0;
    PDNN_CUDA_TRY(cudaMemcpyAsync(&bad, ctl, 4, cudaMemcpyDeviceToHost, s));
    PDNN_CUDA_TRY(cudaStreamSynchronize(s));
    if (bad) { set_error("a label is outside [0, K) or a cluster spans two PEs"); return PDNN_EINVAL; }
    // level-indexed work trees of the placement
    PDNN_CUDA_TRY(cudaMemsetAsync(lvl, 0, 8 * (size_t)K * D, s));
    k_rf_lvl<<<rf_grid(V), 256, 0, s>>>(V, D, g->rank_of, g->level, C.c, part, lvl);
    count_launch();
    launch_fenwick_build(K, D, reinterpret_cast<const long long*>(lvl), tree, s);
    PDNN_LAUNCH_CHECK();
    int32_t nl = 0;
    // (debug build, PDNN_REFINE_TRACE=1) host-timed phases on stderr
    const bool rtrace = debug_knob("PDNN_REFINE_TRACE", 0) != 0;
    auto t_last = std::chrono::steady_clock::now();
    int64_t n_rounds = 0, n_trials = 0;
    auto phase = [&](const char* name) {
        if (!rtrace) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "refine %-10s %9.3f ms  rounds %lld  trials %lld\n", name,
                std::chrono::duration<double, std::milli>(now - t_last).count(), (long long)n_rounds,
                (long long)n_trials);
        t_last = now;
    };
    phase("setup");
    // ---- phase 1: cluster swaps
    if (ns > 0) {
        int32_t* pr = ws_ptr<int32_t>(ws, L.part_rank);
        int64_t* tl = ws_ptr<int64_t>(ws, L.tl_o);
        int64_t* bl = ws_ptr<int64_t>(ws, L.bl_o);
        if ((st = launch_labels(g, part, nullptr, 0, nullptr, pr, s))) return st;
        if ((st = launch_sweep(g, C, pr, tl, bl, ws, L, s))) return st;
        uint64_t* k0 = ws_ptr<uint64_t>(ws, L.rf_keys);
        uint64_t* k1 = k0 + ns;
        int32_t* i0 = ws_ptr<int32_t>(ws, L.rf_ids);
        int32_t* order = i0 + ns;
        RfSec* R = ws_ptr<RfSec>(ws, L.rf_rec);
        int32_t* cnt = ws_ptr<int32_t>(ws, L.rf_cnt);
        int32_t* eoff = ws_ptr<int32_t>(ws, L.rf_eoff);
        int2* ey = ws_ptr<int2>(ws, L.rf_ey);
        long long* ew = ws_ptr<long long>(ws, L.rf_ew);
        uint8_t* marked = ws_ptr<uint8_t>(ws, L.rf_marked);
        k_rf_keys<<<rf_grid(ns), 256, 0, s>>>(K, ns, members, cl_off, tl, k0, i0);
        count_launch();
        PDNN_LAUNCH_CHECK();
        size_t tb = L.rf_temp_bytes;
        PDNN_CUDA_TRY(cub::DeviceRadixSort::SortPairs(ws_ptr<void>(ws, L.rf_temp), tb, k0, k1, i0, order, ns, 0, 64, s));
        count_launch(4);
        const int wgrid = rf_grid((int64_t)ns * 32);
        k_rf_rec<<<wgrid, 256, 0, s>>>(ns, D, order, k1, members, cl_off, cluster_of, g->rank_of, g->orig, g->level, C.c,
                                       tl, g->in_off, g->in_src, g->out_off, g->out_dst, R, cnt);
        count_launch();
        PDNN_LAUNCH_CHECK();
        PDNN_CUDA_TRY(cudaMemsetAsync(cnt + ns, 0, 4, s));
        tb = L.rf_temp_bytes;
        PDNN_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws_ptr<void>(ws, L.rf_temp), tb, cnt, eoff, ns + 1, s));
        count_launch(2);
        k_rf_fill<<<wgrid, 256, 0, s>>>(ns, members, cl_off, cluster_of, g->rank_of, g->orig, g->in_off, g->in_src,
                                        C.in_cost, g->out_off, g->out_dst, C.out_cost, eoff, R, ey, ew);
        count_launch();
        PDNN_CUDA_TRY(cudaMemsetAsync(marked, 0, (size_t)ns, s));
        RfArgs a{};
        a.ns = ns; a.K = K; a.D = D; a.window = window;
        a.R = R; a.ey = ey; a.ew = ew; a.members = members; a.cl_off = cl_off; a.level = g->level;
        a.rank_of = g->rank_of; a.c_rank = C.c; a.part = part; a.tree = tree; a.marked = marked;
        a.log = logd; a.n_log = ctl + 1;
        k_rf_swap<<<1, kRfThreads, 0, s>>>(a);
        count_launch();
        PDNN_LAUNCH_CHECK();
        PDNN_CUDA_TRY(cudaMemcpyAsync(&nl, ctl + 1, 4, cudaMemcpyDeviceToHost, s));
        PDNN_CUDA_TRY(cudaStreamSynchronize(s));
        const int32_t nh = std::min(nl, log_cap);
        if (nh > 0)
            PDNN_CUDA_TRY(cudaMemcpyAsync(log_host, logd, 32 * (size_t)nh, cudaMemcpyDeviceToHost, s));
    }
    phase("swaps");
    // ---- phase 2: node-level passes
    int32_t* cp = ws_ptr<int32_t>(ws, L.cp_nodes);
    int32_t* tn = ws_ptr<int32_t>(ws, L.rf_tn);
    int32_t* tq = ws_ptr<int32_t>(ws, L.rf_tq);
    uint8_t* tdead = ws_ptr<uint8_t>(ws, L.rf_tdead);
    int32_t* elig = ws_ptr<int32_t>(ws, L.rf_elig);
    pdnn_eval_result* res = ws_ptr<pdnn_eval_result>(ws, L.rf_res);
    pdnn_eval_result* resg = ws_ptr<pdnn_eval_result>(ws, L.rf_resg);   // one launch's results
    uint8_t* rows = ws_ptr<uint8_t>(ws, L.rf_rows);
    for (int32_t ps = 0; ps < passes; ++ps) {
        if ((st = rf_sweep_cp(g, C, part, ws, L, cp, ctl + 5, Ld, hash, s))) return st;
        k_rf_copy_L<<<1, 1, 0, s>>>(Ld, L_cur);
        PDNN_CUDA_TRY(cudaMemsetAsync(ctl + 1, 0, 4, s));            // this pass's moves start the device log
        k_rf_trials<<<1, 1024, 0, s>>>(cp, ctl + 5, part, tn, tq, tdead, ctl + 2);
        count_launch(2);
        PDNN_LAUNCH_CHECK();
        for (;;) {
            k_rf_elig<<<1, 1024, 0, s>>>(K, D, ctl + 2, tn, tq, tdead, g->level, g->rank_of, C.c, tree, elig, ctl + 3);
            count_launch();
            PDNN_LAUNCH_CHECK();
            int32_t ne = 0;
            PDNN_CUDA_TRY(cudaMemcpyAsync(&ne, ctl + 3, 4, cudaMemcpyDeviceToHost, s));
            PDNN_CUDA_TRY(cudaStreamSynchronize(s));
            if (ne == 0) break;
            ++n_rounds;
            n_trials += ne;
            // every launch runs the layout's full group (a partial group padded
            // with the current placement): the batched sweep's 2-bit epoch tags
            // rely on every chunk being rewritten at least every other launch --
            // a chunk idle for exactly two launches would hold records with the
            // current tag (stale, yet "ready").  (pdnn_eval_batch keeps this by
            // construction: its partial group always follows a full one, and
            // another batch size is another layout, zeroed by ws_guard.)
            for (int32_t e0 = 0; e0 < ne; e0 += L.B.ng) {
                const int32_t nb = std::min(L.B.ng, ne - e0);
                k_rf_rows<<<rf_grid((int64_t)L.B.ng * V), 256, 0, s>>>(V, L.B.ng, nb, e0, elig, tn, tq, part, rows);
                count_launch();
                PDNN_LAUNCH_CHECK();
                if ((st = launch_bsweep(g, C, 0, L.B.ng, L.B.ng, rows, L.B, ws, resg, s, nullptr, false))) return st;
                PDNN_CUDA_TRY(cudaMemcpyAsync(res + e0, resg, sizeof(pdnn_eval_result) * (size_t)nb,
                                              cudaMemcpyDeviceToDevice, s));
            }
            k_rf_pick<<<1, 1024, 0, s>>>(D, ctl + 3, elig, res, ctl + 2, tn, tq, tdead, g->level, g->rank_of, C.c, part,
                                         tree, L_cur, logd, ctl + 1, ctl + 4);
            count_launch();
            PDNN_LAUNCH_CHECK();
            int32_t moved = 0;
            PDNN_CUDA_TRY(cudaMemcpyAsync(&moved, ctl + 4, 4, cudaMemcpyDeviceToHost, s));
            PDNN_CUDA_TRY(cudaStreamSynchronize(s));
            if (!moved) break;
        }
        int32_t nm = 0;
        PDNN_CUDA_TRY(cudaMemcpyAsync(&nm, ctl + 1, 4, cudaMemcpyDeviceToHost, s));
        PDNN_CUDA_TRY(cudaStreamSynchronize(s));
        const int32_t nh = std::max(0, std::min(nm, log_cap - nl));
        if (nh > 0)
            PDNN_CUDA_TRY(cudaMemcpyAsync(log_host + 4 * (size_t)nl, logd, 32 * (size_t)nh, cudaMemcpyDeviceToHost, s));
        nl += nm;
    }
    phase("passes");
    // L of the final placement
    if ((st = rf_sweep_cp(g, C, part, ws, L, cp, ctl + 5, Ld, hash, s))) return st;
    PDNN_CUDA_TRY(cudaMemcpyAsync(L_host, Ld, 8, cudaMemcpyDeviceToHost, s));
    PDNN_CUDA_TRY(cudaStreamSynchronize(s));
    *n_log = nl;
    return PDNN_OK;
}
