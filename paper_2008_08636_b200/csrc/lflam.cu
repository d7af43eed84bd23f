// lflam.cu -- the LFLAM mapping (Alg. 2; Eq. 2 at
// PAPER.md:366-371): §8(f) NEXT row N4, in reading R21.
//
//   primaries   cluster k < K is PE k (the clusters of pdnn_slice_clusters);
//   order       the secondaries by non-increasing criticality (R19), lower
//               index first;
//   lookahead a secondary sc that is totally-
//               communicating (ext > 0 and one PE takes all of it) or, when
//               CCR >= 10, maximally-communicating (comm(sc, t) * K > ext)
//               joins t, its most communicating PE (lowest on ties), if
//               (a) U >= max(0, work(t) + w(sc) - floor(mean work)),
//               (b) work(t) + w(sc) <= max work, or (c) comm(sc, t) > w(sc),
//               > work(t) and > U; passes repeat while one maps a cluster, at
//               most ceil(log2 |V|) times;
//   balancing   every cluster left joins argmin_pe work(pe, sc) + comm(sc,
//               other PEs) (Eq. 2); ties: the most communicating PE, then
//               the lowest;
//   work(pe,sc) the comp of the nodes on pe whose level is in span(sc) (the
//               levels strictly after the latest parent of sc's first node,
//               strictly before the earliest child of its last node), read
//               from level-indexed binary-indexed trees ("the tree nodes store
//               the weights per level"); U: the same over the
//               nodes of unmapped secondaries other than sc.
//
// B200 design.  Everything a decision reads that no decision
// changes is computed up front, in parallel: the criticality (a labelled sweep
// + per-cluster max, slice.cu), the order (one CUB radix sort), and per
// cluster its span, w(sc), ext(sc) and the flattened list of its external
// edges (one warp per cluster; CUB scan for the offsets).  What is left is the
// algorithm's own sequential chain -- every decision changes the trees and
// the placement the next one reads -- so it runs on ONE warp: the lanes
// gather comm(sc, pe) over the external edges (shared-memory atomics), lane q
// reads PE q's tree range (lane K the unmapped tree), warp shuffles reduce the
// conditions / Eq. 2, and the lanes apply a mapping with atomic tree updates.
// The state (int8 placement, the K + 1 trees) lives in shared memory when it
// fits, else in global memory (volatile loads, L2-coherent); the next
// cluster's static record is prefetched while the current one is decided.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "internal.cuh"

namespace pdnn {

// a secondary's static record, indexed by its position in the criticality order
struct __align__(16) LfRec {
    long long wsc;         // w(sc): total comp of the cluster
    long long ext;         // comm of the edges with exactly one end in the cluster
    int32_t lo, hi;        // span(sc) in levels
    int32_t m0, m1;        // its members' (level, comp) in ml / mc
    int32_t e0, e1;        // its edges to other secondaries in epos / ew
    int32_t k, pad;        // cluster id
};

static int lf_grid(int64_t n, int threads = 256) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 16));
}

// per-(tree, level) comp sums (tree K: the secondaries, all unmapped at the
// start), sum comp / sum comm
__global__ void k_lf_init(int32_t V, int64_t E, int32_t K, int32_t D, const int32_t* __restrict__ rank_of,
                          const int32_t* __restrict__ level, const int64_t* __restrict__ c_rank,
                          const int64_t* __restrict__ in_cost, const int32_t* __restrict__ cluster_of,
                          unsigned long long* __restrict__ lvl, unsigned long long* __restrict__ sums) {
    long long lc = 0, lw = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += stride) {
        const int32_t k = cluster_of[v];
        const long long c = c_rank[rank_of[v]];
        atomicAdd(&lvl[(size_t)(k < K ? k : K) * D + level[v]], (unsigned long long)c);
        lc += c;
    }
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += stride) lw += in_cost[e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lc += __shfl_xor_sync(0xffffffffu, lc, o);
        lw += __shfl_xor_sync(0xffffffffu, lw, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&sums[0], (unsigned long long)lc);
        atomicAdd(&sums[1], (unsigned long long)lw);
    }
}

// Fenwick build from the per-level sums: node i (1-based) of tree q holds the
// levels [i - lowbit(i), i) (0-based)
__global__ void k_lf_build(int32_t T, int32_t D, const long long* __restrict__ lvl, long long* __restrict__ tree) {
    const int64_t n = (int64_t)T * (D + 1);
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const int32_t q = (int32_t)(x / (D + 1)), i = (int32_t)(x % (D + 1));
        long long s = 0;
        if (i > 0)
            for (int32_t l = i - (i & -i); l < i; ++l) s += lvl[(size_t)q * D + l];
        tree[x] = s;
    }
}

// sort keys: criticality descending (the radix sort is stable over the id order)
__global__ void k_lf_keys(int32_t K, int32_t ns, const long long* __restrict__ crit, uint64_t* __restrict__ keys,
                          int32_t* __restrict__ ids) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x) {
        keys[i] = ~(uint64_t)crit[K + i];
        ids[i] = K + i;
    }
}

__global__ void k_lf_pos(int32_t ns, const int32_t* __restrict__ order, int32_t* __restrict__ pos_of) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x) pos_of[order[i]] = i;
}

// one warp per position: span, w(sc), ext(sc); counts of members and of edges
// to other secondaries
__global__ void k_lf_count(int32_t ns, int32_t K, int32_t D, const int32_t* __restrict__ order,
                           const int32_t* __restrict__ members, const int32_t* __restrict__ cl_off,
                           const int32_t* __restrict__ cluster_of, const int32_t* __restrict__ rank_of,
                           const int32_t* __restrict__ orig, const int32_t* __restrict__ level,
                           const int64_t* __restrict__ c_rank, const int32_t* __restrict__ in_off,
                           const int32_t* __restrict__ in_src, const int64_t* __restrict__ in_cost,
                           const int32_t* __restrict__ out_off, const int32_t* __restrict__ out_dst,
                           const int64_t* __restrict__ out_cost, LfRec* __restrict__ R, int32_t* __restrict__ cm,
                           int32_t* __restrict__ ce) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t i = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; i < ns; i += nw) {
        const int32_t k = order[i];
        const int32_t m0 = cl_off[k], m1 = cl_off[k + 1];
        const int32_t rh = rank_of[members[m0]], rt = rank_of[members[m1 - 1]];
        int32_t lo = 0, hi = D - 1;
        for (int32_t e = in_off[rh] + lane; e < in_off[rh + 1]; e += 32) {
            const int32_t p = orig[in_src[e]];
            if (cluster_of[p] != k) lo = max(lo, level[p] + 1);
        }
        for (int32_t e = out_off[rt] + lane; e < out_off[rt + 1]; e += 32) {
            const int32_t x = orig[out_dst[e]];
            if (cluster_of[x] != k) hi = min(hi, level[x] - 1);
        }
        long long wsc = 0, ext = 0;
        int32_t n = 0;
        for (int32_t m = m0 + lane; m < m1; m += 32) {
            const int32_t r = rank_of[members[m]];
            wsc += c_rank[r];
            for (int32_t e = in_off[r]; e < in_off[r + 1]; ++e) {
                const int32_t o = cluster_of[orig[in_src[e]]];
                if (o != k) { ext += in_cost[e]; n += o >= K; }
            }
            for (int32_t e = out_off[r]; e < out_off[r + 1]; ++e) {
                const int32_t o = cluster_of[orig[out_dst[e]]];
                if (o != k) { ext += out_cost[e]; n += o >= K; }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = max(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = min(hi, __shfl_xor_sync(0xffffffffu, hi, o));
            wsc += __shfl_xor_sync(0xffffffffu, wsc, o);
            ext += __shfl_xor_sync(0xffffffffu, ext, o);
            n += __shfl_xor_sync(0xffffffffu, n, o);
        }
        if (lane == 0) {
            LfRec r{};
            r.wsc = wsc; r.ext = ext; r.lo = lo; r.hi = hi; r.k = k;
            R[i] = r;
            cm[i] = m1 - m0;
            ce[i] = n;
        }
    }
}

// one warp per position: members' (level, comp); edges to other secondaries
// (their position, comm); comm to the primaries added into comm[i][pe]
__global__ void k_lf_fill(int32_t ns, int32_t K, const int32_t* __restrict__ order,
                          const int32_t* __restrict__ members, const int32_t* __restrict__ cl_off,
                          const int32_t* __restrict__ cluster_of, const int32_t* __restrict__ pos_of,
                          const int32_t* __restrict__ rank_of, const int32_t* __restrict__ orig,
                          const int32_t* __restrict__ level, const int64_t* __restrict__ c_rank,
                          const int32_t* __restrict__ in_off, const int32_t* __restrict__ in_src,
                          const int64_t* __restrict__ in_cost, const int32_t* __restrict__ out_off,
                          const int32_t* __restrict__ out_dst, const int64_t* __restrict__ out_cost,
                          const int32_t* __restrict__ moff, const int32_t* __restrict__ eoff, LfRec* __restrict__ R,
                          int32_t* __restrict__ ml, long long* __restrict__ mc, int32_t* __restrict__ epos,
                          long long* __restrict__ ew, unsigned long long* __restrict__ comm) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t i = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; i < ns; i += nw) {
        const int32_t k = order[i];
        const int32_t m0 = cl_off[k], m1 = cl_off[k + 1];
        const int32_t mo = moff[i];
        int32_t base = eoff[i];
        if (lane == 0) {
            R[i].m0 = mo; R[i].m1 = mo + (m1 - m0);
            R[i].e0 = base; R[i].e1 = eoff[i + 1];
        }
        for (int32_t mb = m0; mb < m1; mb += 32) {       // warp-uniform trip count
            const int32_t m = mb + lane;
            int32_t n = 0, r = -1;
            if (m < m1) {
                const int32_t u = members[m];
                r = rank_of[u];
                ml[mo + (m - m0)] = level[u];
                mc[mo + (m - m0)] = c_rank[r];
                for (int32_t e = in_off[r]; e < in_off[r + 1]; ++e) {
                    const int32_t o = cluster_of[orig[in_src[e]]];
                    n += o != k && o >= K;
                }
                for (int32_t e = out_off[r]; e < out_off[r + 1]; ++e) {
                    const int32_t o = cluster_of[orig[out_dst[e]]];
                    n += o != k && o >= K;
                }
            }
            int32_t incl = n;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            int32_t p = base + incl - n;
            if (r >= 0) {
                for (int32_t e = in_off[r]; e < in_off[r + 1]; ++e) {
                    const int32_t o = cluster_of[orig[in_src[e]]];
                    if (o == k) continue;
                    if (o < K) atomicAdd(&comm[(size_t)i * K + o], (unsigned long long)in_cost[e]);
                    else { epos[p] = pos_of[o]; ew[p] = in_cost[e]; ++p; }
                }
                for (int32_t e = out_off[r]; e < out_off[r + 1]; ++e) {
                    const int32_t o = cluster_of[orig[out_dst[e]]];
                    if (o == k) continue;
                    if (o < K) atomicAdd(&comm[(size_t)i * K + o], (unsigned long long)out_cost[e]);
                    else { epos[p] = pos_of[o]; ew[p] = out_cost[e]; ++p; }
                }
            }
            base += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
}

// Fenwick queries / updates.  Every lane runs the same trip count (the loops
// are driven by warp-uniform bounds or __any_sync), so the warp never splits:
// with independent thread scheduling a split warp would run the decision's
// shuffles through the divergent (WARPSYNC.COLLECTIVE) path from then on.
__device__ __forceinline__ long long fw_prefix(const volatile long long* t, int32_t i) {   // levels [0, i)
    long long s = 0;
    for (; i > 0; i -= i & -i) s += t[i];
    return s;
}
__device__ __forceinline__ long long fw_range(const volatile long long* t, int32_t lo, int32_t hi) {
    return hi < lo ? 0 : fw_prefix(t, hi + 1) - fw_prefix(t, lo);
}
// tree[tgt] += c and tree[unmapped] -= c at level l for lanes with `on`
template <typename TreeT>
__device__ __forceinline__ void fw_move(TreeT* t_to, TreeT* t_from, int32_t D, int32_t l, long long c, bool on) {
    int32_t i = on ? l + 1 : D + 1;
    while (__any_sync(0xffffffffu, i <= D)) {
        if (i <= D) {
            atomicAdd(reinterpret_cast<unsigned long long*>(const_cast<long long*>(t_to + i)), (unsigned long long)c);
            atomicAdd(reinterpret_cast<unsigned long long*>(const_cast<long long*>(t_from + i)),
                      (unsigned long long)-c);
            i += i & -i;
        }
    }
}

struct LfArgs {
    int32_t K, D, ns, max_iter;
    const LfRec* R;                // [ns] by position
    const int32_t* ml;             // members' levels / comps, by position ranges
    const long long* mc;
    const int32_t* epos;           // edges to other secondaries: their position, comm
    const long long* ew;
    const unsigned long long* sums;   // sum comp, sum comm
    unsigned long long* comm;      // [ns][K] comm(sc, pe), kept current
    long long* tree;               // global trees [K + 1][D + 1]
    int8_t* map;                   // [ns] the PE a position joined
    int32_t* list;                 // [2][ns] the unmapped positions of the next pass
    int32_t* log;                  // [ns][3]
    int32_t* n_log;
    unsigned long long* stats;     // evaluations, passes
    int smem_tree;                 // trees copied into shared memory
    int speculate;                 // lookahead evaluated 32 clusters at a time (see k_lflam)
};

__device__ __forceinline__ LfRec shfl_rec(const LfRec& r, int j) {
    LfRec o;
    o.wsc = __shfl_sync(0xffffffffu, r.wsc, j);
    o.ext = __shfl_sync(0xffffffffu, r.ext, j);
    o.lo = __shfl_sync(0xffffffffu, r.lo, j);
    o.hi = __shfl_sync(0xffffffffu, r.hi, j);
    o.m0 = __shfl_sync(0xffffffffu, r.m0, j);
    o.m1 = __shfl_sync(0xffffffffu, r.m1, j);
    o.e0 = __shfl_sync(0xffffffffu, r.e0, j);
    o.e1 = __shfl_sync(0xffffffffu, r.e1, j);
    o.k = __shfl_sync(0xffffffffu, r.k, j);
    return o;
}

// the sequential decisions on one warp.  The static records of the next 32
// positions of a pass are loaded at once (one per lane) and broadcast; a
// decision reads comm(sc, .) (one row) and the K + 1 tree ranges together.
template <bool kSmemTree>
__global__ void __launch_bounds__(32) k_lflam(LfArgs a) {
    extern __shared__ __align__(16) long long lf_tree_s[];
    const int lane = threadIdx.x;
    const int32_t K = a.K, D = a.D, T = K + 1;
    long long* tree = kSmemTree ? lf_tree_s : a.tree;
    if (kSmemTree)
        for (int32_t x0 = 0; x0 < T * (D + 1); x0 += 32)
            if (x0 + lane < T * (D + 1)) lf_tree_s[x0 + lane] = a.tree[x0 + lane];
    __syncwarp();
    const volatile long long* vtree = tree;
    const volatile long long* vcomm = reinterpret_cast<const volatile long long*>(a.comm);
    const bool high_ccr = (long long)a.sums[1] >= 10 * (long long)a.sums[0];
    int kp = 1;                                      // lanes [0, kp) hold the K PEs
    while (kp < K) kp <<= 1;
    const volatile int32_t* cur = nullptr;           // nullptr: every position, in order
    int32_t n = a.ns, nl = 0, flip = 0;
    unsigned long long evals = 0, passes = 0;
    for (int phase = 0; phase < 2; ++phase) {
        for (int32_t iter = 0; iter < (phase == 0 ? a.max_iter : 1); ++iter) {
            int32_t* nxt = a.list + (size_t)flip * a.ns;
            int32_t nn = 0, nmapped = 0;
            ++passes;
            // target_pri <- target_pri + {sc}: the trees, and comm(sc', tgt) of
            // every secondary sc' it talks to
            auto apply = [&](int32_t p, const LfRec& I, int32_t tgt) {
                for (int32_t m0 = I.m0; m0 < I.m1; m0 += 32) {
                    const int32_t m = m0 + lane;
                    const bool on = m < I.m1;
                    const int32_t l = on ? __ldg(a.ml + m) : 0;
                    const long long c = on ? __ldg(a.mc + m) : 0;
                    fw_move(tree + (size_t)tgt * (D + 1), tree + (size_t)K * (D + 1), D, l, c, on);
                }
                for (int32_t e0 = I.e0; e0 < I.e1; e0 += 32) {
                    const int32_t e = e0 + lane;
                    if (e < I.e1)
                        atomicAdd(a.comm + (size_t)__ldg(a.epos + e) * K + tgt, (unsigned long long)__ldg(a.ew + e));
                }
                if (lane == 0) {
                    a.map[p] = (int8_t)tgt;
                    a.log[3 * nl] = I.k;
                    a.log[3 * nl + 1] = phase;
                    a.log[3 * nl + 2] = tgt;
                }
                ++nl;
                ++nmapped;
                __syncwarp();
            };
            for (int32_t b = 0; b < n; b += 32) {
                const int32_t cnt = min(32, n - b);
                const int32_t idx = min(b + lane, n - 1);      // lanes past the end repeat the last
                const int32_t pl = cur ? cur[idx] : idx;
                const LfRec rl = a.R[pl];
                if (phase == 0 && a.speculate) {
                    // Lookahead, screened 32 at a time: lane l tests position j0 + l's
                    // eligibility (totally / maximally communicating: its comm row
                    // only) against the current state.  Ineligible positions map
                    // nothing and change nothing, so the run before the first
                    // eligible one is settled at once; that one is decided by the
                    // warp as in the sequential loop, and the screen resumes after
                    // it (later lanes are re-tested against the new state).
                    int32_t j0 = 0;
                    while (j0 < cnt) {
                        const bool valid = j0 + lane < cnt;
                        const int32_t jj = valid ? j0 + lane : cnt - 1;
                        const int32_t pj = __shfl_sync(0xffffffffu, pl, jj);
                        const long long ext = __shfl_sync(0xffffffffu, rl.ext, jj);
                        long long bc = -1;
                        {
                            long long cr[PDNN_MAX_PE];
                            const unsigned long long* row = a.comm + (size_t)pj * K;
#pragma unroll
                            for (int32_t q = 0; q < PDNN_MAX_PE; ++q) cr[q] = q < K ? (long long)__ldcg(row + q) : -1;
#pragma unroll
                            for (int32_t q = 0; q < PDNN_MAX_PE; ++q) bc = cr[q] > bc ? cr[q] : bc;
                        }
                        const bool elig = valid && ((ext > 0 && bc == ext) || (high_ccr && bc * K > ext));
                        const unsigned mm = __ballot_sync(0xffffffffu, elig);
                        const int32_t first = mm ? __ffs(mm) - 1 : cnt - j0;   // lanes [0, first): not eligible
                        if (lane < first) nxt[nn + lane] = pj;
                        nn += first;
                        evals += first;
                        __syncwarp();
                        if (!mm) break;
                        j0 += first;
                        // the eligible position: the sequential decision (warp-wide)
                        const int32_t p = __shfl_sync(0xffffffffu, pl, j0);
                        const LfRec I = shfl_rec(rl, j0);
                        ++evals;
                        const long long comm = lane < K ? vcomm[(size_t)p * K + lane] : 0;
                        long long work = fw_range(vtree + (size_t)min(lane, K) * (D + 1), I.lo, I.hi);
                        long long bc2 = lane < K ? comm : -1;
                        int32_t bt = lane;
                        for (int o = kp >> 1; o > 0; o >>= 1) {
                            const long long oc = __shfl_xor_sync(0xffffffffu, bc2, o);
                            const int32_t ot = __shfl_xor_sync(0xffffffffu, bt, o);
                            if (oc > bc2 || (oc == bc2 && ot < bt)) { bc2 = oc; bt = ot; }
                        }
                        bc2 = __shfl_sync(0xffffffffu, bc2, 0);
                        bt = __shfl_sync(0xffffffffu, bt, 0);
                        const long long U = __shfl_sync(0xffffffffu, work, K) - I.wsc;
                        const long long wt = __shfl_sync(0xffffffffu, work, bt);
                        long long sum = lane < K ? work : 0, mx = sum;
                        for (int o = kp >> 1; o > 0; o >>= 1) {
                            sum += __shfl_xor_sync(0xffffffffu, sum, o);
                            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                        }
                        sum = __shfl_sync(0xffffffffu, sum, 0);
                        mx = __shfl_sync(0xffffffffu, mx, 0);
                        long long imb = wt + I.wsc - sum / K;
                        if (imb < 0) imb = 0;
                        const bool ca = U >= imb, cb = wt + I.wsc <= mx;
                        const bool cc = bc2 > I.wsc && bc2 > wt && bc2 > U;
                        if (ca || cb || cc) {
                            apply(p, I, bt);
                        } else {
                            if (lane == 0) nxt[nn] = p;
                            ++nn;
                            __syncwarp();
                        }
                        ++j0;
                    }
                    continue;
                }
                for (int32_t j = 0; j < cnt; ++j) {
                    const int32_t p = __shfl_sync(0xffffffffu, pl, j);
                    const LfRec I = shfl_rec(rl, j);
                    ++evals;
                    // comm(sc, pe) on lane pe; the tree ranges (issued now, used only if
                    // needed): lane q < K PE q, lane K unmapped
                    const long long comm = lane < K ? vcomm[(size_t)p * K + lane] : 0;
                    long long work = fw_range(vtree + (size_t)min(lane, K) * (D + 1), I.lo, I.hi);
                    int32_t tgt = -1;
                    if (phase == 0) {
                        // t = the most communicating PE, lowest on ties
                        long long bc = lane < K ? comm : -1;
                        int32_t bt = lane;
                        for (int o = kp >> 1; o > 0; o >>= 1) {
                            const long long oc = __shfl_xor_sync(0xffffffffu, bc, o);
                            const int32_t ot = __shfl_xor_sync(0xffffffffu, bt, o);
                            if (oc > bc || (oc == bc && ot < bt)) { bc = oc; bt = ot; }
                        }
                        bc = __shfl_sync(0xffffffffu, bc, 0);
                        bt = __shfl_sync(0xffffffffu, bt, 0);
                        const bool totally = I.ext > 0 && bc == I.ext;
                        const bool maximally = bc * K > I.ext;
                        if (totally || (high_ccr && maximally)) {
                            const long long U = __shfl_sync(0xffffffffu, work, K) - I.wsc;
                            const long long wt = __shfl_sync(0xffffffffu, work, bt);
                            long long sum = lane < K ? work : 0, mx = sum;
                            for (int o = kp >> 1; o > 0; o >>= 1) {
                                sum += __shfl_xor_sync(0xffffffffu, sum, o);
                                mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                            }
                            sum = __shfl_sync(0xffffffffu, sum, 0);
                            mx = __shfl_sync(0xffffffffu, mx, 0);
                            long long imb = wt + I.wsc - sum / K;
                            if (imb < 0) imb = 0;
                            const bool ca = U >= imb, cb = wt + I.wsc <= mx;
                            const bool cc = bc > I.wsc && bc > wt && bc > U;
                            if (ca || cb || cc) tgt = bt;
                        }
                    } else {
                        // Eq. 2: min work(pe) + comm to the other PEs; ties: most comm, lowest PE
                        long long tot = comm;
                        for (int o = kp >> 1; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
                        tot = __shfl_sync(0xffffffffu, tot, 0);
                        long long bcost = lane < K ? work + (tot - comm) : LLONG_MAX, bc = comm;
                        int32_t bt = lane;
                        for (int o = kp >> 1; o > 0; o >>= 1) {
                            const long long ocost = __shfl_xor_sync(0xffffffffu, bcost, o);
                            const long long oc = __shfl_xor_sync(0xffffffffu, bc, o);
                            const int32_t ot = __shfl_xor_sync(0xffffffffu, bt, o);
                            if (ocost < bcost || (ocost == bcost && (oc > bc || (oc == bc && ot < bt)))) {
                                bcost = ocost; bc = oc; bt = ot;
                            }
                        }
                        tgt = __shfl_sync(0xffffffffu, bt, 0);
                    }
                    if (tgt < 0) {
                        if (lane == 0) nxt[nn] = p;
                        ++nn;
                        continue;
                    }
                    apply(p, I, tgt);
                }
            }
            __syncwarp();
            cur = nxt;
            n = nn;
            flip ^= 1;
            if (phase == 0 && nmapped == 0) break;
        }
    }
    if (lane == 0) {
        *a.n_log = nl;
        a.stats[0] = evals;
        a.stats[1] = passes;
    }
}

__global__ void k_lf_part(int32_t V, int32_t K, const int32_t* __restrict__ cluster_of,
                          const int32_t* __restrict__ pos_of, const int8_t* __restrict__ map,
                          int32_t* __restrict__ part) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        const int32_t k = cluster_of[v];
        part[v] = k < K ? k : map[pos_of[k]];
    }
}

void launch_fenwick_build(int32_t T, int32_t D, const long long* lvl, long long* tree, cudaStream_t s) {
    k_lf_build<<<lf_grid((int64_t)T * (D + 1)), 256, 0, s>>>(T, D, lvl, tree);
    count_launch();
}

size_t lflam_temp_bytes(int32_t n) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, std::max(n, 1));
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const int32_t*)nullptr, (int32_t*)nullptr, std::max(n, 1) + 1);
    return std::max(a, b);
}

constexpr size_t kLfSmemMax = 200 * 1024;

}  // namespace pdnn

using namespace pdnn;

extern "C" pdnn_status pdnn_lflam(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                                  const int32_t* cluster_of, const int32_t* members, const int32_t* cl_off,
                                  int32_t n_clusters, int32_t K, int32_t* part, int32_t* log, int32_t* n_log,
                                  void* ws, size_t ws_bytes, void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (K < 1 || K > PDNN_MAX_PE || n_clusters < K || n_clusters > g->V + K || !cl_off || !n_log ||
        (g->V > 0 && (!cluster_of || !members || !part)) || (n_clusters > K && !log)) {
        set_error("bad K / n_clusters or null argument");
        return PDNN_EINVAL;
    }
    const WsLayout L = ws_layout(g, PDNN_OP_LFLAM, 0);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    pdnn_status st = ws_guard(ws, 0, 0, L.single_end, L.sig_single, s);
    if (st) return st;
    if ((st = ws_guard(ws, 1, L.single_end, L.total, L.sig_batch, s))) return st;
    const int32_t V = g->V, D = std::max(g->n_levels, 1), nc = n_clusters, ns = nc - K, T = K + 1;
    PDNN_CUDA_TRY(cudaMemsetAsync(n_log, 0, 4, s));
    if (V == 0) return PDNN_OK;
    Costs C;
    if ((st = resolve_costs(g, node_cost, edge_cost, ws, L, s, &C, /*need_blob=*/true))) return st;
    unsigned long long* lvl = ws_ptr<unsigned long long>(ws, L.lf_lvl);
    long long* tree = ws_ptr<long long>(ws, L.lf_tree);
    LfRec* R = ws_ptr<LfRec>(ws, L.lf_rec);
    int32_t* cm = ws_ptr<int32_t>(ws, L.lf_cm);
    int32_t* ce = ws_ptr<int32_t>(ws, L.lf_ce);
    int32_t* moff = ws_ptr<int32_t>(ws, L.lf_moff);
    int32_t* eoff = ws_ptr<int32_t>(ws, L.lf_eoff);
    int32_t* ml = ws_ptr<int32_t>(ws, L.lf_ml);
    long long* mc = ws_ptr<long long>(ws, L.lf_mc);
    int32_t* epos = ws_ptr<int32_t>(ws, L.lf_epos);
    long long* ew = ws_ptr<long long>(ws, L.lf_ew);
    unsigned long long* comm = ws_ptr<unsigned long long>(ws, L.lf_comm);
    long long* crit = ws_ptr<long long>(ws, L.lf_crit);
    uint64_t* k0 = ws_ptr<uint64_t>(ws, L.lf_keys);
    uint64_t* k1 = k0 + std::max(ns, 1);
    int32_t* i0 = ws_ptr<int32_t>(ws, L.lf_ids);
    int32_t* order = i0 + std::max(ns, 1);
    int32_t* pos_of = ws_ptr<int32_t>(ws, L.lf_pos);
    int32_t* list = ws_ptr<int32_t>(ws, L.lf_list);
    int8_t* map = ws_ptr<int8_t>(ws, L.lf_map);
    unsigned long long* sums = ws_ptr<unsigned long long>(ws, L.lf_ctl);     // [0..1] sums, [2..3] stats
    // criticality (R19) and the order
    if ((st = launch_criticality(g, C, cluster_of, nc, reinterpret_cast<int64_t*>(crit), ws, L, s))) return st;
    PDNN_CUDA_TRY(cudaMemsetAsync(sums, 0, 32, s));
    // trees (the primaries on their PEs, every secondary unmapped)
    PDNN_CUDA_TRY(cudaMemsetAsync(lvl, 0, 8 * (size_t)T * D, s));
    k_lf_init<<<lf_grid(std::max<int64_t>(V, g->E)), 256, 0, s>>>(V, g->E, K, D, g->rank_of, g->level, C.c,
                                                                  C.in_cost, cluster_of, lvl, sums);
    count_launch();
    k_lf_build<<<lf_grid((int64_t)T * (D + 1)), 256, 0, s>>>(T, D, reinterpret_cast<const long long*>(lvl), tree);
    count_launch();
    PDNN_LAUNCH_CHECK();
    if (ns > 0) {
        k_lf_keys<<<lf_grid(ns), 256, 0, s>>>(K, ns, crit, k0, i0);
        count_launch();
        PDNN_LAUNCH_CHECK();
        size_t tb = L.lf_temp_bytes;
        PDNN_CUDA_TRY(cub::DeviceRadixSort::SortPairs(ws_ptr<void>(ws, L.lf_temp), tb, k0, k1, i0, order, ns, 0, 64,
                                                      s));
        count_launch(4);
        k_lf_pos<<<lf_grid(ns), 256, 0, s>>>(ns, order, pos_of);
        count_launch();
        // per-position static records, members and edges; comm to the primaries
        const int grid = lf_grid((int64_t)ns * 32);
        k_lf_count<<<grid, 256, 0, s>>>(ns, K, D, order, members, cl_off, cluster_of, g->rank_of, g->orig, g->level,
                                        C.c, g->in_off, g->in_src, C.in_cost, g->out_off, g->out_dst, C.out_cost, R,
                                        cm, ce);
        count_launch();
        PDNN_LAUNCH_CHECK();
        PDNN_CUDA_TRY(cudaMemsetAsync(cm + ns, 0, 4, s));
        PDNN_CUDA_TRY(cudaMemsetAsync(ce + ns, 0, 4, s));
        tb = L.lf_temp_bytes;
        PDNN_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws_ptr<void>(ws, L.lf_temp), tb, cm, moff, ns + 1, s));
        tb = L.lf_temp_bytes;
        PDNN_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws_ptr<void>(ws, L.lf_temp), tb, ce, eoff, ns + 1, s));
        count_launch(4);
        PDNN_CUDA_TRY(cudaMemsetAsync(comm, 0, 8 * (size_t)ns * K, s));
        k_lf_fill<<<grid, 256, 0, s>>>(ns, K, order, members, cl_off, cluster_of, pos_of, g->rank_of, g->orig,
                                       g->level, C.c, g->in_off, g->in_src, C.in_cost, g->out_off, g->out_dst,
                                       C.out_cost, moff, eoff, R, ml, mc, epos, ew, comm);
        count_launch();
        PDNN_LAUNCH_CHECK();
        // the sequential decisions
        int32_t max_iter = 0;
        while ((1ll << max_iter) < (int64_t)V) ++max_iter;    // ceil(log2 |V|)
        if (max_iter < 1) max_iter = 1;
        LfArgs a{};
        a.K = K; a.D = D; a.ns = ns; a.max_iter = max_iter;
        a.R = R; a.ml = ml; a.mc = mc; a.epos = epos; a.ew = ew; a.sums = sums; a.comm = comm; a.tree = tree;
        a.map = map; a.list = list; a.log = log; a.n_log = n_log; a.stats = sums + 2;
        a.speculate = debug_knob("PDNN_LFLAM_SPECULATE", 1);
        const size_t tree_b = (size_t)8 * T * (D + 1);
        size_t smem = 0;
        if (debug_knob("PDNN_LFLAM_GLOBAL", 0) == 0 && tree_b <= kLfSmemMax) { a.smem_tree = 1; smem = tree_b; }
        if (a.smem_tree) {
            if (smem > 48 * 1024)
                PDNN_CUDA_TRY(cudaFuncSetAttribute(k_lflam<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)smem));
            k_lflam<true><<<1, 32, smem, s>>>(a);
        } else {
            k_lflam<false><<<1, 32, 0, s>>>(a);
        }
        count_launch();
        PDNN_LAUNCH_CHECK();
    }
    k_lf_part<<<lf_grid(V), 256, 0, s>>>(V, K, cluster_of, pos_of, map, part);
    count_launch();
    PDNN_LAUNCH_CHECK();
    return PDNN_OK;
}

#ifdef PDNN_DEBUG_KNOBS
// diagnostics (debug-knob builds only): decisions evaluated and passes run by
// the last pdnn_lflam on this workspace
extern "C" pdnn_status pdnn_debug_lflam_stats(const pdnn_graph* g, void* ws, unsigned long long* out_host) {
    const WsLayout L = ws_layout(g, PDNN_OP_LFLAM, 0);
    PDNN_CUDA_TRY(cudaMemcpy(out_host, ws_ptr<unsigned long long>(ws, L.lf_ctl) + 2, 16, cudaMemcpyDeviceToHost));
    return PDNN_OK;
}
#endif
