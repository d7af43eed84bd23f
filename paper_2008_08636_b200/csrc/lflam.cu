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

struct LfInfo {
    long long wsc;   // w(sc): total comp of the cluster
    long long ext;   // comm of the edges with exactly one end in the cluster
    int32_t lo, hi;  // span(sc) in levels
};

static int lf_grid(int64_t n, int threads = 256) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 16));
}

// part8 (primaries' labels, -1 elsewhere), per-(tree, level) comp sums, sum comp / comm
__global__ void k_lf_init(int32_t V, int64_t E, int32_t K, int32_t D, const int32_t* __restrict__ rank_of,
                          const int32_t* __restrict__ level, const int64_t* __restrict__ c_rank,
                          const int64_t* __restrict__ in_cost, const int32_t* __restrict__ cluster_of,
                          int8_t* __restrict__ part8, unsigned long long* __restrict__ lvl,
                          unsigned long long* __restrict__ sums) {
    long long lc = 0, lw = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += stride) {
        const int32_t k = cluster_of[v];
        const int32_t q = k < K ? k : K;
        part8[v] = (int8_t)(k < K ? k : -1);
        const long long c = c_rank[rank_of[v]];
        atomicAdd(&lvl[(size_t)q * D + level[v]], (unsigned long long)c);
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
// levels (i - lowbit(i), i]
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

// one warp per secondary: span, w(sc), ext(sc), external-edge count; members'
// comp and level in member order (the sequential kernel's apply loop)
__global__ void k_lf_cluster(int32_t K, int32_t nc, int32_t D, const int32_t* __restrict__ members,
                             const int32_t* __restrict__ cl_off, const int32_t* __restrict__ cluster_of,
                             const int32_t* __restrict__ rank_of, const int32_t* __restrict__ orig,
                             const int32_t* __restrict__ level, const int64_t* __restrict__ c_rank,
                             const int32_t* __restrict__ in_off, const int32_t* __restrict__ in_src,
                             const int64_t* __restrict__ in_cost, const int32_t* __restrict__ out_off,
                             const int32_t* __restrict__ out_dst, const int64_t* __restrict__ out_cost,
                             LfInfo* __restrict__ info, int32_t* __restrict__ cnt, long long* __restrict__ mc,
                             int32_t* __restrict__ ml) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t k = K + blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; k < nc; k += nw) {
        const int32_t m0 = cl_off[k], m1 = cl_off[k + 1];
        const int32_t h = members[m0], t = members[m1 - 1];
        int32_t lo = 0, hi = D - 1;
        const int32_t rh = rank_of[h], rt = rank_of[t];
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
            const int32_t u = members[m], r = rank_of[u];
            const long long c = c_rank[r];
            wsc += c;
            mc[m] = c;
            ml[m] = level[u];
            for (int32_t e = in_off[r]; e < in_off[r + 1]; ++e)
                if (cluster_of[orig[in_src[e]]] != k) { ext += in_cost[e]; ++n; }
            for (int32_t e = out_off[r]; e < out_off[r + 1]; ++e)
                if (cluster_of[orig[out_dst[e]]] != k) { ext += out_cost[e]; ++n; }
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
            info[k] = LfInfo{wsc, ext, lo, hi};
            cnt[k] = n;
        }
    }
}

// one warp per secondary: its external edges (other end's id, comm) at off[k]
__global__ void k_lf_fill(int32_t K, int32_t nc, const int32_t* __restrict__ members,
                          const int32_t* __restrict__ cl_off, const int32_t* __restrict__ cluster_of,
                          const int32_t* __restrict__ rank_of, const int32_t* __restrict__ orig,
                          const int32_t* __restrict__ in_off, const int32_t* __restrict__ in_src,
                          const int64_t* __restrict__ in_cost, const int32_t* __restrict__ out_off,
                          const int32_t* __restrict__ out_dst, const int64_t* __restrict__ out_cost,
                          const int32_t* __restrict__ off, int32_t* __restrict__ enode, long long* __restrict__ ew) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t k = K + blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; k < nc; k += nw) {
        const int32_t m0 = cl_off[k], m1 = cl_off[k + 1];
        int32_t base = off[k];
        for (int32_t mb = m0; mb < m1; mb += 32) {       // warp-uniform trip count
            const int32_t m = mb + lane;
            int32_t n = 0, r = -1;
            if (m < m1) {
                r = rank_of[members[m]];
                for (int32_t e = in_off[r]; e < in_off[r + 1]; ++e) n += cluster_of[orig[in_src[e]]] != k;
                for (int32_t e = out_off[r]; e < out_off[r + 1]; ++e) n += cluster_of[orig[out_dst[e]]] != k;
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
                    const int32_t x = orig[in_src[e]];
                    if (cluster_of[x] != k) { enode[p] = x; ew[p] = in_cost[e]; ++p; }
                }
                for (int32_t e = out_off[r]; e < out_off[r + 1]; ++e) {
                    const int32_t x = orig[out_dst[e]];
                    if (cluster_of[x] != k) { enode[p] = x; ew[p] = out_cost[e]; ++p; }
                }
            }
            base += __shfl_sync(0xffffffffu, incl, 31);
        }
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

__device__ __forceinline__ long long fw_prefix(const volatile long long* t, int32_t i) {   // levels [0, i)
    long long s = 0;
    for (; i > 0; i -= i & -i) s += t[i];
    return s;
}
__device__ __forceinline__ long long fw_range(const volatile long long* t, int32_t lo, int32_t hi) {
    return hi < lo ? 0 : fw_prefix(t, hi + 1) - fw_prefix(t, lo);
}
__device__ __forceinline__ void fw_add(long long* t, int32_t D, int32_t l, long long v) {
    for (int32_t i = l + 1; i <= D; i += i & -i) atomicAdd(reinterpret_cast<unsigned long long*>(t + i),
                                                           (unsigned long long)v);
}

struct LfArgs {
    int32_t V, K, D, ns, max_iter;
    const int32_t* order;          // [ns] secondaries by criticality
    const LfInfo* info;
    const int32_t* off;            // [nc + 1] external-edge offsets
    const int32_t* enode;
    const long long* ew;
    const int32_t* cl_off;
    const int32_t* members;
    const long long* mc;
    const int32_t* ml;
    const unsigned long long* sums;   // sum comp, sum comm
    int8_t* part8;                 // global placement (in / out)
    long long* tree;               // global trees [K + 1][D + 1]
    int32_t* list;                 // [2][ns] the unmapped clusters of the next pass
    int32_t* log;                  // [ns][3]
    int32_t* n_log;
    int smem_part, smem_tree;      // state copied into shared memory
};

// the sequential decisions on one warp
__global__ void __launch_bounds__(32) k_lflam(LfArgs a) {
    extern __shared__ __align__(16) unsigned char lf_sm[];
    volatile long long* comm_s = reinterpret_cast<long long*>(lf_sm);              // [PDNN_MAX_PE]
    unsigned char* dyn = lf_sm + 8 * PDNN_MAX_PE;
    const int lane = threadIdx.x;
    const int32_t K = a.K, D = a.D, T = K + 1;
    long long* tree = a.tree;
    int8_t* part = a.part8;
    if (a.smem_tree) {
        tree = reinterpret_cast<long long*>(dyn);
        for (int32_t x = lane; x < T * (D + 1); x += 32) tree[x] = a.tree[x];
        dyn += ((size_t)8 * T * (D + 1) + 15) & ~size_t(15);
    }
    if (a.smem_part) {
        part = reinterpret_cast<int8_t*>(dyn);
        for (int32_t x = lane; x < a.V; x += 32) part[x] = a.part8[x];
    }
    __syncwarp();
    const volatile long long* vtree = tree;
    const volatile int8_t* vpart = part;
    const bool high_ccr = (long long)a.sums[1] >= 10 * (long long)a.sums[0];
    const int32_t* cur = a.order;
    int32_t n = a.ns, nl = 0, flip = 0;
    for (int phase = 0; phase < 2; ++phase) {
        for (int32_t iter = 0; iter < (phase == 0 ? a.max_iter : 1); ++iter) {
            int32_t* nxt = a.list + (size_t)flip * a.ns;
            int32_t nn = 0, nmapped = 0;
            // prefetch of the first cluster's static record
            const volatile int32_t* vcur = cur;      // lane 0 wrote it in the previous pass
            int32_t pk = n > 0 ? vcur[0] : 0;
            for (int32_t i = 0; i < n; ++i) {
                const int32_t k = pk;
                const LfInfo I = a.info[k];
                const int32_t e0 = a.off[k], e1 = a.off[k + 1];
                if (i + 1 < n) pk = vcur[i + 1];
                if (lane < K) comm_s[lane] = 0;
                __syncwarp();
                // the tree ranges (independent of comm): lane q < K PE q, lane K unmapped
                long long work = 0;
                if (lane <= K) work = fw_range(vtree + (size_t)lane * (D + 1), I.lo, I.hi);
                for (int32_t e = e0 + lane; e < e1; e += 32) {
                    const int32_t q = vpart[__ldg(a.enode + e)];
                    if (q >= 0) atomicAdd(const_cast<unsigned long long*>(reinterpret_cast<volatile unsigned long long*>(&comm_s[q])),
                                          (unsigned long long)__ldg(a.ew + e));
                }
                __syncwarp();
                const long long comm = lane < K ? comm_s[lane] : 0;
                const long long U = __shfl_sync(0xffffffffu, work, K) - I.wsc;
                if (lane >= K) work = 0;
                long long sum = work, mx = work, tot = comm;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    sum += __shfl_xor_sync(0xffffffffu, sum, o);
                    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                    tot += __shfl_xor_sync(0xffffffffu, tot, o);
                }
                int32_t tgt = -1;
                if (phase == 0) {
                    // t = the most communicating PE, lowest on ties
                    long long bc = lane < K ? comm : -1;
                    int32_t bt = lane;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const long long oc = __shfl_xor_sync(0xffffffffu, bc, o);
                        const int32_t ot = __shfl_xor_sync(0xffffffffu, bt, o);
                        if (oc > bc || (oc == bc && ot < bt)) { bc = oc; bt = ot; }
                    }
                    const long long wt = __shfl_sync(0xffffffffu, work, bt);
                    const bool totally = I.ext > 0 && bc == I.ext;
                    const bool maximally = bc * K > I.ext;
                    if (totally || (high_ccr && maximally)) {
                        long long imb = wt + I.wsc - sum / K;
                        if (imb < 0) imb = 0;
                        const bool ca = U >= imb, cb = wt + I.wsc <= mx;
                        const bool cc = bc > I.wsc && bc > wt && bc > U;
                        if (ca || cb || cc) tgt = bt;
                    }
                } else {
                    // Eq. 2: min work(pe) + comm to the other PEs; ties: most comm, lowest PE
                    long long bcost = lane < K ? work + (tot - comm) : LLONG_MAX, bc = comm;
                    int32_t bt = lane;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const long long ocost = __shfl_xor_sync(0xffffffffu, bcost, o);
                        const long long oc = __shfl_xor_sync(0xffffffffu, bc, o);
                        const int32_t ot = __shfl_xor_sync(0xffffffffu, bt, o);
                        if (ocost < bcost || (ocost == bcost && (oc > bc || (oc == bc && ot < bt)))) {
                            bcost = ocost; bc = oc; bt = ot;
                        }
                    }
                    tgt = bt;
                }
                if (tgt < 0) {
                    if (lane == 0) nxt[nn] = k;
                    ++nn;
                    continue;
                }
                // target_pri <- target_pri + {sc}
                const int32_t m0 = a.cl_off[k], m1 = a.cl_off[k + 1];
                for (int32_t m = m0 + lane; m < m1; m += 32) {
                    const int32_t u = __ldg(a.members + m), l = __ldg(a.ml + m);
                    const long long c = __ldg(a.mc + m);
                    part[u] = (int8_t)tgt;
                    fw_add(tree + (size_t)tgt * (D + 1), D, l, c);
                    fw_add(tree + (size_t)K * (D + 1), D, l, -c);
                }
                if (lane == 0) {
                    a.log[3 * nl] = k;
                    a.log[3 * nl + 1] = phase;
                    a.log[3 * nl + 2] = tgt;
                }
                ++nl;
                ++nmapped;
                __syncwarp();
            }
            __syncwarp();
            cur = nxt;
            n = nn;
            flip ^= 1;
            if (phase == 0 && nmapped == 0) break;
        }
    }
    __syncwarp();
    if (a.smem_part)
        for (int32_t x = lane; x < a.V; x += 32) a.part8[x] = part[x];
    if (lane == 0) *a.n_log = nl;
}

__global__ void k_lf_out(int32_t V, const int8_t* __restrict__ part8, int32_t* __restrict__ part) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) part[v] = part8[v];
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
    int8_t* part8 = ws_ptr<int8_t>(ws, L.lf_part8);
    LfInfo* info = ws_ptr<LfInfo>(ws, L.lf_info);
    int32_t* cnt = ws_ptr<int32_t>(ws, L.lf_cnt);
    int32_t* off = ws_ptr<int32_t>(ws, L.lf_off);
    int32_t* enode = ws_ptr<int32_t>(ws, L.lf_enode);
    long long* ew = ws_ptr<long long>(ws, L.lf_ew);
    long long* mc = ws_ptr<long long>(ws, L.lf_mc);
    int32_t* ml = ws_ptr<int32_t>(ws, L.lf_ml);
    long long* crit = ws_ptr<long long>(ws, L.lf_crit);
    uint64_t* k0 = ws_ptr<uint64_t>(ws, L.lf_keys);
    uint64_t* k1 = k0 + std::max(ns, 1);
    int32_t* i0 = ws_ptr<int32_t>(ws, L.lf_ids);
    int32_t* i1 = i0 + std::max(ns, 1);
    int32_t* list = ws_ptr<int32_t>(ws, L.lf_list);
    unsigned long long* sums = ws_ptr<unsigned long long>(ws, L.lf_ctl);
    // criticality (R19) and the order
    if ((st = launch_criticality(g, C, cluster_of, nc, reinterpret_cast<int64_t*>(crit), ws, L, s))) return st;
    if (ns > 0) {
        k_lf_keys<<<lf_grid(ns), 256, 0, s>>>(K, ns, crit, k0, i0);
        count_launch();
        PDNN_LAUNCH_CHECK();
        size_t tb = L.lf_temp_bytes;
        PDNN_CUDA_TRY(cub::DeviceRadixSort::SortPairs(ws_ptr<void>(ws, L.lf_temp), tb, k0, k1, i0, i1, ns, 0, 64, s));
        count_launch(4);
    }
    // trees and placement of the primaries
    PDNN_CUDA_TRY(cudaMemsetAsync(lvl, 0, 8 * (size_t)T * D, s));
    PDNN_CUDA_TRY(cudaMemsetAsync(sums, 0, 16, s));
    k_lf_init<<<lf_grid(std::max<int64_t>(V, g->E)), 256, 0, s>>>(V, g->E, K, D, g->rank_of, g->level, C.c,
                                                                  C.in_cost, cluster_of, part8, lvl, sums);
    count_launch();
    k_lf_build<<<lf_grid((int64_t)T * (D + 1)), 256, 0, s>>>(T, D, reinterpret_cast<const long long*>(lvl), tree);
    count_launch();
    PDNN_LAUNCH_CHECK();
    // per-secondary static records and external edges
    PDNN_CUDA_TRY(cudaMemsetAsync(cnt, 0, 4 * ((size_t)nc + 1), s));
    if (ns > 0) {
        const int grid = lf_grid((int64_t)ns * 32);
        k_lf_cluster<<<grid, 256, 0, s>>>(K, nc, D, members, cl_off, cluster_of, g->rank_of, g->orig, g->level, C.c,
                                          g->in_off, g->in_src, C.in_cost, g->out_off, g->out_dst, C.out_cost, info,
                                          cnt, mc, ml);
        count_launch();
        PDNN_LAUNCH_CHECK();
    }
    size_t tb = L.lf_temp_bytes;
    PDNN_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws_ptr<void>(ws, L.lf_temp), tb, cnt, off, nc + 1, s));
    count_launch(2);
    if (ns > 0) {
        const int grid = lf_grid((int64_t)ns * 32);
        k_lf_fill<<<grid, 256, 0, s>>>(K, nc, members, cl_off, cluster_of, g->rank_of, g->orig, g->in_off, g->in_src,
                                       C.in_cost, g->out_off, g->out_dst, C.out_cost, off, enode, ew);
        count_launch();
        PDNN_LAUNCH_CHECK();
    }
    // the sequential decisions
    int32_t max_iter = 0;
    while ((1ll << max_iter) < (int64_t)V) ++max_iter;    // ceil(log2 |V|)
    if (max_iter < 1) max_iter = 1;
    LfArgs a{};
    a.V = V; a.K = K; a.D = D; a.ns = ns; a.max_iter = max_iter;
    a.order = i1; a.info = info; a.off = off; a.enode = enode; a.ew = ew; a.cl_off = cl_off; a.members = members;
    a.mc = mc; a.ml = ml; a.sums = sums; a.part8 = part8; a.tree = tree; a.list = list; a.log = log; a.n_log = n_log;
    const size_t tree_b = ((size_t)8 * T * (D + 1) + 15) & ~size_t(15);
    size_t smem = 8 * PDNN_MAX_PE;
    const bool smem_ok = debug_knob("PDNN_LFLAM_GLOBAL", 0) == 0;   // test knob: state in global memory
    if (smem_ok && smem + tree_b <= kLfSmemMax) { a.smem_tree = 1; smem += tree_b; }
    if (smem_ok && a.smem_tree && smem + (size_t)V <= kLfSmemMax) { a.smem_part = 1; smem += (size_t)V; }
    if (smem > 48 * 1024) PDNN_CUDA_TRY(cudaFuncSetAttribute(k_lflam, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                             (int)smem));
    k_lflam<<<1, 32, smem, s>>>(a);
    count_launch();
    PDNN_LAUNCH_CHECK();
    k_lf_out<<<lf_grid(V), 256, 0, s>>>(V, part8, part);
    count_launch();
    PDNN_LAUNCH_CHECK();
    return PDNN_OK;
}
