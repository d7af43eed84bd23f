// graph.cu -- pdnn_build_csr and graph/cost/workspace management (§8(a) rows
// a1, a2): validation, canonical (src,dst) order, Kahn levels on the device
// (frontier kernel with atomic in-degree countdown and warp-aggregated
// appends), level order rank = stable (level, id), rank-space CSRs, and the
// dataflow sweep schedule.
#include <cooperative_groups.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include <cstdlib>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace pdnn {

static thread_local std::string t_last_error;
std::atomic<uint64_t> g_launches{0};
void set_error(const std::string& msg) { t_last_error = msg; }

int sweep_blocks_per_sm(int device, int32_t V, int32_t D);  // sweep.cu

// ------------------------------------------------------------------ kernels
__global__ void k_validate(int64_t E, int32_t V, const int32_t* __restrict__ src,
                           const int32_t* __restrict__ dst, uint64_t* __restrict__ key,
                           int32_t* __restrict__ idx, int32_t* __restrict__ flags) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E;
         k += (int64_t)gridDim.x * blockDim.x) {
        int32_t s = src[k], d = dst[k];
        bool bad = s < 0 || s >= V || d < 0 || d >= V;
        if (bad) atomicOr(&flags[0], 1);
        else if (s == d) atomicOr(&flags[0], 2);
        key[k] = bad ? 0ull : (uint64_t)s * (uint64_t)V + (uint64_t)d;
        idx[k] = (int32_t)k;
    }
}

// canonical arrays + duplicate check + degree histograms
__global__ void k_canon(int64_t E, int32_t V, const uint64_t* __restrict__ key,
                        int32_t* __restrict__ csrc, int32_t* __restrict__ cdst,
                        int32_t* __restrict__ outdeg, int32_t* __restrict__ indeg,
                        int32_t* __restrict__ flags) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E;
         k += (int64_t)gridDim.x * blockDim.x) {
        uint64_t x = key[k];
        if (k > 0 && key[k - 1] == x) atomicOr(&flags[0], 4);
        int32_t s = (int32_t)(x / (uint64_t)V), d = (int32_t)(x % (uint64_t)V);
        csrc[k] = s;
        cdst[k] = d;
        atomicAdd(&outdeg[s], 1);
        atomicAdd(&indeg[d], 1);
    }
}

__global__ void k_offsets_from_canon(int64_t E, const int32_t* __restrict__ csrc,
                                     int32_t* __restrict__ off, int32_t V) {
    // off[v] = first canonical edge with src >= v (canonical order is sorted by src)
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= E;
         k += (int64_t)gridDim.x * blockDim.x) {
        int32_t lo = k == 0 ? 0 : csrc[k - 1] + 1;
        int32_t hi = k == E ? V : csrc[k];
        if (lo < 0 || hi > V) {   // canonical sources are in [0, V): never for a validated input
            printf("k_offsets_from_canon: edge %lld source range [%d, %d] outside [0, %d]\n", (long long)k, lo, hi, V);
            __trap();
        }
        for (int32_t v = lo; v <= hi; ++v) off[v] = (int32_t)k;
    }
}

__device__ __forceinline__ void kahn_append(int32_t s, int32_t* queue, int32_t base, int32_t* cnt) {
    cg::coalesced_group g = cg::coalesced_threads();   // warp-aggregated append
    int32_t off = 0;
    if (g.thread_rank() == 0) off = atomicAdd(cnt, (int32_t)g.size());
    off = g.shfl(off, 0);
    queue[base + off + g.thread_rank()] = s;
}

__device__ __forceinline__ void kahn_relax(int32_t s, int32_t lvl, int32_t* indeg, int32_t* level,
                                           int32_t* queue, int32_t base, int32_t* cnt) {
    if (atomicSub(&indeg[s], 1) == 1) {
        level[s] = lvl + 1;
        kahn_append(s, queue, base, cnt);
    }
}

// Kahn's algorithm, level-synchronous: level l is the frontier of nodes whose
// in-degree dropped to 0 while processing level l-1.
// Frontier sizes go through three rotating counters so that no thread can
// append to the counter another thread is still reading after a barrier:
// level l appends to cnt[(l+1)%3], reads cnt[l%3] at its start, and clears
// cnt[(l+2)%3] (last read before the previous barrier).
// Narrow levels (<= kKahnSolo nodes) are processed by CTA 0 alone, with a
// block barrier per level instead of a grid barrier; the other CTAs wait on a
// flag and rejoin at the next wide level (DNN graphs have thousands of narrow
// levels: C3 4,111 levels x ~7 us of grid barrier before).
constexpr int kKahnSolo = 1024;
constexpr int32_t kKahnOneCtaV = 32768;   // graphs below this many nodes run Kahn on one CTA
__device__ void kahn_level(int32_t lo, int32_t hi, int32_t lvl, int first_warp, int n_warps, int lane,
                           const int32_t* __restrict__ off, const int32_t* __restrict__ dst, int32_t* indeg,
                           int32_t* queue, int32_t* level, int32_t* app) {
    for (int32_t base = lo + first_warp * 32; base < hi; base += n_warps * 32) {
        int32_t idx = base + lane;
        int32_t u = idx < hi ? queue[idx] : -1;
        int32_t s = u >= 0 ? off[u] : 0, t = u >= 0 ? off[u + 1] : 0;
        bool heavy = (t - s) > 32;
        if (!heavy)
            for (int32_t e = s; e < t; ++e) kahn_relax(dst[e], lvl, indeg, level, queue, hi, app);
        unsigned hm = __ballot_sync(0xffffffffu, heavy);
        while (hm) {
            int j = __ffs(hm) - 1;
            hm &= hm - 1;
            int32_t hs = __shfl_sync(0xffffffffu, s, j), ht = __shfl_sync(0xffffffffu, t, j);
            for (int32_t e = hs + lane; e < ht; e += 32)
                kahn_relax(dst[e], lvl, indeg, level, queue, hi, app);
        }
    }
}

__global__ void __launch_bounds__(256) k_kahn(int32_t V, const int32_t* __restrict__ off,
                                              const int32_t* __restrict__ dst,
                                              int32_t* __restrict__ indeg, int32_t* queue,
                                              int32_t* __restrict__ level,
                                              int32_t* __restrict__ level_ptr, int32_t* ctrl) {
    cg::grid_group grid = cg::this_grid();
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nth = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31, warp = tid >> 5, nw = nth >> 5;
    int32_t* cnt = ctrl + 4;   // cnt[0..2], zero on entry
    int32_t* solo = ctrl + 8;  // [0] solo rounds completed, [1] lo, [2] hi, [3] lvl (zero on entry)
    __shared__ int32_t s_lo, s_hi, s_lvl;
    __shared__ int32_t s_eoff[kKahnSolo], s_pre[kKahnSolo + 1], s_q[2][kKahnSolo];
    __shared__ int32_t s_cnt, s_inq;
    for (int v = tid; v < V; v += nth)
        if (indeg[v] == 0) {
            level[v] = 0;
            kahn_append(v, queue, 0, &cnt[0]);
        }
    grid.sync();
    int32_t lo = 0, hi = *(volatile int32_t*)&cnt[0], lvl = 0, rounds = 0;
    while (lo < hi) {
        if (hi - lo <= kKahnSolo) {
            // ---- narrow levels: CTA 0 alone, a block barrier per level
            if (blockIdx.x == 0) {
                if (threadIdx.x == 0) { s_lo = lo; s_hi = hi; s_lvl = lvl; s_inq = 0; }
                __syncthreads();
                for (;;) {
                    const int32_t l0 = s_lo, h0 = s_hi, lv = s_lvl;
                    const bool from_smem = s_inq;   // this level's nodes are also in s_q[cur]
                    if (l0 >= h0 || h0 - l0 > kKahnSolo) break;
                    const int cur = lv & 1;
                    __syncthreads();
                    if (threadIdx.x == 0) { level_ptr[lv] = l0; s_cnt = 0; }
                    // the level's out-edges flattened over the CTA: one relaxation
                    // (one atomic round trip) per thread instead of a loop per node;
                    // the frontier and its counter live in shared memory
                    const int n = h0 - l0;
                    for (int k = threadIdx.x; k < n; k += blockDim.x) {
                        const int32_t u = from_smem ? s_q[cur][k] : queue[l0 + k];
                        const int32_t a0 = off[u];
                        s_eoff[k] = a0;
                        s_pre[k] = off[u + 1] - a0;
                    }
                    __syncthreads();
                    if (threadIdx.x < 32) {   // exclusive scan of the <= kKahnSolo degrees by one warp
                        int32_t run = 0;
                        for (int k0 = 0; k0 < n; k0 += 32) {
                            const int32_t x = k0 + lane < n ? s_pre[k0 + lane] : 0;
                            int32_t incl = x;
#pragma unroll
                            for (int o = 1; o < 32; o <<= 1) {
                                const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                                if (lane >= o) incl += y;
                            }
                            if (k0 + lane < n) s_pre[k0 + lane] = run + incl - x;
                            run += __shfl_sync(0xffffffffu, incl, 31);
                        }
                        if (lane == 0) s_pre[n] = run;
                    }
                    __syncthreads();
                    const int32_t T = s_pre[n];
                    for (int32_t j = threadIdx.x; j < T; j += blockDim.x) {
                        int lo2 = 0, hi2 = n - 1;   // node k with s_pre[k] <= j < s_pre[k + 1]
                        while (lo2 < hi2) {
                            const int mid = (lo2 + hi2 + 1) >> 1;
                            if (s_pre[mid] <= j) lo2 = mid; else hi2 = mid - 1;
                        }
                        const int32_t sv = dst[s_eoff[lo2] + (j - s_pre[lo2])];
                        if (atomicSub(&indeg[sv], 1) == 1) {
                            level[sv] = lv + 1;
                            const int32_t q = atomicAdd(&s_cnt, 1);
                            queue[h0 + q] = sv;
                            if (q < kKahnSolo) s_q[cur ^ 1][q] = sv;
                        }
                    }
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        s_lo = h0;
                        s_hi = h0 + s_cnt;
                        s_lvl = lv + 1;
                        s_inq = 1;
                    }
                    __syncthreads();
                }
                if (threadIdx.x == 0) {
                    solo[1] = s_lo;
                    solo[2] = s_hi;
                    solo[3] = s_lvl;
                    cnt[0] = cnt[1] = cnt[2] = 0;   // grid mode appends from zero
                    __threadfence();
                    atomicAdd(&solo[0], 1);   // release the other CTAs
                }
            } else if (threadIdx.x == 0) {
                long long spins = 0;
                while (*(volatile int32_t*)&solo[0] <= rounds) {
                    __nanosleep(200);
                    if (++spins == (1ll << 25)) {   // ~10 s: report and fail loudly instead of hanging
                        printf("k_kahn: CTA %d waits for narrow round %d (solo %d %d %d %d, V %d)\n", blockIdx.x,
                               rounds, solo[0], solo[1], solo[2], solo[3], V);
                        __trap();
                    }
                }
            }
            __syncthreads();
            __threadfence();
            ++rounds;
            lo = *(volatile int32_t*)&solo[1];
            hi = *(volatile int32_t*)&solo[2];
            lvl = *(volatile int32_t*)&solo[3];
            grid.sync();   // every CTA has read the hand-back before the counters move on
            continue;
        }
        if (tid == 0) {
            level_ptr[lvl] = lo;
            cnt[(lvl + 2) % 3] = 0;
        }
        int32_t* app = &cnt[(lvl + 1) % 3];
        kahn_level(lo, hi, lvl, warp, nw, lane, off, dst, indeg, queue, level, app);
        grid.sync();
        lo = hi;
        hi = lo + *(volatile int32_t*)app;
        ++lvl;
    }
    if (tid == 0) {
        level_ptr[lvl] = hi;
        ctrl[0] = hi;
        ctrl[1] = lvl;
    }
}

__global__ void k_iota(int32_t n, int32_t* __restrict__ a) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

__global__ void k_rank_of(int32_t V, const int32_t* __restrict__ orig, int32_t* __restrict__ rank_of,
                          const int32_t* __restrict__ indeg0, const int32_t* __restrict__ outdeg,
                          int32_t* __restrict__ indeg_r, int32_t* __restrict__ outdeg_r) {
    for (int32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < V; r += gridDim.x * blockDim.x) {
        int32_t v = orig[r];
        rank_of[v] = r;
        indeg_r[r] = indeg0[v];
        outdeg_r[r] = outdeg[v];
    }
}

__global__ void k_rank_keys(int64_t E, int32_t V, const int32_t* __restrict__ csrc,
                            const int32_t* __restrict__ cdst, const int32_t* __restrict__ rank_of,
                            uint64_t* __restrict__ kin, uint64_t* __restrict__ kout,
                            int32_t* __restrict__ idx) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E;
         k += (int64_t)gridDim.x * blockDim.x) {
        uint64_t ru = (uint64_t)rank_of[csrc[k]], rv = (uint64_t)rank_of[cdst[k]];
        kin[k] = rv * (uint64_t)V + ru;   // in-CSR: grouped by head, sorted by tail rank
        kout[k] = ru * (uint64_t)V + rv;  // out-CSR: grouped by tail, sorted by head rank
        idx[k] = (int32_t)k;
    }
}

__global__ void k_split_key(int64_t E, int32_t V, const uint64_t* __restrict__ key,
                            int32_t* __restrict__ other) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E;
         k += (int64_t)gridDim.x * blockDim.x)
        other[k] = (int32_t)(key[k] % (uint64_t)V);
}

// costs -> rank space / CSR order; optional exact validation (R7): every
// cost in [0, 2^62) and sum(comp) + sum(comm) < 2^62.  check[0] = running
// total, check[1] = violation flag.
__device__ __forceinline__ void cost_check(int64_t x, unsigned long long& sum, unsigned long long& bad) {
    const unsigned long long lim = 1ull << 62;
    if (x < 0 || (unsigned long long)x >= lim) { bad = 1; return; }
    sum += (unsigned long long)x;          // < 2^63: cannot wrap
    if (sum >= lim) { bad = 1; sum = lim; }
}

__global__ void k_perm_costs(int32_t V, int64_t E, const int32_t* __restrict__ orig,
                             const int32_t* __restrict__ in_eid, const int32_t* __restrict__ out_eid,
                             const int32_t* __restrict__ perm, const int64_t* __restrict__ nc,
                             const int64_t* __restrict__ ec, int64_t* __restrict__ c_rank,
                             int64_t* __restrict__ in_cost, int64_t* __restrict__ out_cost,
                             unsigned long long* __restrict__ check) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    unsigned long long sum = 0, bad = 0;
    for (int64_t r = tid; r < V; r += nth) {
        int64_t x = nc[orig[r]];
        c_rank[r] = x;
        if (check) cost_check(x, sum, bad);
    }
    for (int64_t e = tid; e < E; e += nth) {
        int32_t a = in_eid[e], b = out_eid[e];
        if (perm) { a = perm[a]; b = perm[b]; }
        in_cost[e] = ec[a];
        int64_t x = ec[b];
        out_cost[e] = x;
        if (check) cost_check(x, sum, bad);   // each edge counted once (out-CSR)
    }
    if (check) {
        if (sum) {
            unsigned long long old = atomicAdd(&check[0], sum);
            if (old >= (1ull << 62) || old + sum >= (1ull << 62)) bad = 1;
        }
        if (bad) atomicOr(&check[1], 1ull);
    }
}

// labels (node-id order, int32 or uint8, or a constant) -> rank space
// (part_rank, the sweep's label array); optional node-id-order int32 copy
__global__ void k_labels(int32_t V, const int32_t* __restrict__ orig, const int32_t* __restrict__ p32,
                         const uint8_t* __restrict__ p8, int32_t fill, int32_t* __restrict__ porig,
                         int32_t* __restrict__ prank) {
    // 4 ranks per thread per round, every gather issued before the first store
    constexpr int U = 4;
    const int32_t nth = gridDim.x * blockDim.x;
    for (int32_t r0 = blockIdx.x * blockDim.x + threadIdx.x; r0 < V; r0 += U * nth) {
        int32_t n[U], lab[U];
#pragma unroll
        for (int u = 0; u < U; ++u) n[u] = r0 + u * nth < V ? __ldg(&orig[r0 + u * nth]) : -1;
#pragma unroll
        for (int u = 0; u < U; ++u)
            lab[u] = n[u] < 0 ? 0 : (p32 ? __ldg(&p32[n[u]]) : (p8 ? (int32_t)__ldg(&p8[n[u]]) : fill));
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (n[u] < 0) continue;
            prank[r0 + u * nth] = lab[u];
            if (porig) porig[n[u]] = lab[u];
        }
    }
}

// Pack the sweep's thread items into their blobs (sweep.cu): per item, one
// 16-byte record per LANE {comp, original id, meta}, then the item's neighbour
// ranks (int32, padded to an even count) and edge costs (int64).  Lane layout:
// node j owns ceil(deg_j / 4) adjacent lanes (chunks of <= 4 edges), starting
// at f_j = sum of the lanes of the nodes before it.  meta = e0 | n_edges << 8
// | j << 11 | chunk << 16 | following lanes of the node << 19.  One warp per item.
__global__ void k_blob(int32_t n_items, const Item* __restrict__ items, const int32_t* __restrict__ in_off,
                       const int32_t* __restrict__ in_src, const int32_t* __restrict__ out_off,
                       const int32_t* __restrict__ out_dst, const int64_t* __restrict__ c,
                       const int64_t* __restrict__ in_cost, const int64_t* __restrict__ out_cost,
                       const int32_t* __restrict__ orig, const int32_t* __restrict__ inodes,
                       unsigned char* __restrict__ blob_in, unsigned char* __restrict__ blob_out) {
    __shared__ uint16_t s_own[8][32];
    const int lane = threadIdx.x & 31, wic = threadIdx.x >> 5;
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    for (int32_t i = blockIdx.x * (blockDim.x >> 5) + wic; i < n_items; i += nwarps) {
        const Item it = items[i];
        if (it.y <= 0) continue;
        const bool fwd = it.x >= 0;
        const int32_t r0 = fwd ? it.x : ~it.x;
        const int32_t* off = fwd ? in_off : out_off;
        const int32_t* src = fwd ? in_src : out_dst;
        const int64_t* cost = fwd ? in_cost : out_cost;
        unsigned char* b = (fwd ? blob_in : blob_out) + (size_t)it.z * 16;
        const int n = it.y, nl = it.w & 0xff, m = (it.w >> 8) & 0xff;
        const bool ix = (it.w & kItemIndexed) != 0;
        // the lane's node (rank): a run of ranks, or listed in inodes (indexed item)
        const int32_t rk = lane < n ? (ix ? inodes[r0 + lane] : r0 + lane) : 0;
        const int32_t base = off[r0];   // (run items: the item's edges are one CSR range)
        const int32_t d = lane < n ? off[rk + 1] - off[rk] : 0;
        const int ln = lane < n ? max(1, (d + 3) >> 2) : 0;
        int ex = d;   // inclusive scan of the degrees: node j's edges start at ex_j - d_j in the item
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, ex, o);
            if (lane >= o) ex += y;
        }
        ex -= d;
        int f = ln;   // inclusive scan of the lanes per node
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, f, o);
            if (lane >= o) f += y;
        }
        f -= ln;
        for (int k = 0; k < ln; ++k) s_own[wic][f + k] = (uint16_t)(lane | k << 5 | (ln - 1 - k) << 8);
        __syncwarp();
        const int o = lane < nl ? s_own[wic][lane] : 0;
        const int j = o & 31, chunk = (o >> 5) & 7, rem = (o >> 8) & 7;
        const int32_t dj = __shfl_sync(0xffffffffu, d, j);
        const int32_t ej = __shfl_sync(0xffffffffu, ex, j);
        const int32_t rj = __shfl_sync(0xffffffffu, rk, j);
        if (lane < nl) {
            const int32_t e0 = ej + 4 * chunk;
            const int32_t ne = min(dj - 4 * chunk, 4);
            int4 rec;
            const int64_t cj = c[rj];
            rec.x = (int32_t)(uint32_t)((uint64_t)cj & 0xffffffffu);
            rec.y = (int32_t)(uint32_t)((uint64_t)cj >> 32);
            rec.z = ix ? rj : orig[rj];   // indexed items carry the rank (the sweep gathers orig)
            rec.w = (int32_t)((uint32_t)e0 | (uint32_t)ne << 8 | (uint32_t)j << 11 | (uint32_t)chunk << 16 |
                              (uint32_t)rem << 19);
            reinterpret_cast<int4*>(b)[lane] = rec;
        }
        int32_t* bn = reinterpret_cast<int32_t*>(b + 16 * nl);
        int64_t* bc = reinterpret_cast<int64_t*>(b + 16 * nl + 4 * ((m + 1) & ~1));
        if (!ix) {
            for (int e = lane; e < ((m + 1) & ~1); e += 32) bn[e] = e < m ? src[base + e] : 0;
            for (int e = lane; e < m; e += 32) bc[e] = cost[base + e];
        } else {
            for (int jj = 0; jj < n; ++jj) {
                const int32_t r = __shfl_sync(0xffffffffu, rk, jj), dd = __shfl_sync(0xffffffffu, d, jj);
                const int32_t e0 = __shfl_sync(0xffffffffu, ex, jj), b0 = off[r];
                for (int e = lane; e < dd; e += 32) {
                    bn[e0 + e] = src[b0 + e];
                    bc[e0 + e] = cost[b0 + e];
                }
            }
            if ((m & 1) && lane == 0) bn[m] = 0;
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ host helpers
namespace {
// Graph memory is stream-ordered (cudaMallocAsync) from the device's default
// pool, whose release threshold is raised once per device so freed blocks stay
// mapped: a later build reuses them instead of mapping fresh pages (round 2:
// the C3 build spent 80-100 ms of ~170 in its ~20 cudaMalloc calls).
cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t s) {
    static std::mutex mu;
    static uint64_t done = 0;   // one bit per device (< 64)
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lock(mu);
        if (dev < 64 && !((done >> dev) & 1)) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            done |= 1ull << dev;
        }
    }
    return cudaMallocAsync(p, std::max<size_t>(bytes, 1), s);
}

struct DevBufs {
    cudaStream_t s = nullptr;
    std::vector<void*> ptrs;
    ~DevBufs() { for (void* p : ptrs) cudaFreeAsync(p, s); }   // stream-ordered after the build's kernels
    template <typename T>
    cudaError_t alloc(T** p, size_t n) {
        void* q = nullptr;
        cudaError_t e = pool_alloc(&q, (std::max<size_t>(n, 1) + 16) * sizeof(T), s);  // +16: TMA slices are widened to 16 B
        if (e == cudaSuccess) { ptrs.push_back(q); *p = static_cast<T*>(q); }
        return e;
    }
    void release(void* p) {  // keep the allocation (ownership moves to the graph)
        ptrs.erase(std::remove(ptrs.begin(), ptrs.end(), p), ptrs.end());
    }
};

int grid_for(int64_t n, int threads = 256, int cap = 148 * 16) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (int)b;
}

void free_graph(pdnn_graph* g) {
    if (!g) return;
    void* ps[] = {g->rank_of, g->orig, g->level, g->perm, g->level_ptr, g->in_off, g->in_src,
                  g->in_eid, g->out_off, g->out_dst, g->out_eid, g->c_rank, g->in_cost,
                  g->out_cost, g->items, g->items_rm, g->inodes, g->hub_nparts, g->heavy_out, g->bitems[0], g->bitems[1], g->bhub_pbase,
                  g->blob[0], g->blob[1]};
    // the graph's memory comes from the stream-ordered pool, where cudaFree does
    // NOT wait for kernels still reading it (unlike a cudaMalloc block): without
    // this barrier a graph dropped right after an asynchronous call went back
    // to the pool while its kernels ran, and the next build reused it
    cudaDeviceSynchronize();
    for (void* p : ps) if (p) cudaFree(p);
    delete g;
}

// Build the dataflow schedule: tl items (levels ascending, in-CSR) and bl
// items (levels descending, out-CSR), interleaved so that every item depends
// only on items with smaller merged index (see sweep.cu).
void build_items(const std::vector<int32_t>& level_ptr, const std::vector<int32_t>& in_off,
                 const std::vector<int32_t>& out_off, std::vector<Item>& items,
                 std::vector<int32_t>& hub_nparts, int max_deg = kTMaxDeg, int max_edges = kTMaxEdges,
                 int max_nodes = 32, int hub_edges = kHEdges, bool split4 = false, bool skip_entry_tl = false,
                 int merge = 1, const std::vector<int32_t>* bl_ready = nullptr,
                 std::vector<int32_t>* inodes = nullptr) {
    const int D = (int)level_ptr.size() - 1;
    std::vector<int32_t> fwave, bwave;   // per item: the hop at which its inputs complete
    auto make = [&](const std::vector<int32_t>& off, bool fwd, std::vector<Item>& out) {
        std::vector<int32_t>& wave = fwd ? fwave : bwave;
        // (skip_entry_tl: level 0 has no predecessors, tl = 0 there; the sweep's
        // prologue publishes those nodes without items)
        for (int li = fwd && skip_entry_tl ? 1 : 0; li < D; ++li) {
            int l = fwd ? li : D - 1 - li;
            int32_t r = level_ptr[l], end = level_ptr[l + 1];
            if (!fwd && l == 0 && bl_ready && inodes && D > 1) {
                // level 0's bl (parameters, constants, entry ops): its nodes'
                // inputs complete at different hops (a parameter feeding level
                // 40 is ready after bl level 40), but a run of consecutive ranks
                // is ready only with its latest node.  Indexed items group the
                // nodes by that hop instead (ranks listed in inodes, blob packed
                // per node); wave = D - m, m = the lowest successor level (D for
                // an exit): every dependency sits at a smaller wave.
                std::vector<std::pair<int32_t, int32_t>> ord;
                ord.reserve(end - r);
                for (int32_t x = r; x < end; ++x) ord.push_back({D - (*bl_ready)[x], x});
                std::stable_sort(ord.begin(), ord.end());
                size_t k = 0;
                while (k < ord.size()) {
                    const int32_t x = ord[k].second;
                    const int32_t deg = off[x + 1] - off[x];
                    if (deg > max_deg) {   // a hub: warp items over its CSR range, as elsewhere
                        int parts = (deg + hub_edges - 1) / hub_edges;
                        int slot = -1;
                        if (parts > 1) { slot = (int)hub_nparts.size(); hub_nparts.push_back(parts); }
                        for (int p = 0; p < parts; ++p) {
                            Item it;
                            it.x = ~x;
                            it.y = parts > 1 ? -1 - slot : 0;
                            it.z = off[x] + p * hub_edges;
                            it.w = std::min<int32_t>(off[x + 1], it.z + hub_edges);
                            out.push_back(it);
                            wave.push_back(ord[k].first);
                        }
                        ++k;
                        continue;
                    }
                    const int32_t base = (int32_t)inodes->size();
                    int32_t n = 0, tot = 0, lanes = 0, wv = 0;
                    while (k + n < ord.size() && n < max_nodes) {
                        const int32_t y = ord[k + n].second;
                        const int32_t d = off[y + 1] - off[y];
                        const int32_t ln = split4 ? std::max(1, (d + 3) / 4) : 1;
                        if (d > max_deg || (n > 0 && (tot + d > max_edges || lanes + ln > 32))) break;
                        inodes->push_back(y);
                        wv = std::max(wv, ord[k + n].first);
                        tot += d;
                        lanes += ln;
                        ++n;
                    }
                    Item it;
                    it.x = ~base;
                    it.y = n;
                    it.z = 0;          // blob offset / lanes are set by the caller
                    it.w = tot | kItemIndexed;
                    out.push_back(it);
                    wave.push_back(wv);
                    k += n;
                }
                continue;
            }
            while (r < end) {
                int32_t deg = off[r + 1] - off[r];
                if (deg > max_deg) {
                    int parts = (deg + hub_edges - 1) / hub_edges;
                    int slot = -1;
                    if (parts > 1) { slot = (int)hub_nparts.size(); hub_nparts.push_back(parts); }
                    for (int p = 0; p < parts; ++p) {
                        Item it;
                        it.x = fwd ? r : ~r;
                        it.y = parts > 1 ? -1 - slot : 0;
                        it.z = off[r] + p * hub_edges;
                        it.w = std::min<int32_t>(off[r + 1], it.z + hub_edges);
                        out.push_back(it);
                        wave.push_back(li);
                    }
                    ++r;
                    continue;
                }
                int32_t n = 0, tot = 0, lanes = 0;
                while (r + n < end && n < max_nodes) {
                    int32_t d = off[r + n + 1] - off[r + n];
                    const int32_t ln = split4 ? std::max(1, (d + 3) / 4) : 1;   // lanes of the node (sweep.cu)
                    if (d > max_deg || (n > 0 && (tot + d > max_edges || lanes + ln > 32))) break;
                    tot += d;
                    lanes += ln;
                    ++n;
                }
                Item it;
                it.x = fwd ? r : ~r;
                it.y = n;
                it.z = off[r];
                it.w = off[r + n];
                out.push_back(it);
                wave.push_back(li);
                r += n;
            }
        }
    };
    std::vector<Item> f, b;
    make(in_off, true, f);
    make(out_off, false, b);
    if (inodes && bl_ready) {   // the indexed level-0 items to their waves (stable: the rest keeps its order)
        std::vector<int32_t> ordb(b.size());
        for (size_t k = 0; k < b.size(); ++k) ordb[k] = (int32_t)k;
        std::stable_sort(ordb.begin(), ordb.end(), [&](int32_t p, int32_t q) { return bwave[p] < bwave[q]; });
        std::vector<Item> b2(b.size());
        std::vector<int32_t> w2(b.size());
        for (size_t k = 0; k < b.size(); ++k) {
            b2[k] = b[ordb[k]];
            w2[k] = bwave[ordb[k]];
        }
        b.swap(b2);
        bwave.swap(w2);
    }
    items.clear();
    items.reserve(f.size() + b.size());
    size_t i = 0, j = 0;
    const size_t nf = f.size(), nb = b.size();
    if (merge == 0) {
        // proportional interleave keeps each list's internal order
        while (i < nf || j < nb) {
            if (j >= nb || (i < nf && i * nb <= j * nf)) items.push_back(f[i++]);
            else items.push_back(b[j++]);
        }
        return;
    }
    // by wave: tl level l and bl level D-1-l complete at the same hop of their
    // chains, so their items are dealt together (a proportional interleave
    // deals the longer list ahead of its time: C4's bl list carries level 0's
    // 10k parameter items, so bl items of later hops sat in front of tl items
    // on the same warps and delayed the tl chain); within a wave,
    // proportionally to the two lists' sizes in that wave (merge 1), or the
    // wave's tl items first (merge 2: C4's last wave pairs tl level 63 with
    // the 10k items of bl level 0)
    while (i < nf || j < nb) {
        const int32_t w = std::min(i < nf ? fwave[i] : INT32_MAX, j < nb ? bwave[j] : INT32_MAX);
        size_t i1 = i, j1 = j;
        while (i1 < nf && fwave[i1] == w) ++i1;
        while (j1 < nb && bwave[j1] == w) ++j1;
        const size_t a = i1 - i, bb = j1 - j;
        size_t x = 0, y = 0;
        while (x < a || y < bb) {
            if (y >= bb || (x < a && (merge == 2 || x * bb <= y * a))) items.push_back(f[i + x++]);
            else items.push_back(b[j + y++]);
        }
        i = i1;
        j = j1;
    }
}
}  // namespace

// ------------------------------------------------------------------ per-device launch properties
int kernel_occupancy(const void* fn, int threads, int dyn_smem) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, int, int>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_tuple(fn, dev, threads, dyn_smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    if (dyn_smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, dyn_smem) != cudaSuccess) cudaGetLastError();
    n = n < 1 ? 1 : n;
    cache[key] = n;
    return n;
}

// ------------------------------------------------------------------ workspace guard
uint64_t layout_sig(const pdnn_graph* g, uint64_t salt, size_t end) {
    const uint64_t w[] = {(uint64_t)g->V, (uint64_t)g->E, (uint64_t)g->n_levels, (uint64_t)g->n_hubs,
                          (uint64_t)g->n_bparts, (uint64_t)g->n_bhubs, (uint64_t)g->num_sms,
                          (uint64_t)g->n_items, (uint64_t)g->n_entry, (uint64_t)end, salt};
    uint64_t h = 0xcbf29ce484222325ull;   // FNV-1a over the words
    for (uint64_t x : w)
        for (int b = 0; b < 8; ++b) { h ^= (x >> (8 * b)) & 0xff; h *= 0x100000001b3ull; }
    return h | 1;   // never 0 (0 = unknown)
}

pdnn_status ws_guard(void* ws, int region, size_t begin, size_t end, uint64_t sig, cudaStream_t s) {
    static std::mutex mu;
    static std::map<std::pair<void*, int>, uint64_t> last;
    bool clear = false;
    {
        std::lock_guard<std::mutex> lock(mu);
        uint64_t& v = last[std::make_pair(ws, region)];
        if (v != sig) { clear = true; v = sig; }
    }
    if (clear && end > begin) PDNN_CUDA_TRY(cudaMemsetAsync(static_cast<char*>(ws) + begin, 0, end - begin, s));
    return PDNN_OK;
}

// ------------------------------------------------------------------ ws layout
WsLayout ws_layout(const pdnn_graph* g, int op, int32_t batch) {
    WsLayout L{};
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
    const size_t V = (size_t)std::max(g->V, 1), E = (size_t)std::max<int64_t>(g->E, 1);
    L.hdr = take(sizeof(WsHeader));
    L.rec = take(16 * V);   // tagged tl+comp [V], then tagged bl [V] (sweep.cu)
    L.hub_acc = take(8 * (size_t)std::max(g->n_hubs, 1));
    L.hub_cnt = take(4 * (size_t)std::max(g->n_hubs, 1));
    L.c_s = take(8 * V);
    L.in_cost_s = take(8 * E);
    L.out_cost_s = take(8 * E);
    L.part_rank = take(4 * V);
    L.blob_s_in = take(g->blob_bytes[0] + 16);    // the sweep's blobs for per-call costs
    L.blob_s_out = take(g->blob_bytes[1] + 16);
    L.tl_o = take(8 * V);
    L.bl_o = take(8 * V);
    L.part_o = take(4 * V);
    L.cp_nodes = take(4 * (size_t)(g->n_levels + 1));
    L.mpot_s = take(8 * V);
    L.emu = take(emulate_ws_bytes(g, 1));
    L.sc_ctl = take(64);
    L.sc_keys = take(16 * V);
    L.sc_ids = take(8 * V);
    L.sc_fwd = take(4 * V);
    L.sc_temp_bytes = slice_sort_temp_bytes(g->V);
    L.sc_temp = take(L.sc_temp_bytes);
    L.cp_grid = 2 * g->num_sms;                // upper bound of the cooperative CP grid (cp.cu)
    L.cp_M = take(8 * (size_t)L.cp_grid);
    L.cp_ctl = take(64);
    L.cp_list = take(4 * V);
    L.cp_pos = take(4 * V);
    L.cp_A = take(8 * V);
    L.cp_d = take(8 * V);
    L.cp_mark = take(V);
    // memory tracker regions for S placements side by side
    auto take_mem = [&](int32_t nseg) {
        L.m_seg = nseg;
        const size_t S = (size_t)nseg;
        L.m_keys = take(8 * V * S);
        L.m_keys_alt = take(8 * V * S);
        L.m_vals = take(4 * V * S);
        L.m_vals_alt = take(4 * V * S);
        L.m_order = take(4 * V * S);
        L.m_pp = take(4 * V * S);
        L.m_relp = take(8 * V * S);
        L.m_rec = take(16 * V * S);
        L.m_pe8 = take(V * S);
        L.m_hist = take(4 * 1024 * 8 * S);                                       // [S][passes][1024] digit bases
        L.m_dtot = take(4 * 32);                                                 // tickets + launch epoch
        L.m_status = take(8 * 1024 * S * ((size_t)ceil_div(g->V, 2048) + 1));  // [S * tiles][1024] look-back
        L.m_tiles = ceil_div(g->V, kMemTile) + 1;
        L.m_tile = take(8 * (size_t)L.m_tiles * PDNN_MAX_PE * S);
        L.m_tile_res = take(sizeof(TileRes) * (size_t)L.m_tiles * PDNN_MAX_PE * S);
        L.m_base = take(8 * (PDNN_MAX_PE * S + 1));
        L.m_ctr = take(4 * (S + 1));
    };
    // the single-placement region: its offsets depend on the graph only, never
    // on the op or the batch, so every single-placement call finds its
    // persistent state (epoch tags, self-resetting counters) where it left it
    take_mem(1);
    L.single_end = off;
    L.sig_single = layout_sig(g, 0, L.single_end);
    int32_t ng_batch = 0;
    const bool refine = op == PDNN_OP_REFINE;
    if (refine) batch = kRefineGroup;   // trial groups of the node-level passes (the batched sweep only)
    const bool batched = (op == PDNN_OP_EVAL_BATCH || op == PDNN_OP_EVAL_BATCH_EMULATED || refine) && batch > 0;
    const bool emulated = op == PDNN_OP_EVAL_BATCH_EMULATED;
    if (batched) {
        const size_t nparts = (size_t)std::max(g->n_bparts, 1);
        const size_t per_cand = V * (1 + 1 + 8 + 8 + 4 + 8 + (emulated ? 24 : 0)) + nparts * 12 + 8;
        int64_t cap = std::max<int64_t>(32, (int64_t)((refine ? kRefineWsBudget : kBatchWsBudget) / per_cand) / 32 * 32);
#ifdef PDNN_DEBUG_KNOBS
        // test / diagnostic knob: cap the candidates per group (exercises the multi-group path)
        static const int64_t group_env = getenv("PDNN_BATCH_GROUP") ? atoll(getenv("PDNN_BATCH_GROUP")) : 0;
        if (group_env > 0) cap = std::min<int64_t>(cap, std::max<int64_t>(32, group_env / 32 * 32));
#endif
        ng_batch = 32 * bsweep_chunks(g, (int32_t)std::min<int64_t>(((int64_t)batch + 31) / 32, cap / 32));
        // the batched region (its own memory-tracker segments + the
        // candidate-parallel state); guarded by its own layout signature
        if (!refine) take_mem(std::min(ng_batch, kMemSegMax));
    }
    L.B = BLayout{};
    if (batched) {
        // candidate-parallel region (bsweep.cu), sized for one group of ng candidates
        const size_t nparts = (size_t)std::max(g->n_bparts, 1), nhubs = (size_t)std::max(g->n_bhubs, 1);
        const int32_t ng = ng_batch;
        const size_t nck = (size_t)ng / 32;
        BLayout& B = L.B;
        B.ng = ng;
        B.hdr = take(sizeof(WsHeader));
        B.lab = take(nck * V * 32);
        B.tlr = take(nck * V * 32 * 8);
        B.blr = take(nck * V * 32 * 8);
        B.nxt = take(nck * V * 32 * 4);
        B.keys = take((size_t)ng * V * 8);
        B.plab = take((size_t)ng * V);
        B.part_val = take(nck * nparts * 32 * 8);
        B.part_idx = take(nck * nparts * 32 * 4);
        B.hub_cnt = take(nck * nhubs * 4);
        B.slots = take((size_t)bsweep_warps(g) * 32 * sizeof(BSlot));
        B.maxst = take((size_t)ng * 8);
        B.emu = emulated ? take(emulate_ws_bytes(g, ng)) : 0;
    }
    if (op == PDNN_OP_RESOLVE_OVERFLOW) {   // scratch of the overflow handler (no persistent state)
        L.ov_mcons = take(8 * V * PDNN_MAX_PE);
        L.ov_a = take(8 * V);
        L.ov_excl = take(V);
        L.ov_small = take(1024);
    }
    if (op == PDNN_OP_LFLAM) {   // scratch of the LFLAM mapping (no persistent state)
        const size_t NC = V + PDNN_MAX_PE + 1, D = (size_t)std::max(g->n_levels, 1);
        L.lf_lvl = take(8 * (PDNN_MAX_PE + 1) * D);
        L.lf_tree = take(8 * (PDNN_MAX_PE + 1) * (D + 1));
        L.lf_rec = take(48 * NC);
        L.lf_cm = take(4 * (NC + 1));
        L.lf_ce = take(4 * (NC + 1));
        L.lf_moff = take(4 * (NC + 1));
        L.lf_eoff = take(4 * (NC + 1));
        L.lf_ml = take(4 * V);
        L.lf_mc = take(8 * V);
        L.lf_epos = take(4 * 2 * E);
        L.lf_ew = take(8 * 2 * E);
        L.lf_comm = take(8 * PDNN_MAX_PE * NC);
        L.lf_crit = take(8 * NC);
        L.lf_keys = take(16 * NC);
        L.lf_ids = take(8 * NC);
        L.lf_pos = take(4 * NC);
        L.lf_list = take(8 * NC);
        L.lf_map = take(NC);
        L.lf_ctl = take(256);
        L.lf_temp_bytes = lflam_temp_bytes((int32_t)NC);
        L.lf_temp = take(L.lf_temp_bytes);
    }
    if (refine) {   // scratch of the refinement (no persistent state besides the batched sweep's)
        const size_t NC = V + PDNN_MAX_PE + 1, D = (size_t)std::max(g->n_levels, 1), NT = 2 * (D + 1);
        L.rf_keys = take(16 * NC);
        L.rf_ids = take(8 * NC);
        L.rf_rec = take(64 * NC);
        L.rf_cnt = take(4 * (NC + 1));
        L.rf_eoff = take(4 * (NC + 1));
        L.rf_ey = take(8 * 2 * E);
        L.rf_ew = take(8 * 2 * E);
        L.rf_marked = take(NC);
        L.rf_temp_bytes = refine_temp_bytes((int32_t)NC);
        L.rf_temp = take(L.rf_temp_bytes);
        L.rf_lvl = take(8 * PDNN_MAX_PE * D);
        L.rf_tree = take(8 * PDNN_MAX_PE * (D + 1));
        L.rf_tn = take(4 * NT);
        L.rf_tq = take(4 * NT);
        L.rf_tdead = take(NT);
        L.rf_elig = take(4 * NT);
        L.rf_res = take(sizeof(pdnn_eval_result) * NT);
        L.rf_rows = take((size_t)std::max(ng_batch, 32) * V);   // one group of trial placements
        L.rf_resg = take(sizeof(pdnn_eval_result) * (size_t)std::max(ng_batch, 32));
        L.rf_log = take(32 * std::max(NC / 2 + 1, NT));
        L.rf_ctl = take(256);
    }
    L.total = off;
    if (op == PDNN_OP_RESOLVE_OVERFLOW) L.sig_batch = layout_sig(g, 0x0F10F10ull, L.total);
    else if (op == PDNN_OP_LFLAM) L.sig_batch = layout_sig(g, 0x1F1A3ull, L.total);
    else if (refine) L.sig_batch = layout_sig(g, 0x2EF1E5ull, L.total);
    else L.sig_batch = ng_batch > 0 ? layout_sig(g, ((uint64_t)ng_batch * 0x9E3779B97F4A7C15ull ^ (uint64_t)L.m_seg) + emulated,
                                            L.total) : 0;
    return L;
}

static void launch_blob(const pdnn_graph* g, const int64_t* c, const int64_t* in_cost, const int64_t* out_cost,
                        unsigned char* blob_in, unsigned char* blob_out, cudaStream_t s) {
    if (g->n_items == 0) return;
    k_blob<<<grid_for((int64_t)g->n_items * 32, 256), 256, 0, s>>>(g->n_items, g->items, g->in_off, g->in_src,
                                                                 g->out_off, g->out_dst, c, in_cost, out_cost,
                                                                 g->orig, g->inodes, blob_in, blob_out);
    count_launch();
}

pdnn_status resolve_costs(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                          void* ws, const WsLayout& L, cudaStream_t s, Costs* out, bool need_blob) {
    if (!node_cost && !edge_cost) {
        if (!g->costs_bound) { set_error("no costs bound to the graph and none given"); return PDNN_EINVAL; }
        *out = Costs{g->c_rank, g->in_cost, g->out_cost, g->blob[0], g->blob[1]};
        return PDNN_OK;
    }
    if (!node_cost || !edge_cost) { set_error("node_cost and edge_cost must both be given or both NULL"); return PDNN_EINVAL; }
    int64_t* c = ws_ptr<int64_t>(ws, L.c_s);
    int64_t* ic = ws_ptr<int64_t>(ws, L.in_cost_s);
    int64_t* oc = ws_ptr<int64_t>(ws, L.out_cost_s);
    unsigned char* bi = ws_ptr<unsigned char>(ws, L.blob_s_in);
    unsigned char* bo = ws_ptr<unsigned char>(ws, L.blob_s_out);
    if (g->V > 0 || g->E > 0) {
        k_perm_costs<<<grid_for(std::max<int64_t>(g->V, g->E)), 256, 0, s>>>(
            g->V, g->E, g->orig, g->in_eid, g->out_eid, nullptr, node_cost, edge_cost, c, ic, oc, nullptr);
        count_launch();
        PDNN_LAUNCH_CHECK();
        if (need_blob) {
            launch_blob(g, c, ic, oc, bi, bo, s);
            PDNN_LAUNCH_CHECK();
        }
    }
    *out = Costs{c, ic, oc, need_blob ? bi : nullptr, need_blob ? bo : nullptr};
    return PDNN_OK;
}

pdnn_status launch_labels(const pdnn_graph* g, const int32_t* part_i32, const uint8_t* part_u8, int32_t fill,
                          int32_t* part_orig_out, int32_t* part_rank, cudaStream_t s) {
    if (g->V == 0) return PDNN_OK;
    k_labels<<<grid_for(g->V, 256, g->num_sms * 16), 256, 0, s>>>(g->V, g->orig, part_i32, part_u8, fill,
                                                                  part_orig_out, part_rank);
    count_launch();
    PDNN_LAUNCH_CHECK();
    return PDNN_OK;
}

}  // namespace pdnn

using namespace pdnn;

// ------------------------------------------------------------------ C ABI
extern "C" {

const char* pdnn_status_string(pdnn_status s) {
    switch (s) {
        case PDNN_OK: return "PDNN_OK";
        case PDNN_EINVAL: return "PDNN_EINVAL";
        case PDNN_ECYCLE: return "PDNN_ECYCLE";
        case PDNN_ENOMEM: return "PDNN_ENOMEM";
        case PDNN_ECUDA: return "PDNN_ECUDA";
        case PDNN_EOVERFLOW: return "PDNN_EOVERFLOW";
        case PDNN_EWORKSPACE: return "PDNN_EWORKSPACE";
    }
    return "PDNN_UNKNOWN";
}

const char* pdnn_last_error(void) { return t_last_error.c_str(); }

uint64_t pdnn_launch_count(void) { return g_launches.load(); }

void pdnn_graph_free(pdnn_graph* g) { free_graph(g); }

pdnn_status pdnn_graph_query(const pdnn_graph* g, int32_t* n, int64_t* m, int32_t* n_levels,
                             int32_t* max_in, int32_t* max_out) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (n) *n = g->V;
    if (m) *m = g->E;
    if (n_levels) *n_levels = g->n_levels;
    if (max_in) *max_in = g->max_in;
    if (max_out) *max_out = g->max_out;
    return PDNN_OK;
}

pdnn_status pdnn_graph_levels(const pdnn_graph* g, int32_t* level_out, void* stream) {
    if (!g || (!level_out && g->V > 0)) { set_error("null argument"); return PDNN_EINVAL; }
    if (g->V == 0) return PDNN_OK;
    PDNN_CUDA_TRY(cudaMemcpyAsync(level_out, g->level, sizeof(int32_t) * g->V,
                                  cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return PDNN_OK;
}

size_t pdnn_workspace_bytes(const pdnn_graph* g, int op, int32_t batch) {
    if (!g) return 0;
    return ws_layout(g, op, batch).total;
}

pdnn_status pdnn_workspace_init(void* ws, size_t ws_bytes, void* stream) {
    if (!ws) { set_error("null workspace"); return PDNN_EWORKSPACE; }
    PDNN_CUDA_TRY(cudaMemsetAsync(ws, 0, ws_bytes, (cudaStream_t)stream));
    PDNN_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    return PDNN_OK;
}

pdnn_status pdnn_build_csr(int32_t V, int64_t E, const int32_t* src, const int32_t* dst,
                           int32_t* perm_out, void* stream, pdnn_graph** out) {
    if (!out) { set_error("out is NULL"); return PDNN_EINVAL; }
    *out = nullptr;
    if (V < 0 || E < 0 || E >= (int64_t(1) << 31)) { set_error("bad sizes"); return PDNN_EINVAL; }
    if (E > 0 && (!src || !dst)) { set_error("null edge arrays"); return PDNN_EINVAL; }
    if (E > 0 && V == 0) { set_error("edges on an empty node set"); return PDNN_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    // (debug build, PDNN_BUILD_TRACE=1) host-timed phases of the build, on stderr
    const bool btrace = debug_knob("PDNN_BUILD_TRACE", 0) != 0;
    auto t_last = std::chrono::steady_clock::now();
    auto phase = [&](const char* name) {
        if (!btrace) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "build %-12s %8.3f ms\n", name, std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    pdnn_graph* g = new (std::nothrow) pdnn_graph();
    if (!g) return PDNN_ENOMEM;
    PDNN_CUDA_TRY(cudaGetDevice(&g->device));
    PDNN_CUDA_TRY(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, g->device));
    g->V = V;
    g->E = E;
    g->rank_bits = bits_for(V > 0 ? (uint64_t)(V - 1) : 0);
    DevBufs tmp, keep;
    tmp.s = keep.s = s;
    const int64_t En = std::max<int64_t>(E, 1);
    uint64_t *key = nullptr, *key2 = nullptr, *kout = nullptr;
    int32_t *idx = nullptr, *csrc = nullptr, *cdst = nullptr, *flags = nullptr, *outdeg = nullptr,
            *indeg = nullptr, *indeg0 = nullptr, *queue = nullptr, *ctrl = nullptr, *idx2 = nullptr,
            *indeg_r = nullptr, *outdeg_r = nullptr, *lvl_sorted = nullptr, *iota = nullptr,
            *out_off_orig = nullptr;
    cudaError_t ce = cudaSuccess;
#define ALLOC(buf, p, n) do { ce = buf.alloc(&(p), (n)); if (ce != cudaSuccess) { free_graph(g); set_error("cudaMalloc failed"); return PDNN_ENOMEM; } } while (0)
    ALLOC(tmp, key, En); ALLOC(tmp, key2, En); ALLOC(tmp, kout, En);
    ALLOC(tmp, idx, En); ALLOC(tmp, idx2, En); ALLOC(tmp, csrc, En); ALLOC(tmp, cdst, En);
    ALLOC(tmp, flags, 4); ALLOC(tmp, outdeg, V + 1); ALLOC(tmp, indeg, V + 1); ALLOC(tmp, indeg0, V + 1);
    ALLOC(tmp, queue, V + 1); ALLOC(tmp, ctrl, 16); ALLOC(tmp, indeg_r, V + 1); ALLOC(tmp, outdeg_r, V + 1);
    ALLOC(tmp, lvl_sorted, V + 1); ALLOC(tmp, iota, V + 1); ALLOC(tmp, out_off_orig, V + 1);
    ALLOC(keep, g->rank_of, V); ALLOC(keep, g->orig, V); ALLOC(keep, g->level, V);
    ALLOC(keep, g->perm, En); ALLOC(keep, g->level_ptr, V + 1);
    ALLOC(keep, g->in_off, V + 1); ALLOC(keep, g->in_src, En); ALLOC(keep, g->in_eid, En);
    ALLOC(keep, g->out_off, V + 1); ALLOC(keep, g->out_dst, En); ALLOC(keep, g->out_eid, En);
#undef ALLOC
    // ownership of `keep` buffers moves to g (freed by free_graph on error)
    keep.ptrs.clear();
    phase("alloc");

    auto fail = [&](pdnn_status st) { free_graph(g); return st; };
#define TRY(expr) do { cudaError_t _e = (expr); if (_e != cudaSuccess) { set_error(std::string(#expr) + ": " + cudaGetErrorString(_e)); return fail(PDNN_ECUDA); } } while (0)
#define CHECK_LAUNCH() do { count_launch(); TRY(cudaGetLastError()); } while (0)

    TRY(cudaMemsetAsync(flags, 0, 16, s));
    TRY(cudaMemsetAsync(ctrl, 0, 64, s));
    TRY(cudaMemsetAsync(outdeg, 0, sizeof(int32_t) * (V + 1), s));
    TRY(cudaMemsetAsync(indeg, 0, sizeof(int32_t) * (V + 1), s));
    // 1. validation + canonical (src,dst) order
    void* cub_tmp = nullptr;
    size_t cub_bytes = 0, need = 0;
    const int key_bits = bits_for(V > 0 ? (uint64_t)V * (uint64_t)V - 1 : 0);
    if (E > 0) {
        k_validate<<<grid_for(E), 256, 0, s>>>(E, V, src, dst, key, idx, flags);
        CHECK_LAUNCH();
        cub::DeviceRadixSort::SortPairs(nullptr, need, key, key2, idx, g->perm, (int)E, 0, key_bits, s);
        cub_bytes = std::max(cub_bytes, need);
        cub::DeviceScan::ExclusiveSum(nullptr, need, indeg_r, g->in_off, V + 1, s);
        cub_bytes = std::max(cub_bytes, need);
        cub::DeviceRadixSort::SortPairs(nullptr, need, lvl_sorted, lvl_sorted, iota, iota, V, 0, 32, s);
        cub_bytes = std::max(cub_bytes, need);
        if (tmp.alloc((char**)&cub_tmp, cub_bytes) != cudaSuccess) return fail(PDNN_ENOMEM);
        TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, key, key2, idx, g->perm, (int)E, 0,
                                            key_bits, s));
        count_launch(4);
        k_canon<<<grid_for(E), 256, 0, s>>>(E, V, key2, csrc, cdst, outdeg, indeg, flags);
        CHECK_LAUNCH();
    } else {
        cub::DeviceScan::ExclusiveSum(nullptr, need, indeg_r, g->in_off, V + 1, s);
        cub_bytes = std::max(cub_bytes, need);
        cub::DeviceRadixSort::SortPairs(nullptr, need, lvl_sorted, lvl_sorted, iota, iota, std::max(V, 1), 0, 32, s);
        cub_bytes = std::max(cub_bytes, need);
        if (tmp.alloc((char**)&cub_tmp, cub_bytes) != cudaSuccess) return fail(PDNN_ENOMEM);
    }
    int32_t hflags[4] = {0, 0, 0, 0};
    TRY(cudaMemcpyAsync(hflags, flags, 16, cudaMemcpyDeviceToHost, s));
    TRY(cudaStreamSynchronize(s));
    if (hflags[0] & 1) { set_error("edge endpoint out of range"); return fail(PDNN_EINVAL); }
    if (hflags[0] & 2) { set_error("self loop"); return fail(PDNN_EINVAL); }
    if (hflags[0] & 4) { set_error("duplicate (src,dst) pair"); return fail(PDNN_EINVAL); }
    if (perm_out && E > 0) TRY(cudaMemcpyAsync(perm_out, g->perm, sizeof(int32_t) * E, cudaMemcpyDeviceToDevice, s));

    phase("validate");
    // 2. Kahn levels (cooperative frontier kernel)
    if (V > 0) {
        k_offsets_from_canon<<<grid_for(E + 1), 256, 0, s>>>(E, csrc, out_off_orig, V);
        CHECK_LAUNCH();
        TRY(cudaMemcpyAsync(indeg0, indeg, sizeof(int32_t) * V, cudaMemcpyDeviceToDevice, s));
        int nb = 0;
        TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_kahn, 256, 0));
        // small graphs: one CTA (every level is processed by CTA 0's block-
        // barrier path anyway; no inter-CTA hand-back, no grid barrier to wait on)
        int kgrid = V < kKahnOneCtaV ? 1 : std::max(1, std::min(nb, 4) * g->num_sms);
        void* args[] = {(void*)&V, (void*)&out_off_orig, (void*)&cdst, (void*)&indeg, (void*)&queue,
                        (void*)&g->level, (void*)&g->level_ptr, (void*)&ctrl};
        TRY(cudaLaunchCooperativeKernel((void*)k_kahn, dim3(kgrid), dim3(256), args, 0, s));
        count_launch();
        int32_t hctrl[2] = {0, 0};
        TRY(cudaMemcpyAsync(hctrl, ctrl, 8, cudaMemcpyDeviceToHost, s));
        TRY(cudaStreamSynchronize(s));
        if (hctrl[0] != V) { set_error("graph has a cycle"); return fail(PDNN_ECYCLE); }
        g->n_levels = hctrl[1];
        phase("kahn");
        // 3. rank = stable (level, id) order
        k_iota<<<grid_for(V), 256, 0, s>>>(V, iota);
        CHECK_LAUNCH();
        const int lbits = bits_for((uint64_t)g->n_levels);
        TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, g->level, lvl_sorted, iota, g->orig, V,
                                            0, lbits, s));
        count_launch(4);
        k_rank_of<<<grid_for(V), 256, 0, s>>>(V, g->orig, g->rank_of, indeg0, outdeg, indeg_r, outdeg_r);
        CHECK_LAUNCH();
        TRY(cudaMemsetAsync(indeg_r + V, 0, 4, s));
        TRY(cudaMemsetAsync(outdeg_r + V, 0, 4, s));
        TRY(cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, indeg_r, g->in_off, V + 1, s));
        TRY(cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, outdeg_r, g->out_off, V + 1, s));
        count_launch(2);
        // 4. rank-space CSRs
        if (E > 0) {
            k_rank_keys<<<grid_for(E), 256, 0, s>>>(E, V, csrc, cdst, g->rank_of, key, kout, idx);
            CHECK_LAUNCH();
            const int kb = bits_for((uint64_t)V * (uint64_t)V - 1);
            TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, key, key2, idx, g->in_eid, (int)E, 0, kb, s));
            k_split_key<<<grid_for(E), 256, 0, s>>>(E, V, key2, g->in_src);
            CHECK_LAUNCH();
            k_iota<<<grid_for(E), 256, 0, s>>>((int32_t)E, idx);
            CHECK_LAUNCH();
            TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, kout, key2, idx, g->out_eid, (int)E, 0, kb, s));
            k_split_key<<<grid_for(E), 256, 0, s>>>(E, V, key2, g->out_dst);
            CHECK_LAUNCH();
            count_launch(8);
        }
    } else {
        TRY(cudaMemsetAsync(g->level_ptr, 0, 4, s));
        TRY(cudaMemsetAsync(g->in_off, 0, 4, s));
        TRY(cudaMemsetAsync(g->out_off, 0, 4, s));
    }
    phase("rank+csr");
    // 5. host-side schedule (level structure + degrees)
    std::vector<int32_t> h_in(V + 1), h_out(V + 1), h_lp(g->n_levels + 1);
    TRY(cudaMemcpyAsync(h_in.data(), g->in_off, 4 * (V + 1), cudaMemcpyDeviceToHost, s));
    TRY(cudaMemcpyAsync(h_out.data(), g->out_off, 4 * (V + 1), cudaMemcpyDeviceToHost, s));
    TRY(cudaMemcpyAsync(h_lp.data(), g->level_ptr, 4 * (g->n_levels + 1), cudaMemcpyDeviceToHost, s));
    TRY(cudaStreamSynchronize(s));
    for (int32_t r = 0; r < V; ++r) {
        g->max_in = std::max(g->max_in, h_in[r + 1] - h_in[r]);
        g->max_out = std::max(g->max_out, h_out[r + 1] - h_out[r]);
    }
    phase("sched-d2h");
    // per rank of level 0: the lowest level among its successors (D for an
    // exit), whose bl completes the node's inputs (indexed bl items)
    std::vector<int32_t> bl_ready;
    const bool ix_items = debug_knob("PDNN_INDEXED_ITEMS", 1) != 0 && g->n_levels > 1 && V > 0;
    if (ix_items) {
        const int32_t n0 = h_lp[1];
        std::vector<int32_t> h_dst((size_t)std::max<int32_t>(h_out[n0], 1));
        if (h_out[n0] > 0)
            TRY(cudaMemcpyAsync(h_dst.data(), g->out_dst, 4 * (size_t)h_out[n0], cudaMemcpyDeviceToHost, s));
        TRY(cudaStreamSynchronize(s));
        bl_ready.assign(n0, g->n_levels);
        for (int32_t r = 0; r < n0; ++r)
            for (int32_t e = h_out[r]; e < h_out[r + 1]; ++e) {
                // level of rank h_dst[e]: level_ptr is sorted
                const int32_t lv = (int32_t)(std::upper_bound(h_lp.begin(), h_lp.end(), h_dst[e]) - h_lp.begin()) - 1;
                bl_ready[r] = std::min(bl_ready[r], lv);
            }
    }
    std::vector<Item> items, items_rm;
    std::vector<int32_t> hubs, hubs_rm, inodes, inodes_rm;
    build_items(h_lp, h_in, h_out, items, hubs, kTMaxDeg, kTMaxEdges, 32, kHEdges, /*split4=*/true,
                /*skip_entry_tl=*/true, debug_knob("PDNN_MERGE_MODE", 2), ix_items ? &bl_ready : nullptr,
                ix_items ? &inodes : nullptr);
    // the K-loop's sweeps remove nodes (their chains are cut short): there the
    // proportional interleave measured faster (C3 K = 8: 18.9 vs 24.1 ms), by
    // wave slower; both orders keep each direction's list order, so the blob
    // offsets below are the same for both
    build_items(h_lp, h_in, h_out, items_rm, hubs_rm, kTMaxDeg, kTMaxEdges, 32, kHEdges, /*split4=*/true,
                /*skip_entry_tl=*/true, debug_knob("PDNN_MERGE_MODE_RM", 0), ix_items ? &bl_ready : nullptr,
                ix_items ? &inodes_rm : nullptr);   // the same bl list and inodes (deterministic)
    phase("sched-items");
    // thread items address their blob (sweep.cu): z = 16-byte offset in the
    // direction's blob, w = lanes | edges << 8
    for (std::vector<Item>* lst : {&items, &items_rm}) {
        size_t boff[2] = {0, 0};
        for (Item& it : *lst) {
            if (it.y <= 0) continue;
            const int d = it.x >= 0 ? 0 : 1;
            const int32_t r0 = d == 0 ? it.x : ~it.x;
            const std::vector<int32_t>& off = d == 0 ? h_in : h_out;
            const bool ix = (it.w & kItemIndexed) != 0;
            const int32_t m = ix ? (it.w & ~kItemIndexed) : it.w - it.z;
            int32_t nl = 0;
            for (int32_t j = 0; j < it.y; ++j) {
                const int32_t x = ix ? inodes[r0 + j] : r0 + j;
                nl += std::max(1, (off[x + 1] - off[x] + 3) / 4);
            }
            const size_t bytes = ((size_t)(16 * nl + 4 * ((m + 1) & ~1) + 8 * m) + 15) & ~(size_t)15;
            if (boff[d] / 16 > 0x7fffffff) { set_error("sweep blob exceeds 32 GB"); return fail(PDNN_ENOMEM); }
            it.z = (int32_t)(boff[d] / 16);
            it.w = nl | m << 8 | (ix ? kItemIndexed : 0);
            boff[d] += bytes;
        }
        g->blob_bytes[0] = boff[0];
        g->blob_bytes[1] = boff[1];
    }
    g->n_items = (int32_t)items.size();
    g->n_hubs = (int32_t)hubs.size();
    std::vector<int32_t> heavy;
    for (int32_t r = 0; r < V; ++r)
        if (h_out[r + 1] - h_out[r] > kMemHeavyDeg) heavy.push_back(r);
    g->n_heavy_out = (int32_t)heavy.size();
    if (pool_alloc((void**)&g->items, sizeof(Item) * std::max<size_t>(items.size(), 1), s) != cudaSuccess ||
        pool_alloc((void**)&g->items_rm, sizeof(Item) * std::max<size_t>(items_rm.size(), 1), s) != cudaSuccess ||
        pool_alloc((void**)&g->hub_nparts, 4 * std::max<size_t>(hubs.size(), 1), s) != cudaSuccess ||
        pool_alloc((void**)&g->heavy_out, 4 * std::max<size_t>(heavy.size(), 1), s) != cudaSuccess)
        return fail(PDNN_ENOMEM);
    if (!items.empty()) TRY(cudaMemcpyAsync(g->items, items.data(), sizeof(Item) * items.size(), cudaMemcpyHostToDevice, s));
    if (!items_rm.empty())
        TRY(cudaMemcpyAsync(g->items_rm, items_rm.data(), sizeof(Item) * items_rm.size(), cudaMemcpyHostToDevice, s));
    if (inodes != inodes_rm) { set_error("sweep schedule: item orders disagree"); return fail(PDNN_EINVAL); }
    g->n_inodes = (int32_t)inodes.size();
    if (pool_alloc((void**)&g->inodes, 4 * std::max<size_t>(inodes.size(), 1), s) != cudaSuccess) return fail(PDNN_ENOMEM);
    if (!inodes.empty())
        TRY(cudaMemcpyAsync(g->inodes, inodes.data(), 4 * inodes.size(), cudaMemcpyHostToDevice, s));
    if (!hubs.empty()) TRY(cudaMemcpyAsync(g->hub_nparts, hubs.data(), 4 * hubs.size(), cudaMemcpyHostToDevice, s));
    if (!heavy.empty()) TRY(cudaMemcpyAsync(g->heavy_out, heavy.data(), 4 * heavy.size(), cudaMemcpyHostToDevice, s));
    phase("sched-blobs");
    g->sweep_grid = sweep_blocks_per_sm(g->device, V, g->n_levels) * g->num_sms;
    // batched (candidate-parallel) sweep schedule: warp = one node x 32 candidates
    {
        std::vector<int32_t> pbase;
        for (int li = 0; li < 2; ++li) {
            std::vector<Item> bitems;
            std::vector<int32_t> bhubs;
            build_items(h_lp, h_in, h_out, bitems, bhubs, kBMaxDeg, kBMaxEdges, li == 0 ? 1 : kBWideNodes, kBHubEdges,
                        false, false, debug_knob("PDNN_BMERGE_MODE", 2));
            if (li == 0) {   // hub splitting does not depend on the nodes per item
                pbase.assign(bhubs.size() + 1, 0);
                for (size_t i = 0; i < bhubs.size(); ++i) pbase[i + 1] = pbase[i] + bhubs[i];
                g->n_bhubs = (int32_t)bhubs.size();
                g->n_bparts = pbase.back();
            }
            g->n_bitems[li] = (int32_t)bitems.size();
            if (pool_alloc((void**)&g->bitems[li], sizeof(Item) * std::max<size_t>(bitems.size(), 1), s) != cudaSuccess)
                return fail(PDNN_ENOMEM);
            if (!bitems.empty())
                TRY(cudaMemcpyAsync(g->bitems[li], bitems.data(), sizeof(Item) * bitems.size(), cudaMemcpyHostToDevice, s));
        }
        if (pool_alloc((void**)&g->bhub_pbase, 4 * pbase.size(), s) != cudaSuccess) return fail(PDNN_ENOMEM);
        TRY(cudaMemcpyAsync(g->bhub_pbase, pbase.data(), 4 * pbase.size(), cudaMemcpyHostToDevice, s));
        g->n_entry = g->n_levels > 0 ? h_lp[1] : 0;
    }
    TRY(cudaStreamSynchronize(s));
#undef TRY
#undef CHECK_LAUNCH
    phase("sched-batch");
    *out = g;
    return PDNN_OK;
}

// pdnn_validate: flags[0] bit 0 = a bad label, bit 1 = a bad kind / negative
// mem, bit 2 = st < 0 or decreasing along an edge, bit 3 = negative cost or
// cost sum >= 2^62, bit 4 = mem sum >= 2^61; flags[1] / flags[2] = sums
__global__ void k_validate_inputs(int32_t V, int64_t E, const int32_t* __restrict__ orig,
                                  const int32_t* __restrict__ out_off, const int32_t* __restrict__ out_dst,
                                  const int64_t* __restrict__ nc, const int64_t* __restrict__ ec,
                                  const int32_t* __restrict__ part, int32_t P, const int64_t* __restrict__ mem,
                                  const uint8_t* __restrict__ kind, const int64_t* __restrict__ st,
                                  unsigned long long* flags) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    unsigned long long f = 0, csum = 0, cbad = 0, msum = 0;
    for (int64_t r = tid; r < V; r += nth) {
        const int32_t u = orig[r];
        if (nc) cost_check(nc[u], csum, cbad);
        if (part) {
            const int32_t l = part[u];
            if (P > 0 ? (l < 0 || l >= P) : (l < 0 && l != PDNN_REMOVED && l != PDNN_UNASSIGNED)) f |= 1;
        }
        if (kind && kind[u] > PDNN_KIND_REFERENCE) f |= 2;
        if (mem) {
            const int64_t m = mem[u];
            if (m < 0) f |= 2;
            else if ((msum += (unsigned long long)m) >= (1ull << 61)) { f |= 16; msum = 1ull << 61; }
        }
        if (st) {
            const int64_t su = st[u];
            if (su < 0) f |= 4;
            for (int32_t e = out_off[r]; e < out_off[r + 1]; ++e)
                if (st[orig[out_dst[e]]] < su) f |= 4;
        }
    }
    if (ec)
        for (int64_t e = tid; e < E; e += nth) cost_check(ec[e], csum, cbad);
    if (cbad) f |= 8;
    if (csum) {
        const unsigned long long old = atomicAdd(&flags[1], csum);
        if (old >= (1ull << 62) || old + csum >= (1ull << 62)) f |= 8;
    }
    if (msum) {
        const unsigned long long old = atomicAdd(&flags[2], msum);
        if (old >= (1ull << 61) || old + msum >= (1ull << 61)) f |= 16;
    }
    if (f) atomicOr(&flags[0], f);
}

pdnn_status pdnn_validate(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                          const int32_t* part, int32_t n_pe, const int64_t* mem, const uint8_t* kind,
                          const int64_t* st, void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (n_pe < 0 || n_pe > PDNN_MAX_PE) { set_error("n_pe must be in [0, 16]"); return PDNN_EINVAL; }
    if ((node_cost == nullptr) != (edge_cost == nullptr)) { set_error("node_cost and edge_cost go together"); return PDNN_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* fl = nullptr;
    PDNN_CUDA_TRY(cudaMalloc(&fl, 32));
    unsigned long long h[3] = {0, 0, 0};
    cudaError_t e = cudaMemsetAsync(fl, 0, 32, s);
    if (e == cudaSuccess && (g->V > 0 || g->E > 0)) {
        k_validate_inputs<<<grid_for(std::max<int64_t>(g->V, g->E)), 256, 0, s>>>(
            g->V, g->E, g->orig, g->out_off, g->out_dst, node_cost, edge_cost, part, n_pe, mem, kind, st, fl);
        count_launch();
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, fl, 24, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(fl);
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return PDNN_ECUDA; }
    if (h[0] & 8) { set_error("negative cost, cost >= 2^62 or sum(comp)+sum(comm) >= 2^62"); return PDNN_EOVERFLOW; }
    if (h[0] & 16) { set_error("sum(mem) >= 2^61"); return PDNN_EOVERFLOW; }
    if (h[0] & 1) { set_error("label out of range"); return PDNN_EINVAL; }
    if (h[0] & 2) { set_error("negative mem or kind not in {0,1,2}"); return PDNN_EINVAL; }
    if (h[0] & 4) { set_error("st negative or decreasing along an edge"); return PDNN_EINVAL; }
    return PDNN_OK;
}

pdnn_status pdnn_graph_set_costs(pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                                 int edge_order, void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if ((g->V > 0 && !node_cost) || (g->E > 0 && !edge_cost)) { set_error("null cost array"); return PDNN_EINVAL; }
    if (edge_order != PDNN_EDGE_ORDER_CANONICAL && edge_order != PDNN_EDGE_ORDER_INPUT) {
        set_error("bad edge_order");
        return PDNN_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (!g->c_rank) {
        if (pool_alloc((void**)&g->c_rank, 8 * ((size_t)std::max(g->V, 1) + 16), s) != cudaSuccess ||
            pool_alloc((void**)&g->in_cost, 8 * ((size_t)std::max<int64_t>(g->E, 1) + 16), s) != cudaSuccess ||
            pool_alloc((void**)&g->out_cost, 8 * ((size_t)std::max<int64_t>(g->E, 1) + 16), s) != cudaSuccess) {
            set_error("cudaMalloc failed");
            return PDNN_ENOMEM;
        }
    }
    if (!g->blob[0]) {
        if (pool_alloc((void**)&g->blob[0], g->blob_bytes[0] + 16, s) != cudaSuccess ||
            pool_alloc((void**)&g->blob[1], g->blob_bytes[1] + 16, s) != cudaSuccess) {
            set_error("cudaMalloc failed");
            return PDNN_ENOMEM;
        }
    }
    unsigned long long* chk = nullptr;
    PDNN_CUDA_TRY(cudaMalloc(&chk, 32));
    PDNN_CUDA_TRY(cudaMemsetAsync(chk, 0, 32, s));
    if (g->V > 0 || g->E > 0) {
        k_perm_costs<<<grid_for(std::max<int64_t>(g->V, g->E)), 256, 0, s>>>(
            g->V, g->E, g->orig, g->in_eid, g->out_eid,
            edge_order == PDNN_EDGE_ORDER_INPUT ? g->perm : nullptr, node_cost, edge_cost, g->c_rank,
            g->in_cost, g->out_cost, chk);
        count_launch();
        if (cudaGetLastError() != cudaSuccess) { cudaFree(chk); set_error("k_perm_costs launch"); return PDNN_ECUDA; }
        launch_blob(g, g->c_rank, g->in_cost, g->out_cost, g->blob[0], g->blob[1], s);
        if (cudaGetLastError() != cudaSuccess) { cudaFree(chk); set_error("k_blob launch"); return PDNN_ECUDA; }
    }
    unsigned long long h[2] = {0, 0};
    cudaMemcpyAsync(h, chk, 16, cudaMemcpyDeviceToHost, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { cudaFree(chk); set_error(cudaGetErrorString(e)); return PDNN_ECUDA; }
    g->costs_bound = false;
    if (h[1]) { cudaFree(chk); set_error("negative cost, cost >= 2^62 or sum(comp)+sum(comm) >= 2^62"); return PDNN_EOVERFLOW; }
    uint64_t total = h[0];
    cudaFree(chk);
    g->cost_total = total;
    g->costs_bound = true;
    return PDNN_OK;
}

}  // extern "C"
