// memory.cu -- the per-PE memory-potential scan (§8(a) row a7): the memory
// consumption tracker of Heuristic I (Eq. 3 at
// PAPER.md:465-481; M_pot in Table 2) in the visit-order
// reading R8-R12 of DESIGN.md.
//
// The tracker is one pass over the nodes in start-time order;
// on the GPU it becomes
//   prep   rank-space labels, sort keys st, residual base per PE
//   sort   stable radix sort of st over level order -> visit order (st, level, id)
//   pos    pos(n) = rank in the visit order
//   edges  per node: last consumer position on each PE (registers, <= 16 PEs),
//          the PE set it is held on, and its release into its last consumer's
//          slot (integer atomics: order-independent, deterministic)
//   scan   a hand-written segmented (per-PE) prefix scan over positions in
//          tiles of 4096: tile sums -> tile prefixes -> per-position M_cons,
//          per-tile peak / argmax / first overflow -> final per-PE reduction.
// M_cons(q,i) = base(q) + sum_{j<i} D_j(q) + acq_i(q) with
//   acq_i(q) = effmem(n_i) if node n_i is held on q from its visit
//   D_i(q)   = acq_i(q) - [q == pe(n_i)] * (relp_i + selfrel_i * effmem(n_i))
#include <cooperative_groups.h>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace pdnn {

struct __align__(16) Rec {
    long long eff;   // effmem of the node visited at this position
    int32_t meta;    // bits 0-15 hold mask, 16-20 home PE, 24 self-release
    int32_t n;       // original id of that node
};

// ---------------------------------------------------------------- prep
// keys = st in level order, payload = (rank << 5) | PE; residual base per PE
// (Eq. 3 term 1); max(st) for the sort's pass count.
__global__ void k_mem_prep(int32_t V, const int32_t* __restrict__ orig, const int32_t* __restrict__ part,
                           const int32_t* __restrict__ part_rank_in, const int64_t* __restrict__ st, bool st_rank,
                           const int64_t* __restrict__ mem, const uint8_t* __restrict__ kind,
                           uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
                           unsigned long long* __restrict__ base, unsigned long long* __restrict__ maxst) {
    __shared__ unsigned long long s_base[PDNN_MAX_PE];
    __shared__ unsigned long long s_max;
    if (threadIdx.x < PDNN_MAX_PE) s_base[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
    unsigned long long mx = 0;
    unsigned long long res[PDNN_MAX_PE];
#pragma unroll
    for (int q = 0; q < PDNN_MAX_PE; ++q) res[q] = 0;
    for (int32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < V; r += gridDim.x * blockDim.x) {
        const int32_t n = orig[r];
        const int32_t h = part_rank_in ? part_rank_in[r] : part[n];
        const uint64_t x = (uint64_t)st[st_rank ? r : n];
        keys[r] = x;
        vals[r] = ((uint32_t)r << 5) | ((uint32_t)h & 31u);
        mx = x > mx ? x : mx;
        if (kind[n] == PDNN_KIND_RESIDUAL) {
            const unsigned long long m = (unsigned long long)mem[n];
#pragma unroll
            for (int q = 0; q < PDNN_MAX_PE; ++q) res[q] += q == h ? m : 0ull;
        }
    }
#pragma unroll
    for (int q = 0; q < PDNN_MAX_PE; ++q) {
        unsigned long long x = res[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0 && x) atomicAdd(&s_base[q], x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
    }
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(&s_max, mx);
    __syncthreads();
    if (threadIdx.x < PDNN_MAX_PE && s_base[threadIdx.x]) atomicAdd(&base[threadIdx.x], s_base[threadIdx.x]);
    if (threadIdx.x == 0 && s_max) atomicMax(maxst, s_max);
}

// ---------------------------------------------------------------- sort
// Stable LSD radix sort of the st keys (8-bit digits) in one cooperative
// launch; the number of passes, ceil(bits(max st) / 8), is decided on the
// device, so a level schedule whose st spans 28 bits costs 4 passes.  Stable
// + level-ordered input => the output is the (st, level, id) visit order.
// Per pass: tile histograms -> per-digit scan over tiles -> stable scatter
// (warp __match_any_sync ranks + per-warp digit counts), 3 grid barriers.
constexpr int kSortThreads = 512, kSortWarps = kSortThreads / 32, kSortPer = 8;
constexpr int kSortTile = kSortThreads * kSortPer, kRadix = 256;

struct SortArgs {
    int32_t V;
    int32_t n_tiles;
    int32_t rounds;   // tile = rounds * kSortThreads keys (one tile per CTA)
    uint64_t* k0;
    uint32_t* v0;
    uint64_t* k1;
    uint32_t* v1;
    uint32_t* order;
    uint32_t* hist;   // [n_tiles][256]
    uint32_t* dtot;   // [256]
    const unsigned long long* maxst;
};

__global__ void __launch_bounds__(kSortThreads) k_mem_sort(SortArgs a) {
    __shared__ uint32_t s_hist[kRadix];
    __shared__ uint32_t s_dbase[kRadix];
    __shared__ uint32_t s_base[kRadix];
    __shared__ uint32_t s_rtot[kRadix];
    __shared__ uint32_t s_wcnt[kSortWarps][kRadix];   // per-warp digit counts (leaders write, then clear)
    __shared__ uint32_t s_pref[kSortWarps][kRadix];   // exclusive prefix over warps (fully rewritten)
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int c = tid; c < kSortWarps * kRadix; c += kSortThreads) (&s_wcnt[0][0])[c] = 0u;
    const unsigned long long mx = *a.maxst;
    const int nbits = mx ? 64 - __clzll((long long)mx) : 0;
    const int npass = (nbits + 7) / 8;
    if (npass == 0) {
        for (int32_t i = blockIdx.x * kSortThreads + tid; i < a.V; i += gridDim.x * kSortThreads) a.order[i] = a.v0[i];
        return;
    }
    for (int p = 0; p < npass; ++p) {
        const uint64_t* ks = (p & 1) ? a.k1 : a.k0;
        const uint32_t* vs = (p & 1) ? a.v1 : a.v0;
        uint64_t* kd = (p & 1) ? a.k0 : a.k1;
        uint32_t* vd = (p & 1) ? a.v0 : a.v1;
        const bool last = p == npass - 1;
        const int sh = 8 * p;
        // phase 1: tile histograms
        for (int t = blockIdx.x; t < a.n_tiles; t += gridDim.x) {
            if (tid < kRadix) s_hist[tid] = 0;
            __syncthreads();
            for (int j = 0; j < a.rounds; ++j) {
                const int32_t i = (t * a.rounds + j) * kSortThreads + tid;
                const int d = i < a.V ? (int)((ks[i] >> sh) & 255) : kRadix;
                const unsigned m = __match_any_sync(0xffffffffu, d);   // one smem atomic per digit per warp
                if (d < kRadix && (m & ((1u << lane) - 1u)) == 0) atomicAdd(&s_hist[d], (uint32_t)__popc(m));
            }
            __syncthreads();
            if (tid < kRadix) a.hist[(size_t)t * kRadix + tid] = s_hist[tid];
            __syncthreads();
        }
        grid.sync();
        // phase 2: exclusive scan over tiles for each digit (one warp per digit)
        {
            const int nwarps = (gridDim.x * kSortThreads) >> 5;
            for (int dg = (blockIdx.x * kSortThreads + tid) >> 5; dg < kRadix; dg += nwarps) {
                uint32_t run = 0;
                for (int t0 = 0; t0 < a.n_tiles; t0 += 32) {
                    const int t = t0 + lane;
                    const uint32_t x = t < a.n_tiles ? a.hist[(size_t)t * kRadix + dg] : 0u;
                    uint32_t incl = x;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    if (t < a.n_tiles) a.hist[(size_t)t * kRadix + dg] = run + incl - x;
                    run += __shfl_sync(0xffffffffu, incl, 31);
                }
                if (lane == 0) a.dtot[dg] = run;
            }
        }
        grid.sync();
        // phase 3: digit bases, then the stable scatter
        if (tid < kRadix) {
            const uint32_t x = a.dtot[tid];
            uint32_t incl = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_rtot[warp] = incl;
            s_dbase[tid] = incl - x;
        }
        __syncthreads();
        if (tid < kRadix) {
            uint32_t add = 0;
            for (int w = 0; w < warp; ++w) add += s_rtot[w];
            s_dbase[tid] += add;
        }
        __syncthreads();
        for (int t = blockIdx.x; t < a.n_tiles; t += gridDim.x) {
            if (tid < kRadix) s_base[tid] = s_dbase[tid] + a.hist[(size_t)t * kRadix + tid];
            for (int j = 0; j < a.rounds; ++j) {
                const int32_t i = (t * a.rounds + j) * kSortThreads + tid;
                const bool valid = i < a.V;
                const uint64_t k = valid ? ks[i] : 0ull;
                const uint32_t v = valid ? vs[i] : 0u;
                const int d = valid ? (int)((k >> sh) & 255) : kRadix;
                const unsigned mask = __match_any_sync(0xffffffffu, d);
                const unsigned lt = mask & ((1u << lane) - 1u);
                if (valid && lt == 0) s_wcnt[warp][d] = __popc(mask);
                __syncthreads();
                if (tid < kRadix) {
                    uint32_t acc = 0;
#pragma unroll
                    for (int w = 0; w < kSortWarps; ++w) {
                        const uint32_t c = s_wcnt[w][tid];
                        s_pref[w][tid] = acc;
                        acc += c;
                    }
                    s_rtot[tid] = acc;
                }
                __syncthreads();
                if (valid) {
                    if (lt == 0) s_wcnt[warp][d] = 0u;   // leaders restore the zero counts
                    const uint32_t dst = s_base[d] + s_pref[warp][d] + __popc(lt);
                    if (last) {
                        a.order[dst] = v;
                    } else {
                        kd[dst] = k;
                        vd[dst] = v;
                    }
                }
                __syncthreads();
                if (tid < kRadix) s_base[tid] += s_rtot[tid];
            }
            __syncthreads();
        }
        grid.sync();
    }
}

int mem_sort_blocks_per_sm() {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_mem_sort, kSortThreads, 0);
    return n < 1 ? 1 : n;
}

// ---------------------------------------------------------------- positions
// pp[r] = (pos(r) << 5) | PE(r): one 4-byte gather gives a successor's
// position and PE in the edge pass
__global__ void k_mem_pos(int32_t V, const uint32_t* __restrict__ order, uint32_t* __restrict__ pp) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < V; i += gridDim.x * blockDim.x) {
        const uint32_t x = order[i];
        pp[x >> 5] = ((uint32_t)i << 5) | (x & 31u);
    }
}

template <int PT>
__device__ __forceinline__ void mem_finish_node(int32_t r, const int32_t (&last)[PT],
                                                const int32_t* __restrict__ orig,
                                                const uint32_t* __restrict__ pp,
                                                const int64_t* __restrict__ mem,
                                                const uint8_t* __restrict__ kind,
                                                unsigned long long* __restrict__ relp, Rec* __restrict__ rec) {
    const int32_t n = orig[r];
    const uint32_t me = pp[r];
    const int32_t h = (int32_t)(me & 31u), pos = (int32_t)(me >> 5);
    const int kd = kind[n];
    const long long eff = kd == PDNN_KIND_REFERENCE ? 0 : mem[n];
    int32_t mask = 0, last_h = -1;
#pragma unroll
    for (int q = 0; q < PT; ++q) {
        if (q == h) last_h = last[q];
        if (last[q] >= 0) {
            if (q != h) mask |= 1 << q;               // remote copy on q (Eq. 3 term 3)
            if (eff > 0 && !(kd == PDNN_KIND_RESIDUAL && q == h))
                atomicAdd(&relp[last[q]], (unsigned long long)eff);  // released after its last consumer on q
        }
    }
    int selfrel = 0;
    if (kd == PDNN_KIND_NORMAL) {
        mask |= 1 << h;                               // held on its own PE from its visit
        selfrel = last_h < 0;                         // ... through its own visit only
    }
    Rec x;
    x.eff = eff;
    x.meta = mask | (h << 16) | (selfrel << 24);
    x.n = n;
    rec[pos] = x;
}

template <int PT>
__global__ void __launch_bounds__(256) k_mem_edges(int32_t V, const int32_t* __restrict__ out_off,
                                                   const int32_t* __restrict__ out_dst,
                                                   const uint32_t* __restrict__ pp,
                                                   const int32_t* __restrict__ orig,
                                                   const int64_t* __restrict__ mem,
                                                   const uint8_t* __restrict__ kind,
                                                   const int32_t* __restrict__ heavy, int32_t n_heavy,
                                                   unsigned long long* __restrict__ relp,
                                                   Rec* __restrict__ rec) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    for (int32_t r = tid; r < V; r += nth) {
        const int32_t s0 = out_off[r], s1 = out_off[r + 1];
        if (s1 - s0 > kTMaxDeg) continue;  // heavy: warp path below
        int32_t last[PT];
#pragma unroll
        for (int q = 0; q < PT; ++q) last[q] = -1;
        for (int32_t e = s0; e < s1; ++e) {
            const uint32_t x = pp[out_dst[e]];
            const int32_t q = (int32_t)(x & 31u), p = (int32_t)(x >> 5);
#pragma unroll
            for (int k = 0; k < PT; ++k) last[k] = (k == q && p > last[k]) ? p : last[k];
        }
        mem_finish_node<PT>(r, last, orig, pp, mem, kind, relp, rec);
    }
    const int lane = threadIdx.x & 31;
    for (int32_t hi = tid >> 5; hi < n_heavy; hi += nth >> 5) {
        const int32_t r = heavy[hi];
        int32_t last[PT];
#pragma unroll
        for (int q = 0; q < PT; ++q) last[q] = -1;
        for (int32_t e = out_off[r] + lane; e < out_off[r + 1]; e += 32) {
            const uint32_t x = pp[out_dst[e]];
            const int32_t q = (int32_t)(x & 31u), p = (int32_t)(x >> 5);
#pragma unroll
            for (int k = 0; k < PT; ++k) last[k] = (k == q && p > last[k]) ? p : last[k];
        }
#pragma unroll
        for (int q = 0; q < PT; ++q) last[q] = __reduce_max_sync(0xffffffffu, last[q]);
        if (lane == 0) mem_finish_node<PT>(r, last, orig, pp, mem, kind, relp, rec);
    }
}

// D_i(q) for one position
template <int PT>
__device__ __forceinline__ void add_delta(long long (&d)[PT], const Rec& x, long long rel) {
    const int32_t mask = x.meta & 0xffff, h = (x.meta >> 16) & 0x1f;
    const long long out = rel + ((x.meta >> 24) & 1 ? x.eff : 0);
#pragma unroll
    for (int q = 0; q < PT; ++q) d[q] += ((mask >> q) & 1 ? x.eff : 0) - (q == h ? out : 0);
}

template <int PT>
__global__ void __launch_bounds__(kMemThreads) k_mem_tile_sums(int32_t V, const Rec* __restrict__ rec,
                                                               const unsigned long long* __restrict__ relp,
                                                               long long* __restrict__ tile_sum) {
    __shared__ long long s_w[kMemThreads / 32][PT];
    long long d[PT];
#pragma unroll
    for (int q = 0; q < PT; ++q) d[q] = 0;
    const int32_t i0 = blockIdx.x * kMemTile + threadIdx.x * kMemPerThread;
    const int32_t i1 = min(V, i0 + kMemPerThread);
    for (int32_t i = i0; i < i1; ++i) add_delta<PT>(d, rec[i], (long long)relp[i]);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < PT; ++q) {
        const long long v = warp_sum_i64(d[q]);
        if (lane == 0) s_w[warp][q] = v;
    }
    __syncthreads();
    if (threadIdx.x < PT) {
        long long t = 0;
        for (int w = 0; w < kMemThreads / 32; ++w) t += s_w[w][threadIdx.x];
        tile_sum[(size_t)blockIdx.x * PDNN_MAX_PE + threadIdx.x] = t;
    }
}

// one CTA per PE: exclusive scan of the tile sums, seeded with the residual
// base (each thread owns a contiguous run of tiles)
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) k_mem_tile_scan(int32_t n_tiles, int32_t P,
                                                                const unsigned long long* __restrict__ base,
                                                                long long* __restrict__ tile_sum) {
    __shared__ long long s_w[kScanThreads / 32];
    const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (n_tiles + kScanThreads - 1) / kScanThreads;
    const int t0 = tid * per, t1 = min(n_tiles, t0 + per);
    long long loc = 0;
    for (int t = t0; t < t1; ++t) loc += tile_sum[(size_t)t * PDNN_MAX_PE + q];
    long long incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    long long run = (long long)base[q] + incl - loc;
    for (int w = 0; w < warp; ++w) run += s_w[w];
    for (int t = t0; t < t1; ++t) {   // in place: sum -> exclusive prefix
        const long long x = tile_sum[(size_t)t * PDNN_MAX_PE + q];
        tile_sum[(size_t)t * PDNN_MAX_PE + q] = run;
        run += x;
    }
}

template <int PT>
__global__ void __launch_bounds__(kMemThreads) k_mem_tile_final(
    int32_t V, int32_t P, const Rec* __restrict__ rec, const unsigned long long* __restrict__ relp,
    const long long* __restrict__ tile_pref, const int64_t* __restrict__ cap_eff,
    int64_t* __restrict__ mpot, int64_t* __restrict__ mcons,
    TileRes* __restrict__ tile_res) {
    __shared__ long long s_w[kMemThreads / 32][PT];
    __shared__ TileRes s_r[kMemThreads / 32][PT];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t i0 = blockIdx.x * kMemTile + threadIdx.x * kMemPerThread;
    const int32_t i1 = min(V, i0 + kMemPerThread);
    long long d[PT];
#pragma unroll
    for (int q = 0; q < PT; ++q) d[q] = 0;
    for (int32_t i = i0; i < i1; ++i) add_delta<PT>(d, rec[i], (long long)relp[i]);
    // block exclusive scan of the per-thread delta vectors
    long long run[PT];
#pragma unroll
    for (int q = 0; q < PT; ++q) {
        long long incl = d[q];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_w[warp][q] = incl;
        run[q] = incl - d[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PT; ++q) {
        long long b = tile_pref[(size_t)blockIdx.x * PDNN_MAX_PE + q];
        for (int w = 0; w < warp; ++w) b += s_w[w][q];
        run[q] += b;
    }
    long long pk[PT], fov[PT];
    int32_t pkp[PT], fo[PT];
    long long cap[PT];
#pragma unroll
    for (int q = 0; q < PT; ++q) {
        pk[q] = 0; pkp[q] = -1; fo[q] = -1; fov[q] = 0;
        cap[q] = q < P ? cap_eff[q] : 0x7fffffffffffffffll;
    }
    for (int32_t i = i0; i < i1; ++i) {
        const Rec x = rec[i];
        const long long rel = (long long)relp[i];
        const int32_t mask = x.meta & 0xffff;
#pragma unroll
        for (int q = 0; q < PT; ++q) {
            const bool acq = (mask >> q) & 1;
            const long long val = run[q] + (acq ? x.eff : 0);
            if (mcons && q < P) mcons[(size_t)q * V + i] = val;
            if ((acq && x.eff > 0) || i == 0) {   // the only places a new max / overflow can start
                if (pkp[q] < 0 || val > pk[q]) { pk[q] = val; pkp[q] = i; }
                if (fo[q] < 0 && val > cap[q]) { fo[q] = i; fov[q] = val; }
            }
        }
        add_delta<PT>(run, x, rel);
        mpot[x.n] = x.eff + rel;                        // M7: own output + released predecessors
    }
    // block reduce per PE: max (lowest position on ties), first overflow
#pragma unroll
    for (int q = 0; q < PT; ++q) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long v2 = __shfl_xor_sync(0xffffffffu, pk[q], o);
            const int32_t p2 = __shfl_xor_sync(0xffffffffu, pkp[q], o);
            if (p2 >= 0 && (pkp[q] < 0 || v2 > pk[q] || (v2 == pk[q] && p2 < pkp[q]))) { pk[q] = v2; pkp[q] = p2; }
            const int32_t f2 = __shfl_xor_sync(0xffffffffu, fo[q], o);
            const long long fv2 = __shfl_xor_sync(0xffffffffu, fov[q], o);
            if (f2 >= 0 && (fo[q] < 0 || f2 < fo[q])) { fo[q] = f2; fov[q] = fv2; }
        }
        if (lane == 0) s_r[warp][q] = TileRes{pk[q], pkp[q], fo[q], fov[q]};
    }
    __syncthreads();
    if (threadIdx.x < PT) {
        const int q = threadIdx.x;
        TileRes t = s_r[0][q];
        for (int w = 1; w < kMemThreads / 32; ++w) {
            const TileRes u = s_r[w][q];
            if (u.peak_pos >= 0 && (t.peak_pos < 0 || u.peak > t.peak || (u.peak == t.peak && u.peak_pos < t.peak_pos))) {
                t.peak = u.peak; t.peak_pos = u.peak_pos;
            }
            if (u.first_over >= 0 && (t.first_over < 0 || u.first_over < t.first_over)) {
                t.first_over = u.first_over; t.over_val = u.over_val;
            }
        }
        tile_res[(size_t)blockIdx.x * PDNN_MAX_PE + q] = t;
    }
}

__device__ __forceinline__ void merge_res(long long& pk, int32_t& pp, int32_t& fo, long long& fv, long long v2,
                                          int32_t p2, int32_t f2, long long fv2) {
    if (p2 >= 0 && (pp < 0 || v2 > pk || (v2 == pk && p2 < pp))) { pk = v2; pp = p2; }
    if (f2 >= 0 && (fo < 0 || f2 < fo)) { fo = f2; fv = fv2; }
}

// one CTA per PE: reduce the per-tile peaks / first overflows
__global__ void __launch_bounds__(kScanThreads) k_mem_final(int32_t n_tiles, int32_t P,
                                                            const TileRes* __restrict__ tile_res,
                                                            const int64_t* __restrict__ cap_eff,
                                                            int64_t* __restrict__ peak, int32_t* __restrict__ peak_pos,
                                                            int32_t* __restrict__ first_over,
                                                            int64_t* __restrict__ over_bytes) {
    __shared__ TileRes s_r[kScanThreads / 32];
    const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    long long pk = 0, fv = 0;
    int32_t pp = -1, fo = -1;
    for (int32_t t = tid; t < n_tiles; t += kScanThreads) {
        const TileRes u = tile_res[(size_t)t * PDNN_MAX_PE + q];
        merge_res(pk, pp, fo, fv, u.peak, u.peak_pos, u.first_over, u.over_val);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        merge_res(pk, pp, fo, fv, __shfl_xor_sync(0xffffffffu, pk, o), __shfl_xor_sync(0xffffffffu, pp, o),
                  __shfl_xor_sync(0xffffffffu, fo, o), __shfl_xor_sync(0xffffffffu, fv, o));
    if (lane == 0) s_r[warp] = TileRes{pk, pp, fo, fv};
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < kScanThreads / 32; ++w) merge_res(pk, pp, fo, fv, s_r[w].peak, s_r[w].peak_pos, s_r[w].first_over, s_r[w].over_val);
        peak[q] = pk;
        peak_pos[q] = pp;
        first_over[q] = fo;
        over_bytes[q] = fo >= 0 ? fv - cap_eff[q] : 0;
    }
}

__global__ void k_mem_empty(int32_t P, int64_t* peak, int32_t* peak_pos, int32_t* first_over, int64_t* over) {
    const int q = threadIdx.x;
    if (q < P) { peak[q] = 0; peak_pos[q] = -1; first_over[q] = -1; over[q] = 0; }
}

template <int PT>
static pdnn_status mem_scan(const pdnn_graph* g, int32_t P, const int64_t* mem, const uint8_t* kind,
                            const int64_t* cap_eff, int64_t* mpot, int64_t* peak, int32_t* peak_pos,
                            int32_t* first_over, int64_t* over_bytes, int64_t* mcons, void* ws,
                            const WsLayout& L, cudaStream_t s) {
    const int32_t V = g->V;
    const uint32_t* pp = ws_ptr<uint32_t>(ws, L.m_pp);
    unsigned long long* relp = ws_ptr<unsigned long long>(ws, L.m_relp);
    Rec* rec = ws_ptr<Rec>(ws, L.m_rec);
    long long* tsum = ws_ptr<long long>(ws, L.m_tile);
    TileRes* tres = ws_ptr<TileRes>(ws, L.m_tile_res);
    const int grid = std::min(ceil_div(V, 256), g->num_sms * 8);
    k_mem_edges<PT><<<grid, 256, 0, s>>>(V, g->out_off, g->out_dst, pp, g->orig, mem, kind, g->heavy_out,
                                         g->n_heavy_out, relp, rec);
    const int tiles = ceil_div(V, kMemTile);
    k_mem_tile_sums<PT><<<tiles, kMemThreads, 0, s>>>(V, rec, relp, tsum);
    k_mem_tile_scan<<<P, kScanThreads, 0, s>>>(tiles, P, ws_ptr<unsigned long long>(ws, L.m_base), tsum);
    k_mem_tile_final<PT><<<tiles, kMemThreads, 0, s>>>(V, P, rec, relp, tsum, cap_eff, mpot, mcons, tres);
    k_mem_final<<<P, kScanThreads, 0, s>>>(tiles, P, tres, cap_eff, peak, peak_pos, first_over, over_bytes);
    count_launch(5);
    PDNN_LAUNCH_CHECK();
    return PDNN_OK;
}

pdnn_status launch_memory(const pdnn_graph* g, const int32_t* part_orig, const int32_t* part_rank_in,
                          int32_t P, const int64_t* mem, const uint8_t* kind, const int64_t* st,
                          const int64_t* cap_eff, int64_t* mpot, int64_t* peak, int32_t* peak_pos,
                          int32_t* first_over, int64_t* over_bytes, int64_t* mcons, void* ws,
                          const WsLayout& L, cudaStream_t s, bool st_rank) {
    const int32_t V = g->V;
    if (V == 0) {
        k_mem_empty<<<1, 32, 0, s>>>(P, peak, peak_pos, first_over, over_bytes);
        count_launch();
        PDNN_LAUNCH_CHECK();
        return PDNN_OK;
    }
    unsigned long long* base = ws_ptr<unsigned long long>(ws, L.m_base);   // [16] base + [1] max st
    PDNN_CUDA_TRY(cudaMemsetAsync(base, 0, 8 * (PDNN_MAX_PE + 1), s));
    PDNN_CUDA_TRY(cudaMemsetAsync(ws_ptr<void>(ws, L.m_relp), 0, 8 * (size_t)V, s));
    const int grid = std::min(ceil_div(V, 256), g->num_sms * 8);
    SortArgs sa;
    static int sort_bpsm = mem_sort_blocks_per_sm();
    const int max_grid = sort_bpsm * g->num_sms;
    sa.V = V;
    sa.rounds = std::max(kSortPer, ceil_div(ceil_div(V, max_grid), kSortThreads));
    sa.n_tiles = ceil_div(V, sa.rounds * kSortThreads);
    sa.k0 = ws_ptr<uint64_t>(ws, L.m_keys);
    sa.k1 = ws_ptr<uint64_t>(ws, L.m_keys_alt);
    sa.v0 = ws_ptr<uint32_t>(ws, L.m_vals);
    sa.v1 = ws_ptr<uint32_t>(ws, L.m_vals_alt);
    sa.order = ws_ptr<uint32_t>(ws, L.m_order);
    sa.hist = ws_ptr<uint32_t>(ws, L.m_hist);
    sa.dtot = ws_ptr<uint32_t>(ws, L.m_dtot);
    sa.maxst = base + PDNN_MAX_PE;
    k_mem_prep<<<grid, 256, 0, s>>>(V, g->orig, part_orig, part_rank_in, st, st_rank, mem, kind, sa.k0, sa.v0, base,
                                    base + PDNN_MAX_PE);
    count_launch();
    PDNN_LAUNCH_CHECK();
    // visit order: stable sort of st over level order == sort by (st, level, id)
    const int sgrid = std::max(1, std::min(sa.n_tiles, max_grid));
    void* args[] = {(void*)&sa};
    PDNN_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_mem_sort, dim3(sgrid), dim3(kSortThreads), args, 0, s));
    count_launch();
    k_mem_pos<<<grid, 256, 0, s>>>(V, sa.order, ws_ptr<uint32_t>(ws, L.m_pp));
    count_launch();
    PDNN_LAUNCH_CHECK();
    if (P <= 2) return mem_scan<2>(g, P, mem, kind, cap_eff, mpot, peak, peak_pos, first_over, over_bytes, mcons, ws, L, s);
    if (P <= 4) return mem_scan<4>(g, P, mem, kind, cap_eff, mpot, peak, peak_pos, first_over, over_bytes, mcons, ws, L, s);
    if (P <= 8) return mem_scan<8>(g, P, mem, kind, cap_eff, mpot, peak, peak_pos, first_over, over_bytes, mcons, ws, L, s);
    return mem_scan<16>(g, P, mem, kind, cap_eff, mpot, peak, peak_pos, first_over, over_bytes, mcons, ws, L, s);
}

}  // namespace pdnn

using namespace pdnn;

extern "C" pdnn_status pdnn_memory_potential(const pdnn_graph* g, const int32_t* part, int32_t n_pe,
                                             const int64_t* mem, const uint8_t* kind, const int64_t* st,
                                             const int64_t* cap_eff, int64_t* mpot, int64_t* peak,
                                             int32_t* peak_pos, int32_t* first_over_pos,
                                             int64_t* over_bytes, int64_t* mcons, void* ws,
                                             size_t ws_bytes, void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (n_pe < 1 || n_pe > PDNN_MAX_PE) { set_error("n_pe must be in [1, 16]"); return PDNN_EINVAL; }
    if (!cap_eff || !peak || !peak_pos || !first_over_pos || !over_bytes ||
        (g->V > 0 && (!part || !mem || !kind || !st || !mpot))) {
        set_error("null argument");
        return PDNN_EINVAL;
    }
    const WsLayout L = ws_layout(g, PDNN_OP_MEMORY, 0);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    return launch_memory(g, part, nullptr, n_pe, mem, kind, st, cap_eff, mpot, peak, peak_pos, first_over_pos,
                         over_bytes, mcons, ws, L, (cudaStream_t)stream);
}
