// memory.cu -- the per-PE memory-potential scan (§8(a) row a7): the memory
// consumption tracker of Heuristic I (Eq. 3 at
// PAPER.md:465-481; M_pot in Table 2) in the visit-order
// reading R8-R12 of DESIGN.md.
//
// The tracker is one pass over the nodes in start-time order;
// on the GPU it becomes
//   prep   rank-space labels, sort keys st, residual base per PE
//   sort   stable radix sort of st over level order -> visit order (st, level, id)
//   pos    pp(n) = (position in the visit order << 5) | PE, written by the sort's last pass
//   edges  per node: last consumer position on each PE (registers, <= 16 PEs),
//          the PE set it is held on, and its release into its last consumer's
//          slot (integer atomics: order-independent, deterministic)
//   scan   a hand-written segmented (per-PE) prefix scan over positions in
//          tiles of 1024: tile sums -> tile prefixes -> per-position M_cons,
//          per-tile peak / argmax / first overflow -> final per-PE reduction.
// M_cons(q,i) = base(q) + sum_{j<i} D_j(q) + acq_i(q) with
//   acq_i(q) = effmem(n_i) if node n_i is held on q from its visit
//   D_i(q)   = acq_i(q) - [q == pe(n_i)] * (relp_i + selfrel_i * effmem(n_i))
//
// Every kernel is segmented: blockIdx.y selects one of S independent
// candidate placements (batched evaluation, row a8) whose per-node arrays sit
// V elements apart; the single-placement call is S = 1.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace pdnn {

struct __align__(16) Rec {
    long long eff;   // effmem of the node visited at this position
    int32_t meta;    // bits 0-15 hold mask, 16-20 home PE, 24 self-release
    int32_t n;       // original id of that node
};

// ---------------------------------------------------------------- prep
// keys = st in level order, PE per rank; residual base per PE
// (Eq. 3 term 1); max(st) over all segments for the sort's pass count.
// Labels come from exactly one source: int32 node-id order, int32 rank order,
// or uint8 rank order (segment-strided); st in node-id order or in rank order
// (segment-strided).
struct PrepArgs {
    int32_t V;
    const int32_t* orig;
    const int32_t* part_i32_orig;
    const int32_t* part_i32_rank;
    const uint8_t* part_u8_rank;
    const int64_t* st_orig;
    const int64_t* st_rank;
    const int64_t* mem;
    const uint8_t* kind;
    uint64_t* keys;
    uint8_t* pe8;                // [S][V] PE per rank
    unsigned long long* base;    // [S][PDNN_MAX_PE]
    unsigned long long* maxst;   // one word for all segments
};

__global__ void k_mem_prep(PrepArgs a) {
    __shared__ unsigned long long s_base[PDNN_MAX_PE];
    __shared__ unsigned long long s_max;
    const size_t so = (size_t)blockIdx.y * a.V;
    if (threadIdx.x < PDNN_MAX_PE) s_base[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
    unsigned long long mx = 0;
    unsigned long long res[PDNN_MAX_PE];
#pragma unroll
    for (int q = 0; q < PDNN_MAX_PE; ++q) res[q] = 0;
    // PDNN_PREP_U ranks per thread per round, every gather issued before the first use
#ifndef PDNN_PREP_U
#define PDNN_PREP_U 4
#endif
    constexpr int U = PDNN_PREP_U;
    const int32_t nth = gridDim.x * blockDim.x;
    for (int32_t r0 = blockIdx.x * blockDim.x + threadIdx.x; r0 < a.V; r0 += U * nth) {
        int32_t n[U], h[U];
        uint64_t x[U];
        int kd[U];
#pragma unroll
        for (int u = 0; u < U; ++u) n[u] = r0 + u * nth < a.V ? __ldg(&a.orig[r0 + u * nth]) : -1;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t r = r0 + u * nth;
            if (n[u] < 0) { h[u] = 0; x[u] = 0; kd[u] = -1; continue; }
            h[u] = a.part_u8_rank ? (int32_t)a.part_u8_rank[so + r]
                                  : (a.part_i32_rank ? a.part_i32_rank[r] : __ldg(&a.part_i32_orig[n[u]]));
            x[u] = (uint64_t)(a.st_rank ? a.st_rank[so + r] : __ldg(&a.st_orig[n[u]]));
            kd[u] = __ldg(&a.kind[n[u]]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (kd[u] < 0) continue;
            const int32_t r = r0 + u * nth;
            a.keys[so + r] = x[u];
            a.pe8[so + r] = (uint8_t)h[u];
            mx = x[u] > mx ? x[u] : mx;
            if (kd[u] == PDNN_KIND_RESIDUAL) {
                const unsigned long long m = (unsigned long long)__ldg(&a.mem[n[u]]);
#pragma unroll
                for (int q = 0; q < PDNN_MAX_PE; ++q) res[q] += q == h[u] ? m : 0ull;
            }
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
    if (threadIdx.x < PDNN_MAX_PE && s_base[threadIdx.x])
        atomicAdd(&a.base[(size_t)blockIdx.y * PDNN_MAX_PE + threadIdx.x], s_base[threadIdx.x]);
    if (threadIdx.x == 0 && s_max) atomicMax(a.maxst, s_max);
}

// ---------------------------------------------------------------- sort
// Lanes of the warp holding the same digit d (d < 0: none), from dbits ballots
// (MATCH.ANY is a low-throughput instruction; ballots issue at full rate).
__device__ __forceinline__ unsigned peer_mask(int d, int dbits) {
    unsigned m = __ballot_sync(0xffffffffu, d >= 0);
    for (int b = 0; b < dbits; ++b) {
        const bool x = (d >> b) & 1;
        const unsigned bal = __ballot_sync(0xffffffffu, x);
        m &= x ? bal : ~bal;
    }
    return d >= 0 ? m : 0u;
}

// Stable LSD radix sort of the st keys of S segments in ONE cooperative
// launch, in the one-sweep style: every pass reads each key once and writes it
// once.  Input: raw st per rank (rank order); output: pp[rank] = (position of
// the node in the visit order << 5) | PE.  Stable + rank-ordered input => the order is
// the (st, level, id) visit order.
//   * packed mode (bits(max st) + bits(V-1) <= 64, decided on the device):
//     pass 0 builds key = st << rb | rank, later passes move 8 bytes per key
//     and only the st bits are sorted (the rank bits are already in order);
//     otherwise (st, rank) pairs, 12 bytes per key;
//   * the st bits are covered by npass = ceil(nbits / 10) passes of <= 10-bit
//     digits; phase 0 histograms every pass's digits in one read and scans
//     them into per-(segment, pass) digit bases;
//   * per pass, CTAs take tiles in ticket order; a tile ranks its keys (warp
//     ballot peer masks against per-warp digit counters + a scan over warps),
//     publishes its digit counts, finds its global offsets by decoupled
//     look-back over the preceding tiles of its segment (epoch-tagged 64-bit
//     status words: no zeroing between launches), reorders the tile in shared
//     memory by digit and writes each digit run out contiguously.
constexpr int kSortThreads = 256, kSortWarps = kSortThreads / 32, kSortPer = 8;
constexpr int kSortTile = kSortThreads * kSortPer;   // 2048 keys per tile
constexpr int kRadixMax = 512, kMaxPass = 7;   // <= 9-bit digits
constexpr int kSortSmem = kSortWarps * kRadixMax * 4      // per-warp digit counters / phase-0 histograms
                          + kSortTile * 8 + kSortTile * 4 // tile keys, values
                          + 3 * kRadixMax * 4             // digit counts, local offsets, global bases
                          + kSortTile * 8 + kSortTile * 4;// the next tile's keys, values (cp.async prefetch)
static_assert(kMaxPass * kRadixMax <= kSortWarps * kRadixMax, "phase-0 histograms fit the counter area");

struct SortArgs {
    int32_t V;
    int32_t S;        // segments
    int32_t tps;      // tiles per segment
    int32_t rb;       // rank bits = bits(V - 1)
    uint64_t* k0;     // raw st on input (rank order)
    uint64_t* k1;
    uint32_t* v0;     // unpacked mode only
    uint32_t* v1;
    uint32_t* pp;                // output: pp[rank] = (pos << 5) | PE (the visit order, inverted)
    const uint8_t* pe8;          // PE per rank
    uint32_t* gbase;             // [S][kMaxPass][kRadixMax] digit totals -> exclusive bases (zeroed by the host)
    uint64_t* status;            // [S * tps][kRadixMax] look-back words
    uint32_t* ticket;            // [kMaxPass] tile tickets (zeroed by the host)
    unsigned long long* epoch;   // launch counter (device-owned)
    const unsigned long long* maxst;
    unsigned long long* trace;   // PDNN_SORT_TRACE=1: per-phase cycles summed over CTAs (diagnostic)
};

__device__ __forceinline__ void cp_async_8(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src),
                 "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_4(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src),
                 "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

#ifndef PDNN_ONESWEEP_MIN_SEG
#define PDNN_ONESWEEP_MIN_SEG 8
#endif
constexpr int kOneSweepMinSeg = PDNN_ONESWEEP_MIN_SEG;
__device__ unsigned long long g_osort_trace[16];
constexpr unsigned long long kStAgg = 1ull << 30, kStInc = 2ull << 30, kStCnt = (1ull << 30) - 1;

__global__ void __launch_bounds__(kSortThreads, 3) k_mem_sort(SortArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* s_wcnt = reinterpret_cast<uint32_t*>(smem_raw);                // [kSortWarps][kRadixMax]
    uint64_t* s_key = reinterpret_cast<uint64_t*>(s_wcnt + kSortWarps * kRadixMax);
    uint32_t* s_val = reinterpret_cast<uint32_t*>(s_key + kSortTile);
    uint32_t* s_cnt = s_val + kSortTile;
    uint32_t* s_loff = s_cnt + kRadixMax;
    uint32_t* s_gb = s_loff + kRadixMax;
    uint64_t* s_pk = reinterpret_cast<uint64_t*>(s_gb + kRadixMax);   // prefetched keys (own slots per thread)
    uint32_t* s_pv = reinterpret_cast<uint32_t*>(s_pk + kSortTile);
    __shared__ uint32_t s_wtot[kSortWarps];
    __shared__ uint32_t s_tile;
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_tiles = a.S * a.tps;
    const unsigned long long mx = *a.maxst;
    const int nbits = mx ? 64 - __clzll((long long)mx) : 0;
    const bool packed = nbits + a.rb <= 64;
    const int npass = (nbits + 8) / 9;
    const int dbits = npass ? (nbits + npass - 1) / npass : 0;
    const int radix = 1 << dbits;
    const uint32_t dmask = (uint32_t)radix - 1u;
    const uint64_t rmask = (1ull << a.rb) - 1;
    const unsigned long long ep0 = *a.epoch;
    if (npass == 0) {   // every st is 0: the visit order is the rank order
        const size_t tot = (size_t)a.S * a.V;
        for (size_t i = (size_t)blockIdx.x * kSortThreads + tid; i < tot; i += (size_t)gridDim.x * kSortThreads)
            a.pp[i] = ((uint32_t)(i % (size_t)a.V) << 5) | (uint32_t)a.pe8[i];
        return;
    }
    // ---- phase 0: digit histograms of every pass (raw st), one read of the keys
    for (int c = tid; c < npass * kRadixMax; c += kSortThreads) s_wcnt[c] = 0u;
    __syncthreads();
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int sg = t / a.tps;
        const size_t so = (size_t)sg * a.V;
        const int32_t i0 = (t % a.tps) * kSortTile;
        for (int j = 0; j < kSortPer; ++j) {
            const int32_t i = i0 + j * kSortThreads + tid;
            const uint64_t st = i < a.V ? a.k0[so + i] : 0ull;
            for (int p = 0; p < npass; ++p) {
                const int d = i < a.V ? (int)((st >> (dbits * p)) & dmask) : -1;
                if (d >= 0) atomicAdd(&s_wcnt[p * kRadixMax + d], 1u);   // (peer-mask aggregation cost more than the conflicts)
            }
        }
        // flush at the end of a segment run of this CTA (next tile in another segment or none)
        const int tn = t + gridDim.x;
        if (tn >= n_tiles || tn / a.tps != sg) {
            __syncthreads();
            for (int c = tid; c < npass * kRadixMax; c += kSortThreads) {
                const uint32_t x = s_wcnt[c];
                if (x) atomicAdd(&a.gbase[((size_t)sg * kMaxPass + c / kRadixMax) * kRadixMax + (c % kRadixMax)], x);
                s_wcnt[c] = 0u;
            }
            __syncthreads();
        }
    }
    grid.sync();
    // exclusive scan of each (segment, pass) digit histogram (one CTA per pair; 4 digits per thread)
    for (int sp = blockIdx.x; sp < a.S * npass; sp += gridDim.x) {
        uint32_t* h = a.gbase + ((size_t)(sp / npass) * kMaxPass + (sp % npass)) * kRadixMax;
        uint32_t x[4], loc = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) { x[q] = 4 * tid + q < radix ? h[4 * tid + q] : 0u; loc += x[q]; }
        uint32_t incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_wtot[warp] = incl;
        __syncthreads();
        uint32_t run = incl - loc;
        for (int w = 0; w < warp; ++w) run += s_wtot[w];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (4 * tid + q < radix) h[4 * tid + q] = run;
            run += x[q];
        }
        __syncthreads();
    }
    for (int c = tid; c < kSortWarps * kRadixMax; c += kSortThreads) s_wcnt[c] = 0u;
    grid.sync();
    long long tr[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tc = 0;
#define PDNN_OSTAMP(ph) if (a.trace && tid == 0) { const long long t_ = clock64(); tr[ph] += t_ - tc; tc = t_; }
    if (a.trace && tid == 0) tc = clock64();
    // ---- the passes
    for (int p = 0; p < npass; ++p) {
        const uint64_t* ks = (p & 1) ? a.k1 : a.k0;
        const uint32_t* vs = (p & 1) ? a.v1 : a.v0;
        uint64_t* kd = (p & 1) ? a.k0 : a.k1;
        uint32_t* vd = (p & 1) ? a.v0 : a.v1;
        const bool last = p == npass - 1;
        const unsigned long long tagp = ((ep0 * kMaxPass + (unsigned long long)p + 1ull) & 0xffffffffull) << 32;
        // the keys of ticket tk into this thread's own prefetch slots (cp.async:
        // the next tile's loads are in flight while the current tile is ranked)
        auto prefetch = [&](int tk) {
            if (tk >= n_tiles) return;
            const int sg = tk % a.S, lt = tk / a.S;
            const size_t so = (size_t)sg * a.V;
            const int32_t t0 = lt * kSortTile;
#pragma unroll
            for (int j = 0; j < kSortPer; ++j) {
                const int e = warp * (32 * kSortPer) + j * 32 + lane;
                const int32_t i = t0 + e;
                const bool valid = i < a.V;
                cp_async_8(&s_pk[e], valid ? (const void*)&ks[so + i] : (const void*)ks, valid);
                if (!packed && p > 0) cp_async_4(&s_pv[e], valid ? (const void*)&vs[so + i] : (const void*)vs, valid);
            }
            cp_async_commit();
        };
        __syncthreads();
        if (tid == 0) s_tile = atomicAdd(&a.ticket[p], 1u);
        __syncthreads();
        int tk = (int)s_tile;
        prefetch(tk);
        for (;;) {
            if (tk >= n_tiles) break;
            cp_async_wait_all();   // this thread's own slots of tile tk
            uint64_t pk8[kSortPer];
            uint32_t pv8[kSortPer];
#pragma unroll
            for (int j = 0; j < kSortPer; ++j) {
                const int e = warp * (32 * kSortPer) + j * 32 + lane;
                pk8[j] = s_pk[e];
                pv8[j] = (!packed && p > 0) ? s_pv[e] : 0u;
            }
            __syncthreads();
            if (tid == 0) s_tile = atomicAdd(&a.ticket[p], 1u);
            __syncthreads();
            const int tkn = (int)s_tile;
            prefetch(tkn);   // overwrites only this thread's own (already read) slots
            PDNN_OSTAMP(7)
            // tickets interleave the segments, so only a few tiles of a segment are
            // in flight at once and the look-back stays shallow
            const int sg = tk % a.S, lt = tk / a.S;
            const int t = sg * a.tps + lt;
            const size_t so = (size_t)sg * a.V;
            const int32_t t0 = lt * kSortTile;
            const int n_valid = min(kSortTile, a.V - t0);
            PDNN_OSTAMP(0)
            // 1. load (warp w owns tile keys [w*256, w*256+256) in 8 rounds of 32)
            uint64_t key[kSortPer];
            uint32_t val[kSortPer];
            int dig[kSortPer];
            uint32_t rk[kSortPer];
            uint32_t* wc = s_wcnt + warp * kRadixMax;
#pragma unroll
            for (int j = 0; j < kSortPer; ++j) {
                const int32_t i = t0 + warp * (32 * kSortPer) + j * 32 + lane;
                const bool valid = i < a.V;
                uint64_t k = valid ? pk8[j] : 0ull;
                uint32_t v = 0;
                if (valid) {
                    if (p == 0) {
                        v = (uint32_t)i;
                        if (packed) k = (k << a.rb) | (uint64_t)i;
                    } else if (!packed) {
                        v = pv8[j];
                    }
                }
                key[j] = k;
                val[j] = v;
                dig[j] = valid ? (int)(((packed ? (k >> a.rb) : k) >> (dbits * p)) & dmask) : -1;
            }
            PDNN_OSTAMP(1)
            // 2. warp-local stable ranks
#pragma unroll
            for (int j = 0; j < kSortPer; ++j) {
                const int d = dig[j];
                const unsigned m = d >= 0 ? __match_any_sync(__activemask(), d) : 0u;   // one instruction vs dbits + 1 ballots
                const uint32_t c0 = d >= 0 ? wc[d] : 0u;
                __syncwarp();
                if (d >= 0 && (m & ((1u << lane) - 1u)) == 0) wc[d] = c0 + (uint32_t)__popc(m);
                __syncwarp();
                rk[j] = c0 + (uint32_t)__popc(m & ((1u << lane) - 1u));
            }
            __syncthreads();
            PDNN_OSTAMP(2)
            // 3. per digit: exclusive over warps (in place) and the tile count
            for (int d = tid; d < radix; d += kSortThreads) {
                uint32_t acc = 0;
#pragma unroll
                for (int w = 0; w < kSortWarps; ++w) {
                    const uint32_t c = s_wcnt[w * kRadixMax + d];
                    s_wcnt[w * kRadixMax + d] = acc;
                    acc += c;
                }
                s_cnt[d] = acc;
                // publish this tile's count (the first tile of a segment publishes its inclusive prefix)
                const unsigned long long w = tagp | (lt == 0 ? kStInc : kStAgg) | (unsigned long long)acc;
                st_relaxed_u64(&a.status[(size_t)t * kRadixMax + d], w);
            }
            __syncthreads();
            // 4. tile-local digit offsets (exclusive scan of the counts; 4 digits per thread)
            {
                uint32_t x[4], loc = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) { x[q] = 4 * tid + q < radix ? s_cnt[4 * tid + q] : 0u; loc += x[q]; }
                uint32_t incl = loc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                if (lane == 31) s_wtot[warp] = incl;
                __syncthreads();
                uint32_t run = incl - loc;
                for (int w = 0; w < warp; ++w) run += s_wtot[w];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (4 * tid + q < radix) s_loff[4 * tid + q] = run;
                    run += x[q];
                }
            }
            PDNN_OSTAMP(3)
            // 5. decoupled look-back over the preceding tiles of the segment; a
            //    thread serves digits tid and tid + kSortThreads, both polls in flight
            {
                static_assert(kRadixMax <= 2 * kSortThreads, "two digits per thread");
                const int d0 = tid, d1 = tid + kSortThreads;
                const bool a0 = d0 < radix, a1 = d1 < radix;
                uint32_t e0 = 0, e1 = 0;
                if (lt > 0) {
                    int j0 = t - 1, j1 = t - 1;
                    bool f0 = !a0, f1 = !a1;
                    while (!(f0 && f1)) {
                        unsigned long long w0 = 0, w1 = 0;
                        if (!f0) w0 = ld_relaxed_u64(&a.status[(size_t)j0 * kRadixMax + d0]);
                        if (!f1) w1 = ld_relaxed_u64(&a.status[(size_t)j1 * kRadixMax + d1]);
                        if (!f0 && (w0 & 0xffffffff00000000ull) == tagp && (w0 & (3ull << 30)) != 0) {
                            e0 += (uint32_t)(w0 & kStCnt);
                            if (w0 & kStInc) f0 = true; else --j0;
                        }
                        if (!f1 && (w1 & 0xffffffff00000000ull) == tagp && (w1 & (3ull << 30)) != 0) {
                            e1 += (uint32_t)(w1 & kStCnt);
                            if (w1 & kStInc) f1 = true; else --j1;
                        }
                    }
                    if (a0) st_relaxed_u64(&a.status[(size_t)t * kRadixMax + d0], tagp | kStInc | (unsigned long long)(e0 + s_cnt[d0]));
                    if (a1) st_relaxed_u64(&a.status[(size_t)t * kRadixMax + d1], tagp | kStInc | (unsigned long long)(e1 + s_cnt[d1]));
                }
                if (a0) s_gb[d0] = a.gbase[((size_t)sg * kMaxPass + p) * kRadixMax + d0] + e0;
                if (a1) s_gb[d1] = a.gbase[((size_t)sg * kMaxPass + p) * kRadixMax + d1] + e1;
            }
            __syncthreads();
            PDNN_OSTAMP(4)
            // 6. reorder the tile by digit in shared memory
#pragma unroll
            for (int j = 0; j < kSortPer; ++j) {
                const int d = dig[j];
                if (d < 0) continue;
                const uint32_t pos = s_loff[d] + wc[d] + rk[j];
                s_key[pos] = key[j];
                if (!packed) s_val[pos] = val[j];
            }
            __syncthreads();
            PDNN_OSTAMP(5)
            // 7. write the digit runs out contiguously
            for (int i = tid; i < n_valid; i += kSortThreads) {
                const uint64_t k = s_key[i];
                const int d = (int)(((packed ? (k >> a.rb) : k) >> (dbits * p)) & dmask);
                const uint32_t dst = s_gb[d] + (uint32_t)i - s_loff[d];
                if (last) {
                    const uint32_t r = packed ? (uint32_t)(k & rmask) : s_val[i];
                    a.pp[so + r] = (dst << 5) | (uint32_t)a.pe8[so + r];   // fused position pass
                } else {
                    kd[so + dst] = k;
                    if (!packed) vd[so + dst] = s_val[i];
                }
            }
            PDNN_OSTAMP(6)
            // 8. clear the per-warp counters for the next tile
            for (int c = tid; c < kSortWarps * radix; c += kSortThreads) s_wcnt[(c >> dbits) * kRadixMax + (c & (radix - 1))] = 0u;
            __syncthreads();
            tk = tkn;
        }
        grid.sync();
    }
    if (a.trace && tid == 0)
        for (int q = 0; q < 8; ++q) atomicAdd(&a.trace[q], (unsigned long long)tr[q]);
#undef PDNN_OSTAMP
    if (blockIdx.x == 0 && tid == 0) *a.epoch = ep0 + 1;
}

// Chunked LSD sort for few segments (S < kOneSweepMinSeg; the single-placement
// call).  One CTA per SM, each owning ONE contiguous chunk of ~V/G keys of the
// current order, so the scan over "all keys before mine" is a scan over G
// chunk histograms that every CTA does for itself.  Per pass, two grid
// barriers:
//   A  histogram of the chunk's digits  -> hist[digit][chunk]
//      -- barrier --
//   B  digit base of the chunk = (keys of smaller digits) + (same digit in
//      earlier chunks), read from the G-column histogram table; then the
//      chunk is ranked stably in sub-tiles of 8,192 keys (ballot peer masks
//      against per-warp counters + a scan over warps) and scattered
//      -- barrier --
// (the round-1 reduce-then-scan variant took four barriers per pass with
// fixed 4,096-key tiles that did not divide evenly over the grid: C4 sort
// 221 us, 40 % of it in grid.sync spins; profiles/r1_*)
constexpr int kChThreads = 512, kChWarps = kChThreads / 32, kChPer = 10;
constexpr int kChTile = kChThreads * kChPer;      // keys per sub-tile
constexpr int kChRadix = 256;                     // <= 8-bit digits
constexpr int kChSmem = (kChWarps * kChRadix + 3 * kChRadix) * 4;
constexpr int kChGrp = 16;                        // chunks per group sum: G <= 32 * 16

struct ChArgs {
    int32_t V;
    int32_t S;
    int32_t rb;       // rank bits = bits(V - 1)
    int32_t cs;       // keys per chunk (chunk c = [c*cs, min(V, (c+1)*cs)))
    uint64_t* k0;     // raw st on input (rank order)
    uint64_t* k1;
    uint32_t* v0;     // unpacked mode only
    uint32_t* v1;
    uint32_t* pp;     // output: pp[rank] = (pos << 5) | PE
    const uint8_t* pe8;
    uint32_t* hist;   // [kChRadix][G]
    const unsigned long long* maxst;
    unsigned long long* trace;   // PDNN_SORT_TRACE=1: per-phase globaltimer stamps of CTAs 0 and G-1 (diagnostic)
};

__device__ unsigned long long g_sort_trace[128];
__device__ unsigned long long g_scan_trace[4 * 4096];   // PDNN_SCAN_TRACE: per tile {start, local done, prefix known, end}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(kChThreads, 2) k_mem_sort_chunk(ChArgs a) {
    extern __shared__ uint32_t sm[];
    uint32_t* s_wcnt = sm;                            // [kChWarps][kChRadix] per-warp counters
    uint32_t* s_base = sm + kChWarps * kChRadix;      // [kChRadix] running global base of each digit
    uint32_t* s_pre = s_base + kChRadix;              // [kChRadix] same digit in earlier chunks
    uint32_t* s_tot = s_pre + kChRadix;               // [kChRadix] digit totals / sub-tile counts
    __shared__ uint32_t s_wsum[kChWarps];
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x, Gp = (G + 3) & ~3;   // Gp: padded row length of the table
    const int ng = (G + kChGrp - 1) / kChGrp;                     // chunk groups (<= 32)
    uint32_t* gs = a.hist + (size_t)kChRadix * Gp;                 // [3][kChRadix][ng] group sums (rotating)
    const unsigned long long mx = *a.maxst;
    const int nbits = mx ? 64 - __clzll((long long)mx) : 0;
    const bool packed = nbits + a.rb <= 64;
    const int npass = (nbits + 7) / 8;
    const int dbits = npass ? (nbits + npass - 1) / npass : 0;
    const int radix = 1 << dbits;
    const uint32_t dmask = (uint32_t)radix - 1u;
    const uint64_t rmask = (1ull << a.rb) - 1;
    if (npass == 0) {   // every st is 0: the visit order is the rank order
        const size_t tot = (size_t)a.S * a.V;
        for (size_t i = (size_t)blockIdx.x * kChThreads + tid; i < tot; i += (size_t)gridDim.x * kChThreads)
            a.pp[i] = ((uint32_t)(i % (size_t)a.V) << 5) | (uint32_t)a.pe8[i];
        return;
    }
    const int32_t lo = min(a.V, c * a.cs), hi = min(a.V, lo + a.cs);
    for (int i = tid; i < kChWarps * kChRadix; i += kChThreads) s_wcnt[i] = 0u;
    for (int sg = 0; sg < a.S; ++sg) {
        const size_t so = (size_t)sg * a.V;
        for (int p = 0; p < npass; ++p) {
            const int gpass = sg * npass + p;   // rotation index of the group-sum buffers
            const uint64_t* ks = (p & 1) ? a.k1 + so : a.k0 + so;
            const uint32_t* vs = (p & 1) ? a.v1 + so : a.v0 + so;
            uint64_t* kd = (p & 1) ? a.k0 + so : a.k1 + so;
            uint32_t* vd = (p & 1) ? a.v0 + so : a.v1 + so;
            const bool last = p == npass - 1;
            const int sh = dbits * p;
            // key / value / digit of element i (pass 0 packs the raw st with its rank)
            auto load = [&](int32_t i, uint64_t& k, uint32_t& v, int& d) {
                const bool valid = i < hi;
                k = valid ? ks[i] : 0ull;
                v = 0;
                if (valid) {
                    if (p == 0) {
                        v = (uint32_t)i;
                        if (packed) k = (k << a.rb) | (uint64_t)i;
                    } else if (!packed) {
                        v = vs[i];
                    }
                }
                d = valid ? (int)(((packed ? (k >> a.rb) : k) >> sh) & dmask) : -1;
            };
            if (a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) a.trace[(blockIdx.x ? 64 : 0) + p * 10 + 0] = gtimer();
            // ---- A: chunk histogram (smem atomics; conflicts within a warp are rare at <= 256 digits)
            // (accumulating the next pass's table in the scatter with one L2 atomic per
            // key was tried: skewed digits -- the 20 % parameter nodes all have st = 0 --
            // made it 3x slower)
            for (int d = tid; d < radix; d += kChThreads) s_tot[d] = 0u;
            __syncthreads();
            for (int32_t t0 = lo; t0 < hi; t0 += kChTile) {
#pragma unroll
                for (int j = 0; j < kChPer; ++j) {
                    uint64_t k;
                    uint32_t v;
                    int d;
                    load(t0 + warp * (32 * kChPer) + j * 32 + lane, k, v, d);
                    if (d >= 0) atomicAdd(&s_tot[d], 1u);
                }
            }
            __syncthreads();
            if (a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) a.trace[(blockIdx.x ? 64 : 0) + p * 10 + 1] = gtimer();
            for (int d = tid; d < radix; d += kChThreads) {
                const uint32_t x = s_tot[d];
                a.hist[(size_t)d * Gp + c] = x;
                if (x) atomicAdd(&gs[(size_t)(gpass % 3) * kChRadix * ng + (size_t)d * ng + c / kChGrp], x);
            }
            {   // the group sums of pass gpass + 1 (last read two passes ago) start from zero
                uint32_t* gz = gs + (size_t)((gpass + 1) % 3) * kChRadix * ng;
                for (int i = c * kChThreads + tid; i < kChRadix * ng; i += G * kChThreads) gz[i] = 0u;
            }
            grid.sync();
            if (a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) a.trace[(blockIdx.x ? 64 : 0) + p * 10 + 2] = gtimer();
            // ---- B1: digit bases of this chunk from the group sums (chunks of
            // earlier groups + the digit's total) and the earlier chunks of its own
            // group: two loads per lane per digit instead of a G-long row
            {
                const int grp = c / kChGrp, g0 = grp * kChGrp;
                const uint32_t* gsp = gs + (size_t)(gpass % 3) * kChRadix * ng;
#pragma unroll 4
                for (int d = warp; d < radix; d += kChWarps) {
                    const uint32_t x = lane < ng ? __ldcg(&gsp[(size_t)d * ng + lane]) : 0u;
                    const uint32_t y = g0 + lane < c ? __ldcg(&a.hist[(size_t)d * Gp + g0 + lane]) : 0u;
                    uint32_t tot = x, pre = (lane < grp ? x : 0u) + y;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        tot += __shfl_xor_sync(0xffffffffu, tot, o);
                        pre += __shfl_xor_sync(0xffffffffu, pre, o);
                    }
                    if (lane == 0) { s_pre[d] = pre; s_tot[d] = tot; }
                }
            }
            __syncthreads();
            if (warp == 0) {   // exclusive scan of the digit totals (<= 8 digits per lane)
                uint32_t x[kChRadix / 32], loc = 0;
#pragma unroll
                for (int q = 0; q < kChRadix / 32; ++q) {
                    const int d = lane * (kChRadix / 32) + q;
                    x[q] = d < radix ? s_tot[d] : 0u;
                    loc += x[q];
                }
                uint32_t incl = loc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                uint32_t run = incl - loc;
#pragma unroll
                for (int q = 0; q < kChRadix / 32; ++q) {
                    const int d = lane * (kChRadix / 32) + q;
                    if (d < radix) s_base[d] = run + s_pre[d];
                    run += x[q];
                }
            }
            __syncthreads();
            if (a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) a.trace[(blockIdx.x ? 64 : 0) + p * 10 + 3] = gtimer();
            // ---- B2: stable rank + scatter, sub-tile by sub-tile
            for (int32_t t0 = lo; t0 < hi; t0 += kChTile) {
                uint64_t key[kChPer];
                uint32_t val[kChPer], rk[kChPer];
                int dig[kChPer];
                uint32_t* wc = s_wcnt + warp * kChRadix;
#pragma unroll
                for (int j = 0; j < kChPer; ++j) load(t0 + warp * (32 * kChPer) + j * 32 + lane, key[j], val[j], dig[j]);
#pragma unroll
                for (int j = 0; j < kChPer; ++j) {
                    const int d = dig[j];
                    const unsigned m = peer_mask(d, dbits);
                    const uint32_t c0 = d >= 0 ? wc[d] : 0u;
                    __syncwarp();
                    if (d >= 0 && (m & ((1u << lane) - 1u)) == 0) wc[d] = c0 + (uint32_t)__popc(m);
                    __syncwarp();
                    rk[j] = c0 + (uint32_t)__popc(m & ((1u << lane) - 1u));
                }
                __syncthreads();
                if (a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) a.trace[(blockIdx.x ? 64 : 0) + p * 10 + 6] = gtimer();
                // exclusive scan over the warps for each digit: kChParts threads per digit
                {
                    constexpr int kChParts = kChThreads / kChRadix, kWp = kChWarps / kChParts;
                    const int d = tid / kChParts, part = tid % kChParts;
                    uint32_t cnt[kWp], loc = 0;
                    if (d < radix) {
#pragma unroll
                        for (int w = 0; w < kWp; ++w) { cnt[w] = s_wcnt[(part * kWp + w) * kChRadix + d]; loc += cnt[w]; }
                    }
                    uint32_t incl = loc;
#pragma unroll
                    for (int o = 1; o < kChParts; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o, kChParts);
                        if (part >= o) incl += y;
                    }
                    const uint32_t total = __shfl_sync(0xffffffffu, incl, kChParts - 1, kChParts);
                    if (d < radix) {
                        uint32_t run = incl - loc;
#pragma unroll
                        for (int w = 0; w < kWp; ++w) {
                            s_wcnt[(part * kWp + w) * kChRadix + d] = run;
                            run += cnt[w];
                        }
                        if (part == 0) s_tot[d] = total;
                    }
                }
                __syncthreads();
                if (a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) a.trace[(blockIdx.x ? 64 : 0) + p * 10 + 7] = gtimer();
#pragma unroll
                for (int j = 0; j < kChPer; ++j) {
                    const int d = dig[j];
                    if (d < 0) continue;
                    const uint32_t dst = s_base[d] + wc[d] + rk[j];
                    if (last) {
                        const uint32_t r = packed ? (uint32_t)(key[j] & rmask) : val[j];
                        a.pp[so + r] = (dst << 5) | (uint32_t)a.pe8[so + r];   // fused position pass
                    } else {
                        kd[dst] = key[j];
                        if (!packed) vd[dst] = val[j];
                    }
                }
                __syncthreads();
                if (a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) a.trace[(blockIdx.x ? 64 : 0) + p * 10 + 8] = gtimer();
                for (int d = tid; d < radix; d += kChThreads) s_base[d] += s_tot[d];
                for (int i = tid; i < kChWarps * radix; i += kChThreads) s_wcnt[(i / radix) * kChRadix + (i % radix)] = 0u;
                __syncthreads();
            }
            if (a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) a.trace[(blockIdx.x ? 64 : 0) + p * 10 + 4] = gtimer();
            grid.sync();
            if (a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) a.trace[(blockIdx.x ? 64 : 0) + p * 10 + 5] = gtimer();
        }
    }
    (void)s_wsum;
}

static int mem_sort_chunk_blocks_per_sm() { return kernel_occupancy((const void*)k_mem_sort_chunk, kChThreads, kChSmem); }
static int mem_sort_blocks_per_sm() { return kernel_occupancy((const void*)k_mem_sort, kSortThreads, kSortSmem); }

// ---------------------------------------------------------------- edges
// (positions: the sort's last pass writes pp[rank] = (pos << 5) | PE, so one
// 4-byte gather gives a successor's position and PE)
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
                                                   const uint32_t* __restrict__ pp_all,
                                                   const int32_t* __restrict__ orig,
                                                   const int64_t* __restrict__ mem,
                                                   const uint8_t* __restrict__ kind,
                                                   const int32_t* __restrict__ heavy, int32_t n_heavy,
                                                   unsigned long long* __restrict__ relp_all,
                                                   Rec* __restrict__ rec_all) {
    const size_t so = (size_t)blockIdx.y * V;
    const uint32_t* pp = pp_all + so;
    unsigned long long* relp = relp_all + so;
    Rec* rec = rec_all + so;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    for (int32_t r = tid; r < V; r += nth) {
        const int32_t s0 = out_off[r], s1 = out_off[r + 1];
        if (s1 - s0 > kMemHeavyDeg) continue;  // heavy: warp path below
        int32_t last[PT];
#pragma unroll
        for (int q = 0; q < PT; ++q) last[q] = -1;
        // successor ids, then their position words, in batches of 4 (most nodes
        // take one batch; 8-wide batches of predicated loads filled the LSU
        // queue: lg_throttle stalls)
        for (int32_t e0 = s0; e0 < s1; e0 += 4) {
            int32_t dv[4];
            uint32_t xv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) dv[k] = e0 + k < s1 ? __ldg(&out_dst[e0 + k]) : -1;
#pragma unroll
            for (int k = 0; k < 4; ++k) xv[k] = dv[k] >= 0 ? pp[dv[k]] : 0xffffffffu;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (dv[k] < 0) break;
                const int32_t q = (int32_t)(xv[k] & 31u), p = (int32_t)(xv[k] >> 5);
#pragma unroll
                for (int j = 0; j < PT; ++j) last[j] = (j == q && p > last[j]) ? p : last[j];
            }
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

__device__ __forceinline__ void merge_res(long long& pk, int32_t& pp, int32_t& fo, long long& fv, long long v2,
                                          int32_t p2, int32_t f2, long long fv2) {
    if (p2 >= 0 && (pp < 0 || v2 > pk || (v2 == pk && p2 < pp))) { pk = v2; pp = p2; }
    if (f2 >= 0 && (fo < 0 || f2 < fo)) { fo = f2; fv = fv2; }
}

// ---------------------------------------------------------------- scan
// ONE single-pass launch per tracker call (all S segments): a CTA takes the
// next tile of 2,048 positions by ticket, computes its per-PE delta sums,
// publishes them, and finds its exclusive per-PE prefix by decoupled
// look-back over the preceding tiles of its segment (warp q serves PE q:
// 32 predecessors per round trip, the nearest inclusive prefix found by
// ballot).  It then emits M_cons / M_pot and the tile's peak and first
// overflow; the last tile of a segment to finish reduces the per-tile
// results into the per-PE outputs.  (Round 1 ran tile sums -> tile scan ->
// tile final -> final reduce: four launches and two reads of the records,
// 97 us on C4.)
//
// Look-back words: (value mod 2^62) | flag << 62 (flag 1 = tile aggregate,
// 2 = inclusive prefix); values are 62-bit two's complement (a tile's
// aggregate is negative when it releases more than it acquires; |M_cons| <
// 2^61 by the cost precondition), zeroed per call together with the tickets.
constexpr unsigned long long kLbAgg = 1ull << 62, kLbInc = 2ull << 62, kLbVal = (1ull << 62) - 1;

// Thread layout of the scan: thread t serves PE q = t % PT over a run of RL
// consecutive positions (run t / PT).  The PT threads of a run read the same
// staged record (a shared-memory broadcast), and each keeps its own PE's
// running sum and candidates in registers, so no per-position work is
// indexed by a data-dependent PE.  (The previous layout -- one thread per run,
// all PEs' sums in shared memory indexed by the hold-mask bits -- spent 16 us
// of a 28 us tile in dependent shared-memory read-modify-writes.)
template <int PT>
struct ScanSmem {
    static constexpr int NR = kMemThreads / PT;     // runs per tile
    static constexpr int RL = kMemTile / NR;        // positions per run
    Rec rec[kMemTile + NR];                         // one pad per run: runs start on different banks
    unsigned long long rel[kMemTile + NR];
#ifndef PDNN_SCAN_UNION
#define PDNN_SCAN_UNION 0   // 1: 4 tiles per SM -- measured slower (C4 tracker 284 vs 271 us; 2 per SM: 279)
#endif
#if PDNN_SCAN_UNION
    union {                                         // (pk is written by a thread after it last reads its
        long long sum[PT][NR];                      //  own sum: sharing the space keeps the tile under
        long long pk[PT][NR];                       //  56 KB, 4 CTAs per SM instead of 3)
    };
#else
    long long sum[PT][NR];
    long long pk[PT][NR];
#endif
    long long fov[PT][NR];
    int32_t pkp[PT][NR];
    int32_t fo[PT][NR];
    long long pref[PT];   // the tile's exclusive prefix per PE
    long long agg[PT];    // the tile's aggregate per PE
    int32_t tile, seg;
    int32_t last;
};

struct ScanArgs {
    int32_t V, P, S, n_tiles;
    const Rec* rec_all;
    const unsigned long long* relp_all;
    const unsigned long long* base_all;   // [S][PDNN_MAX_PE] residual bases (Eq. 3 term 1)
    const int64_t* cap_eff;
    int64_t* mpot;                        // node-id order (S == 1) or nullptr
    int64_t* mcons;                       // [P][V] or nullptr (S == 1)
    unsigned long long* lb;               // [S][n_tiles][PT] look-back words (zeroed)
    TileRes* tres;                        // [S][n_tiles][PT]
    unsigned long long* trace;            // diagnostic (PDNN_SCAN_TRACE=1) or nullptr
    uint32_t* ctr;                        // [0] ticket, [1 + sg] tiles done (zeroed)
    MemOut o;
};

static_assert(!PDNN_SCAN_UNION || sizeof(ScanSmem<8>) <= 56 * 1024, "4 scan tiles per SM (P <= 8)");

template <int PT>
__global__ void __launch_bounds__(kMemThreads) k_mem_scan(ScanArgs a) {
    using SM = ScanSmem<PT>;
    constexpr int NR = SM::NR, RL = SM::RL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SM& sh = *reinterpret_cast<SM*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = tid % PT, run = tid / PT;
    if (tid == 0) {
        const uint32_t t = atomicAdd(&a.ctr[0], 1u);
        // tickets interleave the segments: a tile's predecessor in its segment
        // was ticketed S tickets earlier, so its look-back usually finds an
        // inclusive prefix at once (tiles of one segment are in order)
        sh.seg = (int32_t)(t % (uint32_t)a.S);
        sh.tile = (int32_t)(t / (uint32_t)a.S);
    }
    __syncthreads();
    const int sg = sh.seg, tile = sh.tile;
    if (a.trace && tid == 0 && sg == 0 && tile < 4096) a.trace[4 * tile + 0] = gtimer();
    const size_t so = (size_t)sg * a.V;
    const Rec* rec = a.rec_all + so;
    const unsigned long long* relp = a.relp_all + so;
    unsigned long long* lb = a.lb + (size_t)sg * a.n_tiles * PT;
    const int32_t t0 = tile * kMemTile;
    // 0. stage the tile's records and releases (coalesced, all loads in flight)
#pragma unroll
    for (int k = 0; k < kMemTile / kMemThreads; ++k) {
        const int p = k * kMemThreads + tid;
        if (t0 + p < a.V) {
            sh.rec[p + p / RL] = rec[t0 + p];
            sh.rel[p + p / RL] = relp[t0 + p];
        }
    }
    __syncthreads();
    const int32_t i0 = t0 + run * RL, i1 = min(a.V, i0 + RL);
    const Rec* srec = sh.rec + run * (RL + 1);
    const unsigned long long* srel = sh.rel + run * (RL + 1);
    const bool on = q < a.P;
    // 1. the run's delta sum D(q) = sum of acquisitions on q - releases on q
    long long d = 0;
    if (on)
#pragma unroll 8
        for (int32_t i = i0; i < i1; ++i) {
            const Rec x = srec[i - i0];
            const int h = (x.meta >> 16) & 0x1f;
            d += ((x.meta >> q) & 1) ? x.eff : 0;
            if (h == q) d -= (long long)srel[i - i0] + ((x.meta >> 24) & 1 ? x.eff : 0);
        }
    sh.sum[q][run] = d;
    __syncthreads();
    // 2. exclusive scan over the runs of each PE (warp w: PEs w, w + 8; lane l: runs l*R .. l*R + R - 1)
    constexpr int R = (NR + 31) / 32;
    for (int qq = warp; qq < PT; qq += kMemThreads / 32) {
        long long x[R], loc = 0;
#pragma unroll
        for (int k = 0; k < R; ++k) { const int r = lane * R + k; x[k] = r < NR ? sh.sum[qq][r] : 0; loc += x[k]; }
        long long incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        long long rs = incl - loc;
#pragma unroll
        for (int k = 0; k < R; ++k) { const int r = lane * R + k; if (r < NR) sh.sum[qq][r] = rs; rs += x[k]; }
        const long long agg = __shfl_sync(0xffffffffu, incl, 31);
        if (lane == 0) {
            sh.agg[qq] = agg;
            if (tile == 0) {
                const long long b = (long long)a.base_all[(size_t)sg * PDNN_MAX_PE + qq];
                sh.pref[qq] = b;
                st_relaxed_u64(reinterpret_cast<uint64_t*>(&lb[qq]), kLbInc | ((unsigned long long)(b + agg) & kLbVal));
            } else {
                st_relaxed_u64(reinterpret_cast<uint64_t*>(&lb[(size_t)tile * PT + qq]), kLbAgg | ((unsigned long long)agg & kLbVal));
            }
        }
    }
    if (a.trace && tid == 0 && sg == 0 && tile < 4096) a.trace[4 * tile + 1] = gtimer();
    // 3. decoupled look-back (warp q, 32 predecessors per round trip)
    if (tile > 0) {
        for (int qq = warp; qq < PT; qq += kMemThreads / 32) {
            long long excl = 0;
            int32_t j0 = tile - 1;   // window: tiles j0, j0 - 1, ..., j0 - 31
            for (;;) {
                const int32_t j = j0 - lane;
                // tiles before 0 read as an inclusive zero
                unsigned long long w =
                    j >= 0 ? ld_relaxed_u64(reinterpret_cast<const uint64_t*>(&lb[(size_t)j * PT + qq])) : kLbInc;
                while (__any_sync(0xffffffffu, (w >> 62) == 0)) {   // until every tile of the window has published
                    if ((w >> 62) == 0) w = ld_relaxed_u64(reinterpret_cast<const uint64_t*>(&lb[(size_t)j * PT + qq]));
                }
                const unsigned inc = __ballot_sync(0xffffffffu, (w & kLbInc) != 0);
                const int stop = inc ? __ffs(inc) - 1 : 31;   // nearest inclusive prefix in the window
                long long v = lane <= stop ? (long long)(w << 2) >> 2 : 0;   // 62-bit two's complement
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                excl += v;
                if (inc) break;
                j0 -= 32;
            }
            if (lane == 0) {
                sh.pref[qq] = excl;
                st_relaxed_u64(reinterpret_cast<uint64_t*>(&lb[(size_t)tile * PT + qq]),
                               kLbInc | ((unsigned long long)(excl + sh.agg[qq]) & kLbVal));
            }
        }
    }
    __syncthreads();
    if (a.trace && tid == 0 && sg == 0 && tile < 4096) a.trace[4 * tile + 2] = gtimer();
    // 4. the run again with its prefix: M_cons candidates (acquisitions; position 0),
    //    the optional M_cons row, and M_pot by the home PE's thread
    long long pk = 0, fov = 0;
    int32_t pkp = -1, fo = -1;
    if (on) {
        long long runv = sh.pref[q] + sh.sum[q][run];
        const long long cap = a.cap_eff[q];
#pragma unroll 8
        for (int32_t i = i0; i < i1; ++i) {
            const Rec x = srec[i - i0];
            const int h = (x.meta >> 16) & 0x1f;
            const bool acq = (x.meta >> q) & 1;
            const long long val = runv + (acq ? x.eff : 0);
            if (a.mcons) a.mcons[(size_t)q * a.V + i] = val;
            if ((acq && x.eff > 0) || i == 0) {   // the only places a new max / overflow can start
                if (pkp < 0 || val > pk) { pk = val; pkp = i; }
                if (fo < 0 && val > cap) { fo = i; fov = val; }
            }
            runv += acq ? x.eff : 0;
            if (h == q) {
                const long long rel = (long long)srel[i - i0];
                runv -= rel + ((x.meta >> 24) & 1 ? x.eff : 0);
                if (a.mpot) a.mpot[x.n] = x.eff + rel;   // M7: own output + released predecessors
            }
        }
    }
    sh.pk[q][run] = pk; sh.pkp[q][run] = pkp; sh.fo[q][run] = fo; sh.fov[q][run] = fov;
    __syncthreads();
    // 5. tile reduction per PE (warp w: PEs w, w + 8): max (lowest position on ties), first overflow
    TileRes* tres = a.tres + (size_t)sg * a.n_tiles * PT;
    for (int qq = warp; qq < PT; qq += kMemThreads / 32) {
        long long bp = 0, bf = 0;
        int32_t bpp = -1, bfo = -1;
        for (int r = lane; r < NR; r += 32) merge_res(bp, bpp, bfo, bf, sh.pk[qq][r], sh.pkp[qq][r], sh.fo[qq][r], sh.fov[qq][r]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            merge_res(bp, bpp, bfo, bf, __shfl_xor_sync(0xffffffffu, bp, o), __shfl_xor_sync(0xffffffffu, bpp, o),
                      __shfl_xor_sync(0xffffffffu, bfo, o), __shfl_xor_sync(0xffffffffu, bf, o));
        if (lane == 0) tres[(size_t)tile * PT + qq] = TileRes{bp, bpp, bfo, bf};
    }
    if (a.trace && tid == 0 && sg == 0 && tile < 4096) a.trace[4 * tile + 3] = gtimer();
    // 6. the segment's last tile to finish reduces all its tiles
    __syncthreads();
    if (tid == 0) {
        __threadfence();   // cumulative: the CTA's tres writes (ordered by the barrier) before the count
        sh.last = atomicAdd(&a.ctr[1 + sg], 1u) == (uint32_t)a.n_tiles - 1;
    }
    __syncthreads();
    if (!sh.last) return;
    __threadfence();
    for (int qq = warp; qq < a.P; qq += kMemThreads / 32) {
        long long bp = 0, bf = 0;
        int32_t bpp = -1, bfo = -1;
        for (int t = lane; t < a.n_tiles; t += 32) {
            const TileRes* up = &tres[(size_t)t * PT + qq];   // written by other CTAs: read through L2
            const TileRes u{__ldcg(&up->peak), __ldcg(&up->peak_pos), __ldcg(&up->first_over), __ldcg(&up->over_val)};
            merge_res(bp, bpp, bfo, bf, u.peak, u.peak_pos, u.first_over, u.over_val);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            merge_res(bp, bpp, bfo, bf, __shfl_xor_sync(0xffffffffu, bp, o), __shfl_xor_sync(0xffffffffu, bpp, o),
                      __shfl_xor_sync(0xffffffffu, bfo, o), __shfl_xor_sync(0xffffffffu, bf, o));
        if (lane == 0) {
            const size_t s64 = (size_t)sg * a.o.stride64, s32 = (size_t)sg * a.o.stride32;
            a.o.peak[s64 + qq] = bp;
            a.o.peak_pos[s32 + qq] = bpp;
            a.o.first_over[s32 + qq] = bfo;
            a.o.over_bytes[s64 + qq] = bfo >= 0 ? bf - a.cap_eff[qq] : 0;
        }
    }
}

__global__ void k_mem_empty(int32_t P, MemOut o) {
    const int q = threadIdx.x;
    const size_t s64 = (size_t)blockIdx.x * o.stride64, s32 = (size_t)blockIdx.x * o.stride32;
    if (q < P) { o.peak[s64 + q] = 0; o.peak_pos[s32 + q] = -1; o.first_over[s32 + q] = -1; o.over_bytes[s64 + q] = 0; }
}

template <int PT>
static pdnn_status mem_scan(const pdnn_graph* g, int32_t P, int32_t S, const int64_t* mem, const uint8_t* kind,
                            const int64_t* cap_eff, int64_t* mpot, const MemOut& o, int64_t* mcons,
                            const MemWs& M, cudaStream_t s) {
    const int32_t V = g->V;
    // edge pass grid: up to 64 CTAs per SM over the segments (one node per thread on C4):
    // C4 48.0 -> 45.7 us, C5 x 4096 200.6 -> 190.1 ms (8 / 16 / 32 / 64 per SM measured)
    const int edg_bpsm = debug_knob("PDNN_EDGES_BPSM", 64);
    const int grid = std::min(ceil_div(V, 256), std::max(1, g->num_sms * edg_bpsm / S));
    k_mem_edges<PT><<<dim3(grid, S), 256, 0, s>>>(V, g->out_off, g->out_dst, M.pp, g->orig, mem, kind, g->heavy_out,
                                                  g->n_heavy_out, M.relp, reinterpret_cast<Rec*>(M.rec));
    const int tiles = ceil_div(V, kMemTile);
    ScanArgs sa;
    sa.V = V;
    sa.P = P;
    sa.S = S;
    sa.n_tiles = tiles;
    sa.rec_all = reinterpret_cast<const Rec*>(M.rec);
    sa.relp_all = M.relp;
    sa.base_all = M.base;
    sa.cap_eff = cap_eff;
    sa.mpot = mpot;
    sa.mcons = mcons;
    sa.lb = reinterpret_cast<unsigned long long*>(M.tsum);
    sa.tres = M.tres;
    sa.ctr = M.ctr;
    sa.trace = nullptr;
    if (debug_knob("PDNN_SCAN_TRACE", 0)) cudaGetSymbolAddress((void**)&sa.trace, g_scan_trace);
    sa.o = o;
    PDNN_CUDA_TRY(cudaMemsetAsync(sa.lb, 0, 8 * (size_t)S * tiles * PT, s));
    PDNN_CUDA_TRY(cudaMemsetAsync(sa.ctr, 0, 4 * (size_t)(S + 1), s));
    constexpr int smem = (int)sizeof(ScanSmem<PT>);
    kernel_occupancy((const void*)k_mem_scan<PT>, kMemThreads, smem);   // sets the smem attribute on this device
    k_mem_scan<PT><<<tiles * S, kMemThreads, smem, s>>>(sa);
    count_launch(2);
    PDNN_LAUNCH_CHECK();
    return PDNN_OK;
}

// the whole tracker for S segments (S = 1: a single placement)
pdnn_status launch_memory_seg(const pdnn_graph* g, const MemIn& in, int32_t P, int32_t S, const int64_t* mem,
                              const uint8_t* kind, const int64_t* cap_eff, int64_t* mpot, const MemOut& o,
                              int64_t* mcons, const MemWs& M, cudaStream_t s) {
    const int32_t V = g->V;
    if (V == 0) {
        k_mem_empty<<<S, 32, 0, s>>>(P, o);
        count_launch();
        PDNN_LAUNCH_CHECK();
        return PDNN_OK;
    }
    PDNN_CUDA_TRY(cudaMemsetAsync(M.base, 0, 8 * ((size_t)S * PDNN_MAX_PE + 1), s));
    PDNN_CUDA_TRY(cudaMemsetAsync(M.relp, 0, 8 * (size_t)S * V, s));
    PrepArgs pa;
    pa.V = V;
    pa.orig = g->orig;
    pa.part_i32_orig = in.part_i32_orig;
    pa.part_i32_rank = in.part_i32_rank;
    pa.part_u8_rank = in.part_u8_rank;
    pa.st_orig = in.st_orig;
    pa.st_rank = in.st_rank;
    pa.mem = mem;
    pa.kind = kind;
    pa.keys = M.k0;
    pa.pe8 = M.pe8;
    pa.base = M.base;
    pa.maxst = M.base + (size_t)S * PDNN_MAX_PE;
    // single placement: 2 CTAs per SM, each thread ~20 ranks, so the per-warp
    // residual-base reductions amortise (C4 24.6 -> 19.4 us; 8 / 4 / 1 per SM
    // measured 24.6 / 23.2 / 31.2 us); segmented: 8 per SM over the segments
    const int prep_seg_bpsm = debug_knob("PDNN_PREP_SEG_BPSM", 8);
    const int grid = std::min(ceil_div(V, 256), std::max(1, S == 1 ? g->num_sms * 2 : g->num_sms * prep_seg_bpsm / S));
    k_mem_prep<<<dim3(grid, S), 256, 0, s>>>(pa);
    count_launch();
    PDNN_LAUNCH_CHECK();
    // visit order: stable sort of st over level order == sort by (st, level, id)
    if (S >= kOneSweepMinSeg) {
        SortArgs sa;
        const int sort_bpsm = mem_sort_blocks_per_sm();
        const int max_grid = sort_bpsm * g->num_sms;
        sa.V = V;
        sa.S = S;
        sa.tps = ceil_div(V, kSortTile);
        sa.rb = bits_for((uint64_t)std::max(V - 1, 1));
        sa.k0 = M.k0;
        sa.k1 = M.k1;
        sa.v0 = M.v0;
        sa.v1 = M.v1;
        sa.pp = M.pp;
        sa.pe8 = M.pe8;
        sa.gbase = M.hist;
        sa.status = reinterpret_cast<uint64_t*>(M.sort_status);
        sa.ticket = M.dtot;
        sa.epoch = reinterpret_cast<unsigned long long*>(M.dtot + 16);
        sa.maxst = pa.maxst;
        sa.trace = nullptr;
        if (debug_knob("PDNN_SORT_TRACE", 0)) cudaGetSymbolAddress((void**)&sa.trace, g_osort_trace);
        PDNN_CUDA_TRY(cudaMemsetAsync(M.hist, 0, 4 * (size_t)S * kMaxPass * kRadixMax, s));
        PDNN_CUDA_TRY(cudaMemsetAsync(M.dtot, 0, 4 * 16, s));
        const int sgrid = std::max(1, std::min(sa.tps * S, max_grid));
        void* args[] = {(void*)&sa};
        PDNN_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_mem_sort, dim3(sgrid), dim3(kSortThreads), args, kSortSmem, s));
    } else {
        ChArgs ca;
        const int ch_bpsm = std::max(1, std::min(mem_sort_chunk_blocks_per_sm(), debug_knob("PDNN_CH_BPSM", 2)));
        // one chunk per CTA; >= 2,048 keys per chunk (the barrier, not the chunk, dominates below that)
        const int G = std::max(1, std::min({ch_bpsm * g->num_sms, ceil_div(V, 2048), 32 * kChGrp}));
        ca.V = V;
        ca.S = S;
        ca.rb = bits_for((uint64_t)std::max(V - 1, 1));
        ca.cs = ceil_div(V, G);
        ca.k0 = M.k0;
        ca.k1 = M.k1;
        ca.v0 = M.v0;
        ca.v1 = M.v1;
        ca.pp = M.pp;
        ca.pe8 = M.pe8;
        ca.hist = reinterpret_cast<uint32_t*>(M.sort_status);   // [256][G] counts
        ca.maxst = pa.maxst;
        // the first pass's group sums start from zero (later ones are cleared in the kernel)
        PDNN_CUDA_TRY(cudaMemsetAsync(ca.hist + (size_t)kChRadix * ((G + 3) & ~3), 0,
                                      4 * (size_t)kChRadix * ceil_div(G, kChGrp), s));
        unsigned long long* tr = nullptr;
        if (debug_knob("PDNN_SORT_TRACE", 0)) cudaGetSymbolAddress((void**)&tr, g_sort_trace);
        ca.trace = tr;   // diagnostic only
        void* args[] = {(void*)&ca};
        PDNN_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_mem_sort_chunk, dim3(G), dim3(kChThreads), args, kChSmem, s));
    }
    count_launch();
    PDNN_LAUNCH_CHECK();
    if (P <= 2) return mem_scan<2>(g, P, S, mem, kind, cap_eff, mpot, o, mcons, M, s);
    if (P <= 4) return mem_scan<4>(g, P, S, mem, kind, cap_eff, mpot, o, mcons, M, s);
    if (P <= 8) return mem_scan<8>(g, P, S, mem, kind, cap_eff, mpot, o, mcons, M, s);
    return mem_scan<16>(g, P, S, mem, kind, cap_eff, mpot, o, mcons, M, s);
}

pdnn_status launch_memory(const pdnn_graph* g, const int32_t* part_orig, const int32_t* part_rank_in,
                          int32_t P, const int64_t* mem, const uint8_t* kind, const int64_t* st,
                          const int64_t* cap_eff, int64_t* mpot, int64_t* peak, int32_t* peak_pos,
                          int32_t* first_over, int64_t* over_bytes, int64_t* mcons, void* ws,
                          const WsLayout& L, cudaStream_t s, bool st_rank) {
    MemIn in{};
    in.part_i32_orig = part_rank_in ? nullptr : part_orig;
    in.part_i32_rank = part_rank_in;
    in.st_orig = st_rank ? nullptr : st;
    in.st_rank = st_rank ? st : nullptr;
    MemOut o{peak, peak_pos, first_over, over_bytes, 0, 0};
    return launch_memory_seg(g, in, P, 1, mem, kind, cap_eff, mpot, o, mcons, mem_ws(ws, L), s);
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
        (g->V > 0 && (!part || !mem || !kind || !mpot))) {
        set_error("null argument");
        return PDNN_EINVAL;
    }
    // the tracker's sort packs a visit position as (pos << 5) | PE in 32 bits
    if (g->V >= (1 << 27)) { set_error("the memory tracker needs n_nodes < 2^27"); return PDNN_EINVAL; }
    const WsLayout L = ws_layout(g, PDNN_OP_MEMORY, 0);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    pdnn_status gs = ws_guard(ws, 0, 0, L.single_end, L.sig_single, s);
    if (gs) return gs;
    if (!st && g->V > 0) {
        // default schedule (reading R8): st = tl under the same placement, from
        // a placement-aware sweep with the bound costs
        Costs C;
        if ((gs = resolve_costs(g, nullptr, nullptr, ws, L, s, &C, /*need_blob=*/true))) return gs;
        int32_t* pr = ws_ptr<int32_t>(ws, L.part_rank);
        int64_t* tl = ws_ptr<int64_t>(ws, L.tl_o);
        if ((gs = launch_labels(g, part, nullptr, 0, nullptr, pr, s))) return gs;
        if ((gs = launch_sweep(g, C, pr, tl, ws_ptr<int64_t>(ws, L.bl_o), ws, L, s))) return gs;
        st = tl;
    }
    return launch_memory(g, part, nullptr, n_pe, mem, kind, st, cap_eff, mpot, peak, peak_pos, first_over_pos,
                         over_bytes, mcons, ws, L, s);
}

// diagnostic (PDNN_SORT_TRACE=1): the chunked sort's per-phase timestamps of its last launch
extern "C" int pdnn_debug_sort_trace(unsigned long long* host128) {
    return (int)cudaMemcpyFromSymbol(host128, g_sort_trace, sizeof(g_sort_trace));
}
extern "C" int pdnn_debug_scan_trace(unsigned long long* host16k) {
    return (int)cudaMemcpyFromSymbol(host16k, g_scan_trace, sizeof(g_scan_trace));
}
extern "C" int pdnn_debug_osort_trace(unsigned long long* host16) {
    return (int)cudaMemcpyFromSymbol(host16, g_osort_trace, sizeof(g_osort_trace));
}
