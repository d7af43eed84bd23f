// bsweep.cu -- candidate-parallel weighted-level sweep for batched evaluation
// (§8(a) row a8: refinement / LALB trials).
//
// Same definitions as the single-graph sweep (Table 2):
//   tl(v) = max(0, max_{p in pred(v)} tl(p) + comp(p) + comm'(p,v))
//   bl(u) = comp(u) + max(0, max_{s in succ(u)} comm'(u,s) + bl(s))
// with comm'(u,v) = 0 iff part_b[u] == part_b[v]; every node is alive (batch
// labels are PE ids).  Many candidate placements share one DAG, so the work
// is laid out candidate-minor: a warp processes one node (or a group of
// nodes, one after another) for 32 candidates at once, lane = candidate.  Every
// neighbour gather is then a contiguous 256-byte row (32 x int64) plus a
// 32-byte label row, the neighbour ids and edge costs are warp-uniform, and
// the dependency latency of the DAG is paid once per 32 candidates.
//
// Scheduling: the same dataflow scheme as sweep.cu -- a persistent cooperative
// launch, items in an order where each depends only on smaller indices,
// per-value readiness carried by an epoch tag in bits 62-63 of each record.
// The item index is (node item i, chunk k) -> i * nck + k; with the warp count
// a multiple of nck, warp w always serves chunk w % nck, so its per-candidate
// reductions (entry-node argmax for the CP start, cut communication, max st)
// stay in registers and are flushed once into per-warp slots.
//
// Outputs per chunk: tagged tl+comp and bl records, the bl-tight successor
// nxt (lowest original id, R5) for the CP walk, and the sort keys
// st = tl of the memory tracker in candidate-major rank order.
#include <cstdlib>

#include "internal.cuh"

namespace pdnn {

struct BSweepArgs {
    const Item* items;
    int32_t n_items;
    int32_t nck;          // chunks of 32 candidates in this launch
    int32_t V;
    int32_t n_entry;
    const int32_t* in_off;
    const int32_t* in_src;
    const int32_t* out_off;
    const int32_t* out_dst;
    const int32_t* orig;
    const int64_t* c;
    const int64_t* in_cost;
    const int64_t* out_cost;
    const int32_t* hub_pbase;
    int32_t n_parts;
    int32_t n_hubs;
    const uint8_t* lab;   // [nck][V][32]
    uint64_t* tlr;        // [nck][V][32] tagged tl + comp
    uint64_t* blr;        // [nck][V][32] tagged bl
    int32_t* nxt;         // [nck][V][32] rank of the tight successor, -1 at exits
    int64_t* keys;        // [nck*32][V] st = tl, rank order
    uint8_t* plab;        // [nck*32][V] labels, candidate-major rank order (memory tracker)
    unsigned long long* part_val;  // [nck][n_parts][32]
    int32_t* part_idx;             // [nck][n_parts][32]
    int32_t* hub_cnt;              // [nck][n_hubs]
    BSlot* slots;                  // [n_warps][32]
    WsHeader* hdr;
    int32_t sleep_ns;              // poll back-off: > 0 fixed, < 0 exponential up to -sleep_ns
};

__device__ __forceinline__ void poll_backoff(int32_t cfg, int32_t& ns) {
    if (cfg == 0) return;
    if (ns > 0) __nanosleep(ns);
    ns = cfg > 0 ? cfg : (ns == 0 ? 32 : (ns < -cfg ? 2 * ns : ns));
}

__device__ __forceinline__ uint32_t lab_word(const uint32_t (&lw)[kBMaxNodes / 4], int j) {
    // label words of the item's node rows: row j (32 bytes) = words [8j, 8j+8)
    // held by lanes 8(j%4) .. 8(j%4)+7 in register j/4
    uint32_t w = lw[0];
#pragma unroll
    for (int q = 1; q < kBMaxNodes / 4; ++q) w = (j >> 2) == q ? lw[q] : w;
    return w;
}
__device__ __forceinline__ int node_label(const uint32_t (&lw)[kBMaxNodes / 4], int j, int lane) {
    const uint32_t w = __shfl_sync(0xffffffffu, lab_word(lw, j), 8 * (j & 3) + (lane >> 2));
    return (int)((w >> (8 * (lane & 3))) & 0xffu);
}

struct BAcc {   // per-lane running reductions of a warp (its chunk is fixed)
    int64_t Lb;   // max bl over entry nodes seen
    int32_t Lo, Lr;  // lowest original id / rank attaining it
    int64_t cut;
    int64_t maxst;
};

template <bool FWD>
__device__ __forceinline__ void finalize_node(const BSweepArgs& a, int k, int lane, uint64_t tag, int32_t v,
                                              int64_t cv, int32_t ov, int pv, int64_t best, int32_t bu, BAcc& acc) {
    const size_t row = ((size_t)k * a.V + v) * 32 + lane;
    if (FWD) {
        st_relaxed_u64(&a.tlr[row], tag | (uint64_t)(best + cv));
        a.keys[((size_t)k * 32 + lane) * a.V + v] = best;
        a.plab[((size_t)k * 32 + lane) * a.V + v] = (uint8_t)pv;
        acc.maxst = best > acc.maxst ? best : acc.maxst;
    } else {
        const int64_t b = cv + (best > 0 ? best : 0);
        a.nxt[row] = bu;
        st_relaxed_u64(&a.blr[row], tag | (uint64_t)b);
        if (v < a.n_entry && (b > acc.Lb || (b == acc.Lb && ov < acc.Lo))) {
            acc.Lb = b;
            acc.Lo = ov;
            acc.Lr = v;
        }
    }
}

// relax one batch of <= 8 edges [e0, e1) of ONE node (warp items / hub parts)
template <bool FWD>
__device__ __forceinline__ void relax_node_batch(const BSweepArgs& a, int k, int lane, uint64_t tag,
                                                 const int32_t* nbr, const int64_t* ec, int32_t e0, int32_t e1,
                                                 int pv, int64_t& best, int32_t& bu, int32_t& bo, int64_t& cut) {
    const uint64_t* rec = (FWD ? a.tlr : a.blr) + (size_t)k * a.V * 32 + lane;
    const uint8_t* lab = a.lab + (size_t)k * a.V * 32 + lane;
    const int32_t ne = e1 - e0;
    int32_t nb_l = 0, no_l = 0;
    int64_t w_l = 0;
    if (lane < ne) {
        nb_l = __ldg(&nbr[e0 + lane]);
        w_l = __ldg(&ec[e0 + lane]);
        if (!FWD) no_l = __ldg(&a.orig[nb_l]);
    }
    uint64_t x[8];
    uint32_t lb[8];
    bool rdy[8];
    int32_t uq[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) uq[q] = __shfl_sync(0xffffffffu, nb_l, q);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        x[q] = 0;
        lb[q] = 0;
        ld_relaxed_u64_if(x[q], &rec[(size_t)uq[q] * 32], q < ne);
        ldg_u8_if(lb[q], &lab[(size_t)uq[q] * 32], q < ne);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) rdy[q] = q >= ne || (x[q] & ~kValMask) == tag;
    bool all = true;
#pragma unroll
    for (int q = 0; q < 8; ++q) all = all && rdy[q];
    int32_t ns = 0;
    while (!__all_sync(0xffffffffu, all)) {
        poll_backoff(a.sleep_ns, ns);
        all = true;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            ld_relaxed_u64_if(x[q], &rec[(size_t)uq[q] * 32], !rdy[q]);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            rdy[q] = rdy[q] || (x[q] & ~kValMask) == tag;
            all = all && rdy[q];
        }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int64_t w = __shfl_sync(0xffffffffu, w_l, q);
        const int32_t u = uq[q];
        const int32_t o = __shfl_sync(0xffffffffu, no_l, q);
        if (q < ne) {
            const int64_t cm = (int)lb[q] == pv ? 0 : w;
            const int64_t y = (int64_t)(x[q] & kValMask) + cm;
            if (FWD) {
                best = y > best ? y : best;
            } else {
                if (y > best || (y == best && o < bo)) { best = y; bo = o; bu = u; }
                cut += cm;
            }
        }
    }
}

template <bool FWD>
__device__ __forceinline__ void process_item(const BSweepArgs& a, const Item& it, int k, int lane, uint64_t tag,
                                             BAcc& acc) {
    const int32_t r0 = FWD ? it.x : ~it.x;
    const int32_t* off = FWD ? a.in_off : a.out_off;
    const int32_t* nbr = FWD ? a.in_src : a.out_dst;
    const int64_t* ec = FWD ? a.in_cost : a.out_cost;
    const uint8_t* labk = a.lab + (size_t)k * a.V * 32;
    if (it.y > 0) {
        // ---- a group of n <= 8 nodes with <= 8 edges in total: one batch of gathers
        const int n = it.y;
        const int32_t ne = it.w - it.z;
        int32_t offn_l = 0x7fffffff, nb_l = 0, no_l = 0, ov_l = 0;
        int64_t w_l = 0, c_l = 0;
        if (lane < n) {
            offn_l = __ldg(&off[r0 + lane + 1]);
            c_l = __ldg(&a.c[r0 + lane]);
            ov_l = __ldg(&a.orig[r0 + lane]);
        }
        if (lane < ne) {
            nb_l = __ldg(&nbr[it.z + lane]);
            w_l = __ldg(&ec[it.z + lane]);
            if (!FWD) no_l = __ldg(&a.orig[nb_l]);
        }
        uint32_t lw[kBMaxNodes / 4];
        {
            const uint32_t* rows = reinterpret_cast<const uint32_t*>(labk + (size_t)r0 * 32);
#pragma unroll
            for (int q = 0; q < kBMaxNodes / 4; ++q) {
                const int W = q * 32 + lane;
                lw[q] = W < 8 * n ? __ldg(&rows[W]) : 0u;
            }
        }
        const uint64_t* rec = (FWD ? a.tlr : a.blr) + (size_t)k * a.V * 32 + lane;
        uint64_t x[kBMaxEdges];
        uint32_t lb[kBMaxEdges];
        bool rdy[kBMaxEdges];
        int32_t uq[kBMaxEdges];
#pragma unroll
        for (int q = 0; q < kBMaxEdges; ++q) uq[q] = __shfl_sync(0xffffffffu, nb_l, q);
#pragma unroll
        for (int q = 0; q < kBMaxEdges; ++q) {
            x[q] = 0;
            lb[q] = 0;
            ld_relaxed_u64_if(x[q], &rec[(size_t)uq[q] * 32], q < ne);
            ldg_u8_if(lb[q], &labk[(size_t)uq[q] * 32 + lane], q < ne);
        }
#pragma unroll
        for (int q = 0; q < kBMaxEdges; ++q) rdy[q] = q >= ne || (x[q] & ~kValMask) == tag;
        bool all = true;
#pragma unroll
        for (int q = 0; q < kBMaxEdges; ++q) all = all && rdy[q];
        int32_t ns = 0;
        while (!__all_sync(0xffffffffu, all)) {
            poll_backoff(a.sleep_ns, ns);
            all = true;
#pragma unroll
            for (int q = 0; q < kBMaxEdges; ++q) {
                ld_relaxed_u64_if(x[q], &rec[(size_t)uq[q] * 32], !rdy[q]);
            }
#pragma unroll
            for (int q = 0; q < kBMaxEdges; ++q) {
                rdy[q] = rdy[q] || (x[q] & ~kValMask) == tag;
                all = all && rdy[q];
            }
        }
        // per-node reductions in edge order; nodes own contiguous edge ranges
        int cur = 0;
        int pv = n > 0 ? node_label(lw, 0, lane) : 0;
        int64_t best = FWD ? 0 : -1;
        int32_t bu = -1, bo = 0x7fffffff;
#pragma unroll
        for (int q = 0; q < kBMaxEdges; ++q) {
            if (q < ne) {
                const int32_t e = it.z + q;
                const int j = __popc(__ballot_sync(0xffffffffu, offn_l <= e));   // node of edge e
                while (cur < j) {
                    finalize_node<FWD>(a, k, lane, tag, r0 + cur, __shfl_sync(0xffffffffu, c_l, cur),
                                       __shfl_sync(0xffffffffu, ov_l, cur), pv, best, bu, acc);
                    ++cur;
                    pv = node_label(lw, cur, lane);
                    best = FWD ? 0 : -1;
                    bu = -1;
                    bo = 0x7fffffff;
                }
                const int64_t w = __shfl_sync(0xffffffffu, w_l, q);
                const int32_t u = uq[q];
                const int32_t o = __shfl_sync(0xffffffffu, no_l, q);
                const int64_t cm = (int)lb[q] == pv ? 0 : w;
                const int64_t y = (int64_t)(x[q] & kValMask) + cm;
                if (FWD) {
                    best = y > best ? y : best;
                } else {
                    if (y > best || (y == best && o < bo)) { best = y; bo = o; bu = u; }
                    acc.cut += cm;
                }
            }
        }
        while (cur < n) {
            finalize_node<FWD>(a, k, lane, tag, r0 + cur, __shfl_sync(0xffffffffu, c_l, cur),
                               __shfl_sync(0xffffffffu, ov_l, cur), pv, best, bu, acc);
            ++cur;
            if (cur < n) pv = node_label(lw, cur, lane);
            best = FWD ? 0 : -1;
            bu = -1;
            bo = 0x7fffffff;
        }
        return;
    }
    // ---- one node (y == 0) or one part of a split hub (y < 0): batches of 8 edges
    const int32_t v = r0;
    const int pv = labk[(size_t)v * 32 + lane];
    int64_t best = FWD ? 0 : -1, cut = 0;
    int32_t bu = -1, bo = 0x7fffffff;
    for (int32_t e0 = it.z; e0 < it.w; e0 += 8)
        relax_node_batch<FWD>(a, k, lane, tag, nbr, ec, e0, min(e0 + 8, it.w), pv, best, bu, bo, cut);
    if (!FWD) acc.cut += cut;
    if (it.y < 0) {
        // split hub: publish this part's partial, the last part to finish combines
        const int slot = -it.y - 1;
        const int32_t p = __ldg(&a.hub_pbase[slot]) + (it.z - __ldg(&off[v])) / kBHubEdges;
        const int32_t np = __ldg(&a.hub_pbase[slot + 1]) - __ldg(&a.hub_pbase[slot]);
        const size_t pr = ((size_t)k * a.n_parts + p) * 32 + lane;
        a.part_val[pr] = (unsigned long long)best;
        a.part_idx[pr] = bu;
        __threadfence();
        __syncwarp();
        int done = 0;
        if (lane == 0) done = atomicAdd(&a.hub_cnt[(size_t)k * a.n_hubs + slot], 1);
        done = __shfl_sync(0xffffffffu, done, 0);
        if (done != np - 1) return;
        __threadfence();
        if (lane == 0) a.hub_cnt[(size_t)k * a.n_hubs + slot] = 0;   // self-reset for the next launch
        const int32_t pb = __ldg(&a.hub_pbase[slot]);
        best = FWD ? 0 : -1;
        bu = -1;
        bo = 0x7fffffff;
        for (int32_t q = 0; q < np; ++q) {
            const size_t qr = ((size_t)k * a.n_parts + pb + q) * 32 + lane;
            const int64_t y = (int64_t)__ldcg(&a.part_val[qr]);
            if (FWD) {
                best = y > best ? y : best;
            } else {
                const int32_t u = __ldcg(&a.part_idx[qr]);
                if (u >= 0) {
                    const int32_t o = __ldg(&a.orig[u]);
                    if (y > best || (y == best && o < bo)) { best = y; bo = o; bu = u; }
                }
            }
        }
    }
    finalize_node<FWD>(a, k, lane, tag, v, __ldg(&a.c[v]), __ldg(&a.orig[v]), pv, best, bu, acc);
}

#ifndef PDNN_BSWEEP_MINB
#define PDNN_BSWEEP_MINB 1
#endif
__global__ void __launch_bounds__(kSweepThreads, PDNN_BSWEEP_MINB) k_bsweep(BSweepArgs a) {
    __shared__ uint32_t s_tag;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_tag = ld_relaxed_u32(&a.hdr->epoch) % 3 + 1;
    __syncthreads();
    const uint64_t tag = (uint64_t)s_tag << 62;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int k = gw % a.nck;                 // this warp's chunk (nw % nck == 0)
    const int stride = nw / a.nck;
    BAcc acc;
    acc.Lb = -1;
    acc.Lo = 0x7fffffff;
    acc.Lr = -1;
    acc.cut = 0;
    acc.maxst = 0;
    // the next item's descriptor is loaded one item ahead (off the per-item chain)
    const int32_t i0 = gw / a.nck;
    Item nx = i0 < a.n_items ? a.items[i0] : Item{0, 0, 0, 0};
    for (int32_t i = i0; i < a.n_items; i += stride) {
        const Item it = nx;
        if (i + stride < a.n_items) nx = a.items[i + stride];
        if (it.x >= 0) process_item<true>(a, it, k, lane, tag, acc);
        else process_item<false>(a, it, k, lane, tag, acc);
    }
    BSlot s;
    s.Lb = acc.Lb;
    s.Lo = acc.Lo;
    s.Lr = acc.Lr;
    s.cut = acc.cut;
    s.maxst = acc.maxst;
    a.slots[(size_t)gw * 32 + lane] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t t = atomicAdd(&a.hdr->ticket, 1u);
        if (t == gridDim.x - 1) {
            a.hdr->ticket = 0;
            __threadfence();
            a.hdr->epoch = s_tag;
        }
    }
}

// labels of the chunks: parts uint8 [B][V] (node-id order) -> lab[k][rank][32]
// (candidate-minor); lanes past the batch get label 0 (computed, never read)
__global__ void k_blabels(int32_t V, int32_t nck, int32_t b0, int32_t B, const int32_t* __restrict__ orig,
                          const uint8_t* __restrict__ parts, uint8_t* __restrict__ lab) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < (int64_t)nck * V; t += nwarps) {
        const int k = (int)(t / V);
        const int32_t r = (int32_t)(t % V);
        const int32_t n = __ldg(&orig[r]);
        const int32_t b = b0 + k * 32 + lane;
        lab[t * 32 + lane] = b < B ? __ldg(&parts[(size_t)b * V + n]) : (uint8_t)0;
    }
}

// per chunk (one warp per chunk): combine the warps' slots into L, the CP
// start (lowest-id entry node with bl == L), cut comm and max st, then walk
// the tight-successor chain from the start for the CP length, end and hash
// (cp_hash = sum_k (id_k + 1) * P^k, R16)
__global__ void k_bcp(int32_t V, int32_t nck, int32_t nck_run, int32_t n_warps, int32_t b0, int32_t B, const int32_t* __restrict__ orig,
                      const int32_t* __restrict__ nxt, const BSlot* __restrict__ slots,
                      unsigned long long* __restrict__ maxst, pdnn_eval_result* __restrict__ out,
                      bool write_makespan) {
    const int lane = threadIdx.x & 31;
    const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (k >= nck) return;
    int64_t Lb = -1, cut = 0, mx = 0;
    int32_t Lo = 0x7fffffff, Lr = -1;
    for (int w = k; w < n_warps; w += nck_run) {
        const BSlot s = slots[(size_t)w * 32 + lane];
        if (s.Lb > Lb || (s.Lb == Lb && s.Lo < Lo)) { Lb = s.Lb; Lo = s.Lo; Lr = s.Lr; }
        cut += s.cut;
        mx = s.maxst > mx ? s.maxst : mx;
    }
    const int32_t b = b0 + k * 32 + lane;
    uint64_t h = 0, pk = 1;
    int32_t len = 0, end = -1;
    const int32_t* nk = nxt + (size_t)k * V * 32 + lane;
    for (int32_t u = V > 0 ? Lr : -1; u >= 0;) {
        const int32_t nu = nk[(size_t)u * 32];
        const int32_t o = __ldg(&orig[u]);
        h += (uint64_t)(o + 1) * pk;
        pk *= 0x100000001B3ull;
        ++len;
        end = o;
        u = nu;
    }
    if (b < B) {
        pdnn_eval_result* r = out + (b - b0);
        r->L = V > 0 ? Lb : 0;
        r->cut_comm = cut;
        r->cp_hash = h;
        r->cp_len = len;
        r->cp_start = len > 0 ? Lo : -1;
        r->cp_end = end;
        if (write_makespan) r->makespan = V > 0 ? Lb : 0;   // level schedule: max ft = max(tl + comp) = L
        maxst[b - b0] = (unsigned long long)mx;
    }
}

static int bsweep_blocks_per_sm() { return kernel_occupancy((const void*)k_bsweep, kSweepThreads, 0); }

int bsweep_warps(const pdnn_graph* g) { return bsweep_blocks_per_sm() * g->num_sms * (kSweepThreads / 32); }

// a grid of >= 3/4 of the resident CTAs whose warp count is a multiple of m (0: none)
static int grid_for_chunks(int max_grid, int32_t m) {
    for (int grid = max_grid; 4 * grid >= 3 * max_grid; --grid)
        if (((int64_t)grid * (kSweepThreads / 32)) % m == 0) return grid;
    return 0;
}

int32_t bsweep_chunks(const pdnn_graph* g, int32_t n) {
    const int max_grid = bsweep_blocks_per_sm() * g->num_sms;
    const int32_t nw = max_grid * (kSweepThreads / 32);
    n = std::max<int32_t>(n, 1);
    for (int32_t m = n; m <= nw; ++m)   // terminates: m = nw fits the full grid
        if (grid_for_chunks(max_grid, m)) return m;
    return n;   // more chunks than warps: bsweep_grid reports it
}

int bsweep_grid(const pdnn_graph* g, int32_t nck_run) {
    const int max_grid = debug_knob("PDNN_BSWEEP_CTAS", 0) > 0
                             ? std::min(debug_knob("PDNN_BSWEEP_CTAS", 0), bsweep_blocks_per_sm() * g->num_sms)
                             : bsweep_blocks_per_sm() * g->num_sms;
    int grid = grid_for_chunks(max_grid, nck_run);
    if (!grid)   // (debug grid knob) any grid that fits
        for (grid = max_grid; grid > 0 && ((int64_t)grid * (kSweepThreads / 32)) % nck_run != 0; --grid) {}
    return grid;
}

pdnn_status launch_bsweep(const pdnn_graph* g, const Costs& C, int32_t b0, int32_t nb, int32_t B,
                          const uint8_t* parts, const BLayout& BL, void* ws, pdnn_eval_result* out,
                          cudaStream_t s, const SideStream* side, bool write_makespan) {
    const int32_t V = g->V;
    const int32_t nck_real = (nb + 31) / 32;
    // chunks run: padded so the warp count is a multiple (padded chunks hold
    // no candidate: every lane's b >= B); <= BL.ng / 32 since the padding is monotone
    const int32_t nck = bsweep_chunks(g, nck_real);
    if (nck > BL.ng / 32) { set_error("batched sweep: chunk padding exceeds the workspace group"); return PDNN_EINVAL; }
    uint8_t* lab = ws_ptr<uint8_t>(ws, BL.lab);
    if (V > 0) {
        const int64_t warps = (int64_t)nck * V;
        const int lgrid = (int)std::min<int64_t>((warps + 7) / 8, (int64_t)g->num_sms * 16);
        k_blabels<<<lgrid, 256, 0, s>>>(V, nck, b0, B, g->orig, parts, lab);
        count_launch();
        PDNN_LAUNCH_CHECK();
        BSweepArgs a;
        const int sched = nck >= kBWideChunks ? 1 : 0;
        a.items = g->bitems[sched];
        a.n_items = g->n_bitems[sched];
        a.nck = nck;
        a.V = V;
        a.n_entry = g->n_entry;
        a.in_off = g->in_off;
        a.in_src = g->in_src;
        a.out_off = g->out_off;
        a.out_dst = g->out_dst;
        a.orig = g->orig;
        a.c = C.c;
        a.in_cost = C.in_cost;
        a.out_cost = C.out_cost;
        a.hub_pbase = g->bhub_pbase;
        a.n_parts = std::max(g->n_bparts, 1);
        a.n_hubs = std::max(g->n_bhubs, 1);
        a.lab = lab;
        a.tlr = ws_ptr<uint64_t>(ws, BL.tlr);
        a.blr = ws_ptr<uint64_t>(ws, BL.blr);
        a.nxt = ws_ptr<int32_t>(ws, BL.nxt);
        a.keys = ws_ptr<int64_t>(ws, BL.keys);
        a.plab = ws_ptr<uint8_t>(ws, BL.plab);
        a.part_val = ws_ptr<unsigned long long>(ws, BL.part_val);
        a.part_idx = ws_ptr<int32_t>(ws, BL.part_idx);
        a.hub_cnt = ws_ptr<int32_t>(ws, BL.hub_cnt);
        a.slots = ws_ptr<BSlot>(ws, BL.slots);
        a.hdr = ws_ptr<WsHeader>(ws, BL.hdr);
        a.sleep_ns = debug_knob("PDNN_BPOLL_SLEEP_NS", 0);
        // warps = grid * 8 is a multiple of nck (each warp serves one chunk)
        const int grid = bsweep_grid(g, nck);
        if (grid <= 0) { set_error("batched sweep: no grid fits the chunk count"); return PDNN_EINVAL; }
        void* args[] = {(void*)&a};
        PDNN_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_bsweep, dim3(grid), dim3(kSweepThreads), args, 0, s));
        count_launch();
        const int nwarps = grid * (kSweepThreads / 32);
        // the CP walk is a latency chain of one dependent load per CP node on a
        // handful of warps: run it on a side stream, overlapped with the memory
        // tracker (disjoint result fields); the caller joins it before reusing
        // the workspace
        if (side) {
            PDNN_CUDA_TRY(cudaEventRecord(side->ev_fork, s));
            PDNN_CUDA_TRY(cudaStreamWaitEvent(side->stream, side->ev_fork, 0));
        }
        k_bcp<<<(nck_real + 3) / 4, 128, 0, side ? side->stream : s>>>(V, nck_real, nck, nwarps, b0, b0 + nb, g->orig, a.nxt,
                                                                   a.slots, ws_ptr<unsigned long long>(ws, BL.maxst), out,
                                                                   write_makespan);
        if (side) PDNN_CUDA_TRY(cudaEventRecord(side->ev_join, side->stream));
    } else {
        k_bcp<<<(nck_real + 3) / 4, 128, 0, s>>>(0, nck_real, nck, 0, b0, b0 + nb, g->orig, nullptr, nullptr,
                                            ws_ptr<unsigned long long>(ws, BL.maxst), out, write_makespan);
    }
    count_launch();
    PDNN_LAUNCH_CHECK();
    return PDNN_OK;
}

}  // namespace pdnn
