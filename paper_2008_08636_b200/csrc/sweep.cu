// sweep.cu -- the weighted-level sweep (§8(a) rows a3 + a4).
//
// Definitions (Table 2; Alg. 1 lines 2 / 7):
//   tl(v) = max(0, max_{alive p in pred(v)} tl(p) + comp(p) + comm'(p,v))
//   bl(u) = comp(u) + max(0, max_{alive s in succ(u)} comm'(u,s) + bl(s))
//
// B200 design: one persistent cooperative launch runs
// BOTH passes as a dataflow computation -- no per-level grid barrier.  Work
// items (a level-aligned group of <= 32 nodes, or one part of a high-degree
// node) are dealt round-robin to resident warps in a merged order in which
// every item depends only on items with a smaller index (tl items ascend by
// level over the reverse CSR, bl items descend over the forward CSR).  A
// consumer waits on each needed neighbour value individually: the value and
// its readiness share one 64-bit word (bits 62-63 = the sweep's epoch tag,
// cycling 1..3; values < 2^62), written with st.relaxed.gpu and polled with
// ld.relaxed.gpu.  Static data (offsets, neighbour ids, edge costs, labels)
// is loaded before waiting, so the HBM stream is decoupled from the
// dependency chain; the dependent gathers hit L2.  Hubs are split into
// <= 1024-edge parts reduced by a warp each and combined with a
// self-resetting atomicMax accumulator.
#include "internal.cuh"

namespace pdnn {

struct SweepArgs {
    const Item* items;
    int32_t n_items;
    const int32_t* in_off;
    const int32_t* in_src;
    const int32_t* out_off;
    const int32_t* out_dst;
    const int64_t* c;
    const int64_t* in_cost;
    const int64_t* out_cost;
    const int32_t* part;  // rank space; nullptr = all edges pay comm
    const int32_t* orig;
    uint64_t* tlc;        // tagged tl + comp (rank space)
    uint64_t* bl;         // tagged bl (rank space)
    int64_t* tl_out;      // node-id order (nullable)
    int64_t* bl_out;
    unsigned long long* hub_acc;
    int32_t* hub_cnt;
    const int32_t* hub_nparts;
    WsHeader* hdr;
};

template <bool HAS_PART>
__device__ __forceinline__ void finish_node(const SweepArgs& a, bool fwd, int32_t v, int64_t best,
                                            uint64_t tag, int64_t& lmax) {
    const int64_t c = a.c[v];
    const int32_t ov = a.orig[v];
    if (fwd) {
        const int64_t tlc = best + c;
        st_relaxed_u64(&a.tlc[v], tag | (uint64_t)tlc);
        if (a.tl_out) a.tl_out[ov] = best;
        lmax = tlc > lmax ? tlc : lmax;
    } else {
        const int64_t b = c + best;
        st_relaxed_u64(&a.bl[v], tag | (uint64_t)b);
        if (a.bl_out) a.bl_out[ov] = b;
    }
}

__device__ __forceinline__ void finish_removed(const SweepArgs& a, bool fwd, int32_t v, uint64_t tag) {
    st_relaxed_u64(fwd ? &a.tlc[v] : &a.bl[v], tag);
    int64_t* out = fwd ? a.tl_out : a.bl_out;
    if (out) out[a.orig[v]] = -1;
}

// One warp-synchronous batch of up to 4 edges per lane: edge k of lane l is
// e + k*step (live if < t).  Static data (neighbour, cost, label) is loaded
// first; then every live neighbour value is requested at once and the warp
// re-polls only the values whose tag is not yet this sweep's, in a loop whose
// condition is warp-uniform (__any_sync), so the warp never serialises lanes.
template <bool HAS_PART>
__device__ __forceinline__ void relax_batch(const int32_t* __restrict__ nbr, const int64_t* __restrict__ ec,
                                            const int32_t* __restrict__ part, const uint64_t* val,
                                            int32_t pv, int32_t e, int32_t t, int32_t step, uint64_t tag,
                                            int64_t& best, int64_t& cut) {
    int32_t nb[4];
    int64_t w[4];
    bool live[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int32_t ek = e + k * step;
        live[k] = ek < t;
        nb[k] = live[k] ? __ldg(&nbr[ek]) : 0;
        w[k] = live[k] ? __ldg(&ec[ek]) : 0;
    }
    // neighbour labels and values are requested together (one round trip)
    uint64_t x[4];
    int32_t pp[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        x[k] = live[k] ? ld_relaxed_u64(&val[nb[k]]) : 0;
        pp[k] = (HAS_PART && live[k]) ? __ldg(&part[nb[k]]) : 0;
    }
    int64_t cm[4];
    bool rdy[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (HAS_PART) {
            live[k] = live[k] && pp[k] != PDNN_REMOVED;
            cm[k] = (pp[k] == pv && pv >= 0) ? 0 : w[k];
        } else {
            cm[k] = w[k];
        }
        rdy[k] = !live[k] || (x[k] & ~kValMask) == tag;
    }
    while (__any_sync(0xffffffffu, !(rdy[0] && rdy[1] && rdy[2] && rdy[3]))) {
        __nanosleep(20);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (!rdy[k]) {
                x[k] = ld_relaxed_u64(&val[nb[k]]);
                rdy[k] = (x[k] & ~kValMask) == tag;
            }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (live[k]) {
            const int64_t y = (int64_t)(x[k] & kValMask) + cm[k];
            best = y > best ? y : best;
            cut += cm[k];
        }
}

template <bool HAS_PART>
__global__ void __launch_bounds__(kSweepThreads) k_sweep(SweepArgs a) {
    __shared__ uint32_t s_tag;
    if (threadIdx.x == 0) {
        const uint32_t prev = ld_relaxed_u32(&a.hdr->epoch);
        s_tag = prev % 3 + 1;
        if (blockIdx.x == 0) {  // clear the NEXT epoch's accumulators (unused during this call)
            a.hdr->Lslot[s_tag % 3 + 1] = 0;
            a.hdr->cut[s_tag % 3 + 1] = 0;
        }
    }
    __syncthreads();
    const uint64_t tag = (uint64_t)s_tag << 62;
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    int64_t lmax = 0, cut = 0;

    for (int i = gw; i < a.n_items; i += nw) {
        const Item it = a.items[i];
        const bool fwd = it.x >= 0;
        const int32_t r0 = fwd ? it.x : ~it.x;
        const int32_t* off = fwd ? a.in_off : a.out_off;
        const int32_t* nbr = fwd ? a.in_src : a.out_dst;
        const int64_t* ec = fwd ? a.in_cost : a.out_cost;
        const uint64_t* val = fwd ? a.tlc : a.bl;
        if (it.y > 0) {
            // thread-per-node item: lane j owns node r0 + j (all of one level)
            const bool act = lane < it.y;
            const int32_t v = r0 + lane;
            const int32_t pv = (HAS_PART && act) ? __ldg(&a.part[v]) : 0;
            const bool removed = HAS_PART && act && pv == PDNN_REMOVED;
            const int32_t s0 = act ? __ldg(&off[v]) : 0;
            const int32_t s1 = (act && !removed) ? __ldg(&off[v + 1]) : s0;
            const int32_t maxdeg = __reduce_max_sync(0xffffffffu, s1 - s0);
            int64_t best = 0, c2 = 0;
            for (int32_t k0 = 0; k0 < maxdeg; k0 += 4)   // warp-uniform trip count
                relax_batch<HAS_PART>(nbr, ec, a.part, val, pv, s0 + k0, s1, 1, tag, best, c2);
            if (act) {
                if (removed) {
                    finish_removed(a, fwd, v, tag);
                } else {
                    if (!fwd) cut += c2;
                    finish_node<HAS_PART>(a, fwd, v, best, tag, lmax);
                }
            }
        } else {
            // warp item: edges [z, w) of node r0 (a hub part if y < 0)
            const int32_t v = r0;
            const int32_t pv = HAS_PART ? __ldg(&a.part[v]) : 0;
            if (HAS_PART && pv == PDNN_REMOVED) {
                if (lane == 0 && it.z == __ldg(&off[v])) finish_removed(a, fwd, v, tag);
                continue;
            }
            int64_t best = 0, c2 = 0;
            for (int32_t e0 = it.z; e0 < it.w; e0 += 4 * 32)   // warp-uniform trip count
                relax_batch<HAS_PART>(nbr, ec, a.part, val, pv, e0 + lane, it.w, 32, tag, best, c2);
            if (!fwd) cut += c2;
            best = warp_max_i64(best);
            if (lane == 0) {
                if (it.y == 0) {
                    finish_node<HAS_PART>(a, fwd, v, best, tag, lmax);
                } else {
                    const int slot = -it.y - 1;
                    atomicMax(&a.hub_acc[slot], (unsigned long long)best);
                    __threadfence();
                    const int done = atomicAdd(&a.hub_cnt[slot], 1);
                    if (done == __ldg(&a.hub_nparts[slot]) - 1) {
                        __threadfence();
                        const int64_t b = (int64_t)atomicExch(&a.hub_acc[slot], 0ull);
                        atomicExch(&a.hub_cnt[slot], 0);
                        finish_node<HAS_PART>(a, fwd, v, b, tag, lmax);
                    }
                }
            }
        }
    }
    lmax = warp_max_i64(lmax);
    cut = warp_sum_i64(cut);
    if (lane == 0) {
        if (lmax > 0) atomicMax(&a.hdr->Lslot[s_tag], (unsigned long long)lmax);
        if (cut > 0) atomicAdd(&a.hdr->cut[s_tag], (unsigned long long)cut);
    }
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

int sweep_blocks_per_sm(int device) {
    (void)device;
    int a = 0, b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_sweep<true>, kSweepThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_sweep<false>, kSweepThreads, 0);
    int n = a < b ? a : b;
    return n < 1 ? 1 : n;
}

pdnn_status launch_sweep(const pdnn_graph* g, const Costs& C, const int32_t* part_rank, int64_t* tl,
                         int64_t* bl, void* ws, const WsLayout& L, cudaStream_t s) {
    if (g->V == 0) return PDNN_OK;
    SweepArgs a;
    a.items = g->items;
    a.n_items = g->n_items;
    a.in_off = g->in_off;
    a.in_src = g->in_src;
    a.out_off = g->out_off;
    a.out_dst = g->out_dst;
    a.c = C.c;
    a.in_cost = C.in_cost;
    a.out_cost = C.out_cost;
    a.part = part_rank;
    a.orig = g->orig;
    a.tlc = ws_ptr<uint64_t>(ws, L.tlc);
    a.bl = ws_ptr<uint64_t>(ws, L.bl);
    a.tl_out = tl;
    a.bl_out = bl;
    a.hub_acc = ws_ptr<unsigned long long>(ws, L.hub_acc);
    a.hub_cnt = ws_ptr<int32_t>(ws, L.hub_cnt);
    a.hub_nparts = g->hub_nparts;
    a.hdr = ws_ptr<WsHeader>(ws, L.hdr);
    void* args[] = {(void*)&a};
    const void* fn = part_rank ? (const void*)k_sweep<true> : (const void*)k_sweep<false>;
    PDNN_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(g->sweep_grid), dim3(kSweepThreads), args, 0, s));
    count_launch();
    return PDNN_OK;
}

}  // namespace pdnn

using namespace pdnn;

extern "C" pdnn_status pdnn_weighted_levels(const pdnn_graph* g, const int64_t* node_cost,
                                            const int64_t* edge_cost, const int32_t* part, int64_t* tl,
                                            int64_t* bl, void* ws, size_t ws_bytes, void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (g->V > 0 && (!tl || !bl)) { set_error("null tl/bl"); return PDNN_EINVAL; }
    const WsLayout L = ws_layout(g, PDNN_OP_WEIGHTED_LEVELS, 0);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    Costs C;
    pdnn_status st = resolve_costs(g, node_cost, edge_cost, ws, L, s, &C);
    if (st) return st;
    int32_t* pr = nullptr;
    if (part) {
        pr = ws_ptr<int32_t>(ws, L.part_rank);
        if ((st = launch_to_rank_i32(g, part, pr, s))) return st;
    }
    return launch_sweep(g, C, pr, tl, bl, ws, L, s);
}
