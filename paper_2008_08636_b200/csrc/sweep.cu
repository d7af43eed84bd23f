// sweep.cu -- the weighted-level sweep (§8(a) rows a3 + a4).
//
// Definitions (Table 2; Alg. 1 lines 2 / 7):
//   tl(v) = max(0, max_{alive p in pred(v)} tl(p) + comp(p) + comm'(p,v))
//   bl(u) = comp(u) + max(0, max_{alive s in succ(u)} comm'(u,s) + bl(s))
//
// B200 design: one persistent cooperative launch runs
// BOTH passes as a dataflow computation -- no per-level grid barrier.  Work
// items (a level-aligned run of <= 32 nodes, or one part of a high-degree
// node) are dealt round-robin to resident warps in a merged order in which
// every item depends only on items with a smaller index (tl items ascend by
// level over the reverse CSR, bl items descend over the forward CSR).  A
// consumer waits on each needed neighbour value individually: the value and
// its readiness share one 64-bit word (bits 62-63 = the sweep's epoch tag,
// cycling 1..3; values < 2^62), written with st.relaxed.gpu and polled with
// ld.relaxed.gpu.
//
// Thread items are pre-packed once per cost binding into a contiguous
// per-item "blob" (graph.cu k_blob): one 16-byte record per LANE {comp,
// original id, edge slice of the lane, node index, chunk} -- a node of
// degree d <= 32 owns ceil(d/4) adjacent lanes -- followed by the item's neighbour
// ranks and edge costs.  A warp stages the next item with ONE bulk copy
// (cp.async.bulk, the TMA engine) plus one copy of the item's labels, so the
// per-item work is a shared-memory read per lane, one batch of <= 4 gathers
// per lane, and one store; the HBM stream is decoupled from the dependency
// chain and the dependent gathers hit L2.  Hubs are split into <= 1024-edge
// parts reduced by a warp each and combined with a self-resetting atomicMax.
#include <cooperative_groups.h>

#include "internal.cuh"

namespace pdnn {

struct SweepArgs {
    const Item* items;
    int32_t n_items;
    int32_t V;
    int32_t n_entry;     // ranks [0, n_entry) = level 0: tl = 0, published by the prologue
    const unsigned char* blob_in;    // tl items (reverse CSR), addressed by item.z * 16
    const unsigned char* blob_out;   // bl items (forward CSR)
    // warp items (hub parts) read the CSR directly
    const int32_t* in_off;
    const int32_t* in_src;
    const int32_t* out_off;
    const int32_t* out_dst;
    const int64_t* c;
    const int64_t* in_cost;
    const int64_t* out_cost;
    const int32_t* orig;
    const int32_t* lab;   // rank-space labels; nullptr = every node UNASSIGNED
    const int32_t* lab_src;   // node-id-order labels to convert into `lab` first (nullable)
    uint64_t* rec;        // [2][V] tagged values: rec[v] = tl(v)+comp(v), rec[V+v] = bl(v)
    int64_t* tl_out;      // node-id order
    int64_t* bl_out;
    unsigned long long* hub_acc;
    int32_t* hub_cnt;
    const int32_t* hub_nparts;
    WsHeader* hdr;
    int32_t sleep_ns;     // poll back-off (debug knob; 0 = spin)
    int32_t nowait;       // debug knob: never wait (a streaming-time probe; values are wrong)
    unsigned long long* trace;   // debug knob: per item {start, ready, done} globaltimer stamps (nullable)
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------- TMA staging
constexpr int kBlobMax = 16 * 32 + 4 * kTMaxEdges + 8 * kTMaxEdges;   // lane records + ranks + costs
constexpr int kLabB = 4 * 32 + 16;                                     // <= 32 labels, 16-B widened
constexpr int kRegBlob = 0, kRegLab = kBlobMax, kRegHdr = kRegLab + kLabB;   // hdr: Item + label shift
constexpr int kStageBytes = kRegHdr + 32;
#ifndef PDNN_SWEEP_STAGES
#define PDNN_SWEEP_STAGES 2
#endif
#ifndef PDNN_SWEEP_MINB
#define PDNN_SWEEP_MINB 3
#endif
constexpr int kStages = PDNN_SWEEP_STAGES;
constexpr int kWarpsPerCta = kSweepThreads / 32;
constexpr int kSweepSmem = kWarpsPerCta * kStages * kStageBytes;
static_assert(kStageBytes % 16 == 0 && kBlobMax % 16 == 0, "stage alignment");

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// the blobs are streamed once per sweep: L2 evict-first, so they do not push
// the value records (gathered and polled all sweep long) out of L2
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// Lane 0 stages item `it`: its blob (one copy) and, with labels, the labels of
// its nodes (widened to 16-byte boundaries; the head shift goes in the stage
// header).  Warp items read global memory directly: only the phase completes.
template <bool HAS_LAB>
__device__ __forceinline__ void issue_item(const SweepArgs& a, const Item& it, unsigned char* stage, uint64_t* bar,
                                           uint64_t pol) {
    int32_t shift = 0;
    if (it.y <= 0) {
        mbar_arrive_expect_tx(bar, 0);
    } else {
        const int nl = it.w & 0xff, m = (it.w >> 8) & 0xff;
        const uint32_t bytes = (uint32_t)((16 * nl + 4 * ((m + 1) & ~1) + 8 * m + 15) & ~15);
        const bool fwd = it.x >= 0;
        const int32_t r0 = fwd ? it.x : ~it.x;
        uint32_t lbytes = 0;
        const char* lsrc = nullptr;
        if (HAS_LAB && !(it.w & kItemIndexed)) {   // (indexed items read their nodes' labels per lane)
            const uintptr_t s0 = (uintptr_t)(a.lab + r0), s1 = (uintptr_t)(a.lab + r0 + it.y);
            const uintptr_t lo = s0 & ~(uintptr_t)15, hi = (s1 + 15) & ~(uintptr_t)15;
            lsrc = (const char*)lo;
            lbytes = (uint32_t)(hi - lo);
            shift = (int32_t)((s0 - lo) >> 2);
        }
        mbar_arrive_expect_tx(bar, bytes + lbytes);
        tma_load_1d(stage + kRegBlob, (fwd ? a.blob_in : a.blob_out) + (size_t)it.z * 16, bytes, bar, pol);
        if (HAS_LAB && lbytes) tma_load_1d(stage + kRegLab, lsrc, lbytes, bar, pol);
    }
    *reinterpret_cast<int4*>(stage + kRegHdr) = make_int4(it.x, it.y, it.z, it.w);
    *reinterpret_cast<int32_t*>(stage + kRegHdr + 16) = shift;
}

#ifndef PDNN_SWEEP_LDGSTS
#define PDNN_SWEEP_LDGSTS 0
#endif
// LDGSTS variant (all lanes): the item's blob in 16-byte cp.async chunks and
// its labels in 4-byte ones, one commit group per item
template <bool HAS_LAB>
__device__ __forceinline__ void issue_item_lanes(const SweepArgs& a, const Item& it, unsigned char* stage, int lane) {
    if (it.y > 0) {
        const int nl = it.w & 0xff, m = (it.w >> 8) & 0xff;
        const int chunks = (16 * nl + 4 * ((m + 1) & ~1) + 8 * m + 15) >> 4;
        const bool fwd = it.x >= 0;
        const int32_t r0 = fwd ? it.x : ~it.x;
        const unsigned char* src = (fwd ? a.blob_in : a.blob_out) + (size_t)it.z * 16;
        for (int q = lane; q < chunks; q += 32)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(stage + kRegBlob + 16 * q)),
                         "l"(src + 16 * q) : "memory");
        if (HAS_LAB && lane < it.y && !(it.w & kItemIndexed))
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(stage + kRegLab + 4 * lane)),
                         "l"(a.lab + r0 + lane) : "memory");
    }
    if (lane == 0) {
        *reinterpret_cast<int4*>(stage + kRegHdr) = make_int4(it.x, it.y, it.z, it.w);
        *reinterpret_cast<int32_t*>(stage + kRegHdr + 16) = 0;
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// One warp-synchronous batch of up to 4 edges per lane: edge k of lane l is
// nbr[e + k*step] (live if e + k*step < t).  Every live neighbour value is
// requested at once (and, with labels, the neighbour's label: labels do not
// change during a sweep, so they are read once with the non-coherent path);
// the warp re-polls only the values whose tag is not yet this sweep's, in a
// loop whose condition is warp-uniform (__any_sync), so no lane serialises.
template <bool HAS_LAB>
__device__ __forceinline__ void relax_batch(const int32_t* nbr, const int64_t* ec, const uint64_t* val,
                                            const int32_t* lab, int32_t pv, int32_t e, int32_t t, int32_t step,
                                            uint64_t tag, int64_t& best, int64_t& cut, int32_t sleep_ns,
                                            int32_t nowait) {
    int32_t nb[4];
    int64_t w[4];
    bool live[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int32_t ek = e + k * step;
        live[k] = ek < t;
        nb[k] = live[k] ? nbr[ek] : 0;
        w[k] = live[k] ? ec[ek] : 0;
    }
    uint64_t x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = 0;
    // every load of the batch is issued before the first use
    ld_relaxed_u64_x4(x, &val[nb[0]], &val[nb[1]], &val[nb[2]], &val[nb[3]], live[0], live[1], live[2], live[3]);
    int64_t cm[4];
    if (HAS_LAB) {
        // neighbour labels do not change during a sweep: read once (non-coherent path)
        int32_t pl[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) pl[k] = live[k] ? __ldg(&lab[nb[k]]) : 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            live[k] = live[k] && pl[k] != PDNN_REMOVED;
            cm[k] = (pl[k] == pv && pv >= 0) ? 0 : w[k];
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) cm[k] = w[k];
    }
    bool rdy[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) rdy[k] = !live[k] || (x[k] & ~kValMask) == tag || nowait;
    while (__any_sync(0xffffffffu, !(rdy[0] && rdy[1] && rdy[2] && rdy[3]))) {
        if (sleep_ns > 0) __nanosleep(sleep_ns);
        ld_relaxed_u64_x4(x, &val[nb[0]], &val[nb[1]], &val[nb[2]], &val[nb[3]], !rdy[0], !rdy[1], !rdy[2], !rdy[3]);
#pragma unroll
        for (int k = 0; k < 4; ++k) rdy[k] = rdy[k] || (x[k] & ~kValMask) == tag;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (live[k]) {
            const int64_t y = (int64_t)(x[k] & kValMask) + cm[k];
            best = y > best ? y : best;
            cut += cm[k];
        }
}

// publish node v's value with this sweep's tag
template <bool HAS_LAB>
__device__ __forceinline__ void publish(const SweepArgs& a, bool fwd, int32_t v, int64_t value, int32_t pv, uint64_t tag) {
    (void)pv;
    st_relaxed_u64(a.rec + (fwd ? 0 : (size_t)a.V) + v, tag | (uint64_t)value);
}

// lane record of a thread item (graph.cu k_blob writes them)
struct __align__(16) LaneRec {
    int64_t c;      // comp of the lane's node
    int32_t orig;   // its original id
    uint32_t meta;  // e0 (8) | n_edges (3) | node index (5) | chunk (3) | lanes of the node after this one (3)
};

template <bool HAS_LAB>
__global__ void __launch_bounds__(kSweepThreads, PDNN_SWEEP_MINB) k_sweep(SweepArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_bar[kWarpsPerCta][kStages];
    __shared__ uint32_t s_tag;
    const int lane = threadIdx.x & 31, wic = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        const uint32_t prev = ld_relaxed_u32(&a.hdr->epoch);
        s_tag = prev % 3 + 1;
        if (blockIdx.x == 0) {  // clear the NEXT epoch's accumulators (unused during this call)
            a.hdr->Lslot[s_tag % 3 + 1] = 0;
            a.hdr->cut[s_tag % 3 + 1] = 0;
        }
    }
    if (lane == 0) {
        for (int st = 0; st < kStages; ++st) mbar_init(&s_bar[wic][st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (HAS_LAB && a.lab_src) {
        // the placement's labels into rank space (the former k_labels launch):
        // one grid-stride pass, then a grid barrier before any item stages or
        // gathers a label (labels are read through the non-coherent path below,
        // and no SM has read these lines before this point)
        int32_t* lab_w = const_cast<int32_t*>(a.lab);
        const int32_t nth = gridDim.x * blockDim.x;
        constexpr int U = 4;
        for (int32_t r0 = blockIdx.x * blockDim.x + threadIdx.x; r0 < a.V; r0 += U * nth) {
            int32_t n[U];
#pragma unroll
            for (int u = 0; u < U; ++u) n[u] = r0 + u * nth < a.V ? __ldg(&a.orig[r0 + u * nth]) : -1;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (n[u] >= 0) lab_w[r0 + u * nth] = __ldg(&a.lab_src[n[u]]);
        }
        __threadfence();
        cooperative_groups::this_grid().sync();
    }
    __syncthreads();
    const uint64_t tag = (uint64_t)s_tag << 62;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    unsigned char* wsm = smem + (size_t)wic * kStages * kStageBytes;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int64_t lmax = 0, cut = 0;

    // prologue: level 0 has no predecessors, so tl = 0 there (Table 2 with an
    // empty max); publish tl + comp of every entry node with a grid-stride
    // pass instead of dataflow items
    for (int32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < a.n_entry; r += gridDim.x * blockDim.x) {
        const int32_t o = __ldg(&a.orig[r]);
        if (HAS_LAB && __ldg(&a.lab[r]) == PDNN_REMOVED) {
            st_relaxed_u64(&a.rec[r], tag);
            a.tl_out[o] = -1;
        } else {
            const int64_t c = __ldg(&a.c[r]);
            st_relaxed_u64(&a.rec[r], tag | (uint64_t)c);
            a.tl_out[o] = 0;
            lmax = c > lmax ? c : lmax;
        }
    }

    // descriptors are loaded one iteration before they are issued, so no
    // dependent global load sits on the per-item path
    auto desc = [&](int32_t i) {
        Item d;
        if (i < a.n_items) d = a.items[i];
        else d.x = d.y = d.z = d.w = 0;
        return d;
    };
    for (int k = 0; k < kStages - 1; ++k) {
        const int32_t i = gw + k * nw;
        const Item d = desc(i);
        if (PDNN_SWEEP_LDGSTS) issue_item_lanes<HAS_LAB>(a, i < a.n_items ? d : Item{0, 0, 0, 0}, wsm + k * kStageBytes, lane);
        else if (lane == 0 && i < a.n_items) issue_item<HAS_LAB>(a, d, wsm + k * kStageBytes, &s_bar[wic][k], pol);
    }
    Item nd = desc(gw + (kStages - 1) * nw);
    __syncwarp();
    for (int k = 0;; ++k) {
        const int32_t i = gw + k * nw;
        if (i >= a.n_items) break;
        const int st = k % kStages;
        {
            const int32_t inext = i + (kStages - 1) * nw;
            const int sn = (k + kStages - 1) % kStages;
            if (PDNN_SWEEP_LDGSTS) issue_item_lanes<HAS_LAB>(a, inext < a.n_items ? nd : Item{0, 0, 0, 0}, wsm + sn * kStageBytes, lane);
            else if (lane == 0 && inext < a.n_items) issue_item<HAS_LAB>(a, nd, wsm + sn * kStageBytes, &s_bar[wic][sn], pol);
            nd = desc(inext + nw);   // consumed at the next iteration
        }
        const unsigned char* sb = wsm + st * kStageBytes;
        const int4 itv = *reinterpret_cast<const int4*>(sb + kRegHdr);
        const bool fwd = itv.x >= 0;
        const int32_t r0 = fwd ? itv.x : ~itv.x;
        const uint64_t* val = a.rec + (fwd ? 0 : (size_t)a.V);
        if (PDNN_SWEEP_LDGSTS) {
            asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 1) : "memory");
            __syncwarp();
        } else {
            mbar_wait(&s_bar[wic][st], (uint32_t)((k / kStages) & 1));
        }
        if (itv.y > 0) {
            // thread item: lane <-> (node, chunk of <= 4 edges), from the blob
            const int nl = itv.w & 0xff, m = (itv.w >> 8) & 0xff;
            const bool act = lane < nl;
            const LaneRec lr = act ? reinterpret_cast<const LaneRec*>(sb + kRegBlob)[lane] : LaneRec{0, 0, 0u};
            const int32_t* sNbr = reinterpret_cast<const int32_t*>(sb + kRegBlob + 16 * nl);
            const int64_t* sEc = reinterpret_cast<const int64_t*>(sb + kRegBlob + 16 * nl + 4 * ((m + 1) & ~1));
            const int j = (lr.meta >> 11) & 31;
            // indexed items (bl of level 0, grouped by readiness): the lane
            // record carries the node's rank, its label and id are gathered
            const bool ix = (itv.w & kItemIndexed) != 0;
            const int32_t v = ix ? lr.orig : r0 + j;
            int32_t pv = PDNN_UNASSIGNED;
            if (HAS_LAB && act)
                pv = ix ? __ldg(&a.lab[v])
                        : reinterpret_cast<const int32_t*>(sb + kRegLab)[*reinterpret_cast<const int32_t*>(sb + kRegHdr + 16) + j];
            const bool removed = HAS_LAB && pv == PDNN_REMOVED;
            const int32_t e0 = (int32_t)(lr.meta & 0xff);
            const int32_t e1 = removed ? e0 : e0 + (int32_t)((lr.meta >> 8) & 7);
            int64_t best = 0, c2 = 0;
            unsigned long long t0 = 0;
            if (a.trace && lane == 0) t0 = gtime();
            relax_batch<HAS_LAB>(sNbr, sEc, val, a.lab, pv, e0, e1, 1, tag, best, c2, a.sleep_ns, a.nowait);
            if (a.trace && lane == 0) { a.trace[3 * (size_t)i] = t0; a.trace[3 * (size_t)i + 1] = gtime(); }
            if (!fwd) cut += c2;
            // segmented max over the node's lanes (chunk 0 collects; the lanes
            // of a node are adjacent, rem = lanes of the node after this one)
            const int rem = (int)((lr.meta >> 19) & 7);
            if (__any_sync(0xffffffffu, rem > 0)) {
#pragma unroll
                for (int s2 = 1; s2 < 8; s2 <<= 1) {
                    const int64_t o2 = __shfl_down_sync(0xffffffffu, best, s2);
                    if (s2 <= rem) best = o2 > best ? o2 : best;
                }
            }
            if (act && ((lr.meta >> 16) & 7) == 0) {
                if (removed) {
                    publish<HAS_LAB>(a, fwd, v, 0, pv, tag);
                    (fwd ? a.tl_out : a.bl_out)[ix ? __ldg(&a.orig[v]) : lr.orig] = -1;
                } else if (fwd) {
                    const int64_t tlc = best + lr.c;
                    publish<HAS_LAB>(a, true, v, tlc, pv, tag);
                    a.tl_out[lr.orig] = best;
                    lmax = tlc > lmax ? tlc : lmax;
                } else {
                    const int64_t b = lr.c + best;
                    publish<HAS_LAB>(a, false, v, b, pv, tag);
                    a.bl_out[ix ? __ldg(&a.orig[v]) : lr.orig] = b;
                }
            }
        } else {
            // warp item: edges [z, w) of node r0 (a hub part if y < 0), from global memory
            const int32_t* nbr = fwd ? a.in_src : a.out_dst;
            const int64_t* ec = fwd ? a.in_cost : a.out_cost;
            const int32_t v = r0;
            const int32_t pv = HAS_LAB ? __ldg(&a.lab[v]) : PDNN_UNASSIGNED;
            if (HAS_LAB && pv == PDNN_REMOVED) {
                if (lane == 0 && itv.z == __ldg(&(fwd ? a.in_off : a.out_off)[v])) {
                    publish<HAS_LAB>(a, fwd, v, 0, pv, tag);
                    (fwd ? a.tl_out : a.bl_out)[a.orig[v]] = -1;
                }
            } else {
                int64_t best = 0, c2 = 0;
                for (int32_t e0 = itv.z; e0 < itv.w; e0 += 4 * 32)   // warp-uniform trip count
                    relax_batch<HAS_LAB>(nbr, ec, val, a.lab, pv, e0 + lane, itv.w, 32, tag, best, c2, a.sleep_ns, a.nowait);
                if (!fwd) cut += c2;
                best = warp_max_i64(best);
                if (lane == 0) {
                    bool fin = itv.y == 0;
                    if (!fin) {
                        const int slot = -itv.y - 1;
                        atomicMax(&a.hub_acc[slot], (unsigned long long)best);
                        __threadfence();
                        const int done = atomicAdd(&a.hub_cnt[slot], 1);
                        if (done == __ldg(&a.hub_nparts[slot]) - 1) {
                            __threadfence();
                            best = (int64_t)atomicExch(&a.hub_acc[slot], 0ull);
                            atomicExch(&a.hub_cnt[slot], 0);
                            fin = true;
                        }
                    }
                    if (fin) {
                        const int64_t c = a.c[v];
                        if (fwd) {
                            publish<HAS_LAB>(a, true, v, best + c, pv, tag);
                            a.tl_out[a.orig[v]] = best;
                            lmax = best + c > lmax ? best + c : lmax;
                        } else {
                            publish<HAS_LAB>(a, false, v, c + best, pv, tag);
                            a.bl_out[a.orig[v]] = c + best;
                        }
                    }
                }
            }
        }
        if (a.trace) {   // (debug build) the publish has been issued by now; the max over the warp's lanes
            const unsigned long long t2 = gtime();
            if (lane == 0) a.trace[3 * (size_t)i + 2] = t2;
        }
        __syncwarp();   // the stage is re-filled at the next iteration
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

unsigned long long* g_sweep_trace = nullptr;   // debug build: last trace buffer

static int sweep_occupancy(bool has_lab) {
    return kernel_occupancy(has_lab ? (const void*)k_sweep<true> : (const void*)k_sweep<false>, kSweepThreads,
                            kSweepSmem);
}

// CTAs per SM of the graph's sweep grid.  Deep, narrow graphs are bound by the
// dependency chain, and extra warps only spin: capped at 2 CTAs/SM (round 1:
// C3 3.21 ms at 2 vs 3.78 at 3, C2 1.07 vs 1.17).  Wide graphs (>= kWideLevel
// nodes per level on average) are bound by throughput and take every
// resident CTA.
constexpr int kSweepCtasPerSmDeep = 2;
constexpr int kWideLevel = 2048;
int sweep_blocks_per_sm(int device, int32_t V, int32_t D) {
    (void)device;
    const int a = sweep_occupancy(true), b = sweep_occupancy(false);
    const int n = a < b ? a : b;
    const bool wide = D > 0 && (int64_t)V >= (int64_t)kWideLevel * D;
    return wide || n < kSweepCtasPerSmDeep ? n : kSweepCtasPerSmDeep;
}

pdnn_status launch_sweep(const pdnn_graph* g, const Costs& C, const int32_t* lab_rank, int64_t* tl,
                         int64_t* bl, void* ws, const WsLayout& L, cudaStream_t s, bool removal,
                         const int32_t* lab_src) {
    if (g->V == 0) return PDNN_OK;
    if (!C.blob_in || !C.blob_out) { set_error("sweep: cost blobs not built"); return PDNN_EINVAL; }
    SweepArgs a;
    a.items = removal && g->items_rm ? g->items_rm : g->items;
    a.n_items = g->n_items;
    a.V = g->V;
    a.n_entry = g->n_entry;
    a.blob_in = C.blob_in;
    a.blob_out = C.blob_out;
    a.in_off = g->in_off;
    a.in_src = g->in_src;
    a.out_off = g->out_off;
    a.out_dst = g->out_dst;
    a.c = C.c;
    a.in_cost = C.in_cost;
    a.out_cost = C.out_cost;
    a.orig = g->orig;
    a.lab = lab_rank;
    a.lab_src = lab_rank ? lab_src : nullptr;
    a.rec = ws_ptr<uint64_t>(ws, L.rec);
    a.tl_out = tl;
    a.bl_out = bl;
    a.hub_acc = ws_ptr<unsigned long long>(ws, L.hub_acc);
    a.hub_cnt = ws_ptr<int32_t>(ws, L.hub_cnt);
    a.hub_nparts = g->hub_nparts;
    a.hdr = ws_ptr<WsHeader>(ws, L.hdr);
    a.sleep_ns = debug_knob("PDNN_POLL_SLEEP_NS", 0);
    if (a.sleep_ns < 0) a.sleep_ns = 0;
    a.nowait = debug_knob("PDNN_SWEEP_NOWAIT", 0);
    a.trace = nullptr;
    if (debug_knob("PDNN_SWEEP_TRACE", 0)) {
        static unsigned long long* buf = nullptr;
        static size_t cap = 0;
        if (cap < 3 * (size_t)g->n_items) {
            if (buf) cudaFree(buf);
            cap = 3 * (size_t)g->n_items;
            if (cudaMalloc(&buf, 8 * cap) != cudaSuccess) { buf = nullptr; cap = 0; }
        }
        a.trace = buf;
        g_sweep_trace = buf;
    }
    void* args[] = {(void*)&a};
    const void* fn = lab_rank ? (const void*)k_sweep<true> : (const void*)k_sweep<false>;
    const int occ_max = sweep_occupancy(lab_rank != nullptr) * g->num_sms;
    const int knob = debug_knob("PDNN_SWEEP_CTAS", 0);
    const int grid = std::min(knob > 0 ? knob : g->sweep_grid, occ_max);
    PDNN_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kSweepThreads), args, kSweepSmem, s));
    count_launch();
    return PDNN_OK;
}

}  // namespace pdnn

using namespace pdnn;

// debug build (PDNN_SWEEP_TRACE=1): copy the last sweep's per-item stamps
// {start of the gathers, all inputs ready, published} (3 x n_items ns)
extern "C" int pdnn_debug_sweep_trace(unsigned long long* host, int64_t n) {
    if (!g_sweep_trace) return -1;
    return (int)cudaMemcpy(host, g_sweep_trace, 8 * (size_t)n, cudaMemcpyDeviceToHost);
}
extern "C" int pdnn_debug_sweep_items(const pdnn_graph* g, int32_t* host4) {   // NULL: the item count
    if (!host4) return g->n_items;
    return (int)cudaMemcpy(host4, g->items, sizeof(Item) * (size_t)g->n_items, cudaMemcpyDeviceToHost);
}
// the ranks listed by indexed items (kItemIndexed)
extern "C" int pdnn_debug_sweep_inodes(const pdnn_graph* g, int32_t* host) {
    if (!host) return g->n_inodes;
    return g->n_inodes ? (int)cudaMemcpy(host, g->inodes, 4 * (size_t)g->n_inodes, cudaMemcpyDeviceToHost) : 0;
}
// the same items in the order of the sweeps with REMOVED nodes (the K-loop)
extern "C" int pdnn_debug_sweep_items_rm(const pdnn_graph* g, int32_t* host4) {
    if (!host4) return g->n_items;
    return (int)cudaMemcpy(host4, g->items_rm, sizeof(Item) * (size_t)g->n_items, cudaMemcpyDeviceToHost);
}

extern "C" pdnn_status pdnn_weighted_levels(const pdnn_graph* g, const int64_t* node_cost,
                                            const int64_t* edge_cost, const int32_t* part, int64_t* tl,
                                            int64_t* bl, void* ws, size_t ws_bytes, void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (g->V > 0 && (!tl || !bl)) { set_error("null tl/bl"); return PDNN_EINVAL; }
    const WsLayout L = ws_layout(g, PDNN_OP_WEIGHTED_LEVELS, 0);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    pdnn_status st = ws_guard(ws, 0, 0, L.single_end, L.sig_single, s);
    if (st) return st;
    Costs C;
    if ((st = resolve_costs(g, node_cost, edge_cost, ws, L, s, &C, /*need_blob=*/true))) return st;
    // the labels go into rank space inside the sweep launch (lab_src)
    int32_t* pr = part ? ws_ptr<int32_t>(ws, L.part_rank) : nullptr;
    if (pr && debug_knob("PDNN_FUSED_LABELS", 1) == 0) {   // (debug build: the separate label launch)
        if ((st = launch_labels(g, part, nullptr, 0, nullptr, pr, s))) return st;
        return launch_sweep(g, C, pr, tl, bl, ws, L, s);
    }
    return launch_sweep(g, C, pr, tl, bl, ws, L, s, /*removal=*/false, part);
}
