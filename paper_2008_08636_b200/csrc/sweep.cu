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
#include <cstdlib>

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
    uint64_t* nrec;       // 32 B per rank: {tagged tl+comp, label, tagged bl, label}
    int64_t* tl_out;      // node-id order (nullable)
    int64_t* bl_out;
    unsigned long long* hub_acc;
    int32_t* hub_cnt;
    const int32_t* hub_nparts;
    WsHeader* hdr;
    int32_t sleep_ns;      // poll back-off (PDNN_POLL_SLEEP_NS, default 20)
    int32_t count_spins;   // PDNN_SWEEP_STATS=1: count failed polls into hdr->misc
};

// ---------------------------------------------------------------- TMA staging
// Each warp owns kStages stage buffers in shared memory.  Two items ahead of
// the one it processes, lane 0 issues 1-D bulk copies (cp.async.bulk, the TMA
// engine) of the item's static slices -- offsets, neighbour ids, edge costs,
// node costs, original ids, labels: all contiguous ranges in rank space --
// completing on the stage's mbarrier.  Copies are widened to 16-byte
// boundaries; the consumer indexes past the head misalignment.
constexpr int kStages = 2;
constexpr int kOffB = 192, kNbrB = 544, kEcB = 1056, kCB = 288, kOrigB = 160, kPartB = 160, kHdrB = 48;
constexpr int kRegShift = 16;   // int32[6]: head misalignment of each slice, written by its issuing lane
constexpr int kRegHdr = 0, kRegOff = kHdrB, kRegNbr = kRegOff + kOffB, kRegEc = kRegNbr + kNbrB, kRegC = kRegEc + kEcB,
              kRegOrig = kRegC + kCB, kRegPart = kRegOrig + kOrigB, kStageBytes = kRegPart + kPartB;
constexpr int kWarpsPerCta = kSweepThreads / 32;
constexpr int kSweepSmem = kWarpsPerCta * kStages * kStageBytes;
static_assert(kStageBytes % 16 == 0, "stage alignment");
static_assert(kTMaxEdges * 8 + 16 <= kEcB && kTMaxEdges * 4 + 16 <= kNbrB, "stage sizes");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
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
// The static slices are streamed once per sweep: L2 evict-first, so they do
// not push the node records (gathered and polled all sweep long) out of L2.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    const uint64_t pol = l2_evict_first_policy();
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

struct Slice {  // a 16-byte-widened copy of elements [a, b)
    const char* src;
    uint32_t bytes;
    int32_t shift;  // elements of head misalignment
};
__device__ __forceinline__ Slice make_slice(const void* base, int32_t a, int32_t b, int esize) {
    const uintptr_t s0 = (uintptr_t)base + (uintptr_t)a * esize;
    const uintptr_t s1 = (uintptr_t)base + (uintptr_t)b * esize;
    const uintptr_t lo = s0 & ~(uintptr_t)15, hi = (s1 + 15) & ~(uintptr_t)15;
    Slice sl;
    sl.src = (const char*)lo;
    sl.bytes = b > a ? (uint32_t)(hi - lo) : 0u;
    sl.shift = (int32_t)((s0 - lo) / esize);
    return sl;
}

// per-item slice geometry (computed by the issuing lane; the consumers read the
// head misalignments from the stage header)
template <bool HAS_PART>
struct ItemSlices {
    Slice off, nbr, ec, c, orig, part;
    __device__ __forceinline__ ItemSlices(const SweepArgs& a, const Item& it) {
        const bool fwd = it.x >= 0;
        const int32_t r0 = fwd ? it.x : ~it.x;
        off = make_slice(fwd ? a.in_off : a.out_off, r0, r0 + it.y + 1, 4);
        nbr = make_slice(fwd ? a.in_src : a.out_dst, it.z, it.w, 4);
        ec = make_slice(fwd ? a.in_cost : a.out_cost, it.z, it.w, 8);
        c = make_slice(a.c, r0, r0 + it.y, 8);
        orig = make_slice(a.orig, r0, r0 + it.y, 4);
        if (HAS_PART) part = make_slice(a.part, r0, r0 + it.y, 4);
        else part.bytes = 0, part.shift = 0, part.src = nullptr;
    }
};

// Lane 0 issues the item's bulk copies (cp.async.bulk takes uniform operands:
// spreading the six copies over six lanes serialises them and measured 20 %
// slower on C4) and records each slice's head misalignment in the stage
// header, so the consumer lanes do not recompute the geometry.
template <bool HAS_PART>
__device__ __forceinline__ void issue_item(const SweepArgs& a, const Item& it, unsigned char* stage, uint64_t* bar) {
    *reinterpret_cast<Item*>(stage + kRegHdr) = it;   // the consumer reads its descriptor from here
    if (it.y <= 0) {  // warp items read global memory directly; just complete the phase
        mbar_arrive_expect_tx(bar, 0);
        return;
    }
    const ItemSlices<HAS_PART> sl(a, it);
    int4 sh4;
    sh4.x = sl.off.shift; sh4.y = sl.nbr.shift; sh4.z = sl.ec.shift; sh4.w = sl.c.shift;
    *reinterpret_cast<int4*>(stage + kRegShift) = sh4;
    *reinterpret_cast<int2*>(stage + kRegShift + 16) = make_int2(sl.orig.shift, sl.part.shift);
    mbar_arrive_expect_tx(bar, sl.off.bytes + sl.nbr.bytes + sl.ec.bytes + sl.c.bytes + sl.orig.bytes + sl.part.bytes);
    tma_load_1d(stage + kRegOff, sl.off.src, sl.off.bytes, bar);
    if (sl.nbr.bytes) {
        tma_load_1d(stage + kRegNbr, sl.nbr.src, sl.nbr.bytes, bar);
        tma_load_1d(stage + kRegEc, sl.ec.src, sl.ec.bytes, bar);
    }
    tma_load_1d(stage + kRegC, sl.c.src, sl.c.bytes, bar);
    tma_load_1d(stage + kRegOrig, sl.orig.src, sl.orig.bytes, bar);
    if (HAS_PART) tma_load_1d(stage + kRegPart, sl.part.src, sl.part.bytes, bar);
}

// One warp-synchronous batch of up to 4 edges per lane: edge k of lane l is
// e + k*step (live if < t); NB/EC are the neighbour / cost arrays (global or a
// stage buffer, indexed relative to their own base).  Every live neighbour
// value is requested at once together with its label, and the warp re-polls
// only the values whose tag is not yet this sweep's, in a loop whose condition
// is warp-uniform (__any_sync), so the warp never serialises lanes.
template <bool HAS_PART>
__device__ __forceinline__ void relax_batch(const int32_t* nbr, const int64_t* ec,
                                            const uint64_t* val,
                                            int32_t pv, int32_t e, int32_t t, int32_t step, uint64_t tag,
                                            int64_t& best, int64_t& cut, int32_t sleep_ns, int32_t& spins) {
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
    // value and label share one 16-byte record half: a single gather per edge
    uint64_t x[4], lw[4];
    int32_t pp[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = lw[k] = 0;
    // every load of the batch is issued before the first use
    if (HAS_PART)
        ld_relaxed_v2u64_x4(x, lw, &val[4 * (size_t)nb[0]], &val[4 * (size_t)nb[1]], &val[4 * (size_t)nb[2]],
                            &val[4 * (size_t)nb[3]], live[0], live[1], live[2], live[3]);
    else
        ld_relaxed_u64_x4(x, &val[4 * (size_t)nb[0]], &val[4 * (size_t)nb[1]], &val[4 * (size_t)nb[2]],
                          &val[4 * (size_t)nb[3]], live[0], live[1], live[2], live[3]);
    // the label word's high half is always 0; OR-ing it in keeps the whole
    // 16-byte destination live until the load retires (otherwise ptxas reuses
    // the dead high register at once and the warp stalls on the WAW hazard)
#pragma unroll
    for (int k = 0; k < 4; ++k) pp[k] = (int32_t)(uint32_t)(lw[k] | (lw[k] >> 32));
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
        rdy[k] = !live[k] || (x[k] & ~kValMask) == tag || sleep_ns == -7;   // -7: timing probe, no waits
    }
    int32_t ns = sleep_ns > 0 ? sleep_ns : 0;   // < 0: exponential back-off from 32 ns up to -sleep_ns
    while (__any_sync(0xffffffffu, !(rdy[0] && rdy[1] && rdy[2] && rdy[3]))) {
        ++spins;
        if (ns > 0) __nanosleep(ns);
        if (sleep_ns < 0) ns = ns == 0 ? 32 : (ns < -sleep_ns ? 2 * ns : ns);   // exponential back-off
        ld_relaxed_u64_x4(x, &val[4 * (size_t)nb[0]], &val[4 * (size_t)nb[1]], &val[4 * (size_t)nb[2]],
                          &val[4 * (size_t)nb[3]], !rdy[0], !rdy[1], !rdy[2], !rdy[3]);
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

template <bool HAS_PART>
__device__ __forceinline__ void store_node(const SweepArgs& a, bool fwd, int32_t v, int32_t ov, int64_t c,
                                           int64_t best, uint64_t tag, int64_t& lmax) {
    if (fwd) {
        const int64_t tlc = best + c;
        st_relaxed_u64(&a.nrec[4 * (size_t)v], tag | (uint64_t)tlc);
        if (a.tl_out) a.tl_out[ov] = best;
        lmax = tlc > lmax ? tlc : lmax;
    } else {
        const int64_t b = c + best;
        st_relaxed_u64(&a.nrec[4 * (size_t)v + 2], tag | (uint64_t)b);
        if (a.bl_out) a.bl_out[ov] = b;
    }
}

template <bool HAS_PART, bool STATS>
__global__ void __launch_bounds__(kSweepThreads, 2) k_sweep(SweepArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_bar[kWarpsPerCta][kStages];
    __shared__ uint8_t s_own[kWarpsPerCta][32];   // thread items: lane -> (node, chunk)
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
    __syncthreads();
    const uint64_t tag = (uint64_t)s_tag << 62;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    unsigned char* wsm = smem + (size_t)wic * kStages * kStageBytes;
    int64_t lmax = 0, cut = 0;
    int32_t spins = 0;
    long long t_start = STATS ? clock64() : 0, t_wait = 0, t_proc = 0, t_split = 0, t_relax = 0, t_tail = 0;

    // prologue: stage the first kStages-1 items of this warp.  Descriptors are
    // loaded one iteration before they are issued, so no dependent global load
    // sits on the per-item path.
    auto desc = [&](int32_t i) {
        Item d;
        if (i < a.n_items) d = a.items[i];
        else d.x = d.y = d.z = d.w = 0;
        return d;
    };
    for (int k = 0; k < kStages - 1; ++k) {
        const int32_t i = gw + k * nw;
        const Item d = desc(i);
        if (lane == 0 && i < a.n_items) issue_item<HAS_PART>(a, d, wsm + k * kStageBytes, &s_bar[wic][k]);
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
            if (lane == 0 && inext < a.n_items) issue_item<HAS_PART>(a, nd, wsm + sn * kStageBytes, &s_bar[wic][sn]);
            nd = desc(inext + nw);   // consumed at the next iteration
        }
        const Item it = *reinterpret_cast<const Item*>(wsm + st * kStageBytes + kRegHdr);
        const bool fwd = it.x >= 0;
        const int32_t r0 = fwd ? it.x : ~it.x;
        const uint64_t* val = a.nrec + (fwd ? 0 : 2);
        long long tw0 = STATS ? clock64() : 0;
        mbar_wait(&s_bar[wic][st], (uint32_t)((k / kStages) & 1));
        if (STATS) { const long long t = clock64(); t_wait += t - tw0; tw0 = t; }
        if (it.y > 0) {
            // thread-per-node item from the stage buffer: lane j owns node r0 + j
            const unsigned char* sb = wsm + st * kStageBytes;
            const int32_t* shf = reinterpret_cast<const int32_t*>(sb + kRegShift);
            const int32_t* sOff = reinterpret_cast<const int32_t*>(sb + kRegOff) + shf[0];
            const int32_t* sNbr = reinterpret_cast<const int32_t*>(sb + kRegNbr) + shf[1];
            const int64_t* sEc = reinterpret_cast<const int64_t*>(sb + kRegEc) + shf[2];
            const int64_t* sC = reinterpret_cast<const int64_t*>(sb + kRegC) + shf[3];
            const int32_t* sOrig = reinterpret_cast<const int32_t*>(sb + kRegOrig) + shf[4];
            const int32_t* sPart = reinterpret_cast<const int32_t*>(sb + kRegPart) + (HAS_PART ? shf[5] : 0);
            // lanes <-> (node, chunk of <= 4 edges): a node of degree > 4 gets a
            // second lane, so every lane relaxes at most 4 edges and the whole
            // item takes ONE batch of gathers (one round trip) instead of two
            const int n = it.y;
            const bool nact = lane < n;
            const int32_t ndeg = nact ? sOff[lane + 1] - sOff[lane] : 0;
            const unsigned big = __ballot_sync(0xffffffffu, ndeg > 4);
            uint8_t* own = s_own[wic];
            if (nact) {
                const int f = lane + __popc(big & ((1u << lane) - 1u));
                own[f] = (uint8_t)lane;
                if (ndeg > 4) own[f + 1] = (uint8_t)(lane | 0x80);
            }
            const int nl = n + __popc(big);
            __syncwarp();
            const bool act = lane < nl;
            const int o = act ? own[lane] : 0;
            const int j = o & 31, chunk = o >> 7;
            const int32_t pv = (HAS_PART && act) ? sPart[j] : 0;
            const bool removed = HAS_PART && act && pv == PDNN_REMOVED;
            const int32_t e0 = act ? sOff[j] - it.z + 4 * chunk : 0;
            const int32_t e1 = (act && !removed) ? min(sOff[j + 1] - it.z, e0 + 4) : e0;
            int64_t best = 0, c2 = 0;
            long long tr0 = STATS ? clock64() : 0;
            if (STATS) t_split += tr0 - tw0;
            relax_batch<HAS_PART>(sNbr, sEc, val, pv, e0, e1, 1, tag, best, c2, a.sleep_ns, spins);
            if (STATS) { const long long t = clock64(); t_relax += t - tr0; tr0 = t; }
            if (!fwd) cut += c2;
            // the second chunk's maximum joins its node's first lane
            const int64_t best2 = __shfl_down_sync(0xffffffffu, best, 1);
            const bool first = act && chunk == 0;
            if (first && sOff[j + 1] - sOff[j] > 4) best = best2 > best ? best2 : best;
            if (first) {
                const int32_t v = r0 + j;
                if (removed) {
                    st_relaxed_u64(&a.nrec[4 * (size_t)v + (fwd ? 0 : 2)], tag);
                    int64_t* out = fwd ? a.tl_out : a.bl_out;
                    if (out) out[sOrig[j]] = -1;
                } else {
                    store_node<HAS_PART>(a, fwd, v, sOrig[j], sC[j], best, tag, lmax);
                }
            }
        } else {
            // warp item: edges [z, w) of node r0 (a hub part if y < 0), from global memory
            const int32_t* off = fwd ? a.in_off : a.out_off;
            const int32_t* nbr = fwd ? a.in_src : a.out_dst;
            const int64_t* ec = fwd ? a.in_cost : a.out_cost;
            const int32_t v = r0;
            const int32_t pv = HAS_PART ? __ldg(&a.part[v]) : 0;
            if (HAS_PART && pv == PDNN_REMOVED) {
                if (lane == 0 && it.z == __ldg(&off[v])) {
                    st_relaxed_u64(&a.nrec[4 * (size_t)v + (fwd ? 0 : 2)], tag);
                    int64_t* out = fwd ? a.tl_out : a.bl_out;
                    if (out) out[a.orig[v]] = -1;
                }
            } else {
                int64_t best = 0, c2 = 0;
                for (int32_t e0 = it.z; e0 < it.w; e0 += 4 * 32)   // warp-uniform trip count
                    relax_batch<HAS_PART>(nbr, ec, val, pv, e0 + lane, it.w, 32, tag, best, c2, a.sleep_ns, spins);
                if (!fwd) cut += c2;
                best = warp_max_i64(best);
                if (lane == 0) {
                    bool fin = it.y == 0;
                    if (!fin) {
                        const int slot = -it.y - 1;
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
                    if (fin) store_node<HAS_PART>(a, fwd, v, a.orig[v], a.c[v], best, tag, lmax);
                }
            }
        }
        if (STATS) t_proc += clock64() - tw0;
        if (STATS && it.y > 0) t_tail += 0;   // (tail = proc - split - relax)
        __syncwarp();   // the stage is re-filled at the next iteration
    }
    lmax = warp_max_i64(lmax);
    cut = warp_sum_i64(cut);
    if (STATS && lane == 0) {
        atomicAdd(&a.hdr->misc[0], (unsigned long long)spins);           // warp-level failed polls
        atomicAdd(&a.hdr->misc[1], (unsigned long long)(clock64() - t_start));  // warp busy cycles
        atomicAdd(&a.hdr->misc[2], 1ull);
        atomicAdd(&a.hdr->misc[3], (unsigned long long)t_wait);   // cycles in TMA stage waits
        atomicAdd(&a.hdr->misc[4], (unsigned long long)t_proc);   // cycles processing items
        atomicAdd(&a.hdr->misc[5], (unsigned long long)t_split);  // thread items: TMA ready -> gathers issued
        atomicAdd(&a.hdr->misc[6], (unsigned long long)t_relax);  // thread items: gathers + polls + max
        (void)t_tail;
    }
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

// resident CTAs per SM of one kernel variant (the cooperative grid size)
static int occ_of(const void* fn) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSweepSmem);
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, kSweepThreads, kSweepSmem);
    return n < 1 ? 1 : n;
}

// CTAs per SM of the production variants (the graph's sweep grid).  Deep,
// narrow graphs are bound by the dependency chain, and extra warps only spin:
// capped at 2 CTAs/SM (C3 3.21 ms at 2 vs 3.78 at 3, C2 1.07 vs 1.17).  Wide
// graphs (>= kWideLevel nodes per level on average) are bound by throughput
// and take every resident CTA (C4 0.213 -> 0.195 ms; round-1 measurements).
constexpr int kSweepCtasPerSmDeep = 2;
constexpr int kWideLevel = 2048;
int sweep_blocks_per_sm(int device, int32_t V, int32_t D) {
    (void)device;
    const int a = occ_of((const void*)k_sweep<true, false>), b = occ_of((const void*)k_sweep<false, false>);
    const int n = a < b ? a : b;
    const bool wide = D > 0 && (int64_t)V >= (int64_t)kWideLevel * D;
    return wide || n < kSweepCtasPerSmDeep ? n : kSweepCtasPerSmDeep;
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
    a.nrec = ws_ptr<uint64_t>(ws, L.nrec);
    a.tl_out = tl;
    a.bl_out = bl;
    a.hub_acc = ws_ptr<unsigned long long>(ws, L.hub_acc);
    a.hub_cnt = ws_ptr<int32_t>(ws, L.hub_cnt);
    a.hub_nparts = g->hub_nparts;
    a.hdr = ws_ptr<WsHeader>(ws, L.hdr);
    static const int sleep_env = getenv("PDNN_POLL_SLEEP_NS") ? atoi(getenv("PDNN_POLL_SLEEP_NS")) : 0;
    static const int stats_env = getenv("PDNN_SWEEP_STATS") ? atoi(getenv("PDNN_SWEEP_STATS")) : 0;
    a.sleep_ns = sleep_env;
    a.count_spins = stats_env;
    void* args[] = {(void*)&a};
    const void* fn = part_rank ? (stats_env ? (const void*)k_sweep<true, true> : (const void*)k_sweep<true, false>)
                               : (stats_env ? (const void*)k_sweep<false, true> : (const void*)k_sweep<false, false>);
    static const int ctas_env = getenv("PDNN_SWEEP_CTAS") ? atoi(getenv("PDNN_SWEEP_CTAS")) : 0;
    static const int stats_grid = stats_env ? occ_of(fn) * g->num_sms : 0;   // instrumented variants may fit fewer CTAs
    const int full = stats_env ? std::min(stats_grid, g->sweep_grid) : g->sweep_grid;
    static const int occ_max = occ_of(fn) * g->num_sms;   // experiment knob may exceed the default cap
    const int grid = ctas_env > 0 ? std::min(ctas_env, occ_max) : full;
    PDNN_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kSweepThreads), args, kSweepSmem, s));
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
        if ((st = launch_labels(g, part, nullptr, 0, nullptr, pr, ws, L, s))) return st;
    }
    return launch_sweep(g, C, pr, tl, bl, ws, L, s);
}
