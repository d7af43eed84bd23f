// overflow.cu -- the overflow handler of Memory Heuristic I:
// §8(f) NEXT row N3, in reading R20.
//
// "When the memory consumed exceeds the limit, we deal with the overflow as a
// 0-1 min-knapsack problem" (Eq. 4) with a_j = M_pot(n, t) and c_j = move_cost
// (Eq. 5); "the movement criteria is to pick the node that has the lowest
// move_cost / M_pot(n, t)"; nodes with M_pot > overflow also sit in a heap keyed
// by move_cost and the cheaper of the two tops is chosen; "the selected node is
// moved to another pe if the target pe has sufficient memory to accommodate
// that node memory potential.  Otherwise, the node is not considered again";
// "when a node is moved, the new potentials and memory consumption need to be
// recalculated".
//
// B200 design: the control is sequential (every
// move changes the schedule, the tracker and every potential), so the call is
// a host loop over the library's parallel kernels: per move a placement-aware
// sweep (st = tl, reading R8), the memory tracker with its M_cons matrix,
// M_pot(n, t) of every node at the overflow position (one thread per
// producer, atomics into its last consumer on the overflowing PE), and the
// dual-heap choice as one block-wide reduction (exact move_cost / M_pot
// ordering by 128-bit cross products).  The host reads back a few scalars per
// decision.  SYNCHRONOUS.
#include <algorithm>
#include <vector>

#include "internal.cuh"

namespace pdnn {

// M_pot(n, t) at visit position i on PE q for every node (orig order), R20
__global__ void k_mpot_at(int32_t V, int32_t q, int32_t i, const int32_t* __restrict__ orig,
                          const int32_t* __restrict__ out_off, const int32_t* __restrict__ out_dst,
                          const uint32_t* __restrict__ pp, const int32_t* __restrict__ part,
                          const int64_t* __restrict__ mem, const uint8_t* __restrict__ kind,
                          unsigned long long* __restrict__ a) {
    for (int32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < V; r += gridDim.x * blockDim.x) {
        const int32_t p = orig[r];
        const uint32_t me = pp[r];
        const int32_t pos = (int32_t)(me >> 5);
        const int kd = kind[p];
        if (pos == i && part[p] == q && kd != PDNN_KIND_REFERENCE) atomicAdd(&a[p], (unsigned long long)mem[p]);
        if (pos > i || kd == PDNN_KIND_REFERENCE || (kd == PDNN_KIND_RESIDUAL && part[p] == q)) continue;
        int32_t last = -1, lpos = -1;
        for (int32_t e = out_off[r]; e < out_off[r + 1]; ++e) {
            const uint32_t x = pp[out_dst[e]];
            if ((int32_t)(x & 31u) == q && (int32_t)(x >> 5) > lpos) { lpos = (int32_t)(x >> 5); last = out_dst[e]; }
        }
        if (last >= 0 && lpos >= i) atomicAdd(&a[orig[last]], (unsigned long long)mem[p]);
    }
}

struct Pick {
    int32_t A, B;         // -1: none
    int64_t cA, aA, cB, aB;
};

__device__ __forceinline__ bool ratio_less(int64_t c1, int64_t a1, int32_t n1, int64_t c2, int64_t a2, int32_t n2) {
    if (n2 < 0) return true;
    const __int128 x = (__int128)c1 * a2, y = (__int128)c2 * a1;
    return x < y || (x == y && n1 < n2);
}
__device__ __forceinline__ bool cost_less(int64_t c1, int32_t n1, int64_t c2, int32_t n2) {
    return n2 < 0 || c1 < c2 || (c1 == c2 && n1 < n2);
}

// the two heap tops over the candidates (one CTA): A = min move_cost / M_pot,
// B = min move_cost among M_pot > O (ties by id); move_cost (Eq. 5) = comp(n) +
// the comm of n's edges to predecessors and successors on q
constexpr int kPickThreads = 1024;
__global__ void __launch_bounds__(kPickThreads) k_overflow_pick(
    int32_t V, int32_t q, int64_t O, const int32_t* __restrict__ rank_of, const int32_t* __restrict__ in_off,
    const int32_t* __restrict__ in_src, const int32_t* __restrict__ out_off, const int32_t* __restrict__ out_dst,
    const int64_t* __restrict__ c_rank, const int64_t* __restrict__ in_cost, const int64_t* __restrict__ out_cost,
    const int32_t* __restrict__ part_rank, const int32_t* __restrict__ part, const uint8_t* __restrict__ kind,
    const uint8_t* __restrict__ excl, const unsigned long long* __restrict__ a, Pick* out) {
    __shared__ Pick s_p[kPickThreads / 32];
    Pick m{-1, -1, 0, 0, 0, 0};
    for (int32_t n = threadIdx.x; n < V; n += kPickThreads) {
        if (part[n] != q || kind[n] != PDNN_KIND_NORMAL || excl[n] || a[n] == 0) continue;
        const int64_t an = (int64_t)a[n];
        const int32_t r = rank_of[n];
        int64_t cost = c_rank[r];
        for (int32_t e = in_off[r]; e < in_off[r + 1]; ++e)
            if (part_rank[in_src[e]] == q) cost += in_cost[e];
        for (int32_t e = out_off[r]; e < out_off[r + 1]; ++e)
            if (part_rank[out_dst[e]] == q) cost += out_cost[e];
        if (ratio_less(cost, an, n, m.cA, m.aA, m.A)) { m.A = n; m.cA = cost; m.aA = an; }
        if (an > O && cost_less(cost, n, m.cB, m.B)) { m.B = n; m.cB = cost; m.aB = an; }
    }
    auto merge = [](Pick& x, const Pick& y) {
        if (y.A >= 0 && ratio_less(y.cA, y.aA, y.A, x.cA, x.aA, x.A)) { x.A = y.A; x.cA = y.cA; x.aA = y.aA; }
        if (y.B >= 0 && cost_less(y.cB, y.B, x.cB, x.B)) { x.B = y.B; x.cB = y.cB; x.aB = y.aB; }
    };
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Pick y;
        y.A = __shfl_xor_sync(0xffffffffu, m.A, o);
        y.B = __shfl_xor_sync(0xffffffffu, m.B, o);
        y.cA = __shfl_xor_sync(0xffffffffu, m.cA, o);
        y.aA = __shfl_xor_sync(0xffffffffu, m.aA, o);
        y.cB = __shfl_xor_sync(0xffffffffu, m.cB, o);
        y.aB = __shfl_xor_sync(0xffffffffu, m.aB, o);
        merge(m, y);
    }
    if ((threadIdx.x & 31) == 0) s_p[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        Pick x = s_p[0];
        for (int w = 1; w < kPickThreads / 32; ++w) merge(x, s_p[w]);
        *out = x;
    }
}

// M_cons(k, i) for every PE k (one column of the [P][V] matrix)
__global__ void k_mcons_col(int32_t P, int32_t V, int32_t i, const int64_t* __restrict__ mcons, int64_t* __restrict__ col) {
    if ((int)threadIdx.x < P) col[threadIdx.x] = mcons[(size_t)threadIdx.x * V + i];
}

}  // namespace pdnn

using namespace pdnn;

extern "C" pdnn_status pdnn_resolve_overflow(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                                             const int64_t* mem, const uint8_t* kind, int32_t n_pe,
                                             const int64_t* cap_eff_host, int32_t* part, int32_t max_moves,
                                             int32_t* moves_host, int32_t* n_moves, int32_t* resolved, void* ws,
                                             size_t ws_bytes, void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (n_pe < 1 || n_pe > PDNN_MAX_PE || max_moves < 0 || !cap_eff_host || !n_moves || !resolved ||
        (max_moves > 0 && !moves_host) || (g->V > 0 && (!part || !mem || !kind))) {
        set_error("bad argument");
        return PDNN_EINVAL;
    }
    if (g->V >= (1 << 27)) { set_error("the memory tracker needs n_nodes < 2^27"); return PDNN_EINVAL; }
    const WsLayout L = ws_layout(g, PDNN_OP_RESOLVE_OVERFLOW, 0);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    pdnn_status st = ws_guard(ws, 0, 0, L.single_end, L.sig_single, s);
    if (st) return st;
    // the scratch sits where a batched evaluation keeps its state: claim the
    // region (its next batched call sees another layout and starts fresh)
    if ((st = ws_guard(ws, 1, L.single_end, L.total, L.sig_batch, s))) return st;
    *n_moves = 0;
    *resolved = 0;
    const int32_t V = g->V, P = n_pe;
    if (V == 0) { *resolved = 1; return PDNN_OK; }
    Costs C;
    if ((st = resolve_costs(g, node_cost, edge_cost, ws, L, s, &C, /*need_blob=*/true))) return st;
    int32_t* pr = ws_ptr<int32_t>(ws, L.part_rank);
    int64_t* tl = ws_ptr<int64_t>(ws, L.tl_o);
    int64_t* bl = ws_ptr<int64_t>(ws, L.bl_o);
    int64_t* mpot = ws_ptr<int64_t>(ws, L.mpot_s);
    int64_t* mcons = ws_ptr<int64_t>(ws, L.ov_mcons);
    unsigned long long* a = ws_ptr<unsigned long long>(ws, L.ov_a);
    uint8_t* excl = ws_ptr<uint8_t>(ws, L.ov_excl);
    int64_t* small = ws_ptr<int64_t>(ws, L.ov_small);     // cap[16] peak[16] over[16] col[16]
    int32_t* small32 = ws_ptr<int32_t>(ws, L.ov_small + 64 * 8);   // ppos[16] fo[16]
    Pick* pick = ws_ptr<Pick>(ws, L.ov_small + 96 * 8);
    const MemWs M = mem_ws(ws, L);
    PDNN_CUDA_TRY(cudaMemcpyAsync(small, cap_eff_host, 8 * (size_t)P, cudaMemcpyHostToDevice, s));
    PDNN_CUDA_TRY(cudaMemsetAsync(excl, 0, (size_t)V, s));
    const int grid = std::max(1, std::min(ceil_div(V, 256), g->num_sms * 8));
    int32_t nm = 0;
    for (;;) {
        // schedule (st = tl under the current placement, R8) and the tracker
        if ((st = launch_labels(g, part, nullptr, 0, nullptr, pr, s))) return st;
        if ((st = launch_sweep(g, C, pr, tl, bl, ws, L, s))) return st;
        if ((st = launch_memory(g, part, pr, P, mem, kind, tl, small, mpot, small + 16, small32, small32 + 16,
                                small + 32, mcons, ws, L, s)))
            return st;
        int32_t fo[PDNN_MAX_PE];
        int64_t over[PDNN_MAX_PE];
        PDNN_CUDA_TRY(cudaMemcpyAsync(fo, small32 + 16, 4 * (size_t)P, cudaMemcpyDeviceToHost, s));
        PDNN_CUDA_TRY(cudaMemcpyAsync(over, small + 32, 8 * (size_t)P, cudaMemcpyDeviceToHost, s));
        PDNN_CUDA_TRY(cudaStreamSynchronize(s));
        int32_t q = -1;
        for (int32_t k = 0; k < P; ++k)
            if (fo[k] >= 0 && (q < 0 || fo[k] < fo[q])) q = k;
        if (q < 0) { *resolved = 1; break; }
        if (nm >= max_moves) break;
        const int32_t i = fo[q];
        const int64_t O = over[q];
        // M_pot(n, t) at the overflow, and M_cons(k, t) of every PE
        PDNN_CUDA_TRY(cudaMemsetAsync(a, 0, 8 * (size_t)V, s));
        k_mpot_at<<<grid, 256, 0, s>>>(V, q, i, g->orig, g->out_off, g->out_dst, M.pp, part, mem, kind, a);
        count_launch();
        k_mcons_col<<<1, 32, 0, s>>>(P, V, i, mcons, small + 48);
        count_launch();
        PDNN_LAUNCH_CHECK();
        int64_t col[PDNN_MAX_PE];
        PDNN_CUDA_TRY(cudaMemcpyAsync(col, small + 48, 8 * (size_t)P, cudaMemcpyDeviceToHost, s));
        bool moved = false;
        for (;;) {
            k_overflow_pick<<<1, kPickThreads, 0, s>>>(V, q, O, g->rank_of, g->in_off, g->in_src, g->out_off,
                                                       g->out_dst, C.c, C.in_cost, C.out_cost, pr, part, kind, excl,
                                                       a, pick);
            count_launch();
            PDNN_LAUNCH_CHECK();
            Pick h;
            PDNN_CUDA_TRY(cudaMemcpyAsync(&h, pick, sizeof(Pick), cudaMemcpyDeviceToHost, s));
            PDNN_CUDA_TRY(cudaStreamSynchronize(s));
            if (h.A < 0) break;                                      // run out of nodes
            const bool useB = h.B >= 0 && h.cB < h.cA;
            const int32_t n = useB ? h.B : h.A;
            const int64_t an = useB ? h.aB : h.aA;
            int32_t tgt = -1;
            for (int32_t k = 0; k < P; ++k) {
                if (k == q) continue;
                if (col[k] + an <= cap_eff_host[k] && (tgt < 0 || col[k] < col[tgt])) tgt = k;
            }
            const uint8_t one = 1;
            PDNN_CUDA_TRY(cudaMemcpyAsync(excl + n, &one, 1, cudaMemcpyHostToDevice, s));   // never considered again
            if (nm >= max_moves) break;
            moves_host[3 * nm] = n;
            moves_host[3 * nm + 1] = q;
            moves_host[3 * nm + 2] = tgt;
            ++nm;
            if (tgt >= 0) {
                PDNN_CUDA_TRY(cudaMemcpyAsync(part + n, &tgt, 4, cudaMemcpyHostToDevice, s));
                moved = true;
                break;
            }
        }
        if (!moved) break;
    }
    PDNN_CUDA_TRY(cudaStreamSynchronize(s));
    *n_moves = nm;
    return PDNN_OK;
}
