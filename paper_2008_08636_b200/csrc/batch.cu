// batch.cu -- batched evaluation of candidate placements (§8(a) row a8):
// refinement / LALB trials scored by weighted levels,
// CP, cut communication and the memory tracker with st = tl under each
// candidate.
//
// Candidates are processed in groups of up to BLayout::ng (a multiple of 32,
// sized to the workspace budget).  Per group:
//   1. k_blabels + k_bsweep + k_bcp (bsweep.cu): ONE candidate-parallel
//      persistent launch computes tl / bl / the tight successors of every
//      candidate of the group (lane = candidate), then one warp per 32
//      candidates reduces L, the CP start, cut comm and walks the CP (on a
//      library side stream, overlapped with step 2, joined at the group end);
//   2. the memory tracker (memory.cu), segmented: up to kMemSegMax candidates
//      per launch sequence (prep, one cooperative segmented radix sort of the
//      sweep's st keys, positions, edge pass, per-PE scans);
//   3. k_eval_finish fills the overflow mask and the unused PE slots.
#include <cstdlib>
#include <mutex>

#include "internal.cuh"

namespace pdnn {

const SideStream* side_stream(int device) {
    static std::mutex mu;
    static SideStream ss[64];
    static int state[64] = {0};   // 0 untried, 1 ready, -1 failed
    if (device < 0 || device >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (state[device] == 0) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        const bool ok = cudaStreamCreateWithFlags(&ss[device].stream, cudaStreamNonBlocking) == cudaSuccess &&
                        cudaEventCreateWithFlags(&ss[device].ev_fork, cudaEventDisableTiming) == cudaSuccess &&
                        cudaEventCreateWithFlags(&ss[device].ev_join, cudaEventDisableTiming) == cudaSuccess;
        cudaSetDevice(prev);
        state[device] = ok ? 1 : -1;
        if (!ok) cudaGetLastError();
    }
    return state[device] == 1 ? &ss[device] : nullptr;
}

__global__ void k_eval_finish(int32_t P, pdnn_eval_result* __restrict__ out) {
    pdnn_eval_result* r = out + blockIdx.x;
    const int q = threadIdx.x;
    const bool over = q < P && r->first_over_pos[q] >= 0;
    const unsigned m = __ballot_sync(0xffffffffu, over);
    if (q == 0) r->overflow_mask = (int32_t)m;
    if (q >= P && q < PDNN_MAX_PE) {
        r->peak[q] = 0;
        r->over_bytes[q] = 0;
        r->peak_pos[q] = -1;
        r->first_over_pos[q] = -1;
    }
}

}  // namespace pdnn

using namespace pdnn;

extern "C" pdnn_status pdnn_eval_batch(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                                       const int64_t* mem, const uint8_t* kind, int32_t n_pe,
                                       const int64_t* cap_eff, int32_t batch, const uint8_t* parts,
                                       pdnn_eval_result* out, void* ws, size_t ws_bytes, void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (n_pe < 1 || n_pe > PDNN_MAX_PE || batch < 0) { set_error("bad n_pe / batch"); return PDNN_EINVAL; }
    if (batch > 0 && (!out || !cap_eff || (g->V > 0 && (!parts || !mem || !kind)))) {
        set_error("null argument");
        return PDNN_EINVAL;
    }
    if (g->V >= (1 << 30)) { set_error("batched evaluation needs n_nodes < 2^30"); return PDNN_EINVAL; }
    if (batch == 0) return PDNN_OK;
    const WsLayout L = ws_layout(g, PDNN_OP_EVAL_BATCH, batch);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    Costs C;
    pdnn_status st = resolve_costs(g, node_cost, edge_cost, ws, L, s, &C);
    if (st) return st;
    int64_t* keys = ws_ptr<int64_t>(ws, L.B.keys);
    const uint8_t* plab = ws_ptr<uint8_t>(ws, L.B.plab);
    static const bool no_mem = getenv("PDNN_BATCH_NO_MEM") != nullptr;   // probe: sweep + CP only
    for (int32_t b0 = 0; b0 < batch; b0 += L.B.ng) {
        const int32_t nb = std::min(L.B.ng, batch - b0);
        const SideStream* side = side_stream(g->device);
        if ((st = launch_bsweep(g, C, b0, nb, batch, parts, L.B, ws, out + b0, s, side))) return st;
        if (no_mem) {
            if (side) PDNN_CUDA_TRY(cudaStreamWaitEvent(s, side->ev_join, 0));
            continue;
        }
        // memory tracker on the sweep's st = tl keys, L.m_seg candidates per segmented launch
        for (int32_t j0 = 0; j0 < nb; j0 += L.m_seg) {
            const int32_t S = std::min(L.m_seg, nb - j0);
            MemIn in{};
            in.part_u8_rank = plab + (size_t)j0 * g->V;
            in.st_rank = keys + (size_t)j0 * g->V;
            MemWs M = mem_ws(ws, L);
            M.k0 = reinterpret_cast<uint64_t*>(keys + (size_t)j0 * g->V);   // sort the keys in place
            pdnn_eval_result* r = out + b0 + j0;
            MemOut o{r->peak, r->peak_pos, r->first_over_pos, r->over_bytes, sizeof(pdnn_eval_result) / 8,
                     sizeof(pdnn_eval_result) / 4};
            if ((st = launch_memory_seg(g, in, n_pe, S, mem, kind, cap_eff, nullptr, o, nullptr, M, s))) return st;
            k_eval_finish<<<S, 32, 0, s>>>(n_pe, r);
            count_launch();
            PDNN_LAUNCH_CHECK();
        }
        if (side) PDNN_CUDA_TRY(cudaStreamWaitEvent(s, side->ev_join, 0));   // join the CP walk
    }
    return PDNN_OK;
}
