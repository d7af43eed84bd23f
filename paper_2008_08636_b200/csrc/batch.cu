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
#include <vector>

#include "internal.cuh"

namespace pdnn {

namespace {
std::mutex g_side_mu;
std::vector<SideStream*> g_side_pool;   // idle side streams (all devices); they live for the process
}  // namespace

SideStream* side_acquire(int device) {
    {
        std::lock_guard<std::mutex> lock(g_side_mu);
        for (size_t i = 0; i < g_side_pool.size(); ++i)
            if (g_side_pool[i]->device == device) {
                SideStream* ss = g_side_pool[i];
                g_side_pool.erase(g_side_pool.begin() + (long)i);
                return ss;
            }
    }
    SideStream* ss = new (std::nothrow) SideStream();
    if (!ss) return nullptr;
    ss->device = device;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    const bool ok = cudaStreamCreateWithFlags(&ss->stream, cudaStreamNonBlocking) == cudaSuccess &&
                    cudaEventCreateWithFlags(&ss->ev_fork, cudaEventDisableTiming) == cudaSuccess &&
                    cudaEventCreateWithFlags(&ss->ev_join, cudaEventDisableTiming) == cudaSuccess;
    cudaSetDevice(prev);
    if (!ok) {
        cudaGetLastError();
        delete ss;
        return nullptr;
    }
    return ss;
}

void side_release(SideStream* ss) {
    if (!ss) return;
    std::lock_guard<std::mutex> lock(g_side_mu);
    g_side_pool.push_back(ss);
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
                                       pdnn_eval_result* out, int32_t schedule, void* ws, size_t ws_bytes,
                                       void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (n_pe < 1 || n_pe > PDNN_MAX_PE || batch < 0) { set_error("bad n_pe / batch"); return PDNN_EINVAL; }
    if (schedule != PDNN_SCHEDULE_LEVEL && schedule != PDNN_SCHEDULE_EMULATED) { set_error("bad schedule"); return PDNN_EINVAL; }
    const bool emulated = schedule == PDNN_SCHEDULE_EMULATED;
    if (batch > 0 && (!out || !cap_eff || (g->V > 0 && (!parts || !mem || !kind)))) {
        set_error("null argument");
        return PDNN_EINVAL;
    }
    // the tracker's sort packs a visit position as (pos << 5) | PE in 32 bits
    if (g->V >= (1 << 27)) { set_error("the memory tracker needs n_nodes < 2^27"); return PDNN_EINVAL; }
    if (batch == 0) return PDNN_OK;
    const WsLayout L = ws_layout(g, emulated ? PDNN_OP_EVAL_BATCH_EMULATED : PDNN_OP_EVAL_BATCH, batch);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    pdnn_status st = ws_guard(ws, 1, L.single_end, L.total, L.sig_batch, s);
    if (st) return st;
    Costs C;
    if ((st = resolve_costs(g, node_cost, edge_cost, ws, L, s, &C))) return st;
    int64_t* keys = ws_ptr<int64_t>(ws, L.B.keys);
    const uint8_t* plab = ws_ptr<uint8_t>(ws, L.B.plab);
    const bool no_mem = debug_knob("PDNN_BATCH_NO_MEM", 0) != 0;   // (debug build) sweep + CP only
    // the CP walk runs on a side stream checked out for this call only
    SideStream* side = side_acquire(g->device);
    struct Release { SideStream* s; ~Release() { side_release(s); } } release{side};
    for (int32_t b0 = 0; b0 < batch; b0 += L.B.ng) {
        const int32_t nb = std::min(L.B.ng, batch - b0);
        if ((st = launch_bsweep(g, C, b0, nb, batch, parts, L.B, ws, out + b0, s, side, !emulated))) return st;
        // the emulated FIFO schedule (R17) replaces the sweep's st = tl keys
        // (rank order, candidate-major) and reports the makespan
        if (emulated && (st = launch_emulate(g, C, nullptr, plab, n_pe, nb, ws_ptr<void>(ws, L.B.emu), nullptr,
                                              nullptr, keys, nullptr, out + b0, s)))
            return st;
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
