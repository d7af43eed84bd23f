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
//      candidates reduces L, the CP start, cut comm and walks the CP;
//   2. the memory tracker (memory.cu) per candidate on the sweep's st keys;
//   3. k_eval_finish fills the overflow mask and the unused PE slots.
#include <cstdlib>

#include "internal.cuh"

namespace pdnn {

__global__ void k_eval_finish(int32_t P, pdnn_eval_result* __restrict__ r) {
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
    int32_t* po = ws_ptr<int32_t>(ws, L.part_o);
    int32_t* pr = ws_ptr<int32_t>(ws, L.part_rank);
    int64_t* mpot = ws_ptr<int64_t>(ws, L.mpot_s);
    const int64_t* keys = ws_ptr<int64_t>(ws, L.B.keys);
    for (int32_t b0 = 0; b0 < batch; b0 += L.B.ng) {
        const int32_t nb = std::min(L.B.ng, batch - b0);
        if ((st = launch_bsweep(g, C, b0, nb, batch, parts, L.B, ws, out + b0, s))) return st;
        static const bool no_mem = getenv("PDNN_BATCH_NO_MEM") != nullptr;   // probe: sweep + CP only
        for (int32_t j = 0; j < (no_mem ? 0 : nb); ++j) {
            const int32_t b = b0 + j;
            pdnn_eval_result* r = out + b;
            if ((st = launch_labels(g, nullptr, parts + (size_t)b * g->V, 0, po, pr, ws, L, s))) return st;
            if ((st = launch_memory(g, po, pr, n_pe, mem, kind, keys + (size_t)j * g->V, cap_eff, mpot, r->peak,
                                    r->peak_pos, r->first_over_pos, r->over_bytes, nullptr, ws, L, s, true)))
                return st;
            k_eval_finish<<<1, 32, 0, s>>>(n_pe, r);
            count_launch();
            PDNN_LAUNCH_CHECK();
        }
    }
    return PDNN_OK;
}
