// batch.cu -- batched evaluation of candidate placements (§8(a) row a8):
// refinement / LALB trials scored by weighted levels,
// CP, cut communication and the memory tracker with st = tl under each
// candidate.  This first version streams the candidates through the
// single-graph kernels (sweep -> CP -> memory scan) back to back on the
// caller's stream; each stage is itself a full-GPU kernel.
#include "internal.cuh"

namespace pdnn {

__global__ void k_eval_finish(int32_t P, const int32_t* __restrict__ cp_nodes, const WsHeader* hdr,
                              pdnn_eval_result* __restrict__ r) {
    const int q = threadIdx.x;
    if (q == 0) {
        const uint32_t ep = *(volatile const uint32_t*)&hdr->epoch;
        r->cut_comm = (int64_t)hdr->cut[ep & 3];
        const int32_t n = r->cp_len;
        r->cp_start = n > 0 ? cp_nodes[0] : -1;
        r->cp_end = n > 0 ? cp_nodes[n - 1] : -1;
    }
    __syncthreads();
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
    const WsLayout L = ws_layout(g, PDNN_OP_EVAL_BATCH, batch);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    Costs C;
    pdnn_status st = resolve_costs(g, node_cost, edge_cost, ws, L, s, &C);
    if (st) return st;
    int32_t* po = ws_ptr<int32_t>(ws, L.part_o);
    int32_t* pr = ws_ptr<int32_t>(ws, L.part_rank);
    int64_t* tl = ws_ptr<int64_t>(ws, L.tl_o);
    int64_t* bl = ws_ptr<int64_t>(ws, L.bl_o);
    int32_t* cpn = ws_ptr<int32_t>(ws, L.cp_nodes);
    int64_t* mpot = ws_ptr<int64_t>(ws, L.mpot_s);
    const WsHeader* hdr = ws_ptr<WsHeader>(ws, L.hdr);
    for (int32_t b = 0; b < batch; ++b) {
        pdnn_eval_result* r = out + b;
        if ((st = launch_labels(g, nullptr, parts + (size_t)b * g->V, 0, po, pr, ws, L, s))) return st;
        if ((st = launch_sweep(g, C, pr, tl, bl, ws, L, s))) return st;
        if ((st = launch_cp(g, C, po, tl, bl, cpn, &r->cp_len, &r->L, &r->cp_hash, nullptr, nullptr, nullptr, ws, L, s)))
            return st;
        if ((st = launch_memory(g, po, pr, n_pe, mem, kind, tl, cap_eff, mpot, r->peak, r->peak_pos,
                                r->first_over_pos, r->over_bytes, nullptr, ws, L, s)))
            return st;
        k_eval_finish<<<1, 32, 0, s>>>(n_pe, cpn, hdr, r);
        count_launch();
        PDNN_LAUNCH_CHECK();
    }
    return PDNN_OK;
}
