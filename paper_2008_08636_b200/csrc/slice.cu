// slice.cu -- the whole of Alg. 1 (graph slicing) and the
// criticality of linear clusters: §8(f) NEXT row N2.
//
//   primaries   the K-loop of pdnn_slice (sweep -> CP -> removal, reading R4),
//               each CP appended as cluster j;
//   priorities  one more sweep on G minus the primaries: the stale w_lvl =
//               tl + bl of the secondary phase ("we stop recalculating",
//               PAPER.md:267);
//   secondaries find_heaviest_path with those priorities until every node is
//               in a cluster (reading R18: start = the unvisited node of
//               maximum w_lvl, lowest id on ties; forward by the unvisited
//               successor of maximum w_lvl, then backward from the start by
//               the unvisited predecessor of maximum w_lvl).
//
// B200 design: the sweeps and CPs are the
// library's parallel kernels; the start order is one radix sort of the
// priorities (CUB, a library sort of V keys once per call); the extraction is
// a greedy walk whose every step depends on the previous one (a path may not
// reuse a node an earlier step took), so it runs as ONE warp: the lanes scan
// the current node's neighbours and reduce the highest-priority unvisited one.
// Criticality: a sweep with labels = cluster ids (intra-cluster comm zero, R2)
// and a per-cluster max of tl + bl (reading R19).
#include <cub/device/device_radix_sort.cuh>

#include "internal.cuh"

namespace pdnn {

// CP j (cp_nodes[0, *cp_len)) becomes cluster j: members at the running offset
__global__ void k_append_cluster(const int32_t* __restrict__ cp, const int32_t* __restrict__ cp_len, int32_t j,
                                 int32_t* __restrict__ cluster_of, int32_t* __restrict__ members,
                                 int32_t* __restrict__ cl_off, int32_t* __restrict__ ctl) {
    const int32_t n = *cp_len, m = ctl[0];
    for (int32_t k = threadIdx.x; k < n; k += blockDim.x) {
        const int32_t u = cp[k];
        members[m + k] = u;
        cluster_of[u] = j;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ctl[0] = m + n;
        cl_off[j + 1] = m + n;
    }
}

// sort keys of the secondary phase: alive nodes by w_lvl descending (then id:
// the radix sort is stable over the id order); primaries last
__global__ void k_prio_keys(int32_t V, const int64_t* __restrict__ tl, const int64_t* __restrict__ bl,
                            const int32_t* __restrict__ cluster_of, uint64_t* __restrict__ keys,
                            int32_t* __restrict__ ids) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        keys[v] = cluster_of[v] >= 0 ? ~0ull : (uint64_t)(kValMask - (uint64_t)(tl[v] + bl[v]));
        ids[v] = v;
    }
}

__device__ __forceinline__ bool prio_better(int64_t wa, int32_t a, int64_t wb, int32_t b) {
    return b < 0 || wa > wb || (wa == wb && a < b);
}

// the highest-priority unvisited neighbour of u (warp-wide; -1 if none)
__device__ int32_t warp_best_neighbour(int32_t r, const int32_t* __restrict__ off, const int32_t* __restrict__ nbr,
                                       const int32_t* __restrict__ orig, const int32_t* cluster_of,
                                       const int64_t* __restrict__ tl, const int64_t* __restrict__ bl, int lane) {
    int32_t best = -1;
    int64_t bw = 0;
    for (int32_t e = off[r] + lane; e < off[r + 1]; e += 32) {
        const int32_t s = orig[nbr[e]];
        if (*(volatile const int32_t*)&cluster_of[s] >= 0) continue;
        const int64_t ws = tl[s] + bl[s];
        if (prio_better(ws, s, bw, best)) { best = s; bw = ws; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int32_t ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int64_t ow = __shfl_xor_sync(0xffffffffu, bw, o);
        if (ob >= 0 && prio_better(ow, ob, bw, best)) { best = ob; bw = ow; }
    }
    return best;
}

// The secondary phase on one warp.  ctl[0] = members so far, ctl[1] = clusters.
__global__ void __launch_bounds__(32) k_secondary(int32_t V, const int32_t* __restrict__ order,
                                                  const uint64_t* __restrict__ okeys,
                                                  const int32_t* __restrict__ rank_of,
                                                  const int32_t* __restrict__ orig,
                                                  const int32_t* __restrict__ in_off, const int32_t* __restrict__ in_src,
                                                  const int32_t* __restrict__ out_off,
                                                  const int32_t* __restrict__ out_dst,
                                                  const int64_t* __restrict__ tl, const int64_t* __restrict__ bl,
                                                  int32_t* cluster_of, int32_t* __restrict__ members,
                                                  int32_t* __restrict__ cl_off, int32_t* __restrict__ fwd,
                                                  int32_t* __restrict__ ctl, int32_t* __restrict__ n_clusters) {
    const int lane = threadIdx.x;
    int32_t m = ctl[0], nc = ctl[1];
    for (int32_t i = 0; i < V; ++i) {
        if (okeys[i] == ~0ull) break;                 // primaries sort last
        const int32_t s0 = order[i];
        if (*(volatile int32_t*)&cluster_of[s0] >= 0) continue;   // visited
        if (lane == 0) cluster_of[s0] = nc;
        __syncwarp();
        // forward from the start
        int32_t fw = 0;
        if (lane == 0) fwd[fw] = s0;
        ++fw;
        for (int32_t u = s0;;) {
            const int32_t b = warp_best_neighbour(rank_of[u], out_off, out_dst, orig, cluster_of, tl, bl, lane);
            if (b < 0) break;                         // dead end
            if (lane == 0) { cluster_of[b] = nc; fwd[fw] = b; }
            __syncwarp();
            ++fw;
            u = b;
        }
        // backward from the start (collected reversed, then flipped)
        int32_t bw = 0;
        for (int32_t u = s0;;) {
            const int32_t b = warp_best_neighbour(rank_of[u], in_off, in_src, orig, cluster_of, tl, bl, lane);
            if (b < 0) break;
            if (lane == 0) { cluster_of[b] = nc; members[m + bw] = b; }
            __syncwarp();
            ++bw;
            u = b;
        }
        for (int32_t a = lane; a < bw / 2; a += 32) {
            const int32_t x = members[m + a];
            members[m + a] = members[m + bw - 1 - a];
            members[m + bw - 1 - a] = x;
        }
        for (int32_t k = lane; k < fw; k += 32) members[m + bw + k] = fwd[k];
        __syncwarp();
        m += bw + fw;
        ++nc;
        if (lane == 0) cl_off[nc] = m;
    }
    if (lane == 0) {
        ctl[0] = m;
        ctl[1] = nc;
        *n_clusters = nc;
    }
}

__global__ void k_cluster_max(int32_t V, const int64_t* __restrict__ tl, const int64_t* __restrict__ bl,
                              const int32_t* __restrict__ cluster_of, unsigned long long* __restrict__ crit) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
        atomicMax(&crit[cluster_of[v]], (unsigned long long)(tl[v] + bl[v]));
}

size_t slice_sort_temp_bytes(int32_t V) {
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, std::max(V, 1));
    return need;
}

static int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)); }

}  // namespace pdnn

using namespace pdnn;

extern "C" pdnn_status pdnn_slice_clusters(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                                           int32_t K, int32_t* cluster_of, int32_t* members, int32_t* cl_off,
                                           int32_t* n_clusters, void* ws, size_t ws_bytes, void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (K < 0 || !n_clusters || !cl_off || (g->V > 0 && (!cluster_of || !members))) {
        set_error("bad K or null output");
        return PDNN_EINVAL;
    }
    const WsLayout L = ws_layout(g, PDNN_OP_SLICE_CLUSTERS, 0);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    pdnn_status st = ws_guard(ws, 0, 0, L.single_end, L.sig_single, s);
    if (st) return st;
    Costs C;
    if ((st = resolve_costs(g, node_cost, edge_cost, ws, L, s, &C, /*need_blob=*/true))) return st;
    const int32_t V = g->V;
    int32_t* ctl = ws_ptr<int32_t>(ws, L.sc_ctl);
    PDNN_CUDA_TRY(cudaMemsetAsync(ctl, 0, 16, s));
    PDNN_CUDA_TRY(cudaMemsetAsync(cl_off, 0, 4, s));
    if (V == 0) {
        PDNN_CUDA_TRY(cudaMemsetAsync(cl_off, 0, 4 * ((size_t)K + 1), s));
        PDNN_CUDA_TRY(cudaMemcpyAsync(n_clusters, &K, 4, cudaMemcpyHostToDevice, s));
        PDNN_CUDA_TRY(cudaStreamSynchronize(s));
        return PDNN_OK;
    }
    PDNN_CUDA_TRY(cudaMemsetAsync(cluster_of, 0xff, 4 * (size_t)V, s));   // -1: not in a cluster yet
    int32_t* po = ws_ptr<int32_t>(ws, L.part_o);
    int32_t* pr = ws_ptr<int32_t>(ws, L.part_rank);
    int64_t* tl = ws_ptr<int64_t>(ws, L.tl_o);
    int64_t* bl = ws_ptr<int64_t>(ws, L.bl_o);
    int32_t* cp = ws_ptr<int32_t>(ws, L.cp_nodes);
    int32_t* scal = ws_ptr<int32_t>(ws, L.sc_ctl + 16);                      // cp_len
    int64_t* Ls = ws_ptr<int64_t>(ws, L.sc_ctl + 32);
    uint64_t* hs = ws_ptr<uint64_t>(ws, L.sc_ctl + 48);
    // every node alive and UNASSIGNED (every edge pays, as in the K-loop)
    if ((st = launch_labels(g, nullptr, nullptr, PDNN_UNASSIGNED, po, pr, s))) return st;
    for (int32_t j = 0; j < K; ++j) {
        if ((st = launch_sweep(g, C, pr, tl, bl, ws, L, s, /*removal=*/j > 0))) return st;
        if ((st = launch_cp(g, C, po, tl, bl, cp, scal, Ls, hs, po, pr, ws, L, s))) return st;
        k_append_cluster<<<1, 256, 0, s>>>(cp, scal, j, cluster_of, members, cl_off, ctl);
        count_launch();
        PDNN_LAUNCH_CHECK();
    }
    PDNN_CUDA_TRY(cudaMemcpyAsync(ctl + 1, &K, 4, cudaMemcpyHostToDevice, s));
    // the stale priorities, then the start order
    if ((st = launch_sweep(g, C, pr, tl, bl, ws, L, s, /*removal=*/true))) return st;
    uint64_t* k0 = ws_ptr<uint64_t>(ws, L.sc_keys);
    uint64_t* k1 = k0 + V;
    int32_t* i0 = ws_ptr<int32_t>(ws, L.sc_ids);
    int32_t* i1 = i0 + V;
    k_prio_keys<<<grid_of(V), 256, 0, s>>>(V, tl, bl, cluster_of, k0, i0);
    count_launch();
    PDNN_LAUNCH_CHECK();
    size_t tb = L.sc_temp_bytes;
    PDNN_CUDA_TRY(cub::DeviceRadixSort::SortPairs(ws_ptr<void>(ws, L.sc_temp), tb, k0, k1, i0, i1, V, 0, 64, s));
    count_launch(4);
    k_secondary<<<1, 32, 0, s>>>(V, i1, k1, g->rank_of, g->orig, g->in_off, g->in_src, g->out_off, g->out_dst, tl, bl,
                                 cluster_of, members, cl_off, ws_ptr<int32_t>(ws, L.sc_fwd), ctl, n_clusters);
    count_launch();
    PDNN_LAUNCH_CHECK();
    return PDNN_OK;
}

namespace pdnn {
pdnn_status launch_criticality(const pdnn_graph* g, const Costs& C, const int32_t* cluster_of, int32_t n_clusters,
                               int64_t* crit, void* ws, const WsLayout& L, cudaStream_t s) {
    if (n_clusters > 0) PDNN_CUDA_TRY(cudaMemsetAsync(crit, 0, 8 * (size_t)n_clusters, s));
    if (g->V == 0) return PDNN_OK;
    int32_t* pr = ws_ptr<int32_t>(ws, L.part_rank);
    int64_t* tl = ws_ptr<int64_t>(ws, L.tl_o);
    int64_t* bl = ws_ptr<int64_t>(ws, L.bl_o);
    pdnn_status st;
    // labels = cluster ids: communication inside a cluster is zero (R2, R19)
    if ((st = launch_labels(g, cluster_of, nullptr, 0, nullptr, pr, s))) return st;
    if ((st = launch_sweep(g, C, pr, tl, bl, ws, L, s))) return st;
    k_cluster_max<<<grid_of(g->V), 256, 0, s>>>(g->V, tl, bl, cluster_of, reinterpret_cast<unsigned long long*>(crit));
    count_launch();
    PDNN_LAUNCH_CHECK();
    return PDNN_OK;
}
}  // namespace pdnn

extern "C" pdnn_status pdnn_criticality(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                                        const int32_t* cluster_of, int32_t n_clusters, int64_t* crit, void* ws,
                                        size_t ws_bytes, void* stream) {
    if (!g) { set_error("null graph"); return PDNN_EINVAL; }
    if (n_clusters < 0 || (n_clusters > 0 && !crit) || (g->V > 0 && !cluster_of)) {
        set_error("bad n_clusters or null argument");
        return PDNN_EINVAL;
    }
    const WsLayout L = ws_layout(g, PDNN_OP_WEIGHTED_LEVELS, 0);
    if (!ws || ws_bytes < L.total) { set_error("workspace too small"); return PDNN_EWORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    pdnn_status st = ws_guard(ws, 0, 0, L.single_end, L.sig_single, s);
    if (st) return st;
    if (g->V == 0) {
        if (n_clusters > 0) PDNN_CUDA_TRY(cudaMemsetAsync(crit, 0, 8 * (size_t)n_clusters, s));
        return PDNN_OK;
    }
    Costs C;
    if ((st = resolve_costs(g, node_cost, edge_cost, ws, L, s, &C, /*need_blob=*/true))) return st;
    return launch_criticality(g, C, cluster_of, n_clusters, crit, ws, L, s);
}
