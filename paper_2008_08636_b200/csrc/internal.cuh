// internal.cuh -- shared internals of libpdnn (the CUDA path).  Not part of the
// ABI; include/pdnn.h is.  Nothing here is shared with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>
#include <string>

#include "../../include/pdnn.h"

namespace pdnn {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

#define PDNN_CUDA_TRY(expr)                                                            \
    do {                                                                               \
        cudaError_t _e = (expr);                                                       \
        if (_e != cudaSuccess) {                                                       \
            ::pdnn::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));     \
            return PDNN_ECUDA;                                                         \
        }                                                                              \
    } while (0)

#define PDNN_LAUNCH_CHECK()                                                            \
    do {                                                                               \
        cudaError_t _e = cudaGetLastError();                                           \
        if (_e != cudaSuccess) {                                                       \
            ::pdnn::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e)); \
            return PDNN_ECUDA;                                                         \
        }                                                                              \
    } while (0)

// Diagnostic knobs (grid sizes, trace stamps) read from the environment only in
// a debug build (-DPDNN_DEBUG_KNOBS, `python -m paper_2008_08636_b200.build
// --debug-knobs`); the production library ignores the environment, so no
// variable can change a launch configuration or a result.
#ifdef PDNN_DEBUG_KNOBS
inline int debug_knob(const char* name, int def) {
    const char* v = getenv(name);
    return v ? atoi(v) : def;
}
#else
inline int debug_knob(const char*, int def) { return def; }
#endif

// Per-device launch properties: sets cudaFuncAttributeMaxDynamicSharedMemorySize
// on the CURRENT device (once per kernel, device and size) and returns the
// resident CTAs per SM (>= 1).  Function attributes are per device context, so
// a process driving several GPUs must not cache them process-wide.
int kernel_occupancy(const void* fn, int threads, int dyn_smem);

// ------------------------------------------------------------------ constants
constexpr int kSweepThreads = 256;     // 8 warps per CTA
constexpr int kTMaxDeg = 32;           // thread items: degree <= 32 (a node owns ceil(deg/4) <= 8 lanes)
constexpr int kTMaxEdges = 128;
constexpr int kMemHeavyDeg = 8;        // memory edge pass: out-degree > 8 takes the warp path        // ... and <= 128 edges per item
constexpr int kHEdges = 1024;          // hub items: <= 1024 edges per part
// thread item flag (Item.w bit 30): its nodes are inodes[x' .. x' + y) (x = ~x')
// instead of the rank run [x', x' + y); only bl items of level 0, grouped by
// the level whose bl completes their inputs (graph.cu build_items)
constexpr int32_t kItemIndexed = 1 << 30;
constexpr int kBMaxDeg = 8;           // batched sweep: nodes of degree <= 8 are grouped ...
constexpr int kBMaxEdges = 8;         // ... into items of <= 8 edges (one batch of gathers)
constexpr int kBMaxNodes = 8;         // ... and <= 8 nodes (lane registers hold 8 label rows)
constexpr int kBWideNodes = 2;        // nodes per item of the large-batch schedule
constexpr int kBWideChunks = 32;      // chunks (x32 candidates) from which it is used
constexpr int kBHubEdges = 256;       // batched hub parts: <= 256 edges
constexpr int kCpThreads = 512;
constexpr int kCpU = 4;            // CP kernel: nodes per thread per load round
constexpr uint64_t kValMask = (1ull << 62) - 1;

// sweep work item: x = r0 (tl pass) or ~r0 (bl pass); y > 0: thread-per-node
// item of y nodes; y == 0: single-part warp item; y < 0: hub part of slot -y-1;
// z, w: edge range [z, w) of a warp item.
struct __align__(16) Item { int32_t x, y, z, w; };

// ------------------------------------------------------------------ graph
}  // namespace pdnn

struct pdnn_graph {
    int32_t V = 0;
    int64_t E = 0;
    int32_t n_levels = 0, max_in = 0, max_out = 0;
    int device = 0;
    int rank_bits = 1;
    // original-id space
    int32_t* rank_of = nullptr;   // [V]
    int32_t* orig = nullptr;      // [V] original id of rank r
    int32_t* level = nullptr;     // [V] level of original id
    int32_t* perm = nullptr;      // [E] canonical k -> input index
    // rank space (level order)
    int32_t* level_ptr = nullptr; // [D+1]
    int32_t* in_off = nullptr;    // [V+1]
    int32_t* in_src = nullptr;    // [E] predecessor rank
    int32_t* in_eid = nullptr;    // [E] canonical edge id
    int32_t* out_off = nullptr;   // [V+1]
    int32_t* out_dst = nullptr;   // [E] successor rank
    int32_t* out_eid = nullptr;   // [E]
    // bound costs (rank space / CSR order)
    int64_t* c_rank = nullptr;
    int64_t* in_cost = nullptr;
    int64_t* out_cost = nullptr;
    bool costs_bound = false;
    uint64_t cost_total = 0;      // sum(comp) + sum(comm) of the bound costs
    // dataflow sweep schedule
    pdnn::Item* items = nullptr;    // dealt by wave (sweeps of the whole graph; graph.cu build_items)
    pdnn::Item* items_rm = nullptr; // the same items, proportional interleave (sweeps with REMOVED nodes)
    int32_t* inodes = nullptr;      // ranks of the nodes of "indexed" bl items (kItemIndexed; graph.cu build_items)
    int32_t n_inodes = 0;
    int32_t n_items = 0;
    int32_t n_hubs = 0;
    int32_t* hub_nparts = nullptr;
    int sweep_grid = 0;
    unsigned char* blob[2] = {nullptr, nullptr};   // packed thread items (tl / in-CSR, bl / out-CSR) of the bound costs
    size_t blob_bytes[2] = {0, 0};
    // heavy out-degree nodes (rank) for the memory edge pass
    int32_t* heavy_out = nullptr;
    int32_t n_heavy_out = 0;
    // batched (candidate-parallel) sweep schedule
    // two schedules: [0] one node per thread item (shortest dependency hop: a
    // warp finalises the nodes of an item one after another), [1] up to
    // kBMaxNodes nodes per item (fewer descriptors; for large batches)
    pdnn::Item* bitems[2] = {nullptr, nullptr};
    int32_t n_bitems[2] = {0, 0};
    int32_t n_bhubs = 0, n_bparts = 0;
    int32_t* bhub_pbase = nullptr;  // [n_bhubs + 1] first part slot of each split hub
    int32_t n_entry = 0;            // nodes of level 0 (ranks [0, n_entry))
    int num_sms = 148;
};

namespace pdnn {

// ------------------------------------------------------------------ workspace
struct WsHeader {
    uint32_t epoch;   // tag (1..3) of the last completed sweep; 0 on a fresh ws
    uint32_t ticket;  // sweep CTA completion counter (self-resetting)
    uint32_t cp_ticket;
    uint32_t pad0;
    unsigned long long Lslot[4];  // per-epoch max over alive n of tl(n)+comp(n) (= L)
    unsigned long long cut[4];    // per-epoch sum of comm'(e) over alive edges
    unsigned long long misc[8];
};

#ifndef PDNN_MEM_THREADS
#define PDNN_MEM_THREADS 256
#endif
#ifndef PDNN_MEM_PER_THREAD
#define PDNN_MEM_PER_THREAD 8
#endif
constexpr int kMemThreads = PDNN_MEM_THREADS;
constexpr int kMemPerThread = PDNN_MEM_PER_THREAD;
constexpr int kMemTile = kMemThreads * kMemPerThread;   // positions per scan tile

struct TileRes {          // per (tile, PE) partial of the memory scan
    long long peak;
    int32_t peak_pos;
    int32_t first_over;   // -1 if none in this tile
    long long over_val;   // M_cons at first_over
};

// batched evaluation (bsweep.cu): per-warp reductions and the workspace region
struct BSlot {
    long long Lb;      // max bl over the entry nodes this warp finished (-1: none)
    int32_t Lo, Lr;    // lowest original id / its rank attaining Lb
    long long cut;     // cut communication of the out-edges this warp relaxed
    long long maxst;   // max tl (the memory tracker's st) of the nodes it finished
};
struct BLayout {
    size_t hdr, lab, tlr, blr, nxt, keys, plab, part_val, part_idx, hub_cnt, slots, maxst, emu;
    int32_t ng;        // candidates per group (multiple of 32)
};
constexpr unsigned long long kBatchWsBudget = 32ull << 30;   // bytes of per-group candidate state

struct WsLayout {
    size_t single_end;    // [0, single_end): single-placement region (depends on the graph only)
    uint64_t sig_single, sig_batch;   // layout signatures of the two regions (ws_guard)
    int32_t m_seg;        // placements the memory-tracker region holds (1, or a batch sub-group)
    size_t hdr, rec, hub_acc, hub_cnt, c_s, in_cost_s, out_cost_s, part_rank, blob_s_in, blob_s_out;
    size_t tl_o, bl_o, part_o, cp_nodes, mpot_s;  // slice / batch internals (orig space)
    size_t emu;           // scheduler emulator scratch (one placement)
    size_t sc_ctl, sc_keys, sc_ids, sc_fwd, sc_temp, sc_temp_bytes;   // whole-Alg.1 slicing (slice.cu)
    size_t ov_mcons, ov_a, ov_excl, ov_small;   // overflow handler (overflow.cu), in the batched region
    size_t lf_lvl, lf_tree, lf_rec, lf_cm, lf_ce, lf_moff, lf_eoff, lf_ml, lf_mc, lf_epos, lf_ew, lf_comm, lf_crit,
        lf_keys, lf_ids, lf_pos, lf_list, lf_map, lf_ctl, lf_temp, lf_temp_bytes;   // LFLAM (lflam.cu), batched region
    size_t rf_keys, rf_ids, rf_rec, rf_cnt, rf_eoff, rf_ey, rf_ew, rf_marked, rf_temp, rf_temp_bytes, rf_lvl, rf_tree,
        rf_tn, rf_tq, rf_tdead, rf_elig, rf_res, rf_resg, rf_rows, rf_log, rf_ctl;   // refinement (refine.cu), batched region
    size_t cp_M, cp_ctl, cp_list, cp_pos, cp_A, cp_d, cp_mark;   // CP kernel (cp.cu)
    size_t m_keys, m_keys_alt, m_vals, m_vals_alt, m_order, m_pe8, m_status, m_pp, m_relp, m_rec, m_hist, m_dtot, m_tile,
        m_tile_res, m_base, m_ctr;
    BLayout B;
    size_t total;
    int cp_grid;
    int m_tiles;
    size_t cub_bytes;
};
WsLayout ws_layout(const pdnn_graph* g, int op, int32_t batch);
// Workspace guard.  A workspace region's persistent state (epoch-tagged
// records, self-resetting counters, look-back words) is only valid for the
// layout that wrote it.  The library remembers, per (workspace, region), the
// layout signature of the last call; when it changes (another batch size,
// another graph) the region [begin, end) is zeroed on the stream first, which
// is the documented fresh state.  Host-side, thread-safe; no launch when the
// layout is unchanged.
pdnn_status ws_guard(void* ws, int region, size_t begin, size_t end, uint64_t sig, cudaStream_t s);
uint64_t layout_sig(const pdnn_graph* g, uint64_t salt, size_t end);
// chunks of 32 candidates a batched-sweep launch runs for n real chunks: the
// smallest m >= n that divides the warps of a grid of >= 3/4 of the resident
// CTAs (each warp serves one chunk), so no chunk count starves the launch
int32_t bsweep_chunks(const pdnn_graph* g, int32_t n);
int bsweep_grid(const pdnn_graph* g, int32_t nck_run);

template <typename T>
inline T* ws_ptr(void* ws, size_t off) { return reinterpret_cast<T*>(static_cast<char*>(ws) + off); }

#ifndef PDNN_MEM_SEG_MAX
#define PDNN_MEM_SEG_MAX 64
#endif
constexpr int kMemSegMax = PDNN_MEM_SEG_MAX;   // placements per segmented memory-tracker launch (batched evaluation)

// memory tracker (memory.cu): inputs, outputs and scratch of S segments
struct MemIn {
    const int32_t* part_i32_orig;   // int32 labels, node-id order (single placement)
    const int32_t* part_i32_rank;   // int32 labels, rank order (single placement)
    const uint8_t* part_u8_rank;    // uint8 labels, rank order, S x V
    const int64_t* st_orig;         // st, node-id order (single placement)
    const int64_t* st_rank;         // st, rank order, S x V
};
struct MemOut {
    int64_t* peak;
    int32_t* peak_pos;
    int32_t* first_over;
    int64_t* over_bytes;
    size_t stride64, stride32;      // per-segment strides in int64 / int32 elements
};
struct MemWs {
    uint64_t* k0;
    uint64_t* k1;
    uint32_t* v0;
    uint32_t* v1;
    uint32_t* order;
    uint8_t* pe8;
    uint32_t* pp;
    unsigned long long* relp;
    void* rec;
    uint32_t* hist;          // sort: per-(segment, pass) digit bases
    uint32_t* dtot;          // sort: tickets [16] + launch epoch (8 B, device-owned; never cleared)
    void* sort_status;       // sort: look-back words, [S * tiles][1024] x 8 B
    long long* tsum;
    TileRes* tres;
    unsigned long long* base;       // [S][PDNN_MAX_PE] + max st
    uint32_t* ctr;                  // scan: tile ticket + per-segment tiles done
    int32_t m_tiles;
};
inline MemWs mem_ws(void* ws, const WsLayout& L) {
    MemWs M;
    M.k0 = ws_ptr<uint64_t>(ws, L.m_keys);
    M.k1 = ws_ptr<uint64_t>(ws, L.m_keys_alt);
    M.v0 = ws_ptr<uint32_t>(ws, L.m_vals);
    M.v1 = ws_ptr<uint32_t>(ws, L.m_vals_alt);
    M.order = ws_ptr<uint32_t>(ws, L.m_order);
    M.pe8 = ws_ptr<uint8_t>(ws, L.m_pe8);
    M.pp = ws_ptr<uint32_t>(ws, L.m_pp);
    M.relp = ws_ptr<unsigned long long>(ws, L.m_relp);
    M.rec = ws_ptr<void>(ws, L.m_rec);
    M.hist = ws_ptr<uint32_t>(ws, L.m_hist);
    M.dtot = ws_ptr<uint32_t>(ws, L.m_dtot);
    M.sort_status = ws_ptr<void>(ws, L.m_status);
    M.tsum = ws_ptr<long long>(ws, L.m_tile);
    M.tres = ws_ptr<TileRes>(ws, L.m_tile_res);
    M.base = ws_ptr<unsigned long long>(ws, L.m_base);
    M.ctr = ws_ptr<uint32_t>(ws, L.m_ctr);
    M.m_tiles = L.m_tiles;
    return M;
}

// costs resolved for one call (rank space / CSR order)
struct Costs {
    const int64_t* c;
    const int64_t* in_cost;
    const int64_t* out_cost;
    const unsigned char* blob_in;    // the sweep's packed items (need_blob), else nullptr
    const unsigned char* blob_out;
};
pdnn_status resolve_costs(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                          void* ws, const WsLayout& L, cudaStream_t s, Costs* out, bool need_blob = false);

// kernels shared across translation units (launch wrappers)
// labels -> rank space (part_rank, the sweep's label array); at most one of
// part_i32 / part_u8 is non-null (node-id order), else every label = fill
pdnn_status launch_labels(const pdnn_graph* g, const int32_t* part_i32, const uint8_t* part_u8, int32_t fill,
                          int32_t* part_orig_out, int32_t* part_rank, cudaStream_t s);
// removal: the labels REMOVE nodes (K-loop / slicing sweeps) -> the item order
// measured faster when removed nodes cut the chains (graph.cu build_items)
// lab_src (nullable, node-id order): the sweep converts it into lab_rank itself
// (one pass + a grid barrier at the start of the launch) instead of launch_labels
pdnn_status launch_sweep(const pdnn_graph* g, const Costs& C, const int32_t* lab_rank, int64_t* tl,
                         int64_t* bl, void* ws, const WsLayout& L, cudaStream_t s, bool removal = false,
                         const int32_t* lab_src = nullptr);
pdnn_status launch_cp(const pdnn_graph* g, const Costs& C, const int32_t* part_orig,
                      const int64_t* tl, const int64_t* bl, int32_t* cp_nodes, int32_t* cp_len,
                      int64_t* Lout, uint64_t* hash, int32_t* mark_orig, int32_t* mark_rank,
                      void* ws, const WsLayout& L, cudaStream_t s);
pdnn_status launch_memory(const pdnn_graph* g, const int32_t* part_orig, const int32_t* part_rank_in,
                          int32_t n_pe, const int64_t* mem, const uint8_t* kind, const int64_t* st,
                          const int64_t* cap_eff, int64_t* mpot, int64_t* peak, int32_t* peak_pos,
                          int32_t* first_over, int64_t* over_bytes, int64_t* mcons, void* ws,
                          const WsLayout& L, cudaStream_t s, bool st_rank = false);
int bsweep_warps(const pdnn_graph* g);
pdnn_status launch_memory_seg(const pdnn_graph* g, const MemIn& in, int32_t P, int32_t S, const int64_t* mem,
                              const uint8_t* kind, const int64_t* cap_eff, int64_t* mpot, const MemOut& o,
                              int64_t* mcons, const MemWs& M, cudaStream_t s);
// a library-owned side stream with its own fork / join events, checked out of
// a per-device pool for the duration of ONE call (two concurrent calls never
// share the events, so a fork recorded by one cannot order the other's work)
struct SideStream {
    cudaStream_t stream;
    cudaEvent_t ev_fork, ev_join;
    int device;
};
SideStream* side_acquire(int device);   // nullptr if none could be created
void side_release(SideStream* ss);
// the TF FIFO scheduler emulator (emulate.cu): one warp per placement; labels
// rank-space int32 (one placement) or candidate-major uint8 [n_cand][V]
size_t emulate_ws_bytes(const pdnn_graph* g, int32_t n_cand);
size_t slice_sort_temp_bytes(int32_t V);   // CUB temp storage of the secondary phase's priority sort
size_t lflam_temp_bytes(int32_t n);         // CUB temp storage of LFLAM's criticality sort and edge-count scan
size_t refine_temp_bytes(int32_t n);        // CUB temp storage of the refinement's secondary sort and edge scan
// trial placements per batched-sweep launch of the refinement (refine.cu): up
// to kRefineGroup, fewer when a group's sweep state would pass kRefineWsBudget
// (the batched sweep's depth floor is paid per launch: C3 groups of 256 -> 1,024)
#ifndef PDNN_REFINE_GROUP
#define PDNN_REFINE_GROUP 1024
#endif
constexpr int32_t kRefineGroup = PDNN_REFINE_GROUP;
constexpr unsigned long long kRefineWsBudget = 8ull << 30;
// Fenwick trees [T][D + 1] from per-level sums [T][D] (lflam.cu)
void launch_fenwick_build(int32_t T, int32_t D, const long long* lvl, long long* tree, cudaStream_t s);
// criticality of the clusters (reading R19): a sweep labelled by cluster ids,
// then crit[k] = max over the members of tl + bl (crit zeroed here)
pdnn_status launch_criticality(const pdnn_graph* g, const Costs& C, const int32_t* cluster_of, int32_t n_clusters,
                               int64_t* crit, void* ws, const WsLayout& L, cudaStream_t s);
pdnn_status launch_emulate(const pdnn_graph* g, const Costs& C, const int32_t* lab32, const uint8_t* lab8,
                           int32_t P, int32_t n_cand, void* scratch, int64_t* st_orig, int64_t* ft_orig,
                           int64_t* st_rank, int64_t* makespan, pdnn_eval_result* out, cudaStream_t s);
pdnn_status launch_bsweep(const pdnn_graph* g, const Costs& C, int32_t b0, int32_t nb, int32_t B,
                          const uint8_t* parts, const BLayout& BL, void* ws, pdnn_eval_result* out,
                          cudaStream_t s, const SideStream* side, bool write_makespan);

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// same load without a compiler memory clobber: lets the compiler batch several
// polls (issue all loads, then test the tags) instead of serialising them
__device__ __forceinline__ uint64_t ld_relaxed_u64_nc(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
// predicated loads that write their destination in place (no select / move
// after the load): a poll batch issues every load before the first use
__device__ __forceinline__ void ld_relaxed_u64_if(uint64_t& v, const uint64_t* p, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.relaxed.gpu.global.u64 %0, [%1];\n\t}"
                 : "+l"(v) : "l"(p), "r"((int)pred));
}
__device__ __forceinline__ void ld_relaxed_v2u64_if(uint64_t& a, uint64_t& b, const uint64_t* p, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n\t}"
                 : "+l"(a), "+l"(b) : "l"(p), "r"((int)pred));
}
__device__ __forceinline__ void ldg_u8_if(uint32_t& v, const uint8_t* p, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.u8 %0, [%1];\n\t}"
                 : "+r"(v) : "l"(p), "r"((int)pred));
}
// four predicated 16-byte relaxed loads issued by ONE asm statement, so the
// compiler cannot interleave their consumers (and stall on them) between the
// issues: all four are in flight before the first use
__device__ __forceinline__ void ld_relaxed_v2u64_x4(uint64_t (&a)[4], uint64_t (&b)[4], const uint64_t* p0,
                                                    const uint64_t* p1, const uint64_t* p2, const uint64_t* p3,
                                                    bool q0, bool q1, bool q2, bool q3) {
    asm volatile(
        "{\n\t.reg .pred q0, q1, q2, q3;\n\t"
        "setp.ne.b32 q0, %12, 0;\n\tsetp.ne.b32 q1, %13, 0;\n\t"
        "setp.ne.b32 q2, %14, 0;\n\tsetp.ne.b32 q3, %15, 0;\n\t"
        "@q0 ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%8];\n\t"
        "@q1 ld.relaxed.gpu.global.v2.u64 {%2, %3}, [%9];\n\t"
        "@q2 ld.relaxed.gpu.global.v2.u64 {%4, %5}, [%10];\n\t"
        "@q3 ld.relaxed.gpu.global.v2.u64 {%6, %7}, [%11];\n\t}"
        : "+l"(a[0]), "+l"(b[0]), "+l"(a[1]), "+l"(b[1]), "+l"(a[2]), "+l"(b[2]), "+l"(a[3]), "+l"(b[3])
        : "l"(p0), "l"(p1), "l"(p2), "l"(p3), "r"((int)q0), "r"((int)q1), "r"((int)q2), "r"((int)q3));
}
__device__ __forceinline__ void ld_relaxed_u64_x4(uint64_t (&a)[4], const uint64_t* p0, const uint64_t* p1,
                                                  const uint64_t* p2, const uint64_t* p3, bool q0, bool q1,
                                                  bool q2, bool q3) {
    asm volatile(
        "{\n\t.reg .pred q0, q1, q2, q3;\n\t"
        "setp.ne.b32 q0, %8, 0;\n\tsetp.ne.b32 q1, %9, 0;\n\t"
        "setp.ne.b32 q2, %10, 0;\n\tsetp.ne.b32 q3, %11, 0;\n\t"
        "@q0 ld.relaxed.gpu.global.u64 %0, [%4];\n\t"
        "@q1 ld.relaxed.gpu.global.u64 %1, [%5];\n\t"
        "@q2 ld.relaxed.gpu.global.u64 %2, [%6];\n\t"
        "@q3 ld.relaxed.gpu.global.u64 %3, [%7];\n\t}"
        : "+l"(a[0]), "+l"(a[1]), "+l"(a[2]), "+l"(a[3])
        : "l"(p0), "l"(p1), "l"(p2), "l"(p3), "r"((int)q0), "r"((int)q1), "r"((int)q2), "r"((int)q3));
}
__device__ __forceinline__ void ld_relaxed_v2u64(const uint64_t* p, uint64_t& a, uint64_t& b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_relaxed_v2u64(uint64_t* p, uint64_t a, uint64_t b) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// streaming read-only loads (bypass L1 allocation for one-touch data)
template <typename T>
__device__ __forceinline__ T ldg_stream(const T* p) { return __ldcs(p); }

__device__ __forceinline__ int64_t warp_max_i64(int64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        int64_t x = __shfl_xor_sync(0xffffffffu, v, o);
        v = x > v ? x : v;
    }
    return v;
}
__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

inline int bits_for(uint64_t x) {  // number of bits to represent x (>= 1)
    int b = 1;
    while (b < 64 && (x >> b) != 0) ++b;
    return b;
}
inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace pdnn
