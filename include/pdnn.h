/*
 * pdnn.h -- C ABI of the B200-native weighted-level sweep of ParDNN
 * (arXiv 2008.08636, "A Static Graph Partitioner for Model Parallelism").
 *
 * The library (paper_2008_08636_b200/libpdnn.so, sm_100a CUDA) computes the
 * data-parallel core the paper runs K times during slicing and refinement:
 *
 *   tl(n)  top level  -- costliest path from a source to n, EXCLUDING n
 *   bl(n)  bottom level -- costliest path from n to a sink, INCLUDING n
 *          (Table 2; path length = sum of comp(n) over its
 *          nodes + sum of comm(e) over its edges)
 *   CP     the critical path, extracted with a deterministic tie-break
 *          (Alg. 1 find_heaviest_path with fresh levels)
 *   M_cons / M_pot  the per-PE memory consumption over the visit order and the
 *          per-node memory potential (Eq. 3; Table 2,
 *          PAPER.md:217; tracker pass)
 *
 * Conventions (all calls):
 *  - Node ids are dense int32 in [0, n_nodes); edges are (src, dst) pairs,
 *    n_edges < 2^31.  The graph must be a DAG without self loops or duplicate
 *    pairs (PDNN_EINVAL / PDNN_ECYCLE from pdnn_build_csr).
 *  - Costs are int64: comp(n) and comm(e) in integer nanoseconds, mem(n) in
 *    bytes, all >= 0, with sum(comp) + sum(comm) < 2^62 (so no path length
 *    overflows; pdnn_graph_set_costs checks it and returns PDNN_EOVERFLOW).
 *  - "Canonical edge order" = edges sorted by (src, dst).  pdnn_build_csr
 *    returns the permutation perm[k] = index in the caller's input order of
 *    the k-th canonical edge.
 *  - Pointers are DEVICE pointers unless marked (host).  Arrays are owned by
 *    the caller; the library owns only the opaque pdnn_graph (device-resident
 *    CSR copies, level order and sweep schedule).
 *  - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *    Every call except pdnn_build_csr / pdnn_graph_set_costs /
 *    pdnn_workspace_init is asynchronous and stream-ordered.  Argument errors
 *    are detected on the host before anything is launched and returned
 *    synchronously; no C++ exception crosses the ABI.  Launch failures return
 *    PDNN_ECUDA with detail in pdnn_last_error() (thread-local).
 *  - Scratch: `ws` is a caller-provided device buffer of at least
 *    pdnn_workspace_bytes(g, op, batch) bytes, zero-filled once (e.g.
 *    pdnn_workspace_init) before its first use with a given graph.  The
 *    library keeps small self-resetting state in it between calls (sweep
 *    epoch tags), so a workspace must not be used by two streams at once.
 *
 * Labels `part` (int32[n_nodes], nullable) cover every use in the paper
 * (reading R2/R3):
 *    NULL            every edge pays comm (slicing before placement)
 *    >= 0            PE or cluster id; comm of an edge whose endpoints share a
 *                    label is 0 (criticality PAPER.md:345, refinement PAPER.md:11)
 *    PDNN_REMOVED    node and incident edges deleted (slicing);
 *                    its tl = bl = -1
 *    PDNN_UNASSIGNED alive, never co-located: all its edges pay comm
 */
#ifndef PDNN_H
#define PDNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pdnn_graph pdnn_graph;

typedef enum {
    PDNN_OK = 0,
    PDNN_EINVAL = -1,     /* bad argument, id out of range, self loop, duplicate pair */
    PDNN_ECYCLE = -2,     /* the edge set has a cycle */
    PDNN_ENOMEM = -3,     /* device or host allocation failed */
    PDNN_ECUDA = -4,      /* a CUDA call failed; see pdnn_last_error() */
    PDNN_EOVERFLOW = -5,  /* negative cost or sum(comp)+sum(comm) >= 2^62 */
    PDNN_EWORKSPACE = -6  /* ws is NULL or smaller than pdnn_workspace_bytes() */
} pdnn_status;

enum { PDNN_REMOVED = -1, PDNN_UNASSIGNED = -2, PDNN_MAX_PE = 16 };
enum { PDNN_KIND_NORMAL = 0, PDNN_KIND_RESIDUAL = 1, PDNN_KIND_REFERENCE = 2 };
enum { PDNN_EDGE_ORDER_CANONICAL = 0, PDNN_EDGE_ORDER_INPUT = 1 };
enum {
    PDNN_OP_WEIGHTED_LEVELS = 1,
    PDNN_OP_CRITICAL_PATH = 2,
    PDNN_OP_SLICE = 3,
    PDNN_OP_MEMORY = 4,
    PDNN_OP_EVAL_BATCH = 5,
    PDNN_OP_EMULATE = 6,
    PDNN_OP_EVAL_BATCH_EMULATED = 7,  /* pdnn_eval_batch with PDNN_SCHEDULE_EMULATED */
    PDNN_OP_SLICE_CLUSTERS = 8,
    PDNN_OP_RESOLVE_OVERFLOW = 9,
    PDNN_OP_LFLAM = 10,
    PDNN_OP_REFINE = 11
};
enum { PDNN_SCHEDULE_LEVEL = 0, PDNN_SCHEDULE_EMULATED = 1 };

/* ---------------------------------------------------------------- graph --
 * pdnn_build_csr -- validate the edge list and build the device graph
 * (§8(a) rows a1, a2): canonical (src,dst) edge order, forward and reverse
 * CSR, Kahn topological levels (level(v) = 0 without predecessors, else
 * 1 + max level(pred); the "variant of topological sorting" of PAPER.md:270)
 * computed by a frontier kernel with atomic in-degree countdown and
 * warp-aggregated frontier appends, the level order rank = stable (level, id)
 * order, rank-space CSRs, and the dataflow sweep schedule.
 *   n_nodes, n_edges   sizes (n_nodes >= 0, 0 <= n_edges < 2^31)
 *   src, dst           device int32[n_edges], any order
 *   perm_out           nullable device int32[n_edges]; perm_out[k] = input
 *                      index of the k-th canonical edge
 *   out                (host) receives the graph; NULL on error
 * SYNCHRONOUS on `stream` (reads back the cycle / validation verdict).
 * Errors: PDNN_EINVAL (id out of range, self loop, duplicate pair, bad size),
 *         PDNN_ECYCLE, PDNN_ENOMEM, PDNN_ECUDA. */
pdnn_status pdnn_build_csr(int32_t n_nodes, int64_t n_edges, const int32_t* src,
                           const int32_t* dst, int32_t* perm_out, void* stream,
                           pdnn_graph** out);

void pdnn_graph_free(pdnn_graph* g);

/* Host outputs (each nullable): node / edge count, number of levels D,
 * maximum in- and out-degree. */
pdnn_status pdnn_graph_query(const pdnn_graph* g, int32_t* n_nodes, int64_t* n_edges,
                             int32_t* n_levels, int32_t* max_in, int32_t* max_out);

/* level_out: device int32[n_nodes], level(v) in original id order. */
pdnn_status pdnn_graph_levels(const pdnn_graph* g, int32_t* level_out, void* stream);

/* Bind comp(n) (int64[n_nodes], node-id order) and comm(e) (int64[n_edges],
 * canonical order if edge_order == PDNN_EDGE_ORDER_CANONICAL, else the
 * caller's input order of pdnn_build_csr) to the graph: the library keeps
 * level-ordered copies that the sweeps stream.  SYNCHRONOUS (validates
 * non-negativity and the 2^62 bound: PDNN_EOVERFLOW). */
pdnn_status pdnn_graph_set_costs(pdnn_graph* g, const int64_t* node_cost,
                                 const int64_t* edge_cost, int edge_order, void* stream);

/* Bytes of scratch an op needs (batch is used by PDNN_OP_EVAL_BATCH only). */
size_t pdnn_workspace_bytes(const pdnn_graph* g, int op, int32_t batch);

/* Zero-fill a workspace (cudaMemsetAsync + stream sync).  SYNCHRONOUS. */
pdnn_status pdnn_workspace_init(void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- sweep --
 * pdnn_weighted_levels -- §8(a) rows a3 + a4 (Table 2, PAPER.md:209-211;
 * Alg. 1 lines 2/7):
 *   tl(v) = max(0, max over alive preds p of tl(p) + comp(p) + comm'(p,v))
 *   bl(u) = comp(u) + max(0, max over alive succs s of comm'(u,s) + bl(s))
 * with comm'(u,v) = 0 if part[u] == part[v] >= 0, else comm(u,v).
 *   node_cost, edge_cost  nullable: NULL uses the costs bound by
 *                         pdnn_graph_set_costs; non-NULL (int64, node-id /
 *                         canonical order) are used for this call only
 *   part                  nullable int32[n_nodes] labels (see above)
 *   tl, bl                int64[n_nodes] outputs, node-id order; -1 for
 *                         removed nodes
 * Errors: PDNN_EINVAL (no costs bound and none given), PDNN_EWORKSPACE,
 *         PDNN_ECUDA. */
pdnn_status pdnn_weighted_levels(const pdnn_graph* g, const int64_t* node_cost,
                                 const int64_t* edge_cost, const int32_t* part, int64_t* tl,
                                 int64_t* bl, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------- CP --
 * pdnn_critical_path -- §8(a) row a5 (find_heaviest_path with fresh weighted
 * levels is the CP; reading R5/R6 in DESIGN.md):
 *   L     = max over alive n of tl(n) + bl(n)
 *   start = lowest-id alive node without alive predecessors with bl == L
 *   next  = lowest-id alive successor s of u with comm'(u,s)+bl(s) == bl(u)-comp(u),
 *           until u has no alive successor
 *   cp_hash = sum_k (id_k + 1) * 0x100000001B3^k  (mod 2^64)
 * tl, bl must be the outputs of pdnn_weighted_levels for the same costs and
 * labels.  cp_nodes (int32, capacity >= n_levels) receives the path in
 * order; cp_len (int32), L (int64), cp_hash (uint64) are device scalars.
 * With no alive node: cp_len = 0, L = 0, cp_hash = 0. */
pdnn_status pdnn_critical_path(const pdnn_graph* g, const int64_t* node_cost,
                               const int64_t* edge_cost, const int32_t* part, const int64_t* tl,
                               const int64_t* bl, int32_t* cp_nodes, int32_t* cp_len, int64_t* L,
                               uint64_t* cp_hash, void* ws, size_t ws_bytes, void* stream);

/* pdnn_slice -- §8(a) row a6, the primary phase of graph slicing (Alg. 1,
 * PAPER.md:239-262; reading R4): for j = 0..K-1, sweep the graph minus the
 * paths 0..j-1 with every alive node UNASSIGNED, extract its CP (as
 * pdnn_critical_path) and remove it.  No host round trip between sweeps.
 *   cps     int32[K][cap] (cap >= n_levels), path j in row j
 *   cp_lens int32[K], Ls int64[K], hashes uint64[K]
 * A sweep on an exhausted graph yields cp_len = 0, L = 0, hash = 0. */
pdnn_status pdnn_slice(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                       int32_t K, int32_t cap, int32_t* cps, int32_t* cp_lens, int64_t* Ls,
                       uint64_t* hashes, void* ws, size_t ws_bytes, void* stream);

/* pdnn_slice_clusters -- §8(f) NEXT row N2: the whole of Alg. 1 (PAPER.md:
 * 239-262): the K primaries of pdnn_slice, then -- "we stop recalculating
 * w_lvl(n) for the secondary clusters" -- secondary clusters
 * until every node is in one, each found by find_heaviest_path with the stale
 * priorities w_lvl = tl + bl of G minus the primaries (reading R18: start =
 * the unvisited node of maximum w_lvl, lowest id on ties; forward by the
 * unvisited successor of maximum w_lvl, then backward from the start by the
 * unvisited predecessor of maximum w_lvl; a singleton if neither exists).
 *   cluster_of  int32[n_nodes]: 0..K-1 primaries (empty if the graph runs out),
 *               then the secondaries in extraction order
 *   members     int32[n_nodes]: the nodes cluster by cluster, in path order
 *   cl_off      int32[n_nodes + K + 1]: cluster k = members[cl_off[k], cl_off[k+1])
 *   n_clusters  device int32 scalar
 * The extraction is a greedy walk (one warp); the sweeps and CPs are parallel. */
pdnn_status pdnn_slice_clusters(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                                int32_t K, int32_t* cluster_of, int32_t* members, int32_t* cl_off,
                                int32_t* n_clusters, void* ws, size_t ws_bytes, void* stream);

/* pdnn_criticality -- the criticality of linear clusters (LFLAM):
 * "w_lvl(n) ... recalculated by setting communications within lcs to zeros"
 * (reading R19): a sweep with labels = cluster ids, then
 *   crit[k] = max over n with cluster_of[n] == k of tl(n) + bl(n).
 *   cluster_of  int32[n_nodes], every id in [0, n_clusters);  crit int64[n_clusters] */
pdnn_status pdnn_criticality(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                             const int32_t* cluster_of, int32_t n_clusters, int64_t* crit, void* ws,
                             size_t ws_bytes, void* stream);

/* pdnn_lflam -- §8(f) NEXT row N4: the LFLAM mapping (Alg. 2, PAPER.md:
 * 321-411; Eq. 2 at PAPER.md:366-371) in reading R21: primary k
 * is PE k; the secondaries, in non-increasing criticality (pdnn_criticality,
 * lower index first), go through the locality-first lookahead -- a totally-
 * communicating secondary (or, when sum comm >= 10 sum comp, a maximally-
 * communicating one: comm(sc, t) * K > ext(sc)) joins t, its most
 * communicating PE (lowest on ties), if (a) U >= max(0, work(t) + w(sc) -
 * floor(sum work / K)), (b) work(t) + w(sc) <= max work, or (c) comm(sc, t) >
 * w(sc), > work(t) and > U -- repeated while a pass maps a cluster, at most
 * ceil(log2 n_nodes) passes; every secondary left joins argmin_pe work(pe) +
 * comm(sc, other PEs) (Eq. 2; ties: most communicating, then lowest PE).
 * work(pe) / U = the comp of the nodes on pe / of unmapped secondaries other
 * than sc whose level lies in span(sc) (strictly after the latest parent of
 * the cluster's first node, strictly before the earliest child of its last).
 *   cluster_of, members, cl_off   device, as pdnn_slice_clusters writes them
 *                                 (every node in exactly one cluster; each
 *                                 cluster a path, members in path order)
 *   n_clusters  HOST int32 (K <= n_clusters <= n_nodes + K); 1 <= K <= 16
 *   part        device int32[n_nodes] out: the PE of every node
 *   log         device int32[n_clusters - K][3] out: (cluster, 0 lookahead /
 *               1 balancing, PE) in decision order;  n_log  device int32 out
 * Costs: as pdnn_weighted_levels (NULL = bound costs).  Precondition on
 * device data (not checked): the cluster arrays are a partition of the nodes
 * into paths.  Workspace: pdnn_workspace_bytes(g, PDNN_OP_LFLAM, 0). */
pdnn_status pdnn_lflam(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                       const int32_t* cluster_of, const int32_t* members, const int32_t* cl_off,
                       int32_t n_clusters, int32_t K, int32_t* part, int32_t* log, int32_t* n_log,
                       void* ws, size_t ws_bytes, void* stream);

/* pdnn_refine -- §8(f) NEXT row N4, second half: the refinement of Step 1
 * (appendix "Complexity of Refinement") in reading R22
 * (DESIGN.md), after pdnn_lflam.
 *   Phase 1, cluster swaps: tl under `part`; the secondaries (clusters >= K,
 *   non-empty) sorted by (tl of their first node, id) ("we sort the clusters by
 *   tl(n) of their source nodes ... using binary search"); for every unmarked A
 *   in that order (on PE a) the candidates are the first `window` unmarked B
 *   (sorted order) on a PE b != a with tl(first of B) in [tl(first of A),
 *   tl(last of A) + comp(last of A)]; gain = cut communication before - after
 *   the swap (A's nodes to b, B's to a); the B with the largest gain > 0 (the
 *   earliest on ties) whose swap keeps max(work(a, R), work(b, R)) from rising,
 *   R = the levels the two clusters cover (level-indexed Fenwick trees), is
 *   swapped and both are marked ("not considered again").
 *   Phase 2, `passes` node-level passes (the paper repeats it K times): tl, bl
 *   and the CP (as pdnn_critical_path) under the placement; trials (n, q): a CP
 *   node and the PE of its CP predecessor, then successor, when it differs from
 *   n's; rounds: the live trials whose move keeps work(q, level(n)) + comp(n) <=
 *   max over PEs of work(., level(n)) are scored by L (the batched sweep,
 *   lane = trial); the least L (earliest trial on ties) is applied if it is
 *   below the current L, and n's trials are dropped; else the pass ends.
 *   cluster_of, members, cl_off  device, as pdnn_slice_clusters writes them
 *   n_clusters  HOST int32, K <= n_clusters <= n_nodes + K; 1 <= K <= 16
 *   passes >= 0; 1 <= window <= 1024
 *   part        DEVICE int32[n_nodes] in / out: labels in [0, K), every
 *               cluster's nodes on one PE (PDNN_EINVAL otherwise: checked)
 *   log_host    HOST int64[log_cap][4]: (0, A, B, gain) per swap, then
 *               (1, node, to PE, L after the move) per node move; entries past
 *               log_cap are dropped;  n_log  HOST: the number of decisions
 *   L_host      HOST: L of the final placement
 * Costs: as pdnn_weighted_levels (NULL = bound costs).  SYNCHRONOUS (a host
 * loop over the library's kernels; one read-back per round).  Workspace:
 * pdnn_workspace_bytes(g, PDNN_OP_REFINE, 0). */
pdnn_status pdnn_refine(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                        const int32_t* cluster_of, const int32_t* members, const int32_t* cl_off,
                        int32_t n_clusters, int32_t K, int32_t passes, int32_t window, int32_t* part,
                        int64_t* log_host, int32_t log_cap, int32_t* n_log, int64_t* L_host, void* ws,
                        size_t ws_bytes, void* stream);

/* --------------------------------------------------------------- memory --
 * pdnn_memory_potential -- §8(a) row a7: the memory consumption tracker of
 * Heuristic I (Eq. 3 at PAPER.md:465-481) in the visit-
 * order reading R8-R12 of DESIGN.md:
 *   visit order = sort by (st, level, id); pos(n) its rank
 *   effmem(n)   = 0 for reference nodes, else mem(n)
 *   residual n: held on part[n] over the whole pass; normal n: held on
 *   part[n] from its visit through its last consumer on part[n] (its own
 *   visit if none); any non-reference n with consumers on q != part[n]: held
 *   on q from its visit through its last consumer on q.
 *   M_cons(q,i) = sum over the holdings of q that contain position i.
 * Outputs: mpot[n] = effmem(n) + sum of effmem(p) over predecessors p for
 * which n is the last consumer on part[n] (excluding residual p on part[n]);
 * per PE q: peak[q] = max_i M_cons(q,i), peak_pos[q] = lowest i attaining
 * it, first_over_pos[q] = lowest i with M_cons(q,i) > cap_eff[q] (-1 if
 * none), over_bytes[q] = M_cons(q, first_over_pos[q]) - cap_eff[q] (0 if
 * none); optional mcons int64[n_pe][n_nodes] (nullable).
 *   part     int32[n_nodes], every label in [0, n_pe), 1 <= n_pe <= 16
 *   mem      int64[n_nodes] >= 0 with sum(mem) < 2^61 (every M_cons value and
 *            every scan tile's signed aggregate fits the 62-bit look-back
 *            words);  kind uint8[n_nodes] in {0,1,2}
 *   st       int64[n_nodes] >= 0, non-decreasing along every edge (any real
 *            schedule, e.g. pdnn_emulate's), or NULL: the default st = tl
 *            under `part` (reading R8), computed here with the costs bound by
 *            pdnn_graph_set_costs (PDNN_EINVAL if none are bound)
 *   cap_eff  int64[n_pe] (the 90% capacity)
 * Precondition on device data (not checked): labels in range, kinds valid,
 * st monotone on edges, the sum of mem below 2^61. */
pdnn_status pdnn_memory_potential(const pdnn_graph* g, const int32_t* part, int32_t n_pe,
                                  const int64_t* mem, const uint8_t* kind, const int64_t* st,
                                  const int64_t* cap_eff, int64_t* mpot, int64_t* peak,
                                  int32_t* peak_pos, int32_t* first_over_pos, int64_t* over_bytes,
                                  int64_t* mcons, void* ws, size_t ws_bytes, void* stream);

/* pdnn_resolve_overflow -- §8(f) NEXT row N3: the overflow handler of Memory
 * Heuristic I in reading R20: repeatedly take
 * the earliest overflow (lowest first_over position over the PEs, lowest PE
 * on ties; O = its over_bytes); among the normal nodes on that PE never moved
 * or rejected before, with a = M_pot(n, t) > 0 at that position (Table 2:
 * ancestors' outputs still held for which n is the last consumer on its PE,
 * plus n's own memory at its visit) and c = move_cost (Eq. 5), pick the
 * lowest c / a (ties by id), unless a node with a > O has a strictly smaller
 * c (the second heap); move it to the PE q' != q with M_cons(q', t) + a <=
 * cap_eff[q'] and the least M_cons(q', t) (lowest id on ties), or reject it
 * ("not considered again") and pick again; after every move recompute the
 * schedule (st = tl, reading R8) and the tracker.  Stops when no PE overflows
 * (*resolved = 1), the current overflow has no candidate left, or after
 * max_moves decisions.
 *   mem, kind     device, node-id order;  cap_eff_host  HOST int64[n_pe]
 *   part          DEVICE int32[n_nodes], labels in [0, n_pe): updated in place
 *   moves_host    HOST int32[max_moves][3]: (node, from, to), to = -1 for a
 *                 rejected candidate;  n_moves, resolved  HOST scalars
 * SYNCHRONOUS (a host loop over the library's kernels: a sweep, the tracker,
 * M_pot at the overflow and the dual-heap choice per decision).  Workspace:
 * pdnn_workspace_bytes(g, PDNN_OP_RESOLVE_OVERFLOW, 0). */
pdnn_status pdnn_resolve_overflow(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                                  const int64_t* mem, const uint8_t* kind, int32_t n_pe,
                                  const int64_t* cap_eff_host, int32_t* part, int32_t max_moves,
                                  int32_t* moves_host, int32_t* n_moves, int32_t* resolved, void* ws,
                                  size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- batch --
 * One candidate's evaluation (432 bytes, naturally aligned). */
typedef struct {
    int64_t L;          /* critical-path length under the candidate */
    int64_t cut_comm;   /* sum of comm(e) over edges whose endpoints differ */
    uint64_t cp_hash;
    int32_t cp_len, cp_start, cp_end; /* first / last node of the CP */
    int32_t overflow_mask;            /* bit q set iff first_over_pos[q] >= 0 */
    int64_t peak[PDNN_MAX_PE];        /* PEs >= n_pe: 0 */
    int64_t over_bytes[PDNN_MAX_PE];
    int32_t peak_pos[PDNN_MAX_PE];    /* PEs >= n_pe: -1 */
    int32_t first_over_pos[PDNN_MAX_PE];
    int64_t makespan;   /* max ft of the schedule the tracker used: L for the
                           level schedule, the emulated makespan otherwise */
} pdnn_eval_result;

/* pdnn_eval_batch -- §8(a) row a8: evaluate `batch` candidate placements
 * (refinement / LALB trials): for candidate b with
 * labels parts[b][*] (uint8, in [0, n_pe)): weighted levels, CP, cut comm
 * and the memory tracker under that placement, on the schedule
 *   PDNN_SCHEDULE_LEVEL     st = tl (reading R8); makespan = L
 *   PDNN_SCHEDULE_EMULATED  st = the TF FIFO scheduler emulation (pdnn_emulate,
 *                           reading R17); makespan = its max ft
 * (size the workspace with PDNN_OP_EVAL_BATCH / PDNN_OP_EVAL_BATCH_EMULATED).
 *   parts  uint8[batch][n_nodes];  out  pdnn_eval_result[batch] (device)
 * Costs: as pdnn_weighted_levels (NULL = bound costs). */
pdnn_status pdnn_eval_batch(const pdnn_graph* g, const int64_t* node_cost,
                            const int64_t* edge_cost, const int64_t* mem, const uint8_t* kind,
                            int32_t n_pe, const int64_t* cap_eff, int32_t batch,
                            const uint8_t* parts, pdnn_eval_result* out, int32_t schedule,
                            void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------- emulator --
 * pdnn_emulate -- §8(f) NEXT row N1: the TF FIFO scheduler emulator of Memory
 * Heuristic I in reading R17: every PE runs one
 * node at a time; a node enters the ready queue when its last input arrives,
 *   ready(v) = max(0, max over preds p of ft(p) + comm'(p, v)),
 * the queue is FIFO by entry time, equal entry times ordered by (level, id);
 *   st(v) = max(ready(v), ft(previous node on part[v])),  ft = st + comp.
 *   part      int32[n_nodes], labels in [0, n_pe) (precondition, not checked)
 *   st, ft    int64[n_nodes] outputs, node-id order
 *   makespan  device int64 scalar: max ft (0 for an empty graph)
 * The emulation is sequential per placement (one warp); st feeds
 * pdnn_memory_potential (the paper's tracker visits nodes in st order,
 * PAPER.md:487).  Workspace: pdnn_workspace_bytes(g, PDNN_OP_EMULATE, 0). */
pdnn_status pdnn_emulate(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                         const int32_t* part, int32_t n_pe, int64_t* st, int64_t* ft,
                         int64_t* makespan, void* ws, size_t ws_bytes, void* stream);

/* pdnn_validate -- check, on the device, the data preconditions the
 * asynchronous calls assume but do not check (each array nullable = skipped):
 *   node_cost / edge_cost (int64, node-id / canonical order): every cost >= 0
 *     and sum(comp) + sum(comm) < 2^62 (reading R7)        -> PDNN_EOVERFLOW
 *   mem: every mem >= 0 (PDNN_EINVAL) and sum(mem) < 2^61  -> PDNN_EOVERFLOW
 *   part: with n_pe > 0 every label in [0, n_pe) (the memory tracker, the
 *     batched evaluation, the emulator); with n_pe == 0 every label >= 0,
 *     PDNN_REMOVED or PDNN_UNASSIGNED (the sweep)          -> PDNN_EINVAL
 *   kind: every kind in {0, 1, 2}                          -> PDNN_EINVAL
 *   st: st >= 0 and st(v) >= st(u) on every edge (u, v), so (st, level, id)
 *     is a topological visit order (reading R10)           -> PDNN_EINVAL
 * SYNCHRONOUS on `stream`. */
pdnn_status pdnn_validate(const pdnn_graph* g, const int64_t* node_cost, const int64_t* edge_cost,
                          const int32_t* part, int32_t n_pe, const int64_t* mem, const uint8_t* kind,
                          const int64_t* st, void* stream);

const char* pdnn_status_string(pdnn_status s);
const char* pdnn_last_error(void);

/* Number of kernels this library has launched in the calling process (for the
 * bench's gpu_launches count); monotone, host-side counter. */
uint64_t pdnn_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* PDNN_H */
