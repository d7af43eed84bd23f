/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * The CPU oracle for the weighted-level sweep of ParDNN (arXiv 2008.08636).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It shares no code, header, table or
 * constant with the CUDA library under paper_2008_08636_b200/ (whose public
 * header is include/pdnn.h); the status codes below are restated here, by
 * value, from the readings in DESIGN.md, not included from that header.
 *
 * Every routine is a direct, single-threaded transcription of a definition in
 * PAPER.md (Table 2, Alg. 1, Eq. 3, the tracker pass) in the readings listed
 * in DESIGN.md section "Readings"; see the per-function comments in oracle.c.
 */
#ifndef PDNN_ORACLE_H
#define PDNN_ORACLE_H
#include <stdint.h>

#define OR_OK 0
#define OR_EINVAL (-1)
#define OR_ECYCLE (-2)
#define OR_ENOMEM (-3)
#define OR_EOVERFLOW (-5)

#define OR_REMOVED (-1)
#define OR_UNASSIGNED (-2)
#define OR_MAX_PE 16

#define OR_KIND_NORMAL 0
#define OR_KIND_RESIDUAL 1
#define OR_KIND_REFERENCE 2

typedef struct or_graph or_graph;

/* Result of one candidate evaluation (oracle's own layout; tests compare it
 * field by field with the product's struct). */
typedef struct {
    int64_t L;
    int64_t cut_comm;
    uint64_t cp_hash;
    int32_t cp_len, cp_start, cp_end, overflow_mask;
    int64_t peak[OR_MAX_PE];
    int64_t over_bytes[OR_MAX_PE];
    int32_t peak_pos[OR_MAX_PE];
    int32_t first_over_pos[OR_MAX_PE];
    int64_t makespan;   /* max ft of the schedule the tracker used */
} or_eval_result;

int or_build(int32_t n_nodes, int64_t n_edges, const int32_t* src, const int32_t* dst,
             or_graph** out);
void or_free(or_graph* g);
int32_t or_n_levels(const or_graph* g);
void or_levels(const or_graph* g, int32_t* level_out);
void or_topo(const or_graph* g, int32_t* topo_out);

int or_weighted_levels(const or_graph* g, const int64_t* c, const int64_t* w,
                       const int32_t* part, int64_t* tl, int64_t* bl);
int or_critical_path(const or_graph* g, const int64_t* c, const int64_t* w,
                     const int32_t* part, const int64_t* tl, const int64_t* bl,
                     int32_t* cp, int32_t* cp_len, int64_t* L, uint64_t* cp_hash);
int or_slice(const or_graph* g, const int64_t* c, const int64_t* w, int32_t K,
             int32_t cap, int32_t* cps, int32_t* cp_lens, int64_t* Ls, uint64_t* hashes);
int or_memory(const or_graph* g, const int32_t* part, int32_t n_pe, const int64_t* mem,
              const uint8_t* kind, const int64_t* st, const int64_t* cap_eff,
              int64_t* mpot, int64_t* peak, int32_t* peak_pos, int32_t* first_over,
              int64_t* over_bytes, int64_t* mcons, int32_t* order_out);
/* Whole of Alg. 1 (reading R18): K primaries, then secondary clusters with
 * stale priorities; criticality of clusters (reading R19). */
int or_slice_clusters(const or_graph* g, const int64_t* c, const int64_t* w, int32_t K, int32_t* cluster_of,
                      int32_t* members, int32_t* cl_off, int32_t* n_clusters);
int or_criticality(const or_graph* g, const int64_t* c, const int64_t* w, const int32_t* cluster_of,
                   int32_t n_clusters, int64_t* crit);
/* LFLAM mapping (Alg. 2, Eq. 2; reading R21) of the clusters of
 * or_slice_clusters onto K PEs; log[n][3] = (cluster, phase, pe). */
int or_lflam(const or_graph* g, const int64_t* c, const int64_t* w, const int32_t* cluster_of,
             const int32_t* members, const int32_t* cl_off, int32_t n_clusters, int32_t K, int32_t* part,
             int32_t* log, int32_t* n_log);
/* Refinement (appendix "Complexity of Refinement", reading R22): cluster
 * swaps, then `passes` node-level passes; part in/out; log[n][4] =
 * (0, A, B, gain) / (1, node, to, L); *L_out = L of the final placement. */
int or_refine(const or_graph* g, const int64_t* c, const int64_t* w, const int32_t* cluster_of,
              const int32_t* members, const int32_t* cl_off, int32_t n_clusters, int32_t K, int32_t passes,
              int32_t window, int32_t* part, int64_t* log, int32_t log_cap, int32_t* n_log, int64_t* L_out);
/* Overflow handler of Heuristic I (reading R20); M_pot(n, t) at visit i on q. */
int or_mpot_at(const or_graph* g, const int32_t* part, const int64_t* mem, const uint8_t* kind,
               const int32_t* pos, int32_t q, int32_t i, int64_t* a);
int or_resolve_overflow(const or_graph* g, const int64_t* c, const int64_t* w, const int64_t* mem,
                        const uint8_t* kind, int32_t n_pe, const int64_t* cap_eff, int32_t* part,
                        int32_t max_moves, int32_t* moves, int32_t* n_moves, int32_t* resolved);
/* The TF FIFO scheduler emulator (reading R17): st, ft of
 * every node under the placement `part` (labels in [0, n_pe)), the makespan,
 * and (nullable) the largest ready-queue size seen. */
int or_emulate(const or_graph* g, const int64_t* c, const int64_t* w, const int32_t* part, int32_t n_pe,
               int64_t* st, int64_t* ft, int64_t* makespan, int32_t* max_queue);
int or_eval_batch(const or_graph* g, const int64_t* c, const int64_t* w, const int64_t* mem,
                  const uint8_t* kind, int32_t n_pe, const int64_t* cap_eff, int32_t batch,
                  const uint8_t* parts, or_eval_result* out, int32_t n_threads, int32_t schedule);

#endif
