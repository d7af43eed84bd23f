/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, single-threaded (per
 * graph) CPU oracle for the weighted-level sweep of ParDNN, arXiv 2008.08636.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
 * --impl reference) may load this file's library.  It shares nothing with
 * the CUDA path: no header, helper, table or generator.
 *
 * Citations are PAPER.md line numbers (the paper's LaTeX text) plus the
 * section / table / equation / algorithm they fall in.  Where the paper is
 * silent or ambiguous the reading taken is named R1..R12 and listed in
 * DESIGN.md section "Readings of the paper".
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py
 * (closed forms, brute-force path enumeration on <=20-node DAGs, invariants,
 * and an independent interval-stabbing formulation of Eq. 3); none is
 * "parity unpinned".
 *
 * Integers only: comp(n), comm(e) are int64 nanoseconds, mem(n) int64 bytes
 * (R7).  Precondition: costs >= 0 and sum(comp)+sum(comm) < 2^62 (R7), so no
 * path length overflows; violated -> OR_EOVERFLOW / OR_EINVAL.
 */
#include "oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

struct or_graph {
    int32_t V;
    int64_t E;
    int64_t* pred_off; /* [V+1] */
    int32_t* pred;     /* [E] predecessor node ids, grouped by head node */
    int64_t* pred_eid; /* [E] index of that edge in the caller's input order */
    int64_t* succ_off; /* [V+1] */
    int32_t* succ;     /* [E] */
    int64_t* succ_eid; /* [E] */
    int32_t* topo;     /* [V] Kahn order (FIFO seeded in id order) */
    int32_t* level;    /* [V] */
    int32_t n_levels;
};

/* ------------------------------------------------------------------------ */
/* Graph construction.                                                      */
/* G = (V, E), a DAG of operation nodes (Table 2 at      */
/* PAPER.md:198).  Validation (R9): ids in range, no self loops, no         */
/* duplicate (src,dst) pairs -> OR_EINVAL; a cycle -> OR_ECYCLE.            */
/* ------------------------------------------------------------------------ */

typedef struct { int32_t s, d; } pair_t;
static int cmp_pair(const void* a, const void* b) {
    const pair_t* x = (const pair_t*)a;
    const pair_t* y = (const pair_t*)b;
    if (x->s != y->s) return x->s < y->s ? -1 : 1;
    if (x->d != y->d) return x->d < y->d ? -1 : 1;
    return 0;
}

void or_free(or_graph* g) {
    if (!g) return;
    free(g->pred_off); free(g->pred); free(g->pred_eid);
    free(g->succ_off); free(g->succ); free(g->succ_eid);
    free(g->topo); free(g->level);
    free(g);
}

int or_build(int32_t V, int64_t E, const int32_t* src, const int32_t* dst, or_graph** out) {
    *out = NULL;
    if (V < 0 || E < 0) return OR_EINVAL;
    for (int64_t k = 0; k < E; ++k) {
        if (src[k] < 0 || src[k] >= V || dst[k] < 0 || dst[k] >= V) return OR_EINVAL;
        if (src[k] == dst[k]) return OR_EINVAL;
    }
    /* duplicate pairs: sort a copy and compare neighbours */
    if (E > 1) {
        pair_t* pr = (pair_t*)malloc(sizeof(pair_t) * (size_t)E);
        if (!pr) return OR_ENOMEM;
        for (int64_t k = 0; k < E; ++k) { pr[k].s = src[k]; pr[k].d = dst[k]; }
        qsort(pr, (size_t)E, sizeof(pair_t), cmp_pair);
        for (int64_t k = 1; k < E; ++k)
            if (pr[k].s == pr[k - 1].s && pr[k].d == pr[k - 1].d) { free(pr); return OR_EINVAL; }
        free(pr);
    }
    or_graph* g = (or_graph*)calloc(1, sizeof(or_graph));
    if (!g) return OR_ENOMEM;
    g->V = V; g->E = E;
    g->pred_off = (int64_t*)calloc((size_t)V + 1, sizeof(int64_t));
    g->succ_off = (int64_t*)calloc((size_t)V + 1, sizeof(int64_t));
    g->pred = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E ? E : 1));
    g->succ = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E ? E : 1));
    g->pred_eid = (int64_t*)malloc(sizeof(int64_t) * (size_t)(E ? E : 1));
    g->succ_eid = (int64_t*)malloc(sizeof(int64_t) * (size_t)(E ? E : 1));
    g->topo = (int32_t*)malloc(sizeof(int32_t) * (size_t)(V ? V : 1));
    g->level = (int32_t*)malloc(sizeof(int32_t) * (size_t)(V ? V : 1));
    if (!g->pred_off || !g->succ_off || !g->pred || !g->succ || !g->pred_eid || !g->succ_eid ||
        !g->topo || !g->level) { or_free(g); return OR_ENOMEM; }

    /* adjacency lists, edges kept in input order inside each list */
    for (int64_t k = 0; k < E; ++k) { g->pred_off[dst[k] + 1]++; g->succ_off[src[k] + 1]++; }
    for (int32_t v = 0; v < V; ++v) {
        g->pred_off[v + 1] += g->pred_off[v];
        g->succ_off[v + 1] += g->succ_off[v];
    }
    int64_t* pfill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(V ? V : 1));
    int64_t* sfill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(V ? V : 1));
    for (int32_t v = 0; v < V; ++v) { pfill[v] = g->pred_off[v]; sfill[v] = g->succ_off[v]; }
    for (int64_t k = 0; k < E; ++k) {
        int64_t a = pfill[dst[k]]++;
        g->pred[a] = src[k]; g->pred_eid[a] = k;
        int64_t b = sfill[src[k]]++;
        g->succ[b] = dst[k]; g->succ_eid[b] = k;
    }
    free(pfill); free(sfill);

    /* Kahn's topological sort with a FIFO ready queue seeded in id order --
     * the "variant of topological sorting" of PAPER.md:5 / 270 and the
     * in-degree countdown of the TF scheduler description at PAPER.md:446.
     * level(v) = 0 for nodes without predecessors, else 1 + max level(pred). */
    int64_t* indeg = (int64_t*)malloc(sizeof(int64_t) * (size_t)(V ? V : 1));
    for (int32_t v = 0; v < V; ++v) { indeg[v] = g->pred_off[v + 1] - g->pred_off[v]; g->level[v] = 0; }
    int32_t head = 0, tail = 0;
    for (int32_t v = 0; v < V; ++v) if (indeg[v] == 0) g->topo[tail++] = v;
    while (head < tail) {
        int32_t u = g->topo[head++];
        for (int64_t a = g->succ_off[u]; a < g->succ_off[u + 1]; ++a) {
            int32_t s = g->succ[a];
            if (g->level[u] + 1 > g->level[s]) g->level[s] = g->level[u] + 1;
            if (--indeg[s] == 0) g->topo[tail++] = s;
        }
    }
    free(indeg);
    if (tail != V) { or_free(g); return OR_ECYCLE; }
    g->n_levels = 0;
    for (int32_t v = 0; v < V; ++v) if (g->level[v] + 1 > g->n_levels) g->n_levels = g->level[v] + 1;
    *out = g;
    return OR_OK;
}

int32_t or_n_levels(const or_graph* g) { return g->n_levels; }
void or_levels(const or_graph* g, int32_t* level_out) { memcpy(level_out, g->level, sizeof(int32_t) * (size_t)g->V); }
void or_topo(const or_graph* g, int32_t* topo_out) { memcpy(topo_out, g->topo, sizeof(int32_t) * (size_t)g->V); }

/* ------------------------------------------------------------------------ */
/* Labels (R2, R3): part == NULL -> every edge pays comm (slicing before    */
/* placement).  part[v] >= 0 -> PE / cluster id, comm of an   */
/* edge whose endpoints share it is zero (criticality;       */
/* refinement with PEs).  OR_REMOVED -> node and its incident  */
/* edges deleted (slicing).  OR_UNASSIGNED -> alive, never    */
/* co-located.                                                              */
/* ------------------------------------------------------------------------ */

static int alive(const int32_t* part, int32_t v) { return part == NULL || part[v] != OR_REMOVED; }

static int64_t comm_eff(const int32_t* part, int32_t u, int32_t v, int64_t w) {
    if (part == NULL) return w;
    if (part[u] == OR_UNASSIGNED || part[v] == OR_UNASSIGNED) return w;
    return part[u] == part[v] ? 0 : w;
}

static int check_inputs(const or_graph* g, const int64_t* c, const int64_t* w, const int32_t* part) {
    /* R7: non-negative integer costs whose total stays below 2^62 */
    const int64_t LIM = (int64_t)1 << 62;
    int64_t total = 0;
    for (int32_t v = 0; v < g->V; ++v) {
        if (c[v] < 0) return OR_EINVAL;
        if (c[v] >= LIM - total) return OR_EOVERFLOW;
        total += c[v];
    }
    for (int64_t k = 0; k < g->E; ++k) {
        if (w[k] < 0) return OR_EINVAL;
        if (w[k] >= LIM - total) return OR_EOVERFLOW;
        total += w[k];
    }
    if (part)
        for (int32_t v = 0; v < g->V; ++v)
            if (part[v] < 0 && part[v] != OR_REMOVED && part[v] != OR_UNASSIGNED) return OR_EINVAL;
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Weighted levels, Table 2 and Alg. 1 line 2 / 7        */
/* (PAPER.md:247, 253):                                                     */
/*   tl(n) = length of the costliest path from a source to n, EXCLUDING n;  */
/*   bl(n) = length of the costliest path from n to a sink, INCLUDING n;    */
/*   length = sum comp(n) over the path's nodes + sum comm(e) over edges.   */
/* Computed by the textbook DP over the topological order (the O(V+E)       */
/* "variant of topological sorting"):                         */
/*   tl(v) = max(0, max_{alive p in pred(v)} tl(p) + comp(p) + comm'(p,v))  */
/*   bl(u) = comp(u) + max(0, max_{alive s in succ(u)} comm'(u,s) + bl(s))  */
/* Removed nodes get tl = bl = -1 (R3).                                     */
/* ------------------------------------------------------------------------ */
int or_weighted_levels(const or_graph* g, const int64_t* c, const int64_t* w,
                       const int32_t* part, int64_t* tl, int64_t* bl) {
    int rc = check_inputs(g, c, w, part);
    if (rc) return rc;
    for (int32_t i = 0; i < g->V; ++i) {
        int32_t v = g->topo[i];
        if (!alive(part, v)) { tl[v] = -1; continue; }
        int64_t best = 0;
        for (int64_t a = g->pred_off[v]; a < g->pred_off[v + 1]; ++a) {
            int32_t p = g->pred[a];
            if (!alive(part, p)) continue;
            int64_t len = tl[p] + c[p] + comm_eff(part, p, v, w[g->pred_eid[a]]);
            if (len > best) best = len;
        }
        tl[v] = best;
    }
    for (int32_t i = g->V - 1; i >= 0; --i) {
        int32_t u = g->topo[i];
        if (!alive(part, u)) { bl[u] = -1; continue; }
        int64_t best = 0;
        for (int64_t a = g->succ_off[u]; a < g->succ_off[u + 1]; ++a) {
            int32_t s = g->succ[a];
            if (!alive(part, s)) continue;
            int64_t len = comm_eff(part, u, s, w[g->succ_eid[a]]) + bl[s];
            if (len > best) best = len;
        }
        bl[u] = c[u] + best;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Critical path (Table 2 "CP"; find_heaviest_path with fresh */
/* weighted levels).  Reading R5/R6:                     */
/*   L = max over alive n of tl(n) + bl(n);                                 */
/*   start = lowest-id alive node with no alive predecessor and bl == L;   */
/*   repeat: next = lowest-id alive successor s of u with                   */
/*           comm'(u,s) + bl(s) == bl(u) - comp(u), until u has no alive    */
/*           successor ("until reaching a dead-end").         */
/*   cp_hash = sum_k (id_k + 1) * 0x100000001B3^k  mod 2^64.                */
/* With no alive node: cp_len = 0, L = 0, hash = 0.                         */
/* cp must hold at least n_levels entries.                                  */
/* ------------------------------------------------------------------------ */
int or_critical_path(const or_graph* g, const int64_t* c, const int64_t* w,
                     const int32_t* part, const int64_t* tl, const int64_t* bl,
                     int32_t* cp, int32_t* cp_len, int64_t* L, uint64_t* cp_hash) {
    *cp_len = 0; *L = 0; *cp_hash = 0;
    int64_t best = -1;
    for (int32_t v = 0; v < g->V; ++v)
        if (alive(part, v) && tl[v] + bl[v] > best) best = tl[v] + bl[v];
    if (best < 0) return OR_OK;
    *L = best;
    int32_t start = -1;
    for (int32_t v = 0; v < g->V && start < 0; ++v) {
        if (!alive(part, v) || bl[v] != best) continue;
        int has_pred = 0;
        for (int64_t a = g->pred_off[v]; a < g->pred_off[v + 1]; ++a)
            if (alive(part, g->pred[a])) { has_pred = 1; break; }
        if (!has_pred) start = v;
    }
    if (start < 0) return OR_EINVAL; /* impossible for consistent tl/bl */
    const uint64_t P = 0x100000001B3ull;
    uint64_t h = 0, pw = 1;
    int32_t u = start, n = 0;
    for (;;) {
        cp[n++] = u;
        h += (uint64_t)(u + 1) * pw;
        pw *= P;
        int32_t nxt = -1;
        int any = 0;
        for (int64_t a = g->succ_off[u]; a < g->succ_off[u + 1]; ++a) {
            int32_t s = g->succ[a];
            if (!alive(part, s)) continue;
            any = 1;
            if (comm_eff(part, u, s, w[g->succ_eid[a]]) + bl[s] == bl[u] - c[u])
                if (nxt < 0 || s < nxt) nxt = s;
        }
        if (!any) break;
        if (nxt < 0) return OR_EINVAL; /* inconsistent tl/bl */
        u = nxt;
    }
    *cp_len = n;
    *cp_hash = h;
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Graph slicing, primary phase (Alg. 1; "repeated K      */
/* times").  Reading R4: the weighted levels are          */
/* recomputed AFTER removing the previous path, so sweep j runs on G minus  */
/* primaries 1..j-1; every alive node is UNASSIGNED (all comm counts).      */
/* cps is [K][cap] (cap >= n_levels); a slice that finds an empty graph     */
/* gets cp_len = 0, L = 0, hash = 0.                                        */
/* ------------------------------------------------------------------------ */
int or_slice(const or_graph* g, const int64_t* c, const int64_t* w, int32_t K,
             int32_t cap, int32_t* cps, int32_t* cp_lens, int64_t* Ls, uint64_t* hashes) {
    if (K < 0 || cap < g->n_levels) return OR_EINVAL;
    int32_t V = g->V;
    int32_t* lab = (int32_t*)malloc(sizeof(int32_t) * (size_t)(V ? V : 1));
    int64_t* tl = (int64_t*)malloc(sizeof(int64_t) * (size_t)(V ? V : 1));
    int64_t* bl = (int64_t*)malloc(sizeof(int64_t) * (size_t)(V ? V : 1));
    int rc = OR_OK;
    for (int32_t v = 0; v < V; ++v) lab[v] = OR_UNASSIGNED;
    for (int32_t j = 0; j < K && rc == OR_OK; ++j) {
        rc = or_weighted_levels(g, c, w, lab, tl, bl);
        if (rc) break;
        int32_t* cp = cps + (int64_t)j * cap;
        rc = or_critical_path(g, c, w, lab, tl, bl, cp, &cp_lens[j], &Ls[j], &hashes[j]);
        for (int32_t k = 0; k < cp_lens[j]; ++k) lab[cp[k]] = OR_REMOVED; /* G <- G - path */
    }
    free(lab); free(tl); free(bl);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Graph slicing, whole of Alg. 1 -- NEXT row N2.        */
/* Primaries: the K-loop above (R4).  Then "we stop recalculating w_lvl(n)  */
/* for the secondary clusters": one last recomputation on G  */
/* minus the primaries gives the stale priorities w_lvl = tl + bl (Table 2, */
/* every edge paying comm, as in the K-loop), and secondary clusters are    */
/* extracted "until there is no node left" by               */
/* find_heaviest_path with those priorities: "traversing the graph using   */
/* the computed w_lvls as priorities until reaching a dead-end" (PAPER.md: */
/* 265); "if a path could not be obtained, it returns a single node"       */
/* (PAPER.md:268).  Reading R18 (after SPEC.md:126, 149-150):    */
/* start = the unvisited node of maximum w_lvl (lowest id on ties); extend  */
/* forward by the unvisited successor of maximum w_lvl (lowest id), then    */
/* backward from the start by the unvisited predecessor of maximum w_lvl;   */
/* the path's nodes are marked visited.                                     */
/* Outputs: cluster_of[v] (0..K-1 primaries -- an exhausted graph leaves a  */
/* primary empty -- then the secondaries in extraction order), members      */
/* (cluster by cluster, path order), cl_off[n_clusters + 1].                */
/* ------------------------------------------------------------------------ */
typedef struct { int64_t w; int32_t id; } prio_t;
static int prio_cmp(const void* a, const void* b) {   /* w descending, id ascending */
    const prio_t* x = (const prio_t*)a;
    const prio_t* y = (const prio_t*)b;
    if (x->w != y->w) return x->w > y->w ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

int or_slice_clusters(const or_graph* g, const int64_t* c, const int64_t* w, int32_t K, int32_t* cluster_of,
                      int32_t* members, int32_t* cl_off, int32_t* n_clusters) {
    int32_t V = g->V;
    if (K < 0) return OR_EINVAL;
    size_t n = (size_t)(V ? V : 1);
    int32_t* lab = (int32_t*)malloc(sizeof(int32_t) * n);
    int64_t* tl = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t* bl = (int64_t*)malloc(sizeof(int64_t) * n);
    int32_t* cp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->n_levels + 1));
    prio_t* order = (prio_t*)malloc(sizeof(prio_t) * n);
    int32_t* path = (int32_t*)malloc(sizeof(int32_t) * n);
    if (!lab || !tl || !bl || !cp || !order || !path) {
        free(lab); free(tl); free(bl); free(cp); free(order); free(path);
        return OR_ENOMEM;
    }
    int rc = OR_OK;
    int32_t nc = 0, m = 0;
    for (int32_t v = 0; v < V; ++v) { lab[v] = OR_UNASSIGNED; cluster_of[v] = -1; }
    cl_off[0] = 0;
    /* primaries: Alg. 1 lines 4-7 and 11, K times (R4) */
    for (int32_t j = 0; j < K && rc == OR_OK; ++j) {
        int32_t len = 0;
        int64_t L = 0;
        uint64_t h = 0;
        rc = or_weighted_levels(g, c, w, lab, tl, bl);
        if (rc) break;
        rc = or_critical_path(g, c, w, lab, tl, bl, cp, &len, &L, &h);
        for (int32_t k = 0; k < len; ++k) {
            lab[cp[k]] = OR_REMOVED;
            cluster_of[cp[k]] = nc;
            members[m++] = cp[k];
        }
        cl_off[++nc] = m;
    }
    /* the stale priorities of the secondary phase */
    if (rc == OR_OK) rc = or_weighted_levels(g, c, w, lab, tl, bl);
    if (rc == OR_OK) {
        int32_t no = 0;
        for (int32_t v = 0; v < V; ++v)
            if (lab[v] != OR_REMOVED) { order[no].w = tl[v] + bl[v]; order[no].id = v; ++no; }
        qsort(order, (size_t)no, sizeof(prio_t), prio_cmp);
        for (int32_t i = 0; i < no; ++i) {
            int32_t s0 = order[i].id;
            if (cluster_of[s0] >= 0) continue;            /* visited */
            /* forward from the start, then backward from it */
            int32_t fw = 0;
            path[fw++] = s0;
            cluster_of[s0] = nc;
            for (int32_t u = s0;;) {
                int32_t best = -1;
                for (int64_t a = g->succ_off[u]; a < g->succ_off[u + 1]; ++a) {
                    int32_t s = g->succ[a];
                    if (cluster_of[s] >= 0) continue;
                    if (best < 0 || tl[s] + bl[s] > tl[best] + bl[best] ||
                        (tl[s] + bl[s] == tl[best] + bl[best] && s < best)) best = s;
                }
                if (best < 0) break;                      /* dead end */
                cluster_of[best] = nc;
                path[fw++] = best;
                u = best;
            }
            int32_t bw = 0;                               /* predecessors, collected in reverse */
            for (int32_t u = s0;;) {
                int32_t best = -1;
                for (int64_t a = g->pred_off[u]; a < g->pred_off[u + 1]; ++a) {
                    int32_t p = g->pred[a];
                    if (cluster_of[p] >= 0) continue;
                    if (best < 0 || tl[p] + bl[p] > tl[best] + bl[best] ||
                        (tl[p] + bl[p] == tl[best] + bl[best] && p < best)) best = p;
                }
                if (best < 0) break;
                cluster_of[best] = nc;
                members[m + bw++] = best;                 /* temporarily, reversed below */
                u = best;
            }
            for (int32_t a = 0, b = bw - 1; a < b; ++a, --b) {
                int32_t t = members[m + a]; members[m + a] = members[m + b]; members[m + b] = t;
            }
            for (int32_t k = 0; k < fw; ++k) members[m + bw + k] = path[k];
            m += bw + fw;
            cl_off[++nc] = m;
        }
    }
    *n_clusters = nc;
    free(lab); free(tl); free(bl); free(cp); free(order); free(path);
    return rc;
}

/* Criticality of the clusters (LFLAM): "the length of the   */
/* longest path going from the graph source to its sink and completely     */
/* overlapping with lc ... equivalent to the w_lvl(n) for n in lc, where    */
/* w_lvl(n) is recalculated by setting communications within lcs to zeros  */
/* after the slicing stage".  Reading R19: labels = cluster ids (R2 zeroes  */
/* intra-cluster comm), crit[k] = max over n in cluster k of tl(n) + bl(n). */
int or_criticality(const or_graph* g, const int64_t* c, const int64_t* w, const int32_t* cluster_of,
                   int32_t n_clusters, int64_t* crit) {
    int32_t V = g->V;
    for (int32_t v = 0; v < V; ++v)
        if (cluster_of[v] < 0 || cluster_of[v] >= n_clusters) return OR_EINVAL;
    size_t n = (size_t)(V ? V : 1);
    int64_t* tl = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t* bl = (int64_t*)malloc(sizeof(int64_t) * n);
    if (!tl || !bl) { free(tl); free(bl); return OR_ENOMEM; }
    int rc = or_weighted_levels(g, c, w, cluster_of, tl, bl);
    for (int32_t k = 0; k < n_clusters; ++k) crit[k] = 0;
    if (rc == OR_OK)
        for (int32_t v = 0; v < V; ++v)
            if (tl[v] + bl[v] > crit[cluster_of[v]]) crit[cluster_of[v]] = tl[v] + bl[v];
    free(tl); free(bl);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Memory consumption tracker (Heuristic I; Eq. 3 at       */
/* PAPER.md:465-481; M_pot in Table 2).  Readings R8-R12:      */
/*  M1 st = caller's st (the oracle takes it explicitly).                   */
/*  M2 visit order = nodes sorted by (st, level, id): "visiting all the     */
/*     nodes in the graph in the order of their estimated starting times"   */
/*     (PAPER.md:487); pos(n) = rank in that order.                         */
/*  M3 effmem(n) = 0 for reference nodes ("do not reserve any additional    */
/*     memory"), else mem(n).                                 */
/*  The pass: "A node's memory consumption is added to the   */
/*  cumulative value once it is visited, and subtracted after its last      */
/*  descendent in a certain pe is visited unless it is a res_ns."          */
/*   - residual n: held on pe(n) for the whole pass (Eq. 3 term 1);         */
/*   - normal n: held on pe(n) from its visit until its last consumer on    */
/*     pe(n) has been visited, or just its own visit if it has none there  */
/*     (Eq. 3 terms 2+3);                                                   */
/*   - any non-reference n with consumers on q != pe(n): held on q from its */
/*     visit until its last consumer on q has been visited (Eq. 3 term 3).  */
/*  M_cons(q, i) is the cumulative value on q after the additions of the   */
/*  i-th visit and before its subtractions (closed intervals, "<= t <=").  */
/*  M6 per q: peak = max_i, peak_pos = lowest i attaining it, first_over =  */
/*     lowest i with M_cons > cap_eff[q] (-1 if none), over_bytes =         */
/*     M_cons(q, first_over) - cap_eff[q] (0 if none).                      */
/*  M7 mpot(n) = effmem(n) + sum effmem(p) over predecessors p for which n  */
/*     is the last direct descendant on pe(n), excluding residual p with    */
/*     pe(p) = pe(n) (Table 2 M_pot evaluated at n's own visit).            */
/* part must be in [0, n_pe).  mcons (nullable) is [n_pe][V]; order_out     */
/* (nullable) receives the visit order.                                    */
/* ------------------------------------------------------------------------ */

typedef struct { int64_t st; int32_t level, id; } vkey_t;
static int cmp_vkey(const void* a, const void* b) {
    const vkey_t* x = (const vkey_t*)a;
    const vkey_t* y = (const vkey_t*)b;
    if (x->st != y->st) return x->st < y->st ? -1 : 1;
    if (x->level != y->level) return x->level < y->level ? -1 : 1;
    if (x->id != y->id) return x->id < y->id ? -1 : 1;
    return 0;
}

int or_memory(const or_graph* g, const int32_t* part, int32_t P, const int64_t* mem,
              const uint8_t* kind, const int64_t* st, const int64_t* cap_eff,
              int64_t* mpot, int64_t* peak, int32_t* peak_pos, int32_t* first_over,
              int64_t* over_bytes, int64_t* mcons, int32_t* order_out) {
    int32_t V = g->V;
    if (P < 1 || P > OR_MAX_PE) return OR_EINVAL;
    for (int32_t v = 0; v < V; ++v) {
        if (part[v] < 0 || part[v] >= P) return OR_EINVAL;
        if (mem[v] < 0 || kind[v] > OR_KIND_REFERENCE || st[v] < 0) return OR_EINVAL;
    }
    /* st must not decrease along an edge, otherwise (st, level, id) is not a
     * topological visit order (R10) */
    for (int32_t u = 0; u < V; ++u)
        for (int64_t a = g->succ_off[u]; a < g->succ_off[u + 1]; ++a)
            if (st[g->succ[a]] < st[u]) return OR_EINVAL;

    vkey_t* keys = (vkey_t*)malloc(sizeof(vkey_t) * (size_t)(V ? V : 1));
    int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)(V ? V : 1));
    int64_t* effmem = (int64_t*)malloc(sizeof(int64_t) * (size_t)(V ? V : 1));
    int32_t* last = (int32_t*)malloc(sizeof(int32_t) * (size_t)(V ? V : 1) * (size_t)P);
    if (!keys || !pos || !effmem || !last) { free(keys); free(pos); free(effmem); free(last); return OR_ENOMEM; }

    for (int32_t v = 0; v < V; ++v) { keys[v].st = st[v]; keys[v].level = g->level[v]; keys[v].id = v; }
    qsort(keys, (size_t)V, sizeof(vkey_t), cmp_vkey);                       /* M2 */
    for (int32_t i = 0; i < V; ++i) pos[keys[i].id] = i;
    if (order_out) for (int32_t i = 0; i < V; ++i) order_out[i] = keys[i].id;
    for (int32_t v = 0; v < V; ++v) effmem[v] = kind[v] == OR_KIND_REFERENCE ? 0 : mem[v];   /* M3 */

    /* last[n][q] = position of n's last direct descendant on q, -1 if none */
    for (int64_t k = 0; k < (int64_t)V * P; ++k) last[k] = -1;
    for (int32_t n = 0; n < V; ++n)
        for (int64_t a = g->succ_off[n]; a < g->succ_off[n + 1]; ++a) {
            int32_t u = g->succ[a];
            int32_t* l = &last[(int64_t)n * P + part[u]];
            if (pos[u] > *l) *l = pos[u];
        }

    int64_t cur[OR_MAX_PE];
    for (int32_t q = 0; q < P; ++q) {
        cur[q] = 0; peak[q] = 0; peak_pos[q] = -1; first_over[q] = -1; over_bytes[q] = 0;
    }
    for (int32_t n = 0; n < V; ++n)                                        /* Eq. 3 term 1 */
        if (kind[n] == OR_KIND_RESIDUAL) cur[part[n]] += effmem[n];

    for (int32_t i = 0; i < V; ++i) {
        int32_t n = keys[i].id, h = part[n];
        /* additions at n's visit */
        if (kind[n] == OR_KIND_NORMAL) cur[h] += effmem[n];
        for (int32_t q = 0; q < P; ++q)
            if (q != h && last[(int64_t)n * P + q] >= 0) cur[q] += effmem[n];
        /* record M_cons(q, i) */
        for (int32_t q = 0; q < P; ++q) {
            if (mcons) mcons[(int64_t)q * V + i] = cur[q];
            if (peak_pos[q] < 0 || cur[q] > peak[q]) { peak[q] = cur[q]; peak_pos[q] = i; }
            if (first_over[q] < 0 && cur[q] > cap_eff[q]) { first_over[q] = i; over_bytes[q] = cur[q] - cap_eff[q]; }
        }
        /* subtractions after n's visit, and M_pot(n) (M7) */
        int64_t pot = effmem[n];
        for (int64_t a = g->pred_off[n]; a < g->pred_off[n + 1]; ++a) {
            int32_t p = g->pred[a];
            if (last[(int64_t)p * P + h] != i) continue;      /* n is not p's last descendant on h */
            if (kind[p] == OR_KIND_RESIDUAL && part[p] == h) continue;
            cur[h] -= effmem[p];
            pot += effmem[p];
        }
        if (kind[n] == OR_KIND_NORMAL && last[(int64_t)n * P + h] < 0) cur[h] -= effmem[n];
        mpot[n] = pot;
    }
    free(keys); free(pos); free(effmem); free(last);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Batched evaluation: the oracle steps above, run once per candidate       */
/* placement (refinement / LALB trials).  One          */
/* candidate per host thread; each evaluation is the single-graph sequence: */
/* weighted levels under part_b, CP, memory tracker with st = tl (R8),       */
/* cut_comm = sum comm(e) over edges whose endpoints differ in part_b.      */
/* ------------------------------------------------------------------------ */
/* ------------------------------------------------------------------------ */
/* LFLAM mapping (Alg. 2; Eq. 2) -- NEXT row N4.          */
/* Reading R21: clusters from or_slice_clusters; primary k is   */
/* PE k.  "Level" = the node's depth level; span(sc) = the levels strictly  */
/* after its first node's latest parent and strictly before its last node's */
/* earliest child ([0, D-1] without them); work(pe, sc) = sum comp over     */
/* nodes mapped to pe with level in span(sc) ("binary-indexed-trees, where  */
/* the tree nodes store the weights per level"); U = the same */
/* over the nodes of unmapped secondaries other than sc; comm(sc, pe) = sum */
/* comm of the edges between sc and nodes mapped to pe; ext(sc) = sum comm  */
/* of the edges with exactly one end in sc.  Secondaries are processed in   */
/* non-increasing criticality (R19), lower index first.                     */
/* Locality-first lookahead: eligible = totally-         */
/* communicating (ext > 0 and one pe takes all of it) or, when CCR >= 10,   */
/* maximally-communicating (comm(sc, t) * K > ext); t = the most            */
/* communicating pe (lowest on ties); mapped if (a) U >= max(0, work(t) +   */
/* w(sc) - floor(mean work)), (b) work(t) + w(sc) <= max work, or (c)       */
/* comm(sc, t) > w(sc), > work(t) and > U.  Passes repeat while one maps a  */
/* cluster, at most ceil(log2 |V|) times.  Level-aware       */
/* balancing (Eq. 2): min over pe of work(pe, sc) + comm(sc, other pes);    */
/* ties: the most communicating pe, then the lowest.                        */
/* log: [n][3] = (cluster, phase 0 lookahead / 1 balancing, pe).            */
/* ------------------------------------------------------------------------ */
static void fw_add(int64_t* t, int32_t n, int32_t i, int64_t v) {
    for (++i; i <= n; i += i & -i) t[i] += v;
}
static int64_t fw_pre(const int64_t* t, int32_t i) {   /* sum of levels [0, i) */
    int64_t s = 0;
    for (; i > 0; i -= i & -i) s += t[i];
    return s;
}
static int64_t fw_range(const int64_t* t, int32_t lo, int32_t hi) {   /* [lo, hi] */
    return hi < lo ? 0 : fw_pre(t, hi + 1) - fw_pre(t, lo);
}

int or_lflam(const or_graph* g, const int64_t* c, const int64_t* w, const int32_t* cluster_of,
             const int32_t* members, const int32_t* cl_off, int32_t n_clusters, int32_t K, int32_t* part,
             int32_t* log, int32_t* n_log) {
    int32_t V = g->V, D = g->n_levels;
    if (K < 1 || K > OR_MAX_PE || n_clusters < K) return OR_EINVAL;
    int64_t* crit = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_clusters);
    int64_t* tree = (int64_t*)calloc((size_t)(K + 1) * (size_t)(D + 1), sizeof(int64_t));   /* K pes + unmapped */
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_clusters);
    uint8_t* mapped = (uint8_t*)calloc((size_t)n_clusters, 1);
    if (!crit || !tree || !order || !mapped) { free(crit); free(tree); free(order); free(mapped); return OR_ENOMEM; }
    int rc = or_criticality(g, c, w, cluster_of, n_clusters, crit);
    if (rc) { free(crit); free(tree); free(order); free(mapped); return rc; }
    int64_t* unm = tree + (size_t)K * (D + 1);
    for (int32_t v = 0; v < V; ++v) {
        int32_t k = cluster_of[v];
        part[v] = k < K ? k : -1;
        fw_add(k < K ? tree + (size_t)k * (D + 1) : unm, D, g->level[v], c[v]);
    }
    for (int32_t k = 0; k < K; ++k) mapped[k] = 1;
    /* non-increasing criticality, lower index first (insertion into a sorted list) */
    int32_t ns = 0;
    for (int32_t k = K; k < n_clusters; ++k) order[ns++] = k;
    for (int32_t a = 1; a < ns; ++a) {
        int32_t x = order[a], b = a - 1;
        while (b >= 0 && (crit[order[b]] < crit[x] || (crit[order[b]] == crit[x] && order[b] > x))) {
            order[b + 1] = order[b];
            --b;
        }
        order[b + 1] = x;
    }
    int64_t sum_c = 0, sum_w = 0;
    for (int32_t v = 0; v < V; ++v) sum_c += c[v];
    for (int64_t e = 0; e < g->E; ++e) sum_w += w[e];
    const int high_ccr = sum_w >= 10 * sum_c;
    int32_t max_iter = 0;
    while ((1ll << max_iter) < (int64_t)V) ++max_iter;     /* ceil(log2 |V|) */
    if (max_iter < 1) max_iter = 1;
    int32_t nl = 0;
    for (int phase = 0; phase < 2; ++phase) {
        for (int32_t iter = 0; iter < (phase == 0 ? max_iter : 1); ++iter) {
            int32_t n_mapped = 0;
            for (int32_t oi = 0; oi < ns; ++oi) {
                const int32_t k = order[oi];
                if (mapped[k]) continue;
                const int32_t h = members[cl_off[k]], tl_ = members[cl_off[k + 1] - 1];
                int32_t lo = 0, hi = D - 1;
                for (int64_t a = g->pred_off[h]; a < g->pred_off[h + 1]; ++a)
                    if (cluster_of[g->pred[a]] != k && g->level[g->pred[a]] + 1 > lo) lo = g->level[g->pred[a]] + 1;
                for (int64_t a = g->succ_off[tl_]; a < g->succ_off[tl_ + 1]; ++a)
                    if (cluster_of[g->succ[a]] != k && g->level[g->succ[a]] - 1 < hi) hi = g->level[g->succ[a]] - 1;
                int64_t wsc = 0, comm[OR_MAX_PE], ext = 0;
                for (int32_t q = 0; q < K; ++q) comm[q] = 0;
                for (int32_t m = cl_off[k]; m < cl_off[k + 1]; ++m) {
                    int32_t u = members[m];
                    wsc += c[u];
                    for (int64_t a = g->pred_off[u]; a < g->pred_off[u + 1]; ++a) {
                        int32_t x = g->pred[a];
                        if (cluster_of[x] == k) continue;
                        ext += w[g->pred_eid[a]];
                        if (part[x] >= 0) comm[part[x]] += w[g->pred_eid[a]];
                    }
                    for (int64_t a = g->succ_off[u]; a < g->succ_off[u + 1]; ++a) {
                        int32_t x = g->succ[a];
                        if (cluster_of[x] == k) continue;
                        ext += w[g->succ_eid[a]];
                        if (part[x] >= 0) comm[part[x]] += w[g->succ_eid[a]];
                    }
                }
                int64_t work[OR_MAX_PE], sum = 0, mx = 0, tot_comm = 0;
                for (int32_t q = 0; q < K; ++q) {
                    work[q] = fw_range(tree + (size_t)q * (D + 1), lo, hi);
                    sum += work[q];
                    if (work[q] > mx) mx = work[q];
                    tot_comm += comm[q];
                }
                int32_t tgt = -1;
                if (phase == 0) {
                    int32_t t = 0;
                    for (int32_t q = 1; q < K; ++q) if (comm[q] > comm[t]) t = q;
                    const int totally = ext > 0 && comm[t] == ext;
                    const int maximally = comm[t] * K > ext;
                    if (!(totally || (high_ccr && maximally))) continue;
                    const int64_t U = fw_range(unm, lo, hi) - wsc;
                    int64_t imb = work[t] + wsc - sum / K;
                    if (imb < 0) imb = 0;
                    const int ca = U >= imb, cb = work[t] + wsc <= mx;
                    const int cc = comm[t] > wsc && comm[t] > work[t] && comm[t] > U;
                    if (!(ca || cb || cc)) continue;
                    tgt = t;
                } else {
                    int64_t best = 0;
                    for (int32_t q = 0; q < K; ++q) {
                        const int64_t cost = work[q] + (tot_comm - comm[q]);      /* Eq. 2 */
                        if (tgt < 0 || cost < best || (cost == best && comm[q] > comm[tgt])) { tgt = q; best = cost; }
                    }
                }
                /* target_pri <- target_pri + {sc} */
                mapped[k] = 1;
                ++n_mapped;
                for (int32_t m = cl_off[k]; m < cl_off[k + 1]; ++m) {
                    int32_t u = members[m];
                    part[u] = tgt;
                    fw_add(tree + (size_t)tgt * (D + 1), D, g->level[u], c[u]);
                    fw_add(unm, D, g->level[u], -c[u]);
                }
                log[3 * nl] = k; log[3 * nl + 1] = phase; log[3 * nl + 2] = tgt;
                ++nl;
            }
            if (phase == 0 && n_mapped == 0) break;
        }
    }
    *n_log = nl;
    free(crit); free(tree); free(order); free(mapped);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Refinement (appendix "Complexity of Refinement") -- the  */
/* second half of NEXT row N4, in reading R22:                  */
/* Phase 1, cluster swaps: "we sort the clusters by tl(n) of their source   */
/* nodes to find the clusters within the span of a certain cluster using    */
/* binary search ... Once two clusters are swapped, they are marked and not */
/* considered again ... With each swap the binary-indexed-trees are updated */
/* to reflect the new work loads."  tl under `part` once; the secondaries   */
/* (clusters >= K, non-empty) sorted by (tl(first member), id); span_t(A) = */
/* [tl(h_A), tl(t_A) + comp(t_A)] (h / t = first / last member); for every  */
/* unmarked A in that order (on PE a = part[h_A]) the candidates are the    */
/* first `window` unmarked B != A in sorted order with tl(h_B) in span_t(A) */
/* and part[h_B] = b != a; gain(A, B) = cut comm before - after moving A's  */
/* members to b and B's to a (every edge with an end in A or B, once);      */
/* balance: over the levels R = [min(lvl h_A, lvl h_B), max(lvl t_A, lvl    */
/* t_B)], max(work(a,R) - w(A) + w(B), work(b,R) - w(B) + w(A)) <=          */
/* max(work(a,R), work(b,R)) (work from level-indexed Fenwick trees, w(X) = */
/* comp of X's members); the B with the largest gain > 0 passing the        */
/* balance test (earliest in sorted order on ties) is swapped, both marked. */
/* Phase 2, node level: "The node-level refinement is repeated K times and  */
/* each time we recalculate the weighted levels and the CP.  Upon node      */
/* switching we update the trees."  Per pass: tl, bl, CP (R5) under part,   */
/* L_cur = L; trials (n, q): for CP index k, n = cp[k], q = part of cp[k-1] */
/* then of cp[k+1] when it differs from part[n] (no duplicate (n, q)); then */
/* rounds: the alive trials with work(q, lvl n) + comp(n) <= max_p work(p,  */
/* lvl n) are evaluated (L of part with n moved to q); the least L (earliest */
/* trial on ties) is applied if it is < L_cur (L_cur <- it, n's trials     */
/* dropped, trees updated), else the pass ends.                             */
/* Precondition: every cluster's members share one PE (LFLAM's output).     */
/* log: [n][4] = (0, A, B, gain) swaps, then (1, node, to PE, L) moves.     */
/* ------------------------------------------------------------------------ */
static int64_t rf_level_work(const int64_t* tree, int32_t D, int32_t lo, int32_t hi) {
    (void)D;
    return fw_range(tree, lo, hi);
}

static int64_t rf_L(const or_graph* g, const int64_t* c, const int64_t* w, const int32_t* part, int64_t* tl,
                    int64_t* bl) {
    or_weighted_levels(g, c, w, part, tl, bl);
    int64_t L = 0;
    for (int32_t v = 0; v < g->V; ++v)
        if (tl[v] + bl[v] > L) L = tl[v] + bl[v];
    return L;
}

int or_refine(const or_graph* g, const int64_t* c, const int64_t* w, const int32_t* cluster_of,
              const int32_t* members, const int32_t* cl_off, int32_t n_clusters, int32_t K, int32_t passes,
              int32_t window, int32_t* part, int64_t* log, int32_t log_cap, int32_t* n_log, int64_t* L_out) {
    const int32_t V = g->V, D = g->n_levels;
    *n_log = 0;
    if (K < 1 || K > OR_MAX_PE || n_clusters < K || passes < 0 || window < 1) return OR_EINVAL;
    for (int32_t k = 0; k < n_clusters; ++k)
        for (int32_t m = cl_off[k]; m < cl_off[k + 1]; ++m)
            if (part[members[m]] != part[members[cl_off[k]]]) return OR_EINVAL;
    for (int32_t v = 0; v < V; ++v)
        if (part[v] < 0 || part[v] >= K) return OR_EINVAL;
    int64_t* tl = (int64_t*)malloc(sizeof(int64_t) * (size_t)(V + 1));
    int64_t* bl = (int64_t*)malloc(sizeof(int64_t) * (size_t)(V + 1));
    int64_t* tree = (int64_t*)calloc((size_t)K * (size_t)(D + 1), sizeof(int64_t));
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_clusters + 1));
    uint8_t* marked = (uint8_t*)calloc((size_t)n_clusters + 1, 1);
    int32_t* cp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(D + 1));
    int32_t* tn = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * D + 2));
    int32_t* tq = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * D + 2));
    uint8_t* tdead = (uint8_t*)malloc((size_t)(2 * D + 2));
    int32_t* trial = (int32_t*)malloc(sizeof(int32_t) * (size_t)(V + 1));
    int rc = OR_OK;
    if (!tl || !bl || !tree || !order || !marked || !cp || !tn || !tq || !tdead || !trial) { rc = OR_ENOMEM; goto done; }
    for (int32_t v = 0; v < V; ++v) fw_add(tree + (size_t)part[v] * (D + 1), D, g->level[v], c[v]);
    int32_t nl = 0;
#define RF_LOG(a_, b_, c_, d_)                                                   \
    do {                                                                         \
        if (nl < log_cap) {                                                      \
            log[4 * (int64_t)nl] = (a_); log[4 * (int64_t)nl + 1] = (b_);         \
            log[4 * (int64_t)nl + 2] = (c_); log[4 * (int64_t)nl + 3] = (d_);     \
        }                                                                        \
        ++nl;                                                                    \
    } while (0)

    /* ---- phase 1: cluster swaps ---- */
    or_weighted_levels(g, c, w, part, tl, bl);
    int32_t ns = 0;
    for (int32_t k = K; k < n_clusters; ++k)
        if (cl_off[k + 1] > cl_off[k]) order[ns++] = k;
    for (int32_t a = 1; a < ns; ++a) {   /* insertion sort by (tl(h), id) */
        int32_t x = order[a], b = a - 1;
        const int64_t tx = tl[members[cl_off[x]]];
        while (b >= 0 && (tl[members[cl_off[order[b]]]] > tx ||
                          (tl[members[cl_off[order[b]]]] == tx && order[b] > x))) {
            order[b + 1] = order[b];
            --b;
        }
        order[b + 1] = x;
    }
    for (int32_t oi = 0; oi < ns; ++oi) {
        const int32_t A = order[oi];
        if (marked[A]) continue;
        const int32_t hA = members[cl_off[A]], tA = members[cl_off[A + 1] - 1];
        const int32_t pa = part[hA];
        const int64_t s0 = tl[hA], s1 = tl[tA] + c[tA];
        int64_t wA = 0;
        for (int32_t m = cl_off[A]; m < cl_off[A + 1]; ++m) wA += c[members[m]];
        /* binary search: first sorted position with tl(h) >= s0 */
        int32_t lo = 0, hi = ns;
        while (lo < hi) {
            int32_t mid = (lo + hi) / 2;
            if (tl[members[cl_off[order[mid]]]] < s0) lo = mid + 1; else hi = mid;
        }
        int32_t best = -1;
        int64_t best_gain = 0;
        int32_t seen = 0;
        for (int32_t bi = lo; bi < ns && seen < window; ++bi) {
            const int32_t B = order[bi];
            const int32_t hB = members[cl_off[B]], tB = members[cl_off[B + 1] - 1];
            if (tl[hB] > s1) break;
            if (B == A || marked[B] || part[hB] == pa) continue;
            ++seen;
            const int32_t pb = part[hB];
            /* gain: every edge with an end in A or B, once (edges of A, then edges of B not ending in A) */
            int64_t before = 0, after = 0;
            for (int pass_ = 0; pass_ < 2; ++pass_) {
                const int32_t X = pass_ == 0 ? A : B;
                for (int32_t m = cl_off[X]; m < cl_off[X + 1]; ++m) {
                    const int32_t u = members[m];
                    const int32_t nu = X == A ? pb : pa;
                    for (int dir = 0; dir < 2; ++dir) {
                        const int64_t e0 = dir ? g->succ_off[u] : g->pred_off[u];
                        const int64_t e1 = dir ? g->succ_off[u + 1] : g->pred_off[u + 1];
                        for (int64_t e = e0; e < e1; ++e) {
                            const int32_t y = dir ? g->succ[e] : g->pred[e];
                            const int64_t we = w[dir ? g->succ_eid[e] : g->pred_eid[e]];
                            if (cluster_of[y] == X) continue;   /* both ends move together: never cut */
                            if (X == B && cluster_of[y] == A) continue;   /* counted with A */
                            const int32_t ny = cluster_of[y] == A ? pb : (cluster_of[y] == B ? pa : part[y]);
                            before += part[u] != part[y] ? we : 0;
                            after += nu != ny ? we : 0;
                        }
                    }
                }
            }
            const int64_t gain = before - after;
            if (gain <= 0) continue;
            int64_t wB = 0;
            for (int32_t m = cl_off[B]; m < cl_off[B + 1]; ++m) wB += c[members[m]];
            int32_t rl = g->level[hA] < g->level[hB] ? g->level[hA] : g->level[hB];
            int32_t rh = g->level[tA] > g->level[tB] ? g->level[tA] : g->level[tB];
            const int64_t wa = rf_level_work(tree + (size_t)pa * (D + 1), D, rl, rh);
            const int64_t wb = rf_level_work(tree + (size_t)pb * (D + 1), D, rl, rh);
            const int64_t na = wa - wA + wB, nb = wb - wB + wA;
            const int64_t mb = wa > wb ? wa : wb, mn = na > nb ? na : nb;
            if (mn > mb) continue;
            if (best < 0 || gain > best_gain) { best = B; best_gain = gain; }
        }
        if (best < 0) continue;
        const int32_t pb = part[members[cl_off[best]]];
        for (int32_t m = cl_off[A]; m < cl_off[A + 1]; ++m) {
            const int32_t u = members[m];
            fw_add(tree + (size_t)pa * (D + 1), D, g->level[u], -c[u]);
            fw_add(tree + (size_t)pb * (D + 1), D, g->level[u], c[u]);
            part[u] = pb;
        }
        for (int32_t m = cl_off[best]; m < cl_off[best + 1]; ++m) {
            const int32_t u = members[m];
            fw_add(tree + (size_t)pb * (D + 1), D, g->level[u], -c[u]);
            fw_add(tree + (size_t)pa * (D + 1), D, g->level[u], c[u]);
            part[u] = pa;
        }
        marked[A] = marked[best] = 1;
        RF_LOG(0, A, best, best_gain);
    }

    /* ---- phase 2: node-level refinement, `passes` times ---- */
    int64_t L_cur = 0;
    for (int32_t ps = 0; ps < passes; ++ps) {
        or_weighted_levels(g, c, w, part, tl, bl);
        int32_t cl = 0;
        uint64_t h;
        if ((rc = or_critical_path(g, c, w, part, tl, bl, cp, &cl, &L_cur, &h))) goto done;
        int32_t nt = 0;
        for (int32_t k = 0; k < cl; ++k) {
            const int32_t n = cp[k];
            for (int side = 0; side < 2; ++side) {
                if ((side == 0 && k == 0) || (side == 1 && k == cl - 1)) continue;
                const int32_t q = part[cp[side == 0 ? k - 1 : k + 1]];
                if (q == part[n]) continue;
                if (nt > 0 && tn[nt - 1] == n && tq[nt - 1] == q) continue;
                tn[nt] = n; tq[nt] = q; tdead[nt] = 0; ++nt;
            }
        }
        for (;;) {
            int32_t bt = -1;
            int64_t bL = 0;
            for (int32_t t = 0; t < nt; ++t) {
                if (tdead[t]) continue;
                const int32_t n = tn[t], q = tq[t], l = g->level[n];
                int64_t mx = 0;
                for (int32_t p = 0; p < K; ++p) {
                    const int64_t x = rf_level_work(tree + (size_t)p * (D + 1), D, l, l);
                    if (x > mx) mx = x;
                }
                if (rf_level_work(tree + (size_t)q * (D + 1), D, l, l) + c[n] > mx) continue;
                memcpy(trial, part, sizeof(int32_t) * (size_t)V);
                trial[n] = q;
                const int64_t Lt = rf_L(g, c, w, trial, tl, bl);
                if (bt < 0 || Lt < bL) { bt = t; bL = Lt; }
            }
            if (bt < 0 || bL >= L_cur) break;
            const int32_t n = tn[bt], q = tq[bt];
            fw_add(tree + (size_t)part[n] * (D + 1), D, g->level[n], -c[n]);
            fw_add(tree + (size_t)q * (D + 1), D, g->level[n], c[n]);
            part[n] = q;
            L_cur = bL;
            for (int32_t t = 0; t < nt; ++t)
                if (tn[t] == n) tdead[t] = 1;
            RF_LOG(1, n, q, bL);
        }
    }
#undef RF_LOG
    *L_out = rf_L(g, c, w, part, tl, bl);
    *n_log = nl;
done:
    free(tl); free(bl); free(tree); free(order); free(marked); free(cp); free(tn); free(tq); free(tdead); free(trial);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Overflow handler of Memory Heuristic I -- NEXT row N3. */
/* Reading R20:                                                 */
/*  - M_pot(n, t) (Table 2) at visit position i on q =        */
/*    part[n]: "the summation of the memory occupied by the outputs of n's  */
/*    direct ancestors that are executed before t, and for which n is the   */
/*    last direct descendant in its pe" -- ancestors p with pos(p) <= i <=  */
/*    pos(n), n = p's last consumer on q, p not residual on q -- "plus n's   */
/*    memory consumption if st(n) <= t <= ft(n)" -- effmem(n) if pos(n) = i; */
/*  - the overflow handled next is the earliest first_over position over    */
/*    the PEs (lowest PE on ties); O = its over_bytes (Eq. 4's O);           */
/*  - candidates: normal nodes on that PE, never moved or rejected before,  */
/*    with a = M_pot(n, i) > 0; c = move_cost (Eq. 5): comp(n) + the comm    */
/*    of n's edges to predecessors and successors on the same PE;           */
/*  - "The movement criteria is to pick the node that has the lowest        */
/*    move_cost / M_pot(n, t)" (nodes_heap, ties by id); nodes with a > O   */
/*    sit in a second heap keyed by move_cost; "the top node is removed     */
/*    from both heaps and the one with the least move_cost is chosen" (the  */
/*    nodes_heap top on equal move_cost);                                   */
/*  - "moved to another pe if the target pe has sufficient memory to        */
/*    accommodate that node memory potential": the PE q' != q with          */
/*    M_cons(q', i) + a <= cap_eff[q'] and the least M_cons(q', i) (lowest   */
/*    id on ties); "Otherwise, the node is not considered again";          */
/*  - after a move the schedule (st = tl under the new placement, R8) and   */
/*    the tracker are recomputed and a moved node never      */
/*    moves again; stop when no PE overflows (resolved) or when the         */
/*    current overflow has no candidate left ("we run out of nodes").      */
/* moves: [n][3] = (node, from, to), to = -1 for a rejected candidate.       */
/* ------------------------------------------------------------------------ */
int or_mpot_at(const or_graph* g, const int32_t* part, const int64_t* mem, const uint8_t* kind,
               const int32_t* pos, int32_t q, int32_t i, int64_t* a) {
    int32_t V = g->V;
    for (int32_t n = 0; n < V; ++n) a[n] = 0;
    for (int32_t n = 0; n < V; ++n)   /* n's own memory while it executes (visit i) */
        if (part[n] == q && pos[n] == i && kind[n] != OR_KIND_REFERENCE) a[n] += mem[n];
    for (int32_t p = 0; p < V; ++p) {
        if (pos[p] > i || kind[p] == OR_KIND_REFERENCE) continue;         /* executed before t */
        if (kind[p] == OR_KIND_RESIDUAL && part[p] == q) continue;        /* persists: not freed */
        int32_t last = -1;
        for (int64_t e = g->succ_off[p]; e < g->succ_off[p + 1]; ++e) {
            int32_t s = g->succ[e];
            if (part[s] == q && (last < 0 || pos[s] > pos[last])) last = s;
        }
        if (last >= 0 && pos[last] >= i) a[last] += mem[p];               /* still occupied at t */
    }
    return OR_OK;
}

static int less_ratio(int64_t c1, int64_t a1, int32_t n1, int64_t c2, int64_t a2, int32_t n2) {
    __int128 x = (__int128)c1 * a2, y = (__int128)c2 * a1;   /* c1/a1 < c2/a2, a > 0 */
    return x < y || (x == y && n1 < n2);
}

int or_resolve_overflow(const or_graph* g, const int64_t* c, const int64_t* w, const int64_t* mem,
                        const uint8_t* kind, int32_t P, const int64_t* cap_eff, int32_t* part,
                        int32_t max_moves, int32_t* moves, int32_t* n_moves, int32_t* resolved) {
    int32_t V = g->V;
    if (P < 1 || P > OR_MAX_PE || max_moves < 0) return OR_EINVAL;
    size_t n = (size_t)(V ? V : 1);
    int64_t* tl = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t* bl = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t* mpot = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t* mcons = (int64_t*)malloc(sizeof(int64_t) * n * (size_t)P);
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * n);
    int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * n);
    int64_t* a = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t* cost = (int64_t*)malloc(sizeof(int64_t) * n);
    uint8_t* excl = (uint8_t*)calloc(n, 1);
    if (!tl || !bl || !mpot || !mcons || !order || !pos || !a || !cost || !excl) {
        free(tl); free(bl); free(mpot); free(mcons); free(order); free(pos); free(a); free(cost); free(excl);
        return OR_ENOMEM;
    }
    int rc = OR_OK;
    int32_t nm = 0;
    *resolved = 0;
    for (;;) {
        int64_t peak[OR_MAX_PE], over[OR_MAX_PE];
        int32_t ppos[OR_MAX_PE], fo[OR_MAX_PE];
        rc = or_weighted_levels(g, c, w, part, tl, bl);                       /* st = tl (R8) */
        if (rc) break;
        rc = or_memory(g, part, P, mem, kind, tl, cap_eff, mpot, peak, ppos, fo, over, mcons, order);
        if (rc) break;
        int32_t q = -1;
        for (int32_t k = 0; k < P; ++k)
            if (fo[k] >= 0 && (q < 0 || fo[k] < fo[q])) q = k;
        if (q < 0) { *resolved = 1; break; }
        if (nm >= max_moves) break;
        const int32_t i = fo[q];
        const int64_t O = over[q];
        for (int32_t k = 0; k < V; ++k) pos[order[k]] = k;
        or_mpot_at(g, part, mem, kind, pos, q, i, a);
        for (int32_t v = 0; v < V; ++v) {                                     /* Eq. 5 */
            cost[v] = c[v];
            if (part[v] != q) continue;
            for (int64_t e = g->pred_off[v]; e < g->pred_off[v + 1]; ++e)
                if (part[g->pred[e]] == q) cost[v] += w[g->pred_eid[e]];
            for (int64_t e = g->succ_off[v]; e < g->succ_off[v + 1]; ++e)
                if (part[g->succ[e]] == q) cost[v] += w[g->succ_eid[e]];
        }
        int moved = 0;
        for (;;) {
            int32_t A = -1, B = -1;
            for (int32_t v = 0; v < V; ++v) {
                if (part[v] != q || kind[v] != OR_KIND_NORMAL || excl[v] || a[v] <= 0) continue;
                if (A < 0 || less_ratio(cost[v], a[v], v, cost[A], a[A], A)) A = v;
                if (a[v] > O && (B < 0 || cost[v] < cost[B] || (cost[v] == cost[B] && v < B))) B = v;
            }
            if (A < 0) break;                                  /* run out of nodes */
            const int32_t pick = (B >= 0 && cost[B] < cost[A]) ? B : A;
            int32_t tgt = -1;
            for (int32_t k = 0; k < P; ++k) {
                if (k == q) continue;
                const int64_t m = mcons[(int64_t)k * V + i];
                if (m + a[pick] <= cap_eff[k] && (tgt < 0 || m < mcons[(int64_t)tgt * V + i])) tgt = k;
            }
            excl[pick] = 1;                                    /* never considered again */
            if (nm >= max_moves) break;
            moves[3 * nm] = pick; moves[3 * nm + 1] = q; moves[3 * nm + 2] = tgt;
            ++nm;
            if (tgt >= 0) { part[pick] = tgt; moved = 1; break; }
        }
        if (!moved) break;
    }
    *n_moves = nm;
    free(tl); free(bl); free(mpot); free(mcons); free(order); free(pos); free(a); free(cost); free(excl);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Scheduler emulator (Memory Heuristic I, "Scheduler Emulator",            */
/* PAPER.md:444-449): "TensorFlow scheduler maintains a ready queue that is */
/* initially filled with nodes with no ancestors.  Each node in the graph   */
/* has an in-degree ...  The nodes are executed in FIFO order.  Once a node  */
/* is executed, the in-degrees of its children are decremented by one.  Any */
/* node having an in-degree of zero will be pushed to the queue."  With the  */
/* per-node running times (comp) and communication (comm, paid across PEs, */
/* R2) this yields st(n) and ft(n) under a partitioning (Table 2, PAPER.md: */
/* 198-217), in O(|V| + |E|) node / edge visits.             */
/*                                                                          */
/* Reading R17: each PE executes one node at a time; a node     */
/* enters the ready queue when its last input arrives,                      */
/*     ready(v) = max(0, max over preds p of ft(p) + comm'(p, v)),           */
/* and the queue is FIFO by entry time, equal entry times ordered by        */
/* (level, id) -- the level keeps a zero-duration producer ahead of its     */
/* consumer.  A PE that becomes free takes the earliest entry; so           */
/*     st(v) = max(ready(v), ft(previous node on pe(v))),  ft = st + comp.  */
/* The emulation pops the queue in (ready, level, id) order: every node is  */
/* pushed when its in-degree reaches zero, its ready time is then final,    */
/* and a node's key exceeds each predecessor's key, so a pop never precedes */
/* a later-arriving entry of smaller key.                                   */
/* ------------------------------------------------------------------------ */
typedef struct { int64_t ready; int32_t level, id; } qent_t;
static int qless(const qent_t* a, const qent_t* b) {
    if (a->ready != b->ready) return a->ready < b->ready;
    if (a->level != b->level) return a->level < b->level;
    return a->id < b->id;
}
static void q_push(qent_t* h, int32_t* n, qent_t x) {   /* binary min-heap */
    int32_t i = (*n)++;
    while (i > 0) {
        int32_t p = (i - 1) / 2;
        if (!qless(&x, &h[p])) break;
        h[i] = h[p];
        i = p;
    }
    h[i] = x;
}
static qent_t q_pop(qent_t* h, int32_t* n) {
    qent_t top = h[0], x = h[--(*n)];
    int32_t i = 0;
    for (;;) {
        int32_t c = 2 * i + 1;
        if (c >= *n) break;
        if (c + 1 < *n && qless(&h[c + 1], &h[c])) ++c;
        if (!qless(&h[c], &x)) break;
        h[i] = h[c];
        i = c;
    }
    if (*n > 0) h[i] = x;
    return top;
}

int or_emulate(const or_graph* g, const int64_t* c, const int64_t* w, const int32_t* part, int32_t P,
               int64_t* st, int64_t* ft, int64_t* makespan, int32_t* max_queue) {
    int32_t V = g->V;
    if (P < 1 || P > OR_MAX_PE) return OR_EINVAL;
    for (int32_t v = 0; v < V; ++v)
        if (part[v] < 0 || part[v] >= P || c[v] < 0) return OR_EINVAL;
    int64_t* ready = (int64_t*)calloc((size_t)(V ? V : 1), sizeof(int64_t));
    int64_t* indeg = (int64_t*)malloc(sizeof(int64_t) * (size_t)(V ? V : 1));
    qent_t* heap = (qent_t*)malloc(sizeof(qent_t) * (size_t)(V ? V : 1));
    if (!ready || !indeg || !heap) { free(ready); free(indeg); free(heap); return OR_ENOMEM; }
    int64_t free_at[OR_MAX_PE];
    for (int32_t q = 0; q < P; ++q) free_at[q] = 0;
    int32_t n = 0, peakq = 0, done = 0;
    int64_t span = 0;
    /* the ready queue is initially filled with the nodes with no ancestors */
    for (int32_t v = 0; v < V; ++v) {
        indeg[v] = g->pred_off[v + 1] - g->pred_off[v];
        if (indeg[v] == 0) { qent_t e = {0, g->level[v], v}; q_push(heap, &n, e); }
    }
    while (n > 0) {
        if (n > peakq) peakq = n;
        qent_t e = q_pop(heap, &n);
        int32_t v = e.id, q = part[v];
        st[v] = e.ready > free_at[q] ? e.ready : free_at[q];
        ft[v] = st[v] + c[v];
        free_at[q] = ft[v];
        if (ft[v] > span) span = ft[v];
        ++done;
        /* once a node is executed, the in-degrees of its children drop by one */
        for (int64_t a = g->succ_off[v]; a < g->succ_off[v + 1]; ++a) {
            int32_t s = g->succ[a];
            int64_t arrive = ft[v] + (part[s] == q ? 0 : w[g->succ_eid[a]]);
            if (arrive > ready[s]) ready[s] = arrive;
            if (--indeg[s] == 0) { qent_t x = {ready[s], g->level[s], s}; q_push(heap, &n, x); }
        }
    }
    free(ready); free(indeg); free(heap);
    if (done != V) return OR_ECYCLE;
    *makespan = span;
    if (max_queue) *max_queue = peakq;
    return OR_OK;
}

typedef struct {
    const or_graph* g; const int64_t* c; const int64_t* w; const int64_t* mem; const uint8_t* kind;
    int32_t P; const int64_t* cap_eff; int32_t batch; const uint8_t* parts; or_eval_result* out;
    int32_t next; pthread_mutex_t mu; int rc;
    int32_t schedule;   /* 0: level schedule st = tl (R8); 1: emulated FIFO schedule (R17) */
} batch_ctx;

static int eval_one(batch_ctx* bc, int32_t b, int32_t* part, int64_t* tl, int64_t* bl, int64_t* mpot, int32_t* cp,
                    int64_t* est, int64_t* eft) {
    const or_graph* g = bc->g;
    const uint8_t* pb = bc->parts + (int64_t)b * g->V;
    for (int32_t v = 0; v < g->V; ++v) { if (pb[v] >= bc->P) return OR_EINVAL; part[v] = pb[v]; }
    or_eval_result* r = &bc->out[b];
    memset(r, 0, sizeof(*r));
    int rc = or_weighted_levels(g, bc->c, bc->w, part, tl, bl);
    if (rc) return rc;
    rc = or_critical_path(g, bc->c, bc->w, part, tl, bl, cp, &r->cp_len, &r->L, &r->cp_hash);
    if (rc) return rc;
    r->cp_start = r->cp_len ? cp[0] : -1;
    r->cp_end = r->cp_len ? cp[r->cp_len - 1] : -1;
    int64_t cut = 0;
    for (int32_t u = 0; u < g->V; ++u)
        for (int64_t a = g->succ_off[u]; a < g->succ_off[u + 1]; ++a)
            if (part[u] != part[g->succ[a]]) cut += bc->w[g->succ_eid[a]];
    r->cut_comm = cut;
    int64_t peak[OR_MAX_PE], over[OR_MAX_PE];
    int32_t ppos[OR_MAX_PE], fo[OR_MAX_PE];
    /* the tracker's schedule: the level schedule st = tl (R8), or the emulated
     * FIFO schedule (R17) whose makespan is reported; the level schedule's
     * makespan is max ft = max(tl + comp) = L */
    const int64_t* st = tl;
    r->makespan = r->L;
    if (bc->schedule == 1) {
        rc = or_emulate(g, bc->c, bc->w, part, bc->P, est, eft, &r->makespan, NULL);
        if (rc) return rc;
        st = est;
    }
    rc = or_memory(g, part, bc->P, bc->mem, bc->kind, st, bc->cap_eff, mpot, peak, ppos, fo, over, NULL, NULL);
    if (rc) return rc;
    for (int32_t q = 0; q < OR_MAX_PE; ++q) {
        int in = q < bc->P;
        r->peak[q] = in ? peak[q] : 0;
        r->peak_pos[q] = in ? ppos[q] : -1;
        r->first_over_pos[q] = in ? fo[q] : -1;
        r->over_bytes[q] = in ? over[q] : 0;
        if (in && fo[q] >= 0) r->overflow_mask |= 1 << q;
    }
    return OR_OK;
}

static void* batch_worker(void* arg) {
    batch_ctx* bc = (batch_ctx*)arg;
    int32_t V = bc->g->V;
    size_t n = (size_t)(V ? V : 1);
    int32_t* part = (int32_t*)malloc(sizeof(int32_t) * n);
    int64_t* tl = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t* bl = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t* mpot = (int64_t*)malloc(sizeof(int64_t) * n);
    int32_t* cp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(bc->g->n_levels + 1));
    int64_t* est = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t* eft = (int64_t*)malloc(sizeof(int64_t) * n);
    for (;;) {
        pthread_mutex_lock(&bc->mu);
        int32_t b = bc->next++;
        pthread_mutex_unlock(&bc->mu);
        if (b >= bc->batch) break;
        int rc = eval_one(bc, b, part, tl, bl, mpot, cp, est, eft);
        if (rc) { pthread_mutex_lock(&bc->mu); bc->rc = rc; pthread_mutex_unlock(&bc->mu); }
    }
    free(part); free(tl); free(bl); free(mpot); free(cp); free(est); free(eft);
    return NULL;
}

int or_eval_batch(const or_graph* g, const int64_t* c, const int64_t* w, const int64_t* mem,
                  const uint8_t* kind, int32_t P, const int64_t* cap_eff, int32_t batch,
                  const uint8_t* parts, or_eval_result* out, int32_t n_threads, int32_t schedule) {
    if (P < 1 || P > OR_MAX_PE || batch < 0 || schedule < 0 || schedule > 1) return OR_EINVAL;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    batch_ctx bc = {g, c, w, mem, kind, P, cap_eff, batch, parts, out, 0, PTHREAD_MUTEX_INITIALIZER, OR_OK, schedule};
    pthread_t th[256];
    for (int32_t t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, batch_worker, &bc);
    for (int32_t t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
    return bc.rc;
}
