/*
 * oracle_ft.h -- CPU ORACLE for the Frontier-Tracking (FT) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA product path
 * (paper_2004_10856_b200/, include/ft.h).
 *
 * Paper: arXiv 2004.10856 (TensorOpt).  P:n = /root/reference/PAPER.md line n.
 *   Def. 1 cost frontier
 *   Alg. 1 Reduce
 *   Product / Union
 *   Eq. 4 node elimination
 *   Eq. 5 edge elimination
 *   Eq. 7 heuristic elim (K=1)
 *   marking of the linear graph
 *   Alg. 3 LDP
 *   unroll
 * Readings of ambiguous passages: DESIGN.md section "Readings" (R1..R16).
 *
 * Semantics mirror include/ft.h (same call sequence, same results); names
 * carry the oft_ prefix so both libraries can live in one process.
 */
#ifndef ORACLE_FT_H
#define ORACLE_FT_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { OFT_OK = 0, OFT_EINVAL = -1, OFT_ESTATE = -2, OFT_EPRECOND = -3, OFT_ENOMEM = -4,
       OFT_EOVERFLOW = -6, OFT_ESIZE = -7, OFT_EINTERNAL = -8 };
enum { OFT_NODE = 1, OFT_EDGE = 2, OFT_AUTO = 3, OFT_AUTO_HEUR = 4 };
/* step kinds reported by oft_step_info */
enum { OFT_STEP_NODE = 1, OFT_STEP_EDGE = 2, OFT_STEP_FOLD = 3, OFT_STEP_LDP = 4,
       OFT_STEP_FINAL = 5, OFT_STEP_PAIR = 6, OFT_STEP_BRANCH = 7,
       OFT_STEP_COMPOSE = 8 /* Eq. 6 composite configurations (R21) */,
       OFT_STEP_REMAP = 9 /* an edge re-indexed onto a composite op (R21) */ };

typedef struct oft_graph oft_graph;

/* Graph: n_ops operators with K_i = n_cfgs[i] >= 1 configurations; n_edges
 * directed edges src[e] -> dst[e] (multi-edges allowed, src != dst, acyclic).
 * threads: worker threads over output segments (0 or 1 = single thread). */
int oft_graph_create(int32_t n_ops, const int32_t* n_cfgs, int32_t n_edges,
                     const int32_t* src, const int32_t* dst, int32_t threads,
                     oft_graph** out);
void oft_graph_destroy(oft_graph* g);
/* Eq. 1 operator costs m[K_op], t[K_op] (copied). */
int oft_set_op_costs(oft_graph* g, int32_t op, const int64_t* m, const int64_t* t);
/* Eq. 2 edge costs, row-major [s_src][s_dst]; m may be NULL (= 0). */
int oft_set_edge_costs(oft_graph* g, int32_t edge, const int64_t* m, const int64_t* t);
/* OFT_NODE (id = op), OFT_EDGE (id = edge), OFT_AUTO (id ignored),
 * OFT_AUTO_HEUR: OFT_AUTO, then while the graph is not linear and no exact
 * elimination applies, one heuristic elimination (Eq. 7; lossy)
 * of the unmarked source op with the most out-edges, its configuration
 * fixed to the one of least memory (ties: time, index). */
int oft_eliminate(oft_graph* g, int32_t kind, int32_t id, int32_t* new_edge);
/* LDP + final reduce (cached).  Two-call size pattern: OFT_ESIZE with *n_out. */
int oft_frontier(oft_graph* g, int64_t cap, int64_t* m_out, int64_t* t_out, int64_t* n_out);
/* FT-Elimination instead of LDP: node-eliminate the
 * chain's second op until two ops remain, then reduce over every
 * configuration pair (s_1, s_n) (cached; the graph then has a frontier and
 * oft_frontier returns OFT_ESTATE, and vice versa). */
int oft_frontier_elim(oft_graph* g, int64_t cap, int64_t* m_out, int64_t* t_out, int64_t* n_out);
/* Mini-time query (SS4.1): index of the smallest-time final-frontier
 * tuple with m <= memory_limit (the last such tuple: m ascending, t strictly
 * descending), or -1 if none (infeasible).  Requires a computed frontier. */
int oft_query_mini_time(oft_graph* g, int64_t memory_limit, int64_t* idx_out);
/* Heuristic-elimination configuration rule (R17): policy 0 = least
 * memory (default), 1 = weighted combination alpha*m/M + (1-alpha)*t/T with
 * alpha = num/den (reading R22). */
int oft_set_heuristic(oft_graph* g, int32_t policy, int64_t alpha_num, int64_t alpha_den);
/* Unrolled strategy (config per original op) of final-frontier tuple idx. */
int oft_strategy(oft_graph* g, int64_t tuple_idx, int32_t* cfg_out);
int64_t oft_num_steps(const oft_graph* g);
/* info[0]=kind [1]=nseg [2]=nblk [3]=product tuples [4]=survivors [5]=microseconds */
int oft_step_info(const oft_graph* g, int64_t step, int64_t* info);
/* Output frontier set of a step: seg_off[nseg+1], m/t/bp[survivors]. */
int oft_step_output(const oft_graph* g, int64_t step, int64_t cap, int64_t* seg_off,
                    int64_t* m, int64_t* t, uint64_t* bp);
const char* oft_last_error(const oft_graph* g);

/* Alg. 1 on an explicit tuple list (m, t, id); output sorted by (m, t, id). */
int oft_reduce(int64_t n, const int64_t* m, const int64_t* t, const uint64_t* id,
               int64_t* m_out, int64_t* t_out, uint64_t* id_out, int64_t* n_out);
/* One output segment: reduce( U_k X_k (x) Y_k (x) Z_k ) with ids = position in
 * written product order (R6).  Factor k of X is x_m/x_t[x_off[k]..x_off[k+1]). */
int oft_segment_reduce(int32_t nblk,
                       const int64_t* x_off, const int64_t* x_m, const int64_t* x_t,
                       const int64_t* y_off, const int64_t* y_m, const int64_t* y_t,
                       const int64_t* z_off, const int64_t* z_m, const int64_t* z_t,
                       int64_t cap, int64_t* m_out, int64_t* t_out, uint64_t* id_out,
                       int64_t* n_out);

#ifdef __cplusplus
}
#endif
#endif
