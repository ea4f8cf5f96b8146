/*
 * ft.h -- C-ABI of libft: the B200 (sm_100a) Frontier-Tracking hot path.
 *
 * Paper: "TensorOpt: Exploring the Tradeoffs in Distributed DNN Training with
 * Auto-Parallelism", arXiv 2004.10856.  P:n = line n of the paper text
 * (/root/reference/PAPER.md at build time; not read at run time).
 *
 * The library computes the exact cost frontier (Def. 1) of a
 * computation graph's parallelization strategies by Frontier Tracking:
 * node elimination (Eq. 4), edge elimination (Eq. 5),
 * the exact K=1 case of heuristic elimination (Eq. 7), LDP
 * (Alg. 3) and unroll.  Every elimination / LDP step
 * evaluates, for each configuration pair of the surviving operators, the
 * Product, Union and Reduce (Alg. 1) on
 * the GPU; see DESIGN.md for kernels and readings R1..R16.
 *
 * Conventions (all entry points):
 *  - Every call returns an int status (FT_OK = 0 or a negative FT_E* code);
 *    no C++ exception or abort crosses the ABI.  ft_last_error() returns a
 *    human-readable message for the last failing call on a handle.
 *  - Costs are int64: memory in bytes, time in integer ns (fixed point, R10).
 *    Each input cost must lie in [0, 2^40) and n_ops + n_edges < 2^20, so
 *    every sum of costs is < 2^60 (FT_EOVERFLOW otherwise; FT_EINVAL for a
 *    negative cost).
 *  - Ownership: input arrays are copied before the call returns; output
 *    buffers are caller-allocated HOST memory; sizes use the two-call pattern
 *    (a too-small buffer returns FT_ESIZE with *n_out = required count).
 *    The handle owns all device memory, allocated through ft_options.alloc /
 *    .free when given (else cudaMallocAsync on the handle's stream).
 *  - Strong guarantee: on any error except FT_ECUDA / FT_EINTERNAL the graph
 *    is unchanged.  FT_ECUDA / FT_EINTERNAL poison the handle (every later
 *    call returns the same code).
 *  - A handle is single-threaded; distinct handles are independent.
 *  - Multi-GPU (world > 1): every rank issues the identical call sequence and
 *    every rank returns identical results; each step's configuration pairs
 *    are sharded over ranks and the surviving frontiers are all-gathered over
 *    NCCL (P:663 independence).
 *  - There is no CPU fallback: without a usable CUDA device every call that
 *    needs one returns FT_ECUDA.
 */
#ifndef FT_H
#define FT_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum {
  FT_OK = 0,
  FT_EINVAL = -1,     /* bad argument: ids, src==dst, K<1, negative cost, cycle */
  FT_ESTATE = -2,     /* call order: costs missing at first eliminate, costs after eliminate, ... */
  FT_EPRECOND = -3,   /* elimination precondition violated; graph not linear at ft_frontier */
  FT_ENOMEM = -4,     /* device or host allocation failed */
  FT_ECUDA = -5,      /* CUDA / NCCL runtime error (poisons the handle) */
  FT_EOVERFLOW = -6,  /* cost or size bound violated (R10) */
  FT_ESIZE = -7,      /* output buffer too small; *n_out holds the required count */
  FT_EINTERNAL = -8   /* broken provenance or internal invariant (poisons the handle) */
};

enum { FT_NODE = 1, FT_EDGE = 2, FT_AUTO = 3, FT_AUTO_HEUR = 4 };

/* Step kinds in ft_step_stats records. */
enum { FT_STEP_NODE = 1, FT_STEP_EDGE = 2, FT_STEP_FOLD = 3, FT_STEP_LDP = 4, FT_STEP_FINAL = 5,
       FT_STEP_PAIR = 6 /* FT-Elimination's reduce over configuration pairs */,
       FT_STEP_BRANCH = 7 /* branch elimination, Eq. 6 (merge a one-edge op into its neighbour) */,
       FT_STEP_COMPOSE = 8 /* branch elimination with composite configurations, Eq. 6 (R21) */,
       FT_STEP_REMAP = 9 /* an edge re-indexed onto a composite operator (R21) */ };

typedef struct ft_graph ft_graph; /* opaque, library-owned */

/* Device-memory hooks (ft_options.alloc / .free, e.g. a
 * framework's caching allocator).  alloc returns `bytes` of device memory on
 * the graph's device, usable by work on `stream` (NULL = out of memory ->
 * FT_ENOMEM); free is stream-ordered: work enqueued on `stream` before the
 * call may still read p.  The library calls them with the device current,
 * from the thread that called into it; `ctx` is passed through. */
typedef void* (*ft_alloc_fn)(size_t bytes, void* stream, void* ctx);
typedef void (*ft_free_fn)(void* p, void* stream, void* ctx);

/* All fields optional; a zeroed struct (or NULL) selects defaults. */
typedef struct {
  int32_t device;      /* CUDA device ordinal (default 0) */
  void* stream;        /* cudaStream_t to run on; NULL = library-created stream */
  int32_t rank, world; /* world > 1: SPMD over `world` ranks (one process per GPU) */
  void* nccl_comm;     /* ncclComm_t of the world (required when world > 1) */
  int32_t keep_all;    /* != 0: keep every step's m/t on device (ft_step_output) */
  int32_t profile;     /* != 0: CUDA events between kernel groups (ft_step_stats *_ms) */
  int32_t loopback;    /* != 0 with world > 1 and nccl_comm == NULL: every virtual rank's
                          shard runs in this process on one GPU (partition-invariance tests) */
  ft_alloc_fn alloc;   /* both NULL: cudaMallocAsync / cudaFreeAsync (stream-ordered pool) and a */
  ft_free_fn free;     /*   process-wide per-device scratch; both set: EVERY device allocation of */
  void* alloc_ctx;     /*   the handle, and the pipeline scratch shared by all live handles with the
                            same (alloc, free, ctx) on the device, goes through them; everything is
                            handed back by the time the last such handle is destroyed.  Exactly one
                            of the two set: FT_EINVAL.  A NULL from alloc: FT_ENOMEM, and the handle
                            is poisoned if the failure interrupted a search. */
  int32_t reserved[4];
} ft_options;

/* Per-step statistics (ft_get_stats). */
typedef struct {
  int32_t kind;          /* FT_STEP_* */
  int32_t levels;        /* sample levels used by the reduce */
  int32_t wave;          /* batch of independent steps it ran in */
  int32_t pad;
  int64_t nseg;          /* output segments (configuration pairs / configs) */
  int64_t nblk;          /* blocks (union terms) per segment */
  int64_t tuples;        /* product tuples sum |X||Y||Z| over ALL ranks (the M1 numerator) */
  int64_t survivors;     /* frontier tuples written */
  int64_t candidates;    /* tuples that passed the dominance pre-filter (all levels);
                            wave-level numbers (candidates, launches, *_ms) are
                            booked on the first step of each wave */
  int64_t retries;       /* capacity retries */
  int64_t launches;      /* kernels launched by this step on this rank */
  int64_t max_seg;       /* largest output segment (frontier) of the step */
  int64_t filter_tuples; /* wave: sampled tuples streamed by the pre-filter kernel (this rank) */
  int64_t direct_tuples; /* wave: sampled tuples sorted by the direct kernels (this rank) */
  float kernel_ms;       /* CUDA-event time of the step's kernels on this rank */
  float comm_ms;         /* all-gather time (world > 1) */
  float plan_ms, direct_ms, filter_ms, bucket_ms, compact_ms; /* opt.profile only: k_plan; direct
                            kernels (k_direct*, k_node_*); k_filter alone; bucket sorts + carry +
                            scatter; scans and compaction */
  float host_ms;         /* opt.profile only: host readback + scratch sizing inside the step */
  int64_t path[4];       /* wave: kernel-path counters (this rank) -- shared-order node rows
                            reduced by the packed kernel, ... of them with equal m values,
                            rows sent to the one-CTA-per-row kernel, direct segments sorted
                            by the register-blocked CTA kernel */
} ft_step_stats;

/* Create a graph: n_ops operators, K_i = n_cfgs[i] (1 <= K_i <= 4096)
 * configurations each; n_edges directed edges src[e] -> dst[e]
 * (multi-edges allowed, src != dst, acyclic).  opt may be NULL.
 * Errors: FT_EINVAL, FT_EOVERFLOW, FT_ENOMEM, FT_ECUDA. */
int ft_graph_create(int32_t n_ops, const int32_t* n_cfgs, int32_t n_edges,
                    const int32_t* src, const int32_t* dst, const ft_options* opt,
                    ft_graph** out);
void ft_graph_destroy(ft_graph* g);

/* Validates that every cost is set and uploads all cost tables to the device
 * (done implicitly by the first ft_eliminate / ft_frontier).  Lets a caller
 * time the search with inputs already resident in HBM. */
int ft_prepare(ft_graph* g);

/* All costs at once (fast path; HOST arrays, pinned memory recommended):
 *  op_m/op_t: concatenation over operators 0..n_ops-1 of K_i entries each;
 *  edge_t (and edge_m, NULL = 0 per Eq. 2): concatenation over edges
 *  0..n_edges-1 of K_src*K_dst entries each, row-major [s_src][s_dst].
 * Copied to the device (asynchronously, then validated on the device) before
 * the call returns.  Exclusive with the per-operator / per-edge setters.
 * Errors: FT_EINVAL (negative), FT_EOVERFLOW (>= 2^40), FT_ESTATE, FT_ECUDA. */
int ft_set_costs_all(ft_graph* g, const int64_t* op_m, const int64_t* op_t,
                     const int64_t* edge_m, const int64_t* edge_t);

/* Operator costs, Eq. 1: m[K_op] bytes, t[K_op] ns (host arrays,
 * copied to the device).  Must precede the first ft_eliminate/ft_frontier. */
int ft_set_op_costs(ft_graph* g, int32_t op, const int64_t* m, const int64_t* t);
/* Edge costs, Eq. 2: t[K_src*K_dst] row-major [s_src][s_dst];
 * m may be NULL (= 0 per Eq. 2). */
int ft_set_edge_costs(ft_graph* g, int32_t edge, const int64_t* m, const int64_t* t);

/* One elimination (Alg. 2 lines 4-11):
 *  FT_NODE: id = op with exactly one in-edge and one out-edge, not marked
 *            -> new edge e_hj (Eq. 4).
 *  FT_EDGE: id = edge; merged with the lowest-id other edge of the same
 *           (src, dst) (Eq. 5, binary; X = lower id) -> new edge.
 *  FT_AUTO: id ignored; the deterministic policy of DESIGN.md R9 until no
 *           exact elimination applies: parallel edges (Eq. 5), node
 *           elimination (Eq. 4), the K=1 source fold (Eq. 7, exact for
 *           K=1), branch elimination (Eq. 6: an unmarked op whose only
 *           edge joins it to o_h is merged into o_h, reducing over its
 *           configurations -- reading R14), then branch elimination with
 *           composite configurations (Eq. 6, R21: an unmarked input o_i of
 *           an op o_h with >= 2 inputs, K_h*K_i <= 4096, becomes part of a
 *           new operator o_v = (o_h, o_i) with K_h*K_i configurations; new
 *           operator ids are n_ops, n_ops+1, ... in creation order; the
 *           edges of o_h and o_i move to o_v).
 *  FT_AUTO_HEUR: FT_AUTO without the composite step, then, while the graph
 *           is not linear: one heuristic elimination (Eq. 7, P:618-622;
 *           lossy) -- the unmarked source op with the most out-edges is
 *           fixed to its least-memory configuration (ties: time, index) and
 *           folded into its consumers -- or, if there is no such source, one
 *           composite branch elimination; repeat.
 * New edge ids are n_edges, n_edges+1, ... in creation order (*new_edge,
 * nullable).  Errors: FT_EINVAL, FT_ESTATE, FT_EPRECOND, FT_ENOMEM, FT_ECUDA. */
int ft_eliminate(ft_graph* g, int32_t kind, int32_t id, int32_t* new_edge);

/* LDP (Alg. 3) + final reduce on the remaining chain, computed once and
 * cached.  Writes the frontier F_o: m ascending, t strictly descending,
 * (m, t) unique; cap = capacity of m_out/t_out (host).  FT_EPRECOND if the
 * remaining graph is not a chain. */
int ft_frontier(ft_graph* g, int64_t cap, int64_t* m_out, int64_t* t_out, int64_t* n_out);

/* FT-Elimination (Theorem 2) instead of LDP: on the
 * remaining chain o_1 -> ... -> o_n, node-eliminate (Eq. 4) the second op
 * until two ops remain, then reduce over every configuration pair
 * U_{s_1,s_n} F(e_1n,s_1,s_n) (x) F(o_1,s_1) (x) F(o_n,s_n) (FT_STEP_PAIR:
 * one segment, K_1*K_n blocks).  Same output contract as ft_frontier (the
 * (m, t) frontier is identical: both are exact); computed once and cached.
 * A graph has one final frontier: after ft_frontier_elim, ft_frontier
 * returns FT_ESTATE, and vice versa.  FT_EPRECOND if not a chain. */
int ft_frontier_elim(ft_graph* g, int64_t cap, int64_t* m_out, int64_t* t_out, int64_t* n_out);

/* Configuration rule of heuristic elimination (FT_AUTO_HEUR; Eq. 7,
 * "minimizing the memory consumption of o_i or a weighted
 * combination of different objectives"):
 *  FT_HEUR_MIN_MEMORY (default): the config whose least-memory tuple of
 *    F(o_i, k) has the least m, ties by t, then k (reading R17);
 *  FT_HEUR_WEIGHTED: every tuple x of F(o_i, k) scores
 *    alpha*m_x/M + (1-alpha)*t_x/T with alpha = alpha_num/alpha_den in [0, 1]
 *    and M, T the largest m, t over F(o_i, .) (at least 1), evaluated in IEEE
 *    double (reading R22); least score wins, ties by (m, t), then k.
 * Errors: FT_EINVAL (policy, alpha outside [0, 1] or alpha_den < 1). */
enum { FT_HEUR_MIN_MEMORY = 0, FT_HEUR_WEIGHTED = 1 };
int ft_set_heuristic(ft_graph* g, int32_t policy, int64_t alpha_num, int64_t alpha_den);

/* Mini-time query (SS4.1: "minimizes the per-iteration time while
 * satisfying the memory constraint"): *idx_out = index of the smallest-time
 * final-frontier tuple with m <= memory_limit -- binary search on the
 * staircase (m ascending, t strictly descending: the last feasible tuple) --
 * or -1 when no strategy fits (infeasible is a value, not an error).
 * Requires ft_frontier / ft_frontier_elim (else FT_ESTATE). */
int ft_query_mini_time(ft_graph* g, int64_t memory_limit, int64_t* idx_out);

/* Unroll: configuration index of every ORIGINAL operator for final
 * frontier tuple tuple_idx; cfg_out[n_ops] host.  Requires ft_frontier. */
int ft_strategy(ft_graph* g, int64_t tuple_idx, int32_t* cfg_out);

/* Per-step statistics: buf = ft_step_stats[cap]; two-call size pattern. */
int ft_get_stats(const ft_graph* g, ft_step_stats* buf, int64_t cap, int64_t* n_out);

/* Output frontier set of step `step` (requires opt.keep_all for m/t of
 * consumed sets): seg_off[nseg+1] (host), m/t/bp[survivors] (host, any may be
 * NULL).  bp = provenance id (R6).  cap = capacity of m/t/bp. */
int ft_step_output(ft_graph* g, int64_t step, int64_t cap, int64_t* seg_off, int64_t* m,
                   int64_t* t, uint64_t* bp, int64_t* n_out);

/* Factor provenance of step `step` (debug / parity at full size): for X, Y, Z
 * (i = 0, 1, 2) src[2*i] = kind (0 unit {(0,0)}, 1 original op, 2 original
 * edge, 3 output of an earlier step) and src[2*i+1] = op / edge / step index;
 * params = {kind, KA, KB, KC, nseg, nblk} (block mapping of DESIGN.md "steps"). */
int ft_step_inputs(const ft_graph* g, int64_t step, int64_t* src6, int64_t* params6);

/* Host-side shard plan (no device needed): split `n` units with weights w[n]
 * (int64, >= 0) into `world` contiguous ranges of near-equal weight;
 * bounds[world+1] receives the cut points (bounds[0]=0, bounds[world]=n). */
int ft_shard_plan(int64_t n, const int64_t* w, int32_t world, int64_t* bounds);

/* NCCL bootstrap helpers (so callers need no NCCL headers): rank 0 creates
 * a 128-byte unique id, the caller distributes it (e.g. torch.distributed
 * broadcast), every rank creates its communicator on `device`. */
int ft_nccl_unique_id(uint8_t id_out[128]);
int ft_nccl_comm_init(int32_t world, int32_t rank, const uint8_t id[128], int32_t device,
                      void** comm_out);
int ft_nccl_comm_destroy(void* comm);

const char* ft_last_error(const ft_graph* g);
/* Library version string, e.g. "ft-b200 0.1 sm_100a". */
const char* ft_version(void);

/* ---------------------------------------------------------------------------
 * Edge-cost generation: the step before the FT path.
 * Produces t_x(e_ij, s_i^k, s_j^p) of Eq. 2 (m(e,...) = 0) from
 * the profile-interpolated communication time (reading R18) and
 * tensor re-scheduling as a shortest path over tensor splits (R19).
 * Standalone: no graph handle; all arrays are HOST memory, copied in/out by
 * the call; the computation runs on the current CUDA device (FT_ECUDA
 * without one).  Thread-safe: the per-device buffer pool and pinned staging
 * (library-owned, kept for the process lifetime) are guarded by a mutex.
 * ------------------------------------------------------------------------- */
#define FT_CG_MAX_MESH 6   /* mesh of up to 2^6 = 64 devices */
#define FT_CG_MAX_P 46     /* profiled sizes 2^0 .. 2^P bytes, P <= 46 */
#define FT_CG_MAX_DIMS 4   /* tensor rank */
#define FT_CG_MAX_STATES 160 /* split states per tensor (shared-memory APSP) */

/* Bandwidth profile: for a collective whose device group has
 * 2^c members (c = 1..mesh_log2; the "device partitioning scheme"),
 * bw[c][i] = measured bandwidth in bytes/s (> 0) at data size 2^i, i = 0..P,
 * and latency_ns[c] >= 0.  Row c = 0 is unused (no partners, time 0). */
typedef struct ft_comm_profile {
  int32_t mesh_log2;                                  /* L: 2^L devices, 1..FT_CG_MAX_MESH */
  int32_t P;                                          /* largest profiled size 2^P, 1..FT_CG_MAX_P */
  int64_t latency_ns[FT_CG_MAX_MESH + 1];
  int64_t bw[FT_CG_MAX_MESH + 1][FT_CG_MAX_P + 1];
} ft_comm_profile;

/* comm_time (R18), n queries: t_out[q] = time in integer ns to
 * move bytes[q] per device in a collective over a group of 2^group_log2[q]
 * devices.  0 if bytes == 0 or group_log2 == 0; else with 2^i <= b < 2^(i+1),
 * bw = bw[c][i] + (bw[c][i+1]-bw[c][i])*(b-2^i)/2^i (C integer division;
 * bw[c][P] when i == P) and t = latency_ns[c] + ceil(b*1e9 / bw).
 * Errors: FT_EINVAL (bad profile, group_log2 outside 0..mesh_log2, negative
 * bytes), FT_EOVERFLOW (bytes > 2^P: outside the profile). */
int ft_comm_time(const ft_comm_profile* prof, int64_t n, const int64_t* bytes,
                 const int32_t* group_log2, int64_t* t_out);

/* Split states of a tensor (R19): a = (a_0..a_{D-1}), a_j >= 0,
 * sum a_j <= mesh_log2, 2^a_j divides dims[j]; dim j is split over 2^a_j
 * devices and the tensor is replicated over the remaining 2^(L - sum a).
 * Index = rank in lexicographic order of a.  states_out[cap * ndims]
 * (row-major, may be NULL when cap = 0); *n_out = number of states
 * (two-call pattern, FT_ESIZE if cap too small).  Host only, no device. */
int ft_split_states(int32_t ndims, const int64_t* dims, int32_t mesh_log2, int64_t cap,
                    int32_t* states_out, int64_t* n_out);

/* Re-scheduling edge costs (R19): for n_tensors tensors (tensor τ:
 * ndims[τ] <= FT_CG_MAX_DIMS dims at dims[τ*FT_CG_MAX_DIMS + j] >= 1,
 * elem_bytes[τ] >= 1, product < 2^P) the library builds the state graph
 * whose edges are single collectives -- all-gather on one dim (group 2^c,
 * each device receives shard*(2^c-1) bytes), local slice on one dim (time 0)
 * and all-to-all moving a factor 2^c from dim i to dim j (group 2^c,
 * shard - shard/2^c bytes) -- weighted by ft_comm_time, and solves all-pairs
 * shortest paths on the GPU.  For n_q queries (tensor q_tensor[q], output
 * split q_from[q], required input split q_to[q], state indices of
 * ft_split_states):  t_out[q] = d(from, to) + d(to, from)  (forward
 * re-scheduling plus the backward re-scheduling of the gradient, Eq. 2
 * "both forward pass and backward pass").
 * Errors: FT_EINVAL (bad tensor / query index / profile), FT_EOVERFLOW
 * (tensor bytes > 2^P), FT_ESIZE (a tensor with > FT_CG_MAX_STATES states),
 * FT_ECUDA.  Query indices are validated on the device (FT_EINVAL after
 * the kernels; t_out is then unspecified).  Device buffers are pooled per
 * device across calls (grow-only; calls on one device serialise).  Queries
 * and results stream in chunks of 2^20 through library-owned pinned staging
 * (2 x 20 MB per device), copied by up to 8 host threads. */
int ft_reschedule_costs(const ft_comm_profile* prof, int32_t n_tensors, const int32_t* ndims,
                        const int64_t* dims, const int64_t* elem_bytes, int64_t n_q,
                        const int32_t* q_tensor, const int32_t* q_from, const int32_t* q_to,
                        int64_t* t_out);

/* Gradient-synchronisation operator costs (Eq. 1: m_p and t_s;
 * comm model P:668-671; reading R20): for n_q queries (parameter tensor
 * q_tensor[q] described as in ft_reschedule_costs, split state q_state[q]
 * of ft_split_states) each device stores shard = total / 2^(sum a) bytes,
 * m_out[q] = shard, and all-reduces the gradient over the r = 2^(L - sum a)
 * devices holding the same shard: t_out[q] = ft_comm_time of
 * 2*(shard - shard/r) bytes (ring all-reduce volume) over a group of r
 * (0 when r = 1).  Host arrays; runs on the current device.
 * Errors: FT_EINVAL (bad tensor / state / profile), FT_EOVERFLOW
 * (2 * tensor bytes > 2^P), FT_ESIZE (> FT_CG_MAX_STATES states), FT_ECUDA. */
int ft_sync_costs(const ft_comm_profile* prof, int32_t n_tensors, const int32_t* ndims,
                  const int64_t* dims, const int64_t* elem_bytes, int64_t n_q,
                  const int32_t* q_tensor, const int32_t* q_state, int64_t* m_out,
                  int64_t* t_out);

/* Same as ft_reschedule_costs, but q_tensor / q_from / q_to / t_out are
 * DEVICE pointers (caller-owned, on the current device) and the kernels run
 * on `stream` (cudaStream_t; NULL = legacy default stream).  The tensor
 * descriptions and the profile stay HOST arrays.  Returns after the stream
 * has completed the call's work. */
int ft_reschedule_costs_dev(const ft_comm_profile* prof, int32_t n_tensors, const int32_t* ndims,
                            const int64_t* dims, const int64_t* elem_bytes, int64_t n_q,
                            const int32_t* q_tensor, const int32_t* q_from, const int32_t* q_to,
                            int64_t* t_out, void* stream);

/* Measurement: ft_costgen_profile(1) makes every later ft_reschedule_costs_dev
 * record CUDA events around its two kernels (on the call's stream);
 * ft_costgen_last_times returns the last such call's APSP and gather kernel
 * times in ms on the current device (0 before any profiled call). */
int ft_costgen_profile(int32_t on);
int ft_costgen_last_times(float* apsp_ms, float* gather_ms);

#ifdef __cplusplus
}
#endif
#endif /* FT_H */
