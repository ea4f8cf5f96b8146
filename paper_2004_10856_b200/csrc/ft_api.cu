// ft_api.cu -- libft C-ABI (include/ft.h): graph store, FT_AUTO policy,
// step orchestration on the GPU, multi-GPU exchange, unroll.
//
// Paper: arXiv 2004.10856.  Alg. 2 drives node (Eq.4), edge
// (Eq.5) and exact K=1 heuristic (Eq.7) eliminations, then LDP (Alg.3) and
// unroll.  Every step's Product/Union/Reduce runs in ft_step.cu.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <queue>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include <nccl.h>

#include "../../include/ft.h"
#include "ft_step.h"

namespace {

enum SetKind { S_UNIT = 0, S_OP = 1, S_EDGE = 2, S_STEP = 3 };

struct FSet {
  int kind = S_UNIT;
  int step = -1;
  int a_op = -1, b_op = -1;  // segment -> config mapping for unroll
  int64_t nseg = 0;
  std::vector<int64_t> off;  // host copy of seg_off (lazy for single-rank step outputs)
  bool off_ok = true;
  int64_t* d_off = nullptr;
  int64_t* d_m = nullptr;
  int64_t* d_t = nullptr;
  uint64_t* d_bp = nullptr;
  int wave_buf = -1;         // S_STEP: arena of the wave that produced it
  bool mt_live = true;
  std::vector<uint64_t> h_bp;
  bool h_bp_ok = false;
};

struct StepRec {
  int kind = 0;
  int X = -1, Y = -1, Z = -1, out = -1;
  int64_t KA = 0, KB = 0, KC = 0, nseg = 0, nblk = 0;
  bool done = false;
  ft_step_stats st{};
};

// Ascending set of edge ids with the std::set<int> operations the policy
// uses, in a contiguous vector: operator degrees are small and new edge ids
// are the largest, so inserts append (tree nodes cost ~1 us per policy step
// on C5).
struct IdSet {
  std::vector<int> v;
  std::vector<int>::const_iterator begin() const { return v.begin(); }
  std::vector<int>::const_iterator end() const { return v.end(); }
  size_t size() const { return v.size(); }
  bool empty() const { return v.empty(); }
  void insert(int x) {
    if (v.empty() || v.back() < x) {
      v.push_back(x);
      return;
    }
    auto it = std::lower_bound(v.begin(), v.end(), x);
    if (*it != x) v.insert(it, x);
  }
  void erase(int x) {
    auto it = std::lower_bound(v.begin(), v.end(), x);
    if (it != v.end() && *it == x) v.erase(it);
  }
};

struct PairHash {
  size_t operator()(const std::pair<int, int>& p) const {
    return std::hash<uint64_t>()(((uint64_t)(uint32_t)p.first << 32) | (uint32_t)p.second);
  }
};

struct EdgeRec {
  int src, dst;
  bool alive;
  int set;
};

// One output arena per executed wave: the CSR arrays of all its steps,
// contiguous (step-major), so the multi-GPU all-gather is one broadcast per
// rank and array.  m/t are freed when every set in the wave is consumed.
struct WaveBuf {
  int64_t* m = nullptr;
  int64_t* t = nullptr;
  uint64_t* bp = nullptr;
  int64_t* off = nullptr;
  int live = 0;
};

}  // namespace

struct ft_graph {
  int dev = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int rank = 0, world = 1;
  bool loopback = false;  // world > 1 simulated on one GPU (tests)
  bool no_shared = false;  // FT_NO_SHARED=1 disables the shared-order node path (A/B tests)
  double replicate_tau = 2e7;  // waves below this estimated cost (tuples) are replicated
  std::vector<int> set_edge;   // original edge index of each original edge set (-1 otherwise)
  ncclComm_t comm = nullptr;
  bool keep_all = false;
  int n_ops = 0, n_orig_edges = 0;  // of the input graph; composite ops (R21) get ids n_ops, n_ops+1, ...
  std::vector<int> K;                // per op (original and composite)
  std::vector<std::pair<int, int>> comp;  // composite op (R21): (o_h, o_i), config w = s_h * K_i + s_i
  std::vector<char> op_alive;
  std::vector<int> op_set;
  std::vector<EdgeRec> edges;
  std::vector<IdSet> in_e, out_e;
  // FT_AUTO policy state (R9): positions in the original topological order and
  // ordered candidate sets maintained incrementally
  std::vector<int> pos0, order0;
  std::set<std::pair<int, int>> live_ops;   // (pos0, op)
  std::set<std::pair<int, int>> one_one;    // live ops with one in- and one out-edge
  std::set<std::pair<int, int>> leaf;       // live ops with exactly one edge (branch elimination)
  std::set<std::pair<int, int>> k1src;      // live K=1 sources with out-edges
  std::unordered_map<std::pair<int, int>, IdSet, PairHash> pair_edges;  // (src, dst) -> live edges
  std::set<std::pair<int, int>> multi;      // (pos0 src, pos0 dst) with >= 2 live edges
  std::vector<int> mark_stamp;
  int stamp = 0;
  bool mark_dirty = true;  // the marking must be recomputed (see note_change)
  std::vector<uint8_t> cand;  // refresh(): membership bits of one_one (1), k1src (2), leaf (4)
  struct CommEv {
    int step;
    cudaEvent_t a, b;
  };
  std::vector<CommEv> comm_ev;  // exchange events of sharded waves (read by ft_get_stats)
  std::vector<FSet> sets;
  std::vector<StepRec> steps;
  std::vector<int> pending;       // scheduled, not yet executed steps
  std::vector<WaveBuf> waves;
  std::vector<std::vector<int64_t>> op_m, op_t, e_m, e_t;
  std::vector<char> op_ok, e_ok;
  std::vector<char> e_mzero;  // original edge has m = 0 everywhere (Eq. 2)
  bool started = false, have_final = false;
  int final_mode = 0;  // 1 = LDP (Alg. 3), 2 = FT-Elimination
  int final_set = -1;
  int heur_policy = 0;                 // FT_HEUR_MIN_MEMORY (R17) | FT_HEUR_WEIGHTED (R22)
  int64_t heur_num = 1, heur_den = 2;  // alpha of the weighted rule
  std::vector<int64_t> final_m, final_t;
  int poisoned = 0;
  std::string err;
  ftk::StepRunner* runner = nullptr;  // process-wide per (device, allocator)
  ftk::DevAlloc alloc;                // ft_options.alloc / .free, else cudaMallocAsync
  bool profile = false;
  int64_t* d_costs = nullptr;  // all original costs + iota offsets + unit (alloc_costs)
  std::vector<int64_t> op_off, e_off;  // concatenation offsets of op / edge costs
  int64_t c_unit = 0, c_opm = 0, c_opt = 0, c_em = 0, c_et = 0;
  std::vector<int> op_set0;          // original op sets
  bool host_costs_pending = false;   // per-op/edge setters used: upload at start()
  bool bulk_done = false;            // ft_set_costs_all put every cost on the device
  std::vector<int64_t> h_pin_off;
  int64_t* h_pinned = nullptr;
  int64_t h_pinned_n = 0;
  // host-side wall time by phase (FT_HOST_PROF=1 prints at destroy)
  double hp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int64_t nwaves = 0;
};

namespace {
double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

namespace ftk {
static std::mutex g_reg_mu;
static std::map<std::pair<int, DevAlloc>, StepRunner*> g_runners;
StepRunner* device_runner(int device, const DevAlloc& a) {
  std::lock_guard<std::mutex> l(g_reg_mu);
  const auto key = std::make_pair(device, a);
  auto it = g_runners.find(key);
  if (it != g_runners.end()) {
    it->second->users++;
    return it->second;
  }
  StepRunner* r = new (std::nothrow) StepRunner();
  if (!r) return nullptr;
  r->alloc = a;
  if (cudaSetDevice(device) != cudaSuccess || r->configure() != cudaSuccess) {
    delete r;
    return nullptr;
  }
  r->users = 1;
  g_runners[key] = r;
  return r;
}
void release_runner(int device, const DevAlloc& a) {
  std::lock_guard<std::mutex> l(g_reg_mu);
  auto it = g_runners.find(std::make_pair(device, a));
  if (it == g_runners.end() || --it->second->users > 0 || !a.hooked()) return;
  it->second->release_device();  // scratch back through the hooks (host buffers stay)
}
}  // namespace ftk

namespace {

// Stream-ordered temporaries of one call, handed back on scope exit (also on
// an error return).
struct Temps {
  const ftk::DevAlloc& A;
  cudaStream_t st;
  std::vector<void*> p;
  ~Temps() {
    for (void* q : p) A.put(q, st);
  }
  cudaError_t get(int64_t** out, size_t bytes) {
    const cudaError_t e = A.get((void**)out, bytes, st);
    if (e == cudaSuccess) p.push_back(*out);
    return e;
  }
};

int setf(ft_graph* g, int code, const std::string& m) {
  if (g) g->err = m;
  return code;
}

int cuda_fail(ft_graph* g, cudaError_t e, const char* where) {
  // device memory exhausted (the allocator hook returned NULL, or the pool
  // is empty) -> FT_ENOMEM; either poisons the handle (a wave was cut short)
  const int code = e == cudaErrorMemoryAllocation ? FT_ENOMEM : FT_ECUDA;
  g->poisoned = code;
  g->err = std::string(where) + ": " + cudaGetErrorString(e);
  return code;
}

#define CU(call, where)                                  \
  do {                                                   \
    cudaError_t e__ = (call);                            \
    if (e__ != cudaSuccess) return cuda_fail(g, e__, where); \
  } while (0)

// ---- graph helpers (live adjacency kept incrementally) ----------------------

std::vector<int> topo_order(const ft_graph* g) {
  std::vector<int> deg(g->n_ops, 0);
  std::priority_queue<int, std::vector<int>, std::greater<int>> ready;  // min id first (R9)
  for (int v = 0; v < g->n_ops; ++v) {
    if (!g->op_alive[v]) continue;
    deg[v] = (int)g->in_e[v].size();
    if (deg[v] == 0) ready.push(v);
  }
  std::vector<int> order;
  order.reserve(g->n_ops);
  while (!ready.empty()) {
    int v = ready.top();
    ready.pop();
    order.push_back(v);
    for (int e : g->out_e[v]) {
      int d = g->edges[e].dst;
      if (--deg[d] == 0) ready.push(d);
    }
  }
  return order;
}

// Keeps op v's membership of the policy's candidate sets (one_one, k1src,
// leaf; keyed by topological position) current; touches the ordered sets only
// when a membership changes (cand[v] caches it: most edge updates leave it).
void refresh(ft_graph* g, int v) {
  const std::pair<int, int> key{g->pos0[v], v};
  if ((int)g->cand.size() <= v) g->cand.resize(v + 1, 0);
  const uint8_t have = g->cand[v];
  uint8_t want = 0;
  if (g->op_alive[v]) {
    const size_t ni = g->in_e[v].size(), no = g->out_e[v].size();
    if (ni == 1 && no == 1) want |= 1;
    if (g->K[v] == 1 && ni == 0 && no > 0) want |= 2;
    if (ni + no == 1) want |= 4;
  } else {
    g->live_ops.erase(key);
  }
  if (want == have) return;
  const uint8_t diff = want ^ have;
  if (diff & 1) {
    if (want & 1) g->one_one.insert(key);
    else g->one_one.erase(key);
  }
  if (diff & 2) {
    if (want & 2) g->k1src.insert(key);
    else g->k1src.erase(key);
  }
  if (diff & 4) {
    if (want & 4) g->leaf.insert(key);
    else g->leaf.erase(key);
  }
  g->cand[v] = want;
}

// The marking depends only on the first live operator and on the out-edges
// of marked operators, so it is recomputed only after a change that touches
// a marked operator or the first one (the policy runs O(n) eliminations;
// re-walking the backbone after each one cost ~1 us per step on C5).
inline void note_change(ft_graph* g, int v) {
  if (g->mark_dirty || g->mark_stamp.empty()) return;
  if (g->mark_stamp[v] == g->stamp || (!g->live_ops.empty() && g->live_ops.begin()->second == v))
    g->mark_dirty = true;
}

void kill_edge(ft_graph* g, int e) {
  const int u = g->edges[e].src, v = g->edges[e].dst;
  note_change(g, u);
  note_change(g, v);
  g->edges[e].alive = false;
  g->out_e[u].erase(e);
  g->in_e[v].erase(e);
  auto& pe = g->pair_edges[{u, v}];
  pe.erase(e);
  if (pe.size() < 2) g->multi.erase({g->pos0[u], g->pos0[v]});
  if (pe.empty()) g->pair_edges.erase({u, v});
  refresh(g, u);
  refresh(g, v);
}

int add_edge(ft_graph* g, int s, int d, int set) {
  if (!g->pos0.empty()) {
    note_change(g, s);
    note_change(g, d);
  }
  g->edges.push_back(EdgeRec{s, d, true, set});
  int e = (int)g->edges.size() - 1;
  g->out_e[s].insert(e);
  g->in_e[d].insert(e);
  auto& pe = g->pair_edges[{s, d}];
  pe.insert(e);
  if (pe.size() >= 2 && !g->pos0.empty()) g->multi.insert({g->pos0[s], g->pos0[d]});
  if (!g->pos0.empty()) {
    refresh(g, s);
    refresh(g, d);
  }
  return e;
}

void kill_op(ft_graph* g, int v) {
  note_change(g, v);
  g->op_alive[v] = 0;
  refresh(g, v);
}

// Marking with the R9 order: the first live op, then while the last
// marked op has exactly one downstream op, that op.  Marked ops get the
// current stamp.
void mark_backbone(ft_graph* g) {
  if (!g->mark_dirty) return;  // unchanged since the last walk
  g->mark_dirty = false;
  ++g->stamp;
  if (g->live_ops.empty()) return;
  int v = g->live_ops.begin()->second;
  g->mark_stamp[v] = g->stamp;
  while (true) {
    int only = -1;
    bool several = false;
    for (int e : g->out_e[v]) {
      int d = g->edges[e].dst;
      if (only < 0) only = d;
      else if (d != only) several = true;
    }
    if (only < 0 || several || g->mark_stamp[only] == g->stamp) break;
    g->mark_stamp[only] = g->stamp;
    v = only;
  }
}

// ---- device side ----------------------------------------------------------

// Device cost buffer layout: iota offsets | unit (m,t) | OPM | OPT | EM | ET,
// where OPM/OPT concatenate every operator's Eq.1 costs (K_i each) and EM/ET
// every edge's Eq.2 costs (K_src*K_dst each).  Singleton sets point into it.
int alloc_costs(ft_graph* g) {
  if (g->d_costs) return FT_OK;
  int64_t maxseg = 2, nop = 0, ned = 0;
  g->op_off.assign(g->n_ops + 1, 0);
  g->e_off.assign(g->n_orig_edges + 1, 0);
  for (int i = 0; i < g->n_ops; ++i) {
    maxseg = std::max<int64_t>(maxseg, g->K[i]);
    g->op_off[i + 1] = g->op_off[i] + g->K[i];
  }
  for (int e = 0; e < g->n_orig_edges; ++e) {
    const int64_t n = (int64_t)g->K[g->edges[e].src] * g->K[g->edges[e].dst];
    maxseg = std::max<int64_t>(maxseg, n);
    g->e_off[e + 1] = g->e_off[e] + n;
  }
  nop = g->op_off[g->n_ops];
  ned = g->e_off[g->n_orig_edges];
  g->c_unit = maxseg + 1;
  g->c_opm = g->c_unit + 2;
  g->c_opt = g->c_opm + nop;
  g->c_em = g->c_opt + nop;
  g->c_et = g->c_em + ned;
  const int64_t total = g->c_et + ned;
  CU(cudaSetDevice(g->dev), "cudaSetDevice");
  // stream-ordered pool (release threshold: unlimited) -- a plain
  // cudaMalloc/cudaFree per graph showed ~100 ms driver stalls
  CU(g->alloc.get((void**)&g->d_costs, sizeof(int64_t) * total, g->stream), "cudaMallocAsync(costs)");
  std::vector<int64_t> head(maxseg + 3);
  for (int64_t i = 0; i <= maxseg; ++i) head[i] = i;
  head[maxseg + 1] = 0;
  head[maxseg + 2] = 0;
  CU(cudaMemcpyAsync(g->d_costs, head.data(), sizeof(int64_t) * head.size(), cudaMemcpyHostToDevice,
                     g->stream), "upload costs");
  CU(cudaStreamSynchronize(g->stream), "upload costs");
  int64_t* base = g->d_costs;
  FSet& u = g->sets[0];
  u.d_off = base;
  u.d_m = base + g->c_unit;
  u.d_t = base + g->c_unit + 1;
  for (int i = 0; i < g->n_ops; ++i) {
    FSet& st = g->sets[g->op_set0[i]];
    st.d_off = base;
    st.d_m = base + g->c_opm + g->op_off[i];
    st.d_t = base + g->c_opt + g->op_off[i];
  }
  for (int e = 0; e < g->n_orig_edges; ++e) {
    FSet& st = g->sets[g->edges[e].set];
    st.d_off = base;
    st.d_m = base + g->c_em + g->e_off[e];
    st.d_t = base + g->c_et + g->e_off[e];
  }
  return FT_OK;
}

int start(ft_graph* g) {
  if (g->started) return FT_OK;
  for (int i = 0; i < g->n_ops; ++i)
    if (!g->op_ok[i]) return setf(g, FT_ESTATE, "operator costs missing (op " + std::to_string(i) + ")");
  for (int e = 0; e < g->n_orig_edges; ++e)
    if (!g->e_ok[e]) return setf(g, FT_ESTATE, "edge costs missing (edge " + std::to_string(e) + ")");
  int rc = alloc_costs(g);
  if (rc) return rc;
  if (!g->host_costs_pending) {  // costs already on the device (ft_set_costs_all)
    g->started = true;
    return FT_OK;
  }
  // per-operator / per-edge setters: concatenate on the host, 4 copies
  std::vector<int64_t> a(g->op_off[g->n_ops]), b(g->op_off[g->n_ops]);
  for (int i = 0; i < g->n_ops; ++i) {
    std::copy(g->op_m[i].begin(), g->op_m[i].end(), a.begin() + g->op_off[i]);
    std::copy(g->op_t[i].begin(), g->op_t[i].end(), b.begin() + g->op_off[i]);
  }
  std::vector<int64_t> c(g->e_off[g->n_orig_edges]), d(g->e_off[g->n_orig_edges]);
  for (int e = 0; e < g->n_orig_edges; ++e) {
    std::copy(g->e_m[e].begin(), g->e_m[e].end(), c.begin() + g->e_off[e]);
    std::copy(g->e_t[e].begin(), g->e_t[e].end(), d.begin() + g->e_off[e]);
  }
  int64_t* base = g->d_costs;
  CU(cudaMemcpyAsync(base + g->c_opm, a.data(), sizeof(int64_t) * a.size(), cudaMemcpyHostToDevice, g->stream), "upload");
  CU(cudaMemcpyAsync(base + g->c_opt, b.data(), sizeof(int64_t) * b.size(), cudaMemcpyHostToDevice, g->stream), "upload");
  CU(cudaMemcpyAsync(base + g->c_em, c.data(), sizeof(int64_t) * c.size(), cudaMemcpyHostToDevice, g->stream), "upload");
  CU(cudaMemcpyAsync(base + g->c_et, d.data(), sizeof(int64_t) * d.size(), cudaMemcpyHostToDevice, g->stream), "upload");
  CU(cudaStreamSynchronize(g->stream), "upload costs");
  g->host_costs_pending = false;
  g->started = true;
  return FT_OK;
}

ftk::FacSet fac(const FSet& s) { return ftk::FacSet{s.d_off, s.d_m, s.d_t}; }

// A consumed step output releases its wave arena's m/t once every set of that
// wave has been consumed (bp stays for unroll).
void consume(ft_graph* g, int set) {
  FSet& s = g->sets[set];
  if (s.kind != S_STEP || !s.mt_live) return;
  s.mt_live = false;
  WaveBuf& w = g->waves[s.wave_buf];
  if (--w.live == 0 && !g->keep_all) {
    g->alloc.put(w.m, g->stream);
    g->alloc.put(w.t, g->stream);
    w.m = w.t = nullptr;
  }
}

// Block mapping (host mirror of ftk::block_factor_segs; used for shard
// weights and unroll).
void host_block_segs(const StepRec& r, int64_t sg, int64_t k, int64_t& sx, int64_t& sy,
                     int64_t& sz) {
  if (r.kind == ftk::K_NODE) {
    int64_t w = sg / r.KC, p = sg % r.KC;
    sx = w * r.KB + k; sy = k; sz = k * r.KC + p;
  } else if (r.kind == ftk::K_LDP) {
    sx = k * r.KB + sg; sy = k; sz = sg;
  } else if (r.kind == ftk::K_FINAL) {
    sx = k; sy = 0; sz = 0;
  } else if (r.kind == ftk::K_PAIR) {
    sx = k; sy = k / r.KB; sz = k % r.KB;
  } else if (r.kind == ftk::K_BRANCH) {
    sx = sg; sy = r.KC ? k * r.KA + sg : sg * r.KB + k; sz = k;
  } else if (r.kind == ftk::K_FOLD) {
    sx = sg; sy = r.KB * r.KA + sg; sz = r.KC;
  } else if (r.kind == ftk::K_COMPOSE) {
    const int64_t p = sg / r.KB, q = sg % r.KB;
    sx = p; sy = q * r.KA + p; sz = q;
  } else if (r.kind == ftk::K_REMAP) {
    const int64_t Kv = r.nseg / r.KA, side = r.KC & 1, part = r.KC >> 1;
    const int64_t Kold = part ? r.KB : Kv / r.KB;
    const int64_t w = side == 0 ? sg / r.KA : sg % Kv, y = side == 0 ? sg % r.KA : sg / Kv;
    const int64_t c = part ? w % r.KB : w / r.KB;
    sx = side == 0 ? c * r.KA + y : y * Kold + c;
    sy = 0; sz = 0;
  } else {
    sx = sg; sy = sg; sz = 0;
  }
}

int nccl_fail(ft_graph* g, ncclResult_t nr) {
  g->poisoned = FT_ECUDA;
  g->err = std::string("nccl: ") + ncclGetErrorString(nr);
  return FT_ECUDA;
}

// Device -> host copy ordered after the handle's stream (its work may still be
// in flight: waves do not end with a host sync), then wait for it.
cudaError_t d2h(ft_graph* g, void* dst, const void* src, size_t bytes) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, g->stream);
  return e != cudaSuccess ? e : cudaStreamSynchronize(g->stream);
}

// Host copy of a set's seg_off (single-rank step outputs keep it on the device
// until needed).
int ensure_off(ft_graph* g, int set) {
  FSet& S = g->sets[set];
  if (S.off_ok) return FT_OK;
  S.off.resize(S.nseg + 1);
  if (S.kind == S_OP || S.kind == S_EDGE) {  // original sets: one tuple per segment (built lazily)
    for (int64_t q = 0; q <= S.nseg; ++q) S.off[q] = q;
    S.off_ok = true;
    return FT_OK;
  }
  CU(d2h(g, S.off.data(), S.d_off, sizeof(int64_t) * (S.nseg + 1)), "seg_off d2h");
  S.off_ok = true;
  return FT_OK;
}

// Executes one wave of mutually independent steps as a single batch
// (DESIGN.md 6): shard the wave's segments over ranks, run the pipeline,
// all-gather counts and survivors, gather into the wave arena.
int exec_wave(ft_graph* g, const std::vector<int>& ids) {
  const double h0 = now_ms();
  g->nwaves++;
  const int ns = (int)ids.size();
  // global segment numbering of the wave (step-major)
  std::vector<int64_t> sbase(ns + 1, 0);
  for (int q = 0; q < ns; ++q) sbase[q + 1] = sbase[q] + g->steps[ids[q]].nseg;
  const int64_t NS = sbase[ns];
  // shared-order node path eligibility (k_node_pack / k_node_shared): Y all singletons,
  // Z an original edge with m = 0
  std::vector<char> shared(ns, 0);
  for (int q = 0; q < ns; ++q) {
    const StepRec& r = g->steps[ids[q]];
    if (r.kind != ftk::K_NODE || r.nblk > ftk::NS_MAXBLK) continue;
    const FSet &Y = g->sets[r.Y], &Z = g->sets[r.Z];
    const bool y1 = Y.kind == S_OP || (Y.kind == S_STEP && g->steps[Y.step].done &&
                                       g->steps[Y.step].st.survivors == Y.nseg);
    bool zok = false;
    if (Z.kind == S_EDGE) {
      if (g->set_edge.empty()) {  // original edge of each edge set (built once)
        g->set_edge.assign(g->sets.size(), -1);
        for (int e = 0; e < g->n_orig_edges; ++e)
          if (g->edges[e].set >= 0 && g->edges[e].set < (int)g->set_edge.size())
            g->set_edge[g->edges[e].set] = e;
      }
      const int e = r.Z < (int)g->set_edge.size() ? g->set_edge[r.Z] : -1;
      zok = e >= 0 && g->e_mzero[e] != 0;
    }
    shared[q] = y1 && zok && !g->no_shared;
    if (getenv("FT_DEBUG_SHARED"))
      fprintf(stderr, "[shared] step %d kind %d nblk %lld Y.kind %d y1 %d Z.kind %d zok %d -> %d\n", ids[q],
              r.kind, (long long)r.nblk, Y.kind, (int)y1, Z.kind, (int)zok, (int)shared[q]);
  }
  // Replicated small waves: below tau estimated product tuples
  // every rank computes the whole wave (identical results, no collective).
  // The estimate uses host-known mean segment sizes, identical on all ranks.
  bool replicate = g->world > 1 && !g->loopback;
  if (replicate) {
    double est = 0;
    auto mean_size = [&](int set) {
      const FSet& S = g->sets[set];
      if (S.kind != S_STEP) return 1.0;
      return (double)g->steps[S.step].st.survivors / (double)std::max<int64_t>(S.nseg, 1);
    };
    // shared-order node steps cost ~1/16 per tuple of the generic path
    // (one sort per row, running-min sweeps): sharding them did not pay
    for (int q = 0; q < ns; ++q) {
      const StepRec& r = g->steps[ids[q]];
      est += (shared[q] ? 1.0 / 16 : 1.0) * (double)r.nseg * (double)r.nblk * mean_size(r.X) *
             mean_size(r.Y) * mean_size(r.Z);
    }
    replicate = est < g->replicate_tau;
  }
  const int world = replicate ? 1 : g->world;
  const int rank = replicate ? 0 : g->rank;
  std::vector<int64_t> lo(world + 1, 0);
  lo[world] = NS;
  if (world > 1) {
    // weights = estimated product tuples per segment from host-known mean
    // segment sizes (uniform within a step); any partition gives identical
    // results (ids are shard-invariant, R6) -- the plan only balances load
    auto mean_sz = [&](int set) {
      const FSet& S = g->sets[set];
      if (S.kind != S_STEP) return 1.0;
      return (double)g->steps[S.step].st.survivors / (double)std::max<int64_t>(S.nseg, 1);
    };
    std::vector<int64_t> w(NS, 1);
    int64_t blocks = 0;
    for (int q = 0; q < ns; ++q) blocks += g->steps[ids[q]].nseg * g->steps[ids[q]].nblk;
    if (ns <= 8 && blocks <= (1 << 22)) {
      // few steps (LDP waves, the big ones): exact product tuples per segment
      // from the (replicated) input offsets -- segment costs differ by
      // several x within a step, and the slowest rank sets the wave's time
      for (int q = 0; q < ns; ++q) {
        const StepRec& r = g->steps[ids[q]];
        int rc;
        if ((rc = ensure_off(g, r.X)) || (rc = ensure_off(g, r.Y)) || (rc = ensure_off(g, r.Z))) return rc;
        const FSet &X = g->sets[r.X], &Y = g->sets[r.Y], &Z = g->sets[r.Z];
        const double cap = 4e18 / (double)std::max<int64_t>(NS, 1);
        for (int64_t sg = 0; sg < r.nseg; ++sg) {
          double e = 0;
          for (int64_t k = 0; k < r.nblk; ++k) {
            int64_t sx, sy, sz;
            host_block_segs(r, sg, k, sx, sy, sz);
            e += (double)(X.off[sx + 1] - X.off[sx]) * (double)(Y.off[sy + 1] - Y.off[sy]) *
                 (double)(Z.off[sz + 1] - Z.off[sz]);
          }
          w[sbase[q] + sg] = std::max<int64_t>(1, (int64_t)std::min(e, cap));
        }
      }
    } else {
      for (int q = 0; q < ns; ++q) {
        const StepRec& r = g->steps[ids[q]];
        const double e = (double)r.nblk * mean_sz(r.X) * mean_sz(r.Y) * mean_sz(r.Z);
        const int64_t wi = std::max<int64_t>(1, (int64_t)std::min(e, 4e18 / (double)std::max<int64_t>(NS, 1)));
        for (int64_t sg = 0; sg < r.nseg; ++sg) w[sbase[q] + sg] = wi;
      }
    }
    ft_shard_plan(NS, w.data(), world, lo.data());
  }
  auto make_groups = [&](const std::vector<ftk::StepDev>& v) {
    std::vector<ftk::NodeGroupH> gr;
    int64_t base = 0;
    for (int q = 0; q < ns; ++q) {
      const ftk::StepDev& d = v[q];
      if (d.node_shared && d.seg_hi > d.seg_lo) {
        for (int64_t w = d.seg_lo / d.KC; w <= (d.seg_hi - 1) / d.KC; ++w) {
          const int64_t a0 = std::max(d.seg_lo, w * d.KC), a1 = std::min(d.seg_hi, (w + 1) * d.KC);
          ftk::NodeGroupH G;
          G.step = q;
          G.pad = 0;
          G.w = w;
          G.p_lo = a0 - w * d.KC;
          G.p_hi = a1 - w * d.KC;
          G.gs0 = base + (a0 - d.seg_lo);
          gr.push_back(G);
        }
      }
      base += d.seg_hi - d.seg_lo;
    }
    return gr;
  };
  // step descriptors for the global segment range [a, b) of the wave
  auto make_sd = [&](int64_t a, int64_t b) {
  std::vector<ftk::StepDev> sd(ns);
  for (int q = 0; q < ns; ++q) {
    const StepRec& r = g->steps[ids[q]];
    ftk::StepDev& d = sd[q];
    std::memset(&d, 0, sizeof(d));
    d.kind = r.kind;
    d.node_shared = shared[q];
    d.KA = r.KA;
    d.KB = r.KB;
    d.KC = r.KC;
    d.nseg = r.nseg;
    d.nblk = r.nblk;
    d.X = fac(g->sets[r.X]);
    d.Y = fac(g->sets[r.Y]);
    d.Z = fac(g->sets[r.Z]);
    d.seg_lo = std::min(std::max(a - sbase[q], (int64_t)0), r.nseg);
    d.seg_hi = std::min(std::max(b - sbase[q], (int64_t)0), r.nseg);
  }
  return sd;
  };
  // Multi-rank wave with the device-side exchange: per-segment
  // counts are all-gathered on the device, every rank scans them into the
  // same arena offsets, gathers its own contiguous arena range and broadcasts it.
  if (world > 1 && !g->loopback) {
    std::lock_guard<std::mutex> lock(g->runner->mu);
    g->runner->profile = g->profile;
    std::vector<ftk::StepDev> sd = make_sd(lo[rank], lo[rank + 1]);
    const std::vector<ftk::NodeGroupH> grp = make_groups(sd);
    ftk::StepResult res;
    const double h1 = now_ms();
    cudaError_t ce = g->runner->run(sd, g->stream, &res, nullptr, &grp, true);
    if (ce == cudaErrorInvalidConfiguration)
      return setf(g, FT_EOVERFLOW, "step shape unsupported (a segment sample did not shrink to the direct path within the level plan)");
    if (ce != cudaSuccess) return cuda_fail(g, ce, "step pipeline");
    const double h2 = now_ms();
    cudaEvent_t ca, cb;
    cudaEventCreate(&ca);
    cudaEventCreate(&cb);
    cudaEventRecord(ca, g->stream);
    // the wave arena is registered before its buffers are allocated, so a
    // failure part-way leaves nothing unowned (ft_graph_destroy frees it)
    const int wi = (int)g->waves.size();
    g->waves.emplace_back();
    WaveBuf& wb = g->waves.back();
    // Exchange by two all-gathers: (1) every rank's per-segment
    // {survivor counts, product tuples}, padded to the largest rank range;
    // every rank scans them into the same arena offsets; (2) every rank's
    // survivors, staged contiguously and padded to the largest rank total,
    // then unpacked into the arena (one collective each instead of one
    // broadcast per root and array).
    int64_t *cntg = nullptr, *tupg = nullptr, *pos = nullptr, *sb = nullptr, *stats = nullptr,
            *tmp = nullptr, *hloc = nullptr, *hall = nullptr, *lod = nullptr, *posd = nullptr;
    Temps tmps{g->alloc, g->stream};
    const int64_t nloc = lo[rank + 1] - lo[rank];
    int64_t maxloc = 1;
    for (int q = 0; q < world; ++q) maxloc = std::max<int64_t>(maxloc, lo[q + 1] - lo[q]);
    CU(tmps.get(&cntg, sizeof(int64_t) * std::max<int64_t>(NS, 1)), "alloc");
    CU(tmps.get(&tupg, sizeof(int64_t) * std::max<int64_t>(NS, 1)), "alloc");
    CU(tmps.get(&pos, sizeof(int64_t) * (NS + 1)), "alloc");
    CU(tmps.get(&sb, sizeof(int64_t) * (ns + 1)), "alloc");
    CU(tmps.get(&stats, sizeof(int64_t) * 3 * ns), "alloc");
    CU(tmps.get(&tmp, sizeof(int64_t) * ftk::scan_tmp_elems(NS + 1)), "alloc");
    CU(tmps.get(&hloc, sizeof(int64_t) * 2 * maxloc), "alloc");
    CU(tmps.get(&hall, sizeof(int64_t) * 2 * maxloc * world), "alloc");
    CU(tmps.get(&lod, sizeof(int64_t) * 2 * (world + 1)), "alloc");
    posd = lod + world + 1;
    CU(g->alloc.get((void**)&wb.off, sizeof(int64_t) * (NS + ns), g->stream), "alloc frontier");
    if (nloc > 0) {
      CU(cudaMemcpyAsync(hloc, res.dev_cnt, sizeof(int64_t) * nloc, cudaMemcpyDeviceToDevice, g->stream), "counts");
      CU(cudaMemcpyAsync(hloc + maxloc, res.dev_tup, sizeof(int64_t) * nloc, cudaMemcpyDeviceToDevice, g->stream),
         "counts");
    }
    CU(cudaMemcpyAsync(lod, lo.data(), sizeof(int64_t) * (world + 1), cudaMemcpyHostToDevice, g->stream), "lo");
    CU(cudaMemcpyAsync(sb, sbase.data(), sizeof(int64_t) * (ns + 1), cudaMemcpyHostToDevice, g->stream), "sbase");
    ncclResult_t nr = ncclAllGather(hloc, hall, 2 * maxloc, ncclInt64, g->comm, g->stream);
    if (nr != ncclSuccess) return nccl_fail(g, nr);
    CU(ftk::unpack_counts(hall, maxloc, lod, world, NS, cntg, tupg, g->stream), "unpack counts");
    CU(ftk::wave_offsets(cntg, tupg, NS, ns, sb, pos, wb.off, stats, tmp, g->stream), "wave offsets");
    std::vector<int64_t> hstat(3 * ns), posb(world + 1);
    CU(cudaMemcpyAsync(hstat.data(), stats, sizeof(int64_t) * 3 * ns, cudaMemcpyDeviceToHost, g->stream), "stats");
    for (int q = 0; q <= world; ++q)
      CU(cudaMemcpyAsync(&posb[q], pos + lo[q], sizeof(int64_t), cudaMemcpyDeviceToHost, g->stream), "pos");
    CU(cudaStreamSynchronize(g->stream), "wave offsets");
    std::vector<int64_t> sbeg(ns + 1, 0);
    for (int q = 0; q < ns; ++q) sbeg[q + 1] = sbeg[q] + hstat[3 * q];
    const int64_t total = sbeg[ns];
    int64_t maxn = 1;
    for (int q = 0; q < world; ++q) maxn = std::max<int64_t>(maxn, posb[q + 1] - posb[q]);
    const size_t nb = sizeof(int64_t) * std::max<int64_t>(total, 1);
    CU(g->alloc.get((void**)&wb.m, nb, g->stream), "alloc frontier");
    CU(g->alloc.get((void**)&wb.t, nb, g->stream), "alloc frontier");
    CU(g->alloc.get((void**)&wb.bp, nb, g->stream), "alloc frontier");
    int64_t *sloc = nullptr, *sall = nullptr;
    CU(tmps.get(&sloc, sizeof(int64_t) * 3 * maxn), "alloc");
    CU(tmps.get(&sall, sizeof(int64_t) * 3 * maxn * world), "alloc");
    // this rank's survivors -> staging {m[maxn], t[maxn], bp[maxn]} (positions
    // relative to its arena start posb[rank])
    CU(ftk::gather_range(res.pool, pos, lo[rank], lo[rank + 1], posb[rank + 1] - posb[rank],
                         sloc - posb[rank], sloc + maxn - posb[rank],
                         (uint64_t*)(sloc + 2 * maxn) - posb[rank], g->stream), "gather");
    CU(cudaMemcpyAsync(posd, posb.data(), sizeof(int64_t) * (world + 1), cudaMemcpyHostToDevice, g->stream),
       "posb");
    nr = ncclAllGather(sloc, sall, 3 * maxn, ncclInt64, g->comm, g->stream);
    if (nr != ncclSuccess) return nccl_fail(g, nr);
    CU(ftk::unpack_data(sall, maxn, posd, world, maxn, wb.m, wb.t, wb.bp, g->stream), "unpack survivors");
    cudaEventRecord(cb, g->stream);
    // no host sync at the end of the wave (the next one is stream-ordered);
    // the exchange time is read from the events when stats are requested
    g->runner->fence(g->stream);
    CU(cudaGetLastError(), "wave");
    const float comm_ms = 0;
    g->comm_ev.push_back({ids[0], ca, cb});
    const double h4 = now_ms();
    wb.live = ns;
    for (int q = 0; q < ns; ++q) {
      StepRec& r = g->steps[ids[q]];
      FSet& o = g->sets[r.out];
      o.off_ok = false;
      o.d_off = wb.off + sbase[q] + q;
      o.d_m = wb.m + sbeg[q];
      o.d_t = wb.t + sbeg[q];
      o.d_bp = wb.bp + sbeg[q];
      o.wave_buf = wi;
      r.done = true;
      ft_step_stats& st = r.st;
      st.kind = r.kind;
      st.levels = res.levels;
      st.wave = wi;
      st.nseg = r.nseg;
      st.nblk = r.nblk;
      st.tuples = hstat[3 * q + 2];
      st.max_seg = hstat[3 * q + 1];
      st.survivors = hstat[3 * q];
      st.retries = res.retries;
      if (q == 0) {
        st.candidates = res.candidates;
        st.filter_tuples = res.filter_tuples;
        st.direct_tuples = res.direct_tuples;
        for (int u = 0; u < 4; ++u) st.path[u] = res.path[u];
        st.kernel_ms = res.kernel_ms;
        st.comm_ms = comm_ms;
        st.launches = res.launches + 3;
        st.plan_ms = res.plan_ms;
        st.direct_ms = res.direct_ms;
        st.filter_ms = res.filter_ms;
        st.bucket_ms = res.bucket_ms;
        st.compact_ms = res.compact_ms;
        st.host_ms = res.host_ms;
      }
    }
    for (int q = 0; q < ns; ++q) {
      const StepRec& r = g->steps[ids[q]];
      consume(g, r.X);
      consume(g, r.Y);
      consume(g, r.Z);
    }
    g->hp[0] += h1 - h0;
    g->hp[1] += h2 - h1;
    g->hp[3] += h4 - h2;
    g->hp[4] += now_ms() - h4;
    return FT_OK;
  }
  // Single rank, a replicated wave (every rank computes all of it: no
  // collective), or loopback (every virtual rank's shard runs here).
  std::vector<int> vr;
  if (g->loopback)
    for (int q = 0; q < g->world; ++q) vr.push_back(q);
  else
    vr.push_back(rank);
  ftk::StepResult res, agg;
  const double h1 = now_ms();
  std::lock_guard<std::mutex> lock(g->runner->mu);
  g->runner->profile = g->profile;
  // single rank (or replicated wave): offsets computed on the device straight into the arena
  const bool devoff = world == 1 && !g->loopback;
  const int wi = (int)g->waves.size();
  g->waves.emplace_back();  // registered first: see the multi-rank branch
  WaveBuf& wb = g->waves.back();
  if (devoff)
    CU(g->alloc.get((void**)&wb.off, sizeof(int64_t) * (NS + ns), g->stream), "alloc frontier");
  std::vector<int64_t> cnt(devoff ? 0 : NS, 0), tup(devoff ? 0 : NS, 0);
  std::vector<int64_t> stot(ns, 0), smax(ns, 0), stup(ns, 0);
  std::vector<ftk::StepDev> sd;
  for (size_t v = 0; v < vr.size(); ++v) {
    const int64_t a = lo[vr[v]], b = lo[vr[v] + 1];
    sd = make_sd(a, b);
    const std::vector<ftk::NodeGroupH> grp = make_groups(sd);
    cudaError_t ce = g->runner->run(sd, g->stream, &res, devoff ? wb.off : nullptr, &grp);
    if (ce == cudaErrorInvalidConfiguration)
      return setf(g, FT_EOVERFLOW, "step shape unsupported (a segment sample did not shrink to the direct path within the level plan)");
    if (ce != cudaSuccess) return cuda_fail(g, ce, "step pipeline");
    if (devoff) {
      for (int q = 0; q < ns; ++q) {
        stot[q] = res.step_stats[3 * q];
        smax[q] = res.step_stats[3 * q + 1];
        stup[q] = res.step_stats[3 * q + 2];
      }
    } else {
      for (int64_t i = 0; i < res.nloc; ++i) {  // per-segment survivor counts
        cnt[a + i] = res.counts[i];
        tup[a + i] = res.seg_tuples[i];
      }
    }
    agg.levels = std::max(agg.levels, res.levels);
    agg.candidates += res.candidates;
    agg.filter_tuples += res.filter_tuples;
    agg.direct_tuples += res.direct_tuples;
    for (int u = 0; u < 4; ++u) agg.path[u] += res.path[u];
    agg.kernel_ms += res.kernel_ms;
    agg.launches += res.launches;
    agg.retries += res.retries;
    agg.plan_ms += res.plan_ms;
    agg.direct_ms += res.direct_ms;
    agg.filter_ms += res.filter_ms;
    agg.bucket_ms += res.bucket_ms;
    agg.compact_ms += res.compact_ms;
    agg.host_ms += res.host_ms;
  }
  const double h2 = now_ms();
  // wave arena: step-major CSR
  std::vector<int64_t> hoff(devoff ? 0 : NS + ns, 0);  // per step: nseg+1 offsets (relative)
  std::vector<int64_t> sbeg(ns + 1, 0);                // survivor start of each step in the arena
  for (int q = 0; q < ns; ++q) {
    if (devoff) {
      sbeg[q + 1] = sbeg[q] + stot[q];
      continue;
    }
    int64_t* o = hoff.data() + sbase[q] + q;
    o[0] = 0;
    for (int64_t i = 0; i < g->steps[ids[q]].nseg; ++i) o[i + 1] = o[i] + cnt[sbase[q] + i];
    sbeg[q + 1] = sbeg[q] + o[g->steps[ids[q]].nseg];
    stot[q] = o[g->steps[ids[q]].nseg];
    for (int64_t i = 0; i < g->steps[ids[q]].nseg; ++i) {
      stup[q] += tup[sbase[q] + i];
      smax[q] = std::max<int64_t>(smax[q], cnt[sbase[q] + i]);
    }
  }
  const int64_t total = sbeg[ns];
  const size_t nb = sizeof(int64_t) * std::max<int64_t>(total, 1);
  CU(g->alloc.get((void**)&wb.m, nb, g->stream), "alloc frontier");
  CU(g->alloc.get((void**)&wb.t, nb, g->stream), "alloc frontier");
  CU(g->alloc.get((void**)&wb.bp, nb, g->stream), "alloc frontier");
  if (!devoff) {
    CU(g->alloc.get((void**)&wb.off, sizeof(int64_t) * (NS + ns), g->stream), "alloc frontier");
    CU(cudaMemcpyAsync(wb.off, hoff.data(), sizeof(int64_t) * (NS + ns), cudaMemcpyHostToDevice,
                       g->stream), "upload seg_off");
  }
  auto set_out = [&](std::vector<ftk::StepDev>& v) {
    for (int q = 0; q < ns; ++q) {
      ftk::StepDev& d = v[q];
      d.out_m = wb.m + sbeg[q];
      d.out_t = wb.t + sbeg[q];
      d.out_bp = wb.bp + sbeg[q];
      d.out_off = wb.off + sbase[q] + q + d.seg_lo;
    }
  };
  set_out(sd);
  const double h3 = now_ms();
  CU(g->runner->gather(sd, res, g->stream), "gather");  // last (or only) rank's pool
  for (size_t v = 0; v + 1 < vr.size(); ++v) {           // loopback: re-run the others
    std::vector<ftk::StepDev> sv = make_sd(lo[vr[v]], lo[vr[v] + 1]);
    const std::vector<ftk::NodeGroupH> grp = make_groups(sv);
    cudaError_t ce = g->runner->run(sv, g->stream, &res, nullptr, &grp);
    if (ce != cudaSuccess) return cuda_fail(g, ce, "step pipeline (loopback)");
    set_out(sv);
    CU(g->runner->gather(sv, res, g->stream), "gather");
  }
  // no host sync: the next wave's work is ordered behind this one on the
  // stream, and the host needs nothing from the gather (the runner's fence
  // orders other streams that use the same scratch)
  g->runner->fence(g->stream);
  CU(cudaGetLastError(), "wave");
  const double h4 = now_ms();
  // bookkeeping: sets, stats, consumption
  wb.live = ns;
  for (int q = 0; q < ns; ++q) {
    StepRec& r = g->steps[ids[q]];
    FSet& o = g->sets[r.out];
    if (devoff) {
      o.off_ok = false;  // fetched lazily (unroll, ft_step_output)
    } else {
      o.off.assign(hoff.begin() + sbase[q] + q, hoff.begin() + sbase[q] + q + r.nseg + 1);
      o.off_ok = true;
    }
    o.d_off = wb.off + sbase[q] + q;
    o.d_m = wb.m + sbeg[q];
    o.d_t = wb.t + sbeg[q];
    o.d_bp = wb.bp + sbeg[q];
    o.wave_buf = wi;
    r.done = true;
    ft_step_stats& st = r.st;
    st.kind = r.kind;
    st.levels = agg.levels;
    st.wave = wi;
    st.nseg = r.nseg;
    st.nblk = r.nblk;
    st.tuples = stup[q];
    st.max_seg = smax[q];
    st.survivors = stot[q];
    st.retries = agg.retries;
    if (q == 0) {  // wave-level numbers are booked on the wave's first step
      st.candidates = agg.candidates;
      st.filter_tuples = agg.filter_tuples;
      st.direct_tuples = agg.direct_tuples;
      for (int u = 0; u < 4; ++u) st.path[u] = agg.path[u];
      st.kernel_ms = agg.kernel_ms;
      st.comm_ms = 0;  // no collective: one rank, a replicated wave, or loopback
      st.launches = agg.launches + (int64_t)vr.size();
      st.plan_ms = agg.plan_ms;
      st.direct_ms = agg.direct_ms;
      st.filter_ms = agg.filter_ms;
      st.bucket_ms = agg.bucket_ms;
      st.compact_ms = agg.compact_ms;
      st.host_ms = agg.host_ms;
    }
  }
  for (int q = 0; q < ns; ++q) {
    const StepRec& r = g->steps[ids[q]];
    consume(g, r.X);
    consume(g, r.Y);
    consume(g, r.Z);
  }
  const double h5 = now_ms();
  g->hp[0] += h1 - h0;  // shard plan + descriptors
  g->hp[1] += h2 - h1;  // pipeline (2 syncs inside)
  g->hp[2] += h3 - h2;  // counts -> arena offsets, alloc, upload
  g->hp[3] += h4 - h3;  // gather + sync
  g->hp[4] += h5 - h4;  // bookkeeping
  return FT_OK;
}

// Runs every scheduled step: wave(step) = 1 + max wave of its pending
// producers; each wave is one batched pipeline run.  The results do not
// depend on the grouping (each step is a function of its inputs only).
int flush(ft_graph* g) {
  if (g->pending.empty()) return FT_OK;
  const double f0 = now_ms();
  std::vector<int> wave(g->steps.size(), 0);
  int maxw = 0;
  for (int id : g->pending) {
    const StepRec& r = g->steps[id];
    int w = 1;
    for (int in : {r.X, r.Y, r.Z}) {
      const FSet& S = g->sets[in];
      if (S.kind == S_STEP && !g->steps[S.step].done) w = std::max(w, wave[S.step] + 1);
    }
    wave[id] = w;
    maxw = std::max(maxw, w);
  }
  std::vector<std::vector<int>> groups(maxw + 1);
  for (int id : g->pending) groups[wave[id]].push_back(id);
  g->pending.clear();
  g->hp[5] += now_ms() - f0;  // wave assignment
  for (int w = 1; w <= maxw; ++w) {
    int rc = exec_wave(g, groups[w]);
    if (rc) return rc;
  }
  return FT_OK;
}

// Schedules a step (no GPU work): creates its output set placeholder.
int schedule(ft_graph* g, StepRec r) {
  FSet o;
  o.kind = S_STEP;
  o.step = (int)g->steps.size();
  o.nseg = r.nseg;
  r.out = (int)g->sets.size();
  g->sets.push_back(std::move(o));
  g->steps.push_back(r);
  g->pending.push_back((int)g->steps.size() - 1);
  return r.out;
}

// ---- eliminations (structural; steps are scheduled, then flushed) ----------

int do_node(ft_graph* g, int i, int* new_edge) {  // Eq.4
  int ehi = *g->in_e[i].begin(), eij = *g->out_e[i].begin();
  int h = g->edges[ehi].src, j = g->edges[eij].dst;
  StepRec r;
  r.kind = ftk::K_NODE;
  r.X = g->edges[ehi].set;
  r.Y = g->op_set[i];
  r.Z = g->edges[eij].set;
  r.KA = g->K[h];
  r.KB = g->K[i];
  r.KC = g->K[j];
  r.nseg = r.KA * r.KC;
  r.nblk = r.KB;
  int out = schedule(g, r);
  g->sets[out].a_op = h;
  g->sets[out].b_op = j;
  kill_edge(g, ehi);
  kill_edge(g, eij);
  kill_op(g, i);
  int e = add_edge(g, h, j, out);
  if (new_edge) *new_edge = e;
  return FT_OK;
}

int do_merge(ft_graph* g, int e1, int e2, int* new_edge) {  // Eq.5, binary
  int u = g->edges[e1].src, v = g->edges[e1].dst;
  StepRec r;
  r.kind = ftk::K_EDGE;
  r.X = g->edges[e1].set;
  r.Y = g->edges[e2].set;
  r.Z = 0;
  r.KA = g->K[u];
  r.KB = g->K[v];
  r.nseg = r.KA * r.KB;
  r.nblk = 1;
  int out = schedule(g, r);
  g->sets[out].a_op = u;
  g->sets[out].b_op = v;
  kill_edge(g, e1);
  kill_edge(g, e2);
  int e = add_edge(g, u, v, out);
  if (new_edge) *new_edge = e;
  return FT_OK;
}

// Exact K=1 case of Eq.7: fold the source into every consumer;
// the source's own cost goes to its topologically first consumer (R13).
int do_fold(ft_graph* g, int src, int64_t kstar = 0) {
  std::vector<int> outs(g->out_e[src].begin(), g->out_e[src].end());  // ascending ids
  int first = -1;
  for (int e : outs) {
    int c = g->edges[e].dst;
    if (first < 0 || g->pos0[c] < g->pos0[first]) first = c;
  }
  for (int e : outs) {
    int c = g->edges[e].dst;
    StepRec r;
    r.kind = ftk::K_FOLD;
    r.X = g->op_set[c];
    r.Y = g->edges[e].set;
    r.Z = c == first ? g->op_set[src] : 0;
    r.KA = g->K[c];
    r.KB = kstar;                     // edge segment k* * K_c + p
    r.KC = c == first ? kstar : 0;    // op segment k* (unit set: 0)
    r.nseg = g->K[c];
    r.nblk = 1;
    int out = schedule(g, r);
    g->sets[out].a_op = c;
    g->op_set[c] = out;
    kill_edge(g, e);
  }
  kill_op(g, src);
  return FT_OK;
}

// Eq. 6, reading R14: o_i's only edge e connects it to o_h; it is
// merged into o_h and the union over s_i is reduced at once:
//   F(o_h, s_h) <- reduce(U_{s_i} F(o_h, s_h) (x) F(e, .) (x) F(o_i, s_i)).
int do_branch(ft_graph* g, int i) {
  const bool src = g->in_e[i].empty();  // o_i -> o_h, else o_h -> o_i
  const int e = src ? *g->out_e[i].begin() : *g->in_e[i].begin();
  const int h = src ? g->edges[e].dst : g->edges[e].src;
  StepRec r;
  r.kind = ftk::K_BRANCH;
  r.X = g->op_set[h];
  r.Y = g->edges[e].set;
  r.Z = g->op_set[i];
  r.KA = g->K[h];
  r.KB = g->K[i];
  r.KC = src ? 1 : 0;
  r.nseg = g->K[h];
  r.nblk = g->K[i];
  int out = schedule(g, r);
  g->sets[out].a_op = h;
  g->op_set[h] = out;
  kill_edge(g, e);
  kill_op(g, i);
  return FT_OK;
}

// Re-derives the live graph's topological order after a composite merge
// (R21): Kahn's algorithm, ready ops by (previous position, id); the
// position-keyed candidate sets are rebuilt.
void reorder(ft_graph* g) {
  const int n = (int)g->K.size();
  std::vector<int> indeg(n, 0);
  std::set<std::pair<int, int>> ready;
  for (int v = 0; v < n; ++v)
    if (g->op_alive[v]) {
      indeg[v] = (int)g->in_e[v].size();
      if (indeg[v] == 0) ready.insert({g->pos0[v], v});
    }
  std::vector<int> order;
  while (!ready.empty()) {
    const int u = ready.begin()->second;
    ready.erase(ready.begin());
    order.push_back(u);
    for (int e : g->out_e[u]) {
      const int d = g->edges[e].dst;
      if (--indeg[d] == 0) ready.insert({g->pos0[d], d});
    }
  }
  for (size_t q = 0; q < order.size(); ++q) g->pos0[order[q]] = (int)q;
  g->order0 = order;
  g->mark_dirty = true;
  g->live_ops.clear();
  g->one_one.clear();
  g->leaf.clear();
  g->k1src.clear();
  g->multi.clear();
  std::fill(g->cand.begin(), g->cand.end(), 0);
  for (int v : order) {
    g->live_ops.insert({g->pos0[v], v});
    refresh(g, v);
  }
  for (const auto& kv : g->pair_edges)
    if (kv.second.size() >= 2) g->multi.insert({g->pos0[kv.first.first], g->pos0[kv.first.second]});
}

// A path o_i -> ... -> o_h other than the direct edges (merging o_i into
// o_h would close a cycle).
bool other_path(const ft_graph* g, int i, int h) {
  std::vector<char> seen(g->K.size(), 0);
  std::vector<int> st;
  for (int e : g->out_e[i])
    if (g->edges[e].dst != h) st.push_back(g->edges[e].dst);
  while (!st.empty()) {
    const int u = st.back();
    st.pop_back();
    if (u == h) return true;
    if (seen[u]) continue;
    seen[u] = 1;
    for (int e : g->out_e[u]) st.push_back(g->edges[e].dst);
  }
  return false;
}

// Eq. 6 with composite configurations (reading R21): o_i feeds
// o_h through the single edge e and keeps other edges, so nothing is reduced
// over s_i; o_i and o_h become one operator o_v with configurations
// w = (s_h, s_i) = s_h * K_i + s_i:
//   F(o_v, w) = reduce(F(o_h, s_h) (x) F(e, s_i, s_h) (x) F(o_i, s_i))  (K_COMPOSE)
// and every other edge of o_h or o_i is re-indexed onto o_v (K_REMAP).
int do_compose(ft_graph* g, int i, int h) {
  int e = -1;
  for (int x : g->in_e[h])
    if (g->edges[x].src == i) e = x;
  const int v = (int)g->K.size();
  const int Kv = g->K[h] * g->K[i];
  g->K.push_back(Kv);
  g->op_alive.push_back(1);
  g->in_e.emplace_back();
  g->out_e.emplace_back();
  g->pos0.push_back(g->pos0[h]);
  g->mark_stamp.push_back(0);
  g->comp.push_back({h, i});
  StepRec r;
  r.kind = ftk::K_COMPOSE;
  r.X = g->op_set[h];
  r.Y = g->edges[e].set;
  r.Z = g->op_set[i];
  r.KA = g->K[h];
  r.KB = g->K[i];
  r.nseg = Kv;
  r.nblk = 1;
  const int out = schedule(g, r);
  g->sets[out].a_op = v;
  g->op_set.push_back(out);
  std::set<int> others;  // the other edges of o_h and o_i, ascending id
  for (int o : {h, i}) {
    others.insert(g->in_e[o].begin(), g->in_e[o].end());
    others.insert(g->out_e[o].begin(), g->out_e[o].end());
  }
  others.erase(e);
  kill_edge(g, e);
  for (int x : others) {
    const int src = g->edges[x].src, dst = g->edges[x].dst;
    const int old = (src == h || src == i) ? src : dst;
    const int y = old == src ? dst : src;
    StepRec q;
    q.kind = ftk::K_REMAP;
    q.X = g->edges[x].set;
    q.Y = 0;
    q.Z = 0;
    q.KA = g->K[y];
    q.KB = g->K[i];
    q.KC = (old == src ? 0 : 1) | (old == i ? 2 : 0);
    q.nseg = (int64_t)Kv * g->K[y];
    q.nblk = 1;
    const int so = schedule(g, q);
    const int ns = old == src ? v : y, nd = old == src ? y : v;
    g->sets[so].a_op = ns;
    g->sets[so].b_op = nd;
    kill_edge(g, x);
    add_edge(g, ns, nd, so);
  }
  kill_op(g, h);
  kill_op(g, i);
  reorder(g);
  return FT_OK;
}

// Composite candidate (R21): the topologically first operator o_h with >= 2
// input operators that has an unmarked input o_i with K_h * K_i <= 4096, no
// other path o_i -> o_h, and that is not a source feeding >= 2 operators (a
// broadcast input like BERT's mask, left to heuristic elimination,
// P:618-620); among its inputs the smallest K_i, ties by position.
// Requires a fresh mark_backbone.  Returns 1 = merged, 0 = none.
int compose_step(ft_graph* g) {
  for (const auto& kv : g->live_ops) {
    const int h = kv.second;
    std::set<std::pair<int, int>> ins;
    for (int e : g->in_e[h]) ins.insert({g->pos0[g->edges[e].src], g->edges[e].src});
    if (ins.size() < 2) continue;
    int best = -1;
    for (const auto& pi : ins) {
      const int i = pi.second;
      if (g->mark_stamp[i] == g->stamp || (int64_t)g->K[h] * g->K[i] > 4096 || other_path(g, i, h)) continue;
      if (g->in_e[i].empty()) {
        std::set<int> outs;
        for (int x : g->out_e[i]) outs.insert(g->edges[x].dst);
        if (outs.size() >= 2) continue;
      }
      if (best < 0 || g->K[i] < g->K[best]) best = i;
    }
    if (best >= 0) {
      int rc = do_compose(g, best, h);
      return rc ? rc : 1;
    }
  }
  return 0;
}

// One FT_AUTO elimination (R9).  1 = scheduled, 0 = none applies, <0 error.
// compose = false skips (e) (FT_AUTO_HEUR tries heuristic elimination first).
int auto_step(ft_graph* g, bool compose) {
  mark_backbone(g);
  // (a) parallel edges: topologically first (src, dst), two lowest ids
  if (!g->multi.empty()) {
    const auto key = *g->multi.begin();
    const int u = g->order0[key.first], v = g->order0[key.second];
    const auto& es = g->pair_edges[{u, v}];
    const int e1 = *es.begin(), e2 = *std::next(es.begin());
    int rc = do_merge(g, e1, e2, nullptr);
    return rc ? rc : 1;
  }
  // (b) node elimination: topologically first unmarked 1-in-1-out op
  for (const auto& kv : g->one_one)
    if (g->mark_stamp[kv.second] != g->stamp) {
      int rc = do_node(g, kv.second, nullptr);
      return rc ? rc : 1;
    }
  // (c) K=1 source fold (Eq. 7, exact for K=1)
  if (!g->k1src.empty()) {
    int rc = do_fold(g, g->k1src.begin()->second);
    return rc ? rc : 1;
  }
  // (d) branch elimination (Eq. 6): topologically first unmarked op with one
  //     edge (after the fold, which keeps the backbone intact: DESIGN.md R14)
  for (const auto& kv : g->leaf)
    if (g->mark_stamp[kv.second] != g->stamp) {
      int rc = do_branch(g, kv.second);
      return rc ? rc : 1;
    }
  // (e) branch elimination with composite configurations (Eq. 6, R21)
  return compose ? compose_step(g) : 0;
}

// Heuristic elimination (Eq. 7; lossy, FT_AUTO_HEUR only): the
// unmarked source op with the most out-edges (ties: topological order),
// K >= 2, gets the configuration of least memory -- min over k of the first
// (least-m) tuple of F(o_i, k), ties by its t, then k -- and is folded into
// its consumers.  1 = done, 0 = no candidate, < 0 error.
int heur_step(ft_graph* g) {
  mark_backbone(g);
  int best = -1;
  for (const auto& kv : g->live_ops) {
    const int v = kv.second;
    if (g->mark_stamp[v] == g->stamp || g->K[v] < 2 || !g->in_e[v].empty() || g->out_e[v].empty())
      continue;
    if (best < 0 || g->out_e[v].size() > g->out_e[best].size()) best = v;
  }
  if (best < 0) return 0;
  int rc = flush(g);  // the op's frontier may come from a pending step
  if (rc) return rc;
  const int set = g->op_set[best];
  if ((rc = ensure_off(g, set))) return rc;
  const FSet& S = g->sets[set];
  const int64_t n = S.off[S.nseg];
  std::vector<int64_t> hm(n), ht(n);
  CU(d2h(g, hm.data(), S.d_m, sizeof(int64_t) * n), "d2h");
  CU(d2h(g, ht.data(), S.d_t, sizeof(int64_t) * n), "d2h");
  int64_t ks = 0;
  if (g->heur_policy == 0) {
    for (int64_t k = 1; k < S.nseg; ++k) {
      const int64_t a = S.off[k], b = S.off[ks];
      if (hm[a] < hm[b] || (hm[a] == hm[b] && ht[a] < ht[b])) ks = k;
    }
  } else {
    // R22 (weighted combination): score alpha*m/M + (1-alpha)*t/T per
    // tuple in IEEE double (M, T = largest m, t over F(o_i, .), >= 1; each
    // operation rounded separately, no contraction); least score wins, ties
    // by (m, t), then k
    int64_t M = 1, T = 1;
    for (int64_t q = 0; q < n; ++q) {
      M = std::max(M, hm[q]);
      T = std::max(T, ht[q]);
    }
    const double al = (double)g->heur_num / (double)g->heur_den;
    bool have = false;
    double bs = 0;
    int64_t bm = 0, bt = 0;
    for (int64_t k = 0; k < S.nseg; ++k)
      for (int64_t q = S.off[k]; q < S.off[k + 1]; ++q) {
        const double dm = (double)hm[q] / (double)M, dt = (double)ht[q] / (double)T;
        const double sc = al * dm + (1.0 - al) * dt;
        if (!have || sc < bs || (sc == bs && (hm[q] < bm || (hm[q] == bm && ht[q] < bt)))) {
          have = true;
          bs = sc;
          bm = hm[q];
          bt = ht[q];
          ks = k;
        }
      }
  }
  rc = do_fold(g, best, ks);
  return rc ? rc : 1;
}

// The live graph as a chain o_1 -> ... -> o_n (LDP / FT-Elimination precondition).
int linear_chain(ft_graph* g, std::vector<int>& chain, std::vector<int>& ce) {
  int src = -1, live = 0;
  for (int v = 0; v < (int)g->K.size(); ++v) {
    if (!g->op_alive[v]) continue;
    ++live;
    if (g->in_e[v].empty()) {
      if (src >= 0) return setf(g, FT_EPRECOND, "graph is not linear (several sources)");
      src = v;
    }
  }
  if (src < 0) return setf(g, FT_EPRECOND, "graph is not linear (no source)");
  for (int v = src;;) {
    chain.push_back(v);
    if (g->out_e[v].empty()) break;
    if (g->out_e[v].size() != 1) return setf(g, FT_EPRECOND, "graph is not linear (fan-out)");
    int e = *g->out_e[v].begin();
    int d = g->edges[e].dst;
    if (g->in_e[d].size() != 1) return setf(g, FT_EPRECOND, "graph is not linear (fan-in)");
    ce.push_back(e);
    v = d;
  }
  if ((int)chain.size() != live) return setf(g, FT_EPRECOND, "graph is not linear (disconnected)");
  return FT_OK;
}

// Runs the scheduled steps and fetches the final frontier (one segment).
int finish_final(ft_graph* g, int out, int mode) {
  int rc = flush(g);
  if (rc) return rc;
  g->final_set = out;
  if ((rc = ensure_off(g, out))) return rc;
  const FSet& F = g->sets[out];
  int64_t n = F.off[1];
  g->final_m.resize(n);
  g->final_t.resize(n);
  if (n) {
    CU(cudaMemcpyAsync(g->final_m.data(), F.d_m, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, g->stream), "d2h");
    CU(cudaMemcpyAsync(g->final_t.data(), F.d_t, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, g->stream), "d2h");
    CU(cudaStreamSynchronize(g->stream), "d2h");
  }
  g->have_final = true;
  g->final_mode = mode;
  return FT_OK;
}

// Alg. 3 on the remaining chain, then the final reduce (line 9).
int run_ldp(ft_graph* g) {
  std::vector<int> chain, ce;
  int rc = linear_chain(g, chain, ce);
  if (rc) return rc;
  int cf = g->op_set[chain[0]];  // CF(o_1, s) = F(o_1, s)  (line 3)
  for (size_t i = 1; i < chain.size(); ++i) {
    StepRec r;
    r.kind = ftk::K_LDP;  // line 6: U_k F(e,k,p) (x) CF(o_{i-1},k) (x) F(o_i,p)
    r.X = g->edges[ce[i - 1]].set;
    r.Y = cf;
    r.Z = g->op_set[chain[i]];
    r.KA = g->K[chain[i - 1]];
    r.KB = g->K[chain[i]];
    r.nseg = r.KB;
    r.nblk = r.KA;
    int out = schedule(g, r);
    g->sets[out].a_op = chain[i];
    cf = out;
  }
  StepRec f;
  f.kind = ftk::K_FINAL;  // line 9: reduce(U_s CF(o_n, s))
  f.X = cf;
  f.Y = 0;
  f.Z = 0;
  f.KA = g->K[chain.back()];
  f.nseg = 1;
  f.nblk = f.KA;
  return finish_final(g, schedule(g, f), 1);
}

// FT-Elimination (Theorem 2): node-eliminate (Eq. 4) the
// second op of the remaining chain until o_1 and o_n are left, then reduce
// over every configuration pair: U_{s_1,s_n} F(e_1n,s_1,s_n) (x) F(o_1,s_1)
// (x) F(o_n,s_n) (one segment, K_1*K_n blocks).  One op: reduce(U_s F(o_1,s)).
int run_elim(ft_graph* g) {
  std::vector<int> chain, ce;
  int rc = linear_chain(g, chain, ce);
  if (rc) return rc;
  for (size_t i = 1; i + 1 < chain.size(); ++i)
    if ((rc = do_node(g, chain[i], nullptr))) return rc;
  StepRec f;
  if (chain.size() == 1) {
    f.kind = ftk::K_FINAL;
    f.X = g->op_set[chain[0]];
    f.Y = 0;
    f.Z = 0;
    f.KA = g->K[chain[0]];
    f.nblk = f.KA;
  } else {
    f.kind = ftk::K_PAIR;
    f.X = g->edges[*g->out_e[chain[0]].begin()].set;
    f.Y = g->op_set[chain[0]];
    f.Z = g->op_set[chain.back()];
    f.KA = g->K[chain[0]];
    f.KB = g->K[chain.back()];
    f.nblk = f.KA * f.KB;
  }
  f.nseg = 1;
  return finish_final(g, schedule(g, f), 2);
}

// ---- unroll -----------------------------------------------------------

int fetch_bp(ft_graph* g, FSet& s) {
  if (s.h_bp_ok) return FT_OK;
  if (!s.off_ok) {
    s.off.resize(s.nseg + 1);
    CU(d2h(g, s.off.data(), s.d_off, sizeof(int64_t) * (s.nseg + 1)), "seg_off d2h");
    s.off_ok = true;
  }
  int64_t n = s.off[s.nseg];
  s.h_bp.resize(n);
  if (n) {
    CU(d2h(g, s.h_bp.data(), s.d_bp, sizeof(uint64_t) * n), "bp d2h");
  }
  s.h_bp_ok = true;
  return FT_OK;
}

int put_cfg(ft_graph* g, std::vector<int32_t>& cfg, int op, int64_t c) {
  if (op < 0) return FT_OK;
  if (cfg[op] >= 0 && cfg[op] != c) {
    g->poisoned = FT_EINTERNAL;
    return setf(g, FT_EINTERNAL, "broken provenance (conflicting configs)");
  }
  cfg[op] = (int32_t)c;
  if (op < (int)g->comp.size() && g->comp[op].first >= 0) {  // composite (R21): w = s_h * K_i + s_i
    const int h = g->comp[op].first, i = g->comp[op].second;
    int rc = put_cfg(g, cfg, h, c / g->K[i]);
    return rc ? rc : put_cfg(g, cfg, i, c % g->K[i]);
  }
  return FT_OK;
}

int unroll(ft_graph* g, int set0, int64_t seg0, int64_t idx0, std::vector<int32_t>& cfg) {
  struct Item {
    int set;
    int64_t seg, idx;
  };
  std::vector<Item> todo{{set0, seg0, idx0}};
  while (!todo.empty()) {
    Item it = todo.back();
    todo.pop_back();
    FSet& S = g->sets[it.set];
    if (S.kind == S_UNIT) continue;
    int rc;
    if (S.b_op >= 0) {
      int64_t kb = g->K[S.b_op];
      if ((rc = put_cfg(g, cfg, S.a_op, it.seg / kb)) || (rc = put_cfg(g, cfg, S.b_op, it.seg % kb))) return rc;
    } else if ((rc = put_cfg(g, cfg, S.a_op, it.seg))) {
      return rc;
    }
    if (S.kind != S_STEP) continue;
    if ((rc = fetch_bp(g, S))) return rc;
    const StepRec& r = g->steps[S.step];
    if ((rc = ensure_off(g, r.X)) || (rc = ensure_off(g, r.Y)) || (rc = ensure_off(g, r.Z))) return rc;
    const uint64_t id = S.h_bp[S.off[it.seg] + it.idx];
    const FSet &X = g->sets[r.X], &Y = g->sets[r.Y], &Z = g->sets[r.Z];
    uint64_t acc = 0;
    bool found = false;
    for (int64_t k = 0; k < r.nblk && !found; ++k) {
      int64_t sx, sy, sz;
      host_block_segs(r, it.seg, k, sx, sy, sz);
      uint64_t nx = X.off[sx + 1] - X.off[sx], ny = Y.off[sy + 1] - Y.off[sy],
               nz = Z.off[sz + 1] - Z.off[sz];
      uint64_t n = nx * ny * nz;
      if (id < acc + n) {
        uint64_t rr = id - acc;
        todo.push_back({r.Z, sz, (int64_t)(rr % nz)});
        todo.push_back({r.Y, sy, (int64_t)((rr / nz) % ny)});
        todo.push_back({r.X, sx, (int64_t)(rr / (ny * nz))});
        found = true;
      }
      acc += n;
    }
    if (!found) {
      g->poisoned = FT_EINTERNAL;
      return setf(g, FT_EINTERNAL, "broken provenance (id out of range)");
    }
  }
  return FT_OK;
}

}  // namespace

// =============================================================================
extern "C" {

const char* ft_version(void) { return "ft-b200 0.1 sm_100a"; }

int ft_shard_plan(int64_t n, const int64_t* w, int32_t world, int64_t* bounds) {
  if (n < 0 || world < 1 || !bounds || (n > 0 && !w)) return FT_EINVAL;
  long double tot = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (w[i] < 0) return FT_EINVAL;
    tot += (long double)w[i];
  }
  bounds[0] = 0;
  long double acc = 0;
  int64_t i = 0;
  for (int q = 1; q < world; ++q) {
    long double target = tot * q / world;
    while (i < n && acc + (long double)w[i] / 2 <= target) acc += (long double)w[i++];
    bounds[q] = std::max<int64_t>(i, bounds[q - 1]);
  }
  bounds[world] = n;
  return FT_OK;
}

int ft_graph_create(int32_t n_ops, const int32_t* n_cfgs, int32_t n_edges, const int32_t* src,
                    const int32_t* dst, const ft_options* opt, ft_graph** out) {
  if (!out) return FT_EINVAL;
  *out = nullptr;
  if (n_ops < 1 || n_edges < 0 || !n_cfgs || (n_edges > 0 && (!src || !dst))) return FT_EINVAL;
  if ((int64_t)n_ops + n_edges >= (1 << 20)) return FT_EOVERFLOW;
  for (int i = 0; i < n_ops; ++i)
    if (n_cfgs[i] < 1 || n_cfgs[i] > 4096) return FT_EINVAL;
  for (int e = 0; e < n_edges; ++e)
    if (src[e] < 0 || src[e] >= n_ops || dst[e] < 0 || dst[e] >= n_ops || src[e] == dst[e])
      return FT_EINVAL;
  ft_graph* g = new (std::nothrow) ft_graph();
  if (!g) return FT_ENOMEM;
  g->n_ops = n_ops;
  g->n_orig_edges = n_edges;
  g->K.assign(n_cfgs, n_cfgs + n_ops);
  g->comp.assign(n_ops, {-1, -1});
  g->op_alive.assign(n_ops, 1);
  g->in_e.resize(n_ops);
  g->out_e.resize(n_ops);
  g->op_m.resize(n_ops);
  g->op_t.resize(n_ops);
  g->op_ok.assign(n_ops, 0);
  g->e_m.resize(n_edges);
  g->e_t.resize(n_edges);
  g->e_ok.assign(n_edges, 0);
  g->e_mzero.assign(n_edges, 0);
  FSet unit;
  unit.kind = S_UNIT;
  unit.nseg = 1;
  unit.off = {0, 1};
  g->sets.push_back(unit);
  for (int i = 0; i < n_ops; ++i) {
    g->op_set0.push_back((int)g->sets.size());
    FSet s;
    s.kind = S_OP;
    s.a_op = i;
    s.nseg = g->K[i];
    s.off_ok = false;  // iota, built on demand (ensure_off)
    g->op_set.push_back((int)g->sets.size());
    g->sets.push_back(std::move(s));
  }
  for (int e = 0; e < n_edges; ++e) {
    FSet s;
    s.kind = S_EDGE;
    s.a_op = src[e];
    s.b_op = dst[e];
    s.nseg = (int64_t)g->K[src[e]] * g->K[dst[e]];
    s.off_ok = false;  // iota, built on demand (ensure_off; C5: 9.4e6 entries)
    add_edge(g, src[e], dst[e], (int)g->sets.size());
    g->sets.push_back(std::move(s));
  }
  {
    std::vector<int> order = topo_order(g);
    if ((int)order.size() != n_ops) {
      delete g;
      return FT_EINVAL;  // cycle
    }
    g->order0 = order;
    g->pos0.assign(n_ops, 0);
    for (int q = 0; q < n_ops; ++q) g->pos0[order[q]] = q;
    g->mark_stamp.assign(n_ops, 0);
    for (int v = 0; v < n_ops; ++v) g->live_ops.insert({g->pos0[v], v});
    for (const auto& kv : g->pair_edges)
      if (kv.second.size() >= 2) g->multi.insert({g->pos0[kv.first.first], g->pos0[kv.first.second]});
    for (int v = 0; v < n_ops; ++v) refresh(g, v);
  }
  if (opt) {
    g->dev = opt->device;
    g->rank = opt->rank;
    g->world = opt->world < 1 ? 1 : opt->world;
    g->comm = (ncclComm_t)opt->nccl_comm;
    g->keep_all = opt->keep_all != 0;
    g->profile = opt->profile != 0;
    g->stream = (cudaStream_t)opt->stream;
    if ((opt->alloc == nullptr) != (opt->free == nullptr)) {
      delete g;
      return FT_EINVAL;  // allocator hooks come in pairs
    }
    g->alloc.alloc = opt->alloc;
    g->alloc.free = opt->free;
    g->alloc.ctx = opt->alloc_ctx;
  }
  if (opt && g->world > 1 && !g->comm && opt->loopback) g->loopback = true;
  g->no_shared = getenv("FT_NO_SHARED") != nullptr;
  if (const char* e = getenv("FT_REPLICATE_TAU")) g->replicate_tau = atof(e);
  if (g->world > 1 && !g->loopback && (!g->comm || g->rank < 0 || g->rank >= g->world)) {
    delete g;
    return FT_EINVAL;
  }
  cudaError_t e = cudaSetDevice(g->dev);
  if (e == cudaSuccess && !g->stream) {
    e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
    g->own_stream = e == cudaSuccess;
  }
  if (e == cudaSuccess) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, g->dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    g->runner = ftk::device_runner(g->dev, g->alloc);
    e = g->runner ? cudaSuccess : cudaErrorMemoryAllocation;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete g;
    return FT_ECUDA;
  }
  *out = g;
  return FT_OK;
}

void ft_graph_destroy(ft_graph* g) {
  if (!g) return;
  if (getenv("FT_HOST_PROF"))
    fprintf(stderr,
            "[libft host ms] waves=%lld plan+desc %.2f pipeline %.2f offsets/alloc %.2f gather+sync %.2f "
            "bookkeeping %.2f wave-assign %.2f policy %.2f\n",
            (long long)g->nwaves, g->hp[0], g->hp[1], g->hp[2], g->hp[3], g->hp[4], g->hp[5], g->hp[6]);
  if (getenv("FT_FILTER_STATS") && g->runner)
    fprintf(stderr, "[libft filter] items %llu chunk_tests %llu skipped_elems %llu tested_elems %llu "
            "G_points %llu one_block_warps %llu warps %llu gallops %llu\n",
            g->runner->fstat_acc[0], g->runner->fstat_acc[1], g->runner->fstat_acc[2],
            g->runner->fstat_acc[3], g->runner->fstat_acc[4], g->runner->fstat_acc[5],
            g->runner->fstat_acc[6], g->runner->fstat_acc[7]);
  if (getenv("FT_FILTER_STATS") && g->runner) {
    fprintf(stderr, "[libft buckets] size-class: count/candidates 1 | 2-4 | 5-8 | 9-16 | 17-32 | 33-64 | 65-128 | 129-256 | <=4096 | >4096\n ");
    for (int q = 0; q < 10; ++q)
      fprintf(stderr, " %llu/%llu", g->runner->bstat_acc[0][q], g->runner->bstat_acc[1][q]);
    fprintf(stderr, "\n[libft buckets] key-sort fallbacks to (m, t, id): lane groups %llu, warps %llu\n",
            g->runner->bfall_acc[0], g->runner->bfall_acc[1]);
  }
  if (g->stream) cudaStreamSynchronize(g->stream);
  for (auto& w : g->waves) {
    if (w.m) g->alloc.put(w.m, g->stream);
    if (w.t) g->alloc.put(w.t, g->stream);
    if (w.bp) g->alloc.put(w.bp, g->stream);
    if (w.off) g->alloc.put(w.off, g->stream);
  }
  if (g->d_costs) g->alloc.put(g->d_costs, g->stream);
  if (g->stream) cudaStreamSynchronize(g->stream);  // back to the pool (not the driver)
  for (auto& ev : g->comm_ev) {
    cudaEventDestroy(ev.a);
    cudaEventDestroy(ev.b);
  }
  if (g->runner) ftk::release_runner(g->dev, g->alloc);
  if (g->own_stream) cudaStreamDestroy(g->stream);
  delete g;
}

int ft_set_op_costs(ft_graph* g, int32_t op, const int64_t* m, const int64_t* t) {
  if (!g) return FT_EINVAL;
  if (g->poisoned) return g->poisoned;
  if (g->started) return setf(g, FT_ESTATE, "costs set after elimination began");
  if (op < 0 || op >= g->n_ops || !m || !t) return setf(g, FT_EINVAL, "bad operator or null costs");
  if (g->bulk_done) return setf(g, FT_ESTATE, "costs already set by ft_set_costs_all");
  const int k = g->K[op];
  for (int q = 0; q < k; ++q) {
    if (m[q] < 0 || t[q] < 0) return setf(g, FT_EINVAL, "negative cost");
    if (m[q] >= ((int64_t)1 << 40) || t[q] >= ((int64_t)1 << 40)) return setf(g, FT_EOVERFLOW, "cost >= 2^40");
  }
  g->op_m[op].assign(m, m + k);
  g->op_t[op].assign(t, t + k);
  g->op_ok[op] = 1;
  g->host_costs_pending = true;
  return FT_OK;
}

int ft_set_edge_costs(ft_graph* g, int32_t edge, const int64_t* m, const int64_t* t) {
  if (!g) return FT_EINVAL;
  if (g->poisoned) return g->poisoned;
  if (g->started) return setf(g, FT_ESTATE, "costs set after elimination began");
  if (edge < 0 || edge >= g->n_orig_edges || !t) return setf(g, FT_EINVAL, "bad edge or null costs");
  if (g->bulk_done) return setf(g, FT_ESTATE, "costs already set by ft_set_costs_all");
  const int64_t n = (int64_t)g->K[g->edges[edge].src] * g->K[g->edges[edge].dst];
  for (int64_t q = 0; q < n; ++q) {
    const int64_t mm = m ? m[q] : 0;
    if (mm < 0 || t[q] < 0) return setf(g, FT_EINVAL, "negative cost");
    if (mm >= ((int64_t)1 << 40) || t[q] >= ((int64_t)1 << 40)) return setf(g, FT_EOVERFLOW, "cost >= 2^40");
  }
  if (m) g->e_m[edge].assign(m, m + n);
  else g->e_m[edge].assign(n, 0);
  g->e_mzero[edge] = 1;
  for (int64_t q = 0; q < n; ++q)
    if (g->e_m[edge][q] != 0) g->e_mzero[edge] = 0;
  g->e_t[edge].assign(t, t + n);
  g->e_ok[edge] = 1;
  g->host_costs_pending = true;
  return FT_OK;
}

int ft_set_costs_all(ft_graph* g, const int64_t* op_m, const int64_t* op_t, const int64_t* edge_m,
                     const int64_t* edge_t) {
  if (!g) return FT_EINVAL;
  if (g->poisoned) return g->poisoned;
  if (g->started) return setf(g, FT_ESTATE, "costs set after elimination began");
  if (!op_m || !op_t || (g->n_orig_edges > 0 && !edge_t)) return setf(g, FT_EINVAL, "null cost array");
  if (g->host_costs_pending || g->bulk_done)
    return setf(g, FT_ESTATE, "ft_set_costs_all must be the only cost setter");
  int rc = alloc_costs(g);
  if (rc) return rc;
  const int64_t nop = g->op_off[g->n_ops], ned = g->e_off[g->n_orig_edges];
  int64_t* base = g->d_costs;
  CU(cudaMemcpyAsync(base + g->c_opm, op_m, sizeof(int64_t) * nop, cudaMemcpyHostToDevice, g->stream), "upload");
  CU(cudaMemcpyAsync(base + g->c_opt, op_t, sizeof(int64_t) * nop, cudaMemcpyHostToDevice, g->stream), "upload");
  if (edge_m)
    CU(cudaMemcpyAsync(base + g->c_em, edge_m, sizeof(int64_t) * ned, cudaMemcpyHostToDevice, g->stream), "upload");
  else
    CU(cudaMemsetAsync(base + g->c_em, 0, sizeof(int64_t) * ned, g->stream), "upload");
  CU(cudaMemcpyAsync(base + g->c_et, edge_t, sizeof(int64_t) * ned, cudaMemcpyHostToDevice, g->stream), "upload");
  // validation on the device: R10 bounds, and which edges carry m = 0 (Eq. 2)
  int32_t status = 0;
  std::vector<char> mz(g->n_orig_edges, 1);
  CU(ftk::validate_costs(base + g->c_opm, 2 * nop + 2 * ned, base + g->c_em, g->e_off, g->n_orig_edges,
                         &status, mz.data(), g->stream, g->alloc), "validate costs");
  if (status & 1) return setf(g, FT_EINVAL, "negative cost");
  if (status & 2) return setf(g, FT_EOVERFLOW, "cost >= 2^40");
  for (int i = 0; i < g->n_ops; ++i) g->op_ok[i] = 1;
  for (int e = 0; e < g->n_orig_edges; ++e) {
    g->e_ok[e] = 1;
    g->e_mzero[e] = mz[e];
  }
  g->bulk_done = true;
  return FT_OK;
}

int ft_eliminate(ft_graph* g, int32_t kind, int32_t id, int32_t* new_edge) {
  if (!g) return FT_EINVAL;
  if (g->poisoned) return g->poisoned;
  if (new_edge) *new_edge = -1;
  if (kind != FT_NODE && kind != FT_EDGE && kind != FT_AUTO && kind != FT_AUTO_HEUR)
    return setf(g, FT_EINVAL, "bad kind");
  if (g->have_final) return setf(g, FT_ESTATE, "frontier already computed");
  if (kind == FT_NODE) {
    if (id < 0 || id >= (int)g->K.size() || !g->op_alive[id]) return setf(g, FT_EINVAL, "bad operator");
    mark_backbone(g);
    if (g->mark_stamp[id] == g->stamp || g->in_e[id].size() != 1 || g->out_e[id].size() != 1)
      return setf(g, FT_EPRECOND, "node elimination needs an unmarked op with one in- and one out-edge");
    int rc = start(g);
    if (rc) return rc;
    rc = do_node(g, id, new_edge);
    return rc ? rc : flush(g);
  }
  if (kind == FT_EDGE) {
    if (id < 0 || id >= (int)g->edges.size() || !g->edges[id].alive) return setf(g, FT_EINVAL, "bad edge");
    int other = -1;
    for (int e : g->out_e[g->edges[id].src])
      if (e != id && g->edges[e].dst == g->edges[id].dst) {
        other = e;
        break;
      }
    if (other < 0) return setf(g, FT_EPRECOND, "edge elimination needs a parallel edge");
    int rc = start(g);
    if (rc) return rc;
    rc = do_merge(g, std::min(id, other), std::max(id, other), new_edge);
    return rc ? rc : flush(g);
  }
  int rc = start(g);
  if (rc) return rc;
  const double a0 = now_ms();
  // FT_AUTO: (a)-(e) until none applies.  FT_AUTO_HEUR (R17, R21): (a)-(d);
  // if the graph is not linear, one heuristic elimination, else (e); repeat.
  for (;;) {
    int r = auto_step(g, kind == FT_AUTO);
    if (r < 0) return r;
    if (r == 1) continue;
    if (kind != FT_AUTO_HEUR) break;
    std::vector<int> ch, ce;
    if (linear_chain(g, ch, ce) == FT_OK) break;  // linear: LDP can run
    g->err.clear();
    r = heur_step(g);
    if (r < 0) return r;
    if (r == 1) continue;
    mark_backbone(g);
    r = compose_step(g);
    if (r < 0) return r;
    if (r == 0) break;
  }
  g->hp[6] += now_ms() - a0;  // FT_AUTO policy (scheduling only)
  return flush(g);
}

int ft_frontier(ft_graph* g, int64_t cap, int64_t* m_out, int64_t* t_out, int64_t* n_out) {
  if (!g || !n_out) return FT_EINVAL;
  if (g->poisoned) return g->poisoned;
  int rc = start(g);
  if (rc) return rc;
  if (g->have_final && g->final_mode != 1) return setf(g, FT_ESTATE, "frontier computed by FT-Elimination");
  if (!g->have_final && (rc = run_ldp(g))) return rc;
  const int64_t n = (int64_t)g->final_m.size();
  *n_out = n;
  if (cap < n) return FT_ESIZE;
  if (m_out) std::memcpy(m_out, g->final_m.data(), sizeof(int64_t) * n);
  if (t_out) std::memcpy(t_out, g->final_t.data(), sizeof(int64_t) * n);
  return FT_OK;
}

int ft_frontier_elim(ft_graph* g, int64_t cap, int64_t* m_out, int64_t* t_out, int64_t* n_out) {
  if (!g || !n_out) return FT_EINVAL;
  if (g->poisoned) return g->poisoned;
  int rc = start(g);
  if (rc) return rc;
  if (g->have_final && g->final_mode != 2) return setf(g, FT_ESTATE, "frontier computed by LDP");
  if (!g->have_final && (rc = run_elim(g))) return rc;
  const int64_t n = (int64_t)g->final_m.size();
  *n_out = n;
  if (cap < n) return FT_ESIZE;
  if (m_out) std::memcpy(m_out, g->final_m.data(), sizeof(int64_t) * n);
  if (t_out) std::memcpy(t_out, g->final_t.data(), sizeof(int64_t) * n);
  return FT_OK;
}

int ft_query_mini_time(ft_graph* g, int64_t memory_limit, int64_t* idx_out) {
  if (!g || !idx_out) return FT_EINVAL;
  if (g->poisoned) return g->poisoned;
  if (!g->have_final) return setf(g, FT_ESTATE, "call ft_frontier first");
  // last index with m <= limit (m strictly ascending on the staircase)
  const auto& M = g->final_m;
  *idx_out = (int64_t)(std::upper_bound(M.begin(), M.end(), memory_limit) - M.begin()) - 1;
  return FT_OK;
}

int ft_strategy(ft_graph* g, int64_t tuple_idx, int32_t* cfg_out) {
  if (!g || !cfg_out) return FT_EINVAL;
  if (g->poisoned) return g->poisoned;
  if (!g->have_final) return setf(g, FT_ESTATE, "call ft_frontier first");
  if (tuple_idx < 0 || tuple_idx >= (int64_t)g->final_m.size()) return setf(g, FT_EINVAL, "bad tuple index");
  std::vector<int32_t> cfg(g->K.size(), -1);
  int rc = unroll(g, g->final_set, 0, tuple_idx, cfg);
  if (rc) return rc;
  for (int i = 0; i < g->n_ops; ++i)
    if (cfg[i] < 0) {
      g->poisoned = FT_EINTERNAL;
      return setf(g, FT_EINTERNAL, "broken provenance (operator without config)");
    }
  std::memcpy(cfg_out, cfg.data(), sizeof(int32_t) * g->n_ops);
  return FT_OK;
}

int ft_set_heuristic(ft_graph* g, int32_t policy, int64_t alpha_num, int64_t alpha_den) {
  if (!g) return FT_EINVAL;
  if (g->poisoned) return g->poisoned;
  if (policy != FT_HEUR_MIN_MEMORY && policy != FT_HEUR_WEIGHTED) return setf(g, FT_EINVAL, "bad policy");
  if (policy == FT_HEUR_WEIGHTED && (alpha_den < 1 || alpha_num < 0 || alpha_num > alpha_den))
    return setf(g, FT_EINVAL, "alpha must be in [0, 1]");
  g->heur_policy = policy;
  if (policy == FT_HEUR_WEIGHTED) {
    g->heur_num = alpha_num;
    g->heur_den = alpha_den;
  }
  return FT_OK;
}

int ft_prepare(ft_graph* g) {
  if (!g) return FT_EINVAL;
  if (g->poisoned) return g->poisoned;
  return start(g);
}

int ft_step_inputs(const ft_graph* g, int64_t step, int64_t* src6, int64_t* params6) {
  if (!g || !src6 || !params6) return FT_EINVAL;
  if (step < 0 || step >= (int64_t)g->steps.size()) return FT_EINVAL;
  const StepRec& r = g->steps[step];
  const int ids[3] = {r.X, r.Y, r.Z};
  for (int i = 0; i < 3; ++i) {
    const FSet& S = g->sets[ids[i]];
    src6[2 * i] = S.kind;
    if (S.kind == S_STEP) {
      src6[2 * i + 1] = S.step;
    } else if (S.kind == S_OP) {
      src6[2 * i + 1] = S.a_op;
    } else if (S.kind == S_EDGE) {
      int64_t e = -1;
      for (int q = 0; q < g->n_orig_edges; ++q)
        if (g->edges[q].set == ids[i]) e = q;
      src6[2 * i + 1] = e;
    } else {
      src6[2 * i + 1] = 0;
    }
  }
  params6[0] = r.kind;
  params6[1] = r.KA;
  params6[2] = r.KB;
  params6[3] = r.KC;
  params6[4] = r.nseg;
  params6[5] = r.nblk;
  return FT_OK;
}

int ft_nccl_unique_id(uint8_t id_out[128]) {
  if (!id_out) return FT_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return FT_ECUDA;
  std::memcpy(id_out, &id, sizeof(id) < 128 ? sizeof(id) : 128);
  return FT_OK;
}

int ft_nccl_comm_init(int32_t world, int32_t rank, const uint8_t id[128], int32_t device,
                      void** comm_out) {
  if (!id || !comm_out || world < 1 || rank < 0 || rank >= world) return FT_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return FT_ECUDA;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c;
  if (ncclCommInitRank(&c, world, uid, rank) != ncclSuccess) return FT_ECUDA;
  *comm_out = (void*)c;
  return FT_OK;
}

int ft_nccl_comm_destroy(void* comm) {
  if (!comm) return FT_EINVAL;
  return ncclCommDestroy((ncclComm_t)comm) == ncclSuccess ? FT_OK : FT_ECUDA;
}

int ft_get_stats(const ft_graph* g, ft_step_stats* buf, int64_t cap, int64_t* n_out) {
  if (!g || !n_out) return FT_EINVAL;
  *n_out = (int64_t)g->steps.size();
  if (cap < *n_out) return FT_ESIZE;
  for (size_t i = 0; i < g->steps.size(); ++i)
    if (buf) buf[i] = g->steps[i].st;
  if (buf)
    for (const auto& ev : g->comm_ev) {  // exchange time of each sharded wave (first step)
      float ms = 0;
      if (cudaEventSynchronize(ev.b) == cudaSuccess && cudaEventElapsedTime(&ms, ev.a, ev.b) == cudaSuccess)
        buf[ev.step].comm_ms = ms;
    }
  return FT_OK;
}

int ft_step_output(ft_graph* g, int64_t step, int64_t cap, int64_t* seg_off, int64_t* m, int64_t* t,
                   uint64_t* bp, int64_t* n_out) {
  if (!g || !n_out) return FT_EINVAL;
  if (g->poisoned) return g->poisoned;
  if (step < 0 || step >= (int64_t)g->steps.size()) return setf(g, FT_EINVAL, "bad step");
  int rc0 = ensure_off(g, g->steps[step].out);
  if (rc0) return rc0;
  FSet& S = g->sets[g->steps[step].out];
  const int64_t n = S.off[S.nseg];
  *n_out = n;
  if (cap < n) return FT_ESIZE;
  if (seg_off) std::memcpy(seg_off, S.off.data(), sizeof(int64_t) * (S.nseg + 1));
  if ((m || t) && (S.wave_buf < 0 || !g->waves[S.wave_buf].m))
    return setf(g, FT_ESTATE, "m/t of a consumed set (create with keep_all)");
  if (n) {
    if (m) CU(cudaMemcpyAsync(m, S.d_m, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, g->stream), "d2h");
    if (t) CU(cudaMemcpyAsync(t, S.d_t, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, g->stream), "d2h");
    if (bp) CU(cudaMemcpyAsync(bp, S.d_bp, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, g->stream), "d2h");
    CU(cudaStreamSynchronize(g->stream), "d2h");
  }
  return FT_OK;
}

const char* ft_last_error(const ft_graph* g) { return g ? g->err.c_str() : "null handle"; }

}  // extern "C"
