// oracle_ft.cpp -- plain, slow, obviously-correct CPU oracle of the FT hot path.
//
// TEST INFRASTRUCTURE ONLY (see oracle_ft.h).  Plain loops, std::sort and a
// linear sweep; no blocking, fusion or reordering beyond the paper's
// definitions.  Every function cites the passage it follows.
// P:n = /root/reference/PAPER.md line n; R<n> = DESIGN.md reading n.
#include "oracle_ft.h"

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstring>
#include <functional>
#include <map>
#include <new>
#include <queue>
#include <set>
#include <string>
#include <thread>
#include <vector>

namespace {

// A strategy tuple (S, m, t) of Def. 1.  S is represented by the
// provenance id (R6): the position of the tuple in the written product order
// of the step that produced it; unroll decodes it.
struct Tup {
  int64_t m;
  int64_t t;
  uint64_t id;
};
using Frontier = std::vector<Tup>;

// Alg. 1, with the sort key (m, t, id) of R1/R3: sort ascending,
// v = +inf, keep a tuple iff t < v, then v = t.
Frontier reduce(std::vector<Tup> C) {
  std::sort(C.begin(), C.end(), [](const Tup& a, const Tup& b) {
    if (a.m != b.m) return a.m < b.m;
    if (a.t != b.t) return a.t < b.t;
    return a.id < b.id;
  });
  Frontier F;
  int64_t v = INT64_MAX;  // +inf: all sums are < 2^60 (R10)
  for (const Tup& c : C) {
    if (c.t < v) {
      F.push_back(c);
      v = c.t;
    }
  }
  return F;
}

// A frontier set: one frontier per segment.  Segment layout: op set -> K_op
// segments (config s); edge set e_ij -> K_i*K_j segments, row-major [s_i][s_j];
// cumulative frontier CF(o_i, .) -> K_i segments.
enum SetKind { SET_UNIT = 0, SET_OP = 1, SET_EDGE = 2, SET_STEP = 3 };
struct FSet {
  int kind = SET_UNIT;
  int step = -1;        // producing step (SET_STEP)
  int a_op = -1;        // segment -> configs: op set: cfg(a_op) = seg
  int b_op = -1;        // edge set: cfg(a_op) = seg / K(b_op), cfg(b_op) = seg % K(b_op)
  std::vector<Frontier> seg;
};

// One step of the method.  Block (sigma, k) has factors X = sets[X][sx],
// Y = sets[Y][sy], Z = sets[Z][sz].
struct Step {
  int kind = 0;
  int out = -1, X = -1, Y = -1, Z = -1;
  int64_t KA = 0, KB = 0, KC = 0;  // kind-specific config counts
  int64_t nseg = 0, nblk = 0, tuples = 0, survivors = 0;
  double us = 0;
};

struct Edge {
  int src, dst;
  bool alive;
  int set;
};

}  // namespace

struct oft_graph {
  int n_ops = 0;       // operators so far: originals, then composites (R21)
  int n_orig_ops = 0;  // operators of the input graph
  int n_orig_edges = 0;
  int threads = 1;
  std::vector<int> K;
  std::vector<bool> op_alive;
  std::vector<int> op_set;       // current op frontier set per op
  std::vector<int> orig_op_set;  // original op set (for costs)
  std::vector<Edge> edges;       // original + created
  std::vector<FSet> sets;        // sets[0] = unit {(0,0)}
  std::vector<Step> steps;
  std::vector<bool> op_cost_set, edge_cost_set;
  std::vector<int> pos0;         // position in the live graph's topological order (R9, R21)
  std::vector<std::pair<int, int>> comp;  // composite op (R21): (o_h, o_i), config w = s_h*K_i + s_i
  bool started = false;
  bool have_final = false;
  int final_mode = 0;  // 1 = LDP (Alg. 3), 2 = FT-Elimination
  int final_set = -1;
  int heur_policy = 0;                 // R17 least memory, 1 = weighted (R22)
  int64_t heur_num = 1, heur_den = 2;  // alpha of the weighted rule
  std::string err;
};

namespace {

int fail(oft_graph* g, int code, const std::string& msg) {
  if (g) g->err = msg;
  return code;
}

int64_t seg_size(const oft_graph* g, int set, int64_t seg) {
  return (int64_t)g->sets[set].seg[seg].size();
}

// Factor segments of block k of output segment sigma (Eq.4, Eq.5, Eq.7, Alg.3).
void block_segs(const Step& s, int64_t sigma, int64_t k, int64_t* sx, int64_t* sy, int64_t* sz) {
  switch (s.kind) {
    case OFT_STEP_NODE: {  // Eq.4: sigma = w*K_j + p ; KA=K_h KB=K_i KC=K_j
      int64_t w = sigma / s.KC, p = sigma % s.KC;
      *sx = w * s.KB + k;  // F(e_hi, s_h^w, s_i^k)
      *sy = k;             // F(o_i, s_i^k)
      *sz = k * s.KC + p;  // F(e_ij, s_i^k, s_j^p)
      break;
    }
    case OFT_STEP_EDGE:  // Eq.5 P:600 (binary, R7)
      *sx = sigma; *sy = sigma; *sz = 0;
      break;
    case OFT_STEP_FOLD:  // Eq.7, source fixed to k* = KB: F(o_j,p) (x) F(e,k*,p) [(x) F(o_src,k*)]
      *sx = sigma; *sy = s.KB * s.KA + sigma; *sz = s.KC;  // K=1 fold: KB = KC = 0 (R13)
      break;
    case OFT_STEP_LDP: {  // Alg.3 line 6 P:645; KA=K_{i-1} KB=K_i
      int64_t p = sigma;
      *sx = k * s.KB + p;  // F(e_(i-1)i, s_{i-1}^k, s_i^p)
      *sy = k;             // CF(o_{i-1}, s_{i-1}^k)
      *sz = p;             // F(o_i, s_i^p)
      break;
    }
    case OFT_STEP_FINAL:  // Alg.3 line 9 P:648: reduce(U_s CF(o_n, s))
      *sx = k; *sy = 0; *sz = 0;
      break;
    case OFT_STEP_BRANCH: {  // Eq.6 P:606-613 (reading R14): sigma = s_h, k = s_i
      *sx = sigma;                                            // F(o_h, s_h)
      *sy = s.KC ? k * s.KA + sigma : sigma * s.KB + k;       // F(e, s_i, s_h) | F(e, s_h, s_i)
      *sz = k;                                                // F(o_i, s_i)
      break;
    }
    case OFT_STEP_COMPOSE: {  // Eq.6 P:609-613 (R21): sigma = w = s_h*K_i + s_i, one block
      const int64_t p = sigma / s.KB, k = sigma % s.KB;     // KA = K_h, KB = K_i
      *sx = p;                                              // F(o_h, s_h^p)
      *sy = k * s.KA + p;                                   // F(e_ih, s_i^k, s_h^p)
      *sz = k;                                              // F(o_i, s_i^k)
      break;
    }
    case OFT_STEP_REMAP: {  // R21: an edge of o_h or o_i re-indexed onto the composite o_v
      // KA = K_y (the other endpoint), KB = K_i, KC = side | part << 1: side 0 =
      // o_v is the new edge's source, 1 = its destination; part 0 = the old
      // endpoint was o_h (its config is w / K_i), 1 = o_i (w % K_i)
      const int64_t Kv = s.nseg / s.KA, side = s.KC & 1, part = s.KC >> 1;
      const int64_t Kold = part ? s.KB : Kv / s.KB;
      const int64_t w = side == 0 ? sigma / s.KA : sigma % Kv, y = side == 0 ? sigma % s.KA : sigma / Kv;
      const int64_t c = part ? w % s.KB : w / s.KB;
      *sx = side == 0 ? c * s.KA + y : y * Kold + c;
      *sy = 0;
      *sz = 0;
      break;
    }
    case OFT_STEP_PAIR:  // FT-Elimination P:628: k = s_1 * K_n + s_n over the 2-op graph
      *sx = k;             // F(e_1n, s_1, s_n)
      *sy = k / s.KB;      // F(o_1, s_1)
      *sz = k % s.KB;      // F(o_n, s_n)
      break;
    default:
      *sx = *sy = *sz = 0;
  }
}

// One output segment: Union over blocks k (concatenation) of the
// Product X_k (x) Y_k (x) Z_k in written (x, y, z) order; ids are
// positions (R6); then ONE reduce (R5).
Frontier segment(const oft_graph* g, const Step& s, int64_t sigma) {
  std::vector<Tup> C;
  uint64_t pos = 0;
  for (int64_t k = 0; k < s.nblk; ++k) {
    int64_t sx, sy, sz;
    block_segs(s, sigma, k, &sx, &sy, &sz);
    const Frontier& X = g->sets[s.X].seg[sx];
    const Frontier& Y = g->sets[s.Y].seg[sy];
    const Frontier& Z = g->sets[s.Z].seg[sz];
    for (size_t x = 0; x < X.size(); ++x)
      for (size_t y = 0; y < Y.size(); ++y)
        for (size_t z = 0; z < Z.size(); ++z) {
          C.push_back(Tup{X[x].m + Y[y].m + Z[z].m, X[x].t + Y[y].t + Z[z].t, pos});
          ++pos;
        }
  }
  return reduce(std::move(C));
}

// Runs a step: every output segment independently, statically
// partitioned over threads; results do not depend on the thread count.
int run_step(oft_graph* g, Step s) {
  auto t0 = std::chrono::steady_clock::now();
  FSet out;
  out.kind = SET_STEP;
  out.step = (int)g->steps.size();
  out.seg.resize(s.nseg);
  int T = std::max(1, g->threads);
  if (s.nseg < T) T = (int)std::max<int64_t>(1, s.nseg);
  try {
    if (T == 1) {
      for (int64_t sg = 0; sg < s.nseg; ++sg) out.seg[sg] = segment(g, s, sg);
    } else {
      std::vector<std::thread> th;
      for (int w = 0; w < T; ++w)
        th.emplace_back([&, w]() {
          for (int64_t sg = w; sg < s.nseg; sg += T) out.seg[sg] = segment(g, s, sg);
        });
      for (auto& x : th) x.join();
    }
  } catch (const std::bad_alloc&) {
    return fail(g, OFT_ENOMEM, "out of host memory");
  }
  s.tuples = 0;
  for (int64_t sg = 0; sg < s.nseg; ++sg)
    for (int64_t k = 0; k < s.nblk; ++k) {
      int64_t sx, sy, sz;
      block_segs(s, sg, k, &sx, &sy, &sz);
      s.tuples += seg_size(g, s.X, sx) * seg_size(g, s.Y, sy) * seg_size(g, s.Z, sz);
    }
  s.survivors = 0;
  for (auto& f : out.seg) s.survivors += (int64_t)f.size();
  s.us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  s.out = (int)g->sets.size();
  g->sets.push_back(std::move(out));
  g->steps.push_back(s);
  return OFT_OK;
}

// ---- graph helpers ---------------------------------------------------------

// Live adjacency, rebuilt per elimination (plain O(E)).
struct Adj {
  std::vector<std::vector<int>> in, out;  // live edge ids, ascending
};
Adj build_adj(const oft_graph* g) {
  Adj a;
  a.in.resize(g->n_ops);
  a.out.resize(g->n_ops);
  for (size_t e = 0; e < g->edges.size(); ++e)
    if (g->edges[e].alive) {
      a.out[g->edges[e].src].push_back((int)e);
      a.in[g->edges[e].dst].push_back((int)e);
    }
  return a;
}

// Kahn's topological order with the smallest op id first; computed once on
// the original graph (graph creation).
std::vector<int> topo_order(const oft_graph* g, const Adj& a) {
  std::vector<int> indeg(g->n_ops, 0);
  for (int i = 0; i < g->n_ops; ++i) indeg[i] = (int)a.in[i].size();
  std::priority_queue<int, std::vector<int>, std::greater<int>> q;
  for (int i = 0; i < g->n_ops; ++i)
    if (g->op_alive[i] && indeg[i] == 0) q.push(i);
  std::vector<int> order;
  while (!q.empty()) {
    int u = q.top();
    q.pop();
    order.push_back(u);
    for (int e : a.out[u])
      if (--indeg[g->edges[e].dst] == 0) q.push(g->edges[e].dst);
  }
  return order;
}

// Topological order of the live graph (R9): the original graph's order
// restricted to live operators (eliminations only remove operators and
// replace paths h->i->j by h->j, so it stays a topological order).
std::vector<int> live_order(const oft_graph* g) {
  std::vector<int> order;
  for (int i = 0; i < g->n_ops; ++i)
    if (g->op_alive[i]) order.push_back(i);
  std::sort(order.begin(), order.end(), [g](int a, int b) { return g->pos0[a] < g->pos0[b]; });
  return order;
}

// Marking: mark the topologically first op; while the last marked
// op has exactly one downstream operator, mark it.
std::vector<bool> marking(const oft_graph* g, const Adj& a, const std::vector<int>& topo) {
  std::vector<bool> marked(g->n_ops, false);
  if (topo.empty()) return marked;
  int cur = topo[0];
  marked[cur] = true;
  for (;;) {
    std::set<int> down;
    for (int e : a.out[cur]) down.insert(g->edges[e].dst);
    if (down.size() != 1) break;
    int nxt = *down.begin();
    if (marked[nxt]) break;
    marked[nxt] = true;
    cur = nxt;
  }
  return marked;
}

int new_edge(oft_graph* g, int src, int dst, int set) {
  g->edges.push_back(Edge{src, dst, true, set});
  return (int)g->edges.size() - 1;
}

// Eq. 4: node elimination of o_i.
int do_node(oft_graph* g, const Adj& a, int i, int* out_edge) {
  int ehi = a.in[i][0], eij = a.out[i][0];
  int h = g->edges[ehi].src, j = g->edges[eij].dst;
  Step s;
  s.kind = OFT_STEP_NODE;
  s.X = g->edges[ehi].set;
  s.Y = g->op_set[i];
  s.Z = g->edges[eij].set;
  s.KA = g->K[h]; s.KB = g->K[i]; s.KC = g->K[j];
  s.nseg = s.KA * s.KC;
  s.nblk = s.KB;
  int rc = run_step(g, s);
  if (rc) return rc;
  int so = g->steps.back().out;
  g->sets[so].a_op = h;
  g->sets[so].b_op = j;
  g->edges[ehi].alive = false;
  g->edges[eij].alive = false;
  g->op_alive[i] = false;
  int e = new_edge(g, h, j, so);
  if (out_edge) *out_edge = e;
  return OFT_OK;
}

// Eq. 5, binary merge e1 < e2 (R7).
int do_edge(oft_graph* g, int e1, int e2, int* out_edge) {
  Step s;
  s.kind = OFT_STEP_EDGE;
  s.X = g->edges[e1].set;
  s.Y = g->edges[e2].set;
  s.Z = 0;
  int a = g->edges[e1].src, b = g->edges[e1].dst;
  s.KA = g->K[a]; s.KB = g->K[b];
  s.nseg = s.KA * s.KB;
  s.nblk = 1;
  int rc = run_step(g, s);
  if (rc) return rc;
  int so = g->steps.back().out;
  g->sets[so].a_op = a;
  g->sets[so].b_op = b;
  g->edges[e1].alive = false;
  g->edges[e2].alive = false;
  int e = new_edge(g, a, b, so);
  if (out_edge) *out_edge = e;
  return OFT_OK;
}

// Eq. 7 for a K=1 source (exact, R13): every consumer o_j gets
// F(o_j, p) <- F(o_j, p) (x) F(e, 0, p); the source's own cost is added once,
// to its topologically first consumer.
int do_fold(oft_graph* g, const Adj& a, int src, const std::vector<int>& topo, int64_t kstar = 0) {
  const std::vector<int> out = a.out[src];
  std::vector<int> pos(g->n_ops, 0);
  for (size_t i = 0; i < topo.size(); ++i) pos[topo[i]] = (int)i;
  int first = -1;
  for (int e : out) {
    int c = g->edges[e].dst;
    if (first < 0 || pos[c] < pos[first] || (pos[c] == pos[first] && c < first)) first = c;
  }
  for (int e : out) {  // ascending edge id
    int c = g->edges[e].dst;
    Step s;
    s.kind = OFT_STEP_FOLD;
    s.X = g->op_set[c];
    s.Y = g->edges[e].set;
    s.Z = (c == first) ? g->op_set[src] : 0;
    s.KA = g->K[c];
    s.KB = kstar;                      // edge segment k* * K_c + p
    s.KC = (c == first) ? kstar : 0;   // op segment k* (unit set: 0)
    s.nseg = g->K[c];
    s.nblk = 1;
    int rc = run_step(g, s);
    if (rc) return rc;
    int so = g->steps.back().out;
    g->sets[so].a_op = c;
    g->op_set[c] = so;
    g->edges[e].alive = false;
  }
  g->op_alive[src] = false;
  return OFT_OK;
}

// Eq. 6, reading R14: o_i's only remaining edge is e (to or from
// o_h), so it is merged into o_h.  The paper keeps composite configurations
// (s_h, s_i); since o_i reaches the rest of the graph only through e, the
// union over s_i is reduced at once -- the same (m, t) frontier:
//   F(o_h, s_h) <- reduce(U_{s_i} F(o_h, s_h) (x) F(e, .) (x) F(o_i, s_i)).
int do_branch(oft_graph* g, const Adj& a, int i) {
  const bool src = a.in[i].empty();  // o_i -> o_h, else o_h -> o_i
  const int e = src ? a.out[i][0] : a.in[i][0];
  const int h = src ? g->edges[e].dst : g->edges[e].src;
  Step s;
  s.kind = OFT_STEP_BRANCH;
  s.X = g->op_set[h];
  s.Y = g->edges[e].set;
  s.Z = g->op_set[i];
  s.KA = g->K[h];
  s.KB = g->K[i];
  s.KC = src ? 1 : 0;
  s.nseg = g->K[h];
  s.nblk = g->K[i];
  int rc = run_step(g, s);
  if (rc) return rc;
  int so = g->steps.back().out;
  g->sets[so].a_op = h;
  g->op_set[h] = so;
  g->edges[e].alive = false;
  g->op_alive[i] = false;
  return OFT_OK;
}

// Eq. 6 with composite configurations (reading R21): o_i feeds o_h
// through the single edge e and keeps other edges, so nothing can be reduced
// over s_i; o_i and o_h are replaced by one operator o_v whose configurations
// are the pairs w = (s_h, s_i) (w = s_h * K_i + s_i):
//   F(o_v, w) = reduce(F(o_h, s_h) (x) F(e, s_i, s_h) (x) F(o_i, s_i))
// and every other edge of o_h or o_i is re-indexed onto o_v (F(e', w, .) =
// F(e', s_h or s_i, .)).  The live graph's topological order is recomputed
// (Kahn's algorithm, ready ops by (previous position, id); o_v takes o_h's).
void reorder(oft_graph* g) {
  Adj a = build_adj(g);
  std::vector<int> indeg(g->n_ops, 0);
  std::set<std::pair<int, int>> ready;
  for (int i = 0; i < g->n_ops; ++i)
    if (g->op_alive[i]) {
      indeg[i] = (int)a.in[i].size();
      if (indeg[i] == 0) ready.insert({g->pos0[i], i});
    }
  int pos = 0;
  std::vector<int> np(g->n_ops, INT_MAX);
  while (!ready.empty()) {
    int u = ready.begin()->second;
    ready.erase(ready.begin());
    np[u] = pos++;
    for (int e : a.out[u]) {
      int d = g->edges[e].dst;
      if (--indeg[d] == 0) ready.insert({g->pos0[d], d});
    }
  }
  for (int i = 0; i < g->n_ops; ++i)
    if (g->op_alive[i]) g->pos0[i] = np[i];
}

// Is there a path o_i -> ... -> o_h other than the direct edges?  (Merging
// o_i into o_h would then close a cycle.)
bool other_path(const oft_graph* g, const Adj& a, int i, int h) {
  std::vector<char> seen(g->n_ops, 0);
  std::vector<int> st;
  for (int e : a.out[i])
    if (g->edges[e].dst != h) st.push_back(g->edges[e].dst);
  while (!st.empty()) {
    int u = st.back();
    st.pop_back();
    if (u == h) return true;
    if (seen[u]) continue;
    seen[u] = 1;
    for (int e : a.out[u]) st.push_back(g->edges[e].dst);
  }
  return false;
}

int do_compose(oft_graph* g, const Adj& a, int i, int h) {
  int e = -1;
  for (int x : a.in[h])
    if (g->edges[x].src == i) e = x;
  const int v = g->n_ops;
  g->n_ops++;
  g->K.push_back(g->K[h] * g->K[i]);
  g->op_alive.push_back(true);
  g->pos0.push_back(g->pos0[h]);
  g->comp.resize(g->n_ops, {-1, -1});
  g->comp[v] = {h, i};
  Step s;
  s.kind = OFT_STEP_COMPOSE;
  s.X = g->op_set[h];
  s.Y = g->edges[e].set;
  s.Z = g->op_set[i];
  s.KA = g->K[h];
  s.KB = g->K[i];
  s.nseg = g->K[v];
  s.nblk = 1;
  int rc = run_step(g, s);
  if (rc) return rc;
  g->op_set.push_back(g->steps.back().out);
  g->sets[g->steps.back().out].a_op = v;
  g->edges[e].alive = false;
  // the other edges of o_h and o_i, ascending edge id
  std::set<int> others;
  for (int o : {h, i}) {
    for (int x : a.in[o]) others.insert(x);
    for (int x : a.out[o]) others.insert(x);
  }
  others.erase(e);
  for (int x : others) {
    const int src = g->edges[x].src, dst = g->edges[x].dst;
    const int old = (src == h || src == i) ? src : dst;
    const int y = old == src ? dst : src;
    Step r;
    r.kind = OFT_STEP_REMAP;
    r.X = g->edges[x].set;
    r.Y = 0;
    r.Z = 0;
    r.KA = g->K[y];
    r.KB = g->K[i];
    r.KC = (old == src ? 0 : 1) | (old == i ? 2 : 0);
    r.nseg = (int64_t)g->K[v] * g->K[y];
    r.nblk = 1;
    if ((rc = run_step(g, r))) return rc;
    const int so = g->steps.back().out;
    const int ns = old == src ? v : y, nd = old == src ? y : v;
    g->sets[so].a_op = ns;
    g->sets[so].b_op = nd;
    g->edges[x].alive = false;
    new_edge(g, ns, nd, so);
  }
  g->op_alive[h] = false;
  g->op_alive[i] = false;
  reorder(g);
  return OFT_OK;
}

// Composite branch elimination candidate (R21): the topologically first
// operator o_h with >= 2 input operators that has an unmarked input o_i with
// K_h * K_i <= 4096, no other path o_i -> o_h, and that is not a source
// feeding >= 2 operators (a broadcast input like BERT's attention mask,
// which P:618-620 leaves to heuristic elimination); among its inputs the one
// with the smallest K_i (SPEC: "the input operator with the smaller config
// space"), ties by topological position.  Returns (i, h) or (-1, -1).
std::pair<int, int> compose_candidate(const oft_graph* g, const Adj& a, const std::vector<int>& topo,
                                      const std::vector<bool>& marked) {
  for (int h : topo) {
    std::set<std::pair<int, int>> ins;  // (position, op)
    for (int e : a.in[h]) ins.insert({g->pos0[g->edges[e].src], g->edges[e].src});
    if (ins.size() < 2) continue;
    int best = -1;
    for (auto& pi : ins) {
      const int i = pi.second;
      if (marked[i] || (int64_t)g->K[h] * g->K[i] > 4096 || other_path(g, a, i, h)) continue;
      if (a.in[i].empty()) {  // a source: not if it feeds several operators
        std::set<int> outs;
        for (int e : a.out[i]) outs.insert(g->edges[e].dst);
        if (outs.size() >= 2) continue;
      }
      if (best < 0 || g->K[i] < g->K[best]) best = i;
    }
    if (best >= 0) return {best, h};
  }
  return {-1, -1};
}

int check_started(oft_graph* g) {
  if (g->started) return OFT_OK;
  for (int i = 0; i < g->n_orig_ops; ++i)
    if (!g->op_cost_set[i]) return fail(g, OFT_ESTATE, "missing op costs");
  for (int e = 0; e < g->n_orig_edges; ++e)
    if (!g->edge_cost_set[e]) return fail(g, OFT_ESTATE, "missing edge costs");
  g->started = true;
  return OFT_OK;
}

bool node_eligible(const oft_graph* g, const Adj& a, int i, const std::vector<bool>& marked) {
  if (!g->op_alive[i] || marked[i]) return false;
  return a.in[i].size() == 1 && a.out[i].size() == 1;
}

// FT_AUTO policy (R9; Alg. 2 lines 4-11): one elimination.
// Returns 1 if something was eliminated, 0 if none applies, <0 on error.
// compose = false skips (e) (FT_AUTO_HEUR tries heuristic elimination first).
int auto_one(oft_graph* g, bool compose) {
  Adj a = build_adj(g);
  auto topo = live_order(g);
  auto marked = marking(g, a, topo);  // Alg.2 line 5
  std::vector<int> pos(g->n_ops, INT_MAX);
  for (size_t i = 0; i < topo.size(); ++i) pos[topo[i]] = (int)i;
  // (a) parallel edges: topologically-first (src, dst) pair, two lowest ids.
  std::map<std::pair<int, int>, std::vector<int>> pairs;
  for (size_t e = 0; e < g->edges.size(); ++e)
    if (g->edges[e].alive) pairs[{g->edges[e].src, g->edges[e].dst}].push_back((int)e);
  int be1 = -1, be2 = -1;
  std::pair<int, int> best{INT_MAX, INT_MAX};
  for (auto& kv : pairs) {
    if (kv.second.size() < 2) continue;
    std::pair<int, int> key{pos[kv.first.first], pos[kv.first.second]};
    if (key < best) {
      best = key;
      be1 = kv.second[0];
      be2 = kv.second[1];
    }
  }
  if (be1 >= 0) {
    int rc = do_edge(g, be1, be2, nullptr);
    return rc ? rc : 1;
  }
  // (b) node elimination: topologically-first unmarked op, 1 in-edge, 1 out-edge.
  for (int i : topo)
    if (node_eligible(g, a, i, marked)) {
      int rc = do_node(g, a, i, nullptr);
      return rc ? rc : 1;
    }
  // (c) fold a K=1 source (exact Eq. 7).
  for (int i : topo)
    if (g->op_alive[i] && g->K[i] == 1 && a.in[i].empty() && !a.out[i].empty()) {
      int rc = do_fold(g, a, i, topo);
      return rc ? rc : 1;
    }
  // (d) branch elimination (Eq. 6): topologically-first unmarked op whose
  //     only edge connects it to one neighbour (after the K=1 fold, which keeps
  //     the backbone intact: DESIGN.md R14).
  for (int i : topo)
    if (g->op_alive[i] && !marked[i] && a.in[i].size() + a.out[i].size() == 1) {
      int rc = do_branch(g, a, i);
      return rc ? rc : 1;
    }
  // (e) branch elimination with composite configurations (Eq. 6, R21)
  if (!compose) return 0;
  const auto ih = compose_candidate(g, a, topo, marked);
  if (ih.first >= 0) {
    int rc = do_compose(g, a, ih.first, ih.second);
    return rc ? rc : 1;
  }
  return 0;
}

// (e) alone: one composite branch elimination (R21), 1 = done, 0 = none.
int compose_one(oft_graph* g) {
  Adj a = build_adj(g);
  auto topo = live_order(g);
  auto marked = marking(g, a, topo);
  const auto ih = compose_candidate(g, a, topo, marked);
  if (ih.first < 0) return 0;
  int rc = do_compose(g, a, ih.first, ih.second);
  return rc ? rc : 1;
}

// Heuristic elimination (Eq. 7; lossy, opt-in): the unmarked
// source op with the most out-edges (ties: topological order), K >= 2, gets
// the configuration of least memory -- min over k of the first (least-m)
// tuple of F(o_i, k), ties by its t, then k ("minimizing the memory
// consumption of o_i") -- and is folded into its consumers.  1 = done, 0 =
// no candidate.
int heur_one(oft_graph* g) {
  Adj a = build_adj(g);
  auto topo = live_order(g);
  auto marked = marking(g, a, topo);
  int best = -1;
  for (int i : topo)
    if (g->op_alive[i] && !marked[i] && g->K[i] >= 2 && a.in[i].empty() && !a.out[i].empty() &&
        (best < 0 || a.out[i].size() > a.out[best].size()))
      best = i;
  if (best < 0) return 0;
  const FSet& S = g->sets[g->op_set[best]];
  int64_t ks = 0;
  if (g->heur_policy == 0) {
    for (int64_t k = 1; k < (int64_t)S.seg.size(); ++k) {
      const Tup &x = S.seg[k][0], &y = S.seg[ks][0];
      if (x.m < y.m || (x.m == y.m && x.t < y.t)) ks = k;
    }
  } else {
    // R22 ("a weighted combination of different objectives"): every
    // tuple x of F(o_i, k) scores alpha * m_x / M + (1 - alpha) * t_x / T in
    // IEEE double (M, T = largest m, t over F(o_i, .), at least 1; each
    // operation rounded separately); the config of the least score wins,
    // ties by (m, t) of its tuple, then k.
    int64_t M = 1, T = 1;
    for (const auto& f : S.seg)
      for (const Tup& x : f) {
        M = std::max(M, x.m);
        T = std::max(T, x.t);
      }
    const double al = (double)g->heur_num / (double)g->heur_den;
    bool have = false;
    double bs = 0;
    int64_t bm = 0, bt = 0;
    for (int64_t k = 0; k < (int64_t)S.seg.size(); ++k)
      for (const Tup& x : S.seg[k]) {
        const double dm = (double)x.m / (double)M, dt = (double)x.t / (double)T;
        const double sc = al * dm + (1.0 - al) * dt;
        if (!have || sc < bs || (sc == bs && (x.m < bm || (x.m == bm && x.t < bt)))) {
          have = true;
          bs = sc;
          bm = x.m;
          bt = x.t;
          ks = k;
        }
      }
  }
  int rc = do_fold(g, a, best, topo, ks);
  return rc ? rc : 1;
}

// The live graph as a chain o_1 -> ... -> o_n (LDP precondition).
int chain_of(oft_graph* g, std::vector<int>* chain, std::vector<int>* chain_edges) {
  Adj a = build_adj(g);
  std::vector<int> live;
  for (int i = 0; i < g->n_ops; ++i)
    if (g->op_alive[i]) live.push_back(i);
  int start = -1;
  for (int i : live)
    if (a.in[i].empty()) {
      if (start >= 0) return fail(g, OFT_EPRECOND, "not linear: several sources");
      start = i;
    }
  if (start < 0) return fail(g, OFT_EPRECOND, "not linear: no source");
  int cur = start;
  chain->push_back(cur);
  for (;;) {
    const auto& out = a.out[cur];
    if (out.empty()) break;
    if (out.size() != 1) return fail(g, OFT_EPRECOND, "not linear: op with several out-edges");
    int nx = g->edges[out[0]].dst;
    if (a.in[nx].size() != 1) return fail(g, OFT_EPRECOND, "not linear: op with several in-edges");
    chain_edges->push_back(out[0]);
    chain->push_back(nx);
    cur = nx;
  }
  if (chain->size() != live.size()) return fail(g, OFT_EPRECOND, "not linear: disconnected ops");
  return OFT_OK;
}

// Alg. 3.
int run_ldp(oft_graph* g) {
  std::vector<int> chain, ce;
  int rc = chain_of(g, &chain, &ce);
  if (rc) return rc;
  int cf = g->op_set[chain[0]];  // line 3: CF(o_1, s) = F(o_1, s)
  for (size_t i = 1; i < chain.size(); ++i) {  // lines 4-8
    Step s;
    s.kind = OFT_STEP_LDP;
    s.X = g->edges[ce[i - 1]].set;
    s.Y = cf;
    s.Z = g->op_set[chain[i]];
    s.KA = g->K[chain[i - 1]];
    s.KB = g->K[chain[i]];
    s.nseg = s.KB;
    s.nblk = s.KA;
    rc = run_step(g, s);
    if (rc) return rc;
    cf = g->steps.back().out;
    g->sets[cf].a_op = chain[i];
  }
  Step f;  // line 9
  f.kind = OFT_STEP_FINAL;
  f.X = cf;
  f.Y = 0;
  f.Z = 0;
  f.KA = g->K[chain.back()];
  f.nseg = 1;
  f.nblk = f.KA;
  rc = run_step(g, f);
  if (rc) return rc;
  g->final_set = g->steps.back().out;
  g->have_final = true;
  g->final_mode = 1;
  return OFT_OK;
}

// FT-Elimination (Theorem 2): on the linear graph,
// node-eliminate (Eq.4) the second op of the remaining chain until only
// o_1 and o_n are left, then find the frontier of the two-op graph by
// enumerating every configuration pair: reduce(U_{s_1,s_n} F(e_1n,s_1,s_n)
// (x) F(o_1,s_1) (x) F(o_n,s_n)).  One op: reduce(U_s F(o_1, s)).
int run_elim(oft_graph* g) {
  std::vector<int> chain, ce;
  int rc = chain_of(g, &chain, &ce);
  if (rc) return rc;
  for (size_t i = 1; i + 1 < chain.size(); ++i) {
    Adj a = build_adj(g);
    if ((rc = do_node(g, a, chain[i], nullptr))) return rc;
  }
  Step f;
  if (chain.size() == 1) {
    f.kind = OFT_STEP_FINAL;
    f.X = g->op_set[chain[0]];
    f.Y = 0;
    f.Z = 0;
    f.KA = g->K[chain[0]];
    f.nblk = f.KA;
  } else {
    Adj a = build_adj(g);
    f.kind = OFT_STEP_PAIR;
    f.X = g->edges[a.out[chain[0]][0]].set;
    f.Y = g->op_set[chain[0]];
    f.Z = g->op_set[chain.back()];
    f.KA = g->K[chain[0]];
    f.KB = g->K[chain.back()];
    f.nblk = f.KA * f.KB;
  }
  f.nseg = 1;
  rc = run_step(g, f);
  if (rc) return rc;
  g->final_set = g->steps.back().out;
  g->have_final = true;
  g->final_mode = 2;
  return OFT_OK;
}

// Unroll: walk provenance ids back to original op/edge costs.
int assign(oft_graph* g, std::vector<int32_t>& cfg, int op, int64_t c) {
  if (op < 0) return OFT_OK;
  if (cfg[op] >= 0 && cfg[op] != c) return fail(g, OFT_EINTERNAL, "broken provenance: config conflict");
  cfg[op] = (int32_t)c;
  if (op < (int)g->comp.size() && g->comp[op].first >= 0) {  // composite (R21): w = s_h * K_i + s_i
    const int h = g->comp[op].first, i = g->comp[op].second;
    int rc = assign(g, cfg, h, c / g->K[i]);
    return rc ? rc : assign(g, cfg, i, c % g->K[i]);
  }
  return OFT_OK;
}

int visit(oft_graph* g, std::vector<int32_t>& cfg, int set, int64_t seg, int64_t idx) {
  const FSet& S = g->sets[set];
  if (S.kind == SET_UNIT) return OFT_OK;
  int rc;
  if (S.b_op >= 0) {
    int64_t kb = g->K[S.b_op];
    if ((rc = assign(g, cfg, S.a_op, seg / kb))) return rc;
    if ((rc = assign(g, cfg, S.b_op, seg % kb))) return rc;
  } else if ((rc = assign(g, cfg, S.a_op, seg))) {
    return rc;
  }
  if (S.kind != SET_STEP) return OFT_OK;
  const Step& s = g->steps[S.step];
  uint64_t id = S.seg[seg][idx].id;
  uint64_t start = 0;
  for (int64_t k = 0; k < s.nblk; ++k) {
    int64_t sx, sy, sz;
    block_segs(s, seg, k, &sx, &sy, &sz);
    uint64_t nx = seg_size(g, s.X, sx), ny = seg_size(g, s.Y, sy), nz = seg_size(g, s.Z, sz);
    uint64_t n = nx * ny * nz;
    if (id < start + n) {
      uint64_t r = id - start;
      uint64_t z = r % nz, y = (r / nz) % ny, x = r / (ny * nz);
      if ((rc = visit(g, cfg, s.X, sx, (int64_t)x))) return rc;
      if ((rc = visit(g, cfg, s.Y, sy, (int64_t)y))) return rc;
      return visit(g, cfg, s.Z, sz, (int64_t)z);
    }
    start += n;
  }
  return fail(g, OFT_EINTERNAL, "broken provenance: id out of range");
}

}  // namespace

extern "C" {

int oft_graph_create(int32_t n_ops, const int32_t* n_cfgs, int32_t n_edges, const int32_t* src,
                     const int32_t* dst, int32_t threads, oft_graph** out) {
  if (!out) return OFT_EINVAL;
  *out = nullptr;
  if (n_ops < 1 || n_edges < 0 || !n_cfgs || (n_edges > 0 && (!src || !dst))) return OFT_EINVAL;
  if ((int64_t)n_ops + n_edges >= (1 << 20)) return OFT_EOVERFLOW;  // R10
  for (int i = 0; i < n_ops; ++i)
    if (n_cfgs[i] < 1 || n_cfgs[i] > 4096) return OFT_EINVAL;
  for (int e = 0; e < n_edges; ++e)
    if (src[e] < 0 || src[e] >= n_ops || dst[e] < 0 || dst[e] >= n_ops || src[e] == dst[e])
      return OFT_EINVAL;
  oft_graph* g = new (std::nothrow) oft_graph();
  if (!g) return OFT_ENOMEM;
  g->n_ops = n_ops;
  g->n_orig_ops = n_ops;
  g->comp.assign(n_ops, {-1, -1});
  g->n_orig_edges = n_edges;
  g->threads = threads < 1 ? 1 : threads;
  g->K.assign(n_cfgs, n_cfgs + n_ops);
  g->op_alive.assign(n_ops, true);
  g->op_cost_set.assign(n_ops, false);
  g->edge_cost_set.assign(n_edges, false);
  FSet unit;
  unit.kind = SET_UNIT;
  unit.seg.push_back(Frontier{Tup{0, 0, 0}});
  g->sets.push_back(unit);
  for (int i = 0; i < n_ops; ++i) {
    FSet s;
    s.kind = SET_OP;
    s.a_op = i;
    s.seg.resize(g->K[i]);
    g->op_set.push_back((int)g->sets.size());
    g->sets.push_back(s);
  }
  g->orig_op_set = g->op_set;
  for (int e = 0; e < n_edges; ++e) {
    FSet s;
    s.kind = SET_EDGE;
    s.a_op = src[e];
    s.b_op = dst[e];
    s.seg.resize((size_t)g->K[src[e]] * g->K[dst[e]]);
    g->edges.push_back(Edge{src[e], dst[e], true, (int)g->sets.size()});
    g->sets.push_back(s);
  }
  {
    auto order = topo_order(g, build_adj(g));
    if (order.size() != (size_t)n_ops) {
      delete g;
      return OFT_EINVAL;  // cycle
    }
    g->pos0.assign(n_ops, 0);
    for (int i = 0; i < n_ops; ++i) g->pos0[order[i]] = i;
  }
  *out = g;
  return OFT_OK;
}

void oft_graph_destroy(oft_graph* g) { delete g; }

int oft_set_op_costs(oft_graph* g, int32_t op, const int64_t* m, const int64_t* t) {
  if (!g) return OFT_EINVAL;
  if (g->started) return fail(g, OFT_ESTATE, "costs set after elimination began");
  if (op < 0 || op >= g->n_orig_ops || !m || !t) return fail(g, OFT_EINVAL, "bad op");
  for (int k = 0; k < g->K[op]; ++k) {
    if (m[k] < 0 || t[k] < 0) return fail(g, OFT_EINVAL, "negative cost");
    if (m[k] >= (int64_t(1) << 40) || t[k] >= (int64_t(1) << 40)) return fail(g, OFT_EOVERFLOW, "cost >= 2^40");
  }
  FSet& s = g->sets[g->orig_op_set[op]];
  for (int k = 0; k < g->K[op]; ++k) s.seg[k] = Frontier{Tup{m[k], t[k], 0}};  // F(o_i, s) init
  g->op_cost_set[op] = true;
  return OFT_OK;
}

int oft_set_edge_costs(oft_graph* g, int32_t edge, const int64_t* m, const int64_t* t) {
  if (!g) return OFT_EINVAL;
  if (g->started) return fail(g, OFT_ESTATE, "costs set after elimination began");
  if (edge < 0 || edge >= g->n_orig_edges || !t) return fail(g, OFT_EINVAL, "bad edge");
  int64_t n = (int64_t)g->K[g->edges[edge].src] * g->K[g->edges[edge].dst];
  for (int64_t k = 0; k < n; ++k) {
    int64_t mm = m ? m[k] : 0;
    if (mm < 0 || t[k] < 0) return fail(g, OFT_EINVAL, "negative cost");
    if (mm >= (int64_t(1) << 40) || t[k] >= (int64_t(1) << 40)) return fail(g, OFT_EOVERFLOW, "cost >= 2^40");
  }
  FSet& s = g->sets[g->edges[edge].set];
  for (int64_t k = 0; k < n; ++k) s.seg[k] = Frontier{Tup{m ? m[k] : 0, t[k], 0}};  // Eq.2
  g->edge_cost_set[edge] = true;
  return OFT_OK;
}

int oft_eliminate(oft_graph* g, int32_t kind, int32_t id, int32_t* out_edge) {
  if (!g) return OFT_EINVAL;
  if (out_edge) *out_edge = -1;
  int rc = check_started(g);
  if (rc) return rc;
  if (g->have_final) return fail(g, OFT_ESTATE, "frontier already computed");
  if (kind == OFT_NODE) {
    if (id < 0 || id >= g->n_ops || !g->op_alive[id]) return fail(g, OFT_EINVAL, "bad op");
    Adj a = build_adj(g);
    auto topo = live_order(g);
    auto marked = marking(g, a, topo);
    if (!node_eligible(g, a, id, marked)) return fail(g, OFT_EPRECOND, "node elimination precondition");
    return do_node(g, a, id, out_edge);
  }
  if (kind == OFT_EDGE) {
    if (id < 0 || id >= (int)g->edges.size() || !g->edges[id].alive) return fail(g, OFT_EINVAL, "bad edge");
    int other = -1;
    for (size_t e = 0; e < g->edges.size(); ++e)
      if ((int)e != id && g->edges[e].alive && g->edges[e].src == g->edges[id].src &&
          g->edges[e].dst == g->edges[id].dst) {
        other = (int)e;
        break;
      }
    if (other < 0) return fail(g, OFT_EPRECOND, "edge elimination needs a parallel edge");
    return do_edge(g, std::min(id, other), std::max(id, other), out_edge);
  }
  if (kind == OFT_AUTO || kind == OFT_AUTO_HEUR) {
    // FT_AUTO: (a)-(e) until none applies.  FT_AUTO_HEUR (R17, R21): (a)-(d);
    // if the graph is not linear, one heuristic elimination, else (e); repeat.
    for (;;) {
      int r = auto_one(g, kind == OFT_AUTO);
      if (r < 0) return r;
      if (r == 1) continue;
      if (kind == OFT_AUTO) break;
      std::vector<int> ch, ce;
      if (chain_of(g, &ch, &ce) == OFT_OK) break;  // linear: LDP can run
      g->err.clear();
      r = heur_one(g);
      if (r < 0) return r;
      if (r == 1) continue;
      r = compose_one(g);
      if (r < 0) return r;
      if (r == 0) break;
    }
    return OFT_OK;
  }
  return fail(g, OFT_EINVAL, "bad kind");
}

int oft_frontier(oft_graph* g, int64_t cap, int64_t* m_out, int64_t* t_out, int64_t* n_out) {
  if (!g || !n_out) return OFT_EINVAL;
  int rc = check_started(g);
  if (rc) return rc;
  if (g->have_final && g->final_mode != 1) return fail(g, OFT_ESTATE, "frontier computed by FT-Elimination");
  if (!g->have_final && (rc = run_ldp(g))) return rc;
  const Frontier& F = g->sets[g->final_set].seg[0];
  *n_out = (int64_t)F.size();
  if (cap < (int64_t)F.size()) return OFT_ESIZE;
  for (size_t i = 0; i < F.size(); ++i) {
    if (m_out) m_out[i] = F[i].m;
    if (t_out) t_out[i] = F[i].t;
  }
  return OFT_OK;
}

int oft_frontier_elim(oft_graph* g, int64_t cap, int64_t* m_out, int64_t* t_out, int64_t* n_out) {
  if (!g || !n_out) return OFT_EINVAL;
  int rc = check_started(g);
  if (rc) return rc;
  if (g->have_final && g->final_mode != 2) return fail(g, OFT_ESTATE, "frontier computed by LDP");
  if (!g->have_final && (rc = run_elim(g))) return rc;
  const Frontier& F = g->sets[g->final_set].seg[0];
  *n_out = (int64_t)F.size();
  if (cap < (int64_t)F.size()) return OFT_ESIZE;
  for (size_t i = 0; i < F.size(); ++i) {
    if (m_out) m_out[i] = F[i].m;
    if (t_out) t_out[i] = F[i].t;
  }
  return OFT_OK;
}

int oft_query_mini_time(oft_graph* g, int64_t memory_limit, int64_t* idx_out) {
  if (!g || !idx_out) return OFT_EINVAL;
  if (!g->have_final) return fail(g, OFT_ESTATE, "call oft_frontier first");
  const Frontier& F = g->sets[g->final_set].seg[0];
  int64_t best = -1;  // plain scan: t strictly descends, so the last feasible tuple wins
  for (size_t i = 0; i < F.size(); ++i)
    if (F[i].m <= memory_limit && (best < 0 || F[i].t < F[best].t)) best = (int64_t)i;
  *idx_out = best;
  return OFT_OK;
}

int oft_strategy(oft_graph* g, int64_t idx, int32_t* cfg_out) {
  if (!g || !cfg_out) return OFT_EINVAL;
  if (!g->have_final) return fail(g, OFT_ESTATE, "call oft_frontier first");
  if (idx < 0 || idx >= (int64_t)g->sets[g->final_set].seg[0].size()) return fail(g, OFT_EINVAL, "bad index");
  std::vector<int32_t> cfg(g->n_ops, -1);
  int rc = visit(g, cfg, g->final_set, 0, idx);
  if (rc) return rc;
  for (int i = 0; i < g->n_orig_ops; ++i)
    if (cfg[i] < 0) return fail(g, OFT_EINTERNAL, "broken provenance: op without config");
  std::memcpy(cfg_out, cfg.data(), sizeof(int32_t) * g->n_orig_ops);
  return OFT_OK;
}

int oft_set_heuristic(oft_graph* g, int32_t policy, int64_t alpha_num, int64_t alpha_den) {
  if (!g || (policy != 0 && policy != 1)) return OFT_EINVAL;
  if (policy == 1 && (alpha_den < 1 || alpha_num < 0 || alpha_num > alpha_den))
    return fail(g, OFT_EINVAL, "alpha must be in [0, 1]");
  g->heur_policy = policy;
  if (policy == 1) {
    g->heur_num = alpha_num;
    g->heur_den = alpha_den;
  }
  return OFT_OK;
}

int64_t oft_num_steps(const oft_graph* g) { return g ? (int64_t)g->steps.size() : 0; }

int oft_step_info(const oft_graph* g, int64_t step, int64_t* info) {
  if (!g || !info || step < 0 || step >= (int64_t)g->steps.size()) return OFT_EINVAL;
  const Step& s = g->steps[step];
  info[0] = s.kind; info[1] = s.nseg; info[2] = s.nblk; info[3] = s.tuples;
  info[4] = s.survivors; info[5] = (int64_t)s.us;
  return OFT_OK;
}

int oft_step_output(const oft_graph* g, int64_t step, int64_t cap, int64_t* seg_off, int64_t* m,
                    int64_t* t, uint64_t* bp) {
  if (!g || step < 0 || step >= (int64_t)g->steps.size()) return OFT_EINVAL;
  const FSet& S = g->sets[g->steps[step].out];
  int64_t n = 0;
  for (auto& f : S.seg) n += (int64_t)f.size();
  if (cap < n) return OFT_ESIZE;
  int64_t o = 0;
  for (size_t sg = 0; sg < S.seg.size(); ++sg) {
    if (seg_off) seg_off[sg] = o;
    for (auto& x : S.seg[sg]) {
      if (m) m[o] = x.m;
      if (t) t[o] = x.t;
      if (bp) bp[o] = x.id;
      ++o;
    }
  }
  if (seg_off) seg_off[S.seg.size()] = o;
  return OFT_OK;
}

const char* oft_last_error(const oft_graph* g) { return g ? g->err.c_str() : "null graph"; }

int oft_reduce(int64_t n, const int64_t* m, const int64_t* t, const uint64_t* id, int64_t* m_out,
               int64_t* t_out, uint64_t* id_out, int64_t* n_out) {
  if (n < 0 || !n_out || (n > 0 && (!m || !t))) return OFT_EINVAL;
  std::vector<Tup> C(n);
  for (int64_t i = 0; i < n; ++i) C[i] = Tup{m[i], t[i], id ? id[i] : (uint64_t)i};
  Frontier F = reduce(std::move(C));
  *n_out = (int64_t)F.size();
  for (size_t i = 0; i < F.size(); ++i) {
    if (m_out) m_out[i] = F[i].m;
    if (t_out) t_out[i] = F[i].t;
    if (id_out) id_out[i] = F[i].id;
  }
  return OFT_OK;
}

int oft_segment_reduce(int32_t nblk, const int64_t* x_off, const int64_t* x_m, const int64_t* x_t,
                       const int64_t* y_off, const int64_t* y_m, const int64_t* y_t,
                       const int64_t* z_off, const int64_t* z_m, const int64_t* z_t, int64_t cap,
                       int64_t* m_out, int64_t* t_out, uint64_t* id_out, int64_t* n_out) {
  if (nblk < 0 || !n_out || !x_off || !y_off || !z_off) return OFT_EINVAL;
  std::vector<Tup> C;
  uint64_t pos = 0;
  for (int k = 0; k < nblk; ++k)  // Union of Products, written order
    for (int64_t x = x_off[k]; x < x_off[k + 1]; ++x)
      for (int64_t y = y_off[k]; y < y_off[k + 1]; ++y)
        for (int64_t z = z_off[k]; z < z_off[k + 1]; ++z) {
          C.push_back(Tup{x_m[x] + y_m[y] + z_m[z], x_t[x] + y_t[y] + z_t[z], pos});
          ++pos;
        }
  Frontier F = reduce(std::move(C));
  *n_out = (int64_t)F.size();
  if (cap < (int64_t)F.size()) return OFT_ESIZE;
  for (size_t i = 0; i < F.size(); ++i) {
    if (m_out) m_out[i] = F[i].m;
    if (t_out) t_out[i] = F[i].t;
    if (id_out) id_out[i] = F[i].id;
  }
  return OFT_OK;
}

}  // extern "C"
