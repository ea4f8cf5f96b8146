// oracle_costgen.cpp -- CPU oracle for edge-cost generation (SURVEY 8(f)
// rank 4).  TEST INFRASTRUCTURE: only tests/, smoke() and bench.py's CPU legs
// may call it; it shares no code with the CUDA path (libft's ft_costgen.cu).
//
//  * ocg_comm_time: profile-based communication time, P:668-671 ("we find the
//    integer i satisfying 2^i <= k < 2^(i+1) and use the interpolation of the
//    actual bandwidths at 2^i and 2^(i+1)"), integer reading R18.
//  * ocg_split_states: the nodes of the re-scheduling graph, "different tensor
//    splits", reading R19.
//  * ocg_reschedule_costs: "the optimal communication operations correspond to
//    the shortest path from the output tensor split to the required input
//    tensor split", solved here by textbook Dijkstra (O(S^2) array
//    version) from every source; t_x = d(from,to) + d(to,from) (Eq. 2,
//    P:408-415, forward + backward pass; R19).
#include <cstdint>
#include <vector>

namespace {

constexpr int MAXL = 6, MAXP = 46, MAXD = 4;

struct Profile {
  int32_t L, P;
  int64_t lat[MAXL + 1];
  int64_t bw[MAXL + 1][MAXP + 1];
};

// comm_time(bytes, group 2^c) in integer ns; -1 if bytes is outside the profile.
int64_t comm_time(const Profile* p, int64_t bytes, int c) {
  if (bytes == 0 || c == 0) return 0;
  if (bytes > (int64_t(1) << p->P)) return -1;
  int i = 0;
  while ((int64_t(1) << (i + 1)) <= bytes) i++;  // 2^i <= bytes < 2^(i+1)
  __int128 bw;
  if (i == p->P) {
    bw = p->bw[c][i];
  } else {
    int64_t lo = int64_t(1) << i;
    bw = p->bw[c][i] + (__int128)(p->bw[c][i + 1] - p->bw[c][i]) * (bytes - lo) / lo;
  }
  __int128 num = (__int128)bytes * 1000000000;
  __int128 t = (num + bw - 1) / bw;  // ceil(bytes * 1e9 / bw)
  return p->lat[c] + (int64_t)t;
}

bool profile_ok(const Profile* p) {
  if (p->L < 1 || p->L > MAXL || p->P < 1 || p->P > MAXP) return false;
  for (int c = 1; c <= p->L; c++) {
    if (p->lat[c] < 0) return false;
    for (int i = 0; i <= p->P; i++)
      if (p->bw[c][i] <= 0) return false;
  }
  return true;
}

// Enumerate a = (a_0..a_{D-1}) in lexicographic order (recursion on j).
void enum_states(int D, const int64_t* dims, int L, int j, int used, std::vector<int>& cur,
                 std::vector<std::vector<int>>& out) {
  if (j == D) {
    out.push_back(cur);
    return;
  }
  for (int a = 0; used + a <= L; a++) {
    if (dims[j] % (int64_t(1) << a) != 0) break;  // 2^a must divide dims[j]
    cur[j] = a;
    enum_states(D, dims, L, j + 1, used + a, cur, out);
  }
}

int find_state(const std::vector<std::vector<int>>& S, const std::vector<int>& a) {
  for (size_t s = 0; s < S.size(); s++)
    if (S[s] == a) return (int)s;
  return -1;
}

}  // namespace

extern "C" {

int ocg_comm_time(const void* prof, int64_t n, const int64_t* bytes, const int32_t* group_log2,
                  int64_t* t_out) {
  const Profile* p = (const Profile*)prof;
  if (!profile_ok(p)) return -1;
  for (int64_t q = 0; q < n; q++) {
    if (bytes[q] < 0 || group_log2[q] < 0 || group_log2[q] > p->L) return -1;
    int64_t t = comm_time(p, bytes[q], group_log2[q]);
    if (t < 0) return -6;
    t_out[q] = t;
  }
  return 0;
}

int ocg_split_states(int32_t D, const int64_t* dims, int32_t L, int64_t cap, int32_t* out,
                     int64_t* n_out) {
  if (D < 1 || D > MAXD || L < 1 || L > MAXL) return -1;
  for (int j = 0; j < D; j++)
    if (dims[j] < 1) return -1;
  std::vector<std::vector<int>> S;
  std::vector<int> cur(D, 0);
  enum_states(D, dims, L, 0, 0, cur, S);
  *n_out = (int64_t)S.size();
  if (cap < (int64_t)S.size()) return -7;
  for (size_t s = 0; s < S.size(); s++)
    for (int j = 0; j < D; j++) out[s * D + j] = S[s][j];
  return 0;
}

// All-pairs distances of one tensor's state graph: dist[S*S] (row = source).
int ocg_state_dist(const void* prof, int32_t D, const int64_t* dims, int64_t elem_bytes,
                   int64_t cap, int64_t* dist, int64_t* n_out) {
  const Profile* p = (const Profile*)prof;
  if (!profile_ok(p) || D < 1 || D > MAXD || elem_bytes < 1) return -1;
  int64_t total = elem_bytes;
  for (int j = 0; j < D; j++) {
    if (dims[j] < 1) return -1;
    if (total > ((int64_t(1) << p->P) / dims[j])) return -6;
    total *= dims[j];
  }
  if (total > (int64_t(1) << p->P)) return -6;
  std::vector<std::vector<int>> S;
  std::vector<int> cur(D, 0);
  enum_states(D, dims, p->L, 0, 0, cur, S);
  int64_t n = (int64_t)S.size();
  *n_out = n;
  if (cap < n * n) return -7;
  // Edge list of the state graph: one entry per single collective operation.
  std::vector<std::vector<std::pair<int, int64_t>>> adj(n);
  for (int s = 0; s < n; s++) {
    const std::vector<int>& a = S[s];
    int used = 0;
    for (int j = 0; j < D; j++) used += a[j];
    int64_t shard = total >> used;
    for (int j = 0; j < D; j++) {
      // all-gather on dim j over a group of 2^c devices
      for (int c = 1; c <= a[j]; c++) {
        std::vector<int> b = a;
        b[j] -= c;
        int64_t recv = shard * ((int64_t(1) << c) - 1);
        adj[s].push_back({find_state(S, b), comm_time(p, recv, c)});
      }
      // local slice on dim j (no communication)
      for (int c = 1; used + c <= p->L; c++) {
        std::vector<int> b = a;
        b[j] += c;
        int t = find_state(S, b);
        if (t >= 0) adj[s].push_back({t, 0});
      }
      // all-to-all moving a factor 2^c from dim j to dim k
      for (int k = 0; k < D; k++) {
        if (k == j) continue;
        for (int c = 1; c <= a[j]; c++) {
          std::vector<int> b = a;
          b[j] -= c;
          b[k] += c;
          int t = find_state(S, b);
          if (t < 0) continue;
          int64_t moved = shard - (shard >> c);
          adj[s].push_back({t, comm_time(p, moved, c)});
        }
      }
    }
  }
  const int64_t INF = INT64_MAX;
  for (int src = 0; src < n; src++) {
    int64_t* d = dist + (int64_t)src * n;
    std::vector<char> done(n, 0);
    for (int v = 0; v < n; v++) d[v] = INF;
    d[src] = 0;
    for (int it = 0; it < n; it++) {
      int u = -1;
      for (int v = 0; v < n; v++)
        if (!done[v] && d[v] != INF && (u < 0 || d[v] < d[u])) u = v;
      if (u < 0) break;
      done[u] = 1;
      for (auto& e : adj[u])
        if (d[u] + e.second < d[e.first]) d[e.first] = d[u] + e.second;
    }
  }
  return 0;
}

int ocg_reschedule_costs(const void* prof, int32_t n_tensors, const int32_t* ndims,
                         const int64_t* dims, const int64_t* elem_bytes, int64_t n_q,
                         const int32_t* q_tensor, const int32_t* q_from, const int32_t* q_to,
                         int64_t* t_out) {
  std::vector<std::vector<int64_t>> dist(n_tensors);
  std::vector<int64_t> ns(n_tensors);
  for (int x = 0; x < n_tensors; x++) {
    int64_t n = 0;
    int32_t scratch[1];
    int rc = ocg_split_states(ndims[x], dims + (int64_t)x * MAXD, ((const Profile*)prof)->L, 0,
                              scratch, &n);
    if (rc != 0 && rc != -7) return rc;
    dist[x].resize(n * n);
    rc = ocg_state_dist(prof, ndims[x], dims + (int64_t)x * MAXD, elem_bytes[x], n * n,
                        dist[x].data(), &n);
    if (rc != 0) return rc;
    ns[x] = n;
  }
  for (int64_t q = 0; q < n_q; q++) {
    int x = q_tensor[q];
    if (x < 0 || x >= n_tensors) return -1;
    int64_t n = ns[x];
    if (q_from[q] < 0 || q_from[q] >= n || q_to[q] < 0 || q_to[q] >= n) return -1;
    t_out[q] = dist[x][q_from[q] * n + q_to[q]] + dist[x][q_to[q] * n + q_from[q]];
  }
  return 0;
}

}  // extern "C"

// Gradient synchronisation cost of a parameter tensor (Eq. 1's m_p and t_s,
// P:399-406 with the comm model of P:668-671; reading R20): in split state a
// each device stores shard = total / 2^(sum a) bytes (m_p) and all-reduces
// its gradient with the r = 2^(L - sum a) devices holding the same shard; a
// ring all-reduce moves 2 * (shard - shard / r) bytes per device, timed by
// comm_time over a group of r devices.  r = 1: t_s = 0.
extern "C" int ocg_sync_costs(const void* prof, int32_t n_tensors, const int32_t* ndims,
                              const int64_t* dims, const int64_t* elem_bytes, int64_t n_q,
                              const int32_t* q_tensor, const int32_t* q_state, int64_t* m_out,
                              int64_t* t_out) {
  const Profile* p = (const Profile*)prof;
  if (!profile_ok(p)) return -1;
  for (int64_t q = 0; q < n_q; q++) {
    int x = q_tensor[q];
    if (x < 0 || x >= n_tensors) return -1;
    int D = ndims[x];
    const int64_t* dm = dims + (int64_t)x * MAXD;
    if (D < 1 || D > MAXD || elem_bytes[x] < 1) return -1;
    int64_t total = elem_bytes[x];
    for (int j = 0; j < D; j++) {
      if (dm[j] < 1) return -1;
      if (total > ((int64_t(1) << p->P) / dm[j])) return -6;
      total *= dm[j];
    }
    if (total > (int64_t(1) << (p->P - 1))) return -6;  // 2 * total must fit the profile
    std::vector<std::vector<int>> S;
    std::vector<int> cur(D, 0);
    enum_states(D, dm, p->L, 0, 0, cur, S);
    if (q_state[q] < 0 || q_state[q] >= (int)S.size()) return -1;
    int used = 0;
    for (int j = 0; j < D; j++) used += S[q_state[q]][j];
    int64_t shard = total >> used;
    int u = p->L - used;
    m_out[q] = shard;
    t_out[q] = comm_time(p, 2 * (shard - (shard >> u)), u);
  }
  return 0;
}
