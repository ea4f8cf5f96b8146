// ft_costgen.cu -- edge-cost generation on the GPU:
// t_x(e, s_i^k, s_j^p) of Eq. 2 from the profile-interpolated
// communication time (reading R18) and tensor re-scheduling as a
// shortest path over tensor splits (R19).  C-ABI in include/ft.h.
//
// Kernels:
//   k_cg_comm_time  grid-stride batch of comm_time queries (HBM streaming)
//   k_cg_apsp       one CTA per tensor: build the state graph's weight matrix
//                   in shared memory (one row per source state, moves generated
//                   by the owning thread), then Floyd-Warshall in place in
//                   shared memory (S <= 160: 200 KB of int64), store S x S.
//   k_cg_gather     grid-stride: t_x[q] = d(from,to) + d(to,from).
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstring>
#include <atomic>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/ft.h"

namespace {

constexpr int64_t kInf = INT64_MAX / 4;
constexpr int kApspThreads = 256;

constexpr int kRegWarps = 8;  // warps of the register-resident FW
constexpr int kMaxCode = 7 * 7 * 7 * 7;  // (L+1)^D state codes, L <= 6, D <= 4

struct TensorDesc {
  int64_t total;     // bytes of the whole tensor
  int64_t dist_off;  // offset of its S x S block in the distance buffer
  int32_t state_off; // first row in the state table
  int32_t n_states;
  int32_t ndims;
  int32_t pad;
  int64_t dims[FT_CG_MAX_DIMS];
};

// comm_time (R18): 2^i <= b < 2^(i+1), linear interpolation of bw[c][i],
// bw[c][i+1] in b (C division), then latency + ceil(b * 1e9 / bw).
__device__ inline int64_t cg_time_dev(const ft_comm_profile& p, int64_t b, int c) {
  if (b == 0 || c == 0) return 0;
  const int i = 63 - __clzll(b);
  __int128 bw = p.bw[c][i];
  if (i < p.P) {
    const int64_t lo = int64_t(1) << i;
    bw += (__int128)(p.bw[c][i + 1] - p.bw[c][i]) * (b - lo) / lo;
  }
  const __int128 num = (__int128)b * 1000000000;
  return p.latency_ns[c] + (int64_t)((num + bw - 1) / bw);
}

__global__ void k_cg_comm_time(const ft_comm_profile* __restrict__ prof, int64_t n,
                               const int64_t* __restrict__ bytes, const int32_t* __restrict__ grp,
                               int64_t* __restrict__ out) {
  __shared__ ft_comm_profile p;
  for (int i = threadIdx.x; i < (int)(sizeof(p) / 8); i += blockDim.x)
    reinterpret_cast<int64_t*>(&p)[i] = reinterpret_cast<const int64_t*>(prof)[i];
  __syncthreads();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    out[q] = cg_time_dev(p, bytes[q], grp[q]);
}

// Register-resident Floyd-Warshall for S <= 32*C (C = 2: S <= 64, C = 3:
// S <= 96) with kRegWarps warps: thread (warp w, lane l) owns
// d[w + kRegWarps*r][l + 32c], r < 32*C/kRegWarps, c < C.  Round k publishes
// row k (its owner warp) and column k (lane k%32 of every warp) to
// double-buffered shared rows, one barrier per round; every thread then does
// rows*C min-plus updates from C + rows shared loads.  Writes the result.
template <int C>
__device__ __forceinline__ void fw_registers(const int64_t* __restrict__ d, int S,
                                             int64_t* __restrict__ out, int warp, int lane) {
  constexpr int kRows = 32 * C / kRegWarps;
  __shared__ int64_t rowbuf[2][32 * C], colbuf[2][32 * C];
  int64_t v[kRows][C];
#pragma unroll
  for (int r = 0; r < kRows; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int i = warp + kRegWarps * r, j = lane + 32 * c;
      v[r][c] = (i < S && j < S) ? d[i * S + j] : kInf;
    }
  for (int k = 0; k < S; ++k) {
    const int b = k & 1;
    if ((k % kRegWarps) == warp) {
      const int r = k / kRegWarps;
#pragma unroll
      for (int rr = 0; rr < kRows; ++rr)
        if (rr == r) {
#pragma unroll
          for (int c = 0; c < C; ++c) rowbuf[b][lane + 32 * c] = v[rr][c];
        }
    }
    if ((k & 31) == lane) {
      const int cc = k >> 5;
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        int64_t x = v[r][0];
#pragma unroll
        for (int c = 1; c < C; ++c)
          if (cc == c) x = v[r][c];
        colbuf[b][warp + kRegWarps * r] = x;
      }
    }
    __syncthreads();
    int64_t rk[C];
#pragma unroll
    for (int c = 0; c < C; ++c) rk[c] = rowbuf[b][lane + 32 * c];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const int64_t dik = colbuf[b][warp + kRegWarps * r];
#pragma unroll
      for (int c = 0; c < C; ++c) v[r][c] = min(v[r][c], dik + rk[c]);
    }
  }
#pragma unroll
  for (int r = 0; r < kRows; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int i = warp + kRegWarps * r, j = lane + 32 * c;
      if (i < S && j < S) out[i * S + j] = v[r][c];
    }
}

// One CTA per tensor.  States are packed one byte per dim (a_j <= 6) into
// int32 codes; the lookup table maps the mixed-radix code sum a_j (L+1)^j to
// the state index (-1 = invalid split).
template <int C>
__global__ void __launch_bounds__(kApspThreads, C == 2 ? 3 : 2)
k_cg_apsp(const ft_comm_profile* __restrict__ prof, const TensorDesc* __restrict__ tens,
          const int32_t* __restrict__ states, int64_t* __restrict__ dist) {
  extern __shared__ int64_t smem[];
  __shared__ ft_comm_profile p;
  __shared__ int16_t lut[kMaxCode];
  const TensorDesc td = tens[blockIdx.x];
  const int S = td.n_states, D = td.ndims;
  for (int i = threadIdx.x; i < (int)(sizeof(p) / 8); i += blockDim.x)
    reinterpret_cast<int64_t*>(&p)[i] = reinterpret_cast<const int64_t*>(prof)[i];
  const int L = prof->mesh_log2, R = L + 1;
  int ncode = 1;
  for (int j = 0; j < D; ++j) ncode *= R;
  for (int i = threadIdx.x; i < ncode; i += blockDim.x) lut[i] = -1;
  int64_t* d = smem;  // S x S
  for (int i = threadIdx.x; i < S * S; i += blockDim.x) d[i] = (i / S == i % S) ? 0 : kInf;
  __syncthreads();
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    const int32_t pk = states[td.state_off + s];
    int code = 0, mul = 1;
    for (int j = 0; j < D; ++j, mul *= R) code += ((pk >> (8 * j)) & 0xff) * mul;
    lut[code] = (int16_t)s;
  }
  // A move's time depends only on (sum a, c): shard = total >> sum a.  The
  // 2 x (L+1) x L distinct comm times are computed once, one per thread.
  __shared__ int64_t w_gather[FT_CG_MAX_MESH + 1][FT_CG_MAX_MESH + 1];
  __shared__ int64_t w_a2a[FT_CG_MAX_MESH + 1][FT_CG_MAX_MESH + 1];
  __syncthreads();
  for (int e = threadIdx.x; e < 2 * R * L; e += blockDim.x) {
    const int kind = e / (R * L), u = (e / L) % R, c = e % L + 1;
    const int64_t shard = td.total >> u;
    if (kind == 0)
      w_gather[u][c] = c <= u ? cg_time_dev(p, shard * ((int64_t(1) << c) - 1), c) : 0;
    else
      w_a2a[u][c] = c <= u ? cg_time_dev(p, shard - (shard >> c), c) : 0;
  }
  __syncthreads();
  // Row s of the weight matrix: every single collective out of state s.
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    const int32_t pk = states[td.state_off + s];
    int a[FT_CG_MAX_DIMS], pw[FT_CG_MAX_DIMS];
    int used = 0, code = 0, mul = 1;
    for (int j = 0; j < D; ++j, mul *= R) {
      a[j] = (pk >> (8 * j)) & 0xff;
      pw[j] = mul;
      used += a[j];
      code += a[j] * mul;
    }
    int64_t* row = d + (int64_t)s * S;
    for (int j = 0; j < D; ++j) {
      for (int c = 1; c <= a[j]; ++c) {  // all-gather on dim j, group 2^c
        const int t = lut[code - c * pw[j]];
        const int64_t w = w_gather[used][c];
        if (w < row[t]) row[t] = w;
      }
      for (int c = 1; used + c <= L && a[j] + c <= L; ++c) {  // local slice
        const int t = lut[code + c * pw[j]];
        if (t >= 0) row[t] = 0;
      }
      for (int k = 0; k < D; ++k) {  // all-to-all: factor 2^c from dim j to dim k
        if (k == j) continue;
        for (int c = 1; c <= a[j] && a[k] + c <= L; ++c) {
          const int t = lut[code - c * pw[j] + c * pw[k]];
          if (t < 0) continue;
          const int64_t w = w_a2a[used][c];
          if (w < row[t]) row[t] = w;
        }
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  if (S <= 32 * C && nwarp == kRegWarps) {
    __syncthreads();  // weight matrix complete
    fw_registers<C>(d, S, dist + td.dist_off, warp, lane);
    return;
  }
  // General case: Floyd-Warshall in place in shared memory: row k and column
  // k do not change in round k (d[k][k] = 0), so the in-place update is
  // race-free.  Lane -> column j
  // (a warp reads 32 consecutive int64 of row k), warp -> row i (d[i][k] is a
  // broadcast).
  for (int k = 0; k < S; ++k) {
    __syncthreads();
    const int64_t* rk = d + (int64_t)k * S;
    for (int i = warp; i < S; i += nwarp) {
      int64_t* ri = d + (int64_t)i * S;
      const int64_t dik = ri[k];
      for (int j = lane; j < S; j += 32) {
        const int64_t v = dik + rk[j];
        if (v < ri[j]) ri[j] = v;
      }
    }
  }
  __syncthreads();
  int64_t* out = dist + td.dist_off;
  for (int e = threadIdx.x; e < S * S; e += blockDim.x) out[e] = d[e];
}

__device__ __forceinline__ int64_t cg_one(const TensorDesc* __restrict__ tens, int32_t n_tensors,
                                          const int64_t* __restrict__ dist, int x, int64_t f,
                                          int64_t t, int32_t* bad) {
  if ((unsigned)x >= (unsigned)n_tensors) {  // invalid query: flag, write 0
    *bad = 1;
    return 0;
  }
  const int64_t S = __ldg(&tens[x].n_states), off = __ldg(&tens[x].dist_off);
  if ((uint64_t)f >= (uint64_t)S || (uint64_t)t >= (uint64_t)S) {
    *bad = 1;
    return 0;
  }
  return __ldg(dist + off + f * S + t) + __ldg(dist + off + t * S + f);
}

// Four queries per thread per iteration with 16-byte loads/stores when the
// arrays are 16-byte aligned (independent loads in flight), scalar tail.
__global__ void k_cg_gather(const TensorDesc* __restrict__ tens, int32_t n_tensors,
                            const int64_t* __restrict__ dist, int64_t n,
                            const int32_t* __restrict__ qt, const int32_t* __restrict__ qf,
                            const int32_t* __restrict__ qo, int64_t* __restrict__ out,
                            int32_t* __restrict__ bad) {
  const bool vec = ((reinterpret_cast<uintptr_t>(qt) | reinterpret_cast<uintptr_t>(qf) |
                     reinterpret_cast<uintptr_t>(qo) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = tid; v < n4; v += stride) {
    const int4 x = reinterpret_cast<const int4*>(qt)[v];
    const int4 f = reinterpret_cast<const int4*>(qf)[v];
    const int4 t = reinterpret_cast<const int4*>(qo)[v];
    longlong2 o0, o1;
    o0.x = cg_one(tens, n_tensors, dist, x.x, f.x, t.x, bad);
    o0.y = cg_one(tens, n_tensors, dist, x.y, f.y, t.y, bad);
    o1.x = cg_one(tens, n_tensors, dist, x.z, f.z, t.z, bad);
    o1.y = cg_one(tens, n_tensors, dist, x.w, f.w, t.w, bad);
    reinterpret_cast<longlong2*>(out)[2 * v] = o0;
    reinterpret_cast<longlong2*>(out)[2 * v + 1] = o1;
  }
  for (int64_t q = n4 * 4 + tid; q < n; q += stride)
    out[q] = cg_one(tens, n_tensors, dist, qt[q], qf[q], qo[q], bad);
}

// Gradient-sync op costs (R20): m_p = shard, t_s = comm time of the ring
// all-reduce volume 2*(shard - shard/r) over r = 2^(L - sum a) replicas.
__global__ void k_cg_sync(const ft_comm_profile* __restrict__ prof,
                          const TensorDesc* __restrict__ tens, int32_t n_tensors,
                          const int32_t* __restrict__ states, int64_t n,
                          const int32_t* __restrict__ qt, const int32_t* __restrict__ qs,
                          int64_t* __restrict__ m_out, int64_t* __restrict__ t_out,
                          int32_t* __restrict__ bad) {
  __shared__ ft_comm_profile p;
  for (int i = threadIdx.x; i < (int)(sizeof(p) / 8); i += blockDim.x)
    reinterpret_cast<int64_t*>(&p)[i] = reinterpret_cast<const int64_t*>(prof)[i];
  __syncthreads();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int x = qt[q], s = qs[q];
    if ((unsigned)x >= (unsigned)n_tensors || (unsigned)s >= (unsigned)tens[x].n_states) {
      *bad = 1;
      m_out[q] = 0;
      t_out[q] = 0;
      continue;
    }
    const int32_t pk = states[tens[x].state_off + s];
    const int used = (pk & 0xff) + ((pk >> 8) & 0xff) + ((pk >> 16) & 0xff) + ((pk >> 24) & 0xff);
    const int64_t shard = tens[x].total >> used;
    const int u = p.mesh_log2 - used;
    m_out[q] = shard;
    t_out[q] = cg_time_dev(p, 2 * (shard - (shard >> u)), u);
  }
}

bool profile_valid(const ft_comm_profile* p) {
  if (!p || p->mesh_log2 < 1 || p->mesh_log2 > FT_CG_MAX_MESH || p->P < 1 || p->P > FT_CG_MAX_P)
    return false;
  for (int c = 1; c <= p->mesh_log2; ++c) {
    if (p->latency_ns[c] < 0) return false;
    for (int i = 0; i <= p->P; ++i)
      if (p->bw[c][i] <= 0) return false;
  }
  return true;
}

// Odometer enumeration of the split states in lexicographic order (a_0 most
// significant).  Returns the packed codes (byte j = a_j).
std::vector<int32_t> enum_states(int D, const int64_t* dims, int L) {
  int amax[FT_CG_MAX_DIMS];
  for (int j = 0; j < D; ++j) {
    amax[j] = 0;
    while (amax[j] < L && dims[j] % (int64_t(1) << (amax[j] + 1)) == 0) ++amax[j];
  }
  std::vector<int32_t> out;
  int a[FT_CG_MAX_DIMS] = {0, 0, 0, 0};
  for (;;) {
    int sum = 0;
    for (int j = 0; j < D; ++j) sum += a[j];
    if (sum <= L) {
      int32_t pk = 0;
      for (int j = 0; j < D; ++j) pk |= a[j] << (8 * j);
      out.push_back(pk);
    }
    int j = D - 1;  // increment the least significant digit first
    while (j >= 0 && a[j] == amax[j]) a[j--] = 0;
    if (j < 0) break;
    ++a[j];
  }
  return out;
}

struct DevBufs {
  std::vector<void*> ptrs;
  ~DevBufs() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <class T>
  cudaError_t alloc(T** p, size_t n) {
    void* v = nullptr;
    cudaError_t e = cudaMalloc(&v, n ? n * sizeof(T) : 1);
    if (e == cudaSuccess) ptrs.push_back(v);
    *p = (T*)v;
    return e;
  }
};

// Grow-only device buffers reused across calls (one pool per device; calls
// on the same device serialise on its mutex).
std::atomic<int> g_profile{0};  // ft_costgen_profile

struct Pool {
  std::mutex mu;
  void* buf[8] = {};
  size_t cap[8] = {};
  cudaEvent_t ev[4] = {};     // apsp begin/end, gather begin/end (profiling)
  float last_ms[2] = {0, 0};  // last ft_reschedule_costs_dev: apsp, gather
  cudaError_t get(int slot, size_t bytes, void** out) {
    if (bytes > cap[slot]) {
      const size_t want = std::max(bytes, cap[slot] * 3 / 2);
      if (buf[slot]) cudaFree(buf[slot]);
      buf[slot] = nullptr;
      cap[slot] = 0;
      cudaError_t e = cudaMalloc(&buf[slot], want);
      if (e != cudaSuccess) return e;
      cap[slot] = want;
    }
    *out = buf[slot];
    return cudaSuccess;
  }
};

Pool& pool_for_device() {
  static std::mutex m;
  static Pool* pools[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(m);
  if (!pools[dev & 63]) pools[dev & 63] = new Pool();
  return *pools[dev & 63];
}

#define CG_CHECK(x)                     \
  do {                                  \
    if ((x) != cudaSuccess) {           \
      cudaGetLastError();               \
      return FT_ECUDA;                  \
    }                                   \
  } while (0)

int grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
}

}  // namespace

extern "C" int ft_comm_time(const ft_comm_profile* prof, int64_t n, const int64_t* bytes,
                            const int32_t* group_log2, int64_t* t_out) {
  if (!profile_valid(prof) || n < 0 || (n > 0 && (!bytes || !group_log2 || !t_out)))
    return FT_EINVAL;
  for (int64_t q = 0; q < n; ++q) {
    if (bytes[q] < 0 || group_log2[q] < 0 || group_log2[q] > prof->mesh_log2) return FT_EINVAL;
    if (bytes[q] > (int64_t(1) << prof->P)) return FT_EOVERFLOW;
  }
  if (n == 0) return FT_OK;
  DevBufs B;
  ft_comm_profile* dp;
  int64_t *db, *dt;
  int32_t* dg;
  CG_CHECK(B.alloc(&dp, 1));
  CG_CHECK(B.alloc(&db, n));
  CG_CHECK(B.alloc(&dg, n));
  CG_CHECK(B.alloc(&dt, n));
  CG_CHECK(cudaMemcpy(dp, prof, sizeof(*prof), cudaMemcpyHostToDevice));
  CG_CHECK(cudaMemcpy(db, bytes, n * 8, cudaMemcpyHostToDevice));
  CG_CHECK(cudaMemcpy(dg, group_log2, n * 4, cudaMemcpyHostToDevice));
  k_cg_comm_time<<<grid_for(n), 256>>>(dp, n, db, dg, dt);
  CG_CHECK(cudaGetLastError());
  CG_CHECK(cudaMemcpy(t_out, dt, n * 8, cudaMemcpyDeviceToHost));
  return FT_OK;
}

extern "C" int ft_split_states(int32_t ndims, const int64_t* dims, int32_t mesh_log2, int64_t cap,
                               int32_t* states_out, int64_t* n_out) {
  if (ndims < 1 || ndims > FT_CG_MAX_DIMS || !dims || !n_out || mesh_log2 < 1 ||
      mesh_log2 > FT_CG_MAX_MESH || cap < 0 || (cap > 0 && !states_out))
    return FT_EINVAL;
  for (int j = 0; j < ndims; ++j)
    if (dims[j] < 1) return FT_EINVAL;
  const std::vector<int32_t> st = enum_states(ndims, dims, mesh_log2);
  *n_out = (int64_t)st.size();
  if (cap < (int64_t)st.size()) return FT_ESIZE;
  for (size_t s = 0; s < st.size(); ++s)
    for (int j = 0; j < ndims; ++j) states_out[s * ndims + j] = (st[s] >> (8 * j)) & 0xff;
  return FT_OK;
}

namespace {

// Host-side part shared by both entry points: validate the tensors, enumerate
// their split states, lay out the distance blocks.
int plan_tensors(const ft_comm_profile* prof, int32_t n_tensors, const int32_t* ndims,
                 const int64_t* dims, const int64_t* elem_bytes, std::vector<TensorDesc>& td,
                 std::vector<int32_t>& states, int64_t& dist_total, int& max_s) {
  if (!profile_valid(prof) || n_tensors < 0 || (n_tensors > 0 && (!ndims || !dims || !elem_bytes)))
    return FT_EINVAL;
  const int64_t cap = int64_t(1) << prof->P;
  td.assign(n_tensors, TensorDesc{});
  states.clear();
  dist_total = 0;
  max_s = 0;
  std::vector<int64_t> memo(1 << 15, -1);
  for (int x = 0; x < n_tensors; ++x) {
    TensorDesc& t = td[x];
    t.ndims = ndims[x];
    if (t.ndims < 1 || t.ndims > FT_CG_MAX_DIMS || elem_bytes[x] < 1) return FT_EINVAL;
    int64_t total = elem_bytes[x];
    for (int j = 0; j < t.ndims; ++j) {
      const int64_t dj = dims[(int64_t)x * FT_CG_MAX_DIMS + j];
      if (dj < 1) return FT_EINVAL;
      if (total > cap / dj) return FT_EOVERFLOW;
      total *= dj;
      t.dims[j] = dj;
    }
    t.total = total;
    // The state set depends only on (ndims, min(L, 2-adic valuation of each
    // dim)): tensors with the same signature share one run of state rows.
    int key = t.ndims;
    for (int j = 0; j < t.ndims; ++j) {
      int v = 0;
      while (v < prof->mesh_log2 && t.dims[j] % (int64_t(1) << (v + 1)) == 0) ++v;
      key |= v << (3 + 3 * j);
    }
    if (memo[key] < 0) {
      const std::vector<int32_t> st = enum_states(t.ndims, t.dims, prof->mesh_log2);
      if ((int64_t)st.size() > FT_CG_MAX_STATES) return FT_ESIZE;
      memo[key] = (int64_t)states.size() | ((int64_t)st.size() << 32);
      states.insert(states.end(), st.begin(), st.end());
    }
    t.state_off = (int32_t)(memo[key] & 0xffffffff);
    t.n_states = (int32_t)(memo[key] >> 32);
    t.dist_off = dist_total;
    dist_total += (int64_t)t.n_states * t.n_states;
    if (t.n_states > max_s) max_s = t.n_states;
  }
  return FT_OK;
}

// Device state of one call (pool slots 0..4: profile, descriptors, states,
// distances, error flag).
struct Launch {
  void *dp, *dtd, *dst, *dd, *dbad;
  int32_t n_tensors;
};

// Upload the plan and launch the APSP on `st`.
int launch_apsp(Pool& P, const ft_comm_profile* prof, const std::vector<TensorDesc>& td,
                const std::vector<int32_t>& states, int64_t dist_total, int max_s, cudaStream_t st,
                Launch& L) {
  CG_CHECK(P.get(0, sizeof(*prof), &L.dp));
  CG_CHECK(P.get(1, td.size() * sizeof(TensorDesc), &L.dtd));
  CG_CHECK(P.get(2, states.size() * 4, &L.dst));
  CG_CHECK(P.get(3, (size_t)dist_total * 8, &L.dd));
  CG_CHECK(P.get(4, 4, &L.dbad));
  L.n_tensors = (int32_t)td.size();
  CG_CHECK(cudaMemcpyAsync(L.dp, prof, sizeof(*prof), cudaMemcpyHostToDevice, st));
  CG_CHECK(cudaMemcpyAsync(L.dtd, td.data(), td.size() * sizeof(TensorDesc), cudaMemcpyHostToDevice, st));
  CG_CHECK(cudaMemcpyAsync(L.dst, states.data(), states.size() * 4, cudaMemcpyHostToDevice, st));
  CG_CHECK(cudaMemsetAsync(L.dbad, 0, 4, st));
  const size_t smem = (size_t)max_s * max_s * sizeof(int64_t);
  // Register Floyd-Warshall with 2 columns per lane (S <= 64, 3 CTAs/SM) or
  // 3 (S <= 96, 2 CTAs/SM); larger tensors use the shared-memory path.
  auto kern = max_s <= 64 ? k_cg_apsp<2> : k_cg_apsp<3>;
  CG_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CG_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  kern<<<(int)td.size(), kApspThreads, smem, st>>>((const ft_comm_profile*)L.dp,
                                                  (const TensorDesc*)L.dtd,
                                                  (const int32_t*)L.dst, (int64_t*)L.dd);
  CG_CHECK(cudaGetLastError());
  return FT_OK;
}

int launch_gather(const Launch& L, int64_t n, const int32_t* qt, const int32_t* qf,
                  const int32_t* qo, int64_t* out, cudaStream_t st) {
  k_cg_gather<<<grid_for((n + 3) / 4), 256, 0, st>>>((const TensorDesc*)L.dtd, L.n_tensors,
                                                     (const int64_t*)L.dd, n, qt, qf, qo, out,
                                                     (int32_t*)L.dbad);
  CG_CHECK(cudaGetLastError());
  return FT_OK;
}

int finish(const Launch& L, cudaStream_t st) {
  int32_t bad = 0;
  CG_CHECK(cudaMemcpyAsync(&bad, L.dbad, 4, cudaMemcpyDeviceToHost, st));
  CG_CHECK(cudaStreamSynchronize(st));
  return bad ? FT_EINVAL : FT_OK;
}

// Host copy split over up to 8 threads (pageable <-> pinned staging is bound
// by one core's memcpy bandwidth otherwise).
void par_memcpy(void* dst, const void* src, size_t bytes) {
  const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  const size_t parts = bytes < (size_t(1) << 21) ? 1 : hw;
  if (parts == 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t per = (bytes + parts - 1) / parts;
  for (size_t k = 1; k < parts; ++k) {
    const size_t lo = k * per, n = lo < bytes ? std::min(per, bytes - lo) : 0;
    if (n) th.emplace_back([=] { std::memcpy((char*)dst + lo, (const char*)src + lo, n); });
  }
  std::memcpy(dst, src, std::min(per, bytes));
  for (auto& t : th) t.join();
}

// Pinned host staging for the host-buffer entry: two slots of kChunk queries
// (inputs 12 B, output 8 B per query), grow-once, one set per process.
constexpr int64_t kChunk = int64_t(1) << 20;
struct Staging {
  int32_t* in[2] = {nullptr, nullptr};
  int64_t* out[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int dev = -1;
  cudaError_t init(int device) {
    if (dev == device) return cudaSuccess;
    for (int b = 0; b < 2; ++b) {
      if (in[b]) cudaFreeHost(in[b]);
      if (out[b]) cudaFreeHost(out[b]);
      if (ev[b]) cudaEventDestroy(ev[b]);
      in[b] = nullptr;
      out[b] = nullptr;
      ev[b] = nullptr;
    }
    dev = -1;
    for (int b = 0; b < 2; ++b) {
      cudaError_t e = cudaMallocHost(&in[b], kChunk * 12);
      if (e == cudaSuccess) e = cudaMallocHost(&out[b], kChunk * 8);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    dev = device;
    return cudaSuccess;
  }
};

}  // namespace

extern "C" int ft_reschedule_costs_dev(const ft_comm_profile* prof, int32_t n_tensors,
                                       const int32_t* ndims, const int64_t* dims,
                                       const int64_t* elem_bytes, int64_t n_q,
                                       const int32_t* q_tensor, const int32_t* q_from,
                                       const int32_t* q_to, int64_t* t_out, void* stream) {
  if (n_q < 0 || (n_q > 0 && (!q_tensor || !q_from || !q_to || !t_out))) return FT_EINVAL;
  std::vector<TensorDesc> td;
  std::vector<int32_t> states;
  int64_t dist_total;
  int max_s;
  int rc = plan_tensors(prof, n_tensors, ndims, dims, elem_bytes, td, states, dist_total, max_s);
  if (rc != FT_OK) return rc;
  if (n_q == 0) return FT_OK;
  if (n_tensors == 0) return FT_EINVAL;
  Pool& P = pool_for_device();
  std::lock_guard<std::mutex> lk(P.mu);
  cudaStream_t st = (cudaStream_t)stream;
  const bool prof_on = g_profile.load() != 0;
  if (prof_on && !P.ev[0])
    for (int i = 0; i < 4; ++i) CG_CHECK(cudaEventCreate(&P.ev[i]));
  Launch L;
  if (prof_on) CG_CHECK(cudaEventRecord(P.ev[0], st));
  rc = launch_apsp(P, prof, td, states, dist_total, max_s, st, L);
  if (rc != FT_OK) return rc;
  if (prof_on) {
    CG_CHECK(cudaEventRecord(P.ev[1], st));
    CG_CHECK(cudaEventRecord(P.ev[2], st));
  }
  rc = launch_gather(L, n_q, q_tensor, q_from, q_to, t_out, st);
  if (rc != FT_OK) return rc;
  if (prof_on) CG_CHECK(cudaEventRecord(P.ev[3], st));
  rc = finish(L, st);
  if (rc == FT_OK && prof_on) {
    CG_CHECK(cudaEventElapsedTime(&P.last_ms[0], P.ev[0], P.ev[1]));
    CG_CHECK(cudaEventElapsedTime(&P.last_ms[1], P.ev[2], P.ev[3]));
  }
  return rc;
}

extern "C" int ft_costgen_profile(int32_t on) {
  g_profile.store(on != 0);
  return FT_OK;
}

extern "C" int ft_costgen_last_times(float* apsp_ms, float* gather_ms) {
  if (!apsp_ms || !gather_ms) return FT_EINVAL;
  Pool& P = pool_for_device();
  std::lock_guard<std::mutex> lk(P.mu);
  *apsp_ms = P.last_ms[0];
  *gather_ms = P.last_ms[1];
  return FT_OK;
}

extern "C" int ft_reschedule_costs(const ft_comm_profile* prof, int32_t n_tensors,
                                   const int32_t* ndims, const int64_t* dims,
                                   const int64_t* elem_bytes, int64_t n_q, const int32_t* q_tensor,
                                   const int32_t* q_from, const int32_t* q_to, int64_t* t_out) {
  if (n_q < 0 || (n_q > 0 && (!q_tensor || !q_from || !q_to || !t_out))) return FT_EINVAL;
  std::vector<TensorDesc> td;
  std::vector<int32_t> states;
  int64_t dist_total;
  int max_s;
  int rc = plan_tensors(prof, n_tensors, ndims, dims, elem_bytes, td, states, dist_total, max_s);
  if (rc != FT_OK) return rc;
  if (n_q == 0) return FT_OK;
  if (n_tensors == 0) return FT_EINVAL;
  Pool& P = pool_for_device();
  std::lock_guard<std::mutex> lk(P.mu);
  int dev = 0;
  CG_CHECK(cudaGetDevice(&dev));
  static Staging stage_by_dev[64];
  Staging& SG = stage_by_dev[dev & 63];
  CG_CHECK(SG.init(dev));
  void *dq, *dout;
  CG_CHECK(P.get(5, (size_t)n_q * 12, &dq));
  CG_CHECK(P.get(6, (size_t)n_q * 8, &dout));
  int32_t* dqt = (int32_t*)dq;
  int64_t* dO = (int64_t*)dout;
  cudaStream_t st = cudaStreamPerThread;
  Launch L;
  // The APSP needs only the plan: it runs while the queries stream in.
  rc = launch_apsp(P, prof, td, states, dist_total, max_s, st, L);
  if (rc != FT_OK) return rc;
  // Chunk pipeline through pinned staging: host copies of chunk i overlap
  // the DMA / gather of chunk i-1; results drain two chunks behind.
  const int64_t nch = (n_q + kChunk - 1) / kChunk;
  auto drain = [&](int64_t i) -> int {
    const int b = (int)(i & 1);
    const int64_t lo = i * kChunk, n = std::min(kChunk, n_q - lo);
    CG_CHECK(cudaEventSynchronize(SG.ev[b]));
    par_memcpy(t_out + lo, SG.out[b], n * 8);
    return FT_OK;
  };
  for (int64_t i = 0; i < nch; ++i) {
    const int b = (int)(i & 1);
    if (i >= 2 && (rc = drain(i - 2)) != FT_OK) return rc;
    const int64_t lo = i * kChunk, n = std::min(kChunk, n_q - lo);
    int32_t* in = SG.in[b];
    par_memcpy(in, q_tensor + lo, n * 4);
    par_memcpy(in + n, q_from + lo, n * 4);
    par_memcpy(in + 2 * n, q_to + lo, n * 4);
    int32_t* d = dqt + 3 * lo;
    CG_CHECK(cudaMemcpyAsync(d, in, n * 12, cudaMemcpyHostToDevice, st));
    rc = launch_gather(L, n, d, d + n, d + 2 * n, dO + lo, st);
    if (rc != FT_OK) return rc;
    CG_CHECK(cudaMemcpyAsync(SG.out[b], dO + lo, n * 8, cudaMemcpyDeviceToHost, st));
    CG_CHECK(cudaEventRecord(SG.ev[b], st));
  }
  for (int64_t i = std::max<int64_t>(0, nch - 2); i < nch; ++i)
    if ((rc = drain(i)) != FT_OK) return rc;
  rc = finish(L, st);
  if (rc != FT_OK) return rc;
  return FT_OK;
}

extern "C" int ft_sync_costs(const ft_comm_profile* prof, int32_t n_tensors, const int32_t* ndims,
                             const int64_t* dims, const int64_t* elem_bytes, int64_t n_q,
                             const int32_t* q_tensor, const int32_t* q_state, int64_t* m_out,
                             int64_t* t_out) {
  if (n_q < 0 || (n_q > 0 && (!q_tensor || !q_state || !m_out || !t_out))) return FT_EINVAL;
  std::vector<TensorDesc> td;
  std::vector<int32_t> states;
  int64_t dist_total;
  int max_s;
  int rc = plan_tensors(prof, n_tensors, ndims, dims, elem_bytes, td, states, dist_total, max_s);
  if (rc != FT_OK) return rc;
  for (const TensorDesc& t : td)
    if (t.total > (int64_t(1) << (prof->P - 1))) return FT_EOVERFLOW;
  if (n_q == 0) return FT_OK;
  if (n_tensors == 0) return FT_EINVAL;
  DevBufs B;
  ft_comm_profile* dp;
  TensorDesc* dtd;
  int32_t *dst, *dq, *dbad;
  int64_t *dm, *dt;
  CG_CHECK(B.alloc(&dp, 1));
  CG_CHECK(B.alloc(&dtd, td.size()));
  CG_CHECK(B.alloc(&dst, states.size()));
  CG_CHECK(B.alloc(&dq, 2 * n_q));
  CG_CHECK(B.alloc(&dm, n_q));
  CG_CHECK(B.alloc(&dt, n_q));
  CG_CHECK(B.alloc(&dbad, 1));
  CG_CHECK(cudaMemcpy(dp, prof, sizeof(*prof), cudaMemcpyHostToDevice));
  CG_CHECK(cudaMemcpy(dtd, td.data(), td.size() * sizeof(TensorDesc), cudaMemcpyHostToDevice));
  CG_CHECK(cudaMemcpy(dst, states.data(), states.size() * 4, cudaMemcpyHostToDevice));
  CG_CHECK(cudaMemcpy(dq, q_tensor, n_q * 4, cudaMemcpyHostToDevice));
  CG_CHECK(cudaMemcpy(dq + n_q, q_state, n_q * 4, cudaMemcpyHostToDevice));
  CG_CHECK(cudaMemset(dbad, 0, 4));
  k_cg_sync<<<grid_for(n_q), 256>>>(dp, dtd, (int32_t)td.size(), dst, n_q, dq, dq + n_q, dm, dt,
                                    dbad);
  CG_CHECK(cudaGetLastError());
  int32_t bad = 0;
  CG_CHECK(cudaMemcpy(&bad, dbad, 4, cudaMemcpyDeviceToHost));
  if (bad) return FT_EINVAL;
  CG_CHECK(cudaMemcpy(m_out, dm, n_q * 8, cudaMemcpyDeviceToHost));
  CG_CHECK(cudaMemcpy(t_out, dt, n_q * 8, cudaMemcpyDeviceToHost));
  return FT_OK;
}
