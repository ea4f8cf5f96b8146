// ft_step.cu -- one FT step on the GPU: plan (K0), per-level product +
// dominance pre-filter (K1), bucket sort (K2), Alg.1 sweep (K3), compaction
// (K4), final gather.  See ft_kernels.cuh for the algorithm and DESIGN.md.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>
#include <cooperative_groups/scan.h>

#include "ft_kernels.cuh"
#include "ft_step.h"

namespace ftk {

#ifndef DW_GEN_UNROLL
#define DW_GEN_UNROLL 1  // k_direct_warp: rows generated per unrolled step (A/B builds)
#endif
constexpr int kDwGenUnroll = DW_GEN_UNROLL;

// Launches of the per-level pipeline: with programmatic stream serialisation
// (FT_PDL_ENTRY in every kernel launched here) unless FT_PDL=0.
static bool g_pdl = true;
__constant__ bool g_bskip = true;  // k_blocks: drop blocks dominated as a whole (FT_BLOCK_SKIP=0: keep)
__constant__ bool g_fence = true;  // k_filter: warp-cooperative G lower bound (FT_FENCE=0: per-lane gallop)

template <typename... KArgs, typename... Args>
static inline void launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          Args... args) {
  if (!g_pdl) {
    k<<<grid, block, smem, st>>>(args...);
    return;
  }
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, args...);
}

// ---------------------------------------------------------------------------
// Generic exclusive scan: out[i] = sum_{j<i} in[j] for i in [0, n]; n read
// from *n_dev when given (device-resident counts), else n_host.

constexpr int SCAN_NT = 256, SCAN_ITEMS = 8, SCAN_TILE = SCAN_NT * SCAN_ITEMS;
// scratch layout of a scan over <= n_cap elements: tile states, then the tile counter
__host__ __device__ inline int64_t ntiles_cap_slot(int64_t n_cap) { return (n_cap + SCAN_TILE - 1) / SCAN_TILE; }

// Segment runs the filter path at this level (its direct level is deeper;
// SPECIAL_LEVEL segments are handled by k_node_shared).
__device__ __forceinline__ bool is_filter(int32_t d, int level) {
  return d > level && d < SPECIAL_LEVEL;
}

// Single-pass scan with decoupled look-back: CTAs take tiles in order from
// an atomic counter, publish their tile sum (AGG) and, once the exclusive
// prefix is known, the inclusive prefix (PREF) in one 64-bit word
// (flag << 62 | value); warp 0 looks back 32 predecessors at a time.  The
// tile states and the two counters are zeroed by a memset before each scan.
#define SC_AGG (1ull << 62)
#define SC_PREF (2ull << 62)
#define SC_VAL ((1ull << 62) - 1)

// Element loaders for the scan: a plain array, or a functor that computes
// the element (and stores it for later kernels) while the scan reads it.
// load(): the thread's N elements (0 past n); keep(): stores the loader
// makes for later kernels, issued after the tile's loads.
template <typename T>
struct LoadArr {
  const T* p;
  template <int N>
  __device__ __forceinline__ void load(int64_t base, int64_t n, long long (&v)[N]) const {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = base + i < n ? (long long)p[base + i] : 0;
  }
  template <int N>
  __device__ __forceinline__ void keep(int64_t, int64_t, const long long (&)[N]) const {}
};

// Optional per-element epilogue of the scan: post(i, exclusive prefix, value).
struct NoPost {
  __device__ __forceinline__ void operator()(int64_t, long long, long long) const {}
};

template <typename Load, typename Post = NoPost>
__global__ void __launch_bounds__(SCAN_NT) k_scan1(Load ld, const int64_t* n_dev, int64_t n_host,
                                                   int64_t* out, unsigned long long* state,
                                                   Post post = Post()) {
  FT_PDL_ENTRY();
  __shared__ long long sh[33];
  __shared__ int64_t s_tile;
  __shared__ long long s_pre;
  const int64_t n = n_dev ? min(*n_dev, n_host) : n_host;
  const int64_t ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  unsigned long long* ctr = state + ntiles_cap_slot(n_host);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (ntiles == 0 && blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
  for (;;) {
    if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(ctr, 1ull);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= ntiles) break;
    const int64_t base = tile * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    long long v[SCAN_ITEMS];
    ld.load(base, n, v);
    long long sum = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) sum += v[i];
    long long tot;
    long long ex = block_excl_sum<SCAN_NT>(sum, sh, &tot);
    if (wid == 0) {
      long long pre = 0;
      if (tile == 0) {
        if (lane == 0) atomicExch(state + tile, SC_PREF | (unsigned long long)tot);
      } else {
        if (lane == 0) atomicExch(state + tile, SC_AGG | (unsigned long long)tot);
        int64_t p = tile - 1;
        for (;;) {
          const int64_t q = p - lane;  // lane 0 = nearest predecessor
          const unsigned long long x =
              q >= 0 ? *(volatile unsigned long long*)(state + q) : SC_PREF;
          const unsigned long long fl = x & ~SC_VAL;
          const unsigned pref = __ballot_sync(0xffffffffu, fl == SC_PREF);
          const unsigned ready = __ballot_sync(0xffffffffu, fl != 0);
          const int fp = pref ? __ffs(pref) - 1 : 32;  // nearest inclusive prefix
          const unsigned need = fp == 32 ? 0xffffffffu : (fp == 31 ? 0xffffffffu : ((2u << fp) - 1u));
          if ((ready & need) != need) continue;  // a predecessor has not published yet
          long long c = lane <= fp ? (long long)(x & SC_VAL) : 0;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
          pre += c;
          if (fp < 32) break;
          p -= 32;
        }
        if (lane == 0) atomicExch(state + tile, SC_PREF | (unsigned long long)(pre + tot));
      }
      if (lane == 0) s_pre = pre;
    }
    __syncthreads();
    ex += s_pre;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
      if (base + i < n) {
        out[base + i] = ex;
        post(base + i, ex, v[i]);
      }
      ex += v[i];
    }
    ld.keep(base, n, v);
    if (tile == ntiles - 1 && threadIdx.x == 0) out[n] = s_pre + tot;
    __syncthreads();  // s_tile / s_pre reuse
  }
  // the last CTA out leaves the tile states and counters zeroed for the next
  // scan (every CTA has finished its tiles and look-backs by then)
  __shared__ bool s_last;
  if (threadIdx.x == 0) s_last = atomicAdd(ctr + 1, 1ull) == (unsigned long long)gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    for (int64_t i = threadIdx.x; i < ntiles; i += SCAN_NT) state[i] = 0;
    if (threadIdx.x == 0) {
      ctr[0] = 0;
      ctr[1] = 0;
    }
  }
}

// Two independent exclusive scans of host-sized arrays in ONE launch (the
// per-level bucket-count and work-item scans): tiles [0, tA) belong to A,
// [tA, tA + tB) to B, each with its own decoupled look-back chain; state =
// [tA + tB tile states][tile counter][done counter], left zeroed.
template <typename LoadA, typename LoadB, typename PostB>
__global__ void __launch_bounds__(SCAN_NT) k_scan2(LoadA lda, int64_t nA, int64_t* outA, LoadB ldb, int64_t nB,
                                                   int64_t* outB, unsigned long long* state, PostB postb) {
  FT_PDL_ENTRY();
  __shared__ long long sh[33];
  __shared__ int64_t s_tile;
  __shared__ long long s_pre;
  const int64_t tA = (nA + SCAN_TILE - 1) / SCAN_TILE, tB = (nB + SCAN_TILE - 1) / SCAN_TILE;
  unsigned long long* ctr = state + tA + tB;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (tA == 0) outA[0] = 0;
    if (tB == 0) outB[0] = 0;
  }
  for (;;) {
    if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(ctr, 1ull);
    __syncthreads();
    const int64_t gt = s_tile;
    if (gt >= tA + tB) break;
    const bool isA = gt < tA;
    const int64_t tile = isA ? gt : gt - tA, n = isA ? nA : nB, ntiles = isA ? tA : tB;
    unsigned long long* st = isA ? state : state + tA;
    int64_t* out = isA ? outA : outB;
    const int64_t base = tile * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    long long v[SCAN_ITEMS];
    if (isA) lda.load(base, n, v);
    else ldb.load(base, n, v);
    long long sum = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) sum += v[i];
    long long tot;
    long long ex = block_excl_sum<SCAN_NT>(sum, sh, &tot);
    if (wid == 0) {
      long long pre = 0;
      if (tile == 0) {
        if (lane == 0) atomicExch(st + tile, SC_PREF | (unsigned long long)tot);
      } else {
        if (lane == 0) atomicExch(st + tile, SC_AGG | (unsigned long long)tot);
        int64_t p = tile - 1;
        for (;;) {
          const int64_t q = p - lane;
          const unsigned long long x = q >= 0 ? *(volatile unsigned long long*)(st + q) : SC_PREF;
          const unsigned long long fl = x & ~SC_VAL;
          const unsigned pref = __ballot_sync(0xffffffffu, fl == SC_PREF);
          const unsigned ready = __ballot_sync(0xffffffffu, fl != 0);
          const int fp = pref ? __ffs(pref) - 1 : 32;
          const unsigned need = fp == 32 ? 0xffffffffu : (fp == 31 ? 0xffffffffu : ((2u << fp) - 1u));
          if ((ready & need) != need) continue;
          long long c = lane <= fp ? (long long)(x & SC_VAL) : 0;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
          pre += c;
          if (fp < 32) break;
          p -= 32;
        }
        if (lane == 0) atomicExch(st + tile, SC_PREF | (unsigned long long)(pre + tot));
      }
      if (lane == 0) s_pre = pre;
    }
    __syncthreads();
    ex += s_pre;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
      if (base + i < n) {
        out[base + i] = ex;
        if (!isA) postb(base + i, ex, v[i]);
      }
      ex += v[i];
    }
    if (isA) lda.keep(base, n, v);
    else ldb.keep(base, n, v);
    if (tile == ntiles - 1 && threadIdx.x == 0) out[n] = s_pre + tot;
    __syncthreads();
  }
  __shared__ bool s_last;
  if (threadIdx.x == 0) s_last = atomicAdd(ctr + 1, 1ull) == (unsigned long long)gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    for (int64_t i = threadIdx.x; i < tA + tB; i += SCAN_NT) state[i] = 0;
    if (threadIdx.x == 0) {
      ctr[0] = 0;
      ctr[1] = 0;
    }
  }
}

template <typename LoadA, typename LoadB, typename PostB>
void scan2_excl_fn(LoadA lda, int64_t nA, int64_t* outA, LoadB ldb, int64_t nB, int64_t* outB, int64_t* tmp,
                   cudaStream_t st, PostB postb) {
  const int64_t tiles = (nA + SCAN_TILE - 1) / SCAN_TILE + (nB + SCAN_TILE - 1) / SCAN_TILE;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 148 * 4));
  launch(k_scan2<LoadA, LoadB, PostB>, dim3(grid), dim3(SCAN_NT), 0, st, lda, nA, outA, ldb, nB, outB,
                                                          (unsigned long long*)tmp, postb);
}

// tmp: >= scan_tmp_elems(n_cap) int64 slots, zero on first use (`fresh`
// zeroes it here); every scan leaves it zeroed again.
template <typename Load, typename Post = NoPost>
void scan_excl_fn(Load ld, int64_t* out, const int64_t* n_dev, int64_t n_cap, int64_t* tmp,
                  cudaStream_t st, bool fresh = false, Post post = Post()) {
  const int64_t tiles = (n_cap + SCAN_TILE - 1) / SCAN_TILE;
  if (fresh) cudaMemsetAsync(tmp, 0, sizeof(int64_t) * (size_t)(ntiles_cap_slot(n_cap) + 2), st);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 148 * 4));
  launch(k_scan1<Load, Post>, dim3(grid), dim3(SCAN_NT), 0, st, ld, n_dev, n_cap, out, (unsigned long long*)tmp,
         post);
}

template <typename TIn>
void scan_excl(const TIn* in, int64_t* out, const int64_t* n_dev, int64_t n_cap, int64_t* tmp,
               cudaStream_t st, bool fresh = false) {
  scan_excl_fn(LoadArr<TIn>{in}, out, n_dev, n_cap, tmp, st, fresh);
}

// ---------------------------------------------------------------------------
// K0: plan.  One thread per output segment: block offsets relative to the
// segment (ids, R6), sample sizes per level, the level at which the segment
// is small enough for the direct path.

constexpr int PLAN_BLK_CACHE = 128;  // factor sizes of a segment's blocks cached per warp (k_plan)

__device__ __forceinline__ void plan_seg(const BatchDev& B, int64_t gs, int j, int32_t* seg_d, int32_t* seg_n,
                                         int64_t* blk_rel, int64_t* seg_tuples, StepHdr* hdr,
                                         unsigned long long& sh_D, unsigned long long& sh_tuples,
                                         unsigned long long* sh_filter,
                                         unsigned long long* sh_direct, int (*wn)[3]) {
  // one warp per local output segment (gs, of step j); lanes stride over its blocks
  const int lane = threadIdx.x & 31;
  const StepDev& s = B.steps[j];
  const int64_t li = gs - B.seg_base[j];
  const int64_t sg = s.seg_lo + li;
  int64_t* rel_out = blk_rel + B.blk_base[j] + li * s.nblk;
  // shared-order node path (k_node_pack / k_node_shared): Y, Z singletons, so
  // n = sum_k |X_{w,k}| = X.off[(w+1)K_i] - X.off[w K_i] for every p of row w
  if (s.node_shared && s.nblk <= NS_MAXBLK && s.KB == s.nblk) {
    const int64_t w = sg / s.KC;
    const int64_t rel = s.X.off[(w + 1) * s.KB] - s.X.off[w * s.KB];
    if (rel <= NS_CAP) {
      if (lane == 0) {
        seg_d[gs] = SPECIAL_LEVEL;
        seg_n[gs] = (int32_t)rel;
        seg_tuples[gs] = rel;
        atomicAdd(&sh_tuples, (unsigned long long)rel);
        atomicAdd(&sh_direct[0], (unsigned long long)rel);  // level-0 pool capacity
      }
      return;
    }
  }
  // level 0: block offsets relative to the segment (ids, R6) and the tuple count
  int64_t rel = 0;
  for (int64_t k0 = 0; k0 < s.nblk; k0 += 32) {
    const int64_t k = k0 + lane;
    int64_t nk = 0;
    if (k < s.nblk) {
      const Blk b = load_blk(s, sg, k);
      nk = b.n[0] * b.n[1] * b.n[2];
      if (k < PLAN_BLK_CACHE) {  // the level loop below reuses the factor sizes
        wn[k][0] = (int)min(b.n[0], (int64_t)INT32_MAX);
        wn[k][1] = (int)min(b.n[1], (int64_t)INT32_MAX);
        wn[k][2] = (int)min(b.n[2], (int64_t)INT32_MAX);
      }
    }
    const int64_t inc = warp_incl_sum<long long>(nk);
    if (k < s.nblk) rel_out[k] = rel + inc - nk;
    rel += __shfl_sync(0xffffffffu, inc, 31);
  }
  // shared-order node path (k_node_shared): every segment of row w has the same
  // n = sum_k |X_{w,k}| (Y, Z singletons)
  if (s.node_shared && rel <= NS_CAP && s.nblk <= NS_MAXBLK) {
    if (lane == 0) {
      seg_d[gs] = SPECIAL_LEVEL;
      seg_n[gs] = (int32_t)rel;
      seg_tuples[gs] = rel;
      atomicAdd(&sh_tuples, (unsigned long long)rel);
      atomicAdd(&sh_direct[0], (unsigned long long)rel);  // level-0 pool capacity
    }
    return;
  }
  // levels l = 0, 1, ...: sample size until it fits the direct path.  A
  // segment of more than cdirect blocks never fits (every block keeps >= 1
  // sampled tuple): once the sample stops shrinking, level d has no direct
  // work and an empty output, and level d-1 filters its whole sample against
  // the empty staircase (one bucket per segment, exact in the bucket sorts).
  int d = -1;
  bool empty = false;
  unsigned long long samp = (unsigned long long)rel, prev = ~0ull;
  for (int l = 0; l <= LMAX; ++l) {
    if (l > 0) {
      const int sh = level_shift(l, B.slog0, B.slog);
      unsigned long long loc = 0;
      __syncwarp();
      for (int64_t k = lane; k < s.nblk; k += 32) {
        int64_t n0, n1, n2;
        if (k < PLAN_BLK_CACHE) {
          n0 = wn[k][0];
          n1 = wn[k][1];
          n2 = wn[k][2];
        } else {
          const Blk b = load_blk(s, sg, k);
          n0 = b.n[0];
          n1 = b.n[1];
          n2 = b.n[2];
        }
        loc += (unsigned long long)(samp_cnt(n0, sh) * samp_cnt(n1, sh) * samp_cnt(n2, sh));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) loc += __shfl_xor_sync(0xffffffffu, loc, o);
      samp = loc;
    }
    if (samp <= (unsigned long long)B.cdirect && s.nblk <= B.cdirect) {
      d = l;
      break;
    }
    if (l > 0 && (samp >= prev || l == LMAX)) {
      d = l;
      empty = true;
      break;
    }
    if (lane == 0) atomicAdd(&sh_filter[l], samp);  // level l runs the filter path
    prev = samp;
  }
  if (empty) samp = 0;
  if (lane == 0) {
    if (d < 0) {
      atomicExch(&hdr->bad, 1ull);
      d = LMAX;
    }
    seg_d[gs] = d;
    seg_n[gs] = (int32_t)min(samp, (unsigned long long)INT32_MAX);
    seg_tuples[gs] = rel;
    atomicMax(&sh_D, (unsigned long long)d);
    atomicAdd(&sh_tuples, (unsigned long long)rel);
    atomicAdd(&sh_direct[d], samp);
  }
}

constexpr int PLAN_BASE_CAP = 2048;  // step bases cached in shared memory by k_plan

__global__ void __launch_bounds__(256) k_plan(BatchDev B, int32_t* seg_d, int32_t* seg_n,
                                              int64_t* blk_rel, int64_t* seg_tuples,
                                              StepHdr* hdr) {
  FT_PDL_ENTRY();
  __shared__ unsigned long long sh_D, sh_tuples, sh_filter[LMAX + 1], sh_direct[LMAX + 1];
  __shared__ int64_t s_base[PLAN_BASE_CAP + 1];
  __shared__ int s_wn[8][PLAN_BLK_CACHE][3];  // per warp (256 threads)
  if (threadIdx.x == 0) {
    sh_D = 0;
    sh_tuples = 0;
  }
  if (threadIdx.x <= LMAX) {
    sh_filter[threadIdx.x] = 0;
    sh_direct[threadIdx.x] = 0;
  }
  // step bases in shared memory (a 9-level global binary search per segment
  // dominated node waves with ~1e6 segments); each warp also remembers the
  // step range of its previous segment
  const bool cached = B.nsteps <= PLAN_BASE_CAP;
  if (cached)
    for (int i = threadIdx.x; i <= B.nsteps; i += blockDim.x) s_base[i] = B.seg_base[i];
  __syncthreads();
  // Warps take 32 consecutive segments: each lane first tries the
  // shared-order node shortcut for its own segment (one thread suffices:
  // n = X.off[(w+1)K_i] - X.off[w K_i]), then the warp plans the remaining
  // segments one at a time (plan_seg, lanes over blocks).
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t wglob = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int j = 0;
  int64_t sb = 0, se = -1;
  unsigned long long my_tuples = 0;
  // cw segments per warp pass: 32 when segments are plentiful (node waves,
  // ~1e6 segments), 1 when few (LDP waves: every warp plans its own)
  int64_t cw = B.nseg / nwarps;
  cw = cw < 1 ? 1 : (cw > 32 ? 32 : cw);
  for (int64_t g0 = wglob * cw; g0 < B.nseg; g0 += nwarps * cw) {
    const int64_t gs = lane < cw ? g0 + lane : B.nseg;
    bool done = false;
    if (gs < B.nseg) {
      if (gs < sb || gs >= se) {
        if (cached) {
          int lo = 0, hi = B.nsteps;
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_base[mid] <= gs) lo = mid;
            else hi = mid;
          }
          j = lo;
          sb = s_base[j];
          se = s_base[j + 1];
        } else {
          j = find_base(B.seg_base, B.nsteps, gs);
          sb = B.seg_base[j];
          se = B.seg_base[j + 1];
        }
      }
      const StepDev& s = B.steps[j];
      if (s.node_shared && s.nblk <= NS_MAXBLK && s.KB == s.nblk) {
        const int64_t w = (s.seg_lo + (gs - sb)) / s.KC;
        const int64_t rel = s.X.off[(w + 1) * s.KB] - s.X.off[w * s.KB];
        if (rel <= NS_CAP) {
          seg_d[gs] = SPECIAL_LEVEL;
          seg_n[gs] = (int32_t)rel;
          seg_tuples[gs] = rel;
          my_tuples += (unsigned long long)rel;
          done = true;
        }
      }
    }
    unsigned todo = __ballot_sync(0xffffffffu, gs < B.nseg && !done);  // lanes >= cw: gs = nseg
    while (todo) {
      const int b = __ffs(todo) - 1;
      todo &= todo - 1;
      const int jb = __shfl_sync(0xffffffffu, j, b);
      plan_seg(B, g0 + b, jb, seg_d, seg_n, blk_rel, seg_tuples, hdr, sh_D, sh_tuples, sh_filter, sh_direct,
               s_wn[threadIdx.x >> 5]);
      __syncwarp();  // s_wn reuse by the next segment
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) my_tuples += __shfl_xor_sync(0xffffffffu, my_tuples, o);
  if (lane == 0 && my_tuples) {
    atomicAdd(&sh_tuples, my_tuples);
    atomicAdd(&sh_direct[0], my_tuples);  // level-0 pool capacity
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (sh_D) atomicMax(&hdr->D, sh_D);
    if (sh_tuples) atomicAdd(&hdr->tuples, sh_tuples);
  }
  if (threadIdx.x <= LMAX) {
    if (sh_filter[threadIdx.x]) atomicAdd(&hdr->filter_samp[threadIdx.x], sh_filter[threadIdx.x]);
    if (sh_direct[threadIdx.x]) atomicAdd(&hdr->direct_samp[threadIdx.x], sh_direct[threadIdx.x]);
  }
}

// ---------------------------------------------------------------------------
// Direct path: the whole level-l sample of a segment (<= C_DIRECT tuples) in
// one CTA: product -> bitonic sort on (m,t,id) -> Alg.1 sweep -> compaction.

// Register-blocked CTA sort + Alg. 1 for N = 32 R x (DIRECT_NT / 32) tuples:
// element e = warp*32R + r*32 + lane lives in registers; bitonic stages with
// j < 32 use shuffles, j < 32R register swaps, and only the log2(#warps)
// cross-warp stages per merge exchange through shared memory (x*).  The sweep
// is warp scans with a cross-warp carry; survivors are written by ballot.
template <int R, int JR>
__device__ __forceinline__ void cta_rows_xchg(int64_t (&m)[R], int64_t (&t)[R], uint64_t (&id)[R], int k,
                                              int eb) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (r & JR) continue;
    const int r2 = r | JR;
    const bool up = ((eb | (r << 5)) & k) == 0;
    const bool gt = key_lt(m[r2], t[r2], id[r2], m[r], t[r], id[r]);
    if (gt == up) {
      int64_t a = m[r]; m[r] = m[r2]; m[r2] = a;
      a = t[r]; t[r] = t[r2]; t[r2] = a;
      uint64_t b = id[r]; id[r] = id[r2]; id[r2] = b;
    }
  }
}

template <int R>
__device__ __forceinline__ void cta_bitonic_regs(int64_t (&m)[R], int64_t (&t)[R], uint64_t (&id)[R],
                                                 int64_t* xm, int64_t* xt, uint64_t* xid) {
  constexpr int NW = DIRECT_NT / 32, N = 32 * R * NW;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int eb = wid * 32 * R;
#pragma unroll 1
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32 * R) {  // partner in another warp
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int e = eb + (r << 5) + lane;
          xm[e] = m[r];
          xt[e] = t[r];
          xid[e] = id[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int e = eb + (r << 5) + lane, p = e ^ j;
          const int64_t pm = xm[p], pt = xt[p];
          const uint64_t pi = xid[p];
          const bool up = (e & k) == 0, lower = (e & j) == 0;
          const bool p_lt = key_lt(pm, pt, pi, m[r], t[r], id[r]);
          if ((lower == up) ? p_lt : !p_lt) {
            m[r] = pm;
            t[r] = pt;
            id[r] = pi;
          }
        }
        __syncthreads();
      } else if (j >= 32) {
        const int jr = j >> 5;
        if (jr == 1) cta_rows_xchg<R, 1>(m, t, id, k, eb);
        else if (R >= 4 && jr == 2) cta_rows_xchg<R, (R >= 4 ? 2 : 1)>(m, t, id, k, eb);
        else if (R >= 8 && jr == 4) cta_rows_xchg<R, (R >= 8 ? 4 : 1)>(m, t, id, k, eb);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int64_t pm = __shfl_xor_sync(0xffffffffu, m[r], j);
          const int64_t pt = __shfl_xor_sync(0xffffffffu, t[r], j);
          const uint64_t pi = __shfl_xor_sync(0xffffffffu, id[r], j);
          const int e = eb + (r << 5) + lane;
          const bool up = (e & k) == 0, lower = (e & j) == 0;
          const bool p_lt = key_lt(pm, pt, pi, m[r], t[r], id[r]);
          if ((lower == up) ? p_lt : !p_lt) {
            m[r] = pm;
            t[r] = pt;
            id[r] = pi;
          }
        }
      }
    }
  }
}

template <int R, int JR>
__device__ __forceinline__ void cta_keys_rows(uint64_t (&k)[R], int kk, int eb) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (r & JR) continue;
    const int r2 = r | JR;
    if (r2 >= R) continue;
    const bool up = ((eb | (r << 5)) & kk) == 0;
    const uint64_t a = k[r], b = k[r2];
    const bool sw = up ? (b < a) : (a < b);
    k[r] = sw ? b : a;
    k[r2] = sw ? a : b;
  }
}

// Register-blocked CTA bitonic on single 64-bit keys (same layout as
// cta_bitonic_regs); xk: N keys of shared memory for the cross-warp stages.
template <int R>
__device__ __forceinline__ void cta_bitonic_keys(uint64_t (&k)[R], uint64_t* xk) {
  constexpr int NW = DIRECT_NT / 32, N = 32 * R * NW;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int eb = wid * 32 * R;
#pragma unroll 1
  for (int kk = 2; kk <= N; kk <<= 1) {
#pragma unroll 1
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j >= 32 * R) {  // partner in another warp
#pragma unroll
        for (int r = 0; r < R; ++r) xk[eb + (r << 5) + lane] = k[r];
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int e = eb + (r << 5) + lane;
          const uint64_t pk = xk[e ^ j];
          const bool up = (e & kk) == 0, lower = (e & j) == 0;
          k[r] = (lower == up) ? (pk < k[r] ? pk : k[r]) : (pk > k[r] ? pk : k[r]);
        }
        __syncthreads();
      } else if (j >= 32) {  // rows r, r | jr of this thread (compile-time distances)
        const int jr = j >> 5;
        if (jr == 1) cta_keys_rows<R, 1>(k, kk, eb);
        else if (R >= 4 && jr == 2) cta_keys_rows<R, (R >= 4 ? 2 : 1)>(k, kk, eb);
        else if (R >= 8 && jr == 4) cta_keys_rows<R, (R >= 8 ? 4 : 1)>(k, kk, eb);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint64_t pk = __shfl_xor_sync(0xffffffffu, k[r], j);
          const int e = eb + (r << 5) + lane;
          const bool up = (e & kk) == 0, lower = (e & j) == 0;
          k[r] = (lower == up) ? (pk < k[r] ? pk : k[r]) : (pk > k[r] ? pk : k[r]);
        }
      }
    }
  }
}

template <int R, typename Gen>
__device__ __forceinline__ void cta_sort_sweep(int n, Gen& gen, int64_t* xm, int64_t* xt, uint64_t* xid,
                                               uint64_t* xk, long long* sh, const LevelDev& L,
                                               int64_t gs, int64_t* s_start, int kspan) {
  constexpr int NW = DIRECT_NT / 32;
  constexpr int EB = R >= 8 ? 11 : 10;  // bits of the element index e < N = 32 R NW
  constexpr uint64_t EM = (1ull << EB) - 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int eb = wid * 32 * R;
  int64_t m[R], t[R];
  uint64_t id[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    m[r] = INF;
    t[r] = INF;
    id[r] = ~0ull;
  }
  // Tuples are staged in x*; the sort runs on 64-bit keys ((m - m0) << EB | e)
  // (m0 = the sample's least m, e < N <= 2048) and t, id are gathered by e.
  // Frontier m grows with the eliminated subgraph (sums up to 2^60, R10), so
  // the packing is used only when the sample's m span fits in kspan (<= 53)
  // bits; otherwise, and when two tuples share m (the key order is then not
  // the (m, t, id) order), the staged tuples are sorted on the full key.
  long long lmin = INF, lmax = -1;
#pragma unroll 1
  for (int r = 0; r < R; ++r) {
    const int e = eb + (r << 5) + lane;
    if (e < n) {
      int64_t vm, vt;
      uint64_t vi;
      gen(e, vm, vt, vi);
      xm[e] = vm;
      xt[e] = vt;
      xid[e] = vi;
      lmin = vm < lmin ? vm : lmin;
      lmax = vm > lmax ? vm : lmax;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long a = __shfl_xor_sync(0xffffffffu, lmin, o), b = __shfl_xor_sync(0xffffffffu, lmax, o);
    lmin = a < lmin ? a : lmin;
    lmax = b > lmax ? b : lmax;
  }
  if (lane == 0) {
    sh[wid] = lmin;
    sh[NW + wid] = lmax;
  }
  __syncthreads();
  long long m0 = INF, m1 = -1;
  for (int w = 0; w < NW; ++w) {
    m0 = sh[w] < m0 ? sh[w] : m0;
    m1 = sh[NW + w] > m1 ? sh[NW + w] : m1;
  }
  const bool wide = ((unsigned long long)(m1 - m0) >> (kspan < 63 - EB ? kspan : 63 - EB)) != 0;
  uint64_t k[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = eb + (r << 5) + lane;
    k[r] = e < n ? ((uint64_t)(xm[e] - m0) << EB) | (uint64_t)e : ~0ull;
  }
  __syncthreads();  // sh reuse
  bool tie = false;
  if (!wide) {
    cta_bitonic_keys<R>(k, xk);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = eb + (r << 5) + lane;
      if (e < n) {
        const int src = (int)(k[r] & EM);
        m[r] = (int64_t)(k[r] >> EB) + m0;
        t[r] = xt[src];
        id[r] = xid[src];
      }
      uint64_t prev = __shfl_up_sync(0xffffffffu, k[r], 1);
      const uint64_t rowlast = __shfl_sync(0xffffffffu, k[r > 0 ? r - 1 : 0], 31);
      if (lane == 0) prev = r > 0 ? rowlast : ~0ull;
      if (e < n && prev != ~0ull && (prev >> EB) == (k[r] >> EB)) tie = true;
    }
    if (lane == 31) sh[wid] = (long long)(k[R - 1] >> EB);  // last key m of the warp (padding: all ones)
    __syncthreads();
    if (wid > 0 && lane == 0 && eb < n && (long long)(k[0] >> EB) == sh[wid - 1]) tie = true;
  }
  if (__syncthreads_or(tie || wide)) {  // exact sort on (m, t, id)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = eb + (r << 5) + lane;
      m[r] = e < n ? xm[e] : INF;
      t[r] = e < n ? xt[e] : INF;
      id[r] = e < n ? xid[e] : ~0ull;
    }
    __syncthreads();
    cta_bitonic_regs<R>(m, t, id, xm, xt, xid);
  }
  // Alg. 1: keep iff t < min of all earlier t (earlier warps via sh)
  long long wmin = INF;
#pragma unroll
  for (int r = 0; r < R; ++r) wmin = t[r] < wmin ? t[r] : wmin;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long u = __shfl_xor_sync(0xffffffffu, wmin, o);
    wmin = u < wmin ? u : wmin;
  }
  if (lane == 0) sh[wid] = wmin;
  __syncthreads();
  long long carry = INF;
  for (int w = 0; w < wid; ++w) carry = sh[w] < carry ? sh[w] : carry;
  unsigned bal[R];
  int cnt = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const long long inc = warp_incl_min(t[r]);
    long long ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = INF;
    const long long v = ex < carry ? ex : carry;
    bal[r] = __ballot_sync(0xffffffffu, eb + (r << 5) + lane < n && t[r] < v);
    const long long rowmin = __shfl_sync(0xffffffffu, inc, 31);
    carry = rowmin < carry ? rowmin : carry;
    cnt += __popc(bal[r]);
  }
  __syncthreads();  // sh reused for the per-warp counts
  if (lane == 0) sh[wid] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int w = 0; w < NW; ++w) tot += sh[w];
    const unsigned long long st0 = atomicAdd(L.out.cursor, (unsigned long long)tot);
    int64_t base = -1;
    if ((int64_t)(st0 + tot) > L.out.cap) atomicExch(&L.hdr->overflow, 1ull);
    else base = (int64_t)st0;
    atomicAdd(&L.hdr->out_total[L.level], (unsigned long long)tot);
    L.out.start[gs] = base;
    L.out.cnt[gs] = tot;
    *s_start = base;
    atomicAdd(&L.hdr->dreg, 1ull);
  }
  __syncthreads();
  const int64_t base = *s_start;
  if (base >= 0) {
    int64_t off = base;
    for (int w = 0; w < wid; ++w) off += sh[w];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if ((bal[r] >> lane) & 1u) {
        const int64_t d = off + __popc(bal[r] & ((1u << lane) - 1u));
        L.out.m[d] = m[r];
        L.out.t[d] = t[r];
        L.out.id[d] = id[r];
      }
      off += __popc(bal[r]);
    }
  }
  __syncthreads();  // sh / x* / s_start reuse
}

constexpr int DIRECT_MAXBLK = 128;  // per-block info cached in smem up to this many blocks
static size_t direct_smem(int cap) { return (size_t)cap * (3 * 8 + 4 + 4) + 8; }

__global__ void __launch_bounds__(DIRECT_NT, 3) k_direct(BatchDev B, LevelDev L) {
  FT_PDL_ENTRY();
  extern __shared__ int64_t dyn_direct[];  // capacity B.cdirect (runtime)
  int64_t* sm = dyn_direct;
  int64_t* stt = sm + B.cdirect;
  uint64_t* sid = (uint64_t*)(stt + B.cdirect);
  int* kf = (int*)(sid + B.cdirect);
  int* pre = kf + B.cdirect;  // [B.cdirect + 1]
  __shared__ int64_t bo[DIRECT_MAXBLK][3];  // factor offsets
  __shared__ int bn[DIRECT_MAXBLK][3];      // factor sizes
  __shared__ int bc[DIRECT_MAXBLK][3];      // sampled counts
  __shared__ long long sh[33];
  __shared__ int64_t s_start;
  __shared__ int64_t s_list[DIRECT_NT];
  __shared__ int s_nl;
  const int st = L.st;
  // one parallel pass over tw segments' seg_d picks this level's CTA-direct
  // segments (most waves have few among many)
  int64_t tw = B.nseg / ((int64_t)gridDim.x * 4);
  tw = tw < 1 ? 1 : (tw > DIRECT_NT ? DIRECT_NT : tw);
  // the CTA's segments are b, b + G, b + 2G, ... (G = grid; spreads a step's
  // heavy segments over CTAs), examined tw at a time
  for (int64_t t0 = 0; (int64_t)blockIdx.x + t0 * gridDim.x < B.nseg; t0 += tw) {
    if (threadIdx.x == 0) s_nl = 0;
    __syncthreads();
    {
      const int64_t g = (int64_t)blockIdx.x + (t0 + threadIdx.x) * gridDim.x;
      if (threadIdx.x < tw && g < B.nseg && L.seg_d[g] == L.level && L.seg_n[g] > L.warp2)
        s_list[atomicAdd(&s_nl, 1)] = g;
    }
    __syncthreads();
    const int nl = s_nl;
    for (int q = 0; q < nl; ++q) {
    const int64_t gs = s_list[q];
    if (L.hdr->overflow) return;
    const int j = find_base(B.seg_base, B.nsteps, gs);
    const StepDev& s = B.steps[j];
    const int64_t li = gs - B.seg_base[j];
    const int64_t sg = s.seg_lo + li;
    const int nblk = (int)s.nblk;
    const int64_t* rel = L.blk_rel + B.blk_base[j] + li * s.nblk;
    const bool cached = nblk <= DIRECT_MAXBLK;
    // block sample sizes -> inclusive prefix in pre[1..nblk]
    for (int k = threadIdx.x; k < nblk; k += DIRECT_NT) {
      Blk b = load_blk(s, sg, k);
      const int c0 = (int)samp_cnt(b.n[0], st), c1 = (int)samp_cnt(b.n[1], st),
                c2 = (int)samp_cnt(b.n[2], st);
      pre[k + 1] = c0 * c1 * c2;
      if (cached) {
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          bo[k][f] = b.o[f];
          bn[k][f] = (int)b.n[f];
        }
        bc[k][0] = c0;
        bc[k][1] = c1;
        bc[k][2] = c2;
      }
    }
    if (threadIdx.x == 0) pre[0] = 0;
    __syncthreads();
    {
      const int per = (nblk + DIRECT_NT - 1) / DIRECT_NT;
      const int lo = min(nblk, (int)threadIdx.x * per), hi = min(nblk, lo + per);
      long long loc = 0;
      for (int k = lo; k < hi; ++k) loc += pre[k + 1];
      long long tot;
      int off = (int)block_excl_sum<DIRECT_NT>(loc, sh, &tot);
      for (int k = lo; k < hi; ++k) {
        off += pre[k + 1];
        pre[k + 1] = off;
      }
      __syncthreads();
    }
    const int n = pre[nblk];
    int N = 1;
    while (N < n) N <<= 1;
    // tuple i of the level-l sample (block k = largest with pre[k] <= i)
    auto gen = [&](int i, int64_t& om, int64_t& ot, uint64_t& oid) {
      int lo = 0, hi = nblk;
      while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (pre[mid] <= i) lo = mid;
        else hi = mid;
      }
      const int k = lo;
      Blk b;
      int cy, cz;
      if (cached) {
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          b.o[f] = bo[k][f];
          b.n[f] = bn[k][f];
        }
        cy = bc[k][1];
        cz = bc[k][2];
      } else {
        b = load_blk(s, sg, k);
        cy = (int)samp_cnt(b.n[1], st);
        cz = (int)samp_cnt(b.n[2], st);
      }
      const int r = i - pre[k];  // < C_DIRECT: 32-bit index math
      const int jz = r % cz, q2 = r / cz, jy = q2 % cy, jx = q2 / cy;
      const int64_t x = samp_idx(jx, b.n[0], st), y = samp_idx(jy, b.n[1], st),
                    z = samp_idx(jz, b.n[2], st);
      make_tuple(s, b, rel[k], x, y, z, om, ot, oid);
    };
    if ((N == 2 * DIRECT_NT || N == 4 * DIRECT_NT || N == 8 * DIRECT_NT) && N <= B.cdirect) {
      uint64_t* xk = (uint64_t*)kf;  // kf + pre (>= 8 N bytes) are free after generation
      if (N == 2 * DIRECT_NT) cta_sort_sweep<2>(n, gen, sm, stt, sid, xk, sh, L, gs, &s_start, B.kspan);
      else if (N == 4 * DIRECT_NT) cta_sort_sweep<4>(n, gen, sm, stt, sid, xk, sh, L, gs, &s_start, B.kspan);
      else cta_sort_sweep<8>(n, gen, sm, stt, sid, xk, sh, L, gs, &s_start, B.kspan);
      continue;
    }
    for (int i = threadIdx.x; i < N; i += DIRECT_NT) {
      if (i < n) {
        gen(i, sm[i], stt[i], sid[i]);
      } else {
        sm[i] = INF;
        stt[i] = INF;
        sid[i] = ~0ull;
      }
    }
    __syncthreads();
    bitonic_smem<DIRECT_NT>(sm, stt, sid, N);
    const int cnt = alg1_sweep_smem<DIRECT_NT>(stt, n, INF, kf, sh);
    if (threadIdx.x == 0) {
      unsigned long long st0 = atomicAdd(L.out.cursor, (unsigned long long)cnt);
      if ((int64_t)(st0 + cnt) > L.out.cap) {
        atomicExch(&L.hdr->overflow, 1ull);
        s_start = -1;
      } else {
        s_start = (int64_t)st0;
      }
      atomicAdd(&L.hdr->out_total[L.level], (unsigned long long)cnt);
      L.out.start[gs] = s_start;
      L.out.cnt[gs] = cnt;
    }
    __syncthreads();
    const int64_t o = s_start;
    if (o >= 0)
      for (int i = threadIdx.x; i < n; i += DIRECT_NT)
        if (kf[i]) {
          int64_t d = o + kf[i] - 1;
          L.out.m[d] = sm[i];
          L.out.t[d] = stt[i];
          L.out.id[d] = sid[i];
        }
    __syncthreads();
    }
    __syncthreads();  // s_nl / s_list reuse
  }
}

// Direct path for small segments (<= WARP_DIRECT tuples): one warp, R rows of
// 32 tuples in registers (element e = r*32 + lane), bitonic sort on (m,t,id)
// by shuffles, Alg. 1 sweep by warp scans, ballot compaction.  No barriers.
// Stages run as runtime loops (only the R rows are unrolled): a fully
// unrolled network for R = 1..8 inlined into every caller made the kernels
// ~600 KB of SASS and instruction-fetch bound.
template <int R, int JR>
__device__ __forceinline__ void warp_bitonic_rows(int64_t (&m)[R], int64_t (&t)[R], uint64_t (&id)[R],
                                                  int k) {
  // partner rows r and r|JR (j = 32*JR >= 32; k >= 64 so `up` depends on r only)
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (r & JR) continue;
    const int r2 = r | JR;
    const bool up = ((r << 5) & k) == 0;
    const bool gt = key_lt(m[r2], t[r2], id[r2], m[r], t[r], id[r]);
    if (gt == up) {
      int64_t a = m[r]; m[r] = m[r2]; m[r2] = a;
      a = t[r]; t[r] = t[r2]; t[r2] = a;
      uint64_t b = id[r]; id[r] = id[r2]; id[r2] = b;
    }
  }
}

template <int R>
__device__ __forceinline__ void warp_bitonic(int64_t (&m)[R], int64_t (&t)[R], uint64_t (&id)[R]) {
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int k = 2; k <= R * 32; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int jr = j >> 5;
        if (jr == 1) warp_bitonic_rows<R, 1>(m, t, id, k);
        else if (R >= 4 && jr == 2) warp_bitonic_rows<R, (R >= 4 ? 2 : 1)>(m, t, id, k);
        else if (R >= 8 && jr == 4) warp_bitonic_rows<R, (R >= 8 ? 4 : 1)>(m, t, id, k);
        else if (R >= 16) warp_bitonic_rows<R, (R >= 16 ? 8 : 1)>(m, t, id, k);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int64_t pm = __shfl_xor_sync(0xffffffffu, m[r], j);
          const int64_t pt = __shfl_xor_sync(0xffffffffu, t[r], j);
          const uint64_t pi = __shfl_xor_sync(0xffffffffu, id[r], j);
          const int e = (r << 5) | lane;
          const bool up = (e & k) == 0, lower = (e & j) == 0;
          const bool p_lt = key_lt(pm, pt, pi, m[r], t[r], id[r]);
          // lower element of an ascending pair keeps the min, etc.
          const bool take_partner = (lower == up) ? p_lt : !p_lt;
          if (take_partner) {
            m[r] = pm;
            t[r] = pt;
            id[r] = pi;
          }
        }
      }
    }
  }
}

// Warp bitonic on single 64-bit keys, R rows of 32 (element e = r*32 + lane).
// Row exchanges (j >= 32) take the row distance as a template parameter so
// that every register-array index is a compile-time constant (a runtime
// index would put the array in local memory).
template <int R, int JR>
__device__ __forceinline__ void warp_keys_rows(uint64_t (&k)[R], int kk) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (r & JR) continue;
    const int r2 = r | JR;
    if (r2 >= R) continue;
    const bool up = ((r << 5) & kk) == 0;
    const uint64_t a = k[r], b = k[r2];
    const bool sw = up ? (b < a) : (a < b);
    k[r] = sw ? b : a;
    k[r2] = sw ? a : b;
  }
}

template <int R>
__device__ __forceinline__ void warp_bitonic_keys(uint64_t (&k)[R]) {
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int kk = 2; kk <= R * 32; kk <<= 1) {
#pragma unroll 1
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int jr = j >> 5;
        if (jr == 1) warp_keys_rows<R, 1>(k, kk);
        else if (R >= 4 && jr == 2) warp_keys_rows<R, (R >= 4 ? 2 : 1)>(k, kk);
        else if (R >= 8 && jr == 4) warp_keys_rows<R, (R >= 8 ? 4 : 1)>(k, kk);
        else if (R >= 16) warp_keys_rows<R, (R >= 16 ? 8 : 1)>(k, kk);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint64_t pk = __shfl_xor_sync(0xffffffffu, k[r], j);
          const int e = (r << 5) | lane;
          const bool up = (e & kk) == 0, lower = (e & j) == 0;
          k[r] = (lower == up) ? (pk < k[r] ? pk : k[r]) : (pk > k[r] ? pk : k[r]);
        }
      }
    }
  }
}

constexpr int WARP_BLK_CACHE = 64;
constexpr size_t DW_SMEM = 8 * 2 * WARP_DIRECT * 8;  // t/id staging of k_direct_warp  // block descriptors cached per warp

// Alg. 1 sweep over R rows of 32 sorted elements (element e = r*32 + lane,
// t[r] in order; padding t = INF) and ballot compaction into the level pool;
// out(r, d) writes element (r, lane) to pool slot d.
template <int R, typename Out>
__device__ __forceinline__ void warp_sweep_write(const LevelDev& L, int64_t gs, int n, const int64_t (&t)[R],
                                                 Out out) {
  const int lane = threadIdx.x & 31;
  long long carry = INF;
  unsigned keep = 0;  // bit r: element (r, lane) kept
  int cnt = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const long long inc = warp_incl_min(t[r]);
    long long ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = INF;
    const long long v = ex < carry ? ex : carry;
    const bool k = ((r << 5) | lane) < n && t[r] < v;
    keep |= (unsigned)k << r;
    const long long rowmin = __shfl_sync(0xffffffffu, inc, 31);
    carry = rowmin < carry ? rowmin : carry;
    cnt += __popc(__ballot_sync(0xffffffffu, k));
  }
  int64_t base = 0;
  if (lane == 0) {
    unsigned long long st0 = atomicAdd(L.out.cursor, (unsigned long long)cnt);
    if ((int64_t)(st0 + cnt) > L.out.cap) {
      atomicExch(&L.hdr->overflow, 1ull);
      base = -1;
    } else {
      base = (int64_t)st0;
    }
    atomicAdd(&L.hdr->out_total[L.level], (unsigned long long)cnt);
    L.out.start[gs] = base;
    L.out.cnt[gs] = cnt;
  }
  base = __shfl_sync(0xffffffffu, base, 0);
  if (base < 0) return;
  int off = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const bool k = (keep >> r) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, k);
    if (k) out(r, base + off + __popc(bal & ((1u << lane) - 1u)));
    off += __popc(bal);
  }
}

// Exact (m, t, id) warp bitonic over R rows of 32 elements that carry only
// (m, e): t and id of element e are staged in wt / wi and read only when two
// m values are equal (padding: m = INF, ordered by e).  Register footprint:
// R x (64 + 32) bits, so the full-key sort does not spill.
template <int R>
__device__ __forceinline__ bool pair_lt(int64_t ma, int ea, int64_t mb, int eb, const int64_t* wt,
                                        const uint64_t* wi) {
  if (ma != mb) return ma < mb;
  if (ma == INF) return ea < eb;
  const int64_t ta = wt[ea], tb = wt[eb];
  if (ta != tb) return ta < tb;
  return wi[ea] < wi[eb];
}

template <int R, int JR>
__device__ __forceinline__ void warp_pairs_rows(int64_t (&m)[R], int (&e)[R], int kk, const int64_t* wt,
                                                const uint64_t* wi) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (r & JR) continue;
    const int r2 = r | JR;
    if (r2 >= R) continue;
    const bool up = ((r << 5) & kk) == 0;
    const bool sw = up ? pair_lt<R>(m[r2], e[r2], m[r], e[r], wt, wi)
                       : pair_lt<R>(m[r], e[r], m[r2], e[r2], wt, wi);
    if (sw) {
      const int64_t a = m[r]; m[r] = m[r2]; m[r2] = a;
      const int b = e[r]; e[r] = e[r2]; e[r2] = b;
    }
  }
}

template <int R>
__device__ __forceinline__ void warp_bitonic_pairs(int64_t (&m)[R], int (&e)[R], const int64_t* wt,
                                                   const uint64_t* wi) {
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int kk = 2; kk <= R * 32; kk <<= 1) {
#pragma unroll 1
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int jr = j >> 5;
        if (jr == 1) warp_pairs_rows<R, 1>(m, e, kk, wt, wi);
        else if (R >= 4 && jr == 2) warp_pairs_rows<R, (R >= 4 ? 2 : 1)>(m, e, kk, wt, wi);
        else if (R >= 8 && jr == 4) warp_pairs_rows<R, (R >= 8 ? 4 : 1)>(m, e, kk, wt, wi);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int64_t pm = __shfl_xor_sync(0xffffffffu, m[r], j);
          const int pe = __shfl_xor_sync(0xffffffffu, e[r], j);
          const int x = (r << 5) | lane;
          const bool up = (x & kk) == 0, lower = (x & j) == 0;
          const bool p_lt = pair_lt<R>(pm, pe, m[r], e[r], wt, wi);
          if ((lower == up) ? p_lt : !p_lt) {
            m[r] = pm;
            e[r] = pe;
          }
        }
      }
    }
  }
}

template <int R>
__device__ void warp_direct_seg(const BatchDev& B, const LevelDev& L, int64_t gs, int n, int* wpre,
                                Blk* wblk, int64_t* wt, uint64_t* wi) {
  const int lane = threadIdx.x & 31;
  const int st = L.st;
  const int j = find_base(B.seg_base, B.nsteps, gs);
  const StepDev& s = B.steps[j];
  const int64_t li = gs - B.seg_base[j];
  const int64_t sg = s.seg_lo + li;
  const int nblk = (int)s.nblk;  // <= n <= WARP_DIRECT
  const int64_t* rel = L.blk_rel + B.blk_base[j] + li * s.nblk;
  // per-block sample sizes -> inclusive prefix (warp scan in chunks of 32)
  int run = 0;
  for (int k0 = 0; k0 < nblk; k0 += 32) {
    const int k = k0 + lane;
    int c = 0;
    if (k < nblk) {
      Blk b = load_blk(s, sg, k);
      c = (int)(samp_cnt(b.n[0], st) * samp_cnt(b.n[1], st) * samp_cnt(b.n[2], st));
      if (k < WARP_BLK_CACHE) wblk[k] = b;
    }
    const int inc = warp_incl_sum<int>(c);
    if (k < nblk) wpre[k + 1] = run + inc;
    run += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) wpre[0] = 0;
  __syncwarp();
  // tuple e of the sample (block: largest lo with wpre[lo] <= e)
  const StepDev* sp = &s;
  auto gen = [&](int e, int64_t& vm, int64_t& vt, uint64_t& vi) {
    int lo = 0, hi = nblk;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (wpre[mid] <= e) lo = mid;
      else hi = mid;
    }
    const Blk b = lo < WARP_BLK_CACHE ? wblk[lo] : load_blk(*sp, sg, lo);
    const int rr = e - wpre[lo];
    const int cy = (int)samp_cnt(b.n[1], st), cz = (int)samp_cnt(b.n[2], st);
    const int jz = rr % cz, q = rr / cz, jy = q % cy, jx = q / cy;
    make_tuple(*sp, b, rel[lo], samp_idx(jx, b.n[0], st), samp_idx(jy, b.n[1], st),
               samp_idx(jz, b.n[2], st), vm, vt, vi);
  };
  // Sort 64-bit keys ((m - m0) << 9 | e), m0 = the sample's least m, with t
  // and id staged in wt/wi by e; after the sort an element carries (m, e).
  // A sample whose m span needs more than B.kspan bits (frontier m reaches
  // 2^60, R10), or with equal m values (detected after the sort: the key
  // order is then not the (m, t, id) order), is (re)sorted exactly on (m, e)
  // pairs with t / id looked up by e on equal m (warp_bitonic_pairs).
  uint64_t k[R];
  long long lmin = INF, lmax = -1;
#pragma unroll
  for (int r = 0; r < R; ++r) k[r] = ~0ull;
  // rows generated DW_GEN_UNROLL at a time, so that the factor loads of
  // several rows are in flight together (each row is a chain of dependent
  // loads: block search, offsets, factor values)
#pragma unroll kDwGenUnroll
  for (int r = 0; r < R; ++r) {
    const int e = (r << 5) | lane;
    if (e < n) {
      int64_t vm, vt;
      uint64_t vi;
      gen(e, vm, vt, vi);
      wt[e] = vt;
      wi[e] = vi;
      lmin = vm < lmin ? vm : lmin;
      lmax = vm > lmax ? vm : lmax;
#pragma unroll
      for (int q2 = 0; q2 < R; ++q2)
        if (q2 == r) k[q2] = (uint64_t)vm;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long a = __shfl_xor_sync(0xffffffffu, lmin, o), b = __shfl_xor_sync(0xffffffffu, lmax, o);
    lmin = a < lmin ? a : lmin;
    lmax = b > lmax ? b : lmax;
  }
  const bool wide = ((unsigned long long)(lmax - lmin) >> B.kspan) != 0;
  __syncwarp();
  int64_t m[R];
  int ix[R];
  bool tie = false;
  if (!wide) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = (r << 5) | lane;
      if (e < n) k[r] = ((k[r] - (uint64_t)lmin) << 9) | (uint64_t)e;
    }
    warp_bitonic_keys<R>(k);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = (r << 5) | lane;
      uint64_t prev = __shfl_up_sync(0xffffffffu, k[r], 1);
      const uint64_t rowlast = __shfl_sync(0xffffffffu, k[r > 0 ? r - 1 : 0], 31);
      if (lane == 0) prev = r > 0 ? rowlast : ~0ull;
      if (e < n && prev != ~0ull && (prev >> 9) == (k[r] >> 9)) tie = true;
      m[r] = e < n ? (int64_t)(k[r] >> 9) + lmin : INF;
      ix[r] = e < n ? (int)(k[r] & 511u) : e;
    }
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = (r << 5) | lane;
      m[r] = e < n ? (int64_t)k[r] : INF;
      ix[r] = e;
    }
  }
  if (__any_sync(0xffffffffu, tie || wide)) warp_bitonic_pairs<R>(m, ix, wt, wi);  // exact (m, t, id)
  int64_t t[R];
#pragma unroll
  for (int r = 0; r < R; ++r) t[r] = ((r << 5) | lane) < n ? wt[ix[r]] : INF;
  warp_sweep_write<R>(L, gs, n, t, [&](int r, int64_t d) {
#pragma unroll
    for (int q = 0; q < R; ++q)
      if (q == r) {
        L.out.m[d] = m[q];
        L.out.t[d] = t[q];
        L.out.id[d] = wi[ix[q]];
      }
  });
}

__global__ void __launch_bounds__(256, 3) k_direct_warp(BatchDev B, LevelDev L) {
  FT_PDL_ENTRY();
  __shared__ int pre_all[8][WARP_DIRECT + 1];
  __shared__ Blk blk_all[8][WARP_BLK_CACHE];
  extern __shared__ int64_t dyn_dw[];  // per warp: t[WARP_DIRECT], id[WARP_DIRECT]
  int64_t* wt = dyn_dw + (threadIdx.x >> 5) * 2 * WARP_DIRECT;
  uint64_t* wi = (uint64_t*)(wt + WARP_DIRECT);
  const int wid = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * 8;
  int64_t tw = B.nseg / nw;
  tw = tw < 1 ? 1 : (tw > 32 ? 32 : tw);
  const int64_t w0 = (int64_t)blockIdx.x * 8 + wid;  // segments w0 + j * nw, tw per ballot
  for (int64_t t0 = 0; w0 + t0 * nw < B.nseg; t0 += tw) {
    const int64_t g = w0 + (t0 + lane) * nw;
    int nn = 0;
    if (lane < tw && g < B.nseg && L.seg_d[g] == L.level) {
      nn = L.seg_n[g];
      if (nn == 0) {  // empty-staircase level of a very wide segment (k_plan)
        L.out.start[g] = 0;
        L.out.cnt[g] = 0;
      }
    }
    unsigned bal = __ballot_sync(0xffffffffu, nn > 0 && nn <= WARP_DIRECT);
    while (bal) {
      const int b = __ffs(bal) - 1;
      bal &= bal - 1;
      const int64_t gs = w0 + (t0 + b) * nw;
      const int n = __shfl_sync(0xffffffffu, nn, b);
      if (L.hdr->overflow) return;
      if (n <= 32) warp_direct_seg<1>(B, L, gs, n, pre_all[wid], blk_all[wid], wt, wi);
      else if (n <= 64) warp_direct_seg<2>(B, L, gs, n, pre_all[wid], blk_all[wid], wt, wi);
      else if (n <= 128) warp_direct_seg<4>(B, L, gs, n, pre_all[wid], blk_all[wid], wt, wi);
      else warp_direct_seg<8>(B, L, gs, n, pre_all[wid], blk_all[wid], wt, wi);
      __syncwarp();
    }
  }
}

// Shared-order node elimination (Eq. 4) for steps whose Y = F(o_i,k) are
// singletons and Z = F(e_ij,k,p) is an original edge with m = 0 (Eq. 2): for a
// fixed w, every segment (w,p) holds the same tuples (k, x) with the same m and
// id = rel_k + x; only t = t_x + t_y + t_z(k,p) depends on p.  The (m, id)
// order is sorted once per w; if no two tuples share m it equals the
// (m, t, id) order of every p and Alg. 1 is one running-min sweep per p.
//
// k_node_pack (common case): a CTA takes a pack of up to 256/ceil32(K_j) rows
// w of one step; each row (<= WARP_DIRECT tuples) is sorted by one warp in
// registers, t_z(k, p) is staged once per step in shared memory and reused
// across the CTA's packs, and one thread per (w, p) runs Alg. 1 as a
// sequential running min, recording keep bits; survivors are then written
// warp-cooperatively (coalesced).  Rows with more than WARP_DIRECT tuples, an
// m span wider than the packed keys hold, or an oversized t_z table go to
// k_node_shared (one CTA per row, full int64 keys, exact group rule for ties)
// through a device list.
constexpr int NP_NT = 256;
constexpr int NP_WORDS = WARP_DIRECT / 32;
constexpr int NP_ROWS = 8;
constexpr int64_t NP_ZT_CAP = 8192;  // t_z table entries staged per step (64 KB)

__host__ __device__ inline int np_tpr(int64_t np) { return (int)((np + 31) / 32 * 32); }
__host__ __device__ inline size_t np_smem(int rmax, int64_t ztn) {
  return (size_t)ztn * 8 + (size_t)rmax * (WARP_DIRECT * 20 + NS_MAXBLK * 8 + (NS_MAXBLK + 1) * 4) +
         (size_t)NP_WORDS * NP_NT * 4;
}

// One row: generate its (<= WARP_DIRECT) tuples, sort 64-bit keys
// ((m - m0) << 9 | e) in registers (m0 = the row's least m) and gather t_xy
// and the block by e (= the tuple id rel_k + x, R6).  Ties in m need no
// re-sort: the sweep applies the exact equal-m group rule, which scans the
// whole group.  Returns bit 0: equal m values; bit 1: the row's m span needs
// more than kspan bits (frontier m reaches 2^60, R10) -- the caller then
// hands the row to k_node_shared, which sorts the full int64 m.
template <int R>
__device__ __forceinline__ int np_row_sort(const StepDev& s, const int* pre, const int64_t* bo,
                                           const int64_t* ym, const int64_t* yt, int nblk, int n,
                                           int64_t* sm, int64_t* stxy, uint32_t* sidk, int kspan) {
  const int lane = threadIdx.x & 31;
  uint64_t key[R];
  long long lmin = INF, lmax = -1;
#pragma unroll
  for (int r = 0; r < R; ++r) key[r] = ~0ull;
#pragma unroll 1
  for (int r = 0; r < R && (r << 5) < n; ++r) {
    const int e = (r << 5) | lane;
    if (e < n) {
      int lo = 0, hi = nblk;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (pre[mid] <= e) lo = mid;
        else hi = mid;
      }
      const int x = e - pre[lo];
      const int64_t vm = __ldg(s.X.m + bo[lo] + x) + ym[lo];
      stxy[e] = __ldg(s.X.t + bo[lo] + x) + yt[lo];  // staged by e
      sidk[e] = (uint32_t)lo;
      lmin = vm < lmin ? vm : lmin;
      lmax = vm > lmax ? vm : lmax;
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (q == r) key[q] = (uint64_t)vm;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long a = __shfl_xor_sync(0xffffffffu, lmin, o), b = __shfl_xor_sync(0xffffffffu, lmax, o);
    lmin = a < lmin ? a : lmin;
    lmax = b > lmax ? b : lmax;
  }
  if (((unsigned long long)(lmax - lmin) >> kspan) != 0) return 2;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = (r << 5) | lane;
    if (e < n) key[r] = ((key[r] - (uint64_t)lmin) << 9) | (uint64_t)e;
  }
  __syncwarp();
  warp_bitonic_keys<R>(key);
  int64_t t[R];
  uint32_t kb[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = (r << 5) | lane;
    const int src = (int)(key[r] & 511u);
    t[r] = e < n ? stxy[src] : INF;
    kb[r] = e < n ? sidk[src] : 0u;
  }
  __syncwarp();  // all gathers before the sorted rows are written back
  bool tie = false;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    uint64_t nk = __shfl_down_sync(0xffffffffu, key[r], 1);
    const uint64_t n0 = r + 1 < R ? __shfl_sync(0xffffffffu, key[r + 1 < R ? r + 1 : r], 0) : ~0ull;
    if (lane == 31) nk = n0;
    const int e = (r << 5) | lane;
    const bool same_next = e + 1 < n && (nk >> 9) == (key[r] >> 9);
    if (same_next) tie = true;
    if (e < n) {  // id | k << 16 | (last of its equal-m group) << 31
      sm[e] = (int64_t)(key[r] >> 9) + lmin;
      stxy[e] = t[r];
      sidk[e] = (uint32_t)(key[r] & 511u) | (kb[r] << 16) | (same_next ? 0u : 0x80000000u);
    }
  }
  return __any_sync(0xffffffffu, tie) ? 1 : 0;
}

__global__ void __launch_bounds__(NP_NT, 3) k_node_pack(BatchDev B, LevelDev L, const NodeGroup* packs,
                                                     int npacks, int rmax, int64_t ztn,
                                                     NodeGroup* big) {
  FT_PDL_ENTRY();
  extern __shared__ int64_t dyn_np[];
  int64_t* ztab = dyn_np;                                        // [ztn] t_z(k, p) at k*tpr+pl
  int64_t* sm = ztab + ztn;                                      // [rmax][WARP_DIRECT]
  int64_t* stxy = sm + (size_t)rmax * WARP_DIRECT;               // [rmax][WARP_DIRECT]
  int64_t* bo = stxy + (size_t)rmax * WARP_DIRECT;               // [rmax][NS_MAXBLK]
  uint32_t* sidk = (uint32_t*)(bo + (size_t)rmax * NS_MAXBLK);   // [rmax][WARP_DIRECT]
  int* pre = (int*)(sidk + (size_t)rmax * WARP_DIRECT);          // [rmax][NS_MAXBLK + 1]
  uint32_t* kbits = (uint32_t*)(pre + (size_t)rmax * (NS_MAXBLK + 1));  // [NP_WORDS][NP_NT]
  __shared__ int64_t ym[NS_MAXBLK], yt[NS_MAXBLK];
  __shared__ int soff[NP_NT];
  __shared__ int row_n[NP_ROWS];
  __shared__ bool row_tie[NP_ROWS];
  __shared__ long long sh[33];
  __shared__ int64_t s_base;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int p0 = (int)((int64_t)npacks * blockIdx.x / gridDim.x);
  const int p1 = (int)((int64_t)npacks * (blockIdx.x + 1) / gridDim.x);
  int cur = -1;
  int64_t cur_lo = -1, cur_hi = -1;
  for (int pi = p0; pi < p1; ++pi) {
    if (L.hdr->overflow) return;
    const NodeGroup P = packs[pi];
    const StepDev& s = B.steps[P.step];
    const int nblk = (int)s.nblk;
    const int64_t np = P.p_hi - P.p_lo;
    const int tpr = np_tpr(np);
    const int nw = P.pad;
    const bool fits = np <= NP_NT && (int64_t)nblk * tpr <= ztn && nw <= rmax;
    // per-step tables t_z(k, p_lo + pl), Y = F(o_i, k); a rank boundary can cut
    // a row, so the cache key includes the p range
    if ((P.step != cur || P.p_lo != cur_lo || P.p_hi != cur_hi) && fits) {
      for (int64_t q = threadIdx.x; q < (int64_t)nblk * tpr; q += NP_NT) {
        const int k = (int)(q / tpr), pl = (int)(q - (int64_t)k * tpr);
        ztab[q] = pl < np ? s.Z.t[s.Z.off[(int64_t)k * s.KC + P.p_lo + pl]] : 0;
      }
      for (int k = threadIdx.x; k < nblk; k += NP_NT) {
        const int64_t oy = s.Y.off[k];
        ym[k] = s.Y.m[oy];
        yt[k] = s.Y.t[oy];
      }
      cur = P.step;
      cur_lo = P.p_lo;
      cur_hi = P.p_hi;
    }
    __syncthreads();
    // one warp per row: block prefix, register sort, tie check
    for (int r = wid; r < nw; r += NP_NT / 32) {
      const int64_t gsr = P.gs0 + (int64_t)r * np;
      int n = 0;
      if (L.seg_d[gsr] == SPECIAL_LEVEL) {
        n = L.seg_n[gsr];
        bool ok = fits && n <= WARP_DIRECT;
        if (ok) {
          int* pr = pre + r * (NS_MAXBLK + 1);
          int64_t* b = bo + r * NS_MAXBLK;
          int run = 0;
          for (int k0 = 0; k0 < nblk; k0 += 32) {
            const int k = k0 + lane;
            int c = 0;
            if (k < nblk) {
              const int64_t sx = (P.w + r) * s.KB + k;
              const int64_t o = s.X.off[sx];
              b[k] = o;
              c = (int)(s.X.off[sx + 1] - o);
            }
            const int inc = warp_incl_sum<int>(c);
            if (k < nblk) pr[k + 1] = run + inc;
            run += __shfl_sync(0xffffffffu, inc, 31);
          }
          if (lane == 0) pr[0] = 0;
          __syncwarp();
          int64_t* rm = sm + r * WARP_DIRECT;
          int64_t* rt = stxy + r * WARP_DIRECT;
          uint32_t* ri = sidk + r * WARP_DIRECT;
          int rc;
          if (n <= 32) rc = np_row_sort<1>(s, pr, b, ym, yt, nblk, n, rm, rt, ri, B.kspan);
          else if (n <= 64) rc = np_row_sort<2>(s, pr, b, ym, yt, nblk, n, rm, rt, ri, B.kspan);
          else if (n <= 128) rc = np_row_sort<4>(s, pr, b, ym, yt, nblk, n, rm, rt, ri, B.kspan);
          else rc = np_row_sort<8>(s, pr, b, ym, yt, nblk, n, rm, rt, ri, B.kspan);
          ok = rc != 2;  // wide m span: k_node_shared
          if (lane == 0 && ok) {
            row_tie[r] = rc != 0;
            atomicAdd(&L.hdr->ns_rows, 1ull);
            if (rc) atomicAdd(&L.hdr->ns_tie, 1ull);
          }
        }
        if (!ok) {  // large rows / tables: one CTA per row in k_node_shared
          if (lane == 0) {
            NodeGroup G;
            G.step = P.step;
            G.pad = 0;
            G.w = P.w + r;
            G.p_lo = P.p_lo;
            G.p_hi = P.p_hi;
            G.gs0 = gsr;
            big[atomicAdd(&L.hdr->ns_big, 1ull)] = G;
          }
          n = 0;
        }
      }
      if (lane == 0) row_n[r] = n;
    }
    __syncthreads();
    // Alg. 1 for segment (w, p): running min over the shared (m, id) order
    const int r = threadIdx.x / tpr, pl = threadIdx.x - r * tpr;
    const int n = r < nw ? row_n[r] : 0;
    const bool act = n > 0 && pl < np;
    int cnt = 0;
    if (act && !row_tie[r]) {
      const int64_t* rt = stxy + r * WARP_DIRECT;
      const uint32_t* ri = sidk + r * WARP_DIRECT;
      long long carry = INF;
      for (int c0 = 0; c0 < n; c0 += 32) {
        uint32_t word = 0;
        const int ce = min(32, n - c0);
#pragma unroll 4
        for (int b = 0; b < ce; ++b) {
          const int i = c0 + b;
          const long long t = rt[i] + ztab[((ri[i] >> 16) & 0x7fffu) * tpr + pl];
          if (t < carry) {
            word |= 1u << b;
            carry = t;
          }
        }
        kbits[(c0 >> 5) * NP_NT + threadIdx.x] = word;
        cnt += __popc(word);
      }
    } else if (act) {
      // equal m values: Alg. 1 under (m, t, id) keeps only the (t, id)-least
      // tuple of an equal-m group, iff its t is below every earlier t
      const int64_t* rt = stxy + r * WARP_DIRECT;
      const uint32_t* ri = sidk + r * WARP_DIRECT;
      for (int c0 = 0; c0 < n; c0 += 32) kbits[(c0 >> 5) * NP_NT + threadIdx.x] = 0;
      long long carry = INF, bt = INF;
      int bi = 0;
      uint32_t bid = 0xffffffffu;
      for (int i = 0; i < n; ++i) {
        const uint32_t v = ri[i];
        const long long t = rt[i] + ztab[((v >> 16) & 0x7fffu) * tpr + pl];
        const uint32_t id = v & 0xffffu;
        if (t < bt || (t == bt && id < bid)) {
          bt = t;
          bi = i;
          bid = id;
        }
        if (v >> 31) {
          if (bt < carry) {
            kbits[(bi >> 5) * NP_NT + threadIdx.x] |= 1u << (bi & 31);
            carry = bt;
            ++cnt;
          }
          bt = INF;
          bid = 0xffffffffu;
        }
      }
    }
    long long tot;
    const int ex = (int)block_excl_sum<NP_NT>(cnt, sh, &tot);
    soff[threadIdx.x] = ex;
    if (threadIdx.x == 0) {
      int64_t base = -1;
      const unsigned long long st0 = tot ? atomicAdd(L.out.cursor, (unsigned long long)tot) : 0ull;
      if ((int64_t)(st0 + tot) > L.out.cap) atomicExch(&L.hdr->overflow, 1ull);
      else base = (int64_t)st0;
      if (tot) atomicAdd(&L.hdr->out_total[0], (unsigned long long)tot);
      s_base = base;
    }
    __syncthreads();
    const int64_t base = s_base;
    if (act) {
      const int64_t gs = P.gs0 + (int64_t)r * np + pl;
      L.out.start[gs] = base < 0 ? -1 : base + ex;
      L.out.cnt[gs] = cnt;
    }
    if (base >= 0) {
      // survivors of (r, pl), coalesced: lane = bit within a 32-tuple word
      for (int j = wid; j < nw * tpr; j += NP_NT / 32) {
        const int rr = j / tpr, pp = j - rr * tpr;
        const int nn = row_n[rr];
        if (nn == 0 || pp >= np) continue;
        int off = soff[j];
        const int64_t* rm = sm + rr * WARP_DIRECT;
        const int64_t* rt = stxy + rr * WARP_DIRECT;
        const uint32_t* ri = sidk + rr * WARP_DIRECT;
        for (int c0 = 0; c0 < nn; c0 += 32) {
          const uint32_t word = kbits[(c0 >> 5) * NP_NT + j];
          if ((word >> lane) & 1u) {
            const int i = c0 + lane;
            const uint32_t v = ri[i];
            const int64_t d = base + off + __popc(word & ((1u << lane) - 1u));
            L.out.m[d] = rm[i];
            L.out.t[d] = rt[i] + ztab[((v >> 16) & 0x7fffu) * tpr + pp];
            L.out.id[d] = (uint64_t)(v & 0xffffu);
          }
          off += __popc(word);
        }
      }
    }
    __syncthreads();
  }
}

constexpr size_t NS_SMEM = (size_t)NS_CAP * (5 * 8 + 4 + 2 + 2);
static_assert(sizeof(NodeGroup) == sizeof(NodeGroupH), "NodeGroup layout");

__global__ void __launch_bounds__(DIRECT_NT) k_node_shared(BatchDev B, LevelDev L,
                                                           const NodeGroup* groups) {
  FT_PDL_ENTRY();
  const int ngroups = (int)L.hdr->ns_big;  // rows k_node_pack handed over
  extern __shared__ int64_t dyn_ns[];
  int64_t* sm = dyn_ns;                            // [NS_CAP] m (sorted by (m, id))
  uint64_t* sid = (uint64_t*)(sm + NS_CAP);        // [NS_CAP] id
  int64_t* stxy = (int64_t*)(sid + NS_CAP);        // [NS_CAP] t_x + t_y
  int64_t* tt = stxy + NS_CAP;                     // [NS_CAP] t for this p
  int64_t* mincl = tt + NS_CAP;                    // [NS_CAP] inclusive prefix-min of tt (ties)
  int* kf = (int*)(mincl + NS_CAP);                // [NS_CAP] keep flags -> positions
  int16_t* sk = (int16_t*)(kf + NS_CAP);           // [NS_CAP] block of each tuple
  int16_t* gst = sk + NS_CAP;                      // [NS_CAP] start of the equal-m group
  __shared__ int64_t zt[NS_MAXBLK];
  __shared__ int64_t wzt[DIRECT_NT / 32][NS_MAXBLK];  // per-warp t_z(k, p)
  __shared__ int pre[NS_MAXBLK + 1];
  __shared__ int64_t bo[NS_MAXBLK];
  __shared__ int64_t bym[NS_MAXBLK], byt[NS_MAXBLK];
  __shared__ long long sh[33];
  __shared__ int s_tie;
  __shared__ int64_t s_start;
  for (int gi = blockIdx.x; gi < ngroups; gi += gridDim.x) {
    const NodeGroup G = groups[gi];
    if (L.seg_d[G.gs0] != SPECIAL_LEVEL) continue;  // uniform per group
    if (L.hdr->overflow) return;
    const StepDev& s = B.steps[G.step];
    const int nblk = (int)s.nblk;
    // blocks: X = F(e_hi, w, k) (runs), Y = F(o_i, k), Z = F(e_ij, k, p)
    for (int k = threadIdx.x; k < nblk; k += DIRECT_NT) {
      const int64_t sx = G.w * s.KB + k;
      const int64_t o = s.X.off[sx];
      bo[k] = o;
      pre[k + 1] = (int)(s.X.off[sx + 1] - o);
      const int64_t oy = s.Y.off[k];
      bym[k] = s.Y.m[oy];
      byt[k] = s.Y.t[oy];
    }
    if (threadIdx.x == 0) {
      pre[0] = 0;
      s_tie = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 0; k < nblk; ++k) pre[k + 1] += pre[k];
    __syncthreads();
    const int n = pre[nblk];
    int N = 1;
    while (N < n) N <<= 1;
    for (int i = threadIdx.x; i < N; i += DIRECT_NT) {
      if (i < n) {
        int lo = 0, hi = nblk;
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (pre[mid] <= i) lo = mid;
          else hi = mid;
        }
        const int x = i - pre[lo];
        sm[i] = __ldg(s.X.m + bo[lo] + x) + bym[lo];
        stxy[i] = __ldg(s.X.t + bo[lo] + x) + byt[lo];
        sid[i] = (uint64_t)(pre[lo] + x);  // id = rel_k + x  (|Y| = |Z| = 1, R6)
        sk[i] = (int16_t)lo;
      } else {
        sm[i] = INF;
        stxy[i] = INF;
        sid[i] = ~0ull;
        sk[i] = 0;
      }
    }
    __syncthreads();
    // bitonic sort by (m, id), carrying (t_xy, k)
    for (int kk = 2; kk <= N; kk <<= 1) {
      for (int jj = kk >> 1; jj > 0; jj >>= 1) {
        for (int i = threadIdx.x; i < N; i += DIRECT_NT) {
          const int l = i ^ jj;
          if (l > i) {
            const bool up = (i & kk) == 0;
            const bool gt = sm[l] < sm[i] || (sm[l] == sm[i] && sid[l] < sid[i]);
            if (gt == up) {
              int64_t a = sm[i]; sm[i] = sm[l]; sm[l] = a;
              a = stxy[i]; stxy[i] = stxy[l]; stxy[l] = a;
              uint64_t b = sid[i]; sid[i] = sid[l]; sid[l] = b;
              int16_t c = sk[i]; sk[i] = sk[l]; sk[l] = c;
            }
          }
        }
        __syncthreads();
      }
    }
    // equal-m groups (rare): gst[i] = first index of i's group
    for (int i = threadIdx.x; i < n; i += DIRECT_NT) {
      int g0 = i;
      while (g0 > 0 && sm[g0 - 1] == sm[i]) --g0;
      gst[i] = (int16_t)g0;
      if (g0 != i) s_tie = 1;
    }
    __syncthreads();
    const bool tie = s_tie != 0;
    if (!tie) {
      // distinct m: the (m, id) order is every p's (m, t, id) order; one warp
      // per p runs Alg. 1 as a warp-scan sweep (count pass, then write pass)
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
      for (int64_t p = G.p_lo + wid; p < G.p_hi; p += DIRECT_NT / 32) {
        const int64_t gs = G.gs0 + (p - G.p_lo);
        for (int k = lane; k < nblk; k += 32) wzt[wid][k] = s.Z.t[s.Z.off[(int64_t)k * s.KC + p]];
        __syncwarp();
        long long carry = INF;
        int cnt = 0;
        for (int c0 = 0; c0 < n; c0 += 32) {
          const int i = c0 + lane;
          const long long t = i < n ? stxy[i] + wzt[wid][sk[i]] : INF;
          const long long inc = warp_incl_min(t);
          long long ex = __shfl_up_sync(0xffffffffu, inc, 1);
          if (lane == 0) ex = INF;
          const bool keep = i < n && t < (ex < carry ? ex : carry);
          cnt += __popc(__ballot_sync(0xffffffffu, keep));
          const long long rm = __shfl_sync(0xffffffffu, inc, 31);
          carry = rm < carry ? rm : carry;
        }
        int64_t base = 0;
        if (lane == 0) {
          unsigned long long st0 = atomicAdd(L.out.cursor, (unsigned long long)cnt);
          if ((int64_t)(st0 + cnt) > L.out.cap) {
            atomicExch(&L.hdr->overflow, 1ull);
            base = -1;
          } else {
            base = (int64_t)st0;
          }
          atomicAdd(&L.hdr->out_total[0], (unsigned long long)cnt);
          L.out.start[gs] = base;
          L.out.cnt[gs] = cnt;
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= 0) {
          carry = INF;
          int off = 0;
          for (int c0 = 0; c0 < n; c0 += 32) {
            const int i = c0 + lane;
            const long long t = i < n ? stxy[i] + wzt[wid][sk[i]] : INF;
            const long long inc = warp_incl_min(t);
            long long ex = __shfl_up_sync(0xffffffffu, inc, 1);
            if (lane == 0) ex = INF;
            const bool keep = i < n && t < (ex < carry ? ex : carry);
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) {
              const int64_t d = base + off + __popc(bal & ((1u << lane) - 1u));
              L.out.m[d] = sm[i];
              L.out.t[d] = t;
              L.out.id[d] = sid[i];
            }
            off += __popc(bal);
            const long long rm = __shfl_sync(0xffffffffu, inc, 31);
            carry = rm < carry ? rm : carry;
          }
        }
        __syncwarp();
      }
      __syncthreads();
      continue;
    }
    for (int64_t p = G.p_lo; p < G.p_hi; ++p) {
      const int64_t gs = G.gs0 + (p - G.p_lo);
      for (int k = threadIdx.x; k < nblk; k += DIRECT_NT) {
        const int64_t sz = (int64_t)k * s.KC + p;
        zt[k] = s.Z.t[s.Z.off[sz]];
      }
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += DIRECT_NT) tt[i] = stxy[i] + zt[sk[i]];
      __syncthreads();
      int cnt;
      if (!tie) {
        // distinct m: the (m, id) order is the (m, t, id) order -> Alg. 1 directly
        cnt = alg1_sweep_smem<DIRECT_NT>(tt, n, INF, kf, sh);
      } else {
        // Alg. 1 under (m, t, id) on the (m, id) order: only the (t, id)-least
        // tuple of an equal-m group can survive, iff its t is below every t of
        // the earlier groups.
        {
          const int per = (n + DIRECT_NT - 1) / DIRECT_NT;
          const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
          long long lmin = INF;
          for (int i = lo; i < hi; ++i) lmin = tt[i] < lmin ? tt[i] : lmin;
          long long v = block_excl_min<DIRECT_NT>(lmin, sh);
          for (int i = lo; i < hi; ++i) {
            v = tt[i] < v ? tt[i] : v;
            mincl[i] = v;
          }
        }
        __syncthreads();
        int c = 0;
        const int per = (n + DIRECT_NT - 1) / DIRECT_NT;
        const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
        for (int i = lo; i < hi; ++i) {
          const int g0 = gst[i];
          bool best = true;
          for (int jx = g0; jx < n && sm[jx] == sm[i]; ++jx)
            if (jx != i && (tt[jx] < tt[i] || (tt[jx] == tt[i] && sid[jx] < sid[i]))) best = false;
          const long long before = g0 > 0 ? mincl[g0 - 1] : INF;
          kf[i] = best && tt[i] < before;
          c += kf[i];
        }
        long long tot;
        long long off = block_excl_sum<DIRECT_NT>(c, sh, &tot);
        int q = (int)off;
        for (int i = lo; i < hi; ++i)
          if (kf[i]) kf[i] = ++q;
        __syncthreads();
        cnt = (int)tot;
      }
      if (threadIdx.x == 0) {
        unsigned long long st0 = atomicAdd(L.out.cursor, (unsigned long long)cnt);
        if ((int64_t)(st0 + cnt) > L.out.cap) {
          atomicExch(&L.hdr->overflow, 1ull);
          s_start = -1;
        } else {
          s_start = (int64_t)st0;
        }
        atomicAdd(&L.hdr->out_total[0], (unsigned long long)cnt);
        L.out.start[gs] = s_start;
        L.out.cnt[gs] = cnt;
      }
      __syncthreads();
      const int64_t o = s_start;
      if (o >= 0)
        for (int i = threadIdx.x; i < n; i += DIRECT_NT)
          if (kf[i]) {
            const int64_t d = o + kf[i] - 1;
            L.out.m[d] = sm[i];
            L.out.t[d] = tt[i];
            L.out.id[d] = sid[i];
          }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// Filter path, level l < d_sigma.


// Long factor = the one with most sampled indices; runs = product of the other two.
__device__ __forceinline__ void run_shape(const Blk& b, int st, int& lf, int& fa, int& fb, int64_t& cL,
                                          int64_t& cA, int64_t& cB) {
  // scalars and selects only: an indexed local array would live in local memory
  const int64_t c0 = samp_cnt(b.n[0], st), c1 = samp_cnt(b.n[1], st), c2 = samp_cnt(b.n[2], st);
  lf = 0;
  if (c1 > c0) lf = 1;
  if (c2 > (lf == 1 ? c1 : c0)) lf = 2;
  fa = lf == 0 ? 1 : 0;
  fb = lf == 2 ? 1 : 2;
  cL = lf == 0 ? c0 : (lf == 1 ? c1 : c2);
  cA = fa == 0 ? c0 : c1;
  cB = fb == 2 ? c2 : c1;
}

// Work items of the filter: L.run_item consecutive sampled indices of one run
// (a multiple of CHUNK, chosen per level so that the grid has enough threads).
// Per-segment bucket counts nb are computed by the bucket-base scan's loader
// and stored for the later kernels; per-block work-item counts wcnt come from
// k_blocks.
struct LoadNb {
  LevelDev L;
  template <int N>
  __device__ __forceinline__ void load(int64_t base, int64_t n, long long (&v)[N]) const {
#pragma unroll
    for (int i = 0; i < N; ++i)
      v[i] = base + i < n && is_filter(L.seg_d[base + i], L.level) ? L.in.cnt[base + i] + 1 : 0;
  }
  template <int N>
  __device__ __forceinline__ void keep(int64_t base, int64_t n, const long long (&v)[N]) const {
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (base + i < n) L.nb[base + i] = v[i];
  }
};

// Warp-start block hints for k_filter: hint[c] = the block of filter item
// 32c (largest beta with wo[beta] <= 32c) and hint[hcap + c] its step, one
// thread per hint, so that a k_filter warp finds its items' blocks and steps
// with a few loads instead of binary searches over all blocks and steps at
// the head of its dependent-load chain.  (Written
// first in the work-offset scan's epilogue: serial per block, ~30 us per
// LDP level.)
__global__ void __launch_bounds__(256) k_hints(BatchDev B, LevelDev L) {
  FT_PDL_ENTRY();
  const int64_t nbl = B.nblk, W = L.wo[nbl];
  const int64_t nh = min((W + 31) >> 5, L.hcap);
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nh; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = c << 5;
    int64_t lo = 0, hi = nbl;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (L.wo[mid] <= x) lo = mid;
      else hi = mid;
    }
    L.whint[c] = (int32_t)lo;
    L.whint[L.hcap + c] = find_base(B.blk_base, B.nsteps, lo);  // its step
  }
}

// K1: product + pre-filter, output-sensitive run walk.  A work item is a
// range of one run (short-factor indices fixed, long factor sweeping: m
// strictly ascending, t strictly descending).  For element x let g be the
// last G point with m_g <= m_x (pointer advanced by galloping; G is a
// staircase).  If g strictly dominates x, it also strictly dominates every
// later element with t >= t_g (their m exceeds m_g), so the walk jumps to
// the first element with t < t_g (binary search on t).  Otherwise x is a
// candidate: emitted with bucket = #G points with m <= m_x.
constexpr int EPRE = 2;  // run elements loaded ahead in k_filter's element test (4: spills at 80 regs)

// lower_bound(G[0, g), x) for every lane of a warp whose lanes share G (the
// 32 items of a warp pass lie in one block, ~90% of passes): one coalesced
// load of 32 fences (the last point of each of 32 slices), a 5-step search
// over them by shuffles, then a per-lane binary search inside one slice --
// ~log2(g / 32) dependent loads instead of a gallop over all of G.
__device__ __forceinline__ int warp_lower_bound(const int64_t* G, int g, int64_t x) {
  const int lane = threadIdx.x & 31;
  const int s1 = (g + 31) >> 5;
  const int64_t f = G[min((lane + 1) * s1, g) - 1];
  int c = 0;  // fences below x
#pragma unroll
  for (int b = 16; b > 0; b >>= 1) {
    const int64_t v = __shfl_sync(0xffffffffu, f, c + b - 1);
    if (v < x) c += b;
  }
  if (__shfl_sync(0xffffffffu, f, 31) < x) return g;
  int a0 = c * s1, a1 = min((c + 1) * s1, g) - 1;  // G[a1] >= x
  if (a1 - a0 > 8) {  // second level: 8 sub-fences of the slice, independent loads
    const int s2 = (a1 - a0 + 8) >> 3;
    int c2 = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) c2 += G[min(a0 + (k + 1) * s2, a1 + 1) - 1] < x;
    // G[a0 + c2 * s2 - 1] < x (c2 > 0), G[min(a0 + (c2 + 1) * s2, a1 + 1) - 1] >= x
    const int b0 = a0 + c2 * s2;
    a1 = min(b0 + s2, a1 + 1) - 1;
    a0 = b0;
  }
  while (a0 < a1) {
    const int mid = (a0 + a1) >> 1;
    if (G[mid] < x) a0 = mid + 1;
    else a1 = mid;
  }
  return a0;
}

// Per-block work-item counts of a filter level (wcnt[beta], scanned next into
// the work offsets) with a block-level pre-filter: one thread per block, so
// the G lower bounds of all blocks are in flight at once (as the scan's
// loader, each thread ran 8 of them back to back); a warp whose 32 blocks
// share one segment searches G cooperatively.
__global__ void __launch_bounds__(256) k_blocks(BatchDev B, LevelDev L) {
  FT_PDL_ENTRY();
  const int64_t nbl = B.nblk;
  const int lane = threadIdx.x & 31;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); b0 < nbl; b0 += gstride) {
    const int64_t beta = b0 + lane;
    const bool valid = beta < nbl;
    const int64_t bb = valid ? beta : nbl - 1;
    const int j = find_base(B.blk_base, B.nsteps, bb);
    const StepDev& s = B.steps[j];
    const int64_t lb = bb - B.blk_base[j];
    const int64_t li = lb / s.nblk, k = lb - li * s.nblk;
    const int64_t lseg = B.seg_base[j] + li;
    const bool filt = valid && is_filter(L.seg_d[lseg], L.level);
    const Blk b = load_blk(s, s.seg_lo + li, k);
    int lf, fa, fb;
    int64_t cL, cA, cB;
    run_shape(b, L.st, lf, fa, fb, cL, cA, cB);
    long long w = filt ? cA * cB * ((cL + L.run_item - 1) / L.run_item) : 0;
    const bool need = w > 0 && g_bskip;
    int64_t mlo = 0, tlo = 0;
    if (need) {
      // Block-level pre-filter: every sampled tuple of the block has m >= the
      // sum of the factors' first m and t >= the sum of their last t (factor
      // segments are staircases and each sample keeps indices 0 and n-1).
      // The last G point with m below that bound has the least t among them;
      // if it is <= the t bound it strictly dominates the whole block, which
      // then emits no candidate -- the outcome of K1's chunk test on every
      // item of the block, without the items (C5: 92 M items -> 30 M).
      mlo = __ldg(s.X.m + b.o[0]) + __ldg(s.Y.m + b.o[1]) + __ldg(s.Z.m + b.o[2]);
      tlo = __ldg(s.X.t + b.o[0] + b.n[0] - 1) + __ldg(s.Y.t + b.o[1] + b.n[1] - 1) +
            __ldg(s.Z.t + b.o[2] + b.n[2] - 1);
    }
    if (g_bskip) {
      const int64_t l0 = __shfl_sync(0xffffffffu, lseg, 0);
      const bool same = __all_sync(0xffffffffu, valid && lseg == l0);
      const int64_t g0 = L.in.start[lseg];
      const int g = (int)L.in.cnt[lseg];
      int q = 0;
      if (same) {
        if (g > 0 && __any_sync(0xffffffffu, need)) q = warp_lower_bound(L.in.m + g0, g, mlo);
      } else if (need) {
        const int64_t* Gm = L.in.m + g0;
        int a1 = g;
        while (q < a1) {
          const int mid = (q + a1) >> 1;
          if (Gm[mid] < mlo) q = mid + 1;
          else a1 = mid;
        }
      }
      if (need && q > 0 && L.in.t[g0 + q - 1] <= tlo) w = 0;
    }
    if (valid) L.wcnt[beta] = w;
  }
}

__device__ __forceinline__ void filter_body(const BatchDev& B, const LevelDev& L) {
  namespace cg = cooperative_groups;
  if (L.hdr->overflow) return;
  if (L.bucket_base[B.nseg] > L.bcap) {  // more buckets than scratch: grow and retry
    atomicExch(&L.hdr->overflow, 1ull);
    return;
  }
  const int64_t nbl = B.nblk;
  const int64_t W = L.wo[nbl];
  const int sh = L.st;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (int64_t wbase = (int64_t)blockIdx.x * blockDim.x; wbase < W; wbase += gstride) {
    const int64_t w0 = wbase + (threadIdx.x & ~31);  // first item of this warp
    if (w0 >= W) break;
    // blocks of the warp's items: hint[w0/32] holds the block of item w0 and
    // hint[w0/32 + 1] that of item w0 + 32 (k_hints);
    // beyond the hint table, two full binary searches per warp.  Then a
    // bounded binary search per lane.
    const int64_t c0 = w0 >> 5;
    int64_t blo, bhi;  // wo[blo] <= w0 + lane < wo[bhi]
    int jlo = 0, jhi = B.nsteps;  // steps of the warp's blocks: [jlo, jhi)
    if (c0 + 1 < L.hcap) {
      blo = L.whint[c0];
      jlo = L.whint[L.hcap + c0];
      if (w0 + 32 < W) {
        bhi = (int64_t)L.whint[c0 + 1] + 1;
        jhi = L.whint[L.hcap + c0 + 1] + 1;
      } else {
        bhi = nbl;
      }
    } else {
      int64_t lo = 0;
      if (lane == 0 || lane == 31) {
        const int64_t x = lane == 0 ? w0 : min(w0 + 31, W - 1);
        int64_t hi = nbl;  // largest beta with wo[beta] <= x
        while (hi - lo > 1) {
          const int64_t mid = (lo + hi) >> 1;
          if (L.wo[mid] <= x) lo = mid;
          else hi = mid;
        }
      }
      blo = __shfl_sync(0xffffffffu, lo, 0);
      bhi = __shfl_sync(0xffffffffu, lo, 31) + 1;
    }
    const int64_t w = w0 + lane;
    // all 32 items in one block (hence one G): cooperative first lower bound
    const bool one = g_fence && bhi - blo <= 1 && w0 + 32 <= W;
    if (L.fstats) {  // warp passes, and those whose items all lie in one block
      const unsigned act = __ballot_sync(0xffffffffu, w < W);
      if (lane == 0) {
        atomicAdd(&L.hdr->fstat[6], 1ull);
        if (bhi - blo <= 1 && act == 0xffffffffu) atomicAdd(&L.hdr->fstat[5], 1ull);
      }
    }
    if (w >= W) continue;
    int64_t lo = blo;
    int64_t hi = bhi;  // wo[lo] <= w < wo[hi]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (L.wo[mid] <= w) lo = mid;
      else hi = mid;
    }
    const int64_t beta = lo, wl = w - L.wo[beta];
    int jstep = jlo;  // largest j in [jlo, jhi) with blk_base[j] <= beta
    for (int jh = jhi; jh - jstep > 1;) {
      const int mid = (jstep + jh) >> 1;
      if (__ldg(B.blk_base + mid) <= beta) jstep = mid;
      else jh = mid;
    }
    const StepDev& s = B.steps[jstep];
    const int64_t lb = beta - B.blk_base[jstep];
    const int64_t li0 = lb / s.nblk, k = lb - li0 * s.nblk;
    const int64_t li = B.seg_base[jstep] + li0;  // local segment (pools, buckets)
    const Blk b = load_blk(s, s.seg_lo + li0, k);
    const int64_t rel = L.blk_rel[beta];
    int lf, fa, fb;
    int64_t cL, cA, cB;
    run_shape(b, sh, lf, fa, fb, cL, cA, cB);
    // factor pointers without dynamic register-array indexing
    const int64_t* const fm[3] = {s.X.m, s.Y.m, s.Z.m};
    const int64_t* const ft[3] = {s.X.t, s.Y.t, s.Z.t};
    const int64_t oL = lf == 0 ? b.o[0] : (lf == 1 ? b.o[1] : b.o[2]);
    const int nL = (int)(lf == 0 ? b.n[0] : (lf == 1 ? b.n[1] : b.n[2]));
    // samp_idx32 over the long factor with its sample count hoisted
    const int cL0 = (int)(((int64_t)nL + ((int64_t)1 << sh) - 1) >> sh);
    auto sidx = [cL0](int j, int n, int shv) { return j < cL0 ? (int)((int64_t)j << shv) : n - 1; };
    const int64_t oA = fa == 0 ? b.o[0] : b.o[1];
    const int64_t nA = fa == 0 ? b.n[0] : b.n[1];
    const int64_t oB = fb == 2 ? b.o[2] : b.o[1];
    const int64_t nB = fb == 2 ? b.n[2] : b.n[1];
    const int64_t RI = L.run_item;
    const int64_t nch = (cL + RI - 1) / RI;
    int64_t run, ch, ja, jb;
    if (((wl | nch | cB) >> 31) == 0) {  // 32-bit division fast path
      const unsigned r32 = (unsigned)wl / (unsigned)nch;
      run = r32;
      ch = wl - (int64_t)r32 * nch;
      const unsigned a32 = r32 / (unsigned)cB;
      ja = a32;
      jb = run - (int64_t)a32 * cB;
    } else {
      run = wl / nch;
      ch = wl - run * nch;
      ja = run / cB;
      jb = run - ja * cB;
    }
    const int ia = (int)samp_idx(ja, nA, sh), ib = (int)samp_idx(jb, nB, sh);
    const int64_t* Am = fa == 0 ? fm[0] : fm[1];
    const int64_t* At = fa == 0 ? ft[0] : ft[1];
    const int64_t* Bm = fb == 2 ? fm[2] : fm[1];
    const int64_t* Bt = fb == 2 ? ft[2] : ft[1];
    const int64_t* Lm = (lf == 0 ? fm[0] : (lf == 1 ? fm[1] : fm[2])) + oL;
    const int64_t* Lt = (lf == 0 ? ft[0] : (lf == 1 ? ft[1] : ft[2])) + oL;
    const int64_t ms = __ldg(Am + oA + ia) + __ldg(Bm + oB + ib);
    const int64_t ts = __ldg(At + oA + ia) + __ldg(Bt + oB + ib);
    // (x, y, z) index of the tuple for the id (R6): the long factor varies
    const int ny = (int)b.n[1], nz = (int)b.n[2];
    const int j0 = (int)(ch * RI), j1 = (int)min(ch * RI + RI, cL);
    const int64_t* Gm = L.in.m + L.in.start[li];
    const int64_t* Gt = L.in.t + L.in.start[li];
    const int g = (int)L.in.cnt[li];
    const int64_t bb = L.bucket_base[li];
    const int64_t gml = g > 0 ? Gm[g - 1] : INF;  // largest G m (interpolation)
    // q: #G points with m < m of the current chunk start (galloping lower bound)
    int q = 0;
    int jj = j0;
    bool exact = false;  // q = lower_bound(mf) of the first chunk already
    if (one && g > 0) {  // warp-uniform: every lane of the warp is here
      q = warp_lower_bound(Gm, g, ms + __ldg(Lm + sidx(j0, nL, sh)));
      exact = true;
    }
    unsigned c_tests = 0, c_skip = 0, c_elem = 0, c_gallop = 0;
    while (jj < j1) {
      ++c_tests;
      const int je = min(jj + CHUNK, j1);
      const int64_t mf = ms + __ldg(Lm + sidx(jj, nL, sh));
      const int64_t tl = ts + __ldg(Lt + sidx(je - 1, nL, sh));
      const bool known = exact;
      exact = false;
      if (!known && q < g && Gm[q] < mf) {  // lower_bound(mf) in G, starting at q
        {  // short advances are the common case: probe q+1..q+4 with independent loads
          const int64_t v1 = q + 1 < g ? Gm[q + 1] : INF, v2 = q + 2 < g ? Gm[q + 2] : INF;
          const int64_t v3 = q + 3 < g ? Gm[q + 3] : INF, v4 = q + 4 < g ? Gm[q + 4] : INF;
          if (v1 >= mf) { q += 1; goto g_done; }
          if (v2 >= mf) { q += 2; goto g_done; }
          if (v3 >= mf) { q += 3; goto g_done; }
          if (v4 >= mf) { q += 4; goto g_done; }
          q += 4;  // Gm[q] < mf still: interpolation / gallop from here
        }
        ++c_gallop;
        if (g - q > 16) {
          // one interpolation probe between Gm[q] and Gm[g-1] (G's m values are
          // spread over the segment's range); the gallop then starts there
          const int64_t mq = Gm[q];
          if (gml < mf) {
            q = g;
            goto g_done;
          }
          int e = q + (int)((double)(mf - mq) / (double)(gml - mq) * (double)(g - 1 - q));
          e = e <= q ? q + 1 : (e > g - 1 ? g - 1 : e);
          if (Gm[e] < mf) {
            q = e;
          } else {  // lower bound in (q, e]: gallop down from e
            int stp = 1;
            while (e - stp > q && Gm[e - stp] >= mf) stp <<= 1;
            int a0 = e - stp < q ? q + 1 : e - stp + 1, a1 = e - (stp >> 1);
            // Gm[a1] >= mf (or a1 == e), lower bound in [a0, a1]
            while (a0 < a1) {
              const int mid = (a0 + a1) >> 1;
              if (Gm[mid] < mf) a0 = mid + 1;
              else a1 = mid;
            }
            q = a0;
            goto g_done;
          }
        }
        int step = 1;
        while (q + step < g && Gm[q + step] < mf) step <<= 1;
        int a0 = q + (step >> 1) + 1, a1 = min(q + step, g);
        while (a0 < a1) {
          const int mid = (a0 + a1) >> 1;
          if (Gm[mid] < mf) a0 = mid + 1;
          else a1 = mid;
        }
        q = a0;
      }
    g_done:
      if (q > 0 && Gt[q - 1] <= tl) {
        // G[q-1] (m < mf) strictly dominates the whole chunk and every later
        // element with t >= its t: gallop along the run to the first t below it.
        const int64_t tg = Gt[q - 1];
        if (ts + __ldg(Lt + sidx(j1 - 1, nL, sh)) >= tg) {  // common: the rest of the item
          c_skip += j1 - jj;
          jj = j1;
          continue;
        }
        int step = 1, last = je - 1;  // t(last) >= tg
        while (last + step < j1 && ts + __ldg(Lt + sidx(last + step, nL, sh)) >= tg) {
          last += step;
          step <<= 1;
        }
        int a0 = last + 1, a1 = min(last + step, j1);  // first index with t < tg in [a0, a1]
        while (a0 < a1) {
          const int mid = (a0 + a1) >> 1;
          if (ts + __ldg(Lt + sidx(mid, nL, sh)) >= tg) a0 = mid + 1;
          else a1 = mid;
        }
        c_skip += a0 - jj;
        jj = a0;
        continue;
      }
      c_elem += je - jj;
      // element-level test of the chunk: p = #G points with m <= m_x; the
      // run elements are loaded EPRE at a time ahead of the (dependent) G walk
      int p = q;
      // G[p] and G[p-1] kept in registers: consecutive run elements mostly
      // share p, so the walk and the dominance test reload only when p moves
      // (and G[p+1] one step ahead: a one-point advance does not wait for a load)
      int64_t gmp = p < g ? Gm[p] : INF, gmn = p + 1 < g ? Gm[p + 1] : INF;
      int64_t gmq = p > 0 ? Gm[p - 1] : 0, gtq = p > 0 ? Gt[p - 1] : INF;
      unsigned surv = 0;  // bit j - jj: run element j is a candidate
      uint64_t pdel = 0;  // 4 bits per candidate: min(p - q, 15) (its bucket, for the emission)
      for (int j4 = jj; j4 < je; j4 += EPRE) {
        int64_t em[EPRE], et[EPRE];
#pragma unroll
        for (int u = 0; u < EPRE; ++u) {
          const int iu = sidx(min(j4 + u, je - 1), nL, sh);
          em[u] = __ldg(Lm + iu);
          et[u] = __ldg(Lt + iu);
        }
#pragma unroll
        for (int u = 0; u < EPRE; ++u) {
          if (j4 + u >= je) break;
          const int64_t m = ms + em[u];
          const int64_t t = ts + et[u];
          if (gmp <= m) {
            do {
              gmq = gmp;
              ++p;
              gmp = gmn;
              gmn = p + 1 < g ? Gm[p + 1] : INF;
            } while (gmp <= m);
            gtq = Gt[p - 1];
          }
          if (!(p > 0 && (gtq < t || (gtq == t && gmq < m)))) {
            const int x = j4 + u - jj;
            surv |= 1u << x;
            pdel |= (uint64_t)min(p - q, 15) << (4 * x);
          }
        }
      }
      if (surv) {
        // one slot reservation per chunk for the coalesced threads (instead of
        // one per candidate), then the candidates are re-derived (L1 hits)
        cg::coalesced_group grp = cg::coalesced_threads();
        const unsigned nsv = __popc(surv);
        const unsigned off = cg::exclusive_scan(grp, nsv);
        const unsigned tot = grp.shfl(off + nsv, grp.size() - 1);
        unsigned long long base = 0;
        if (grp.thread_rank() == 0) base = atomicAdd(L.cand_cursor, (unsigned long long)tot);
        base = grp.shfl(base, 0) + off;
        int pp = q;
        while (surv) {
          const int b = __ffs(surv) - 1;
          surv &= surv - 1;
          const int il = sidx(jj + b, nL, sh);
          const int64_t m = ms + __ldg(Lm + il);
          const int64_t t = ts + __ldg(Lt + il);
          const int dp = (int)(pdel >> (4 * b)) & 15;  // p - q from the element test
          if (dp < 15) {
            pp = q + dp;
          } else {  // p >= q + 15: walk on from there
            pp = max(pp, q + 15);
            while (pp < g && Gm[pp] <= m) ++pp;
          }
          int64_t x, y, z;  // (x, y, z) in 64 bits for the id
          if (lf == 0) { x = il; y = ia; z = ib; }
          else if (lf == 1) { x = ia; y = il; z = ib; }
          else { x = ia; y = ib; z = il; }
          const uint64_t id = (uint64_t)(rel + (x * ny + y) * nz + z);
          const int64_t gb = bb + pp;
          const unsigned long long idx = base++;
          if ((int64_t)idx < L.cand_cap) {
            atomicAdd(L.bcount + gb, 1u);  // no return value: slots are taken in k_carry_scatter
            atomicMin(L.bmin + gb, (long long)t);
            L.cm[idx] = m;
            L.ct[idx] = t;
            L.cid[idx] = id;
            L.cgb[idx] = gb;
          }
        }
      }
      jj = je;
    }
    if (L.fstats) {
      atomicAdd(&L.hdr->fstat[0], 1ull);
      atomicAdd(&L.hdr->fstat[1], c_tests);
      atomicAdd(&L.hdr->fstat[2], c_skip);
      atomicAdd(&L.hdr->fstat[3], c_elem);
      atomicAdd(&L.hdr->fstat[4], (unsigned long long)g);
      atomicAdd(&L.hdr->fstat[7], (unsigned long long)c_gallop);
    }
  }
}

// Two register budgets for the same body (A/B: FT_FILTER_REGS=64 selects the
// 64-register variant, 8 CTAs of 128 threads per SM; default 80 registers).
__global__ void __launch_bounds__(128, 6) k_filter(BatchDev B, LevelDev L) { FT_PDL_ENTRY(); filter_body(B, L); }
__global__ void __launch_bounds__(128, 8) k_filter64(BatchDev B, LevelDev L) { FT_PDL_ENTRY(); filter_body(B, L); }


// Carry per bucket: exclusive prefix-min of bucket minima within the segment
// (the running minimum v of Alg.1 entering each bucket).
// After the bucket-offset scan: (1) the carry of every bucket = exclusive
// prefix-min of the bucket minima within its segment (Alg. 1's running
// minimum v entering the bucket), one CTA per segment; (2) every candidate
// moved into its bucket (grid-stride; a slot inside the bucket is taken by
// handing the bucket's count back down -- the order inside a bucket is
// irrelevant, buckets are sorted by (m, t, id) next).  One launch.
__constant__ unsigned char kBminFill[8] = {BMIN_FILL, BMIN_FILL, BMIN_FILL, BMIN_FILL,
                                           BMIN_FILL, BMIN_FILL, BMIN_FILL, BMIN_FILL};

__global__ void __launch_bounds__(256) k_carry_scatter(BatchDev B, LevelDev L, int64_t* ncand) {
  FT_PDL_ENTRY();
  __shared__ long long sh[33];
  __shared__ long long chunk_min;
  const unsigned long long cc = *(volatile unsigned long long*)L.cand_cursor;  // final: k_filter is done
  const int64_t n = (int64_t)cc < L.cand_cap ? (int64_t)cc : L.cand_cap;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // candidate and bucket totals (after k_filter)
    L.hdr->cand_total[L.level] = cc;
    L.hdr->bucket_total[L.level] = L.bucket_base[B.nseg];
    if ((int64_t)cc > L.cand_cap) atomicExch(&L.hdr->overflow, 1ull);
    *ncand = n;
  }
  if ((int64_t)cc > L.cand_cap || L.hdr->overflow) return;
  const int64_t nloc = B.nseg;
  for (int64_t li = blockIdx.x; li < nloc; li += gridDim.x) {
    if (!is_filter(L.seg_d[li], L.level)) continue;
    const int64_t b0 = L.bucket_base[li], nb = L.nb[li];
    long long carry = INF;
    for (int64_t c0 = 0; c0 < nb; c0 += 256) {
      const int64_t i = c0 + threadIdx.x;
      const long long v = i < nb ? L.bmin[b0 + i] : INF;
      const long long ex = block_excl_min<256>(v, sh);
      if (i < nb) {
        L.bcarry[b0 + i] = ex < carry ? ex : carry;
        L.bmin[b0 + i] = *(const long long*)kBminFill;  // back to the reset state
      }
      if (threadIdx.x == 255) chunk_min = v < ex ? v : ex;
      __syncthreads();
      carry = chunk_min < carry ? chunk_min : carry;
      __syncthreads();
    }
  }
  // consecutive candidates mostly share a bucket (k_filter emits a chunk's
  // candidates contiguously): lanes with equal buckets take their slots with
  // one atomic (warp-aggregated), the leader handing out ranks
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < n; i0 += gstride) {
    const int64_t i = i0 + lane;
    const bool act = i < n;
    const int64_t gb = act ? L.cgb[i] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, gb);
    const int leader = __ffs(peers) - 1;
    unsigned top = 0;
    if (act && lane == leader) top = atomicSub(L.bcount + gb, (unsigned)__popc(peers));
    top = __shfl_sync(0xffffffffu, top, leader);
    if (act) {
      const unsigned rank = __popc(peers & ((1u << lane) - 1u));
      const int64_t d = L.boff[gb] + (int64_t)(top - 1u - rank);
      L.gm[d] = L.cm[i];
      L.gt[d] = L.ct[i];
      L.gid[d] = L.cid[i];
    }
  }
}

// K2+K3 for buckets of 33..WARP_DIRECT candidates: one warp per bucket,
// register bitonic sort by shuffles (R rows of 32), Alg.1 sweep with the
// bucket's carry.  The sort runs on single 64-bit keys (m << 8 | e) when
// every m fits in B.kspan bits (<= 55) and the bucket's m values are distinct
// (then the key order is the (m, t, id) order, R1/R3/R6); otherwise on the
// full (m, t, id) triple.  Only kept elements are written back (k_compact
// reads nothing else); larger buckets go to the CTA kernels.
template <int R>
__device__ __forceinline__ void warp_bucket(const LevelDev& L, int64_t bkt, int64_t c, int64_t base, int kspan) {
  const int lane = threadIdx.x & 31;
  const int sb = kspan < 55 ? kspan : 55;
  uint64_t k[R];
  bool fits = true;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = (r << 5) | lane;
    k[r] = ~0ull;
    if (e < c) {
      const uint64_t v = (uint64_t)L.gm[base + e];
      fits = fits && (v >> sb) == 0;
      k[r] = (v << 8) | (uint64_t)e;
    }
  }
  bool keyed = __all_sync(0xffffffffu, fits);
  if (keyed) {
    warp_bitonic_keys<R>(k);
    bool tie = false;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = (r << 5) | lane;
      uint64_t prev = __shfl_up_sync(0xffffffffu, k[r], 1);
      const uint64_t rowlast = __shfl_sync(0xffffffffu, k[r > 0 ? r - 1 : 0], 31);
      if (lane == 0) prev = r > 0 ? rowlast : ~0ull;
      if (e < c && prev != ~0ull && (prev >> 8) == (k[r] >> 8)) tie = true;
    }
    keyed = !__any_sync(0xffffffffu, tie);
  }
  int64_t m[R], t[R];
  uint64_t id[R];
  if (keyed) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = (r << 5) | lane;
      const int ix = (int)(k[r] & 255u);
      m[r] = e < c ? (int64_t)(k[r] >> 8) : INF;
      t[r] = e < c ? L.gt[base + ix] : INF;
      id[r] = e < c ? L.gid[base + ix] : ~0ull;
    }
  } else {
    if (L.fstats && lane == 0) atomicAdd(&L.hdr->bfall[1], 1ull);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = (r << 5) | lane;
      m[r] = e < c ? L.gm[base + e] : INF;
      t[r] = e < c ? L.gt[base + e] : INF;
      id[r] = e < c ? L.gid[base + e] : ~0ull;
    }
    warp_bitonic<R>(m, t, id);
  }
  __syncwarp();  // every read of the bucket precedes the in-place writes
  long long carry = L.bcarry[bkt];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = (r << 5) | lane;
    const long long inc = warp_incl_min(t[r]);
    long long ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = INF;
    const long long v = ex < carry ? ex : carry;
    if (e < c) {
      const bool kf = t[r] < v;
      L.gflag[base + e] = kf;
      if (kf) {
        L.gm[base + e] = m[r];
        L.gt[base + e] = t[r];
        L.gid[base + e] = id[r];
      }
    }
    const long long rowmin = __shfl_sync(0xffffffffu, inc, 31);
    carry = rowmin < carry ? rowmin : carry;
  }
}

// Buckets of 2..32 candidates: the 32/S buckets of one size class
// (S/2, S] of a 32-bucket tile are sorted together, one per S-lane group
// (bitonic with shuffles inside the group, segmented warp scans for Alg. 1).
// Keys as in warp_bucket (m << 5 | e; the (m, t, id) network for the whole
// warp pass when some m needs more than B.kspan bits or a group has equal m;
// always for pairs, where the triple network is the cheaper one).
template <int S>
__device__ __forceinline__ void bucket_groups(const LevelDev& L, int64_t c, int64_t b0, int* slist, int kspan) {
  const int lane = threadIdx.x & 31;
  const bool mine = c > S / 2 && c <= S;
  const unsigned mask = __ballot_sync(0xffffffffu, mine);
  if (mask == 0) return;
  if (mine) slist[__popc(mask & ((1u << lane) - 1u))] = lane;
  __syncwarp();
  const int n = __popc(mask);
  constexpr int G = 32 / S;
  const int g = lane / S, e = lane & (S - 1);
  const int sb = kspan < 58 ? kspan : 58;
  for (int p0 = 0; p0 < n; p0 += G) {
    const int q = p0 + g;
    const int src = q < n ? slist[q] : 0;
    const int64_t cc = __shfl_sync(0xffffffffu, c, src);
    int64_t m = INF, t = INF, base = 0;
    uint64_t id = ~0ull;
    long long carry = INF;
    const int64_t bk = b0 + src;
    const bool valid = q < n && e < cc;
    if (q < n) {
      base = L.boff[bk];
      carry = L.bcarry[bk];
      if (e < cc) {
        m = L.gm[base + e];
        t = L.gt[base + e];
        id = L.gid[base + e];
      }
    }
    const bool fits = S > 2 && (!valid || ((uint64_t)m >> sb) == 0);
    uint64_t key = valid ? ((uint64_t)m << 5) | (uint64_t)e : ~0ull;
#pragma unroll
    for (int k = 2; k <= (S > 2 ? S : 1); k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        const uint64_t pk = __shfl_xor_sync(0xffffffffu, key, j);
        const bool up = (e & k) == 0, lower = (e & j) == 0;
        key = (lower == up) ? (pk < key ? pk : key) : (pk > key ? pk : key);
      }
    }
    const uint64_t pv = S > 2 ? __shfl_up_sync(0xffffffffu, key, 1, S) : 0;
    const bool tie = e > 0 && key != ~0ull && (pv >> 5) == (key >> 5);
    if (__all_sync(0xffffffffu, fits && !tie)) {
      const int from = (lane & ~(S - 1)) | (int)(key & (S - 1));
      const int64_t tt = __shfl_sync(0xffffffffu, t, from);
      const uint64_t ii = __shfl_sync(0xffffffffu, id, from);
      if (key != ~0ull) {
        m = (int64_t)(key >> 5);
        t = tt;
        id = ii;
      } else {
        m = INF;
        t = INF;
        id = ~0ull;
      }
    } else {
      if (S > 2 && L.fstats && lane == 0) atomicAdd(&L.hdr->bfall[0], 1ull);
#pragma unroll
      for (int k = 2; k <= S; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
          const int64_t pm = __shfl_xor_sync(0xffffffffu, m, j);
          const int64_t pt = __shfl_xor_sync(0xffffffffu, t, j);
          const uint64_t pi = __shfl_xor_sync(0xffffffffu, id, j);
          const bool up = (e & k) == 0, lower = (e & j) == 0;
          const bool p_lt = key_lt(pm, pt, pi, m, t, id);
          if ((lower == up) ? p_lt : !p_lt) {
            m = pm;
            t = pt;
            id = pi;
          }
        }
      }
    }
    long long inc = t;
#pragma unroll
    for (int d = 1; d < S; d <<= 1) {
      const long long u = __shfl_up_sync(0xffffffffu, inc, d, S);
      if (e >= d) inc = u < inc ? u : inc;
    }
    long long ex = __shfl_up_sync(0xffffffffu, inc, 1, S);
    if (e == 0) ex = INF;
    const long long v = ex < carry ? ex : carry;
    __syncwarp();  // every read of the pass's buckets precedes the in-place writes
    if (q < n && e < cc) {
      const bool kf = t < v;
      L.gflag[base + e] = kf;
      if (kf) {
        L.gm[base + e] = m;
        L.gt[base + e] = t;
        L.gid[base + e] = id;
      }
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(256, 3) k_bucket_small(BatchDev Bt, LevelDev L) {
  FT_PDL_ENTRY();
  if (L.hdr->overflow) return;
  __shared__ int slist_all[8][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int* slist = slist_all[wid];
  const int64_t B = min(L.bucket_base[Bt.nseg], L.bcap);
  const int64_t nw = (int64_t)gridDim.x * 8;
  // tiles of T buckets per warp: T = 1 (a warp per bucket) while there are
  // few buckets, up to 32 when there are many (size classes batch up)
  int64_t T = B / (2 * nw);
  T = T < 1 ? 1 : (T > 32 ? 32 : T);
  const int64_t ntile = (B + T - 1) / T;
  for (int64_t tile = (int64_t)blockIdx.x * 8 + wid; tile < ntile; tile += nw) {
    const int64_t b0 = tile * T;
    const int64_t bkt = b0 + lane;
    const int64_t c = lane < T && bkt < B ? L.boff[bkt + 1] - L.boff[bkt] : 0;
    if (L.fstats && c > 0) {
      const int cls = c == 1 ? 0 : c <= 4 ? 1 : c <= 8 ? 2 : c <= 16 ? 3 : c <= 32 ? 4 : c <= 64 ? 5
                      : c <= 128 ? 6 : c <= 256 ? 7 : c <= 4096 ? 8 : 9;
      atomicAdd(&L.hdr->bstat[0][cls], 1ull);
      atomicAdd(&L.hdr->bstat[1][cls], (unsigned long long)c);
    }
    if (c > WARP_DIRECT) L.large_list[atomicAdd(L.large_n, 1ull)] = bkt;
    if (c == 1) {  // a single candidate: kept iff below the carry
      const int64_t base = L.boff[bkt];
      L.gflag[base] = L.gt[base] < L.bcarry[bkt] ? 1 : 0;
    }
    bucket_groups<2>(L, c, b0, slist, Bt.kspan);
    bucket_groups<4>(L, c, b0, slist, Bt.kspan);
    bucket_groups<8>(L, c, b0, slist, Bt.kspan);
    bucket_groups<16>(L, c, b0, slist, Bt.kspan);
    bucket_groups<32>(L, c, b0, slist, Bt.kspan);
    unsigned big = __ballot_sync(0xffffffffu, c > 32 && c <= WARP_DIRECT);
    while (big) {
      const int src = __ffs(big) - 1;
      big &= big - 1;
      const int64_t cb = __shfl_sync(0xffffffffu, c, src);
      const int64_t bk = b0 + src;
      const int64_t base = L.boff[bk];
      if (cb <= 64) warp_bucket<2>(L, bk, cb, base, Bt.kspan);
      else if (cb <= 128) warp_bucket<4>(L, bk, cb, base, Bt.kspan);
      else warp_bucket<8>(L, bk, cb, base, Bt.kspan);
    }
  }
}

// K2+K3 for buckets of 33..BUCKET_SMEM candidates: one CTA, bitonic in smem.
// Register-blocked sort + Alg. 1 of one bucket of c <= 32 R x 8 candidates
// (in place in gm/gt/gid, keep flags in gflag; carry from earlier buckets).
template <int R>
__device__ __forceinline__ void cta_bucket_regs(const LevelDev& L, int64_t bkt, int64_t c, int64_t base,
                                                int64_t* xm, int64_t* xt, uint64_t* xid,
                                                long long* sh) {
  constexpr int NW = DIRECT_NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int eb = wid * 32 * R;
  int64_t m[R], t[R];
  uint64_t id[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = eb + (r << 5) + lane;
    if (e < c) {
      m[r] = L.gm[base + e];
      t[r] = L.gt[base + e];
      id[r] = L.gid[base + e];
    } else {
      m[r] = INF;
      t[r] = INF;
      id[r] = ~0ull;
    }
  }
  cta_bitonic_regs<R>(m, t, id, xm, xt, xid);
  long long wmin = INF;
#pragma unroll
  for (int r = 0; r < R; ++r) wmin = t[r] < wmin ? t[r] : wmin;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long u = __shfl_xor_sync(0xffffffffu, wmin, o);
    wmin = u < wmin ? u : wmin;
  }
  if (lane == 0) sh[wid] = wmin;
  __syncthreads();
  long long carry = L.bcarry[bkt];
  for (int w = 0; w < wid; ++w) carry = sh[w] < carry ? sh[w] : carry;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = eb + (r << 5) + lane;
    const long long inc = warp_incl_min(t[r]);
    long long ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = INF;
    const long long v = ex < carry ? ex : carry;
    if (e < c) {
      const bool kf = t[r] < v;
      L.gflag[base + e] = kf;
      if (kf) {  // k_compact reads kept elements only
        L.gm[base + e] = m[r];
        L.gt[base + e] = t[r];
        L.gid[base + e] = id[r];
      }
    }
    const long long rowmin = __shfl_sync(0xffffffffu, inc, 31);
    carry = rowmin < carry ? rowmin : carry;
  }
  (void)NW;
  __syncthreads();  // sh / x* reuse
}

template <int NT>
__device__ void bucket_huge_one(const LevelDev& L, int64_t bkt, int64_t* sm, int64_t* stt, uint64_t* sid,
                                long long* sh);

__global__ void __launch_bounds__(DIRECT_NT, 3) k_bucket_large(LevelDev L) {
  FT_PDL_ENTRY();
  extern __shared__ int64_t dyn[];
  int64_t* sm = dyn;
  int64_t* stt = sm + BUCKET_SMEM;
  uint64_t* sid = (uint64_t*)(stt + BUCKET_SMEM);
  int* kf = (int*)(sid + BUCKET_SMEM);
  __shared__ long long sh[33];
  if (L.hdr->overflow) return;
  const int64_t nl = *L.large_n;
  for (int64_t e = blockIdx.x; e < nl; e += gridDim.x) {
    const int64_t bkt = L.large_list[e];
    const int64_t c = L.boff[bkt + 1] - L.boff[bkt];
    if (c > BUCKET_SMEM) {  // huge: tiles + global merges in this CTA (rare)
      bucket_huge_one<DIRECT_NT>(L, bkt, sm, stt, sid, sh);
      __syncthreads();
      continue;
    }
    const int64_t base = L.boff[bkt];
    int N = 1;
    while (N < c) N <<= 1;
    if (N <= 2 * DIRECT_NT) {  // c <= 512
      cta_bucket_regs<2>(L, bkt, c, base, sm, stt, sid, sh);
      continue;
    }
    if (N == 4 * DIRECT_NT) {  // c <= 1024
      cta_bucket_regs<4>(L, bkt, c, base, sm, stt, sid, sh);
      continue;
    }
    for (int i = threadIdx.x; i < N; i += DIRECT_NT) {
      if (i < c) {
        sm[i] = L.gm[base + i];
        stt[i] = L.gt[base + i];
        sid[i] = L.gid[base + i];
      } else {
        sm[i] = INF;
        stt[i] = INF;
        sid[i] = ~0ull;
      }
    }
    __syncthreads();
    bitonic_smem<DIRECT_NT>(sm, stt, sid, N);
    alg1_sweep_smem<DIRECT_NT>(stt, (int)c, L.bcarry[bkt], kf, sh);
    for (int i = threadIdx.x; i < c; i += DIRECT_NT) {
      L.gflag[base + i] = kf[i] != 0;
      if (kf[i]) {
        L.gm[base + i] = sm[i];
        L.gt[base + i] = stt[i];
        L.gid[base + i] = sid[i];
      }
    }
    __syncthreads();
  }
}

// K2+K3 for a huge bucket (> BUCKET_SMEM candidates), one CTA of NT threads
// (called from k_bucket_large): smem-sorted tiles, then pairwise merges
// through the (dead) candidate arrays as scratch, then Alg. 1 with carry.
template <int NT>
__device__ void bucket_huge_one(const LevelDev& L, int64_t bkt, int64_t* sm, int64_t* stt, uint64_t* sid,
                                long long* sh) {
  {
    const int64_t c = L.boff[bkt + 1] - L.boff[bkt];
    const int64_t base = L.boff[bkt];
    if (threadIdx.x == 0) atomicAdd(&L.hdr->huge, 1ull);
    // 1) sort tiles of BUCKET_SMEM
    for (int64_t t0 = 0; t0 < c; t0 += BUCKET_SMEM) {
      const int64_t n = min((int64_t)BUCKET_SMEM, c - t0);
      for (int i = threadIdx.x; i < BUCKET_SMEM; i += NT) {
        if (i < n) {
          sm[i] = L.gm[base + t0 + i];
          stt[i] = L.gt[base + t0 + i];
          sid[i] = L.gid[base + t0 + i];
        } else {
          sm[i] = INF;
          stt[i] = INF;
          sid[i] = ~0ull;
        }
      }
      __syncthreads();
      bitonic_smem<NT>(sm, stt, sid, BUCKET_SMEM);
      for (int i = threadIdx.x; i < n; i += NT) {
        L.gm[base + t0 + i] = sm[i];
        L.gt[base + t0 + i] = stt[i];
        L.gid[base + t0 + i] = sid[i];
      }
      __syncthreads();
    }
    // 2) merge passes: src/dst alternate between grouped and candidate arrays
    int64_t *am = L.gm + base, *at = L.gt + base;
    uint64_t* ai = L.gid + base;
    int64_t *bm = L.cm + base, *bt = L.ct + base;
    uint64_t* bi = L.cid + base;
    for (int64_t wdt = BUCKET_SMEM; wdt < c; wdt <<= 1) {
      for (int64_t i = threadIdx.x; i < c; i += NT) {
        const int64_t r0 = (i / (2 * wdt)) * 2 * wdt;
        const int64_t mid = min(r0 + wdt, c), r1 = min(r0 + 2 * wdt, c);
        const bool left = i < mid;
        const int64_t o0 = left ? mid : r0, o1 = left ? r1 : mid;
        // rank of key i in the other run
        int64_t lo = o0, hi = o1;
        while (lo < hi) {
          int64_t q = (lo + hi) >> 1;
          if (key_lt(am[q], at[q], ai[q], am[i], at[i], ai[i])) lo = q + 1;
          else hi = q;
        }
        const int64_t pos = r0 + (left ? (i - r0) : (i - mid)) + (lo - o0);
        bm[pos] = am[i];
        bt[pos] = at[i];
        bi[pos] = ai[i];
      }
      __syncthreads();
      int64_t* x = am; am = bm; bm = x;
      x = at; at = bt; bt = x;
      uint64_t* y = ai; ai = bi; bi = y;
    }
    if (am != L.gm + base) {
      for (int64_t i = threadIdx.x; i < c; i += NT) {
        L.gm[base + i] = am[i];
        L.gt[base + i] = at[i];
        L.gid[base + i] = ai[i];
      }
      __syncthreads();
    }
    // 3) Alg.1 sweep in chunks with carry
    long long carry = L.bcarry[bkt];
    __shared__ long long s_carry_h;
    for (int64_t c0 = 0; c0 < c; c0 += NT) {
      const int64_t i = c0 + threadIdx.x;
      const long long v = i < c ? L.gt[base + i] : INF;
      long long ex = block_excl_min<NT>(v, sh);
      long long pv = ex < carry ? ex : carry;
      if (i < c) L.gflag[base + i] = v < pv ? 1 : 0;
      if (threadIdx.x == NT - 1) s_carry_h = v < pv ? v : pv;
      __syncthreads();
      carry = s_carry_h;
      __syncthreads();
    }
  }
}

// Survivors of the filter path go to the level pool at the fixed offset
// `base` = this level's direct-sample total (the direct kernels' outputs,
// reserved by cursor atomics, never exceed it; the pool holds both).
// Survivors of the filter path go to the level pool at the fixed offset
// `base` = this level's direct-sample total (the direct kernels' outputs,
// reserved by cursor atomics, never exceed it; the pool holds both), and
// every filter segment's pool range is recorded (one launch).
__global__ void k_compact(BatchDev B, LevelDev L, const int64_t* gpos, const int64_t* ncand, int64_t base) {
  FT_PDL_ENTRY();
  const int64_t n = *ncand;
  const int64_t g0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gstride = (int64_t)gridDim.x * blockDim.x;
  if (g0 == 0) {
    const int64_t tot = gpos[n];
    atomicAdd(&L.hdr->out_total[L.level], (unsigned long long)tot);
    if (base + tot > L.out.cap) atomicExch(&L.hdr->overflow, 1ull);
    *L.cand_cursor = 0;  // ready for the next filter level
    *L.large_n = 0;
  }
  for (int64_t li = g0; li < B.nseg; li += gstride) {
    if (!is_filter(L.seg_d[li], L.level)) continue;
    const int64_t b0 = L.bucket_base[li], b1 = b0 + L.nb[li];
    const int64_t lo = L.boff[b0], hi = L.boff[b1];
    L.out.start[li] = base + gpos[lo];
    L.out.cnt[li] = gpos[hi] - gpos[lo];
  }
  if (L.hdr->overflow) return;
  for (int64_t i = g0; i < n; i += gstride) {
    if (gpos[i + 1] != gpos[i] && base + gpos[i] < L.out.cap) {
      const int64_t d = base + gpos[i];
      L.out.m[d] = L.gm[i];
      L.out.t[d] = L.gt[i];
      L.out.id[d] = L.gid[i];
    }
  }
}

// Final gather of the level-0 pool into every step's CSR output set (one
// warp per segment).
__global__ void __launch_bounds__(256) k_gather(BatchDev B, Pool P) {
  FT_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t gs = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gs < B.nseg; gs += nw) {
    const int j = find_base(B.seg_base, B.nsteps, gs);
    const StepDev& s = B.steps[j];
    const int64_t li = gs - B.seg_base[j];
    const int64_t src = P.start[gs], n = P.cnt[gs], d = s.out_off[li];
    for (int64_t i = lane; i < n; i += 32) {
      s.out_m[d + i] = P.m[src + i];
      s.out_t[d + i] = P.t[src + i];
      s.out_bp[d + i] = P.id[src + i];
    }
  }
}

// Single-rank gather: the arena is in `pos` order (step-major exclusive scan
// of the survivor counts), so output element i belongs to the segment gs with
// pos[gs] <= i < pos[gs+1].  Tiles of 2048 outputs: one binary search per CTA
// for the tile's segment range, then a short search per element.
__global__ void __launch_bounds__(256) k_gather_flat(BatchDev B, Pool P, const int64_t* pos,
                                                     int64_t* om, int64_t* ot, uint64_t* obp) {
  FT_PDL_ENTRY();
  __shared__ int64_t seg_lo_s, seg_hi_s;
  const int64_t total = pos[B.nseg];
  const int64_t ntiles = (total + 2047) / 2048;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t t0 = tile * 2048, t1 = min(t0 + 2048, total);
    if (threadIdx.x < 2) {  // segment containing t0 (thread 0) and t1-1 (thread 1)
      const int64_t x = threadIdx.x == 0 ? t0 : t1 - 1;
      int64_t lo = 0, hi = B.nseg;  // largest gs with pos[gs] <= x
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (pos[mid] <= x) lo = mid;
        else hi = mid;
      }
      if (threadIdx.x == 0) seg_lo_s = lo;
      else seg_hi_s = lo;
    }
    __syncthreads();
    const int64_t slo = seg_lo_s, shi = seg_hi_s;
    for (int64_t i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
      int64_t lo = slo, hi = shi + 1;
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (pos[mid] <= i) lo = mid;
        else hi = mid;
      }
      const int64_t src = P.start[lo] + (i - pos[lo]);
      om[i] = P.m[src];
      ot[i] = P.t[src];
      obp[i] = P.id[src];
    }
    __syncthreads();
  }
}

// Device-side wave offsets (single rank): from the level-0 survivor counts
// and their exclusive scan `pos` (step-major = arena order), write every
// step's relative CSR offsets into the arena offset array (step j's nseg+1
// entries start at seg_base[j] + j) and per-step totals / max / tuples.
__global__ void k_wave_off(BatchDev B, const int64_t* cnt, const int64_t* seg_tuples,
                           const int64_t* pos, int64_t* off, int64_t* step_arr) {
  FT_PDL_ENTRY();
  const int64_t gs = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gs >= B.nseg) return;
  const int j = find_base(B.seg_base, B.nsteps, gs);
  const int64_t sb = B.seg_base[j], se = B.seg_base[j + 1];
  const int64_t base = pos[sb];
  off[sb + j + (gs - sb)] = pos[gs] - base;
  if (gs == se - 1) {
    off[sb + j + (gs - sb) + 1] = pos[se] - base;
    step_arr[3 * j] = pos[se] - base;
  }
  // per-step max / sum: one atomic per run of equal j within the warp
  unsigned long long mx = (unsigned long long)cnt[gs], sm = (unsigned long long)seg_tuples[gs];
  const unsigned act = __activemask();
  const unsigned same = __match_any_sync(act, j);
  // segments are step-major, so `same` is a contiguous run of lanes [a, b];
  // after offset o lane i holds [i, min(i + 2o - 1, b)]
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long m2 = __shfl_down_sync(act, mx, o), s2 = __shfl_down_sync(act, sm, o);
    const int src = (threadIdx.x & 31) + o;
    if (src < 32 && ((same >> src) & 1u)) {
      mx = m2 > mx ? m2 : mx;
      sm += s2;
    }
  }
  if ((threadIdx.x & 31) == __ffs(same) - 1) {
    atomicMax((unsigned long long*)&step_arr[3 * j + 1], mx);
    atomicAdd((unsigned long long*)&step_arr[3 * j + 2], sm);
  }
}

static int grid_for(int64_t n, int nt, int maxg);

// ---------------------------------------------------------------------------
// Cost validation for ft_set_costs_all (R10 bounds; edges with m = 0).

__global__ void k_validate(const int64_t* d, int64_t n, int32_t* status) {
  int bits = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = d[i];
    if (v < 0) bits |= 1;
    if (v >= ((int64_t)1 << 40)) bits |= 2;
  }
  bits = __reduce_or_sync(0xffffffffu, bits);
  if ((threadIdx.x & 31) == 0 && bits) atomicOr(status, bits);
}

__global__ void k_edge_mzero(const int64_t* em, const int64_t* e_off, int ne, char* mz) {
  for (int e = blockIdx.x; e < ne; e += gridDim.x) {
    int nz = 0;
    for (int64_t i = e_off[e] + threadIdx.x; i < e_off[e + 1]; i += blockDim.x) nz |= em[i] != 0;
    nz = __syncthreads_or(nz);
    if (threadIdx.x == 0) mz[e] = nz ? 0 : 1;
  }
}

cudaError_t validate_costs(const int64_t* d, int64_t n, const int64_t* em,
                           const std::vector<int64_t>& e_off, int ne, int32_t* status_host,
                           char* mz_host, cudaStream_t st, const DevAlloc& A) {
  int32_t* dstat = nullptr;
  int64_t* doff = nullptr;
  char* dmz = nullptr;
  cudaError_t e = A.get((void**)&dstat, sizeof(int32_t) + 16, st);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(dstat, 0, sizeof(int32_t), st);
  if (n > 0) k_validate<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(d, n, dstat);
  if (ne > 0) {
    if ((e = A.get((void**)&doff, sizeof(int64_t) * (ne + 1), st)) != cudaSuccess) return e;
    if ((e = A.get((void**)&dmz, ne, st)) != cudaSuccess) return e;
    cudaMemcpyAsync(doff, e_off.data(), sizeof(int64_t) * (ne + 1), cudaMemcpyHostToDevice, st);
    k_edge_mzero<<<std::min(ne, 148 * 8), 128, 0, st>>>(em, doff, ne, dmz);
    cudaMemcpyAsync(mz_host, dmz, ne, cudaMemcpyDeviceToHost, st);
  }
  cudaMemcpyAsync(status_host, dstat, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  A.put(dstat, st);
  A.put(doff, st);
  A.put(dmz, st);
  return cudaGetLastError();
}

// Multi-rank exchange helpers (device offsets over the whole wave).
__global__ void __launch_bounds__(256) k_gather_range(Pool P, const int64_t* pos, int64_t lo, int64_t hi,
                                                      int64_t* om, int64_t* ot, uint64_t* obp) {
  __shared__ int64_t seg_lo_s, seg_hi_s;
  const int64_t a0 = pos[lo], a1 = pos[hi];
  const int64_t ntiles = (a1 - a0 + 2047) / 2048;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t t0 = a0 + tile * 2048, t1 = min(t0 + 2048, a1);
    if (threadIdx.x < 2) {
      const int64_t x = threadIdx.x == 0 ? t0 : t1 - 1;
      int64_t l = lo, h = hi;  // largest gs in [lo, hi) with pos[gs] <= x
      while (h - l > 1) {
        const int64_t mid = (l + h) >> 1;
        if (pos[mid] <= x) l = mid;
        else h = mid;
      }
      if (threadIdx.x == 0) seg_lo_s = l;
      else seg_hi_s = l;
    }
    __syncthreads();
    const int64_t slo = seg_lo_s, shi = seg_hi_s;
    for (int64_t i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
      int64_t l = slo, h = shi + 1;
      while (h - l > 1) {
        const int64_t mid = (l + h) >> 1;
        if (pos[mid] <= i) l = mid;
        else h = mid;
      }
      const int64_t src = P.start[l - lo] + (i - pos[l]);
      om[i] = P.m[src];
      ot[i] = P.t[src];
      obp[i] = P.id[src];
    }
    __syncthreads();
  }
}

cudaError_t wave_offsets(const int64_t* cnt, const int64_t* tup, int64_t NS, int ns,
                         const int64_t* sbase_dev, int64_t* pos, int64_t* off, int64_t* stats,
                         int64_t* scan_tmp, cudaStream_t st) {
  BatchDev B{};
  B.seg_base = sbase_dev;
  B.nsteps = ns;
  B.nseg = NS;
  scan_excl<int64_t>(cnt, pos, nullptr, NS, scan_tmp, st, true);  // freshly allocated scratch
  cudaMemsetAsync(stats, 0, sizeof(int64_t) * 3 * ns, st);
  k_wave_off<<<grid_for(NS, 256, 1 << 30), 256, 0, st>>>(B, cnt, tup, pos, off, stats);
  return cudaGetLastError();
}

cudaError_t gather_range(const Pool& P, const int64_t* pos, int64_t lo, int64_t hi, int64_t nout,
                         int64_t* om, int64_t* ot, uint64_t* obp, cudaStream_t st) {
  if (hi <= lo || nout <= 0) return cudaSuccess;
  k_gather_range<<<grid_for(nout, 2048, 148 * 16), 256, 0, st>>>(P, pos, lo, hi, om, ot, obp);
  return cudaGetLastError();
}

int64_t scan_tmp_elems(int64_t n) { return ntiles_cap_slot(n) + 8; }

// Multi-rank exchange by all-gathers: rank q's block of the
// gathered buffer holds its segments' {counts[maxloc], tuples[maxloc]}; wave
// segment gs of rank q (lo[q] <= gs < lo[q+1]) is local segment gs - lo[q].
__global__ void k_unpack_counts(const int64_t* all, int64_t maxloc, const int64_t* lo, int world, int64_t NS,
                                int64_t* cnt, int64_t* tup) {
  for (int64_t gs = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gs < NS;
       gs += (int64_t)gridDim.x * blockDim.x) {
    int q = 0;
    while (q + 1 < world && lo[q + 1] <= gs) ++q;
    const int64_t* blk = all + (int64_t)q * 2 * maxloc;
    cnt[gs] = blk[gs - lo[q]];
    tup[gs] = blk[maxloc + gs - lo[q]];
  }
}

// Rank q's staged survivors {m[cap], t[cap], bp[cap]} (gathered) -> the wave
// arena at [posb[q], posb[q+1]) (blockIdx.y = q).
__global__ void k_unpack_data(const int64_t* all, int64_t cap, const int64_t* posb, int64_t* om, int64_t* ot,
                              uint64_t* obp) {
  const int q = blockIdx.y;
  const int64_t a0 = posb[q], n = posb[q + 1] - a0;
  const int64_t* blk = all + (int64_t)q * 3 * cap;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    om[a0 + i] = blk[i];
    ot[a0 + i] = blk[cap + i];
    obp[a0 + i] = (uint64_t)blk[2 * cap + i];
  }
}

cudaError_t unpack_counts(const int64_t* all, int64_t maxloc, const int64_t* lo_dev, int world, int64_t NS,
                          int64_t* cnt, int64_t* tup, cudaStream_t st) {
  if (NS <= 0) return cudaSuccess;
  k_unpack_counts<<<grid_for(NS, 256, 148 * 8), 256, 0, st>>>(all, maxloc, lo_dev, world, NS, cnt, tup);
  return cudaGetLastError();
}

cudaError_t unpack_data(const int64_t* all, int64_t cap, const int64_t* posb_dev, int world, int64_t maxn,
                        int64_t* om, int64_t* ot, uint64_t* obp, cudaStream_t st) {
  if (maxn <= 0) return cudaSuccess;
  k_unpack_data<<<dim3(grid_for(maxn, 256, 148 * 4), world), 256, 0, st>>>(all, cap, posb_dev, om, ot, obp);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Host side

// Grow-only scratch with geometric growth: reallocation happens O(log size)
// times per process, not per step.  Callers have synchronised the stream
// since the buffer's last use (every wave ends with a stream sync).
static cudaError_t grow_raw(const DevAlloc& A, cudaStream_t st, void** p, size_t* have, size_t need,
                            size_t hw) {
  if (need <= *have && *p) return cudaSuccess;
  // after a release (hooked runners hand their scratch back when their last
  // graph goes), the first growth goes straight to the previous capacity:
  // one allocation of a size a caching allocator has seen before
  size_t nb = std::max<size_t>({need, 2 * *have, (size_t)1 << 16, hw});
  if (*p) {
    A.put(*p, st, true);
    *p = nullptr;
    *have = 0;
  }
  cudaError_t e = A.get(p, nb, st, true);
  if (e == cudaSuccess) *have = nb;
  return e;
}

#define GROW(buf, T, n)                                                         \
  do {                                                                          \
    cudaError_t e__ = grow_raw(alloc, st, (void**)&buf.p, &buf.bytes, sizeof(T) * (size_t)(n), buf.hw); \
    if (e__ != cudaSuccess) return e__;                                         \
  } while (0)

StepRunner::StepRunner() {}
StepRunner::~StepRunner() { release(); }

void StepRunner::release() {
  release_device();
  if (hdr_host) cudaFreeHost(hdr_host);
  hdr_host = nullptr;
  if (cnt_host) cudaFreeHost(cnt_host);
  cnt_host = nullptr;
  cnt_host_n = 0;
  if (step_host_p) cudaFreeHost(step_host_p);
  step_host_p = nullptr;
  step_host.clear();
  for (auto& e : pev)
    if (e) {
      cudaEventDestroy(e);
      e = nullptr;
    }
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  ev0 = ev1 = nullptr;
  if (fence_ev) cudaEventDestroy(fence_ev);
  fence_ev = nullptr;
}

void StepRunner::release_device() {
  Buf* all[] = {&seg_d, &seg_n, &blk_rel, &seg_tuples, &hdr, &poolA_m, &poolA_t, &poolA_id, &poolA_start,
                &poolA_cnt, &poolB_m, &poolB_t, &poolB_id, &poolB_start, &poolB_cnt, &cursors,
                &nb, &bucket_base, &wcnt, &wo, &bcount, &bmin, &boff, &bcarry, &cm, &ct, &cid,
                &cgb, &gm, &gt, &gid, &gflag, &large_list, &scan_tmp, &ncand,
                &dst_off, &steps_dev, &base_dev, &pos, &step_arr, &groups_dev, &packs_dev, &big_dev, &whint};
  for (Buf* b : all) {
    if (b->p) alloc.put(b->p, nullptr, true);
    b->p = nullptr;
    b->hw = std::max(b->hw, b->bytes);
    b->bytes = 0;
  }
}

static int grid_for(int64_t n, int nt, int maxg) {
  int64_t g = (n + nt - 1) / nt;
  if (g < 1) g = 1;
  if (g > maxg) g = maxg;
  return (int)g;
}

cudaError_t StepRunner::run(const std::vector<StepDev>& steps, cudaStream_t st, StepResult* res,
                            int64_t* dev_off, const std::vector<NodeGroupH>* groups, bool keep_dev) {
  int64_t nl = 0;  // kernel launches
  int pgroup[64];
  if (fence_ev && fence_st != st) cudaStreamWaitEvent(st, fence_ev, 0);  // scratch last used on another stream
  npev = 0;
  auto mark = [&](int group) {  // group of the interval that starts here
    if (!profile || npev >= 64) return;
    if (!pev[npev]) cudaEventCreate(&pev[npev]);
    cudaEventRecord(pev[npev], st);
    pgroup[npev] = group;
    ++npev;
  };
  // batch layout: local segments / blocks numbered consecutively over steps
  const int nsteps = (int)steps.size();
  h_base.assign(2 * (nsteps + 1), 0);
  for (int j = 0; j < nsteps; ++j) {
    const int64_t ns = steps[j].seg_hi - steps[j].seg_lo;
    h_base[j + 1] = h_base[j] + ns;
    h_base[nsteps + 1 + j + 1] = h_base[nsteps + 1 + j] + ns * steps[j].nblk;
  }
  const int64_t nloc = h_base[nsteps];
  const int64_t nbl = h_base[2 * nsteps + 1];
  cudaError_t e;
  if (!ev0) {
    if ((e = cudaEventCreate(&ev0)) != cudaSuccess) return e;
    if ((e = cudaEventCreate(&ev1)) != cudaSuccess) return e;
  }
  if (!hdr_host) {
    if ((e = cudaMallocHost((void**)&hdr_host, sizeof(StepHdr))) != cudaSuccess) return e;
  }
  res->nloc = nloc;
  res->retries = 0;
  if (nloc == 0) {
    res->total = 0;
    res->levels = 0;
    res->tuples = 0;
    res->candidates = 0;
    res->kernel_ms = 0;
    return cudaSuccess;
  }
  GROW(steps_dev, StepDev, nsteps);
  GROW(base_dev, int64_t, 2 * (nsteps + 1));
  cudaMemcpyAsync(steps_dev.p, steps.data(), sizeof(StepDev) * nsteps, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(base_dev.p, h_base.data(), sizeof(int64_t) * 2 * (nsteps + 1),
                  cudaMemcpyHostToDevice, st);
  BatchDev s;
  s.steps = (const StepDev*)steps_dev.p;
  s.seg_base = (const int64_t*)base_dev.p;
  s.blk_base = (const int64_t*)base_dev.p + nsteps + 1;
  s.nsteps = nsteps;
  s.slog = slog;
  s.slog0 = slog0;
  {  // test hook: FT_KEY_SPAN_BITS < 53 forces the full-key sorts (read per wave)
    const char* ks = getenv("FT_KEY_SPAN_BITS");
    s.kspan = ks ? std::max(0, std::min(53, atoi(ks))) : 53;
  }
  // waves of few segments (LDP: one per configuration) take a larger direct
  // capacity: one filter level fewer per segment, and few CTAs sort in smem
  // (A/B: a global 2048 helped C5's LDP waves but slowed C4's 6e4-segment
  // node waves, 52 -> 58 ms)
  const int cd = nloc <= small_wave_segs ? std::min(C_DIRECT, cdirect_small) : cdirect;
  s.cdirect = cd;
  s.nseg = nloc;
  s.nblk = nbl;
  batch = s;
  GROW(seg_d, int32_t, nloc);
  GROW(seg_n, int32_t, nloc);
  const int ngroups = groups ? (int)groups->size() : 0;
  // k_node_pack: consecutive full rows w of one step, up to NP_NT/ceil32(K_j) per pack
  std::vector<NodeGroup> packs;
  int np_rmax = 1;
  int64_t np_ztn = 0;
  if (ngroups) {
    for (int gi = 0; gi < ngroups; ++gi) {
      const NodeGroup& G = (*groups)[gi];
      const StepDev& d = steps[G.step];
      const int64_t np = G.p_hi - G.p_lo;
      const int tpr = np_tpr(np);
      const int64_t zt = d.nblk * (int64_t)tpr;
      if (np <= NP_NT && zt <= NP_ZT_CAP) np_ztn = std::max(np_ztn, zt);
      const int rcap = np <= NP_NT ? std::min(NP_ROWS, NP_NT / tpr) : 1;
      if (!packs.empty()) {
        NodeGroup& P = packs.back();
        if (P.step == G.step && P.p_lo == G.p_lo && P.p_hi == G.p_hi && G.p_lo == 0 && G.p_hi == d.KC &&
            G.w == P.w + P.pad && G.gs0 == P.gs0 + P.pad * np && P.pad < rcap) {
          ++P.pad;
          np_rmax = std::max(np_rmax, P.pad);
          continue;
        }
      }
      NodeGroup P = G;
      P.pad = 1;
      packs.push_back(P);
    }
    GROW(groups_dev, NodeGroup, ngroups);  // rows handed to k_node_shared
    GROW(packs_dev, NodeGroup, packs.size());
    cudaMemcpyAsync(packs_dev.p, packs.data(), sizeof(NodeGroup) * packs.size(), cudaMemcpyHostToDevice, st);
  }
  GROW(blk_rel, int64_t, nbl);
  GROW(seg_tuples, int64_t, nloc);
  GROW(hdr, StepHdr, 1);
  StepHdr* H = (StepHdr*)hdr.p;
  cudaEventRecord(ev0, st);
  mark(0);
  cudaMemsetAsync(H, 0, sizeof(StepHdr), st);
  ++nl;
  launch(k_plan, dim3(grid_for(nloc * 32, 256, 148 * 8)), dim3(256), 0, st, s, (int32_t*)seg_d.p, (int32_t*)seg_n.p,
                                                            (int64_t*)blk_rel.p,
                                                            (int64_t*)seg_tuples.p, H);
  cudaMemcpyAsync(hdr_host, H, sizeof(StepHdr), cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  mark(5);  // host: readback + scratch sizing
  if (hdr_host->bad) return cudaErrorInvalidConfiguration;
  const int D = (int)hdr_host->D;
  res->levels = D + 1;
  res->tuples = (int64_t)hdr_host->tuples;
  int64_t need_filter = 0, need_out = 0;
  for (int l = 0; l <= D; ++l) need_filter = std::max<int64_t>(need_filter, hdr_host->filter_samp[l]);
  unsigned long long plan_copy[2 * (LMAX + 1)];
  for (int l = 0; l <= LMAX; ++l) {
    plan_copy[l] = hdr_host->direct_samp[l];
    plan_copy[LMAX + 1 + l] = hdr_host->filter_samp[l];
  }
  // warp-start hints of the filter items (k_hints): W <= the level's sample
  // (an item holds >= 1 sampled element), capped at 4 M entries (16 MB);
  // warps beyond it search
  const int64_t hcap = nbl < ((int64_t)1 << 31) ? std::min<int64_t>(need_filter / 32 + 2, 1 << 22) : 0;
  for (int attempt = 0;; ++attempt) {
    const int64_t cand_cap = std::min<int64_t>(need_filter, cand_budget);
    need_out = 0;
    for (int l = 0; l <= D; ++l)
      need_out = std::max<int64_t>(need_out, (int64_t)plan_copy[l] +
                                                 std::min<int64_t>(plan_copy[LMAX + 1 + l], cand_cap));
    need_out = std::max<int64_t>(need_out, out_budget);
    const int64_t bcap = std::max<int64_t>(need_out + nloc + 1, bucket_budget);
    GROW(poolA_m, int64_t, need_out);
    GROW(poolA_t, int64_t, need_out);
    GROW(poolA_id, uint64_t, need_out);
    GROW(poolB_m, int64_t, need_out);
    GROW(poolB_t, int64_t, need_out);
    GROW(poolB_id, uint64_t, need_out);
    GROW(poolA_start, int64_t, nloc);
    GROW(poolA_cnt, int64_t, nloc);
    GROW(poolB_start, int64_t, nloc);
    GROW(poolB_cnt, int64_t, nloc);
    // [0..8): cand / large cursors (k_compact resets them per level); [8 + l]:
    // the output cursor of level l (no memset between a wave's kernels: PDL)
    GROW(cursors, unsigned long long, 8 + LMAX + 1);
    cudaMemsetAsync(cursors.p, 0, sizeof(unsigned long long) * (8 + LMAX + 1), st);
    if (D > 0) {
      GROW(nb, int64_t, nloc);
      GROW(bucket_base, int64_t, nloc + 1);
      GROW(wcnt, int64_t, std::max<int64_t>(nbl, 1));
      GROW(wo, int64_t, nbl + 1);
      {  // bucket counters / minima live in their reset state between levels
         // (k_carry_scatter hands every count back to 0 and every minimum to
         // INF); fresh or retried scratch is reset here
        const size_t ob = bcount.bytes, om = bmin.bytes;
        GROW(bcount, unsigned int, bcap);
        GROW(bmin, long long, bcap);
        if (bcount.bytes != ob || attempt > 0) cudaMemsetAsync(bcount.p, 0, bcount.bytes, st);
        if (bmin.bytes != om || attempt > 0) cudaMemsetAsync(bmin.p, BMIN_FILL, bmin.bytes, st);
      }
      GROW(boff, int64_t, bcap + 1);
      GROW(bcarry, long long, bcap);
      GROW(cm, int64_t, cand_cap);
      GROW(ct, int64_t, cand_cap);
      GROW(cid, uint64_t, cand_cap);
      GROW(cgb, int64_t, cand_cap + 1);
      GROW(gm, int64_t, cand_cap);
      GROW(gt, int64_t, cand_cap);
      GROW(gid, uint64_t, cand_cap);
      GROW(gflag, uint8_t, cand_cap + 1);
      GROW(large_list, int64_t, bcap);
      GROW(whint, int32_t, 2 * hcap);  // blocks, then their steps
      GROW(ncand, int64_t, 2);
    }
    // scan scratch: the largest single scan, or the bucket-count + work-item pair
    const int64_t scan_n = std::max<int64_t>({nloc + nbl + 2 * SCAN_TILE, bcap + 1, cand_cap + 1});
    {  // scan scratch: zeroed when (re)allocated -- compare the capacity, not the
       // address (a larger allocation can come back at the same address); scans
       // leave it zeroed
      const size_t old_bytes = scan_tmp.bytes;
      GROW(scan_tmp, int64_t, scan_n / SCAN_TILE + 8);
      if (scan_tmp.bytes != old_bytes) cudaMemsetAsync(scan_tmp.p, 0, scan_tmp.bytes, st);
    }
    unsigned long long* cur = (unsigned long long*)cursors.p;
    if (attempt > 0) {
      cudaMemsetAsync(H, 0, sizeof(StepHdr), st);
      launch(k_plan, dim3(grid_for(nloc * 32, 256, 148 * 8)), dim3(256), 0, st, s, (int32_t*)seg_d.p, (int32_t*)seg_n.p,
                                                                (int64_t*)blk_rel.p,
                                                                (int64_t*)seg_tuples.p, H);
    }
    Pool pools[2];
    pools[0] = Pool{(int64_t*)poolA_m.p, (int64_t*)poolA_t.p, (uint64_t*)poolA_id.p,
                    (int64_t*)poolA_start.p, (int64_t*)poolA_cnt.p, cur + 0, need_out};
    pools[1] = Pool{(int64_t*)poolB_m.p, (int64_t*)poolB_t.p, (uint64_t*)poolB_id.p,
                    (int64_t*)poolB_start.p, (int64_t*)poolB_cnt.p, cur + 1, need_out};
    for (int l = D; l >= 0; --l) {
      LevelDev L;
      std::memset(&L, 0, sizeof(L));
      L.level = l;
      L.st = level_shift(l, slog0, slog);
      L.warp2 = WARP_DIRECT;
      L.fstats = fstats;
      {  // ~item_div work items per resident thread (148 SMs x 2048 threads)
        const int64_t tot = (int64_t)plan_copy[LMAX + 1 + l];
        int64_t ri = tot / (int64_t)(148 * 2048) / item_div;
        ri = std::max<int64_t>(CHUNK, std::min<int64_t>(item_max, ri));
        L.run_item = (int)((ri + CHUNK - 1) / CHUNK * CHUNK);
      }
      L.seg_d = (const int32_t*)seg_d.p;
      L.seg_n = (const int32_t*)seg_n.p;
      L.blk_rel = (const int64_t*)blk_rel.p;
      L.in = pools[(l + 1) & 1];
      L.out = pools[l & 1];
      L.hdr = H;
      L.out.cursor = cur + 8 + l;
      mark(1);
      nl += 2;
      if (l == 0 && ngroups) {
        ++nl;
        ++nl;
        const int npk = (int)packs.size();
        launch(k_node_pack, dim3(std::min(npk, pack_grid)), dim3(NP_NT), np_smem(np_rmax, np_ztn), st, 
            s, L, (const NodeGroup*)packs_dev.p, npk, np_rmax, np_ztn, (NodeGroup*)groups_dev.p);
        launch(k_node_shared, dim3(std::min(ngroups, 148 * 2)), dim3(DIRECT_NT), NS_SMEM, st, 
            s, L, (const NodeGroup*)groups_dev.p);
      }
      launch(k_direct_warp, dim3(grid_for(nloc, 8, 148 * 8)), dim3(256), DW_SMEM, st, s, L);
      launch(k_direct, dim3(grid_for(nloc, 1, 148 * 8)), dim3(DIRECT_NT), direct_smem(cd), st, s, L);
      if (l < D) {
        L.nb = (int64_t*)nb.p;
        L.bucket_base = (int64_t*)bucket_base.p;
        L.wcnt = (int64_t*)wcnt.p;
        L.wo = (int64_t*)wo.p;
        L.bcount = (unsigned int*)bcount.p;
        L.bmin = (long long*)bmin.p;
        L.boff = (int64_t*)boff.p;
        L.bcarry = (long long*)bcarry.p;
        L.bcap = bcap;
        L.cm = (int64_t*)cm.p;
        L.ct = (int64_t*)ct.p;
        L.cid = (uint64_t*)cid.p;
        L.cgb = (int64_t*)cgb.p;
        L.cand_cursor = cur + 2;
        L.cand_cap = cand_cap;
        L.gm = (int64_t*)gm.p;
        L.gt = (int64_t*)gt.p;
        L.gid = (uint64_t*)gid.p;
        L.gflag = (uint8_t*)gflag.p;
        L.large_list = (int64_t*)large_list.p;
        L.large_n = cur + 3;
        L.whint = (int32_t*)whint.p;
        L.hcap = hcap;
        int64_t* nc = (int64_t*)ncand.p;
        int64_t* tmp = (int64_t*)scan_tmp.p;
        mark(4);  // scans (bucket bases, work offsets) count as scan/compaction time
        nl += 3;  // block work counts, scan(+nb) and work-offset scan in one launch, filter
        launch(k_blocks, dim3(grid_for(nbl, 256, 148 * 8)), dim3(256), 0, st, s, L);
        scan2_excl_fn(LoadNb{L}, nloc, L.bucket_base, LoadArr<int64_t>{L.wcnt}, nbl, L.wo, tmp, st, NoPost());
        ++nl;
        launch(k_hints, dim3(148 * 4), dim3(256), 0, st, s, L);
        mark(2);  // filter_ms: k_filter alone
        if (filter_regs64) launch(k_filter64, dim3(filter_grid), dim3(128), 0, st, s, L);
        else launch(k_filter, dim3(filter_grid), dim3(128), 0, st, s, L);
        // bucket offsets over B buckets (B on device)
        mark(3);
        nl += 4;  // scan, carry+scatter, 2 bucket sorts (huge buckets inside k_bucket_large)
        scan_excl<unsigned int>(L.bcount, L.boff, L.bucket_base + nloc, bcap, tmp, st);
        launch(k_carry_scatter, dim3(148 * 8), dim3(256), 0, st, s, L, nc);  // + candidate total
        launch(k_bucket_small, dim3(148 * 8), dim3(256), 0, st, s, L);
        const size_t lsm = (size_t)BUCKET_SMEM * (3 * sizeof(int64_t) + sizeof(int));
        launch(k_bucket_large, dim3(148 * 2), dim3(DIRECT_NT), lsm, st, L);
        // positions of survivors: scan flags in place into gpos (reuse cgb as gpos)
        mark(4);
        nl += 2;  // scan, compact (+ segment ranges)
        int64_t* gpos = (int64_t*)cgb.p;  // candidate gb is dead after scatter
        scan_excl<uint8_t>(L.gflag, gpos, nc, cand_cap, tmp, st);
        const int64_t cbase = (int64_t)plan_copy[l];  // direct outputs of level l stay below
        launch(k_compact, dim3(148 * 8), dim3(256), 0, st, s, L, gpos, nc, cbase);
      }
    }
    mark(-1);
    cudaEventRecord(ev1, st);
    // read back header + level-0 per-segment counts
    if (cnt_host_n < nloc) {
      if (cnt_host) cudaFreeHost(cnt_host);
      if ((e = cudaMallocHost((void**)&cnt_host, sizeof(int64_t) * 2 * nloc)) != cudaSuccess) return e;
      cnt_host_n = nloc;
    }
    if (dev_off) {  // offsets on the device; only per-step totals come back
      GROW(pos, int64_t, nloc + 1);
      GROW(step_arr, int64_t, 3 * nsteps);
      if ((int64_t)step_host.size() < 3 * nsteps) {
        if (step_host_p) cudaFreeHost(step_host_p);
        if ((e = cudaMallocHost((void**)&step_host_p, sizeof(int64_t) * 3 * nsteps)) != cudaSuccess) return e;
        step_host.assign(3 * nsteps, 0);
      }
      scan_excl<int64_t>(pools[0].cnt, (int64_t*)pos.p, nullptr, nloc, (int64_t*)scan_tmp.p, st);
      cudaMemsetAsync(step_arr.p, 0, sizeof(int64_t) * 3 * nsteps, st);
      launch(k_wave_off, dim3(grid_for(nloc, 256, 1 << 30)), dim3(256), 0, st, s, pools[0].cnt, (int64_t*)seg_tuples.p,
                                                               (int64_t*)pos.p, dev_off,
                                                               (int64_t*)step_arr.p);
      nl += 2;  // scan, wave_off
      cudaMemcpyAsync(hdr_host, H, sizeof(StepHdr), cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(step_host_p, step_arr.p, sizeof(int64_t) * 3 * nsteps, cudaMemcpyDeviceToHost, st);
    } else if (keep_dev) {  // multi-rank device exchange: counts stay on the device
      cudaMemcpyAsync(hdr_host, H, sizeof(StepHdr), cudaMemcpyDeviceToHost, st);
    } else {
      cudaMemcpyAsync(hdr_host, H, sizeof(StepHdr), cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(cnt_host, pools[0].cnt, sizeof(int64_t) * nloc, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(cnt_host + nloc, seg_tuples.p, sizeof(int64_t) * nloc, cudaMemcpyDeviceToHost, st);
    }
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (!hdr_host->overflow) {
      res->pool = pools[0];
      res->candidates = 0;
      for (int l = 0; l < D; ++l) res->candidates += (int64_t)hdr_host->cand_total[l];
      if (fstats) {
        for (int q = 0; q < 10; ++q) {
          bstat_acc[0][q] += hdr_host->bstat[0][q];
          bstat_acc[1][q] += hdr_host->bstat[1][q];
        }
        bfall_acc[0] += hdr_host->bfall[0];
        bfall_acc[1] += hdr_host->bfall[1];
        for (int q = 0; q < 8; ++q) fstat_acc[q] += hdr_host->fstat[q];
      }
      res->filter_tuples = res->direct_tuples = 0;
      for (int l = 0; l <= D; ++l) {
        res->filter_tuples += (int64_t)plan_copy[LMAX + 1 + l];
        res->direct_tuples += (int64_t)plan_copy[l];
      }
      res->huge = (int64_t)hdr_host->huge;
      res->path[0] = (int64_t)hdr_host->ns_rows;
      res->path[1] = (int64_t)hdr_host->ns_tie;
      res->path[2] = (int64_t)hdr_host->ns_big;
      res->path[3] = (int64_t)hdr_host->dreg;
      int64_t tot = 0;
      if (dev_off) {
        res->counts = nullptr;
        res->seg_tuples = nullptr;
        res->step_stats = step_host_p;
        for (int q = 0; q < nsteps; ++q) tot += step_host_p[3 * q];
      } else if (keep_dev) {
        res->counts = nullptr;
        res->seg_tuples = nullptr;
        res->step_stats = nullptr;
        res->dev_cnt = pools[0].cnt;
        res->dev_tup = (const int64_t*)seg_tuples.p;
      } else {
        res->counts = cnt_host;
        res->seg_tuples = cnt_host + nloc;
        res->step_stats = nullptr;
        for (int64_t i = 0; i < nloc; ++i) tot += cnt_host[i];
      }
      res->total = tot;
      float ms = 0;
      cudaEventElapsedTime(&ms, ev0, ev1);
      res->kernel_ms = ms;
      res->launches = nl;
      res->plan_ms = res->direct_ms = res->filter_ms = res->bucket_ms = res->compact_ms = 0;
      res->host_ms = 0;
      for (int q = 0; q + 1 < npev; ++q) {
        float d = 0;
        cudaEventElapsedTime(&d, pev[q], pev[q + 1]);
        float* dst[6] = {&res->plan_ms, &res->direct_ms, &res->filter_ms, &res->bucket_ms,
                         &res->compact_ms, &res->host_ms};
        if (pgroup[q] >= 0 && pgroup[q] < 6) *dst[pgroup[q]] += d;
      }
      return cudaSuccess;
    }
    // grow budgets and retry
    res->retries++;
    int64_t mc = 0, mo = 0, mb = 0;
    for (int l = 0; l <= D; ++l) {
      mc = std::max<int64_t>(mc, hdr_host->cand_total[l]);
      mo = std::max<int64_t>(mo, hdr_host->out_total[l]);
      mb = std::max<int64_t>(mb, hdr_host->bucket_total[l]);
    }
    cand_budget = std::max<int64_t>(cand_budget * 2, mc + mc / 4);
    out_budget = std::max<int64_t>(out_budget * 2, mo + mo / 4);
    bucket_budget = std::max<int64_t>(bucket_budget * 2, mb + mb / 4);
    if (attempt > 16) return cudaErrorMemoryAllocation;
  }
}

cudaError_t StepRunner::gather(const std::vector<StepDev>& steps, const StepResult& r,
                               cudaStream_t st) {
  if (r.nloc == 0) return cudaSuccess;
  if (r.step_stats) {  // device-offset mode: arena is contiguous in pos order
    launch(k_gather_flat, dim3(grid_for(r.total, 2048, 148 * 16)), dim3(256), 0, st, 
        batch, r.pool, (const int64_t*)pos.p, steps[0].out_m, steps[0].out_t, steps[0].out_bp);
    return cudaGetLastError();
  }
  // the output pointers changed: refresh the step array (same batch layout)
  cudaMemcpyAsync(steps_dev.p, steps.data(), sizeof(StepDev) * steps.size(), cudaMemcpyHostToDevice,
                  st);
  launch(k_gather, dim3(grid_for(r.nloc, 8, 148 * 16)), dim3(256), 0, st, batch, r.pool);
  return cudaGetLastError();
}

cudaError_t StepRunner::configure() {
  fstats = getenv("FT_FILTER_STATS") != nullptr;
  if (const char* e = getenv("FT_PDL")) g_pdl = atoi(e) != 0;
  if (const char* e = getenv("FT_BLOCK_SKIP")) {
    const bool v = atoi(e) != 0;
    cudaMemcpyToSymbol(g_bskip, &v, sizeof(v));
  }
  if (const char* e = getenv("FT_FENCE")) {
    const bool v = atoi(e) != 0;
    cudaMemcpyToSymbol(g_fence, &v, sizeof(v));
  }
  if (const char* e = getenv("FT_PACK_GRID")) pack_grid = std::max(1, atoi(e));  // tests: packs per CTA
  filter_regs64 = getenv("FT_FILTER_REGS") && atoi(getenv("FT_FILTER_REGS")) == 64;
  filter_grid = 148 * 128;  // A/B after the block pre-filter (C5 / C4 ms, items <= 256): 148x256 47.8 / 36.2, 148x128 46.0 / 34.4, 148x64 46.4 / 34.8
  if (const char* e = getenv("FT_FILTER_GRID")) filter_grid = std::max(148, atoi(e));
  if (const char* e = getenv("FT_ITEM_MAX")) item_max = std::max(16, atoi(e));
  if (const char* e = getenv("FT_ITEM_DIV")) item_div = std::max(1, atoi(e));
  {
    cudaError_t e0 = cudaFuncSetAttribute(k_node_shared, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)NS_SMEM);
    if (e0 != cudaSuccess) return e0;
    e0 = cudaFuncSetAttribute(k_node_pack, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)np_smem(NP_ROWS, NP_ZT_CAP));
    if (e0 != cudaSuccess) return e0;
    e0 = cudaFuncSetAttribute(k_direct_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DW_SMEM);
    if (e0 != cudaSuccess) return e0;
  }
  if (const char* e = getenv("FT_SLOG")) slog = std::max(1, std::min(6, atoi(e)));
  if (const char* e = getenv("FT_SLOG0")) slog0 = std::max(1, std::min(6, atoi(e)));
  // direct capacities are powers of two: a sample of n tuples is sorted as
  // the next power of two N >= n, which must fit the capacity
  auto pow2_floor = [](int v) {
    int p = 256;
    while (p * 2 <= v) p *= 2;
    return p;
  };
  if (const char* e = getenv("FT_CDIRECT")) cdirect = pow2_floor(std::min(C_DIRECT, atoi(e)));
  if (const char* e = getenv("FT_SMALL_WAVE")) small_wave_segs = std::max(0, atoi(e));
  if (const char* e = getenv("FT_CDIRECT_SMALL")) cdirect_small = pow2_floor(std::min(C_DIRECT, atoi(e)));
  {
    cudaError_t e0 = cudaFuncSetAttribute(k_direct, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)direct_smem(C_DIRECT));
    if (e0 != cudaSuccess) return e0;
  }
  const size_t lsm = (size_t)BUCKET_SMEM * (3 * sizeof(int64_t) + sizeof(int));
  cudaError_t e = cudaFuncSetAttribute(k_bucket_large, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)lsm);
  if (e != cudaSuccess) return e;
  return cudaSuccess;
}

}  // namespace ftk
