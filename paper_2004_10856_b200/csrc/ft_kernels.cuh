// ft_kernels.cuh -- sm_100a kernels of the FT hot path (arXiv 2004.10856).
//
// One FT step (node elimination Eq.4, edge elimination Eq.5
// P:599-603, K=1 fold Eq.7, LDP step Alg.3 line 6 P:645, final
// reduce Alg.3 line 9 P:648) computes, for every output segment sigma,
//
//     F_sigma = reduce( U_k  X_k (x) Y_k (x) Z_k )                    (R5)
//
// with Product (x), Union U and Reduce = Alg.1
// under the key (m, t, id) (R1, R3, R6).  DESIGN.md "pipeline" explains the
// exact sampled-staircase pre-filter used here; in short, per segment:
//
//   level D (coarsest sample, <= C_DIRECT tuples): direct CTA sort+scan.
//   level l < D: G = frontier of the level-(l+1) sample (real tuples);
//     K1 product kernel expands the level-l sample run by run, drops every
//     tuple strictly dominated by G (a chunk at a time when possible) and
//     bins survivors by G interval ("bucket");  K2 sorts each bucket by
//     (m,t,id);  K3 applies Alg.1's running minimum with the bucket's carry
//     (exclusive prefix-min over earlier buckets);  K4 compacts.
//   Because G consists of real tuples of the segment, a tuple strictly
//   dominated by G is beaten in Alg.1 and reduce(candidates) = reduce(all).
//
// No tensor cores: the path is integer compare/add work.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ftk {

constexpr int64_t INF = INT64_MAX;
constexpr int LMAX = 12;            // max sample level
constexpr int C_DIRECT = 4096;      // max direct (single-CTA) segment capacity (dynamic smem)
constexpr int WARP_DIRECT = 256;    // direct segments up to this size: one warp each (R <= 8)
constexpr int NS_CAP = 2048;        // shared-order node path: tuples per (step, w) group
constexpr int NS_MAXBLK = 128;      // ... and blocks (K_i)
constexpr int SPECIAL_LEVEL = 60;   // seg_d of segments handled by the shared-order node path
constexpr int DIRECT_NT = 256;      // threads of the direct / bucket CTA kernels
constexpr int CHUNK = 16;           // run elements per filter work item
constexpr int BUCKET_SMEM = 4096;   // largest bucket sorted in shared memory
constexpr int BMIN_FILL = 0x7F;     // memset byte: 0x7F7F..7F > any t (< 2^60)

// Programmatic dependent launch (PDL): the pipeline's kernels are launched
// with programmatic stream serialisation, so a kernel's CTAs are dispatched
// while its predecessor still runs.  Every such kernel opens with this: wait
// until the predecessor grid has completed and its writes are visible (before
// ANY global access -- reads of its outputs and writes of its inputs alike),
// then let the successor launch.  Without the launch attribute both are no-ops.
#define FT_PDL_ENTRY()                                          \
  do {                                                          \
    asm volatile("griddepcontrol.wait;" ::: "memory");          \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
  } while (0)

enum { K_NODE = 1, K_EDGE = 2, K_FOLD = 3, K_LDP = 4, K_FINAL = 5, K_PAIR = 6, K_BRANCH = 7, K_COMPOSE = 8,
       K_REMAP = 9 };

// A frontier set on the device (CSR): segment s = [off[s], off[s+1]).
struct FacSet {
  const int64_t* off;
  const int64_t* m;
  const int64_t* t;
};

// One FT step of a batch ("wave" of independent steps).
struct StepDev {
  int kind;
  int node_shared;  // NODE step with singleton F(o_i,k) and original m=0 edge F(e_ij,k,p)
  int64_t KA, KB, KC, nseg, nblk;
  int64_t seg_lo, seg_hi;  // this rank's output segments [seg_lo, seg_hi)
  FacSet X, Y, Z;
  // gather destination (set after the survivor counts are known)
  int64_t* out_m;
  int64_t* out_t;
  uint64_t* out_bp;
  const int64_t* out_off;  // [seg_hi - seg_lo] offsets of this rank's segments in the output
};

// A batch of steps; local segments / blocks are numbered consecutively over
// the steps: step j owns segments [seg_base[j], seg_base[j+1]) and blocks
// [blk_base[j], blk_base[j+1]) (blocks of a segment are contiguous).
struct BatchDev {
  const StepDev* steps;
  const int64_t* seg_base;  // [nsteps+1]
  const int64_t* blk_base;  // [nsteps+1]
  int nsteps;
  int slog;                 // sample stride at level l >= 1: 2^(slog0 + slog*(l-1))
  int slog0;
  int cdirect;              // direct-path capacity (<= C_DIRECT)
  int kspan;                // single-key sorts pack (m - m_min) when it fits in kspan bits
  int64_t nseg;             // local segments over all steps
  int64_t nblk;             // local blocks over all steps
};

// Step header written by the plan kernel, read back by the host.
struct StepHdr {
  unsigned long long D;                       // max level over segments (atomicMax)
  unsigned long long tuples;                  // product tuples of this rank's segments
  unsigned long long direct_samp[LMAX + 1];   // sum of sample sizes of DIRECT segments at l
  unsigned long long filter_samp[LMAX + 1];   // sum of sample sizes of FILTER segments at l
  unsigned long long overflow;                // != 0: some capacity was exceeded
  unsigned long long bad;                     // != 0: unsupported shape (nblk > C_DIRECT)
  unsigned long long cand_total[LMAX + 1];    // candidates emitted per level (may exceed cap)
  unsigned long long out_total[LMAX + 1];     // level outputs
  unsigned long long bucket_total[LMAX + 1];  // buckets per level
  unsigned long long huge;                    // buckets sorted by the global-memory path
  unsigned long long bstat[2][10];            // bucket count / candidates by size class (stats)
  unsigned long long bfall[2];                // key-sorted bucket sorts redone on (m, t, id): lane groups, warps (stats)
  unsigned long long fstat[8];                // filter work counters (FT_FILTER_STATS): work
                                              // items, chunk tests, skipped chunks' elements,
                                              // elements tested one by one; G points over items,
                                              // warp passes with all 32 items in one block, warp
                                              // passes, chunk tests past the 4-point G probe
  unsigned long long ns_big;                  // rows handed from k_node_pack to k_node_shared
  unsigned long long ns_rows;                 // rows reduced by k_node_pack
  unsigned long long ns_tie;                  // ... of which with equal m values (group rule)
  unsigned long long dreg;                    // k_direct segments sorted register-blocked
};

// Per-level pool of per-segment results (G of the next finer level, or the
// step output at level 0).
struct Pool {
  int64_t* m;
  int64_t* t;
  uint64_t* id;
  int64_t* start;                 // [nseg]
  int64_t* cnt;                   // [nseg]
  unsigned long long* cursor;
  int64_t cap;
};

struct LevelDev {
  int level;
  int st;      // log2 of the sample stride
  int run_item;  // filter work-item length (sampled run elements)
  int warp2;     // largest direct segment handled by the warp kernels
  int fstats;    // collect filter work counters
  const int32_t* seg_d;
  const int32_t* seg_n;  // sample size at the direct level
  const int64_t* blk_rel;
  Pool in;     // level l+1 output (G), valid when level < D
  Pool out;
  // filter / bucket scratch
  int64_t* nb;           // [nseg]  buckets per segment (g+1 for FILTER)
  int64_t* bucket_base;  // [nseg+1]
  int64_t* wcnt;         // [nblocks]
  int64_t* wo;           // [nblocks+1]
  unsigned int* bcount;  // [bcap]
  long long* bmin;       // [bcap]
  int64_t* boff;         // [bcap+1]
  long long* bcarry;     // [bcap]
  int64_t bcap;
  int64_t* cm;
  int64_t* ct;
  uint64_t* cid;
  int64_t* cgb;
  unsigned long long* cand_cursor;
  int64_t cand_cap;
  int64_t* gm;           // grouped (bucket-ordered) candidates
  int64_t* gt;
  uint64_t* gid;
  uint8_t* gflag;        // keep flags (0/1), scanned -> positions
  int64_t* large_list;
  unsigned long long* large_n;
  int32_t* whint;        // [2 hcap] block of filter item 32c (k_filter warp starts), then its step
  int64_t hcap;
  int64_t* scratch;      // global-memory sort scratch (huge buckets)
  int64_t scratch_cap;
  StepHdr* hdr;
};

// ---------------------------------------------------------------------------
// helpers

// Largest j in [0, n) with base[j] <= x (base ascending, base[0] = 0).
__device__ __forceinline__ int find_base(const int64_t* base, int n, int64_t x) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (__ldg(base + mid) <= x) lo = mid;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ bool key_lt(int64_t am, int64_t at, uint64_t ai, int64_t bm, int64_t bt,
                                       uint64_t bi) {
  if (am != bm) return am < bm;
  if (at != bt) return at < bt;
  return ai < bi;
}

// Factor segments of block k of output segment sigma (Eq.4, Eq.5, Eq.7, Alg.3).
__device__ __forceinline__ void block_factor_segs(const StepDev& s, int64_t sg, int64_t k,
                                                  int64_t& sx, int64_t& sy, int64_t& sz) {
  if (s.kind == K_NODE) {          // sigma = w*K_j + p ; X=F(e_hi,w,k) Y=F(o_i,k) Z=F(e_ij,k,p)
    int64_t w, p;
    if ((sg >> 31) == 0 && (s.KC >> 31) == 0) {  // 32-bit division fast path
      const unsigned q = (unsigned)sg / (unsigned)s.KC;
      w = q;
      p = sg - (int64_t)q * s.KC;
    } else {
      w = sg / s.KC;
      p = sg - w * s.KC;
    }
    sx = w * s.KB + k;
    sy = k;
    sz = k * s.KC + p;
  } else if (s.kind == K_LDP) {    // sigma = p ; X=F(e,k,p) Y=CF(o_{i-1},k) Z=F(o_i,p)
    sx = k * s.KB + sg;
    sy = k;
    sz = sg;
  } else if (s.kind == K_FINAL) {  // X = CF(o_n, k)
    sx = k;
    sy = 0;
    sz = 0;
  } else if (s.kind == K_BRANCH) { // Eq. 6 (R14): sigma = s_h, k = s_i; KC = o_i is the edge's source
    sx = sg;                         // F(o_h, s_h)
    sy = s.KC ? k * s.KA + sg : sg * s.KB + k;  // F(e, s_i, s_h) | F(e, s_h, s_i)
    sz = k;                          // F(o_i, s_i)
  } else if (s.kind == K_PAIR) {   // FT-Elimination: k = s_1*K_n + s_n
    const int64_t s1 = (k >> 31) == 0 && (s.KB >> 31) == 0 ? (int64_t)((unsigned)k / (unsigned)s.KB) : k / s.KB;
    sx = k;                          // F(e_1n, s_1, s_n)
    sy = s1;                         // F(o_1, s_1)
    sz = k - s1 * s.KB;              // F(o_n, s_n)
  } else if (s.kind == K_COMPOSE) {  // Eq. 6 composite (R21): sigma = w = s_h*K_i + s_i, one block
    const int64_t p = sg / s.KB, q = sg - p * s.KB;  // KA = K_h, KB = K_i
    sx = p;                          // F(o_h, s_h)
    sy = q * s.KA + p;               // F(e_ih, s_i, s_h)
    sz = q;                          // F(o_i, s_i)
  } else if (s.kind == K_REMAP) {  // R21: an edge of o_h / o_i re-indexed onto the composite o_v
    // KA = K_y (other endpoint), KB = K_i, KC = side | part << 1 (side 0: o_v is
    // the source; part 0: the old endpoint was o_h -> w / K_i, 1: o_i -> w % K_i)
    const int64_t Kv = s.nseg / s.KA, side = s.KC & 1, part = s.KC >> 1;
    const int64_t Kold = part ? s.KB : Kv / s.KB;
    const int64_t w = side == 0 ? sg / s.KA : sg % Kv, y = side == 0 ? sg % s.KA : sg / Kv;
    const int64_t c = part ? w % s.KB : w / s.KB;
    sx = side == 0 ? c * s.KA + y : y * Kold + c;
    sy = 0;
    sz = 0;
  } else if (s.kind == K_FOLD) {   // Eq. 7, source fixed to k* = KB: X=o_j, Y=F(e,k*,p), Z=o_src(k*)|unit
    sx = sg;
    sy = s.KB * s.KA + sg;           // K=1 fold: KB = KC = 0 (R13)
    sz = s.KC;
  } else {                         // K_EDGE (X=e1, Y=e2)
    sx = sg;
    sy = sg;
    sz = 0;
  }
}

struct Blk {
  int64_t o[3];
  int64_t n[3];
};

__device__ __forceinline__ Blk load_blk(const StepDev& s, int64_t sg, int64_t k) {
  int64_t sx, sy, sz;
  block_factor_segs(s, sg, k, sx, sy, sz);
  Blk b;
  b.o[0] = s.X.off[sx];
  b.n[0] = s.X.off[sx + 1] - b.o[0];
  b.o[1] = s.Y.off[sy];
  b.n[1] = s.Y.off[sy + 1] - b.o[1];
  b.o[2] = s.Z.off[sz];
  b.n[2] = s.Z.off[sz + 1] - b.o[2];
  return b;
}

// log2 of the sample stride of level l (level 0 = everything).
__host__ __device__ __forceinline__ int level_shift(int l, int slog0, int slog) {
  return l == 0 ? 0 : slog0 + slog * (l - 1);
}

// Sampled index set at stride st = 2^sh: {0, st, 2st, ...} U {n-1}.
// (The level-l sample of every factor; nested across levels.)
__device__ __forceinline__ int64_t samp_cnt(int64_t n, int sh) {
  if (sh == 0 || n <= 1) return n;
  const int64_t st = (int64_t)1 << sh;
  int64_t c = (n + st - 1) >> sh;
  if ((n - 1) & (st - 1)) ++c;
  return c;
}
__device__ __forceinline__ int64_t samp_idx(int64_t j, int64_t n, int sh) {
  const int64_t c0 = (n + ((int64_t)1 << sh) - 1) >> sh;
  return j < c0 ? (j << sh) : n - 1;
}

// 32-bit variant for indices inside one factor segment (a segment frontier
// holds < 2^31 tuples); the stride 2^sh itself may exceed 2^31.
__device__ __forceinline__ int samp_idx32(int j, int n, int sh) {
  const int64_t c0 = ((int64_t)n + ((int64_t)1 << sh) - 1) >> sh;
  return j < c0 ? (int)((int64_t)j << sh) : n - 1;
}

__device__ __forceinline__ const int64_t* fac_m(const StepDev& s, int f) {
  return f == 0 ? s.X.m : (f == 1 ? s.Y.m : s.Z.m);
}
__device__ __forceinline__ const int64_t* fac_t(const StepDev& s, int f) {
  return f == 0 ? s.X.t : (f == 1 ? s.Y.t : s.Z.t);
}

// Product tuple for actual factor indices (x, y, z) of block b; id =
// lexicographic (k, x, y, z) rank within the segment (R6).
__device__ __forceinline__ void make_tuple(const StepDev& s, const Blk& b, int64_t rel, int64_t x,
                                           int64_t y, int64_t z, int64_t& m, int64_t& t,
                                           uint64_t& id) {
  m = __ldg(s.X.m + b.o[0] + x) + __ldg(s.Y.m + b.o[1] + y) + __ldg(s.Z.m + b.o[2] + z);
  t = __ldg(s.X.t + b.o[0] + x) + __ldg(s.Y.t + b.o[1] + y) + __ldg(s.Z.t + b.o[2] + z);
  id = (uint64_t)(rel + (x * b.n[1] + y) * b.n[2] + z);
}

template <typename T>
__device__ __forceinline__ T warp_incl_sum(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += u;
  }
  return v;
}
__device__ __forceinline__ long long warp_incl_min(long long v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    long long u = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v = u < v ? u : v;
  }
  return v;
}

// Block-wide exclusive scans (all threads must call).  sh: >= 33 slots.
template <int NT>
__device__ __forceinline__ long long block_excl_min(long long v, long long* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long inc = warp_incl_min(v);
  if (lane == 31) sh[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    long long w = lane < NT / 32 ? sh[lane] : INF;
    long long wi = warp_incl_min(w);
    long long we = __shfl_up_sync(0xffffffffu, wi, 1);
    if (lane == 0) we = INF;
    if (lane < NT / 32) sh[lane] = we;
  }
  __syncthreads();
  long long ex = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) ex = INF;
  long long wpre = sh[wid];
  __syncthreads();
  return ex < wpre ? ex : wpre;
}
template <int NT>
__device__ __forceinline__ long long block_excl_sum(long long v, long long* sh, long long* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long inc = warp_incl_sum(v);
  if (lane == 31) sh[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    long long w = lane < NT / 32 ? sh[lane] : 0;
    long long wi = warp_incl_sum(w);
    if (lane < NT / 32) sh[lane] = wi - w;
    if (lane == NT / 32 - 1) sh[32] = wi;
  }
  __syncthreads();
  long long r = inc - v + sh[wid];
  *total = sh[32];
  __syncthreads();
  return r;
}

// Bitonic sort of N (power of 2) keys in shared memory, ascending (m, t, id).
template <int NT>
__device__ void bitonic_smem(int64_t* m, int64_t* t, uint64_t* id, int N) {
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < N; i += NT) {
        int l = i ^ j;
        if (l > i) {
          bool up = (i & k) == 0;
          bool gt = key_lt(m[l], t[l], id[l], m[i], t[i], id[i]);
          if (gt == up) {
            int64_t a = m[i]; m[i] = m[l]; m[l] = a;
            a = t[i]; t[i] = t[l]; t[l] = a;
            uint64_t b = id[i]; id[i] = id[l]; id[l] = b;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Alg.1 sweep over n sorted keys in smem with carry-in v0 (lines 4-8,
// P:490-494): keep[i] = t[i] < min(v0, t[0..i-1]).  Each thread owns a
// contiguous range.  Writes keep flags into kf (int smem), returns count.
template <int NT>
__device__ int alg1_sweep_smem(const int64_t* t, int n, long long v0, int* kf, long long* sh) {
  const int per = (n + NT - 1) / NT;
  const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
  long long lmin = INF;
  for (int i = lo; i < hi; ++i) lmin = t[i] < lmin ? t[i] : lmin;
  long long pre = block_excl_min<NT>(lmin, sh);
  long long v = pre < v0 ? pre : v0;
  int c = 0;
  for (int i = lo; i < hi; ++i) {
    int k = t[i] < v;
    kf[i] = k;
    c += k;
    if (k) v = t[i];
  }
  long long tot;
  long long off = block_excl_sum<NT>(c, sh, &tot);
  // convert flags to output positions (+1; 0 = dropped)
  int p = (int)off;
  for (int i = lo; i < hi; ++i) {
    if (kf[i]) kf[i] = ++p;
  }
  __syncthreads();
  return (int)tot;
}

}  // namespace ftk
