// ft_step.h -- host interface of the per-step GPU pipeline (internal).
#pragma once
#include <cstdint>
#include <mutex>
#include <vector>
#include <cuda_runtime.h>

#include "ft_kernels.cuh"

namespace ftk {

struct StepResult {
  int64_t nloc = 0;        // segments computed on this rank
  int64_t total = 0;       // survivors over those segments
  int64_t tuples = 0;      // product tuples over those segments
  int64_t candidates = 0;  // pre-filter survivors over all levels
  int64_t filter_tuples = 0, direct_tuples = 0;  // sampled tuples per kernel family
  int64_t huge = 0;        // buckets that took the global-memory sort
  int64_t path[4] = {0, 0, 0, 0};  // shared rows: packed, packed with m ties, CTA fallback;
                                   // register-blocked k_direct segments
  int64_t retries = 0;
  int levels = 0;
  int64_t launches = 0;
  float kernel_ms = 0;
  float plan_ms = 0, direct_ms = 0, filter_ms = 0, bucket_ms = 0, compact_ms = 0, host_ms = 0;
  const int64_t* counts = nullptr;  // host (pinned) per-segment survivor counts [nloc]
  const int64_t* seg_tuples = nullptr;  // host (pinned) per-segment product tuples [nloc]
  const int64_t* step_stats = nullptr;  // device-offset mode: per step {survivors, max, tuples}
  const int64_t* dev_cnt = nullptr;     // keep_dev mode: per-local-segment counts (device)
  const int64_t* dev_tup = nullptr;     // keep_dev mode: per-local-segment tuples (device)
  Pool pool;                        // level-0 pool (device)
};

// Device memory: the caller's hooks (ft_options.alloc / .free) when set, else
// the stream-ordered pool (cudaMallocAsync) or, for grow-only scratch,
// cudaMalloc.
struct DevAlloc {
  void* (*alloc)(size_t, void*, void*) = nullptr;
  void (*free)(void*, void*, void*) = nullptr;
  void* ctx = nullptr;
  bool hooked() const { return alloc != nullptr; }
  cudaError_t get(void** p, size_t bytes, cudaStream_t st, bool scratch = false) const {
    if (alloc) {
      *p = alloc(bytes ? bytes : 1, (void*)st, ctx);
      return *p ? cudaSuccess : cudaErrorMemoryAllocation;
    }
    return scratch ? cudaMalloc(p, bytes) : cudaMallocAsync(p, bytes, st);
  }
  void put(void* p, cudaStream_t st, bool scratch = false) const {
    if (!p) return;
    if (free) free(p, (void*)st, ctx);
    else if (scratch) cudaFree(p);
    else cudaFreeAsync(p, st);
  }
  bool operator<(const DevAlloc& o) const {
    if (alloc != o.alloc) return (uintptr_t)alloc < (uintptr_t)o.alloc;
    if (free != o.free) return (uintptr_t)free < (uintptr_t)o.free;
    return (uintptr_t)ctx < (uintptr_t)o.ctx;
  }
};

// Process-wide scratch + pipeline per (CUDA device, allocator), shared by all
// graphs with that pair (its mutex is held for a whole wave; see ft_api.cu).
class StepRunner;
StepRunner* device_runner(int device, const DevAlloc& a);
// A graph is done with its runner: a hooked runner (caller allocator) hands its
// device scratch back through the hooks when its last graph is destroyed (so
// every hooked allocation is returned by then); the default runner keeps its
// scratch for the process lifetime.
void release_runner(int device, const DevAlloc& a);

// One (step, w) row of a shared-order node elimination (k_node_shared).
struct NodeGroup {
  int32_t step;
  int32_t pad;
  int64_t w, p_lo, p_hi;  // p range [p_lo, p_hi) of this rank's segments in row w
  int64_t gs0;            // local segment index of (w, p_lo)
};
using NodeGroupH = NodeGroup;

// Multi-rank device exchange: exclusive scan of the wave's per-segment counts
// (step-major) into pos[0..NS], CSR offsets into `off` (arena layout) and
// per-step {survivors, max, tuples} into stats[3*ns] (device).
cudaError_t wave_offsets(const int64_t* cnt, const int64_t* tup, int64_t NS, int ns,
                         const int64_t* sbase_dev, int64_t* pos, int64_t* off, int64_t* stats,
                         int64_t* scan_tmp, cudaStream_t st);
// Copies this rank's level-0 pool (global segments [lo, hi)) into the arena at pos.
cudaError_t gather_range(const Pool& P, const int64_t* pos, int64_t lo, int64_t hi, int64_t nout,
                         int64_t* om, int64_t* ot, uint64_t* obp, cudaStream_t st);
int64_t scan_tmp_elems(int64_t n);
// All-gather exchange helpers: gathered per-rank count blocks
// -> per-segment counts / tuples; gathered per-rank survivor blocks -> arena.
cudaError_t unpack_counts(const int64_t* all, int64_t maxloc, const int64_t* lo_dev, int world, int64_t NS,
                          int64_t* cnt, int64_t* tup, cudaStream_t st);
cudaError_t unpack_data(const int64_t* all, int64_t cap, const int64_t* posb_dev, int world, int64_t maxn,
                        int64_t* om, int64_t* ot, uint64_t* obp, cudaStream_t st);

// Validates costs on the device (bit 0: negative, bit 1: >= 2^40) and reports
// per edge whether its memory costs are all zero.
cudaError_t validate_costs(const int64_t* d, int64_t n, const int64_t* em,
                           const std::vector<int64_t>& e_off, int ne, int32_t* status_host,
                           char* mz_host, cudaStream_t st, const DevAlloc& A);

class StepRunner {
 public:
  StepRunner();
  ~StepRunner();
  cudaError_t configure();
  // Runs a batch of independent steps, each for its segments [seg_lo,
  // seg_hi); on success res->counts (local segments, in batch order) and
  // res->pool describe the results (valid until the next run).
  // dev_off != nullptr (single rank): write the wave's CSR offsets on the device
  // (arena layout) and return only per-step totals in res->step_stats.
  cudaError_t run(const std::vector<StepDev>& steps, cudaStream_t st, StepResult* res,
                  int64_t* dev_off = nullptr, const std::vector<NodeGroupH>* groups = nullptr,
                  bool keep_dev = false);
  // Gathers the level-0 pool into each step's CSR output (steps[j].out_*).
  cudaError_t gather(const std::vector<StepDev>& steps, const StepResult& r, cudaStream_t st);
  void release();
  void release_device();  // device scratch only (hooked runners, last graph gone)
  // Marks the end of a wave's use of the scratch on stream st; the next run()
  // on another stream waits for it (waves do not end with a host sync).
  void fence(cudaStream_t st) {
    if (!fence_ev) cudaEventCreateWithFlags(&fence_ev, cudaEventDisableTiming);
    cudaEventRecord(fence_ev, st);
    fence_st = st;
  }

  int slog = 3;                       // sample stride x8 per level beyond level 1 (A/B after the block
                                      // pre-filter, C5 / C4 ms: x8 44.6 / 33.8, x16 45.4 / 34.4, x32 48.3 / 38.3)
  int slog0 = 2;                      // level-1 stride 2^slog0 = 4 (tight G for level 0)
  int cdirect = 512;                  // direct-path capacity of large waves (power of 2 <= C_DIRECT;
                                      // A/B: 512 beats 1024 on C4 by 1 ms, C5 equal)
  int small_wave_segs = 4096;         // waves with <= this many segments: capacity cdirect_small (A/B: 4096 > 1024 > 0)
  int cdirect_small = 2048;           // direct capacity of waves of <= small_wave_segs segments
  int fstats = 0;                     // FT_FILTER_STATS: accumulate filter work counters
  int filter_grid = 148 * 128;         // CTAs of k_filter (grid-stride; set in configure())
  int pack_grid = 148 * 6;             // CTAs of k_node_pack (each takes a contiguous pack range; A/B: 888 > 592 > 444 > 296 on C5)
  bool filter_regs64 = false;          // k_filter64 (64 registers) instead of k_filter (80)
  int item_max = 256;                 // filter work item: max sampled run elements
  int item_div = 16;                  // ... and target items per resident thread (A/B: 256/16 best since
                                      // the block pre-filter; was 512/4)
  unsigned long long fstat_acc[8] = {};
  unsigned long long bstat_acc[2][10] = {};
  unsigned long long bfall_acc[2] = {};
  bool profile = false;               // events between kernel groups
  DevAlloc alloc;                     // scratch memory (set once at creation)
  std::mutex mu;                      // held by a graph for a whole wave
  int users = 0;                      // live graphs (device_runner / release_runner)
  int64_t cand_budget = 16 << 20;     // candidate capacity (grown on overflow)
  int64_t out_budget = 1 << 20;
  int64_t bucket_budget = 1 << 20;

 private:
  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
    size_t hw = 0;  // capacity before the last release_device: re-grown in one step
  };
  Buf seg_d, seg_n, blk_rel, seg_tuples, hdr;
  Buf poolA_m, poolA_t, poolA_id, poolA_start, poolA_cnt;
  Buf poolB_m, poolB_t, poolB_id, poolB_start, poolB_cnt;
  Buf cursors, nb, bucket_base, wcnt, wo, bcount, bmin, boff, bcarry;
  Buf cm, ct, cid, cgb, gm, gt, gid, gflag, large_list, scan_tmp, ncand, dst_off;
  Buf steps_dev, base_dev, pos, step_arr, groups_dev, packs_dev, big_dev, whint;
  std::vector<int64_t> step_host;
  int64_t* step_host_p = nullptr;
  std::vector<int64_t> h_base;
  BatchDev batch{};
  StepHdr* hdr_host = nullptr;
  int64_t* cnt_host = nullptr;
  int64_t cnt_host_n = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t fence_ev = nullptr;
  cudaStream_t fence_st = nullptr;
  cudaEvent_t pev[64] = {};
  int npev = 0;
};

}  // namespace ftk
