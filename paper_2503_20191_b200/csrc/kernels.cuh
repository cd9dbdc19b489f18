// Device kernels of the batched simulator (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/maya_b200.h"
#include "soa.h"

namespace maya {

// ExecOp.w sentinels
static const uint64_t EXEC_BAD = ~0ull << 2;             // KERN whose estimator failed
static const uint64_t EXEC_NONE = ((~0ull) >> 2) << 2;   // WAIT on a never-recorded event
static const uint64_t EXEC_OVF = EXEC_BAD - 4;           // folded kernel run whose composite
                                                         // leaves int64 (the run's times do too)

// Device view of one uploaded batch (all pointers into the device arena).
struct DevBatch {
  const JobHdr *jobs;
  const RankRec *ranks;
  const uint32_t *rank_comm;
  const CommRec *comms;
  const SlotRec *wfeats;      // unique call records (wire features)
  const Walker *walkers;      // heaviest stream first
  const uint32_t *wids;       // rank-major (rank, stream) -> walker index
  const RepHdr *reps;
  const Op *ops;
  const StreamRange *streams;
  const uint32_t *coll_lc;
  const uint32_t *coll_idx;
  const uint32_t *coll_wf;    // per rep collective: batch-global wire feature if it folds (NO_WF)
  const SyncRec *syncs;
  const uint32_t *counts;
  const MemRec *mems;
  const Feature *feats;
  const uint32_t *feat_meta;
  const KBlock *blocks;       // kernel blocks (batch-global fid lists)
  const uint32_t *blk_fids;
  int64_t *blk_ab;            // per block: (A, Brel) composite after the estimator
  const RankColl *rcolls;
  const uint32_t *rcslot;     // batch-global call slot of each rank-collective entry
  RCX *rcx;                   // entry + wire time of each rank-collective entry (resolve)
  ExecOp *exec;
  // scratch / outputs
  uint32_t *feat_d32;          // per feature: duration (ns) when < DUR32_WIDE, else DUR32_*
  int64_t *feat_ns;            // per feature: the duration when feat_d32 is DUR32_WIDE
  int64_t *wire;
  int64_t *fire;
  int64_t *delay;
  uint8_t *spill;             // per-job global spill (JobHdr.wstate = byte offset)
  CollSlot *cslots;
  RepOut *repout;
  int64_t *tl_start;
  int64_t *tl_end;
  maya_job_result *results;
  const int32_t *order;       // CTA -> job (largest first)
  const LaneJob *lane_jobs;   // per job: lane-scheduler layout choice
  const uint32_t *lane_wslot; // per walker: ring slot word (soa.h)
  const uint32_t *lane_perm;  // per job: lane -> FIFO tables
  const GridPart *grid_parts; // grid jobs: one entry per part (CTA)
  GridSync *gsync;            // per job (grid jobs only)
  const uint32_t *comm_part;  // per comm: the grid part holding all its members, else ~0
  uint8_t *lane_gctx;         // per walker: 64 B FIFO context when not in shared memory
  uint8_t *lane_gst;          // per walker: 48 B FIFO state when LANE_ST_GLOBAL
  ChainMacro *macros;         // chain jobs, folded runs: each FIFO's macro ops (chain_macro_kernel)
  const FoldChunk *chunks;    // fold work items (one per 1,024 ops of a FIFO)
  uint32_t n_chunks;
  uint32_t *clen;             // folded FIFO lengths (fold_kernel) or null: unfolded ops
  uint32_t *ccounts;          // host-sync dispatch counts in folded indices (with clen)
  int32_t *err_flag;          // any estimator failure
  uint32_t n_jobs, n_reps, n_feats, n_slots, n_blocks, n_wfeats;
  uint64_t n_ops, n_rcolls;
};

// Roofline constants of one (device, dtype, op kind) class, for the straight-
// line fast path of the estimator (kernels.cu estimate_fast):
// compute = ceil(flops * K / D) with K = 1e9 * eff_den, D = peak * eff_num
// (= the reference's ceil(ceil(flops * 1e9 * den / peak) / num)), exact while
// flops <= maxf; memory = ceil(bytes * 1e9 / H).  D == 0 / H == 0: no fast path.
// M* = floor(2^64 / y), ~0 for y == 1 (kernels.cu ceil_div_magic).
struct EstClass {
  uint64_t K, D, MD, maxf, H, MH;
};

// feature durations are stored in 4 B (the common case: below 4.29 s) with
// two escapes: WIDE = read the 8 B value from feat_ns, FAIL = EstimationError
static constexpr uint32_t DUR32_WIDE = 0xfffffffeu, DUR32_FAIL = 0xffffffffu;
// err_flag bits: 1 = a feature estimate failed, 2 = a wire estimate failed,
// ERR_WIDE_DUR = some feature duration needs its 8-byte escape (not an error)
static constexpr int32_t ERR_WIDE_DUR = 4;

struct DevTables {
  const EstClass *cls;         // [device][MAYA_MAX_DTYPES][n_op_kinds]
  const DevTables *gtab;       // this table's copy in device memory (the general
                               // estimator reads it there: no per-thread param copy)
  maya_device_params devs[8];
  int64_t eff_num[64];
  int64_t eff_den[64];
  int32_t n_devs, n_op_kinds;
  int64_t overhead_ns;
  // reciprocals for the quotient estimates of the roofline (corrected exactly):
  // 1 / peak_flops[dtype], 1 / eff_num[op], 1 / hbm_bytes_per_s (0: none)
  double inv_peak[8][MAYA_MAX_DTYPES];
  double inv_num[64];
  double inv_hbm[8];
  // exact division by these invariant divisors: M = floor(2^64 / y) (0: y == 1)
  uint64_t mag_peak[8][MAYA_MAX_DTYPES];
  uint64_t mag_num[64];
  uint64_t mag_hbm[8];
  // 64-bit fast-path bounds per op kind: flops * 1e9 * eff_den and
  // peak * eff_num stay below 2^64
  uint64_t max_flops[64];
  uint64_t max_peak[64];
};

void launch_estimate(const DevBatch &b, const DevTables &t, cudaStream_t s);
void launch_memscan(const DevBatch &b, cudaStream_t s);
int sched_variant(uint32_t n_walkers, uint32_t n_ranks);   // 0..3
void launch_resolve(const DevBatch &b, cudaStream_t s);
void launch_schedule_variant(const DevBatch &b, int variant, const int32_t *order, uint32_t n,
                             int record, uint32_t smem, cudaStream_t s);
uint32_t sched_smem_cap();
void launch_schedule_lane_warp(const DevBatch &b, const int32_t *order, uint32_t n,
                               uint32_t warps_per_cta, uint32_t region, int record,
                               cudaStream_t s);
void launch_schedule_lane(const DevBatch &b, const int32_t *order, uint32_t n, uint32_t threads,
                          int record, uint32_t smem, cudaStream_t s);
// grid jobs: parts [p0, p1) of b.grid_parts in one cooperative launch
int launch_schedule_grid(const DevBatch &b, uint32_t p0, uint32_t p1, int record, uint32_t smem,
                         cudaStream_t s);
// chain jobs (sched_chain.cu): the macro ops of every FIFO of the n jobs
// order[0..n) (folded runs), then one CTA per job, whole job on chip
void launch_chain_macros(const DevBatch &b, const int32_t *order, uint32_t n, uint32_t max_fifos,
                         cudaStream_t s);
void launch_schedule_chain(const DevBatch &b, const int32_t *order, uint32_t n, uint32_t threads,
                           int record, uint32_t smem, cudaStream_t s);
int grid_max_ctas(uint32_t smem);   // co-resident CTAs of the grid kernel at this smem
int prof_read(unsigned long long *out8, int reset);   // MAYA_PROFILE builds only
int lane_prof_read(unsigned long long *out8, int reset);
int chain_prof_read(unsigned long long *out8, int reset);
void launch_topk(const DevBatch &b, int k, maya_topk_entry *out, int32_t *n_out, void *scratch,
                 cudaStream_t s);
size_t topk_scratch_bytes(uint32_t n_jobs, int k);
// per-rank busy statistics from a recorded timeline (stats.cu): out[4 * rank] =
// compute, comm, busy (unions), peak memory
size_t rank_stats_scratch_bytes(uint64_t n_tl, uint32_t n_ranks);
int launch_rank_stats(const DevBatch &b, const uint64_t *rank_seg, uint32_t n_ranks,
                      uint64_t n_tl, void *scratch, size_t scratch_bytes, int64_t *out,
                      cudaStream_t s);

}  // namespace maya
