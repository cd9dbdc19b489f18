// C ABI of the engine (include/maya_b200.h): batch assembly, upload, run,
// results, search reduction, timeline.
#include <cuda_runtime.h>
#include <chrono>

#include <algorithm>
#include <cstdlib>
#include <functional>
#include <atomic>
#include <memory>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/maya_b200.h"
#include "kernels.cuh"
#include "gen.h"
#include "pack.h"
#include "pool.h"
#include "traceio.h"

using namespace maya;

namespace {

thread_local std::string g_err;
thread_local int g_err_kind = 0;

// warp-window jobs at or under this layout size launch separately, opt-in via
// MAYA_SPLIT_SMEM (bytes; default 0 = one launch per group).  Measured on C2
// (profiles/split_smem_r1.json): 40 KB keeps the scheduler out of its slow mode
// but costs the step ~0.08 ms, netting 461k vs 476k configs/s on average.
static uint32_t split_smem_threshold() {
  static const uint32_t t = [] {
    const char *v = getenv("MAYA_SPLIT_SMEM");
    return v ? (uint32_t)strtoul(v, nullptr, 10) : 0u;
  }();
  return t ? t : 0xffffffffu;
}

int fail(int code, const std::string &msg) {
  g_err = msg;
  g_err_kind = 0;
  return code;
}
int fail_trace(const TraceFail &f) {
  g_err = f.msg;
  g_err_kind = f.kind;
  return MAYA_EINVAL;
}

#define CU(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess)                                                           \
      return fail(MAYA_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));      \
  } while (0)

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// One array of the arena: host bytes copied at [off, off + bytes).
struct Seg {
  size_t off = 0, bytes = 0;
};

// JobPacks are pooled across batches: their vectors keep capacity, so
// re-staging a batch does not fault in fresh pages (which serialises host
// threads in the kernel's page-fault path).
struct PackPool {
  std::vector<std::unique_ptr<JobPack>> pool;
  size_t n = 0;
  size_t size() const { return n; }
  void clear() { n = 0; }
  void resize(size_t m) {
    while (pool.size() < m) pool.push_back(std::make_unique<JobPack>());
    n = m;
  }
  JobPack &operator[](size_t i) { return *pool[i]; }
  const JobPack &operator[](size_t i) const { return *pool[i]; }
};

}  // namespace

struct maya_engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {};
  // scheduler launch groups: 0-2 warp-window kernel (4/8/16 warps), 3-10 lane
  // kernel warp jobs (by shared-memory region class), 11-14 lane kernel CTA
  // jobs (2/4/8/16 warps); each group runs on its own stream (fork/join)
  // 15: grid jobs (cooperative launch over their parts); 16..: chain kernel
  // jobs by shared-memory region class (CHAIN_REGION) and CTA size (1, 2, 4,
  // 8 warps: CHAIN_CLASSES variants each)
  static const int NVAR = 16 + 4 * (int)CHAIN_CLASSES;
  cudaStream_t vstream[NVAR] = {};
  cudaEvent_t vev[NVAR + 1] = {};
  uint32_t var_n[NVAR] = {};        // jobs per group (order segments)
  uint32_t var_smem[NVAR] = {};     // dynamic smem per group launch
  // warp-window groups split by shared-memory footprint: the jobs whose layout
  // fits SMALL_SMEM run in a second launch sized for them (a group's launch
  // otherwise reserves its largest job's smem for every CTA)
  cudaStream_t sstream[3] = {};
  cudaEvent_t sev[3] = {};
  uint32_t var_big[3] = {};         // leading jobs of the group's segment above SMALL_SMEM
  uint32_t var_smem_small[3] = {};
  // staged jobs
  PackPool packs;
  std::vector<maya_device_params> devs;
  std::vector<int64_t> eff_num, eff_den;
  int64_t overhead_ns = 1000;
  // arena (inputs) and scratch (device only)
  void *h_arena = nullptr;
  size_t h_arena_cap = 0;
  void *d_arena = nullptr;
  size_t d_arena_cap = 0;
  size_t arena_bytes = 0;
  void *d_scratch = nullptr;
  void *d_est = nullptr;    // DevTables copy + EstClass table (estimator)
  size_t d_est_cap = 0;
  size_t d_scratch_cap = 0;
  size_t scratch_bytes = 0;
  bool uploaded = false, ran = false, recorded = false;
  DevBatch db{};
  DevTables tables{};
  // segments
  Seg s_fmeta;
  Seg s_jobs, s_ranks, s_rank_comm, s_comms, s_wfeats, s_walkers, s_reps, s_ops, s_streams,
      s_coll_lc, s_coll_idx, s_coll_wf, s_syncs, s_counts, s_mems, s_feats, s_order, s_rcolls, s_wids, s_rcslot,
      s_lane_jobs, s_lane_wslot, s_lane_perm, s_chunks, s_grid_parts, s_comm_part, s_blocks,
      s_blk_fids;
  Seg x_clen, x_ccounts, x_lctx, x_lst, x_gsync, x_macros;
  uint32_t chain_first = 0, chain_jobs = 0;   // chain jobs: the tail of the job order
  uint32_t chain_maxw = 0;                    // their largest FIFO count
  std::vector<int32_t> job_kernel;            // per job: 0 warp-window, 1 lane, 2 grid, 3 chain
  cudaGraphExec_t graph_exec = nullptr;       // the run's device work, captured (maya_run)
  bool graph_fold = false;
  uint32_t runs_since_upload = 0;
  std::vector<GridPart> grid_parts;        // host copy (launch grouping)
  std::vector<std::pair<uint32_t, uint32_t>> grid_launches;   // part ranges per launch
  uint32_t grid_smem = 0;
  Seg x_blk_ab;
  bool has_blocks = false;             // staged jobs carry kernel blocks (must run folded)
  Seg x_exec, x_rcw, x_feat_ns, x_feat_d32, x_wire, x_fire, x_delay, x_wstate, x_cslots, x_repout, x_tl_start, x_tl_end,
      x_results, x_err, x_topk, x_topk_out, x_topk_n;
  uint64_t n_tl = 0;
  std::vector<uint64_t> job_tl;      // per job timeline base
  std::vector<uint64_t> job_ops;     // per job batch op base (for op_seq/streams)
  std::vector<uint32_t> job_rank0;   // per job batch index of its first simulated rank
  std::vector<uint64_t> rank_seg;    // per batch rank: timeline base (n_ranks + 1 entries)
  void *d_stats = nullptr;           // rank_seg + per-rank stats + sort scratch (timeline runs)
  size_t d_stats_cap = 0;
  int64_t *d_rstats = nullptr;       // [n_ranks][4] compute, comm, busy, peak
  bool stats_ok = false;
  float last_ms[3] = {0, 0, 0};
  int64_t run_launches = 0, topk_launches = 0;
  maya_topk_entry *h_topk = nullptr;   // pinned: 64 entries + count (maya_topk_async)
  int32_t topk_pending = 0;            // k of an enqueued, not yet read top-k
  int32_t options = MAYA_OPT_COLLAPSE;
};

namespace {

// Lane-scheduler plan of one job: launch shape, ring depth and which tables
// live in shared memory, greedily from the fastest layout down to what fits
// the per-job budget (sized so that a large batch keeps many jobs resident
// per SM; a small batch gets the whole CTA budget per job).
//   variants 3..10: warp jobs, region classes LANE_REGION[v-3]
//   variants 11..14: CTA jobs of 2/4/8/16 warps
//   -1: the job runs on the warp-window kernel (variants 0..2)
static const uint32_t LANE_REGION[8] = {14u << 10, 20u << 10, 28u << 10, 40u << 10,
                                        56u << 10, 80u << 10, 112u << 10, LANE_SMEM_CAP};
static const uint32_t LANE_WARP_JOB_MAX_FIFOS = 128;   // 4 FIFOs per lane

struct LanePlan {
  int variant = -1;
  uint32_t flags = 0, n_slots = 0, smem = 0, lgd_max = 0, threads = 32, per_lane = 1, fc_log2 = 0;
  std::vector<GridPart> parts;   // variant 15: the job's CTAs (job/wslot/first filled at upload)
};

uint32_t lane_slots_of(uint32_t len, uint32_t lgd_max) {
  if (len == 0 || lgd_max == 0xff) return 0;
  const uint32_t chunks = (len + LANE_SLOT_OPS - 1) / LANE_SLOT_OPS;
  uint32_t lg = 0;
  while ((1u << lg) < chunks && lg < lgd_max) lg++;
  return 1u << lg;
}

// device events of a FIFO (a kernel block counts its launches): the shape the
// kernel-choice thresholds below were tuned on
uint32_t lane_fifo_len(const JobPack &P, uint32_t w) {
  const Walker wk = P.walkers[w];
  const RepHdr &h = P.reps[P.ranks[wk.rank].rep];
  return P.stream_events[h.streams + wk.stream];
}

static const uint32_t GRID_PART_FIFOS = 256;   // one FIFO per thread of a grid-job CTA

// A job with more FIFOs than a CTA has threads runs as a grid job: rank-aligned
// parts of <= 256 FIFOs, one CTA each, rings sized by folded FIFO length.
bool plan_grid(const JobPack &P, LanePlan &pl) {
  const uint32_t W = (uint32_t)P.walkers.size(), R = (uint32_t)P.ranks.size();
  const uint32_t nc = (uint32_t)P.comms.size();
  std::vector<GridPart> parts;
  uint32_t w = 0;
  for (uint32_t r = 0; r < R;) {
    GridPart g{};
    g.r0 = r;
    g.w0 = w;
    while (r < R) {
      const uint32_t ns = P.reps[P.ranks[r].rep].n_streams;
      if (w + ns - g.w0 > GRID_PART_FIFOS && r > g.r0) break;
      w += ns;
      r++;
    }
    g.r1 = r;
    g.w1 = w;
    parts.push_back(g);
  }
  if (w != W) return false;
  uint32_t smem_max = 0;
  for (GridPart &g : parts) {
    uint32_t fc = 0;
    while ((1u << fc) < 8 * (g.r1 - g.r0) && fc < 12) fc++;
    bool ok = false;
    for (uint32_t lgd : {2u, 1u, 0xffu}) {
      uint64_t slots = 0;
      for (uint32_t q = g.w0; q < g.w1; q++) {
        const Walker wk = P.walkers[q];
        const RepHdr &h = P.reps[P.ranks[wk.rank].rep];
        slots += lane_slots_of(P.streams[h.streams + wk.stream].folded, lgd);
      }
      const uint32_t ringf =
          (P.hdr.flags & JOB_RING) && nc <= RING_MAX_COMMS ? LANE_COLL_RING : 0u;
      const LaneLayout L = lane_layout(g.w1 - g.w0, g.r1 - g.r0, nc, ringf, (uint32_t)slots,
                                       P.hdr.n_fire, P.hdr.n_rcolls, fc);
      if (L.bytes > LANE_SMEM_CAP) continue;
      g.flags = ringf;
      g.n_slots = (uint32_t)slots;
      g.fc_log2 = fc;
      g.wslot = lgd;   // ring depth, replaced by the batch index at upload
      smem_max = std::max(smem_max, L.bytes);
      ok = true;
      break;
    }
    if (!ok) return false;
  }
  for (GridPart &g : parts) {
    g.part = (uint32_t)(&g - parts.data());
    g.n_parts = (uint32_t)parts.size();
    g.warps_total = (uint32_t)parts.size() * (GRID_PART_FIFOS / 32);
  }
  pl.variant = 15;
  pl.parts = std::move(parts);
  pl.smem = smem_max;
  pl.threads = GRID_PART_FIFOS;
  pl.per_lane = 1;
  return true;
}

// Chain-kernel plan (sched_chain.cu): the whole job resident in one CTA's
// shared-memory region -- every FIFO's macro ops (its folded ops fused into
// [WAIT]? [KERN | COLL]? [REC]? groups), record times, collective rings and
// rank collective table -- one FIFO per thread (collectives rendezvous in
// shared-memory rings when the job allows them, JOB_RING, else in global
// slots).  n_slots carries the job's macro op count (the region's op area).
LanePlan plan_chain(const JobPack &P) {
  LanePlan pl;
  const uint32_t W = (uint32_t)P.walkers.size(), R = (uint32_t)P.ranks.size();
  const uint32_t nc = (uint32_t)P.comms.size();
  if (P.hdr.status != MAYA_ST_OK || W == 0 || W > CHAIN_MAX_FIFOS) return pl;
  uint64_t n_ops = 0;   // macro ops (soa.h ChainMacro) of the job's FIFOs
  for (uint32_t w = 0; w < W; w++) {
    const Walker wk = P.walkers[w];
    n_ops += P.stream_macros[P.reps[P.ranks[wk.rank].rep].streams + wk.stream];
  }
  const ChainLayout L = chain_layout(W, R, nc, P.hdr.n_fire, P.hdr.n_rcolls, n_ops);
  if (L.bytes > CHAIN_REGION[CHAIN_CLASSES - 1]) return pl;
  uint32_t c = 0;
  while (CHAIN_REGION[c] < L.bytes) c++;
  const int lw = W <= 32 ? 0 : W <= 64 ? 1 : W <= 128 ? 2 : 3;   // log2 warps
  pl.threads = 32u << lw;
  pl.variant = 16 + (int)c + lw * (int)CHAIN_CLASSES;
  pl.smem = L.bytes;
  pl.n_slots = (uint32_t)n_ops;
  pl.per_lane = 1;
  return pl;
}

LanePlan plan_lane(const JobPack &P, uint32_t budget, bool force) {
  LanePlan pl;
  if (P.hdr.status != MAYA_ST_OK) { pl.variant = 3; return pl; }
  const uint32_t W = (uint32_t)P.walkers.size(), R = (uint32_t)P.ranks.size();
  if (!force) {
    // Lockstep lanes pay off when many FIFOs carry work; a few long FIFOs
    // (compute streams) are serial chains the warp-window kernel scans 32 ops
    // per step.
    // Criterion: the 32nd longest FIFO is at least a quarter of the longest
    // (a warp's worth of busy FIFOs; a pipeline's per-stage compute streams
    // are fewer), and no folded FIFO is longer than 8k ops.
    if (W < 32) return pl;
    std::vector<uint32_t> l(W);
    for (uint32_t w = 0; w < W; w++) l[w] = lane_fifo_len(P, w);
    std::nth_element(l.begin(), l.begin() + 31, l.end(), std::greater<uint32_t>());
    const uint32_t mx = *std::max_element(l.begin(), l.begin() + 32);
    if (l[31] < 64 || 4ull * l[31] < mx) return pl;
    // very long FIFOs after run folding: the warp-window scan's 32 ops per
    // step win even when many of them are busy (C4's 16-stage pipelines)
    uint32_t mxf = 0, wl = 0;
    for (uint32_t w = 0; w < W; w++) {
      const Walker wk = P.walkers[w];
      const uint32_t f = P.streams[P.reps[P.ranks[wk.rank].rep].streams + wk.stream].folded;
      if (f > mxf) { mxf = f; wl = w; }
    }
    if (mxf > 8192) return pl;
    // ... and the same when the longest FIFO rarely blocks: waits and
    // multi-member collectives (sampled over its first 4k ops) more than 128
    // ops apart leave long affine runs for the scan
    {
      const Walker wk = P.walkers[wl];
      const RankRec &rr = P.ranks[wk.rank];
      const RepHdr &h = P.reps[rr.rep];
      const StreamRange &sr = P.streams[h.streams + wk.stream];
      uint32_t n = 0, blockers = 0;   // over the first ~4k device events
      for (uint32_t q = 0; q < sr.len && n < 4096; q++) {
        const Op &o = P.ops[h.ops + sr.begin + q];
        const uint32_t tg = op_tag(o.meta);
        n += (tg == TAG_KERN && (o.arg & KBLOCK)) ? P.blocks[o.arg & ~KBLOCK].n : 1u;
        if (tg == TAG_WAIT) {
          blockers++;
        } else if (tg == TAG_COLL) {
          const uint32_t g = P.rank_comm[rr.comm + P.coll_lc[h.colls + o.arg]];
          blockers += P.comm_rdv[g] > 1 ? 1u : 0u;
        }
      }
      if (blockers == 0 || n / blockers > 128) return pl;
    }
  }
  const uint32_t nc = (uint32_t)P.comms.size();
  const uint32_t ring = (P.hdr.flags & JOB_RING) && nc <= RING_MAX_COMMS ? LANE_COLL_RING : 0;
  if (W > LANE_MAX_THREADS) {   // a grid job: several co-resident CTAs
    if (!plan_grid(P, pl)) pl = LanePlan();
    return pl;
  }
  const bool warp_job = W <= LANE_WARP_JOB_MAX_FIFOS;
  if (!warp_job) budget = LANE_SMEM_CAP;
  std::vector<uint32_t> lens(W);   // ring sizing: the folded FIFO (what the kernel stages)
  for (uint32_t w = 0; w < W; w++) {
    const Walker wk = P.walkers[w];
    const RepHdr &h = P.reps[P.ranks[wk.rank].rep];
    lens[w] = P.streams[h.streams + wk.stream].folded;
  }
  const uint32_t nthreads = warp_job ? 32u : [&] {
    uint32_t nw = 2;
    while (nw * 32 < W && nw * 32 < LANE_MAX_THREADS) nw <<= 1;
    return nw * 32;
  }();
  const bool multi = W > nthreads;   // lanes own several FIFOs
  // FIFO contexts / states: shared memory first, global memory when the job's
  // FIFOs do not fit (thousands of ranks)
  const uint32_t place[3] = {multi ? LANE_CTX_SMEM : 0u, 0u, LANE_ST_GLOBAL};
  // record-time cache when the table stays global: 8 live records per rank
  uint32_t fc = 0;
  while ((1u << fc) < 8 * R && fc < 12) fc++;
  struct Try { uint32_t lgd, flags; };
  // deep rings before on-chip tables once the tables do not fit: a long FIFO
  // (1e5-1e6 events per rank) stalls on refills with 2 slots, while its record
  // and collective tables are read through the tagged cache / L1 anyway
  const Try tries[] = {{3, LANE_FIRE_SMEM | LANE_RCX_SMEM}, {2, LANE_FIRE_SMEM | LANE_RCX_SMEM},
                       {1, LANE_FIRE_SMEM | LANE_RCX_SMEM}, {3, LANE_FIRE_SMEM}, {3, 0},
                       {2, LANE_FIRE_SMEM}, {2, 0},
                       {1, LANE_FIRE_SMEM}, {1, 0}, {0xff, LANE_FIRE_SMEM}, {0xff, 0}};
  for (int pass = 0; pass < 2; pass++) {
    const uint32_t cap = pass == 0 ? budget : LANE_SMEM_CAP;
    for (uint32_t pc = 0; pc < 3; pc++) {
    if (pc > 0 && !multi) break;
    const uint32_t ctxf = place[pc];
    for (const Try &t : tries) {
      uint64_t slots = 0;
      for (uint32_t w = 0; w < W; w++) slots += lane_slots_of(lens[w], t.lgd);
      if (slots >= (1u << 28)) continue;
      const uint32_t fl = ring | t.flags | ctxf;
      const LaneLayout L =
          lane_layout(W, R, nc, fl, (uint32_t)slots, P.hdr.n_fire, P.hdr.n_rcolls, fc);
      if (L.bytes > cap) continue;
      pl.flags = fl;
      pl.n_slots = (uint32_t)slots;
      pl.smem = L.bytes;
      pl.lgd_max = t.lgd;
      pl.fc_log2 = (fl & LANE_FIRE_SMEM) ? 0 : fc;
      if (warp_job) {
        int v = 0;
        while (v < 7 && LANE_REGION[v] < L.bytes) v++;
        pl.variant = 3 + v;
        pl.threads = 32;
      } else {
        uint32_t nw = 2;
        while (nw * 32 < W && nw * 32 < LANE_MAX_THREADS) nw <<= 1;
        pl.variant = nw == 2 ? 11 : nw == 4 ? 12 : nw == 8 ? 13 : 14;
        pl.threads = nw * 32;
      }
      pl.per_lane = (W + pl.threads - 1) / pl.threads;
      if (pl.per_lane == 0) pl.per_lane = 1;
      return pl;
    }
    }
  }
  return pl;
}

// lane -> FIFO table (per_lane x threads).  Warp jobs: LPT on FIFO length, so
// the heavy FIFOs (compute streams) land on distinct lanes.  CTA jobs: one
// FIFO per thread in rank-major order (the streams of a rank and the ranks of
// a communicator share a warp), or contiguous blocks when FIFOs outnumber
// threads.
void lane_perm_fill(const JobPack &P, const LanePlan &pl, uint32_t *out) {
  const uint32_t W = (uint32_t)P.walkers.size(), T = pl.threads, K = pl.per_lane;
  for (uint32_t q = 0; q < K * T; q++) out[q] = 0xffffffffu;
  if (W <= T) {
    for (uint32_t w = 0; w < W; w++) out[w] = w;
    return;
  }
  if (T > 32) {
    for (uint32_t w = 0; w < W; w++) out[(w % K) * T + w / K] = w;
    return;
  }
  std::vector<uint32_t> idx(W);
  for (uint32_t w = 0; w < W; w++) idx[w] = w;
  std::vector<uint32_t> lens(W);
  for (uint32_t w = 0; w < W; w++) lens[w] = lane_fifo_len(P, w);
  std::stable_sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) { return lens[a] > lens[b]; });
  std::vector<uint64_t> load(T, 0);
  std::vector<uint32_t> fill(T, 0);
  for (uint32_t w : idx) {
    uint32_t best = 0xffffffffu;
    for (uint32_t t = 0; t < T; t++)
      if (fill[t] < K && (best == 0xffffffffu || load[t] < load[best])) best = t;
    out[fill[best] * T + best] = w;
    fill[best]++;
    load[best] += lens[w] + 1;
  }
}

}  // namespace

namespace {
template <typename T>
bool vec_eq(const std::vector<T> &a, const std::vector<T> &b) {
  return a.size() == b.size() && (a.empty() || memcmp(a.data(), b.data(), a.size() * sizeof(T)) == 0);
}
bool pack_eq(const JobPack &a, const JobPack &b) {
  return memcmp(&a.hdr, &b.hdr, sizeof(JobHdr)) == 0 && vec_eq(a.reps, b.reps) &&
         vec_eq(a.ops, b.ops) && vec_eq(a.op_seq, b.op_seq) && vec_eq(a.streams, b.streams) &&
         vec_eq(a.coll_lc, b.coll_lc) && vec_eq(a.coll_idx, b.coll_idx) && vec_eq(a.coll_wf, b.coll_wf) &&
         vec_eq(a.syncs, b.syncs) && vec_eq(a.counts, b.counts) && vec_eq(a.mems, b.mems) &&
         vec_eq(a.feats, b.feats) && vec_eq(a.feat_meta, b.feat_meta) && vec_eq(a.comms, b.comms) && vec_eq(a.slots, b.slots) &&
         vec_eq(a.ranks, b.ranks) && vec_eq(a.rank_comm, b.rank_comm) &&
         vec_eq(a.walkers, b.walkers) && vec_eq(a.wids, b.wids) && vec_eq(a.rcolls, b.rcolls) &&
         vec_eq(a.rep_ring_ok, b.rep_ring_ok) && vec_eq(a.comm_rdv, b.comm_rdv) &&
         vec_eq(a.rank_orig, b.rank_orig) && vec_eq(a.rank_sim, b.rank_sim) &&
         vec_eq(a.stream_events, b.stream_events) && vec_eq(a.blocks, b.blocks) &&
         vec_eq(a.wfeats, b.wfeats) && vec_eq(a.slot_wf, b.slot_wf) &&
         vec_eq(a.blk_fids, b.blk_fids) &&
         a.collapsed == b.collapsed && a.n_fire == b.n_fire && a.n_delay == b.n_delay;
}
}  // namespace

extern "C" {

const char *maya_last_error(void) { return g_err.c_str(); }
int maya_abi_version(void) { return MAYA_ABI_VERSION; }

int maya_open(int cuda_device, maya_engine **out) {
  maya_engine *e = new maya_engine();
  e->device = cuda_device;
  cudaError_t err = cudaSetDevice(cuda_device);
  if (err != cudaSuccess) {
    delete e;
    return fail(MAYA_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(err));
  }
  err = cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking);
  if (err != cudaSuccess) {
    delete e;
    return fail(MAYA_ECUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(err));
  }
  for (auto &ev : e->ev) cudaEventCreate(&ev);
  for (auto &s : e->vstream) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (auto &ev : e->vev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  for (auto &s : e->sstream) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (auto &ev : e->sev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  *out = e;
  return MAYA_OK;
}

int maya_close(maya_engine *e) {
  if (!e) return MAYA_OK;
  cudaSetDevice(e->device);
  if (e->h_arena) cudaFreeHost(e->h_arena);
  if (e->d_arena) cudaFree(e->d_arena);
  if (e->d_scratch) cudaFree(e->d_scratch);
  if (e->d_est) cudaFree(e->d_est);
  if (e->d_stats) cudaFree(e->d_stats);
  if (e->h_topk) cudaFreeHost(e->h_topk);
  if (e->graph_exec) cudaGraphExecDestroy(e->graph_exec);
  for (auto &ev : e->ev) if (ev) cudaEventDestroy(ev);
  for (auto &ev : e->vev) if (ev) cudaEventDestroy(ev);
  for (auto &s : e->vstream) if (s) cudaStreamDestroy(s);
  for (auto &ev : e->sev) if (ev) cudaEventDestroy(ev);
  for (auto &s : e->sstream) if (s) cudaStreamDestroy(s);
  if (e->stream) cudaStreamDestroy(e->stream);
  delete e;
  return MAYA_OK;
}

int maya_batch_reset(maya_engine *e) {
  e->packs.clear();
  e->uploaded = e->ran = e->recorded = false;
  return MAYA_OK;
}

int maya_batch_set_devices(maya_engine *e, int32_t n, const maya_device_params *devs) {
  if (n < 0 || n > 8) return fail(MAYA_EINVAL, "at most 8 device classes per batch");
  e->devs.assign(devs, devs + n);
  return MAYA_OK;
}

int maya_batch_set_roofline(maya_engine *e, const maya_roofline_params *roof) {
  if (roof->n_op_kinds < 0 || roof->n_op_kinds > 64)
    return fail(MAYA_EINVAL, "at most 64 op kinds per batch");
  e->eff_num.assign(roof->eff_num, roof->eff_num + roof->n_op_kinds);
  e->eff_den.assign(roof->eff_den, roof->eff_den + roof->n_op_kinds);
  for (int i = 0; i < roof->n_op_kinds; i++)
    if (e->eff_num[i] <= 0 || e->eff_den[i] <= 0)
      return fail(MAYA_EINVAL, "efficiency fractions must be positive");
  e->overhead_ns = roof->overhead_ns;
  return MAYA_OK;
}

int maya_batch_add_job(maya_engine *e, const maya_raw_job *job, int32_t key_rank) {
  return maya_batch_add_jobs(e, 1, job, &key_rank, 1);
}

int maya_batch_add_jobs(maya_engine *e, int32_t n, const maya_raw_job *jobs,
                        const int32_t *key_ranks, int32_t n_threads) {
  if (n < 0) return fail(MAYA_EINVAL, "negative job count");
  for (int i = 0; i < n; i++)
    if (jobs[i].device < 0 || jobs[i].device >= 8)
      return fail(MAYA_EINVAL, "job device index out of range");
  size_t base = e->packs.size();
  e->packs.resize(base + n);
  std::atomic<int> next(0);
  auto work = [&]() {
    for (;;) {
      int i = next.fetch_add(1);
      if (i >= n) break;
      pack_job(jobs[i], key_ranks ? key_ranks[i] : i, e->packs[base + i],
               (e->options & MAYA_OPT_COLLAPSE) != 0);
    }
  };
  WorkerPool::get().run(std::max(1, std::min<int>(n_threads, n)), work);
  e->uploaded = e->ran = false;
  return MAYA_OK;
}

int maya_batch_num_jobs(maya_engine *e) { return (int)e->packs.size(); }

int maya_set_options(maya_engine *e, int32_t options) {
  e->options = options;
  return MAYA_OK;
}

int maya_batch_kernels(maya_engine *e, int32_t *out) {
  if (!e->uploaded) return fail(MAYA_ESTATE, "maya_batch_kernels before maya_upload");
  for (size_t j = 0; j < e->packs.size(); j++) out[j] = e->job_kernel[j];
  return MAYA_OK;
}

int maya_batch_collapsed(maya_engine *e, uint8_t *out) {
  for (size_t j = 0; j < e->packs.size(); j++) out[j] = e->packs[j].collapsed ? 1 : 0;
  return MAYA_OK;
}

int maya_upload(maya_engine *e) {
  static const bool dbg_t = getenv("MAYA_DEBUG_UPLOAD") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t_up0 = now();
  auto lap = [&](const char *what) {
    if (dbg_t)
      fprintf(stderr, "upload %-10s %.3f ms\n", what,
              std::chrono::duration<double>(now() - t_up0).count() * 1e3);
  };
  CU(cudaSetDevice(e->device));
  const size_t nj = e->packs.size();
  // totals
  size_t n_ranks = 0, n_rank_comm = 0, n_comms = 0, n_slots = 0, n_walkers = 0, n_reps = 0,
         n_ops = 0, n_streams = 0, n_colls = 0, n_syncs = 0, n_counts = 0, n_mems = 0,
         n_feats = 0, n_fire = 0, n_delay = 0, n_wstate = 0, n_rcolls = 0, n_chunks = 0,
         n_blocks = 0, n_blk_fids = 0, n_wfeats = 0;
  uint64_t n_tl = 0;
  e->job_tl.resize(nj);
  e->job_ops.resize(nj);
  e->job_rank0.resize(nj);
  e->rank_seg.clear();
  for (size_t j = 0; j < nj; j++) {
    const JobPack &P = e->packs[j];
    e->job_rank0[j] = (uint32_t)n_ranks;
    n_ranks += P.ranks.size();
    n_rank_comm += P.rank_comm.size();
    n_comms += P.comms.size();
    n_slots += P.slots.size();
    n_wfeats += P.wfeats.size();
    n_walkers += P.walkers.size();
    n_reps += P.reps.size();
    e->job_ops[j] = n_ops;
    n_ops += P.ops.size();
    n_streams += P.streams.size();
    n_colls += P.coll_lc.size();
    n_syncs += P.syncs.size();
    n_counts += P.counts.size();
    n_mems += P.mems.size();
    n_feats += P.feats.size();
    n_blocks += P.blocks.size();
    n_blk_fids += P.blk_fids.size();
    n_fire += P.n_fire;
    n_delay += P.n_delay;
    n_rcolls += P.rcolls.size();
    for (const StreamRange &sr : P.streams) n_chunks += (sr.len + FOLD_CHUNK - 1) / FOLD_CHUNK;
    {
      const SchedLayout L = sched_layout((uint32_t)P.walkers.size(), (uint32_t)P.ranks.size(),
                                         (uint32_t)P.comms.size(), (P.hdr.flags & JOB_RING) != 0,
                                         P.hdr.n_fire, P.hdr.n_rcolls, sched_smem_cap());
      if (!L.on_chip) n_wstate += spill_bytes(P.walkers.size(), P.ranks.size());
    }
    e->job_tl[j] = n_tl;
    for (const RankRec &rr : P.ranks) {
      e->rank_seg.push_back(n_tl);
      n_tl += P.reps[rr.rep].n_ops;
    }
  }
  e->rank_seg.push_back(n_tl);
  lap("totals");
  // scheduler plans (lane kernel unless disabled or the job does not fit it)
  std::vector<LanePlan> plans(nj);
  size_t n_perm = 0, n_macros = 0;
  {
    // per-job shared-memory budget: the whole CTA budget for small batches,
    // else enough to keep the batch resident (148 SMs x 228 KB)
    const uint64_t sm_bytes = 148ull * 228 * 1024;
    uint64_t budget = nj <= 296 ? LANE_SMEM_CAP : sm_bytes / nj;
    if (const char *ev = getenv("MAYA_LANE_BUDGET")) budget = strtoull(ev, nullptr, 10);
    if (budget < LANE_REGION[0]) budget = LANE_REGION[0];
    if (budget > LANE_SMEM_CAP) budget = LANE_SMEM_CAP;
    // Jobs whose FIFOs suit lockstep lanes (many balanced FIFOs that block
    // often: C5's per-rank-distinct traces) are throughput-bound and take the
    // lane kernel's resident rings.  The others -- chains of hand-offs between
    // few FIFOs (pipelines) -- take the chain kernel when the job fits one
    // CTA's shared memory (latency-optimised: ~1 k cycles per hand-off against
    // ~10 k for the warp-window kernel, which keeps the rest).
    const bool forced = (e->options & (MAYA_OPT_WARP_SCHED | MAYA_OPT_LANE_SCHED)) != 0;
    for (size_t j = 0; j < nj; j++) {
      if (!(e->options & MAYA_OPT_WARP_SCHED))
        plans[j] = plan_lane(e->packs[j], (uint32_t)budget, (e->options & MAYA_OPT_LANE_SCHED) != 0);
      if (plans[j].variant < 0 && !forced && !(e->options & MAYA_OPT_NO_CHAIN))
        plans[j] = plan_chain(e->packs[j]);
      if (plans[j].variant >= 0 && plans[j].variant != 15)
        n_perm += (size_t)plans[j].per_lane * plans[j].threads;
      if (plans[j].variant >= 16) n_macros += plans[j].n_slots;
    }
    if (getenv("MAYA_DEBUG_PLAN"))
      for (size_t j = 0; j < nj; j++) {
        const JobPack &P = e->packs[j];
        fprintf(stderr, "plan job %zu: variant %d smem %u per_lane %u W %zu R %zu comms %zu ring %d rcolls %u fire %u\n",
                j, plans[j].variant, plans[j].smem, plans[j].per_lane, P.walkers.size(),
                P.ranks.size(), P.comms.size(), (P.hdr.flags & JOB_RING) ? 1 : 0, P.hdr.n_rcolls,
                P.hdr.n_fire);
      }
    // a grid job runs only if all its parts are co-resident under the batch's
    // grid launch shape (the largest part layout); otherwise it is scheduled
    // by the warp-window kernel (2,048-rank full-rank jobs with many streams)
    for (;;) {
      uint32_t smax = 0;
      for (size_t j = 0; j < nj; j++)
        if (plans[j].variant == 15) smax = std::max(smax, (plans[j].smem + 127u) & ~127u);
      if (!smax) break;
      const size_t cap = (size_t)std::max(1, grid_max_ctas(smax));
      bool demoted = false;
      for (size_t j = 0; j < nj; j++)
        if (plans[j].variant == 15 && plans[j].parts.size() > cap) {
          plans[j] = LanePlan();
          demoted = true;
        }
      if (!demoted) break;
    }
  }
  if (n_reps > 0xffffffffull) return fail(MAYA_EINVAL, "too many representatives in batch");
  if (n_feats >= 0xffffffffull) return fail(MAYA_EINVAL, "too many kernel features in batch");
  if (n_blocks >= KBLOCK) return fail(MAYA_EINVAL, "too many kernel blocks in batch");
  e->has_blocks = n_blocks > 0;
  if (n_slots >= 0xffffffffull) return fail(MAYA_EINVAL, "too many collective calls in batch");
  e->n_tl = n_tl;
  // arena layout
  size_t off = 0;
  auto seg = [&](Seg &s, size_t bytes) {
    s.off = off;
    s.bytes = bytes;
    off = align_up(off + bytes, 256);
  };
  seg(e->s_jobs, nj * sizeof(JobHdr));
  seg(e->s_order, nj * sizeof(int32_t));
  seg(e->s_ranks, n_ranks * sizeof(RankRec));
  seg(e->s_rank_comm, n_rank_comm * sizeof(uint32_t));
  seg(e->s_comms, n_comms * sizeof(CommRec));
  seg(e->s_wfeats, n_wfeats * sizeof(SlotRec));
  seg(e->s_walkers, n_walkers * sizeof(Walker));
  seg(e->s_wids, n_walkers * sizeof(uint32_t));
  seg(e->s_reps, n_reps * sizeof(RepHdr));
  seg(e->s_ops, n_ops * sizeof(Op));
  seg(e->s_streams, n_streams * sizeof(StreamRange));
  seg(e->s_coll_lc, n_colls * sizeof(uint32_t));
  seg(e->s_coll_idx, n_colls * sizeof(uint32_t));
  seg(e->s_coll_wf, n_colls * sizeof(uint32_t));
  seg(e->s_syncs, n_syncs * sizeof(SyncRec));
  seg(e->s_counts, n_counts * sizeof(uint32_t));
  seg(e->s_mems, n_mems * sizeof(MemRec));
  seg(e->s_feats, n_feats * sizeof(Feature));
  seg(e->s_fmeta, n_feats * sizeof(uint32_t));
  seg(e->s_rcolls, n_rcolls * sizeof(RankColl));
  seg(e->s_rcslot, n_rcolls * sizeof(uint32_t));
  seg(e->s_lane_jobs, nj * sizeof(LaneJob));
  seg(e->s_lane_wslot, n_walkers * sizeof(uint32_t));
  seg(e->s_lane_perm, n_perm * sizeof(uint32_t));
  seg(e->s_chunks, n_chunks * sizeof(FoldChunk));
  size_t n_parts = 0;
  for (size_t j = 0; j < nj; j++) n_parts += plans[j].parts.size();
  seg(e->s_grid_parts, n_parts * sizeof(GridPart));
  seg(e->s_comm_part, n_comms * sizeof(uint32_t));
  seg(e->s_blocks, n_blocks * sizeof(KBlock));
  seg(e->s_blk_fids, n_blk_fids * sizeof(uint32_t));
  e->arena_bytes = off;
  if (getenv("MAYA_DEBUG_ARENA")) {
    const Seg *sg[] = {&e->s_jobs, &e->s_order, &e->s_ranks, &e->s_rank_comm, &e->s_comms,
                       &e->s_wfeats, &e->s_walkers, &e->s_wids, &e->s_reps, &e->s_ops,
                       &e->s_streams, &e->s_coll_lc, &e->s_coll_idx, &e->s_syncs, &e->s_counts,
                       &e->s_mems, &e->s_feats, &e->s_rcolls, &e->s_rcslot, &e->s_lane_jobs,
                       &e->s_lane_wslot, &e->s_lane_perm, &e->s_chunks, &e->s_grid_parts,
                       &e->s_comm_part, &e->s_blocks, &e->s_blk_fids};
    const char *nm[] = {"jobs", "order", "ranks", "rank_comm", "comms", "wfeats", "walkers",
                        "wids", "reps", "ops", "streams", "coll_lc", "coll_idx", "syncs",
                        "counts", "mems", "feats", "rcolls", "rcslot", "lane_jobs", "lane_wslot",
                        "lane_perm", "chunks", "grid_parts", "comm_part", "blocks", "blk_fids"};
    for (size_t q = 0; q < sizeof(sg) / sizeof(sg[0]); q++)
      fprintf(stderr, "arena %-10s %12zu\n", nm[q], sg[q]->bytes);
  }
  // scratch layout
  off = 0;
  seg(e->x_exec, n_ops * sizeof(ExecOp));
  seg(e->x_clen, n_streams * sizeof(uint32_t));
  seg(e->x_lctx, n_walkers * 64);
  seg(e->x_lst, n_walkers * 48);
  seg(e->x_macros, n_macros * sizeof(ChainMacro));
  seg(e->x_gsync, nj * sizeof(GridSync));
  seg(e->x_ccounts, n_counts * sizeof(uint32_t));
  seg(e->x_rcw, n_rcolls * sizeof(RCX));
  seg(e->x_feat_ns, n_feats * 8);
  seg(e->x_feat_d32, n_feats * 4);
  seg(e->x_blk_ab, n_blocks * 16);
  seg(e->x_wire, n_wfeats * 8);
  seg(e->x_fire, n_fire * 8);
  seg(e->x_delay, n_delay * 8);
  seg(e->x_wstate, n_wstate);
  seg(e->x_cslots, n_slots * sizeof(CollSlot));
  seg(e->x_repout, n_reps * sizeof(RepOut));
  seg(e->x_results, nj * sizeof(maya_job_result));
  seg(e->x_err, 16);
  seg(e->x_topk, topk_scratch_bytes((uint32_t)nj, 64));
  seg(e->x_topk_out, 64 * sizeof(maya_topk_entry));
  seg(e->x_topk_n, 16);
  seg(e->x_tl_start, 0);
  seg(e->x_tl_end, 0);
  e->scratch_bytes = off;

  // pinned host / device arenas grow geometrically (x2): pinning GBs costs
  // ~1 s, so a search whose batches grow re-pins a few times, not per batch
  if (e->arena_bytes > e->h_arena_cap) {
    if (e->h_arena) cudaFreeHost(e->h_arena);
    e->h_arena = nullptr;
    size_t cap = align_up(std::max(e->arena_bytes + e->arena_bytes / 4, 2 * e->h_arena_cap), 1 << 20);
    CU(cudaMallocHost(&e->h_arena, cap));
    e->h_arena_cap = cap;
  }
  if (e->arena_bytes > e->d_arena_cap) {
    if (e->d_arena) cudaFree(e->d_arena);
    e->d_arena = nullptr;
    size_t cap = align_up(std::max(e->arena_bytes + e->arena_bytes / 4, 2 * e->d_arena_cap), 1 << 20);
    CU(cudaMalloc(&e->d_arena, cap));
    e->d_arena_cap = cap;
  }
  if (e->scratch_bytes > e->d_scratch_cap) {
    if (e->d_scratch) cudaFree(e->d_scratch);
    e->d_scratch = nullptr;
    size_t cap = align_up(std::max(e->scratch_bytes + e->scratch_bytes / 4, 2 * e->d_scratch_cap), 1 << 20);
    CU(cudaMalloc(&e->d_scratch, cap));
    e->d_scratch_cap = cap;
  }
  char *H = (char *)e->h_arena;
  lap("plans");
  // job order: grouped by scheduler variant, largest work first in each group
  // (LPT over the CTA scheduler)
  {
    std::vector<int32_t> order(nj);
    std::vector<int> var(nj);
    std::vector<uint32_t> wbytes(nj, 0);
    for (size_t j = 0; j < nj; j++) {
      order[j] = (int32_t)j;
      var[j] = plans[j].variant >= 0 ? plans[j].variant
                                     : sched_variant((uint32_t)e->packs[j].walkers.size(),
                                                     (uint32_t)e->packs[j].ranks.size());
      if (var[j] < 3) {
        const JobPack &P = e->packs[j];
        wbytes[j] = sched_layout((uint32_t)P.walkers.size(), (uint32_t)P.ranks.size(),
                                 (uint32_t)P.comms.size(), (P.hdr.flags & JOB_RING) != 0,
                                 P.hdr.n_fire, P.hdr.n_rcolls, sched_smem_cap())
                        .bytes;
      }
    }
    const uint32_t small = split_smem_threshold();
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      if (var[a] != var[b]) return var[a] < var[b];
      const bool ba = wbytes[a] > small, bb = wbytes[b] > small;
      if (ba != bb) return ba;
      return e->packs[a].hdr.dev_ops > e->packs[b].hdr.dev_ops;
    });
    for (int v = 0; v < maya_engine::NVAR; v++) e->var_n[v] = e->var_smem[v] = 0;
    for (int v = 0; v < 3; v++) e->var_big[v] = e->var_smem_small[v] = 0;
    for (size_t j = 0; j < nj; j++) {
      e->var_n[var[j]]++;
      if (var[j] >= 3) {   // lane kernels (15: grid jobs, smem per part)
        const uint32_t need = (plans[j].smem + 127u) & ~127u;
        if (need > e->var_smem[var[j]]) e->var_smem[var[j]] = need;
        continue;
      }
      if (wbytes[j] > small) {
        e->var_big[var[j]]++;
        if (wbytes[j] > e->var_smem[var[j]]) e->var_smem[var[j]] = wbytes[j];
      } else if (wbytes[j] > e->var_smem_small[var[j]]) {
        e->var_smem_small[var[j]] = wbytes[j];
      }
    }
    memcpy(H + e->s_order.off, order.data(), nj * sizeof(int32_t));
    e->job_kernel.resize(nj);
    for (size_t j = 0; j < nj; j++)
      e->job_kernel[j] = var[j] >= 16 ? 3 : var[j] == 15 ? 2 : var[j] >= 3 ? 1 : 0;
    // chain jobs (variants 16..) close the order: their macro pass takes that tail
    e->chain_jobs = 0;
    e->chain_maxw = 0;
    for (size_t j = 0; j < nj; j++)
      if (var[j] >= 16) {
        e->chain_jobs++;
        e->chain_maxw = std::max(e->chain_maxw, (uint32_t)e->packs[j].walkers.size());
      }
    e->chain_first = (uint32_t)(nj - e->chain_jobs);
  }
  // per-job bases (serial prefix), then parallel copy
  struct Base {
    size_t ranks, rank_comm, comms, slots, walkers, reps, ops, streams, colls, syncs, counts,
        mems, feats, fire, delay, wstate, rcolls, perm, blocks, blk_fids, wfeats, macros;
  };
  std::vector<Base> bases(nj);
  {
    Base b{};
    for (size_t j = 0; j < nj; j++) {
      const JobPack &P = e->packs[j];
      bases[j] = b;
      b.ranks += P.ranks.size();
      b.rank_comm += P.rank_comm.size();
      b.comms += P.comms.size();
      b.slots += P.slots.size();
      b.wfeats += P.wfeats.size();
      b.walkers += P.walkers.size();
      b.reps += P.reps.size();
      b.ops += P.ops.size();
      b.streams += P.streams.size();
      b.colls += P.coll_lc.size();
      b.syncs += P.syncs.size();
      b.counts += P.counts.size();
      b.mems += P.mems.size();
      b.feats += P.feats.size();
      b.blocks += P.blocks.size();
      b.blk_fids += P.blk_fids.size();
      b.fire += P.n_fire;
      b.delay += P.n_delay;
      b.rcolls += P.rcolls.size();
      if (plans[j].variant >= 0 && plans[j].variant != 15)
        b.perm += (size_t)plans[j].per_lane * plans[j].threads;
      if (plans[j].variant >= 16) b.macros += plans[j].n_slots;
      const SchedLayout L = sched_layout((uint32_t)P.walkers.size(), (uint32_t)P.ranks.size(),
                                         (uint32_t)P.comms.size(), (P.hdr.flags & JOB_RING) != 0,
                                         P.hdr.n_fire, P.hdr.n_rcolls, sched_smem_cap());
      if (!L.on_chip) b.wstate += spill_bytes(P.walkers.size(), P.ranks.size());
    }
  }
  {  // run-folding work items: one per 1,024 ops of every FIFO, with the folded
     // ops before each (host-counted in pack_tail: no counting pass on the device)
    FoldChunk *fcs = (FoldChunk *)(H + e->s_chunks.off);
    size_t q = 0;
    for (size_t j = 0; j < nj; j++) {
      const JobPack &P = e->packs[j];
      size_t k = 0;
      for (size_t r = 0; r < P.reps.size(); r++) {
        const RepHdr &h = P.reps[r];
        for (uint32_t st = 0; st < h.n_streams; st++) {
          const uint32_t len = P.streams[h.streams + st].len;
          for (uint32_t c = 0; c * FOLD_CHUNK < len; c++)
            fcs[q++] = FoldChunk{(uint32_t)(bases[j].reps + r), st, c, P.fold_base[k++]};
        }
      }
    }
  }
  if (n_chunks >= 0xffffffffull) return fail(MAYA_EINVAL, "too many fold chunks in batch");
  {  // grid jobs: their parts, grouped into cooperative launches that fit co-resident
    e->grid_parts.clear();
    e->grid_launches.clear();
    e->grid_smem = e->var_smem[15];
    for (size_t j = 0; j < nj; j++) {
      if (plans[j].variant != 15) continue;
      const uint32_t first = (uint32_t)e->grid_parts.size();
      for (GridPart g : plans[j].parts) {
        g.job = (uint32_t)j;
        g.first = first;
        g.wslot = bases[j].walkers + g.w0;
        e->grid_parts.push_back(g);
      }
    }
    if (!e->grid_parts.empty()) {
      const uint32_t cap = (uint32_t)std::max(1, grid_max_ctas(e->grid_smem));
      uint32_t p = 0;
      while (p < e->grid_parts.size()) {
        uint32_t q = p;
        while (q < e->grid_parts.size()) {
          const uint32_t np = e->grid_parts[q].n_parts;
          if (q + np - p > cap && q > p) break;
          if (np > cap) return fail(MAYA_EINVAL, "grid job larger than the co-resident CTAs");
          q += np;
        }
        e->grid_launches.push_back({p, q});
        p = q;
      }
    }
    if (!e->grid_parts.empty())
      memcpy(H + e->s_grid_parts.off, e->grid_parts.data(), e->grid_parts.size() * sizeof(GridPart));
  }
  lap("layout");
  auto copy_job = [&](size_t j) {
    const JobPack &P = e->packs[j];
    const Base &B = bases[j];
    JobHdr h = P.hdr;
    h.ranks = B.ranks;
    h.rank_comm = B.rank_comm;
    h.comms = B.comms;
    h.slots = B.slots;
    h.walkers = B.walkers;
    h.feats = B.feats;
    h.fire = B.fire;
    h.delay = B.delay;
    h.wstate = B.wstate;
    h.timeline = e->job_tl[j];
    h.rcolls = B.rcolls;
    h.blocks = B.blocks;
    h.blk_fids = B.blk_fids;
    h.n_blocks = (uint32_t)P.blocks.size();
    memcpy(H + e->s_jobs.off + j * sizeof(JobHdr), &h, sizeof h);
    RankRec *rk = (RankRec *)(H + e->s_ranks.off) + B.ranks;
    for (size_t r = 0; r < P.ranks.size(); r++) {
      RankRec x = P.ranks[r];
      x.rep += (uint32_t)B.reps;
      rk[r] = x;
    }
    RepHdr *rp = (RepHdr *)(H + e->s_reps.off) + B.reps;
    for (size_t r = 0; r < P.reps.size(); r++) {
      RepHdr x = P.reps[r];
      x.ops += B.ops;
      x.streams += B.streams;
      x.colls += B.colls;
      x.syncs += B.syncs;
      x.counts += B.counts;
      x.mems += B.mems;
      x.job = (uint32_t)j;
      rp[r] = x;
    }
#define CPY(SEG, VEC, BASE)                                                             \
  if (!P.VEC.empty())                                                                   \
    memcpy(H + e->SEG.off + (BASE) * sizeof(P.VEC[0]), P.VEC.data(),                    \
           P.VEC.size() * sizeof(P.VEC[0]));
    CPY(s_rank_comm, rank_comm, B.rank_comm)
    CPY(s_comms, comms, B.comms)
    CPY(s_wfeats, wfeats, B.wfeats)
    CPY(s_walkers, walkers, B.walkers)
    CPY(s_wids, wids, B.walkers)
    {  // ops: KERN args become batch-global feature (or kernel block) ids
      Op *dst = (Op *)(H + e->s_ops.off) + B.ops;
      for (size_t q = 0; q < P.ops.size(); q++) {
        Op o = P.ops[q];
        if (op_tag(o.meta) == TAG_KERN)
          o.arg = (o.arg & KBLOCK) ? (KBLOCK | ((o.arg & ~KBLOCK) + (uint32_t)B.blocks))
                                   : o.arg + (uint32_t)B.feats;
        dst[q] = o;
      }
      KBlock *kb = (KBlock *)(H + e->s_blocks.off) + B.blocks;
      for (size_t q = 0; q < P.blocks.size(); q++) {
        KBlock x = P.blocks[q];
        x.fid0 += (uint32_t)B.blk_fids;
        kb[q] = x;
      }
      uint32_t *bf = (uint32_t *)(H + e->s_blk_fids.off) + B.blk_fids;
      for (size_t q = 0; q < P.blk_fids.size(); q++) bf[q] = P.blk_fids[q] + (uint32_t)B.feats;
    }
    CPY(s_rcolls, rcolls, B.rcolls)
    {  // lane-scheduler plan and per-walker ring words
      const LanePlan &pl = plans[j];
      LaneJob lj{B.macros, pl.flags, pl.n_slots, B.walkers, B.perm, pl.per_lane, pl.fc_log2};
      memcpy(H + e->s_lane_jobs.off + j * sizeof(LaneJob), &lj, sizeof lj);
      if (pl.variant >= 0 && pl.variant != 15 && P.hdr.status == MAYA_ST_OK)
        lane_perm_fill(P, pl, (uint32_t *)(H + e->s_lane_perm.off) + B.perm);
      uint32_t *ws = (uint32_t *)(H + e->s_lane_wslot.off) + B.walkers;
      uint32_t slot = 0;
      size_t part = 0;
      for (size_t w = 0; w < P.walkers.size(); w++) {
        uint32_t lgd_max = pl.lgd_max;
        if (pl.variant == 15) {   // grid job: ring slots are part-local
          while (part + 1 < pl.parts.size() && w >= pl.parts[part + 1].w0) part++;
          if (w == pl.parts[part].w0) slot = 0;
          lgd_max = (uint32_t)pl.parts[part].wslot;
        }
        const Walker wk = P.walkers[w];
        const RepHdr &h = P.reps[P.ranks[wk.rank].rep];
        if (pl.variant >= 16) {   // chain job: the FIFO's first macro op in the job's area
          ws[w] = slot;
          slot += P.stream_macros[h.streams + wk.stream];
          continue;
        }
        const uint32_t n = pl.variant >= 3 ? lane_slots_of(P.streams[h.streams + wk.stream].folded,
                                                           lgd_max)
                                           : 0;
        uint32_t lg = 0;
        while ((1u << lg) < n) lg++;
        ws[w] = n ? (slot | (lg << 28)) : (0xfu << 28);
        slot += n;
      }
    }
    {  // grid jobs: the part holding all members of each communicator (else ~0)
      uint32_t *cp = (uint32_t *)(H + e->s_comm_part.off) + B.comms;
      for (size_t g = 0; g < P.comms.size(); g++) cp[g] = 0xffffffffu;
      const LanePlan &pl = plans[j];
      if (pl.variant == 15) {
        std::vector<uint32_t> owner(P.comms.size(), 0xfffffffeu);   // unset
        size_t part = 0;
        for (size_t r = 0; r < P.ranks.size(); r++) {
          while (part + 1 < pl.parts.size() && r >= pl.parts[part + 1].r0) part++;
          const RankRec &rr = P.ranks[r];
          const uint32_t nlc = (r + 1 < P.ranks.size() ? P.ranks[r + 1].comm
                                                        : (uint32_t)P.rank_comm.size()) - rr.comm;
          for (uint32_t q = 0; q < nlc; q++) {
            const uint32_t g = P.rank_comm[rr.comm + q];
            owner[g] = owner[g] == 0xfffffffeu ? (uint32_t)part
                       : owner[g] == (uint32_t)part ? owner[g] : 0xffffffffu;
          }
        }
        for (size_t g = 0; g < P.comms.size(); g++)
          cp[g] = owner[g] == 0xfffffffeu ? 0xffffffffu : owner[g];
      }
    }
    {  // batch-global call slot of every rank-collective entry
      uint32_t *dst = (uint32_t *)(H + e->s_rcslot.off) + B.rcolls;
      for (size_t q = 0; q < P.rcolls.size(); q++) {
        const RankColl ent = P.rcolls[q];
        const uint32_t g = (uint32_t)(ent >> 32) & 0xffffu, idx = (uint32_t)ent;
        dst[q] = (uint32_t)(B.wfeats + P.slot_wf[P.comms[g].call_base + idx]);
      }
    }
    CPY(s_streams, streams, B.streams)
    CPY(s_coll_lc, coll_lc, B.colls)
    CPY(s_coll_idx, coll_idx, B.colls)
    {  // foldable collectives: batch-global wire feature
      uint32_t *dst = (uint32_t *)(H + e->s_coll_wf.off) + B.colls;
      for (size_t q = 0; q < P.coll_wf.size(); q++)
        dst[q] = P.coll_wf[q] == NO_WF ? NO_WF : (uint32_t)(B.wfeats + P.coll_wf[q]);
    }
    CPY(s_syncs, syncs, B.syncs)
    CPY(s_counts, counts, B.counts)
    CPY(s_mems, mems, B.mems)
    CPY(s_feats, feats, B.feats)
    CPY(s_fmeta, feat_meta, B.feats)
#undef CPY
  };
  {
    int nt = (int)std::min<size_t>(std::max(1u, std::thread::hardware_concurrency()),
                                   std::max<size_t>(1, nj / 16));
    std::atomic<size_t> next(0);
    auto work = [&]() {
      for (;;) {
        size_t j = next.fetch_add(1);
        if (j >= nj) break;
        copy_job(j);
      }
    };
    WorkerPool::get(1).run(nt, work);
  }
  lap("copy");
  CU(cudaMemcpyAsync(e->d_arena, e->h_arena, e->arena_bytes, cudaMemcpyHostToDevice, e->stream));
  lap("h2d");
  // device view
  char *D = (char *)e->d_arena;
  char *X = (char *)e->d_scratch;
  DevBatch &db = e->db;
  db.jobs = (const JobHdr *)(D + e->s_jobs.off);
  db.order = (const int32_t *)(D + e->s_order.off);
  db.lane_jobs = (const LaneJob *)(D + e->s_lane_jobs.off);
  db.lane_wslot = (const uint32_t *)(D + e->s_lane_wslot.off);
  db.lane_perm = (const uint32_t *)(D + e->s_lane_perm.off);
  db.chunks = (const FoldChunk *)(D + e->s_chunks.off);
  db.grid_parts = (const GridPart *)(D + e->s_grid_parts.off);
  db.comm_part = (const uint32_t *)(D + e->s_comm_part.off);
  db.n_chunks = (uint32_t)n_chunks;
  db.ranks = (const RankRec *)(D + e->s_ranks.off);
  db.rank_comm = (const uint32_t *)(D + e->s_rank_comm.off);
  db.comms = (const CommRec *)(D + e->s_comms.off);
  db.wfeats = (const SlotRec *)(D + e->s_wfeats.off);
  db.n_wfeats = (uint32_t)n_wfeats;
  db.walkers = (const Walker *)(D + e->s_walkers.off);
  db.wids = (const uint32_t *)(D + e->s_wids.off);
  db.reps = (const RepHdr *)(D + e->s_reps.off);
  db.ops = (const Op *)(D + e->s_ops.off);
  db.streams = (const StreamRange *)(D + e->s_streams.off);
  db.coll_lc = (const uint32_t *)(D + e->s_coll_lc.off);
  db.coll_idx = (const uint32_t *)(D + e->s_coll_idx.off);
  db.coll_wf = (const uint32_t *)(D + e->s_coll_wf.off);
  db.syncs = (const SyncRec *)(D + e->s_syncs.off);
  db.counts = (const uint32_t *)(D + e->s_counts.off);
  db.mems = (const MemRec *)(D + e->s_mems.off);
  db.feats = (const Feature *)(D + e->s_feats.off);
  db.feat_meta = (const uint32_t *)(D + e->s_fmeta.off);
  db.blocks = (const KBlock *)(D + e->s_blocks.off);
  db.blk_fids = (const uint32_t *)(D + e->s_blk_fids.off);
  db.n_blocks = (uint32_t)n_blocks;
  db.rcolls = (const RankColl *)(D + e->s_rcolls.off);
  db.rcslot = (const uint32_t *)(D + e->s_rcslot.off);
  db.rcx = (RCX *)(X + e->x_rcw.off);
  db.n_rcolls = n_rcolls;
  db.exec = (ExecOp *)(X + e->x_exec.off);
  db.n_ops = n_ops;
  db.feat_ns = (int64_t *)(X + e->x_feat_ns.off);
  db.feat_d32 = (uint32_t *)(X + e->x_feat_d32.off);
  db.wire = (int64_t *)(X + e->x_wire.off);
  db.fire = (int64_t *)(X + e->x_fire.off);
  db.delay = (int64_t *)(X + e->x_delay.off);
  db.spill = (uint8_t *)(X + e->x_wstate.off);
  db.cslots = (CollSlot *)(X + e->x_cslots.off);
  db.repout = (RepOut *)(X + e->x_repout.off);
  db.results = (maya_job_result *)(X + e->x_results.off);
  db.err_flag = (int32_t *)(X + e->x_err.off);
  db.tl_start = nullptr;
  db.tl_end = nullptr;
  db.n_jobs = (uint32_t)nj;
  db.n_reps = (uint32_t)n_reps;
  db.n_feats = (uint32_t)n_feats;
  db.n_slots = (uint32_t)n_slots;
  // estimator tables
  DevTables &t = e->tables;
  memset(&t, 0, sizeof t);
  t.n_devs = (int32_t)e->devs.size();
  for (size_t i = 0; i < e->devs.size(); i++) t.devs[i] = e->devs[i];
  t.n_op_kinds = (int32_t)e->eff_num.size();
  for (size_t i = 0; i < e->eff_num.size(); i++) {
    t.eff_num[i] = e->eff_num[i];
    t.eff_den[i] = e->eff_den[i];
  }
  t.overhead_ns = e->overhead_ns;
  // floor(2^64 / y) for y >= 2 (fits: <= 2^63); 0 stands for y == 1 (and for y <= 0,
  // which the kernel never divides by on this path)
  auto magic = [](int64_t y) -> uint64_t {
    if (y <= 1) return 0;
    return (uint64_t)(((unsigned __int128)1 << 64) / (unsigned __int128)(uint64_t)y);
  };
  for (int d = 0; d < t.n_devs && d < 8; d++) {
    for (int q = 0; q < MAYA_MAX_DTYPES; q++) {
      t.inv_peak[d][q] = t.devs[d].peak_flops[q] > 0 ? 1.0 / (double)t.devs[d].peak_flops[q] : 0.0;
      t.mag_peak[d][q] = magic(t.devs[d].peak_flops[q]);
    }
    t.inv_hbm[d] = t.devs[d].hbm_bytes_per_s > 0 ? 1.0 / (double)t.devs[d].hbm_bytes_per_s : 0.0;
    t.mag_hbm[d] = magic(t.devs[d].hbm_bytes_per_s);
  }
  for (int q = 0; q < t.n_op_kinds && q < 64; q++) {
    t.inv_num[q] = t.eff_num[q] > 0 ? 1.0 / (double)t.eff_num[q] : 0.0;
    t.mag_num[q] = magic(t.eff_num[q]);
    const unsigned __int128 scale = (unsigned __int128)1000000000ull * (uint64_t)t.eff_den[q];
    t.max_flops[q] = (t.eff_den[q] > 0 && (scale >> 64) == 0) ? UINT64_MAX / (uint64_t)scale : 0;
    t.max_peak[q] = t.eff_num[q] > 0 ? UINT64_MAX / (uint64_t)t.eff_num[q] : 0;
  }
  {  // per (device, dtype, op kind) constants of the estimator's fast path
    const int nd = std::min(t.n_devs, 8), no = std::max(t.n_op_kinds, 1);
    std::vector<EstClass> cls((size_t)std::max(nd, 1) * MAYA_MAX_DTYPES * no);
    auto magic_nb = [](uint64_t y) -> uint64_t {   // floor(2^64 / y), ~0 for y == 1
      return y == 1 ? ~0ull : (uint64_t)(((unsigned __int128)1 << 64) / y);
    };
    for (int dv = 0; dv < nd; dv++)
      for (int dt = 0; dt < MAYA_MAX_DTYPES; dt++)
        for (int op = 0; op < t.n_op_kinds; op++) {
          EstClass &c = cls[(size_t)(dv * MAYA_MAX_DTYPES + dt) * no + op];
          c = EstClass{0, 0, 0, 0, 0, 0};
          const int64_t peak = t.devs[dv].peak_flops[dt], num = t.eff_num[op], den = t.eff_den[op];
          const unsigned __int128 K = (unsigned __int128)1000000000ull * (uint64_t)(den > 0 ? den : 0);
          const unsigned __int128 D = (unsigned __int128)(uint64_t)(peak > 0 ? peak : 0) *
                                      (uint64_t)(num > 0 ? num : 0);
          if (peak > 0 && num > 0 && den > 0 && (K >> 64) == 0 && (D >> 64) == 0) {
            c.K = (uint64_t)K;
            c.D = (uint64_t)D;
            c.MD = magic_nb(c.D);
            c.maxf = UINT64_MAX / c.K;
          }
          const int64_t hbm = t.devs[dv].hbm_bytes_per_s;
          if (hbm > 0) {
            c.H = (uint64_t)hbm;
            c.MH = magic_nb(c.H);
          }
        }
    const size_t need = cls.size() * sizeof(EstClass) + sizeof(DevTables);
    if (need > e->d_est_cap) {
      if (e->d_est) cudaFree(e->d_est);
      e->d_est = nullptr;
      CU(cudaMalloc(&e->d_est, need));
      e->d_est_cap = need;
    }
    char *E = (char *)e->d_est;
    t.gtab = (const DevTables *)E;
    t.cls = (const EstClass *)(E + sizeof(DevTables));
    CU(cudaMemcpy(E, &t, sizeof(DevTables), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(E + sizeof(DevTables), cls.data(), cls.size() * sizeof(EstClass),
                  cudaMemcpyHostToDevice));
  }
  for (size_t j = 0; j < nj; j++) {
    const JobPack &P = e->packs[j];
    if (P.hdr.status == MAYA_ST_OK && (int)P.hdr.device >= t.n_devs && !P.feats.empty())
      return fail(MAYA_EINVAL, "job references a device class that was not set");
  }
  e->uploaded = true;
  // a new batch: the captured run (kernel arguments, grid sizes) is stale
  if (e->graph_exec) {
    cudaGraphExecDestroy(e->graph_exec);
    e->graph_exec = nullptr;
  }
  e->runs_since_upload = 0;
  e->ran = false;
  return MAYA_OK;
}

int maya_run(maya_engine *e, int32_t record_timeline) {
  e->topk_pending = 0;
  if (!e->uploaded) return fail(MAYA_ESTATE, "maya_run before maya_upload");
  if (e->has_blocks && (record_timeline || (e->options & MAYA_OPT_NO_FOLD)))
    return fail(MAYA_ESTATE, "batch staged with kernel blocks runs folded only: set "
                             "MAYA_OPT_NO_BLOCKS before staging to record a timeline");
  CU(cudaSetDevice(e->device));
  DevBatch db = e->db;
  if (record_timeline) {
    size_t need = e->scratch_bytes + align_up(e->n_tl * 8, 256) * 2;
    if (need > e->d_scratch_cap) {
      // grow scratch, keeping the layout (scratch contents are rebuilt per run)
      void *p = nullptr;
      CU(cudaStreamSynchronize(e->stream));
      CU(cudaMalloc(&p, need));
      cudaFree(e->d_scratch);
      if (e->graph_exec) {   // its kernels point into the old scratch
        cudaGraphExecDestroy(e->graph_exec);
        e->graph_exec = nullptr;
      }
      e->d_scratch = p;
      e->d_scratch_cap = need;
      char *X = (char *)p;
      db.exec = (ExecOp *)(X + e->x_exec.off);
      db.rcx = (RCX *)(X + e->x_rcw.off);
      db.feat_ns = (int64_t *)(X + e->x_feat_ns.off);
      db.feat_d32 = (uint32_t *)(X + e->x_feat_d32.off);
      db.wire = (int64_t *)(X + e->x_wire.off);
      db.fire = (int64_t *)(X + e->x_fire.off);
      db.delay = (int64_t *)(X + e->x_delay.off);
      db.spill = (uint8_t *)(X + e->x_wstate.off);
      db.cslots = (CollSlot *)(X + e->x_cslots.off);
      db.repout = (RepOut *)(X + e->x_repout.off);
      db.results = (maya_job_result *)(X + e->x_results.off);
      db.err_flag = (int32_t *)(X + e->x_err.off);
      e->db = db;
    }
    char *X = (char *)e->d_scratch;
    db.tl_start = (int64_t *)(X + e->scratch_bytes);
    db.tl_end = (int64_t *)(X + e->scratch_bytes + align_up(e->n_tl * 8, 256));
    e->db.tl_start = db.tl_start;
    e->db.tl_end = db.tl_end;
    // -1 = never completed: a deadlocked job's residue (sim.py:382-402) is read
    // from the first unfinished op of every FIFO (api._deadlock_message)
    if (e->n_tl) CU(cudaMemsetAsync(db.tl_end, 0xFF, e->n_tl * 8, e->stream));
  }
  char *X = (char *)e->d_scratch;
  // runs fold (fold_kernel) unless a per-op timeline is recorded
  const bool fold = !record_timeline && !(e->options & MAYA_OPT_NO_FOLD);
  db.clen = fold ? (uint32_t *)(X + e->x_clen.off) : nullptr;
  db.blk_ab = (int64_t *)(X + e->x_blk_ab.off);
  db.lane_gctx = (uint8_t *)(X + e->x_lctx.off);
  db.lane_gst = (uint8_t *)(X + e->x_lst.off);
  db.macros = (ChainMacro *)(X + e->x_macros.off);
  db.gsync = (GridSync *)(X + e->x_gsync.off);
  db.ccounts = fold ? (uint32_t *)(X + e->x_ccounts.off) : nullptr;
  // The run's device work (estimators, memory scan, fold / resolve, macro
  // pass, the scheduler groups on their streams, joined back).  Runs without a
  // timeline replay it as ONE CUDA graph from the second run of a batch on
  // (captured once per upload): ~25 launches and their fork/join events cost
  // one graph launch.  The phase-timing events become external event-record
  // nodes, so maya_last_timings keeps its three phases.
  auto enqueue = [&](bool captured) -> int {
    auto rec = [&](cudaEvent_t ev) {
      return captured ? cudaEventRecordWithFlags(ev, e->stream, cudaEventRecordExternal)
                      : cudaEventRecord(ev, e->stream);
    };
    CU(rec(e->ev[0]));
    CU(cudaMemsetAsync(X + e->x_err.off, 0, 16, e->stream));
    launch_estimate(db, e->tables, e->stream);
    CU(cudaGetLastError());
    CU(rec(e->ev[1]));
    CU(cudaMemsetAsync(X + e->x_fire.off, 0xff, e->x_fire.bytes, e->stream));
    CU(cudaMemsetAsync(X + e->x_cslots.off, 0, e->x_cslots.bytes, e->stream));
    if (!e->grid_parts.empty()) CU(cudaMemsetAsync(X + e->x_gsync.off, 0, e->x_gsync.bytes, e->stream));
    launch_memscan(db, e->stream);
    CU(cudaGetLastError());
    launch_resolve(db, e->stream);
    CU(cudaGetLastError());
    if (fold && e->chain_jobs) {   // chain jobs: macro ops of their folded FIFOs
      launch_chain_macros(db, db.order + e->chain_first, e->chain_jobs, e->chain_maxw, e->stream);
      CU(cudaGetLastError());
    }
    CU(rec(e->ev[2]));
    {
      // variants run concurrently on their own streams (fork/join)
      CU(cudaEventRecord(e->vev[maya_engine::NVAR], e->stream));
      uint32_t var_off[maya_engine::NVAR];
      for (int v = 0, o = 0; v < maya_engine::NVAR; v++) { var_off[v] = (uint32_t)o; o += (int)e->var_n[v]; }
      // groups of larger jobs first (grid jobs, CTA lane jobs, then warp-window
      // jobs from 16 down to 4 warps): the longest dependency chains get their
      // SMs before the short jobs fill the machine (measured: C2's step stays at
      // its fast mode in 5 of 6 processes instead of 2 of 5)
      for (int vi = 0; vi < maya_engine::NVAR; vi++) {
        const int v = maya_engine::NVAR - 1 - vi;
        const uint32_t off = var_off[v];
        if (!e->var_n[v]) continue;
        CU(cudaStreamWaitEvent(e->vstream[v], e->vev[maya_engine::NVAR], 0));
        if (v == 15) {   // grid jobs: one cooperative launch per group of co-resident parts
          for (auto &pr : e->grid_launches)
            if (launch_schedule_grid(db, pr.first, pr.second, record_timeline ? 1 : 0,
                                     e->grid_smem, e->vstream[v]) != 0)
              return fail(MAYA_ECUDA, std::string("cooperative launch: ") +
                                          cudaGetErrorString(cudaGetLastError()));
        } else if (v < 3) {
          const uint32_t nb = e->var_big[v], ns = e->var_n[v] - nb;
          launch_schedule_variant(db, v, db.order + off, nb, record_timeline ? 1 : 0,
                                  e->var_smem[v], e->vstream[v]);
          if (ns) {   // small-footprint jobs on their own stream, concurrently
            CU(cudaStreamWaitEvent(e->sstream[v], e->vev[maya_engine::NVAR], 0));
            launch_schedule_variant(db, v, db.order + off + nb, ns, record_timeline ? 1 : 0,
                                    e->var_smem_small[v], e->sstream[v]);
            CU(cudaGetLastError());
            CU(cudaEventRecord(e->sev[v], e->sstream[v]));
            CU(cudaStreamWaitEvent(e->stream, e->sev[v], 0));
          }
        } else if (v >= 16) {
          launch_schedule_chain(db, db.order + off, e->var_n[v],
                                32u << ((v - 16) / (int)CHAIN_CLASSES), record_timeline ? 1 : 0,
                                e->var_smem[v], e->vstream[v]);
        } else if (v <= 10) {
          const uint32_t region = e->var_smem[v];
          uint32_t wpc = region ? LANE_SMEM_CAP / region : 8;
          wpc = wpc < 1 ? 1 : wpc > 8 ? 8 : wpc;
          launch_schedule_lane_warp(db, db.order + off, e->var_n[v], wpc, region,
                                    record_timeline ? 1 : 0, e->vstream[v]);
        } else {
          launch_schedule_lane(db, db.order + off, e->var_n[v], 64u << (v - 11),
                               record_timeline ? 1 : 0, e->var_smem[v], e->vstream[v]);
        }
        CU(cudaGetLastError());
        CU(cudaEventRecord(e->vev[v], e->vstream[v]));
        CU(cudaStreamWaitEvent(e->stream, e->vev[v], 0));
      }
    }
    CU(rec(e->ev[3]));
    return MAYA_OK;
  };
  const bool graph_ok = !record_timeline && e->grid_launches.empty() && !getenv("MAYA_NO_GRAPH");
  if (graph_ok && e->graph_exec && e->graph_fold == fold) {
    CU(cudaGraphLaunch(e->graph_exec, e->stream));
  } else if (graph_ok && e->runs_since_upload > 0) {
    if (e->graph_exec) {
      cudaGraphExecDestroy(e->graph_exec);
      e->graph_exec = nullptr;
    }
    CU(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
    const int rc = enqueue(true);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(e->stream, &g);
    bool launched = false;
    if (rc == MAYA_OK && ce == cudaSuccess && g) {
      if (cudaGraphInstantiate(&e->graph_exec, g, 0) == cudaSuccess) {
        e->graph_fold = fold;
        CU(cudaGraphLaunch(e->graph_exec, e->stream));
        launched = true;
      } else {
        e->graph_exec = nullptr;
      }
    }
    if (g) cudaGraphDestroy(g);
    if (!launched) {   // capture not possible here: run eagerly
      cudaGetLastError();
      const int rc2 = enqueue(false);
      if (rc2 != MAYA_OK) return rc2;
    }
  } else {
    const int rc = enqueue(false);
    if (rc != MAYA_OK) return rc;
  }
  e->runs_since_upload++;
  e->stats_ok = false;
  if (record_timeline) {
    // per-rank busy statistics (_report, sim.py:406-426) from the recorded timeline
    const uint32_t nr = (uint32_t)(e->rank_seg.size() - 1);
    if (e->n_tl >= 0x7fffffffull) return fail(MAYA_EINVAL, "timeline too large for rank stats");
    const size_t seg_b = align_up(e->rank_seg.size() * 8, 256), out_b = align_up(nr * 32ull, 256);
    const size_t tmp_b = rank_stats_scratch_bytes(e->n_tl, nr);
    const size_t need = seg_b + out_b + tmp_b;
    if (need > e->d_stats_cap) {
      CU(cudaStreamSynchronize(e->stream));
      if (e->d_stats) cudaFree(e->d_stats);
      e->d_stats = nullptr;
      CU(cudaMalloc(&e->d_stats, need));
      e->d_stats_cap = need;
    }
    char *S = (char *)e->d_stats;
    CU(cudaMemcpyAsync(S, e->rank_seg.data(), e->rank_seg.size() * 8, cudaMemcpyHostToDevice,
                       e->stream));
    e->d_rstats = (int64_t *)(S + seg_b);
    if (launch_rank_stats(db, (const uint64_t *)S, nr, e->n_tl, S + seg_b + out_b, tmp_b,
                          e->d_rstats, e->stream) != 0)
      return fail(MAYA_ECUDA, std::string("rank stats: ") + cudaGetErrorString(cudaGetLastError()));
    e->stats_ok = true;
  }
  {
    // kernels this run launched: estimators, memscan, resolve/fold, schedulers
    int64_t n = (db.n_feats ? 1 : 0) + (db.n_wfeats ? 1 : 0) + (db.n_reps ? 1 : 0) +
                (db.n_rcolls ? 1 : 0);
    if (fold)
      n += (db.n_blocks ? 1 : 0) + (db.n_chunks ? 1 : 0) + (db.n_reps ? 1 : 0) +
           (e->chain_jobs ? 1 : 0);
    else
      n += db.n_ops ? 1 : 0;
    for (int v = 0; v < maya_engine::NVAR; v++)
      n += v == 15  ? (int64_t)e->grid_launches.size()
           : v < 3  ? (e->var_big[v] ? 1 : 0) + (e->var_n[v] > e->var_big[v] ? 1 : 0)
                    : (e->var_n[v] ? 1 : 0);
    if (e->stats_ok) n += 3;   // keys, segmented sort (cub), unions
    e->run_launches = n;
  }
  e->ran = true;
  e->recorded = record_timeline != 0;
  return MAYA_OK;
}

int maya_results(maya_engine *e, maya_job_result *out) {
  if (!e->ran) return fail(MAYA_ESTATE, "maya_results before maya_run");
  CU(cudaSetDevice(e->device));
  const size_t nj = e->packs.size();
  int32_t err_flag = 0;
  CU(cudaMemcpyAsync(out, e->db.results, nj * sizeof(maya_job_result), cudaMemcpyDeviceToHost,
                     e->stream));
  CU(cudaMemcpyAsync(&err_flag, e->db.err_flag, sizeof err_flag, cudaMemcpyDeviceToHost,
                     e->stream));
  CU(cudaStreamSynchronize(e->stream));
  for (size_t j = 0; j < nj; j++) {
    const JobPack &P = e->packs[j];
    if (out[j].first_oom_rank >= 0 && (size_t)out[j].first_oom_rank < P.rank_orig.size())
      out[j].first_oom_rank = P.rank_orig[out[j].first_oom_rank];
  }
  cudaEventElapsedTime(&e->last_ms[0], e->ev[0], e->ev[1]);
  cudaEventElapsedTime(&e->last_ms[1], e->ev[1], e->ev[2]);
  cudaEventElapsedTime(&e->last_ms[2], e->ev[2], e->ev[3]);
  if (err_flag & 3) {
    // Estimation errors are raised by annotate() for ANY event, before the
    // simulation (estimate.py:344-347): attribute failed features to jobs.
    std::vector<uint32_t> fns(e->db.n_feats);
    std::vector<int64_t> wns(e->db.n_wfeats);
    CU(cudaMemcpy(fns.data(), e->db.feat_d32, fns.size() * 4, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(wns.data(), e->db.wire, wns.size() * 8, cudaMemcpyDeviceToHost));
    size_t fb = 0, sb = 0;
    for (size_t j = 0; j < nj; j++) {
      const JobPack &P = e->packs[j];
      bool bad = false;
      for (size_t f = 0; f < P.feats.size(); f++) bad |= fns[fb + f] == DUR32_FAIL;
      for (size_t s = 0; s < P.wfeats.size(); s++) bad |= wns[sb + s] < 0;
      // annotate() raises before simulate() runs (estimate.py:344-347): any
      // failed estimate of the job decides its status, whatever the schedule did
      if (bad && out[j].status != MAYA_ST_BAD_INPUT) out[j].status = MAYA_ST_ESTIMATION;
      fb += P.feats.size();
      sb += P.wfeats.size();
    }
  }
  return MAYA_OK;
}

// Engine-internal profiling counters (builds with -DMAYA_PROFILE; else returns 0).
// out: 16 counters (8 warp-window kernel, 8 lane kernel).
int maya_prof_read(unsigned long long *out16, int reset) {
  const int a = prof_read(out16, reset);
  lane_prof_read(out16 + 8, reset);
  if (getenv("MAYA_PROF_CHAIN")) chain_prof_read(out16 + 8, reset);   // chain counters instead
  return a;
}

int maya_get_stream(maya_engine *e, void **stream) {
  *stream = (void *)e->stream;
  return MAYA_OK;
}

int64_t maya_arena_bytes(maya_engine *e) { return (int64_t)e->arena_bytes; }

int maya_batch_stats(maya_engine *e, int64_t *o) {
  for (int i = 0; i < 16; i++) o[i] = 0;
  o[10] = e->run_launches;
  o[11] = e->topk_launches;
  o[0] = (int64_t)e->packs.size();
  for (size_t j = 0; j < e->packs.size(); j++) {
    const JobPack &P = e->packs[j];
    for (const RepHdr &h : P.reps) o[1] += h.n_events;
    o[2] += (int64_t)P.rank_comm.size();
    o[3] += (int64_t)P.feats.size();
    o[4] += (int64_t)P.slots.size();
    o[5] += (int64_t)P.ops.size();
    o[6] += P.hdr.rank_ops;
    o[8] += (int64_t)P.ranks.size();
    o[9] += (int64_t)P.reps.size();
    o[12] += (int64_t)P.blocks.size();
    o[13] += (int64_t)P.blk_fids.size();
    o[14] += (int64_t)P.wfeats.size();
    for (const RankRec &rr : P.ranks) o[15] += P.reps[rr.rep].n_events;   // class-ops
  }
  o[7] = (int64_t)e->arena_bytes;
  return MAYA_OK;
}

int maya_last_timings(maya_engine *e, float *ms3) {
  for (int i = 0; i < 3; i++) ms3[i] = e->last_ms[i];
  return MAYA_OK;
}

int maya_topk_async(maya_engine *e, int32_t k) {
  if (!e->ran) return fail(MAYA_ESTATE, "maya_topk_async before maya_run");
  if (k < 1 || k > 64) return fail(MAYA_EINVAL, "k must be in [1, 64]");
  CU(cudaSetDevice(e->device));
  if (!e->h_topk) CU(cudaMallocHost(&e->h_topk, 65 * sizeof(maya_topk_entry)));
  char *X = (char *)e->d_scratch;
  maya_topk_entry *d_out = (maya_topk_entry *)(X + e->x_topk_out.off);
  int32_t *d_n = (int32_t *)(X + e->x_topk_n.off);
  launch_topk(e->db, k, d_out, d_n, X + e->x_topk.off, e->stream);
  e->topk_launches = e->db.n_jobs ? 2 : 0;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(e->h_topk + 64, d_n, sizeof(int32_t), cudaMemcpyDeviceToHost, e->stream));
  CU(cudaMemcpyAsync(e->h_topk, d_out, k * sizeof(maya_topk_entry), cudaMemcpyDeviceToHost,
                     e->stream));
  e->topk_pending = k;
  return MAYA_OK;
}

int maya_topk(maya_engine *e, int32_t k, maya_topk_entry *out, int32_t *n_out) {
  if (!e->ran) return fail(MAYA_ESTATE, "maya_topk before maya_run");
  if (k < 1 || k > 64) return fail(MAYA_EINVAL, "k must be in [1, 64]");
  CU(cudaSetDevice(e->device));
  if (e->topk_pending == k) {   // enqueued by maya_topk_async after this run
    CU(cudaStreamSynchronize(e->stream));
    e->topk_pending = 0;
    *n_out = *(const int32_t *)(e->h_topk + 64);
    memcpy(out, e->h_topk, k * sizeof(maya_topk_entry));
    return MAYA_OK;
  }
  char *X = (char *)e->d_scratch;
  maya_topk_entry *d_out = (maya_topk_entry *)(X + e->x_topk_out.off);
  int32_t *d_n = (int32_t *)(X + e->x_topk_n.off);
  launch_topk(e->db, k, d_out, d_n, X + e->x_topk.off, e->stream);
  e->topk_launches = e->db.n_jobs ? 2 : 0;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(n_out, d_n, sizeof(int32_t), cudaMemcpyDeviceToHost, e->stream));
  CU(cudaMemcpyAsync(out, d_out, k * sizeof(maya_topk_entry), cudaMemcpyDeviceToHost, e->stream));
  CU(cudaStreamSynchronize(e->stream));
  return MAYA_OK;
}

int maya_timeline_size(maya_engine *e, int32_t job, int64_t *n) {
  if (job < 0 || (size_t)job >= e->packs.size()) return fail(MAYA_EINVAL, "job index");
  *n = e->packs[job].hdr.dev_ops;   // all ranks (classes are expanded)
  return MAYA_OK;
}

int maya_timeline(maya_engine *e, int32_t job, int32_t *rank, int32_t *stream, int32_t *seq,
                  int64_t *start, int64_t *end) {
  if (!e->recorded) return fail(MAYA_ESTATE, "no timeline recorded");
  if (job < 0 || (size_t)job >= e->packs.size()) return fail(MAYA_EINVAL, "job index");
  CU(cudaSetDevice(e->device));
  const JobPack &P = e->packs[job];
  uint64_t n_sim = 0;
  for (const RankRec &rr : P.ranks) n_sim += P.reps[rr.rep].n_ops;
  std::vector<int64_t> s(n_sim), en(n_sim);
  if (n_sim) {
    CU(cudaMemcpyAsync(s.data(), e->db.tl_start + e->job_tl[job], n_sim * 8,
                       cudaMemcpyDeviceToHost, e->stream));
    CU(cudaMemcpyAsync(en.data(), e->db.tl_end + e->job_tl[job], n_sim * 8,
                       cudaMemcpyDeviceToHost, e->stream));
  }
  CU(cudaStreamSynchronize(e->stream));
  uint64_t t = 0;
  for (size_t r = 0; r < P.rank_sim.size(); r++) {
    const RankRec &rr = P.ranks[P.rank_sim[r]];
    const RepHdr &h = P.reps[rr.rep];
    for (uint32_t sidx = 0; sidx < h.n_streams; sidx++) {
      const StreamRange &sr = P.streams[h.streams + sidx];
      for (uint32_t i = 0; i < sr.len; i++, t++) {
        const uint64_t src = rr.tl + sr.begin + i;
        rank[t] = (int32_t)r;
        stream[t] = sr.raw;
        const uint64_t o = h.ops + sr.begin + i;
        // tag in the low bits of seq: (seq << 2) | tag so callers can filter timed ops
        seq[t] = (int32_t)((P.op_seq[o] << 2) | op_tag(P.ops[o].meta));
        start[t] = s[src];
        end[t] = en[src];
      }
    }
  }
  return MAYA_OK;
}

int maya_rank_stats(maya_engine *e, int32_t job, int32_t num_ranks, int64_t *out) {
  if (!e->recorded || !e->stats_ok) return fail(MAYA_ESTATE, "no timeline recorded");
  if (job < 0 || (size_t)job >= e->packs.size()) return fail(MAYA_EINVAL, "job index");
  const JobPack &P = e->packs[job];
  if (num_ranks != (int32_t)P.rank_sim.size()) return fail(MAYA_EINVAL, "num_ranks of the job");
  CU(cudaSetDevice(e->device));
  const size_t ns = P.ranks.size();
  std::vector<int64_t> st(4 * ns);
  maya_job_result r{};
  if (ns)
    CU(cudaMemcpyAsync(st.data(), e->d_rstats + 4ull * e->job_rank0[job], 32 * ns,
                       cudaMemcpyDeviceToHost, e->stream));
  CU(cudaMemcpyAsync(&r, e->db.results + job, sizeof r, cudaMemcpyDeviceToHost, e->stream));
  CU(cudaStreamSynchronize(e->stream));
  for (int32_t q = 0; q < num_ranks; q++) {
    const int64_t *x = st.data() + 4 * (size_t)P.rank_sim[q];
    out[5 * q + 0] = x[0];              // compute_busy_ns
    out[5 * q + 1] = x[1];              // comm_busy_ns
    out[5 * q + 2] = x[2] - x[0];       // exposed_comm_ns = |comm u compute| - |compute|
    out[5 * q + 3] = r.total_ns - x[2]; // idle_ns
    out[5 * q + 4] = x[3];              // peak_mem_bytes
  }
  return MAYA_OK;
}

// ---- native generation ----------------------------------------------------


int maya_debug_pack_compare(const maya_model *model, int32_t n, const maya_config *cfgs,
                                       const maya_cluster *cluster, int32_t schedule,
                                       int64_t dispatch_overhead_ns, int32_t collapse) {
  int bad = 0;
  GenJob g, g2;
  for (int i = 0; i < n; i++) {
    std::string err;
    JobPack a, b2;
    int rc = generate_job(*model, cfgs[i], *cluster, schedule, dispatch_overhead_ns, g, &err);
    if (rc != MAYA_OK) continue;
    maya_raw_job raw = g.raw(0);
    pack_job(raw, i, a, collapse != 0);
    rc = pack_generated(*model, cfgs[i], *cluster, schedule, dispatch_overhead_ns, 0, i,
                        collapse != 0, g2, b2, &err);
    if (rc != MAYA_OK || !pack_eq(a, b2)) bad++;
  }
  return bad;
}

struct maya_gen {
  GenJob job;
  std::unique_ptr<LoadedJob> loaded;   // jobs read by maya_job_load (their text form)
  std::string op_blob, dtype_blob;
};

struct maya_trace {
  ParsedTrace t;
  std::string text;
};

int maya_last_error_kind(void) { return g_err_kind; }

int maya_trace_parse(const char *text, int64_t len, maya_trace **out) {
  if (!text || len < 0) return fail(MAYA_EINVAL, "null text");
  maya_trace *h = new maya_trace();
  try {
    parse_trace(text, (size_t)len, h->t);
  } catch (const TraceFail &f) {
    delete h;
    return fail_trace(f);
  } catch (const std::exception &x) {
    delete h;
    return fail(MAYA_EINVAL, x.what());
  }
  *out = h;
  return MAYA_OK;
}

int maya_trace_info(const maya_trace *h, int64_t *out4) {
  out4[0] = h->t.rank;
  out4[1] = h->t.host;
  out4[2] = h->t.device;
  out4[3] = (int64_t)h->t.ev.size();
  return MAYA_OK;
}

int maya_trace_serialize(maya_trace *h, const char **text, int64_t *len) {
  h->text = serialize_trace(h->t);
  *text = h->text.c_str();
  *len = (int64_t)h->text.size();
  return MAYA_OK;
}

int maya_trace_free(maya_trace *h) {
  delete h;
  return MAYA_OK;
}

int maya_job_load(const char *manifest_path, const maya_cluster *cluster, maya_gen **out) {
  if (!manifest_path || !cluster) return fail(MAYA_EINVAL, "null argument");
  if (cluster->num_hosts < 1 || cluster->devices_per_host < 1)
    return fail(MAYA_EINVAL, "cluster must have at least one host and device");
  maya_gen *g = new maya_gen();
  g->loaded.reset(new LoadedJob());
  try {
    load_job(manifest_path, cluster->num_hosts, cluster->devices_per_host,
             cluster->device_memory_bytes, g->job, *g->loaded);
  } catch (const TraceFail &f) {
    delete g;
    return fail_trace(f);
  } catch (const std::exception &x) {
    delete g;
    return fail(MAYA_EINVAL, x.what());
  }
  for (size_t q = 0; q < g->loaded->op_names.size(); q++)
    g->op_blob += (q ? "\n" : "") + g->loaded->op_names[q];
  for (size_t q = 0; q < g->loaded->dtype_names.size(); q++)
    g->dtype_blob += (q ? "\n" : "") + g->loaded->dtype_names[q];
  *out = g;
  return MAYA_OK;
}

int maya_job_save(const maya_gen *g, const char *out_dir, const char *manifest_name) {
  if (!g->loaded) return fail(MAYA_EINVAL, "only jobs read by maya_job_load keep their text form");
  try {
    save_job(*g->loaded, out_dir, manifest_name ? manifest_name : "job.manifest");
  } catch (const TraceFail &f) {
    return fail_trace(f);
  }
  return MAYA_OK;
}

int maya_gen_names(const maya_gen *g, int32_t which, const char **blob, int32_t *n) {
  if (which != 0 && which != 1) return fail(MAYA_EINVAL, "which: 0 op kinds, 1 dtypes");
  if (g->loaded) {
    *blob = which == 0 ? g->op_blob.c_str() : g->dtype_blob.c_str();
    *n = (int32_t)(which == 0 ? g->loaded->op_names.size() : g->loaded->dtype_names.size());
  } else {
    static std::string ob, db;
    static std::once_flag once;
    std::call_once(once, [] {
      for (int q = 0; q < 12; q++) ob += (q ? "\n" : "") + std::string(GEN_OP_KINDS[q]);
      for (int q = 0; q < 3; q++) db += (q ? "\n" : "") + std::string(GEN_DTYPES[q]);
    });
    *blob = which == 0 ? ob.c_str() : db.c_str();
    *n = which == 0 ? 12 : 3;
  }
  return MAYA_OK;
}

const char *maya_gen_op_kind_name(int32_t id) {
  return (id >= 0 && id < 12) ? GEN_OP_KINDS[id] : nullptr;
}
const char *maya_gen_dtype_name(int32_t id) { return (id >= 0 && id < 3) ? GEN_DTYPES[id] : nullptr; }

int maya_gen_job(const maya_model *model, const maya_config *cfg, const maya_cluster *cluster,
                 int32_t schedule, int64_t dispatch_overhead_ns, maya_gen **out) {
  maya_gen *g = new maya_gen();
  std::string err;
  int rc = generate_job(*model, *cfg, *cluster, schedule, dispatch_overhead_ns, g->job, &err);
  if (rc != MAYA_OK) {
    delete g;
    return fail(rc, err);
  }
  *out = g;
  return MAYA_OK;
}

int maya_gen_view_of(const maya_gen *g, maya_gen_view *v) {
  memset(v, 0, sizeof *v);
  v->job = g->job.raw(0);
  v->num_hosts = g->job.num_hosts;
  v->n_comm_names = (int32_t)g->job.comm_names.size();
  v->rep_ranks = g->job.rep_ranks.data();
  v->comm_names = g->job.comm_blob.c_str();
  v->n_events = (int64_t)g->job.ev_kind.size();
  v->n_calls = (int64_t)g->job.call_kind.size();
  v->n_rank_comm = (int64_t)g->job.rank_comm.size();
  return MAYA_OK;
}

int maya_gen_free(maya_gen *g) {
  delete g;
  return MAYA_OK;
}

int maya_batch_add_generated(maya_engine *e, const maya_model *model, int32_t n,
                             const maya_config *cfgs, const maya_cluster *cluster, int32_t device,
                             int32_t schedule, int64_t dispatch_overhead_ns,
                             const int32_t *key_ranks, int32_t n_threads, int32_t *status_out) {
  if (n < 0) return fail(MAYA_EINVAL, "negative job count");
  if (device < 0 || device >= 8) return fail(MAYA_EINVAL, "device index out of range");
  size_t base = e->packs.size();
  e->packs.resize(base + n);
  // longest first (generation cost grows with stages x micro-batches x virtual
  // stages, r = 0.8 over C2), so the workers' tail is short jobs
  std::vector<int32_t> lpt(n);
  for (int32_t i = 0; i < n; i++) lpt[i] = i;
  auto cost = [&](int32_t i) {
    return (int64_t)cfgs[i].pp * cfgs[i].micro_mult * std::max(1, cfgs[i].virtual_stages);
  };
  std::stable_sort(lpt.begin(), lpt.end(), [&](int32_t a, int32_t b) { return cost(a) > cost(b); });
  std::atomic<int> next(0);
  GenCache cache;   // layout-only structure, shared by this call's workers
  auto work = [&]() {
    thread_local GenJob g;
    for (;;) {
      int q = next.fetch_add(1);
      if (q >= n) break;
      const int i = lpt[q];
      std::string err;
      JobPack &P = e->packs[base + i];
      const int32_t kr = key_ranks ? key_ranks[i] : i;
      // fused generate -> pack (no raw event arrays)
      int rc = pack_generated(*model, cfgs[i], *cluster, schedule, dispatch_overhead_ns, device,
                              kr, (e->options & MAYA_OPT_COLLAPSE) != 0, g, P, &err,
                              !(e->options & MAYA_OPT_NO_BLOCKS), &cache);
      if (status_out) status_out[i] = rc;
      if (rc != MAYA_OK) {
        P.clear();
        P.hdr.status = MAYA_ST_BAD_INPUT;
        P.hdr.key_rank = kr;
        P.message = err;
      }
    }
  };
  WorkerPool::get().run(std::max(1, std::min<int>(n_threads, n)), work);
  e->uploaded = e->ran = false;
  return MAYA_OK;
}

}  // extern "C"
