// Chain scheduler (sm_100a): latency-bound jobs, whole job resident in one
// CTA's shared memory, ONE THREAD PER FIFO, lockstep iterations.
//
// Same semantics as sched_warp_kernel (kernels.cu) and the lane kernels
// (sched_lane.cu) -- the event-driven simulator of pkg/src/dltsim/sim.py:222-402
// evaluated as a monotone max-plus fixpoint:
//     ready = max(dispatch, done(prev op on the stream))
//     KERN  done = ready + dur          REC  fire = done = ready
//     WAIT  done = max(ready, fire)     COLL done = max_members(ready) + wire
// -- shaped for jobs whose time is a CHAIN of hand-offs between few FIFOs
// (pipeline stages after rank-class collapse: C2's pp8 jobs hand each
// microbatch stage to stage; after run folding their critical path is ~1,500
// dependent ops).  The cost that matters is the latency of ONE op on that
// path, so:
//   * the whole job lives in the CTA's shared memory: every FIFO's folded op
//     stream (one cp.async.bulk per FIFO at entry, completed on one mbarrier),
//     record times, collective rings, the rank collective table;
//   * one thread per FIFO (1 or 2 warps), and every iteration each thread
//     evaluates the op at the head of its FIFO with the SAME predicated
//     instruction sequence whatever the op kind -- no divergent per-kind
//     paths (measured: a divergent "run each FIFO until it blocks" loop costs
//     the union of all lanes' paths, ~1.1k cycles per critical op); only the
//     rendezvous atomics of a multi-member collective branch;
//   * the next op of each FIFO is prefetched into registers when the current
//     one retires, so an iteration's dependent chain is one table load
//     (record time / collective entry) plus a few integer ops;
//   * a hand-off (record -> wait, last collective arrival) is visible to the
//     consumer in the next iteration (__syncwarp / bar.sync between iterations).
// Host syncs, termination and deadlock follow the round protocol of the other
// kernels: an iteration in which no thread progresses ends the round, host
// syncs are resolved (sim.py:243-283), and a round without progress with work
// left is the reference's SimDeadlockError (sim.py:382-402).
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace maya {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int64_t CNEG = INT64_MIN / 4;             // -inf of the max-plus evaluation
constexpr int64_t CLIM = (int64_t)1 << 62;          // operands below: no sum leaves int64

#ifdef MAYA_PROFILE
// [0] kernel cycles [1] iterations [2] iteration cycles [3] ops retired
// [4] rounds [5] setup cycles
__device__ unsigned long long g_cprof[8];
#endif

__device__ __forceinline__ uint32_t sm_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ int64_t lds_vol_s64(const void *p) {
  int64_t v;
  asm volatile("ld.volatile.shared.s64 %0, [%1];" : "=l"(v) : "r"(sm_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds_vol_u32(const void *p) {
  uint32_t v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(sm_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void sts_vol_s64(void *p, int64_t v) {
  asm volatile("st.volatile.shared.s64 [%0], %1;" ::"r"(sm_u32(p)), "l"(v) : "memory");
}

struct ChainSh {
  const JobHdr *J;
  CollSlot *ring;          // 2 per communicator
  uint32_t *hostk;         // resolved host syncs per rank
  uint32_t *fst_i;         // FIFO states at round end (host syncs read them)
  int64_t *fst_x;
  int64_t *fire;           // job's record times
  const RCX *rcx;          // job's rank-collective table
  int64_t *delay;          // job's host-delay table (global)
};

// Resolve the host syncs of rank r that the FIFO states allow (sim.py:243-263,
// 272-283): H' = max(H, X), host time = gap prefix + delay.
__device__ bool chain_host_step(const DevBatch &b, const ChainSh &sh, uint32_t r) {
  const JobHdr &J = *sh.J;
  const RankRec rr = b.ranks[J.ranks + r];
  const RepHdr &h = b.reps[rr.rep];
  uint32_t k = sh.hostk[r];
  if (k >= h.n_syncs) return false;
  int64_t *delay = sh.delay + rr.delay;
  int64_t d = delay[k];
  bool adv = false;
  while (k < h.n_syncs) {
    const SyncRec s = b.syncs[h.syncs + k];
    int64_t X = INT64_MIN;
    bool ok = true;
    if (s.type == SYNC_ESYNC) {
      if (s.arg == NO_REC) {
        ok = false;
      } else {
        X = lds_vol_s64(sh.fire + rr.fire + s.arg);
        ok = X >= 0;
      }
    } else {
      uint32_t s0 = 0, s1 = h.n_streams;
      if (s.type == SYNC_SSYNC) {
        if (s.arg == NO_REC) { s0 = s1 = 0; } else { s0 = s.arg; s1 = s.arg + 1; }
      }
      for (uint32_t ls = s0; ls < s1; ls++) {
        const uint32_t cnt = (b.clen ? b.ccounts : b.counts)[h.counts + s.cnt + ls];
        if (cnt == 0) continue;
        const uint32_t w = rr.walker + ls;
        if (sh.fst_i[w] < cnt) { ok = false; break; }
        if (sh.fst_x[w] > X) X = sh.fst_x[w];
      }
    }
    if (!ok) break;
    if (X > s.gpre + d) d = X - s.gpre;
    k++;
    delay[k] = d;
    adv = true;
  }
  sh.hostk[r] = k;
  return adv;
}

template <int NW>
__device__ __forceinline__ bool group_any(bool v) {
  if (NW == 1) {
    __syncwarp();
    return __any_sync(FULL, v);
  }
  return __syncthreads_or(v) != 0;
}
template <int NW>
__device__ __forceinline__ int group_max(int v) {
  if (NW == 1) {
    __syncwarp();
    return (int)__reduce_max_sync(FULL, (unsigned)v);
  }
  __shared__ int s_m;
  if (threadIdx.x == 0) s_m = 0;
  __syncthreads();
  if (v) atomicMax(&s_m, v);
  __syncthreads();
  const int r = s_m;
  __syncthreads();
  return r;
}
template <int NW>
__device__ __forceinline__ void group_sync() {
  if (NW == 1) __syncwarp();
  else __syncthreads();
}

}  // namespace

// One CTA of NW warps per job; thread t owns FIFO perm[t] (LaneJob.per_lane
// == 1).  The region is laid out by chain_layout (soa.h); lane_wslot holds
// each FIFO's first op in the op area.
// RES: folded runs, every FIFO's ops staged on chip; REC: record the timeline
// (unfolded ops, read from global memory).
template <int NW, bool RES, bool REC>
__global__ void __launch_bounds__(NW * 32) sched_chain_kernel(DevBatch b, const int32_t *order) {
  extern __shared__ __align__(128) uint8_t dsm[];
  const uint32_t tid = threadIdx.x, nt = NW * 32;
#ifdef MAYA_PROFILE
  const long long t_start = clock64();
#endif
  const uint32_t j = (uint32_t)order[blockIdx.x];
  const JobHdr &J = b.jobs[j];
  maya_job_result *res = b.results + j;
  if (J.status != MAYA_ST_OK) {
    if (tid == 0) {
      maya_job_result r = {};
      r.status = J.status;
      r.first_oom_rank = -1;
      r.first_oom_seq = -1;
      r.rank_ops = J.rank_ops;
      *res = r;
    }
    return;
  }
  const LaneJob LJ = b.lane_jobs[j];
  const uint32_t W = J.n_walkers, R = J.n_ranks;
  constexpr bool resident = RES;
  const ChainLayout L = chain_layout(W, R, J.n_comms, J.n_fire, J.n_rcolls, LJ.n_slots);
  ChainSh sh;
  sh.J = &J;
  sh.ring = (CollSlot *)(dsm + L.ring);
  sh.hostk = (uint32_t *)(dsm + L.hostk);
  sh.fst_i = (uint32_t *)(dsm + L.fst_i);
  sh.fst_x = (int64_t *)(dsm + L.fst_x);
  sh.fire = (int64_t *)(dsm + L.fire);
  sh.rcx = (const RCX *)(dsm + L.rcx);
  sh.delay = b.delay + J.delay;
  uint64_t *bar = (uint64_t *)(dsm + L.bar);
  ExecOp *sops = (ExecOp *)(dsm + L.ops);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_u32(bar)), "r"(nt) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  group_sync<NW>();
  // this thread's FIFO: loop invariants and walker state in registers
  const uint32_t w = b.lane_perm[LJ.perm + tid];
  const bool valid = w != 0xffffffffu;
  const ExecOp *ops = nullptr;
  const uint32_t *cnt = nullptr;
  uint64_t tl = 0;
  uint32_t len = 0, rank = 0, ns = 0, nsync = 0, fb = 0, rcb = 0, dlb = 0;
  const ExecOp *src = nullptr;
  if (valid) {
    const Walker wk = b.walkers[J.walkers + w];
    const RankRec rr = b.ranks[J.ranks + wk.rank];
    const RepHdr &h = b.reps[rr.rep];
    const StreamRange sr = b.streams[h.streams + wk.stream];
    len = resident ? b.clen[h.streams + wk.stream] : sr.len;
    cnt = (resident ? b.ccounts : b.counts) + h.counts + wk.stream;
    tl = J.timeline + rr.tl + sr.begin;
    rank = wk.rank;
    ns = h.n_streams;
    nsync = h.n_syncs;
    fb = rr.fire;
    rcb = rr.rslot;
    dlb = rr.delay;
    src = b.exec + h.ops + sr.begin;
    ops = resident ? sops + b.lane_wslot[J.walkers + w] : src;
  }
  const uint32_t ops_sm = RES && valid ? sm_u32(ops) : 0u;
  // op streams (each thread its FIFO) and the collective table (thread 0),
  // all bulk copies in flight at once
  const uint32_t bytes = (resident && valid ? len * 16u : 0u) + (tid == 0 ? J.n_rcolls * 16u : 0u);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(bar)),
               "r"(bytes)
               : "memory");
  if (tid == 0 && J.n_rcolls)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(sm_u32(dsm + L.rcx)),
        "l"(b.rcx + J.rcolls), "r"(J.n_rcolls * 16u), "r"(sm_u32(bar))
        : "memory");
  if (resident && valid && len)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(sm_u32(ops)),
        "l"(src), "r"(len * 16u), "r"(sm_u32(bar))
        : "memory");
  // tables: record times unfired, rings empty, no host sync resolved
  for (uint32_t q = tid; q < J.n_fire; q += nt) sh.fire[q] = -1;
  for (uint32_t q = tid; q < 2 * J.n_comms; q += nt) sh.ring[q] = CollSlot{0, 0, 0};
  for (uint32_t r = tid; r < R; r += nt) {
    sh.hostk[r] = 0;
    sh.delay[b.ranks[J.ranks + r].delay] = 0;
  }
  for (uint32_t q = tid; q < W; q += nt) {
    sh.fst_i[q] = 0;
    sh.fst_x[q] = 0;
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(sm_u32(bar))
          : "memory");
  }
  group_sync<NW>();
#ifdef MAYA_PROFILE
  if (tid == 0) atomicAdd(&g_cprof[5], (unsigned long long)(clock64() - t_start));
  unsigned long long n_it = 0, c_it = 0, n_ops = 0;
#endif

  int64_t x = 0, cdel = 0;
  uint32_t i = 0, seg = 0, bound = valid ? (nsync ? cnt[0] : len) : 0, lim = 0;
  bool posted = false;
  // the op at the head of the FIFO, prefetched when its predecessor retires
  auto load_op = [&](uint32_t q) -> ExecOp {
    if (RES) {
      uint64_t a, c;
      asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(c) : "r"(ops_sm + q * 16u));
      return ExecOp{(int64_t)a, c};
    }
    const longlong2 v = __ldg(reinterpret_cast<const longlong2 *>(ops + q));
    return ExecOp{v.x, (uint64_t)v.y};
  };
  ExecOp nxt{0, 0};
  if (valid && len) nxt = load_op(0);
  int err = 0;
  int64_t rounds = 0;
  const uint32_t fire_sm = sm_u32(sh.fire + fb), rcx_sm = sm_u32(sh.rcx + rcb);
  for (;;) {
    bool progress = false;
    for (uint32_t r = tid; r < R; r += nt) progress |= chain_host_step(b, sh, r);
    group_sync<NW>();
    if (valid) {
      const uint32_t hk = sh.hostk[rank];
      lim = hk < nsync ? cnt[hk * ns] : len;
    }
    if (err) lim = i;   // a failed FIFO stops (the job's status is the error)
    for (;;) {
#ifdef MAYA_PROFILE
      const long long t0 = clock64();
#endif
      bool prog = false;
      if (i < lim) {
        if (i >= bound) {   // next host-sync segment (rare)
          while (i >= bound && seg < nsync) {
            seg++;
            cdel = sh.delay[dlb + seg];
            bound = seg < nsync ? cnt[seg * ns] : len;
          }
        }
        // one predicated evaluation for every op kind
        const uint32_t tag = (uint32_t)(nxt.w & 3u);
        const uint32_t pay32 = (uint32_t)(nxt.w >> 2);    // REC/WAIT/COLL index
        const int64_t rdisp = nxt.disp + cdel;
        const int64_t ready = x > rdisp ? x : rdisp;
        const bool isK = tag == TAG_KERN, isR = tag == TAG_REC, isW = tag == TAG_WAIT,
                   isC = tag == TAG_COLL;
        int64_t fv = -1;   // WAIT: the record time (never-recorded: stays -1, blocks forever)
        if (isW && (nxt.w >> 2) != (EXEC_NONE >> 2))
          asm volatile("ld.volatile.shared.s64 %0, [%1];" : "=l"(fv) : "r"(fire_sm + pay32 * 8u) : "memory");
        uint64_t ent = 1ull << 48;
        int64_t wire = 0;
        if (isC)
          asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(ent), "=l"(wire) : "r"(rcx_sm + pay32 * 16u));
        const uint32_t nr = (uint32_t)(ent >> 48);
        bool ok = isK || isR || fv >= 0 || (isC && nr == 1);
        int64_t base = ready > fv ? ready : fv;
        if (isC && nr != 1) {                      // collective rendezvous (sim.py:326-343)
          const uint32_t g = (uint32_t)(ent >> 32) & 0xffffu, idx = (uint32_t)ent;
          CollSlot *cs = sh.ring + 2 * g + (idx & 1u);
          const uint32_t target = ((idx >> 1) + 1u) * nr;
          bool done_c;
          if (!posted) {
            atomicMax(&cs->maxarr, (unsigned long long)ready);
            __threadfence_block();
            const uint32_t old = atomicAdd(&cs->count, 1u);
            posted = true;
            prog = true;
            if (old + 1 > target) err = MAYA_ST_INTERNAL;
            done_c = old + 1 == target;
          } else {
            done_c = lds_vol_u32(&cs->count) >= target;
          }
          if (done_c) {
            __threadfence_block();
            base = (int64_t)lds_vol_s64(&cs->maxarr);
          }
          ok = done_c && !err;
        }
        const int64_t add = isK ? (int64_t)(nxt.w >> 2) : wire;   // (wire = 0 unless COLL)
        if (isK && nxt.w >= EXEC_OVF) {            // EXEC_OVF / EXEC_BAD (cold)
          err = nxt.w == EXEC_BAD ? MAYA_ST_ESTIMATION : MAYA_ST_OVERFLOW;
          ok = false;
        }
        if (ok && (base >= CLIM || add >= CLIM) && add > INT64_MAX - base) {
          err = MAYA_ST_OVERFLOW;
          ok = false;
        }
        if (ok) {
          const int64_t done = base + add;
          if (isR)
            asm volatile("st.volatile.shared.s64 [%0], %1;" ::"r"(fire_sm + pay32 * 8u), "l"(ready) : "memory");
          if (REC) {
            b.tl_start[tl + i] = ready;
            b.tl_end[tl + i] = done;
          }
          x = done;
          posted = false;
          i++;
          if (i < len) nxt = load_op(i);
          prog = true;
#ifdef MAYA_PROFILE
          n_ops++;
#endif
        }
        if (err) lim = i;
      }
      const bool anyp = group_any<NW>(prog);
#ifdef MAYA_PROFILE
      n_it++;
      c_it += clock64() - t0;
#endif
      if (!anyp) break;
      progress = true;
    }
    if (valid) {
      sh.fst_i[w] = i;
      sh.fst_x[w] = x;
    }
    rounds++;
    err = group_max<NW>(err);
    if (err) break;
    if (!group_any<NW>(progress)) break;
  }
  // x is monotone along a FIFO: its last value is the FIFO's latest completion
  int64_t tmax = x;
#ifdef MAYA_PROFILE
  if (tid == 0) {
    atomicAdd(&g_cprof[0], (unsigned long long)(clock64() - t_start));
    atomicAdd(&g_cprof[1], n_it);
    atomicAdd(&g_cprof[2], c_it);
    atomicAdd(&g_cprof[4], (unsigned long long)rounds);
  }
  atomicAdd(&g_cprof[3], n_ops);
#endif
  // epilogue: unfinished FIFOs or host syncs = deadlock; host end time, peak
  // memory, first OOM (sim.py:235-242, 365-366)
  __shared__ int s_incomplete, s_oom_rank;
  __shared__ unsigned long long s_tmax;
  __shared__ long long s_peak, s_oom_t;
  if (tid == 0) {
    s_incomplete = 0;
    s_oom_rank = INT32_MAX;
    s_tmax = 0;
    s_peak = 0;
    s_oom_t = INT64_MAX;
  }
  group_sync<NW>();
  bool incomplete = valid && i < len;
  int64_t oom_t = INT64_MAX, peak = 0;
  int32_t oom_rank = INT32_MAX;
  for (uint32_t r = tid; r < R; r += nt) {
    const RankRec rr = b.ranks[J.ranks + r];
    const RepHdr &h = b.reps[rr.rep];
    if (sh.hostk[r] < h.n_syncs) { incomplete = true; continue; }
    const int64_t hend = h.gend + sh.delay[rr.delay + h.n_syncs];
    if (hend > tmax) tmax = hend;
    const RepOut ro = b.repout[rr.rep];
    if (ro.peak > peak) peak = ro.peak;
    if (ro.first_exceed >= 0) {
      const MemRec m = b.mems[h.mems + ro.first_exceed];
      const int64_t t = m.gpre + sh.delay[rr.delay + m.seg];
      if (t < oom_t || (t == oom_t && (int32_t)r < oom_rank)) {
        oom_t = t;
        oom_rank = (int32_t)r;
      }
    }
  }
  if (incomplete) s_incomplete = 1;
  atomicMax(&s_tmax, (unsigned long long)tmax);
  atomicMax(&s_peak, (long long)peak);
  if (oom_rank != INT32_MAX) atomicMin(&s_oom_t, (long long)oom_t);
  group_sync<NW>();
  if (oom_rank != INT32_MAX && oom_t == s_oom_t) atomicMin(&s_oom_rank, oom_rank);
  group_sync<NW>();
  if (tid == 0) {
    const bool inc = s_incomplete != 0;
    maya_job_result r = {};
    r.status = err ? err : (inc ? MAYA_ST_DEADLOCK : MAYA_ST_OK);
    r.total_ns = (int64_t)s_tmax;
    r.peak_mem_bytes = s_peak;
    r.first_oom_rank = -1;
    r.first_oom_seq = -1;
    if (s_oom_rank != INT32_MAX && !inc) {
      const RankRec rr = b.ranks[J.ranks + s_oom_rank];
      const RepHdr &h = b.reps[rr.rep];
      r.oom = 1;
      r.first_oom_rank = s_oom_rank;
      r.first_oom_seq = (int32_t)b.mems[h.mems + b.repout[rr.rep].first_exceed].seq;
    }
    r.dispatched_ops = J.dev_ops;
    r.completed_ops = J.dev_ops;
    r.rank_ops = J.rank_ops;
    r.rounds = rounds;
    *res = r;
  }
}

int chain_prof_read(unsigned long long *out8, int reset) {
#ifdef MAYA_PROFILE
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out8, g_cprof, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_cprof, z, sizeof z);
  }
  return 1;
#else
  (void)out8;
  (void)reset;
  return 0;
#endif
}

void launch_schedule_chain(const DevBatch &b, const int32_t *order, uint32_t n, uint32_t threads,
                           int record, uint32_t smem, cudaStream_t s) {
  if (!n) return;
  static bool attr = false;
  if (!attr) {
    const int cap = (int)CHAIN_REGION[CHAIN_CLASSES - 1];
    cudaFuncSetAttribute(sched_chain_kernel<1, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(sched_chain_kernel<2, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(sched_chain_kernel<1, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(sched_chain_kernel<2, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(sched_chain_kernel<1, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(sched_chain_kernel<2, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    attr = true;
  }
  const bool res = b.clen != nullptr;   // folded runs (never with a timeline)
  if (threads <= 32) {
    if (record) sched_chain_kernel<1, false, true><<<n, 32, smem, s>>>(b, order);
    else if (res) sched_chain_kernel<1, true, false><<<n, 32, smem, s>>>(b, order);
    else sched_chain_kernel<1, false, false><<<n, 32, smem, s>>>(b, order);
  } else {
    if (record) sched_chain_kernel<2, false, true><<<n, 64, smem, s>>>(b, order);
    else if (res) sched_chain_kernel<2, true, false><<<n, 64, smem, s>>>(b, order);
    else sched_chain_kernel<2, false, false><<<n, 64, smem, s>>>(b, order);
  }
}

}  // namespace maya
