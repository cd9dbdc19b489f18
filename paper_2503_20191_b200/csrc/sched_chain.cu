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
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_u32(bar)), "r"(nt) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  group_sync<NW>();
  // this thread's FIFO: loop invariants and walker state in registers
  const uint32_t w = b.lane_perm[LJ.perm + tid];
  const bool valid = w != 0xffffffffu;
  const ExecOp *ops = nullptr;       // global ExecOps (the FIFO's ops, folded when RES)
  const uint32_t *cnt = nullptr;
  uint64_t tl = 0;
  uint32_t len = 0, rank = 0, ns = 0, nsync = 0, fb = 0, rcb = 0, dlb = 0;
  uint32_t nops = 0;                 // the FIFO's (folded) ops
  uint32_t mac_sm = 0;               // RES: its macro area (shared memory)
  const ChainMacro *mac_g = nullptr; // RES: its macro ops (global)
  int err = 0;
  if (valid) {
    const Walker wk = b.walkers[J.walkers + w];
    const RankRec rr = b.ranks[J.ranks + wk.rank];
    const RepHdr &h = b.reps[rr.rep];
    const StreamRange sr = b.streams[h.streams + wk.stream];
    nops = RES ? b.clen[h.streams + wk.stream] : sr.len;
    cnt = (RES ? b.ccounts : b.counts) + h.counts + wk.stream;
    tl = J.timeline + rr.tl + sr.begin;
    rank = wk.rank;
    ns = h.n_streams;
    nsync = h.n_syncs;
    fb = rr.fire;
    rcb = rr.rslot;
    dlb = rr.delay;
    ops = b.exec + h.ops + sr.begin;
    len = nops;
    if (RES) {   // the FIFO's macro ops (chain_macro_kernel), host-planned count
      const uint32_t m0 = b.lane_wslot[J.walkers + w];
      const uint32_t m1 = w + 1 < W ? b.lane_wslot[J.walkers + w + 1] : LJ.n_slots;
      len = m1 - m0;
      mac_sm = sm_u32(dsm + L.ops) + m0 * (uint32_t)sizeof(ChainMacro);
      mac_g = b.macros + LJ.mbase + m0;
      if (len == 0 && nops > 0) err = MAYA_ST_INTERNAL;   // plan and fold disagree
    }
  }
  // op streams (each thread its FIFO) and the collective table (thread 0),
  // all bulk copies in flight at once
  const uint32_t bytes = (RES && valid ? len * (uint32_t)sizeof(ChainMacro) : 0u) +
                         (tid == 0 ? J.n_rcolls * 16u : 0u);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(bar)),
               "r"(bytes)
               : "memory");
  if (tid == 0 && J.n_rcolls)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(sm_u32(dsm + L.rcx)),
        "l"(b.rcx + J.rcolls), "r"(J.n_rcolls * 16u), "r"(sm_u32(bar))
        : "memory");
  if (RES && valid && len)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(mac_sm),
        "l"(mac_g), "r"(len * (uint32_t)sizeof(ChainMacro)), "r"(sm_u32(bar))
        : "memory");
  // tables: record times unfired, rings empty, no host sync resolved
  for (uint32_t q = tid; q < J.n_fire; q += nt) sh.fire[q] = -1;
  if (J.n_comms <= RING_MAX_COMMS)
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
#ifdef MAYA_PROFILE
  const long long t_copied = clock64();
  if (tid == 0) atomicAdd(&g_cprof[6], (unsigned long long)(t_copied - t_start));
#endif
  if (RES && valid && len && !err) {   // the macro pass flags a FIFO it could not fuse
    uint32_t k0;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(k0) : "r"(mac_sm + 40u) : "memory");
    if (k0 == CM_FAIL) err = MAYA_ST_INTERNAL;
  }
  group_sync<NW>();
#ifdef MAYA_PROFILE
  if (tid == 0) atomicAdd(&g_cprof[5], (unsigned long long)(clock64() - t_start));
  if (tid == 0) atomicAdd(&g_cprof[7], (unsigned long long)(clock64() - t_copied));
  unsigned long long n_it = 0, c_it = 0, n_ops = 0;
#endif

  int64_t x = 0, cdel = 0;
  uint32_t i = 0, iops = 0, seg = 0, bound = valid ? (nsync ? cnt[0] : nops) : 0, lim = 0;
  bool posted = false;
  // the unit at the head of the FIFO (a macro op; without folding, one op),
  // prefetched when its predecessor retires
  auto load_unit = [&](uint32_t q) -> ChainMacro {
    ChainMacro c;
    if (RES) {
      const uint32_t a = mac_sm + q * (uint32_t)sizeof(ChainMacro);
      uint64_t r1, dk, rr, wr;
      uint32_t cidx, end, kind, pad;
      asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(r1), "=l"(dk) : "r"(a) : "memory");
      asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(rr), "=l"(wr) : "r"(a + 16u) : "memory");
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(cidx), "=r"(end), "=r"(kind), "=r"(pad) : "r"(a + 32u) : "memory");
      c = ChainMacro{(int64_t)r1, (int64_t)dk, (int64_t)rr, (uint32_t)wr, (uint32_t)(wr >> 32),
                     cidx, end, kind, 0};
      return c;
    }
    const longlong2 v = __ldg(reinterpret_cast<const longlong2 *>(ops + q));
    const uint64_t wv = (uint64_t)v.y;
    const uint32_t tag = (uint32_t)(wv & 3u);
    const uint64_t pay = wv >> 2;
    c = ChainMacro{CNEG, 0, CNEG, 0, 0, 0, q + 1, 0, 0};
    if (tag == TAG_REC) {
      c.kind = CM_REC;
      c.rr = v.x;
      c.ridx = (uint32_t)pay;
    } else {
      c.r1 = v.x;
      if (tag == TAG_KERN) {
        c.kind = CM_KERN | (wv == EXEC_BAD ? CM_BAD : 0u) | (wv == EXEC_OVF ? CM_OVF : 0u);
        c.dk = (int64_t)pay;
      } else if (tag == TAG_COLL) {
        c.kind = CM_COLL;
        c.cidx = (uint32_t)pay;
      } else {
        c.kind = CM_WAIT | (pay == (EXEC_NONE >> 2) ? CM_NEVER : 0u);
        c.widx = (uint32_t)pay;
      }
    }
    return c;
  };
  ChainMacro cm{};
  if (valid && len && !err) cm = load_unit(0);
  int64_t rounds = 0;
  const uint32_t fire_sm = sm_u32(sh.fire + fb), rcx_sm = sm_u32(sh.rcx + rcb);
  const bool ring = (J.flags & JOB_RING) && J.n_comms <= RING_MAX_COMMS;
  for (;;) {
    bool progress = false;
    for (uint32_t r = tid; r < R; r += nt) progress |= chain_host_step(b, sh, r);
    group_sync<NW>();
    if (valid) {
      const uint32_t hk = sh.hostk[rank];
      lim = hk < nsync ? cnt[hk * ns] : nops;   // in (folded) ops
    }
    if (err) lim = iops;   // a failed FIFO stops (the job's status is the error)
    for (;;) {
#ifdef MAYA_PROFILE
      const long long t0 = clock64();
#endif
      bool prog = false;
      if (i < len && iops < lim) {
        if (iops >= bound) {   // next host-sync segment (rare)
          while (iops >= bound && seg < nsync) {
            seg++;
            cdel = sh.delay[dlb + seg];
            bound = seg < nsync ? cnt[seg * ns] : nops;
          }
        }
        // one predicated evaluation of the unit [WAIT]? [KERN | COLL]? [REC]?
        const uint32_t kind = cm.kind;
        const int64_t r1 = cm.r1 + cdel;
        const int64_t ready0 = x > r1 ? x : r1;
        int64_t fv = -1;   // WAIT: the record time (never recorded: stays -1, blocks forever)
        if ((kind & (CM_WAIT | CM_NEVER)) == CM_WAIT)
          asm volatile("ld.volatile.shared.s64 %0, [%1];" : "=l"(fv) : "r"(fire_sm + cm.widx * 8u) : "memory");
        const bool wait_ok = !(kind & CM_WAIT) || fv >= 0;
        const int64_t ready = ready0 > fv ? ready0 : fv;
        uint64_t ent = 1ull << 48;
        int64_t wire = 0;
        if (kind & CM_COLL)
          asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(ent), "=l"(wire) : "r"(rcx_sm + cm.cidx * 16u));
        const uint32_t nr = (uint32_t)(ent >> 48);
        bool ok = wait_ok;
        int64_t base = ready;
        if ((kind & CM_COLL) && nr != 1 && wait_ok) {   // collective rendezvous (sim.py:326-343)
          const uint32_t g = (uint32_t)(ent >> 32) & 0xffffu, idx = (uint32_t)ent;
          // shared-memory rings (2 slots per communicator, cumulative counts)
          // when every rank issues a communicator's calls in order from one
          // stream (JOB_RING); else one global slot per call
          // (explicit address spaces: a generic pointer would make every
          // atomic and volatile load generic, system scope)
          uint32_t target, old = 0, cnt = 0;
          uint64_t mx = 0;
          if (ring) {
            const uint32_t cs = sm_u32(sh.ring + 2 * g + (idx & 1u));
            target = ((idx >> 1) + 1u) * nr;
            if (!posted) {
              asm volatile("atom.shared.max.u64 %0, [%1], %2;" : "=l"(mx) : "r"(cs), "l"((uint64_t)ready) : "memory");
              asm volatile("fence.acq_rel.cta;" ::: "memory");
              asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(cs + 8u) : "memory");
              cnt = old + 1;
            } else {
              asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(cnt) : "r"(cs + 8u) : "memory");
            }
            if (cnt >= target) {
              asm volatile("fence.acq_rel.cta;" ::: "memory");
              asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(mx) : "r"(cs) : "memory");
            }
          } else {
            CollSlot *cs = b.cslots + J.slots + b.comms[J.comms + g].call_base + idx;
            target = nr;
            if (!posted) {
              asm volatile("atom.global.max.u64 %0, [%1], %2;" : "=l"(mx) : "l"(&cs->maxarr), "l"((uint64_t)ready) : "memory");
              asm volatile("fence.acq_rel.cta;" ::: "memory");
              asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(&cs->count) : "memory");
              cnt = old + 1;
            } else {
              asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(cnt) : "l"(&cs->count) : "memory");
            }
            if (cnt >= target) {
              asm volatile("fence.acq_rel.cta;" ::: "memory");
              asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(mx) : "l"(&cs->maxarr) : "memory");
            }
          }
          if (!posted) {
            posted = true;
            prog = true;
            if (cnt > target) err = MAYA_ST_INTERNAL;
          }
          const bool done_c = cnt >= target && !err;
          if (done_c) base = (int64_t)mx;
          ok = done_c;
        }
        const int64_t add = (kind & CM_KERN) ? cm.dk : wire;   // (wire = 0 unless COLL)
        if (kind & (CM_BAD | CM_OVF)) {            // a failed estimate / overflowed run (cold)
          err = (kind & CM_BAD) ? MAYA_ST_ESTIMATION : MAYA_ST_OVERFLOW;
          ok = false;
        }
        if (ok && (base >= CLIM || add >= CLIM) && add > INT64_MAX - base) {
          err = MAYA_ST_OVERFLOW;
          ok = false;
        }
        if (ok) {
          const int64_t v = base + add;
          const int64_t rr = cm.rr + cdel;
          const int64_t done = (kind & CM_REC) && rr > v ? rr : v;
          if (kind & CM_REC)
            asm volatile("st.volatile.shared.s64 [%0], %1;" ::"r"(fire_sm + cm.ridx * 8u), "l"(done) : "memory");
          if (REC) {   // (timeline runs: one op per unit)
            b.tl_start[tl + i] = kind == CM_REC ? done : ready0;
            b.tl_end[tl + i] = done;
          }
          x = done;
          posted = false;
          iops = cm.end;
          i++;
          if (i < len) cm = load_unit(i);
          prog = true;
#ifdef MAYA_PROFILE
          n_ops++;
#endif
        }
        if (err) lim = iops;
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
      sh.fst_i[w] = iops;
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
  bool incomplete = valid && i < len;   // (units: macro ops or ops)
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

// ---------------------------------------------------------------------------
// Macro pass: the folded ops of every FIFO of a chain job grouped into macro
// ops (soa.h MacroFuse), written to DevBatch.macros for the chain kernel to
// bulk-copy.  One CTA per chain job, a warp per FIFO in turn (8 warps).  The
// rule is local -- an op joins the macro of the op before it (same segment)
// iff it is a body after a WAIT or a REC after a WAIT or a body, so a macro
// has at most 3 members -- hence chunks of 32 ops: lanes 0-29 lead macros
// whose members all lie in the chunk, and the next chunk starts at the first
// op no written macro covers.  Grid: `parts` CTAs of 8 warps per chain job
// (enough for its largest FIFO count), one warp per FIFO, so every FIFO of the
// batch is fused at once.
static constexpr uint32_t MACRO_WARPS = 8;

__global__ void __launch_bounds__(MACRO_WARPS * 32) chain_macro_kernel(DevBatch b,
                                                                       const int32_t *order,
                                                                       uint32_t parts) {
  const uint32_t PARTS = parts;
  const uint32_t j = (uint32_t)order[blockIdx.x / PARTS];
  const JobHdr &J = b.jobs[j];
  const uint32_t lane = threadIdx.x & 31u, W = J.n_walkers;
  const uint32_t w = (blockIdx.x % PARTS) * MACRO_WARPS + (threadIdx.x >> 5);
  if (J.status != MAYA_ST_OK || w >= W) return;
  const LaneJob LJ = b.lane_jobs[j];
  {
    const Walker wk = b.walkers[J.walkers + w];
    const RankRec rr = b.ranks[J.ranks + wk.rank];
    const RepHdr &h = b.reps[rr.rep];
    const StreamRange sr = b.streams[h.streams + wk.stream];
    const uint32_t nops = b.clen[h.streams + wk.stream];
    const ExecOp *ops = b.exec + h.ops + sr.begin;
    const uint32_t *cnt = b.ccounts + h.counts + wk.stream;
    const uint32_t ns = h.n_streams, nsync = h.n_syncs;
    const uint32_t m0 = b.lane_wslot[J.walkers + w];
    const uint32_t len = (w + 1 < W ? b.lane_wslot[J.walkers + w + 1] : LJ.n_slots) - m0;
    ChainMacro *out = b.macros + LJ.mbase + m0;
    // the first four sync boundaries (a segment: the syncs whose count <= q)
    const uint32_t bnd = lane < nsync && lane < 4u ? cnt[lane * ns] : 0xffffffffu;
    const uint32_t fb0 = __shfl_sync(FULL, bnd, 0), fb1 = __shfl_sync(FULL, bnd, 1),
                   fb2 = __shfl_sync(FULL, bnd, 2), fb3 = __shfl_sync(FULL, bnd, 3);
    uint32_t m_base = 0, p_cls = 4, p_seg = 0;   // macros written, op before the chunk
    bool fail = false;
    for (uint32_t q0 = 0; q0 < nops && !fail;) {
      const uint32_t q = q0 + lane;
      const bool have = q < nops;
      longlong2 v = make_longlong2(0, 0);
      if (have) v = __ldg(reinterpret_cast<const longlong2 *>(ops + q));
      const uint64_t dsp = (uint64_t)v.x, wv = (uint64_t)v.y;
      uint32_t sg = (q >= fb0) + (q >= fb1) + (q >= fb2) + (q >= fb3);
      if (have && nsync > 4) {   // many host syncs: binary search
        uint32_t lo = 0, hi = nsync;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (cnt[mid * ns] <= q) lo = mid + 1; else hi = mid;
        }
        sg = lo;
      }
      const uint32_t tag = (uint32_t)(wv & 3u);
      const uint32_t cls = !have ? 5u : tag == TAG_KERN ? 0u : tag == TAG_COLL ? 1u
                         : tag == TAG_REC ? 2u : 3u;
      uint32_t pc = __shfl_up_sync(FULL, cls, 1), ps = __shfl_up_sync(FULL, sg, 1);
      if (lane == 0) { pc = p_cls; ps = p_seg; }
      const bool body = cls <= 1u;
      const bool joins = have && pc < 4u && ps == sg &&
                         ((body && pc == 3u) || (cls == 2u && (pc == 3u || pc <= 1u)));
      const bool lead = have && lane < 30u && !joins;
      const uint32_t j1 = __shfl_down_sync(FULL, joins ? 1u : 0u, 1);
      const uint32_t j2 = __shfl_down_sync(FULL, joins ? 1u : 0u, 2);
      const uint64_t d1 = __shfl_down_sync(FULL, dsp, 1), w1 = __shfl_down_sync(FULL, wv, 1);
      const uint64_t d2 = __shfl_down_sync(FULL, dsp, 2), w2 = __shfl_down_sync(FULL, wv, 2);
      const uint32_t nmem = 1u + ((lane < 31u && j1) ? 1u + ((lane < 30u && j2) ? 1u : 0u) : 0u);
      const unsigned lm = __ballot_sync(FULL, lead);
      const uint32_t midx = m_base + __popc(lm & ((1u << lane) - 1u));
      if (lead && midx < len) {
        ChainMacro c{CNEG, 0, CNEG, 0, 0, 0, q + nmem, 0, 0};
#pragma unroll
        for (uint32_t k = 0; k < 3; k++) {
          if (k >= nmem) break;
          const uint64_t dk = k == 0 ? dsp : k == 1 ? d1 : d2;
          const uint64_t wk2 = k == 0 ? wv : k == 1 ? w1 : w2;
          const uint32_t tk = (uint32_t)(wk2 & 3u);
          const uint64_t pay = wk2 >> 2;
          if (tk == TAG_REC) {
            c.kind |= CM_REC;
            c.rr = (int64_t)dk;
            c.ridx = (uint32_t)pay;
          } else {
            if ((int64_t)dk > c.r1) c.r1 = (int64_t)dk;
            if (tk == TAG_KERN) {
              c.kind |= CM_KERN | (wk2 == EXEC_BAD ? CM_BAD : 0u) | (wk2 == EXEC_OVF ? CM_OVF : 0u);
              c.dk = (int64_t)pay;
            } else if (tk == TAG_COLL) {
              c.kind |= CM_COLL;
              c.cidx = (uint32_t)pay;
            } else {
              c.kind |= CM_WAIT | (pay == (EXEC_NONE >> 2) ? CM_NEVER : 0u);
              c.widx = (uint32_t)pay;
            }
          }
        }
        longlong2 *o = reinterpret_cast<longlong2 *>(out + midx);
        o[0] = make_longlong2(c.r1, c.dk);
        o[1] = make_longlong2(c.rr, (long long)(((uint64_t)c.ridx << 32) | c.widx));
        o[2] = make_longlong2((long long)(((uint64_t)c.end << 32) | c.cidx), (long long)c.kind);
      }
      m_base += __popc(lm);
      fail = m_base > len;
      const uint32_t cov = __reduce_max_sync(FULL, lead ? lane + nmem : 0u);
      p_cls = __shfl_sync(FULL, cls, cov - 1);
      p_seg = __shfl_sync(FULL, sg, cov - 1);
      q0 += cov;
    }
    if ((fail || m_base != len) && len && lane == 0) out[0].kind = CM_FAIL;
  }
}

void launch_chain_macros(const DevBatch &b, const int32_t *order, uint32_t n, uint32_t max_fifos,
                         cudaStream_t s) {
  const uint32_t parts = (max_fifos + MACRO_WARPS - 1) / MACRO_WARPS;
  if (n && parts) chain_macro_kernel<<<n * parts, MACRO_WARPS * 32, 0, s>>>(b, order, parts);
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
#define CHAIN_ATTR(NW)                                                                                  \
  cudaFuncSetAttribute(sched_chain_kernel<NW, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap); \
  cudaFuncSetAttribute(sched_chain_kernel<NW, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap); \
  cudaFuncSetAttribute(sched_chain_kernel<NW, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    CHAIN_ATTR(1) CHAIN_ATTR(2) CHAIN_ATTR(4) CHAIN_ATTR(8)
#undef CHAIN_ATTR
    attr = true;
  }
  const bool res = b.clen != nullptr;   // folded runs (never with a timeline)
#define CHAIN_LAUNCH(NW)                                                                     \
  do {                                                                                       \
    if (record) sched_chain_kernel<NW, false, true><<<n, NW * 32, smem, s>>>(b, order);      \
    else if (res) sched_chain_kernel<NW, true, false><<<n, NW * 32, smem, s>>>(b, order);    \
    else sched_chain_kernel<NW, false, false><<<n, NW * 32, smem, s>>>(b, order);            \
  } while (0)
  if (threads <= 32) CHAIN_LAUNCH(1);
  else if (threads <= 64) CHAIN_LAUNCH(2);
  else if (threads <= 128) CHAIN_LAUNCH(4);
  else CHAIN_LAUNCH(8);
#undef CHAIN_LAUNCH
}

}  // namespace maya
