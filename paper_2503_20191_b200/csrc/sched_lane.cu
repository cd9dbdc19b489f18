// Lane-parallel max-plus scheduler (sm_100a): ONE LANE PER (rank, stream) FIFO.
//
// Same semantics as sched_warp_kernel (kernels.cu) -- the event-driven
// simulator of pkg/src/dltsim/sim.py:222-402 evaluated as a monotone max-plus
// fixpoint --
//     ready = max(dispatch, done(prev op on the stream))
//     KERN  done = ready + dur          REC  fire = done = ready
//     WAIT  done = max(ready, fire)     COLL done = max_members(ready) + wire
// but mapped for throughput on jobs with many balanced FIFOs: every lane owns
// one (or a few) FIFOs and the lanes step in LOCKSTEP, each retiring at most
// one op of each of its FIFOs per step, so the warp executes one short,
// mostly convergent op-evaluation sequence per step for up to 32 FIFOs, and a
// record -> wait or collective hand-off between FIFOs costs one step (shared
// memory), not a cross-warp wake-up.  (Jobs dominated by one long FIFO -- a
// compute stream -- go to the warp-window kernel instead, which scans 32 ops
// of one FIFO per step; the engine chooses per job.)  Two launch shapes:
//   * warp jobs  (sched_lane_warp_kernel): one WARP simulates one job; a CTA
//     holds several independent jobs, each in its own shared-memory region,
//     so many small jobs (C2 configs, C5 8-rank sweeps) are resident per SM;
//   * CTA jobs   (sched_lane_cta_kernel): one CTA of 2..16 warps per job.
// FIFOs are assigned to lanes by the host (LPT on op count, soa.h LaneJob).
//
// Trace staging: each FIFO owns a ring of 8-op (128 B) shared-memory slots,
// filled by cp.async.bulk (the TMA bulk-copy engine) and completed on one
// mbarrier per slot; a lane refills a slot as soon as it has consumed it, so
// up to D-1 slots per FIFO are in flight while it computes.  The collective
// rendezvous slots live in shared memory; record times live in shared memory
// when they fit, else in global memory fronted by a tagged shared-memory cache
// (a wait almost always reads a record of the last few steps); the per-rank
// collective table is staged in shared memory or read through L1.
//
// Host syncs, termination and deadlock follow the round protocol of the warp
// kernel: the group iterates while any lane progresses (or waits for bytes in
// flight); when the group is idle the round ends, host syncs are resolved
// (sim.py:243-283), and a round without progress and with work left is the
// reference's SimDeadlockError (sim.py:382-402).
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace maya {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t SLOT = LANE_SLOT_OPS;           // ops per ring slot
constexpr uint32_t SLOT_LG = 3;
constexpr uint32_t SMASK = SLOT - 1;
static_assert((1u << SLOT_LG) == SLOT, "slot size");

template <typename T>
__device__ __forceinline__ T vld(const T *p) {
  return *(const volatile T *)p;
}
template <typename T>
__device__ __forceinline__ void vst(T *p, T v) {
  *(volatile T *)p = v;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// Global-memory accesses other threads (or other CTAs of a grid job) race on:
// relaxed at GPU scope (a generic volatile access would be system scope).
__device__ __forceinline__ uint32_t ld_relaxed_u32(const void *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int64_t ld_relaxed_s64(const void *p) {
  int64_t v;
  asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Collective rendezvous slot (sim.py:326-343) on a shared-memory ring or a
// global slot, with explicit address spaces: post = max(maxarr, ready) then
// count += 1 (release), returning the new count; count / maxarr reads acquire.
__device__ __forceinline__ uint32_t rdv_post(bool shared, CollSlot *cs, uint64_t ready) {
  uint32_t old;
  uint64_t mx;
  if (shared) {
    const uint32_t a = smem_u32(cs);
    asm volatile("atom.shared.max.u64 %0, [%1], %2;" : "=l"(mx) : "r"(a), "l"(ready) : "memory");
    asm volatile("fence.acq_rel.cta;" ::: "memory");
    asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(a + 8u) : "memory");
  } else {
    asm volatile("atom.global.max.u64 %0, [%1], %2;" : "=l"(mx) : "l"(&cs->maxarr), "l"(ready) : "memory");
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(&cs->count) : "memory");
  }
  (void)mx;
  return old + 1;
}
__device__ __forceinline__ uint32_t rdv_count(bool shared, const CollSlot *cs) {
  if (shared) {
    uint32_t v;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&cs->count)) : "memory");
    return v;
  }
  return ld_relaxed_u32(&cs->count);
}
__device__ __forceinline__ int64_t rdv_max(bool shared, const CollSlot *cs) {
  int64_t v;
  if (shared) {
    asm volatile("fence.acq_rel.cta;" ::: "memory");
    asm volatile("ld.volatile.shared.s64 %0, [%1];" : "=l"(v) : "r"(smem_u32(&cs->maxarr)) : "memory");
  } else {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    v = ld_relaxed_s64(&cs->maxarr);
  }
  return v;
}

__device__ __forceinline__ void mbar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// TMA bulk copy global -> shared, completion on the slot's mbarrier.  The
// slot's previous contents were consumed into registers by this same thread
// before the refill is issued (program order + data dependence).
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes,
                                          uint64_t *bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct __align__(16) LCtx {   // loop invariants of one FIFO (64 B)
  const ExecOp *ops;          // first op of the stream
  const uint32_t *cnt;        // counts of the rep, this stream (stride ns)
  uint64_t tl;                // timeline row of the first op
  uint32_t len, rank, ns, nsync;
  uint32_t ring, lgd;         // first ring slot, log2(slots) (0xff: no ring)
  uint32_t fire, rc;          // job-local record-table / collective-table base of the rank
  uint32_t delay, pad;        // job-local host-delay base of the rank
};
static_assert(sizeof(LCtx) == 64, "LCtx");

struct __align__(16) LSt {    // walker state (48 B)
  int64_t x;                  // completion time of the last op
  int64_t cdel;               // host delay of sync segment `seg`
  uint32_t i, bound, seg, flags;   // flags: ST_POSTED | ST_WFIRE | ST_WCOUNT
  uint32_t lim;               // dispatch limit for the resolved host syncs (per round)
  uint32_t wtgt;              // blocked: record index (ST_WFIRE) or arrival target (ST_WCOUNT)
  const uint32_t *waddr;      // blocked on ST_WCOUNT: the rendezvous counter
};
enum : uint32_t {
  ST_POSTED = 1,              // our arrival at op i's collective is posted
  ST_WFIRE = 2,               // op i waits for record wtgt
  ST_WCOUNT = 4,              // op i waits for *waddr >= wtgt
};
static_assert(sizeof(LSt) == 48, "LSt");

enum { ADV_IDLE = 0, ADV_PROG = 1, ADV_DATA = 2 };
#ifndef LANE_SUBSTEPS
#define LANE_SUBSTEPS 1
#endif
// Lockstep sub-steps per warp vote.  A job's steps are dependency-bound (~9
// of 32 lanes retire an op per step on C5), so several sub-steps between the
// votes let hand-offs inside the warp resolve without paying the votes and
// the round bookkeeping each time.  Warp jobs on folded runs and CTA jobs: 8
// (C5 8 x 10 k: 2.26 -> 2.20 ms; CTA jobs, 64 x 10 k: 2.23 -> 1.98 ms); grid
// jobs: 3 (512 x 10 k: 1.35 -> 1.23 ms, 2,048 x 1 k: 0.17 -> 0.155 ms).
#ifndef LANE_WARP_SUBSTEPS
#define LANE_WARP_SUBSTEPS 8
#endif
#ifndef LANE_GRID_SUBSTEPS
#define LANE_GRID_SUBSTEPS 3
#endif

#ifdef MAYA_PROFILE
// [0] loop cycles [1] group steps [2] data-only steps [3] step cycles
// [4] ops retired [5] data waits [6] (unused) [7] blocked visits
__device__ unsigned long long g_lprof[8];
#endif

struct FireEnt {              // tagged record-time cache entry
  int64_t val;
  int64_t tag;                // job-local record index, -1 empty
};

struct LaneSh {
  const JobHdr *J;
  CollSlot *ring;             // rendezvous rings (2 per comm) or null -> global slots
  const uint32_t *cb;         // call_base per comm (smem)
  uint32_t *hostk;
  LSt *st;
  LCtx *ctx;
  uint64_t *bars;
  ExecOp *rdata;
  int64_t *fire;              // record times: whole table in smem, or global backing
  FireEnt *fcache;            // tagged cache when `fire` is global
  uint32_t fmask;             // cache entries - 1
  const RCX *rcx;             // smem or global collective table
  int64_t *delay;             // job's host-delay table (global)
  const uint32_t *perm;       // lane -> FIFOs (K per lane, stride = group threads); null: w0 + lane
  uint32_t K;
  uint32_t w0, w1;            // the FIFOs of this group (a grid job's part; else the job)
  const uint32_t *comm_part;  // grid jobs: part holding all members of each comm (else global slots)
  uint32_t part;
  int record;
  bool fire_sm, rcx_sm;       // fire / rcx tables in shared memory
};

// ---- typed accesses --------------------------------------------------------

__device__ __forceinline__ int64_t ld_vol_shared_s64(const void *p) {
  int64_t v;
  asm volatile("ld.volatile.shared.s64 %0, [%1];" : "=l"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_vol_shared_u32(const void *p) {
  uint32_t v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ int64_t ld_vol_global_s64(const void *p) {
  int64_t v;
  asm volatile("ld.volatile.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Record times (REC writes, WAIT/ESYNC read).  When the job's table does not
// fit shared memory it lives in global memory, written through, and a tagged
// direct-mapped shared-memory cache answers the reads: a wait normally reads a
// record of the last few steps.  A cache miss is NOT proof that the record is
// unfired (a colliding record may have replaced the entry), so a miss reports
// "not yet" and the exact global lookup runs on a blocked wait's first step of
// every round -- a wait that missed is re-examined before the round can end
// idle, so no deadlock is declared on a stale miss.
__device__ __forceinline__ void fire_store(const LaneSh &sh, uint32_t idx, int64_t v) {
  if (sh.fire_sm) {
    asm volatile("st.volatile.shared.s64 [%0], %1;" ::"r"(smem_u32(sh.fire + idx)), "l"(v)
                 : "memory");
  } else {
    asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(sh.fire + idx), "l"(v) : "memory");
    asm volatile("st.volatile.shared.v2.s64 [%0], {%1, %2};" ::"r"(
                     smem_u32(sh.fcache + (idx & sh.fmask))),
                 "l"(v), "l"((int64_t)idx)
                 : "memory");
  }
}

// record time of job-local record index idx; -1: not fired (or, with
// full == false and a global table, not in the cache)
__device__ __forceinline__ int64_t fire_load(const LaneSh &sh, uint32_t idx, bool full) {
  if (sh.fire_sm) return ld_vol_shared_s64(sh.fire + idx);
  int64_t v, t;
  asm volatile("ld.volatile.shared.v2.s64 {%0, %1}, [%2];"
               : "=l"(v), "=l"(t)
               : "r"(smem_u32(sh.fcache + (idx & sh.fmask)))
               : "memory");
  if (t == (int64_t)idx) return v;
  return full ? ld_relaxed_s64(sh.fire + idx) : -1;
}

__device__ __forceinline__ RCX ld_rcx(const RCX *p, bool smem) {
  RCX r;
  if (smem) {
    uint64_t a, b2;
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b2) : "r"(smem_u32(p)));
    r.ent = a;
    r.wire = (int64_t)b2;
  } else {
    const longlong2 v = __ldg(reinterpret_cast<const longlong2 *>(p));
    r.ent = (uint64_t)v.x;
    r.wire = v.y;
  }
  return r;
}

// dispatch limit of a FIFO for the host syncs resolved so far
__device__ __forceinline__ uint32_t fifo_limit(const LaneSh &sh, const LCtx &c) {
  const uint32_t hk = sh.hostk[c.rank];
  return hk < c.nsync ? c.cnt[hk * c.ns] : c.len;
}

// Retire at most one op of FIFO (c, s).  IDLE: blocked or finished; DATA: the
// op's chunk is still in flight; PROG: an op retired or an arrival was posted.
struct RcxPf {                // next collective-table entry of a FIFO, prefetched
  RCX rx;
  uint32_t key;               // job-local table index of rx (0xFFFFFFFF: none)
};

// FAST: folded runs and no timeline (the kernel prelude and the timeline
// stores are compiled out); else both are decided at run time.
template <bool FAST = false>
__device__ __forceinline__ int lane_step(const DevBatch &b, const LaneSh &sh, const LCtx &c,
                                         LSt &s, int64_t &tmax, int &err, bool full,
                                         RcxPf *pf) {
  if (s.i >= s.lim) return ADV_IDLE;
  // a blocked op re-checks only its wake condition
  if (s.flags & ST_WFIRE) {
    if (fire_load(sh, s.wtgt, full) < 0) return ADV_IDLE;
    s.flags &= ~ST_WFIRE;
  } else if (s.flags & ST_WCOUNT) {
    const uint32_t cnt = __isShared(s.waddr) ? (uint32_t)ld_vol_shared_u32(s.waddr) : ld_relaxed_u32(s.waddr);
    if (cnt < s.wtgt) return ADV_IDLE;
    s.flags &= ~ST_WCOUNT;
  }
  while (s.i >= s.bound && s.seg < c.nsync) {   // next host-sync segment (rare)
    s.seg++;
    s.cdel = sh.delay[c.delay + s.seg];
    s.bound = s.seg < c.nsync ? c.cnt[s.seg * c.ns] : c.len;
  }
  longlong2 v;
  const bool ring = c.lgd != 0xffu;
  if (!FAST && ring && (s.i & SMASK) != 0 && !sh.record && !b.clen) {   // folded runs: no prelude
    // kernel prelude: up to 3 kernel ops of the staged chunk, operands < 2^61
    // (no sum can leave int64), before the one general op below
    constexpr int64_t LIM = (int64_t)1 << 61;
    const uint32_t slot = c.ring + ((s.i >> SLOT_LG) & ((1u << c.lgd) - 1u));
    const longlong2 *q = reinterpret_cast<const longlong2 *>(&sh.rdata[slot * SLOT]);
    uint32_t end = (s.i | SMASK) + 1u;
    end = min(end, min(s.lim, s.bound > s.i ? s.bound : s.lim));
    end = min(end, s.i + 3u);
    int64_t x = s.x;
    uint32_t i = s.i;
    for (; i < end; i++) {
      const longlong2 u = q[i & SMASK];
      const uint64_t wu = (uint64_t)u.y;
      const int64_t d = (int64_t)(wu >> 2);
      if ((wu & 3u) != TAG_KERN || d >= LIM || u.x >= LIM || x >= LIM || s.cdel >= LIM) break;
      const int64_t rd = u.x + s.cdel;
      x = (x > rd ? x : rd) + d;
    }
    if (i != s.i) {
      s.x = x;
      if (x > tmax) tmax = x;
      s.i = i;
      if ((i & SMASK) == 0 || i >= s.lim) {   // chunk end (refill) or limit: finish the step
        if ((i & SMASK) == 0) {
          const uint32_t dm = (1u << c.lgd) - 1u;
          const uint32_t nc = (i >> SLOT_LG) - 1u + (dm + 1u);
          const uint32_t first = nc << SLOT_LG;
          if (first < c.len) {
            const uint32_t n = min(SLOT, c.len - first);
            const uint32_t sl = c.ring + (nc & dm);
            bulk_load(&sh.rdata[sl * SLOT], c.ops + first, n * 16u, &sh.bars[sl]);
          }
        }
        return ADV_PROG;
      }
      if (i >= s.bound && s.seg < c.nsync) return ADV_PROG;
    }
  }
  if (ring) {
    const uint32_t chunk = s.i >> SLOT_LG, slot = c.ring + (chunk & ((1u << c.lgd) - 1u));
    if ((s.i & SMASK) == 0 && !mbar_test(&sh.bars[slot], (chunk >> c.lgd) & 1u)) return ADV_DATA;
    v = *reinterpret_cast<const longlong2 *>(&sh.rdata[slot * SLOT + (s.i & SMASK)]);
  } else {
    v = __ldg(reinterpret_cast<const longlong2 *>(c.ops + s.i));
    if ((s.i & 7u) == 0 && s.i + 16 < c.len)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(c.ops + s.i + 16));
  }
  const uint64_t wv = (uint64_t)v.y;
  const uint32_t tag = (uint32_t)(wv & 3u);
  const uint64_t pay = wv >> 2;
  const int64_t rdisp = v.x + s.cdel;
  const int64_t ready = s.x > rdisp ? s.x : rdisp;
  int64_t done;
  if (tag == TAG_KERN) {
    if (wv == EXEC_BAD) { err = MAYA_ST_ESTIMATION; return ADV_IDLE; }
    if (wv == EXEC_OVF) { err = MAYA_ST_OVERFLOW; return ADV_IDLE; }
    const int64_t d = (int64_t)pay;
    if (d > INT64_MAX - ready) { err = MAYA_ST_OVERFLOW; return ADV_IDLE; }
    done = ready + d;
  } else if (tag == TAG_REC) {
    fire_store(sh, c.fire + (uint32_t)pay, ready);
    done = ready;
  } else if (tag == TAG_WAIT) {
    if (pay == (EXEC_NONE >> 2)) return ADV_IDLE;   // never recorded: blocks forever
    const int64_t f = fire_load(sh, c.fire + (uint32_t)pay, full);
    if (f < 0) {
      s.flags |= ST_WFIRE;
      s.wtgt = c.fire + (uint32_t)pay;
      return ADV_IDLE;
    }
    done = ready > f ? ready : f;
  } else {                                         // collective rendezvous (sim.py:326-343)
    const uint32_t key = c.rc + (uint32_t)pay;
    const RCX rx = (pf && pf->key == key) ? pf->rx : ld_rcx(&sh.rcx[key], sh.rcx_sm);
    const int64_t w8 = rx.wire;
    const uint32_t nr = (uint32_t)(rx.ent >> 48);
    const uint32_t g = (uint32_t)(rx.ent >> 32) & 0xffffu;
    const uint32_t idx = (uint32_t)rx.ent;
    if (nr == 1) {
      if (w8 > INT64_MAX - ready) { err = MAYA_ST_OVERFLOW; return ADV_IDLE; }
      done = ready + w8;
    } else {
      CollSlot *cs;
      uint32_t target;
      const bool on_chip = sh.ring && (!sh.comm_part || sh.comm_part[g] == sh.part);
      if (on_chip) {   // on-chip rendezvous
        cs = sh.ring + 2 * g + (idx & 1u);
        target = ((idx >> 1) + 1u) * nr;
      } else {
        cs = b.cslots + sh.J->slots + sh.cb[g] + idx;
        target = nr;
      }
      if (!(s.flags & ST_POSTED)) {
        const uint32_t cnt = rdv_post(on_chip, cs, (uint64_t)ready);
        s.flags |= ST_POSTED;
        if (cnt > target) { err = MAYA_ST_INTERNAL; return ADV_IDLE; }
        if (cnt < target) {                         // posted; completes in a later step
          s.flags |= ST_WCOUNT;
          s.wtgt = target;
          s.waddr = &cs->count;
          return ADV_PROG;
        }
      } else if (rdv_count(on_chip, cs) < target) {
        s.flags |= ST_WCOUNT;
        s.wtgt = target;
        s.waddr = &cs->count;
        return ADV_IDLE;
      }
      const int64_t m = rdv_max(on_chip, cs);
      if (w8 > INT64_MAX - m) { err = MAYA_ST_OVERFLOW; return ADV_IDLE; }
      done = m + w8;
      s.flags &= ~ST_POSTED;
    }
    // collectives of a FIFO are consecutive in the table (pack.cpp): fetch the
    // next one now, it is consumed dozens of steps later
    if (pf && key + 1 < sh.J->n_rcolls) {
      pf->rx = ld_rcx(&sh.rcx[key + 1], sh.rcx_sm);
      pf->key = key + 1;
    }
  }
  if (!FAST && sh.record) {
    b.tl_start[c.tl + s.i] = ready;
    b.tl_end[c.tl + s.i] = done;
  }
  s.x = done;
  if (done > tmax) tmax = done;
  s.i++;
  if (ring && (s.i & SMASK) == 0) {   // chunk s.i/16 - 1 consumed: refill its slot D chunks ahead
    const uint32_t dm = (1u << c.lgd) - 1u;
    const uint32_t nc = (s.i >> SLOT_LG) - 1u + (dm + 1u);
    const uint32_t first = nc << SLOT_LG;
    if (first < c.len) {
      const uint32_t n = min(SLOT, c.len - first);
      const uint32_t slot = c.ring + (nc & dm);
      bulk_load(&sh.rdata[slot * SLOT], c.ops + first, n * 16u, &sh.bars[slot]);
    }
  }
  return ADV_PROG;
}

// Resolve the host syncs of rank r that the stream states allow
// (sim.py:243-263, 272-283): H' = max(H, X), host time = gap prefix + delay.
__device__ bool lane_host_step(const DevBatch &b, const LaneSh &sh, uint32_t r) {
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
        X = fire_load(sh, rr.fire + s.arg, true);
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
        const LSt &ws = sh.st[rr.walker + ls];
        if (ws.i < cnt) { ok = false; break; }
        if (ws.x > X) X = ws.x;
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

// Set up the job's shared-memory region (group-strided: tid in [0, nt)).
// The FIFOs [w0, w1) and ranks [r0, r1) of job j (the whole job, or one part of
// a grid job); state and host-sync arrays are indexed with job-local numbers.
__device__ void lane_setup(const DevBatch &b, uint32_t j, uint8_t *base, uint32_t tid,
                           uint32_t nt, LaneSh &sh, int record, LCtx &own, const LaneJob &LJ,
                           uint32_t w0, uint32_t w1, uint32_t r0, uint32_t r1) {
  const JobHdr &J = b.jobs[j];
  const LaneLayout L = lane_layout(w1 - w0, r1 - r0, J.n_comms, LJ.flags, LJ.n_slots, J.n_fire,
                                   J.n_rcolls, LJ.fc_log2);
  sh.J = &J;
  sh.ring = (LJ.flags & LANE_COLL_RING) ? (CollSlot *)(base + L.ring) : nullptr;
  uint32_t *cb = (uint32_t *)(base + L.cb);
  for (uint32_t g = tid; g < J.n_comms; g += nt) cb[g] = b.comms[J.comms + g].call_base;
  sh.cb = cb;
  if (sh.ring)
    for (uint32_t q = tid; q < 2 * J.n_comms; q += nt) sh.ring[q] = CollSlot{0, 0, 0};
  sh.hostk = (uint32_t *)(base + L.hostk) - r0;
  sh.st = (LJ.flags & LANE_ST_GLOBAL) ? (LSt *)(b.lane_gst + (size_t)J.walkers * 48)
                                      : (LSt *)(base + L.state) - w0;
  sh.w0 = w0;
  sh.w1 = w1;
  sh.comm_part = nullptr;
  sh.part = 0;
  // several FIFOs per lane: contexts in shared memory, else in global memory
  // (one FIFO per lane keeps its context in registers)
  sh.ctx = (LJ.flags & LANE_CTX_SMEM) ? (LCtx *)(base + L.ctx)
           : LJ.per_lane > 1          ? (LCtx *)(b.lane_gctx + (size_t)J.walkers * 64)
                                      : nullptr;
  sh.bars = (uint64_t *)(base + L.bars);
  sh.rdata = (ExecOp *)(base + L.rdata);
  sh.fire_sm = (LJ.flags & LANE_FIRE_SMEM) != 0;
  sh.fire = sh.fire_sm ? (int64_t *)(base + L.fire) : b.fire + J.fire;
  sh.fcache = (FireEnt *)(base + L.fcache);
  sh.fmask = LJ.fc_log2 ? (1u << LJ.fc_log2) - 1u : 0u;
  sh.rcx_sm = (LJ.flags & LANE_RCX_SMEM) != 0;
  sh.rcx = sh.rcx_sm ? (const RCX *)(base + L.rcx) : b.rcx + J.rcolls;
  sh.delay = b.delay + J.delay;
  sh.perm = b.lane_perm + LJ.perm;
  sh.K = LJ.per_lane;
  sh.record = record;
  if (sh.fire_sm)
    for (uint32_t q = tid; q < J.n_fire; q += nt) sh.fire[q] = -1;
  else if (LJ.fc_log2)
    for (uint32_t q = tid; q <= sh.fmask; q += nt) sh.fcache[q] = FireEnt{-1, -1};
  if (sh.rcx_sm) {
    const RCX *src = b.rcx + J.rcolls;
    RCX *dst = (RCX *)(base + L.rcx);
    for (uint32_t q = tid; q < J.n_rcolls; q += nt) dst[q] = src[q];
  }
  for (uint32_t r = r0 + tid; r < r1; r += nt) {
    sh.delay[b.ranks[J.ranks + r].delay] = 0;
    sh.hostk[r] = 0;
  }
  const uint32_t *wslot = b.lane_wslot + LJ.wslot - w0;
  for (uint32_t w = w0 + tid; w < w1; w += nt) {
    const Walker wk = b.walkers[J.walkers + w];
    const RankRec rr = b.ranks[J.ranks + wk.rank];
    const RepHdr &h = b.reps[rr.rep];
    const StreamRange sr = b.streams[h.streams + wk.stream];
    LCtx c;
    c.ops = b.exec + h.ops + sr.begin;
    c.cnt = (b.clen ? b.ccounts : b.counts) + h.counts + wk.stream;
    c.tl = J.timeline + rr.tl + sr.begin;
    c.len = b.clen ? b.clen[h.streams + wk.stream] : sr.len;
    c.rank = wk.rank;
    c.ns = h.n_streams;
    c.nsync = h.n_syncs;
    const uint32_t ws = wslot[w];
    c.ring = ws & 0x0fffffffu;
    c.lgd = (ws >> 28) == 0xfu ? 0xffu : (ws >> 28);
    c.fire = rr.fire;
    c.rc = rr.rslot;
    c.delay = rr.delay;
    c.pad = 0;
    if (sh.ctx) sh.ctx[w] = c;
    if (w == w0 + tid) own = c;   // one FIFO per lane: the context stays in registers
    LSt s{};
    s.bound = c.nsync ? c.cnt[0] : c.len;
    sh.st[w] = s;
    if (c.lgd != 0xffu) {
      for (uint32_t q = 0; q < (1u << c.lgd); q++) mbar_init(&sh.bars[c.ring + q]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      // prime the ring: the first D chunks
      for (uint32_t q = 0; q < (1u << c.lgd) && (q << SLOT_LG) < c.len; q++) {
        const uint32_t n = min(SLOT, c.len - (q << SLOT_LG));
        bulk_load(&sh.rdata[(c.ring + q) * SLOT], c.ops + (q << SLOT_LG), n * 16u, &sh.bars[c.ring + q]);
      }
    }
  }
}

// Wait for every bulk copy still targeting the region (no copy may land in
// shared memory after the job's CTA has exited); flag unfinished FIFOs.
__device__ bool lane_drain(const LaneSh &sh, uint32_t tid, uint32_t nt, const LCtx &own) {
  bool incomplete = false;
  for (uint32_t w = sh.w0 + tid; w < sh.w1; w += nt) {
    const LCtx c = sh.ctx ? sh.ctx[w] : own;
    const LSt s = sh.st[w];
    if (s.i < c.len) incomplete = true;
    if (c.lgd == 0xffu) continue;
    const uint32_t D = 1u << c.lgd;
    const uint32_t nchunks = (c.len + SMASK) >> SLOT_LG;
    const uint32_t issued = min(nchunks, (s.i >> SLOT_LG) + D);   // first D + one per chunk consumed
    for (uint32_t k = issued > D ? issued - D : 0; k < issued; k++)
      while (!mbar_test(&sh.bars[c.ring + (k & (D - 1))], (k >> c.lgd) & 1u)) {
      }
  }
  return incomplete;
}

// The FIFOs of one lane: K == 1 keeps the FIFO in registers for a whole
// round; K > 1 steps each FIFO from its shared-memory state.
struct LaneFifos {
  LCtx c;
  LSt s;
  RcxPf pf;
  bool one, valid;
};

__device__ __forceinline__ void fifos_begin_round(const LaneSh &sh, uint32_t tid, uint32_t nt,
                                                  LaneFifos &f) {
  if (f.one) {
    if (f.valid) {
      f.s = sh.st[sh.w0 + tid];
      f.s.lim = fifo_limit(sh, f.c);
    }
    return;
  }
  for (uint32_t k = 0; k < sh.K; k++) {
    const uint32_t w = sh.perm[k * nt + tid];
    if (w == 0xffffffffu) break;
    sh.st[w].lim = fifo_limit(sh, sh.ctx[w]);
  }
}

__device__ __forceinline__ void fifos_end_round(const LaneSh &sh, uint32_t tid, LaneFifos &f) {
  if (f.one && f.valid) sh.st[sh.w0 + tid] = f.s;
}

template <bool FAST = false, int SUB = LANE_SUBSTEPS>
__device__ __forceinline__ void fifos_step(const DevBatch &b, const LaneSh &sh, uint32_t tid,
                                           uint32_t nt, LaneFifos &f, int64_t &tmax, int &err,
                                           bool &prog, bool &data, bool full) {
  if (f.one) {
    // SUB lockstep sub-steps per group step: a hand-off between
    // FIFOs of the warp (record -> wait, last collective arrival) resolves
    // within one step; the __syncwarp orders the sub-steps' shared-memory
    // accesses across lanes
#pragma unroll 1
    for (int m = 0; m < SUB; m++) {
      int a = ADV_IDLE;
      if (f.valid) {
        a = lane_step<FAST>(b, sh, f.c, f.s, tmax, err, full && m == 0, sh.rcx_sm ? nullptr : &f.pf);
      }
      prog |= a == ADV_PROG;
      data |= a == ADV_DATA;
      __syncwarp();
    }
    return;
  }
  for (uint32_t k = 0; k < sh.K; k++) {
    const uint32_t w = sh.perm[k * nt + tid];
    if (w == 0xffffffffu) break;
    LSt s = sh.st[w];
    if (s.i >= s.lim) continue;
    const LCtx c = sh.ctx[w];
    int a = lane_step<FAST>(b, sh, c, s, tmax, err, full, nullptr);
    if (a != ADV_IDLE || err || (s.flags & (ST_WFIRE | ST_WCOUNT))) sh.st[w] = s;
    prog |= a == ADV_PROG;
    data |= a == ADV_DATA;
    if (err) break;
  }
}

struct EpiVals {       // per-thread partials of the job epilogue
  int64_t tmax;
  int64_t oom_t;
  int64_t peak;
  int32_t oom_rank;
  bool incomplete;
};

__device__ void epi_ranks(const DevBatch &b, const LaneSh &sh, uint32_t tid, uint32_t nt,
                          EpiVals &v, uint32_t r0, uint32_t r1) {
  const JobHdr &J = *sh.J;
  for (uint32_t r = r0 + tid; r < r1; r += nt) {
    const RankRec rr = b.ranks[J.ranks + r];
    const RepHdr &h = b.reps[rr.rep];
    const uint32_t k = sh.hostk[r];
    if (k < h.n_syncs) { v.incomplete = true; continue; }
    const int64_t hend = h.gend + sh.delay[rr.delay + h.n_syncs];
    if (hend > v.tmax) v.tmax = hend;
    const RepOut ro = b.repout[rr.rep];
    if (ro.peak > v.peak) v.peak = ro.peak;
    if (ro.first_exceed >= 0) {
      const MemRec m = b.mems[h.mems + ro.first_exceed];
      const int64_t t = m.gpre + sh.delay[rr.delay + m.seg];
      if (t < v.oom_t || (t == v.oom_t && (int32_t)r < v.oom_rank)) {
        v.oom_t = t;
        v.oom_rank = (int32_t)r;
      }
    }
  }
}

__device__ void write_result(const DevBatch &b, const JobHdr &J, maya_job_result *res, int err,
                             bool incomplete, int64_t tmax, int64_t peak, int32_t oom_rank,
                             int64_t rounds) {
  maya_job_result r = {};
  r.status = err ? err : (incomplete ? MAYA_ST_DEADLOCK : MAYA_ST_OK);
  r.total_ns = tmax;
  r.peak_mem_bytes = peak;
  r.first_oom_rank = -1;
  r.first_oom_seq = -1;
  if (oom_rank != INT32_MAX && !incomplete) {
    const RankRec rr = b.ranks[J.ranks + oom_rank];
    const RepHdr &h = b.reps[rr.rep];
    r.oom = 1;
    r.first_oom_rank = oom_rank;
    r.first_oom_seq = (int32_t)b.mems[h.mems + b.repout[rr.rep].first_exceed].seq;
  }
  r.dispatched_ops = J.dev_ops;
  r.completed_ops = J.dev_ops;
  r.rank_ops = J.rank_ops;
  r.rounds = rounds;
  *res = r;
}

__device__ void write_preset(const JobHdr &J, maya_job_result *res) {
  maya_job_result r = {};
  r.status = J.status;
  r.first_oom_rank = -1;
  r.first_oom_seq = -1;
  r.rank_ops = J.rank_ops;
  *res = r;
}

__device__ __forceinline__ int64_t warp_max64(int64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const int64_t u = __shfl_xor_sync(FULL, v, o);
    v = u > v ? u : v;
  }
  return v;
}

__device__ __forceinline__ void fifos_init(const LaneSh &sh, uint32_t tid, LaneFifos &f,
                                           const LCtx &own) {
  f.one = sh.K == 1;
  f.valid = false;
  f.pf.key = 0xffffffffu;
  if (f.one) {
    const uint32_t w = sh.perm ? sh.perm[tid] : (sh.w0 + tid < sh.w1 ? sh.w0 + tid : 0xffffffffu);
    f.valid = w != 0xffffffffu;   // (identity: w == w0 + tid when K == 1)
    if (f.valid) f.c = own;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// warp jobs: CTA = blockDim/32 independent jobs, one shared-memory region each

#ifndef LANE_WARP_MINB
#define LANE_WARP_MINB 2
#endif
template <bool FAST>
__global__ void __launch_bounds__(256, LANE_WARP_MINB) sched_lane_warp_kernel(DevBatch b, const int32_t *order,
                                                              uint32_t n_jobs, uint32_t region,
                                                              int record) {
  extern __shared__ __align__(128) uint8_t dsm[];
  const uint32_t lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const uint32_t slot = blockIdx.x * (blockDim.x >> 5) + wp;
  if (slot >= n_jobs) return;
  const uint32_t j = (uint32_t)order[slot];
  const JobHdr &J = b.jobs[j];
  maya_job_result *res = b.results + j;
  if (J.status != MAYA_ST_OK) {
    if (lane == 0) write_preset(J, res);
    return;
  }
  LaneSh sh;
#ifdef MAYA_PROFILE
  const long long tstart = clock64();
#endif
  LCtx own{};
  const LaneJob LJ = b.lane_jobs[j];
  lane_setup(b, j, dsm + wp * region, lane, 32, sh, record, own, LJ, 0, J.n_walkers, 0,
             J.n_ranks);
  __syncwarp();
  LaneFifos f;
  fifos_init(sh, lane, f, own);
  const uint32_t R = J.n_ranks;
  int64_t tmax = 0;
  int err = 0;
  int64_t rounds = 0;
  for (;;) {
    bool progress = false;
    for (uint32_t r = lane; r < R; r += 32) progress |= lane_host_step(b, sh, r);
    __syncwarp();
    fifos_begin_round(sh, lane, 32, f);
    for (bool full = true;; full = false) {
      bool prog = false, data = false;
#ifdef MAYA_PROFILE
      const long long t0 = clock64();
#endif
      fifos_step<FAST, FAST ? LANE_WARP_SUBSTEPS : LANE_SUBSTEPS>(b, sh, lane, 32, f, tmax, err,
                                                                  prog, data, full);
      __syncwarp();
      const bool ap = __any_sync(FULL, prog), ad = __any_sync(FULL, data);
#ifdef MAYA_PROFILE
      {
        const unsigned nops = __popc(__ballot_sync(FULL, prog));
        if (lane == 0) {
          atomicAdd(&g_lprof[3], (unsigned long long)(clock64() - t0));
          atomicAdd(&g_lprof[1], 1ull);
          atomicAdd(&g_lprof[4], (unsigned long long)nops);
          if (!ap && ad) atomicAdd(&g_lprof[2], 1ull);
        }
      }
#endif
      if (__any_sync(FULL, err != 0)) break;
      if (ap) {
        progress = true;
        continue;
      }
      if (!ad) break;
    }
    fifos_end_round(sh, lane, f);
    __syncwarp();
    rounds++;
    if (__any_sync(FULL, err != 0)) {
      err = (int)__reduce_max_sync(FULL, (unsigned)err);
      break;
    }
    if (!__any_sync(FULL, progress)) break;
  }
#ifdef MAYA_PROFILE
  if (lane == 0) atomicAdd(&g_lprof[0], (unsigned long long)(clock64() - tstart));
#endif
  bool incomplete = lane_drain(sh, lane, 32, own);
  __syncwarp();
  EpiVals v{tmax, INT64_MAX, 0, INT32_MAX, incomplete};
  epi_ranks(b, sh, lane, 32, v, 0, J.n_ranks);
  incomplete = __any_sync(FULL, v.incomplete);
  const int64_t tm = warp_max64(v.tmax);
  const int64_t pk = warp_max64(v.peak);
  // first OOM: min (time, rank)
  int64_t ot = v.oom_t;
  int32_t orank = v.oom_rank;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const int64_t t2 = __shfl_xor_sync(FULL, ot, o);
    const int32_t r2 = __shfl_xor_sync(FULL, orank, o);
    if (t2 < ot || (t2 == ot && r2 < orank)) { ot = t2; orank = r2; }
  }
  if (lane == 0) write_result(b, J, res, err, incomplete, tm, pk, orank, rounds);
}

// ---------------------------------------------------------------------------
// CTA jobs: one CTA of 2..16 warps per job

__global__ void __launch_bounds__(LANE_MAX_THREADS, 1)
    sched_lane_cta_kernel(DevBatch b, const int32_t *order, int record) {
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ unsigned long long s_tmax;
  __shared__ int s_err, s_incomplete, s_active, s_oom_rank;
  __shared__ long long s_peak, s_oom_t;

  const uint32_t j = (uint32_t)order[blockIdx.x];
  const JobHdr &J = b.jobs[j];
  maya_job_result *res = b.results + j;
  const uint32_t tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
  const uint32_t NW = nt >> 5;
  if (J.status != MAYA_ST_OK) {
    if (tid == 0) write_preset(J, res);
    return;
  }
  LaneSh sh;
  LCtx own{};
  const LaneJob LJ = b.lane_jobs[j];
  lane_setup(b, j, dsm, tid, nt, sh, record, own, LJ, 0, J.n_walkers, 0, J.n_ranks);
  if (tid == 0) {
    s_tmax = 0;
    s_err = 0;
    s_incomplete = 0;
    s_peak = 0;
    s_oom_t = INT64_MAX;
    s_oom_rank = INT32_MAX;
  }
  __syncthreads();
  LaneFifos f;
  fifos_init(sh, tid, f, own);
  const uint32_t R = J.n_ranks;
  int64_t tmax = 0;
  int err = 0;
  int64_t rounds = 0;
  for (;;) {
    int progress = 0;
    for (uint32_t r = tid; r < R; r += nt) progress |= lane_host_step(b, sh, r);
    if (tid == 0) s_active = (int)NW;
    __syncthreads();
    fifos_begin_round(sh, tid, nt, f);
    bool idle = false;
    for (uint32_t spin = 0;; spin++) {
      bool prog = false, data = false;
      fifos_step<false, LANE_WARP_SUBSTEPS>(b, sh, tid, nt, f, tmax, err, prog, data,
                                            spin == 0 && !idle);
      if (__any_sync(FULL, err != 0)) {
        if (err) atomicMax(&s_err, err);
        __syncwarp();
      }
      if (vld(&s_err) != 0) {
        if (!idle && lane == 0) atomicSub(&s_active, 1);
        break;
      }
      if (__any_sync(FULL, prog)) {
        progress = 1;
        if (idle) {
          if (lane == 0) atomicAdd(&s_active, 1);
          idle = false;
        }
        spin = 0;
        continue;
      }
      if (__any_sync(FULL, data)) continue;     // bytes in flight: not idle
      if (!idle) {
        if (lane == 0) atomicSub(&s_active, 1);
        idle = true;
      }
      __syncwarp();
      if (vld(&s_active) <= 0) break;
      if (spin > 16) __nanosleep(64);
    }
    fifos_end_round(sh, tid, f);
    rounds++;
    if (vld(&s_err) != 0) progress = 0;
    if (!__syncthreads_or(progress)) break;
  }
  if (lane_drain(sh, tid, nt, own)) s_incomplete = 1;
  EpiVals v{tmax, INT64_MAX, 0, INT32_MAX, false};
  epi_ranks(b, sh, tid, nt, v, 0, J.n_ranks);
  if (v.incomplete) s_incomplete = 1;
  atomicMax(&s_tmax, (unsigned long long)v.tmax);
  atomicMax(&s_peak, (long long)v.peak);
  if (v.oom_rank != INT32_MAX) atomicMin(&s_oom_t, (long long)v.oom_t);
  __syncthreads();
  if (v.oom_rank != INT32_MAX && v.oom_t == s_oom_t) atomicMin(&s_oom_rank, v.oom_rank);
  __syncthreads();
  if (tid == 0)
    write_result(b, J, res, s_err, s_incomplete != 0, (int64_t)s_tmax, s_peak, s_oom_rank, rounds);
}


// ---------------------------------------------------------------------------
// grid jobs: a job too large for one CTA runs on several co-resident CTAs
// (rank-aligned FIFO ranges, one FIFO per thread).  The round protocol of the
// CTA kernel is lifted to the job: one job-wide counter of walking warps in
// global memory, collectives through global slots, and a job-wide barrier
// between rounds (host syncs, termination and deadlock decided there).

static constexpr uint32_t GRID_THREADS = 256;

__device__ void grid_barrier(GridSync *gs, uint32_t n_parts, int reset_active) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = vld(&gs->gen);
    __threadfence();
    if (atomicAdd(&gs->arrive, 1u) == n_parts - 1) {
      vst(&gs->arrive, 0u);
      if (reset_active >= 0) {
        vst(&gs->active, reset_active);
        vst(&gs->progress, 0);
      }
      __threadfence();
      atomicAdd(&gs->gen, 1u);
    } else {
      while (vld(&gs->gen) == g) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(GRID_THREADS, 1)
    sched_lane_grid_kernel(DevBatch b, uint32_t p0, int record) {
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ unsigned long long s_tmax;
  __shared__ int s_err, s_incomplete, s_oom_rank, s_any;
  __shared__ long long s_peak, s_oom_t;
  const GridPart P = b.grid_parts[p0 + blockIdx.x];
  const uint32_t j = P.job;
  const JobHdr &J = b.jobs[j];
  GridSync *gs = b.gsync + j;
  const uint32_t tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
  LaneJob LJ{};
  LJ.flags = P.flags;
  LJ.n_slots = P.n_slots;
  LJ.wslot = P.wslot;
  LJ.per_lane = 1;
  LJ.fc_log2 = P.fc_log2;
  LaneSh sh;
  LCtx own{};
  lane_setup(b, j, dsm, tid, nt, sh, record, own, LJ, P.w0, P.w1, P.r0, P.r1);
  sh.perm = nullptr;
  sh.K = 1;
  if (sh.ring) {   // communicators whose members all live in this part meet on chip
    sh.comm_part = b.comm_part + J.comms;
    sh.part = P.part;
  }
  if (tid == 0) {
    s_tmax = 0;
    s_err = 0;
    s_incomplete = 0;
    s_peak = 0;
    s_oom_t = INT64_MAX;
    s_oom_rank = INT32_MAX;
  }
  LaneFifos f;
  fifos_init(sh, tid, f, own);
  if (P.part == 0 && tid == 0) {   // the job-wide minima start at +inf (scratch is zeroed)
    vst(&gs->oom_t, (long long)INT64_MAX);
    vst(&gs->oom_rank, (int)INT32_MAX);
  }
  grid_barrier(gs, P.n_parts, (int)P.warps_total);
  int64_t tmax = 0;
  int err = 0;
  int64_t rounds = 0;
  for (;;) {
    int progress = 0;
    for (uint32_t r = P.r0 + tid; r < P.r1; r += nt) progress |= lane_host_step(b, sh, r);
    __syncthreads();
    fifos_begin_round(sh, tid, nt, f);
    bool idle = false;
    for (uint32_t spin = 0;; spin++) {
      bool prog = false, data = false;
      fifos_step<false, LANE_GRID_SUBSTEPS>(b, sh, tid, nt, f, tmax, err, prog, data,
                                            spin == 0 && !idle);
      if (__any_sync(FULL, err != 0)) {
        if (err && lane == 0) atomicMax(&gs->err, err);
        if (err) atomicMax(&s_err, err);
        __syncwarp();
      }
      if ((int)ld_relaxed_u32(&gs->err) != 0) {
        if (!idle && lane == 0) atomicSub(&gs->active, 1);
        break;
      }
      if (__any_sync(FULL, prog)) {
        progress = 1;
        if (idle) {
          if (lane == 0) atomicAdd(&gs->active, 1);
          idle = false;
        }
        spin = 0;
        continue;
      }
      if (__any_sync(FULL, data)) continue;     // bytes in flight: not idle
      if (!idle) {
        if (lane == 0) atomicSub(&gs->active, 1);
        idle = true;
      }
      __syncwarp();
      if ((int)ld_relaxed_u32(&gs->active) <= 0) break;   // every warp of the job is idle
      if (spin > 16) __nanosleep(128);
    }
    fifos_end_round(sh, tid, f);
    rounds++;
    if (__syncthreads_or(progress) && tid == 0) atomicOr(&gs->progress, 1);
    grid_barrier(gs, P.n_parts, -1);            // the round is over everywhere
    if (tid == 0) s_any = vld(&gs->progress) && !vld(&gs->err);
    grid_barrier(gs, P.n_parts, (int)P.warps_total);   // read; reset for the next round
    if (!s_any) break;
  }
  if (lane_drain(sh, tid, nt, own)) s_incomplete = 1;
  EpiVals v{tmax, INT64_MAX, 0, INT32_MAX, false};
  epi_ranks(b, sh, tid, nt, v, P.r0, P.r1);
  if (v.incomplete) s_incomplete = 1;
  atomicMax(&s_tmax, (unsigned long long)v.tmax);
  atomicMax(&s_peak, (long long)v.peak);
  if (v.oom_rank != INT32_MAX) atomicMin(&s_oom_t, (long long)v.oom_t);
  __syncthreads();
  if (tid == 0) {
    atomicMax(&gs->tmax, s_tmax);
    atomicMax(&gs->peak, s_peak);
    atomicMin(&gs->oom_t, s_oom_t);
    if (s_incomplete) atomicOr(&gs->incomplete, 1);
  }
  grid_barrier(gs, P.n_parts, -1);
  const long long got = vld(&gs->oom_t);
  if (v.oom_rank != INT32_MAX && v.oom_t == got) atomicMin(&s_oom_rank, v.oom_rank);
  __syncthreads();
  if (tid == 0 && s_oom_rank != INT32_MAX) atomicMin(&gs->oom_rank, s_oom_rank);
  grid_barrier(gs, P.n_parts, -1);
  if (P.part == 0 && tid == 0)
    write_result(b, J, b.results + j, vld(&gs->err), vld(&gs->incomplete) != 0,
                 (int64_t)vld(&gs->tmax), vld(&gs->peak), vld(&gs->oom_rank), rounds);
}

int grid_max_ctas(uint32_t smem) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sched_lane_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)LANE_SMEM_CAP);
    attr = true;
  }
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sched_lane_grid_kernel, GRID_THREADS,
                                                smem);
  return per_sm * sms;
}

int launch_schedule_grid(const DevBatch &b, uint32_t p0, uint32_t p1, int record, uint32_t smem,
                         cudaStream_t s) {
  if (p1 <= p0) return 0;
  grid_max_ctas(smem);   // sets the shared-memory attribute
  DevBatch bb = b;
  uint32_t pp = p0;
  int rec = record;
  void *args[] = {&bb, &pp, &rec};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void *)sched_lane_grid_kernel,
                                                    dim3(p1 - p0), dim3(GRID_THREADS), args,
                                                    smem, s);
  return e == cudaSuccess ? 0 : -1;
}

int lane_prof_read(unsigned long long *out8, int reset) {
#ifdef MAYA_PROFILE
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out8, g_lprof, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_lprof, z, sizeof z);
  }
  return 1;
#else
  (void)out8;
  (void)reset;
  return 0;
#endif
}

void launch_schedule_lane_warp(const DevBatch &b, const int32_t *order, uint32_t n,
                               uint32_t warps_per_cta, uint32_t region, int record,
                               cudaStream_t s) {
  if (!n) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sched_lane_warp_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)LANE_SMEM_CAP);
    cudaFuncSetAttribute(sched_lane_warp_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)LANE_SMEM_CAP);
    attr = true;
  }
  const uint32_t grid = (n + warps_per_cta - 1) / warps_per_cta;
  if (b.clen && !record)   // folded runs, no timeline
    sched_lane_warp_kernel<true><<<grid, warps_per_cta * 32, warps_per_cta * region, s>>>(
        b, order, n, region, 0);
  else
    sched_lane_warp_kernel<false><<<grid, warps_per_cta * 32, warps_per_cta * region, s>>>(
        b, order, n, region, record);
}

void launch_schedule_lane(const DevBatch &b, const int32_t *order, uint32_t n, uint32_t threads,
                          int record, uint32_t smem, cudaStream_t s) {
  if (!n) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sched_lane_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)LANE_SMEM_CAP);
    attr = true;
  }
  sched_lane_cta_kernel<<<n, threads, smem, s>>>(b, order, record);
}

}  // namespace maya
