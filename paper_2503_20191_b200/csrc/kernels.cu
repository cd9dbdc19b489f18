// sm_100a kernels of the batched trace-driven simulator.
//
//   estimate_features  RooflineEstimator.estimate_kernel  estimate.py:120-134
//   estimate_wire      collective_estimate                estimate.py:79-100
//   memscan            memory accounting of _advance_host sim.py:235-242
//   schedule           simulate()/_Sim.run as a max-plus fixpoint   sim.py:222-380
//   topk               _rank / SearchResult.best           search.py:349-357
//
// The scheduler exploits that the event-driven simulation is a monotone
// max-plus system: every op's completion time is
//     ready = max(dispatch, done(prev op on the stream))
//     KERN  done = ready + dur          REC  fire = done = ready
//     WAIT  done = max(ready, fire)     COLL done = max_members(ready) + wire
// and host dispatch time is the gap prefix plus the delay accumulated at host
// syncs.  One CTA simulates one job; each thread walks (rank, stream) FIFOs
// until it meets an unresolved dependency; CTA-wide rounds separate host-sync
// resolution from stream progress, and collectives rendezvous through
// atomics on a per-(comm, call) slot.  A round without progress and with work
// left is exactly the reference's deadlock condition (sim.py:382-402).
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace maya {

typedef unsigned __int128 u128;

// ---------------------------------------------------------------------------
// exact integer helpers (estimate.py:_ceil_div with Python big ints)

__device__ __forceinline__ bool mul_u128_u64(u128 a, uint64_t b, u128 *r) {
  uint64_t alo = (uint64_t)a, ahi = (uint64_t)(a >> 64);
  u128 p0 = (u128)alo * b;
  u128 p1 = (u128)ahi * b;
  if ((uint64_t)(p1 >> 64) != 0) return false;
  u128 hi = (u128)(uint64_t)p1 << 64;
  u128 s = p0 + hi;
  if (s < p0) return false;
  *r = s;
  return true;
}

// ceil(a / b) into int64; false on overflow
__device__ __forceinline__ bool ceil_div_i64(u128 a, u128 b, int64_t *out) {
  u128 q = a / b;
  if (q * b != a) q += 1;
  if (q > (u128)INT64_MAX) return false;
  *out = (int64_t)q;
  return true;
}

// ---------------------------------------------------------------------------
// estimators

__global__ void estimate_features_kernel(DevBatch b, DevTables t) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b.n_feats) return;
  Feature f = b.feats[i];
  if (f.fixed >= 0) { b.feat_ns[i] = f.fixed; return; }
  const maya_device_params &dev = t.devs[f.device];
  int64_t compute = 0, memory = 0;
  bool ok = true;
  if (f.flops > 0) {
    int64_t peak = (f.dtype >= 0 && f.dtype < MAYA_MAX_DTYPES) ? dev.peak_flops[f.dtype] : 0;
    if (peak <= 0 || f.op_kind < 0 || f.op_kind >= t.n_op_kinds) {
      ok = false;  // EstimationError: no peak rate for dtype (estimate.py:124-127)
    } else {
      u128 num, den;
      ok = mul_u128_u64((u128)(uint64_t)f.flops * 1000000000ull, (uint64_t)t.eff_den[f.op_kind],
                        &num);
      den = (u128)(uint64_t)peak * (uint64_t)t.eff_num[f.op_kind];
      if (ok) ok = ceil_div_i64(num, den, &compute);
    }
  }
  if (ok && f.bytes > 0)
    ok = ceil_div_i64((u128)(uint64_t)f.bytes * 1000000000ull, (u128)(uint64_t)dev.hbm_bytes_per_s,
                      &memory);
  int64_t m = compute > memory ? compute : memory;
  if (ok && m > INT64_MAX - t.overhead_ns) ok = false;
  if (!ok) {
    b.feat_ns[i] = -1;
    atomicOr(b.err_flag, 1);
    return;
  }
  b.feat_ns[i] = m + t.overhead_ns;
}

__global__ void estimate_wire_kernel(DevBatch b, DevTables t) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b.n_slots) return;
  SlotRec s = b.slots[i];
  if (s.kind < 0) { b.wire[i] = 0; return; }
  if (s.fixed >= 0) { b.wire[i] = s.fixed; return; }
  int64_t n = s.nranks;
  if (n < 1) { b.wire[i] = -1; atomicOr(b.err_flag, 2); return; }
  if (n == 1) { b.wire[i] = 0; return; }
  const maya_device_params &dev = t.devs[s.device];
  int li = s.topo == 0 ? 0 : 1;  // mixed priced at inter-host rates (cluster.py:55-59)
  uint64_t a = (uint64_t)dev.alpha_ns[li], beta = (uint64_t)dev.beta_bytes_per_s[li];
  uint64_t steps = (s.kind == 0) ? 2 * (uint64_t)(n - 1) : (s.kind <= 2 ? (uint64_t)(n - 1) : 1);
  u128 num;
  bool ok = mul_u128_u64((u128)(uint64_t)s.bytes * 1000000000ull, steps, &num);
  u128 den = (s.kind <= 2) ? (u128)(uint64_t)n * beta : (u128)beta;
  int64_t bw = 0;
  if (ok) ok = ceil_div_i64(num, den, &bw);
  u128 lat = (u128)steps * a;
  if (ok && (lat > (u128)INT64_MAX || (int64_t)lat > INT64_MAX - bw)) ok = false;
  if (!ok) { b.wire[i] = -1; atomicOr(b.err_flag, 2); return; }
  b.wire[i] = (int64_t)lat + bw;
}

void launch_estimate(const DevBatch &b, const DevTables &t, cudaStream_t s) {
  if (b.n_feats) estimate_features_kernel<<<(b.n_feats + 255) / 256, 256, 0, s>>>(b, t);
  if (b.n_slots) estimate_wire_kernel<<<(b.n_slots + 255) / 256, 256, 0, s>>>(b, t);
}

// ---------------------------------------------------------------------------
// memory: peak = max(0, max prefix of deltas); first prefix > capacity.
// One warp per representative trace.

__global__ void memscan_kernel(DevBatch b) {
  uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (warp >= b.n_reps) return;
  const RepHdr h = b.reps[warp];
  const int64_t cap = b.jobs[h.job].capacity;
  int64_t run = 0, peak = 0;
  int32_t first = -1;
  for (uint32_t base = 0; base < h.n_mems; base += 32) {
    uint32_t k = base + lane;
    int64_t v = k < h.n_mems ? b.mems[h.mems + k].delta : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    int64_t s = run + v;
    int64_t m = (k < h.n_mems) ? s : INT64_MIN;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      int64_t u = __shfl_xor_sync(0xffffffffu, m, o);
      m = u > m ? u : m;
    }
    if (m > peak) peak = m;
    if (first < 0) {
      unsigned bal = __ballot_sync(0xffffffffu, k < h.n_mems && s > cap);
      if (bal) first = (int32_t)(base + __ffs(bal) - 1);
    }
    run = __shfl_sync(0xffffffffu, s, 31);
  }
  if (lane == 0) b.repout[warp] = RepOut{peak, first, 0};
}

void launch_memscan(const DevBatch &b, cudaStream_t s) {
  if (b.n_reps) memscan_kernel<<<(b.n_reps * 32 + 255) / 256, 256, 0, s>>>(b);
}

// ---------------------------------------------------------------------------
// scheduler

static constexpr int SCHED_THREADS = 256;

template <typename T>
__device__ __forceinline__ T vload(const T *p) {
  return *(const volatile T *)p;
}
template <typename T>
__device__ __forceinline__ void vstore(T *p, T v) {
  *(volatile T *)p = v;
}

struct SchedCtx {
  const JobHdr *J;
  WState *ws;        // [n_walkers] walkers, then [n_ranks] host states (i = resolved syncs)
  int64_t *fire;     // job base
  int64_t *delay;    // job base
  int record;
};

// Advance one (rank, stream) walker as far as its dependencies allow.
// Returns true if it made progress; sets *err on estimation/overflow/internal.
__device__ bool advance_walker(const DevBatch &b, const SchedCtx &c, uint32_t w, int64_t &tmax,
                               int &err) {
  const JobHdr &J = *c.J;
  const Walker wk = b.walkers[J.walkers + w];
  const RankRec rr = b.ranks[J.ranks + wk.rank];
  const RepHdr &h = b.reps[rr.rep];
  const StreamRange sr = b.streams[h.streams + wk.stream];
  WState st = c.ws[w];
  if (st.i >= sr.len) return false;
  const uint32_t hk = vload(&c.ws[J.n_walkers + wk.rank].i);
  const Op *ops = b.ops + h.ops + sr.begin;
  int64_t *fire = c.fire + rr.fire;
  const int64_t *delay = c.delay + rr.delay;
  int64_t x = st.x;
  uint32_t i = st.i, flags = st.flags;
  uint32_t cseg = 0;
  int64_t cdel = 0;
  bool adv = false;
  while (i < sr.len) {
    const Op op = ops[i];
    const uint32_t seg = op_seg(op.meta);
    if (seg > hk) break;  // not dispatched yet: host blocked at an earlier sync
    if (seg != cseg) { cseg = seg; cdel = delay[seg]; }
    int64_t ready = op.disp + cdel;
    if (ready < x) ready = x;
    int64_t nx;
    const uint32_t tag = op_tag(op.meta);
    if (tag == TAG_KERN) {
      const int64_t d = b.feat_ns[J.feats + op.arg];
      if (d < 0) { err = MAYA_ST_ESTIMATION; break; }
      if (d > INT64_MAX - ready) { err = MAYA_ST_OVERFLOW; break; }
      nx = ready + d;
    } else if (tag == TAG_REC) {
      vstore(&fire[op.arg], ready);
      nx = ready;
    } else if (tag == TAG_WAIT) {
      if (op.arg == NO_REC) break;
      const int64_t f = vload(&fire[op.arg]);
      if (f < 0) break;
      nx = ready > f ? ready : f;
    } else {  // TAG_COLL: rendezvous of all members (sim.py:326-343)
      const uint32_t lc = b.coll_lc[h.colls + op.arg];
      const uint32_t ci = b.coll_idx[h.colls + op.arg];
      const uint32_t g = b.rank_comm[J.rank_comm + rr.comm + lc];
      const CommRec cm = b.comms[J.comms + g];
      const uint64_t slot = J.slots + cm.call_base + ci;
      CollSlot *cs = b.cslots + slot;
      if (!(flags & 1u)) {
        atomicMax(&cs->maxarr, (unsigned long long)ready);
        __threadfence_block();
        const uint32_t old = atomicAdd(&cs->count, 1u);
        flags |= 1u;
        adv = true;
        if (old + 1 > (uint32_t)cm.nranks) { err = MAYA_ST_INTERNAL; break; }
        if (old + 1 < (uint32_t)cm.nranks) break;
      } else if (vload(&cs->count) < (uint32_t)cm.nranks) {
        break;
      }
      __threadfence_block();
      const int64_t m = (int64_t)vload(&cs->maxarr);
      const int64_t wt = b.wire[slot];
      if (wt > INT64_MAX - m) { err = MAYA_ST_OVERFLOW; break; }
      nx = m + wt;
      flags = 0;
    }
    if (c.record) {
      const uint64_t t = J.timeline + rr.tl + sr.begin + i;
      b.tl_start[t] = ready;
      b.tl_end[t] = nx;
    }
    x = nx;
    i++;
    adv = true;
  }
  c.ws[w] = WState{x, i, flags};
  if (x > tmax) tmax = x;
  return adv;
}

// Resolve as many host syncs of rank r as the stream states allow
// (sim.py:243-263, 272-283): H' = max(H, X) with H = gap prefix + delay.
__device__ bool advance_host(const DevBatch &b, const SchedCtx &c, uint32_t r) {
  const JobHdr &J = *c.J;
  const RankRec rr = b.ranks[J.ranks + r];
  const RepHdr &h = b.reps[rr.rep];
  if (h.n_syncs == 0) return false;
  uint32_t k = c.ws[J.n_walkers + r].i;
  if (k >= h.n_syncs) return false;
  int64_t d = c.delay[rr.delay + k];
  bool adv = false;
  while (k < h.n_syncs) {
    const SyncRec s = b.syncs[h.syncs + k];
    int64_t X = INT64_MIN;
    bool ok = true;
    if (s.type == SYNC_ESYNC) {
      if (s.arg == NO_REC) {
        ok = false;
      } else {
        X = vload(&c.fire[rr.fire + s.arg]);
        ok = X >= 0;
      }
    } else {
      uint32_t s0 = 0, s1 = h.n_streams;
      if (s.type == SYNC_SSYNC) {
        if (s.arg == NO_REC) { s0 = s1 = 0; } else { s0 = s.arg; s1 = s.arg + 1; }
      }
      for (uint32_t ls = s0; ls < s1; ls++) {
        const uint32_t cnt = b.counts[h.counts + s.cnt + ls];
        if (cnt == 0) continue;
        const WState w = c.ws[rr.walker + ls];
        if (w.i < cnt) { ok = false; break; }
        if (w.x > X) X = w.x;
      }
    }
    if (!ok) break;
    if (X > s.gpre + d) d = X - s.gpre;
    k++;
    c.delay[rr.delay + k] = d;
    adv = true;
  }
  c.ws[J.n_walkers + r].i = k;
  return adv;
}

__global__ void __launch_bounds__(SCHED_THREADS) schedule_kernel(DevBatch b, int record) {
  __shared__ WState s_states[SMEM_STATES];
  __shared__ unsigned long long s_tmax;
  __shared__ int s_err, s_incomplete;
  __shared__ long long s_oom_t;
  __shared__ int s_oom_rank;
  __shared__ long long s_peak;

  const uint32_t j = b.order ? (uint32_t)b.order[blockIdx.x] : blockIdx.x;
  const JobHdr &J = b.jobs[j];
  maya_job_result *res = b.results + j;
  if (J.status != MAYA_ST_OK) {
    if (threadIdx.x == 0) {
      maya_job_result r = {};
      r.status = J.status;
      r.first_oom_rank = -1;
      r.first_oom_seq = -1;
      r.rank_ops = J.rank_ops;
      *res = r;
    }
    return;
  }
  const uint32_t W = J.n_walkers, R = J.n_ranks, S = W + R;
  SchedCtx c;
  c.J = &J;
  c.ws = (S <= (uint32_t)SMEM_STATES) ? s_states : b.wstate + J.wstate;
  c.fire = b.fire + J.fire;
  c.delay = b.delay + J.delay;
  c.record = record;
  const uint32_t tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) {
    s_tmax = 0;
    s_err = 0;
    s_incomplete = 0;
    s_oom_t = INT64_MAX;
    s_oom_rank = INT32_MAX;
    s_peak = 0;
  }
  for (uint32_t w = tid; w < S; w += nt) c.ws[w] = WState{0, 0, 0};
  for (uint32_t r = tid; r < R; r += nt) c.delay[b.ranks[J.ranks + r].delay] = 0;
  __syncthreads();

  int64_t tmax = 0;
  int err = 0;
  int64_t rounds = 0;
  for (;;) {
    int progress = 0;
    for (uint32_t r = tid; r < R; r += nt) progress |= advance_host(b, c, r);
    __syncthreads();
    for (uint32_t w = tid; w < W; w += nt) progress |= advance_walker(b, c, w, tmax, err);
    rounds++;
    if (err) { atomicMax(&s_err, err); progress = 0; }
    if (!__syncthreads_or(progress)) break;
  }
  // completion + host end time (the trailing gaps extend the makespan, sim.py:365-366)
  for (uint32_t w = tid; w < W; w += nt) {
    const Walker wk = b.walkers[J.walkers + w];
    const RankRec rr = b.ranks[J.ranks + wk.rank];
    const StreamRange sr = b.streams[b.reps[rr.rep].streams + wk.stream];
    if (c.ws[w].i < sr.len) s_incomplete = 1;
  }
  for (uint32_t r = tid; r < R; r += nt) {
    const RankRec rr = b.ranks[J.ranks + r];
    const RepHdr &h = b.reps[rr.rep];
    const uint32_t k = c.ws[W + r].i;
    if (k < h.n_syncs) { s_incomplete = 1; continue; }
    const int64_t hend = h.gend + c.delay[rr.delay + h.n_syncs];
    if (hend > tmax) tmax = hend;
    const RepOut ro = b.repout[rr.rep];
    atomicMax(&s_peak, (long long)ro.peak);
    if (ro.first_exceed >= 0) {
      const MemRec m = b.mems[h.mems + ro.first_exceed];
      const int64_t t = m.gpre + c.delay[rr.delay + m.seg];
      atomicMin(&s_oom_t, (long long)t);
    }
  }
  atomicMax(&s_tmax, (unsigned long long)tmax);
  __syncthreads();
  for (uint32_t r = tid; r < R; r += nt) {
    const RankRec rr = b.ranks[J.ranks + r];
    const RepOut ro = b.repout[rr.rep];
    if (ro.first_exceed >= 0 && !s_incomplete) {
      const RepHdr &h = b.reps[rr.rep];
      const MemRec m = b.mems[h.mems + ro.first_exceed];
      if (m.gpre + c.delay[rr.delay + m.seg] == s_oom_t) atomicMin(&s_oom_rank, (int)r);
    }
  }
  __syncthreads();
  if (tid == 0) {
    maya_job_result r = {};
    r.status = s_err ? s_err : (s_incomplete ? MAYA_ST_DEADLOCK : MAYA_ST_OK);
    r.total_ns = (int64_t)s_tmax;
    r.peak_mem_bytes = s_peak;
    r.first_oom_rank = -1;
    r.first_oom_seq = -1;
    if (s_oom_rank != INT32_MAX) {
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

void launch_schedule(const DevBatch &b, int record, cudaStream_t s) {
  if (b.n_jobs) schedule_kernel<<<b.n_jobs, SCHED_THREADS, 0, s>>>(b, record);
}

// ---------------------------------------------------------------------------
// search reduction: k best jobs by (class, time, key_rank) where class 0 =
// OK, non-OOM, time > 0; class 1 = OK, non-OOM, time == 0 (MFU 0.0 sorts
// after every positive MFU, search.py:784, sim.py:493-494).  Two passes:
// per-CTA top-k by repeated argmin, then one CTA merges the candidates.

struct Cand {
  unsigned long long k0;  // class << 63 | time
  uint32_t k1;            // key_rank
  int32_t job;
};

__device__ __forceinline__ bool cand_less(const Cand &a, const Cand &b) {
  return a.k0 < b.k0 || (a.k0 == b.k0 && (a.k1 < b.k1 || (a.k1 == b.k1 && a.job < b.job)));
}

static constexpr int TOPK_THREADS = 256;
static constexpr int TOPK_MAX = 64;
static constexpr int TOPK_CHUNK = 2048;

__device__ Cand block_argmin(Cand v) {
  __shared__ Cand sh[TOPK_THREADS / 32];
  for (int o = 16; o; o >>= 1) {
    Cand u;
    u.k0 = __shfl_xor_sync(0xffffffffu, v.k0, o);
    u.k1 = __shfl_xor_sync(0xffffffffu, v.k1, o);
    u.job = __shfl_xor_sync(0xffffffffu, v.job, o);
    if (cand_less(u, v)) v = u;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? sh[lane] : Cand{~0ull, ~0u, INT32_MAX};
    for (int o = 16; o; o >>= 1) {
      Cand u;
      u.k0 = __shfl_xor_sync(0xffffffffu, v.k0, o);
      u.k1 = __shfl_xor_sync(0xffffffffu, v.k1, o);
      u.job = __shfl_xor_sync(0xffffffffu, v.job, o);
      if (cand_less(u, v)) v = u;
    }
    if (lane == 0) sh[0] = v;
  }
  __syncthreads();
  return sh[0];
}

__device__ Cand make_cand(const DevBatch &b, uint32_t j) {
  const maya_job_result r = b.results[j];
  if (r.status != MAYA_ST_OK || r.oom) return Cand{~0ull, ~0u, INT32_MAX};
  unsigned long long k0 = r.total_ns > 0 ? (unsigned long long)r.total_ns : (1ull << 63);
  return Cand{k0, (uint32_t)b.jobs[j].key_rank, (int32_t)j};
}

// pass 1: each CTA takes TOPK_CHUNK jobs and emits its k best
__global__ void topk_local_kernel(DevBatch b, int k, Cand *cand) {
  __shared__ Cand items[TOPK_CHUNK];
  const uint32_t base = blockIdx.x * TOPK_CHUNK;
  const uint32_t n = min((uint32_t)TOPK_CHUNK, b.n_jobs - base);
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) items[i] = make_cand(b, base + i);
  __syncthreads();
  for (int q = 0; q < k; q++) {
    Cand best{~0ull, ~0u, INT32_MAX};
    int at = -1;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
      if (cand_less(items[i], best)) { best = items[i]; at = (int)i; }
    Cand m = block_argmin(best);
    if (at >= 0 && best.job == m.job && m.job != INT32_MAX) items[at] = Cand{~0ull, ~0u, INT32_MAX};
    if (threadIdx.x == 0) cand[blockIdx.x * k + q] = m;
    __syncthreads();
  }
}

// pass 2: one CTA merges all candidates
__global__ void topk_merge_kernel(Cand *cand, uint32_t n, int k, maya_topk_entry *out,
                                  int32_t *n_out, const DevBatch b) {
  int found = 0;
  for (int q = 0; q < k; q++) {
    Cand best{~0ull, ~0u, INT32_MAX};
    int at = -1;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
      if (cand_less(cand[i], best)) { best = cand[i]; at = (int)i; }
    Cand m = block_argmin(best);
    if (m.job == INT32_MAX) break;
    if (at >= 0 && best.job == m.job) cand[at] = Cand{~0ull, ~0u, INT32_MAX};
    if (threadIdx.x == 0) {
      out[q] = maya_topk_entry{b.results[m.job].total_ns, (int32_t)m.k1, m.job};
    }
    found++;
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_out = found;
}

size_t topk_scratch_bytes(uint32_t n_jobs, int k) {
  size_t blocks = (n_jobs + TOPK_CHUNK - 1) / TOPK_CHUNK;
  return (blocks * (size_t)k + 1) * sizeof(Cand);
}

void launch_topk(const DevBatch &b, int k, maya_topk_entry *out, int32_t *n_out, void *scratch,
                 cudaStream_t s) {
  if (k > TOPK_MAX) k = TOPK_MAX;
  uint32_t blocks = (b.n_jobs + TOPK_CHUNK - 1) / TOPK_CHUNK;
  Cand *cand = (Cand *)scratch;
  if (blocks == 0) {
    cudaMemsetAsync(n_out, 0, sizeof(int32_t), s);
    return;
  }
  topk_local_kernel<<<blocks, TOPK_THREADS, 0, s>>>(b, k, cand);
  topk_merge_kernel<<<1, TOPK_THREADS, 0, s>>>(cand, blocks * k, k, out, n_out, b);
}

}  // namespace maya
