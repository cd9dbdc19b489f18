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

// ceil(a / b) into int64; false on overflow.  Fast path for a, b < 2^64 and a
// quotient < 2^52: a double-precision estimate corrected exactly with 128-bit
// products (the estimate is within +-2 of the true quotient); otherwise the
// exact 128-bit division.
__device__ __forceinline__ bool ceil_div_i64(u128 a, u128 b, int64_t *out) {
  if ((a >> 64) == 0 && (b >> 64) == 0 && (uint64_t)b != 0) {
    const uint64_t x = (uint64_t)a, y = (uint64_t)b;
    const double qd = (double)x / (double)y;
    if (qd < 4503599627370496.0) {   // 2^52
      uint64_t q = (uint64_t)qd;
      u128 p = (u128)q * y;
      while (p > (u128)x) { q--; p -= y; }
      while (p + y <= (u128)x) { q++; p += y; }
      if (p != (u128)x) q++;
      *out = (int64_t)q;
      return true;
    }
  }
  u128 q = a / b;
  if (q * b != a) q += 1;
  if (q > (u128)INT64_MAX) return false;
  *out = (int64_t)q;
  return true;
}

// ceil(a / b) for a, b < 2^64 with a reciprocal estimate inv ~ 1/b: the
// double quotient a * inv is within a few units of the true one when it is
// below 2^50, then corrected exactly with 64 x 64 -> 128-bit products;
// anything else goes through ceil_div_i64.
__device__ __forceinline__ bool ceil_div_inv(uint64_t x, uint64_t y, double inv, int64_t *out) {
  const double qd = (double)x * inv;
  if (inv > 0.0 && qd < 1125899906842624.0) {   // 2^50
    uint64_t q = (uint64_t)qd;
    // p = q * y as (hi, lo); fix q until q * y <= x < (q + 1) * y
    uint64_t lo = q * y, hi = __umul64hi(q, y);
    while (hi != 0 || lo > x) {
      q--;
      const uint64_t nlo = lo - y;
      hi -= (nlo > lo) ? 1u : 0u;
      lo = nlo;
    }
    while (true) {   // (q + 1) * y <= x ?
      const uint64_t nlo = lo + y;
      if (nlo < lo || nlo > x) break;
      lo = nlo;
      q++;
    }
    if (lo != x) q++;
    *out = (int64_t)q;
    return true;
  }
  return ceil_div_i64((u128)x, (u128)y, out);
}

// ceil(x / y) for y >= 1 with the host-made magic M = floor(2^64 / y) (M == 0:
// y == 1).  q0 = floor(x * M / 2^64) satisfies x/y - 1 < q0 <= x/y (M > 2^64/y - 1
// and x < 2^64), so q0 is floor(x / y) or one less and one conditional
// subtraction fixes it; branch-free, ~12 instructions.
__device__ __forceinline__ uint64_t ceil_div_magic(uint64_t x, uint64_t y, uint64_t M) {
  if (M == 0) return x;
  uint64_t q = __umul64hi(x, M);
  uint64_t r = x - q * y;
  const bool c = r >= y;
  q += c ? 1u : 0u;
  r -= c ? y : 0u;
  return q + (r != 0 ? 1u : 0u);
}
// The same with M = ~0 standing for y == 1 (EstClass): then q0 = x - 1 for x >= 1
// (x * (2^64 - 1) / 2^64 = x - x / 2^64), still within one, so no branch.
__device__ __forceinline__ uint64_t ceil_div_magic_nb(uint64_t x, uint64_t y, uint64_t M) {
  uint64_t q = __umul64hi(x, M);
  uint64_t r = x - q * y;
  const bool c = r >= y;
  q += c ? 1u : 0u;
  r -= c ? y : 0u;
  return q + (r != 0 ? 1u : 0u);
}

// ---------------------------------------------------------------------------
// estimators

// a feature's duration as written by estimate_features_kernel (-1: failed)
__device__ __forceinline__ int64_t feat_dur(const DevBatch &b, uint32_t i) {
  const uint32_t w = b.feat_d32[i];
  if (w < DUR32_WIDE) return (int64_t)w;
  return w == DUR32_FAIL ? -1 : b.feat_ns[i];
}

// one feature's roofline duration (-1 on EstimationError / overflow)
__device__ __noinline__ int64_t estimate_one(const DevTables &t, longlong2 fv, uint32_t meta) {
  if (meta & FMETA_FIXED) return fv.x;
  struct { int64_t flops, bytes; int32_t op_kind, dtype, device; } f{
      fv.x, fv.y, fmeta_op(meta), fmeta_dtype(meta), fmeta_device(meta)};
  const maya_device_params &dev = t.devs[f.device];
  int64_t compute = 0, memory = 0;
  bool ok = true;
  if (f.flops > 0) {
    int64_t peak = (f.dtype >= 0 && f.dtype < MAYA_MAX_DTYPES) ? dev.peak_flops[f.dtype] : 0;
    if (peak <= 0 || f.op_kind < 0 || f.op_kind >= t.n_op_kinds) {
      ok = false;  // EstimationError: no peak rate for dtype (estimate.py:124-127)
    } else if ((uint64_t)f.flops <= t.max_flops[f.op_kind] && t.eff_num[f.op_kind] > 0) {
      // 64-bit fast path: X = flops * 1e9 * den fits (host bound);
      // ceil(X / (peak * num)) = ceil(ceil(X / peak) / num), both by invariant divisors
      const uint64_t X = (uint64_t)f.flops * (1000000000ull * (uint64_t)t.eff_den[f.op_kind]);
      const uint64_t q1 = ceil_div_magic(X, (uint64_t)peak, t.mag_peak[f.device][f.dtype]);
      const uint64_t q = ceil_div_magic(q1, (uint64_t)t.eff_num[f.op_kind], t.mag_num[f.op_kind]);
      ok = q <= (uint64_t)INT64_MAX;
      compute = (int64_t)q;
    } else {
      u128 num, den;
      ok = mul_u128_u64((u128)(uint64_t)f.flops * 1000000000ull, (uint64_t)t.eff_den[f.op_kind],
                        &num);
      den = (u128)(uint64_t)peak * (uint64_t)t.eff_num[f.op_kind];
      if (ok && (num >> 64) == 0 && (den >> 64) == 0)
        ok = ceil_div_inv((uint64_t)num, (uint64_t)den,
                          t.inv_peak[f.device][f.dtype] * t.inv_num[f.op_kind], &compute);
      else if (ok)
        ok = ceil_div_i64(num, den, &compute);
    }
  }
  if (ok && f.bytes > 0) {
    const u128 mb = (u128)(uint64_t)f.bytes * 1000000000ull;
    if ((mb >> 64) == 0 && dev.hbm_bytes_per_s > 0) {
      const uint64_t q = ceil_div_magic((uint64_t)mb, (uint64_t)dev.hbm_bytes_per_s,
                                        t.mag_hbm[f.device]);
      ok = q <= (uint64_t)INT64_MAX;
      memory = (int64_t)q;
    } else {
      ok = ceil_div_i64(mb, (u128)(uint64_t)dev.hbm_bytes_per_s, &memory);
    }
  }
  int64_t m = compute > memory ? compute : memory;
  if (ok && m > INT64_MAX - t.overhead_ns) ok = false;
  return ok ? m + t.overhead_ns : -1;
}

// Straight-line fast path: one invariant division per term through the class
// table (EstClass); every other case (bad ids, no rate, wide products) takes
// the general routine above, so the results are the same.
__device__ __forceinline__ int64_t estimate_fast(const DevTables &t, longlong2 fv, uint32_t meta) {
  if (meta & FMETA_FIXED) return fv.x;
  const int32_t op = fmeta_op(meta), dt = fmeta_dtype(meta), dv = fmeta_device(meta);
  if (op < t.n_op_kinds && dt < MAYA_MAX_DTYPES && dv < t.n_devs) {
    // < 8 x 16 x 4096 entries: 32-bit index arithmetic
    const EstClass *c = t.cls + (uint32_t)((dv * MAYA_MAX_DTYPES + dt) * t.n_op_kinds + op);
    const ulonglong2 kd = __ldg(reinterpret_cast<const ulonglong2 *>(c));
    const ulonglong2 mm = __ldg(reinterpret_cast<const ulonglong2 *>(c) + 1);
    const ulonglong2 hh = __ldg(reinterpret_cast<const ulonglong2 *>(c) + 2);
    const bool fok = fv.x <= 0 || (kd.y != 0 && (uint64_t)fv.x <= mm.y);
    const bool bok = fv.y <= 0 || (hh.x != 0 && (uint64_t)fv.y <= 18446744073ull);
    if (fok && bok) {
      const uint64_t comp = fv.x > 0 ? ceil_div_magic_nb((uint64_t)fv.x * kd.x, kd.y, mm.x) : 0;
      const uint64_t mem = fv.y > 0 ? ceil_div_magic_nb((uint64_t)fv.y * 1000000000ull, hh.x, hh.y) : 0;
      if (comp > (uint64_t)INT64_MAX || mem > (uint64_t)INT64_MAX) return -1;
      const int64_t m = (int64_t)(comp > mem ? comp : mem);
      return m > INT64_MAX - t.overhead_ns ? -1 : m + t.overhead_ns;
    }
  }
  return estimate_one(*t.gtab, fv, meta);
}

// EST_PER features per thread, all loads issued before the arithmetic (memory-
// level parallelism: the kernel streams 20 B in and 8 B out per feature)
static constexpr uint32_t EST_PER = 4;
__global__ void __launch_bounds__(256) estimate_features_kernel(DevBatch b, DevTables t) {
  const uint32_t base = blockIdx.x * (256 * EST_PER) + threadIdx.x;
  longlong2 fv[EST_PER];
  uint32_t meta[EST_PER];
#pragma unroll
  for (uint32_t k = 0; k < EST_PER; k++) {
    const uint32_t i = base + k * 256;
    if (i < b.n_feats) {
      fv[k] = __ldg(reinterpret_cast<const longlong2 *>(b.feats) + i);
      meta[k] = __ldg(b.feat_meta + i);
    }
  }
  bool bad = false, wide = false;
#pragma unroll
  for (uint32_t k = 0; k < EST_PER; k++) {
    const uint32_t i = base + k * 256;
    if (i < b.n_feats) {
      const int64_t v = estimate_fast(t, fv[k], meta[k]);
      // 4 B per duration (DUR32_*): the fold / resolve passes read them back
      uint32_t w = (uint32_t)v;
      if (v < 0) {
        w = DUR32_FAIL;
        bad = true;
      } else if (v >= (int64_t)DUR32_WIDE) {
        w = DUR32_WIDE;
        b.feat_ns[i] = v;
        wide = true;
      }
      b.feat_d32[i] = w;
    }
  }
  if (bad || wide) atomicOr(b.err_flag, (bad ? 1 : 0) | (wide ? ERR_WIDE_DUR : 0));
}

__global__ void estimate_wire_kernel(DevBatch b, DevTables t) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b.n_wfeats) return;
  SlotRec s = b.wfeats[i];
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
  if (b.n_feats)
    estimate_features_kernel<<<(b.n_feats + 256 * EST_PER - 1) / (256 * EST_PER), 256, 0, s>>>(b, t);
  if (b.n_wfeats) estimate_wire_kernel<<<(b.n_wfeats + 255) / 256, 256, 0, s>>>(b, t);
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
//
// resolve: Op + estimator output -> ExecOp (duration inlined), one thread per op.

__global__ void resolve_kernel(DevBatch b) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b.n_ops) return;
  const Op op = b.ops[i];
  const uint32_t tag = op_tag(op.meta);
  uint64_t pay;
  if (tag == TAG_KERN) {
    const int64_t d = feat_dur(b, op.arg);   // batch-global feature id
    pay = (d < 0 || d >= (int64_t)(EXEC_BAD >> 2)) ? (EXEC_BAD >> 2) : (uint64_t)d;
  } else {
    pay = (op.arg == NO_REC) ? (EXEC_NONE >> 2) : (uint64_t)op.arg;
  }
  b.exec[i] = ExecOp{op.disp, (pay << 2) | tag};
}

// wire time of every (rank, rep collective) entry, gathered once per run
__global__ void resolve_colls_kernel(DevBatch b) {
  uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= b.n_rcolls) return;
  b.rcx[e] = RCX{b.rcolls[e], b.wire[b.rcslot[e]]};
}

template <typename T>
__device__ __forceinline__ T vload(const T *p) {
  return *(const volatile T *)p;
}
template <typename T>
__device__ __forceinline__ void vstore(T *p, T v) {
  *(volatile T *)p = v;
}

static constexpr unsigned FULL = 0xffffffffu;
#ifndef MAYA_WIDE_FAILS
#define MAYA_WIDE_FAILS 2u   // failed 128-op windows after which a FIFO stops trying them
#endif

#ifdef MAYA_PROFILE
// per-batch cycle counters: [0] walk windows, [1] slow ops, [2] idle sleep,
// [3] sweeps (skip checks + ctx), [4] windows, [5] slow-op calls, [6] wakes, [7] passes
// accumulated per thread (lane 0 of each warp) and flushed once at kernel exit
__device__ unsigned long long g_prof[8];
// window sub-phases (lane 0): [0] segment advance + wide attempt, [1] load + classify
// (to the blocker ballot), [2] scan, [3] blockers + commit
__device__ unsigned long long g_prof_sub[8];   // [4] wide attempts, [5] failed wide cycles
#define PROF_T(v) long long v = clock64()
#define PROF_ADD(i, v) (prof_acc[i] += (unsigned long long)(v))
#else
#define PROF_T(v)
#define PROF_ADD(i, v)
#endif
static constexpr int64_t NEG = INT64_MIN / 4;          // -inf of the max-plus scan
static constexpr int64_t LIM_T = (int64_t)1 << 60;     // times beyond: exact serial path
static constexpr uint64_t LIM_D = (uint64_t)1 << 56;   // durations beyond: exact serial path
static constexpr uint64_t LIM_W = (uint64_t)1 << 52;   // wide-window duration guard

// Per-walker state (one (rank, stream) FIFO), kept in shared memory (or the
// global spill) between rounds; uniform across the lanes of the warp.
struct WSt {
  int64_t x;              // completion time of the last op processed
  int64_t cdel;           // host delay of the current sync segment
  uint32_t i, flags, seg, bound;
  const void *wa;         // wake condition of a blocked walker: counter / record entry
  uint32_t wt;            // target count
  uint32_t wk;            // WAKE_*
};
enum { WAKE_NONE = 0, WAKE_COUNT = 1, WAKE_FIRE = 2, WAKE_ROUND = 3 };
static_assert(sizeof(WSt) == WSTATE_BYTES, "WSt layout");

// Walker context: loop-invariant pointers of one (rank, stream) FIFO
// (cached in shared memory for on-chip jobs).
struct WCtx {
  const ExecOp *ops;      // stream's first op
  int64_t *fire;          // rank's record table
  const int64_t *delay;   // rank's host-delay table (n_syncs + 1)
  const RCX *rc;          // rank's collective entries + wire times (smem or global)
  const uint32_t *cnt;    // counts[0][stream] of the rep (stride ns)
  uint64_t tl;            // timeline row of the stream's first op
  uint32_t len, rank, ns, nsync;
};
static_assert(sizeof(WCtx) == WCTX_BYTES, "WCtx layout");

struct JobSh {            // per-CTA view of the job
  const JobHdr *J;
  CollSlot *ring;         // smem rings (2 per comm) or null -> global slots
  const uint32_t *cb;     // call_base per comm (smem u32, or CommRec stride in global)
  uint32_t cb_stride;
  uint32_t *hostk;        // resolved host syncs per rank
  WSt *st;                // walker states
  const uint32_t *wid;    // rank-major (rank, stream) position -> walker index
  WCtx *ctx;              // cached contexts (smem) or null
  int64_t *fire;          // job's record-time table (smem or global)
  const RCX *rcx;         // job's rank-collective table (smem or global)
  unsigned *epoch;        // CTA progress epoch
  int record;
};

__device__ __forceinline__ void load_ctx(const DevBatch &b, const JobHdr &J, uint32_t w,
                                         int record, WCtx &c, int64_t *fire_job,
                                         const RCX *rcx_job) {
  const Walker wk = b.walkers[J.walkers + w];
  const RankRec rr = b.ranks[J.ranks + wk.rank];
  const RepHdr &h = b.reps[rr.rep];
  const StreamRange sr = b.streams[h.streams + wk.stream];
  c.ops = b.exec + h.ops + sr.begin;
  c.fire = fire_job + rr.fire;
  c.delay = b.delay + J.delay + rr.delay;
  c.rc = rcx_job + rr.rslot;
  c.cnt = (b.clen ? b.ccounts : b.counts) + h.counts + wk.stream;
  c.len = b.clen ? b.clen[h.streams + wk.stream] : sr.len;
  c.rank = wk.rank;
  c.ns = h.n_streams;
  c.nsync = h.n_syncs;
  c.tl = J.timeline + rr.tl + sr.begin;
  (void)record;
}

enum { STEP_OK = 0, STEP_BLOCK = 1, STEP_ERR = 2 };

struct SlowRes {
  int64_t nx;       // completion time
  uint32_t code;    // status | flags << 2 | adv << 3 | err << 4 | wake kind << 8
  uint32_t wt;      // wake target (WAKE_COUNT)
  const void *wa;   // wake address
};

__device__ __forceinline__ ExecOp load_exec(const ExecOp *p) {
  const longlong2 v = __ldg(reinterpret_cast<const longlong2 *>(p));
  return ExecOp{v.x, (uint64_t)v.y};
}

// Warp-cooperative walker: advance one (rank, stream) FIFO 32 records at a
// time.  Every op whose inputs are already known is a max-plus affine map of
// the stream clock x (ready = max(x, disp)):
//   kernel                       x -> max(x + d, disp + d)
//   record                       x -> max(x, disp)            (fire = result)
//   wait on a fired event f      x -> max(x, max(disp, f))
//   collective, one member class x -> max(x + w, disp + w)
//   collective, all others in    x -> max(x + w, max(disp, M) + w)
// so a window is one segmented inclusive scan of (a, b) pairs across the
// lanes (5 shuffle steps).  Their inputs (fired times, slot counters, wire
// times) are loaded lane-parallel first; only true blockers -- waits on
// unfired events, arrivals that are not the last, overflow-checked kernels --
// are applied in order by lane 0, and segments restart after them.
__device__ bool warp_walk(const DevBatch &b, const JobSh &sh, const WCtx &c, WSt &s,
                          int64_t &tmax, int &err, uint32_t lane
#ifdef MAYA_PROFILE
                          , unsigned long long *prof_acc
#endif
                          ) {
  if (s.i >= c.len) return false;
  const JobHdr &J = *sh.J;
  const uint32_t hk = sh.hostk[c.rank];
  const uint32_t limit = hk < c.nsync ? c.cnt[hk * c.ns] : c.len;
  bool adv = false;
  bool streaming = false;   // the last window committed 32 ops: try 128-op windows
  // no 128-op window has failed in this walk, and the FIFO has not failed two
  // (WSt.flags bits 4-5 count failures): a failed one costs a 2 KB load and its
  // dependent gathers, ~2.5 k cycles, and FIFOs that block often keep failing
  bool wide_ok = ((s.flags >> 4) & 3u) < MAYA_WIDE_FAILS;
  s.wk = WAKE_ROUND;   // until something else is known: wait for the next round
  while (s.i < limit) {
    PROF_T(t_win);
    while (s.i >= s.bound && s.seg < c.nsync) {  // next host-sync segment
      s.seg++;
      s.cdel = c.delay[s.seg];
      s.bound = s.seg < c.nsync ? c.cnt[s.seg * c.ns] : c.len;
    }
    const uint32_t end = s.bound < limit ? s.bound : limit;
    // ---- wide window: 128 ops (4 per lane) when none of them blocks --------
    // Every op is an affine max-plus map x -> max(x + A, B); a lane composes
    // its 4 maps, the warp scans the 32 compositions (5 shuffle steps) and each
    // lane expands its own 4.  Records fire in the expansion; a wait on an
    // unfired event, a multi-member collective or a guard miss anywhere in the
    // block sends the block back to the 32-op window below.
    // the next 2 KB of this FIFO into L1 while this window computes (one line per lane)
    if (lane < 16 && s.i + 128u + lane * 8u < c.len)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(c.ops + s.i + 128u + lane * 8u));
    if (streaming && end - s.i >= 128u && s.x < LIM_T) {
#ifdef MAYA_PROFILE
      const long long t_wide = clock64();
      if (lane == 0) atomicAdd(&g_prof_sub[4], 1ull);
#endif
      int64_t A4[4], B4[4], rd4[4];
      uint32_t rec4 = 0;
      bool blk = false;
      const ExecOp *base = c.ops + s.i + lane * 4u;
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const ExecOp ek = load_exec(base + k);
        const uint32_t tg = (uint32_t)(ek.w & 3);
        const uint64_t py = ek.w >> 2;
        const int64_t rd = ek.disp + s.cdel;
        rd4[k] = rd;
        A4[k] = 0;
        B4[k] = rd;
        if (rd >= LIM_T) blk = true;
        if (tg == TAG_KERN) {
          if (py >= LIM_W) blk = true;   // 128 x 2^52 + 2^60 stays far below 2^63
          A4[k] = (int64_t)py;
          B4[k] = rd + (int64_t)py;
        } else if (tg == TAG_REC) {
          rec4 |= 1u << k;
        } else if (tg == TAG_WAIT) {
          const int64_t f = py == (EXEC_NONE >> 2) ? -1 : vload(&c.fire[py]);
          if (f < 0) blk = true;
          else if (f > rd) B4[k] = f;
        } else {
          const RCX rx = c.rc[py];
          if ((uint32_t)(rx.ent >> 48) != 1u || rx.wire >= (int64_t)LIM_W) blk = true;
          A4[k] = rx.wire;
          B4[k] = rd + rx.wire;
        }
      }
      if (!__any_sync(FULL, blk)) {
        // compose the lane's 4 maps, then an inclusive warp scan
        int64_t A = A4[0], B = B4[0];
#pragma unroll
        for (int k = 1; k < 4; k++) {
          const int64_t nb = B + A4[k];
          B = nb > B4[k] ? nb : B4[k];
          A += A4[k];
        }
#pragma unroll
        for (uint32_t off = 1; off < 32; off <<= 1) {
          const int64_t A2 = __shfl_up_sync(FULL, A, off);
          const int64_t B2 = __shfl_up_sync(FULL, B, off);
          if (lane >= off) {
            const int64_t nb = B2 + A;
            B = nb > B ? nb : B;
            A = A2 + A;
          }
        }
        // exclusive prefix applied to the walker's clock
        int64_t Ae = __shfl_up_sync(FULL, A, 1), Be = __shfl_up_sync(FULL, B, 1);
        int64_t x = s.x;
        if (lane > 0) {
          const int64_t v = x + Ae;
          x = v > Be ? v : Be;
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const int64_t ready = x > rd4[k] ? x : rd4[k];
          const int64_t v = x + A4[k];
          const int64_t d = v > B4[k] ? v : B4[k];
          if (rec4 & (1u << k)) {
            const uint64_t py = (load_exec(base + k).w) >> 2;
            vstore(&c.fire[py], d);
          }
          if (sh.record) {
            b.tl_start[c.tl + s.i + lane * 4u + k] = ready;
            b.tl_end[c.tl + s.i + lane * 4u + k] = d;
          }
          x = d;
        }
        s.x = __shfl_sync(FULL, x, 31);
#ifdef MAYA_PROFILE
        if (lane == 0) { PROF_ADD(6, 1); PROF_ADD(7, 128); PROF_ADD(0, clock64() - t_win); PROF_ADD(4, 1); }
#endif
        s.i += 128u;
        s.flags &= ~1u;
        adv = true;
        if (__any_sync(FULL, rec4 != 0)) __threadfence_block();
        s.wk = WAKE_ROUND;
        continue;
      }
      streaming = false;
      wide_ok = false;
      if (((s.flags >> 4) & 3u) < 3u) s.flags += 16u;
#ifdef MAYA_PROFILE
      if (lane == 0) atomicAdd(&g_prof_sub[5], (unsigned long long)(clock64() - t_wide));
#endif
    }
#ifdef MAYA_PROFILE
    long long t_a = clock64();
#endif
    const uint32_t n = min(32u, end - s.i);
    const bool valid = lane < n;
    ExecOp e{0, 0};
    if (valid) e = load_exec(c.ops + s.i + lane);
    if (lane < 4 && s.i + 32 + lane * 8 < c.len)   // next window's lines into L1
      asm volatile("prefetch.global.L1 [%0];" ::"l"(c.ops + s.i + 32 + lane * 8));
    const uint32_t tag = (uint32_t)(e.w & 3);
    const uint64_t pay = e.w >> 2;
    const int64_t rdisp = e.disp + s.cdel;
    // lane-parallel classification: affine map (A, B), side effect, or blocker
    int64_t A = 0, B = NEG, w8 = 0;
    uint32_t fx = 0;            // side effect at commit: 1 record fire, 2 post last arrival
    uint32_t target = 0;
    CollSlot *cs = nullptr;
    bool blocker = false;
    if (valid) {
      if (s.x >= LIM_T || rdisp >= LIM_T) {
        blocker = true;
      } else if (tag == TAG_KERN) {
        if (pay >= LIM_D) blocker = true;      // also EXEC_BAD
        else { A = (int64_t)pay; B = rdisp + A; }
      } else if (tag == TAG_REC) {
        A = 0; B = rdisp; fx = 1;
      } else if (tag == TAG_WAIT) {
        const int64_t f = pay == (EXEC_NONE >> 2) ? -1 : vload(&c.fire[pay]);
        if (f < 0) blocker = true;
        else { A = 0; B = rdisp > f ? rdisp : f; }
      } else {
        const RCX rx = c.rc[pay];
        const RankColl ent = rx.ent;
        w8 = rx.wire;
        const uint32_t nr = (uint32_t)(ent >> 48);
        const uint32_t g = (uint32_t)(ent >> 32) & 0xffffu;
        const uint32_t idx = (uint32_t)ent;
        if (w8 >= (int64_t)LIM_D) {
          blocker = true;
        } else if (nr == 1) {                  // one member (class): no wait
          A = w8; B = rdisp + w8;
        } else {
          if (sh.ring) {
            cs = sh.ring + 2 * g + (idx & 1u);
            target = ((idx >> 1) + 1u) * nr;
          } else {
            cs = b.cslots + J.slots + sh.cb[g * sh.cb_stride] + idx;
            target = nr;
          }
          const uint32_t cnt = vload(&cs->count);
          if (lane == 0 && (s.flags & 1u)) {   // our arrival already posted
            if (cnt >= target) { A = NEG; B = (int64_t)vload(&cs->maxarr) + w8; }
            else blocker = true;
          } else if (cnt + 1 == target) {      // every other member is in: we complete it
            const int64_t m = (int64_t)vload(&cs->maxarr);
            A = w8; B = (rdisp > m ? rdisp : m) + w8; fx = 2;
          } else {
            blocker = true;
          }
        }
      }
    }
    const uint32_t bmask = __ballot_sync(FULL, blocker);
#ifdef MAYA_PROFILE
    long long t_b = clock64();
#endif
    if (blocker) { A = 0; B = NEG; }
    // segmented inclusive scan; segments start at lane 0 and after each
    // blocker: lane L absorbs lane L - off while that lane is in its segment
    // (L - off >= start of L's segment), so no flag travels with the values
    const uint32_t starts = (bmask << 1) | 1u;
    const int32_t seg0 = 31 - __clz(starts & (0xffffffffu >> (31 - lane)));
#pragma unroll
    for (uint32_t off = 1; off < 32; off <<= 1) {
      const int64_t A2 = __shfl_up_sync(FULL, A, off);
      const int64_t B2 = __shfl_up_sync(FULL, B, off);
      if ((int32_t)lane - (int32_t)off >= seg0) {
        const int64_t nb = B2 + A;
        B = nb > B ? nb : B;
        A = A2 + A;
      }
    }
#ifdef MAYA_PROFILE
    long long t_c = clock64();
#endif
    // finalize segments; apply blockers in order
    int64_t xin = s.x, d = 0;
    uint32_t p = 0, commit = n, spec = bmask;
    bool blocked = false;
    for (;;) {
      const uint32_t q = spec ? (uint32_t)(__ffs(spec) - 1) : n;
      const bool in_seg = lane >= p && lane < q;
      if (in_seg) {
        const int64_t v = xin + A;
        d = v > B ? v : B;
      }
      int64_t prev = __shfl_up_sync(FULL, d, 1);
      if (lane == p) prev = xin;
      if (in_seg && fx) {
        if (fx == 1) {
          vstore(&c.fire[pay], d);
        } else {
          const int64_t ready = rdisp > prev ? rdisp : prev;
          atomicMax(&cs->maxarr, (unsigned long long)ready);
          __threadfence_block();
          if (atomicAdd(&cs->count, 1u) + 1 != target) err = MAYA_ST_INTERNAL;
        }
      }
      if (sh.record && in_seg) {
        b.tl_start[c.tl + s.i + lane] = rdisp > prev ? rdisp : prev;
        b.tl_end[c.tl + s.i + lane] = d;
      }
      // one warp reduction for both: side effects made (bit 0), error (bit 1)
      const uint32_t ev = __reduce_or_sync(FULL, ((in_seg && fx) ? 1u : 0u) | (err != 0 ? 2u : 0u));
      if (ev & 1u) {
        adv = true;
        __threadfence_block();
      }
      if (ev & 2u) {
        err = __reduce_max_sync(FULL, (unsigned)err);
        blocked = true;
        commit = q;
        break;
      }
      if (q >= n) break;
      spec &= spec - 1;
      // blocker q: applied by lane 0 (sim.py:311-343 semantics)
      const int64_t xq = q > p ? __shfl_sync(FULL, d, q - 1) : xin;
      const int64_t qd = __shfl_sync(FULL, rdisp, q);
      const uint64_t qw = __shfl_sync(FULL, e.w, q);
      const int64_t qw8 = __shfl_sync(FULL, w8, q);
      const int64_t ready = qd > xq ? qd : xq;
      const uint32_t qtag = (uint32_t)(qw & 3);
      const uint64_t qpay = qw >> 2;
      PROF_T(t_slow);
      int64_t nx = 0;
      uint32_t stc = STEP_OK, wk = WAKE_NONE, wt = 0, eno = 0;
      const void *wa = nullptr;
      if (ready >= LIM_T || (qtag == TAG_KERN)) {    // exact, overflow-checked
        int64_t dd = 0;
        if (qtag == TAG_KERN) {
          if (qw == EXEC_BAD) { stc = STEP_ERR; eno = MAYA_ST_ESTIMATION; }
          else if (qw == EXEC_OVF) { stc = STEP_ERR; eno = MAYA_ST_OVERFLOW; }
          dd = (int64_t)qpay;
        }
        if (stc == STEP_OK && qtag == TAG_KERN) {
          if (dd > INT64_MAX - ready) { stc = STEP_ERR; eno = MAYA_ST_OVERFLOW; }
          else nx = ready + dd;
        }
      }
      if (stc == STEP_OK && qtag != TAG_KERN) {
        if (qtag == TAG_REC) {
          if (lane == 0) vstore(&c.fire[qpay], ready);
          nx = ready;
        } else if (qtag == TAG_WAIT) {
          const int64_t f = qpay == (EXEC_NONE >> 2) ? -1 : vload(&c.fire[qpay]);
          if (f < 0) {
            stc = STEP_BLOCK;
            s.flags &= ~1u;
            wk = qpay == (EXEC_NONE >> 2) ? WAKE_ROUND : WAKE_FIRE;
            wa = qpay == (EXEC_NONE >> 2) ? nullptr : &c.fire[qpay];
          } else {
            nx = ready > f ? ready : f;
          }
        } else {                                   // collective rendezvous
          const RankColl ent = c.rc[qpay].ent;
          const uint32_t nr = (uint32_t)(ent >> 48);
          const uint32_t g = (uint32_t)(ent >> 32) & 0xffffu;
          const uint32_t idx = (uint32_t)ent;
          if (nr == 1) {
            if (qw8 > INT64_MAX - ready) { stc = STEP_ERR; eno = MAYA_ST_OVERFLOW; }
            else nx = ready + qw8;
          } else {
            CollSlot *qs;
            uint32_t tgt;
            if (sh.ring) {
              qs = sh.ring + 2 * g + (idx & 1u);
              tgt = ((idx >> 1) + 1u) * nr;
            } else {
              qs = b.cslots + J.slots + sh.cb[g * sh.cb_stride] + idx;
              tgt = nr;
            }
            uint32_t code = 0;
            int64_t m = 0;
            const bool posted = q == 0 && (s.flags & 1u);   // flag belongs to the op at s.i
            if (lane == 0) {
              bool done = true;
              if (!posted) {
                atomicMax(&qs->maxarr, (unsigned long long)ready);
                __threadfence_block();
                const uint32_t old = atomicAdd(&qs->count, 1u);
                code |= 2u;
                if (old + 1 > tgt) code |= 4u;
                else if (old + 1 < tgt) done = false;
              } else if (vload(&qs->count) < tgt) {
                done = false;
              }
              if (done && !(code & 4u)) {
                __threadfence_block();
                m = (int64_t)vload(&qs->maxarr);
                code |= 1u;
              }
            }
            code = __shfl_sync(FULL, code, 0);
            m = __shfl_sync(FULL, m, 0);
            if (code & 2u) adv = true;
            if (code & 4u) { stc = STEP_ERR; eno = MAYA_ST_INTERNAL; }
            else if (!(code & 1u)) {
              stc = STEP_BLOCK; wk = WAKE_COUNT; wt = tgt; wa = &qs->count;
              s.flags = (s.flags & ~1u) | ((posted || (code & 2u)) ? 1u : 0u);   // for the new s.i (= this op)
            }
            else if (qw8 > INT64_MAX - m) { stc = STEP_ERR; eno = MAYA_ST_OVERFLOW; }
            else { nx = m + qw8; }
          }
        }
      }
#ifdef MAYA_PROFILE
      if (lane == 0) { PROF_ADD(1, clock64() - t_slow); PROF_ADD(5, 1); }
#endif
      if (stc != STEP_OK) {
        if (stc == STEP_ERR) err = (int)eno;
        if (stc == STEP_ERR && q > 0) s.flags &= ~1u;
        s.wk = wk;
        s.wt = wt;
        s.wa = wa;
        blocked = true;
        commit = q;
        break;
      }
      if (lane == q) {
        d = nx;
        if (sh.record) {
          b.tl_start[c.tl + s.i + lane] = ready;
          b.tl_end[c.tl + s.i + lane] = nx;
        }
      }
      xin = nx;
      p = q + 1;
    }
#ifdef MAYA_PROFILE
    if (lane == 0) PROF_ADD(7, commit);
#endif
#ifdef MAYA_PROFILE
    if (lane == 0) {
      const long long t_d = clock64();
      atomicAdd(&g_prof_sub[0], (unsigned long long)(t_a - t_win));
      atomicAdd(&g_prof_sub[1], (unsigned long long)(t_b - t_a));
      atomicAdd(&g_prof_sub[2], (unsigned long long)(t_c - t_b));
      atomicAdd(&g_prof_sub[3], (unsigned long long)(t_d - t_c));
    }
#endif
    streaming = wide_ok && !blocked && commit == 32u;
    if (commit > 0) {
      s.x = __shfl_sync(FULL, d, commit - 1);
      s.i += commit;
      adv = true;
      // the arrival flag belongs to the op at s.i: a committed op 0 completed it;
      // a blocker at q > 0 set it for the new s.i
      if (!blocked) s.flags &= ~1u;
    }
#ifdef MAYA_PROFILE
    if (lane == 0) { PROF_ADD(0, clock64() - t_win); PROF_ADD(4, 1); }
#endif
    if (blocked) break;
    s.wk = WAKE_ROUND;
  }
  if (s.x > tmax) tmax = s.x;
  return adv;
}

// Resolve as many host syncs of rank r as the stream states allow
// (sim.py:243-263, 272-283): H' = max(H, X), H = gap prefix + delay.
__device__ bool host_step(const DevBatch &b, const JobSh &sh, uint32_t r, int64_t *delay_job) {
  const JobHdr &J = *sh.J;
  const RankRec rr = b.ranks[J.ranks + r];
  const RepHdr &h = b.reps[rr.rep];
  uint32_t k = sh.hostk[r];
  if (k >= h.n_syncs) return false;
  int64_t *delay = delay_job + rr.delay;
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
        X = vload(&sh.fire[rr.fire + s.arg]);
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
        const WSt &ws = sh.st[sh.wid[rr.walker + ls]];
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

template <int NW>
__global__ void __launch_bounds__(NW * 32, 16 / NW) sched_warp_kernel(DevBatch b, const int32_t *order,
                                                             int record, uint32_t smem_cap) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ unsigned long long s_tmax;
  __shared__ int s_err, s_incomplete, s_oom_rank, s_active;
  __shared__ unsigned s_epoch;
  __shared__ long long s_oom_t, s_peak;

  const uint32_t j = (uint32_t)order[blockIdx.x];
  const JobHdr &J = b.jobs[j];
  maya_job_result *res = b.results + j;
  const uint32_t tid = threadIdx.x, nt = NW * 32, lane = tid & 31, wp = tid >> 5;
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
  const uint32_t W = J.n_walkers, R = J.n_ranks;
  const SchedLayout L = sched_layout(W, R, J.n_comms, (J.flags & JOB_RING) != 0, J.n_fire,
                                     J.n_rcolls, smem_cap);
  const bool on_chip = L.on_chip;
  uint8_t *base = on_chip ? dsm : b.spill + J.wstate;
  JobSh sh;
  sh.J = &J;
  sh.ring = (on_chip && L.ring_on) ? (CollSlot *)(dsm + L.ring) : nullptr;
  if (on_chip) {
    uint32_t *cb = (uint32_t *)(dsm + L.cb);
    for (uint32_t g = tid; g < J.n_comms; g += nt) cb[g] = b.comms[J.comms + g].call_base;
    sh.cb = cb;
    sh.cb_stride = 1;
  } else {
    sh.cb = &b.comms[J.comms].call_base;
    sh.cb_stride = sizeof(CommRec) / 4;
  }
  if (sh.ring)
    for (uint32_t q = tid; q < 2 * J.n_comms; q += nt) sh.ring[q] = CollSlot{0, 0, 0};
  sh.hostk = (uint32_t *)(base + (on_chip ? L.hostk : 0));
  sh.st = (WSt *)(base + (on_chip ? L.state : ((4 * R + 15) & ~15u)));
  sh.wid = b.wids + J.walkers;
  sh.ctx = on_chip ? (WCtx *)(dsm + L.ctx) : nullptr;
  sh.fire = L.fire_on ? (int64_t *)(dsm + L.fire) : b.fire + J.fire;
  sh.rcx = L.rcx_on ? (const RCX *)(dsm + L.rcx) : b.rcx + J.rcolls;
  if (L.fire_on)
    for (uint32_t q = tid; q < J.n_fire; q += nt) ((int64_t *)(dsm + L.fire))[q] = -1;
  if (L.rcx_on) {   // stage the job's collective table (contiguous, 16 B records)
    const RCX *src = b.rcx + J.rcolls;
    RCX *dst = (RCX *)(dsm + L.rcx);
    for (uint32_t q = tid; q < J.n_rcolls; q += nt) dst[q] = src[q];
  }
  sh.epoch = &s_epoch;
  sh.record = record;
  if (tid == 0) {
    s_tmax = 0;
    s_err = 0;
    s_incomplete = 0;
    s_oom_t = INT64_MAX;
    s_oom_rank = INT32_MAX;
    s_peak = 0;
    s_epoch = 0;
  }
  int64_t *delay_job = b.delay + J.delay;
  for (uint32_t r = tid; r < R; r += nt) {
    delay_job[b.ranks[J.ranks + r].delay] = 0;
    sh.hostk[r] = 0;
  }
  for (uint32_t w = tid; w < W; w += nt) {
    WCtx c;
    load_ctx(b, J, w, 0, c, sh.fire, sh.rcx);
    sh.st[w] = WSt{0, 0, 0, 0, 0, c.nsync ? c.cnt[0] : c.len, nullptr, 0, WAKE_NONE};
    if (sh.ctx) sh.ctx[w] = c;
  }
  __syncthreads();

  int64_t tmax = 0;
  int err = 0;
  int64_t rounds = 0;
#ifdef MAYA_PROFILE
  unsigned long long prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  uint32_t my_wb = 0, my_we = 0;   // walkers of this warp's first rank
  if (wp < R) {
    const RankRec rr = b.ranks[J.ranks + wp];
    my_wb = rr.walker;
    my_we = rr.walker + b.reps[rr.rep].n_streams;
  }
  for (;;) {
    int progress = 0;
    for (uint32_t r = tid; r < R; r += nt) progress |= host_step(b, sh, r, delay_job);
    if (tid == 0) s_active = (int)min(R, (uint32_t)NW);
    __syncthreads();
    if (wp < R) {
      // a warp sweeps its FIFOs while anything in the CTA makes progress; an
      // idle warp sleeps on the progress epoch; when every warp is idle the
      // round ends (host syncs, termination and deadlock are decided there)
      bool fresh = true;   // first sweep of the round re-examines every walker
      for (;;) {
        bool pass = false;
        PROF_T(t_sweep);
        for (uint32_t r = wp; r < R; r += NW) {
          uint32_t wb = my_wb, we = my_we;
          if (r != wp) {
            const RankRec rr = b.ranks[J.ranks + r];
            wb = rr.walker;
            we = rr.walker + b.reps[rr.rep].n_streams;
          }
          // lane-parallel wake check of up to 32 FIFOs, then walk the ready ones
          for (uint32_t w0 = wb; w0 < we; w0 += 32) {
            bool can = false;
            if (w0 + lane < we) {
              const uint32_t w = w0 + lane;
              const uint32_t wk = sh.st[w].wk;
              can = !(wk == WAKE_ROUND && !fresh);
              if (can && wk == WAKE_COUNT)
                can = vload((const uint32_t *)sh.st[w].wa) >= sh.st[w].wt;
              else if (can && wk == WAKE_FIRE)
                can = vload((const int64_t *)sh.st[w].wa) >= 0;
              if (can && sh.ctx) can = sh.st[w].i < sh.ctx[w].len;
            }
            unsigned ready = __ballot_sync(FULL, can);
            while (ready) {
            const uint32_t w = w0 + (uint32_t)(__ffs(ready) - 1);
            ready &= ready - 1;
            WSt s = sh.st[w];
            WCtx c;
            if (sh.ctx) {
              c = sh.ctx[w];
            } else {
              load_ctx(b, J, w, record, c, sh.fire, sh.rcx);
            }
            pass |= warp_walk(b, sh, c, s, tmax, err, lane
#ifdef MAYA_PROFILE
                              , prof_acc
#endif
                              );
            __syncwarp();
            if (lane == 0) sh.st[w] = s;
            __syncwarp();
            }
          }
        }
        if (err) {
          if (lane == 0) atomicSub(&s_active, 1);
          break;
        }
#ifdef MAYA_PROFILE
        if (lane == 0) { PROF_ADD(3, clock64() - t_sweep); }
#endif
        fresh = false;
        if (pass) {
          progress = 1;
          continue;
        }
        int wake = 0;
        PROF_T(t_idle);
        // idle: poll the wake conditions of this warp's blocked walkers (lane
        // parallel) until one holds, or until no warp of the CTA is walking
        if (lane == 0) atomicSub(&s_active, 1);
        __syncwarp();
        unsigned ns = 32;
        for (int poll = 0;; poll++) {
          bool any = false;
          for (uint32_t r = wp; r < R && !any; r += NW) {
            uint32_t wb = my_wb, we = my_we;
            if (r != wp) {
              const RankRec rr = b.ranks[J.ranks + r];
              wb = rr.walker;
              we = rr.walker + b.reps[rr.rep].n_streams;
            }
            for (uint32_t w = wb + lane; w < we; w += 32) {
              const uint32_t wk = sh.st[w].wk;
              if (wk == WAKE_COUNT)
                any |= vload((const uint32_t *)sh.st[w].wa) >= sh.st[w].wt;
              else if (wk == WAKE_FIRE)
                any |= vload((const int64_t *)sh.st[w].wa) >= 0;
            }
          }
          if (__any_sync(FULL, any)) {
            wake = 1;
            break;
          }
          if (vload(&s_active) <= 0) break;
#ifndef MAYA_POLL_SPIN
          if (poll >= 32) {
            __nanosleep(ns);
            if (ns < 256) ns <<= 1;
          }
#endif
        }
        if (wake && lane == 0) atomicAdd(&s_active, 1);
        wake = __shfl_sync(FULL, wake, 0);
#ifdef MAYA_PROFILE
        if (lane == 0) { PROF_ADD(2, clock64() - t_idle); }
#endif
        if (!wake) break;
      }
    }
    rounds++;
    if (err) { atomicMax(&s_err, err); progress = 0; }
    if (!__syncthreads_or(progress)) break;
  }
#ifdef MAYA_PROFILE
  if (lane == 0)
    for (int q = 0; q < 8; q++) atomicAdd(&g_prof[q], prof_acc[q]);
#endif
  for (uint32_t w = tid; w < W; w += nt) {
    const Walker wk = b.walkers[J.walkers + w];
    const RankRec rr = b.ranks[J.ranks + wk.rank];
    const uint64_t si = b.reps[rr.rep].streams + wk.stream;
    const uint32_t len = b.clen ? b.clen[si] : b.streams[si].len;
    if (sh.st[w].i < len) s_incomplete = 1;
  }
  // epilogue: host end time, peak memory, first OOM (sim.py:235-242, 365-366)
  for (uint32_t r = tid; r < R; r += nt) {
    const RankRec rr = b.ranks[J.ranks + r];
    const RepHdr &h = b.reps[rr.rep];
    const uint32_t k = sh.hostk[r];
    if (k < h.n_syncs) { s_incomplete = 1; continue; }
    const int64_t hend = h.gend + delay_job[rr.delay + h.n_syncs];
    if (hend > tmax) tmax = hend;
    const RepOut ro = b.repout[rr.rep];
    atomicMax(&s_peak, (long long)ro.peak);
    if (ro.first_exceed >= 0) {
      const MemRec m = b.mems[h.mems + ro.first_exceed];
      atomicMin(&s_oom_t, (long long)(m.gpre + delay_job[rr.delay + m.seg]));
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
      if (m.gpre + delay_job[rr.delay + m.seg] == s_oom_t) atomicMin(&s_oom_rank, (int)r);
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

static const uint32_t SCHED_SMEM_CAP = 112 * 1024;

int sched_variant(uint32_t W, uint32_t R) {
  (void)W;
  const uint32_t nw = sched_warps(R);
  return nw == 4 ? 0 : nw == 8 ? 1 : 2;
}

// ---------------------------------------------------------------------------
// Affine run folding (the resolve pass of runs without a timeline).
//
// A kernel op is the max-plus map x -> max(x + d, disp + delay + d); a run of
// kernel ops of one FIFO inside one host-sync segment (one `delay`) composes
// to ONE such map, x -> max(x + A, B0 + delay) with A = sum d and
// B0 = fold of (disp + d).  The fold is written as a kernel op with
// d' = A, disp' = B0 - A, so both schedulers consume it unchanged and produce
// identical times (same maps, composed earlier).  One warp per FIFO streams
// its 16-byte ops once (segmented warp scan of the (A, B0) pairs), writes the
// folded FIFO in place of the ExecOp array (same base), its length (clen) and
// the per-sync dispatch counts in folded indices (ccounts: counts[k][s] =
// number of ops with segment <= k, so a segment change is a fold boundary).
// Runs are cut every 1,024 ops and only durations < 2^40 fold, so A < 2^50.
// Per-op fold eligibility and run starts of one 32-op window.  Eligibility
// reads the op only (a kernel whose gap prefix is < 2^61), so the counting
// pass does not gather durations; the writing pass saturates the composite at
// 2^62 and writes EXEC_OVF when it leaves int64 (every op time of the run
// does too: done >= sum of durations, done >= B0), and a failed estimate
// saturates as well (the job's status is ESTIMATION whatever the schedule).
static constexpr int64_t FOLD_SAT = (int64_t)1 << 62;
__device__ __forceinline__ int64_t sat_add(int64_t x, int64_t y) {   // x, y in [0, FOLD_SAT]
  const int64_t s = x + y;
  return s > FOLD_SAT ? FOLD_SAT : s;
}

// Both passes give each lane 32 consecutive ops of the 1,024-op chunk and walk
// them sequentially (a few instructions per op, not a warp scan per 32 ops);
// the warp combines the 32 lane results once per chunk.
// Collectives enter runs too when the packer marked them OP_FOLDC (their rep's
// coll_wf entry names a wire feature: every simulated rank meets them alone):
// done = ready + wire is the kernel map with d = wire.
__device__ __forceinline__ bool op_foldable(const Op &o, const uint32_t *) {
  return o.disp < ((int64_t)1 << 61) && (op_tag(o.meta) == TAG_KERN || (o.meta & OP_FOLDC));
}

// Kernel blocks (soa.h KBLOCK): the composite of a block's n kernels, kernel k
// dispatched k*gap after the first, relative to the first kernel's disp:
// A = sum d_k, Brel = fold of (k*gap + d_k) -- the same saturating maps the
// fold pass composes op by op, composed once per interned block (affine
// max-plus composition is associative, so the folded FIFO is identical up to
// where runs are cut, and the schedule is exact either way).  One warp per
// block: each lane composes a contiguous slice, then a shuffle tree.
__global__ void block_compose_kernel(DevBatch b) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= b.n_blocks) return;
  const KBlock kb = b.blocks[i];
  const uint32_t *fp = b.blk_fids + kb.fid0;
  const uint32_t per = (kb.n + 31) / 32, k0 = lane * per, k1 = min(kb.n, k0 + per);
  int64_t A = 0, B = 0;
  bool any = false;
  for (uint32_t k = k0; k < k1; k++) {
    const int64_t d = feat_dur(b, fp[k]);
    const int64_t de = (d < 0 || d > FOLD_SAT) ? FOLD_SAT : d;
    const int64_t bk = sat_add((int64_t)k * kb.gap, de);   // k * gap < 2^61 (packer)
    if (!any) {
      A = de;
      B = bk;
      any = true;
    } else {
      const int64_t nb = sat_add(B, de);
      B = nb > bk ? nb : bk;
      A = sat_add(A, de);
    }
  }
  // left-to-right tree: lane L absorbs lane L + off (identity: empty slice)
#pragma unroll
  for (uint32_t off = 1; off < 32; off <<= 1) {
    const int64_t A2 = __shfl_down_sync(FULL, A, off), B2 = __shfl_down_sync(FULL, B, off);
    const bool any2 = __shfl_down_sync(FULL, any, off);
    if ((lane & (2 * off - 1)) == 0 && lane + off < 32 && any2) {
      if (any) {
        const int64_t nb = sat_add(B, A2);
        B = nb > B2 ? nb : B2;
        A = sat_add(A, A2);
      } else {
        A = A2;
        B = B2;
        any = true;
      }
    }
  }
  if (lane == 0) {
    b.blk_ab[2 * (size_t)i] = A;
    b.blk_ab[2 * (size_t)i + 1] = B;
  }
}

// One pass: fold and write each chunk at its offset (FoldChunk.out, counted by
// the host packer with the same rule, pack.cpp); sync counts; lengths.
// 128-op windows, 4 consecutive ops per lane: a lane composes its 4 maps
// sequentially (branch-free), the warp scans the 32 lane composites once, and
// each lane writes the runs that end among its ops.
// BLOCKS: the batch has kernel blocks (KBLOCK ops enter as their composites);
// without, the kernel is the plain per-op fold.
template <bool BLOCKS>
__global__ void __launch_bounds__(128) fold_write_kernel(DevBatch b) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= b.n_chunks) return;
  const FoldChunk fc = b.chunks[c];
  const RepHdr &h = b.reps[fc.rep];
  const uint32_t ns = h.n_streams, nsync = h.n_syncs;
  const StreamRange sr = b.streams[h.streams + fc.st];
  const Op *in = b.ops + h.ops + sr.begin;
  const uint32_t *cw = b.coll_wf + h.colls;
  ExecOp *out = b.exec + h.ops + sr.begin;
  uint32_t *cc = b.ccounts + h.counts + fc.st;
  const uint32_t n = sr.len;
  const uint32_t lo = fc.chunk * FOLD_CHUNK, hi = min(n, lo + FOLD_CHUNK);
  uint32_t outpos = fc.out;   // folded ops of the FIFO before this window (host-counted)
  // no failed or wide duration in the batch (estimate_features_kernel's flags):
  // every feature's duration is its 4-byte word
  const bool plain = (*(volatile const int32_t *)b.err_flag & (1 | ERR_WIDE_DUR)) == 0;
  // carry from the previous window: last op's segment / foldability, open run
  uint32_t cseg = lo > 0 ? op_seg(in[lo - 1].meta) : 0;
  bool cfold = false;            // the chunk's first op always starts a run
  int64_t cA = 0, cB = 0;        // composite of the run open at the window edge
  for (uint32_t base = lo; base < hi; base += 128) {
    const uint32_t j0 = base + lane * 4u;
    Op o[4];
    int64_t d[4], bx[4];   // bx >= 0: a kernel block's Brel (d is its A)
    bool v[4], f[4], st[4];
    uint32_t sg[4];
#pragma unroll
    for (int t = 0; t < 4; t++) {
      v[t] = j0 + t < hi;
      o[t] = v[t] ? in[j0 + t] : Op{0, 0, 0};
      sg[t] = op_seg(o[t].meta);
      f[t] = v[t] && op_foldable(o[t], cw);
      d[t] = 0;
      bx[t] = -1;
      if (f[t] && op_tag(o[t].meta) == TAG_COLL) {
        d[t] = b.wire[cw[o[t].arg]];   // < 0: failed estimate, saturates (host sets ESTIMATION)
        if (d[t] < 0) d[t] = FOLD_SAT;
      } else if (v[t] && op_tag(o[t].meta) == TAG_KERN) {
        if (BLOCKS && (o[t].arg & KBLOCK)) {
          const longlong2 ab =
              *reinterpret_cast<const longlong2 *>(b.blk_ab + 2 * (size_t)(o[t].arg & ~KBLOCK));
          d[t] = ab.x;
          bx[t] = ab.y;
        } else {
          d[t] = plain ? (int64_t)b.feat_d32[o[t].arg] : feat_dur(b, o[t].arg);
        }
      }
    }
    // previous op of each of the lane's ops
    uint32_t psg = __shfl_up_sync(FULL, sg[3], 1);
    bool pf = __shfl_up_sync(FULL, f[3], 1);
    if (lane == 0) {
      psg = cseg;
      pf = cfold;
    }
    uint32_t nst = 0;   // starts among the lane's ops
#pragma unroll
    for (int t = 0; t < 4; t++) {
      const uint32_t ps = t ? sg[t - 1] : psg;
      const bool pfo = t ? f[t - 1] : pf;
      st[t] = v[t] && (j0 + t == lo || !f[t] || !pfo || sg[t] != ps);
      nst += st[t] ? 1u : 0u;
    }
    // lane composite of its last run (restarts at each start), affine pairs
    int64_t A = 0, B = 0;
    bool hs = false;     // the lane has a start
#pragma unroll
    for (int t = 0; t < 4; t++) {
      if (!v[t]) continue;
      const int64_t de = (d[t] < 0 || d[t] > FOLD_SAT) ? FOLD_SAT : d[t];
      const int64_t a = f[t] ? de : 0,
                    bb = f[t] ? sat_add(o[t].disp, (BLOCKS && bx[t] >= 0) ? bx[t] : de) : 0;
      if (st[t]) {
        A = a;
        B = bb;
        hs = true;
      } else {
        const int64_t nb = sat_add(B, a);
        B = nb > bb ? nb : bb;
        A = sat_add(A, a);
      }
    }
    // output index base of the lane: exclusive scan of start counts
    uint32_t incl = nst;
#pragma unroll
    for (uint32_t off = 1; off < 32; off <<= 1) {
      const uint32_t x = __shfl_up_sync(FULL, incl, off);
      if (lane >= off) incl += x;
    }
    const uint32_t obase = outpos + incl - nst;
    // incoming composite of the run open at the lane's first op
    int64_t sA = A, sB = B;
    bool sfl = hs || !v[0];
    if (lane == 0 && !hs) {   // continue the carried run
      const int64_t nb = sat_add(cB, sA);
      sB = nb > sB ? nb : sB;
      sA = sat_add(cA, sA);
      sfl = true;
    }
#pragma unroll
    for (uint32_t off = 1; off < 32; off <<= 1) {
      const int64_t A2 = __shfl_up_sync(FULL, sA, off);
      const int64_t B2 = __shfl_up_sync(FULL, sB, off);
      const bool f2 = __shfl_up_sync(FULL, sfl, off);
      if (lane >= off && !sfl) {
        const int64_t nb = sat_add(B2, sA);
        sB = nb > sB ? nb : sB;
        sA = sat_add(A2, sA);
        sfl = f2;
      }
    }
    int64_t iA = __shfl_up_sync(FULL, sA, 1), iB = __shfl_up_sync(FULL, sB, 1);
    if (lane == 0) {
      iA = cA;
      iB = cB;
    }
    // start flag of the op after the lane's last op
    bool nxt = __shfl_down_sync(FULL, st[0], 1);
    if (lane == 31 || j0 + 4 >= hi) nxt = true;   // window / chunk edge: resolved below
    // walk the lane's ops: write runs that end here, sync counts
    uint32_t oidx = obase - 1;
    int64_t rA = iA, rB = iB;
#pragma unroll
    for (int t = 0; t < 4; t++) {
      if (!v[t]) continue;
      const int64_t de = (d[t] < 0 || d[t] > FOLD_SAT) ? FOLD_SAT : d[t];
      const int64_t a = f[t] ? de : 0,
                    bb = f[t] ? sat_add(o[t].disp, (BLOCKS && bx[t] >= 0) ? bx[t] : de) : 0;
      if (st[t]) {
        oidx++;
        rA = a;
        rB = bb;
        const uint32_t ps = t ? sg[t - 1] : psg;
        if (sg[t] != ps)
          for (uint32_t k = ps; k < sg[t] && k < nsync; k++) cc[(size_t)k * ns] = oidx;
      } else {
        const int64_t nb = sat_add(rB, a);
        rB = nb > bb ? nb : bb;
        rA = sat_add(rA, a);
      }
      const bool ends = t < 3 ? (!v[t + 1] || st[t + 1]) : nxt;
      // a foldable run reaching the window edge (not the chunk end) stays open
      const bool edge = (t == 3 || !v[t + 1]) && (lane == 31 || j0 + t + 1 >= base + 128) &&
                        j0 + t + 1 < hi;
      if (ends && !(f[t] && edge)) {
        if (f[t]) {
          out[oidx] = (rA >= FOLD_SAT || rB >= FOLD_SAT)
                          ? ExecOp{0, EXEC_OVF}
                          : ExecOp{rB - rA, ((uint64_t)rA << 2) | TAG_KERN};
        } else {
          const uint32_t tag = op_tag(o[t].meta);
          const bool bad = d[t] < 0 || d[t] >= (int64_t)(EXEC_BAD >> 2);
          uint64_t pay;
          if (BLOCKS && tag == TAG_KERN && bx[t] >= 0) pay = EXEC_OVF >> 2;   // blocks always fold
          else if (tag == TAG_KERN) pay = bad ? (EXEC_BAD >> 2) : (uint64_t)d[t];
          else pay = (o[t].arg == NO_REC) ? (EXEC_NONE >> 2) : (uint64_t)o[t].arg;
          out[oidx] = ExecOp{o[t].disp, (pay << 2) | tag};
        }
      }
    }
    // carry to the next window: the last valid op of the window
    const uint32_t nwin = min(128u, hi - base);
    const uint32_t ll = (nwin - 1) >> 2, lt = (nwin - 1) & 3;
    const uint32_t sgl = lt == 0 ? sg[0] : lt == 1 ? sg[1] : lt == 2 ? sg[2] : sg[3];
    const bool fl = lt == 0 ? f[0] : lt == 1 ? f[1] : lt == 2 ? f[2] : f[3];
    const uint32_t lseg = __shfl_sync(FULL, sgl, ll);
    const bool lfold = __shfl_sync(FULL, fl, ll);
    const int64_t lA = __shfl_sync(FULL, rA, ll), lB = __shfl_sync(FULL, rB, ll);
    const uint32_t ltotal = __shfl_sync(FULL, incl, 31);
    // the next window's first op decides whether the carried run ends
    const bool more = base + 128 < hi;
    bool next_start = true;
    if (more) {
      const Op on = in[base + 128];
      next_start = !op_foldable(on, cw) || !lfold || op_seg(on.meta) != lseg;
    }
    if (lfold && lane == 0) {
      if (!more || next_start) {
        const uint32_t last_idx = outpos + ltotal - 1;
        out[last_idx] = (lA >= FOLD_SAT || lB >= FOLD_SAT)
                              ? ExecOp{0, EXEC_OVF}
                              : ExecOp{lB - lA, ((uint64_t)lA << 2) | TAG_KERN};
      }
    }
    cseg = lseg;
    cfold = lfold && more && !next_start;
    cA = lA;
    cB = lB;
    outpos += ltotal;
  }
  if (hi == n) {   // the FIFO's last chunk: counts of the remaining syncs, length
    const uint32_t last_seg = n > 0 ? cseg : 0;
    for (uint32_t k = last_seg + lane; k < nsync; k += 32) cc[(size_t)k * ns] = outpos;
    if (lane == 0) b.clen[h.streams + fc.st] = outpos;
  }
}

// FIFOs without ops have no chunk: their counts are 0, their length 0
__global__ void fold_empty_kernel(DevBatch b) {
  const uint32_t rep = blockIdx.x * blockDim.y + threadIdx.y;
  if (rep >= b.n_reps) return;
  const RepHdr &h = b.reps[rep];
  for (uint32_t st = 0; st < h.n_streams; st++) {
    if (b.streams[h.streams + st].len) continue;
    for (uint32_t k = threadIdx.x; k < h.n_syncs; k += 32)
      b.ccounts[h.counts + (size_t)k * h.n_streams + st] = 0;
    if (threadIdx.x == 0) b.clen[h.streams + st] = 0;
  }
}

void launch_resolve(const DevBatch &b, cudaStream_t s) {
  if (b.clen) {
    if (b.n_blocks)
      block_compose_kernel<<<(unsigned)((b.n_blocks * 32ull + 255) / 256), 256, 0, s>>>(b);
    if (b.n_chunks) {
      const unsigned gw = (unsigned)((b.n_chunks * 32ull + 127) / 128);
      if (b.n_blocks) fold_write_kernel<true><<<gw, 128, 0, s>>>(b);
      else fold_write_kernel<false><<<gw, 128, 0, s>>>(b);
    }
    if (b.n_reps) fold_empty_kernel<<<(b.n_reps + 7) / 8, dim3(32, 8), 0, s>>>(b);
  } else if (b.n_ops) {
    resolve_kernel<<<(unsigned)((b.n_ops + 255) / 256), 256, 0, s>>>(b);
  }
  if (b.n_rcolls)
    resolve_colls_kernel<<<(unsigned)((b.n_rcolls + 255) / 256), 256, 0, s>>>(b);
}

template <int NW>
static void launch_nw(const DevBatch &b, const int32_t *order, uint32_t n, int record,
                      uint32_t smem, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sched_warp_kernel<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SCHED_SMEM_CAP);
    attr = true;
  }
  sched_warp_kernel<NW><<<n, NW * 32, smem, s>>>(b, order, record, smem);
}

void launch_schedule_variant(const DevBatch &b, int variant, const int32_t *order, uint32_t n,
                             int record, uint32_t smem, cudaStream_t s) {
  if (!n) return;
  if (smem > SCHED_SMEM_CAP) smem = SCHED_SMEM_CAP;
  switch (variant) {
    case 0: launch_nw<4>(b, order, n, record, smem, s); break;
    case 1: launch_nw<8>(b, order, n, record, smem, s); break;
    default: launch_nw<16>(b, order, n, record, smem, s); break;
  }
}

uint32_t sched_smem_cap() { return SCHED_SMEM_CAP; }

extern "C" int maya_prof_read_sub(unsigned long long *out4, int reset) {
#ifdef MAYA_PROFILE
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out4, g_prof_sub, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_prof_sub, z, sizeof z);
  }
  return 1;
#else
  (void)out4;
  (void)reset;
  return 0;
#endif
}

int prof_read(unsigned long long *out8, int reset) {
#ifdef MAYA_PROFILE
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out8, g_prof, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_prof, z, sizeof z);
  }
  return 1;
#else
  (void)out8;
  (void)reset;
  return 0;
#endif
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
