// Per-rank busy statistics of the reference's _report (sim.py:406-473) on the
// device, from the timeline the scheduler recorded:
//   compute_busy = |union of kernel intervals|          (_union_len, :412)
//   comm_busy    = |union of collective intervals|      (_merge, :413-414)
//   busy         = |union of all timed intervals|       (:417)
//   exposed_comm = |comm \ compute| = busy - compute_busy   (_subtract_len, :415-416)
//   idle         = total - busy                         (:421)
// A union length over intervals sorted by start is sum_i max(0, e_i - max(s_i,
// M_{i-1})) with M the running max of the ends: one segmented sort of each
// simulated rank's (start, end|class) pairs, then one warp per rank walks its
// sorted intervals 32 at a time with three max-scans (all / compute / comm).
// Record and wait ops carry zero-length intervals: they never contribute and
// never raise a later term (their end <= every later start).
#include <cub/cub.cuh>

#include "kernels.cuh"

namespace maya {

namespace {

// (start, end << 2 | class) per timeline slot; class 0 compute, 1 comm, 2 untimed
__global__ void stats_keys_kernel(DevBatch b, const uint64_t *rank_seg, uint32_t n_ranks,
                                  int64_t *keys, uint64_t *vals) {
  for (uint32_t q = blockIdx.x; q < n_ranks; q += gridDim.x) {
    const uint64_t s0 = rank_seg[q], s1 = rank_seg[q + 1];
    const RepHdr &h = b.reps[b.ranks[q].rep];
    for (uint64_t k = threadIdx.x; k < s1 - s0; k += blockDim.x) {
      const uint32_t tag = op_tag(b.ops[h.ops + k].meta);
      const int64_t a = b.tl_start[s0 + k];
      int64_t e = b.tl_end[s0 + k];
      uint64_t cls = tag == TAG_KERN ? 0 : tag == TAG_COLL ? 1 : 2;
      if (cls == 2 || e < a) e = a;
      keys[s0 + k] = a;
      vals[s0 + k] = ((uint64_t)e << 2) | cls;
    }
  }
}

__device__ __forceinline__ int64_t smax(int64_t a, int64_t b) { return a > b ? a : b; }

// one warp per simulated rank: out[q] = {compute, comm, busy, peak}
__global__ void stats_union_kernel(DevBatch b, const uint64_t *rank_seg, uint32_t n_ranks,
                                   const int64_t *keys, const uint64_t *vals, int64_t *out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= n_ranks) return;
  const uint64_t s0 = rank_seg[q], s1 = rank_seg[q + 1];
  const int64_t NEG = INT64_MIN / 4;
  int64_t m[3] = {NEG, NEG, NEG};          // running max end before this window
  int64_t acc[3] = {0, 0, 0};
  for (uint64_t base = s0; base < s1; base += 32) {
    const uint64_t k = base + lane;
    int64_t a = 0, e = NEG;
    uint32_t cls = 2;
    if (k < s1) {
      a = keys[k];
      const uint64_t v = vals[k];
      e = (int64_t)(v >> 2);
      cls = (uint32_t)(v & 3);
    }
    // x = 0: every interval; 1: compute; 2: comm
#pragma unroll
    for (int x = 0; x < 3; x++) {
      const bool in = k < s1 && (x == 0 || (uint32_t)(x - 1) == cls);
      int64_t inc = in ? e : NEG;
#pragma unroll
      for (uint32_t off = 1; off < 32; off <<= 1) {
        const int64_t o = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc = smax(inc, o);
      }
      int64_t exc = __shfl_up_sync(0xffffffffu, inc, 1);
      exc = lane == 0 ? m[x] : smax(exc, m[x]);
      if (in) {
        const int64_t c = e - smax(a, exc);
        if (c > 0) acc[x] += c;
      }
      m[x] = smax(m[x], __shfl_sync(0xffffffffu, inc, 31));
    }
  }
#pragma unroll
  for (int x = 0; x < 3; x++)
#pragma unroll
    for (uint32_t off = 16; off > 0; off >>= 1) acc[x] += __shfl_down_sync(0xffffffffu, acc[x], off);
  if (lane == 0) {
    out[4 * q + 0] = acc[1];
    out[4 * q + 1] = acc[2];
    out[4 * q + 2] = acc[0];
    out[4 * q + 3] = b.repout[b.ranks[q].rep].peak;
  }
}

}  // namespace

size_t rank_stats_scratch_bytes(uint64_t n_tl, uint32_t n_ranks) {
  size_t tmp = 0;
  cub::DeviceSegmentedSort::SortPairs(nullptr, tmp, (const int64_t *)nullptr, (int64_t *)nullptr,
                                      (const uint64_t *)nullptr, (uint64_t *)nullptr, (int)n_tl,
                                      (int)n_ranks, (const uint64_t *)nullptr,
                                      (const uint64_t *)nullptr);
  return 32 * n_tl + tmp + 1024;
}

int launch_rank_stats(const DevBatch &b, const uint64_t *rank_seg, uint32_t n_ranks,
                      uint64_t n_tl, void *scratch, size_t scratch_bytes, int64_t *out,
                      cudaStream_t s) {
  if (n_ranks == 0) return 0;
  char *p = (char *)scratch;
  auto take = [&](size_t bytes) {
    char *r = p;
    p += (bytes + 255) & ~(size_t)255;
    return r;
  };
  int64_t *k_in = (int64_t *)take(8 * n_tl), *k_out = (int64_t *)take(8 * n_tl);
  uint64_t *v_in = (uint64_t *)take(8 * n_tl), *v_out = (uint64_t *)take(8 * n_tl);
  size_t tmp = scratch_bytes - (size_t)(p - (char *)scratch);
  stats_keys_kernel<<<n_ranks < 4096 ? n_ranks : 4096, 256, 0, s>>>(b, rank_seg, n_ranks, k_in,
                                                                      v_in);
  if (cub::DeviceSegmentedSort::SortPairs(p, tmp, k_in, k_out, v_in, v_out, (int)n_tl,
                                          (int)n_ranks, rank_seg, rank_seg + 1, s) != cudaSuccess)
    return -1;
  stats_union_kernel<<<(n_ranks + 7) / 8, 256, 0, s>>>(b, rank_seg, n_ranks, k_out, v_out, out);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace maya
