// Native restatement of the reference's synthetic frontend and collator:
//   validate_config            pkg/src/dltsim/workload.py:168-208
//   rank coords / comm ids     workload.py:226-278
//   unique_workers             workload.py:281-298
//   kernel inventory           workload.py:316-378 (_gemm, _elem, _layer_fwd_kernels,
//                              _embed/_head_fwd_kernels, _bwd_of)
//   memory model               workload.py:381-445
//   pipeline_order             workload.py:450-505
//   _TraceBuilder / generate_trace  workload.py:510-780
//   collate (groups, calls, comm_map)  pkg/src/dltsim/collate.py:256-372
//   topology_of                pkg/src/dltsim/cluster.py:79-92
// Output is a raw job identical, event for event, to
// rawtrace.from_reference(collate(*generate_representatives(...))) — checked
// by tests/test_gen.py against the reference's own traces.
#include "gen.h"

#include <algorithm>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <tuple>
#include <unordered_map>

namespace maya {

const char *const GEN_OP_KINDS[12] = {"gemm", "layernorm", "softmax", "gelu", "add", "embed",
                                      "cross_entropy", "optimizer_step", "memcpy_h2d",
                                      "memcpy_d2h", "memcpy_d2d", "memset"};
const char *const GEN_DTYPES[3] = {"bf16", "fp16", "fp32"};

enum { OK_GEMM = 0, OK_LAYERNORM, OK_SOFTMAX, OK_GELU, OK_ADD, OK_EMBED, OK_CROSS_ENTROPY,
       OK_OPTIMIZER, OK_MEMCPY_H2D, OK_MEMCPY_D2H, OK_MEMCPY_D2D, OK_MEMSET };
enum { DT_FP32 = 2 };
enum { K_ALLREDUCE = 0, K_ALLGATHER, K_REDUCESCATTER, K_BROADCAST, K_SENDRECV };
enum { STREAM_COMPUTE = 0, STREAM_GRAD_COMM = 1, FIRST_P2P_STREAM = 2 };

namespace {

struct GenFail {
  std::string msg;
};

typedef __int128 i128;

inline int64_t chk(i128 v) {
  if (v > (i128)INT64_MAX || v < -(i128)INT64_MAX) throw GenFail{"generated size overflows int64"};
  return (int64_t)v;
}

// Python floor division for the (always non-negative) sizes used here.
inline int64_t fdiv(i128 a, i128 b) {
  i128 q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
  return chk(q);
}


KSpec gemm(i128 m, i128 n, i128 k, i128 esz) {  // workload.py:316-318
  return KSpec{OK_GEMM, chk(2 * m * n * k), chk(esz * (m * k + k * n + m * n))};
}
KSpec elem(int op, i128 elems, i128 flops_per, i128 esz, i128 rw = 2) {  // :321-324
  return KSpec{op, chk(flops_per * elems), chk(rw * elems * esz)};
}

struct Shape {
  i128 s, h, v, esz, L;
};

std::vector<KSpec> layer_fwd(const Shape &M, i128 b, i128 tp, bool sp) {  // :327-348
  const i128 s = M.s, h = M.h, esz = M.esz;
  const i128 u = sp ? tp : 1;
  std::vector<KSpec> ks;
  ks.push_back(elem(OK_LAYERNORM, fdiv(b * s * h, u), 8, esz));
  ks.push_back(gemm(b * s, fdiv(3 * h, tp), h, esz));
  ks.push_back(KSpec{OK_GEMM, fdiv(2 * b * s * s * h, tp),
                     chk(esz * (fdiv(2 * b * s * h, tp) + fdiv(b * s * s, tp)))});
  ks.push_back(elem(OK_SOFTMAX, fdiv(b * s * s, tp), 5, esz));
  ks.push_back(KSpec{OK_GEMM, fdiv(2 * b * s * s * h, tp),
                     chk(esz * (fdiv(b * s * s, tp) + fdiv(2 * b * s * h, tp)))});
  ks.push_back(gemm(b * s, h, fdiv(h, tp), esz));
  ks.push_back(elem(OK_ADD, fdiv(b * s * h, u), 1, esz, 3));
  ks.push_back(elem(OK_LAYERNORM, fdiv(b * s * h, u), 8, esz));
  ks.push_back(gemm(b * s, fdiv(4 * h, tp), h, esz));
  ks.push_back(elem(OK_GELU, fdiv(4 * b * s * h, tp), 8, esz));
  ks.push_back(gemm(b * s, h, fdiv(4 * h, tp), esz));
  ks.push_back(elem(OK_ADD, fdiv(b * s * h, u), 1, esz, 3));
  return ks;
}

KSpec embed_fwd(const Shape &M, i128 b, i128 tp, bool sp) {  // :351-354
  const i128 u = sp ? tp : 1;
  return KSpec{OK_EMBED, 0, chk((i128)fdiv(b * M.s * M.h * M.esz, u) + b * M.s * 8)};
}

std::vector<KSpec> head_fwd(const Shape &M, i128 b, i128 tp, bool sp) {  // :357-364
  const i128 u = sp ? tp : 1;
  std::vector<KSpec> ks;
  ks.push_back(elem(OK_LAYERNORM, fdiv(b * M.s * M.h, u), 8, M.esz));
  ks.push_back(gemm(b * M.s, fdiv(M.v, tp), M.h, M.esz));
  ks.push_back(elem(OK_CROSS_ENTROPY, fdiv(b * M.s * M.v, tp), 5, M.esz));
  return ks;
}

std::vector<KSpec> bwd_of(const std::vector<KSpec> &fwd, size_t a, size_t e) {  // :367-378
  std::vector<KSpec> out;
  for (size_t q = e; q-- > a;) {
    const KSpec &k = fwd[q];
    if (k.op == OK_GEMM) {
      out.push_back(k);
      out.push_back(k);
    } else {
      out.push_back(KSpec{k.op, chk((i128)2 * k.flops), chk((i128)k.bytes + k.bytes / 2)});
    }
  }
  return out;
}

i128 layer_stash_elems(const Shape &M, i128 b, i128 tp, bool sp, bool rc) {  // :381-387
  const i128 s = M.s, h = M.h, u = sp ? tp : 1;
  if (rc) return fdiv(b * s * h, u);
  return (i128)fdiv(12 * b * s * h, tp) + fdiv(2 * b * s * s, tp) + fdiv(5 * b * s * h, u);
}

struct Chunk {
  int64_t vs, layers;
  bool has_embed, has_head;
};

std::vector<Chunk> device_chunks(const Shape &M, int p, int v, int stage) {  // :400-408
  const int64_t total_vs = (int64_t)p * v;
  const int64_t lpc = fdiv(M.L, total_vs);
  std::vector<Chunk> out;
  for (int c = 0; c < v; c++) {
    int64_t vs = stage + (int64_t)c * p;
    out.push_back(Chunk{vs, lpc, vs == 0, vs == total_vs - 1});
  }
  return out;
}

int64_t chunk_stash_bytes(const Shape &M, const maya_config &c, i128 b, const Chunk &ch) {
  const i128 tp = c.tp, u = c.seq_parallel ? tp : 1;  // :411-420
  i128 elems = (i128)ch.layers * layer_stash_elems(M, b, tp, c.seq_parallel, c.act_recompute);
  if (ch.has_head && !c.act_recompute)
    elems += (i128)fdiv(M.s * b * M.v, tp) + fdiv(b * M.s * M.h, u);
  return chk(elems * M.esz);
}

int64_t device_param_elems(const Shape &M, const maya_config &c, int stage) {  // :423-434
  const i128 h = M.h, v = M.v;
  const i128 per_layer = fdiv(12 * h * h, c.tp);
  i128 total = 0;
  for (const Chunk &ch : device_chunks(M, c.pp, c.virtual_stages, stage)) {
    total += (i128)ch.layers * per_layer;
    if (ch.has_embed) total += fdiv(v * h, c.tp);
    if (ch.has_head) total += fdiv(v * h, c.tp);
  }
  return chk(total);
}

enum Phase { FWD = 0, BWD = 1 };
struct Step {
  int phase;
  int64_t mb;
  int chunk;
};

// workload.py:450-505
std::vector<Step> pipeline_order(int schedule, int64_t p, int64_t m, int64_t v, int64_t stage) {
  std::vector<Step> order;
  if (schedule == 0) {
    if (v != 1) throw GenFail{"gpipe schedule runs with virtual_stages == 1"};
    for (int64_t j = 0; j < m; j++) order.push_back({FWD, j, 0});
    for (int64_t j = 0; j < m; j++) order.push_back({BWD, j, 0});
    return order;
  }
  if (schedule == 1) {
    if (v != 1) throw GenFail{"1f1b schedule runs with virtual_stages == 1"};
    if (m < p) throw GenFail{"1f1b with too few microbatches has no steady state"};
    int64_t warmup = std::min(p - 1 - stage, m);
    for (int64_t j = 0; j < warmup; j++) order.push_back({FWD, j, 0});
    for (int64_t i = 0; i < m - warmup; i++) {
      order.push_back({FWD, warmup + i, 0});
      order.push_back({BWD, i, 0});
    }
    for (int64_t j = m - warmup; j < m; j++) order.push_back({BWD, j, 0});
    return order;
  }
  if (schedule == 2) {
    if (v < 2) throw GenFail{"interleaved schedule requires virtual_stages > 1"};
    if (m % p != 0) throw GenFail{"interleaved schedule needs microbatches % pp == 0"};
    const int64_t total = m * v, group = p * v;
    auto fwd_step = [&](int64_t st) {
      return Step{FWD, st % p + (st / group) * p, (int)((st % group) / p)};
    };
    auto bwd_step = [&](int64_t st) {
      return Step{BWD, st % p + (st / group) * p, (int)(v - 1 - (st % group) / p)};
    };
    int64_t warmup = std::min(total, (p - stage - 1) * 2 + (v - 1) * p);
    for (int64_t i = 0; i < warmup; i++) order.push_back(fwd_step(i));
    for (int64_t i = 0; i < total - warmup; i++) {
      order.push_back(fwd_step(warmup + i));
      order.push_back(bwd_step(i));
    }
    for (int64_t i = total - warmup; i < total; i++) order.push_back(bwd_step(i));
    return order;
  }
  throw GenFail{"unknown schedule"};
}

// -- rank coordinates and communicators (workload.py:226-278)

struct Coords {
  int64_t t, d, p;
};

inline int64_t rank_of(const Coords &C, int64_t i, int64_t j, int64_t k) {
  return k * C.t * C.d + j * C.t + i;
}

enum CommType { C_TP = 0, C_DP, C_PF, C_PB };
struct CommRole {
  int type;
  int64_t a, b, c;  // TP: stage, dp; DP: tp, stage; PF/PB: boundary, tp, dp
  int32_t nranks, my_rank;
};

std::string comm_name(const CommRole &r) {
  char buf[96];
  switch (r.type) {
    case C_TP: snprintf(buf, sizeof buf, "tp.p%lld.d%lld", (long long)r.a, (long long)r.b); break;
    case C_DP: snprintf(buf, sizeof buf, "dp.t%lld.p%lld", (long long)r.a, (long long)r.b); break;
    case C_PF:
      snprintf(buf, sizeof buf, "pf%lld.t%lld.d%lld", (long long)r.a, (long long)r.b,
               (long long)r.c);
      break;
    default:
      snprintf(buf, sizeof buf, "pb%lld.t%lld.d%lld", (long long)r.a, (long long)r.b,
               (long long)r.c);
  }
  return buf;
}

void worker_comms(const Coords &C, int64_t v, int64_t rank, std::vector<CommRole> &out) {
  const int64_t i = rank % C.t, j = (rank / C.t) % C.d, k = rank / (C.t * C.d);
  out.clear();
  if (C.t > 1) out.push_back({C_TP, k, j, 0, (int32_t)C.t, (int32_t)i});
  if (C.d > 1) out.push_back({C_DP, i, k, 0, (int32_t)C.d, (int32_t)j});
  const int64_t total_vs = C.p * v;
  for (int64_t c = 0; c < v; c++) {
    int64_t vs = k + c * C.p;
    if (vs > 0) {
      out.push_back({C_PF, vs - 1, i, j, 2, 1});
      out.push_back({C_PB, vs - 1, i, j, 2, 0});
    }
    if (vs < total_vs - 1) {
      out.push_back({C_PF, vs, i, j, 2, 0});
      out.push_back({C_PB, vs, i, j, 2, 1});
    }
  }
}

// members of a communicator by position (resolved by collate from CommInits)
std::vector<int64_t> comm_members(const Coords &C, const CommRole &r) {
  std::vector<int64_t> m;
  switch (r.type) {
    case C_TP:
      for (int64_t i = 0; i < C.t; i++) m.push_back(rank_of(C, i, r.b, r.a));
      break;
    case C_DP:
      for (int64_t j = 0; j < C.d; j++) m.push_back(rank_of(C, r.a, j, r.b));
      break;
    case C_PF:  // position 0 sends (holds vs == boundary), 1 receives
      m.push_back(rank_of(C, r.b, r.c, r.a % C.p));
      m.push_back(rank_of(C, r.b, r.c, (r.a + 1) % C.p));
      break;
    default:    // PB: position 0 holds vs == boundary + 1 (sends gradients)
      m.push_back(rank_of(C, r.b, r.c, (r.a + 1) % C.p));
      m.push_back(rank_of(C, r.b, r.c, r.a % C.p));
  }
  return m;
}

// Rank of x's decimal string among the decimal strings of 0..65535 (string
// order: "1" < "10" < "11" < "2"); a monotone map of the name order of one
// numeric field, built once per process.
const uint16_t *decimal_string_rank() {
  static std::vector<uint16_t> rank;
  static std::once_flag once;
  std::call_once(once, [] {
    std::vector<std::pair<std::string, uint32_t>> v(65536);
    for (uint32_t x = 0; x < 65536; x++) v[x] = {std::to_string(x), x};
    std::sort(v.begin(), v.end());
    rank.resize(65536);
    for (uint32_t q = 0; q < 65536; q++) rank[v[q].second] = (uint16_t)q;
  });
  return rank.data();
}

// Sort key equal to the order of comm_name(r) strings.  Field separators are
// '.' (below every digit) and each name kind has a fixed shape, so comparing
// names = comparing (kind, field ranks) lexicographically.
uint64_t comm_order_key(const CommRole &r) {
  const uint16_t *R = decimal_string_rank();
  auto f = [&](int64_t x) -> uint64_t {
    if (x < 0 || x > 65535) throw GenFail{"communicator coordinate beyond 65535"};
    return R[x];
  };
  switch (r.type) {   // "dp" < "pb" < "pf" < "tp"
    case C_DP: return (0ull << 48) | (f(r.a) << 32) | (f(r.b) << 16);
    case C_PB: return (1ull << 48) | (f(r.a) << 32) | (f(r.b) << 16) | f(r.c);
    case C_PF: return (2ull << 48) | (f(r.a) << 32) | (f(r.b) << 16) | f(r.c);
    default: return (3ull << 48) | (f(r.a) << 32) | (f(r.b) << 16);
  }
}

// topology_of over the communicator's members (cluster.py:85-92), no lists kept
int8_t comm_topology(const Coords &C, const CommRole &r, int64_t dph, std::vector<int64_t> &hosts) {
  hosts.clear();
  switch (r.type) {
    case C_TP:
      for (int64_t i = 0; i < C.t; i++) hosts.push_back(rank_of(C, i, r.b, r.a) / dph);
      break;
    case C_DP:
      for (int64_t j = 0; j < C.d; j++) hosts.push_back(rank_of(C, r.a, j, r.b) / dph);
      break;
    case C_PF:
      hosts.push_back(rank_of(C, r.b, r.c, r.a % C.p) / dph);
      hosts.push_back(rank_of(C, r.b, r.c, (r.a + 1) % C.p) / dph);
      break;
    default:
      hosts.push_back(rank_of(C, r.b, r.c, (r.a + 1) % C.p) / dph);
      hosts.push_back(rank_of(C, r.b, r.c, r.a % C.p) / dph);
  }
  const size_t n = hosts.size();
  std::sort(hosts.begin(), hosts.end());
  const size_t u = (size_t)(std::unique(hosts.begin(), hosts.end()) - hosts.begin());
  return u == 1 ? 0 : (u == n ? 1 : 2);
}

// -- _TraceBuilder (workload.py:510-568)

struct Builder {
  std::vector<uint8_t> &kind;
  std::vector<int32_t> &stream;
  std::vector<int64_t> &f;
  EventSink *sink;
  int64_t overhead;
  int32_t dtype;
  std::vector<int32_t> comm_nranks;          // per local comm
  std::vector<int64_t> call_idx;             // per local comm
  std::vector<std::vector<std::pair<int8_t, int64_t>>> calls;  // per local comm
  std::vector<int64_t> next_version, last_version;   // by event id (small)
  int64_t next_alloc = 0;
  // kernel blocks (sinks that take them): the open run of kernel launches, as
  // segments of the trace's kernel lists (run-length coded).  A run whose
  // segments repeat an earlier run of this trace (a layer body of the next
  // microbatch) is emitted by its block id, without building or hashing its
  // launch list; the packer interns the list itself the first time.
  bool blocks = false;
  int32_t run_stream = 0;
  struct Seg {
    const KSpec *p;
    uint32_t n, rep;
    bool operator==(const Seg &o) const { return p == o.p && n == o.n && rep == o.rep; }
  };
  std::vector<Seg> rsegs;
  size_t run_n = 0;
  bool run_owned = false;          // a segment points at a temporary: never memoised
  std::vector<KSpec> run;          // materialised launch list (first occurrence)
  std::vector<KSpec> singles;      // copies of single launches passed by value
  struct Memo {
    uint64_t h;
    uint32_t seg0, nseg, id;
  };
  std::vector<Memo> memo;
  std::vector<Seg> memo_segs;

  void flush() {
    if (rsegs.empty()) return;
    const int64_t gap = overhead > 0 ? overhead : 0;
    uint64_t h = 0x9e3779b97f4a7c15ull;
    for (const Seg &g : rsegs)
      h = (h ^ ((uint64_t)(uintptr_t)g.p + ((uint64_t)g.n << 40) + ((uint64_t)g.rep << 52))) *
          0xff51afd7ed558ccdull;
    if (!run_owned)
      for (const Memo &m : memo)
        if (m.h == h && m.nseg == rsegs.size() &&
            std::equal(rsegs.begin(), rsegs.end(), memo_segs.begin() + m.seg0)) {
          if (sink->kernel_block_id(run_stream, m.id, run_n, gap)) {
            rsegs.clear();
            run_n = 0;
            return;
          }
          break;
        }
    run.clear();
    for (const Seg &g : rsegs)
      for (uint32_t r = 0; r < g.rep; r++) run.insert(run.end(), g.p, g.p + g.n);
    const uint32_t id = sink->kernel_block(run_stream, run.data(), run.size(), gap, dtype);
    if (id != ~0u && !run_owned) {
      memo.push_back(Memo{h, (uint32_t)memo_segs.size(), (uint32_t)rsegs.size(), id});
      memo_segs.insert(memo_segs.end(), rsegs.begin(), rsegs.end());
    }
    rsegs.clear();
    run_n = 0;
    run_owned = false;
    singles.clear();
  }
  void ev(uint8_t k, int32_t s, int64_t a, int64_t b = 0, int64_t c = 0, int64_t d = 0) {
    if (sink) {
      if (!rsegs.empty()) flush();
      sink->ev(k, s, a, b, c, d);
      return;
    }
    kind.push_back(k);
    stream.push_back(s);
    const size_t n = f.size();
    f.resize(n + 4);
    int64_t *p = f.data() + n;
    p[0] = a;
    p[1] = b;
    p[2] = c;
    p[3] = d;
  }
  void gap() {
    if (overhead > 0) ev(MAYA_EV_HOSTGAP, 0, overhead);
  }
  // a launch of a kernel list that lives for the whole trace
  void kernel(int32_t s, const KSpec &k) { kernels(s, &k, 1); }
  // a launch passed by value (a temporary): copied, its run never memoised
  void kernel_tmp(int32_t s, const KSpec &k) {
    if (blocks) {
      if (!rsegs.empty() && run_stream != s) flush();
      singles.reserve(16);
      if (singles.size() == singles.capacity()) flush();   // keep earlier segment pointers valid
      singles.push_back(k);
      run_owned = true;
      kernels(s, &singles.back(), 1);
      return;
    }
    kernels(s, &k, 1);
  }
  // n consecutive launches on stream s (one segment of the open run in block mode)
  void kernels(int32_t s, const KSpec *k, size_t n) {
    if (blocks) {
      if (!rsegs.empty() && run_stream != s) flush();
      run_stream = s;
      if (!rsegs.empty() && rsegs.back().p == k && rsegs.back().n == n) rsegs.back().rep++;
      else rsegs.push_back(Seg{k, (uint32_t)n, 1});
      run_n += n;
      return;
    }
    for (size_t i = 0; i < n; i++) {
      gap();
      ev(MAYA_EV_KERNEL, s, k[i].op, dtype, k[i].flops, k[i].bytes);
    }
  }
  void memcpy_h2d(int32_t s, int64_t n) {
    gap();
    ev(MAYA_EV_MEMCPY, s, OK_MEMCPY_H2D, DT_FP32, 0, n);
  }
  void memset_(int32_t s, int64_t n) {
    gap();
    ev(MAYA_EV_MEMSET, s, OK_MEMSET, DT_FP32, 0, n);
  }
  void collective(int32_t s, int lc, int kind_, int64_t n) {
    int64_t idx = call_idx[lc]++;
    ev(MAYA_EV_COLLECTIVE, s, lc, idx, kind_, n);
    calls[lc].emplace_back((int8_t)kind_, n);
  }
  void record(int32_t s, int64_t e) {
    if ((size_t)e >= next_version.size()) {
      next_version.resize(e + 1, 0);
      last_version.resize(e + 1, 0);
    }
    int64_t ver = next_version[e];
    next_version[e] = ver + 1;
    last_version[e] = ver;
    ev(MAYA_EV_RECORD, s, e, ver);
  }
  void wait_last(int32_t s, int64_t e) { ev(MAYA_EV_WAIT, s, e, last_version[e]); }
  int64_t alloc(int64_t n) {
    int64_t aid = next_alloc++;
    ev(MAYA_EV_MEMALLOC, 0, aid, n);
    return aid;
  }
  void free_(int64_t aid) { ev(MAYA_EV_MEMFREE, 0, aid); }
};

struct RepCalls {
  std::vector<std::vector<std::pair<int8_t, int64_t>>> calls;  // per local comm
};

// The builder side of a phase template (generate_trace): the template id in
// the packer, and the calls, event versions and allocations a replay adds.
struct BTpl {
  int id = -2;                                   // -2: not captured, -1: not replayable
  int tries = 0;                                 // captures attempted (the first occurrence
                                                 // of a phase often opens communicators)
  // the calls a replay appends: runs (lc, [begin, end) of call_data), by lc
  std::vector<std::pair<int, std::pair<uint32_t, uint32_t>>> call_runs;
  std::vector<std::pair<int8_t, int64_t>> call_data;     // (kind, bytes)
  std::vector<std::pair<int64_t, int64_t>> vers; // (event id, records)
  int64_t allocs = 0;
};
typedef std::array<int64_t, 20> TplKey;
// The phase templates of one job, shared by its reps: a worker-thread object
// reset per job, whose entries (and their vectors' capacity) are reused; a
// deque keeps the BTpl addresses the generator holds stable as it grows.
struct JobTpls {
  struct Ent {
    uint64_t hash = 0;
    TplKey key{};
    BTpl tpl;
  };
  std::deque<Ent> store;
  size_t used = 0;
  void reset() { used = 0; }
  BTpl &operator[](const TplKey &k) {
    uint64_t h = 1469598103934665603ull;
    for (int64_t x : k) h = (h ^ (uint64_t)x) * 1099511628211ull;
    for (size_t i = 0; i < used; i++)
      if (store[i].hash == h && store[i].key == k) return store[i].tpl;
    if (used == store.size()) store.emplace_back();
    Ent &e = store[used++];
    e.hash = h;
    e.key = k;
    BTpl &b = e.tpl;
    b.id = -2;
    b.tries = 0;
    b.call_runs.clear();
    b.call_data.clear();
    b.vers.clear();
    b.allocs = 0;
    return b;
  }
};

// workload.py:571-780 for one representative rank; appends events.
// A few dozen keyed entries per trace (communicator roles, p2p streams,
// event ids): a flat vector searched linearly, no node allocation per entry.
template <class K, class V>
struct FlatMap {
  std::vector<std::pair<K, V>> v;
  const V *get(const K &k) const {
    for (const auto &e : v)
      if (e.first == k) return &e.second;
    return nullptr;
  }
  std::pair<V *, bool> emplace(const K &k, const V &val) {
    for (auto &e : v)
      if (e.first == k) return {&e.second, false};
    v.emplace_back(k, val);
    return {&v.back().second, true};
  }
  V &operator[](const K &k) { return *emplace(k, V{}).first; }
};

void generate_trace(const Shape &M, const maya_config &cfg, const Coords &C, int schedule,
                    int64_t rank, int64_t overhead, int32_t dtype, GenJob &G, RepCalls &rc,
                    EventSink *sink, JobTpls *jtpl) {
  const int64_t t = C.t, d = C.d;
  const int64_t i = rank % t, j = (rank / t) % d, stage = rank / (t * d);
  const int64_t p = cfg.pp, v = cfg.virtual_stages, total_vs = p * v;
  const int64_t m = (int64_t)cfg.micro_mult * cfg.pp;
  const i128 b = fdiv(cfg.global_batch, (i128)d * m);
  const i128 s = M.s, h = M.h, esz = M.esz;
  const bool sp = cfg.seq_parallel != 0;
  const i128 u = sp ? t : 1;

  Builder B{G.ev_kind, G.ev_stream, G.ev_f, sink, overhead, dtype, {}, {}, {}, {}, {}, 0};
  std::vector<std::vector<std::pair<int8_t, int64_t>>> spare = std::move(rc.calls);   // capacity
  B.blocks = sink && sink->takes_blocks();
  {  // reserve for this trace: ~ (2 x kernels per layer-microbatch) + specials
    const size_t est = (size_t)(cfg.micro_mult) * (size_t)cfg.pp * (size_t)(M.L / cfg.pp + 2) *
                           (cfg.act_recompute ? 110 : 80) + 4096;
    if (sink) {
      sink->rep_begin(est);
    } else {
      G.ev_kind.reserve(G.ev_kind.size() + est);
      G.ev_stream.reserve(G.ev_stream.size() + est);
      G.ev_f.reserve(G.ev_f.size() + 4 * est);
    }
  }
  std::vector<CommRole> roles;
  worker_comms(C, v, rank, roles);
  // local comm index of each role (first CommInit of a comm id); keyed by the
  // role's integer fields, which comm_name spells out one to one
  FlatMap<std::tuple<int, int64_t, int64_t, int64_t>, int> local;
  for (const CommRole &r : roles) {
    int lc = (int)B.comm_nranks.size();
    if (!local.emplace(std::make_tuple(r.type, r.a, r.b, r.c), lc).second)
      throw GenFail{"duplicate communicator"};
    B.comm_nranks.push_back(r.nranks);
    B.call_idx.push_back(0);
    if (B.calls.size() < spare.size()) {
      B.calls.push_back(std::move(spare[B.calls.size()]));
      B.calls.back().clear();
    } else {
      B.calls.emplace_back();
    }
    B.ev(MAYA_EV_COMMINIT, 0, lc, r.nranks, r.my_rank);
  }
  auto lc_of = [&](int type, int64_t a, int64_t b2, int64_t c2) {
    const int *q = local.get(std::make_tuple(type, a, b2, c2));
    if (!q) throw GenFail{"communicator missing from worker_comms"};
    return *q;
  };

  std::vector<Chunk> chunks = device_chunks(M, (int)p, (int)v, (int)stage);
  FlatMap<std::pair<int64_t, int>, int32_t> p2p_stream;  // (boundary, role) -> stream
  FlatMap<std::pair<int, int64_t>, int64_t> eid;         // (key kind, boundary) -> id
  enum { R_FIN = 0, R_BOUT, R_FOUT, R_BIN };
  enum { E_FIN = 0, E_BOUT, E_FOUT, E_BIN, E_GRADS, E_DP_DONE, E_OPT_DONE, E_AG_DONE };
  int32_t next_stream = FIRST_P2P_STREAM;
  int64_t next_eid = 0;
  for (const Chunk &ch : chunks) {
    if (ch.vs > 0) {
      p2p_stream[{ch.vs - 1, R_FIN}] = next_stream++;
      p2p_stream[{ch.vs - 1, R_BOUT}] = next_stream++;
      eid[{E_FIN, ch.vs - 1}] = next_eid++;
      eid[{E_BOUT, ch.vs - 1}] = next_eid++;
    }
    if (ch.vs < total_vs - 1) {
      p2p_stream[{ch.vs, R_FOUT}] = next_stream++;
      p2p_stream[{ch.vs, R_BIN}] = next_stream++;
      eid[{E_FOUT, ch.vs}] = next_eid++;
      eid[{E_BIN, ch.vs}] = next_eid++;
    }
  }
  for (int key : {E_GRADS, E_DP_DONE, E_OPT_DONE, E_AG_DONE}) eid[{key, -1}] = next_eid++;

  // static allocations (device_memory_bytes, :437-445)
  const int64_t params = device_param_elems(M, cfg, (int)stage);
  int64_t opt = chk((i128)12 * params);
  if (cfg.dist_optimizer) opt = -fdiv(-(i128)opt, d);
  B.alloc(chk((i128)params * esz));
  const int64_t grads_bytes = chk((i128)params * 4);
  B.alloc(grads_bytes);
  B.alloc(opt);
  B.memset_(STREAM_COMPUTE, grads_bytes);

  const int64_t p2p_payload = fdiv(b * s * h * esz, u);
  const int64_t tp_coll_bytes = chk(b * s * h * esz);
  const int64_t loss_reduce_bytes = chk(b * s * 8);
  const int tp_lc = t > 1 ? lc_of(C_TP, stage, j, 0) : -1;
  // activation allocation handle of each (chunk, micro-batch), -1: none
  std::vector<int64_t> act_ids(chunks.size() * (size_t)m, -1);
  auto act = [&](int c, int64_t mb) -> int64_t & { return act_ids[(size_t)c * (size_t)m + (size_t)mb]; };

  // the kernel lists are a pure function of (model shape, micro-batch size,
  // tp, sp): memoised per worker thread (128-bit shape arithmetic per rep
  // otherwise); a shape that overflows throws before it is stored
  struct KSets {
    std::vector<KSpec> lks, hks, mlp_bwd, attn_bwd, head_bwd;
    KSpec eks;
  };
  thread_local std::map<std::array<int64_t, 8>, KSets> ks_memo;
  const std::array<int64_t, 8> ks_key{(int64_t)M.s, (int64_t)M.h, (int64_t)M.v, (int64_t)M.esz,
                                      (int64_t)M.L, (int64_t)b, (int64_t)t, sp ? 1 : 0};
  auto ks_it = ks_memo.find(ks_key);
  if (ks_it == ks_memo.end()) {
    KSets k;
    k.lks = layer_fwd(M, b, t, sp);
    k.hks = head_fwd(M, b, t, sp);
    k.eks = embed_fwd(M, b, t, sp);
    k.mlp_bwd = bwd_of(k.lks, 7, 12);
    k.attn_bwd = bwd_of(k.lks, 0, 7);
    k.head_bwd = bwd_of(k.hks, 0, 3);
    if (ks_memo.size() > 4096) ks_memo.clear();
    ks_it = ks_memo.emplace(ks_key, std::move(k)).first;
  }
  const std::vector<KSpec> &lks = ks_it->second.lks;
  const std::vector<KSpec> &hks = ks_it->second.hks;
  const KSpec eks = ks_it->second.eks;
  const std::vector<KSpec> &mlp_bwd = ks_it->second.mlp_bwd;
  const std::vector<KSpec> &attn_bwd = ks_it->second.attn_bwd;
  const std::vector<KSpec> &head_bwd = ks_it->second.head_bwd;

  auto tp_pair_fwd = [&]() {
    if (t > 1) B.collective(STREAM_COMPUTE, tp_lc, sp ? K_REDUCESCATTER : K_ALLREDUCE, tp_coll_bytes);
  };
  auto tp_gather_fwd = [&]() {
    if (t > 1 && sp) B.collective(STREAM_COMPUTE, tp_lc, K_ALLGATHER, tp_coll_bytes);
  };
  auto emit_layer_fwd = [&]() {
    if (t == 1) {   // no tensor-parallel collectives between the launches
      B.kernels(STREAM_COMPUTE, lks.data(), 12);
      return;
    }
    B.kernel(STREAM_COMPUTE, lks[0]);
    tp_gather_fwd();
    B.kernels(STREAM_COMPUTE, &lks[1], 5);
    tp_pair_fwd();
    B.kernels(STREAM_COMPUTE, &lks[6], 2);
    tp_gather_fwd();
    B.kernels(STREAM_COMPUTE, &lks[8], 3);
    tp_pair_fwd();
    B.kernel(STREAM_COMPUTE, lks[11]);
  };
  auto emit_layer_fwd_compute_only = [&]() {
    B.kernels(STREAM_COMPUTE, lks.data(), lks.size());
  };
  auto emit_head_fwd = [&](bool compute_only) {
    B.kernel(STREAM_COMPUTE, hks[0]);
    if (!compute_only) tp_gather_fwd();
    B.kernel(STREAM_COMPUTE, hks[1]);
    B.kernel(STREAM_COMPUTE, hks[2]);
    if (!compute_only && t > 1) B.collective(STREAM_COMPUTE, tp_lc, K_ALLREDUCE, loss_reduce_bytes);
  };
  auto emit_layer_bwd = [&]() {
    if (t > 1) B.collective(STREAM_COMPUTE, tp_lc, sp ? K_ALLGATHER : K_ALLREDUCE, tp_coll_bytes);
    B.kernels(STREAM_COMPUTE, mlp_bwd.data(), mlp_bwd.size());
    if (t > 1 && sp) B.collective(STREAM_COMPUTE, tp_lc, K_REDUCESCATTER, tp_coll_bytes);
    if (t > 1) B.collective(STREAM_COMPUTE, tp_lc, sp ? K_ALLGATHER : K_ALLREDUCE, tp_coll_bytes);
    B.kernels(STREAM_COMPUTE, attn_bwd.data(), attn_bwd.size());
    if (t > 1 && sp) B.collective(STREAM_COMPUTE, tp_lc, K_REDUCESCATTER, tp_coll_bytes);
  };
  auto emit_forward = [&](int64_t mb, int chunk_id) {
    const Chunk &ch = chunks[chunk_id];
    const int64_t vs = ch.vs;
    act(chunk_id, mb) = B.alloc(chunk_stash_bytes(M, cfg, b, ch));
    if (vs > 0) {
      int32_t fin = p2p_stream[{vs - 1, R_FIN}];
      B.collective(fin, lc_of(C_PF, vs - 1, i, j), K_SENDRECV, p2p_payload);
      B.record(fin, eid[{E_FIN, vs - 1}]);
      B.wait_last(STREAM_COMPUTE, eid[{E_FIN, vs - 1}]);
    } else {
      B.memcpy_h2d(STREAM_COMPUTE, chk(b * s * 8));
      B.kernel(STREAM_COMPUTE, eks);
    }
    for (int64_t l = 0; l < ch.layers; l++) emit_layer_fwd();
    if (ch.has_head) emit_head_fwd(false);
    if (vs < total_vs - 1) {
      int32_t fout = p2p_stream[{vs, R_FOUT}];
      B.record(STREAM_COMPUTE, eid[{E_FOUT, vs}]);
      B.wait_last(fout, eid[{E_FOUT, vs}]);
      B.collective(fout, lc_of(C_PF, vs, i, j), K_SENDRECV, p2p_payload);
    }
  };
  auto emit_backward = [&](int64_t mb, int chunk_id) {
    const Chunk &ch = chunks[chunk_id];
    const int64_t vs = ch.vs;
    if (vs < total_vs - 1) {
      int32_t bin = p2p_stream[{vs, R_BIN}];
      B.collective(bin, lc_of(C_PB, vs, i, j), K_SENDRECV, p2p_payload);
      B.record(bin, eid[{E_BIN, vs}]);
      B.wait_last(STREAM_COMPUTE, eid[{E_BIN, vs}]);
    }
    if (cfg.act_recompute) {
      if (ch.has_embed) B.kernel(STREAM_COMPUTE, eks);
      for (int64_t l = 0; l < ch.layers; l++) emit_layer_fwd_compute_only();
      if (ch.has_head) emit_head_fwd(true);
    }
    if (ch.has_head)
      B.kernels(STREAM_COMPUTE, head_bwd.data(), head_bwd.size());
    for (int64_t l = 0; l < ch.layers; l++) emit_layer_bwd();
    if (ch.has_embed) B.kernel(STREAM_COMPUTE, eks);
    if (vs > 0) {
      int32_t bout = p2p_stream[{vs - 1, R_BOUT}];
      B.record(STREAM_COMPUTE, eid[{E_BOUT, vs - 1}]);
      B.wait_last(bout, eid[{E_BOUT, vs - 1}]);
      B.collective(bout, lc_of(C_PB, vs - 1, i, j), K_SENDRECV, p2p_payload);
    }
    int64_t &h = act(chunk_id, mb);
    B.free_(h);
    h = -1;
  };

  // Phase templates (kernel-block sinks): every forward / backward of one
  // chunk emits the same events up to counters, so the packer captures the
  // first occurrence and stamps the later ones; the builder replays its own
  // side -- call lists and call numbers, event versions, allocation handles
  // (pack.cpp RepPacker::phase_*).  Templates are shared by the job's reps:
  // a phase's events are fixed by its chunk's shape and the local indices it
  // touches (streams, event ids, communicators) -- the key -- and the
  // config-wide kernel lists and sizes, so isomorphic pipeline stages (every
  // middle stage) pack each phase once per job.
  // (kernel-block mode always cuts runs at phase boundaries, replay or not, so
  // both pack the same kernel blocks)
  const bool tpl_on = B.blocks && jtpl;
  const bool replay = tpl_on && sink->replays();
  std::vector<BTpl *> btpl(tpl_on ? 2 * chunks.size() : 0);
  if (tpl_on)
    for (size_t c = 0; c < chunks.size(); c++) {
      const Chunk &ch = chunks[c];
      const int64_t vs = ch.vs;
      const bool in = vs > 0, out = vs < total_vs - 1;
      for (int ph = 0; ph < 2; ph++) {
        const TplKey key{ph, ch.layers, ch.has_embed ? 1 : 0, ch.has_head ? 1 : 0, in, out,
                         in ? p2p_stream[{vs - 1, R_FIN}] : -1,
                         in ? p2p_stream[{vs - 1, R_BOUT}] : -1,
                         out ? p2p_stream[{vs, R_FOUT}] : -1,
                         out ? p2p_stream[{vs, R_BIN}] : -1,
                         in ? eid[{E_FIN, vs - 1}] : -1, in ? eid[{E_BOUT, vs - 1}] : -1,
                         out ? eid[{E_FOUT, vs}] : -1, out ? eid[{E_BIN, vs}] : -1,
                         in ? lc_of(C_PF, vs - 1, i, j) : -1, in ? lc_of(C_PB, vs - 1, i, j) : -1,
                         out ? lc_of(C_PF, vs, i, j) : -1, out ? lc_of(C_PB, vs, i, j) : -1,
                         tp_lc, chunk_stash_bytes(M, cfg, b, ch)};
        btpl[2 * c + (ph == 0 ? 0 : 1)] = &(*jtpl)[key];
      }
    }
  std::vector<size_t> calls0;
  std::vector<int64_t> vers0;
  // the order is a pure function of (schedule, p, m, v, stage): memoised per
  // worker thread (configs of a batch share their pipeline shapes); a failing
  // shape throws before it is stored
  thread_local std::map<std::array<int64_t, 5>, std::vector<Step>> po_memo;
  const std::array<int64_t, 5> po_key{schedule, p, m, v, stage};
  auto po_it = po_memo.find(po_key);
  if (po_it == po_memo.end()) {
    if (po_memo.size() > 4096) po_memo.clear();
    po_it = po_memo.emplace(po_key, pipeline_order(schedule, p, m, v, stage)).first;
  }
  for (const Step &st : po_it->second) {
    if (!tpl_on) {
      if (st.phase == FWD) emit_forward(st.mb, st.chunk);
      else emit_backward(st.mb, st.chunk);
      continue;
    }
    BTpl &bt = *btpl[2 * st.chunk + (st.phase == FWD ? 0 : 1)];
    B.flush();   // phases start and end outside a kernel run
    if (replay && bt.id >= 0 && sink->phase_replay(bt.id, B.next_alloc)) {
      act(st.chunk, st.mb) = st.phase == FWD ? B.next_alloc : -1;   // its one allocation
      B.next_alloc += bt.allocs;
      for (const auto &run : bt.call_runs) {   // one range append per communicator
        auto &dst = B.calls[run.first];
        dst.insert(dst.end(), bt.call_data.begin() + run.second.first,
                   bt.call_data.begin() + run.second.second);
        B.call_idx[run.first] += (int64_t)(run.second.second - run.second.first);
      }
      for (const auto &e : bt.vers) {
        B.next_version[e.first] += e.second;
        B.last_version[e.first] = B.next_version[e.first] - 1;
      }
      continue;
    }
    const bool capture = replay && bt.id < 0 && bt.tries < 3;
    if (capture) {
      sink->phase_begin(B.next_alloc);
      calls0.resize(B.calls.size());
      for (size_t lc = 0; lc < B.calls.size(); lc++) calls0[lc] = B.calls[lc].size();
      vers0 = B.next_version;
    }
    const int64_t aid0 = B.next_alloc;
    if (st.phase == FWD) emit_forward(st.mb, st.chunk);
    else emit_backward(st.mb, st.chunk);
    B.flush();
    if (capture) {
      bt.tries++;
      bt.call_runs.clear();
      bt.call_data.clear();
      bt.vers.clear();
      bt.id = sink->phase_end();
      bt.allocs = B.next_alloc - aid0;
      if (st.phase == FWD && bt.allocs != 1) bt.id = -1;   // replay assumes one activation alloc
      // call lists in issue order across communicators are not needed: each
      // communicator's list is appended in its own order
      for (size_t lc = 0; lc < B.calls.size(); lc++) {
        if (B.calls[lc].size() <= calls0[lc]) continue;
        const uint32_t b0 = (uint32_t)bt.call_data.size();
        bt.call_data.insert(bt.call_data.end(), B.calls[lc].begin() + calls0[lc], B.calls[lc].end());
        bt.call_runs.push_back({(int)lc, {b0, (uint32_t)bt.call_data.size()}});
      }
      for (size_t e = 0; e < B.next_version.size(); e++) {
        const int64_t before = e < vers0.size() ? vers0[e] : 0;
        if (B.next_version[e] != before) bt.vers.push_back({(int64_t)e, B.next_version[e] - before});
      }
    }
  }

  // gradient reduction and optimizer step (:757-777)
  const int64_t grad_comm_bytes = chk((i128)params * esz);
  if (d > 1) {
    const int dp_lc = lc_of(C_DP, i, stage, 0);
    B.record(STREAM_COMPUTE, eid[{E_GRADS, -1}]);
    B.wait_last(STREAM_GRAD_COMM, eid[{E_GRADS, -1}]);
    B.collective(STREAM_GRAD_COMM, dp_lc, cfg.dist_optimizer ? K_REDUCESCATTER : K_ALLREDUCE,
                 grad_comm_bytes);
    B.record(STREAM_GRAD_COMM, eid[{E_DP_DONE, -1}]);
    B.wait_last(STREAM_COMPUTE, eid[{E_DP_DONE, -1}]);
  }
  B.kernel_tmp(STREAM_COMPUTE, KSpec{OK_OPTIMIZER, chk((i128)6 * params), chk((i128)16 * params)});
  if (d > 1 && cfg.dist_optimizer) {
    const int dp_lc = lc_of(C_DP, i, stage, 0);
    B.record(STREAM_COMPUTE, eid[{E_OPT_DONE, -1}]);
    B.wait_last(STREAM_GRAD_COMM, eid[{E_OPT_DONE, -1}]);
    B.collective(STREAM_GRAD_COMM, dp_lc, K_ALLGATHER, grad_comm_bytes);
    B.record(STREAM_GRAD_COMM, eid[{E_AG_DONE, -1}]);
    B.wait_last(STREAM_COMPUTE, eid[{E_AG_DONE, -1}]);
  }
  B.ev(MAYA_EV_DSYNC, 0, 0);
  rc.calls = std::move(B.calls);
  if (sink) sink->rep_end();
}

// workload.py:168-208 (cluster divisibility + model + schedule rules)
void validate(const maya_model &model, const maya_config &c, int64_t n, int schedule) {
  if (std::min({(int64_t)c.tp, (int64_t)c.pp, (int64_t)c.micro_mult, (int64_t)c.virtual_stages,
                c.global_batch}) < 1)
    throw GenFail{"tp/pp/micro_mult/virtual_stages/global_batch must be >= 1"};
  if (n % ((int64_t)c.tp * c.pp) != 0) throw GenFail{"tp*pp does not divide device count"};
  const int64_t d = n / ((int64_t)c.tp * c.pp), m = (int64_t)c.micro_mult * c.pp;
  std::string errs;
  if (c.global_batch % (d * m) != 0) errs += "global_batch not divisible by dp*microbatches; ";
  if (model.hidden_size % c.tp) errs += "hidden_size not divisible by tp; ";
  if (model.seq_len % c.tp) errs += "seq_len not divisible by tp; ";
  if (model.vocab_size % c.tp) errs += "vocab_size not divisible by tp; ";
  if (model.num_layers % ((int64_t)c.pp * c.virtual_stages))
    errs += "num_layers not divisible by pp*virtual_stages; ";
  if (c.virtual_stages > 1 && c.pp == 1) errs += "virtual_stages > 1 requires pp > 1; ";
  if (schedule == 2 && c.virtual_stages == 1) errs += "interleaved schedule requires virtual_stages > 1; ";
  if (schedule != 2 && c.virtual_stages > 1) errs += "schedule requires virtual_stages == 1; ";
  if (schedule == 1 && m < c.pp) errs += "1f1b needs microbatches >= pp for warmup; ";
  if (!errs.empty()) throw GenFail{errs};
}

}  // namespace

namespace {

// The communicators of a job (collate.py:297-323): one per distinct role over
// all ranks, in the reference's global (name) order, with the stage and local
// index of its position-0 member (whose calls become the group's call table),
// its topology, and every rank's local -> global translation.
struct CommStruct {
  std::vector<CommRole> role;
  std::vector<int32_t> nranks, first_stage, first_lc;
  std::vector<int8_t> topo;
  std::vector<int64_t> rank_comm_off;
  std::vector<int32_t> rank_comm;
  // distinct (first stage, first local index) pairs and how many comms take
  // their calls from each (total call count = sum of mult x calls of the pair)
  std::vector<int32_t> pair_stage, pair_lc, pair_mult;
  std::string error;
};

std::shared_ptr<const CommStruct> build_comm_struct(const Coords &C, int64_t v, int64_t n,
                                                    int64_t dph) {
  auto cs = std::make_shared<CommStruct>();
  // Roles are keyed by integers (each communicator's name spells its fields
  // out one to one)
  auto role_key = [](const CommRole &r) -> uint64_t {
    return ((uint64_t)r.type << 60) | ((uint64_t)r.a << 40) | ((uint64_t)r.b << 20) |
           (uint64_t)r.c;
  };
  struct CInfo {
    CommRole role;
    int32_t stage_of_first;  // stage of position-0 rank
    int32_t lc_of_first;     // local comm index of the role in that rank's rep
  };
  // role key -> comm (discovery order): open addressing, sized for every
  // (rank, role) pair, so the table never grows
  std::vector<CInfo> infos;
  std::vector<int32_t> comm_of;                  // per rank, per local comm: discovery index
  std::vector<int64_t> rk_off(n + 1, 0);
  const size_t roles_per_rank = 2 + 4 * (size_t)v;
  size_t cap = 64;
  while (cap < 2 * (size_t)n * roles_per_rank) cap <<= 1;
  std::vector<uint64_t> hkey(cap, ~0ull);
  std::vector<int32_t> hval(cap, -1);
  auto slot_of = [&](uint64_t key) {
    size_t h = (size_t)((key * 0x9E3779B97F4A7C15ull) >> 20) & (cap - 1);
    while (hkey[h] != key && hkey[h] != ~0ull) h = (h + 1) & (cap - 1);
    return h;
  };
  std::vector<CommRole> roles;
  for (int64_t r = 0; r < n; r++) {
    worker_comms(C, v, r, roles);
    for (size_t q = 0; q < roles.size(); q++) {
      const uint64_t key = role_key(roles[q]);
      const size_t h = slot_of(key);
      if (hkey[h] == ~0ull) {
        hkey[h] = key;
        hval[h] = (int32_t)infos.size();
        infos.push_back(CInfo{roles[q], -1, -1});
      }
      comm_of.push_back(hval[h]);
      CInfo &ci = infos[hval[h]];
      if (roles[q].my_rank == 0 && ci.stage_of_first < 0) {
        ci.role = roles[q];
        ci.stage_of_first = (int32_t)(r / (C.t * C.d));
        ci.lc_of_first = (int32_t)q;
      }
    }
    rk_off[r + 1] = (int64_t)comm_of.size();
  }
  // JobTrace.groups order = sorted by name (collate.py:323).  The names are
  // "dp.t<i>.p<k>" < "pb<v>.t<i>.d<j>" < "pf<v>.t<i>.d<j>" < "tp.p<k>.d<j>", so the
  // string order is the order of (kind, decimal-string rank of each field):
  // an integer key per communicator, no names needed
  std::vector<uint64_t> okey(infos.size());
  for (size_t g = 0; g < infos.size(); g++) okey[g] = comm_order_key(infos[g].role);
  std::vector<int32_t> order(infos.size());
  for (size_t g = 0; g < order.size(); g++) order[g] = (int32_t)g;
  std::sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return okey[x] < okey[y]; });
  std::vector<int32_t> gid_of(infos.size());
  std::vector<int64_t> hosts_buf;
  for (size_t gi = 0; gi < order.size(); gi++) {
    const int32_t g0 = order[gi];
    gid_of[g0] = (int32_t)gi;
    const CInfo &ci = infos[g0];
    if (ci.stage_of_first < 0) {
      cs->error = "communicator without a position-0 member";
      return cs;
    }
    cs->role.push_back(ci.role);
    cs->nranks.push_back(ci.role.nranks);
    cs->first_stage.push_back(ci.stage_of_first);
    cs->first_lc.push_back(ci.lc_of_first);
    cs->topo.push_back(comm_topology(C, ci.role, dph, hosts_buf));
  }
  cs->rank_comm_off.push_back(0);
  for (int64_t r = 0; r < n; r++) {
    for (int64_t q = rk_off[r]; q < rk_off[r + 1]; q++) cs->rank_comm.push_back(gid_of[comm_of[q]]);
    cs->rank_comm_off.push_back((int64_t)cs->rank_comm.size());
  }
  {
    std::map<std::pair<int32_t, int32_t>, int32_t> mult;
    for (size_t g = 0; g < cs->first_stage.size(); g++) mult[{cs->first_stage[g], cs->first_lc[g]}]++;
    for (const auto &kv : mult) {
      cs->pair_stage.push_back(kv.first.first);
      cs->pair_lc.push_back(kv.first.second);
      cs->pair_mult.push_back(kv.second);
    }
  }
  return cs;
}

}  // namespace

maya_raw_job GenJob::raw(int32_t device) const {
  maya_raw_job r{};
  r.num_ranks = num_ranks;
  r.devices_per_host = devices_per_host;
  r.capacity = capacity;
  r.device = device;
  r.n_reps = (int32_t)rep_ranks.size();
  r.rank_rep = rank_rep.data();
  r.ev_off = ev_off.data();
  r.ev_kind = ev_kind.data();
  r.ev_stream = ev_stream.data();
  r.ev_f = ev_f.data();
  r.n_comms = (int32_t)comm_nranks.size();
  r.comm_nranks = comm_nranks.data();
  r.comm_topo = comm_topo.data();
  r.call_off = call_off.data();
  r.call_kind = call_kind.data();
  r.call_bytes = call_bytes.data();
  r.rank_comm_off = rank_comm_off.data();
  r.rank_comm = rank_comm.data();
  r.kernel_ns = nullptr;
  r.wire_ns = nullptr;
  return r;
}

int generate_job(const maya_model &model, const maya_config &cfg, const maya_cluster &cl,
                 int32_t schedule, int64_t overhead, GenJob &G, std::string *err,
                 EventSink *sink, GenCache *cache) {
  G.clear();   // keep capacity: a worker thread reuses one GenJob across configs
  try {
    if (cl.num_hosts < 1 || cl.devices_per_host < 1) throw GenFail{"empty cluster"};
    if (model.dtype < 0 || model.dtype > 2) throw GenFail{"unknown dtype"};
    const int64_t n = (int64_t)cl.num_hosts * cl.devices_per_host;
    if (schedule < 0) schedule = cfg.virtual_stages > 1 ? 2 : 1;  // default_schedule
    validate(model, cfg, n, schedule);
    Shape M{model.seq_len, model.hidden_size, model.vocab_size,
            model.dtype == 2 ? 4 : 2, model.num_layers};
    Coords C{cfg.tp, n / ((int64_t)cfg.tp * cfg.pp), cfg.pp};
    G.num_ranks = (int32_t)n;
    G.num_hosts = cl.num_hosts;
    G.devices_per_host = cl.devices_per_host;
    G.capacity = cl.device_memory_bytes;
    // representatives: one per stage (unique_workers, :281-298)
    std::vector<RepCalls> rcalls(cfg.pp);
    // the previous config's call lists (this worker's GenJob) lend their
    // capacity to this one's (generate_trace reuses them, cleared)
    for (size_t k = 0; k < rcalls.size() && k < G.rep_calls.size(); k++)
      rcalls[k].calls = std::move(G.rep_calls[k]);
    thread_local JobTpls jtpl;   // phase templates of the job
    jtpl.reset();
    G.ev_off.push_back(0);
    for (int k = 0; k < cfg.pp; k++) {
      int64_t rep = rank_of(C, 0, 0, k);
      G.rep_ranks.push_back(rep);
      generate_trace(M, cfg, C, schedule, rep, overhead, model.dtype, G, rcalls[k], sink, &jtpl);
      G.ev_off.push_back((int64_t)G.ev_kind.size());
    }
    G.rank_rep.resize(n);
    for (int64_t r = 0; r < n; r++) G.rank_rep[r] = (int32_t)(r / (C.t * C.d));
    // communicators: every role of every rank (collate.py:297-322), their
    // global order, topology and each rank's translation -- a function of the
    // parallel layout only, shared across the batch's configurations (cache)
    std::shared_ptr<const CommStruct> cs;
    if (cache && sink) {
      const std::array<int64_t, 6> key{1, C.t, C.d, C.p, cfg.virtual_stages, cl.devices_per_host};
      cs = cache->get<CommStruct>(key, [&] { return build_comm_struct(C, cfg.virtual_stages, n, cl.devices_per_host); });
    } else {
      cs = build_comm_struct(C, cfg.virtual_stages, n, cl.devices_per_host);
    }
    if (!cs->error.empty()) throw GenFail{cs->error};
    if (cache && sink) {   // lazy call tables (GenJob::comm_calls)
      G.lazy_calls = true;
      G.comm_nranks = cs->nranks;
      G.comm_topo = cs->topo;
      G.comm_first_stage = cs->first_stage;
      G.comm_first_lc = cs->first_lc;
      G.rep_calls.resize(rcalls.size());
      for (size_t k = 0; k < rcalls.size(); k++) G.rep_calls[k] = std::move(rcalls[k].calls);
      int64_t nc = 0;
      for (size_t q = 0; q < cs->pair_stage.size(); q++)
        nc += (int64_t)cs->pair_mult[q] * (int64_t)G.rep_calls[cs->pair_stage[q]][cs->pair_lc[q]].size();
      G.n_calls_total = nc;
      G.rank_comm_off = cs->rank_comm_off;
      G.rank_comm = cs->rank_comm;
      return MAYA_OK;
    }
    G.call_off.push_back(0);
    for (size_t gi = 0; gi < cs->nranks.size(); gi++) {
      G.comm_nranks.push_back(cs->nranks[gi]);
      G.comm_topo.push_back(cs->topo[gi]);
      const auto &cl2 = rcalls[cs->first_stage[gi]].calls[cs->first_lc[gi]];
      for (auto &kb : cl2) {
        G.call_kind.push_back(kb.first);
        G.call_bytes.push_back(kb.second);
      }
      G.call_off.push_back((int64_t)G.call_kind.size());
      if (!sink) {
        const std::string nm = comm_name(cs->role[gi]);
        G.comm_names.push_back(nm);
        G.comm_blob += nm;
        G.comm_blob += '\n';
      }
    }
    G.rank_comm_off = cs->rank_comm_off;
    G.rank_comm = cs->rank_comm;
  } catch (const GenFail &f) {
    if (err) *err = f.msg;
    return MAYA_EINVAL;
  }
  return MAYA_OK;
}

}  // namespace maya
