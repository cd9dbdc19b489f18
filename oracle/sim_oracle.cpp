// ORACLE — test infrastructure only.  Not part of the product path.
//
// CPU restatement of the reference's event-driven simulator and estimators,
// consuming the raw-job arrays of include/maya_b200.h:
//   * kernel roofline           pkg/src/dltsim/estimate.py:120-134 (_ceil_div :63-64)
//   * alpha-beta collectives    pkg/src/dltsim/estimate.py:79-100, cluster.py:55-59
//   * annotate error order      pkg/src/dltsim/estimate.py:329-361
//   * _compile_rank             pkg/src/dltsim/sim.py:135-174
//   * _advance_host             pkg/src/dltsim/sim.py:222-270
//   * _check_host_drain         pkg/src/dltsim/sim.py:272-283
//   * _fire / _try_start / _pump pkg/src/dltsim/sim.py:287-353
//   * run / _check_residue      pkg/src/dltsim/sim.py:357-402
//   * _report / _merge / _union_len / _subtract_len  sim.py:406-473
// The heap (t, tie, kind, rank, stream) and the worklist are kept, so event
// ordering (and hence the timeline order and first_oom) follows the reference.
// Only the only-in-tests pieces may import this (tests/, smoke(), bench.py's
// cpu_baseline / --impl reference leg).  Parity pinned by tests/golden/.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <deque>
#include <queue>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>
#include <algorithm>
#include <thread>
#include <atomic>

#include "../include/maya_b200.h"

typedef unsigned __int128 u128;
typedef __int128 i128;

namespace {

enum Tag { GAP, MEM, KERN, COLL, REC, WAIT, ESYNC, SSYNC, DSYNC };

struct Op {
  int tag;
  int32_t stream;
  int64_t val;    // GAP dur, MEM delta, KERN dur
  int64_t seq;
  int64_t e, v;   // REC/WAIT/ESYNC
  int64_t gkey;   // COLL global call index
  int32_t name;   // KERN: op-kind id (or -1-kernelclass); COLL: kind id
};

struct Stream {
  std::deque<int> queue;
  int running = -1;
  int64_t start = 0;
  bool waiting = false;
  uint64_t wait_key = 0;
  bool drained() const { return running < 0 && queue.empty() && !waiting; }
};

struct Waiter { bool host; int rank; int stream; };

struct HeapEv {
  int64_t t; int64_t tie; int kind; int rank; int stream;  // kind 0 host, 1 end
  bool operator>(const HeapEv &o) const {
    if (t != o.t) return t > o.t;
    return tie > o.tie;
  }
};

struct Interval { int cls; int stream; int32_t name; int64_t seq; int64_t a, b; };

struct Fail { int status; std::string msg; };

static inline int64_t ceil_div_u128(u128 a, u128 b) {
  u128 q = a / b + ((a % b) ? 1 : 0);
  if (q > (u128)INT64_MAX) throw Fail{MAYA_ST_OVERFLOW, "duration overflows int64"};
  return (int64_t)q;
}

static inline u128 mul_chk(u128 a, u128 b) {
  u128 r;
  if (__builtin_mul_overflow(a, b, &r)) throw Fail{MAYA_ST_OVERFLOW, "128-bit overflow in estimator"};
  return r;
}

// estimate.py:120-134
static int64_t roofline(const maya_device_params &dev, const maya_roofline_params &roof,
                        int64_t op_kind, int64_t dtype, int64_t flops, int64_t bytes) {
  int64_t compute = 0;
  if (flops > 0) {
    int64_t peak = (dtype >= 0 && dtype < MAYA_MAX_DTYPES) ? dev.peak_flops[dtype] : 0;
    if (peak <= 0) throw Fail{MAYA_ST_ESTIMATION, "no peak rate for dtype"};
    if (op_kind < 0 || op_kind >= roof.n_op_kinds) throw Fail{MAYA_ST_BAD_INPUT, "op kind id"};
    u128 num = mul_chk(mul_chk((u128)flops, (u128)1000000000ULL), (u128)roof.eff_den[op_kind]);
    u128 den = mul_chk((u128)peak, (u128)roof.eff_num[op_kind]);
    compute = ceil_div_u128(num, den);
  }
  int64_t memory = 0;
  if (bytes > 0) memory = ceil_div_u128(mul_chk((u128)bytes, (u128)1000000000ULL),
                                        (u128)dev.hbm_bytes_per_s);
  int64_t m = compute > memory ? compute : memory;
  if (m > INT64_MAX - roof.overhead_ns) throw Fail{MAYA_ST_OVERFLOW, "duration overflows int64"};
  return m + roof.overhead_ns;
}

// estimate.py:79-100
static int64_t collective(const maya_device_params &dev, int kind, int64_t bytes, int64_t n,
                          int topo) {
  if (n < 1) throw Fail{MAYA_ST_ESTIMATION, "collective with nranks < 1"};
  if (n == 1) return 0;
  int li = topo == 0 ? 0 : 1;
  u128 a = (u128)dev.alpha_ns[li], beta = (u128)dev.beta_bytes_per_s[li];
  u128 nn = (u128)n;
  u128 r;
  if (kind == 0) {
    r = mul_chk(2 * (nn - 1), a) +
        (u128)ceil_div_u128(mul_chk(mul_chk(2 * (nn - 1), (u128)bytes), 1000000000ULL),
                            mul_chk(nn, beta));
  } else if (kind == 1 || kind == 2) {
    r = mul_chk(nn - 1, a) +
        (u128)ceil_div_u128(mul_chk(mul_chk(nn - 1, (u128)bytes), 1000000000ULL),
                            mul_chk(nn, beta));
  } else if (kind == 3 || kind == 4) {
    r = a + (u128)ceil_div_u128(mul_chk((u128)bytes, 1000000000ULL), beta);
  } else {
    throw Fail{MAYA_ST_ESTIMATION, "unknown collective kind"};
  }
  if (r > (u128)INT64_MAX) throw Fail{MAYA_ST_OVERFLOW, "wire time overflows int64"};
  return (int64_t)r;
}

struct Sim {
  const maya_raw_job &job;
  const maya_device_params &dev;
  int R;
  std::vector<int64_t> kernel_ns;  // per event
  std::vector<int64_t> wire;       // per call
  std::vector<std::vector<Op>> ops;
  std::vector<size_t> host_idx;
  std::vector<int> host_blocked;   // 0 none, 1 gap, 2 event, 3 ssync, 4 dsync
  std::vector<int32_t> host_block_stream;
  std::vector<uint64_t> host_block_key;
  std::vector<char> host_finished;
  std::vector<std::vector<std::pair<int32_t, Stream>>> streams;  // creation order
  std::priority_queue<HeapEv, std::vector<HeapEv>, std::greater<HeapEv>> heap;
  int64_t tie = 0, now = 0, max_t = 0;
  std::unordered_set<uint64_t> fired;
  std::unordered_map<uint64_t, std::vector<Waiter>> event_waiters;
  std::unordered_map<int64_t, std::vector<std::pair<int, int>>> arrivals;
  std::vector<int64_t> arrival_order;  // insertion order for residue
  std::deque<std::pair<int, int>> worklist;
  std::unordered_set<uint64_t> on_worklist;
  std::vector<int64_t> mem, peak;
  int first_oom_rank = -1; int64_t first_oom_seq = -1;
  int64_t dispatched = 0, completed = 0;
  std::vector<std::vector<Interval>> intervals;

  Sim(const maya_raw_job &j, const maya_device_params &d) : job(j), dev(d), R(j.num_ranks) {}

  static uint64_t ekey(int rank, int64_t e, int64_t v) {
    if (e < 0 || e >= (1 << 20) || v < 0 || v >= (1 << 20))
      throw Fail{MAYA_ST_BAD_INPUT, "event id/version out of oracle range"};
    return ((uint64_t)rank << 40) | ((uint64_t)e << 20) | (uint64_t)v;
  }

  Stream *find_stream(int rank, int32_t s) {
    for (auto &p : streams[rank]) if (p.first == s) return &p.second;
    return nullptr;
  }
  Stream &stream(int rank, int32_t s) {
    Stream *st = find_stream(rank, s);
    if (st) return *st;
    streams[rank].emplace_back(s, Stream());
    return streams[rank].back().second;
  }

  void push(int64_t t, int kind, int rank, int s) { tie++; heap.push({t, tie, kind, rank, s}); }

  void mark(int rank, int s) {
    uint64_t k = ((uint64_t)rank << 32) | (uint32_t)s;
    if (on_worklist.insert(k).second) worklist.emplace_back(rank, s);
  }

  // sim.py:135-174
  void compile_rank(int rank) {
    int rep = job.rank_rep[rank];
    int64_t b = job.ev_off[rep], e = job.ev_off[rep + 1];
    std::unordered_map<int64_t, int64_t> alloc_bytes;
    std::vector<Op> &out = ops[rank];
    for (int64_t i = b; i < e; i++) {
      const int64_t *f = job.ev_f + 4 * i;
      int k = job.ev_kind[i];
      int32_t s = job.ev_stream[i];
      int64_t seq = i - b;
      Op op{};
      op.seq = seq; op.stream = s; op.name = -1;
      switch (k) {
        case MAYA_EV_HOSTGAP: op.tag = GAP; op.val = f[0]; break;
        case MAYA_EV_KERNEL: case MAYA_EV_MEMCPY: case MAYA_EV_MEMSET:
          op.tag = KERN; op.val = kernel_ns[i]; op.name = (int32_t)f[0]; break;
        case MAYA_EV_MEMALLOC: alloc_bytes[f[0]] = f[1]; op.tag = MEM; op.val = f[1]; break;
        case MAYA_EV_MEMFREE: {
          auto it = alloc_bytes.find(f[0]);
          if (it == alloc_bytes.end()) throw Fail{MAYA_ST_INTERNAL, "free of unallocated handle"};
          op.tag = MEM; op.val = -it->second; break;
        }
        case MAYA_EV_COMMINIT: continue;
        case MAYA_EV_COLLECTIVE: {
          int64_t lc = f[0];
          int64_t cb = job.rank_comm_off[rank], ce = job.rank_comm_off[rank + 1];
          if (lc < 0 || cb + lc >= ce) throw Fail{MAYA_ST_BAD_INPUT, "collective comm index"};
          int g = job.rank_comm[cb + lc];
          int64_t ncall = job.call_off[g + 1] - job.call_off[g];
          if (f[1] < 0 || f[1] >= ncall) throw Fail{MAYA_ST_BAD_INPUT, "collective call index"};
          op.tag = COLL; op.gkey = job.call_off[g] + f[1]; op.name = (int32_t)f[2];
          break;
        }
        case MAYA_EV_RECORD: op.tag = REC; op.e = f[0]; op.v = f[1]; break;
        case MAYA_EV_WAIT: op.tag = WAIT; op.e = f[0]; op.v = f[1]; break;
        case MAYA_EV_ESYNC: op.tag = ESYNC; op.e = f[0]; op.v = f[1]; break;
        case MAYA_EV_SSYNC: op.tag = SSYNC; break;
        case MAYA_EV_DSYNC: op.tag = DSYNC; break;
        default: throw Fail{MAYA_ST_BAD_INPUT, "unknown event kind"};
      }
      out.push_back(op);
    }
  }

  bool all_drained(int rank) {
    for (auto &p : streams[rank]) if (!p.second.drained()) return false;
    return true;
  }

  // sim.py:222-270
  void advance_host(int rank) {
    host_blocked[rank] = 0;
    std::vector<Op> &o = ops[rank];
    size_t &idx = host_idx[rank];
    while (idx < o.size()) {
      Op &op = o[idx];
      switch (op.tag) {
        case GAP:
          idx++;
          if (op.val > 0) { host_blocked[rank] = 1; push(now + op.val, 0, rank, -1); return; }
          break;
        case MEM:
          mem[rank] += op.val;
          if (mem[rank] > peak[rank]) peak[rank] = mem[rank];
          if (mem[rank] > job.capacity && first_oom_rank < 0) {
            first_oom_rank = rank; first_oom_seq = op.seq;
          }
          idx++;
          break;
        case ESYNC: {
          uint64_t key = ekey(rank, op.e, op.v);
          if (fired.count(key)) { idx++; }
          else {
            host_blocked[rank] = 2; host_block_key[rank] = key;
            event_waiters[key].push_back({true, rank, -1});
            return;
          }
          break;
        }
        case SSYNC: {
          Stream *st = find_stream(rank, op.stream);
          if (!st || st->drained()) idx++;
          else { host_blocked[rank] = 3; host_block_stream[rank] = op.stream; return; }
          break;
        }
        case DSYNC:
          if (all_drained(rank)) idx++;
          else { host_blocked[rank] = 4; return; }
          break;
        default:
          stream(rank, op.stream).queue.push_back((int)idx);
          dispatched++;
          mark(rank, op.stream);
          idx++;
      }
    }
    host_finished[rank] = 1;
  }

  // sim.py:272-283
  void check_host_drain(int rank) {
    if (host_blocked[rank] == 0 || host_finished[rank]) return;
    if (host_blocked[rank] == 3) {
      Stream *st = find_stream(rank, host_block_stream[rank]);
      if (!st || st->drained()) advance_host(rank);
    } else if (host_blocked[rank] == 4) {
      if (all_drained(rank)) advance_host(rank);
    }
  }

  // sim.py:287-300
  void fire(int rank, int64_t e, int64_t v) {
    uint64_t key = ekey(rank, e, v);
    fired.insert(key);
    auto it = event_waiters.find(key);
    if (it == event_waiters.end()) return;
    std::vector<Waiter> ws = std::move(it->second);
    event_waiters.erase(it);
    for (auto &w : ws) {
      if (!w.host) {
        Stream &st = stream(w.rank, w.stream);
        if (st.waiting && st.wait_key == key) {
          st.waiting = false;
          st.queue.pop_front();
          completed++;
          mark(w.rank, w.stream);
        }
      } else {
        advance_host(w.rank);
      }
    }
  }

  // sim.py:302-347
  void try_start(int rank, int s) {
    Stream *stp = &stream(rank, s);
    while (stp->running < 0 && !stp->waiting && !stp->queue.empty()) {
      Op &op = ops[rank][stp->queue.front()];
      if (op.tag == REC) {
        stp->queue.pop_front();
        completed++;
        fire(rank, op.e, op.v);
        stp = &stream(rank, s);   // fire may create streams (vector realloc)
      } else if (op.tag == WAIT) {
        uint64_t key = ekey(rank, op.e, op.v);
        if (fired.count(key)) { stp->queue.pop_front(); completed++; }
        else {
          stp->waiting = true; stp->wait_key = key;
          event_waiters[key].push_back({false, rank, s});
          break;
        }
      } else if (op.tag == KERN) {
        stp->running = stp->queue.front();
        stp->queue.pop_front();
        stp->start = now;
        if (op.val > INT64_MAX - now) throw Fail{MAYA_ST_OVERFLOW, "time overflow"};
        push(now + op.val, 1, rank, s);
        break;
      } else if (op.tag == COLL) {
        stp->running = stp->queue.front();
        stp->queue.pop_front();
        stp->start = now;
        auto ins = arrivals.emplace(op.gkey, std::vector<std::pair<int, int>>());
        if (ins.second) arrival_order.push_back(op.gkey);
        auto &members = ins.first->second;
        members.emplace_back(rank, s);
        int64_t g = 0;
        // comm of this call: find by call_off (binary search)
        {
          int lo = 0, hi = job.n_comms - 1;
          while (lo < hi) {
            int mid = (lo + hi + 1) / 2;
            if (job.call_off[mid] <= op.gkey) lo = mid; else hi = mid - 1;
          }
          g = lo;
        }
        int n = job.comm_nranks[g];
        if ((int)members.size() > n) throw Fail{MAYA_ST_INTERNAL, "internal error: too many arrivals"};
        if ((int)members.size() == n) {
          int64_t w = wire[op.gkey];
          if (w > INT64_MAX - now) throw Fail{MAYA_ST_OVERFLOW, "time overflow"};
          int64_t end = now + w;
          std::vector<std::pair<int, int>> ms = std::move(members);
          arrivals.erase(op.gkey);
          for (auto &m : ms) push(end, 1, m.first, m.second);
        }
        break;
      } else {
        throw Fail{MAYA_ST_INTERNAL, "internal error: op tag on stream"};
      }
    }
    if (stp->drained()) check_host_drain(rank);
  }

  void pump() {
    while (!worklist.empty()) {
      auto p = worklist.front();
      worklist.pop_front();
      on_worklist.erase(((uint64_t)p.first << 32) | (uint32_t)p.second);
      try_start(p.first, p.second);
    }
  }

  void run() {
    ops.resize(R); host_idx.assign(R, 0); host_blocked.assign(R, 0);
    host_block_stream.assign(R, 0); host_block_key.assign(R, 0); host_finished.assign(R, 0);
    streams.resize(R); mem.assign(R, 0); peak.assign(R, 0); intervals.resize(R);
    for (int r = 0; r < R; r++) { compile_rank(r); host_finished[r] = ops[r].empty(); }
    for (int r = 0; r < R; r++) advance_host(r);
    pump();
    while (!heap.empty()) {
      HeapEv ev = heap.top();
      heap.pop();
      now = ev.t;
      if (ev.t > max_t) max_t = ev.t;
      if (ev.kind == 0) {
        advance_host(ev.rank);
      } else {
        Stream &st = stream(ev.rank, ev.stream);
        Op &op = ops[ev.rank][st.running];
        st.running = -1;
        completed++;
        intervals[ev.rank].push_back({op.tag == COLL ? 1 : 0, ev.stream, op.name, op.seq,
                                      st.start, ev.t});
        mark(ev.rank, ev.stream);
      }
      pump();
    }
  }

  // sim.py:382-402 — returns a residue message or empty string
  std::string residue() {
    std::string out;
    char buf[256];
    for (int r = 0; r < R; r++) {
      if (!host_finished[r]) {
        const char *why = host_blocked[r] == 1 ? "gap" : host_blocked[r] == 2 ? "event"
                        : host_blocked[r] == 3 ? "ssync" : host_blocked[r] == 4 ? "dsync" : "None";
        snprintf(buf, sizeof buf, "rank %d: host blocked on %s\n", r, why);
        out += buf;
      }
      std::vector<std::pair<int32_t, Stream *>> ss;
      for (auto &p : streams[r]) ss.emplace_back(p.first, &p.second);
      std::sort(ss.begin(), ss.end(), [](auto &a, auto &b) { return a.first < b.first; });
      for (auto &p : ss) {
        Stream &st = *p.second;
        if (st.waiting) {
          snprintf(buf, sizeof buf, "rank %d stream %d: waiting on event (%d, %lld, %lld)\n", r,
                   p.first, r, (long long)((st.wait_key >> 20) & 0xFFFFF),
                   (long long)(st.wait_key & 0xFFFFF));
          out += buf;
        } else if (st.running >= 0 && ops[r][st.running].tag == COLL) {
          snprintf(buf, sizeof buf, "rank %d stream %d: stalled in collective %lld\n", r, p.first,
                   (long long)ops[r][st.running].gkey);
          out += buf;
        } else if (!st.queue.empty() || st.running >= 0) {
          snprintf(buf, sizeof buf, "rank %d stream %d: %zu ops queued\n", r, p.first,
                   st.queue.size());
          out += buf;
        }
      }
    }
    std::vector<int64_t> keys;
    for (auto &kv : arrivals) keys.push_back(kv.first);
    std::sort(keys.begin(), keys.end());
    for (int64_t k : keys) {
      auto &m = arrivals[k];
      int lo = 0, hi = job.n_comms - 1;
      while (lo < hi) { int mid = (lo + hi + 1) / 2; if (job.call_off[mid] <= k) lo = mid; else hi = mid - 1; }
      snprintf(buf, sizeof buf, "collective %lld: %zu/%d arrived\n", (long long)k, m.size(),
               job.comm_nranks[lo]);
      out += buf;
    }
    return out;
  }
};

static std::vector<std::pair<int64_t, int64_t>> merge(std::vector<std::pair<int64_t, int64_t>> iv) {
  std::sort(iv.begin(), iv.end());
  std::vector<std::pair<int64_t, int64_t>> out;
  for (auto &p : iv) {
    if (p.second <= p.first) continue;
    if (!out.empty() && p.first <= out.back().second) {
      if (p.second > out.back().second) out.back().second = p.second;
    } else {
      out.push_back(p);
    }
  }
  return out;
}

static int64_t union_len(std::vector<std::pair<int64_t, int64_t>> iv) {
  int64_t t = 0;
  for (auto &p : merge(std::move(iv))) t += p.second - p.first;
  return t;
}

static int64_t subtract_len(const std::vector<std::pair<int64_t, int64_t>> &base,
                            const std::vector<std::pair<int64_t, int64_t>> &cut) {
  int64_t total = 0;
  size_t ci = 0;
  for (auto &ab : base) {
    int64_t a = ab.first, b = ab.second, pos = a;
    while (ci < cut.size() && cut[ci].second <= pos) ci++;
    size_t k = ci;
    while (pos < b) {
      if (k >= cut.size() || cut[k].first >= b) { total += b - pos; break; }
      int64_t ca = cut[k].first, cb = cut[k].second;
      if (ca > pos) total += ca - pos;
      pos = std::max(pos, cb);
      k++;
    }
  }
  return total;
}

thread_local std::string g_err;

}  // namespace

extern "C" {

const char *oracle_last_error(void) { return g_err.c_str(); }

// estimate.py:329-361 over one job: fills kernel_ns[E] (-1 for non-kernel
// events) and wire[n_calls] (-1 for unused slots).  Returns status.
int oracle_annotate(const maya_raw_job *job, const maya_device_params *dev,
                    const maya_roofline_params *roof, int64_t *kernel_ns, int64_t *wire,
                    int64_t *err_rep, int64_t *err_seq) {
  *err_rep = -1; *err_seq = -1;
  int64_t E = job->ev_off[job->n_reps];
  try {
    for (int rep = 0; rep < job->n_reps; rep++) {
      for (int64_t i = job->ev_off[rep]; i < job->ev_off[rep + 1]; i++) {
        int k = job->ev_kind[i];
        kernel_ns[i] = -1;
        if (k != MAYA_EV_KERNEL && k != MAYA_EV_MEMCPY && k != MAYA_EV_MEMSET) continue;
        if (job->kernel_ns) { kernel_ns[i] = job->kernel_ns[i]; continue; }
        const int64_t *f = job->ev_f + 4 * i;
        *err_rep = rep; *err_seq = i - job->ev_off[rep];
        kernel_ns[i] = roofline(*dev, *roof, f[0], f[1], f[2], f[3]);
      }
    }
    *err_rep = -1; *err_seq = -1;
    int64_t nc = job->call_off[job->n_comms];
    for (int g = 0; g < job->n_comms; g++) {
      for (int64_t c = job->call_off[g]; c < job->call_off[g + 1]; c++) {
        wire[c] = -1;
        if (job->call_kind[c] < 0) continue;
        if (job->wire_ns) { wire[c] = job->wire_ns[c]; continue; }
        wire[c] = collective(*dev, job->call_kind[c], job->call_bytes[c], job->comm_nranks[g],
                             job->comm_topo[g]);
      }
    }
    (void)nc; (void)E;
  } catch (const Fail &f) {
    g_err = f.msg;
    return f.status;
  }
  return MAYA_ST_OK;
}

// Full annotate + simulate of one job.  rank_stats: [R][5] compute_busy,
// comm_busy, exposed_comm, idle, peak_mem (may be NULL).  Timeline arrays
// (may be NULL) need capacity >= number of timed ops; *n_timeline receives
// the count.  Timeline rows follow the reference: per rank, in end-event
// order (sim.py:375, 425-426).  name = op-kind id (kernels) or kind id (comm).
int oracle_simulate(const maya_raw_job *job, const maya_device_params *dev,
                    const maya_roofline_params *roof, maya_job_result *out,
                    int64_t *rank_stats, int32_t *tl_rank, int32_t *tl_stream, int64_t *tl_seq,
                    int64_t *tl_start, int64_t *tl_end, int32_t *tl_class, int64_t *n_timeline,
                    char *msg, int32_t msglen) {
  memset(out, 0, sizeof *out);
  out->first_oom_rank = -1; out->first_oom_seq = -1;
  if (msg && msglen) msg[0] = 0;
  int64_t E = job->ev_off[job->n_reps];
  int64_t rank_ops = 0;
  for (int r = 0; r < job->num_ranks; r++) {
    int rep = job->rank_rep[r];
    rank_ops += job->ev_off[rep + 1] - job->ev_off[rep];
  }
  out->rank_ops = rank_ops;
  Sim sim(*job, *dev);
  sim.kernel_ns.assign(E, -1);
  sim.wire.assign(job->call_off[job->n_comms], -1);
  int64_t er, es;
  int st = oracle_annotate(job, dev, roof, sim.kernel_ns.data(), sim.wire.data(), &er, &es);
  if (st != MAYA_ST_OK) {
    out->status = st;
    if (msg && msglen) {
      if (er >= 0) snprintf(msg, msglen, "rank-rep %lld seq %lld: %s", (long long)er,
                            (long long)es, g_err.c_str());
      else snprintf(msg, msglen, "%s", g_err.c_str());
    }
    return 0;
  }
  try {
    sim.run();
    std::string res = sim.residue();
    if (!res.empty()) {
      out->status = MAYA_ST_DEADLOCK;
      if (msg && msglen) snprintf(msg, msglen, "%s", res.c_str());
    }
  } catch (const Fail &f) {
    out->status = f.status;
    if (msg && msglen) snprintf(msg, msglen, "%s", f.msg.c_str());
    return 0;
  }
  out->total_ns = sim.max_t;
  int64_t pk = 0;
  for (int r = 0; r < sim.R; r++) pk = std::max(pk, sim.peak[r]);
  out->peak_mem_bytes = pk;
  out->oom = sim.first_oom_rank >= 0;
  out->first_oom_rank = sim.first_oom_rank;
  out->first_oom_seq = (int32_t)sim.first_oom_seq;
  out->dispatched_ops = sim.dispatched;
  out->completed_ops = sim.completed;
  int64_t nt = 0;
  for (int r = 0; r < sim.R; r++) {
    auto &ivs = sim.intervals[r];
    if (rank_stats) {
      std::vector<std::pair<int64_t, int64_t>> comp, comm, all;
      for (auto &iv : ivs) {
        (iv.cls ? comm : comp).emplace_back(iv.a, iv.b);
        all.emplace_back(iv.a, iv.b);
      }
      auto comm_m = merge(comm);
      int64_t comm_len = 0;
      for (auto &p : comm_m) comm_len += p.second - p.first;
      int64_t *rs = rank_stats + 5 * r;
      rs[0] = union_len(comp);
      rs[1] = comm_len;
      rs[2] = subtract_len(comm_m, merge(comp));
      rs[3] = sim.max_t - union_len(all);
      rs[4] = sim.peak[r];
    }
    if (tl_start) {
      for (auto &iv : ivs) {
        tl_rank[nt] = r; tl_stream[nt] = iv.stream; tl_seq[nt] = iv.seq;
        tl_start[nt] = iv.a; tl_end[nt] = iv.b; if (tl_class) tl_class[nt] = iv.cls;
        nt++;
      }
    } else {
      nt += (int64_t)ivs.size();
    }
  }
  if (n_timeline) *n_timeline = nt;
  return 0;
}

// Multi-threaded batch (the CPU baseline): n jobs, results only.
int oracle_simulate_many(int32_t n, const maya_raw_job *jobs, const maya_device_params *devs,
                         const maya_roofline_params *roof, maya_job_result *out,
                         int32_t n_threads) {
  std::atomic<int> next(0);
  auto work = [&]() {
    for (;;) {
      int i = next.fetch_add(1);
      if (i >= n) break;
      oracle_simulate(&jobs[i], &devs[jobs[i].device], roof, &out[i], nullptr, nullptr, nullptr,
                      nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0);
    }
  };
  if (n_threads <= 1) { work(); return 0; }
  std::vector<std::thread> th;
  for (int t = 0; t < n_threads; t++) th.emplace_back(work);
  for (auto &t : th) t.join();
  return 0;
}

}  // extern "C"
