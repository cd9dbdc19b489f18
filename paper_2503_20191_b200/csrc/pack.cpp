// Host-side ingestion of one collated job into the device SoA (soa.h).
//
// Restates, per representative trace, what the reference's _compile_rank
// (pkg/src/dltsim/sim.py:135-174) and _advance_host (sim.py:222-270) derive
// from the event list, but splits it by dependence on timing:
//   * host gaps  -> per-op dispatch offset `disp` (sim.py:229-234: a gap > 0
//                   delays every later dispatch by its duration; gaps <= 0 are
//                   skipped);
//   * MemAlloc/MemFree -> signed deltas (sim.py:152-156, 235-242);
//   * Event/Stream/DeviceSynchronize -> the sync program (sim.py:243-263);
//   * kernel-class, Collective, EventRecord, StreamWaitEvent -> stream-major
//     device ops (sim.py:264-269, 302-347).
// Kernel-class features are deduplicated per job so the estimator kernel runs
// once per unique (op_kind, dtype, flops, bytes) (estimate.py:329-352).
#include "pack.h"

#include <cstring>
#include <unordered_map>

namespace maya {

namespace {

struct FeatKey {
  int64_t a, b, c, d;
  bool operator==(const FeatKey &o) const { return a == o.a && b == o.b && c == o.c && d == o.d; }
};
struct FeatHash {
  size_t operator()(const FeatKey &k) const {
    uint64_t h = 1469598103934665603ull;
    for (int64_t v : {k.a, k.b, k.c, k.d}) {
      h ^= (uint64_t)v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
      h *= 1099511628211ull;
    }
    return (size_t)h;
  }
};

struct Fail {
  int32_t status;
  std::string msg;
};

inline bool add_overflows(int64_t a, int64_t b) { return b > 0 && a > INT64_MAX - b; }

struct RepBuild {
  std::vector<int32_t> raw_of;                 // local stream -> raw handle
  std::vector<std::vector<Op>> sops;           // per local stream
  std::vector<std::vector<uint32_t>> sseq;
  int last_raw = INT32_MIN, last_local = -1;

  int local_stream(int32_t raw, bool create) {
    if (raw == last_raw) return last_local;
    for (size_t i = 0; i < raw_of.size(); i++)
      if (raw_of[i] == raw) { last_raw = raw; last_local = (int)i; return (int)i; }
    if (!create) return -1;
    raw_of.push_back(raw);
    sops.emplace_back();
    sseq.emplace_back();
    last_raw = raw;
    last_local = (int)raw_of.size() - 1;
    return last_local;
  }
};

void pack_rep(const maya_raw_job &job, int rep, JobPack &P,
              std::unordered_map<FeatKey, uint32_t, FeatHash> &feat_map,
              std::unordered_map<int64_t, uint32_t> &fixed_map, uint32_t &n_local_comms) {
  const int64_t b = job.ev_off[rep], e = job.ev_off[rep + 1];
  RepHdr h{};
  h.n_events = (uint32_t)(e - b);
  h.job = 0;
  // record ordinals (trace.py:453-459: each (event, version) recorded once)
  std::unordered_map<uint64_t, uint32_t> rec;
  auto ekey = [](int64_t ev, int64_t ver) -> uint64_t {
    if (ev < 0 || ev > 0x7fffffff || ver < 0 || ver > 0x7fffffff)
      throw Fail{MAYA_ST_BAD_INPUT, "event id/version outside [0, 2^31)"};
    return ((uint64_t)ev << 32) | (uint64_t)ver;
  };
  n_local_comms = 0;
  for (int64_t i = b; i < e; i++) {
    const int k = job.ev_kind[i];
    if (k == MAYA_EV_RECORD) {
      const int64_t *f = job.ev_f + 4 * i;
      auto ins = rec.emplace(ekey(f[0], f[1]), (uint32_t)rec.size());
      if (!ins.second)
        throw Fail{MAYA_ST_BAD_INPUT, "event (" + std::to_string(f[0]) + ", v" +
                                          std::to_string(f[1]) + ") recorded twice"};
    } else if (k == MAYA_EV_COMMINIT) {
      n_local_comms = std::max<uint32_t>(n_local_comms, (uint32_t)job.ev_f[4 * i] + 1);
    }
  }
  h.n_recs = (uint32_t)rec.size();
  auto ord = [&](const int64_t *f) -> uint32_t {
    auto it = rec.find(ekey(f[0], f[1]));
    return it == rec.end() ? NO_REC : it->second;
  };

  RepBuild RB;
  std::vector<std::vector<uint32_t>> snap;  // per sync: ops dispatched per local stream
  std::unordered_map<int64_t, int64_t> alloc;
  std::unordered_map<uint64_t, uint32_t> coll_seen;
  const uint64_t coll0 = P.coll_lc.size();
  int64_t gpre = 0;
  uint32_t seg = 0;
  const uint64_t mem0 = P.mems.size(), sync0 = P.syncs.size();
  for (int64_t i = b; i < e; i++) {
    const int k = job.ev_kind[i];
    const int64_t *f = job.ev_f + 4 * i;
    const uint32_t seq = (uint32_t)(i - b);
    auto emit = [&](uint32_t tag, uint32_t arg) {
      int ls = RB.local_stream(job.ev_stream[i], true);
      if (seg >= (1u << 30)) throw Fail{MAYA_ST_BAD_INPUT, "too many host syncs"};
      RB.sops[ls].push_back(Op{gpre, arg, tag | (seg << 2)});
      RB.sseq[ls].push_back(seq);
    };
    auto sync = [&](uint32_t type, uint32_t arg) {
      std::vector<uint32_t> c(RB.sops.size());
      for (size_t s = 0; s < c.size(); s++) c[s] = (uint32_t)RB.sops[s].size();
      snap.push_back(std::move(c));
      P.syncs.push_back(SyncRec{gpre, type, arg, 0, 0});
      seg++;
    };
    switch (k) {
      case MAYA_EV_HOSTGAP:
        if (f[0] > 0) {
          if (add_overflows(gpre, f[0])) throw Fail{MAYA_ST_OVERFLOW, "host gaps overflow int64"};
          gpre += f[0];
        }
        break;
      case MAYA_EV_KERNEL:
      case MAYA_EV_MEMCPY:
      case MAYA_EV_MEMSET: {
        uint32_t fid;
        if (job.kernel_ns) {
          int64_t d = job.kernel_ns[i];
          if (d < 0)
            throw Fail{MAYA_ST_ESTIMATION, "rank " + std::to_string(rep) + " seq " +
                                               std::to_string(seq) + ": negative duration " +
                                               std::to_string(d)};
          auto it = fixed_map.find(d);
          if (it == fixed_map.end()) {
            fid = (uint32_t)P.feats.size();
            fixed_map.emplace(d, fid);
            P.feats.push_back(Feature{0, 0, d, -1, -1, (int16_t)job.device});
          } else {
            fid = it->second;
          }
        } else {
          FeatKey key{f[0], f[1], f[2], f[3]};
          auto it = feat_map.find(key);
          if (it == feat_map.end()) {
            fid = (uint32_t)P.feats.size();
            feat_map.emplace(key, fid);
            P.feats.push_back(Feature{f[2], f[3], -1, (int32_t)f[0], (int16_t)f[1],
                                      (int16_t)job.device});
          } else {
            fid = it->second;
          }
        }
        emit(TAG_KERN, fid);
        break;
      }
      case MAYA_EV_MEMALLOC:
        alloc[f[0]] = f[1];
        P.mems.push_back(MemRec{f[1], gpre, seg, seq});
        break;
      case MAYA_EV_MEMFREE: {
        auto it = alloc.find(f[0]);
        if (it == alloc.end())
          throw Fail{MAYA_ST_INTERNAL, "MemFree of unallocated handle " + std::to_string(f[0])};
        P.mems.push_back(MemRec{-it->second, gpre, seg, seq});
        break;
      }
      case MAYA_EV_RECORD: emit(TAG_REC, ord(f)); break;
      case MAYA_EV_WAIT: emit(TAG_WAIT, ord(f)); break;
      case MAYA_EV_ESYNC: sync(SYNC_ESYNC, ord(f)); break;
      case MAYA_EV_SSYNC: {
        int ls = RB.local_stream(job.ev_stream[i], false);
        sync(SYNC_SSYNC, ls < 0 ? NO_REC : (uint32_t)ls);
        break;
      }
      case MAYA_EV_DSYNC: sync(SYNC_DSYNC, 0); break;
      case MAYA_EV_COMMINIT: break;
      case MAYA_EV_COLLECTIVE: {
        if (f[0] < 0 || (uint64_t)f[0] >= n_local_comms)
          throw Fail{MAYA_ST_BAD_INPUT, "collective on comm without CommInit"};
        if (f[1] < 0 || f[1] > 0x7fffffff) throw Fail{MAYA_ST_BAD_INPUT, "call_idx range"};
        uint64_t ck = ((uint64_t)f[0] << 32) | (uint64_t)f[1];
        if (!coll_seen.emplace(ck, 0).second)
          throw Fail{MAYA_ST_BAD_INPUT, "collective (comm, call_idx) issued twice by one rank"};
        uint32_t ci = (uint32_t)(P.coll_lc.size() - coll0);
        P.coll_lc.push_back((uint32_t)f[0]);
        P.coll_idx.push_back((uint32_t)f[1]);
        emit(TAG_COLL, ci);
        break;
      }
      default:
        throw Fail{MAYA_ST_BAD_INPUT, "unknown event kind " + std::to_string(k)};
    }
  }
  // stream-major op layout
  h.ops = P.ops.size();
  h.streams = P.streams.size();
  h.n_streams = (uint32_t)RB.sops.size();
  uint32_t pos = 0;
  for (size_t s = 0; s < RB.sops.size(); s++) {
    P.streams.push_back(StreamRange{pos, (uint32_t)RB.sops[s].size(), RB.raw_of[s], 0});
    P.ops.insert(P.ops.end(), RB.sops[s].begin(), RB.sops[s].end());
    P.op_seq.insert(P.op_seq.end(), RB.sseq[s].begin(), RB.sseq[s].end());
    pos += (uint32_t)RB.sops[s].size();
  }
  h.n_ops = pos;
  h.colls = coll0;
  h.n_colls = (uint32_t)(P.coll_lc.size() - coll0);
  h.syncs = sync0;
  h.n_syncs = (uint32_t)(P.syncs.size() - sync0);
  h.counts = P.counts.size();
  for (size_t k = 0; k < snap.size(); k++) {
    P.syncs[sync0 + k].cnt = (uint32_t)(P.counts.size() - h.counts);
    for (uint32_t s = 0; s < h.n_streams; s++)
      P.counts.push_back(s < snap[k].size() ? snap[k][s] : 0u);
  }
  h.mems = mem0;
  h.n_mems = (uint32_t)(P.mems.size() - mem0);
  h.gend = gpre;
  P.reps.push_back(h);
}

}  // namespace

void pack_job(const maya_raw_job &job, int32_t key_rank, JobPack &P) {
  P = JobPack();
  JobHdr &H = P.hdr;
  H.key_rank = key_rank;
  H.capacity = job.capacity;
  H.device = (uint32_t)job.device;
  H.n_ranks = (uint32_t)job.num_ranks;
  H.status = MAYA_ST_OK;
  try {
    if (job.num_ranks < 0 || job.n_reps < 0) throw Fail{MAYA_ST_BAD_INPUT, "negative sizes"};
    std::unordered_map<FeatKey, uint32_t, FeatHash> feat_map;
    std::unordered_map<int64_t, uint32_t> fixed_map;
    std::vector<uint32_t> rep_comms(job.n_reps);
    for (int rep = 0; rep < job.n_reps; rep++) {
      pack_rep(job, rep, P, feat_map, fixed_map, rep_comms[rep]);
      P.reps.back().job = 0;
    }
    // communicators and their call slots (JobTrace.groups / .calls)
    const int64_t n_calls = job.call_off[job.n_comms];
    if (n_calls > 0x7fffffff) throw Fail{MAYA_ST_BAD_INPUT, "too many group calls"};
    for (int g = 0; g < job.n_comms; g++) {
      CommRec c{job.comm_nranks[g], job.comm_topo[g], (uint32_t)job.call_off[g],
                (uint32_t)(job.call_off[g + 1] - job.call_off[g])};
      if (c.topo < 0 || c.topo > 2) throw Fail{MAYA_ST_BAD_INPUT, "topology class"};
      P.comms.push_back(c);
      for (int64_t s = job.call_off[g]; s < job.call_off[g + 1]; s++) {
        int64_t fixed = -1;
        if (job.wire_ns && job.call_kind[s] >= 0) {
          fixed = job.wire_ns[s];
          if (fixed < 0) throw Fail{MAYA_ST_BAD_INPUT, "negative host wire time"};
        }
        if (job.call_kind[s] > 4) throw Fail{MAYA_ST_BAD_INPUT, "collective kind"};
        P.slots.push_back(SlotRec{job.call_bytes[s], fixed, job.call_kind[s], c.nranks, c.topo,
                                  job.device});
      }
    }
    // ranks
    uint64_t fire = 0, delay = 0, walk = 0, tl = 0;
    int64_t rank_ops = 0, dev_ops = 0;
    for (int r = 0; r < job.num_ranks; r++) {
      int rep = job.rank_rep[r];
      if (rep < 0 || rep >= job.n_reps) throw Fail{MAYA_ST_BAD_INPUT, "rank_rep out of range"};
      const RepHdr &h = P.reps[rep];
      int64_t cb = job.rank_comm_off[r], ce = job.rank_comm_off[r + 1];
      if ((uint64_t)(ce - cb) < rep_comms[rep])
        throw Fail{MAYA_ST_BAD_INPUT, "rank lacks comm translation"};
      RankRec rr{(uint32_t)rep, (uint32_t)P.rank_comm.size(), (uint32_t)fire, (uint32_t)delay,
                 (uint32_t)walk, (uint32_t)tl};
      for (int64_t q = cb; q < ce; q++) {
        int32_t g = job.rank_comm[q];
        if (g < 0 || g >= job.n_comms) throw Fail{MAYA_ST_BAD_INPUT, "rank_comm out of range"};
        P.rank_comm.push_back((uint32_t)g);
      }
      for (uint32_t s = 0; s < h.n_streams; s++) P.walkers.push_back(Walker{(uint32_t)r, s});
      P.ranks.push_back(rr);
      fire += h.n_recs;
      delay += h.n_syncs + 1;
      walk += h.n_streams;
      tl += h.n_ops;
      rank_ops += h.n_events;
      dev_ops += h.n_ops;
      if (fire > 0xffffffffull || delay > 0xffffffffull || tl > 0xffffffffull)
        throw Fail{MAYA_ST_BAD_INPUT, "job too large for 32-bit per-job tables"};
    }
    // each collective of a rep must address a real call slot for every rank
    for (int r = 0; r < job.num_ranks; r++) {
      const RepHdr &h = P.reps[job.rank_rep[r]];
      const RankRec &rr = P.ranks[r];
      for (uint32_t c = 0; c < h.n_colls; c++) {
        uint32_t g = P.rank_comm[rr.comm + P.coll_lc[h.colls + c]];
        if (P.coll_idx[h.colls + c] >= P.comms[g].n_calls ||
            P.slots[P.comms[g].call_base + P.coll_idx[h.colls + c]].kind < 0)
          throw Fail{MAYA_ST_BAD_INPUT, "collective call missing from the job's call table"};
      }
    }
    H.n_comms = (uint32_t)P.comms.size();
    H.n_slots = (uint32_t)P.slots.size();
    H.n_walkers = (uint32_t)P.walkers.size();
    H.n_feats = (uint32_t)P.feats.size();
    H.rank_ops = rank_ops;
    H.dev_ops = dev_ops;
    P.n_fire = fire;
    P.n_delay = delay;
  } catch (const Fail &f) {
    H.status = f.status;
    P.message = f.msg;
    int64_t rank_ops = 0;
    for (int r = 0; r < job.num_ranks && job.n_reps > 0; r++) {
      int rep = job.rank_rep[r];
      if (rep >= 0 && rep < job.n_reps) rank_ops += job.ev_off[rep + 1] - job.ev_off[rep];
    }
    // keep nothing else: the scheduler skips jobs whose status is preset
    JobPack empty;
    empty.hdr = H;
    empty.hdr.rank_ops = rank_ops;
    empty.hdr.n_ranks = 0;
    empty.message = P.message;
    P = std::move(empty);
  }
}

}  // namespace maya
