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

#include <algorithm>
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

// Per-stream op lists of one rep.  Reused across reps by a thread's packer:
// reset() keeps every list's capacity (no regrowth per rep).
struct RepBuild {
  std::vector<int32_t> raw_of;                 // local stream -> raw handle
  std::vector<std::vector<Op>> sops;           // per local stream (first n_live used)
  std::vector<std::vector<uint32_t>> sseq;
  std::vector<uint32_t> sev;                   // per local stream: device events (blocks expanded)
  size_t n_live = 0;
  int last_raw = INT32_MIN, last_local = -1;
  size_t reserve_hint = 0;

  void reset(size_t hint) {
    raw_of.clear();
    sev.clear();
    for (size_t i = 0; i < n_live; i++) {
      sops[i].clear();
      sseq[i].clear();
    }
    n_live = 0;
    last_raw = INT32_MIN;
    last_local = -1;
    reserve_hint = hint;
  }
  size_t size() const { return n_live; }

  int local_stream(int32_t raw, bool create) {
    if (raw == last_raw) return last_local;
    for (size_t i = 0; i < raw_of.size(); i++)
      if (raw_of[i] == raw) { last_raw = raw; last_local = (int)i; return (int)i; }
    if (!create) return -1;
    raw_of.push_back(raw);
    sev.push_back(0);
    if (n_live == sops.size()) {
      sops.emplace_back();
      sseq.emplace_back();
    }
    n_live++;
    if (n_live == 1 && sops[0].capacity() < reserve_hint) {   // usually the compute stream
      sops[0].reserve(reserve_hint);
      sseq[0].reserve(reserve_hint);
    }
    last_raw = raw;
    last_local = (int)raw_of.size() - 1;
    return last_local;
  }
};

struct FeatCacheEnt {
  int64_t k[4];
  uint32_t fid;
};

// Job-level kernel-feature dedup (estimate.py:329-352 runs the estimator per
// event; we run it once per unique (op_kind, dtype, flops, bytes)).
struct FeatState {
  std::unordered_map<FeatKey, uint32_t, FeatHash> feat_map;
  std::unordered_map<int64_t, uint32_t> fixed_map;
  std::unordered_map<uint64_t, uint32_t> blk_map;    // launch-list hash -> kernel block id
  struct BlkKey {
    size_t spec0;
    uint32_t n;
    int32_t dtype;
    int64_t gap;
  };
  std::vector<BlkKey> blk_keys;                      // per block id: its launch list
  std::vector<KSpec> blk_specs;
  struct BlkCacheEnt {
    uint64_t h;
    uint32_t id;
  };
  BlkCacheEnt bcache[256];                           // direct-mapped, in front of blk_map
  FeatCacheEnt fcache[64];
  void clear() {
    feat_map.clear();
    fixed_map.clear();
    blk_map.clear();
    blk_keys.clear();
    blk_specs.clear();
    for (auto &e : bcache) e.id = UINT32_MAX;
    for (auto &ce : fcache) ce.fid = UINT32_MAX;
  }
};

// Ops of a FIFO after the device folds its affine runs (kernels.cu
// fold_write_kernel: the same rule): kernels, and collectives whose coll_wf
// entry names a wire feature, whose gap prefix is below 2^61, join the run of
// the op before them within one host-sync segment; runs are cut every
// FOLD_CHUNK ops.  coll_wf: the rep's per-collective entries (null: none).
uint32_t folded_len(const Op *v, uint32_t n, const uint32_t *coll_wf) {
  uint32_t folded = 0, ps = 0;
  bool pf = false;
  for (uint32_t i = 0; i < n; i++) {
    const uint32_t tg = op_tag(v[i].meta);
    const bool f = v[i].disp < ((int64_t)1 << 61) &&
                   (tg == TAG_KERN || (tg == TAG_COLL && coll_wf && coll_wf[v[i].arg] != NO_WF));
    const uint32_t sg = op_seg(v[i].meta);
    folded += (i % FOLD_CHUNK == 0 || !f || !pf || sg != ps) ? 1u : 0u;
    pf = f;
    ps = sg;
  }
  return folded;
}

// Per-event half of the packer for ONE representative trace, in trace order.
// pack_job drives it from raw event arrays (ordinals precomputed by a first
// pass, so a wait may precede its record); the fused generator drives it
// directly (ordinals assigned at the record: every generated wait follows its
// record, workload.py:510-568).
struct RepPacker {
  JobPack *P = nullptr;
  FeatState *F = nullptr;
  int32_t device = 0;
  RepHdr h{};
  RepBuild RB;
  bool fly = false;                                  // ordinals on the fly
  std::unordered_map<uint64_t, uint32_t> rec;        // (event, version) -> ordinal
  std::vector<std::vector<uint32_t>> rec_small;      // fly mode: [event][version]
  uint32_t n_recs = 0, n_local_comms = 0;
  std::vector<std::vector<uint32_t>> snap;
  std::unordered_map<int64_t, int64_t> alloc_big;
  std::vector<int64_t> alloc_small;
  std::unordered_map<uint64_t, uint32_t> coll_seen;
  std::vector<int32_t> comm_stream;
  std::vector<int64_t> comm_next;
  bool ring_ok = true;
  uint64_t coll0 = 0, mem0 = 0, sync0 = 0;
  int64_t gpre = 0;
  uint32_t seg = 0, seq = 0, n_devev = 0;
  bool keep_seq = true;   // event seq per op, for timelines (not kept with kernel blocks)

  static uint64_t ekey(int64_t ev, int64_t ver) {
    if (ev < 0 || ev > 0x7fffffff || ver < 0 || ver > 0x7fffffff)
      throw Fail{MAYA_ST_BAD_INPUT, "event id/version outside [0, 2^31)"};
    return ((uint64_t)ev << 32) | (uint64_t)ver;
  }

  // ---- phase templates (fused generator, kernel-block mode) ----------------
  // A microbatch phase of the synthetic frontend (forward or backward of one
  // model chunk, workload.py:571-756) emits the same events every time up to
  // counters: gap prefix, event seq, record ordinals, collective indices and
  // call numbers, allocation handles.  The first occurrence is packed event by
  // event and captured as a template of relative records; later occurrences
  // are stamped from it (no per-event work).  A phase that changes packer
  // state a template cannot carry (a new stream, a sync, a first use of a
  // communicator, an out-of-order collective, a wait on an earlier phase's
  // record) is never replayed.
  struct PhaseTpl {
    bool ok = false;
    uint32_t seg = 0;
    std::vector<std::vector<Op>> ops;        // per stream, relative fields
    size_t nst = 0;                          // streams the template covers
    std::vector<int32_t> raw;                // their trace stream handles (templates are
                                             // shared by the reps of a job, whose local
                                             // stream numbering may differ)
    std::vector<uint32_t> sev;               // per stream: device events added
    std::vector<uint32_t> coll_lc, coll_rel; // new collective entries (call_idx - comm_next)
    std::vector<std::pair<uint32_t, uint32_t>> lc_adv;   // (lc, calls issued)
    std::vector<MemRec> mems;                // gpre / seq relative
    std::vector<std::pair<int64_t, int64_t>> allocs;     // (handle - aid base, size)
    int64_t dgpre = 0;
    uint32_t dseq = 0, ddevev = 0, drecs = 0;
  };
  std::vector<PhaseTpl> tpls;   // the first ntpl are this job's (objects reused: no
  size_t ntpl = 0;              // allocation per job); job_begin() resets
  std::vector<int> rmap;        // replay: template stream -> local stream
  bool cap = false;
  int64_t cap_aid = 0;
  struct Snap {
    int64_t gpre;
    uint32_t seq, devev, recs, seg;
    size_t colls, mems, nst;
    bool ring_ok;
  } snap0{};
  std::vector<size_t> cap_size;
  std::vector<uint32_t> cap_sev;
  std::vector<int64_t> cap_next;
  std::vector<std::pair<int64_t, int64_t>> cap_allocs;

  void phase_begin(int64_t aid_base) {
    cap = true;
    cap_aid = aid_base;
    snap0 = Snap{gpre, seq, n_devev, n_recs, seg, P->coll_lc.size(), P->mems.size(), RB.size(),
                 ring_ok};
    cap_size.resize(RB.size());
    cap_sev.resize(RB.size());
    for (size_t q = 0; q < RB.size(); q++) {
      cap_size[q] = RB.sops[q].size();
      cap_sev[q] = RB.sev[q];
    }
    cap_next = comm_next;
    cap_allocs.clear();
  }
  int phase_end() {
    cap = false;
    if (ntpl == tpls.size()) tpls.emplace_back();
    PhaseTpl &t = tpls[ntpl];
    t.ok = false;
    for (auto &v : t.ops) v.clear();
    t.sev.clear();
    t.raw.clear();
    t.coll_lc.clear();
    t.coll_rel.clear();
    t.lc_adv.clear();
    t.mems.clear();
    t.allocs.clear();
    // A first occurrence may open streams and communicators (their local
    // indices and issuing streams are then fixed for every later occurrence,
    // which finds them open) and may clear ring_ok (sticky); it must not
    // cross a host sync or issue collectives out of order.
    t.ok = seg == snap0.seg && coll_seen.empty() && gpre >= snap0.gpre && !keep_seq;
    if (!t.ok) return -1;
    const uint32_t c0 = (uint32_t)(snap0.colls - coll0);
    t.seg = seg;
    if (t.ops.size() < RB.size()) t.ops.resize(RB.size());
    t.nst = RB.size();
    t.sev.resize(RB.size());
    t.raw.assign(RB.raw_of.begin(), RB.raw_of.begin() + RB.size());
    for (size_t q = 0; q < RB.size(); q++) {
      const size_t k0 = q < snap0.nst ? cap_size[q] : 0;
      t.sev[q] = RB.sev[q] - (q < snap0.nst ? cap_sev[q] : 0u);
      for (size_t k = k0; k < RB.sops[q].size(); k++) {
        Op o = RB.sops[q][k];
        o.disp -= snap0.gpre;
        const uint32_t tg = op_tag(o.meta);
        if (tg == TAG_REC || tg == TAG_WAIT) {
          if (o.arg == NO_REC || o.arg < snap0.recs) return -1;   // an earlier phase's record
          o.arg -= snap0.recs;
        } else if (tg == TAG_COLL) {
          o.arg -= c0;
        }
        t.ops[q].push_back(o);
      }
    }
    for (size_t k = snap0.colls; k < P->coll_lc.size(); k++) {
      const uint32_t lc = P->coll_lc[k];
      t.coll_lc.push_back(lc);
      t.coll_rel.push_back((uint32_t)(P->coll_idx[k] - (lc < cap_next.size() ? cap_next[lc] : 0)));
    }
    for (uint32_t lc = 0; lc < comm_next.size(); lc++) {
      const int64_t before = lc < cap_next.size() ? cap_next[lc] : 0;
      if (comm_next[lc] != before) t.lc_adv.push_back({lc, (uint32_t)(comm_next[lc] - before)});
    }
    for (size_t k = snap0.mems; k < P->mems.size(); k++) {
      MemRec m = P->mems[k];
      m.gpre -= snap0.gpre;
      m.seq -= snap0.seq;
      t.mems.push_back(m);
    }
    t.allocs = cap_allocs;
    t.dgpre = gpre - snap0.gpre;
    t.dseq = seq - snap0.seq;
    t.ddevev = n_devev - snap0.devev;
    t.drecs = n_recs - snap0.recs;
    return (int)ntpl++;
  }
  // stamp template `id` at the current state; false: not here (the caller
  // emits the phase event by event)
  bool phase_replay(int id, int64_t aid_base) {
    const PhaseTpl &t = tpls[id];
    if (seg != t.seg) return false;
    // the run-folding limit and block fits (kernel_block) assume gap prefixes
    // well below 2^61: replay only far from it
    if (gpre > ((int64_t)1 << 59) - t.dgpre) return false;
    // the streams and communicators the template touches must be open here
    rmap.resize(t.nst);
    for (size_t q = 0; q < t.nst; q++) {
      rmap[q] = -1;
      if (t.ops[q].empty() && t.sev[q] == 0) continue;
      rmap[q] = RB.local_stream(t.raw[q], false);
      if (rmap[q] < 0) return false;
    }
    for (const auto &a : t.lc_adv)
      if (a.first >= comm_next.size()) return false;
    const uint32_t cb = (uint32_t)(P->coll_lc.size() - coll0);
    // per tag: what the op's arg is relative to (KERN: nothing, COLL: the
    // rep's collective count, REC/WAIT: the record count)
    const uint32_t addv[4] = {0u, cb, n_recs, n_recs};
    for (size_t q = 0; q < t.nst; q++) {
      if (rmap[q] < 0) continue;
      std::vector<Op> &dst = RB.sops[rmap[q]];
      const size_t n0 = dst.size(), n = t.ops[q].size();
      dst.resize(n0 + n);
      Op *d = dst.data() + n0;
      const Op *src = t.ops[q].data();
      for (size_t k = 0; k < n; k++) {
        Op o = src[k];
        o.disp += gpre;
        o.arg += addv[o.meta & 3u];
        d[k] = o;
      }
      RB.sev[rmap[q]] += t.sev[q];
    }
    {
      const size_t c0 = P->coll_lc.size(), n = t.coll_lc.size();
      P->coll_lc.resize(c0 + n);
      P->coll_idx.resize(c0 + n);
      uint32_t *lc = P->coll_lc.data() + c0, *ix = P->coll_idx.data() + c0;
      for (size_t k = 0; k < n; k++) {
        lc[k] = t.coll_lc[k];
        ix[k] = (uint32_t)(t.coll_rel[k] + comm_next[t.coll_lc[k]]);
      }
    }
    for (const auto &a : t.lc_adv) comm_next[a.first] += a.second;
    {
      const size_t m0 = P->mems.size(), n = t.mems.size();
      P->mems.resize(m0 + n);
      MemRec *d = P->mems.data() + m0;
      for (size_t k = 0; k < n; k++) {
        MemRec m = t.mems[k];
        m.gpre += gpre;
        m.seq += seq;
        d[k] = m;
      }
    }
    for (const auto &a : t.allocs) {
      const int64_t h = aid_base + a.first;
      if (h >= 0 && h < (1 << 20)) {
        if ((size_t)h >= alloc_small.size()) alloc_small.resize(h + 64, INT64_MIN);
        alloc_small[h] = a.second;
      } else {
        alloc_big[h] = a.second;
      }
    }
    gpre += t.dgpre;
    seq += t.dseq;
    n_devev += t.ddevev;
    n_recs += t.drecs;
    return true;
  }

  void job_begin() { ntpl = 0; }
  void begin(JobPack &pk, FeatState &fs, int32_t dev, bool on_the_fly, size_t reserve_hint) {
    cap = false;
    keep_seq = true;
    P = &pk;
    F = &fs;
    device = dev;
    h = RepHdr{};
    h.job = 0;
    RB.reset(reserve_hint);
    fly = on_the_fly;
    rec.clear();
    for (auto &v : rec_small) v.clear();   // keep the per-event capacity
    n_recs = 0;
    n_local_comms = 0;
    snap.clear();
    alloc_big.clear();
    alloc_small.clear();
    coll_seen.clear();
    comm_stream.clear();
    comm_next.clear();
    ring_ok = true;
    coll0 = P->coll_lc.size();
    mem0 = P->mems.size();
    sync0 = P->syncs.size();
    gpre = 0;
    seg = 0;
    seq = 0;
    n_devev = 0;
  }

  // raw mode: the first pass over the rep's events
  void add_record(int64_t ev, int64_t ver) {
    auto ins = rec.emplace(ekey(ev, ver), n_recs);
    if (!ins.second)
      throw Fail{MAYA_ST_BAD_INPUT, "event (" + std::to_string(ev) + ", v" +
                                        std::to_string(ver) + ") recorded twice"};
    n_recs++;
  }
  void set_local_comms(uint32_t n) {
    n_local_comms = n;
    comm_stream.assign(n, INT32_MIN);
    comm_next.assign(n, 0);
  }

  uint32_t ord(const int64_t *f) {
    if (fly && f[0] >= 0 && f[0] < 4096 && f[1] >= 0 && f[1] < (1 << 20)) {
      if ((size_t)f[0] < rec_small.size() && (size_t)f[1] < rec_small[f[0]].size())
        return rec_small[f[0]][f[1]];
      return NO_REC;
    }
    auto it = rec.find(ekey(f[0], f[1]));
    return it == rec.end() ? NO_REC : it->second;
  }
  uint32_t record_fly(const int64_t *f) {
    if (f[0] >= 0 && f[0] < 4096 && f[1] >= 0 && f[1] < (1 << 20)) {
      if ((size_t)f[0] >= rec_small.size()) rec_small.resize(f[0] + 1);
      auto &v = rec_small[f[0]];
      if ((size_t)f[1] >= v.size()) v.resize(f[1] + 1, NO_REC);
      if (v[f[1]] != NO_REC)
        throw Fail{MAYA_ST_BAD_INPUT, "event (" + std::to_string(f[0]) + ", v" +
                                          std::to_string(f[1]) + ") recorded twice"};
      v[f[1]] = n_recs;
      return n_recs++;
    }
    add_record(f[0], f[1]);
    return n_recs - 1;
  }

  void emit(int32_t stream, uint32_t tag, uint32_t arg) {
    int ls = RB.local_stream(stream, true);
    if (seg >= (1u << 29)) throw Fail{MAYA_ST_BAD_INPUT, "too many host syncs"};
    RB.sops[ls].push_back(Op{gpre, arg, tag | (seg << 2)});
    if (keep_seq) RB.sseq[ls].push_back(seq);
    RB.sev[ls]++;
    n_devev++;
  }
  void sync(uint32_t type, uint32_t arg) {
    std::vector<uint32_t> c(RB.size());
    for (size_t s = 0; s < c.size(); s++) c[s] = (uint32_t)RB.sops[s].size();
    snap.push_back(std::move(c));
    P->syncs.push_back(SyncRec{gpre, type, arg, 0, 0});
    seg++;
  }

  // job-local id of roofline feature (op kind, dtype, flops, bytes)
  uint32_t feature(const int64_t *f) {
    // direct-mapped cache in front of the hash map: kernel templates repeat
    const uint64_t hk = ((uint64_t)f[2] * 0x9e3779b97f4a7c15ull) ^ (uint64_t)f[3] ^
                        ((uint64_t)f[0] << 48) ^ ((uint64_t)f[1] << 56);
    FeatCacheEnt &ce = F->fcache[(hk >> 58) & 63];
    if (ce.fid != UINT32_MAX && ce.k[0] == f[0] && ce.k[1] == f[1] && ce.k[2] == f[2] &&
        ce.k[3] == f[3])
      return ce.fid;
    uint32_t fid;
    FeatKey key{f[0], f[1], f[2], f[3]};
    auto it = F->feat_map.find(key);
    if (it == F->feat_map.end()) {
      fid = (uint32_t)P->feats.size();
      F->feat_map.emplace(key, fid);
      if (f[0] < 0 || f[0] > 0xfff || f[1] < 0 || f[1] > 0xff || device < 0 || device > 0xff)
        throw Fail{MAYA_ST_BAD_INPUT, "op kind / dtype / device id outside the feature meta word"};
      P->feats.push_back(Feature{f[2], f[3]});
      P->feat_meta.push_back(fmeta((int32_t)f[0], (int32_t)f[1], device));
    } else {
      fid = it->second;
    }
    ce = FeatCacheEnt{{f[0], f[1], f[2], f[3]}, fid};
    return fid;
  }

  // A run of n kernel launches on one stream, each after a host gap of `gap`
  // (the events [HostGap(gap) if gap > 0, KernelLaunch] x n): ONE KBLOCK op
  // whose disp is the first kernel's, the block interned per job.  Single
  // kernels, and runs reaching the fold limit of the gap prefix (2^61), go
  // through the per-event path (kernels.cu op_foldable).
  bool block_fits(size_t n, int64_t gap) const {
    return gap >= 0 && n >= 2 && n < (1u << 24) &&
           (gap == 0 || (int64_t)n <= (((int64_t)1 << 61) - 1 - gpre) / gap);
  }
  // emit interned block `id` (n launches, host gap `gap` before each)
  void emit_block(int32_t stream, uint32_t id, size_t n, int64_t gap) {
    gpre += gap;                     // the first kernel's gap
    seq += gap > 0 ? 1 : 0;
    emit(stream, TAG_KERN, KBLOCK | id);
    gpre += (int64_t)(n - 1) * gap;
    seq += (uint32_t)((n - 1) * (gap > 0 ? 2 : 1) + 1);
    n_devev += (uint32_t)(n - 1);
    RB.sev[RB.local_stream(stream, false)] += (uint32_t)(n - 1);
  }
  bool kernel_block_id(int32_t stream, uint32_t id, size_t n, int64_t gap) {
    if (!block_fits(n, gap)) return false;
    emit_block(stream, id, n, gap);
    return true;
  }
  uint32_t kernel_block(int32_t stream, const KSpec *ks, size_t n, int64_t gap, int32_t dtype) {
    const bool fits = block_fits(n, gap);
    if (!fits) {
      for (size_t i = 0; i < n; i++) {
        if (gap > 0) {
          const int64_t g[4] = {gap, 0, 0, 0};
          event(MAYA_EV_HOSTGAP, 0, g, -1, false);
        }
        const int64_t f[4] = {ks[i].op, dtype, ks[i].flops, ks[i].bytes};
        event(MAYA_EV_KERNEL, stream, f, -1, false);
      }
      return ~0u;
    }
    // intern by the launch list itself: a repeated layer body costs a hash
    // and a compare, no per-kernel feature lookups
    uint64_t h0 = 1469598103934665603ull ^ (uint64_t)gap, h1 = (uint64_t)n << 8 | (uint32_t)dtype,
             h2 = 0x9e3779b97f4a7c15ull;
    for (size_t i = 0; i < n; i++) {   // three independent multiply chains
      h0 = (h0 ^ (uint64_t)ks[i].op) * 1099511628211ull;
      h1 = (h1 ^ (uint64_t)ks[i].flops) * 0xff51afd7ed558ccdull;
      h2 = (h2 ^ (uint64_t)ks[i].bytes) * 0xc4ceb9fe1a85ec53ull;
    }
    const uint64_t hsh = h0 ^ (h1 >> 1) ^ (h2 << 1) ^ (h1 * 31) ^ (h2 >> 7);
    uint32_t id = UINT32_MAX, cand = UINT32_MAX;
    FeatState::BlkCacheEnt &ce = F->bcache[(hsh ^ (hsh >> 29)) & 255];
    if (ce.id != UINT32_MAX && ce.h == hsh) {
      cand = ce.id;
    } else {
      auto it = F->blk_map.find(hsh);
      if (it != F->blk_map.end()) cand = it->second;
    }
    if (cand != UINT32_MAX) {
      const FeatState::BlkKey &bk = F->blk_keys[cand];
      if (bk.n == n && bk.gap == gap && bk.dtype == dtype &&
          memcmp(F->blk_specs.data() + bk.spec0, ks, n * sizeof(KSpec)) == 0) {
        id = cand;
        ce = FeatState::BlkCacheEnt{hsh, cand};
      }
    }
    if (id == UINT32_MAX) {
      id = (uint32_t)P->blocks.size();
      if (id >= KBLOCK) throw Fail{MAYA_ST_BAD_INPUT, "too many kernel blocks"};
      P->blocks.push_back(KBlock{(uint32_t)P->blk_fids.size(), (uint32_t)n, gap});
      F->blk_keys.push_back(FeatState::BlkKey{F->blk_specs.size(), (uint32_t)n, dtype, gap});
      for (size_t i = 0; i < n; i++) {
        const int64_t f[4] = {ks[i].op, dtype, ks[i].flops, ks[i].bytes};
        P->blk_fids.push_back(feature(f));
      }
      F->blk_specs.insert(F->blk_specs.end(), ks, ks + n);
      if (F->blk_map.emplace(hsh, id).second) ce = FeatState::BlkCacheEnt{hsh, id};
      // (a colliding hash keeps its first block interned; later ones stay unshared)
    }
    emit_block(stream, id, n, gap);
    return id;
  }

  // one event (trace.py:71-151 as rawtrace.py arrays); host_ns >= 0: a
  // host-computed duration for a kernel-class event (annotate() with another
  // EstimatorInterface)
  void event(int k, int32_t stream, const int64_t *f, int64_t host_ns, bool has_host) {
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
        if (has_host) {
          if (host_ns < 0)
            throw Fail{MAYA_ST_ESTIMATION, "seq " + std::to_string(seq) + ": negative duration " +
                                               std::to_string(host_ns)};
          auto it = F->fixed_map.find(host_ns);
          if (it == F->fixed_map.end()) {
            fid = (uint32_t)P->feats.size();
            F->fixed_map.emplace(host_ns, fid);
            P->feats.push_back(Feature{host_ns, 0});
            P->feat_meta.push_back(FMETA_FIXED | fmeta(0, 0, device));
          } else {
            fid = it->second;
          }
        } else {
          fid = feature(f);
        }
        emit(stream, TAG_KERN, fid);
        break;
      }
      case MAYA_EV_MEMALLOC:
        if (cap) cap_allocs.push_back({f[0] - cap_aid, f[1]});
        if (f[0] >= 0 && f[0] < (1 << 20)) {
          if ((size_t)f[0] >= alloc_small.size()) alloc_small.resize(f[0] + 64, INT64_MIN);
          alloc_small[f[0]] = f[1];
        } else {
          alloc_big[f[0]] = f[1];
        }
        P->mems.push_back(MemRec{f[1], gpre, seg, seq});
        break;
      case MAYA_EV_MEMFREE: {
        int64_t sz = INT64_MIN;
        if (f[0] >= 0 && (size_t)f[0] < alloc_small.size()) {
          sz = alloc_small[f[0]];
        } else {
          auto it = alloc_big.find(f[0]);
          if (it != alloc_big.end()) sz = it->second;
        }
        if (sz == INT64_MIN)
          throw Fail{MAYA_ST_INTERNAL, "MemFree of unallocated handle " + std::to_string(f[0])};
        P->mems.push_back(MemRec{-sz, gpre, seg, seq});
        break;
      }
      case MAYA_EV_RECORD: emit(stream, TAG_REC, fly ? record_fly(f) : ord(f)); break;
      case MAYA_EV_WAIT: emit(stream, TAG_WAIT, ord(f)); break;
      case MAYA_EV_ESYNC: sync(SYNC_ESYNC, ord(f)); break;
      case MAYA_EV_SSYNC: {
        int ls = RB.local_stream(stream, false);
        sync(SYNC_SSYNC, ls < 0 ? NO_REC : (uint32_t)ls);
        break;
      }
      case MAYA_EV_DSYNC: sync(SYNC_DSYNC, 0); break;
      case MAYA_EV_COMMINIT:
        if (fly && f[0] >= 0 && (uint64_t)f[0] >= n_local_comms && f[0] < (1 << 20)) {
          n_local_comms = (uint32_t)f[0] + 1;
          comm_stream.resize(n_local_comms, INT32_MIN);
          comm_next.resize(n_local_comms, 0);
        }
        break;
      case MAYA_EV_COLLECTIVE: {
        if (f[0] < 0 || (uint64_t)f[0] >= n_local_comms)
          throw Fail{MAYA_ST_BAD_INPUT, "collective on comm without CommInit"};
        if (f[1] < 0 || f[1] > 0x7fffffff) throw Fail{MAYA_ST_BAD_INPUT, "call_idx range"};
        // (comm, call_idx) issued twice by one rank?  Calls issued in order
        // 0, 1, 2, ... (the common case) cannot repeat; others go to the map.
        const bool in_order = comm_next[f[0]] == f[1] && !(comm_stream[f[0]] == INT32_MIN && f[1] != 0);
        if (!in_order || !coll_seen.empty()) {
          uint64_t ck = ((uint64_t)f[0] << 32) | (uint64_t)f[1];
          if (coll_seen.empty()) {   // first out-of-order call: enter the earlier in-order ones
            for (uint32_t c = 0; c < n_local_comms; c++)
              for (int64_t q = 0; q < comm_next[c] && comm_stream[c] != INT32_MIN; q++)
                coll_seen.emplace(((uint64_t)c << 32) | (uint64_t)q, 0);
          }
          if (!coll_seen.emplace(ck, 0).second)
            throw Fail{MAYA_ST_BAD_INPUT, "collective (comm, call_idx) issued twice by one rank"};
        }
        if (comm_stream[f[0]] == INT32_MIN) comm_stream[f[0]] = stream;
        if (comm_stream[f[0]] != stream || comm_next[f[0]] != f[1]) ring_ok = false;
        if (comm_next[f[0]] <= f[1]) comm_next[f[0]] = f[1] + 1;
        uint32_t ci = (uint32_t)(P->coll_lc.size() - coll0);
        P->coll_lc.push_back((uint32_t)f[0]);
        P->coll_idx.push_back((uint32_t)f[1]);
        emit(stream, TAG_COLL, ci);
        break;
      }
      default:
        throw Fail{MAYA_ST_BAD_INPUT, "unknown event kind " + std::to_string(k)};
    }
    seq++;
  }

  void finish() {
    h.n_events = seq;
    h.n_devev = n_devev;
    h.n_recs = n_recs;
    // collectives renumbered stream-major: the collectives of one FIFO are
    // consecutive in the per-rank collective tables, so a walker reads (and
    // prefetches) its entries sequentially
    {
      const uint32_t nc = (uint32_t)(P->coll_lc.size() - coll0);
      thread_local std::vector<uint32_t> lc, ix;   // scratch, capacity kept per worker
      lc.resize(nc);
      ix.resize(nc);
      uint32_t next = 0;
      for (size_t si = 0; si < RB.size(); si++)
        for (Op &o : RB.sops[si])
          if (op_tag(o.meta) == TAG_COLL) {
            lc[next] = P->coll_lc[coll0 + o.arg];
            ix[next] = P->coll_idx[coll0 + o.arg];
            o.arg = next++;
          }
      std::copy(lc.begin(), lc.end(), P->coll_lc.begin() + coll0);
      std::copy(ix.begin(), ix.end(), P->coll_idx.begin() + coll0);
    }
    // stream-major op layout
    h.ops = P->ops.size();
    h.streams = P->streams.size();
    h.n_streams = (uint32_t)RB.size();
    uint32_t pos = 0;
    for (size_t s = 0; s < RB.size(); s++) {
      // (folded: set by pack_tail once the foldable collectives are known)
      P->streams.push_back(StreamRange{pos, (uint32_t)RB.sops[s].size(), RB.raw_of[s], 0});
      P->stream_events.push_back(RB.sev[s]);
      P->ops.insert(P->ops.end(), RB.sops[s].begin(), RB.sops[s].end());
      if (keep_seq) P->op_seq.insert(P->op_seq.end(), RB.sseq[s].begin(), RB.sseq[s].end());
      pos += (uint32_t)RB.sops[s].size();
    }
    h.n_ops = pos;
    h.colls = coll0;
    h.n_colls = (uint32_t)(P->coll_lc.size() - coll0);
    h.syncs = sync0;
    h.n_syncs = (uint32_t)(P->syncs.size() - sync0);
    h.counts = P->counts.size();
    for (size_t k = 0; k < snap.size(); k++) {
      P->syncs[sync0 + k].cnt = (uint32_t)(P->counts.size() - h.counts);
      for (uint32_t s = 0; s < h.n_streams; s++)
        P->counts.push_back(s < snap[k].size() ? snap[k][s] : 0u);
    }
    h.mems = mem0;
    h.n_mems = (uint32_t)(P->mems.size() - mem0);
    h.gend = gpre;
    P->reps.push_back(h);
    P->rep_ring_ok.push_back(ring_ok ? 1 : 0);
  }
};

void pack_rep(const maya_raw_job &job, int rep, JobPack &P, FeatState &F, RepPacker &RP,
              uint32_t &n_local_comms) {
  const int64_t b = job.ev_off[rep], e = job.ev_off[rep + 1];
  RP.begin(P, F, job.device, false, (size_t)(e - b) / 2 + 16);
  // first pass: record ordinals (trace.py:453-459: each (event, version)
  // recorded once) and the number of local communicators
  uint32_t nlc = 0;
  for (int64_t i = b; i < e; i++) {
    const int k = job.ev_kind[i];
    if (k == MAYA_EV_RECORD) {
      const int64_t *f = job.ev_f + 4 * i;
      RP.add_record(f[0], f[1]);
    } else if (k == MAYA_EV_COMMINIT) {
      nlc = std::max<uint32_t>(nlc, (uint32_t)job.ev_f[4 * i] + 1);
    }
  }
  RP.set_local_comms(nlc);
  for (int64_t i = b; i < e; i++)
    RP.event(job.ev_kind[i], job.ev_stream[i], job.ev_f + 4 * i,
             job.kernel_ns ? job.kernel_ns[i] : -1, job.kernel_ns != nullptr);
  RP.finish();
  n_local_comms = nlc;
}

}  // namespace

// --- exact rank-class collapse -------------------------------
//
// Equitable refinement: colour = representative trace; refine by, for each
// CommInit of the rank's representative in order, (topology, multiset of member
// colours).  Ranks of one class see identical inputs at every step of the
// max-plus iteration, so their op times are identical (Kleene iteration from a
// class-constant start stays class-constant).  The reduced job simulates one
// rank per class; communicators reached from class members at the same local
// index are identified (union-find) and must resolve consistently, otherwise
// the job is simulated full-rank.  A collective of a reduced communicator
// waits for one arrival per member class; its wire time keeps the real nranks
// and topology.
struct SimView {
  std::vector<int32_t> rank_orig;              // sim rank -> original rank
  std::vector<int32_t> rank_sim;               // original rank -> sim rank
  std::vector<std::vector<int32_t>> rank_comm; // sim rank -> sim comm per local index
  std::vector<int32_t> comm_real;              // sim comm -> a real comm (calls, topo, nranks)
  std::vector<int32_t> comm_rdv;               // sim comm -> arrivals per call
};

namespace {

struct DSU {
  std::vector<int32_t> p;
  explicit DSU(int n) : p(n) { for (int i = 0; i < n; i++) p[i] = i; }
  int find(int x) { while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; } return x; }
  void unite(int a, int b) { a = find(a); b = find(b); if (a != b) p[std::max(a, b)] = std::min(a, b); }
};

uint64_t mix64(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  return h * 0xff51afd7ed558ccdull;
}

// lazy: the job's call tables live in the generator (GenJob lazy_calls); then
// *structural reports whether every identified pair of communicators takes its
// calls from the same (representative, local index) -- equal for every
// configuration of the layout, so the view is shareable (GenCache).
bool build_collapsed(const maya_raw_job &job, const std::vector<uint32_t> &rep_comms,
                     SimView &V, const GenJob *lazy = nullptr, bool *structural = nullptr) {
  if (structural) *structural = true;
  const int R = job.num_ranks, G = job.n_comms;
  if (R <= 1) return false;
  std::vector<std::vector<int32_t>> members(G);
  for (int r = 0; r < R; r++)
    for (int64_t q = job.rank_comm_off[r]; q < job.rank_comm_off[r + 1]; q++)
      members[job.rank_comm[q]].push_back(r);
  std::vector<int32_t> color(R);
  int ncol = 0;
  {
    std::unordered_map<int32_t, int32_t> m;
    for (int r = 0; r < R; r++) {
      auto it = m.emplace(job.rank_rep[r], (int32_t)m.size()).first;
      color[r] = it->second;
    }
    ncol = (int)m.size();
  }
  // per iteration: communicator signatures (topology, sorted member colours),
  // then each rank's signature (colour, comm signatures by local index) laid
  // out flat; equal signatures (hash, then exact) get one new colour
  std::vector<uint64_t> csig(G), sig, rh(R);
  std::vector<int64_t> soff(R + 1);
  std::vector<int32_t> buf, ncolor(R), first_of, next_of(R);
  std::unordered_map<uint64_t, int32_t> head;   // signature hash -> first rank
  for (int iter = 0; iter < 64; iter++) {
    for (int g = 0; g < G; g++) {
      buf.clear();
      for (int32_t m : members[g]) buf.push_back(color[m]);
      std::sort(buf.begin(), buf.end());
      uint64_t h = mix64(0x51ed, (uint64_t)job.comm_topo[g]);
      for (int32_t x : buf) h = mix64(h, (uint64_t)x);
      csig[g] = h;
    }
    sig.clear();
    for (int r = 0; r < R; r++) {
      soff[r] = (int64_t)sig.size();
      sig.push_back((uint64_t)color[r]);
      for (int64_t q = job.rank_comm_off[r]; q < job.rank_comm_off[r + 1]; q++)
        sig.push_back(csig[job.rank_comm[q]]);
      uint64_t h = 0x9e37;
      for (int64_t q = soff[r]; q < (int64_t)sig.size(); q++) h = mix64(h, sig[q]);
      rh[r] = h;
    }
    soff[R] = (int64_t)sig.size();
    auto same_sig = [&](int a, int b2) {
      const int64_t la = soff[a + 1] - soff[a], lb = soff[b2 + 1] - soff[b2];
      return la == lb && std::equal(sig.begin() + soff[a], sig.begin() + soff[a + 1],
                                    sig.begin() + soff[b2]);
    };
    head.clear();
    int n2 = 0;
    for (int r = 0; r < R; r++) {
      next_of[r] = -1;
      auto ins = head.emplace(rh[r], r);
      int found = -1;
      if (!ins.second) {   // walk the ranks already seen with this hash
        int o = ins.first->second, last = o;
        for (; o >= 0; last = o, o = next_of[o])
          if (same_sig(o, r)) { found = ncolor[o]; break; }
        if (found < 0) next_of[last] = r;
      }
      if (found < 0) found = n2++;
      ncolor[r] = found;
    }
    bool stable = n2 == ncol;
    color.swap(ncolor);
    ncol = n2;
    if (stable) break;
    if (iter == 63) return false;
  }
  if (ncol == R) return false;  // nothing to collapse
  // class representatives: lowest rank
  std::vector<int32_t> rho(ncol, -1);
  for (int r = 0; r < R; r++)
    if (rho[color[r]] < 0) rho[color[r]] = r;
  // identify communicators reached at the same local index by class members
  DSU dsu(G);
  for (int r = 0; r < R; r++) {
    const int p = rho[color[r]];
    const int64_t nr = job.rank_comm_off[r + 1] - job.rank_comm_off[r];
    if (nr != job.rank_comm_off[p + 1] - job.rank_comm_off[p]) return false;
    for (int64_t k = 0; k < nr; k++)
      dsu.unite(job.rank_comm[job.rank_comm_off[r] + k], job.rank_comm[job.rank_comm_off[p] + k]);
  }
  // every reduced comm: one local index per member class, equal call tables
  std::unordered_map<int32_t, int32_t> sim_of;   // dsu root -> sim comm
  V = SimView();
  V.rank_sim.assign(color.begin(), color.end());
  for (int c = 0; c < ncol; c++) {
    const int p = rho[c];
    V.rank_orig.push_back(p);
    std::vector<int32_t> lc;
    std::vector<int32_t> roots;
    for (int64_t q = job.rank_comm_off[p]; q < job.rank_comm_off[p + 1]; q++) {
      const int32_t g = job.rank_comm[q];
      const int32_t root = dsu.find(g);
      for (int32_t x : roots)
        if (x == root) return false;  // two local comms of one class fold together
      roots.push_back(root);
      auto it = sim_of.find(root);
      if (it == sim_of.end()) {
        it = sim_of.emplace(root, (int32_t)V.comm_real.size()).first;
        V.comm_real.push_back(g);
        V.comm_rdv.push_back(0);
      }
      lc.push_back(it->second);
    }
    V.rank_comm.push_back(std::move(lc));
  }
  // arrivals per call = number of member classes; check group consistency
  std::vector<std::vector<int32_t>> cls_of(V.comm_real.size());
  for (int g = 0; g < G; g++) {
    auto it = sim_of.find(dsu.find(g));
    if (it == sim_of.end()) continue;
    const int32_t sg = it->second, g0 = V.comm_real[sg];
    if (job.comm_topo[g] != job.comm_topo[g0] || job.comm_nranks[g] != job.comm_nranks[g0])
      return false;
    if (lazy) {
      if (lazy->comm_first_stage[g] != lazy->comm_first_stage[g0] ||
          lazy->comm_first_lc[g] != lazy->comm_first_lc[g0]) {
        if (structural) *structural = false;
        if (lazy->comm_calls(g) != lazy->comm_calls(g0)) return false;
      }
    } else {
      const int64_t n0 = job.call_off[g0 + 1] - job.call_off[g0];
      if (job.call_off[g + 1] - job.call_off[g] != n0) return false;
      for (int64_t i = 0; i < n0; i++) {
        const int64_t a = job.call_off[g] + i, b = job.call_off[g0] + i;
        if (job.call_kind[a] != job.call_kind[b] || job.call_bytes[a] != job.call_bytes[b])
          return false;
        if (job.wire_ns && job.wire_ns[a] != job.wire_ns[b]) return false;
      }
    }
    for (int32_t m : members[g]) cls_of[sg].push_back(color[m]);
  }
  for (size_t sg = 0; sg < cls_of.size(); sg++) {
    auto &v = cls_of[sg];
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    V.comm_rdv[sg] = (int32_t)v.size();
    // each member class's representative must reach this comm exactly once
    for (int32_t cl : v) {
      int hits = 0;
      for (int32_t x : V.rank_comm[cl]) hits += (x == (int32_t)sg);
      if (hits != 1) return false;
    }
  }
  (void)rep_comms;
  return true;
}

void full_view(const maya_raw_job &job, SimView &V) {
  V = SimView();
  for (int r = 0; r < job.num_ranks; r++) {
    V.rank_orig.push_back(r);
    V.rank_sim.push_back(r);
    std::vector<int32_t> lc;
    for (int64_t q = job.rank_comm_off[r]; q < job.rank_comm_off[r + 1]; q++)
      lc.push_back(job.rank_comm[q]);
    V.rank_comm.push_back(std::move(lc));
  }
  for (int g = 0; g < job.n_comms; g++) {
    V.comm_real.push_back(g);
    V.comm_rdv.push_back(job.comm_nranks[g]);
  }
}

}  // namespace

namespace {

// Job-level half of the packer: validation, rank classes, communicators, call
// slots, simulated ranks, per-rank collective tables, walkers.  Reads only the
// job tables of `job` (not its events); the reps are already in P.
// Kernel features renumbered in stream-major first use: consecutive kernel ops
// of a FIFO then read consecutive duration entries on the device (the fold
// pass gathers one per op), which matters when features are mostly unique.
void renumber_features(JobPack &P) {
  const uint32_t nf = (uint32_t)P.feats.size();
  if (nf < 2 || !P.blocks.empty()) return;   // block jobs: few per-op gathers remain
  std::vector<uint32_t> nid(nf, UINT32_MAX);
  uint32_t next = 0;
  for (Op &o : P.ops) {
    if (op_tag(o.meta) != TAG_KERN) continue;
    uint32_t &m = nid[o.arg];
    if (m == UINT32_MAX) m = next++;
    o.arg = m;
  }
  for (uint32_t f = 0; f < nf; f++)
    if (nid[f] == UINT32_MAX) nid[f] = next++;   // unused (cannot happen; keep total)
  std::vector<Feature> nf2(nf);
  std::vector<uint32_t> nm2(nf);
  for (uint32_t f = 0; f < nf; f++) {
    nf2[nid[f]] = P.feats[f];
    nm2[nid[f]] = P.feat_meta[f];
  }
  P.feats.swap(nf2);
  P.feat_meta.swap(nm2);
}

// A collapse (or full) view with its outcome, shareable across the jobs of a
// batch with the same parallel layout (GenCache).
struct CachedView {
  SimView V;
  bool collapsed = false;
  bool shareable = true;   // false: each job of the layout computes its own view
};

void pack_tail(const maya_raw_job &job, JobPack &P, bool collapse,
               const std::vector<uint32_t> &rep_comms, const CachedView *shared = nullptr,
               const GenJob *lazy = nullptr) {
  JobHdr &H = P.hdr;
  renumber_features(P);
    // validate rank tables
  for (int r = 0; r < job.num_ranks; r++) {
    int rep = job.rank_rep[r];
    if (rep < 0 || rep >= job.n_reps) throw Fail{MAYA_ST_BAD_INPUT, "rank_rep out of range"};
    int64_t cb = job.rank_comm_off[r], ce = job.rank_comm_off[r + 1];
    if ((uint64_t)(ce - cb) < rep_comms[rep])
      throw Fail{MAYA_ST_BAD_INPUT, "rank lacks comm translation"};
    for (int64_t q = cb; q < ce; q++)
      if (job.rank_comm[q] < 0 || job.rank_comm[q] >= job.n_comms)
        throw Fail{MAYA_ST_BAD_INPUT, "rank_comm out of range"};
  }
  const int64_t n_calls = lazy ? lazy->n_calls_total : job.call_off[job.n_comms];
  if (n_calls > 0x7fffffff) throw Fail{MAYA_ST_BAD_INPUT, "too many group calls"};
  // the ranks / communicators the scheduler simulates (collapsed or full)
  SimView Vown;
  const SimView *Vp = &Vown;
  if (shared) {
    Vp = &shared->V;
    P.collapsed = shared->collapsed;
  } else {
    P.collapsed = collapse && build_collapsed(job, rep_comms, Vown, lazy);
    if (!P.collapsed) full_view(job, Vown);
  }
  const SimView &V = *Vp;
  P.rank_orig = V.rank_orig;
  P.rank_sim = V.rank_sim;
  // communicators and their call slots (JobTrace.groups / .calls)
  for (size_t sg = 0; sg < V.comm_real.size(); sg++) {
    const int g = V.comm_real[sg];
    if (lazy) {   // the generator's call list of the comm (no wire_ns on this path)
      const auto &calls = lazy->comm_calls(g);
      CommRec cr{job.comm_nranks[g], job.comm_topo[g], (uint32_t)P.slots.size(),
                 (uint32_t)calls.size()};
      if (cr.topo < 0 || cr.topo > 2) throw Fail{MAYA_ST_BAD_INPUT, "topology class"};
      P.comms.push_back(cr);
      P.comm_rdv.push_back(V.comm_rdv[sg]);
      for (const auto &kb : calls) {
        if (kb.first > 4) throw Fail{MAYA_ST_BAD_INPUT, "collective kind"};
        P.slots.push_back(SlotRec{kb.second, -1, kb.first, cr.nranks, cr.topo, job.device});
      }
      continue;
    }
    CommRec cr{job.comm_nranks[g], job.comm_topo[g], (uint32_t)P.slots.size(),
               (uint32_t)(job.call_off[g + 1] - job.call_off[g])};
    if (cr.topo < 0 || cr.topo > 2) throw Fail{MAYA_ST_BAD_INPUT, "topology class"};
    P.comms.push_back(cr);
    P.comm_rdv.push_back(V.comm_rdv[sg]);
    for (int64_t s = job.call_off[g]; s < job.call_off[g + 1]; s++) {
      int64_t fixed = -1;
      if (job.wire_ns && job.call_kind[s] >= 0) {
        fixed = job.wire_ns[s];
        if (fixed < 0) throw Fail{MAYA_ST_BAD_INPUT, "negative host wire time"};
      }
      if (job.call_kind[s] > 4) throw Fail{MAYA_ST_BAD_INPUT, "collective kind"};
      P.slots.push_back(SlotRec{job.call_bytes[s], fixed, job.call_kind[s], cr.nranks, cr.topo,
                                job.device});
    }
  }
  // wire features: the unique call records of the job (collective_estimate
  // depends on kind, bytes, nranks, topology and device only), one wire time
  // each on the device; slots keep an index.  A job has a handful: the last
  // match, then a scan of the (short) list, then a hash map past 32 entries.
  {
    auto same = [](const SlotRec &a, const SlotRec &b) {
      return a.bytes == b.bytes && a.fixed == b.fixed && a.kind == b.kind &&
             a.nranks == b.nranks && a.topo == b.topo && a.device == b.device;
    };
    struct WH {
      size_t operator()(const SlotRec &k) const {
        return std::hash<int64_t>()(k.bytes * 0x9E3779B97F4A7C15ll ^ k.fixed ^
                                    ((int64_t)k.kind << 40) ^ ((int64_t)k.nranks << 20) ^
                                    ((int64_t)k.topo << 56) ^ ((int64_t)k.device << 60));
      }
    };
    struct WE {
      bool operator()(const SlotRec &a, const SlotRec &b) const {
        return a.bytes == b.bytes && a.fixed == b.fixed && a.kind == b.kind &&
               a.nranks == b.nranks && a.topo == b.topo && a.device == b.device;
      }
    };
    std::unordered_map<SlotRec, uint32_t, WH, WE> wmap;
    P.slot_wf.resize(P.slots.size());
    uint32_t last = UINT32_MAX;
    for (size_t q = 0; q < P.slots.size(); q++) {
      const SlotRec &r = P.slots[q];
      uint32_t id = UINT32_MAX;
      if (last != UINT32_MAX && same(P.wfeats[last], r)) {
        id = last;
      } else if (P.wfeats.size() <= 32) {
        for (uint32_t w = 0; w < P.wfeats.size(); w++)
          if (same(P.wfeats[w], r)) { id = w; break; }
        if (id == UINT32_MAX && P.wfeats.size() == 32)   // switching to the map
          for (uint32_t w = 0; w < 32; w++) wmap.emplace(P.wfeats[w], w);
      } else {
        auto it = wmap.find(r);
        if (it != wmap.end()) id = it->second;
      }
      if (id == UINT32_MAX) {
        id = (uint32_t)P.wfeats.size();
        P.wfeats.push_back(r);
        if (P.wfeats.size() > 32) wmap.emplace(r, id);
      }
      P.slot_wf[q] = last = id;
    }
  }
  // work accounting over ALL ranks (sim.py:183-184)
  int64_t rank_ops = 0, dev_ops = 0;
  for (int r = 0; r < job.num_ranks; r++) {
    const RepHdr &h = P.reps[job.rank_rep[r]];
    rank_ops += h.n_events;
    dev_ops += h.n_devev;
  }
  // simulated ranks
  uint64_t fire = 0, delay = 0, walk = 0, tl = 0;
  for (size_t sr = 0; sr < V.rank_orig.size(); sr++) {
    const int rep = job.rank_rep[V.rank_orig[sr]];
    const RepHdr &h = P.reps[rep];
    RankRec rr{(uint32_t)rep, (uint32_t)P.rank_comm.size(), (uint32_t)fire, (uint32_t)delay,
               (uint32_t)walk, (uint32_t)tl, 0, 0};
    for (int32_t g : V.rank_comm[sr]) P.rank_comm.push_back((uint32_t)g);
    for (uint32_t s = 0; s < h.n_streams; s++) P.walkers.push_back(Walker{(uint32_t)sr, s});
    P.ranks.push_back(rr);
    fire += h.n_recs;
    delay += h.n_syncs + 1;
    walk += h.n_streams;
    tl += h.n_ops;
    if (fire > 0xffffffffull || delay > 0xffffffffull || tl > 0xffffffffull)
      throw Fail{MAYA_ST_BAD_INPUT, "job too large for 32-bit per-job tables"};
  }
  // each collective of a rep must address a real call slot for every rank;
  // per-rank collective tables (arrivals | comm | call_idx)
  bool ring = P.comms.size() <= 0xffff;
  for (uint8_t ok : P.rep_ring_ok) ring = ring && ok;
  for (size_t sr = 0; sr < P.ranks.size(); sr++) {
    RankRec &rr = P.ranks[sr];
    const RepHdr &h = P.reps[rr.rep];
    rr.rslot = (uint32_t)P.rcolls.size();
    for (uint32_t c2 = 0; c2 < h.n_colls; c2++) {
      uint32_t g = P.rank_comm[rr.comm + P.coll_lc[h.colls + c2]];
      uint32_t idx = P.coll_idx[h.colls + c2];
      if (idx >= P.comms[g].n_calls || P.slots[P.comms[g].call_base + idx].kind < 0)
        throw Fail{MAYA_ST_BAD_INPUT, "collective call missing from the job's call table"};
      int64_t nr = P.comm_rdv[g];
      if (nr < 1 || nr > 0xffff || g > 0xffff)
        throw Fail{MAYA_ST_BAD_INPUT, "communicator too large for the engine"};
      if (ring && (uint64_t)(P.comms[g].n_calls / 2 + 1) * (uint64_t)nr > 0xffffffffull)
        ring = false;
      P.rcolls.push_back(((uint64_t)nr << 48) | ((uint64_t)g << 32) | idx);
    }
    if (P.rcolls.size() > 0xffffffffull) throw Fail{MAYA_ST_BAD_INPUT, "too many collectives"};
  }
  // Collectives every simulated rank of a rep meets alone (the communicator is
  // one member class: done = ready + wire, no rendezvous, sim.py:326-343 with
  // one arrival) and with the same wire feature are affine maps of the stream
  // clock, exactly like kernels: the fold pass composes them into kernel runs
  // (kernels.cu fold_*), so a tensor-parallel layer body of a collapsed job is
  // one op.  Folded FIFO lengths (ring sizing) follow the same rule.
  {
    P.coll_wf.assign(P.coll_lc.size(), NO_WF);
    std::vector<uint8_t> seen(P.reps.size(), 0);
    for (size_t sr = 0; sr < P.ranks.size(); sr++) {
      const RankRec &rr = P.ranks[sr];
      const RepHdr &h = P.reps[rr.rep];
      for (uint32_t c2 = 0; c2 < h.n_colls; c2++) {
        const RankColl ent = P.rcolls[rr.rslot + c2];
        const uint32_t g = (uint32_t)(ent >> 32) & 0xffffu, idx = (uint32_t)ent;
        const uint32_t wf = (ent >> 48) == 1 ? P.slot_wf[P.comms[g].call_base + idx] : NO_WF - 1;
        uint32_t &cw = P.coll_wf[h.colls + c2];
        if (!seen[rr.rep]) cw = wf;
        else if (cw != wf) cw = NO_WF - 1;
      }
      seen[rr.rep] = 1;
    }
    bool any = false;
    for (uint32_t &cw : P.coll_wf) {
      if (cw == NO_WF - 1) cw = NO_WF;
      any |= cw != NO_WF;
    }
    P.stream_macros.assign(P.streams.size(), 0);
    P.fold_base.clear();
    // one pass per FIFO: flag the foldable collectives (OP_FOLDC) and count the
    // ops it keeps after the device folds its runs (kernels.cu fold_write_kernel:
    // the same rule, folded_len), for sizing the schedulers' staging
    for (const RepHdr &h : P.reps)
      for (uint32_t s = 0; s < h.n_streams; s++) {
        StreamRange &st = P.streams[h.streams + s];
        Op *v = P.ops.data() + h.ops + st.begin;
        const uint32_t *cw = P.coll_wf.data() + h.colls;
        uint32_t folded = 0, ps = 0, macros = 0;
        bool pf = false;
        MacroFuse mf;
        for (uint32_t i = 0; i < st.len; i++) {
          const uint32_t tg = op_tag(v[i].meta);
          if (any && tg == TAG_COLL && cw[v[i].arg] != NO_WF) v[i].meta |= OP_FOLDC;
          const bool f = v[i].disp < ((int64_t)1 << 61) &&
                         (tg == TAG_KERN || (v[i].meta & OP_FOLDC));
          const uint32_t sg = op_seg(v[i].meta);
          if (i % FOLD_CHUNK == 0) P.fold_base.push_back(folded);   // the fold pass's chunk
          if (i % FOLD_CHUNK == 0 || !f || !pf || sg != ps) {   // a folded op starts here
            folded++;
            // its class for the chain kernel's macro fusion (kernel: a folded run)
            const uint32_t cls = f ? 0u : tg == TAG_KERN ? 0u : tg == TAG_COLL ? 1u
                                 : tg == TAG_REC ? 2u : 3u;
            macros += mf.push(cls, sg) ? 1u : 0u;
          }
          pf = f;
          ps = sg;
        }
        st.folded = folded;
        P.stream_macros[h.streams + s] = macros;
      }
  }
  // walkers rank-major: a scheduler warp owns whole ranks
  P.wids.resize(P.walkers.size());
  for (size_t w = 0; w < P.walkers.size(); w++) P.wids[w] = (uint32_t)w;
  H.flags = ring ? JOB_RING : 0;
  H.n_rcolls = (uint32_t)P.rcolls.size();
  H.n_fire = (uint32_t)fire;
  H.n_ranks = (uint32_t)P.ranks.size();
  H.n_comms = (uint32_t)P.comms.size();
  H.n_slots = (uint32_t)P.slots.size();
  H.n_walkers = (uint32_t)P.walkers.size();
  H.n_feats = (uint32_t)P.feats.size();
  H.rank_ops = rank_ops;
  H.dev_ops = dev_ops;
  P.n_fire = fire;
  P.n_delay = delay;
}

void pack_fail(const maya_raw_job &job, JobPack &P, const Fail &f) {
  JobHdr &H = P.hdr;
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

void pack_header(const maya_raw_job &job, int32_t key_rank, JobPack &P) {
  P.clear();
  JobHdr &H = P.hdr;
  H.key_rank = key_rank;
  H.capacity = job.capacity;
  H.device = (uint32_t)job.device;
  H.n_ranks = (uint32_t)job.num_ranks;
  H.status = MAYA_ST_OK;
}

// Generator events straight into the packer (no raw event arrays).
struct PackSink final : EventSink {
  JobPack *P;
  FeatState *F;
  RepPacker *RP;
  int32_t device;
  std::vector<uint32_t> *rep_comms;
  bool blocks = false;
  bool takes_blocks() const override { return blocks; }
  uint32_t kernel_block(int32_t s, const KSpec *ks, size_t n, int64_t gap, int32_t dtype) override {
    return RP->kernel_block(s, ks, n, gap, dtype);
  }
  bool kernel_block_id(int32_t s, uint32_t id, size_t n, int64_t gap) override {
    return RP->kernel_block_id(s, id, n, gap);
  }
  bool replays() const override { return blocks && replay; }
  void phase_begin(int64_t aid_base) override { RP->phase_begin(aid_base); }
  int phase_end() override { return RP->phase_end(); }
  bool phase_replay(int id, int64_t aid_base) override { return RP->phase_replay(id, aid_base); }
  bool replay = true;
  void rep_begin(size_t est_events) override {
    RP->begin(*P, *F, device, true, est_events / 2 + 16);
    RP->keep_seq = !blocks;   // block batches never record a timeline (engine.cu)
  }
  void ev(uint8_t k, int32_t s, int64_t a, int64_t b, int64_t c, int64_t d) override {
    const int64_t f[4] = {a, b, c, d};
    RP->event(k, s, f, -1, false);
  }
  void rep_end() override {
    RP->finish();
    P->reps.back().job = 0;
    rep_comms->push_back(RP->n_local_comms);
  }
};

}  // namespace

bool g_phase_replay = true;

void pack_job(const maya_raw_job &job, int32_t key_rank, JobPack &P, bool collapse) {
  pack_header(job, key_rank, P);
  try {
    if (job.num_ranks < 0 || job.n_reps < 0) throw Fail{MAYA_ST_BAD_INPUT, "negative sizes"};
    thread_local FeatState F;
    thread_local RepPacker RP;
    F.clear();
    std::vector<uint32_t> rep_comms(job.n_reps);
    for (int rep = 0; rep < job.n_reps; rep++) {
      pack_rep(job, rep, P, F, RP, rep_comms[rep]);
      P.reps.back().job = 0;
    }
    pack_tail(job, P, collapse, rep_comms);
  } catch (const Fail &f) {
    pack_fail(job, P, f);
  }
}

int pack_generated(const maya_model &model, const maya_config &cfg, const maya_cluster &cl,
                   int32_t schedule, int64_t overhead, int32_t device, int32_t key_rank,
                   bool collapse, GenJob &G, JobPack &P, std::string *err, bool blocks,
                   GenCache *cache) {
  thread_local FeatState F;
  thread_local RepPacker RP;
  F.clear();
  std::vector<uint32_t> rep_comms;
  P.clear();
  PackSink sink;
  sink.P = &P;
  sink.F = &F;
  sink.RP = &RP;
  sink.device = device;
  sink.rep_comms = &rep_comms;
  sink.blocks = blocks;
  sink.replay = g_phase_replay;
  RP.job_begin();   // phase templates are shared by the job's reps
  int rc;
  try {
    rc = generate_job(model, cfg, cl, schedule, overhead, G, err, &sink, cache);
  } catch (const Fail &f) {   // packer error inside the generator's event stream
    maya_raw_job raw = G.raw(device);
    pack_header(raw, key_rank, P);
    pack_fail(raw, P, f);
    if (err) *err = f.msg;
    return MAYA_OK;
  }
  if (rc != MAYA_OK) return rc;
  maya_raw_job raw = G.raw(device);
  // keep the packed reps: pack_header clears P, so set the header by hand
  JobHdr &H = P.hdr;
  H = JobHdr{};
  H.key_rank = key_rank;
  H.capacity = raw.capacity;
  H.device = (uint32_t)device;
  H.n_ranks = (uint32_t)raw.num_ranks;
  H.status = MAYA_ST_OK;
  try {
    std::shared_ptr<const CachedView> view;
    const GenJob *lazy = G.lazy_calls ? &G : nullptr;
    if (cache && lazy) {
      // The view depends on rank -> rep, the communicator tables, each rep's
      // local communicator count -- functions of the layout -- and on the
      // identified communicators having equal call tables, which holds for
      // every configuration of the layout when each identified pair takes its
      // calls from the same (representative, local index); otherwise each job
      // builds its own (shareable = false).
      const int64_t n = (int64_t)cl.num_hosts * cl.devices_per_host;
      const std::array<int64_t, 6> key{collapse ? 2 : 3, cfg.tp, n / ((int64_t)cfg.tp * cfg.pp),
                                       cfg.pp, cfg.virtual_stages, cl.devices_per_host};
      view = cache->get<CachedView>(key, [&] {
        auto cv = std::make_shared<CachedView>();
        bool structural = true;
        cv->collapsed = collapse && build_collapsed(raw, rep_comms, cv->V, lazy, &structural);
        if (!cv->collapsed) full_view(raw, cv->V);
        cv->shareable = structural;
        return cv;
      });
      if (!view->shareable) view.reset();
    }
    pack_tail(raw, P, collapse, rep_comms, view.get(), lazy);
  } catch (const Fail &f) {
    pack_fail(raw, P, f);
  }
  return MAYA_OK;
}

}  // namespace maya
