// Native trace generation (row f1 of SURVEY §8f): the synthetic Megatron-style
// frontend of pkg/src/dltsim/workload.py plus the group resolution of
// collate.py, producing a raw job (include/maya_b200.h) directly.
#pragma once
#include <array>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/maya_b200.h"

namespace maya {

// Fixed string tables of generated jobs (ids used in ev_f).
extern const char *const GEN_OP_KINDS[12];
extern const char *const GEN_DTYPES[3];

struct GenJob {
  int32_t num_ranks = 0, num_hosts = 0, devices_per_host = 0;
  int64_t capacity = 0;
  std::vector<int64_t> rep_ranks;
  std::vector<int32_t> rank_rep;
  std::vector<int64_t> ev_off;
  std::vector<uint8_t> ev_kind;
  std::vector<int32_t> ev_stream;
  std::vector<int64_t> ev_f;
  std::vector<std::string> comm_names;
  std::vector<int32_t> comm_nranks;
  std::vector<int8_t> comm_topo;
  std::vector<int64_t> call_off;
  std::vector<int8_t> call_kind;
  std::vector<int64_t> call_bytes;
  std::vector<int64_t> rank_comm_off;
  std::vector<int32_t> rank_comm;
  std::string comm_blob;  // comm names joined by '\n'
  // Lazy call tables (fused path with a GenCache): every communicator's call
  // table is the call list of its position-0 member's representative at that
  // member's local communicator index (collate.py:323-340), so the per-comm
  // tables (thousands of communicators at 2,048 ranks) are not materialised:
  // call_off / call_kind / call_bytes stay empty and readers go through
  // rep_calls[comm_first_stage[g]][comm_first_lc[g]] (materialize_calls()
  // builds the arrays when a reader needs them).
  bool lazy_calls = false;
  std::vector<std::vector<std::vector<std::pair<int8_t, int64_t>>>> rep_calls;
  std::vector<int32_t> comm_first_stage, comm_first_lc;
  int64_t n_calls_total = 0;
  const std::vector<std::pair<int8_t, int64_t>> &comm_calls(size_t g) const {
    return rep_calls[comm_first_stage[g]][comm_first_lc[g]];
  }
  void materialize_calls() {
    if (!lazy_calls || !call_off.empty()) return;
    call_off.push_back(0);
    for (size_t g = 0; g < comm_first_stage.size(); g++) {
      for (const auto &kb : comm_calls(g)) {
        call_kind.push_back(kb.first);
        call_bytes.push_back(kb.second);
      }
      call_off.push_back((int64_t)call_kind.size());
    }
  }

  maya_raw_job raw(int32_t device) const;
  void clear() {
    num_ranks = num_hosts = devices_per_host = 0;
    capacity = 0;
    rep_ranks.clear(); rank_rep.clear(); ev_off.clear(); ev_kind.clear(); ev_stream.clear();
    ev_f.clear(); comm_names.clear(); comm_nranks.clear(); comm_topo.clear(); call_off.clear();
    call_kind.clear(); call_bytes.clear(); rank_comm_off.clear(); rank_comm.clear();
    // rep_calls keeps its lists (read only while lazy_calls): the next config's
    // generator reuses their capacity (gen.cpp generate_job)
    lazy_calls = false; comm_first_stage.clear(); comm_first_lc.clear();
    n_calls_total = 0;
    comm_blob.clear();
  }
};

// One kernel launch of the generator's inventory (workload.py:316-378).
struct KSpec {          // no padding: launch lists compare with memcmp (pack.cpp)
  int64_t op;
  int64_t flops, bytes;
};

// Receives the events of each representative trace in order instead of the
// raw arrays (the fused generate -> pack path, pack.cpp pack_generated).
struct EventSink {
  virtual ~EventSink() {}
  virtual void rep_begin(size_t est_events) = 0;
  virtual void ev(uint8_t k, int32_t s, int64_t a, int64_t b, int64_t c, int64_t d) = 0;
  virtual void rep_end() = 0;
  // A sink that takes kernel blocks receives each maximal run of kernel
  // launches on one stream (with nothing else in between) as ONE call: the
  // events [HostGap(gap) if gap > 0, KernelLaunch(ks[i], dtype)] for i < n.
  virtual bool takes_blocks() const { return false; }
  // Returns the block's id (interned per job), or ~0u if the run went through
  // the per-event path.
  virtual uint32_t kernel_block(int32_t, const KSpec *, size_t, int64_t, int32_t) { return ~0u; }
  // The same run again (its launch list interned as `id` by an earlier
  // kernel_block of this trace): emit it by id.  False: not possible here (the
  // caller then sends the launch list).
  virtual bool kernel_block_id(int32_t, uint32_t, size_t, int64_t) { return false; }
  // Phase templates (kernel-block sinks): the generator brackets each
  // microbatch phase with phase_begin / phase_end (which returns a template id,
  // or -1 if the phase cannot be replayed) and later asks phase_replay(id) to
  // stamp an identical phase (false: emit it event by event).  aid_base: the
  // first allocation handle the phase uses.
  virtual bool replays() const { return false; }
  virtual void phase_begin(int64_t) {}
  virtual int phase_end() { return -1; }
  virtual bool phase_replay(int, int64_t) { return false; }
};

// Per-batch cache of structure that depends only on the parallel layout
// (tp, dp, pp, virtual stages, devices per host), not on the trace: the
// communicator tables of generate_job and the packer's rank-class collapse.
// Shared by the batch's worker threads; one per maya_batch_add_generated call.
struct GenCache {
  std::mutex mu;
  std::map<std::array<int64_t, 6>, std::shared_ptr<const void>> entries;
  template <class T, class F>
  std::shared_ptr<const T> get(const std::array<int64_t, 6> &key, F build) {
    {
      std::lock_guard<std::mutex> g(mu);
      auto it = entries.find(key);
      if (it != entries.end()) return std::static_pointer_cast<const T>(it->second);
    }
    std::shared_ptr<const T> v = build();   // outside the lock (threads may race: same value)
    std::lock_guard<std::mutex> g(mu);
    auto ins = entries.emplace(key, v);
    return std::static_pointer_cast<const T>(ins.first->second);
  }
};

// Returns 0 or a negative code with *err set (invalid configuration).  With a
// sink, the events go to the sink and out's event arrays stay empty (its job
// tables -- reps, communicators, calls, rank translation -- are filled).
int generate_job(const maya_model &model, const maya_config &cfg, const maya_cluster &cl,
                 int32_t schedule, int64_t dispatch_overhead_ns, GenJob &out, std::string *err,
                 EventSink *sink = nullptr, GenCache *cache = nullptr);

}  // namespace maya
