// Host-side ingestion: raw job (reference schema as arrays) -> device SoA.
#pragma once
#include <string>
#include <vector>

#include "../../include/maya_b200.h"
#include "gen.h"
#include "soa.h"

namespace maya {

// Everything one job contributes to a batch; all indices are job-local.
struct JobPack {
  JobHdr hdr{};
  std::vector<RepHdr> reps;
  std::vector<Op> ops;
  std::vector<uint32_t> op_seq;        // event seq of each op (timeline)
  std::vector<StreamRange> streams;
  std::vector<uint32_t> stream_events; // host only: device events per stream (blocks expanded)
  std::vector<uint32_t> stream_macros; // host only: chain-kernel macro ops per stream (soa.h)
  std::vector<uint32_t> fold_base;     // per stream, per 1,024-op chunk: folded ops before it
  std::vector<uint32_t> coll_lc, coll_idx;
  std::vector<uint32_t> coll_wf;       // per rep collective: job-local wire feature when every
                                       // simulated rank of the rep meets it alone (one member
                                       // class, no rendezvous) with that wire time, else ~0 --
                                       // the fold pass composes it like a kernel (soa.h)
  std::vector<SyncRec> syncs;
  std::vector<uint32_t> counts;
  std::vector<MemRec> mems;
  std::vector<Feature> feats;
  std::vector<uint32_t> feat_meta;     // fmeta() per feature (soa.h)
  std::vector<KBlock> blocks;          // interned kernel blocks (soa.h KBLOCK)
  std::vector<uint32_t> blk_fids;      // their feature ids, job-local
  std::vector<CommRec> comms;
  std::vector<SlotRec> slots;          // host only: one per (comm, call_idx) group call
  std::vector<SlotRec> wfeats;         // unique call records of the job (uploaded)
  std::vector<uint32_t> slot_wf;       // per slot: its wire feature
  std::vector<RankRec> ranks;
  std::vector<uint32_t> rank_comm;
  std::vector<Walker> walkers;         // rank-major (rank, local stream)
  std::vector<uint32_t> wids;          // rank-major (rank, stream) -> index into walkers
  std::vector<RankColl> rcolls;        // per rank, per rep collective
  std::vector<uint8_t> rep_ring_ok;    // per rep: every comm used from one stream, idx 0,1,..
  std::vector<int32_t> comm_rdv;        // arrivals per call of each simulated comm
  std::vector<int32_t> rank_orig;       // simulated rank -> original rank
  std::vector<int32_t> rank_sim;        // original rank -> simulated rank
  bool collapsed = false;               // ranks are classes
  uint64_t n_fire = 0, n_delay = 0;
  std::string message;                 // why status != OK

  void clear() {   // keeps capacity (see engine.cu PackPool)
    hdr = JobHdr{};
    reps.clear(); ops.clear(); op_seq.clear(); streams.clear(); stream_events.clear(); stream_macros.clear(); fold_base.clear(); coll_lc.clear();
    coll_idx.clear(); coll_wf.clear(); syncs.clear(); counts.clear(); mems.clear(); feats.clear(); feat_meta.clear(); comms.clear();
    blocks.clear(); blk_fids.clear();
    slots.clear(); wfeats.clear(); slot_wf.clear(); ranks.clear(); rank_comm.clear(); walkers.clear(); wids.clear();
    rcolls.clear(); rep_ring_ok.clear(); comm_rdv.clear(); rank_orig.clear(); rank_sim.clear();
    collapsed = false;
    n_fire = n_delay = 0;
    message.clear();
  }
};

// Pack one job.  Never throws; input problems become hdr.status + message.
void pack_job(const maya_raw_job &job, int32_t key_rank, JobPack &out, bool collapse);

// Generate one configuration (gen.cpp) and pack it in the same pass: the
// generator's events go straight into the per-rep packer, never through raw
// event arrays.  Same JobPack as generate_job + pack_job (tests/test_gen.py).
// Returns generate_job's code (invalid configuration: <0 with *err set).
// With blocks, runs of kernel launches become interned kernel blocks (one
// KBLOCK op each): the batch must then be run folded (no timeline).
// Phase templates in pack_generated's kernel-block mode (default on; tests
// compare against the event-by-event packing).
extern bool g_phase_replay;

int pack_generated(const maya_model &model, const maya_config &cfg, const maya_cluster &cl,
                   int32_t schedule, int64_t overhead, int32_t device, int32_t key_rank,
                   bool collapse, GenJob &scratch, JobPack &out, std::string *err,
                   bool blocks = false, GenCache *cache = nullptr);

}  // namespace maya
