// Device kernels of the batched simulator (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/maya_b200.h"
#include "soa.h"

namespace maya {

// Device view of one uploaded batch (all pointers into the device arena).
struct DevBatch {
  const JobHdr *jobs;
  const RankRec *ranks;
  const uint32_t *rank_comm;
  const CommRec *comms;
  const SlotRec *slots;
  const Walker *walkers;
  const RepHdr *reps;
  const Op *ops;
  const StreamRange *streams;
  const uint32_t *coll_lc;
  const uint32_t *coll_idx;
  const SyncRec *syncs;
  const uint32_t *counts;
  const MemRec *mems;
  const Feature *feats;
  // scratch / outputs
  int64_t *feat_ns;
  int64_t *wire;
  int64_t *fire;
  int64_t *delay;
  WState *wstate;
  CollSlot *cslots;
  RepOut *repout;
  int64_t *tl_start;
  int64_t *tl_end;
  maya_job_result *results;
  const int32_t *order;       // CTA -> job (largest first)
  int32_t *err_flag;          // any estimator failure
  uint32_t n_jobs, n_reps, n_feats, n_slots;
};

struct DevTables {
  maya_device_params devs[8];
  int64_t eff_num[64];
  int64_t eff_den[64];
  int32_t n_devs, n_op_kinds;
  int64_t overhead_ns;
};

void launch_estimate(const DevBatch &b, const DevTables &t, cudaStream_t s);
void launch_memscan(const DevBatch &b, cudaStream_t s);
void launch_schedule(const DevBatch &b, int record, cudaStream_t s);
void launch_topk(const DevBatch &b, int k, maya_topk_entry *out, int32_t *n_out, void *scratch,
                 cudaStream_t s);
size_t topk_scratch_bytes(uint32_t n_jobs, int k);

}  // namespace maya
