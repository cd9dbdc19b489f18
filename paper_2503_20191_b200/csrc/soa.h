// Device-resident structure-of-arrays for a batch of collated jobs.
//
// Layout decisions (DESIGN.md §Data layout):
//  * Only DEVICE ops (kernel-class, collective, record, wait) reach the
//    scheduler.  Host gaps are folded into a per-op dispatch offset `disp`
//    (prefix sum of gaps, timing independent), memory ops go to a separate
//    per-rep delta list (peak memory is a prefix-max scan, independent of
//    timing), CommInit is dropped (sim.py:157-158), host syncs become a short
//    per-rep "sync program".
//  * Device ops are stored STREAM-MAJOR per representative trace: each local
//    stream's ops are contiguous, in FIFO (= host) order, so a stream walker
//    streams through 16-byte records.
//  * Every index inside a record is rep- or job-local; bases live in headers,
//    so per-job packing is embarrassingly parallel and batch assembly is a
//    memcpy.
#pragma once
#include <stdint.h>

#ifndef __CUDACC__
#ifndef __host__
#define __host__
#endif
#ifndef __device__
#define __device__
#endif
#endif

namespace maya {

enum OpTag : uint32_t { TAG_KERN = 0, TAG_COLL = 1, TAG_REC = 2, TAG_WAIT = 3 };
enum SyncType : uint32_t { SYNC_ESYNC = 0, SYNC_SSYNC = 1, SYNC_DSYNC = 2 };

static const uint32_t NO_REC = 0xFFFFFFFFu;
// jobs whose walker + rank states fit are scheduled out of shared memory
static const uint32_t SMEM_STATES = 2560;

// 16-byte device op record.
struct alignas(16) Op {
  int64_t disp;    // sum of host gaps before this op in host order (ns)
  uint32_t arg;    // KERN: job-local feature id; COLL: rep-local coll index;
                   // REC/WAIT: rep-local record ordinal (NO_REC: never recorded)
  uint32_t meta;   // tag (2 bits) | sync segment << 2
};

__host__ __device__ inline uint32_t op_tag(uint32_t meta) { return meta & 3u; }
__host__ __device__ inline uint32_t op_seg(uint32_t meta) { return meta >> 2; }

struct StreamRange {
  uint32_t begin;  // rep-local op index
  uint32_t len;
  int32_t raw;     // stream handle in the trace
  uint32_t pad;
};

struct SyncRec {
  int64_t gpre;     // gap prefix at the sync position
  uint32_t type;    // SyncType
  uint32_t arg;     // SSYNC: local stream (or NO_REC if the stream never ran an op);
                    // ESYNC: record ordinal (NO_REC if never recorded)
  uint32_t cnt;     // index into counts: n_streams entries, ops dispatched per stream
  uint32_t pad;
};

struct MemRec {
  int64_t delta;
  int64_t gpre;
  uint32_t seg;
  uint32_t seq;
};

struct RepHdr {
  uint64_t ops;        // batch op index of first op
  uint64_t streams;    // batch StreamRange index
  uint64_t colls;      // batch coll-table index
  uint64_t syncs;      // batch SyncRec index
  uint64_t counts;     // batch counts index
  uint64_t mems;       // batch MemRec index
  int64_t gend;        // total host gaps of the trace
  uint32_t n_ops, n_streams, n_recs, n_colls, n_syncs, n_mems;
  uint32_t n_events, job;
};

// Kernel feature (one per unique (op kind, dtype, flops, bytes) of a job, or a
// host-provided duration).
struct Feature {
  int64_t flops;
  int64_t bytes;
  int64_t fixed;       // >= 0: host duration; -1: roofline
  int32_t op_kind;
  int16_t dtype;
  int16_t device;
};

struct CommRec {
  int32_t nranks;
  int32_t topo;
  uint32_t call_base;  // job-local slot index of call 0
  uint32_t n_calls;
};

struct SlotRec {       // one (comm, call_idx) group call
  int64_t bytes;
  int64_t fixed;       // >= 0: host wire time; -1: alpha-beta
  int32_t kind;        // -1: unused slot
  int32_t nranks;
  int32_t topo;
  int32_t device;
};

struct RankRec {
  uint32_t rep;        // batch rep index
  uint32_t comm;       // job-local index into rank_comm
  uint32_t fire;       // job-local fire-table base
  uint32_t delay;      // job-local delay-table base (n_syncs + 1 entries)
  uint32_t walker;     // job-local index of this rank's first walker
  uint32_t tl;         // job-local timeline base (sum of device ops of lower ranks)
};

struct JobHdr {
  uint64_t ranks;      // batch RankRec index
  uint64_t rank_comm;  // batch rank_comm index
  uint64_t comms;      // batch CommRec index
  uint64_t slots;      // batch slot index
  uint64_t walkers;    // batch walker index (uint32 job-local rank per walker + local stream)
  uint64_t feats;      // batch feature index
  uint64_t fire;       // batch fire-table base (int64 entries)
  uint64_t delay;      // batch delay-table base (int64 entries)
  uint64_t wstate;     // batch walker-state base
  uint64_t timeline;   // batch timeline base (per rank-op slots), if recorded
  int64_t capacity;
  int64_t rank_ops;
  int64_t dev_ops;     // sum over ranks of device ops (dispatched == completed when OK)
  uint32_t n_ranks, n_comms, n_slots, n_walkers, n_feats, device;
  int32_t key_rank;
  int32_t status;      // pre-set by the packer (BAD_INPUT, INTERNAL) else 0
};

struct Walker {
  uint32_t rank;       // job-local
  uint32_t stream;     // local stream index of rank's rep
};

struct WState {        // per-walker scheduler state
  int64_t x;           // completion time of the last op processed
  uint32_t i;          // next op (stream-relative)
  uint32_t flags;      // bit0: arrival posted for the collective at i
};

struct CollSlot {      // collective rendezvous (sim.py:326-343)
  unsigned long long maxarr;
  uint32_t count;
  uint32_t pad;
};

struct RepOut {        // memory scan result per representative
  int64_t peak;
  int32_t first_exceed;   // MemRec index (rep-local) of first mem > capacity, -1 none
  int32_t pad;
};

}  // namespace maya
