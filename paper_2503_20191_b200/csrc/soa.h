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
static const uint32_t NO_WF = 0xFFFFFFFFu;   // coll_wf: the collective does not fold
// Op.arg flag of a KERN op that stands for a kernel BLOCK: n consecutive
// kernel launches of one stream, each after a host gap of `gap` ns, with no
// other event in between (the generator's layer bodies).  Blocks are interned
// per job (KBlock); the device folds each into one affine map after the
// estimator (kernels.cu block_compose_kernel).  Only in batches that fold.
static const uint32_t KBLOCK = 0x80000000u;
struct KBlock {
  uint32_t fid0;       // job-local index of its first feature id in the job's block fid list
  uint32_t n;          // kernels (>= 2)
  int64_t gap;         // host gap before each kernel (ns)
};
// On-chip layout of one job inside a scheduler CTA (shared by the engine,
// which sizes dynamic shared memory, and the kernel).  When the whole layout
// does not fit the CTA's dynamic shared memory, host-sync counters and walker
// states go to a per-job global spill area of spill_bytes() and collectives
// rendezvous through global slots.
struct SchedLayout {
  uint32_t ring, cb, hostk, state, ctx, fire, rcx, bytes;   // byte offsets / total
  bool on_chip;     // walker state/contexts, host-sync counters in smem
  bool ring_on;     // collectives rendezvous in smem rings
  bool fire_on;     // event-record times in smem
  bool rcx_on;      // per-rank collective entries + wire times in smem
};
static const uint32_t RING_MAX_COMMS = 4096;
static const uint32_t WSTATE_BYTES = 48;
static const uint32_t WCTX_BYTES = 64;
__host__ __device__ inline uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }
// Greedy: the walker core must fit; then record times; then collective tables.
__host__ __device__ inline SchedLayout sched_layout(uint32_t W, uint32_t R, uint32_t n_comms,
                                                    bool ring_flag, uint32_t n_fire,
                                                    uint32_t n_rcolls, uint32_t cap) {
  SchedLayout L{};
  L.ring_on = ring_flag && n_comms <= RING_MAX_COMMS;
  uint64_t off = 0;
  L.ring = (uint32_t)off;
  if (L.ring_on) off += 32ull * n_comms;
  L.cb = (uint32_t)off;
  off = align16((uint32_t)(off + 4ull * n_comms));
  L.hostk = (uint32_t)off;
  off = align16((uint32_t)(off + 4ull * R));
  L.state = (uint32_t)off;
  off += (uint64_t)WSTATE_BYTES * W;
  L.ctx = (uint32_t)off;
  off += (uint64_t)WCTX_BYTES * W;
  L.on_chip = off <= cap;
  if (!L.on_chip) {
    L.ring_on = false;
    L.bytes = 0;
    return L;
  }
  L.fire = (uint32_t)off;
  if (off + 8ull * n_fire <= cap) {
    L.fire_on = true;
    off += 8ull * n_fire;
  }
  L.rcx = (uint32_t)off;
  if (off + 16ull * n_rcolls <= cap) {
    L.rcx_on = true;
    off += 16ull * n_rcolls;
  }
  L.bytes = (uint32_t)off;
  return L;
}
// global spill (hostk + states) for jobs whose layout exceeds the CTA budget
inline uint64_t spill_bytes(uint64_t W, uint64_t R) {
  return ((4 * R + 15) & ~15ull) + WSTATE_BYTES * W + 16;
}
// warps per scheduler CTA for a job with R ranks (4..16, power of two): a
// warp owns all stream FIFOs of its ranks (they are coupled by event
// record/wait; ranks couple only through collectives)
__host__ __device__ inline uint32_t sched_warps(uint32_t R) {
  uint32_t nw = 4;
  while (nw < R && nw < 16) nw <<= 1;
  return nw;
}

// ---- lane-parallel scheduler (sched_lane.cu) ---------------------------------
// One CTA per job, one lane per (rank, stream) FIFO; a FIFO stages its ops in
// a ring of 8-op (128 B) shared-memory slots filled by bulk copies.
static const uint32_t LANE_MAX_THREADS = 512;
static const uint32_t LANE_SMEM_CAP = 220 * 1024;
static const uint32_t LANE_SLOT_OPS = 8;
enum LaneFlags : uint32_t {
  LANE_COLL_RING = 1,   // collectives rendezvous in shared-memory rings
  LANE_FIRE_SMEM = 2,   // record times in shared memory
  LANE_RCX_SMEM = 4,    // per-rank collective table in shared memory
  LANE_CTX_SMEM = 8,    // FIFO contexts in shared memory (lanes own several FIFOs)
  LANE_ST_GLOBAL = 16,  // FIFO states in global memory (jobs with thousands of FIFOs)
};
struct LaneJob {
  uint64_t mbase;       // chain jobs: batch index of the job's first macro op (DevBatch.macros)
  uint32_t flags;       // LaneFlags
  uint32_t n_slots;     // ring slots of the job (sum over FIFOs)
  uint64_t wslot;       // batch index of the job's first per-walker ring word
  uint64_t perm;        // batch index of the job's lane -> FIFO table
  uint32_t per_lane;    // FIFOs per lane (table is per_lane x group threads, 0xFFFFFFFF pad)
  uint32_t fc_log2;     // record-time cache entries (log2; 0: none) when LANE_FIRE_SMEM is off
};
// One CTA of a grid job (a job too large for one CTA): a rank-aligned range
// of its FIFOs.  All parts of a grid job are co-resident (cooperative launch);
// collectives rendezvous in global slots and rounds end at a job-wide barrier.
struct GridPart {
  uint32_t job, part, n_parts, warps_total;   // warps_total: all parts of the job
  uint32_t w0, w1, r0, r1;                    // job-local FIFO and rank ranges
  uint32_t flags, n_slots, fc_log2, first;    // first: batch index of the job's part 0
  uint64_t wslot;                             // batch index of the part's ring words
};
// Job-wide synchronisation of a grid job (scratch, zeroed every run).
struct GridSync {
  unsigned arrive, gen;
  int active, progress;
  int err, incomplete;
  int oom_rank, rounds;
  unsigned long long tmax;
  long long peak, oom_t;
};

// Chain-kernel macro ops: the folded FIFO grouped greedily into
// [WAIT]? [KERN | COLL]? [REC]? within one host-sync segment (sched_chain.cu
// chain_macro_kernel builds them; the host counts them with the same rule to
// size the shared-memory region).  One macro op is one lockstep iteration:
//   ready = max(x, r1 + delay, fire[widx]);  body: + dk | rendezvous + wire;
//   out = max(body, rr + delay);  fire[ridx] = out.
struct alignas(16) ChainMacro {
  int64_t r1;        // max dispatch (gap prefix) of the WAIT and body ops (INT64_MIN/4: none)
  int64_t dk;        // KERN duration (folded run)
  int64_t rr;        // REC dispatch (INT64_MIN/4: none)
  uint32_t widx;     // WAIT: rep-local record ordinal
  uint32_t ridx;     // REC: rep-local record ordinal
  uint32_t cidx;     // COLL: rep-local collective index
  uint32_t end;      // folded ops of the FIFO up to and including this macro
  uint32_t kind;     // CM_* bits
  uint32_t pad;
};
static_assert(sizeof(ChainMacro) == 48, "ChainMacro");
enum : uint32_t {
  CM_WAIT = 1, CM_REC = 2, CM_KERN = 4, CM_COLL = 8,
  CM_NEVER = 16,     // the WAIT's event is never recorded: blocks forever
  CM_BAD = 32,       // the kernel's estimate failed (EXEC_BAD)
  CM_OVF = 64,       // the folded run's composite overflowed (EXEC_OVF)
  CM_FAIL = 0xffffffffu,   // (first macro's kind) the macro pass disagreed with the plan
};
// op classes of the fusion rule: 0 kernel (incl. folded runs), 1 collective,
// 2 record, 3 wait.  Greedy state machine (one per FIFO, reset per segment).
struct MacroFuse {
  int state = 0;             // 0 closed, 1 open after a WAIT, 2 open after a body
  uint32_t seg = 0xffffffffu;
  // true: op of class `cls` in segment `sg` starts a new macro
  __host__ __device__ bool push(uint32_t cls, uint32_t sg) {
    if (sg != seg) { seg = sg; state = 0; }
    const bool body = cls <= 1;
    if (state == 1 && (body || cls == 2)) { state = body ? 2 : 0; return false; }
    if (state == 2 && cls == 2) { state = 0; return false; }
    state = cls == 3 ? 1 : body ? 2 : 0;
    return true;
  }
};

// ---- chain scheduler (sched_chain.cu) ---------------------------------------
// Latency-bound jobs (few FIFOs, frequent hand-offs: pipeline stages) run with
// one warp per job and EVERYTHING resident in shared memory: the folded op
// stream of every FIFO, record times, collective rings and the rank
// collective table.  Per-walker word (lane_wslot): the FIFO's first op in the
// region's op area.  Region classes by footprint.
static const uint32_t CHAIN_MAX_FIFOS = 256;  // one FIFO per thread, 1, 2, 4 or 8 warps
static const uint32_t CHAIN_CLASSES = 10;
static const uint32_t CHAIN_REGION[CHAIN_CLASSES] = {8u << 10,  12u << 10, 16u << 10, 24u << 10,
                                                     32u << 10, 48u << 10, 64u << 10, 96u << 10,
                                                     144u << 10, 220u << 10};
struct ChainLayout {
  uint32_t bar, ring, hostk, fst_i, fst_x, fire, rcx, ops, bytes;
};
__host__ __device__ inline ChainLayout chain_layout(uint32_t W, uint32_t R, uint32_t n_comms,
                                                    uint32_t n_fire, uint32_t n_rcolls,
                                                    uint64_t n_ops) {
  ChainLayout L{};
  uint64_t off = 0;
  L.bar = 0;
  off = 16;
  L.ring = (uint32_t)off;
  off += 32ull * (n_comms <= RING_MAX_COMMS ? n_comms : 0);   // 2 CollSlot per communicator
  L.hostk = (uint32_t)off;
  off = (off + 4ull * R + 15) & ~15ull;
  L.fst_i = (uint32_t)off;
  off = (off + 4ull * W + 15) & ~15ull;
  L.fst_x = (uint32_t)off;
  off += 8ull * W;
  off = (off + 15) & ~15ull;
  L.fire = (uint32_t)off;
  off = (off + 8ull * n_fire + 15) & ~15ull;
  L.rcx = (uint32_t)off;
  off += 16ull * n_rcolls;
  L.ops = (uint32_t)off;
  off += sizeof(ChainMacro) * n_ops;   // n_ops: the job's macro ops (folded runs: resident)
  L.bytes = off > 0xffffffffull ? 0xffffffffu : (uint32_t)off;
  return L;
}

// per-walker ring word: first slot (job-local, 28 bits) | log2(slots) << 28
// (0xF << 28: the FIFO reads global memory directly)
struct LaneLayout {
  uint32_t ring, cb, hostk, state, ctx, bars, rdata, fire, fcache, rcx, bytes;
};
__host__ __device__ inline LaneLayout lane_layout(uint32_t W, uint32_t R, uint32_t n_comms,
                                                  uint32_t flags, uint32_t n_slots,
                                                  uint32_t n_fire, uint32_t n_rcolls,
                                                  uint32_t fc_log2) {
  LaneLayout L{};
  uint64_t off = 0;
  L.ring = (uint32_t)off;
  if (flags & LANE_COLL_RING) off += 32ull * n_comms;
  L.cb = (uint32_t)off;
  off = (off + 4ull * n_comms + 15) & ~15ull;
  L.hostk = (uint32_t)off;
  off = (off + 4ull * R + 15) & ~15ull;
  L.state = (uint32_t)off;
  if (!(flags & LANE_ST_GLOBAL)) off += 48ull * W;
  L.ctx = (uint32_t)off;
  if (flags & LANE_CTX_SMEM) off += 64ull * W;
  L.bars = (uint32_t)off;
  off = (off + 8ull * n_slots + 127) & ~127ull;
  L.rdata = (uint32_t)off;
  off += 16ull * LANE_SLOT_OPS * n_slots;
  L.fire = (uint32_t)off;
  if (flags & LANE_FIRE_SMEM) off += (8ull * n_fire + 15) & ~15ull;
  L.fcache = (uint32_t)off;
  if (!(flags & LANE_FIRE_SMEM) && fc_log2) off += 16ull << fc_log2;
  L.rcx = (uint32_t)off;
  if (flags & LANE_RCX_SMEM) off += 16ull * n_rcolls;
  L.bytes = off > 0xffffffffull ? 0xffffffffu : (uint32_t)off;
  return L;
}

// One 1,024-op chunk of one FIFO for the run-folding pass (kernels.cu):
// runs are cut at chunk starts, so chunks fold independently.
static const uint32_t FOLD_CHUNK = 1024;
struct FoldChunk {
  uint32_t rep;        // batch rep index
  uint32_t st;         // local stream
  uint32_t chunk;      // chunk index within the FIFO
  uint32_t out;        // folded ops of the FIFO before this chunk (host-counted, pack.cpp)
};

// 16-byte device op record.
struct alignas(16) Op {
  int64_t disp;    // sum of host gaps before this op in host order (ns)
  uint32_t arg;    // KERN: job-local feature id; COLL: rep-local coll index;
                   // REC/WAIT: rep-local record ordinal (NO_REC: never recorded)
  uint32_t meta;   // tag (2 bits) | sync segment << 2
};

// meta bit 31 (OP_FOLDC): a collective that folds into kernel runs (pack.cpp
// coll_wf: every simulated rank of the rep meets it alone), so the fold pass's
// eligibility test reads the op only; segments stay below 2^29.
static const uint32_t OP_FOLDC = 0x80000000u;
__host__ __device__ inline uint32_t op_tag(uint32_t meta) { return meta & 3u; }
__host__ __device__ inline uint32_t op_seg(uint32_t meta) { return (meta >> 2) & 0x1FFFFFFFu; }

struct StreamRange {
  uint32_t begin;  // rep-local op index
  uint32_t len;
  int32_t raw;     // stream handle in the trace
  uint32_t folded; // ops after the device folds kernel runs (ring sizing)
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
  uint32_t n_devev;    // device events (kernel-class, collective, record, wait): n_ops
                       // plus the kernels hidden in blocks
  uint32_t pad3;
};

// Kernel feature (one per unique (op kind, dtype, flops, bytes) of a job, or a
// host-provided duration): 16 B of operands plus a 4 B meta word in a parallel
// array, so the estimator streams 20 B per feature.
struct Feature {
  int64_t flops;       // FMETA_FIXED: the host duration
  int64_t bytes;
};
static const uint32_t FMETA_FIXED = 0x80000000u;
__host__ __device__ inline uint32_t fmeta(int32_t op_kind, int32_t dtype, int32_t device) {
  return ((uint32_t)op_kind & 0xfffu) | (((uint32_t)dtype & 0xffu) << 12) |
         (((uint32_t)device & 0xffu) << 20);
}
__host__ __device__ inline int32_t fmeta_op(uint32_t m) { return (int32_t)(m & 0xfffu); }
__host__ __device__ inline int32_t fmeta_dtype(uint32_t m) { return (int32_t)((m >> 12) & 0xffu); }
__host__ __device__ inline int32_t fmeta_device(uint32_t m) { return (int32_t)((m >> 20) & 0xffu); }

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
  uint32_t rslot;      // job-local base of this rank's collective table (one per rep coll)
  uint32_t pad;
};

// Scheduler op record, produced on device by the resolve pass from Op and the
// estimator output: everything a walker needs, no dependent gathers.
struct alignas(16) ExecOp {
  int64_t disp;        // gap prefix (host dispatch offset)
  uint64_t w;          // tag (2 bits) | payload << 2: KERN duration, REC/WAIT ordinal,
                       // COLL rep-local collective index
};

// Per-(rank, rep collective) entry: nranks << 48 | job-local comm << 32 | call_idx
typedef uint64_t RankColl;

enum JobFlags : uint32_t { JOB_RING = 1 };  // collectives rendezvous in shared-memory rings

struct JobHdr {
  uint64_t ranks;      // batch RankRec index
  uint64_t rank_comm;  // batch rank_comm index
  uint64_t comms;      // batch CommRec index
  uint64_t slots;      // batch slot index
  uint64_t walkers;    // batch walker index (uint32 job-local rank per walker + local stream)
  uint64_t feats;      // batch feature index
  uint64_t fire;       // batch fire-table base (int64 entries)
  uint64_t delay;      // batch delay-table base (int64 entries)
  uint64_t wstate;     // byte offset of the job's spill area (scheduler state overflow)
  uint64_t timeline;   // batch timeline base (per rank-op slots), if recorded
  uint64_t rcolls;     // batch RankColl base
  int64_t capacity;
  int64_t rank_ops;
  int64_t dev_ops;     // sum over ranks of device ops (dispatched == completed when OK)
  uint32_t n_ranks, n_comms, n_slots, n_walkers, n_feats, device;
  int32_t key_rank;
  int32_t status;      // pre-set by the packer (BAD_INPUT, INTERNAL) else 0
  uint32_t flags;      // JobFlags
  uint32_t n_rcolls;
  uint32_t n_fire;     // record-time entries of the simulated ranks
  uint32_t n_blocks;   // kernel blocks (KBlock) of the job
  uint64_t blocks;     // batch KBlock index
  uint64_t blk_fids;   // batch index into the block feature-id list
};

// per-(rank, rep collective) entry with its wire time (resolve_colls_kernel)
struct RCX {
  uint64_t ent;        // RankColl
  int64_t wire;
};

struct Walker {
  uint32_t rank;       // job-local
  uint32_t stream;     // local stream index of rank's rep
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
