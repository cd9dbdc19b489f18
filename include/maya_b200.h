/*
 * maya_b200.h — C ABI of the B200 batched trace-driven simulator engine.
 *
 * The engine replaces, for a batch of collated jobs, the reference call chain
 *     annotate(job, RooflineEstimator())      pkg/src/dltsim/estimate.py:329-361
 *     simulate(annotated, cluster)            pkg/src/dltsim/sim.py:476-485
 *     _rank(trials) / SearchResult.best       pkg/src/dltsim/search.py:349-357, 337-339
 * i.e. the body of PipelineEvaluator.__call__ after trace generation
 * (search.py:200-209).  Plain pointers and sizes only; every function returns
 * 0 on success or a negative MAYA_E* code, with maya_last_error() giving a
 * thread-local message.
 *
 * Inputs are "raw jobs": the JobTrace/AnnotatedJob fields the simulator reads,
 * flattened to integer arrays (see paper_2503_20191_b200/rawtrace.py for the
 * event payload table).  String ids (op kinds, dtypes) are batch-global and
 * resolved by the caller.
 */
#ifndef MAYA_B200_H
#define MAYA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MAYA_ABI_VERSION 1
#define MAYA_MAX_DTYPES 16

/* return codes */
#define MAYA_OK 0
#define MAYA_EINVAL -1      /* malformed input (reference would raise ValueError/KeyError) */
#define MAYA_ECUDA -2       /* CUDA runtime failure */
#define MAYA_ENOMEM -3
#define MAYA_ESTATE -4      /* call order violated */

/* per-job status (maya_job_result.status) */
#define MAYA_ST_OK 0
#define MAYA_ST_DEADLOCK 1      /* sim.py:382-402 SimDeadlockError */
#define MAYA_ST_INTERNAL 2      /* sim.py:334-337 / 345 RuntimeError */
#define MAYA_ST_ESTIMATION 3    /* estimate.py EstimationError (missing dtype peak, bad collective) */
#define MAYA_ST_OVERFLOW 4      /* a time or intermediate left the representable range */
#define MAYA_ST_BAD_INPUT 5     /* trace shape the engine does not represent */

/* event kinds (trace.py:160-174 order) */
enum {
  MAYA_EV_HOSTGAP = 0, MAYA_EV_KERNEL, MAYA_EV_MEMALLOC, MAYA_EV_MEMFREE, MAYA_EV_MEMCPY,
  MAYA_EV_MEMSET, MAYA_EV_RECORD, MAYA_EV_WAIT, MAYA_EV_ESYNC, MAYA_EV_SSYNC, MAYA_EV_DSYNC,
  MAYA_EV_COMMINIT, MAYA_EV_COLLECTIVE
};

/* DeviceClass (cluster.py:39-59) in integer form. */
typedef struct maya_device_params {
  int64_t peak_flops[MAYA_MAX_DTYPES]; /* by batch dtype id; 0 = no peak for this dtype */
  int64_t hbm_bytes_per_s;
  int64_t alpha_ns[2];                 /* [0] intra_host, [1] inter_host; mixed -> inter */
  int64_t beta_bytes_per_s[2];
} maya_device_params;

/* RooflineEstimator (estimate.py:103-134): efficiency as exact fractions
 * (Fraction(str(eff)), estimate.py:114-115) per batch op-kind id. */
typedef struct maya_roofline_params {
  int32_t n_op_kinds;
  const int64_t *eff_num;
  const int64_t *eff_den;
  int64_t overhead_ns;
} maya_roofline_params;

/* One collated job (JobTrace + optional AnnotatedJob durations). */
typedef struct maya_raw_job {
  int32_t num_ranks;
  int32_t devices_per_host;
  int64_t capacity;            /* device_memory_bytes for the OOM check (sim.py:239) */
  int32_t device;              /* index into the device table */
  int32_t n_reps;
  const int32_t *rank_rep;     /* [num_ranks] representative of each rank */
  const int64_t *ev_off;       /* [n_reps + 1] */
  const uint8_t *ev_kind;      /* [E] MAYA_EV_* */
  const int32_t *ev_stream;    /* [E] */
  const int64_t *ev_f;         /* [E][4] payload, rawtrace.py table */
  int32_t n_comms;
  const int32_t *comm_nranks;  /* [n_comms] */
  const int8_t *comm_topo;     /* [n_comms] 0 intra, 1 inter, 2 mixed */
  const int64_t *call_off;     /* [n_comms + 1] */
  const int8_t *call_kind;     /* [n_calls] 0..4, -1 unused */
  const int64_t *call_bytes;   /* [n_calls] */
  const int64_t *rank_comm_off;/* [num_ranks + 1] */
  const int32_t *rank_comm;    /* global comm of each CommInit of the rank's rep */
  const int64_t *kernel_ns;    /* [E] host durations, or NULL -> roofline on device */
  const int64_t *wire_ns;      /* [n_calls] host wire times, or NULL -> alpha-beta on device */
} maya_raw_job;

/* SimReport fields the search consumes (sim.py:59-72, search.py:209). */
typedef struct maya_job_result {
  int64_t total_ns;
  int64_t peak_mem_bytes;
  int32_t oom;
  int32_t status;              /* MAYA_ST_* */
  int32_t first_oom_rank;      /* -1 if none */
  int32_t first_oom_seq;
  int64_t dispatched_ops;
  int64_t completed_ops;
  int64_t rank_ops;            /* sum over ranks of rep trace length (work units) */
  int64_t rounds;              /* scheduler rounds used (engine diagnostic) */
} maya_job_result;

/* Top-k entry of the search reduction (search.py:349-357 order). */
typedef struct maya_topk_entry {
  int64_t time_ns;
  int32_t key_rank;            /* position of config.key() among the batch's keys */
  int32_t job;                 /* job index in the batch */
} maya_topk_entry;

typedef struct maya_engine maya_engine;

const char *maya_last_error(void);
int maya_abi_version(void);

/* Engine lifetime: one engine per CUDA device, not re-entrant. */
int maya_open(int cuda_device, maya_engine **out);
int maya_close(maya_engine *eng);

/* Batch assembly (host).  maya_batch_add_job packs a raw job into the
 * engine's pinned staging SoA; pointers need only live for the call. */
int maya_batch_reset(maya_engine *eng);
int maya_batch_set_devices(maya_engine *eng, int32_t n, const maya_device_params *devs);
int maya_batch_set_roofline(maya_engine *eng, const maya_roofline_params *roof);
int maya_batch_add_job(maya_engine *eng, const maya_raw_job *job, int32_t key_rank);
int maya_batch_add_jobs(maya_engine *eng, int32_t n, const maya_raw_job *jobs,
                        const int32_t *key_ranks, int32_t n_threads);
int maya_batch_num_jobs(maya_engine *eng);

/* Engine options (apply to jobs staged afterwards). */
#define MAYA_OPT_COLLAPSE 1   /* exact rank-class collapse (default on) */
#define MAYA_OPT_WARP_SCHED 2 /* schedule every job with the warp-window kernel instead of
                                 the lane-parallel kernel (A/B and parity testing) */
#define MAYA_OPT_NO_FOLD 8    /* keep one scheduler op per trace op (no affine run folding;
                                 A/B testing -- runs are never folded when a timeline is recorded) */
#define MAYA_OPT_LANE_SCHED 4 /* schedule every job that fits with the lane-parallel kernel
                                 (default: per job, by the shape of its FIFOs) */
#define MAYA_OPT_NO_BLOCKS 16 /* generated jobs: one op per kernel launch instead of interned
                                 kernel blocks (runs of launches of one stream, folded on the
                                 device); required to record a timeline of generated jobs */
#define MAYA_OPT_NO_CHAIN 32  /* never use the chain kernel (latency-bound jobs resident in one
                                 warp's shared memory); default: every job that fits it, unless
                                 MAYA_OPT_WARP_SCHED / MAYA_OPT_LANE_SCHED force a kernel */
int maya_set_options(maya_engine *eng, int32_t options);
/* Per staged job: 1 if it is simulated as rank classes. */
int maya_batch_collapsed(maya_engine *eng, uint8_t *out);
/* After maya_upload, per staged job: the scheduler kernel chosen for it --
   0 warp-window, 1 lane-parallel (warp or CTA job), 2 grid job, 3 chain. */
int maya_batch_kernels(maya_engine *eng, int32_t *out);

/* Upload the staged batch to HBM (the H2D leg). */
int maya_upload(maya_engine *eng);

/* Run estimators + memory scan + scheduler (+ timeline if record != 0) on the
 * resident batch; asynchronous on the engine stream. */
int maya_run(maya_engine *eng, int32_t record_timeline);

/* Download per-job results (the D2H leg); synchronises the engine stream. */
int maya_results(maya_engine *eng, maya_job_result *out);

/* Fused search reduction on device: the k best jobs by
 * (time_ns asc, key_rank asc) over OK, non-OOM jobs with time_ns > 0 first,
 * then time_ns == 0 jobs (their MFU is 0.0, search.py:784 / sim.py:493-494). */
int maya_topk(maya_engine *eng, int32_t k, maya_topk_entry *out, int32_t *n_out);

/* Enqueue the same reduction after the last maya_run without waiting; the
 * next maya_topk with the same k returns its result (stream order keeps it
 * behind the run, so a host can stage the next batch meanwhile). */
int maya_topk_async(maya_engine *eng, int32_t k);
/* Timeline of one job after maya_run(record_timeline=1): per timed op
 * (rank, stream, seq, start, end), ordered by rank then stream then FIFO. */
int maya_timeline_size(maya_engine *eng, int32_t job, int64_t *n);
int maya_timeline(maya_engine *eng, int32_t job, int32_t *rank, int32_t *stream,
                  int32_t *seq, int64_t *start, int64_t *end);

/* Per-rank statistics of _report (sim.py:406-426, RankStats sim.py:50-56) of
 * one job after maya_run(record_timeline=1), computed on the device from the
 * recorded timeline (segmented sort + union scans, stats.cu).  out is
 * [num_ranks][5]: compute_busy_ns, comm_busy_ns, exposed_comm_ns, idle_ns,
 * peak_mem_bytes, in the job's original rank numbering. */
int maya_rank_stats(maya_engine *eng, int32_t job, int32_t num_ranks, int64_t *out);
/* The engine's CUDA stream (cudaStream_t) so callers can time on it. */
int maya_get_stream(maya_engine *eng, void **stream);

/* Bytes of the staged SoA arena (what maya_upload copies host -> device). */
int64_t maya_arena_bytes(maya_engine *eng);

/* Batch totals of the staged batch: [0] jobs, [1] sum of rep trace events,
 * [2] sum over ranks of rep CommInits, [3] kernel features, [4] group-call
 * slots, [5] device op records (stream-major; a kernel block is one record),
 * [6] rank-ops, [7] arena bytes, [8] ranks, [9] reps, [10] kernels launched by
 * the last maya_run, [11] kernels launched by the last maya_topk, [12] kernel
 * blocks, [13] block feature ids, [14] wire features (unique call records),
 * [15] executed class-ops: sum over SIMULATED ranks (rank classes of collapsed
 * jobs) of their rep trace length (rank-ops [6] counts every rank). */
int maya_batch_stats(maya_engine *eng, int64_t *out16);

/* Scheduler phase counters of instrumented builds (-DMAYA_PROFILE); returns
 * 0 (and leaves out8 untouched) in product builds. */
int maya_prof_read(unsigned long long *out16, int reset);  /* 8 warp-window + 8 lane counters */

/* Device time of the last maya_run, per phase (ms): estimate, memscan, schedule. */
int maya_last_timings(maya_engine *eng, float *ms3);

/* ---- native trace generation (workload.py frontend + collate.py) -------- */

/* ModelSpec (workload.py:96-128); dtype 0 bf16, 1 fp16, 2 fp32. */
typedef struct maya_model {
  int64_t num_layers, hidden_size, seq_len, vocab_size;
  int32_t dtype;
  int32_t pad;
} maya_model;

/* ConfigPoint (workload.py:131-165). */
typedef struct maya_config {
  int32_t tp, pp, micro_mult, virtual_stages;
  int32_t act_recompute, seq_parallel, dist_optimizer;
  int32_t pad;
  int64_t global_batch;
} maya_config;

/* ClusterSpec (cluster.py:62-92) without the device class. */
typedef struct maya_cluster {
  int32_t num_hosts, devices_per_host;
  int64_t device_memory_bytes;
} maya_cluster;

/* schedule: -1 default_schedule (workload.py:218-221), 0 gpipe, 1 1f1b, 2 interleaved */
typedef struct maya_gen maya_gen;

typedef struct maya_gen_view {
  maya_raw_job job;        /* device = 0; kernel_ns = wire_ns = NULL */
  int32_t num_hosts;
  int32_t n_comm_names;
  const int64_t *rep_ranks;
  const char *comm_names;  /* n_comm_names names joined by '\n' (sorted, = JobTrace.groups) */
  int64_t n_events;
  int64_t n_calls;
  int64_t n_rank_comm;
} maya_gen_view;

/* Op-kind / dtype id tables used by generated jobs' ev_f. */
const char *maya_gen_op_kind_name(int32_t id);
const char *maya_gen_dtype_name(int32_t id);

int maya_gen_job(const maya_model *model, const maya_config *cfg, const maya_cluster *cluster,
                 int32_t schedule, int64_t dispatch_overhead_ns, maya_gen **out);
int maya_gen_view_of(const maya_gen *g, maya_gen_view *view);
int maya_gen_free(maya_gen *g);

/* ---- text traces and job manifests (trace.py:282-495, collate.py:256-431) --
 * Native parse_trace / serialize_trace / validate_trace and save_job /
 * load_job + collate.  Errors return MAYA_EINVAL with maya_last_error() set to
 * the reference's exception message and maya_last_error_kind() to its class. */
#define MAYA_ERR_PARSE 1        /* TraceParseError (trace.py:209-212) */
#define MAYA_ERR_VALIDATION 2   /* TraceValidationError (trace.py:215-220) */
#define MAYA_ERR_COLLATION 3    /* CollationError (collate.py:42) */
#define MAYA_ERR_RANGE 4        /* an integer the engine's int64/int32 fields cannot hold */
#define MAYA_ERR_IO 5           /* file missing / unwritable (FileNotFoundError) */
int maya_last_error_kind(void);
typedef struct maya_trace maya_trace;
/* parse_trace + validate_trace of one rank_<r>.trace text (universal newlines). */
int maya_trace_parse(const char *text, int64_t len, maya_trace **out);
/* [0] global rank, [1] host, [2] device, [3] events */
int maya_trace_info(const maya_trace *t, int64_t *out4);
/* serialize_trace; the text is owned by t (valid until the next call or free). */
int maya_trace_serialize(maya_trace *t, const char **text, int64_t *len);
int maya_trace_free(maya_trace *t);
/* load_job(manifest, cluster): the rank traces, dup expansion and collate, into
 * a raw job (maya_gen_view_of; string tables via maya_gen_names). */
int maya_job_load(const char *manifest_path, const maya_cluster *cluster, maya_gen **out);
/* save_job of a loaded job: rank_<r>.trace per representative + manifest. */
int maya_job_save(const maya_gen *g, const char *out_dir, const char *manifest_name);
/* '\n'-joined op-kind (which 0) or dtype (which 1) names of a job's ev_f ids. */
int maya_gen_names(const maya_gen *g, int32_t which, const char **blob, int32_t *n);
/* Generate + pack n configs straight into the engine batch (no host round
 * trip through arrays).  status_out[i] receives 0 or MAYA_EINVAL for an
 * invalid configuration (ConfigError, workload.py:168-208); such jobs are
 * staged with status MAYA_ST_BAD_INPUT. */
int maya_batch_add_generated(maya_engine *eng, const maya_model *model, int32_t n,
                             const maya_config *cfgs, const maya_cluster *cluster,
                             int32_t device, int32_t schedule, int64_t dispatch_overhead_ns,
                             const int32_t *key_ranks, int32_t n_threads, int32_t *status_out);

/* Test hook: packs each config through the fused generate->pack path and
 * through generate + pack_job, and returns how many packs differ (0 expected). */
int maya_debug_pack_compare(const maya_model *model, int32_t n, const maya_config *cfgs,
                            const maya_cluster *cluster, int32_t schedule,
                            int64_t dispatch_overhead_ns, int32_t collapse);

#ifdef __cplusplus
}
#endif
#endif
