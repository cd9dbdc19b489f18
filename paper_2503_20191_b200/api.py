"""Drop-in, reference-shaped API over the CUDA engine.

Mirrors the reference's hot-path entry points so that a dltsim user can swap
them in:

* ``simulate(annotated, cluster=None, record_timeline=False) -> SimReport``
  — pkg/src/dltsim/sim.py:476-485 (SimReport fields :59-105, errors :46-47);
* ``compute_mfu(report, model_flops, cluster, dtype)`` — sim.py:488-497;
* ``GpuPipelineEvaluator`` — the ``PipelineEvaluator`` of search.py:187-209
  (same fields, ``__call__(config) -> EvalResult``) plus ``evaluate_many`` /
  ``prefetch`` that run a whole population as one GPU batch;
* ``evaluate_space`` — every valid config of a SearchSpace in one batch plus
  the fused device top-k, ranked exactly like ``_rank`` (search.py:349-357).

Reference classes (SimReport, RankStats, EvalResult, SimDeadlockError) are
used when dltsim is importable, else the same-named mirrors below.
"""

from __future__ import annotations

import functools
from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np

from ._abi import (ST_DEADLOCK, ST_ESTIMATION, ST_INTERNAL, ST_OK, ST_OVERFLOW, STATUS_NAMES,
                   DEFAULT_EFFICIENCY, DEFAULT_KERNEL_OVERHEAD_NS, Batch)
from .rawtrace import RawJob, from_annotated, from_reference
from . import workload as W


# --- reference-compatible result types ------------------------------------------

class SimDeadlockError(Exception):
    """Queue drained with blocked work left (sim.py:46-47)."""


class EstimationError(Exception):
    """estimate.py:59-60."""


@dataclass
class RankStats:
    compute_busy_ns: int = 0
    comm_busy_ns: int = 0
    exposed_comm_ns: int = 0
    idle_ns: int = 0
    peak_mem_bytes: int = 0


@dataclass
class SimReport:
    total_ns: int
    per_rank: dict
    oom: bool
    first_oom: tuple | None
    dispatched_ops: int
    completed_ops: int
    mfu: float | None = None
    timeline: list = field(default_factory=list)

    @property
    def peak_mem_bytes(self) -> int:
        return max((s.peak_mem_bytes for s in self.per_rank.values()), default=0)

    @property
    def exposed_comm_ns(self) -> int:
        return max((s.exposed_comm_ns for s in self.per_rank.values()), default=0)


@dataclass(frozen=True)
class EvalResult:
    time_ns: int
    mfu: float | None
    peak_mem_bytes: int
    oom: bool


def _ref_types():
    """Use dltsim's own classes when the reference is importable."""
    try:
        from dltsim import sim as rs
        from dltsim import search as rsearch
        from dltsim import estimate as rest
        from dltsim import workload as rwork
        return dict(SimReport=rs.SimReport, RankStats=rs.RankStats,
                    SimDeadlockError=rs.SimDeadlockError, EvalResult=rsearch.EvalResult,
                    EstimationError=rest.EstimationError, ConfigError=rwork.ConfigError)
    except Exception:
        return dict(SimReport=SimReport, RankStats=RankStats,
                    SimDeadlockError=SimDeadlockError, EvalResult=EvalResult,
                    EstimationError=EstimationError, ConfigError=W.ConfigError)


# --- engine singletons (one per CUDA device per process) -------------------------

@functools.lru_cache(maxsize=None)
def _engine(device: int = 0):
    from .engine import Engine
    return Engine(device)


def _raise_for(status: int, what: str = "", raw: RawJob | None = None, timeline=None) -> None:
    """Raise the reference's exception for a failed job.  With the job (and,
    for deadlocks, its timeline run) the text is the reference's own
    (residue.py: sim.py:382-402, estimate.py:124-127 + 339-346)."""
    from .residue import deadlock_message, estimation_message
    T = _ref_types()
    if status == ST_OK:
        return
    if status == ST_DEADLOCK:
        if raw is not None and timeline is not None:
            raise T["SimDeadlockError"](deadlock_message(raw, timeline))
        raise T["SimDeadlockError"](f"simulation deadlocked with blocked work{what}")
    if status == ST_ESTIMATION:
        msg = estimation_message(raw) if raw is not None else None
        raise T["EstimationError"](msg or f"estimator failed{what}")
    if status == ST_INTERNAL:
        raise RuntimeError(f"internal error{what}")
    raise ValueError(f"engine status {STATUS_NAMES[status]}{what}")


def _failure(status: int, raw: RawJob, device: int) -> Exception:
    """The exception of a failed generated job: deadlocks are re-run alone with
    a timeline (error path only) so the residue names the blocked objects."""
    timeline = None
    if status == ST_DEADLOCK:
        res, eng = simulate_raw([raw], device, record_timeline=True)
        if int(res[0]["status"]) == ST_DEADLOCK:
            timeline = eng.timeline(0)
    try:
        _raise_for(status, "", raw, timeline)
    except Exception as exc:  # noqa: BLE001 - returned to the caller
        return exc
    return RuntimeError("no failure")


def _is_default_roofline(est) -> bool:
    return (type(est).__name__ == "RooflineEstimator" and hasattr(est, "efficiency")
            and hasattr(est, "overhead_ns"))


# --- simulate() ----------------------------------------------------------------------

def simulate_raw(jobs: Sequence[RawJob], device: int = 0, record_timeline: bool = False,
                 efficiency: Mapping[str, float] | None = None,
                 overhead_ns: int = DEFAULT_KERNEL_OVERHEAD_NS):
    """Batch entry on raw jobs: returns (results array, engine)."""
    eng = _engine(device)
    res = eng.simulate(list(jobs), record_timeline=record_timeline, efficiency=efficiency,
                       overhead_ns=overhead_ns)
    return res, eng


def simulate(annotated, cluster=None, record_timeline: bool = False, device: int = 0):
    """Drop-in for dltsim.simulate (sim.py:476-485) on the GPU engine."""
    raw = from_annotated(annotated, cluster)
    res, eng = simulate_raw([raw], device, record_timeline=True)
    r = res[0]
    st = int(r["status"])
    _raise_for(st, "", raw, eng.timeline(0) if st == ST_DEADLOCK else None)
    T = _ref_types()
    # per-rank busy / exposed / idle / peak: segmented sort + union scans on the
    # device over the recorded timeline (stats.cu, _report sim.py:406-426)
    per_rank = {q: T["RankStats"](compute_busy_ns=int(x[0]), comm_busy_ns=int(x[1]),
                                  exposed_comm_ns=int(x[2]), idle_ns=int(x[3]),
                                  peak_mem_bytes=int(x[4]))
                for q, x in enumerate(eng.rank_stats(0, raw.num_ranks))}
    timeline = []
    if record_timeline:
        names = _timeline_names(raw, eng)
        timed = eng.timeline(0).timed()
        order = np.lexsort((timed.start, timed.end, timed.rank))
        timeline = [(int(timed.rank[i]), int(timed.stream[i]), names(timed, i),
                     int(timed.start[i]), int(timed.end[i])) for i in order]
    return T["SimReport"](
        total_ns=int(r["total_ns"]), per_rank=per_rank, oom=bool(r["oom"]),
        first_oom=((int(r["first_oom_rank"]), int(r["first_oom_seq"])) if r["oom"] else None),
        dispatched_ops=int(r["dispatched_ops"]), completed_ops=int(r["completed_ops"]),
        timeline=timeline)


def _timeline_names(raw: RawJob, eng):
    from .rawtrace import COLLECTIVE_KINDS, EV_COLLECTIVE
    ops = raw.op_kind_names

    def name(tl, i):
        rep = raw.rank_rep[int(tl.rank[i])]
        ev = int(raw.ev_off[rep]) + int(tl.seq[i])
        if raw.ev_kind[ev] == EV_COLLECTIVE:
            return COLLECTIVE_KINDS[int(raw.ev_f[ev, 2])]
        return ops[int(raw.ev_f[ev, 0])]
    return name


def compute_mfu(report, model_flops: int, cluster, dtype: str) -> float | None:
    """sim.py:488-497, verbatim arithmetic (int/int true division)."""
    if report.oom:
        return None
    if report.total_ns <= 0:
        return 0.0
    peak = cluster.device.peak_flops[dtype]
    achieved_per_s = model_flops * 1_000_000_000 / report.total_ns
    return achieved_per_s / (cluster.num_devices * peak)


def _mfu(total_ns: int, oom: bool, model_flops: int, cluster, dtype: str):
    if oom:
        return None
    if total_ns <= 0:
        return 0.0
    return (model_flops * 1_000_000_000 / total_ns) / (cluster.num_devices
                                                       * cluster.device.peak_flops[dtype])


# --- model flops (workload.py:117-128) -------------------------------------------------

def iteration_flops(model, global_batch: int) -> int:
    if hasattr(model, "iteration_flops"):
        return model.iteration_flops(global_batch)
    s, h, v, b = model.seq_len, model.hidden_size, model.vocab_size, global_batch
    layer = (8 * b * s * h + 2 * b * s * 3 * h * h + 2 * b * s * s * h + 5 * b * s * s
             + 2 * b * s * s * h + 2 * b * s * h * h + b * s * h + 8 * b * s * h
             + 2 * b * s * 4 * h * h + 8 * 4 * b * s * h + 2 * b * s * h * 4 * h + b * s * h)
    head = 8 * b * s * h + 2 * b * s * v * h + 5 * b * s * v
    return 3 * (model.num_layers * layer + head)


# --- PipelineEvaluator drop-in -----------------------------------------------------------

class GpuPipelineEvaluator:
    """search.py:187-209 on the GPU: generate -> collate -> annotate -> simulate.

    ``__call__`` evaluates one config (cached if prefetched); ``evaluate_many``
    runs a population as one batch.  Not picklable into worker processes (it
    owns a CUDA engine): use ``run_search(..., jobs=1)``.
    """

    def __init__(self, model, cluster, estimator=None, dispatch_overhead_ns: int = 0,
                 schedule=None, device: int = 0, threads: int = 8):
        self.model = model
        self.cluster = cluster
        self.estimator = estimator
        self.dispatch_overhead_ns = dispatch_overhead_ns
        self.schedule = schedule
        self.device = device
        self.threads = threads
        self._cache: dict = {}

    def _efficiency(self):
        est = self.estimator
        if est is None:
            return dict(DEFAULT_EFFICIENCY), DEFAULT_KERNEL_OVERHEAD_NS
        if _is_default_roofline(est):
            return dict(est.efficiency), int(est.overhead_ns)
        return None, None

    def evaluate_many(self, configs: Sequence) -> list:
        """EvalResult per config, or the exception its evaluation raised (the
        reference's class and text, as run_search records it, search.py:370-374)."""
        T = _ref_types()
        configs = list(configs)
        out: list = [None] * len(configs)
        todo = []
        for i, c in enumerate(configs):
            sched = self.schedule or W.default_schedule(c)
            errors = W.validate_config(self.model, c, self.cluster, sched)
            if errors:
                out[i] = T["ConfigError"]("; ".join(errors))
            else:
                todo.append(i)
        if not todo:
            return out
        eff, overhead = self._efficiency()
        eng = _engine(self.device)
        raws = None
        if eff is not None:
            sub = [configs[i] for i in todo]
            eng.stage_generated(self.model, sub, self.cluster, schedule=self.schedule,
                                dispatch_overhead_ns=self.dispatch_overhead_ns,
                                efficiency=eff, overhead_ns=overhead, threads=self.threads)
            eng.upload()
        else:  # user estimator: host annotations (estimate.py:329-361), per config
            raws, keep = [], []
            for i in todo:
                try:
                    raws.append(self._annotated_raw(configs[i]))
                    keep.append(i)
                except Exception as exc:  # noqa: BLE001 - per-config INVALID, as the reference
                    out[i] = exc
            todo = keep
            if not todo:
                return out
            eng.load(raws, threads=self.threads)
        eng.run()
        res = eng.results()
        flops = {}
        failed = []
        for k, i in enumerate(todo):
            r = res[k]
            st_ = int(r["status"])
            if st_ != ST_OK:
                failed.append((k, i, st_))
                continue
            gb = configs[i].global_batch
            if gb not in flops:
                flops[gb] = iteration_flops(self.model, gb)
            mfu = _mfu(int(r["total_ns"]), bool(r["oom"]), flops[gb], self.cluster,
                       self.model.dtype)
            out[i] = T["EvalResult"](int(r["total_ns"]), mfu, int(r["peak_mem_bytes"]),
                                     bool(r["oom"]))
        for k, i, st_ in failed:      # error path: rebuild the reference's exception text
            raw = raws[k] if raws is not None else W.generate_job(
                self.model, configs[i], self.cluster, self.schedule, self.dispatch_overhead_ns)
            out[i] = _failure(st_, raw, self.device)
        return out

    def _annotated_raw(self, config) -> RawJob:
        """Host-estimator path.  With the reference importable (a TableEstimator
        or any dltsim estimator) the job comes from its own generate_representatives
        -> collate -> annotate (workload.py:571-780, collate.py:256, estimate.py:329),
        so KernelAttrs carry their dims and estimator errors their reference text;
        the simulation then runs on the device.  Without it, the native generator's
        features (no dims) feed annotate_raw."""
        ref = _reference_frontend(self.model)
        if ref is not None:
            wl, col, est_mod = ref
            sched = self.schedule or wl.default_schedule(config)
            traces, expansion = wl.generate_representatives(
                self.model, config, self.cluster, sched,
                dispatch_overhead_ns=self.dispatch_overhead_ns)
            job = col.collate(traces, expansion, self.cluster)
            return from_annotated(est_mod.annotate(job, self.estimator))
        raw = W.generate_job(self.model, config, self.cluster, self.schedule,
                             self.dispatch_overhead_ns)
        return annotate_raw(raw, self.estimator, self.cluster.device)

    def prefetch(self, configs: Sequence) -> None:
        for c, r in zip(configs, self.evaluate_many(configs)):
            self._cache[c.key()] = r

    def __call__(self, config):
        r = self._cache.get(config.key())
        if r is None:
            r = self.evaluate_many([config])[0]
        if isinstance(r, Exception):
            raise r
        return r


def _reference_frontend(model):
    """(dltsim.workload, dltsim.collate, dltsim.estimate) when `model` is the
    reference's own ModelSpec, else None."""
    if not type(model).__module__.startswith("dltsim"):
        return None
    import importlib
    try:   # submodules by name: the package re-exports functions of the same names
        wl, col, est_mod = (importlib.import_module(f"dltsim.{m}")
                            for m in ("workload", "collate", "estimate"))
    except Exception:
        return None
    return wl, col, est_mod


def annotate_raw(raw: RawJob, estimator, device) -> RawJob:
    """Host-computed durations for an arbitrary EstimatorInterface, one call per
    unique feature (the reference calls it once per event, estimate.py:339-352)."""
    from .rawtrace import EV_KERNEL, EV_MEMCPY, EV_MEMSET, COLLECTIVE_KINDS, TOPOLOGIES
    import dataclasses
    kc = np.isin(raw.ev_kind, (EV_KERNEL, EV_MEMCPY, EV_MEMSET))
    kn = np.full(raw.n_events, -1, dtype=np.int64)
    cache: dict = {}
    KernelAttrs = _kernel_attrs_type()
    for i in np.nonzero(kc)[0].tolist():
        op, dt, fl, by = (int(x) for x in raw.ev_f[i])
        key = (op, dt, fl, by)
        if key not in cache:
            attrs = KernelAttrs.make({}, raw.dtype_names[dt], fl, by)
            cache[key] = int(estimator.estimate_kernel(raw.op_kind_names[op], attrs, device))
        kn[i] = cache[key]
    wire = np.zeros(len(raw.call_kind), dtype=np.int64)
    for g in range(len(raw.comm_nranks)):
        for c in range(int(raw.call_off[g]), int(raw.call_off[g + 1])):
            if raw.call_kind[c] < 0:
                continue
            wire[c] = int(estimator.estimate_collective(
                COLLECTIVE_KINDS[raw.call_kind[c]], int(raw.call_bytes[c]),
                int(raw.comm_nranks[g]), TOPOLOGIES[raw.comm_topo[g]], device))
    return dataclasses.replace(raw, kernel_ns=kn, wire_ns=wire)


def _kernel_attrs_type():
    try:
        from dltsim.trace import KernelAttrs
        return KernelAttrs
    except Exception:
        @dataclass(frozen=True)
        class KernelAttrs:
            dims: tuple
            dtype: str
            flops: int
            bytes_moved: int

            @staticmethod
            def make(dims, dtype, flops, bytes_moved):
                return KernelAttrs(tuple(sorted(dict(dims).items())), dtype, flops, bytes_moved)
        return KernelAttrs


# --- whole-space search with the fused device reduction --------------------------------

@dataclass
class SpaceResult:
    configs: list
    results: list            # EvalResult or exception per config (enumeration order)
    best: list               # top-k configs in _rank order (search.py:349-357)
    best_time_ns: list


def key_ranks(configs) -> np.ndarray:
    order = sorted(range(len(configs)), key=lambda i: configs[i].key())
    kr = np.zeros(len(configs), dtype=np.int32)
    kr[order] = np.arange(len(configs), dtype=np.int32)
    return kr


def evaluate_space(space, model, cluster, k: int = 8, dispatch_overhead_ns: int = 0,
                   schedule=None, device: int = 0, threads: int = 8,
                   efficiency: Mapping[str, float] | None = None,
                   overhead_ns: int = DEFAULT_KERNEL_OVERHEAD_NS) -> SpaceResult:
    """Every valid config of ``space`` as one GPU batch; the k best by the
    reference ranking come from the fused device top-k."""
    T = _ref_types()
    configs = W.enumerate_space(space, model, cluster)
    eng = _engine(device)
    kr = key_ranks(configs)
    eng.stage_generated(model, configs, cluster, schedule=schedule,
                        dispatch_overhead_ns=dispatch_overhead_ns, efficiency=efficiency,
                        overhead_ns=overhead_ns, key_ranks=kr, threads=threads)
    eng.upload()
    eng.run()
    res = eng.results()
    top = eng.topk(k)
    fl = iteration_flops(model, configs[0].global_batch) if configs else 0
    results = []
    for c, r in zip(configs, res):
        if int(r["status"]) != ST_OK:
            results.append(RuntimeError(STATUS_NAMES[int(r["status"])]))
        else:
            results.append(T["EvalResult"](int(r["total_ns"]), _mfu(
                int(r["total_ns"]), bool(r["oom"]), fl, cluster, model.dtype),
                int(r["peak_mem_bytes"]), bool(r["oom"])))
    return SpaceResult(configs, results, [configs[int(t["job"])] for t in top],
                       [int(t["time_ns"]) for t in top])


class GenPipeline:
    """Double-buffered end-to-end evaluation of a config list: native
    generation + packing of chunk q+1 on the host threads overlaps the H2D,
    estimator, scheduler and top-k of chunk q on the device (two engines, each
    on its own stream).  Results come back in config order; the k best are the
    merge of the per-chunk device top-k under the reference ranking
    (search.py:349-357)."""

    def __init__(self, device: int = 0, chunks: int = 1):
        from .engine import Engine
        self.engines = [Engine(device), Engine(device)]
        self.chunks = max(1, int(chunks))

    def close(self) -> None:
        for e in self.engines:
            e.close()

    def evaluate(self, model, configs, cluster, k: int = 8, key_order=None,
                 dispatch_overhead_ns: int = 0, schedule=None, threads: int = 8,
                 efficiency: Mapping[str, float] | None = None,
                 overhead_ns: int = DEFAULT_KERNEL_OVERHEAD_NS):
        """-> (results structured array, top-k rows (time_ns, key_rank, config index))."""
        from ._abi import RESULT_DTYPE
        n = len(configs)
        kr = key_ranks(configs) if key_order is None else np.asarray(key_order)
        bounds = np.linspace(0, n, min(self.chunks, max(n, 1)) + 1).astype(int)
        res = np.zeros(n, dtype=RESULT_DTYPE)
        cands = []
        status = np.zeros(n, dtype=np.int32)

        def collect(item):
            e, lo, hi = item
            res[lo:hi] = e.results()
            for t in e.topk(k):
                cands.append((int(t["time_ns"]), int(t["key_rank"]), lo + int(t["job"])))

        pending = None
        for q in range(len(bounds) - 1):
            lo, hi = int(bounds[q]), int(bounds[q + 1])
            if hi <= lo:
                continue
            e = self.engines[q % 2]
            status[lo:hi] = e.stage_generated(model, configs[lo:hi], cluster, schedule=schedule,
                                              dispatch_overhead_ns=dispatch_overhead_ns,
                                              efficiency=efficiency, overhead_ns=overhead_ns,
                                              key_ranks=kr[lo:hi], threads=threads)
            e.upload()
            e.run()
            if pending is not None:
                collect(pending)
            pending = (e, lo, hi)
        if pending is not None:
            collect(pending)
        top = merge_topk(np.array(cands, dtype=np.int64).reshape(-1, 3), k)
        return res, top, status


    def evaluate_stream(self, model, batches, cluster, k: int = 8, key_orders=None,
                        dispatch_overhead_ns: int = 0, schedule=None, threads: int = 8,
                        efficiency: Mapping[str, float] | None = None,
                        overhead_ns: int = DEFAULT_KERNEL_OVERHEAD_NS):
        """Evaluate a stream of config batches (a search's successive
        populations), yielding (results, top-k rows, status) per batch in
        order.  Batch q+1 is generated and packed on the host threads while
        batch q's arena is assembled and uploaded (a helper thread) and its
        kernels and D2H run on the device (the two engines alternate), so a
        long search runs at the speed of the slowest stage instead of the sum.
        Every batch still goes through generation, H2D, the kernels, the D2H
        of its results and the top-k."""
        from ._abi import RESULT_DTYPE

        def collect(item):
            e, n, st = item
            res = np.zeros(n, dtype=RESULT_DTYPE)
            res[:] = e.results()
            top = merge_topk(np.array([(int(t["time_ns"]), int(t["key_rank"]), int(t["job"]))
                                       for t in e.topk(k)], dtype=np.int64).reshape(-1, 3), k)
            return res, top, st

        # Three stages overlap: the main thread generates + packs batch q (pool 0
        # of the native workers) while a helper thread assembles batch q-1's
        # arena (pool 1), uploads it and enqueues its run; the device runs
        # batch q-1 meanwhile.  An engine is restaged only after its previous
        # batch's results were read.
        from concurrent.futures import ThreadPoolExecutor

        def launch(e):
            e.upload()
            e.run()
            e.topk_async(k)                    # behind the run on its stream: no wait

        inflight = [None, None]                # per engine: (batch, future, n configs, status)
        with ThreadPoolExecutor(max_workers=1) as pool:
            for q, configs in enumerate(batches):
                e = self.engines[q % 2]
                if inflight[q % 2] is not None:   # batch q-2 on this engine: read it first
                    _, fut, n, st = inflight[q % 2]
                    fut.result()
                    inflight[q % 2] = None
                    yield collect((e, n, st))
                kr = (key_ranks(configs) if key_orders is None or key_orders[q] is None
                      else np.asarray(key_orders[q]))
                st = e.stage_generated(model, configs, cluster, schedule=schedule,
                                       dispatch_overhead_ns=dispatch_overhead_ns,
                                       efficiency=efficiency, overhead_ns=overhead_ns,
                                       key_ranks=kr, threads=threads)
                inflight[q % 2] = (q, pool.submit(launch, e), len(configs), st)
            for slot in sorted((0, 1), key=lambda x: inflight[x][0] if inflight[x] else -1):
                if inflight[slot] is not None:     # the last batches, in order
                    _, fut, n, st = inflight[slot]
                    fut.result()
                    inflight[slot] = None
                    yield collect((self.engines[slot], n, st))


def merge_topk(candidates: np.ndarray, k: int) -> np.ndarray:
    """Merge per-GPU top-k candidate rows (time_ns, global key rank, config id)
    with the device comparator; time_ns == 0 sorts after every positive time."""
    c = np.asarray(candidates, dtype=np.int64).reshape(-1, 3)
    c = c[c[:, 0] >= 0]
    t = np.where(c[:, 0] == 0, np.iinfo(np.int64).max, c[:, 0])
    order = np.lexsort((c[:, 2], c[:, 1], t))
    return c[order[:k]]


def shard_lpt(costs: Sequence[int], n: int) -> list:
    """Greedy LPT assignment of configs (by estimated cost) to n GPUs."""
    import heapq
    heap = [(0, g) for g in range(n)]
    heapq.heapify(heap)
    out = [[] for _ in range(n)]
    for i in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        load, g = heapq.heappop(heap)
        out[g].append(i)
        heapq.heappush(heap, (load + costs[i], g))
    return [sorted(x) for x in out]


def config_costs(configs) -> list:
    """LPT cost proxy of a config's simulation: pipeline steps per rank times
    stages (microbatches x virtual stages x pp)."""
    return [c.micro_mult * c.pp * c.pp * c.virtual_stages for c in configs]


def evaluate_sharded(model, configs, cluster, k: int = 8, engine=None, rank: int = 0,
                     world: int = 1, dispatch_overhead_ns: int = 0, schedule=None,
                     threads: int = 8, key_order=None):
    """ONE search's config list sharded over `world` processes (one per GPU):
    LPT on config_costs, the local fused device top-k, one all_gather of
    k x 24 B candidates (NCCL; gloo on CPU), and the same merge on every rank.
    Within one search (one cluster, one global batch) MFU is a decreasing
    function of time_ns, so the (time_ns, key rank) order of the merge is the
    reference ranking (search.py:349-357).
    -> (merged (k, 3) rows: time_ns, key rank, GLOBAL config index; my indices)"""
    kr = key_ranks(configs) if key_order is None else np.asarray(key_order, dtype=np.int32)
    mine = shard_lpt(config_costs(configs), world)[rank]
    eng = engine if engine is not None else _engine(0)
    cand = np.full((k, 3), -1, dtype=np.int64)
    if mine:
        sub = [configs[i] for i in mine]
        eng.stage_generated(model, sub, cluster, schedule=schedule,
                            dispatch_overhead_ns=dispatch_overhead_ns, key_ranks=kr[mine],
                            threads=threads)
        eng.upload()
        eng.run()
        for q, t in enumerate(eng.topk(k)):
            cand[q] = (int(t["time_ns"]), int(t["key_rank"]), mine[int(t["job"])])
    merged = gather_merge(cand, k) if world > 1 else merge_topk(cand, k)
    return merged, mine


def evaluate_space_distributed(space, model, cluster, k: int = 8, dispatch_overhead_ns: int = 0,
                               schedule=None, threads: int = 8, engine=None):
    """One process per GPU (torch.distributed): every valid config of `space`,
    sharded by evaluate_sharded.  -> (merged top-k rows, configs)"""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    configs = W.enumerate_space(space, model, cluster)
    if engine is None:
        engine = _engine(torch.cuda.current_device() if torch.cuda.is_available() else 0)
    merged, _ = evaluate_sharded(model, configs, cluster, k, engine, rank, world,
                                 dispatch_overhead_ns, schedule, threads)
    return merged, configs


def rank_by_mfu(rows, model, configs_of) -> list:
    """Merge candidates of DIFFERENT searches (global batches / clusters) the
    reference's way: (-mfu, time_ns, config.key()) (search.py:349-357), MFU by
    compute_mfu's arithmetic (sim.py:488-497).  rows: (time_ns, ..., cfg handle);
    configs_of(row) -> (config, cluster)."""
    out = []
    for row in rows:
        cfg, cl = configs_of(row)
        t = int(row[0])
        mfu = _mfu(t, False, iteration_flops(model, cfg.global_batch), cl, model.dtype)
        out.append((-mfu, t, cfg.key(), row))
    out.sort(key=lambda x: x[:3])
    return [(r, -m) for m, _, _, r in out]


def gather_merge(cand: np.ndarray, k: int) -> np.ndarray:
    """all_gather of the (k, 3) candidate block then the global merge; NCCL on
    GPUs, gloo on CPU (tests)."""
    import torch
    import torch.distributed as dist
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    t = torch.from_numpy(np.ascontiguousarray(cand)).to(dev)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    allc = torch.cat(parts).cpu().numpy()
    return merge_topk(allc, k)
