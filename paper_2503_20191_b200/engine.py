"""Python handle on the CUDA engine (libmaya_b200.so, C ABI in include/maya_b200.h).

There is no CPU fallback: if the extension is missing or no CUDA device is
usable, construction raises.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np

from ._abi import (Batch, DeviceParamsC, JobResultC, RawJobC, RooflineC, TopkEntryC,
                   RESULT_DTYPE, TOPK_DTYPE, DEFAULT_KERNEL_OVERHEAD_NS)
from .rawtrace import RawJob
from .workload import ConfigC

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MAYA_LIB_PATH") or os.path.join(_HERE, "libmaya_b200.so")
_lib = None

EXPORTED = (
    "maya_last_error", "maya_abi_version", "maya_open", "maya_close", "maya_batch_reset",
    "maya_batch_set_devices", "maya_batch_set_roofline", "maya_batch_add_job",
    "maya_batch_add_jobs", "maya_batch_num_jobs", "maya_upload", "maya_run", "maya_results",
    "maya_topk", "maya_timeline_size", "maya_timeline", "maya_last_timings",
    "maya_get_stream", "maya_arena_bytes", "maya_gen_job", "maya_gen_view_of", "maya_gen_free",
    "maya_gen_op_kind_name", "maya_gen_dtype_name", "maya_batch_add_generated",
    "maya_batch_stats", "maya_set_options", "maya_batch_collapsed", "maya_batch_kernels",
    "maya_prof_read",
    "maya_debug_pack_compare", "maya_rank_stats", "maya_last_error_kind", "maya_trace_parse",
    "maya_trace_info", "maya_trace_serialize", "maya_trace_free", "maya_job_load",
    "maya_job_save", "maya_gen_names", "maya_topk_async",
)


SCHEDS = ("auto", "nochain", "lane", "warp")


class EngineError(RuntimeError):
    pass


def lib():
    """Load the in-tree extension; raise loudly if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise EngineError(f"CUDA extension {LIB_PATH} is missing: run `python __graft_entry__.py` "
                          f"(build) or `make -C paper_2503_20191_b200/csrc`")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp = C.c_void_p
    L.maya_last_error.restype = C.c_char_p
    L.maya_open.argtypes = [C.c_int, P(vp)]
    L.maya_close.argtypes = [vp]
    L.maya_batch_reset.argtypes = [vp]
    L.maya_batch_set_devices.argtypes = [vp, C.c_int32, P(DeviceParamsC)]
    L.maya_batch_set_roofline.argtypes = [vp, P(RooflineC)]
    L.maya_batch_add_job.argtypes = [vp, P(RawJobC), C.c_int32]
    L.maya_batch_add_jobs.argtypes = [vp, C.c_int32, P(RawJobC), P(C.c_int32), C.c_int32]
    L.maya_batch_num_jobs.argtypes = [vp]
    L.maya_upload.argtypes = [vp]
    L.maya_run.argtypes = [vp, C.c_int32]
    L.maya_results.argtypes = [vp, P(JobResultC)]
    L.maya_topk.argtypes = [vp, C.c_int32, P(TopkEntryC), P(C.c_int32)]
    L.maya_timeline_size.argtypes = [vp, C.c_int32, P(C.c_int64)]
    L.maya_timeline.argtypes = [vp, C.c_int32, P(C.c_int32), P(C.c_int32), P(C.c_int32),
                                P(C.c_int64), P(C.c_int64)]
    L.maya_last_timings.argtypes = [vp, P(C.c_float)]
    L.maya_get_stream.argtypes = [vp, P(vp)]
    L.maya_arena_bytes.argtypes = [vp]
    L.maya_arena_bytes.restype = C.c_int64
    L.maya_batch_stats.argtypes = [vp, P(C.c_int64)]
    L.maya_set_options.argtypes = [vp, C.c_int32]
    L.maya_batch_collapsed.argtypes = [vp, P(C.c_uint8)]
    L.maya_batch_kernels.argtypes = [vp, P(C.c_int32)]
    L.maya_rank_stats.argtypes = [vp, C.c_int32, C.c_int32, P(C.c_int64)]
    L.maya_topk_async.argtypes = [vp, C.c_int32]
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc != 0:
        raise EngineError(f"maya error {rc}: {lib().maya_last_error().decode()}")


@dataclass
class Timeline:
    rank: np.ndarray
    stream: np.ndarray
    seq: np.ndarray
    tag: np.ndarray       # 0 kernel-class, 1 collective, 2 record, 3 wait
    start: np.ndarray
    end: np.ndarray

    def timed(self) -> "Timeline":
        """Only the ops the reference records (kernels and collectives, sim.py:375)."""
        m = self.tag <= 1
        return Timeline(self.rank[m], self.stream[m], self.seq[m], self.tag[m], self.start[m],
                        self.end[m])


_GEN_BATCHES: dict = {}


def _generated_batch(device, efficiency, overhead_ns) -> Batch:
    """The estimator tables and device record of a generated batch (read-only
    once built: the native calls copy them), shared by every batch with the
    same device class, efficiency table and kernel overhead."""
    from .rawtrace import DeviceParams
    # keyed by the device object's identity (the entry keeps it alive, so the
    # id cannot be reused while cached) and its rates (a frozen dataclass whose
    # peak_flops mapping could still be edited), and the efficiency table
    try:
        key = (id(device), tuple(sorted(getattr(device, "peak_flops", {}).items())),
               getattr(device, "hbm_bytes_per_s", None),
               None if efficiency is None else tuple(sorted(efficiency.items())), int(overhead_ns))
        hash(key)
    except TypeError:
        key = None
    hit = _GEN_BATCHES.get(key) if key is not None else None
    if hit is not None and hit[0] is device:
        return hit[1]
    b = Batch([], efficiency, overhead_ns)
    b.devices.append(DeviceParams.from_reference(device))
    b.c_devices = (DeviceParamsC * 1)()
    b._fill_device(b.c_devices[0], b.devices[0])
    if key is not None:
        if len(_GEN_BATCHES) > 64:
            _GEN_BATCHES.clear()
        _GEN_BATCHES[key] = (device, b)
    return b


class Engine:
    """One engine per CUDA device (C ABI: maya_open ... maya_close)."""

    def __init__(self, device: int = 0, collapse: bool = True, sched: str = "auto",
                 fold: bool = True, blocks: bool = True):
        L = lib()
        self._h = C.c_void_p()
        _check(L.maya_open(int(device), C.byref(self._h)))
        if sched not in SCHEDS:
            raise ValueError(f"sched must be one of {SCHEDS}, not {sched!r}")
        self._collapse = bool(collapse)
        self._sched = sched
        self._fold = bool(fold)
        self._blocks = bool(blocks)
        self._apply_options()
        self.device = device
        self.batch: Batch | None = None
        self.n_jobs = 0

    def set_collapse(self, on: bool) -> None:
        """Exact rank-class collapse of deduplicated jobs."""
        self._collapse = bool(on)
        self._apply_options()

    def set_sched(self, sched: str) -> None:
        """Scheduler kernel: 'auto' (per job, default: the chain kernel where the
        job fits it, else lane-parallel or warp-window by the shape of its
        FIFOs), 'nochain' (auto without the chain kernel), 'lane' (lane-parallel
        wherever it fits) or 'warp' (warp-window for every job)."""
        if sched not in SCHEDS:
            raise ValueError(f"sched must be one of {SCHEDS}, not {sched!r}")
        self._sched = sched
        self._apply_options()

    def set_blocks(self, on: bool) -> None:
        """Generated jobs carry interned kernel blocks (runs of launches of one
        stream, folded on the device).  Off: one op per launch, which a
        timeline recording of generated jobs needs."""
        self._blocks = bool(on)
        self._apply_options()

    def _apply_options(self) -> None:
        opts = ((1 if self._collapse else 0) | (2 if self._sched == "warp" else 0)
                | (4 if self._sched == "lane" else 0) | (0 if self._fold else 8)
                | (16 if not (self._blocks and self._fold) else 0)
                | (32 if self._sched == "nochain" else 0))
        _check(lib().maya_set_options(self._h, opts))

    KERNELS = ("warp", "lane", "grid", "chain")

    def kernels(self) -> list:
        """Scheduler kernel of each staged job (after upload): 'warp'
        (warp-window), 'lane' (lane-parallel), 'grid' (multi-CTA lane job) or
        'chain' (latency-bound job resident in one CTA's shared memory)."""
        out = np.zeros(max(self.n_jobs, 1), dtype=np.int32)
        _check(lib().maya_batch_kernels(self._h, out.ctypes.data_as(C.POINTER(C.c_int32))))
        return [self.KERNELS[int(v)] for v in out[:self.n_jobs]]

    def collapsed(self) -> np.ndarray:
        out = np.zeros(max(self.n_jobs, 1), dtype=np.uint8)
        _check(lib().maya_batch_collapsed(self._h, out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out[:self.n_jobs].astype(bool)

    def close(self) -> None:
        if self._h:
            lib().maya_close(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- batch ------------------------------------------------------------------

    def load(self, jobs: Sequence[RawJob] | Batch, efficiency: Mapping[str, float] | None = None,
             overhead_ns: int = DEFAULT_KERNEL_OVERHEAD_NS,
             key_ranks: Sequence[int] | None = None, threads: int = 8) -> None:
        """Pack jobs (host, multi-threaded) and upload them to HBM."""
        b = jobs if isinstance(jobs, Batch) else Batch(jobs, efficiency, overhead_ns)
        self.stage(b, key_ranks, threads)
        self.upload()

    def stage(self, b: Batch, key_ranks: Sequence[int] | None = None, threads: int = 8) -> None:
        L = lib()
        self.batch = b
        n = len(b.jobs)
        _check(L.maya_batch_reset(self._h))
        _check(L.maya_batch_set_devices(self._h, len(b.devices), b.c_devices))
        _check(L.maya_batch_set_roofline(self._h, C.byref(b.c_roof)))
        kr = (np.arange(n, dtype=np.int32) if key_ranks is None
              else np.ascontiguousarray(key_ranks, dtype=np.int32))
        _check(L.maya_batch_add_jobs(self._h, n, b.c_jobs, kr.ctypes.data_as(C.POINTER(C.c_int32)),
                                     int(threads)))
        self.n_jobs = n

    def upload(self) -> None:
        _check(lib().maya_upload(self._h))

    def run(self, record_timeline: bool = False) -> None:
        _check(lib().maya_run(self._h, 1 if record_timeline else 0))

    def results(self) -> np.ndarray:
        out = np.zeros(self.n_jobs, dtype=RESULT_DTYPE)
        _check(lib().maya_results(self._h, out.ctypes.data_as(C.POINTER(JobResultC))))
        return out

    def simulate(self, jobs: Sequence[RawJob] | Batch, record_timeline: bool = False,
                 **kw) -> np.ndarray:
        self.load(jobs, **kw)
        self.run(record_timeline)
        return self.results()

    def topk(self, k: int) -> np.ndarray:
        out = np.zeros(k, dtype=TOPK_DTYPE)
        n = C.c_int32()
        _check(lib().maya_topk(self._h, int(k), out.ctypes.data_as(C.POINTER(TopkEntryC)),
                               C.byref(n)))
        return out[:n.value]

    def timeline(self, job: int) -> Timeline:
        L = lib()
        n = C.c_int64()
        _check(L.maya_timeline_size(self._h, int(job), C.byref(n)))
        n = n.value
        rank = np.zeros(max(n, 1), np.int32)
        stream = np.zeros(max(n, 1), np.int32)
        seq = np.zeros(max(n, 1), np.int32)
        start = np.zeros(max(n, 1), np.int64)
        end = np.zeros(max(n, 1), np.int64)
        P = C.POINTER
        _check(L.maya_timeline(self._h, int(job), rank.ctypes.data_as(P(C.c_int32)),
                               stream.ctypes.data_as(P(C.c_int32)),
                               seq.ctypes.data_as(P(C.c_int32)),
                               start.ctypes.data_as(P(C.c_int64)),
                               end.ctypes.data_as(P(C.c_int64))))
        return Timeline(rank[:n], stream[:n], seq[:n] >> 2, seq[:n] & 3, start[:n], end[:n])

    def topk_async(self, k: int) -> None:
        """Enqueue the top-k after the last run; the next topk(k) returns it."""
        _check(lib().maya_topk_async(self._h, int(k)))

    def rank_stats(self, job: int, num_ranks: int) -> np.ndarray:
        """Per-rank (compute_busy, comm_busy, exposed_comm, idle, peak_mem) of one
        job, computed on the device after run(record_timeline=True)."""
        out = np.zeros((max(num_ranks, 1), 5), np.int64)
        _check(lib().maya_rank_stats(self._h, int(job), int(num_ranks),
                                     out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out[:num_ranks]

    def stream_handle(self) -> int:
        s = C.c_void_p()
        _check(lib().maya_get_stream(self._h, C.byref(s)))
        return s.value or 0

    def batch_stats(self) -> dict:
        o = (C.c_int64 * 16)()
        _check(lib().maya_batch_stats(self._h, o))
        keys = ("jobs", "rep_events", "rank_comms", "features", "slots", "device_ops",
                "rank_ops", "arena_bytes", "ranks", "reps", "run_launches", "topk_launches",
                "kernel_blocks", "block_fids", "wire_features", "class_ops")
        return {k: int(v) for k, v in zip(keys, o)}

    def arena_bytes(self) -> int:
        return int(lib().maya_arena_bytes(self._h))

    def stage_generated(self, model, configs, cluster, schedule=None,
                        dispatch_overhead_ns: int = 5000, efficiency=None,
                        overhead_ns: int = DEFAULT_KERNEL_OVERHEAD_NS,
                        key_ranks=None, threads: int = 8) -> np.ndarray:
        """Generate + pack configs natively into the batch (no RawJob round trip).
        Returns per-config generation status (0 ok, <0 invalid config)."""
        from .workload import _gen_lib, cluster_c, configs_array, model_c, schedule_code
        L = _gen_lib()
        b = _generated_batch(cluster.device, efficiency, overhead_ns)
        self.batch = b
        n = len(configs)
        _check(L.maya_batch_reset(self._h))
        _check(L.maya_batch_set_devices(self._h, 1, b.c_devices))
        _check(L.maya_batch_set_roofline(self._h, C.byref(b.c_roof)))
        cfgs_np = configs_array(configs)
        cfgs = cfgs_np.ctypes.data_as(C.POINTER(ConfigC))
        kr = (np.arange(n, dtype=np.int32) if key_ranks is None
              else np.ascontiguousarray(key_ranks, dtype=np.int32))
        st = np.zeros(max(n, 1), dtype=np.int32)
        P = C.POINTER
        _check(L.maya_batch_add_generated(
            self._h, C.byref(model_c(model)), n, cfgs, C.byref(cluster_c(cluster)), 0,
            schedule_code(schedule), int(dispatch_overhead_ns),
            kr.ctypes.data_as(P(C.c_int32)), int(threads), st.ctypes.data_as(P(C.c_int32))))
        self.n_jobs = n
        return st[:n]

    def last_timings_ms(self) -> tuple[float, float, float]:
        t = (C.c_float * 3)()
        _check(lib().maya_last_timings(self._h, t))
        return tuple(t)
