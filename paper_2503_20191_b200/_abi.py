"""ctypes mirror of include/maya_b200.h and the batch marshaller.

``Batch`` turns a list of RawJob into the C structs of the ABI, interning
op-kind and dtype strings batch-wide and building the device table and the
roofline efficiency table (exact fractions of ``str(eff)``, as
``RooflineEstimator._eff`` does at ``pkg/src/dltsim/estimate.py:114-115``).
"""

from __future__ import annotations

import ctypes as C
from fractions import Fraction
from typing import Mapping, Sequence

import numpy as np

from .rawtrace import EV_KERNEL, EV_MEMCPY, EV_MEMSET, RawJob

MAX_DTYPES = 16

ST_OK, ST_DEADLOCK, ST_INTERNAL, ST_ESTIMATION, ST_OVERFLOW, ST_BAD_INPUT = range(6)
STATUS_NAMES = ("ok", "deadlock", "internal", "estimation", "overflow", "bad_input")

# estimate.py:37-56
DEFAULT_KERNEL_OVERHEAD_NS = 1000
DEFAULT_EFFICIENCY = {
    "gemm": 0.6, "layernorm": 0.8, "softmax": 0.8, "gelu": 0.8, "add": 0.8,
    "embed": 0.8, "cross_entropy": 0.8, "optimizer_step": 0.8, "memcpy_h2d": 0.8,
    "memcpy_d2h": 0.8, "memcpy_d2d": 0.8, "memset": 0.8,
}
FALLBACK_EFFICIENCY = 0.5

P = C.POINTER


class DeviceParamsC(C.Structure):
    _fields_ = [("peak_flops", C.c_int64 * MAX_DTYPES), ("hbm_bytes_per_s", C.c_int64),
                ("alpha_ns", C.c_int64 * 2), ("beta_bytes_per_s", C.c_int64 * 2)]


class RooflineC(C.Structure):
    _fields_ = [("n_op_kinds", C.c_int32), ("eff_num", P(C.c_int64)),
                ("eff_den", P(C.c_int64)), ("overhead_ns", C.c_int64)]


class RawJobC(C.Structure):
    _fields_ = [
        ("num_ranks", C.c_int32), ("devices_per_host", C.c_int32), ("capacity", C.c_int64),
        ("device", C.c_int32), ("n_reps", C.c_int32),
        ("rank_rep", P(C.c_int32)), ("ev_off", P(C.c_int64)), ("ev_kind", P(C.c_uint8)),
        ("ev_stream", P(C.c_int32)), ("ev_f", P(C.c_int64)),
        ("n_comms", C.c_int32), ("comm_nranks", P(C.c_int32)), ("comm_topo", P(C.c_int8)),
        ("call_off", P(C.c_int64)), ("call_kind", P(C.c_int8)), ("call_bytes", P(C.c_int64)),
        ("rank_comm_off", P(C.c_int64)), ("rank_comm", P(C.c_int32)),
        ("kernel_ns", P(C.c_int64)), ("wire_ns", P(C.c_int64)),
    ]


class JobResultC(C.Structure):
    _fields_ = [("total_ns", C.c_int64), ("peak_mem_bytes", C.c_int64), ("oom", C.c_int32),
                ("status", C.c_int32), ("first_oom_rank", C.c_int32),
                ("first_oom_seq", C.c_int32), ("dispatched_ops", C.c_int64),
                ("completed_ops", C.c_int64), ("rank_ops", C.c_int64), ("rounds", C.c_int64)]


class TopkEntryC(C.Structure):
    _fields_ = [("time_ns", C.c_int64), ("key_rank", C.c_int32), ("job", C.c_int32)]


RESULT_DTYPE = np.dtype([("total_ns", "<i8"), ("peak_mem_bytes", "<i8"), ("oom", "<i4"),
                         ("status", "<i4"), ("first_oom_rank", "<i4"), ("first_oom_seq", "<i4"),
                         ("dispatched_ops", "<i8"), ("completed_ops", "<i8"),
                         ("rank_ops", "<i8"), ("rounds", "<i8")])
assert RESULT_DTYPE.itemsize == C.sizeof(JobResultC)

TOPK_DTYPE = np.dtype([("time_ns", "<i8"), ("key_rank", "<i4"), ("job", "<i4")])
assert TOPK_DTYPE.itemsize == C.sizeof(TopkEntryC)


def _ptr(a: np.ndarray | None, ctype):
    if a is None:
        return C.cast(None, P(ctype))
    assert a.flags.c_contiguous
    return a.ctypes.data_as(P(ctype))


def efficiency_fraction(value) -> Fraction:
    return Fraction(str(value))


class Batch:
    """Marshal RawJobs for one ABI call; keeps every array alive."""

    def __init__(self, jobs: Sequence[RawJob], efficiency: Mapping[str, float] | None = None,
                 overhead_ns: int = DEFAULT_KERNEL_OVERHEAD_NS):
        self.jobs = list(jobs)
        self.efficiency = dict(DEFAULT_EFFICIENCY if efficiency is None else efficiency)
        self.overhead_ns = int(overhead_ns)
        self.op_kinds: list[str] = []
        self.dtypes: list[str] = []
        self._op_id: dict[str, int] = {}
        self._dt_id: dict[str, int] = {}
        self._keep: list = []
        self.devices: list = []
        # generated jobs use fixed id tables (csrc/gen.cpp): intern them first
        from .workload import GEN_DTYPES, GEN_OP_KINDS
        self._intern(GEN_OP_KINDS, self.op_kinds, self._op_id)
        self._intern(GEN_DTYPES, self.dtypes, self._dt_id)
        self._dev_id: dict = {}
        self.c_jobs = (RawJobC * len(self.jobs))()
        for i, job in enumerate(self.jobs):
            self._fill(i, job)
        self.c_devices = (DeviceParamsC * max(1, len(self.devices)))()
        for i, dev in enumerate(self.devices):
            self._fill_device(self.c_devices[i], dev)
        n = len(self.op_kinds)
        self.eff_num = np.ones(max(1, n), dtype=np.int64)
        self.eff_den = np.ones(max(1, n), dtype=np.int64)
        for k, name in enumerate(self.op_kinds):
            fr = efficiency_fraction(self.efficiency.get(name, FALLBACK_EFFICIENCY))
            if fr <= 0:
                raise ValueError(f"non-positive efficiency for {name!r}")
            if fr.numerator >= 1 << 63 or fr.denominator >= 1 << 63:
                raise OverflowError(f"efficiency fraction of {name!r} exceeds int64")
            self.eff_num[k] = fr.numerator
            self.eff_den[k] = fr.denominator
        self.c_roof = RooflineC(n, _ptr(self.eff_num, C.c_int64), _ptr(self.eff_den, C.c_int64),
                                self.overhead_ns)

    def _intern(self, names, table, ids):
        out = np.empty(len(names), dtype=np.int64)
        for i, n in enumerate(names):
            if n not in ids:
                ids[n] = len(table)
                table.append(n)
            out[i] = ids[n]
        return out

    def _fill(self, i: int, job: RawJob) -> None:
        opmap = self._intern(job.op_kind_names, self.op_kinds, self._op_id)
        dtmap = self._intern(job.dtype_names, self.dtypes, self._dt_id)
        if len(self.dtypes) > MAX_DTYPES:
            raise ValueError(f"more than {MAX_DTYPES} dtypes in one batch")
        ev_f = job.ev_f
        kc = np.isin(job.ev_kind, (EV_KERNEL, EV_MEMCPY, EV_MEMSET))
        if kc.any() and (not np.array_equal(opmap, np.arange(len(opmap)))
                         or not np.array_equal(dtmap, np.arange(len(dtmap)))):
            ev_f = ev_f.copy()
            ev_f[kc, 0] = opmap[ev_f[kc, 0]]
            ev_f[kc, 1] = dtmap[ev_f[kc, 1]]
        ev_f = np.ascontiguousarray(ev_f, dtype=np.int64)
        dkey = (job.device.name, tuple(sorted(job.device.peak_flops.items())),
                job.device.hbm_bytes_per_s, job.device.intra_alpha_ns, job.device.intra_beta,
                job.device.inter_alpha_ns, job.device.inter_beta)
        if dkey not in self._dev_id:
            self._dev_id[dkey] = len(self.devices)
            self.devices.append(job.device)
        arrs = dict(
            rank_rep=np.ascontiguousarray(job.rank_rep, dtype=np.int32),
            ev_off=np.ascontiguousarray(job.ev_off, dtype=np.int64),
            ev_kind=np.ascontiguousarray(job.ev_kind, dtype=np.uint8),
            ev_stream=np.ascontiguousarray(job.ev_stream, dtype=np.int32),
            ev_f=ev_f,
            comm_nranks=np.ascontiguousarray(job.comm_nranks, dtype=np.int32),
            comm_topo=np.ascontiguousarray(job.comm_topo, dtype=np.int8),
            call_off=np.ascontiguousarray(job.call_off, dtype=np.int64),
            call_kind=np.ascontiguousarray(job.call_kind, dtype=np.int8),
            call_bytes=np.ascontiguousarray(job.call_bytes, dtype=np.int64),
            rank_comm_off=np.ascontiguousarray(job.rank_comm_off, dtype=np.int64),
            rank_comm=np.ascontiguousarray(job.rank_comm, dtype=np.int32),
            kernel_ns=None if job.kernel_ns is None else np.ascontiguousarray(job.kernel_ns,
                                                                               dtype=np.int64),
            wire_ns=None if job.wire_ns is None else np.ascontiguousarray(job.wire_ns,
                                                                           dtype=np.int64),
        )
        self._keep.append(arrs)
        c = self.c_jobs[i]
        c.num_ranks = job.num_ranks
        c.devices_per_host = job.devices_per_host
        c.capacity = job.capacity
        c.device = self._dev_id[dkey]
        c.n_reps = job.n_reps
        c.n_comms = len(job.comm_nranks)
        types = dict(rank_rep=C.c_int32, ev_off=C.c_int64, ev_kind=C.c_uint8,
                     ev_stream=C.c_int32, ev_f=C.c_int64, comm_nranks=C.c_int32,
                     comm_topo=C.c_int8, call_off=C.c_int64, call_kind=C.c_int8,
                     call_bytes=C.c_int64, rank_comm_off=C.c_int64, rank_comm=C.c_int32,
                     kernel_ns=C.c_int64, wire_ns=C.c_int64)
        for name, ct in types.items():
            setattr(c, name, _ptr(arrs[name], ct))

    def _fill_device(self, c: DeviceParamsC, dev) -> None:
        for name, peak in dev.peak_flops.items():
            if name in self._dt_id:
                c.peak_flops[self._dt_id[name]] = int(peak)
        c.hbm_bytes_per_s = dev.hbm_bytes_per_s
        c.alpha_ns[0] = dev.intra_alpha_ns
        c.alpha_ns[1] = dev.inter_alpha_ns
        c.beta_bytes_per_s[0] = dev.intra_beta
        c.beta_bytes_per_s[1] = dev.inter_beta

    def device_of(self, i: int) -> DeviceParamsC:
        return self.c_devices[self.c_jobs[i].device]

    def unknown_op_kinds(self) -> list[str]:
        return sorted(k for k in self.op_kinds if k not in self.efficiency)
