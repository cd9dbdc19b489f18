"""ORACLE — test infrastructure only (never imported by the product path).

ctypes wrapper over oracle/_build/liboracle.so, the C++ restatement of the
reference's event-driven simulator (pkg/src/dltsim/sim.py) and estimators
(pkg/src/dltsim/estimate.py).  Pinned against the reference itself through
the golden fixtures under tests/golden/ (tests/test_oracle_golden.py).

Allowed importers: tests/, __graft_entry__.smoke(), and bench.py's
cpu_baseline / --impl reference legs.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Mapping, Sequence

import numpy as np

from paper_2503_20191_b200._abi import (Batch, DeviceParamsC, JobResultC, RawJobC, RooflineC,
                                        RESULT_DTYPE, DEFAULT_KERNEL_OVERHEAD_NS)
from paper_2503_20191_b200.rawtrace import RawJob

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        P = C.POINTER
        L.oracle_simulate.argtypes = [
            P(RawJobC), P(DeviceParamsC), P(RooflineC), P(JobResultC), P(C.c_int64),
            P(C.c_int32), P(C.c_int32), P(C.c_int64), P(C.c_int64), P(C.c_int64),
            P(C.c_int32), P(C.c_int64), C.c_char_p, C.c_int32]
        L.oracle_simulate_many.argtypes = [C.c_int32, P(RawJobC), P(DeviceParamsC), P(RooflineC),
                                           P(JobResultC), C.c_int32]
        L.oracle_annotate.argtypes = [P(RawJobC), P(DeviceParamsC), P(RooflineC), P(C.c_int64),
                                      P(C.c_int64), P(C.c_int64), P(C.c_int64)]
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def simulate(job: RawJob, efficiency: Mapping[str, float] | None = None,
             overhead_ns: int = DEFAULT_KERNEL_OVERHEAD_NS, timeline: bool = False) -> dict:
    """annotate + simulate one job on the CPU oracle."""
    b = Batch([job], efficiency, overhead_ns)
    L = lib()
    res = JobResultC()
    R = job.num_ranks
    stats = np.zeros((R, 5), dtype=np.int64)
    n_tl = C.c_int64(0)
    msg = C.create_string_buffer(4096)
    cap = job.rank_ops() + 1
    tl = None
    if timeline:
        tl = dict(rank=np.zeros(cap, np.int32), stream=np.zeros(cap, np.int32),
                  seq=np.zeros(cap, np.int64), start=np.zeros(cap, np.int64),
                  end=np.zeros(cap, np.int64), cls=np.zeros(cap, np.int32))
        args = (_p(tl["rank"], C.c_int32), _p(tl["stream"], C.c_int32), _p(tl["seq"], C.c_int64),
                _p(tl["start"], C.c_int64), _p(tl["end"], C.c_int64), _p(tl["cls"], C.c_int32))
    else:
        args = (None,) * 6
    L.oracle_simulate(C.byref(b.c_jobs[0]), C.byref(b.device_of(0)), C.byref(b.c_roof),
                      C.byref(res), _p(stats, C.c_int64), *args, C.byref(n_tl), msg, 4096)
    out = {name: getattr(res, name) for name, _ in JobResultC._fields_}
    out["rank_stats"] = stats
    out["message"] = msg.value.decode()
    out["op_kinds"] = list(b.op_kinds)
    if timeline:
        n = n_tl.value
        out["timeline"] = {k: v[:n].copy() for k, v in tl.items()}
    return out


def annotate(job: RawJob, efficiency: Mapping[str, float] | None = None,
             overhead_ns: int = DEFAULT_KERNEL_OVERHEAD_NS):
    """(status, kernel_ns[E], wire[n_calls]) from the oracle estimators."""
    b = Batch([job], efficiency, overhead_ns)
    E = job.n_events
    kn = np.zeros(max(E, 1), dtype=np.int64)
    wn = np.zeros(max(int(job.call_off[-1]), 1), dtype=np.int64)
    er, es = C.c_int64(), C.c_int64()
    st = lib().oracle_annotate(C.byref(b.c_jobs[0]), C.byref(b.device_of(0)), C.byref(b.c_roof),
                               _p(kn, C.c_int64), _p(wn, C.c_int64), C.byref(er), C.byref(es))
    return st, kn[:E], wn[:int(job.call_off[-1])]


def simulate_many(jobs: Sequence[RawJob], efficiency: Mapping[str, float] | None = None,
                  overhead_ns: int = DEFAULT_KERNEL_OVERHEAD_NS, threads: int = 1,
                  batch: Batch | None = None) -> np.ndarray:
    b = batch if batch is not None else Batch(jobs, efficiency, overhead_ns)
    out = np.zeros(len(b.jobs), dtype=RESULT_DTYPE)
    lib().oracle_simulate_many(len(b.jobs), b.c_jobs, b.c_devices, C.byref(b.c_roof),
                               out.ctypes.data_as(C.POINTER(JobResultC)), int(threads))
    return out
