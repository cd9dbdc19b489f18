"""RawJob: the collated job trace as flat integer arrays.

This is the host-side interchange between the reference schema and the
engine.  It restates, as arrays, exactly the fields ``simulate()`` reads from
an ``AnnotatedJob`` (reference ``pkg/src/dltsim/estimate.py:314-326``) and its
``JobTrace`` (``pkg/src/dltsim/collate.py:215-253``):

* one event list per representative worker (``JobTrace.reps``), each event a
  ``kind`` code, a ``stream`` and four int64 payload fields (the dataclass
  fields of ``pkg/src/dltsim/trace.py:71-151``, see ``EV_*`` below);
* ``rank_rep``: representative of every rank (``JobTrace.rep_of``,
  ``collate.py:234-235``);
* ``rank_comm``: per rank, the global communicator of each CommInit of its
  representative, in trace order (``JobTrace.comm_map``, ``collate.py:223``,
  consumed by ``_compile_rank`` at ``sim.py:159-161``);
* communicator table (``JobTrace.groups``: nranks and topology class) and the
  call table (``JobTrace.calls``: kind and bytes per ``(comm, call_idx)``);
* optional host-computed annotations ``kernel_ns`` (per event) and
  ``wire_ns`` (per call) for estimators other than the roofline.

Event payload layout (``f`` is int64[E, 4]):

============  ===================  =========================================
kind          stream               f0, f1, f2, f3
============  ===================  =========================================
HOSTGAP       0                    duration_ns
KERNEL        stream               op_kind id, dtype id, flops, bytes_moved
MEMALLOC      0                    alloc_id, bytes
MEMFREE       0                    alloc_id
MEMCPY        stream               op_kind id (memcpy_<dir>), dtype id (fp32), 0, bytes
MEMSET        stream               op_kind id (memset), dtype id (fp32), 0, bytes
RECORD        stream               event_id, version
WAIT          stream               event_id, version
ESYNC         0                    event_id, version
SSYNC         stream               -
DSYNC         0                    -
COMMINIT      0                    local comm index, nranks, my_rank
COLLECTIVE    stream               local comm index, call_idx, kind id, bytes
============  ===================  =========================================

The Memcpy/Memset rows carry the ``kernel_view`` mapping of
``estimate.py:300-311`` already applied, so every kernel-class event has the
same (op_kind, dtype, flops, bytes) feature.  "local comm index" is the
position of the comm id among the representative's CommInit events.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np

# Event kind codes (order of trace.EVENT_KINDS, pkg/src/dltsim/trace.py:160-174).
EV_HOSTGAP, EV_KERNEL, EV_MEMALLOC, EV_MEMFREE, EV_MEMCPY, EV_MEMSET, \
    EV_RECORD, EV_WAIT, EV_ESYNC, EV_SSYNC, EV_DSYNC, EV_COMMINIT, \
    EV_COLLECTIVE = range(13)

EVENT_CLASS_NAMES = (
    "HostGap", "KernelLaunch", "MemAlloc", "MemFree", "Memcpy", "Memset",
    "EventRecord", "StreamWaitEvent", "EventSynchronize", "StreamSynchronize",
    "DeviceSynchronize", "CommInit", "Collective",
)
_KIND_OF_CLASS = {name: i for i, name in enumerate(EVENT_CLASS_NAMES)}

# trace.py:42 and cluster.py:19-23
COLLECTIVE_KINDS = ("AllReduce", "AllGather", "ReduceScatter", "Broadcast", "SendRecv")
TOPOLOGIES = ("intra_host", "inter_host", "mixed")
MEMCPY_OP_KINDS = {"H2D": "memcpy_h2d", "D2H": "memcpy_d2h", "D2D": "memcpy_d2d"}

INT64_MAX = (1 << 63) - 1


def _i64(v: int, what: str) -> int:
    if not (-(1 << 63) <= v <= INT64_MAX):
        raise OverflowError(f"{what} = {v} does not fit in int64")
    return v


@dataclass(frozen=True)
class DeviceParams:
    """Integer performance envelope of a DeviceClass (cluster.py:39-59)."""

    name: str
    peak_flops: Mapping[str, int]
    hbm_bytes_per_s: int
    intra_alpha_ns: int
    intra_beta: int
    inter_alpha_ns: int
    inter_beta: int

    @staticmethod
    def from_reference(dev) -> "DeviceParams":
        intra, inter = dev.links["intra_host"], dev.links["inter_host"]
        return DeviceParams(str(dev.name), dict(dev.peak_flops), int(dev.hbm_bytes_per_s),
                            int(intra.alpha_ns), int(intra.beta_bytes_per_s),
                            int(inter.alpha_ns), int(inter.beta_bytes_per_s))


@dataclass
class RawJob:
    num_hosts: int
    devices_per_host: int
    capacity: int                      # device_memory_bytes used for OOM
    device: DeviceParams
    rep_ranks: np.ndarray              # int64[n_reps] global rank of each representative
    rank_rep: np.ndarray               # int32[R] representative index of each rank
    ev_off: np.ndarray                 # int64[n_reps + 1]
    ev_kind: np.ndarray                # uint8[E]
    ev_stream: np.ndarray              # int32[E]
    ev_f: np.ndarray                   # int64[E, 4]
    op_kind_names: list                # op kind strings (KERNEL/MEMCPY/MEMSET f0)
    dtype_names: list                  # dtype strings (f1)
    comm_names: list                   # global communicator ids, sorted
    comm_nranks: np.ndarray            # int32[G]
    comm_topo: np.ndarray              # int8[G] index into TOPOLOGIES
    call_off: np.ndarray               # int64[G + 1]; call (g, idx) -> call_off[g] + idx
    call_kind: np.ndarray              # int8[n_calls] index into COLLECTIVE_KINDS, -1 = unused
    call_bytes: np.ndarray             # int64[n_calls]
    rank_comm_off: np.ndarray          # int64[R + 1]
    rank_comm: np.ndarray              # int32[...] global comm of each rep CommInit
    kernel_ns: np.ndarray | None = None    # int64[E] host annotations, -1 elsewhere
    wire_ns: np.ndarray | None = None      # int64[n_calls]
    name: str = ""

    @property
    def num_ranks(self) -> int:
        return int(self.rank_rep.shape[0])

    @property
    def n_reps(self) -> int:
        return int(self.rep_ranks.shape[0])

    @property
    def n_events(self) -> int:
        return int(self.ev_kind.shape[0])

    def rep_events(self, rep: int) -> slice:
        return slice(int(self.ev_off[rep]), int(self.ev_off[rep + 1]))

    def rank_ops(self) -> int:
        """Sum over ranks of the representative trace length: the unit of work
        the reference simulator performs (sim.py:183-184)."""
        lens = np.diff(self.ev_off)
        return int(lens[self.rank_rep].sum())

    def call_index(self, comm: int, idx: int) -> int:
        return int(self.call_off[comm]) + idx

    # -- persistence ----------------------------------------------------------

    def to_arrays(self, prefix: str = "") -> dict:
        d = {}
        for f in dataclasses.fields(self):
            v = getattr(self, f.name)
            if isinstance(v, np.ndarray):
                d[prefix + f.name] = v
        d[prefix + "meta"] = np.array([self.num_hosts, self.devices_per_host, self.capacity],
                                      dtype=np.int64)
        dev = self.device
        d[prefix + "device"] = np.array(
            [dev.hbm_bytes_per_s, dev.intra_alpha_ns, dev.intra_beta,
             dev.inter_alpha_ns, dev.inter_beta], dtype=np.int64)
        d[prefix + "strings"] = np.array(
            [repr({"op_kind_names": list(self.op_kind_names),
                   "dtype_names": list(self.dtype_names),
                   "comm_names": list(self.comm_names),
                   "device_name": dev.name,
                   "peak_flops": dict(dev.peak_flops),
                   "name": self.name})])
        return d

    @staticmethod
    def from_arrays(d: Mapping, prefix: str = "") -> "RawJob":
        import ast
        s = ast.literal_eval(str(d[prefix + "strings"][0]))
        meta = [int(x) for x in d[prefix + "meta"]]
        dv = [int(x) for x in d[prefix + "device"]]
        dev = DeviceParams(s["device_name"], s["peak_flops"], dv[0], dv[1], dv[2], dv[3], dv[4])
        arrays = {}
        for f in dataclasses.fields(RawJob):
            key = prefix + f.name
            if f.name in ("kernel_ns", "wire_ns"):
                arrays[f.name] = np.asarray(d[key]) if key in d else None
            elif key in d and f.name not in ("device",):
                arrays[f.name] = np.asarray(d[key])
        return RawJob(num_hosts=meta[0], devices_per_host=meta[1], capacity=meta[2],
                      device=dev, op_kind_names=list(s["op_kind_names"]),
                      dtype_names=list(s["dtype_names"]), comm_names=list(s["comm_names"]),
                      name=s.get("name", ""), **arrays)

    def with_capacity(self, capacity: int) -> "RawJob":
        return dataclasses.replace(self, capacity=int(capacity))


def save_jobs(path: str, jobs: Sequence[RawJob], extra: Mapping | None = None) -> None:
    d = {"n_jobs": np.array([len(jobs)])}
    for i, job in enumerate(jobs):
        d.update(job.to_arrays(f"j{i}."))
    if extra:
        d.update(extra)
    np.savez_compressed(path, **d)


def load_jobs(path: str) -> tuple[list[RawJob], dict]:
    with np.load(path, allow_pickle=False) as z:
        d = {k: z[k] for k in z.files}
    n = int(d["n_jobs"][0])
    jobs = [RawJob.from_arrays(d, f"j{i}.") for i in range(n)]
    extra = {k: v for k, v in d.items() if not k.startswith("j") and k != "n_jobs"}
    return jobs, extra


# --- adapter from the reference's Python objects ---------------------------------

class _Interner:
    def __init__(self):
        self.names: list[str] = []
        self.ids: dict[str, int] = {}

    def __call__(self, name: str) -> int:
        i = self.ids.get(name)
        if i is None:
            i = self.ids[name] = len(self.names)
            self.names.append(name)
        return i


def from_reference(job, *, kernel_ns: Mapping | None = None, wire_ns: Mapping | None = None,
                   capacity: int | None = None, name: str = "") -> RawJob:
    """Flatten a reference ``JobTrace`` (duck-typed: no dltsim import needed).

    ``kernel_ns``/``wire_ns`` are ``AnnotatedJob.kernel_ns``/``wire_ns``
    (estimate.py:324-325) when the durations were computed on the host.
    Raises ValueError for inputs the reference would reject or that the
    engine cannot represent (documented in DESIGN.md §Boundary).
    """
    cluster = job.cluster
    rep_ranks = sorted(job.reps)
    rep_index = {r: i for i, r in enumerate(rep_ranks)}
    all_ranks = job.all_ranks()
    if all_ranks != list(range(len(all_ranks))):
        raise ValueError("job ranks must be 0..R-1")
    rank_rep = np.array([rep_index[job.rep_of(r)] for r in all_ranks], dtype=np.int32)

    comm_names = sorted(job.groups)
    comm_id = {c: i for i, c in enumerate(comm_names)}
    comm_nranks = np.array([job.groups[c].nranks for c in comm_names], dtype=np.int32)
    comm_topo = np.array([TOPOLOGIES.index(job.groups[c].topology) for c in comm_names],
                         dtype=np.int8)
    ncalls = [0] * len(comm_names)
    for (c, idx) in job.calls:
        if c not in comm_id:
            raise ValueError(f"call on unknown comm {c}")
        if idx < 0:
            raise ValueError(f"negative call_idx on {c}")
        ncalls[comm_id[c]] = max(ncalls[comm_id[c]], idx + 1)
    call_off = np.zeros(len(comm_names) + 1, dtype=np.int64)
    call_off[1:] = np.cumsum(ncalls)
    n_calls = int(call_off[-1])
    call_kind = np.full(n_calls, -1, dtype=np.int8)
    call_bytes = np.zeros(n_calls, dtype=np.int64)
    wire = np.full(n_calls, -1, dtype=np.int64) if wire_ns is not None else None
    for (c, idx), (kind, nbytes) in job.calls.items():
        k = int(call_off[comm_id[c]]) + idx
        call_kind[k] = COLLECTIVE_KINDS.index(kind)
        call_bytes[k] = _i64(nbytes, "collective bytes")
        if wire is not None:
            wire[k] = _i64(wire_ns[(c, idx)], "wire_ns")

    ops = _Interner()
    dts = _Interner()
    kinds: list[int] = []
    streams: list[int] = []
    fs: list[tuple[int, int, int, int]] = []
    kns: list[int] = []
    ev_off = [0]
    rep_local_comms: list[list[str]] = []
    for rep in rep_ranks:
        trace = job.reps[rep]
        local: dict[str, int] = {}
        order: list[str] = []
        for ev in trace.events:
            if type(ev).__name__ == "CommInit" and ev.comm_id not in local:
                local[ev.comm_id] = len(order)
                order.append(ev.comm_id)
        rep_local_comms.append(order)
        for seq, ev in enumerate(trace.events):
            cls = type(ev).__name__
            k = _KIND_OF_CLASS.get(cls)
            if k is None:
                raise TypeError(f"unhandled event {type(ev)!r}")
            s = int(getattr(ev, "stream", 0))
            if k == EV_HOSTGAP:
                f = (_i64(ev.duration_ns, "gap"), 0, 0, 0)
            elif k == EV_KERNEL:
                a = ev.attrs
                f = (ops(ev.op_kind), dts(a.dtype), _i64(a.flops, "flops"),
                     _i64(a.bytes_moved, "bytes_moved"))
            elif k == EV_MEMALLOC:
                f = (_i64(ev.alloc_id, "alloc_id"), _i64(ev.bytes, "alloc bytes"), 0, 0)
            elif k == EV_MEMFREE:
                f = (_i64(ev.alloc_id, "alloc_id"), 0, 0, 0)
            elif k == EV_MEMCPY:
                f = (ops(MEMCPY_OP_KINDS[ev.direction]), dts("fp32"), 0,
                     _i64(ev.bytes, "memcpy bytes"))
            elif k == EV_MEMSET:
                f = (ops("memset"), dts("fp32"), 0, _i64(ev.bytes, "memset bytes"))
            elif k in (EV_RECORD, EV_WAIT, EV_ESYNC):
                f = (_i64(ev.event_id, "event_id"), _i64(ev.version, "version"), 0, 0)
            elif k in (EV_SSYNC, EV_DSYNC):
                f = (0, 0, 0, 0)
            elif k == EV_COMMINIT:
                f = (local[ev.comm_id], int(ev.nranks), int(ev.my_rank), 0)
            else:  # Collective
                if ev.comm_id not in local:
                    raise ValueError(f"rank {rep} seq {seq}: collective on comm "
                                     f"{ev.comm_id} without CommInit")
                f = (local[ev.comm_id], _i64(ev.call_idx, "call_idx"),
                     COLLECTIVE_KINDS.index(ev.kind), _i64(ev.bytes, "collective bytes"))
            kinds.append(k)
            streams.append(s)
            fs.append(f)
            if kernel_ns is not None:
                kns.append(int(kernel_ns.get((rep, seq), -1))
                           if k in (EV_KERNEL, EV_MEMCPY, EV_MEMSET) else -1)
        ev_off.append(len(kinds))

    rank_comm: list[int] = []
    rank_comm_off = [0]
    for r in all_ranks:
        cm = job.comm_map[r]
        for c in rep_local_comms[rank_rep[r]]:
            rank_comm.append(comm_id[cm[c][0]])
        rank_comm_off.append(len(rank_comm))

    dev = DeviceParams.from_reference(cluster.device)
    E = len(kinds)
    return RawJob(
        num_hosts=int(cluster.num_hosts), devices_per_host=int(cluster.devices_per_host),
        capacity=int(capacity if capacity is not None else cluster.device_memory_bytes),
        device=dev,
        rep_ranks=np.array(rep_ranks, dtype=np.int64), rank_rep=rank_rep,
        ev_off=np.array(ev_off, dtype=np.int64),
        ev_kind=np.array(kinds, dtype=np.uint8),
        ev_stream=np.array(streams, dtype=np.int32),
        ev_f=np.array(fs, dtype=np.int64).reshape(E, 4),
        op_kind_names=ops.names, dtype_names=dts.names, comm_names=comm_names,
        comm_nranks=comm_nranks, comm_topo=comm_topo, call_off=call_off,
        call_kind=call_kind, call_bytes=call_bytes,
        rank_comm_off=np.array(rank_comm_off, dtype=np.int64),
        rank_comm=np.array(rank_comm, dtype=np.int32),
        kernel_ns=np.array(kns, dtype=np.int64) if kernel_ns is not None else None,
        wire_ns=wire, name=name)


def from_annotated(annotated, cluster=None, name: str = "") -> RawJob:
    """Flatten an ``AnnotatedJob`` keeping its host-computed durations.

    ``cluster`` mirrors ``simulate``'s override (sim.py:476-485): only its
    memory capacity is used, and its device count must match.
    """
    job = annotated.job
    cap = None
    if cluster is not None:
        if cluster.num_devices != job.cluster.num_devices:
            raise ValueError("cluster does not match the collated job")
        cap = cluster.device_memory_bytes
    return from_reference(job, kernel_ns=annotated.kernel_ns, wire_ns=annotated.wire_ns,
                          capacity=cap, name=name)


def raw_digest(job: RawJob) -> str:
    """Content hash of a RawJob independent of string-table ordering."""
    import hashlib
    h = hashlib.sha256()
    f = job.ev_f.copy()
    kc = np.isin(job.ev_kind, (EV_KERNEL, EV_MEMCPY, EV_MEMSET))
    used_ops: list = []
    used_dts: list = []
    if kc.any():
        used_ops = sorted(set(job.op_kind_names[i] for i in np.unique(job.ev_f[kc, 0])))
        used_dts = sorted(set(job.dtype_names[i] for i in np.unique(job.ev_f[kc, 1])))
        om = np.array([used_ops.index(n) if n in used_ops else -1 for n in job.op_kind_names])
        dm = np.array([used_dts.index(n) if n in used_dts else -1 for n in job.dtype_names])
        f[kc, 0] = om[f[kc, 0]]
        f[kc, 1] = dm[f[kc, 1]]
    h.update(repr((used_ops, used_dts, job.num_hosts, job.devices_per_host, job.capacity,
                   list(job.comm_names))).encode())
    for a in (job.rep_ranks, job.rank_rep, job.ev_off, job.ev_kind, job.ev_stream, f,
              job.comm_nranks, job.comm_topo, job.call_off, job.call_kind, job.call_bytes,
              job.rank_comm_off, job.rank_comm):
        h.update(np.ascontiguousarray(a, dtype=np.int64).tobytes())
    return h.hexdigest()
