"""Duck-typed stand-ins for the reference's trace/collation classes (same class
and field names as pkg/src/dltsim/trace.py, collate.py, cluster.py,
estimate.py), rebuilt from a RawJob so the drop-in ``simulate(annotated)``
path can be tested where the reference is not installed (the GPU box)."""
from dataclasses import dataclass, field

from paper_2503_20191_b200.rawtrace import (COLLECTIVE_KINDS, TOPOLOGIES, EV_COLLECTIVE,
                                            EV_COMMINIT, EV_DSYNC, EV_ESYNC, EV_HOSTGAP,
                                            EV_KERNEL, EV_MEMALLOC, EV_MEMCPY, EV_MEMFREE,
                                            EV_MEMSET, EV_RECORD, EV_SSYNC, EV_WAIT)


@dataclass(frozen=True)
class KernelAttrs:
    dims: tuple
    dtype: str
    flops: int
    bytes_moved: int


@dataclass(frozen=True)
class HostGap:
    duration_ns: int


@dataclass(frozen=True)
class KernelLaunch:
    stream: int
    op_kind: str
    attrs: KernelAttrs


@dataclass(frozen=True)
class MemAlloc:
    alloc_id: int
    bytes: int


@dataclass(frozen=True)
class MemFree:
    alloc_id: int


@dataclass(frozen=True)
class Memcpy:
    stream: int
    direction: str
    bytes: int


@dataclass(frozen=True)
class Memset:
    stream: int
    bytes: int


@dataclass(frozen=True)
class EventRecord:
    stream: int
    event_id: int
    version: int


@dataclass(frozen=True)
class StreamWaitEvent:
    stream: int
    event_id: int
    version: int


@dataclass(frozen=True)
class EventSynchronize:
    event_id: int
    version: int


@dataclass(frozen=True)
class StreamSynchronize:
    stream: int


@dataclass(frozen=True)
class DeviceSynchronize:
    pass


@dataclass(frozen=True)
class CommInit:
    comm_id: str
    nranks: int
    my_rank: int


@dataclass(frozen=True)
class Collective:
    stream: int
    comm_id: str
    call_idx: int
    kind: str
    bytes: int
    nranks: int


@dataclass(frozen=True)
class WorkerTrace:
    global_rank: int
    host_index: int
    device_index: int
    events: tuple


@dataclass(frozen=True)
class LinkClass:
    alpha_ns: int
    beta_bytes_per_s: int


@dataclass(frozen=True)
class DeviceClass:
    name: str
    peak_flops: dict
    hbm_bytes_per_s: int
    links: dict


@dataclass(frozen=True)
class ClusterSpec:
    num_hosts: int
    devices_per_host: int
    device_memory_bytes: int
    device: DeviceClass

    @property
    def num_devices(self):
        return self.num_hosts * self.devices_per_host


@dataclass(frozen=True)
class CommGroup:
    comm_id: str
    nranks: int
    ranks: tuple
    topology: str


@dataclass(frozen=True)
class JobTrace:
    cluster: ClusterSpec
    reps: dict
    dup_of: dict
    comm_map: dict
    groups: dict
    calls: dict

    def all_ranks(self):
        return sorted(list(self.reps) + list(self.dup_of))

    def rep_of(self, rank):
        return self.dup_of.get(rank, rank)


@dataclass(frozen=True)
class AnnotatedJob:
    job: JobTrace
    kernel_ns: dict
    wire_ns: dict
    warnings: tuple = ()


_DIRS = {"memcpy_h2d": "H2D", "memcpy_d2h": "D2H", "memcpy_d2d": "D2D"}


def to_reference_like(raw, kernel_ns=None, wire_ns=None):
    """Inverse of rawtrace.from_reference (durations default to the raw's)."""
    d = raw.device
    dev = DeviceClass(d.name, dict(d.peak_flops), d.hbm_bytes_per_s,
                      {"intra_host": LinkClass(d.intra_alpha_ns, d.intra_beta),
                       "inter_host": LinkClass(d.inter_alpha_ns, d.inter_beta)})
    cluster = ClusterSpec(raw.num_hosts, raw.devices_per_host, raw.capacity, dev)
    reps, rep_local = {}, []
    kn = {} if kernel_ns is None else kernel_ns
    for rep in range(raw.n_reps):
        rank = int(raw.rep_ranks[rep])
        sl = raw.rep_events(rep)
        local = []
        # local comm names of this rep: from a rank that uses the rep
        r0 = int(list(raw.rank_rep).index(rep))
        cb = int(raw.rank_comm_off[r0])
        evs = []
        for seq, (k, s, f) in enumerate(zip(raw.ev_kind[sl].tolist(), raw.ev_stream[sl].tolist(),
                                            raw.ev_f[sl].tolist())):
            if k == EV_HOSTGAP:
                ev = HostGap(f[0])
            elif k == EV_KERNEL:
                ev = KernelLaunch(s, raw.op_kind_names[f[0]],
                                  KernelAttrs((), raw.dtype_names[f[1]], f[2], f[3]))
            elif k == EV_MEMALLOC:
                ev = MemAlloc(f[0], f[1])
            elif k == EV_MEMFREE:
                ev = MemFree(f[0])
            elif k == EV_MEMCPY:
                ev = Memcpy(s, _DIRS[raw.op_kind_names[f[0]]], f[3])
            elif k == EV_MEMSET:
                ev = Memset(s, f[3])
            elif k == EV_RECORD:
                ev = EventRecord(s, f[0], f[1])
            elif k == EV_WAIT:
                ev = StreamWaitEvent(s, f[0], f[1])
            elif k == EV_ESYNC:
                ev = EventSynchronize(f[0], f[1])
            elif k == EV_SSYNC:
                ev = StreamSynchronize(s)
            elif k == EV_DSYNC:
                ev = DeviceSynchronize()
            elif k == EV_COMMINIT:
                g = int(raw.rank_comm[cb + f[0]]) if rank == r0 else None
                name = raw.comm_names[int(raw.rank_comm[int(raw.rank_comm_off[rank]) + f[0]])]
                ev = CommInit(name, f[1], f[2])
            else:
                name = raw.comm_names[int(raw.rank_comm[int(raw.rank_comm_off[rank]) + f[0]])]
                ev = Collective(s, name, f[1], COLLECTIVE_KINDS[f[2]], f[3],
                                int(raw.comm_nranks[int(raw.rank_comm[int(raw.rank_comm_off[rank]) + f[0]])]))
            if k in (EV_KERNEL, EV_MEMCPY, EV_MEMSET) and raw.kernel_ns is not None and kernel_ns is None:
                kn[(rank, seq)] = int(raw.kernel_ns[sl.start + seq])
            evs.append(ev)
        reps[rank] = WorkerTrace(rank, *divmod(rank, raw.devices_per_host), tuple(evs))
    dup_of, comm_map = {}, {}
    for r in range(raw.num_ranks):
        rep = int(raw.rep_ranks[raw.rank_rep[r]])
        if r != rep:
            dup_of[r] = rep
        rep_names = [raw.comm_names[int(g)] for g in
                     raw.rank_comm[int(raw.rank_comm_off[rep]):int(raw.rank_comm_off[rep + 1])]]
        own = [raw.comm_names[int(g)] for g in
               raw.rank_comm[int(raw.rank_comm_off[r]):int(raw.rank_comm_off[r + 1])]]
        comm_map[r] = {a: (b, 0) for a, b in zip(rep_names, own)}
    groups = {name: CommGroup(name, int(raw.comm_nranks[g]), (), TOPOLOGIES[raw.comm_topo[g]])
              for g, name in enumerate(raw.comm_names)}
    calls, wn = {}, {} if wire_ns is None else wire_ns
    for g, name in enumerate(raw.comm_names):
        for c in range(int(raw.call_off[g]), int(raw.call_off[g + 1])):
            if raw.call_kind[c] >= 0:
                idx = c - int(raw.call_off[g])
                calls[(name, idx)] = (COLLECTIVE_KINDS[raw.call_kind[c]], int(raw.call_bytes[c]))
                if raw.wire_ns is not None and wire_ns is None:
                    wn[(name, idx)] = int(raw.wire_ns[c])
    job = JobTrace(cluster, reps, dup_of, comm_map, groups, calls)
    return AnnotatedJob(job, kn, wn)
