"""Host-side mirror of the reference frontend API used around the hot path.

* ModelSpec / ConfigPoint / ClusterSpec / DeviceClass mirrors with the same
  fields as pkg/src/dltsim/workload.py:96-165 and cluster.py:29-92 (reference
  objects are accepted anywhere, duck-typed);
* validate_config / default_schedule / SearchSpace / enumerate_space
  restated from workload.py:168-221 and search.py:44-79 (pure host logic);
* generate_job: the native (C++) trace generator — workload.py:571-791 plus
  collate.py:256-372 — producing a RawJob without building Python events.
"""

from __future__ import annotations

import ctypes as C
import enum
import itertools
from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np

from .rawtrace import DeviceParams, RawJob

DEFAULT_DISPATCH_OVERHEAD_NS = 5000      # workload.py:69
DTYPE_SIZES = {"fp32": 4, "fp16": 2, "bf16": 2}
GEN_DTYPE_IDS = {"bf16": 0, "fp16": 1, "fp32": 2}
GEN_OP_KINDS = ("gemm", "layernorm", "softmax", "gelu", "add", "embed", "cross_entropy",
                "optimizer_step", "memcpy_h2d", "memcpy_d2h", "memcpy_d2d", "memset")
GEN_DTYPES = ("bf16", "fp16", "fp32")


class ConfigError(Exception):
    pass


class ScheduleKind(enum.Enum):
    GPIPE = "gpipe"
    ONE_F_ONE_B = "1f1b"
    INTERLEAVED_ONE_F_ONE_B = "interleaved"


_SCHED_CODE = {"gpipe": 0, "1f1b": 1, "interleaved": 2}


@dataclass(frozen=True)
class LinkClass:
    alpha_ns: int
    beta_bytes_per_s: int


@dataclass(frozen=True)
class DeviceClass:
    name: str
    peak_flops: Mapping[str, int]
    hbm_bytes_per_s: int
    links: Mapping[str, LinkClass]

    def link(self, topology: str) -> LinkClass:
        return self.links["inter_host" if topology == "mixed" else topology]


@dataclass(frozen=True)
class ClusterSpec:
    num_hosts: int
    devices_per_host: int
    device_memory_bytes: int
    device: DeviceClass

    @property
    def num_devices(self) -> int:
        return self.num_hosts * self.devices_per_host

    def placement(self, global_rank: int) -> tuple[int, int]:
        return divmod(global_rank, self.devices_per_host)


@dataclass(frozen=True)
class ModelSpec:
    name: str
    num_layers: int
    hidden_size: int
    seq_len: int
    vocab_size: int
    dtype: str = "bf16"

    @property
    def elem_size(self) -> int:
        return DTYPE_SIZES[self.dtype]


@dataclass(frozen=True)
class ConfigPoint:
    tp: int
    pp: int
    micro_mult: int
    virtual_stages: int
    act_recompute: bool
    seq_parallel: bool
    dist_optimizer: bool
    global_batch: int

    @property
    def microbatches(self) -> int:
        return self.micro_mult * self.pp

    def dp(self, cluster) -> int:
        return cluster.num_devices // (self.tp * self.pp)

    def key(self) -> tuple:
        return (self.tp, self.pp, self.micro_mult, self.virtual_stages, self.act_recompute,
                self.seq_parallel, self.dist_optimizer, self.global_batch)

    def label(self) -> str:
        flags = "".join(c if on else "-" for c, on in
                        (("r", self.act_recompute), ("s", self.seq_parallel),
                         ("z", self.dist_optimizer)))
        return (f"tp{self.tp}.pp{self.pp}.mm{self.micro_mult}"
                f".vs{self.virtual_stages}.{flags}")


# presets (pkg/src/dltsim/presets/*.yaml)
_DEVICE_PRESETS = {
    "fast": DeviceClass("fast", {"bf16": 990_000_000_000_000, "fp16": 990_000_000_000_000,
                                 "fp32": 67_000_000_000_000}, 3_350_000_000_000,
                        {"intra_host": LinkClass(2000, 400_000_000_000),
                         "inter_host": LinkClass(6000, 50_000_000_000)}),
    "slow": DeviceClass("slow", {"bf16": 125_000_000_000_000, "fp16": 125_000_000_000_000,
                                 "fp32": 15_700_000_000_000}, 900_000_000_000,
                        {"intra_host": LinkClass(3000, 150_000_000_000),
                         "inter_host": LinkClass(9000, 12_000_000_000)}),
}
_MODEL_PRESETS = {
    "gpt3-18.4b": ModelSpec("gpt3-18.4b", 40, 6144, 2048, 51200, "bf16"),
    "gpt3-2.7b": ModelSpec("gpt3-2.7b", 32, 2560, 2048, 51200, "bf16"),
    "tiny": ModelSpec("tiny", 8, 512, 512, 8192, "bf16"),
}


def load_device_preset(name: str) -> DeviceClass:
    try:
        return _DEVICE_PRESETS[name]
    except KeyError:
        raise ValueError(f"unknown device preset {name!r}") from None


def load_model_preset(name: str) -> ModelSpec:
    try:
        return _MODEL_PRESETS[name]
    except KeyError:
        raise ConfigError(f"unknown model preset {name!r}") from None


def _sched_name(schedule) -> str | None:
    if schedule is None:
        return None
    return getattr(schedule, "value", schedule)


def validate_config(model, config, cluster, schedule=None) -> list[str]:
    """workload.py:168-208, message for message."""
    errors = []
    if min(config.tp, config.pp, config.micro_mult, config.virtual_stages,
           config.global_batch) < 1:
        errors.append("tp/pp/micro_mult/virtual_stages/global_batch must be >= 1")
        return errors
    n = cluster.num_devices
    if n % (config.tp * config.pp) != 0:
        errors.append(f"tp*pp = {config.tp * config.pp} does not divide "
                      f"device count {n}")
        return errors
    d = n // (config.tp * config.pp)
    m = config.micro_mult * config.pp
    if config.global_batch % (d * m) != 0:
        errors.append(f"global_batch {config.global_batch} not divisible by "
                      f"dp*microbatches = {d}*{m}")
    if model is not None:
        if model.hidden_size % config.tp != 0:
            errors.append(f"hidden_size {model.hidden_size} not divisible by tp {config.tp}")
        if model.seq_len % config.tp != 0:
            errors.append(f"seq_len {model.seq_len} not divisible by tp {config.tp}")
        if model.vocab_size % config.tp != 0:
            errors.append(f"vocab_size {model.vocab_size} not divisible by tp {config.tp}")
        if model.num_layers % (config.pp * config.virtual_stages) != 0:
            errors.append(f"num_layers {model.num_layers} not divisible by "
                          f"pp*virtual_stages = {config.pp}*{config.virtual_stages}")
    if config.virtual_stages > 1 and config.pp == 1:
        errors.append("virtual_stages > 1 requires pp > 1 (interleaving needs a pipeline)")
    sname = _sched_name(schedule)
    if sname is not None:
        if sname == "interleaved" and config.virtual_stages == 1:
            errors.append("interleaved schedule requires virtual_stages > 1")
        if sname != "interleaved" and config.virtual_stages > 1:
            errors.append(f"schedule {sname} requires virtual_stages == 1")
        if sname == "1f1b" and m < config.pp:
            errors.append("1f1b needs microbatches >= pp for warmup")
    return errors


def default_schedule(config) -> ScheduleKind:
    if config.virtual_stages > 1:
        return ScheduleKind.INTERLEAVED_ONE_F_ONE_B
    return ScheduleKind.ONE_F_ONE_B


@dataclass(frozen=True)
class SearchSpace:
    """search.py:44-63 (default knob table)."""

    tp: tuple = (1, 2, 4, 8)
    pp: tuple = (1, 2, 4, 8)
    micro_mult: tuple = (1, 2, 4, 6, 8)
    virtual_stages: tuple = (1, 2, 4)
    act_recompute: tuple = (True, False)
    seq_parallel: tuple = (True, False)
    dist_optimizer: tuple = (True, False)
    global_batch: int = 512

    def points(self) -> list[ConfigPoint]:
        return [ConfigPoint(tp, pp, mm, vs, rc, sp, dz, self.global_batch)
                for tp, pp, mm, vs, rc, sp, dz in itertools.product(
                    self.tp, self.pp, self.micro_mult, self.virtual_stages,
                    self.act_recompute, self.seq_parallel, self.dist_optimizer)]


def enumerate_space(space, model, cluster, with_invalid: bool = False):
    """search.py:66-79: valid points in itertools.product order."""
    points = space.points()
    if not points:
        raise ValueError("empty search space")
    annotated = [(c, validate_config(model, c, cluster)) for c in points]
    if with_invalid:
        return annotated
    return [c for c, reasons in annotated if not reasons]


# --- native generation ------------------------------------------------------------

class ModelC(C.Structure):
    _fields_ = [("num_layers", C.c_int64), ("hidden_size", C.c_int64), ("seq_len", C.c_int64),
                ("vocab_size", C.c_int64), ("dtype", C.c_int32), ("pad", C.c_int32)]


class ConfigC(C.Structure):
    _fields_ = [("tp", C.c_int32), ("pp", C.c_int32), ("micro_mult", C.c_int32),
                ("virtual_stages", C.c_int32), ("act_recompute", C.c_int32),
                ("seq_parallel", C.c_int32), ("dist_optimizer", C.c_int32), ("pad", C.c_int32),
                ("global_batch", C.c_int64)]


class ClusterC(C.Structure):
    _fields_ = [("num_hosts", C.c_int32), ("devices_per_host", C.c_int32),
                ("device_memory_bytes", C.c_int64)]


def model_c(model) -> ModelC:
    if model.dtype not in GEN_DTYPE_IDS:
        raise ConfigError(f"unknown dtype {model.dtype!r}")
    return ModelC(int(model.num_layers), int(model.hidden_size), int(model.seq_len),
                  int(model.vocab_size), GEN_DTYPE_IDS[model.dtype], 0)


def config_c(cfg) -> ConfigC:
    return ConfigC(int(cfg.tp), int(cfg.pp), int(cfg.micro_mult), int(cfg.virtual_stages),
                   int(bool(cfg.act_recompute)), int(bool(cfg.seq_parallel)),
                   int(bool(cfg.dist_optimizer)), 0, int(cfg.global_batch))


CONFIG_DTYPE = np.dtype([("tp", "<i4"), ("pp", "<i4"), ("micro_mult", "<i4"),
                         ("virtual_stages", "<i4"), ("act_recompute", "<i4"),
                         ("seq_parallel", "<i4"), ("dist_optimizer", "<i4"), ("pad", "<i4"),
                         ("global_batch", "<i8")])


def configs_array(configs) -> np.ndarray:
    """maya_config[n] (ConfigC layout) for a config list, built in one pass
    (ctypes structs one by one cost ~3 us per config)."""
    a = np.zeros(max(len(configs), 1), dtype=CONFIG_DTYPE)
    if configs:
        a[:len(configs)] = [(c.tp, c.pp, c.micro_mult, c.virtual_stages, bool(c.act_recompute),
                             bool(c.seq_parallel), bool(c.dist_optimizer), 0, c.global_batch)
                            for c in configs]
    return a


def cluster_c(cluster) -> ClusterC:
    return ClusterC(int(cluster.num_hosts), int(cluster.devices_per_host),
                    int(cluster.device_memory_bytes))


def schedule_code(schedule) -> int:
    s = _sched_name(schedule)
    return -1 if s is None else _SCHED_CODE[s]


def _gen_lib():
    from ._abi import RawJobC
    from .engine import lib
    L = lib()
    if not hasattr(L, "_gen_ready"):
        P = C.POINTER

        class GenViewC(C.Structure):
            _fields_ = [("job", RawJobC), ("num_hosts", C.c_int32), ("n_comm_names", C.c_int32),
                        ("rep_ranks", P(C.c_int64)), ("comm_names", C.c_char_p),
                        ("n_events", C.c_int64), ("n_calls", C.c_int64),
                        ("n_rank_comm", C.c_int64)]
        L.maya_gen_job.argtypes = [P(ModelC), P(ConfigC), P(ClusterC), C.c_int32, C.c_int64,
                                   P(C.c_void_p)]
        L.maya_gen_view_of.argtypes = [C.c_void_p, P(GenViewC)]
        L.maya_gen_free.argtypes = [C.c_void_p]
        L.maya_batch_add_generated.argtypes = [
            C.c_void_p, P(ModelC), C.c_int32, P(ConfigC), P(ClusterC), C.c_int32, C.c_int32,
            C.c_int64, P(C.c_int32), C.c_int32, P(C.c_int32)]
        L._GenViewC = GenViewC
        L._gen_ready = True
    return L


def _copy(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def generate_job(model, config, cluster, schedule=None,
                 dispatch_overhead_ns: int = DEFAULT_DISPATCH_OVERHEAD_NS,
                 name: str = "") -> RawJob:
    """RawJob of collate(*generate_representatives(model, config, cluster,
    schedule or default_schedule(config))) — natively."""
    errors = validate_config(model, config, cluster,
                             schedule if schedule is not None else default_schedule(config))
    if errors:
        raise ConfigError("; ".join(errors))
    L = _gen_lib()
    h = C.c_void_p()
    rc = L.maya_gen_job(C.byref(model_c(model)), C.byref(config_c(config)),
                        C.byref(cluster_c(cluster)), schedule_code(schedule),
                        int(dispatch_overhead_ns), C.byref(h))
    if rc != 0:
        raise ConfigError(L.maya_last_error().decode())
    try:
        v = L._GenViewC()
        L.maya_gen_view_of(h, C.byref(v))
        j = v.job
        R, nrep, E = j.num_ranks, j.n_reps, v.n_events
        G, ncall = v.n_comm_names, v.n_calls
        names = v.comm_names.decode().split("\n")[:G]
        raw = RawJob(
            num_hosts=v.num_hosts, devices_per_host=j.devices_per_host, capacity=j.capacity,
            device=DeviceParams.from_reference(cluster.device),
            rep_ranks=_copy(v.rep_ranks, nrep, np.int64),
            rank_rep=_copy(j.rank_rep, R, np.int32),
            ev_off=_copy(j.ev_off, nrep + 1, np.int64),
            ev_kind=_copy(j.ev_kind, E, np.uint8),
            ev_stream=_copy(j.ev_stream, E, np.int32),
            ev_f=_copy(j.ev_f, 4 * E, np.int64).reshape(E, 4),
            op_kind_names=list(GEN_OP_KINDS), dtype_names=list(GEN_DTYPES),
            comm_names=names,
            comm_nranks=_copy(j.comm_nranks, G, np.int32),
            comm_topo=_copy(j.comm_topo, G, np.int8),
            call_off=_copy(j.call_off, G + 1, np.int64),
            call_kind=_copy(j.call_kind, ncall, np.int8),
            call_bytes=_copy(j.call_bytes, ncall, np.int64),
            rank_comm_off=_copy(j.rank_comm_off, R + 1, np.int64),
            rank_comm=_copy(j.rank_comm, v.n_rank_comm, np.int32),
            name=name or config.label())
    finally:
        L.maya_gen_free(h)
    return raw
