"""Text traces and job manifests through the native loader.

Mirrors the reference's I/O entry points with the engine's data types:

* ``parse_trace_text(text) -> ParsedTrace``   parse_trace + validate_trace
  (``pkg/src/dltsim/trace.py:282-397``, ``:406-495``); ``.serialize()`` is
  ``serialize_trace`` (``trace.py:282-290``);
* ``load_job(manifest_path, cluster) -> LoadedJob``  load_job + collate
  (``pkg/src/dltsim/collate.py:256-372``, ``:405-431``); ``.raw()`` is the
  ``RawJob`` that ``rawtrace.from_reference(load_job(...))`` gives, without
  building WorkerTrace objects; ``.save(out_dir)`` is ``save_job``
  (``collate.py:377-402``).

Errors carry the reference's messages.  The exception classes subclass
dltsim's own (TraceParseError, TraceValidationError, CollationError) when the
reference package is importable, so ``except dltsim.trace.TraceError`` keeps
working.  Integers that do not fit int64 raise OverflowError (the reference
keeps Python ints; the engine's fields are int64).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .rawtrace import DeviceParams, RawJob


def _ref_bases():
    try:
        from dltsim.collate import CollationError as CE
        from dltsim.trace import TraceParseError as PE, TraceValidationError as VE
        return PE, VE, CE
    except Exception:
        return Exception, Exception, Exception


_PE, _VE, _CE = _ref_bases()


class TraceParseError(_PE):
    """trace.py:209-212; str() is "line <n>: <message>"."""

    def __init__(self, line_no: int, message: str):
        Exception.__init__(self, f"line {line_no}: {message}")
        self.line_no = line_no


class TraceValidationError(_VE):
    """trace.py:215-220; str() is "invalid trace: seq <i>: [<rule>] <message>; ..."."""

    def __init__(self, message: str):
        Exception.__init__(self, message)
        self.violations = None


class CollationError(_CE):
    """collate.py:42."""

    def __init__(self, message: str):
        Exception.__init__(self, message)


ERR_PARSE, ERR_VALIDATION, ERR_COLLATION, ERR_RANGE, ERR_IO = 1, 2, 3, 4, 5


def _lib():
    from .engine import lib
    from .workload import ClusterC, _gen_lib
    L = _gen_lib()
    if not hasattr(L, "_traceio_ready"):
        P = C.POINTER
        vp = C.c_void_p
        L.maya_last_error_kind.restype = C.c_int
        L.maya_trace_parse.argtypes = [C.c_char_p, C.c_int64, P(vp)]
        L.maya_trace_info.argtypes = [vp, P(C.c_int64)]
        L.maya_trace_serialize.argtypes = [vp, P(C.c_char_p), P(C.c_int64)]
        L.maya_trace_free.argtypes = [vp]
        L.maya_job_load.argtypes = [C.c_char_p, P(ClusterC), P(vp)]
        L.maya_job_save.argtypes = [vp, C.c_char_p, C.c_char_p]
        L.maya_gen_names.argtypes = [vp, C.c_int32, P(C.c_char_p), P(C.c_int32)]
        L._traceio_ready = True
    return L


def _raise(L) -> None:
    kind = L.maya_last_error_kind()
    msg = L.maya_last_error().decode("utf-8", "replace")
    if kind == ERR_PARSE:
        head, _, rest = msg.partition(": ")
        raise TraceParseError(int(head.split()[1]), rest)
    if kind == ERR_VALIDATION:
        raise TraceValidationError(msg)
    if kind == ERR_COLLATION:
        raise CollationError(msg)
    if kind == ERR_RANGE:
        raise OverflowError(msg)
    if kind == ERR_IO:
        raise FileNotFoundError(msg)
    raise ValueError(msg)


class ParsedTrace:
    """One parsed and validated worker trace (native)."""

    def __init__(self, handle, lib):
        self._h, self._L = handle, lib
        info = (C.c_int64 * 4)()
        lib.maya_trace_info(handle, info)
        self.global_rank, self.host_index, self.device_index, self.n_events = (int(x) for x in info)

    def serialize(self) -> str:
        p, n = C.c_char_p(), C.c_int64()
        self._L.maya_trace_serialize(self._h, C.byref(p), C.byref(n))
        return C.string_at(p, n.value).decode("utf-8")

    def close(self) -> None:
        if self._h:
            self._L.maya_trace_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def parse_trace_text(text: str | bytes) -> ParsedTrace:
    """parse_trace(io.StringIO(text)) natively (universal newlines)."""
    L = _lib()
    b = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    if L.maya_trace_parse(b, len(b), C.byref(h)) != 0:
        _raise(L)
    return ParsedTrace(h, L)


def _copy(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


class LoadedJob:
    """A job read from a manifest: its raw arrays and its text form."""

    def __init__(self, handle, lib, cluster):
        self._h, self._L, self.cluster = handle, lib, cluster

    def _names(self, which: int) -> list:
        p, n = C.c_char_p(), C.c_int32()
        self._L.maya_gen_names(self._h, which, C.byref(p), C.byref(n))
        return p.value.decode().split("\n")[:n.value] if n.value else []

    def raw(self, name: str = "") -> RawJob:
        """The RawJob of rawtrace.from_reference(load_job(manifest, cluster))."""
        L = self._L
        v = L._GenViewC()
        L.maya_gen_view_of(self._h, C.byref(v))
        j = v.job
        R, nrep, E = j.num_ranks, j.n_reps, v.n_events
        G, ncall = v.n_comm_names, v.n_calls
        names = v.comm_names.decode().split("\n")[:G] if G else []
        return RawJob(
            num_hosts=v.num_hosts, devices_per_host=j.devices_per_host, capacity=j.capacity,
            device=DeviceParams.from_reference(self.cluster.device),
            rep_ranks=_copy(v.rep_ranks, nrep, np.int64),
            rank_rep=_copy(j.rank_rep, R, np.int32),
            ev_off=_copy(j.ev_off, nrep + 1, np.int64),
            ev_kind=_copy(j.ev_kind, E, np.uint8),
            ev_stream=_copy(j.ev_stream, E, np.int32),
            ev_f=_copy(j.ev_f, 4 * E, np.int64).reshape(E, 4),
            op_kind_names=self._names(0), dtype_names=self._names(1), comm_names=names,
            comm_nranks=_copy(j.comm_nranks, G, np.int32),
            comm_topo=_copy(j.comm_topo, G, np.int8),
            call_off=_copy(j.call_off, G + 1, np.int64),
            call_kind=_copy(j.call_kind, ncall, np.int8),
            call_bytes=_copy(j.call_bytes, ncall, np.int64),
            rank_comm_off=_copy(j.rank_comm_off, R + 1, np.int64),
            rank_comm=_copy(j.rank_comm, v.n_rank_comm, np.int32), name=name)

    def save(self, out_dir: str, manifest_name: str = "job.manifest") -> str:
        """save_job (collate.py:377-402): rank_<r>.trace per representative + manifest."""
        import os
        if self._L.maya_job_save(self._h, out_dir.encode(), manifest_name.encode()) != 0:
            _raise(self._L)
        return os.path.join(out_dir, manifest_name)

    def close(self) -> None:
        if self._h:
            self._L.maya_gen_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def load_job(manifest_path: str, cluster) -> LoadedJob:
    """load_job(manifest_path, cluster) (collate.py:405-431) natively."""
    from .workload import cluster_c
    L = _lib()
    h = C.c_void_p()
    if L.maya_job_load(str(manifest_path).encode(), C.byref(cluster_c(cluster)), C.byref(h)) != 0:
        _raise(L)
    return LoadedJob(h, L, cluster)


def load_raw_job(manifest_path: str, cluster, name: str = "") -> RawJob:
    """Manifest -> RawJob for the engine (Engine.simulate / api.simulate_raw)."""
    job = load_job(manifest_path, cluster)
    try:
        return job.raw(name)
    finally:
        job.close()
