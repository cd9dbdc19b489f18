"""Native text trace / manifest I/O against the reference.

CPU tests through the C ABI (the loader has no device code): the fixtures
under tests/golden/traceio* were produced by the reference itself
(tests/golden/make_traceio_golden.py): save_job() directories, the RawJob of
rawtrace.from_reference(load_job(...)), and the exception class + message of
every parse / validation / collation failure case.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

TRACEIO = os.path.join(GOLDEN, "traceio")


def _meta():
    from paper_2503_20191_b200.rawtrace import load_jobs
    jobs, extra = load_jobs(os.path.join(GOLDEN, "traceio_jobs.npz"))
    return jobs, json.loads(str(extra["meta"][0]))


def _cluster(nh, dph):
    from paper_2503_20191_b200 import workload as W
    return W.ClusterSpec(nh, dph, 80 * 2 ** 30, W.load_device_preset("fast"))


ARRAYS = ("rep_ranks", "rank_rep", "ev_off", "ev_kind", "ev_stream", "ev_f", "comm_nranks",
          "comm_topo", "call_off", "call_kind", "call_bytes", "rank_comm_off", "rank_comm")


@pytest.mark.parametrize("i", range(4))
def test_load_job_matches_reference(i):
    from paper_2503_20191_b200 import traceio
    from paper_2503_20191_b200.rawtrace import raw_digest
    jobs, meta = _meta()
    m, want = meta[i], jobs[i]
    got = traceio.load_raw_job(os.path.join(TRACEIO, m["name"], "job.manifest"),
                               _cluster(m["num_hosts"], m["devices_per_host"]), name=m["name"])
    for a in ARRAYS:
        assert np.array_equal(getattr(got, a), getattr(want, a)), (m["name"], a)
    assert got.op_kind_names == list(want.op_kind_names)
    assert got.dtype_names == list(want.dtype_names)
    assert got.comm_names == list(want.comm_names)
    assert (got.num_hosts, got.devices_per_host, got.capacity) == \
        (want.num_hosts, want.devices_per_host, want.capacity)
    assert raw_digest(got) == m["digest"]


@pytest.mark.parametrize("i", range(4))
def test_save_job_round_trip_is_byte_identical(i, tmp_path):
    """load (native) -> save (native) reproduces the reference's save_job files."""
    from paper_2503_20191_b200 import traceio
    _, meta = _meta()
    m = meta[i]
    src = os.path.join(TRACEIO, m["name"])
    job = traceio.load_job(os.path.join(src, "job.manifest"),
                           _cluster(m["num_hosts"], m["devices_per_host"]))
    job.save(str(tmp_path))
    assert sorted(os.listdir(tmp_path)) == sorted(os.listdir(src))
    for f in os.listdir(src):
        assert open(os.path.join(tmp_path, f), "rb").read() == \
            open(os.path.join(src, f), "rb").read(), f


def test_trace_serialize_round_trip():
    from paper_2503_20191_b200 import traceio
    d = os.path.join(TRACEIO, "pp4vs2_16r_2h")
    n = 0
    for f in sorted(os.listdir(d)):
        if not f.endswith(".trace"):
            continue
        text = open(os.path.join(d, f)).read()
        t = traceio.parse_trace_text(text)
        assert t.serialize() == text
        assert t.global_rank == int(f[5:-6])
        n += 1
    assert n >= 4


def _error_cases():
    return json.load(open(os.path.join(GOLDEN, "traceio_errors.json")))


def test_trace_errors_match_reference():
    from paper_2503_20191_b200 import traceio
    checked = 0
    for case in _error_cases():
        if "text" not in case:
            continue
        kind, msg = case["kind"], case["message"]
        if kind == "ok":
            try:
                traceio.parse_trace_text(case["text"])
            except OverflowError:
                # documented restriction: integers beyond int64 (the reference keeps Python ints)
                assert "99999999999999999999" in case["text"]
            checked += 1
            continue
        exc = {"parse": traceio.TraceParseError,
               "validation": traceio.TraceValidationError}[kind]
        with pytest.raises(exc) as ei:
            traceio.parse_trace_text(case["text"])
        assert str(ei.value) == msg, (case["text"], str(ei.value), msg)
        checked += 1
    assert checked >= 40


def test_manifest_errors_match_reference(tmp_path):
    from paper_2503_20191_b200 import traceio
    base = os.path.join(TRACEIO, "tp2pp2_8r")
    checked = 0
    for case in _error_cases():
        if "manifest" not in case:
            continue
        d = tmp_path / case["case"]
        d.mkdir()
        for f in os.listdir(base):
            body = case["manifest"] if f == "job.manifest" else \
                case["traces"].get(f, open(os.path.join(base, f)).read())
            (d / f).write_text(body)
        cl = _cluster(case["num_hosts"], case["devices_per_host"])
        if case["kind"] == "ok":
            traceio.load_raw_job(str(d / "job.manifest"), cl)
        else:
            exc = {"collation": traceio.CollationError, "parse": traceio.TraceParseError,
                   "validation": traceio.TraceValidationError}[case["kind"]]
            with pytest.raises(exc) as ei:
                traceio.load_raw_job(str(d / "job.manifest"), cl)
            assert str(ei.value) == case["message"], case["case"]
        checked += 1
    assert checked >= 10


def test_missing_trace_file(tmp_path):
    from paper_2503_20191_b200 import traceio
    (tmp_path / "job.manifest").write_text("dltsim-job v1 ranks=1\nworker rank=0 file=nope.trace\n")
    with pytest.raises(FileNotFoundError):
        traceio.load_job(str(tmp_path / "job.manifest"), _cluster(1, 1))


@pytest.mark.gpu
def test_loaded_job_simulates_like_generated():
    """A manifest read natively simulates to the reference's result for the
    same job (C1: total 9,846,585 ns, peak 4,822,794,240 B)."""
    from paper_2503_20191_b200 import traceio
    from paper_2503_20191_b200.engine import Engine
    raw = traceio.load_raw_job(os.path.join(TRACEIO, "c1_gpt2_2r", "job.manifest"), _cluster(1, 2))
    eng = Engine(0)
    r = eng.simulate([raw])[0]
    eng.close()
    assert int(r["status"]) == 0
    assert int(r["total_ns"]) == 9846585
    assert int(r["peak_mem_bytes"]) == 4822794240
