"""The chain scheduler (csrc/sched_chain.cu) against the reference's outputs.

The chain kernel runs latency-bound jobs with the whole job resident in one
CTA's shared memory and one thread per FIFO.  On folded runs it evaluates
macro ops ([WAIT]? [KERN|COLL]? [REC]?, built by chain_macro_kernel); with a
timeline it evaluates one op per step.  The engine picks it per batch
('auto'); these tests check that it is really chosen where expected and that
its results equal the reference's (golden fixtures from pkg/src/dltsim) on
every golden family, folded and with a timeline, deadlocks included, and on
C4-shaped pipelines of up to 256 FIFOs (8 warps).
"""
import json
import os

import numpy as np
import pytest

from paper_2503_20191_b200._abi import STATUS_NAMES

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FAMILIES = ["unit", "syncfree", "multirank", "workload", "synth"]


def _check(res, exps):
    bad = []
    for r, exp in zip(res, exps):
        st = STATUS_NAMES[r["status"]]
        if st != exp["status"]:
            bad.append((exp["name"], st, exp["status"]))
            continue
        if st != "ok":
            continue
        for key in ("total_ns", "peak_mem_bytes"):
            if int(r[key]) != exp[key]:
                bad.append((exp["name"], key, int(r[key]), exp[key]))
        if bool(r["oom"]) != exp["oom"]:
            bad.append((exp["name"], "oom"))
    assert not bad, bad[:10]


@pytest.mark.parametrize("collapse", [True, False])
@pytest.mark.parametrize("timeline", [False, True])
def test_chain_matches_reference(golden, collapse, timeline):
    """Every golden family under 'auto': the small jobs run on the chain kernel
    (macro ops when folded, one op per step with a timeline)."""
    from paper_2503_20191_b200.engine import Engine
    used = 0
    for name in FAMILIES:
        jobs, exps = golden(name)
        e = Engine(0, collapse=collapse, sched="auto")
        try:
            res = e.simulate(jobs, record_timeline=timeline)
            used += e.kernels().count("chain")
        finally:
            e.close()
        _check(res, exps)
    assert used > 100


def test_chain_deadlocks_folded(golden):
    """Deadlocking jobs on the folded (macro-op) path: status deadlock."""
    from paper_2503_20191_b200.engine import Engine
    jobs, exps = golden("deadlock")
    e = Engine(0, sched="auto")
    try:
        res = e.simulate(jobs)
        kinds = e.kernels()
    finally:
        e.close()
    assert kinds.count("chain") >= 50
    assert all(STATUS_NAMES[s] == "deadlock" for s in res["status"])


def test_chain_runs_c2_and_matches_reference():
    """All 512 C2 configs (pipelines: chain-shaped) run on the chain kernel and give the
    reference's results (c2_results.json made by the reference itself)."""
    from paper_2503_20191_b200 import workload as W
    from paper_2503_20191_b200.engine import Engine
    model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
    cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
    cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
    gold = json.load(open(os.path.join(GOLDEN, "c2_results.json")))
    out = {}
    for sched in ("auto", "nochain"):
        e = Engine(0, sched=sched)
        try:
            e.stage_generated(model, cfgs, cluster, dispatch_overhead_ns=5000, threads=8)
            e.upload()
            kinds = e.kernels()
            e.run()
            out[sched] = e.results()
        finally:
            e.close()
        if sched == "auto":
            assert kinds.count("chain") == 512
        else:
            assert "chain" not in kinds
    for sched, res in out.items():
        for r, g in zip(res, gold):
            assert (int(r["total_ns"]), int(r["peak_mem_bytes"]), bool(r["oom"])) == \
                (g["total_ns"], g["peak_mem_bytes"], g["oom"]), sched


def test_chain_declined_for_throughput_jobs():
    """Jobs shaped for lockstep lanes (many balanced FIFOs that block often:
    8-rank x 10k-event per-rank-distinct traces, C5) keep the lane kernel's
    rings, in a large batch or alone; the CPU oracle agrees on the results."""
    from oracle import oracle
    from paper_2503_20191_b200.engine import Engine
    from paper_2503_20191_b200.synth import c5_job
    base = [c5_job(8, 10000, cfg=c) for c in range(4)]
    for jobs in ([base[q % 4] for q in range(256)], base[:2]):
        e = Engine(0, sched="auto")
        try:
            res = e.simulate(jobs)
            kinds = e.kernels()
        finally:
            e.close()
        assert set(kinds) == {"lane"}
        for q in range(min(4, len(jobs))):
            o = oracle.simulate(base[q])
            assert int(res[q]["total_ns"]) == o["total_ns"]
            assert int(res[q]["peak_mem_bytes"]) == o["peak_mem_bytes"]


def test_chain_c4_pipelines_match_reference():
    """C4 lattice configs (Llama-70B shape, 256-2,048 ranks, up to 16 stages x
    10 virtual stages) pinned to the reference (scale_big_results.json /
    scale_results.json, made by pkg/src/dltsim): the ones that fit run on the
    chain kernel with 1-8 warps and give the reference's totals."""
    import json
    from paper_2503_20191_b200 import workload as W
    from paper_2503_20191_b200.engine import Engine
    rows = []
    for name in ("scale_results.json", "scale_big_results.json"):
        path = os.path.join(GOLDEN, name)
        if os.path.exists(path):
            rows += json.load(open(path))
    used = 0
    for r in rows:
        m = W.ModelSpec(*r["model"])
        cl = W.ClusterSpec(r["ranks"] // 8, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
        e = Engine(0, sched="auto")
        try:
            e.stage_generated(m, [W.ConfigPoint(*r["key"])], cl, dispatch_overhead_ns=5000, threads=4)
            e.upload()
            kind = e.kernels()[0]
            e.run()
            res = e.results()[0]
        finally:
            e.close()
        used += kind == "chain"
        assert int(res["total_ns"]) == r["total_ns"], (r["key"], kind)
        assert int(res["peak_mem_bytes"]) == r["peak_mem_bytes"], (r["key"], kind)
    assert used >= 10
