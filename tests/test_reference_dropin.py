"""The drop-in driven by the REAL reference objects (oracle/_ref/dltsim, the
unmodified reference copied by oracle/Makefile `ref`; it travels to the GPU
box with the snapshot).

* run_search (search.py:381-444) with GpuPipelineEvaluator produces the same
  trial records -- statuses, times, MFU, peak memory, pruning provenance,
  error strings -- as with the reference's own PipelineEvaluator, for three
  strategies;
* a TableEstimator trained with profile_mode_annotate (workload.py:815-835)
  gives the same EvalResults on both evaluators (host-estimator path: the
  reference's annotate with full KernelAttrs incl. dims, then the device);
* a device without a peak for the model dtype gives the reference's
  EstimationError text on the device-roofline path;
* api.simulate on real AnnotatedJobs equals dltsim.simulate (report fields,
  per-rank stats, timeline), and raises the reference's SimDeadlockError text.

Each comparison runs the reference here, live (CPU), beside the engine.
"""
import hashlib
import os
import sys

import pytest

from conftest import REPO

REF = os.path.join(REPO, "oracle", "_ref")


def _ref():
    if not os.path.isdir(os.path.join(REF, "dltsim")):
        pytest.skip("oracle/_ref not built (make -C oracle ref where /root/reference exists)")
    for p in (REF, os.path.join(REF, "reftests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import dltsim  # noqa: F401
    return dltsim


def test_reference_copy_is_unmodified():
    _ref()
    man = os.path.join(REF, "MANIFEST.sha256")
    with open(man) as f:
        rows = [ln.split() for ln in f if ln.strip()]
    assert rows
    for digest, rel in rows:
        with open(os.path.join(REF, rel), "rb") as g:
            assert hashlib.sha256(g.read()).hexdigest() == digest, rel
        src = os.path.join("/root/reference/pkg/src" if rel.startswith("dltsim")
                           else "/root/reference/pkg/tests", rel.split("/", 1)[1]
                           if rel.startswith("reftests") else rel)
        if os.path.exists(src):   # build container: byte-identical to the reference
            with open(src, "rb") as g:
                assert hashlib.sha256(g.read()).hexdigest() == digest, rel


def _small():
    from dltsim.cluster import ClusterSpec, load_device_preset
    from dltsim.workload import ModelSpec
    model = ModelSpec("t", num_layers=8, hidden_size=128, seq_len=64, vocab_size=512)
    cluster = ClusterSpec(2, 8, 2 * 2 ** 30, load_device_preset("fast"))
    return model, cluster


def _trials(result):
    return [(t.config, t.status, t.time_ns, t.mfu, t.peak_mem_bytes, t.provenance, t.tactic,
             t.premise, t.error) for t in result.trials]


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["grid", "random", "evolutionary"])
def test_run_search_with_gpu_evaluator_equals_reference(strategy):
    _ref()
    from dltsim.estimate import RooflineEstimator
    from dltsim.search import (PipelineEvaluator, SearchSpace, StopRule, enumerate_space,
                               make_strategy, run_search)
    from paper_2503_20191_b200.api import GpuPipelineEvaluator
    model, cluster = _small()
    space = SearchSpace(global_batch=32)
    ref_ev = PipelineEvaluator(model, cluster, RooflineEstimator(), dispatch_overhead_ns=2000)
    gpu_ev = GpuPipelineEvaluator(model, cluster, RooflineEstimator(), dispatch_overhead_ns=2000)
    gpu_ev.prefetch(enumerate_space(space, model, cluster))   # one GPU batch
    kw = dict(jobs=1, use_tactics=True, stop=StopRule(window=40, top_k=3))
    want = run_search(space, ref_ev, make_strategy(strategy, seed=7), model, cluster, **kw)
    got = run_search(space, gpu_ev, make_strategy(strategy, seed=7), model, cluster, **kw)
    assert _trials(got) == _trials(want)
    assert [t.config for t in got.ranked] == [t.config for t in want.ranked]
    assert got.best.config == want.best.config
    assert got.stopped_early == want.stopped_early


@pytest.mark.gpu
def test_table_estimator_path_equals_reference():
    _ref()
    from dltsim.estimate import RooflineEstimator, TableEstimator, ProfileTable, roofline_estimate
    from dltsim.search import PipelineEvaluator, SearchSpace, enumerate_space
    from dltsim.workload import default_schedule, generate_representatives, profile_mode_annotate
    from paper_2503_20191_b200.api import GpuPipelineEvaluator
    model, cluster = _small()
    dev = cluster.device
    eff = {"gemm": 0.37, "layernorm": 0.61, "softmax": 0.5, "gelu": 0.73, "add": 0.8}

    def oracle(op, attrs):
        return roofline_estimate(op, attrs, dev, efficiency=eff, overhead_ns=1700)
    configs = enumerate_space(SearchSpace(global_batch=32), model, cluster)
    table = ProfileTable()
    for cfg in configs[::9]:           # profile a subset: the rest interpolates
        traces, _ = generate_representatives(model, cfg, cluster, default_schedule(cfg),
                                             dispatch_overhead_ns=2000)
        for tr in traces:
            for row in profile_mode_annotate(tr, oracle, dev.name).rows:
                table.add(row)
    est = TableEstimator(table, RooflineEstimator(overhead_ns=900))
    ref_ev = PipelineEvaluator(model, cluster, est, dispatch_overhead_ns=2000)
    gpu_ev = GpuPipelineEvaluator(model, cluster, est, dispatch_overhead_ns=2000)
    sample = configs[::3]
    got = gpu_ev.evaluate_many(sample)
    for cfg, g in zip(sample, got):
        assert g == ref_ev(cfg), cfg


@pytest.mark.gpu
def test_estimation_error_text_equals_reference():
    _ref()
    from dltsim.cluster import ClusterSpec, DeviceClass, LinkClass
    from dltsim.estimate import RooflineEstimator
    from dltsim.search import PipelineEvaluator, SearchSpace, enumerate_space
    from paper_2503_20191_b200.api import GpuPipelineEvaluator
    model, cl = _small()
    d = cl.device
    nobf16 = DeviceClass("nobf16", {"fp32": 10 ** 14}, d.hbm_bytes_per_s,
                         {"intra_host": LinkClass(1000, 10 ** 11),
                          "inter_host": LinkClass(5000, 10 ** 10)})
    cluster = ClusterSpec(2, 8, 2 * 2 ** 30, nobf16)
    configs = enumerate_space(SearchSpace(global_batch=32), model, cluster)[::11]
    ref_ev = PipelineEvaluator(model, cluster, RooflineEstimator(), dispatch_overhead_ns=2000)
    got = GpuPipelineEvaluator(model, cluster, RooflineEstimator(),
                               dispatch_overhead_ns=2000).evaluate_many(configs)
    for cfg, g in zip(configs, got):
        with pytest.raises(Exception) as ei:
            ref_ev(cfg)
        assert isinstance(g, Exception), cfg
        assert type(g).__name__ == type(ei.value).__name__
        assert str(g) == str(ei.value), cfg


def _annotated_jobs():
    from dltsim.cluster import ClusterSpec, load_device_preset
    from dltsim.collate import collate
    from dltsim.estimate import RooflineEstimator, annotate
    from dltsim.search import SearchSpace, enumerate_space
    from dltsim.workload import ModelSpec, default_schedule, generate_representatives
    out = []
    model, cluster = _small()
    for cfg in enumerate_space(SearchSpace(global_batch=32), model, cluster)[::23]:
        tr, ex = generate_representatives(model, cfg, cluster, default_schedule(cfg),
                                          dispatch_overhead_ns=2000)
        out.append((annotate(collate(tr, ex, cluster), RooflineEstimator()), None))
    m = ModelSpec("gpt2-small", 12, 768, 1024, 50304, "bf16")
    c = ClusterSpec(1, 2, 80 * 2 ** 30, load_device_preset("fast"))
    cfg = enumerate_space(SearchSpace(global_batch=8), m, c)[0]
    tr, ex = generate_representatives(m, cfg, c, default_schedule(cfg), dispatch_overhead_ns=5000)
    ann = annotate(collate(tr, ex, c), RooflineEstimator())
    out.append((ann, None))
    out.append((ann, ClusterSpec(1, 2, 3 * 2 ** 30, load_device_preset("fast"))))  # OOM override
    return out


@pytest.mark.gpu
def test_api_simulate_on_reference_annotated_jobs():
    _ref()
    from dltsim.sim import simulate as ref_simulate
    from paper_2503_20191_b200 import api
    for ann, cluster in _annotated_jobs():
        want = ref_simulate(ann, cluster, record_timeline=True)
        got = api.simulate(ann, cluster, record_timeline=True)
        assert type(got).__name__ == "SimReport"
        for k in ("total_ns", "oom", "first_oom", "dispatched_ops", "completed_ops",
                  "peak_mem_bytes", "exposed_comm_ns"):
            assert getattr(got, k) == getattr(want, k), k
        assert got.per_rank == want.per_rank
        assert sorted(got.timeline) == sorted(want.timeline)


@pytest.mark.gpu
def test_api_simulate_raises_reference_deadlock():
    _ref()
    from builders import FixedEstimator, toy_cluster
    from dltsim.collate import collate
    from dltsim.estimate import annotate
    from dltsim.sim import SimDeadlockError, simulate as ref_simulate
    from dltsim.trace import Collective, CommInit, WorkerTrace
    from paper_2503_20191_b200 import api
    cluster = toy_cluster(1, 2)
    mk = lambda rank, order: WorkerTrace(rank, 0, rank, (   # noqa: E731 (test_sim.py:191-200)
        CommInit("x", 2, rank), CommInit("y", 2, rank),
        Collective(0, order[0], 0, "AllReduce", 8, 2),
        Collective(0, order[1], 0, "AllReduce", 8, 2),
    ))
    ann = annotate(collate([mk(0, ("x", "y")), mk(1, ("y", "x"))], {}, cluster),
                   FixedEstimator({}, coll_ns=10))
    with pytest.raises(SimDeadlockError) as want:
        ref_simulate(ann)
    with pytest.raises(SimDeadlockError) as got:
        api.simulate(ann)
    assert str(got.value) == str(want.value)


@pytest.mark.gpu
def test_search_run_search_delegates_to_reference_runner():
    """search.run_search with the reference's own strategy objects runs the
    reference's runner (strategies, tactics, early stop, ranking) over one
    engine batch, and equals the reference run with its own evaluator."""
    _ref()
    from dltsim.estimate import RooflineEstimator
    from dltsim.search import (PipelineEvaluator, SearchSpace, StopRule, make_strategy,
                               run_search as ref_run_search)
    from paper_2503_20191_b200 import search as S
    from paper_2503_20191_b200.api import GpuPipelineEvaluator
    model, cluster = _small()
    space = SearchSpace(global_batch=32)
    for name in ("grid", "evolutionary"):
        want = ref_run_search(space, PipelineEvaluator(model, cluster, RooflineEstimator(), 2000),
                              make_strategy(name, seed=3), model, cluster,
                              stop=StopRule(window=30, top_k=3))
        got = S.run_search(space, GpuPipelineEvaluator(model, cluster, RooflineEstimator(), 2000),
                           make_strategy(name, seed=3), model, cluster,
                           stop=StopRule(window=30, top_k=3))
        assert type(got).__module__.startswith("dltsim")
        assert _trials(got) == _trials(want)
