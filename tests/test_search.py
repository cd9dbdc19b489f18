"""Batched search runner (search.py) against the reference's run_search.

tests/golden/search_golden.json holds dltsim.search.run_search's own trial
sequences for seven scenarios (grid / random / evolutionary strategies,
tactics on and off, early stopping, max_trials, jobs=4 batches), driven by the
reference's evaluator results for the C2 lattice (make_search_golden.py).  The
CPU tests replay them with the same table evaluator; the GPU test evaluates
every trial on the engine (bulk speculative batches) and must reproduce them.
"""
import json
import os

import pytest

from conftest import GOLDEN


def _golden():
    return json.load(open(os.path.join(GOLDEN, "search_golden.json")))


def _bad(key) -> bool:          # tests/golden/make_search_golden.py: bad_key
    tp, pp, mm, vs = key[:4]
    return tp == 2 and pp == 4 and mm == 6


class TableEvaluator:
    def __init__(self, evals):
        from paper_2503_20191_b200.api import EvalResult
        self.results = {tuple(k): EvalResult(t, m, p, o) for k, t, m, p, o in evals}

    def __call__(self, config):
        k = config.key()
        if _bad(k):
            raise ValueError(f"synthetic failure for {config.label()}")
        return self.results[k]


def _setup():
    from paper_2503_20191_b200 import workload as W
    model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
    cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
    return W, model, cluster


def _run(sc, evaluator):
    from paper_2503_20191_b200 import search as S
    W, model, cluster = _setup()
    stop = S.StopRule(*sc["stop"]) if sc["stop"] else None
    return S.run_search(W.SearchSpace(global_batch=512), evaluator,
                        S.make_strategy(sc["strategy"], sc["seed"]), model, cluster,
                        jobs=sc["jobs"], use_tactics=sc["tactics"], stop=stop,
                        max_trials=sc["max_trials"], deterministic=sc["deterministic"])


def _rows(res):
    return [[list(t.config.key()), t.status.value, t.time_ns, t.mfu, t.peak_mem_bytes,
             t.provenance, t.tactic, list(t.premise.key()) if t.premise else None, t.error]
            for t in res.trials]


def _check(sc, res):
    got = _rows(res)
    assert len(got) == len(sc["trials"]), (sc["name"], len(got), len(sc["trials"]))
    for i, (a, b) in enumerate(zip(got, sc["trials"])):
        assert a == b, (sc["name"], i, a, b)
    assert [list(t.config.key()) for t in res.ranked] == sc["ranked"], sc["name"]
    assert res.stopped_early == sc["stopped_early"], sc["name"]


@pytest.mark.parametrize("i", range(7))
def test_run_search_matches_reference(i):
    g = _golden()
    sc = g["scenarios"][i]
    _check(sc, _run(sc, TableEvaluator(g["evals"])))


def test_tactics_and_stop_exercised():
    g = _golden()
    tactics = {t[6] for sc in g["scenarios"] for t in sc["trials"] if t[6]}
    assert {"oom-without-seq-parallel", "dist-optimizer-runtime",
            "more-microbatches-runtime"} <= tactics
    assert any(sc["stopped_early"] for sc in g["scenarios"])
    assert any(t[1] == "invalid" for t in g["scenarios"][0]["trials"])


class GpuTable:
    """The engine's results for the 512 golden configs; the same failures as
    the golden evaluator elsewhere (KeyError beyond the table, synthetic ones)."""

    def __init__(self, evals):
        from paper_2503_20191_b200.api import GpuPipelineEvaluator
        W, model, cluster = _setup()
        self.keys = {tuple(k) for k, *_ in evals}
        self.gpu = GpuPipelineEvaluator(model, cluster, dispatch_overhead_ns=5000)
        self.calls = 0

    def _fail(self, config):
        k = config.key()
        if _bad(k):
            return ValueError(f"synthetic failure for {config.label()}")
        if k not in self.keys:
            return KeyError(k)
        return None

    def evaluate_many(self, configs):
        self.calls += 1
        ok = [c for c in configs if self._fail(c) is None]
        res = dict(zip([c.key() for c in ok], self.gpu.evaluate_many(ok)))
        return [self._fail(c) or res[c.key()] for c in configs]

    def __call__(self, config):
        r = self.evaluate_many([config])[0]
        if isinstance(r, Exception):
            raise r
        return r


@pytest.mark.gpu
@pytest.mark.parametrize("i", [0, 2, 4, 6])
def test_run_search_on_gpu_matches_reference(i):
    g = _golden()
    sc = g["scenarios"][i]
    ev = GpuTable(g["evals"])
    _check(sc, _run(sc, ev))
    # bulk: grid / random in one engine batch, evolutionary one batch per population
    if sc["strategy"] != "evolutionary":
        assert ev.calls == 1


def _cma(evaluator):
    from paper_2503_20191_b200 import search as S
    W, model, cluster = _setup()
    return S.cma_search(W.SearchSpace(global_batch=512), evaluator, model, cluster,
                        popsize=64, generations=10, seed=1)


def test_cma_search_finds_the_best_region():
    g = _golden()
    gens = _cma(TableEvaluator(g["evals"]))
    assert len(gens) == 10
    ranked = sorted(((m, tuple(k)) for k, t, m, p, o in g["evals"] if not o and not _bad(k)),
                    key=lambda x: (-x[0], x[1]))
    top = {k for _, k in ranked[:10]}
    assert gens[-1].best.key() in top
    assert gens[-1].best_mfu == pytest.approx(max(m for m, _ in ranked), rel=0.02)


@pytest.mark.gpu
def test_cma_search_on_gpu_follows_the_same_trajectory():
    g = _golden()
    a = _cma(TableEvaluator(g["evals"]))
    b = _cma(GpuTable(g["evals"]))
    for x, y in zip(a, b):
        assert [c.key() for c in x.configs] == [c.key() for c in y.configs]
        assert x.mfu == y.mfu
        assert x.best.key() == y.best.key()
