"""Golden fixtures for the batched search runner, made by
running the REAL reference's run_search in this container:

    python tests/golden/make_search_golden.py [--ref /root/reference/pkg]

The evaluator is the reference's own C2 results (c2_results.json: every one of
the 512 configs evaluated by dltsim's PipelineEvaluator), served from a table,
with MFU from dltsim's compute_mfu; a few keys raise to exercise INVALID.  For
each scenario (strategy x tactics x stop rule x max_trials x jobs) the file
stores the reference's trial sequence, ranking and early-stop flag.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

SCENARIOS = [
    {"name": "grid_tactics", "strategy": "grid", "seed": 0, "tactics": True, "stop": None,
     "max_trials": None, "jobs": 1, "deterministic": False},
    {"name": "grid_plain", "strategy": "grid", "seed": 0, "tactics": False, "stop": None,
     "max_trials": None, "jobs": 1, "deterministic": False},
    {"name": "random_stop", "strategy": "random", "seed": 3, "tactics": True, "stop": [20, 5],
     "max_trials": None, "jobs": 1, "deterministic": False},
    {"name": "random_max", "strategy": "random", "seed": 11, "tactics": True, "stop": None,
     "max_trials": 100, "jobs": 1, "deterministic": False},
    {"name": "evolutionary", "strategy": "evolutionary", "seed": 5, "tactics": True,
     "stop": None, "max_trials": None, "jobs": 1, "deterministic": False},
    {"name": "evolutionary_stop", "strategy": "evolutionary", "seed": 7, "tactics": True,
     "stop": [30, 5], "max_trials": None, "jobs": 1, "deterministic": False},
    {"name": "grid_jobs4_det", "strategy": "grid", "seed": 0, "tactics": True, "stop": None,
     "max_trials": None, "jobs": 4, "deterministic": True},
]


def bad_key(key) -> bool:
    """Configs whose evaluation raises (INVALID trials)."""
    tp, pp, mm, vs = key[:4]
    return tp == 2 and pp == 4 and mm == 6


class TableEvaluator:
    """Picklable evaluator (run_search with jobs > 1 uses a process pool)."""

    def __init__(self, results):
        self.results = results

    def __call__(self, config):
        k = config.key()
        if bad_key(k):
            raise ValueError(f"synthetic failure for {config.label()}")
        return self.results[k]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    args = ap.parse_args()
    sys.path.insert(0, os.path.join(args.ref, "src"))
    from dltsim.cluster import ClusterSpec, load_device_preset
    from dltsim.search import (EvalResult, SearchSpace, StopRule, make_strategy, run_search)
    from dltsim.sim import SimReport, compute_mfu
    from dltsim.workload import ModelSpec

    model = ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
    cluster = ClusterSpec(1, 8, 80 * 2 ** 30, load_device_preset("fast"))
    table = {tuple(r["key"]): r for r in json.load(open(os.path.join(HERE, "c2_results.json")))}
    results = {}
    for key, r in table.items():
        rep = SimReport(total_ns=r["total_ns"], per_rank={}, oom=r["oom"], first_oom=None,
                        dispatched_ops=0, completed_ops=0)
        mfu = compute_mfu(rep, model.iteration_flops(key[7]), cluster, model.dtype)
        results[key] = EvalResult(r["total_ns"], mfu, r["peak_mem_bytes"], r["oom"])

    evaluator = TableEvaluator(results)

    space = SearchSpace(global_batch=512)
    out = {"evals": [[list(k), v.time_ns, v.mfu, v.peak_mem_bytes, v.oom]
                     for k, v in sorted(results.items())], "scenarios": []}
    for sc in SCENARIOS:
        stop = StopRule(*sc["stop"]) if sc["stop"] else None
        res = run_search(space, evaluator, make_strategy(sc["strategy"], sc["seed"]), model,
                         cluster, jobs=sc["jobs"], use_tactics=sc["tactics"], stop=stop,
                         max_trials=sc["max_trials"], deterministic=sc["deterministic"])

        def rec(t):
            return [list(t.config.key()), t.status.value, t.time_ns, t.mfu, t.peak_mem_bytes,
                    t.provenance, t.tactic, list(t.premise.key()) if t.premise else None,
                    t.error]
        out["scenarios"].append(dict(sc, trials=[rec(t) for t in res.trials],
                                     ranked=[list(t.config.key()) for t in res.ranked],
                                     stopped_early=res.stopped_early))
        print(sc["name"], len(res.trials), "trials, stopped", res.stopped_early,
              "best", res.best.config.key() if res.best else None)
    with open(os.path.join(HERE, "search_golden.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    sys.modules.setdefault("make_search_golden", sys.modules["__main__"])
    main()
