"""The UNMODIFIED reference (oracle/_ref/dltsim, copied from /root/reference by
oracle/Makefile `ref`) timed on the host cores -- TEST / MEASUREMENT
INFRASTRUCTURE ONLY.  Used by bench.py's reference arm (--impl reference) and
its cpu_baseline leg; never by the product.

Nothing here imports paper_2503_20191_b200 (the engine's .so stays unloaded in
these processes): the workload is built with the reference's own
enumerate_space, and the two legs are the reference's own calls
(BASELINE.md §3):

* e2e      -- PipelineEvaluator.__call__(config)        search.py:200-209
              (generate -> collate -> annotate -> simulate -> compute_mfu)
* sim-only -- simulate(annotate(job, RooflineEstimator()))  sim.py:476-485,
              estimate.py:329-361, on jobs generated + collated before the
              timed region.

Throughput mode runs N forked worker processes (N = host cores), each with a
fixed shard of the sample; one pass = every worker evaluates its shard, timed
from the start signal to the last worker's completion.
"""
from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")

C2_MODEL = ("gpt3-1.3b", 24, 2048, 2048, 51200, "bf16")


def available() -> str | None:
    """None when the reference copy is importable, else why not."""
    if not os.path.isdir(os.path.join(REF, "dltsim")):
        return "oracle/_ref/dltsim missing (run `make -C oracle ref` where /root/reference exists)"
    return None


def _ref_path():
    if REF not in sys.path:
        sys.path.insert(0, REF)


def c2_workload():
    """BASELINE C2 with the reference's own API: (model, cluster, configs[:512])."""
    _ref_path()
    from dltsim.cluster import ClusterSpec, load_device_preset
    from dltsim.search import SearchSpace, enumerate_space
    from dltsim.workload import ModelSpec
    model = ModelSpec(*C2_MODEL)
    cluster = ClusterSpec(1, 8, 80 * 2 ** 30, load_device_preset("fast"))
    return model, cluster, enumerate_space(SearchSpace(global_batch=512), model, cluster)[:512]


def _worker(conn, mode: str, idx: list):
    _ref_path()
    from dltsim.collate import collate
    from dltsim.estimate import RooflineEstimator, annotate
    from dltsim.search import PipelineEvaluator
    from dltsim.sim import simulate
    from dltsim.workload import default_schedule, generate_representatives
    model, cluster, configs = c2_workload()
    cfgs = [configs[i] for i in idx]
    est = RooflineEstimator()
    jobs = None
    if mode == "sim":   # generation + collation outside the timed region
        jobs = []
        for c in cfgs:
            tr, ex = generate_representatives(model, c, cluster, default_schedule(c),
                                              dispatch_overhead_ns=5000)
            jobs.append(collate(tr, ex, cluster))
    ev = PipelineEvaluator(model, cluster, est, dispatch_overhead_ns=5000)
    conn.send("ready")
    while True:
        msg = conn.recv()
        if msg == "stop":
            break
        out = []
        if mode == "sim":
            for j in jobs:
                rep = simulate(annotate(j, est))
                out.append((rep.total_ns, rep.peak_mem_bytes, rep.oom))
        else:
            for c in cfgs:
                r = ev(c)
                out.append((r.time_ns, r.peak_mem_bytes, r.oom))
        conn.send(out)
    conn.close()


class Pool:
    """N persistent forked workers with fixed shards of `idx` (round-robin)."""

    def __init__(self, mode: str, idx: list, n: int):
        ctx = mp.get_context("fork")
        self.n = max(1, min(n, len(idx)))
        self.shards = [idx[w::self.n] for w in range(self.n)]
        self.conns, self.procs = [], []
        for w in range(self.n):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_worker, args=(b, mode, self.shards[w]), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        for c in self.conns:
            assert c.recv() == "ready"

    def run_pass(self):
        """-> (seconds, {config index: (time_ns, peak, oom)})"""
        t0 = time.perf_counter()
        for c in self.conns:
            c.send("go")
        res = {}
        for w, c in enumerate(self.conns):
            for i, r in zip(self.shards[w], c.recv()):
                res[i] = r
        return time.perf_counter() - t0, res

    def close(self):
        for c in self.conns:
            c.send("stop")
        for p in self.procs:
            p.join(timeout=10)


def sample_indices(k: int, n_total: int = 512) -> list:
    """k configs spread evenly over the 512 C2 configs (enumeration order)."""
    k = max(1, min(k, n_total))
    return sorted({(q * n_total) // k for q in range(k)})


def parity(res: dict) -> dict:
    """The reference arm's own results against the committed reference goldens
    (tests/golden/c2_results.json, made in the build container)."""
    path = os.path.join(os.path.dirname(HERE), "tests", "golden", "c2_results.json")
    try:
        with open(path) as f:
            gold = json.load(f)
    except OSError:
        return {"checked": 0}
    bad = sum(1 for i, (t, p, o) in res.items()
              if (gold[i]["total_ns"], gold[i]["peak_mem_bytes"], gold[i]["oom"]) != (t, p, o))
    return {"checked": len(res), "mismatches": bad}


def _sample_weight(idx: list):
    """Mean rank-ops of the sampled configs over the mean of all 512 (from the
    committed reference goldens): > 1 means the sample is heavier than the batch."""
    path = os.path.join(os.path.dirname(HERE), "tests", "golden", "c2_results.json")
    try:
        with open(path) as f:
            gold = json.load(f)
    except OSError:
        return None
    mean_all = sum(r["rank_ops"] for r in gold) / len(gold)
    return round(sum(gold[i]["rank_ops"] for i in idx) / len(idx) / mean_all, 4)


def measure(mode: str, n_workers: int, per_worker: int, passes: int, warmup: int = 1) -> dict:
    """Throughput of one leg: `passes` timed passes of n_workers x per_worker
    configs (after `warmup` untimed passes)."""
    idx = sample_indices(n_workers * per_worker)
    pool = Pool(mode, idx, n_workers)
    try:
        for _ in range(warmup):
            pool.run_pass()
        times, res = [], {}
        for _ in range(passes):
            dt, res = pool.run_pass()
            times.append(dt)
    finally:
        pool.close()
    t = sum(times) / len(times)
    return {"configs_per_s": round(len(idx) / t, 3), "seconds_per_pass": round(t, 4),
            "sample_rank_ops_vs_all_512": _sample_weight(idx),
            "configs_per_pass": len(idx), "workers": pool.n, "passes": passes,
            "times": [round(x, 4) for x in times], "parity": parity(res)}
