"""Pin C3 / C4 at their full rank counts to the REAL reference (container only).

    python tests/golden/make_scale_golden.py [--ref /root/reference/pkg] [--jobs 4]

Writes tests/golden/scale_big_results.json: seeded samples of the BASELINE
C3 lattice (GPT-3 18.4B, act_recompute, global_batch 1024/2048) at 256, 512
and 1,024 ranks (8 configs each) and of the C4 lattice (Llama-3-70B-shaped,
interleaved + sequence parallel) at 512, 1,024 and 2,048 ranks
(6 configs each, global_batch 2,048-16,384), every config <= 50 M rank-ops so
the reference's per-rank op lists (sim.py:135-174) fit in host RAM.  The C4
picks are chosen greedily to cover pp=16, virtual_stages 4/5/10, micro_mult
2-16, act_recompute and dist_optimizer on and off, and every global batch.

For each config the reference runs generate_representatives -> collate ->
annotate(RooflineEstimator) -> simulate (workload.py:571-780, collate.py:256,
estimate.py:329, sim.py:476) in its own process; the row stores total_ns,
peak memory, oom, rank_ops and the digest of the collated job (rawtrace.
raw_digest), exactly as scale_results.json does for 64-256 ranks.

Config SELECTION uses the native generator's rank-op count (a size filter
only); every stored number comes from the reference.
"""
from __future__ import annotations

import argparse
import json
import os
import random
import sys
import time
from concurrent.futures import ProcessPoolExecutor, as_completed

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

C3_MODEL = ("gpt3-18.4b", 40, 6144, 2048, 51200, "bf16")
C4_MODEL = ("llama3-70b-shaped", 80, 8192, 8192, 128256, "bf16")
C4_KNOBS = dict(tp=(1, 2, 4, 8), pp=(2, 4, 8, 16), micro_mult=tuple(range(1, 17)),
                virtual_stages=(2, 4, 5, 10), act_recompute=(True, False), seq_parallel=(True,),
                dist_optimizer=(True, False))
MAX_RANK_OPS = 50_000_000


def _features(tag, cfg, gb):
    f = {f"gb{gb}"}
    if tag == "C4":
        f |= {f"pp{cfg.pp}", f"vs{cfg.virtual_stages}", f"rc{int(cfg.act_recompute)}",
              f"dz{int(cfg.dist_optimizer)}", f"tp{cfg.tp}"}
        f.add("mm1" if cfg.micro_mult == 1 else "mm2-4" if cfg.micro_mult <= 4 else
              "mm5-8" if cfg.micro_mult <= 8 else "mm9-16")
    else:
        f |= {f"pp{cfg.pp}", f"tp{cfg.tp}", f"mm{min(cfg.micro_mult, 4)}",
              f"dz{int(cfg.dist_optimizer)}", f"sp{int(cfg.seq_parallel)}"}
    return f


def pick():
    """(tag, model tuple, ranks, key) picks; seeded, size-filtered, coverage-greedy."""
    from paper_2503_20191_b200 import workload as W
    fast = W.load_device_preset("fast")
    rng = random.Random(20261017)
    picks = []
    plan = [("C3", C3_MODEL, n, (1024, 2048), 8, dict(act_recompute=(True,)))
            for n in (256, 512, 1024)]
    plan += [("C4", C4_MODEL, n, (2048, 4096, 8192, 16384), 6, C4_KNOBS)
             for n in (512, 1024, 2048)]
    for tag, mt, n, gbs, quota, knobs in plan:
        model = W.ModelSpec(*mt)
        c = W.ClusterSpec(n // 8, 8, 80 * 2 ** 30, fast)
        cands = []
        for gb in gbs:
            for cfg in W.enumerate_space(W.SearchSpace(**knobs, global_batch=gb), model, c):
                cands.append((gb, cfg))
        rng.shuffle(cands)
        sized = []
        for gb, cfg in cands:
            if len(sized) >= 40 * quota:
                break
            ops = W.generate_job(model, cfg, c, dispatch_overhead_ns=5000).rank_ops()
            if ops <= MAX_RANK_OPS:
                sized.append((gb, cfg, ops))
        covered = set()
        chosen = []
        for _ in range(quota):
            # first maximal in the seeded shuffle order: random tie-break
            best = max(sized, key=lambda t: len(_features(tag, t[1], t[0]) - covered))
            sized.remove(best)
            covered |= _features(tag, best[1], best[0])
            chosen.append(best)
        for gb, cfg, ops in chosen:
            picks.append((tag, mt, n, list(cfg.key()), ops))
        print(f"{tag} {n}: {[(c.label(), o) for _, c, o in chosen]}", flush=True)
    return picks


def run_one(ref, tag, mt, n, key):
    sys.path.insert(0, os.path.join(ref, "src"))
    from dltsim.cluster import ClusterSpec, load_device_preset
    from dltsim.collate import collate
    from dltsim.estimate import RooflineEstimator, annotate
    from dltsim.sim import simulate
    from dltsim.workload import ConfigPoint, ModelSpec, default_schedule, generate_representatives
    from paper_2503_20191_b200.rawtrace import from_reference, raw_digest
    t0 = time.time()
    m = ModelSpec(*mt)
    c = ClusterSpec(n // 8, 8, 80 * 2 ** 30, load_device_preset("fast"))
    cfg = ConfigPoint(*key)
    tr, ex = generate_representatives(m, cfg, c, default_schedule(cfg), dispatch_overhead_ns=5000)
    job = collate(tr, ex, c)
    digest = raw_digest(from_reference(job))
    rank_ops = sum(len(job.trace_of(r).events) for r in job.all_ranks())
    rep = simulate(annotate(job, RooflineEstimator()))
    return {"set": tag, "model": list(mt), "ranks": n, "key": key, "total_ns": rep.total_ns,
            "peak_mem_bytes": rep.peak_mem_bytes, "oom": rep.oom, "rank_ops": rank_ops,
            "raw_sha256": digest, "ref_seconds": round(time.time() - t0, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default=os.environ.get("MAYA_REF", "/root/reference/pkg"))
    ap.add_argument("--jobs", type=int, default=4)
    args = ap.parse_args()
    picks = pick()
    out = os.path.join(HERE, "scale_big_results.json")
    rows = []
    t0 = time.time()
    # largest first so the pool's tail is short
    picks.sort(key=lambda p: -p[4])
    with ProcessPoolExecutor(args.jobs) as ex:
        futs = {ex.submit(run_one, args.ref, t, m, n, k): (t, n, k) for t, m, n, k, _ in picks}
        for f in as_completed(futs):
            r = f.result()
            rows.append(r)
            print(f"  {r['set']} {r['ranks']} {r['key']}: {r['total_ns']} ns, "
                  f"{r['rank_ops']} rank-ops, {r['ref_seconds']} s "
                  f"({len(rows)}/{len(picks)}, {time.time() - t0:.0f} s)", flush=True)
    rows.sort(key=lambda r: (r["set"], r["ranks"], r["key"]))
    with open(out, "w") as f:
        json.dump(rows, f)
    print(f"wrote {out}: {len(rows)} configs in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
