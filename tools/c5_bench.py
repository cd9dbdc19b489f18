"""C5 synthetic sweep: scheduler time, HBM GB/s, parity vs the oracle (sampled).

    python tools/c5_bench.py [RxNxB ...]      (env SCHED=lane|warp|both, default both)
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2503_20191_b200.synth import c5_job
from paper_2503_20191_b200.engine import Engine

sizes = [(8, 10000, 64), (64, 10000, 16), (8, 100000, 16), (512, 1000, 16), (64, 100000, 2),
         (8, 10000, 1024)]
if len(sys.argv) > 1:
    sizes = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1:]]
scheds = {"both": ["auto", "warp"]}.get(os.environ.get("SCHED", "both"), [os.environ.get("SCHED")])
eng = Engine(0)
peak = 6650.0
for R, n, B in sizes:
    t = time.time()
    jobs = [c5_job(R, n, cfg=c) for c in range(min(B, 64))]
    jobs = [jobs[c % len(jobs)] for c in range(B)]
    tg = time.time() - t
    for sched in scheds:
        eng.set_sched(sched)
        eng.load(jobs, threads=16)
        st = eng.batch_stats()
        for _ in range(2):
            eng.run(); r = eng.results()
        ts = []
        for _ in range(5):
            eng.run(); r = eng.results(); ts.append(eng.last_timings_ms())
        est, mem, sched_ms = [float(np.median(x)) for x in zip(*ts)]
        alg = 16 * st["rep_events"] + 4 * st["rank_comms"] + 16 * (st["features"] + st["slots"]) + 24 * st["jobs"]
        ok = int((r["status"] == 0).sum())
        from oracle import oracle
        bad = 0
        for j in range(min(2, B)):
            o = oracle.simulate(jobs[j])
            bad += int(o["total_ns"] != int(r["total_ns"][j]) or o["peak_mem_bytes"] != int(r["peak_mem_bytes"][j]))
        print(f"C5[{sched}] R={R} n={n} B={B}: events {st['rep_events']/1e6:.1f}M dev_ops {st['device_ops']/1e6:.1f}M "
              f"sched {sched_ms:.3f} ms (est {est:.3f}, mem+resolve {mem:.3f}) -> {alg/sched_ms/1e6:.0f} GB/s alg "
              f"({alg/sched_ms/1e6/peak*100:.1f}% of {peak}), rank-ops/s {st['rank_ops']/sched_ms*1e3:.3g}, "
              f"ok {ok}/{B}, oracle mismatches {bad}, rounds {int(r['rounds'].max())}, gen {tg:.1f}s", flush=True)
