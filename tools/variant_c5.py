"""C5 scheduler time with an alternative build of the engine (tuning experiments)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20191_b200 import engine as E
E.LIB_PATH = E.LIB_PATH.replace("libmaya_b200.so", sys.argv[1])
import numpy as np
from paper_2503_20191_b200.synth import c5_job
eng = E.Engine(0)
for spec in sys.argv[2:]:
    R, n, B = (int(x) for x in spec.split("x"))
    jobs = [c5_job(R, n, cfg=c) for c in range(min(B, 64))]
    eng.load([jobs[c % len(jobs)] for c in range(B)], threads=16)
    ts = []
    for _ in range(5):
        eng.run(); r = eng.results(); ts.append(eng.last_timings_ms()[2])
    st = eng.batch_stats()
    alg = 16 * st["rep_events"] + 4 * st["rank_comms"] + 16 * (st["features"] + st["slots"]) + 24 * st["jobs"]
    ms = float(np.median(ts[2:]))
    print(sys.argv[1], spec, f"sched {ms:.3f} ms -> {alg/ms/1e6:.0f} GB/s ({alg/ms/1e6/6650*100:.1f}%) ok {(r['status']==0).sum()}", flush=True)
