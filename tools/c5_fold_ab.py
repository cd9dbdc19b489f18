"""C5 step with and without run folding (resolve pass + unfolded lane scheduler)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20191_b200.synth import c5_job
from paper_2503_20191_b200.engine import Engine
R, n, B = (int(x) for x in sys.argv[1].split("x"))
jobs = [c5_job(R, n, cfg=c) for c in range(min(B, 64))]
for fold in (True, False):
    eng = Engine(0, fold=fold)
    eng.load([jobs[c % len(jobs)] for c in range(B)], threads=16)
    for _ in range(3):
        eng.run(); r = eng.results()
    t = eng.last_timings_ms()
    print(sys.argv[1], "fold" if fold else "nofold", [round(x, 3) for x in t], round(sum(t), 3), int(r["status"].max()), int(r["total_ns"].sum() % 1000003), flush=True)
    eng.close()
