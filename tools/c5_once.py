"""One C5 batch, N runs (for ncu captures): python tools/c5_once.py RxNxB [runs] (env SCHED)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20191_b200.synth import c5_job
from paper_2503_20191_b200.engine import Engine
R, n, B = (int(x) for x in sys.argv[1].split("x"))
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
jobs = [c5_job(R, n, cfg=c) for c in range(min(B, 64))]
eng = Engine(0, sched=os.environ.get("SCHED", "auto"))
eng.load([jobs[c % len(jobs)] for c in range(B)], threads=16)
for _ in range(runs):
    eng.run(); r = eng.results()
print(sys.argv[1], eng.last_timings_ms(), int(r["status"].max()))
