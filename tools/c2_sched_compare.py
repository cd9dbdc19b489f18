"""C2 step under each scheduler choice (auto / forced lane / forced warp):
per-phase device ms (estimators, fold, schedulers), results compared.

    python tools/c2_sched_compare.py [runs]
"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.engine import Engine

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 10
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
out = {}
ref = None
for sched in ("auto", "nochain", "lane", "warp"):
    eng = Engine(0, collapse=True, sched=sched)
    eng.stage_generated(model, cfgs, cluster, dispatch_overhead_ns=5000, threads=16)
    eng.upload()
    ts = []
    for _ in range(runs):
        eng.run()
        r = eng.results()
        ts.append(eng.last_timings_ms())
    tot = np.array([x["total_ns"] for x in r]) if isinstance(r, list) else r["total_ns"].copy()
    if ref is None:
        ref = tot
    ts = np.array(ts)
    out[sched] = {"ms_median": [round(float(v), 4) for v in np.median(ts, axis=0)],
                  "ms_min": [round(float(v), 4) for v in ts.min(axis=0)],
                  "equal_to_auto": bool(np.array_equal(tot, ref))}
    print(sched, json.dumps(out[sched]), flush=True)
    del eng
print(json.dumps(out))
