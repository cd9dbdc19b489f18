"""Run C2 configs selected by label (or 'all') a few times on one engine, for
ncu captures of one scheduler.  SCHED=auto|lane|warp picks the kernel.

    python tools/one_c2.py tp1.pp8.mm8.vs1.r-- [runs]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.engine import Engine

lab = sys.argv[1]
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
sub = cfgs if lab == "all" else [c for c in cfgs if c.label() == lab]
eng = Engine(0, sched=os.environ.get("SCHED", "auto"))
eng.stage_generated(model, sub, cluster, dispatch_overhead_ns=5000, threads=8)
eng.upload()
for _ in range(runs):
    eng.run()
    r = eng.results()
print(lab, len(sub), "sched ms", eng.last_timings_ms(), "total_ns", r["total_ns"][:4])
