"""Run one C2 config (or a label filter) repeatedly; for ncu source profiles."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.engine import Engine
label = sys.argv[1] if len(sys.argv) > 1 else "tp1.pp1.mm8.vs1.rsz"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = [c for c in W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
        if c.label() == label]
eng = Engine(0, sched=os.environ.get("SCHED", "auto"), blocks=os.environ.get("BLOCKS", "1") == "1")
eng.stage_generated(model, cfgs, cluster, dispatch_overhead_ns=5000)
print(eng.batch_stats())
eng.upload()
for _ in range(reps):
    eng.run(); r = eng.results()
    print(label, eng.last_timings_ms(), r["total_ns"], r["rounds"])
