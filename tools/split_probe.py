"""Per-phase timings of the C2 step (engine events + a step event pair), for
comparing scheduler launch layouts: MAYA_SPLIT_SMEM=T python tools/split_probe.py"""
import os, sys, time, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.engine import Engine
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
eng = Engine(0)
eng.stage_generated(model, cfgs, cluster, dispatch_overhead_ns=5000, threads=16)
eng.upload()
st = eng.batch_stats()
ph, host, tot = [], [], []
for i in range(15):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.run()
    t1 = time.perf_counter()
    eng.topk(8)
    t2 = time.perf_counter()
    if i >= 3:
        ph.append(eng.last_timings_ms()); host.append((t1 - t0) * 1e3); tot.append((t2 - t0) * 1e3)
med = lambda xs: round(statistics.median(xs), 4)
print(os.environ.get("MAYA_SPLIT_SMEM"), "phases", [med([p[k] for p in ph]) for k in range(3)],
      "host enqueue ms", med(host), "run+topk wall ms", med(tot), "launches", st["run_launches"])
