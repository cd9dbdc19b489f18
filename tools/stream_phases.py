"""Host-side time of each call in the streamed C2 e2e loop (GenPipeline.evaluate_stream)."""
import os, sys, time, statistics
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.api import GenPipeline, key_ranks
from paper_2503_20191_b200 import engine as EN
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
kr = key_ranks(cfgs)
T = {}
def wrap(name):
    f = getattr(EN.Engine, name)
    def g(self, *a, **k):
        t0 = time.perf_counter(); r = f(self, *a, **k)
        T.setdefault(name, []).append((time.perf_counter() - t0) * 1e3); return r
    setattr(EN.Engine, name, g)
for n in ("stage_generated", "upload", "run", "topk_async", "results", "topk"):
    wrap(n)
pipe = GenPipeline(0)
th = len(os.sched_getaffinity(0))
for it in range(2):
    T.clear()
    t0 = time.perf_counter()
    for _ in pipe.evaluate_stream(model, [cfgs] * 20, cluster, k=8, key_orders=[kr] * 20,
                                  dispatch_overhead_ns=5000, threads=th):
        pass
    wall = (time.perf_counter() - t0) * 1e3 / 20
print("threads", th, "ms/step", round(wall, 3),
      {k: round(statistics.median(v), 3) for k, v in T.items()})
