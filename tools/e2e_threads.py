"""C2 e2e (GenPipeline stream) ms/step per generation thread count, interleaved rounds."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200 import api
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
kr = api.key_ranks(cfgs)
pipe = api.GenPipeline(0)
K = 20
settings = [int(x) for x in sys.argv[1].split(",")]
res = {t: [] for t in settings}
for _ in pipe.evaluate_stream(model, [cfgs] * 3, cluster, k=8, key_orders=[kr] * 3, dispatch_overhead_ns=5000, threads=16):
    pass
for rnd in range(5):
    for th in settings:
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in pipe.evaluate_stream(model, [cfgs] * K, cluster, k=8, key_orders=[kr] * K, dispatch_overhead_ns=5000, threads=th):
            pass
        torch.cuda.synchronize()
        res[th].append((time.perf_counter() - t0) * 1000 / K)
for th in settings:
    v = sorted(res[th])
    print(th, "threads: median", round(v[len(v) // 2], 3), "ms/step, all", [round(x, 2) for x in res[th]])
