"""C2 e2e through api.GenPipeline.evaluate_stream (K steps after 3 warm-up steps), ms/step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200 import api
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
kr = api.key_ranks(cfgs)
th = int(os.environ.get("GEN_THREADS", len(os.sched_getaffinity(0))))
pipe = api.GenPipeline(0)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for _ in pipe.evaluate_stream(model, [cfgs] * 3, cluster, k=8, key_orders=[kr] * 3, dispatch_overhead_ns=5000, threads=th):
    pass
out = []
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in pipe.evaluate_stream(model, [cfgs] * K, cluster, k=8, key_orders=[kr] * K, dispatch_overhead_ns=5000, threads=th):
        pass
    torch.cuda.synchronize()
    out.append((time.perf_counter() - t0) * 1000 / K)
print(os.environ.get("MAYA_COPY_THREADS", "default"), "gen", th, "ms/step", [round(x, 3) for x in out], "configs/s", round(512 / min(out) * 1000))
