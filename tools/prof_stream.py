import cProfile, pstats, os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.api import GenPipeline, key_ranks
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
kr = key_ranks(cfgs)
pipe = GenPipeline(0)
th = len(os.sched_getaffinity(0))
for _ in pipe.evaluate_stream(model, [cfgs] * 3, cluster, k=8, key_orders=[kr] * 3, dispatch_overhead_ns=5000, threads=th):
    pass
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in pipe.evaluate_stream(model, [cfgs] * 20, cluster, k=8, key_orders=[kr] * 20, dispatch_overhead_ns=5000, threads=th):
    pass
pr.disable()
print("ms/step", (time.perf_counter() - t0) * 1000 / 20)
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
