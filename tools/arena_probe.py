import os, sys
sys.path.insert(0, "/root/repo")
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.engine import Engine
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
eng = Engine(0)
eng.stage_generated(model, cfgs, cluster, dispatch_overhead_ns=5000, threads=16)
eng.upload()
