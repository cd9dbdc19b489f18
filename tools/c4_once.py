"""One C4 lattice batch, N runs (for ncu captures): python tools/c4_once.py RANKS GB [runs]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.engine import Engine
from scale_bench import C4_MODEL, C4_KNOBS
n, gb = int(sys.argv[1]), int(sys.argv[2])
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cluster = W.ClusterSpec(n // 8, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(**C4_KNOBS, global_batch=gb), C4_MODEL, cluster)
eng = Engine(0)
eng.stage_generated(C4_MODEL, cfgs, cluster, dispatch_overhead_ns=5000, threads=16)
eng.upload()
for _ in range(runs):
    eng.run(); eng.results()
print(len(cfgs), eng.last_timings_ms())
import collections
print("kernels", collections.Counter(eng.kernels()))
