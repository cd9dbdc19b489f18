"""Host-side breakdown of the e2e path (gen+pack, arena copy + H2D, run, D2H)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.engine import Engine
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
threads = int(sys.argv[1]) if len(sys.argv) > 1 else len(os.sched_getaffinity(0))
eng = Engine(0)
for it in range(4):
    t0 = time.perf_counter()
    eng.stage_generated(model, cfgs, cluster, dispatch_overhead_ns=5000, threads=threads)
    t1 = time.perf_counter()
    eng.upload()
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    eng.run()
    r = eng.results()
    t3 = time.perf_counter()
    eng.topk(8)
    t4 = time.perf_counter()
    print(f"threads {threads}: gen+pack {1e3*(t1-t0):.1f} ms, upload(copy+H2D enqueue) {1e3*(t2-t1):.1f} ms, "
          f"run+results {1e3*(t3-t2):.1f} ms, topk {1e3*(t4-t3):.1f} ms, total {1e3*(t4-t0):.1f} ms, "
          f"arena {eng.arena_bytes()/1e6:.1f} MB, kernel ms {eng.last_timings_ms()}")
