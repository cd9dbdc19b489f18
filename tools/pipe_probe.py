"""Per-phase host timings of api.GenPipeline on C2 (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.api import GenPipeline, key_ranks
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
kr = key_ranks(cfgs)
threads = len(os.sched_getaffinity(0))
for chunks in (1, 2, 4, 8):
    pipe = GenPipeline(0, chunks=chunks)
    for it in range(4):
        e = pipe.engines
        t0 = time.perf_counter()
        pipe.evaluate(model, cfgs, cluster, k=8, key_order=kr, dispatch_overhead_ns=5000, threads=threads)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
    # phase probe of one chunk
    n = 512 // chunks
    eng = pipe.engines[0]
    t0 = time.perf_counter(); eng.stage_generated(model, cfgs[:n], cluster, dispatch_overhead_ns=5000, key_ranks=kr[:n], threads=threads)
    t1 = time.perf_counter(); eng.upload(); t2 = time.perf_counter(); eng.run(); t3 = time.perf_counter(); eng.results(); t4 = time.perf_counter()
    print(f"chunks {chunks}: evaluate {1e3*(t1-t0):.1f} ms total-last ... stage {1e3*(t1-t0):.1f} upload {1e3*(t2-t1):.1f} run-enqueue {1e3*(t3-t2):.1f} results {1e3*(t4-t3):.1f} kernels {eng.last_timings_ms()}", flush=True)
    t0 = time.perf_counter()
    pipe.evaluate(model, cfgs, cluster, k=8, key_order=kr, dispatch_overhead_ns=5000, threads=threads)
    torch.cuda.synchronize()
    print(f"   full evaluate {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
    pipe.close()
