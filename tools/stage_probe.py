"""Where stage_generated's host time goes (C2 512 configs): Python-side
conversion vs the native generate+pack call, per thread count."""
import os, sys, time, statistics
import ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.engine import Engine, _check
from paper_2503_20191_b200.workload import _gen_lib, cluster_c, configs_array, model_c, schedule_code
from paper_2503_20191_b200.workload import ConfigC
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
eng = Engine(0)
L = _gen_lib()
for th in (1, 4, 8, 16):
    tc, tg, ts = [], [], []
    for _ in range(6):
        t0 = time.perf_counter()
        arr = configs_array(cfgs)
        t1 = time.perf_counter()
        eng.stage_generated(model, cfgs, cluster, dispatch_overhead_ns=5000, threads=th)
        t2 = time.perf_counter()
        _check(L.maya_batch_reset(eng._h))
        n = len(cfgs)
        kr = np.arange(n, dtype=np.int32)
        st = np.zeros(n, dtype=np.int32)
        P = C.POINTER
        t3 = time.perf_counter()
        _check(L.maya_batch_add_generated(eng._h, C.byref(model_c(model)), n,
               arr.ctypes.data_as(P(ConfigC)), C.byref(cluster_c(cluster)), 0, schedule_code(None),
               5000, kr.ctypes.data_as(P(C.c_int32)), th, st.ctypes.data_as(P(C.c_int32))))
        t4 = time.perf_counter()
        tc.append((t1 - t0) * 1e3); tg.append((t2 - t1) * 1e3); ts.append((t4 - t3) * 1e3)
    print(f"threads {th}: configs_array {statistics.median(tc):.3f} ms, stage_generated "
          f"{statistics.median(tg):.3f} ms, native add_generated {statistics.median(ts):.3f} ms", flush=True)
