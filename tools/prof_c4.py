"""Scheduler phase counters (instrumented build) for one C4 lattice batch."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20191_b200 import engine as E
E.LIB_PATH = E.LIB_PATH.replace("libmaya_b200.so", "libmaya_b200_prof.so")
from paper_2503_20191_b200 import workload as W
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from scale_bench import C4_MODEL, C4_KNOBS
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
gb = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
cluster = W.ClusterSpec(n // 8, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(**C4_KNOBS, global_batch=gb), C4_MODEL, cluster)
L = E.lib()
L.maya_prof_read.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
eng = E.Engine(0)
eng.stage_generated(C4_MODEL, cfgs, cluster, dispatch_overhead_ns=5000, threads=16)
eng.upload()
eng.run(); eng.results()
buf = (C.c_ulonglong * 16)(); sub = (C.c_ulonglong * 8)()
L.maya_prof_read(buf, 1); L.maya_prof_read_sub(sub, 1)
eng.run(); r = eng.results()
L.maya_prof_read(buf, 1); L.maya_prof_read_sub(sub, 1)
names = ["walk_cyc", "slow_cyc", "idle_cyc", "sweep_cyc", "windows", "slow_calls", "wide_windows", "ops_committed"]
print(f"C4 n={n} gb={gb}: {len(cfgs)} configs, sched ms {eng.last_timings_ms()[2]:.3f}",
      dict(zip(names, list(buf)[:8])), "lane", list(buf)[8:], "sub", list(sub))
