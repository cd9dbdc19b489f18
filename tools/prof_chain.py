"""Counters of the chain scheduler (instrumented build, make prof) on C2 configs."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MAYA_PROF_CHAIN"] = "1"
from paper_2503_20191_b200 import engine as E
E.LIB_PATH = E.LIB_PATH.replace("libmaya_b200.so", "libmaya_b200_prof.so")
from paper_2503_20191_b200 import workload as W
L = E.lib()
L.maya_prof_read.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
eng = E.Engine(0)
names = ["kernel_cyc", "steps", "step_cyc", "ops", "rounds", "setup_cyc", "copied_cyc", "fuse_cyc"]  # steps = lockstep iterations
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
for lab in sys.argv[1:]:
    sub = cfgs if lab == "all" else [c for c in cfgs if c.label() == lab]
    eng.stage_generated(model, sub, cluster, dispatch_overhead_ns=5000)
    eng.upload()
    buf = (C.c_ulonglong * 16)()
    eng.run(); eng.results(); L.maya_prof_read(buf, 1)
    eng.run(); eng.results(); L.maya_prof_read(buf, 1)
    d = dict(zip(names, list(buf)[8:]))
    st = max(d["steps"], 1)
    print(lab, "sched ms", round(eng.last_timings_ms()[2], 3), d, "cyc/step", d["step_cyc"] // st,
          "ops/step", round(d["ops"] / st, 2), flush=True)
