"""Per-phase counters of the lane scheduler (instrumented build, make prof)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20191_b200 import engine as E
E.LIB_PATH = E.LIB_PATH.replace("libmaya_b200.so", "libmaya_b200_prof.so")
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.synth import c5_job
L = E.lib()
L.maya_prof_read.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
eng = E.Engine(0, sched=os.environ.get("SCHED", "auto"))
names = ["loop_cyc", "iters", "data_iters", "pass_cyc", "ops", "data_ret", "prog_visits", "blk_visits"]
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]

def show(tag):
    eng.run(); eng.results()
    buf = (C.c_ulonglong * 16)()
    L.maya_prof_read(buf, 1)
    eng.run(); eng.results()
    L.maya_prof_read(buf, 1)
    d = dict(zip(names, list(buf)[8:]))
    it = max(d["iters"], 1)
    print(tag, "sched ms", round(eng.last_timings_ms()[2], 3), d,
          "cyc/iter", d["pass_cyc"] // it, "ops/iter", round(d["ops"] / it, 1), flush=True)

for spec in sys.argv[1:]:
    if spec.startswith("c2:"):
        lab = spec[3:]
        sub = cfgs if lab == "all" else [c for c in cfgs if c.label() == lab]
        eng.stage_generated(model, sub, cluster, dispatch_overhead_ns=5000)
        eng.upload()
    else:
        R, n, B = (int(x) for x in spec.split("x"))
        jobs = [c5_job(R, n, cfg=c) for c in range(min(B, 64))]
        eng.load([jobs[c % len(jobs)] for c in range(B)], threads=16)
    show(spec)
