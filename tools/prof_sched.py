"""Per-phase cycle breakdown of the scheduler (instrumented build)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MAYA_LIB"] = "prof"
from paper_2503_20191_b200 import engine as E
E.LIB_PATH = E.LIB_PATH.replace("libmaya_b200.so", "libmaya_b200_prof.so")
from paper_2503_20191_b200 import workload as W
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
L = E.lib()
L.maya_prof_read.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
eng = E.Engine(0)
names = ["walk_cyc", "slow_cyc", "idle_cyc", "sweep_cyc", "windows", "slow_calls", "wide_windows", "ops_committed"]
for label in (sys.argv[1:] if len(sys.argv) > 1 else ([] if os.environ.get("C5") else ["tp2.pp2.mm8.vs4.rsz", "tp1.pp8.mm8.vs1.rsz"])):
    sub = [c for c in cfgs if c.label() == label]
    eng.stage_generated(model, sub, cluster, dispatch_overhead_ns=5000)
    eng.upload()
    eng.run(); eng.results()
    buf = (C.c_ulonglong * 16)()
    L.maya_prof_read(buf, 1)
    eng.run(); r = eng.results()
    L.maya_prof_read(buf, 1)
    sub = (C.c_ulonglong * 8)()
    if hasattr(L, "maya_prof_read_sub"):
        L.maya_prof_read_sub(sub, 1)
        eng.run(); eng.results()
        L.maya_prof_read_sub(sub, 1)
    print(label, "sched ms", round(eng.last_timings_ms()[2], 3), dict(zip(names, list(buf))),
          "window sub-phases (seg/wide, load+classify, scan, blockers+commit, wide attempts, failed-wide cycles):", list(sub))

if os.environ.get("C5"):
    from paper_2503_20191_b200.synth import c5_job
    for spec in os.environ["C5"].split(","):
        R, n, B = (int(x) for x in spec.split("x"))
        jobs = [c5_job(R, n, cfg=c) for c in range(B)]
        eng.load(jobs, threads=16)
        eng.run(); eng.results()
        buf = (C.c_ulonglong * 16)()
        L.maya_prof_read(buf, 1)
        eng.run(); r = eng.results()
        L.maya_prof_read(buf, 1)
        st = eng.batch_stats()
        print(f"C5 {spec} sched ms", round(eng.last_timings_ms()[2], 3), "dev_ops", st["device_ops"],
              dict(zip(names, list(buf))))
