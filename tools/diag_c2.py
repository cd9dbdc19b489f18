"""Diagnostics for the C2 batch: rounds per config, kernel time by subset."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.engine import Engine

model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]
eng = Engine(0, collapse=("--full" not in sys.argv), sched=os.environ.get("SCHED", "auto"),
             blocks=os.environ.get("BLOCKS", "1") == "1")

def run(sub, reps=5):
    eng.stage_generated(model, sub, cluster, dispatch_overhead_ns=5000)
    st = eng.batch_stats()
    eng.upload()
    ts = []
    for _ in range(reps):
        eng.run(); r = eng.results(); ts.append(eng.last_timings_ms())
    return r, st, [statistics.median(x) for x in zip(*ts)]

r, st, t = run(cfgs)
print("all", len(cfgs), st, "ms est/mem/sched", t, "collapsed", int(eng.collapsed().sum()))
rounds = r["rounds"]
print("rounds: max", rounds.max(), "median", np.median(rounds), "mean", rounds.mean())
order = np.argsort(-rounds)
for i in order[:10]:
    print(cfgs[i].label(), "rounds", rounds[i], "rank_ops", r["rank_ops"][i])
for name, pred in [("tp1pp1", lambda c: c.tp == 1 and c.pp == 1), ("tp8", lambda c: c.tp == 8),
                   ("pp8", lambda c: c.pp == 8), ("pp1", lambda c: c.pp == 1),
                   ("vs4", lambda c: c.virtual_stages == 4)]:
    sub = [c for c in cfgs if pred(c)]
    if not sub: continue
    rs, st2, t2 = run(sub)
    print(name, len(sub), "sched ms", t2[2], "max rounds", rs["rounds"].max(), "rank_ops", st2["rank_ops"])
# single slowest config alone
i = int(order[0])
rs, st2, t2 = run([cfgs[i]])
print("slowest alone", cfgs[i].label(), t2, rs["rounds"])
i = int(np.argmax(r["rank_ops"]))
rs, st2, t2 = run([cfgs[i]])
print("largest alone", cfgs[i].label(), t2, rs["rounds"], rs["rank_ops"])
