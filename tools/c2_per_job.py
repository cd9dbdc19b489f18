"""Each C2 config alone: scheduler ms under the warp-window and lane kernels,
with the packed job's size.  Finds the configs that set the C2 step.

    python tools/c2_per_job.py [n_configs]
"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.engine import Engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
cfgs = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:n]
scheds = os.environ.get("SCHEDS", "warp,lane").split(",")
engs = {s: Engine(0, collapse=True, sched=s) for s in scheds}
rows = []
for i, c in enumerate(cfgs):
    row = {"i": i, "cfg": [c.tp, c.pp, c.micro_mult, c.virtual_stages, int(c.act_recompute),
                           int(c.seq_parallel), int(c.dist_optimizer)]}
    for s, eng in engs.items():
        eng.stage_generated(model, [c], cluster, dispatch_overhead_ns=5000, threads=1)
        eng.upload()
        best = 1e9
        for _ in range(3):
            eng.run()
            r = eng.results()
            best = min(best, eng.last_timings_ms()[2])
        row[s] = round(best, 4)
        row["rounds"] = int(r["rounds"][0])
    st = engs[scheds[0]].batch_stats()
    row.update(ranks=st["ranks"], ops=st["device_ops"], rank_ops=st["rank_ops"])
    rows.append(row)
rows.sort(key=lambda r: -r[scheds[0]])
for r in rows[:25]:
    print(json.dumps(r))
print("sum", scheds[0], round(sum(r[scheds[0]] for r in rows), 3), "max", rows[0][scheds[0]])
json.dump(rows, open("gpurun_out/c2_per_job.json", "w"))
