"""C3 / C4 lattices through the engine: configs/s on one GPU.

    python tools/scale_bench.py [c3|c4|both] [--sample K]

C3: GPT-3 18.4B, clusters 64..1024 ranks (8 per host), SearchSpace(act_recompute=(True,),
    global_batch in {1024, 2048}) -> 4,088 valid configs.
C4: Llama-3-70B-shaped (80 x 8192, seq 8192, vocab 128256), clusters 256..2048 ranks,
    knobs of tests/golden/make_golden.py C4_KNOBS, global_batch 1024..16384 -> 15,936 configs.
Per (cluster, global_batch) batch: native generation + packing on host threads (collapsed
jobs), H2D, estimators + scheduler + top-k on the device.  Reports device-resident
configs/s (kernel time) and end-to-end configs/s (host gen/pack + H2D + kernels + D2H).
"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.engine import Engine

C3_MODEL = W.ModelSpec("gpt3-18.4b", 40, 6144, 2048, 51200, "bf16")
C4_MODEL = W.ModelSpec("llama3-70b-shaped", 80, 8192, 8192, 128256, "bf16")
C4_KNOBS = dict(tp=(1, 2, 4, 8), pp=(2, 4, 8, 16), micro_mult=tuple(range(1, 17)),
                virtual_stages=(2, 4, 5, 10), act_recompute=(True, False), seq_parallel=(True,),
                dist_optimizer=(True, False))


def lattices(which):
    fast = W.load_device_preset("fast")
    out = []
    if which in ("c3", "both"):
        for n in (64, 128, 256, 512, 1024):
            c = W.ClusterSpec(n // 8, 8, 80 * 2 ** 30, fast)
            for gb in (1024, 2048):
                cfgs = W.enumerate_space(W.SearchSpace(act_recompute=(True,), global_batch=gb),
                                         C3_MODEL, c)
                out.append(("C3", C3_MODEL, c, gb, cfgs))
    if which in ("c4", "both"):
        for n in (256, 512, 1024, 2048):
            c = W.ClusterSpec(n // 8, 8, 80 * 2 ** 30, fast)
            for gb in (1024, 2048, 4096, 8192, 16384):
                cfgs = W.enumerate_space(W.SearchSpace(**C4_KNOBS, global_batch=gb), C4_MODEL, c)
                out.append(("C4", C4_MODEL, c, gb, cfgs))
    return out


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c3"
    sample = 0
    if "--sample" in sys.argv:
        sample = int(sys.argv[sys.argv.index("--sample") + 1])
    threads = len(os.sched_getaffinity(0))
    eng = Engine(0)
    tot = {}
    for tag, model, cluster, gb, cfgs in lattices(which):
        if sample:
            cfgs = cfgs[::max(1, len(cfgs) // sample)][:sample]
        if not cfgs:
            continue
        t0 = time.perf_counter()
        st = eng.stage_generated(model, cfgs, cluster, dispatch_overhead_ns=5000, threads=threads)
        t1 = time.perf_counter()
        eng.upload()
        eng.run()
        res = eng.results()
        top = eng.topk(8)
        t2 = time.perf_counter()
        ks = []
        for _ in range(3):
            eng.run()
            eng.results()
            ks.append(sum(eng.last_timings_ms()))
        stats = eng.batch_stats()
        kms = float(np.median(ks))
        n = len(cfgs)
        ok = int((res["status"] == 0).sum())
        oom = int(res["oom"].sum())
        d = tot.setdefault(tag, {"configs": 0, "kernel_ms": 0.0, "e2e_s": 0.0, "rank_ops": 0,
                                 "ok": 0, "oom": 0, "collapsed": 0})
        d["configs"] += n
        d["kernel_ms"] += kms
        d["e2e_s"] += t2 - t0
        d["rank_ops"] += stats["rank_ops"]
        d["ok"] += ok
        d["oom"] += oom
        d["collapsed"] += int(eng.collapsed().sum())
        print(f"{tag} n={cluster.num_devices:5d} gb={gb:5d}: {n:5d} configs, ok {ok}, oom {oom}, "
              f"rank-ops {stats['rank_ops']/1e6:9.1f}M, sim ranks {stats['ranks']}, "
              f"kernels {kms:8.3f} ms ({n / kms * 1e3:10.0f} cfg/s), gen+pack {t1 - t0:6.2f} s, "
              f"e2e {t2 - t0:6.2f} s ({n / (t2 - t0):8.0f} cfg/s), best {int(top[0]['time_ns']) if len(top) else -1}",
              flush=True)
    for tag, d in tot.items():
        d["device_configs_per_s"] = round(d["configs"] / (d["kernel_ms"] / 1e3), 1)
        d["e2e_configs_per_s"] = round(d["configs"] / d["e2e_s"], 1)
        d["rank_ops_per_s_device"] = round(d["rank_ops"] / (d["kernel_ms"] / 1e3), 1)
        print(json.dumps({tag: d}), flush=True)


if __name__ == "__main__":
    main()
