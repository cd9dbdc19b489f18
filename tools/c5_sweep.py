"""C5 synthetic sweep (BASELINE configs[4]): throughput vs trace size on one GPU.

Each point: R ranks x N events/rank, B configs per batch (B chosen to fill the
GPU within memory; `distinct` seeds tiled, every config with its own arena
copy).  Reports the scheduler kernel time and the whole step (estimators +
fold/resolve + schedulers), configs/s, rank-ops/s and the HBM roofline
fraction of the scheduler (algorithmic bytes).  Writes
profiles/c5_sweep_r1.json and prints a markdown table.
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2503_20191_b200.engine import Engine
from paper_2503_20191_b200.synth import c5_job

# (ranks, events/rank, max configs, distinct seeds).  The batch holds
# min(max configs, what fits BUDGET_GB of device arena) configurations: a long-
# trace point runs as many configs as HBM holds (one job per warp / CTA / grid).
GRID = [(8, 1000, 8192, 64), (8, 10000, 4096, 64), (8, 100000, 2368, 16), (8, 1000000, 296, 4),
        (64, 1000, 2048, 64), (64, 10000, 592, 32), (64, 100000, 148, 8), (64, 1000000, 16, 2),
        (512, 1000, 296, 16), (512, 10000, 64, 8), (512, 100000, 8, 2), (512, 1000000, 1, 1),
        (2048, 1000, 74, 4), (2048, 10000, 16, 2), (2048, 100000, 2, 1), (2048, 1000000, 1, 1)]
BUDGET_GB = float(os.environ.get("C5_BUDGET_GB", "60"))
BYTES_PER_EVENT = 40      # device arena + scratch per trace event (measured: arena_bytes)


def _peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0   # B200_PROFILING.md fallback


PEAK = _peak()


def main():
    only = sys.argv[1:]
    eng = Engine(0)
    rows = []
    for R, n, B, distinct in GRID:
        if only and f"{R}x{n}" not in only:
            continue
        B = max(1, min(B, int(BUDGET_GB * 1e9 / (BYTES_PER_EVENT * R * n))))
        t0 = time.time()
        base = [c5_job(R, n, cfg=c) for c in range(min(B, distinct))]
        jobs = [base[c % len(base)] for c in range(B)]
        tg = time.time() - t0
        eng.load(jobs, threads=len(os.sched_getaffinity(0)))
        st = eng.batch_stats()
        ts = []
        for _ in range(4):
            eng.run()
            r = eng.results()
            ts.append(eng.last_timings_ms())
        est, pre, sched = [float(np.median([t[k] for t in ts[1:]])) for k in range(3)]
        alg = (16 * st["rep_events"] + 4 * st["rank_comms"] + 16 * (st["features"] + st["slots"])
               + 24 * st["jobs"])
        step = est + pre + sched
        row = {"ranks": R, "events_per_rank": n, "configs": B, "distinct_seeds": len(base),
               "rank_ops": st["rank_ops"], "sched_ms": round(sched, 4), "step_ms": round(step, 4),
               "configs_per_s": round(B / step * 1e3, 1),
               "rank_ops_per_s": round(st["rank_ops"] / step * 1e3, 1),
               "sched_gbs": round(alg / sched / 1e6, 1),
               "sched_frac": round(alg / sched / 1e6 / PEAK, 4),
               "step_frac": round(alg / step / 1e6 / PEAK, 4),
               "ok": int((r["status"] == 0).sum()), "gen_s": round(tg, 1),
               "arena_gb": round(st["arena_bytes"] / 1e9, 2)}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del jobs, base
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                       "c5_sweep_r2.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(rows, f, indent=1)
    print("| ranks | events/rank | configs | sched ms | step ms | configs/s | rank-ops/s | sched % HBM | step % HBM |")
    print("|---|---|---|---|---|---|---|---|---|")
    for x in rows:
        print(f"| {x['ranks']} | {x['events_per_rank']} | {x['configs']} | {x['sched_ms']} | {x['step_ms']} | "
              f"{x['configs_per_s']:.0f} | {x['rank_ops_per_s']:.3g} | {100 * x['sched_frac']:.1f} | "
              f"{100 * x['step_frac']:.1f} |")


if __name__ == "__main__":
    main()
