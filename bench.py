#!/usr/bin/env python
"""Benchmark of the B200 batched simulator on the BASELINE C2 workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): GPT-3 1.3B
(24 x 2048, seq 2048, vocab 51200, bf16) on ClusterSpec(1, 8, 80 GiB, "fast"),
the first 512 valid configs of enumerate_space(SearchSpace(global_batch=512)),
5 us dispatch gaps, RooflineEstimator.  One STEP = evaluate the whole
512-config batch: kernel-roofline + alpha-beta estimators, memory scan,
max-plus scheduler, and the fused top-k search reduction.  Under torchrun
each rank evaluates its own 512-config search (weak scaling): rank r uses
global_batch 512 * 2**r (identical lattice validity, same op counts), and the
per-rank top-k candidates are merged with one NCCL all_gather.

value  = configs/s with traces resident in HBM (CUDA events, L2 flushed
         between timed steps by a 256 MiB write on the engine stream).
e2e    = configs/s through the C ABI from the config list: native trace
         generation + SoA packing (host, C++ threads), H2D of the arena,
         kernels, D2H of results and the top-k.
Reference arm: the UNMODIFIED reference (dltsim, copied to oracle/_ref by
oracle/Makefile) on all host cores, one forked worker process per core:
PipelineEvaluator.__call__ over a bounded, evenly spaced sample of the 512 C2
configs per step (oracle/refbench.py); no module of the product is loaded.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

N_CONFIGS = 512
TOPK = 8
MODEL = ("gpt3-1.3b", 24, 2048, 2048, 51200, "bf16")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--threads", type=int, default=0, help="host threads (0 = all)")
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="0 = 3 x --steps (at least 30): a host-bound step of ~3.5 ms needs "
                         "~0.1 s of timed steps to average out host scheduling jitter")
    ap.add_argument("--cpu-seconds", type=float, default=5.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 lattice sub-line")
    # 4,736 configs = 2 full waves of the lane scheduler (148 SMs x 2 CTAs x 8
    # one-warp jobs): a batch that is a whole number of waves leaves no tail
    ap.add_argument("--c5", default="8x10000x4736",
                    help="C5 synthetic sweep point RANKSxOPSxCONFIGS for the HBM-roofline line "
                         "('' to skip)")
    return ap.parse_args()


def bench_config(world: int) -> dict:
    return {"workload": "C2: GPT-3 1.3B (24x2048, seq 2048, vocab 51200) on 1x8 'fast' 80 GiB; "
                        "enumerate_space(SearchSpace(global_batch=512*2**rank))[:512]; 5 us gaps; "
                        "RooflineEstimator",
            "configs_per_gpu": N_CONFIGS, "ranks_per_config": 8, "topk": TOPK,
            "l2": "flushed between timed steps (256 MiB write on the engine stream)",
            "parallelism": f"config-sharded x{world}"}


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def workload(rank: int):
    from paper_2503_20191_b200 import workload as W
    model = W.ModelSpec(*MODEL)
    cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
    gb = 512 * (2 ** rank)
    configs = W.enumerate_space(W.SearchSpace(global_batch=gb), model, cluster)[:N_CONFIGS]
    return model, cluster, configs


def key_ranks(configs):
    order = sorted(range(len(configs)), key=lambda i: configs[i].key())
    kr = [0] * len(configs)
    for pos, i in enumerate(order):
        kr[i] = pos
    return kr


class ClockSampler:
    """nvidia-smi clocks + throttle reasons around and during the timed region.

    nvidia-smi runs from start() with a 10 ms period; a reader thread stamps
    every line with the host clock, and stop(t0, t1) keeps the samples taken
    inside [t0, t1].  A region shorter than the sampling period falls back to
    the samples that bracket it (marked so)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.rows = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
        except OSError:
            self.proc = None
            return

        def reader():
            for line in self.proc.stdout:
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 9:
                    self.rows.append((time.perf_counter(), p))
        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        t_end = time.perf_counter() + 2.0   # wait for the first sample
        while not self.rows and time.perf_counter() < t_end:
            time.sleep(0.01)

    def stop(self, t0: float, t1: float) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.05)
        self.proc.terminate()
        self.proc.wait()
        if self.thread:
            self.thread.join(timeout=1.0)
        inside = [p for t, p in self.rows if t0 <= t <= t1]
        window = "timed region"
        if not inside:
            before = [p for t, p in self.rows if t < t0][-1:]
            after = [p for t, p in self.rows if t > t1][:1]
            inside = before + after
            window = "samples bracketing the timed region (shorter than the 10 ms period)"
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in inside if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in inside)
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in inside for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": reasons, "samples": len(inside), "window": window}


def load_golden_c2():
    path = os.path.join(REPO, "tests", "golden", "c2_results.json")
    with open(path) as f:
        return json.load(f)


def parity_c2(configs, res) -> dict:
    """Rank-0 batch against the reference's own C2 results (tests/golden)."""
    gold = {tuple(r["key"]): r for r in load_golden_c2()}
    bad = 0
    for cfg, r in zip(configs, res):
        g = gold[tuple(cfg.key())]
        if (int(r["status"]) != 0 or int(r["total_ns"]) != g["total_ns"]
                or int(r["peak_mem_bytes"]) != g["peak_mem_bytes"] or bool(r["oom"]) != g["oom"]):
            bad += 1
    ok = [g for g in gold.values() if not g["oom"]]
    ok.sort(key=lambda g: (g["total_ns"], tuple(g["key"])))
    return {"checked": len(configs), "mismatches": bad, "reference_best": ok[0]["key"],
            "reference_best_ns": ok[0]["total_ns"]}


def _gen_jobs(model, cluster, configs, threads):
    """Native generator (ctypes releases the GIL) on a thread pool."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2503_20191_b200 import workload as W
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(lambda c: W.generate_job(model, c, cluster, dispatch_overhead_ns=5000),
                           configs))


def port_baseline(model, cluster, configs, seconds: float, threads: int) -> dict:
    """Secondary CPU figure: the oracle port (oracle/sim_oracle.cpp, a C++
    restatement of the reference's event-driven simulate + annotate) on the
    host cores, on jobs pre-built by the native generator."""
    from oracle import oracle
    from paper_2503_20191_b200._abi import Batch
    t0 = time.perf_counter()
    jobs = _gen_jobs(model, cluster, configs, threads)
    t_gen = time.perf_counter() - t0
    b = Batch(jobs)
    t1 = time.perf_counter()
    reps = 0
    while True:
        oracle.simulate_many(jobs, threads=threads, batch=b)
        reps += 1
        if time.perf_counter() - t1 > seconds:
            break
    t_sim = (time.perf_counter() - t1) / reps
    n = len(jobs)
    rank_ops = sum(j.rank_ops() for j in jobs)
    return {"value": round(n / t_sim, 2), "unit": "configs/s", "cores": threads, "kind": "port",
            "sample": f"all {n} C2 configs per pass, {reps} passes, pre-built jobs",
            "trace_ops_per_s": round(rank_ops / t_sim, 1),
            "gen_plus_sim_configs_per_s": round(n / (t_sim + t_gen), 2)}


REF_PER_WORKER = 4      # C2 configs per worker process per reference pass (~1-2 s)


def reference_legs(cores: int, e2e_passes: int, warmup: int, extra: bool) -> dict:
    """The unmodified reference (oracle/_ref/dltsim) on the host cores: e2e
    PipelineEvaluator.__call__ with `cores` worker processes (the headline
    leg), and, with `extra`, 1-core e2e and sim-only legs (oracle/refbench.py)."""
    from oracle import refbench
    out = {"e2e": refbench.measure("e2e", cores, REF_PER_WORKER, e2e_passes, warmup)}
    if extra:
        out["e2e_1core"] = refbench.measure("e2e", 1, 6, 1, 0)
        out["sim_only"] = refbench.measure("sim", cores, REF_PER_WORKER, 2, 1)
        out["sim_only_1core"] = refbench.measure("sim", 1, 6, 1, 0)
    return out


def _ref_sample_text(legs: dict, cores: int) -> str:
    e = legs["e2e"]
    return (f"{e['configs_per_pass']} of the 512 C2 configs (evenly spaced in enumeration "
            f"order) per pass, {e['workers']} forked worker processes x {REF_PER_WORKER} "
            f"configs, {e['passes']} timed passes: dltsim PipelineEvaluator.__call__ "
            f"(generate -> collate -> annotate(RooflineEstimator) -> simulate -> compute_mfu, "
            f"search.py:200-209), unmodified reference copied to oracle/_ref")


def cpu_baseline(cores: int) -> dict:
    """Our arm's cpu_baseline: the reference itself on the box's cores (bounded sample)."""
    from oracle import refbench
    why = refbench.available()
    if why:
        return {"value": None, "unit": "configs/s", "cores": cores, "kind": "reference",
                "sample": why}
    legs = reference_legs(cores, 2, 1, extra=True)
    return {"value": legs["e2e"]["configs_per_s"], "unit": "configs/s", "cores": cores,
            "kind": "reference", "sample": _ref_sample_text(legs, cores),
            "e2e_1core_configs_per_s": legs["e2e_1core"]["configs_per_s"],
            "sim_only_configs_per_s": legs["sim_only"]["configs_per_s"],
            "sim_only_1core_configs_per_s": legs["sim_only_1core"]["configs_per_s"],
            "parity_vs_golden": legs["e2e"]["parity"]}


def bench_reference(args):
    """--impl reference: the unmodified reference (dltsim, oracle/_ref) on the
    host cores, rank 0 only.  No module of the product is imported here, so
    libmaya_b200.so is never loaded in this process or its workers."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import refbench
    n = args.gpus
    cores = args.threads or host_threads()
    why = refbench.available()
    if why:
        print(json.dumps({"impl": "reference", "unavailable": why}), flush=True)
        return
    legs = reference_legs(cores, max(1, args.steps), max(0, args.warmup), extra=True)
    e = legs["e2e"]
    val = e["configs_per_s"]
    line = {
        "impl": "reference", "metric": "simulated configs/sec", "value": val,
        "unit": "configs/s", "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * e["seconds_per_pass"], 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic: the reference's own trace generator (dltsim.workload)",
        "config": bench_config(1),
        "step": f"one pass over a bounded sample of the workload ({e['configs_per_pass']} "
                f"configs); value = configs per second over the timed passes",
        "cpu_baseline": {"value": val, "unit": "configs/s", "cores": cores, "kind": "reference",
                         "sample": _ref_sample_text(legs, cores)},
        "e2e": {"value": val, "unit": "configs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "legs": legs,
        "full_batch_seconds_extrapolated": round(512 / val, 2),
    }
    print(json.dumps(line), flush=True)


def measured_peak_hbm():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def ncu_traffic():
    """dram bytes per launch of the scheduler from the committed ncu summary."""
    path = os.path.join(REPO, "profiles", "schedule_kernel_ncu_r2.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def c5_sweep(spec: str, steps: int, dev_index: int) -> dict:
    """C5: per-rank-distinct synthetic traces, the workload the
    HBM-roofline claim is made on.  Scheduler-kernel time only (CUDA events on
    the engine's streams), inputs resident in HBM, L2 flushed between runs."""
    import numpy as np
    import torch
    from paper_2503_20191_b200.engine import Engine
    from paper_2503_20191_b200.synth import c5_job
    R, n, B = (int(x) for x in spec.split("x"))
    distinct = min(B, 64)
    jobs = [c5_job(R, n, cfg=c) for c in range(distinct)]
    eng = Engine(dev_index)
    eng.load([jobs[c % distinct] for c in range(B)], threads=host_threads())
    st = eng.batch_stats()
    dev = torch.device("cuda", dev_index)
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=dev)
    for _ in range(2):
        eng.run()
        r = eng.results()
    ok = int((r["status"] == 0).sum())
    sched, pre, est = [], [], []
    for i in range(max(3, steps)):
        with torch.cuda.stream(stream):
            flush.fill_(i & 0xff)
        eng.run()
        eng.results()
        t = eng.last_timings_ms()
        est.append(t[0])
        pre.append(t[1])
        sched.append(t[2])
    ms = statistics.median(sched)
    fold_ms = statistics.median(pre)
    est_ms = statistics.median(est)
    alg = (16 * st["rep_events"] + 4 * st["rank_comms"] + 16 * (st["features"] + st["slots"])
           + 24 * st["jobs"])
    peak, peak_kind = measured_peak_hbm()
    step_ms = est_ms + fold_ms + ms
    achieved = alg / (step_ms / 1000) / 1e9
    eng.close()
    del flush
    traffic = c5_ncu_traffic(R, n, B)
    return {"workload": f"C5 synthetic: {R} ranks x {n} events/rank, {B} configs per batch "
                        f"({distinct} distinct seeds tiled; every config has its own arena copy; "
                        f"the default batch is 2 full waves of the lane scheduler: "
                        f"148 SMs x 16 resident one-warp jobs x 2)",
            "configs_per_s": round(B / (step_ms / 1000), 1),
            "rank_ops_per_s": round(st["rank_ops"] / (step_ms / 1000), 1),
            "class_ops_per_s": round(st["class_ops"] / (step_ms / 1000), 1),
            "ok": ok, "configs": B,
            "step_ms": {"estimators": round(est_ms, 4), "memscan+fold+resolve": round(fold_ms, 4),
                        "schedulers": round(ms, 4), "total": round(step_ms, 4)},
            "roofline": {"bound": "hbm",
                         "kernels": "the whole step: estimate_features + fold_write (one pass) "
                                    "+ sched_lane_warp (+ small tables), i.e. every kernel that "
                                    "reads the algorithmic bytes",
                         "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "peak_source": peak_kind,
                         "algorithmic_bytes_per_step": alg,
                         "traffic": traffic.get("step_dram_bytes"),
                         "traffic_over_algorithmic": (round(traffic["step_dram_bytes"] / alg, 3)
                                                      if traffic.get("step_dram_bytes") else None),
                         "per_kernel": traffic.get("per_kernel"),
                         "traffic_source": traffic.get("source"),
                         "note": "algorithmic bytes = 16 B x rep events + tables (DESIGN.md "
                                 "roofline) over the step's device time; per_kernel: ncu "
                                 "dram__bytes and time of one cold launch each (committed "
                                 "profile of the same workload)"},
            "scheduler_only": {"ms": round(ms, 4),
                               "input_frac": round(alg / (ms / 1000) / 1e9 / peak, 4),
                               "note": "algorithmic bytes over the scheduler kernel alone -- NOT "
                                       "a roofline of that kernel: the estimator and fold "
                                       "kernels stream those bytes; the scheduler reads the "
                                       "folded ops (per_kernel)"}}


def c5_ncu_traffic(R: int, n: int, B: int) -> dict:
    """Per-kernel DRAM bytes of the C5 step from the committed ncu launch list
    (profiles/c5_step_kernels_r2.json, tools/ncu_summary.py), when it was
    captured on this workload shape."""
    path = os.path.join(REPO, "profiles", "c5_step_kernels_r2.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return {}
    if d.get("workload") not in (None, f"{R}x{n}x{B}"):
        return {}
    per = {k: {"ms": round(v["mean_ms"], 4),
               "dram_bytes": int(v["dram_read_bytes"] + v["dram_write_bytes"])}
           for k, v in d["kernels"].items()}
    return {"step_dram_bytes": sum(v["dram_bytes"] for v in per.values()), "per_kernel": per,
            "source": "profiles/c5_step_kernels_r2.json (" + str(d.get("source")) + ")"}


def c3_lattice(dev_index: int, threads: int, rank: int = 0, world: int = 1) -> dict:
    """C3 (BASELINE configs[2]): GPT-3 18.4B, all 4,088 configs of the
    64-1,024-rank lattices (act_recompute on, global batch 1,024 / 2,048).
    Each of the 10 lattice searches is sharded over the `world` GPUs (strong
    scaling: LPT shards, local fused top-k, one NCCL all_gather of k x 24 B,
    api.evaluate_sharded's merge); the overall best is merged across searches by
    MFU (api.rank_by_mfu).  device: per search, the max over GPUs of its kernel
    time (median of 3 runs, inputs resident), summed; e2e: per search, the max
    over GPUs of generation + packing + H2D + kernels + D2H + top-k on a warm
    engine, summed.  With world > 1, rank 0 re-runs every search alone and
    checks the sharded top-k is identical."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2503_20191_b200 import workload as W
    from paper_2503_20191_b200.api import (config_costs, gather_merge, key_ranks, merge_topk,
                                           rank_by_mfu, shard_lpt)
    from paper_2503_20191_b200.engine import Engine
    model = W.ModelSpec("gpt3-18.4b", 40, 6144, 2048, 51200, "bf16")
    fast = W.load_device_preset("fast")
    searches = []
    for n in (64, 128, 256, 512, 1024):
        cl = W.ClusterSpec(n // 8, 8, 80 * 2 ** 30, fast)
        for gb in (1024, 2048):
            cfgs = W.enumerate_space(W.SearchSpace(act_recompute=(True,), global_batch=gb),
                                     model, cl)
            kr = key_ranks(cfgs)
            mine = shard_lpt(config_costs(cfgs), world)[rank]
            searches.append((cl, cfgs, kr, mine))
    eng = Engine(dev_index)
    dev = torch.device("cuda", dev_index)

    def rmax(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def once(cl, cfgs, kr, idx):
        cand = np.full((TOPK, 3), -1, dtype=np.int64)
        if not idx:
            return None, cand
        eng.stage_generated(model, [cfgs[i] for i in idx], cl, dispatch_overhead_ns=5000,
                            key_ranks=kr[idx], threads=threads)
        eng.upload()
        eng.run()
        r = eng.results()
        for q, t in enumerate(eng.topk(TOPK)):
            cand[q] = (int(t["time_ns"]), int(t["key_rank"]), idx[int(t["job"])])
        return r, cand
    for cl, cfgs, kr, mine in searches:          # warm: size the arenas once
        once(cl, cfgs, kr, mine)
    e2e_s, dev_ms, n_ok, rank_ops, class_ops = 0.0, 0.0, 0, 0, 0
    merged_all = []
    for q, (cl, cfgs, kr, mine) in enumerate(searches):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        r, cand = once(cl, cfgs, kr, mine)
        merged = gather_merge(cand, TOPK) if world > 1 else merge_topk(cand, TOPK)
        e2e_s += rmax(time.perf_counter() - t0)
        ks = []
        for _ in range(3):
            if mine:
                eng.run()
                eng.results()
                ks.append(sum(eng.last_timings_ms()))
            else:
                ks.append(0.0)
        dev_ms += rmax(statistics.median(ks))
        if r is not None:
            n_ok += int((r["status"] == 0).sum())
            bs = eng.batch_stats()
            rank_ops += bs["rank_ops"]
            class_ops += bs["class_ops"]
        merged_all.append(merged)
    n_cfg = sum(len(c) for _, c, _, _ in searches)
    rows = [(int(m[0]), q, int(m[2])) for q, mg in enumerate(merged_all) for m in mg if m[0] >= 0]
    ranked = rank_by_mfu(rows, model,
                         lambda row: (searches[row[1]][1][row[2]], searches[row[1]][0]))
    best_row, best_mfu = ranked[0]
    best_cfg = searches[best_row[1]][1][best_row[2]]
    out = {"workload": "C3: GPT-3 18.4B (40 x 6144, seq 2048), 64-1,024 ranks (8 per host), "
                       "SearchSpace(act_recompute=(True,), global_batch=1024|2048), 5 us gaps, "
                       "RooflineEstimator; 10 lattice searches",
           "configs": n_cfg, "gpus": world,
           "sharding": "each search's configs LPT-sharded over the GPUs (strong scaling), local "
                       "fused top-k, NCCL all_gather of k x 24 B, merge; best across searches "
                       "by MFU (reference _rank order)",
           "device_configs_per_s": round(n_cfg / (dev_ms / 1000), 1),
           "e2e_configs_per_s": round(n_cfg / e2e_s, 1),
           "best": {"key": list(best_cfg.key()), "ranks": searches[best_row[1]][0].num_devices,
                    "time_ns": best_row[0], "mfu": best_mfu}}
    if rank == 0:
        out["ok_on_rank0"] = n_ok
        out["rank_ops_per_s_device_rank0"] = round(rank_ops / (dev_ms / 1000), 1)
        out["class_ops_per_s_device_rank0"] = round(class_ops / (dev_ms / 1000), 1)
    if world > 1 and rank == 0:      # the sharded top-k equals one GPU's
        same = True
        for (cl, cfgs, kr, _), mg in zip(searches, merged_all):
            _, cand = once(cl, cfgs, kr, list(range(len(cfgs))))
            same &= bool(np.array_equal(merge_topk(cand, TOPK), mg))
        out["sharded_topk_equals_single_gpu"] = same
    eng.close()
    return out


def bench_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2503_20191_b200.engine import Engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    threads = args.threads or max(1, host_threads() // max(1, world))

    model, cluster, configs = workload(rank)
    kr = key_ranks(configs)
    eng = Engine(local)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=dev)
    st = eng.stage_generated(model, configs, cluster, dispatch_overhead_ns=5000, key_ranks=kr,
                             threads=threads)
    assert (st == 0).all(), "invalid configs in the C2 lattice"
    eng.upload()
    stats = eng.batch_stats()
    n_collapsed = int(eng.collapsed().sum())
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)

    def step():
        eng.run()
        return eng.topk(TOPK)

    for _ in range(max(3, args.warmup)):
        step()
    res = eng.results()
    parity = parity_c2(configs, res) if rank == 0 else None
    st2 = eng.batch_stats()
    launches_per_step = st2["run_launches"] + st2["topk_launches"]

    # --- device-resident throughput -------------------------------------------------
    sampler = ClockSampler(local)
    sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_region0 = time.perf_counter()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    sched_ms = []
    top = None
    for i in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(i & 0xff)          # L2 flush, outside the timed window
            ev[i][0].record(stream)
        top = step()
        ev[i][1].record(stream)
        sched_ms.append(eng.last_timings_ms()[2])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_region1 = time.perf_counter()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    clocks = sampler.stop(t_region0, t_region1)
    ms = sum(step_ms) / len(step_ms)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())

    # search reduction across GPUs: all_gather of k x 24 B candidates (NCCL).
    # Each GPU searched its own global batch (512 * 2**rank), so the merge ranks
    # by MFU as the reference's _rank does (search.py:349-357; api.rank_by_mfu)
    from paper_2503_20191_b200.api import rank_by_mfu
    cand = np.full((TOPK, 3), -1, dtype=np.int64)
    for q, e in enumerate(top):
        cand[q] = (int(e["time_ns"]), rank, int(e["job"]))
    if world > 1:
        tc = torch.from_numpy(cand).to(dev)
        parts = [torch.empty_like(tc) for _ in range(world)]
        dist.all_gather(parts, tc)
        allc = torch.cat(parts).cpu().numpy()
    else:
        allc = cand
    by_rank = {r: workload(r)[2] for r in range(world)}
    ranked = rank_by_mfu([tuple(int(x) for x in row) for row in allc if row[0] >= 0], model,
                         lambda row: (by_rank[row[1]][row[2]], cluster))
    best, best_mfu = ranked[0]
    best_rank, best_cfg = best[1], by_rank[best[1]][best[2]]

    # --- the same batch on the full-rank path (no class collapse) -------------------
    full = None
    if rank == 0:
        eng.set_collapse(False)
        eng.stage_generated(model, configs, cluster, dispatch_overhead_ns=5000, key_ranks=kr,
                            threads=threads)
        eng.upload()
        for _ in range(2):
            eng.run()
            rf = eng.results()
        fms = []
        for _ in range(max(3, args.steps // 2)):
            with torch.cuda.stream(stream):
                flush.fill_(1)
                a = torch.cuda.Event(enable_timing=True)
                a.record(stream)
            eng.run()
            eng.topk(TOPK)
            z = torch.cuda.Event(enable_timing=True)
            z.record(stream)
            z.synchronize()
            fms.append(a.elapsed_time(z))
        same = bool((rf["total_ns"] == res["total_ns"]).all() and (rf["status"] == res["status"]).all())
        full = {"value": round(N_CONFIGS / (statistics.mean(fms) / 1000), 2), "unit": "configs/s",
                "ms_per_step": round(statistics.mean(fms), 4),
                "trace_ops_per_s": round(stats["rank_ops"] / (statistics.mean(fms) / 1000), 1),
                "class_ops_per_s": round(eng.batch_stats()["class_ops"]
                                         / (statistics.mean(fms) / 1000), 1),
                "identical_results_to_collapsed": same}
        eng.set_collapse(True)
        eng.stage_generated(model, configs, cluster, dispatch_overhead_ns=5000, key_ranks=kr,
                            threads=threads)
        eng.upload()

    # --- end to end through the public API with host buffers ------------------------
    # api.GenPipeline.evaluate_stream over K successive 512-config batches (a
    # search's populations): every step generates + packs on the host threads,
    # copies its arena H2D, runs the kernels, reads its results and top-k D2H;
    # step k+1's host work overlaps step k's device work (two engines).  Timed on
    # the host clock over the K steps, device synchronised on both sides.
    from paper_2503_20191_b200.api import GenPipeline
    pipe = GenPipeline(local, chunks=1)
    e2e_steps = args.e2e_steps or max(30, 3 * args.steps)
    for _ in pipe.evaluate_stream(model, [configs] * 6, cluster, k=TOPK, key_orders=[kr] * 6,
                                  dispatch_overhead_ns=5000, threads=threads):
        pass
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_best = None
    t0 = time.perf_counter()
    outs = []
    for pres, ptop, _ in pipe.evaluate_stream(model, [configs] * e2e_steps, cluster, k=TOPK,
                                              key_orders=[kr] * e2e_steps,
                                              dispatch_overhead_ns=5000, threads=threads):
        outs.append((pres, ptop))
    torch.cuda.synchronize()
    e2e_ms = [(time.perf_counter() - t0) * 1000 / e2e_steps]
    pres, ptop = outs[-1]
    e2e_best = (int(ptop[0][0]), int(ptop[0][1])) if len(ptop) else None
    e2e_same = all(bool((p_["total_ns"] == res["total_ns"]).all()
                        and (p_["status"] == res["status"]).all()) for p_, _ in outs)
    pipe.close()
    e = torch.tensor([sum(e2e_ms) / len(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e, op=dist.ReduceOp.MAX)
        dist.barrier()
    e2e_ms_max = float(e.item())

    c3 = None if args.no_c3 else c3_lattice(local, threads, rank, world)

    if rank == 0:
        n_total = N_CONFIGS * world
        value = n_total / (ms_max / 1000)
        rank_ops = stats["rank_ops"]
        # algorithmic bytes of one step: the packed input read
        # once -- 16 B per device op record (a kernel block is one record, plus 16 B
        # per interned block and 4 B per block feature id) -- and the tables
        alg_bytes = (16 * stats["device_ops"] + 16 * stats["kernel_blocks"]
                     + 4 * stats["block_fids"] + 4 * stats["rank_comms"]
                     + 32 * (stats["features"] + stats["wire_features"]) + 24 * stats["jobs"])
        sched = statistics.median(sched_ms)
        peak, peak_kind = measured_peak_hbm()
        achieved = alg_bytes / (sched / 1000) / 1e9
        line = {
            "metric": "simulated configs/sec", "value": round(value, 2), "unit": "configs/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": round(ms_max, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64",
            "data": "synthetic: native restatement of the reference trace generator "
                    "(event-for-event identical, tests/test_gen.py)",
            "config": dict(bench_config(world), rank_ops_per_gpu=rank_ops),
            "trace_ops_per_s": round(rank_ops * world / (ms_max / 1000), 1),
            "class_ops_per_s": round(stats["class_ops"] * world / (ms_max / 1000), 1),
            "ops_note": "trace_ops_per_s: rank-ops (sum over ALL ranks of the rep trace length, "
                        "the reference's work unit); class_ops_per_s: the ops the engine "
                        "executed (rank classes of collapsed jobs, SURVEY 7.8)",
            "e2e": {"value": round(n_total / (e2e_ms_max / 1000), 2), "unit": "configs/s",
                    "ms_per_step": round(e2e_ms_max, 3), "steps": e2e_steps,
                    "h2d_bytes_per_step": int(stats["arena_bytes"]),
                    "d2h_bytes_per_step": int(N_CONFIGS * 64 + TOPK * 16),
                    "path": "api.GenPipeline.evaluate_stream: per step, config list -> fused "
                            "native gen+pack (C++ threads) -> H2D -> kernels -> D2H results + "
                            "top-k; step k+1's generation overlaps step k's arena assembly + upload (helper thread) and device work",
                    "identical_results_to_device_step": e2e_same,
                    "best": list(e2e_best) if e2e_best else None},
            "roofline": {"bound": "hbm", "kernel": "sched_chain_kernel",
                         "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 5), "traffic": ncu_traffic(),
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "kernel_ms": round(sched, 4), "peak_source": peak_kind,
                         "note": "C2 is latency-bound: the step is the slowest job's chain of "
                                 "stage hand-offs (~800 lockstep iterations of the chain "
                                 "kernel for pp8 x 64 microbatches); dedup, kernel blocks and "
                                 "folding make the compulsory bytes << work"},
            "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
            "rounds": {"max": int(res["rounds"].max()), "median": float(np.median(res["rounds"]))},
            "best": {"rank": best_rank, "key": list(best_cfg.key()), "time_ns": int(best[0]),
                     "mfu": best_mfu},
            "class_collapse": {"collapsed_configs": int(n_collapsed), "simulated_ranks":
                               stats["ranks"], "note": "exact rank-class collapse (SURVEY 7.8), "
                               "verified per config; value/e2e use it"},
            "full_rank": full,
            "parity": parity,
        }
        if world == 1 and args.c5:
            line["c5"] = c5_sweep(args.c5, args.steps, local)
        if c3 is not None:
            line["c3"] = c3
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(host_threads())
            line["cpu_baseline"]["port"] = port_baseline(model, cluster, configs,
                                                         args.cpu_seconds, host_threads())
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
