"""Generate the golden fixtures by running the REAL reference in this container.

Usage (container only — /root/reference does not exist on the GPU box):

    python tests/golden/make_golden.py [--ref /root/reference/pkg] [--c2]

Imports ``dltsim`` from ``<ref>/src`` and its test helpers (``builders.py``,
``listsched.py``) from ``<ref>/tests``; builds every case below with the
reference's own API, runs ``annotate``/``simulate`` there, and stores the
flattened job (rawtrace.RawJob) together with the reference's outputs:

* unit.npz        — the hand-built known-answer traces of tests/test_sim.py
                    (pkg/tests/test_sim.py:263-459), GPipe/1F1B closed forms
                    (:483-502), deadlock (:415-438) and OOM (:441-459) cases.
* syncfree.npz    — 200 + 200 random single-worker traces, seeds 20260811
                    (test_sim.py:506-518) and 0xACCE97 (test_acceptance.py:246-257),
                    RooflineEstimator on toy_cluster(1, 1).
* multirank.npz   — seeded random multi-rank jobs with collectives, cross-stream
                    events, host syncs and memory (deadlocks kept as status cases).
* workload.npz    — C1 (GPT-2 small, 2 ranks) and a spread of generated
                    Megatron-style configs (acceptance criterion-4 lattice and
                    GPT-3 1.3B / C2 samples) with RooflineEstimator.
* deadlock.npz    — >= 60 deadlocking multi-rank jobs (crossed collective orders,
                    events recorded behind stalled ops, host syncs on them,
                    partial arrivals; 2-256 ranks) with SimDeadlockError's text.
* estimators.json — estimate.py known answers (pkg/tests/test_estimate.py:27-117)
                    plus a seeded sweep of roofline/alpha-beta values.
* c2_results.json — (--c2) reference results for all 512 C2 configs (BASELINE C2).

Outputs stored per job: status, total_ns, peak_mem_bytes, oom, first_oom,
dispatched/completed ops, per-rank stats and (small jobs) the timeline.
"""

from __future__ import annotations

import argparse
import hashlib
import itertools
import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)


def setup(ref: str):
    sys.path.insert(0, os.path.join(ref, "src"))
    sys.path.insert(0, os.path.join(ref, "tests"))


def run_case(name, job, est, cluster=None, timeline_limit=4000):
    """Run the reference on a JobTrace; return (RawJob, expected dict)."""
    from dltsim.estimate import annotate, EstimationError, RooflineEstimator
    from dltsim.sim import simulate, SimDeadlockError
    from paper_2503_20191_b200.rawtrace import from_reference, from_annotated

    exp = {"name": name}
    is_roof = type(est) is RooflineEstimator and est == RooflineEstimator()
    try:
        ann = annotate(job, est)
    except EstimationError as exc:
        raw = from_reference(job, name=name)
        exp.update(status="estimation", message=str(exc))
        return raw, exp
    raw = (from_reference(job, name=name,
                          capacity=None if cluster is None else cluster.device_memory_bytes)
           if is_roof else from_annotated(ann, cluster, name=name))
    try:
        rep = simulate(ann, cluster, record_timeline=True)
    except SimDeadlockError as exc:
        exp.update(status="deadlock", message=str(exc))
        return raw, exp
    except RuntimeError as exc:
        exp.update(status="internal", message=str(exc))
        return raw, exp
    exp.update(status="ok", total_ns=rep.total_ns, peak_mem_bytes=rep.peak_mem_bytes,
               oom=rep.oom, first_oom=list(rep.first_oom) if rep.first_oom else None,
               dispatched_ops=rep.dispatched_ops, completed_ops=rep.completed_ops,
               rank_stats=[[s.compute_busy_ns, s.comm_busy_ns, s.exposed_comm_ns, s.idle_ns,
                            s.peak_mem_bytes] for _, s in sorted(rep.per_rank.items())])
    if len(rep.timeline) <= timeline_limit:
        exp["timeline"] = [[r, s, a, b] for r, s, _, a, b in rep.timeline]
        exp["timeline_names"] = [n for _, _, n, _, _ in rep.timeline]
    return raw, exp


def save(path, cases):
    import numpy as np
    from paper_2503_20191_b200.rawtrace import save_jobs
    jobs = [c[0] for c in cases]
    exps = [c[1] for c in cases]
    save_jobs(path, jobs, {"expected": np.array([json.dumps(exps)])})
    print(f"wrote {path}: {len(jobs)} jobs, {sum(j.n_events for j in jobs)} events")


# --- unit cases (pkg/tests/test_sim.py) -------------------------------------------

def unit_cases():
    from dltsim.collate import collate
    from dltsim.estimate import RooflineEstimator
    from dltsim.trace import (Collective, CommInit, DeviceSynchronize, EventRecord,
                              EventSynchronize, HostGap, KernelAttrs, KernelLaunch, MemAlloc,
                              MemFree, StreamSynchronize, StreamWaitEvent, WorkerTrace)
    from dltsim.workload import ScheduleKind
    from builders import FixedEstimator, toy_cluster, uniform_pipeline_traces

    GIGA = 10 ** 9

    def K(stream, op="k", flops=0, nbytes=0):
        return KernelLaunch(stream, op, KernelAttrs.make({}, "bf16", flops, nbytes))

    cases = []

    def single(name, events, durations, cluster=None, coll_ns=0):
        cluster = cluster or toy_cluster(1, 1)
        job = collate([WorkerTrace(0, 0, 0, tuple(events))], {}, cluster)
        cases.append(run_case(name, job, FixedEstimator(durations, coll_ns=coll_ns)))

    single("empty", [], {})
    single("serial_gap_kernel", [HostGap(2000), K(0, "k")], {"k": 10_000})
    single("two_streams", [K(0, "a"), K(1, "b")], {"a": 100_000, "b": 80_000})
    single("same_stream", [K(0, "a"), K(0, "b")], {"a": 100_000, "b": 80_000})
    single("gap_blocks_host", [K(0, "a"), HostGap(50_000), K(1, "b")],
           {"a": 100_000, "b": 10_000})
    single("trailing_gap", [K(0, "k"), HostGap(500_000)], {"k": 1000})
    single("no_lost_events", [K(0, "a"), K(1, "b"), K(0, "a")], {"a": 10, "b": 20})
    single("wait_chains", [K(0, "a"), EventRecord(0, 0, 0), StreamWaitEvent(1, 0, 0),
                           K(1, "b")], {"a": 50_000, "b": 30_000})
    single("wait_after_fired", [K(0, "a"), EventRecord(0, 0, 0), K(0, "c"),
                                StreamWaitEvent(1, 0, 0), K(1, "b")],
           {"a": 10_000, "b": 5_000, "c": 40_000})
    single("esync", [K(0, "a"), EventRecord(0, 0, 0), EventSynchronize(0, 0), HostGap(5_000),
                     K(1, "b")], {"a": 20_000, "b": 1_000})
    single("ssync", [K(0, "a"), StreamSynchronize(0), K(1, "b")], {"a": 30_000, "b": 1_000})
    single("dsync_idle", [DeviceSynchronize(), K(0, "a")], {"a": 1_000})
    single("dsync_all", [K(0, "a"), K(1, "b"), DeviceSynchronize(), K(2, "c")],
           {"a": 30_000, "b": 40_000, "c": 1_000})
    single("event_version_reuse", [K(0, "a"), EventRecord(0, 0, 0), StreamWaitEvent(1, 0, 0),
                                   K(1, "b"), K(0, "a"), EventRecord(0, 0, 1),
                                   StreamWaitEvent(1, 0, 1), K(1, "b")],
           {"a": 10_000, "b": 1_000})
    single("solo_collective", [CommInit("solo", 1, 0), Collective(0, "solo", 0, "AllReduce", 1024, 1),
                               K(0, "k")], {"k": 5_000}, coll_ns=123_456)
    single("ssync_unknown_stream", [K(0, "a"), StreamSynchronize(7), HostGap(10), K(1, "b")],
           {"a": 30_000, "b": 1_000})
    single("esync_unrecorded_deadlock", [K(0, "a"), EventSynchronize(3, 0), K(1, "b")],
           {"a": 1, "b": 1})
    single("wait_unrecorded_deadlock", [K(0, "a"), StreamWaitEvent(0, 3, 0), K(0, "b")],
           {"a": 1, "b": 1})
    single("wait_before_record", [StreamWaitEvent(1, 0, 0), K(1, "b"), HostGap(7000),
                                  K(0, "a"), EventRecord(0, 0, 0)], {"a": 11_000, "b": 3_000})
    single("record_same_stream_after_wait_deadlock",
           [StreamWaitEvent(0, 0, 0), K(0, "a"), EventRecord(0, 0, 0)], {"a": 5})
    single("zero_duration_chain", [K(0, "z"), K(1, "z"), EventRecord(0, 1, 0),
                                   StreamWaitEvent(1, 1, 0), K(1, "z"), HostGap(0),
                                   DeviceSynchronize()], {"z": 0})
    single("esync_then_ssync", [HostGap(100), K(0, "a"), EventRecord(0, 0, 0), K(1, "b"),
                                EventSynchronize(0, 0), StreamSynchronize(1), HostGap(3),
                                K(0, "a"), DeviceSynchronize(), HostGap(9)],
           {"a": 1000, "b": 5000})

    # memory (test_sim.py:441-459)
    single("oom_third_alloc", [MemAlloc(i, 10 * GIGA) for i in range(3)], {},
           cluster=toy_cluster(1, 1, mem_bytes=25 * GIGA))
    single("free_then_alloc", [MemAlloc(0, 10 * GIGA), MemFree(0), MemAlloc(1, 20 * GIGA)], {},
           cluster=toy_cluster(1, 1, mem_bytes=25 * GIGA))
    single("continue_after_oom", [MemAlloc(0, 2048), K(0, "k")], {"k": 9_000},
           cluster=toy_cluster(1, 1, mem_bytes=1024))
    single("oom_after_gap", [HostGap(500), MemAlloc(0, 100), HostGap(7), MemAlloc(1, 100),
                             MemFree(0), MemAlloc(2, 50)], {},
           cluster=toy_cluster(1, 1, mem_bytes=180))

    # collectives (test_sim.py:351-413)
    def two_worker(name, t0ev, t1ev, durations, wire_ns):
        cluster = toy_cluster(1, 2)
        job = collate([WorkerTrace(0, 0, 0, tuple(t0ev)), WorkerTrace(1, 0, 1, tuple(t1ev))],
                      {}, cluster)
        cases.append(run_case(name, job, FixedEstimator(durations, coll_ns=wire_ns)))

    two_worker("lockstep", [CommInit("c1", 2, 0), K(0, "pre"),
                            Collective(0, "c1", 0, "AllReduce", 1 << 20, 2)],
               [CommInit("c1", 2, 1), K(0, "slow"), Collective(0, "c1", 0, "AllReduce", 1 << 20, 2)],
               {"pre": 10_000, "slow": 50_000}, 15_000)
    two_worker("overlap_blocked_comm", [CommInit("c1", 2, 0),
                                        Collective(1, "c1", 0, "AllReduce", 1 << 20, 2), K(0, "big")],
               [CommInit("c1", 2, 1), K(0, "slow"), Collective(1, "c1", 0, "AllReduce", 1 << 20, 2)],
               {"big": 100_000, "slow": 90_000}, 5_000)
    mk = lambda rank, order: [CommInit("x", 2, rank), CommInit("y", 2, rank),
                              Collective(0, order[0], 0, "AllReduce", 8, 2),
                              Collective(0, order[1], 0, "AllReduce", 8, 2)]
    two_worker("crossed_deadlock", mk(0, ("x", "y")), mk(1, ("y", "x")), {}, 10)
    two_worker("crossed_streams_ok",
               [CommInit("x", 2, 0), CommInit("y", 2, 0),
                Collective(1, "x", 0, "AllReduce", 8, 2), Collective(2, "y", 0, "AllReduce", 8, 2)],
               [CommInit("x", 2, 1), CommInit("y", 2, 1),
                Collective(1, "y", 0, "AllReduce", 8, 2), Collective(2, "x", 0, "AllReduce", 8, 2)],
               {}, 10)
    two_worker("coll_then_esync",
               [CommInit("x", 2, 0), K(0, "a"), Collective(0, "x", 0, "AllGather", 8, 2),
                EventRecord(0, 0, 0), EventSynchronize(0, 0), HostGap(50), K(1, "a")],
               [CommInit("x", 2, 1), HostGap(70_000), Collective(0, "x", 0, "AllGather", 8, 2),
                DeviceSynchronize(), K(0, "a")],
               {"a": 2_000}, 777)

    # pipeline closed forms (test_sim.py:483-502, test_acceptance.py:260-270)
    for sched, pm, tf, tb in (
            [(ScheduleKind.GPIPE, (p, m), 3_000, 5_000) for p in (1, 2, 4, 8) for m in (1, 2, 4, 8, 16)]
            + [(ScheduleKind.ONE_F_ONE_B, pm, 1000, 2000) for pm in ((2, 4), (4, 8))]):
        p, m = pm
        cluster = toy_cluster(1, p)
        job = collate(uniform_pipeline_traces(p, m, sched), {}, cluster)
        cases.append(run_case(f"{sched.value}_p{p}_m{m}", job,
                              FixedEstimator({"fwd": tf, "bwd": tb}, coll_ns=0)))
    cluster = toy_cluster(1, 2)
    job = collate(uniform_pipeline_traces(2, 4, ScheduleKind.ONE_F_ONE_B), {}, cluster)
    cases.append(run_case("accounting_1f1b", job,
                          FixedEstimator({"fwd": 1000, "bwd": 2000}, coll_ns=500)))
    # estimator error surfaces through annotate (estimate.py:344-347)
    job = collate([WorkerTrace(0, 0, 0, (K(0, "gemm", flops=10), KernelLaunch(
        0, "gemm", KernelAttrs.make({}, "fp16x", 10, 0))))], {}, toy_cluster(1, 1))
    cases.append(run_case("missing_dtype", job, RooflineEstimator()))
    return cases


def syncfree_cases():
    from dltsim.collate import collate
    from dltsim.estimate import RooflineEstimator, annotate
    from builders import random_syncfree_trace, toy_cluster
    from listsched import list_schedule_total
    cases = []
    for seed in (20260811, 0xACCE97):
        rng = random.Random(seed)
        for i in range(200):
            trace = random_syncfree_trace(rng)
            cluster = toy_cluster(1, 1)
            job = collate([trace], {}, cluster)
            raw, exp = run_case(f"syncfree_{seed}_{i}", job, RooflineEstimator(), timeline_limit=0)
            ann = annotate(job, RooflineEstimator())
            exp["list_schedule_total"] = list_schedule_total(
                trace, {seq: ns for (_, seq), ns in ann.kernel_ns.items()})
            cases.append((raw, exp))
    return cases


def random_multirank_job(rng: random.Random, n_ranks: int, n_steps: int, n_hosts: int = 1,
                         reorder=None):
    """Seeded random valid multi-rank job: collectives in a shared global order
    on random streams, cross-stream events, host syncs, memory, gaps."""
    from dltsim.cluster import ClusterSpec
    from dltsim.collate import collate
    from dltsim.trace import (Collective, CommInit, DeviceSynchronize, EventRecord,
                              EventSynchronize, HostGap, KernelAttrs, KernelLaunch, MemAlloc,
                              MemFree, Memcpy, Memset, StreamSynchronize, StreamWaitEvent,
                              WorkerTrace, validate_trace)
    from builders import toy_device
    dph = max(1, n_ranks // n_hosts)
    cluster = ClusterSpec(n_hosts, dph, rng.choice([2 ** 40, 3 * 2 ** 30]), toy_device())
    R = cluster.num_devices
    comms = [("world", tuple(range(R)))]
    if R >= 2:
        for a in range(0, R - 1, 2):
            comms.append((f"pair{a}", (a, a + 1)))
        comms.append(("odd", tuple(range(1, R, 2))))
        comms.append(("solo0", (0,)))
    # global collective program: (comm index, kind, bytes)
    kinds = ("AllReduce", "AllGather", "ReduceScatter", "Broadcast", "SendRecv")
    program = [(rng.randrange(len(comms)), rng.choice(kinds), rng.randrange(1, 1 << 24))
               for _ in range(max(1, n_steps // 6))]
    traces = []
    for r in range(R):
        ev = []
        my = [(i, c) for i, c in enumerate(comms) if r in c[1]]
        for i, (cid, members) in my:
            ev.append(CommInit(cid, len(members), members.index(r)))
        call = {cid: 0 for cid, _ in comms}
        ver = {}
        recorded = []
        live = []
        na = 0
        prog = [p for p in program if r in comms[p[0]][1]]
        if reorder is not None:
            prog = reorder(r, prog)
        pi = 0
        nstreams = rng.randrange(1, 5)
        lrng = random.Random(rng.randrange(1 << 30))
        for step in range(n_steps):
            roll = lrng.random()
            if roll < 0.25:
                ev.append(HostGap(lrng.choice([0, lrng.randrange(0, 20_000)])))
            elif roll < 0.55:
                ev.append(KernelLaunch(lrng.randrange(nstreams), lrng.choice(("gemm", "gelu", "mystery")),
                                       KernelAttrs.make({"elems": 1}, lrng.choice(("bf16", "fp32")),
                                                        lrng.randrange(0, 1 << 32),
                                                        lrng.randrange(0, 1 << 26))))
            elif roll < 0.60:
                ev.append(Memcpy(lrng.randrange(nstreams), lrng.choice(("H2D", "D2H", "D2D")),
                                 lrng.randrange(1, 1 << 22)))
            elif roll < 0.62:
                ev.append(Memset(lrng.randrange(nstreams), lrng.randrange(1, 1 << 20)))
            elif roll < 0.72 and pi < len(prog):
                ci, kind, nbytes = prog[pi]
                pi += 1
                cid, members = comms[ci]
                ev.append(Collective(lrng.randrange(nstreams), cid, call[cid], kind, nbytes,
                                     len(members)))
                call[cid] += 1
            elif roll < 0.80:
                e = lrng.randrange(4)
                v = ver.get(e, 0)
                ver[e] = v + 1
                ev.append(EventRecord(lrng.randrange(nstreams), e, v))
                recorded.append((e, v))
            elif roll < 0.87 and recorded:
                e, v = lrng.choice(recorded[-3:])
                ev.append(StreamWaitEvent(lrng.randrange(nstreams), e, v))
            elif roll < 0.89 and recorded:
                e, v = lrng.choice(recorded)
                ev.append(EventSynchronize(e, v))
            elif roll < 0.91:
                ev.append(StreamSynchronize(lrng.randrange(nstreams + 1)))
            elif roll < 0.92:
                ev.append(DeviceSynchronize())
            elif roll < 0.97 or not live:
                ev.append(MemAlloc(na, lrng.randrange(1, 1 << 30)))
                live.append(na)
                na += 1
            else:
                ev.append(MemFree(live.pop(lrng.randrange(len(live)))))
        while pi < len(prog):
            ci, kind, nbytes = prog[pi]
            pi += 1
            cid, members = comms[ci]
            ev.append(Collective(lrng.randrange(nstreams), cid, call[cid], kind, nbytes,
                                 len(members)))
            call[cid] += 1
        if lrng.random() < 0.7:
            ev.append(DeviceSynchronize())
        host, dev = cluster.placement(r)
        tr = WorkerTrace(r, host, dev, tuple(ev))
        assert not validate_trace(tr), validate_trace(tr)[:3]
        traces.append(tr)
    return collate(traces, {}, cluster), cluster


def multirank_cases():
    from dltsim.estimate import RooflineEstimator
    from builders import FixedEstimator
    cases = []
    rng = random.Random(0x5EED2026)
    for i in range(160):
        R = rng.choice([1, 2, 3, 4, 6, 8])
        nh = rng.choice([1, 2]) if R % 2 == 0 else 1
        job, cluster = random_multirank_job(rng, R, rng.randrange(5, 160), nh)
        est = RooflineEstimator() if i % 3 else FixedEstimator(
            {"gemm": rng.randrange(1, 9000), "gelu": 0}, default_ns=rng.randrange(0, 3000),
            coll_ns=rng.randrange(0, 40_000))
        cases.append(run_case(f"multirank_{i}", job, est))
    return cases


def _crossed(rng: random.Random, prog: list, swaps: int) -> list:
    """Per-rank collective order with `swaps` random adjacent transpositions of
    calls on DIFFERENT communicators (per-comm call_idx order stays valid, so
    collate accepts the job; crossings between ranks deadlock it)."""
    prog = list(prog)
    for _ in range(swaps):
        if len(prog) < 2:
            break
        i = rng.randrange(len(prog) - 1)
        if prog[i][0] != prog[i + 1][0]:
            prog[i], prog[i + 1] = prog[i + 1], prog[i]
    return prog


def random_deadlock_job(rng: random.Random, n_ranks: int, n_steps: int, n_hosts: int = 1):
    """random_multirank_job with the even ranks' collective order locally
    crossed (calls on different communicators swapped): the reference
    deadlocks on most of them -- crossed collectives, streams waiting on
    events recorded behind a stalled op, host syncs on such streams/events,
    partial arrivals."""
    seed = rng.randrange(1 << 30)
    swaps = rng.randrange(1, 4)

    def reorder(r, prog):
        if r % 2:
            return prog
        return _crossed(random.Random(seed ^ (r * 7919)), prog, swaps)
    return random_multirank_job(rng, n_ranks, n_steps, n_hosts, reorder=reorder)


def deadlock_cases():
    """>= 50 deadlocking multi-rank jobs (2-8 ranks) plus larger ones (160 and
    256 ranks, hundreds of stream FIFOs: the lane scheduler runs them as grid
    jobs), with the reference's SimDeadlockError text."""
    from dltsim.estimate import RooflineEstimator
    from builders import FixedEstimator
    cases = []
    rng = random.Random(0xDEAD10C)
    tries = 0
    while len(cases) < 60 and tries < 2000:
        tries += 1
        R = rng.choice([2, 3, 4, 6, 8])
        nh = rng.choice([1, 2]) if R % 2 == 0 else 1
        job, cluster = random_deadlock_job(rng, R, rng.randrange(10, 120), nh)
        est = RooflineEstimator() if tries % 3 else FixedEstimator(
            {"gemm": rng.randrange(1, 9000), "gelu": 0}, default_ns=rng.randrange(0, 3000),
            coll_ns=rng.randrange(0, 40_000))
        raw, exp = run_case(f"deadlock_{len(cases)}", job, est)
        if exp["status"] == "deadlock":
            cases.append((raw, exp))
    big = 0
    while big < 3 and tries < 4000:
        tries += 1
        R = (160, 256, 256)[big]
        job, cluster = random_deadlock_job(rng, R, rng.randrange(30, 60), R // 8)
        raw, exp = run_case(f"deadlock_big_{big}", job, RooflineEstimator(), timeline_limit=0)
        if exp["status"] == "deadlock":
            cases.append((raw, exp))
            big += 1
    print(f"  deadlock: {len(cases)} cases from {tries} tries")
    return cases


def workload_cases():
    from dltsim.cluster import ClusterSpec, load_device_preset
    from dltsim.collate import collate
    from dltsim.estimate import RooflineEstimator
    from dltsim.search import SearchSpace, enumerate_space
    from dltsim.workload import (ConfigPoint, ModelSpec, default_schedule,
                                 generate_representatives, validate_config)
    cases = []
    fast = load_device_preset("fast")
    est = RooflineEstimator()
    # C1
    m = ModelSpec("gpt2-small", 12, 768, 1024, 50304, "bf16")
    c = ClusterSpec(1, 2, 80 * 2 ** 30, fast)
    cfg = ConfigPoint(1, 1, 1, 1, False, False, False, 8)
    tr, ex = generate_representatives(m, cfg, c, default_schedule(cfg), dispatch_overhead_ns=5000)
    cases.append(run_case("C1", collate(tr, ex, c), est))
    # acceptance criterion-4 lattice (test_acceptance.py:289-315), every 4th config
    model = ModelSpec("t", num_layers=8, hidden_size=128, seq_len=64, vocab_size=512)
    cluster = ClusterSpec(2, 8, 2 * 2 ** 30, fast)
    n = 0
    for tp, pp in itertools.product((1, 2, 4), repeat=2):
        for mm, vs in itertools.product((1, 2), (1, 2)):
            for rc, sp, dz in itertools.product((False, True), repeat=3):
                cfg = ConfigPoint(tp, pp, mm, vs, rc, sp, dz, 32)
                if validate_config(model, cfg, cluster):
                    continue
                n += 1
                if n % 4:
                    continue
                sched = default_schedule(cfg)
                tr, ex = generate_representatives(model, cfg, cluster, sched)
                cases.append(run_case(f"lattice_{cfg.label()}", collate(tr, ex, cluster), est,
                                      timeline_limit=0))
    # GPT-3 1.3B C2 samples (every 37th of the first 512 valid configs)
    m = ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
    c = ClusterSpec(1, 8, 80 * 2 ** 30, fast)
    cfgs = enumerate_space(SearchSpace(global_batch=512), m, c)[:512]
    for cfg in cfgs[::37]:
        tr, ex = generate_representatives(m, cfg, c, default_schedule(cfg),
                                          dispatch_overhead_ns=5000)
        cases.append(run_case(f"C2_{cfg.label()}", collate(tr, ex, c), est, timeline_limit=0))
    return cases


def synth_cases():
    """C5 synthetic per-rank-distinct jobs, validated and simulated by the reference."""
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    from dltsim import trace as T
    from dltsim.cluster import ClusterSpec, load_device_preset
    from dltsim.collate import collate
    from dltsim.estimate import RooflineEstimator
    from paper_2503_20191_b200.synth import c5_job
    from refmirror import to_reference_like

    def conv(ev):
        n = type(ev).__name__
        if n == "KernelLaunch":
            return T.KernelLaunch(ev.stream, ev.op_kind, T.KernelAttrs.make(
                {}, ev.attrs.dtype, ev.attrs.flops, ev.attrs.bytes_moved))
        return getattr(T, n)(**ev.__dict__)

    cases = []
    for cfg, (R, n) in enumerate([(8, 640), (16, 1280), (24, 320), (3, 2000), (64, 640)]):
        raw = c5_job(R, n, cfg=cfg)
        ann = to_reference_like(raw)
        traces = []
        for r, wt in sorted(ann.job.reps.items()):
            tr = T.WorkerTrace(r, *divmod(r, raw.devices_per_host),
                               tuple(conv(e) for e in wt.events))
            assert not T.validate_trace(tr)
            traces.append(tr)
        cl = ClusterSpec(raw.num_hosts, raw.devices_per_host, raw.capacity,
                         load_device_preset("fast"))
        cases.append(run_case(raw.name, collate(traces, {}, cl), RooflineEstimator(),
                              timeline_limit=0))
    return cases


def estimator_cases():
    from fractions import Fraction
    from dltsim.cluster import DeviceClass, LinkClass, load_device_preset
    from dltsim.estimate import RooflineEstimator, collective_estimate, EstimationError
    from dltsim.trace import KernelAttrs
    GIGA = 10 ** 9
    out = {"kernel": [], "collective": []}

    def dev_json(d):
        return {"name": d.name, "peak_flops": dict(d.peak_flops), "hbm": d.hbm_bytes_per_s,
                "intra": [d.links["intra_host"].alpha_ns, d.links["intra_host"].beta_bytes_per_s],
                "inter": [d.links["inter_host"].alpha_ns, d.links["inter_host"].beta_bytes_per_s]}

    d1 = DeviceClass("d", {"bf16": GIGA}, GIGA, {"intra_host": LinkClass(0, GIGA),
                                                 "inter_host": LinkClass(0, GIGA)})
    d2 = DeviceClass("d", {"bf16": 100 * 10 ** 12}, GIGA, {"intra_host": LinkClass(0, GIGA),
                                                           "inter_host": LinkClass(0, GIGA)})
    d3 = DeviceClass("d", {"bf16": GIGA}, GIGA, {"intra_host": LinkClass(0, 100 * 2 ** 30),
                                                 "inter_host": LinkClass(0, 100 * 2 ** 30)})
    fast, slow = load_device_preset("fast"), load_device_preset("slow")
    from builders import toy_device
    toy = toy_device()

    def kern(dev, op, dtype, flops, nbytes, overhead=1000, eff=None):
        est = RooflineEstimator(eff, overhead) if eff else RooflineEstimator(overhead_ns=overhead)
        try:
            v = est.estimate_kernel(op, KernelAttrs.make({}, dtype, flops, nbytes), dev)
        except EstimationError:
            v = None
        out["kernel"].append({"device": dev_json(dev), "op": op, "dtype": dtype, "flops": flops,
                              "bytes": nbytes, "overhead": overhead,
                              "efficiency": dict(est.efficiency), "expected": v})

    kern(d1, "memcpy_h2d", "bf16", 0, GIGA, 500)          # 1,000,000,500
    kern(d2, "gemm", "bf16", 2 * 4096 ** 3, 1, 0)          # 2,290,650
    kern(toy, "gemm", "bf16", 0, 0, 777)                   # 777
    kern(toy, "mystery", "bf16", 10 ** 12, 0, 0)           # fallback 1/2
    kern(toy, "gemm", "fp16x", 10, 0, 1000)                # missing dtype
    rng = random.Random(77)
    for _ in range(300):
        dev = rng.choice([fast, slow, toy, d2])
        op = rng.choice(["gemm", "layernorm", "memset", "mystery", "optimizer_step"])
        flops = rng.choice([0, rng.randrange(1 << 40), rng.randrange(1 << 62),
                            1_100_000_000_000_000])
        nbytes = rng.choice([0, rng.randrange(1 << 34), rng.randrange(1 << 60)])
        eff = rng.choice([None, {"gemm": 0.123456789, "layernorm": 0.999},
                          {"gemm": 1, "memset": 0.25}])
        kern(dev, op, rng.choice(["bf16", "fp32", "fp16"]), flops, nbytes,
             rng.choice([0, 1000, 12345]), eff)

    def coll(dev, kind, nbytes, n, topo):
        try:
            v = collective_estimate(kind, nbytes, n, topo, dev)
        except EstimationError:
            v = None
        out["collective"].append({"device": dev_json(dev), "kind": kind, "bytes": nbytes,
                                  "nranks": n, "topology": topo, "expected": v})

    coll(d3, "AllReduce", 2 ** 30, 4, "intra_host")       # 15,000,000
    for topo in ("intra_host", "inter_host", "mixed"):
        for n in (1, 2, 4, 8, 16, 2048):
            for e in range(10, 61, 5):
                for kind in ("AllReduce", "AllGather", "ReduceScatter", "Broadcast", "SendRecv"):
                    coll(rng.choice([fast, slow, toy]), kind, 2 ** e + rng.randrange(1000), n, topo)
    return out


def c2_results():
    """Reference results for the 512 C2 configs (BASELINE C2), + trace digests."""
    from dltsim.cluster import ClusterSpec, load_device_preset
    from dltsim.collate import collate
    from dltsim.estimate import RooflineEstimator, annotate
    from dltsim.search import SearchSpace, enumerate_space
    from dltsim.sim import simulate
    from dltsim.trace import dumps_trace
    from dltsim.workload import ModelSpec, default_schedule, generate_representatives
    m = ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
    c = ClusterSpec(1, 8, 80 * 2 ** 30, load_device_preset("fast"))
    cfgs = enumerate_space(SearchSpace(global_batch=512), m, c)[:512]
    rows = []
    t0 = time.time()
    for cfg in cfgs:
        tr, ex = generate_representatives(m, cfg, c, default_schedule(cfg), dispatch_overhead_ns=5000)
        job = collate(tr, ex, c)
        rep = simulate(annotate(job, RooflineEstimator()))
        digest = hashlib.sha256("".join(dumps_trace(t) for t in tr).encode()).hexdigest()
        from paper_2503_20191_b200.rawtrace import from_reference, raw_digest
        raw_sha = raw_digest(from_reference(job))
        rows.append({"key": list(cfg.key()), "total_ns": rep.total_ns,
                     "peak_mem_bytes": rep.peak_mem_bytes, "oom": rep.oom,
                     "n_events": sum(len(t.events) for t in tr),
                     "rank_ops": sum(len(job.trace_of(r).events) for r in job.all_ranks()),
                     "trace_sha256": digest, "raw_sha256": raw_sha})
    print(f"C2: {len(rows)} configs in {time.time() - t0:.1f}s")
    return rows


# C3 / C4 lattices, shared with tools/scale_bench.py and tests/test_scale.py
C3_MODEL = ("gpt3-18.4b", 40, 6144, 2048, 51200, "bf16")
C4_MODEL = ("llama3-70b-shaped", 80, 8192, 8192, 128256, "bf16")
C4_KNOBS = dict(tp=(1, 2, 4, 8), pp=(2, 4, 8, 16), micro_mult=tuple(range(1, 17)),
                virtual_stages=(2, 4, 5, 10), act_recompute=(True, False), seq_parallel=(True,),
                dist_optimizer=(True, False))


def scale_results():
    """Reference results for C3/C4-shaped configs at 64-256 ranks (the reference
    runs 1-10 s per config here), with the digest of each collated job."""
    from dltsim.cluster import ClusterSpec, load_device_preset
    from dltsim.collate import collate
    from dltsim.estimate import RooflineEstimator, annotate
    from dltsim.search import SearchSpace, enumerate_space
    from dltsim.sim import simulate
    from dltsim.workload import ModelSpec, default_schedule, generate_representatives
    from paper_2503_20191_b200.rawtrace import from_reference, raw_digest
    fast = load_device_preset("fast")
    rows = []
    picks = []
    m3 = ModelSpec(*C3_MODEL)
    for n, every in ((64, 17), (128, 41)):
        c = ClusterSpec(n // 8, 8, 80 * 2 ** 30, fast)
        cfgs = enumerate_space(SearchSpace(act_recompute=(True,), global_batch=1024), m3, c)
        picks += [("C3", m3, c, cfg) for cfg in cfgs[::every]]
    m4 = ModelSpec(*C4_MODEL)
    c = ClusterSpec(32, 8, 80 * 2 ** 30, fast)
    cfgs = enumerate_space(SearchSpace(**C4_KNOBS, global_batch=1024), m4, c)
    small = [cfg for cfg in cfgs if cfg.micro_mult == 1 and cfg.pp <= 8]
    picks += [("C4", m4, c, cfg) for cfg in small[::7][:4]]
    t0 = time.time()
    for tag, m, c, cfg in picks:
        tr, ex = generate_representatives(m, cfg, c, default_schedule(cfg), dispatch_overhead_ns=5000)
        job = collate(tr, ex, c)
        rep = simulate(annotate(job, RooflineEstimator()))
        rows.append({"set": tag, "model": list((m.name, m.num_layers, m.hidden_size, m.seq_len,
                                                m.vocab_size, m.dtype)),
                     "ranks": c.num_devices, "key": list(cfg.key()), "total_ns": rep.total_ns,
                     "peak_mem_bytes": rep.peak_mem_bytes, "oom": rep.oom,
                     "rank_ops": sum(len(job.trace_of(r).events) for r in job.all_ranks()),
                     "raw_sha256": raw_digest(from_reference(job))})
        print(f"  {tag} {c.num_devices} {cfg.label()}: {rep.total_ns} ns ({time.time() - t0:.1f}s)",
              flush=True)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default=os.environ.get("MAYA_REF", "/root/reference/pkg"))
    ap.add_argument("--c2", action="store_true", help="also compute c2_results.json (~3 min)")
    ap.add_argument("--only", default="")
    ap.add_argument("--scale", action="store_true", help="also compute scale_results.json (C3/C4)")
    args = ap.parse_args()
    setup(args.ref)
    only = set(args.only.split(",")) if args.only else None
    todo = [("unit", unit_cases), ("syncfree", syncfree_cases), ("multirank", multirank_cases),
            ("workload", workload_cases), ("synth", synth_cases), ("deadlock", deadlock_cases)]
    for name, fn in todo:
        if only and name not in only:
            continue
        t0 = time.time()
        save(os.path.join(HERE, f"{name}.npz"), fn())
        print(f"  {name}: {time.time() - t0:.1f}s")
    if not only or "estimators" in only:
        with open(os.path.join(HERE, "estimators.json"), "w") as f:
            json.dump(estimator_cases(), f)
    if args.scale:
        with open(os.path.join(HERE, "scale_results.json"), "w") as f:
            json.dump(scale_results(), f)
    if args.c2:
        rows = c2_results()
        with open(os.path.join(HERE, "c2_results.json"), "w") as f:
            json.dump(rows, f)


if __name__ == "__main__":
    main()
