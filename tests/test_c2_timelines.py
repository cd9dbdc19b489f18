"""Dependency order on C2- and C3-shaped jobs: the engine's per-(rank, stream)
op timelines equal the CPU oracle's (the restatement of the reference's
event-driven simulator, pinned to the reference by tests/test_oracle_golden.py)
on the C2 configs whose pipelines hand off the most (8 stages x 64
micro-batches, interleaved 2- and 4-chunk schedules, tensor parallel with
sequence parallelism), and on a 64-rank GPT-3 18.4B config -- on every
scheduler kernel, collapsed (classes expanded to ranks) and full-rank.
"""
import pytest

pytestmark = pytest.mark.gpu

C2_LABELS = ["tp1.pp8.mm8.vs1.r--", "tp2.pp4.mm8.vs2.rs-", "tp2.pp2.mm8.vs4.rsz",
             "tp1.pp4.mm8.vs2.r--", "tp8.pp1.mm8.vs1.rsz", "tp4.pp2.mm4.vs2.-s-"]


def _rows(tl):
    d = {}
    for r, s, a, b in tl:
        d.setdefault((int(r), int(s)), []).append((int(a), int(b)))
    return d


def _jobs():
    from paper_2503_20191_b200 import workload as W
    model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
    cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
    cfgs = {c.label(): c for c in W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)}
    jobs = [W.generate_job(model, cfgs[lab], cluster, dispatch_overhead_ns=5000)
            for lab in C2_LABELS if lab in cfgs]
    m3 = W.ModelSpec("gpt3-18.4b", 40, 6144, 2048, 51200, "bf16")
    c3 = W.ClusterSpec(8, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
    jobs.append(W.generate_job(m3, W.ConfigPoint(8, 8, 1, 1, True, False, True, 1024), c3,
                               dispatch_overhead_ns=5000))
    return jobs


@pytest.mark.parametrize("sched", ["auto", "lane", "warp"])
@pytest.mark.parametrize("collapse", [True, False])
def test_c2_timelines_match_oracle(sched, collapse):
    from oracle import oracle
    from paper_2503_20191_b200.engine import Engine
    jobs = _jobs()
    assert len(jobs) >= 6
    e = Engine(0, collapse=collapse, sched=sched)
    try:
        res = e.simulate(jobs, record_timeline=True)
        kinds = e.kernels()
        for q, job in enumerate(jobs):
            o = oracle.simulate(job, timeline=True)
            assert int(res[q]["status"]) == o["status"]
            assert int(res[q]["total_ns"]) == o["total_ns"], (q, sched)
            tl = e.timeline(q).timed()
            got = _rows(zip(tl.rank, tl.stream, tl.start, tl.end))
            ot = o["timeline"]
            want = _rows(zip(ot["rank"], ot["stream"], ot["start"], ot["end"]))
            assert got == want, (q, sched, collapse)
    finally:
        e.close()
    if sched == "auto":
        assert "chain" in kinds
