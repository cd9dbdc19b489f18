"""Pin the CPU oracle (oracle/sim_oracle.cpp) to the reference's own outputs.

The fixtures were produced by running the reference (pkg/src/dltsim) in the
build container (tests/golden/make_golden.py); this test needs no reference.
"""
import pytest

from oracle import oracle

STATUS = {0: "ok", 1: "deadlock", 2: "internal", 3: "estimation", 4: "overflow", 5: "bad_input"}


def check(job, exp):
    got = oracle.simulate(job, timeline="timeline" in exp)
    assert STATUS[got["status"]] == exp["status"], (exp["name"], got["message"], exp.get("message"))
    if exp["status"] != "ok":
        return
    assert got["total_ns"] == exp["total_ns"], exp["name"]
    assert got["peak_mem_bytes"] == exp["peak_mem_bytes"], exp["name"]
    assert bool(got["oom"]) == exp["oom"], exp["name"]
    if exp["first_oom"] is not None:
        assert [got["first_oom_rank"], got["first_oom_seq"]] == exp["first_oom"], exp["name"]
    assert got["dispatched_ops"] == exp["dispatched_ops"]
    assert got["completed_ops"] == exp["completed_ops"]
    assert got["rank_stats"].tolist() == exp["rank_stats"], exp["name"]
    if "timeline" in exp:
        tl = got["timeline"]
        rows = [[int(r), int(s), int(a), int(b)] for r, s, a, b in
                zip(tl["rank"], tl["stream"], tl["start"], tl["end"])]
        assert rows == exp["timeline"], exp["name"]


@pytest.mark.parametrize("name", ["unit", "syncfree", "multirank", "workload", "synth", "deadlock"])
def test_oracle_matches_reference(golden, name):
    jobs, exps = golden(name)
    for job, exp in zip(jobs, exps):
        check(job, exp)


def test_syncfree_list_scheduler(golden):
    # pkg/tests/listsched.py: the reference's independent oracle agrees too
    jobs, exps = golden("syncfree")
    for job, exp in zip(jobs, exps):
        assert exp["total_ns"] == exp["list_schedule_total"]
