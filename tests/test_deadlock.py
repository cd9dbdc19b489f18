"""Deadlock parity: status AND the reference's SimDeadlockError text.

tests/golden/deadlock.npz holds 63 deadlocking multi-rank jobs made by the
reference itself (make_golden.py deadlock_cases: crossed collective orders,
streams waiting on events recorded behind stalled collectives, host
ESYNC/SSYNC/DSYNC blocked on them, partial arrivals; 2-8 ranks plus 160- and
256-rank jobs that the lane scheduler runs as grid jobs).  unit.npz adds the
hand-built deadlock cases of the reference's test_sim.py.

Every job runs on every scheduler (auto, forced lane/grid, forced warp),
collapsed and full-rank; the residue text is rebuilt from the device run's
timeline (residue.deadlock_message) and must equal the reference's message
character for character (sim.py:382-402).
"""
import pytest

from paper_2503_20191_b200._abi import STATUS_NAMES
from paper_2503_20191_b200.residue import deadlock_message


def test_deadlock_goldens_are_deadlocks(golden):
    jobs, exps = golden("deadlock")
    assert len(jobs) >= 60
    assert all(e["status"] == "deadlock" for e in exps)
    assert max(j.num_ranks for j in jobs) >= 256


@pytest.mark.gpu
@pytest.mark.parametrize("collapse", [True, False])
@pytest.mark.parametrize("sched", ["auto", "lane", "warp"])
def test_deadlock_residue_matches_reference(golden, collapse, sched):
    from paper_2503_20191_b200.engine import Engine
    jobs, exps = golden("deadlock")
    ujobs, uexps = golden("unit")
    for j, e in zip(ujobs, uexps):
        if e["status"] == "deadlock":
            jobs = jobs + [j]
            exps = exps + [e]
    eng = Engine(0, collapse=collapse, sched=sched)
    try:
        res = eng.simulate(jobs, record_timeline=True)
        bad = []
        for q, (job, exp) in enumerate(zip(jobs, exps)):
            st = STATUS_NAMES[res[q]["status"]]
            if st != "deadlock":
                bad.append((exp["name"], st))
                continue
            msg = deadlock_message(job, eng.timeline(q))
            if msg != exp["message"]:
                bad.append((exp["name"], msg[:300], exp["message"][:300]))
        assert not bad, bad[:3]
    finally:
        eng.close()


@pytest.mark.gpu
def test_simulate_raises_reference_deadlock_text(golden):
    """api path: SimDeadlockError with the residue (through simulate_raw +
    _raise_for, as api.simulate does for an AnnotatedJob)."""
    from paper_2503_20191_b200 import api
    jobs, exps = golden("deadlock")
    for job, exp in list(zip(jobs, exps))[:8]:
        res, eng = api.simulate_raw([job], record_timeline=True)
        with pytest.raises(Exception) as ei:
            api._raise_for(int(res[0]["status"]), "", job, eng.timeline(0))
        assert type(ei.value).__name__ == "SimDeadlockError"
        assert str(ei.value) == exp["message"]
