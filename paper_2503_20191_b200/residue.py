"""Reference-exact error texts for jobs the engine ends with a failure status.

The engine reports a per-job status code; the reference raises exceptions
whose text names the failing objects, and ``run_search`` stores that text in
INVALID trial records (search.py:370-374).  These functions rebuild the texts
from the job and the engine's final device state:

* ``deadlock_message`` -- ``_check_residue`` (sim.py:382-402).  A timeline
  run marks every device op the schedulers completed (``maya_run`` presets
  each op's end time to -1); the deadlocked state of the reference is the same
  least fixpoint, so per rank the host's blocking sync is the first one whose
  condition fails on the completed set (sim.py:243-263), and per stream the
  first dispatched, uncompleted op is the WAIT it waits on or the collective
  it is stalled in (sim.py:302-343).
* ``estimation_message`` -- the roofline estimator's missing-dtype error as
  ``annotate`` re-raises it (estimate.py:124-127, 339-346): the first
  kernel-class event, reps in rank order, with flops > 0 and no peak rate.

Error paths only: the formatting reads the RawJob on the host; every time in
it comes from the device run.
"""
from __future__ import annotations

import numpy as np

from .rawtrace import (EV_COLLECTIVE, EV_DSYNC, EV_ESYNC, EV_KERNEL, EV_MEMCPY, EV_MEMSET,
                       EV_RECORD, EV_SSYNC, EV_WAIT, RawJob)

_DEVICE_OPS = (EV_KERNEL, EV_MEMCPY, EV_MEMSET, EV_COLLECTIVE, EV_RECORD, EV_WAIT)


def deadlock_message(raw: RawJob, timeline) -> str:
    """``SimDeadlockError`` text of a deadlocked job from its timeline run
    (``Engine.timeline(job)``: every device op of every rank, end -1 when the
    op never completed)."""
    done_by_rank: dict[int, set] = {}
    m = timeline.end >= 0
    for r, q in zip(timeline.rank[m].tolist(), timeline.seq[m].tolist()):
        done_by_rank.setdefault(r, set()).add(q)
    stuck: list[str] = []
    arrivals: dict[tuple, list] = {}
    kinds, streams, f = raw.ev_kind, raw.ev_stream, raw.ev_f
    for r in range(raw.num_ranks):
        rep = int(raw.rank_rep[r])
        lo, hi = int(raw.ev_off[rep]), int(raw.ev_off[rep + 1])
        done = done_by_rank.get(r, set())
        comms = raw.rank_comm[int(raw.rank_comm_off[r]):int(raw.rank_comm_off[r + 1])]
        fired = set()
        queues: dict[int, list] = {}      # stream -> dispatched seqs (FIFO order)

        def drained(s):
            q = queues.get(s)
            return q is None or all(x in done for x in q)

        blocked = None
        for seq in range(hi - lo):
            e = lo + seq
            k = int(kinds[e])
            if k in _DEVICE_OPS:
                queues.setdefault(int(streams[e]), []).append(seq)
                if k == EV_RECORD and seq in done:
                    fired.add((int(f[e, 0]), int(f[e, 1])))
        # host replay over the final state (sim.py:222-270)
        for seq in range(hi - lo):
            e = lo + seq
            k = int(kinds[e])
            if k == EV_ESYNC:
                key = (int(f[e, 0]), int(f[e, 1]))
                if key not in fired:
                    blocked = ("event", (r, key[0], key[1]))
            elif k == EV_SSYNC:
                s = int(streams[e])
                if not _drained_before(queues.get(s), done, seq):
                    blocked = ("ssync", s)
            elif k == EV_DSYNC:
                if not all(_drained_before(q, done, seq) for q in queues.values()):
                    blocked = ("dsync", None)
            if blocked is not None:
                host_pc = seq
                break
        else:
            host_pc = hi - lo
        if blocked is not None:
            stuck.append(f"rank {r}: host blocked on {blocked}")
        for s in sorted(queues):
            q = [x for x in queues[s] if x < host_pc]   # dispatched before the host stopped
            if not q:
                continue
            pending = [x for x in q if x not in done]
            if not pending:
                continue
            e = lo + pending[0]
            k = int(kinds[e])
            if k == EV_WAIT:
                stuck.append(f"rank {r} stream {s}: waiting on event "
                             f"{(r, int(f[e, 0]), int(f[e, 1]))}")
            elif k == EV_COLLECTIVE:
                gkey = (raw.comm_names[int(comms[int(f[e, 0])])], int(f[e, 1]))
                stuck.append(f"rank {r} stream {s}: stalled in collective {gkey}")
                arrivals.setdefault(gkey, []).append(r)
            else:
                stuck.append(f"rank {r} stream {s}: {len(pending)} ops queued")
    names = {n: i for i, n in enumerate(raw.comm_names)}
    for gkey, members in sorted(arrivals.items()):
        need = int(raw.comm_nranks[names[gkey[0]]])
        stuck.append(f"collective {gkey}: {len(members)}/{need} arrived ({sorted(members)})")
    return "simulation deadlocked with blocked work:\n  " + "\n  ".join(stuck)


def _drained_before(q, done, pc) -> bool:
    """Stream drained at host position pc: every op it dispatched before pc done."""
    if q is None:
        return True
    return all(x in done for x in q if x < pc)


def estimation_message(raw: RawJob) -> str | None:
    """``EstimationError`` text of the roofline estimator on this job, or None."""
    kc = np.isin(raw.ev_kind, (EV_KERNEL, EV_MEMCPY, EV_MEMSET))
    peaks = raw.device.peak_flops
    bad_dt = np.array([n not in peaks for n in raw.dtype_names] + [False], dtype=bool)
    dt = np.where(kc, raw.ev_f[:, 1], len(raw.dtype_names))
    hit = kc & (raw.ev_f[:, 2] > 0) & bad_dt[dt]
    if not hit.any():
        return None
    for rep in np.argsort(raw.rep_ranks, kind="stable").tolist():
        lo, hi = int(raw.ev_off[rep]), int(raw.ev_off[rep + 1])
        idx = np.nonzero(hit[lo:hi])[0]
        if len(idx):
            e = lo + int(idx[0])
            return (f"rank {int(raw.rep_ranks[rep])} seq {int(idx[0])}: device "
                    f"{raw.device.name!r} has no peak rate for dtype "
                    f"{raw.dtype_names[int(raw.ev_f[e, 1])]!r}")
    return None
