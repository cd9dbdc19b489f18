"""C5: synthetic per-rank-distinct traces, generated straight
to RawJob arrays with NumPy (no Python event objects).

Per rank r (seed 20261017 + r), ``ops_per_rank`` events in blocks of 64:
59 regular events then the DP-bucket pattern of workload.py:761-767 —
EventRecord(s0), StreamWaitEvent(s1), AllReduce on s1 over the 8-rank comm of
consecutive ranks, EventRecord(s1), StreamWaitEvent(s0).  Regular events are
~49 % HostGap(5000), ~48 % KernelLaunch on streams 0-3 with features drawn as
in pkg/tests/builders.py:133-136 (flops U[0, 2^30), bytes U[0, 2^24)), and
MemAlloc/MemFree pairs.  Collective sizes come from a per-comm seed so every
member issues an identical call sequence (collate.py:352-364).  A trailing
DeviceSynchronize ends each trace.  Every rank is its own representative.
"""

from __future__ import annotations

import numpy as np

from .rawtrace import (EV_COLLECTIVE, EV_COMMINIT, EV_DSYNC, EV_HOSTGAP, EV_KERNEL,
                       EV_MEMALLOC, EV_MEMFREE, EV_RECORD, EV_WAIT, DeviceParams, RawJob)

SEED = 20261017
BLOCK = 64
PATTERN = 5
GROUP = 8

FAST = DeviceParams("fast", {"bf16": 990_000_000_000_000, "fp16": 990_000_000_000_000,
                             "fp32": 67_000_000_000_000}, 3_350_000_000_000,
                    2000, 400_000_000_000, 6000, 50_000_000_000)


def _rank_events(r: int, n_blocks: int, comm_bytes: np.ndarray, cfg: int = 0):
    """(kind, stream, f[4]) for one rank: 1 CommInit + n_blocks*64 + 1 DSYNC."""
    rng = np.random.default_rng(SEED + r + 100_003 * cfg)
    nreg = BLOCK - PATTERN
    n = n_blocks * BLOCK
    kind = np.empty(n, dtype=np.uint8)
    stream = np.zeros(n, dtype=np.int32)
    f = np.zeros((n, 4), dtype=np.int64)
    pos = np.arange(n) % BLOCK
    blk = np.arange(n) // BLOCK
    reg = pos < nreg
    roll = rng.random(n)
    # regular events: gap / kernel / memory
    is_gap = reg & (roll < 0.51)
    is_mem = reg & (roll >= 0.99)
    is_kern = reg & ~is_gap & ~is_mem
    kind[is_gap] = EV_HOSTGAP
    f[is_gap, 0] = 5000
    kind[is_kern] = EV_KERNEL
    nk = int(is_kern.sum())
    stream[is_kern] = rng.integers(0, 4, size=nk)
    f[is_kern, 0] = 0                                    # op kind "gemm"
    f[is_kern, 1] = 0                                    # bf16
    f[is_kern, 2] = rng.integers(0, 1 << 30, size=nk)
    f[is_kern, 3] = rng.integers(0, 1 << 24, size=nk)
    # memory: alternate alloc / free of one buffer at a time
    mpos = np.nonzero(is_mem)[0]
    alloc = (np.arange(len(mpos)) % 2) == 0
    aid = np.arange(len(mpos)) // 2
    kind[mpos] = np.where(alloc, EV_MEMALLOC, EV_MEMFREE)
    f[mpos, 0] = aid
    f[mpos[alloc], 1] = rng.integers(1, 1 << 28, size=int(alloc.sum()))
    if len(mpos) % 2 == 1:                               # unmatched trailing alloc -> gap
        last = mpos[-1]
        kind[last] = EV_HOSTGAP
        f[last] = (5000, 0, 0, 0)
    # the DP-bucket pattern per block
    p = ~reg
    q = pos - nreg
    kind[p & (q == 0)] = EV_RECORD
    kind[p & (q == 1)] = EV_WAIT
    kind[p & (q == 2)] = EV_COLLECTIVE
    kind[p & (q == 3)] = EV_RECORD
    kind[p & (q == 4)] = EV_WAIT
    stream[p & (q == 0)] = 0
    stream[p & ((q == 1) | (q == 2) | (q == 3))] = 1
    stream[p & (q == 4)] = 0
    ev01 = p & ((q == 0) | (q == 1))
    ev23 = p & ((q == 3) | (q == 4))
    f[ev01, 0] = 0
    f[ev01, 1] = blk[ev01]
    f[ev23, 0] = 1
    f[ev23, 1] = blk[ev23]
    c = p & (q == 2)
    f[c, 0] = 0                                          # local comm index
    f[c, 1] = blk[c]                                     # call_idx
    f[c, 2] = 0                                          # AllReduce
    f[c, 3] = comm_bytes[blk[c]]
    return kind, stream, f


def c5_job(n_ranks: int, ops_per_rank: int, name: str = "", cfg: int = 0) -> RawJob:
    """One C5 configuration: n_ranks per-rank-distinct traces of ~ops_per_rank events
    (``cfg`` varies the seeds so a batch holds distinct configurations)."""
    n_blocks = max(1, ops_per_rank // BLOCK)
    n_comms = (n_ranks + GROUP - 1) // GROUP
    kinds, streams, fs, off = [], [], [], [0]
    comm_bytes = [np.random.default_rng([SEED, 7, g, cfg]).integers(1, 1 << 28, size=n_blocks)
                  for g in range(n_comms)]
    for r in range(n_ranks):
        g = r // GROUP
        size = min(GROUP, n_ranks - GROUP * g)
        k, s, f = _rank_events(r, n_blocks, comm_bytes[g], cfg)
        head_f = np.array([[0, size, r - GROUP * g, 0]], dtype=np.int64)
        kinds += [np.array([EV_COMMINIT], np.uint8), k, np.array([EV_DSYNC], np.uint8)]
        streams += [np.zeros(1, np.int32), s, np.zeros(1, np.int32)]
        fs += [head_f, f, np.zeros((1, 4), np.int64)]
        off.append(off[-1] + len(k) + 2)
    ev_kind = np.concatenate(kinds)
    comm_nranks = np.array([min(GROUP, n_ranks - GROUP * g) for g in range(n_comms)], np.int32)
    call_off = np.arange(n_comms + 1, dtype=np.int64) * n_blocks
    return RawJob(
        num_hosts=n_comms, devices_per_host=GROUP if n_ranks >= GROUP else n_ranks,
        capacity=80 * 2 ** 30, device=FAST,
        rep_ranks=np.arange(n_ranks, dtype=np.int64),
        rank_rep=np.arange(n_ranks, dtype=np.int32),
        ev_off=np.array(off, dtype=np.int64), ev_kind=ev_kind,
        ev_stream=np.concatenate(streams), ev_f=np.concatenate(fs),
        op_kind_names=["gemm"], dtype_names=["bf16"],
        comm_names=[f"c5.g{g:05d}" for g in range(n_comms)],
        comm_nranks=comm_nranks, comm_topo=np.zeros(n_comms, np.int8),
        call_off=call_off, call_kind=np.zeros(n_comms * n_blocks, np.int8),
        call_bytes=np.concatenate(comm_bytes).astype(np.int64),
        rank_comm_off=np.arange(n_ranks + 1, dtype=np.int64),
        rank_comm=(np.arange(n_ranks) // GROUP).astype(np.int32),
        name=name or f"C5.r{n_ranks}.n{ops_per_rank}.c{cfg}")
