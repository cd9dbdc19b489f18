"""Device estimators (estimate_features_kernel / estimate_wire_kernel, exact
u128 arithmetic with a double-precision fast path) against the reference's own
estimator outputs (tests/golden/estimators.json: RooflineEstimator known
answers and random cases up to 1.3e18 flops; collective_estimate for every
kind, 2..2048 ranks, three topology classes)."""
import json
import os
from collections import defaultdict

import numpy as np
import pytest

from paper_2503_20191_b200.rawtrace import (EV_COLLECTIVE, EV_COMMINIT, EV_KERNEL, DeviceParams,
                                            RawJob, TOPOLOGIES, COLLECTIVE_KINDS)
from paper_2503_20191_b200._abi import STATUS_NAMES

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def cases():
    with open(os.path.join(GOLDEN, "estimators.json")) as f:
        return json.load(f)


def dev(d):
    return DeviceParams(d["name"], dict(d["peak_flops"]), d["hbm"], d["intra"][0], d["intra"][1],
                        d["inter"][0], d["inter"][1])


def kernel_job(c):
    op_kinds = sorted(c["efficiency"])
    if c["op"] not in op_kinds:
        op_kinds.append(c["op"])
    dtypes = [c["dtype"]]
    f = np.array([[op_kinds.index(c["op"]), 0, c["flops"], c["bytes"]]], dtype=np.int64)
    return RawJob(num_hosts=1, devices_per_host=1, capacity=2 ** 62, device=dev(c["device"]),
                  rep_ranks=np.zeros(1, np.int64), rank_rep=np.zeros(1, np.int32),
                  ev_off=np.array([0, 1], np.int64), ev_kind=np.array([EV_KERNEL], np.uint8),
                  ev_stream=np.zeros(1, np.int32), ev_f=f, op_kind_names=op_kinds,
                  dtype_names=dtypes, comm_names=[], comm_nranks=np.zeros(0, np.int32),
                  comm_topo=np.zeros(0, np.int8), call_off=np.zeros(1, np.int64),
                  call_kind=np.zeros(0, np.int8), call_bytes=np.zeros(0, np.int64),
                  rank_comm_off=np.zeros(2, np.int64), rank_comm=np.zeros(0, np.int32),
                  name=f"k{c['op']}")


def coll_job(c):
    n = c["nranks"]
    dph = n if c["topology"] == "intra_host" else 1
    f = np.array([[0, n, 0, 0], [0, 0, COLLECTIVE_KINDS.index(c["kind"]), c["bytes"]]], np.int64)
    return RawJob(num_hosts=max(1, n // dph), devices_per_host=dph, capacity=2 ** 62,
                  device=dev(c["device"]), rep_ranks=np.zeros(1, np.int64),
                  rank_rep=np.zeros(n, np.int32), ev_off=np.array([0, 2], np.int64),
                  ev_kind=np.array([EV_COMMINIT, EV_COLLECTIVE], np.uint8),
                  ev_stream=np.zeros(2, np.int32), ev_f=f, op_kind_names=["gemm"],
                  dtype_names=["bf16"], comm_names=["c"], comm_nranks=np.array([n], np.int32),
                  comm_topo=np.array([TOPOLOGIES.index(c["topology"])], np.int8),
                  call_off=np.array([0, 1], np.int64),
                  call_kind=np.array([COLLECTIVE_KINDS.index(c["kind"])], np.int8),
                  call_bytes=np.array([c["bytes"]], np.int64),
                  rank_comm_off=np.arange(n + 1, dtype=np.int64),
                  rank_comm=np.zeros(n, np.int32), name=f"c{c['kind']}{n}")


def test_kernel_estimator_matches_reference():
    from paper_2503_20191_b200.engine import Engine
    groups = defaultdict(list)
    for c in cases()["kernel"]:
        groups[(c["overhead"], json.dumps(c["efficiency"], sort_keys=True))].append(c)
    eng = Engine(0)
    bad = []
    for (overhead, eff), cs in groups.items():
        res = eng.simulate([kernel_job(c) for c in cs], efficiency=json.loads(eff),
                           overhead_ns=overhead)
        for c, r in zip(cs, res):
            st = STATUS_NAMES[int(r["status"])]
            if c["expected"] is None:
                if st != "estimation":
                    bad.append((c["op"], c["flops"], st))
            elif st != "ok" or int(r["total_ns"]) != c["expected"]:
                bad.append((c["op"], c["flops"], c["bytes"], st, int(r["total_ns"]), c["expected"]))
    eng.close()
    assert not bad, bad[:5]


def test_collective_estimator_matches_reference():
    from paper_2503_20191_b200.engine import Engine
    eng = Engine(0)
    cs = cases()["collective"]
    res = eng.simulate([coll_job(c) for c in cs])
    bad = [(c["kind"], c["nranks"], c["topology"], int(r["total_ns"]), c["expected"])
           for c, r in zip(cs, res)
           if STATUS_NAMES[int(r["status"])] != "ok" or int(r["total_ns"]) != c["expected"]]
    eng.close()
    assert not bad, bad[:5]


def _roofline_exact(flops, nbytes, peak, eff, hbm, overhead):
    """estimate.py:120-134 in exact integers: max(ceil(flops*1e9/(peak*eff)),
    ceil(bytes*1e9/hbm)) + overhead, eff as Fraction(str(eff))."""
    from fractions import Fraction
    fr = Fraction(str(eff))
    cdiv = lambda a, b: -(-a // b)
    comp = cdiv(flops * 10 ** 9 * fr.denominator, peak * fr.numerator) if flops > 0 else 0
    mem = cdiv(nbytes * 10 ** 9, hbm) if nbytes > 0 else 0
    return max(comp, mem) + overhead


def test_kernel_estimator_fast_path_boundaries():
    """The estimator's straight-line path (kernels.cu estimate_fast: one
    invariant division per term through EstClass) hands every case it cannot
    do exactly to the general u128 routine: flops at and past floor(2^64 / K),
    bytes at and past 2^64 / 1e9, K = 1e9 * den or D = peak * num past 2^64,
    divisors of 1 (the ~0 magic), zero terms.  Each result equals the
    reference formula in exact integer arithmetic."""
    from paper_2503_20191_b200.engine import Engine
    U64 = 2 ** 64 - 1
    out = []
    for peak, hbm, eff in [(10 ** 15, 8 * 10 ** 12, 0.7), (1, 1, 1.0), (3, 7, 0.5),
                           (2_250_000_000_000_000, 7_700_000_000_000, 0.123456789),
                           (10 ** 15, 10 ** 12, 0.1234567891234), (999_999_999_989, 3, 0.75)]:
        from fractions import Fraction
        fr = Fraction(str(eff))
        K = 10 ** 9 * fr.denominator
        maxf = U64 // K
        flops_cases = {0, 1, 12345, maxf - 1, maxf, maxf + 1, 2 * maxf + 3, 10 ** 12}
        bytes_cases = {0, 1, 18446744073, 18446744074, 10 ** 11}
        for fl in sorted(flops_cases):
            for by in sorted(bytes_cases):
                if fl < 0 or fl >= 2 ** 63 or by >= 2 ** 63:
                    continue
                exp = _roofline_exact(fl, by, peak, eff, hbm, 500)
                if exp >= 2 ** 62 - 1:   # the schedulers' documented range (a
                    continue             # duration >= 2^62 ns reports OVERFLOW)
                out.append({"device": {"name": "d", "peak_flops": {"bf16": peak}, "hbm": hbm,
                                       "intra": [0, 10 ** 9], "inter": [0, 10 ** 9]},
                            "op": "gemm", "dtype": "bf16", "flops": fl, "bytes": by,
                            "overhead": 500, "efficiency": {"gemm": eff}, "expected": exp})
    assert len(out) > 100
    groups = defaultdict(list)
    for c in out:
        groups[(json.dumps(c["device"], sort_keys=True), json.dumps(c["efficiency"]))].append(c)
    eng = Engine(0)
    bad = []
    try:
        for (_, eff), cs in groups.items():
            res = eng.simulate([kernel_job(c) for c in cs], efficiency=json.loads(eff),
                               overhead_ns=500)
            for c, r in zip(cs, res):
                st = STATUS_NAMES[int(r["status"])]
                if st != "ok" or int(r["total_ns"]) != c["expected"]:
                    bad.append((c["flops"], c["bytes"], c["device"]["peak_flops"], st,
                                int(r["total_ns"]), c["expected"]))
    finally:
        eng.close()
    assert not bad, bad[:5]
