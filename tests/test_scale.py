"""C3 / C4 shapes: GPT-3 18.4B and Llama-3-70B-shaped configs at
64-256 ranks, pinned to the reference's own results (tests/golden/
scale_results.json, made by tests/golden/make_golden.py --scale).

* CPU: the native generator's collated job hashes to the reference's digest;
* GPU: the engine (collapsed and full-rank) reproduces total_ns, peak memory
  and the OOM flag bit-exactly, and the batched top-k equals the reference's
  (time, key) order over the sample.
"""
import json
import os

import numpy as np
import pytest

from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.rawtrace import raw_digest

from conftest import GOLDEN


def rows():
    with open(os.path.join(GOLDEN, "scale_results.json")) as f:
        return json.load(f)


def point(r):
    model = W.ModelSpec(*r["model"])
    cluster = W.ClusterSpec(r["ranks"] // 8, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
    return model, cluster, W.ConfigPoint(*r["key"])


def test_scale_generator_digests_match_reference():
    bad = []
    for r in rows():
        model, cluster, cfg = point(r)
        job = W.generate_job(model, cfg, cluster, dispatch_overhead_ns=5000)
        assert job.rank_ops() == r["rank_ops"], cfg
        if raw_digest(job) != r["raw_sha256"]:
            bad.append((r["set"], r["ranks"], cfg.label()))
    assert not bad, bad[:5]


@pytest.mark.gpu
@pytest.mark.parametrize("collapse", [True, False])
@pytest.mark.parametrize("blocks", [True, False])
def test_scale_engine_matches_reference(collapse, blocks):
    """C3/C4-shaped configs at 64-256 ranks against the reference's results,
    with and without kernel blocks (interned launch runs, soa.h KBLOCK)."""
    from paper_2503_20191_b200.engine import Engine
    rs = rows()
    eng = Engine(0, collapse=collapse, blocks=blocks)
    bad = []
    groups = {}
    for i, r in enumerate(rs):
        groups.setdefault((tuple(r["model"]), r["ranks"]), []).append(i)
    got = {}
    for (_, _), idx in groups.items():
        model, cluster, _ = point(rs[idx[0]])
        cfgs = [point(rs[i])[2] for i in idx]
        st = eng.stage_generated(model, cfgs, cluster, dispatch_overhead_ns=5000)
        assert (st == 0).all()
        eng.upload()
        eng.run()
        res = eng.results()
        for q, i in enumerate(idx):
            got[i] = res[q]
    for i, r in enumerate(rs):
        g = got[i]
        if (int(g["status"]) != 0 or int(g["total_ns"]) != r["total_ns"]
                or int(g["peak_mem_bytes"]) != r["peak_mem_bytes"] or bool(g["oom"]) != r["oom"]):
            bad.append((r["set"], r["ranks"], r["key"], int(g["status"]), int(g["total_ns"]),
                        r["total_ns"]))
    eng.close()
    assert not bad, bad[:5]
