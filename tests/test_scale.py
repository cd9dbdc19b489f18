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


# --- full rank counts: C3 at 256-1,024 ranks, C4 at 512-2,048 ranks -------------------
# tests/golden/scale_big_results.json (make_scale_golden.py): 24 C3 + 18 C4 configs
# of up to 46.5 M rank-ops each, covering pp=16, virtual stages 4/5/10, micro_mult
# 2-16, act_recompute / dist_optimizer on and off, global batch 2,048-16,384.

def big_rows():
    with open(os.path.join(GOLDEN, "scale_big_results.json")) as f:
        return json.load(f)


def test_scale_big_goldens_cover_the_lattices():
    rs = big_rows()
    c3 = {r["ranks"] for r in rs if r["set"] == "C3"}
    c4 = [r for r in rs if r["set"] == "C4"]
    assert c3 == {256, 512, 1024}
    assert {r["ranks"] for r in c4} == {512, 1024, 2048}
    assert {r["key"][1] for r in c4} >= {16}                      # pp = 16
    assert {r["key"][3] for r in c4} >= {4, 5, 10}                # virtual stages
    assert max(r["key"][2] for r in c4) >= 8                      # micro_mult
    assert {r["key"][7] for r in c4} >= {2048, 4096, 8192, 16384}


def test_scale_big_generator_digests_match_reference():
    bad = []
    for r in big_rows():
        model, cluster, cfg = point(r)
        job = W.generate_job(model, cfg, cluster, dispatch_overhead_ns=5000)
        if job.rank_ops() != r["rank_ops"] or raw_digest(job) != r["raw_sha256"]:
            bad.append((r["set"], r["ranks"], cfg.label()))
    assert not bad, bad[:5]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["auto", "full-rank", "lane", "warp", "no-blocks"])
def test_scale_big_engine_matches_reference(mode):
    """C3/C4 at their full rank counts against the reference, on every scheduler
    path: collapsed (auto), full-rank (grid jobs for the lane kernel at 512+
    ranks), forced lane, forced warp-window, and without kernel blocks."""
    from paper_2503_20191_b200.engine import Engine
    rs = big_rows()
    eng = Engine(0, collapse=mode != "full-rank",
                 sched={"lane": "lane", "warp": "warp"}.get(mode, "auto"),
                 blocks=mode != "no-blocks")
    groups = {}
    for i, r in enumerate(rs):
        groups.setdefault((tuple(r["model"]), r["ranks"]), []).append(i)
    bad = []
    for idx in groups.values():
        model, cluster, _ = point(rs[idx[0]])
        cfgs = [point(rs[i])[2] for i in idx]
        st = eng.stage_generated(model, cfgs, cluster, dispatch_overhead_ns=5000)
        assert (st == 0).all()
        eng.upload()
        eng.run()
        res = eng.results()
        for q, i in enumerate(idx):
            g, r = res[q], rs[i]
            if (int(g["status"]) != 0 or int(g["total_ns"]) != r["total_ns"]
                    or int(g["peak_mem_bytes"]) != r["peak_mem_bytes"]
                    or bool(g["oom"]) != r["oom"] or int(g["rank_ops"]) != r["rank_ops"]):
                bad.append((r["set"], r["ranks"], r["key"], int(g["status"]),
                            int(g["total_ns"]), r["total_ns"]))
    eng.close()
    assert not bad, bad[:5]


@pytest.mark.gpu
def test_scale_big_topk_is_reference_order():
    """One batch per (set, ranks): the device top-k equals the reference's
    (time_ns, key) order over the pinned configs."""
    from paper_2503_20191_b200.api import key_ranks
    from paper_2503_20191_b200.engine import Engine
    rs = big_rows()
    eng = Engine(0)
    groups = {}
    for i, r in enumerate(rs):
        groups.setdefault((r["set"], r["ranks"]), []).append(i)
    for idx in groups.values():
        cfgs = [point(rs[i])[2] for i in idx]
        clusters = {point(rs[i])[1].num_devices for i in idx}
        assert len(clusters) == 1
        model, cluster, _ = point(rs[idx[0]])
        kr = key_ranks(cfgs)
        eng.stage_generated(model, cfgs, cluster, dispatch_overhead_ns=5000, key_ranks=kr)
        eng.upload()
        eng.run()
        eng.results()
        top = eng.topk(len(idx))
        ok = [i for i in idx if not rs[i]["oom"]]
        want = sorted(ok, key=lambda i: (rs[i]["total_ns"] if rs[i]["total_ns"] > 0
                                         else 1 << 62, tuple(rs[i]["key"])))
        got = [idx[int(t["job"])] for t in top]
        assert got == want
    eng.close()
