"""Native trace generator (csrc/gen.cpp) == the reference frontend + collator.

Host-only (no GPU): the generator is C++ host code in libmaya_b200.so.
* every one of the 512 C2 configs hashes to the digest of the reference's
  own collated job (tests/golden/c2_results.json, raw_sha256);
* when the reference is importable (build container), event-level equality
  on a spread of lattices, schedules and clusters.
"""
import itertools
import json
import os
import sys

import numpy as np
import pytest

from paper_2503_20191_b200 import workload as W
from paper_2503_20191_b200.rawtrace import raw_digest

from conftest import GOLDEN

REF = os.environ.get("MAYA_REF", "/root/reference/pkg")


def c2_space():
    model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
    cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
    return model, cluster, W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster)[:512]


def test_c2_digests_match_reference():
    with open(os.path.join(GOLDEN, "c2_results.json")) as f:
        gold = json.load(f)
    model, cluster, cfgs = c2_space()
    assert [tuple(g["key"]) for g in gold] == [c.key() for c in cfgs]
    bad = []
    for cfg, g in zip(cfgs, gold):
        job = W.generate_job(model, cfg, cluster, dispatch_overhead_ns=5000)
        assert job.rank_ops() == g["rank_ops"]
        if raw_digest(job) != g["raw_sha256"]:
            bad.append(cfg.label())
    assert not bad, bad[:5]


def test_invalid_config_raises_config_error():
    model, cluster, _ = c2_space()
    with pytest.raises(W.ConfigError, match="global_batch"):
        W.generate_job(model, W.ConfigPoint(1, 1, 6, 1, False, False, False, 512), cluster)


def test_validate_matches_enumeration_counts():
    # search.py:66-79 over the default lattice: 1,920 points, 576 valid for C2
    model, cluster, cfgs = c2_space()
    allp = W.enumerate_space(W.SearchSpace(global_batch=512), model, cluster, with_invalid=True)
    assert len(allp) == 1920
    assert sum(1 for _, r in allp if not r) == 576


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "src", "dltsim")),
                    reason="reference not present (GPU box)")
def test_generator_event_level_vs_reference():
    sys.path.insert(0, os.path.join(REF, "src"))
    from dltsim.cluster import ClusterSpec, load_device_preset
    from dltsim.collate import collate
    from dltsim.workload import (ConfigPoint, ModelSpec, ScheduleKind, default_schedule,
                                 generate_representatives, validate_config)
    from paper_2503_20191_b200.rawtrace import from_reference
    cases = []
    m = ModelSpec("t", 8, 128, 64, 512)
    for hosts, dph, dev in ((2, 8, "fast"), (4, 2, "slow"), (1, 4, "fast")):
        cl = ClusterSpec(hosts, dph, 2 ** 34, load_device_preset(dev))
        for tp, pp, mm, vs in itertools.product((1, 2, 4), (1, 2, 4), (1, 2), (1, 2)):
            for rc, sp, dz in ((False, False, False), (True, True, True), (False, True, False)):
                cfg = ConfigPoint(tp, pp, mm, vs, rc, sp, dz, 64)
                if validate_config(m, cfg, cl):
                    continue
                cases.append((m, cfg, cl, None))
    cl = ClusterSpec(1, 4, 2 ** 34, load_device_preset("fast"))
    for p, mm in ((2, 2), (4, 1)):
        cases.append((m, ConfigPoint(1, p, mm, 1, False, False, False, 64), cl, ScheduleKind.GPIPE))
    for model, cfg, cl, sched in cases:
        s = sched or default_schedule(cfg)
        tr, ex = generate_representatives(model, cfg, cl, s, dispatch_overhead_ns=777)
        ref = from_reference(collate(tr, ex, cl))
        got = W.generate_job(model, cfg, cl, schedule=s, dispatch_overhead_ns=777)
        assert raw_digest(ref) == raw_digest(got), (cfg, s)


def _pack_compare(model, cfgs, cluster, collapse, schedule=None, overhead=5000):
    import ctypes as C
    from paper_2503_20191_b200.workload import (ConfigC, cluster_c, config_c, model_c,
                                                schedule_code, _gen_lib)
    L = _gen_lib()
    L.maya_debug_pack_compare.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                          C.c_int32, C.c_int64, C.c_int32]
    arr = (ConfigC * len(cfgs))(*[config_c(c) for c in cfgs])
    m, cl = model_c(model), cluster_c(cluster)
    return L.maya_debug_pack_compare(C.byref(m), len(cfgs), arr, C.byref(cl),
                                     schedule_code(schedule), overhead, int(collapse))


@pytest.mark.parametrize("collapse", [True, False])
def test_fused_generate_pack_equals_generate_then_pack(collapse):
    """engine's maya_batch_add_generated packs generator events on the fly
    (pack.cpp pack_generated); it must produce byte-identical JobPacks to
    generate_job + pack_job on the C2 lattice and the C3/C4 golden configs."""
    model, cluster, cfgs = c2_space()
    assert _pack_compare(model, cfgs, cluster, collapse) == 0
    with open(os.path.join(GOLDEN, "scale_results.json")) as f:
        rows = json.load(f)
    for r in rows[::3]:
        m = W.ModelSpec(*r["model"])
        cl = W.ClusterSpec(r["ranks"] // 8, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
        assert _pack_compare(m, [W.ConfigPoint(*r["key"])], cl, collapse) == 0, r["key"]
    # small lattices, every schedule, odd overheads
    m = W.ModelSpec("t", 8, 128, 64, 512)
    cl = W.ClusterSpec(2, 8, 2 ** 34, W.load_device_preset("fast"))
    small = W.enumerate_space(W.SearchSpace(global_batch=64), m, cl)
    assert _pack_compare(m, small, cl, collapse, overhead=777) == 0
    assert _pack_compare(m, small, cl, collapse, overhead=0) == 0
