"""Multi-GPU host logic on CPU: LPT sharding and the all_gather + merge of
per-GPU top-k candidates (gloo, world_size 2)."""
import os

import numpy as np
import torch.multiprocessing as mp

from paper_2503_20191_b200.api import merge_topk, shard_lpt


def test_shard_lpt_balances_and_covers():
    rng = np.random.default_rng(3)
    costs = rng.integers(1, 100, size=101).tolist()
    parts = shard_lpt(costs, 4)
    flat = sorted(i for p in parts for i in p)
    assert flat == list(range(101))
    loads = [sum(costs[i] for i in p) for p in parts]
    assert max(loads) - min(loads) <= max(costs)


def test_merge_topk_order():
    c = np.array([[5, 2, 0], [0, 1, 1], [5, 1, 2], [3, 9, 3], [-1, -1, -1]])
    m = merge_topk(c, 3)
    # time asc, key asc; time 0 (MFU 0.0) after every positive time
    assert m[:, 2].tolist() == [3, 2, 0]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2503_20191_b200.api import gather_merge
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(rank)
    k = 4
    cand = np.stack([rng.integers(1, 50, size=k), rng.integers(0, 1000, size=k),
                     rank * 100 + np.arange(k)], axis=1).astype(np.int64)
    merged = gather_merge(cand, k)
    q.put((rank, cand, merged))
    dist.destroy_process_group()


def test_gather_merge_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29611
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    allc = np.concatenate([c for _, c, _ in out])
    want = merge_topk(allc, 4)
    for _, _, merged in out:
        assert np.array_equal(merged, want)


class _StubEngine:
    """CPU stand-in for the engine in the sharding test: a deterministic
    'time' per config (with ties) and the device top-k's (time, key rank) order."""

    def stage_generated(self, model, cfgs, cluster, key_ranks=None, **kw):
        self.cfgs, self.kr = list(cfgs), np.asarray(key_ranks)

    def upload(self):
        pass

    def run(self):
        pass

    def topk(self, k):
        from paper_2503_20191_b200._abi import TOPK_DTYPE
        t = np.array([stub_time(c) for c in self.cfgs], dtype=np.int64)
        order = np.lexsort((self.kr, t))[:k]
        out = np.zeros(len(order), dtype=TOPK_DTYPE)
        out["time_ns"] = t[order]
        out["key_rank"] = self.kr[order]
        out["job"] = order
        return out


def stub_time(c):
    return 1 + (c.tp * 131 + c.pp * 31 + c.micro_mult * 7 + c.virtual_stages * 3
                + c.act_recompute + 2 * c.seq_parallel + 4 * c.dist_optimizer) % 97


def _c2_space():
    from paper_2503_20191_b200 import workload as W
    model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
    cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
    return W.SearchSpace(global_batch=512), model, cluster


def _shard_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2503_20191_b200.api import evaluate_space_distributed
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    space, model, cluster = _c2_space()
    merged, configs = evaluate_space_distributed(space, model, cluster, k=8, engine=_StubEngine())
    q.put((rank, merged))
    dist.destroy_process_group()


def test_evaluate_space_distributed_gloo_world2_equals_single():
    """One search sharded over 2 processes (LPT + all_gather + merge) selects the
    same top-k, in the same order, as the whole search on one process."""
    from paper_2503_20191_b200 import workload as W
    from paper_2503_20191_b200.api import evaluate_sharded
    space, model, cluster = _c2_space()
    configs = W.enumerate_space(space, model, cluster)
    single, _ = evaluate_sharded(model, configs, cluster, 8, _StubEngine())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_shard_worker, args=(r, 2, 29613, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=180) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for _, merged in out:
        assert np.array_equal(merged, single)
    # ties on time are broken by the config key, as the reference's _rank
    times = [stub_time(configs[int(i)]) for i in single[:, 2]]
    keys = [configs[int(i)].key() for i in single[:, 2]]
    assert list(zip(times, keys)) == sorted(zip(times, keys))


def test_rank_by_mfu_matches_reference_rank():
    """Candidates of searches with different global batches merge in the
    reference's _rank order (search.py:349-357), not by time."""
    import sys
    import pytest
    from conftest import REPO
    ref = os.path.join(REPO, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "dltsim")):
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, ref)
    from dltsim.search import TrialRecord, TrialStatus, _rank
    from dltsim.sim import compute_mfu
    from paper_2503_20191_b200 import workload as W
    from paper_2503_20191_b200.api import rank_by_mfu
    model = W.ModelSpec("gpt3-1.3b", 24, 2048, 2048, 51200)
    cluster = W.ClusterSpec(1, 8, 80 * 2 ** 30, W.load_device_preset("fast"))
    rng = np.random.default_rng(5)
    cfgs = {gb: W.enumerate_space(W.SearchSpace(global_batch=gb), model, cluster)[:40]
            for gb in (512, 1024)}
    rows = [(int(rng.integers(1, 4) * 10 ** 9 * (gb // 512)), gb, i)
            for gb in (512, 1024) for i in range(40)]
    got = [cfgs[r[1]][r[2]] for r, _ in rank_by_mfu(rows, model,
                                                     lambda r: (cfgs[r[1]][r[2]], cluster))]

    class Rep:
        def __init__(self, t):
            self.total_ns, self.oom = t, False
    recs = []
    for t, gb, i in rows:
        from dltsim.workload import ModelSpec as RefModel
        flops = RefModel("gpt3-1.3b", 24, 2048, 2048, 51200).iteration_flops(gb)
        mfu = compute_mfu(Rep(t), flops, cluster, model.dtype)
        recs.append(TrialRecord(cfgs[gb][i], TrialStatus.COMPLETED, time_ns=t, mfu=mfu))
    assert got == [r.config for r in _rank(recs)]
