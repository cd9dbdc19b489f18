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
