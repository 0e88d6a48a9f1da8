"""Multi-rank plumbing of the batch x head sharding (CPU, gloo, world size 2 and 3).

The compute step is a CPU stand-in that depends on the query head AND on the
K/V head it is paired with, so a wrong GQA mapping, a wrong slice or a wrong
gather order changes the result.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_03950_b200.sharding import dma_attention_sharded, plan_shard


def stand_in(q, k, v, cfg):
    """O[h] = q[h] * 2 + mean(k[h // g]) + v[h // g]  (per head, GQA-aware)."""
    g = q.shape[1] // k.shape[1]
    kk = k.repeat_interleave(g, dim=1)
    vv = v.repeat_interleave(g, dim=1)
    return q * 2 + kk.mean(dim=(2, 3), keepdim=True) + vv


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, shapes, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for i, (B, H, KVH, L, D) in enumerate(shapes):
            g = torch.Generator().manual_seed(100 + i)
            q = torch.randn(B, H, L, D, generator=g)
            k = torch.randn(B, KVH, L, D, generator=g)
            v = torch.randn(B, KVH, L, D, generator=g)
            out, shard = dma_attention_sharded(q, k, v, None, compute=stand_in)
            want = stand_in(q, k, v, None)
            results[(rank, i)] = bool(torch.equal(out, want)) and tuple(out.shape) == (B, H, L, D)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gather_matches_unsharded(world):
    shapes = [(2, 8, 2, 16, 8), (1, 32, 8, 8, 4), (3, 4, 4, 8, 4), (1, 6, 3, 4, 4)]
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), shapes, results), nprocs=world, join=True)
    assert len(results) == world * len(shapes)
    assert all(results.values()), dict(results)


def test_plan_shard_partition():
    for B, H, KVH in [(1, 32, 8), (8, 64, 64), (3, 12, 4), (1, 1, 1)]:
        for W in (1, 2, 3, 4, 8):
            shards = [plan_shard(B, H, KVH, W, r) for r in range(W)]
            covered = [u for s in shards for u in range(s.start, s.stop)]
            assert covered == list(range(B * KVH))
            sizes = [s.stop - s.start for s in shards]
            assert max(sizes) - min(sizes) <= 1
            for s in shards:  # q heads of a unit are exactly its GQA group
                assert s.q_heads.stop - s.q_heads.start == (s.stop - s.start) * (H // KVH)
    with pytest.raises(ValueError):
        plan_shard(1, 6, 4, 2, 0)
