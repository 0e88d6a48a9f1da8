"""Batch x head sharding of the DMA forward across ranks (one process per GPU).

Every (batch, head) of the forward is independent (the reference is a
single-head function, attention.py:282; query tiles and heads never exchange
data), so the multi-GPU path is a partition plus one output gather:

* the unit of work is a (batch, kv-head) pair, so the H/KVH query heads that
  share a K/V head stay on one rank and GQA K/V are never duplicated;
* rank r of W owns a contiguous range of the flattened units; in the flattened
  ``[B*H]`` query-head index those are the contiguous heads
  ``[start*g, stop*g)`` (g = H/KVH) and K/V heads ``[start, stop)``;
* the hot path has no collective; ``gather`` reassembles O with one
  ``all_gather_into_tensor`` (NCCL over NVLink on B200 boxes, gloo in the CPU
  tests).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    """Rank-local slice of a [B, H, L, D] problem (flattened head ranges)."""

    rank: int
    world: int
    units: int          # B * KVH
    group: int          # H / KVH
    start: int          # first (b, kvh) unit
    stop: int           # one past the last unit

    @property
    def q_heads(self) -> slice:
        return slice(self.start * self.group, self.stop * self.group)

    @property
    def kv_heads(self) -> slice:
        return slice(self.start, self.stop)

    @property
    def max_units(self) -> int:
        return -(-self.units // self.world)


def plan_shard(batch: int, heads: int, kv_heads: int, world: int, rank: int) -> Shard:
    """Contiguous, balanced split of the B*KVH units (the first units % world ranks get one more)."""
    if heads % kv_heads:
        raise ValueError(f"heads {heads} not divisible by kv_heads {kv_heads}")
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    units = batch * kv_heads
    base, extra = divmod(units, world)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return Shard(rank, world, units, heads // kv_heads, start, stop)


def local_inputs(q, k, v, shard: Shard):
    """This rank's q/k/v as [1, heads_local, L, D] views (q [B,H,L,D], k/v [B,KVH,L,D])."""
    B, H, Lq, D = q.shape
    _, KVH, Lk, _ = k.shape
    qf = q.reshape(B * H, Lq, D)[shard.q_heads]
    kf = k.reshape(B * KVH, Lk, k.shape[-1])[shard.kv_heads]
    vf = v.reshape(B * KVH, Lk, v.shape[-1])[shard.kv_heads]
    return qf.unsqueeze(0), kf.unsqueeze(0), vf.unsqueeze(0)


def gather(o_local, shard: Shard, batch: int, heads: int, group=None):
    """all_gather the per-rank O shards ([1, heads_local, L, DV]) into O [B, H, L, DV] on every rank."""
    import torch
    import torch.distributed as dist

    _, hl, L, DV = o_local.shape
    per = shard.max_units * shard.group  # padded heads per rank (uneven splits)
    buf = o_local.new_zeros((per, L, DV))
    buf[:hl] = o_local[0]
    out = o_local.new_empty((shard.world * per, L, DV))
    dist.all_gather_into_tensor(out, buf.contiguous(), group=group)
    pieces = []
    for r in range(shard.world):
        s = plan_shard(batch, heads, heads // shard.group, shard.world, r)
        n = (s.stop - s.start) * s.group
        pieces.append(out[r * per:r * per + n])
    return torch.cat(pieces).reshape(batch, heads, L, DV)


def dma_attention_sharded(q, k, v, cfg, group=None, compute=None, gather_output=True):
    """Sharded forward: this rank runs its (b, kv-head) slice, then O is all-gathered.

    ``compute(q, k, v, cfg)`` defaults to ``paper_2604_03950_b200.dma_attention``
    (the sm_100a kernel); tests inject a CPU stand-in to check the plumbing.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if compute is None:
        from .attention import dma_attention, kv_split_count

        # every rank takes the whole problem's KV split count (small problems): the gathered
        # O is then bit-identical to one device call over the whole problem at any world size
        n_split = kv_split_count(q.shape, k.shape, v.shape, cfg)

        def compute(ql, kl, vl, c):
            return dma_attention(ql, kl, vl, c, kv_split=n_split)
    B, H = q.shape[0], q.shape[1]
    shard = plan_shard(B, H, k.shape[1], world, rank)
    ql, kl, vl = local_inputs(q, k, v, shard)
    o_local = compute(ql, kl, vl, cfg)
    if not gather_output or world == 1:
        return o_local, shard
    return gather(o_local, shard, B, H, group), shard
