"""Multi-GPU sharding of the attention hot path.

The unit of work is a (sequence b, layer, kv-head h) cache; units are fully
independent in prefill, selection, quantization and decode (
pipeline.cpp:141-163), so the path shards with NO collective:

* batch-major: rank r owns sequences [r*B/N, (r+1)*B/N) when N divides B;
* when B < N, sequences are replicated across groups of N/B ranks and the
  kv-heads of a sequence are split across the group (Hkv/(N/B) each).  Only
  then does a consumer that needs the full hidden vector of a sequence need an
  exchange: gather_heads() all-gathers the per-rank [B_local, Hq_local, d]
  outputs (NCCL over NVLink on the GPU box, gloo in the CPU tests).

One process per GPU; torch.distributed is the plumbing.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    seqs: Tuple[int, ...]      # global sequence ids owned (or shared) by this rank
    kv_heads: Tuple[int, ...]  # kv-heads of those sequences computed by this rank
    group: int                 # ranks sharing each sequence (1 = pure batch sharding)

    def units(self, layers: int, batch: int, n_kv_heads: int) -> List[int]:
        """Global unit ids u = (layer * batch + b) * n_kv_heads + h owned by this rank."""
        return [(l * batch + b) * n_kv_heads + h for l in range(layers) for b in self.seqs for h in self.kv_heads]


def plan(batch: int, n_kv_heads: int, world: int, rank: int) -> Shard:
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if batch >= world:
        if batch % world:
            raise ValueError(f"batch {batch} not divisible by world {world}")
        per = batch // world
        return Shard(rank, world, tuple(range(rank * per, (rank + 1) * per)), tuple(range(n_kv_heads)), 1)
    if world % batch:
        raise ValueError(f"world {world} not divisible by batch {batch}")
    group = world // batch
    if n_kv_heads % group:
        raise ValueError(f"{n_kv_heads} kv-heads cannot be split over {group} ranks")
    hp = n_kv_heads // group
    b, j = divmod(rank, group)
    return Shard(rank, world, (b,), tuple(range(j * hp, (j + 1) * hp)), group)


_SEQ_GROUPS = {}


def seq_groups(shard: Shard):
    """The process groups of ranks sharing a sequence ([b*group, (b+1)*group) for each b).
    dist.new_group is collective over the whole world, so every rank creates every group
    (once, cached) and uses its own."""
    import torch.distributed as dist
    key = (shard.world, shard.group)
    if key not in _SEQ_GROUPS:
        _SEQ_GROUPS[key] = [dist.new_group(list(range(b * shard.group, (b + 1) * shard.group)))
                            for b in range(shard.world // shard.group)]
    return _SEQ_GROUPS[key]


def gather_heads(local_out, shard: Shard, group_ranks=None):
    """All-gather per-head outputs [B_local, Hq_local, d] into [B_local, Hq, d] across the
    ranks sharing a sequence (only needed when batch < world).  group_ranks: the process
    group of this rank's sequence; None builds the sequence groups (collective: every rank
    of the world must call it the same number of times)."""
    import torch
    import torch.distributed as dist
    if shard.group == 1:
        return local_out
    if group_ranks is None:
        group_ranks = seq_groups(shard)[shard.rank // shard.group]
    parts = [torch.empty_like(local_out) for _ in range(shard.group)]
    dist.all_gather(parts, local_out.contiguous(), group=group_ranks)
    return torch.cat(parts, dim=1)
