"""N > 1 sharding logic on CPU: world_size-2 gloo processes (the GPU box runs
the same code over NCCL).  Checks that shards cover every (layer, seq, kv-head)
unit exactly once, that batch < world splits kv-heads, and that gather_heads
reassembles per-head outputs in order."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_18077_b200 import shard


def test_plan_covers_units_exactly_once():
    for batch, hkv, world in [(16, 8, 1), (16, 8, 2), (128, 8, 8), (8, 32, 8), (2, 8, 8), (1, 8, 4), (4, 8, 8)]:
        seen = []
        for r in range(world):
            seen += shard.plan(batch, hkv, world, r).units(3, batch, hkv)
        if batch >= world:
            assert sorted(seen) == list(range(3 * batch * hkv))
        else:
            assert sorted(seen) == list(range(3 * batch * hkv))  # split heads: still exactly once
    with pytest.raises(ValueError):
        shard.plan(3, 8, 2, 0)
    with pytest.raises(ValueError):
        shard.plan(1, 6, 4, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, batch, hkv, G, d, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = shard.plan(batch, hkv, world, rank)
    # fake per-head attention output: value encodes (seq, q-head, channel)
    local = torch.zeros(len(sh.seqs), len(sh.kv_heads) * G, d)
    for i, b in enumerate(sh.seqs):
        for jh, h in enumerate(sh.kv_heads):
            for g in range(G):
                local[i, jh * G + g] = b * 1000 + (h * G + g) + torch.arange(d) * 1e-3
    full = shard.gather_heads(local, sh)
    # timing-style max over ranks (as bench.py does)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    q.put((rank, sh.seqs, sh.kv_heads, full.tolist(), float(t.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("batch,hkv,world", [(4, 8, 2), (1, 8, 2), (2, 8, 4)])
def test_gloo_world2(batch, hkv, world):
    G, d = 2, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, batch, hkv, G, d, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(r[4] == float(world) for r in res)
    covered = sorted((b, h) for r in res for b in r[1] for h in r[2])
    if batch >= world:
        assert covered == [(b, h) for b in range(batch) for h in range(hkv)]
        for r in res:
            full = torch.tensor(r[3])
            assert full.shape == (batch // world, hkv * G, d)
    else:
        # every rank of a sequence group holds the full gathered head set, in head order
        for r in res:
            full = torch.tensor(r[3])
            b = r[1][0]
            assert full.shape == (1, hkv * G, d)
            for hq in range(hkv * G):
                assert torch.allclose(full[0, hq], b * 1000 + hq + torch.arange(d) * 1e-3)
