"""bench.py's output contract (one JSON line, the keys the driver and the judge read)."""
import json
import os
import subprocess
import sys

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_line():
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "1"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    for k in ("metric", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "config", "cpu_baseline", "e2e"):
        assert k in d
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_b200_arm_line():
    d = _line(["--steps", "3", "--warmup", "3", "--no-prefill", "--no-cpu-baseline"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0.2 < r["frac"] < 1.05
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-6
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_b200_arm_lwm_shard_line():
    """configs[4]'s per-GPU shard (one LWM-Text-7B sequence, 32 MHA heads, 256K context)."""
    d = _line(["--workload", "lwm-7b", "--steps", "3", "--warmup", "3", "--no-prefill", "--no-cpu-baseline"])
    assert "LWM-Text-7B" in d["metric"] and d["config"]["context"] == 262144 and d["config"]["batch_per_gpu"] == 1
    assert d["value"] > 0 and 0.2 < d["roofline"]["frac"] < 1.05


def _rank_logic_worker(rank, world, port, q):
    import argparse

    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import bench
    got = {}
    for wl, batch in (("llama3-8b", None), ("llama3-8b", 1), ("lwm-7b", None)):
        args = argparse.Namespace(workload=wl, batch=batch)
        sh, firsts, upl = bench.rank_units(args, rank, world)
        units = [f + j for f in firsts for j in range(upl)]
        got[(wl, batch)] = (bench.global_batch(args, world), units)
    m = bench.dist_max(float(rank + 1), world)
    bench.barrier(world)
    q.put((rank, got, m))
    dist.destroy_process_group()


def test_bench_rank_logic_gloo_world2():
    """bench.py's own N > 1 logic on two gloo ranks: the default N > 1 workload is configs[2]'s
    global batch 128 (configs[4]: 8), the ranks' unit ranges (shard.plan, contiguous per layer)
    cover every global (layer, seq, kv-head) unit exactly once, and timings reduce as the max
    over ranks."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_logic_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=180) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[2] == 2.0 for r in res)
    for key, (layers, hkv) in {("llama3-8b", None): (32, 8), ("llama3-8b", 1): (32, 8), ("lwm-7b", None): (32, 32)}.items():
        B = res[0][1][key][0]
        assert B == {("llama3-8b", None): 128, ("llama3-8b", 1): 1, ("lwm-7b", None): 8}[key]
        units = sorted(u for r in res for u in r[1][key][1])
        assert units == list(range(layers * B * hkv)), key


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with two ranks (the reference arm
    runs on rank 0 only and reports n_gpus 2 and configs[2]'s global batch)."""
    d = _line(["--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "1", "--no-config0",
               "--cpu-units-per-layer", "1"], timeout=900)
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 128 and d["impl"] == "reference"
