"""World-size-2 gloo tests (CPU) of the batch-shard driver's host logic:
shard ranges, the setup broadcast of a stretched CSR, MAX-over-ranks timing,
and the generator's shard invariance (image n is identical on any rank)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1802_10280_b200 import inputs, shard, workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L = workloads.TINY
        if rank == 0:
            import oracle
            w = inputs.layer_weights("tiny", L, 800)
            rp, ci, v = oracle.csr_stretch(w, L.H, L.W, L.stride, L.pad)
            b = inputs.bias("tiny", "tiny", L.M)
            t = shard.broadcast_csr(rp, ci, v, b, "cpu")
        else:
            t = shard.broadcast_csr(None, None, None, None, "cpu")
        digest = [x.numpy().tobytes() for x in t]
        a, bnd = shard.shard_range(128, rank, world)
        x = inputs.activations("tiny", "tiny", a, bnd - a, L.C, L.H, L.W)
        mx = shard.max_over_ranks(10.0 + rank, "cpu")
        q.put((rank, digest, (a, bnd), x.tobytes(), mx))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_broadcast_shard_max():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict()
    for _ in range(world):
        r = q.get(timeout=240)
        res[r[0]] = r
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1]                      # identical CSR + bias on both ranks
    assert res[0][2] == (0, 64) and res[1][2] == (64, 128)
    L = workloads.TINY
    full = inputs.activations("tiny", "tiny", 0, 128, L.C, L.H, L.W)
    assert res[0][3] + res[1][3] == full.tobytes()    # shards tile the global batch exactly
    assert res[0][4] == res[1][4] == 11.0


@pytest.mark.parametrize("n,w", [(128, 1), (128, 3), (7, 4), (0, 2), (16, 8)])
def test_shard_range_partition(n, w):
    rs = [shard.shard_range(n, r, w) for r in range(w)]
    assert rs[0][0] == 0 and rs[-1][1] == n
    for (a, b), (c, d) in zip(rs, rs[1:]):
        assert b == c
    sizes = [b - a for a, b in rs]
    assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_bench_strong_scaling_ranges(world):
    # bench.py's default: the GLOBAL batch 128 is split across ranks (strong scaling), every image once
    import argparse
    import bench
    wl = workloads.workload("resnet50")
    args = argparse.Namespace(batch=None, weak=False)
    seen = []
    for r in range(world):
        n0, B, GB = bench.batch_range(args, wl, r, world)
        assert GB == 128 and B == 128 // world
        seen += list(range(n0, n0 + B))
    assert seen == list(range(128))
    args.weak = True
    assert bench.batch_range(args, wl, 1, world) == (128, 128, 128 * world)


def test_bench_jit_tunings_per_workload():
    # host logic of bench.py's tuning lists: ResNet-50 (v1 and v1.5) compiles its three stage winners,
    # every other workload the full list; every entry parses into <= 18 escoin_csr_jit tunables, and the
    # split-channel entries ask for "auto count, only where a split is needed" (ks = -2, index 17)
    import sys
    sys.argv = ["bench.py", "--workload", "resnet50"]
    import bench
    assert bench.parse().jit_tunings == bench.RESNET_JIT_TUNINGS
    sys.argv = ["bench.py", "--workload", "googlenet"]
    assert bench.parse().jit_tunings == bench.DEFAULT_JIT_TUNINGS
    sys.argv = ["bench.py", "--workload", "alexnet", "--jit-tunings", "0;32,1"]
    assert bench.parse().jit_tunings == "0;32,1"
    for wl in ["resnet50", "resnet50_v15", "alexnet", "googlenet", "googlenet_1x1"]:
        entries = [[int(v) for v in t.split(",")] for t in bench.jit_tunings_for(wl).split(";") if t.strip() != "0"]
        assert entries and all(len(e) <= 18 for e in entries)
    ks = [e for e in ([int(v) for v in t.split(",")] for t in bench.DEFAULT_JIT_TUNINGS.split(";") if t != "0")
          if len(e) == 18]
    assert len(ks) == 2 and all(e[17] == -2 for e in ks)
    assert len(bench.RESNET_JIT_TUNINGS.split(";")) == 3
