"""CPU, world_size 2 over gloo: the multi-GPU host path (contiguous env shards,
no hot-path collective, end-of-run gather of per-env results) reproduces the
single-process batch exactly. The per-shard compute here is the C oracle (the
checker); on the GPU box bench.py plugs in the CUDA path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_20304_b200.sharding import run_sharded, shard_range


def test_shard_ranges_partition():
    for n in (0, 1, 7, 65536, 1048576 + 3):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_env, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from cases import manifold_cases  # noqa: F401
    from oracle import Oracle
    from paper_2602_20304_b200 import api
    from paper_2602_20304_b200 import workloads as W
    from paper_2602_20304_b200.scene import SmoothingConfig

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ws = W.box_box(n_env)
    meshes = [api.surface_from_spec(b).mesh for b in ws.bodies]
    s = [Oracle.Surface(m.vertices, m.edges, b.sdf, b.vertex_topk, b.edge_topk)
         for m, b in zip(meshes, ws.bodies)]
    p1, p2 = ws.poses(n_env)  # generated in global env order, then sliced

    def compute(lo, hi):
        r = Oracle.manifold_batch(s[0], s[1], p1, p2[lo:hi], SmoothingConfig(), threads=1,
                                  want_meta=False)
        return torch.as_tensor(r["mean_dist"])

    full = run_sharded(compute, n_env, rank, world)
    q.put((rank, full.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_process():
    n_env = 37  # uneven shards
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_env, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import Oracle
    from paper_2602_20304_b200 import api
    from paper_2602_20304_b200 import workloads as W
    from paper_2602_20304_b200.scene import SmoothingConfig
    ws = W.box_box(n_env)
    meshes = [api.surface_from_spec(b).mesh for b in ws.bodies]
    s = [Oracle.Surface(m.vertices, m.edges, b.sdf, b.vertex_topk, b.edge_topk)
         for m, b in zip(meshes, ws.bodies)]
    p1, p2 = ws.poses(n_env)
    ref = Oracle.manifold_batch(s[0], s[1], p1, p2, SmoothingConfig(), threads=1)["mean_dist"]
    for r in (0, 1):
        assert np.array_equal(res[r], ref)  # bitwise: per-env results are shard-independent
