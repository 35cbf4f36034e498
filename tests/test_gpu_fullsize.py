"""GPU parity at the BASELINE configs' full sizes (BASELINE.json configs C and
D), every env against the C oracle on the same seeded inputs, plus the host
paths a deployment exercises around the kernels:

* config C: the four mixed-primitive buckets, 65,536 envs each (262,144);
  provenance (soft top-K src) bit-exact;
* config D: the drop scene's 10 body pairs x 32,768 envs, forward; the pose
  Jacobian kernel's primal at full size and its tangents against the
  reference's own generate_manifold<Dual12> on a scattered sample of envs;
* the host-buffer C-ABI call from several host threads at once (leased
  scratch) reproduces the single-threaded results bitwise;
* two processes on the GPU (world size 2, gloo for the end-of-run gather) each
  run their contiguous env shard through the CUDA path; the gathered per-env
  results equal the 1-process batch bitwise.
"""
import os
import socket
import threading

import numpy as np
import pytest
import torch

from helpers import assert_parity, assert_parity_conditioned
from oracle import Oracle, Ref
from test_gpu_jvp import jac_report
from paper_2602_20304_b200 import api
from paper_2602_20304_b200 import workloads as W
from paper_2602_20304_b200.scene import SmoothingConfig

pytestmark = pytest.mark.gpu
CHUNK = 16384


def oracle_surfaces(bodies, api_surfaces):
    return [Oracle.Surface(a.mesh.vertices, a.mesh.edges, b.sdf, b.vertex_topk, b.edge_topk)
            for a, b in zip(api_surfaces, bodies)]


@pytest.mark.parametrize("kind", W.MIXED_KINDS)
def test_config_c_bucket_full_size(cuda, kind):
    n = 65536
    ws = W.mixed_bucket(kind, n)
    a = [api.surface_from_spec(b) for b in ws.bodies]
    o = oracle_surfaces(ws.bodies, a)
    p1, p2 = ws.poses(n)
    cfg = SmoothingConfig()
    r = api.generate_manifold_batch(a[0], a[1], torch.as_tensor(p1, device="cuda"),
                                    torch.as_tensor(p2, device="cuda"), cfg, want_src=True)
    torch.cuda.synchronize()
    got = r["contacts"].cpu().numpy()
    src = r["src"].cpu().numpy()
    mean = r["mean_dist"].cpu().numpy()
    for lo in range(0, n, CHUNK):
        ref = Oracle.manifold_batch(o[0], o[1], p1, p2[lo:lo + CHUNK], cfg)

        def reeval(e, delta, lo=lo):
            return Oracle.manifold(o[0], o[1], p1[0], p2[lo + e] + delta, cfg)["contacts"]

        assert_parity_conditioned(got[lo:lo + CHUNK], ref["contacts"], reeval, what=f"config C {kind} envs {lo}+")
        assert np.array_equal(src[lo:lo + CHUNK], ref["meta"][..., 2:]), f"{kind}: provenance differs"
        assert np.allclose(mean[lo:lo + CHUNK], ref["mean_dist"], rtol=1e-5, atol=1e-6)


@pytest.fixture(scope="module")
def drop():
    n = 32768
    sc = W.drop_scene(n)
    bodies = [api.surface_from_spec(b) for b in sc.bodies]
    o = oracle_surfaces(sc.bodies, bodies)
    P = sc.poses(n)
    pairs = api.scene_pairs(len(bodies), sc.is_static())
    return dict(n=n, sc=sc, bodies=bodies, o=o, P=P, pairs=pairs)


def test_config_d_forward_full_size(cuda, drop):
    d = drop
    outs = api.generate_manifold_scene_batch(d["bodies"], torch.as_tensor(d["P"], device="cuda"), SmoothingConfig(),
                                             is_static=d["sc"].is_static(), want_src=True)
    torch.cuda.synchronize()
    for q, (i, j) in enumerate(d["pairs"]):
        got = outs[q]["contacts"].cpu().numpy()
        src = outs[q]["src"].cpu().numpy()
        ref = Oracle.manifold_batch(d["o"][i], d["o"][j], d["P"][:, i], d["P"][:, j], SmoothingConfig())

        def reeval(e, delta, i=i, j=j):
            return Oracle.manifold(d["o"][i], d["o"][j], d["P"][e, i], d["P"][e, j] + delta, SmoothingConfig())["contacts"]

        assert_parity_conditioned(got, ref["contacts"], reeval, what=f"config D pair {q} ({i},{j})")
        assert np.array_equal(src, ref["meta"][..., 2:])


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref (the compiled reference) not built")
def test_config_d_jvp_full_size(cuda, drop):
    d = drop
    cfg = SmoothingConfig()
    rs = [Ref.Surface(Ref.Mesh.box(b.mesh.box_half, b.mesh.subdivisions, b.mesh.quad_edges), b.sdf, b.vertex_topk,
                      b.edge_topk) for b in d["sc"].bodies]
    outs = api.generate_manifold_scene_jvp_batch(d["bodies"], torch.as_tensor(d["P"], device="cuda"), cfg,
                                                 is_static=d["sc"].is_static())
    torch.cuda.synchronize()
    idx = np.linspace(0, d["n"] - 1, 12).astype(int)
    for q, (i, j) in enumerate(d["pairs"]):
        got = outs[q]["contacts"].cpu().numpy()
        tan = outs[q]["tangents"].cpu().numpy()
        assert np.isfinite(tan).all()
        ref = Oracle.manifold_batch(d["o"][i], d["o"][j], d["P"][:, i], d["P"][:, j], cfg, want_meta=False)

        def reeval(e, delta, i=i, j=j):
            return Oracle.manifold(d["o"][i], d["o"][j], d["P"][e, i], d["P"][e, j] + delta, cfg)["contacts"]

        assert_parity_conditioned(got, ref["contacts"], reeval, what=f"config D JVP primal, pair {q}")
        # tangents vs the reference's own generate_manifold<Dual12> (compiled into
        # oracle/_ref) on a scattered sample of envs, with tests/test_gpu_jvp.py's
        # Frobenius tolerance per contact field
        for e in idx:
            ref_j = Ref.manifold_jvp(rs[i], rs[j], d["P"][e, i], d["P"][e, j], cfg)
            rep = jac_report(tan[e], ref_j["tangents"])
            assert max(rep.values()) <= 1.0, (q, int(e), rep)


def test_host_buffer_calls_from_many_threads(cuda):
    """cmgb_manifold_batch_host from 6 host threads at once (leased scratch,
    per-call pipeline streams): every thread's result equals the serial one."""
    n = 4096
    ws = W.box_box(n)
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    p1, p2 = ws.poses(n)
    jobs = [np.ascontiguousarray(p2[(k * 97) % n:][: n // 2]) for k in range(6)]
    serial = [api.generate_manifold_batch_host(s1, s2, p1, j, SmoothingConfig()) for j in jobs]
    C = api.layout(s1, s2)["n_contacts"]
    serial_c = []
    for j in jobs:
        c = np.empty((len(j), C, 8), np.float32)
        api.generate_manifold_batch_host(s1, s2, p1, j, SmoothingConfig(), contacts_out=c)
        serial_c.append(c)
    res = [None] * len(jobs)
    errs = []

    def work(k):
        try:
            c = np.empty((len(jobs[k]), C, 8), np.float32)
            m = api.generate_manifold_batch_host(s1, s2, p1, jobs[k], SmoothingConfig(), contacts_out=c,
                                                 stream=torch.cuda.Stream())
            res[k] = (m, c)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    for _ in range(3):
        ts = [threading.Thread(target=work, args=(k,)) for k in range(len(jobs))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errs, errs
        for k in range(len(jobs)):
            assert np.array_equal(res[k][0], serial[k])
            assert np.array_equal(res[k][1], serial_c[k])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cuda_rank(rank, world, port, n_env, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist

    from paper_2602_20304_b200.sharding import gather_shards, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ws = W.box_box(n_env)
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    p1, p2 = ws.poses(n_env)  # global env order, then sliced
    lo, hi = shard_range(n_env, rank, world)
    r = api.generate_manifold_batch(s1, s2, torch.as_tensor(p1, device="cuda"),
                                    torch.as_tensor(np.ascontiguousarray(p2[lo:hi]), device="cuda"), SmoothingConfig())
    torch.cuda.synchronize()
    full = gather_shards(r["mean_dist"].cpu(), n_env, rank, world)
    q.put((rank, full.numpy(), r["contacts"].cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_cuda_path_match_single_process(cuda):
    import torch.multiprocessing as mp

    n_env = 4099  # uneven shards
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cuda_rank, args=(r, 2, port, n_env, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        rank, mean, contacts = q.get(timeout=300)
        res[rank] = (mean, contacts)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ws = W.box_box(n_env)
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    p1, p2 = ws.poses(n_env)
    one = api.generate_manifold_batch(s1, s2, torch.as_tensor(p1, device="cuda"), torch.as_tensor(p2, device="cuda"),
                                      SmoothingConfig())
    torch.cuda.synchronize()
    ref_mean = one["mean_dist"].cpu().numpy()
    ref_c = one["contacts"].cpu().numpy()
    for r in (0, 1):
        assert np.array_equal(res[r][0], ref_mean)  # the gathered per-env results, bitwise
    assert np.array_equal(np.concatenate([res[0][1], res[1][1]]), ref_c)  # shards, bitwise
