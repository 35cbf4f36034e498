"""The host-buffer scene call (cmgb_manifold_scene_batch_host: host poses in,
each pair's per-env mean distance out, a lead env chunk then the rest on two
pipeline streams) must return exactly what the device-buffer scene call
(cmgb_manifold_scene_batch) computes for the same poses, across the chunk
boundary."""
import numpy as np
import pytest

from paper_2602_20304_b200 import api
from paper_2602_20304_b200 import workloads as W
from paper_2602_20304_b200.scene import SmoothingConfig


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 300, 5000])
def test_scene_host_matches_device(cuda, n):
    import torch

    sc = W.drop_scene(n)
    bodies = [api.surface_from_spec(b) for b in sc.bodies]
    poses = np.ascontiguousarray(sc.poses(n), dtype=np.float64)
    cfg = SmoothingConfig()
    got = api.generate_manifold_scene_batch_host(bodies, poses, cfg, is_static=sc.is_static())
    ref = api.generate_manifold_scene_batch(bodies, torch.as_tensor(poses, device=cuda), cfg,
                                            is_static=sc.is_static())
    torch.cuda.synchronize()
    assert got.shape == (len(ref), n)
    for q, r in enumerate(ref):
        assert np.array_equal(got[q], r["mean_dist"].cpu().numpy()), q


@pytest.mark.gpu
def test_scene_host_rejects_bad_arguments(cuda):
    sc = W.drop_scene(4)
    bodies = [api.surface_from_spec(b) for b in sc.bodies]
    poses = np.asarray(sc.poses(4), np.float64)
    with pytest.raises(ValueError):
        api.generate_manifold_scene_batch_host(bodies[:-1], poses)
    with pytest.raises(ValueError):
        api.generate_manifold_scene_batch_host(bodies, poses, mean_out=np.empty((1, 4), np.float32))
    with pytest.raises(Exception):
        api.generate_manifold_scene_batch_host(bodies, poses, pairs=np.array([[0, 9]], np.int32))
