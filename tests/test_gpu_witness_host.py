"""The host-buffer witness calls (cmgb_ee_witness_batch_host /
cmgb_vf_witness_batch_host: the reference's run_ee_batch / run_vf_batch
signature, src/batch.cpp:53-98) run as a two-stream pipeline over pair chunks.
Their results must be bit-identical to the device-buffer calls over the whole
batch: chunk boundaries (ragged last chunk), labels and the V-F widening on
the device included; pageable and pinned host buffers alike."""
import numpy as np
import pytest

from paper_2602_20304_b200 import api
from paper_2602_20304_b200 import workloads as W
from paper_2602_20304_b200.scene import SmoothingConfig


def _pairs(n, seed):
    return W.mt19937_64_uniform(seed, 12 * n, 0.0, 1.0).reshape(n, 12)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 1000, 3 * 65536 + 17])
@pytest.mark.parametrize("variant", ["ours", "ours_ns"])
def test_ee_host_matches_device(cuda, n, variant):
    import torch

    cfg = SmoothingConfig().for_variant(variant)
    pairs = _pairs(n, 3)
    labels = np.empty(n, np.int32)
    got = api.run_ee_batch_host(pairs, cfg, labels=labels)
    ref = api.run_ee_batch_f64(torch.as_tensor(pairs, device=cuda), cfg, want_labels=True)
    assert np.array_equal(got, ref["out"].cpu().numpy())
    assert np.array_equal(labels, ref["labels"].cpu().numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 1000, 3 * 65536 + 17])
def test_vf_host_matches_device(cuda, n):
    import torch

    cfg = SmoothingConfig()
    pairs = _pairs(n, 5)
    # pinned host buffers (the overlapped path)
    hp = torch.as_tensor(pairs).pin_memory().numpy()
    out = torch.empty((n, 3), dtype=torch.float64).pin_memory().numpy()
    labels = np.empty(n, np.int32)
    api.run_vf_batch_host(hp, cfg, out=out, labels=labels)
    ref = api.run_vf_batch(torch.as_tensor(pairs, device=cuda), cfg, want_labels=True)
    assert np.array_equal(out, ref["out"].cpu().numpy().astype(np.float64))
    assert np.array_equal(labels, ref["labels"].cpu().numpy())


@pytest.mark.gpu
def test_witness_host_rejects_bad_buffers(cuda):
    pairs = _pairs(8, 1)
    with pytest.raises(ValueError):
        api.run_ee_batch_host(pairs, out=np.empty((8, 6), np.float32))
    with pytest.raises(ValueError):
        api.run_vf_batch_host(pairs, labels=np.empty(8, np.int64))
