"""GPU Siddon densifier (qrb_siddon_densify) vs the host restatement."""

import numpy as np
import pytest

from paper_1907_01891_b200 import ct_system as cs

pytestmark = pytest.mark.gpu


def host_dense_device(g, lda):
    import torch
    r, c, v = cs.siddon_coo(g)
    a = torch.zeros((g.n_pixels, lda), dtype=torch.float64, device="cuda")
    a.view(-1).index_put_((torch.from_numpy(c * lda + r).cuda(),), torch.from_numpy(v).cuda())
    return a


@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_gpu_siddon_bit_identical_to_host(cfg):
    import torch
    g = cs.config_geometry(cfg)
    lda = (g.n_rays + 31) // 32 * 32
    ref = host_dense_device(g, lda)
    got = cs.densify_device(g, lda)
    diff = (got != ref).sum().item()
    assert diff == 0, f"{diff} entries differ (max {float((got - ref).abs().max()):.3e})"


@pytest.mark.parametrize("world", [2, 3])
def test_gpu_siddon_block_cyclic_columns(world):
    import torch
    from paper_1907_01891_b200 import dist as qd
    g = cs.config_geometry(1)
    lda = (g.n_rays + 31) // 32 * 32
    full = cs.densify_device(g, lda)
    for rank in range(world):
        part = cs.densify_device(g, lda, rank=rank, world=world, nb=128)
        assert torch.equal(part, qd.scatter_block_cyclic(full, g.n_pixels, 128, rank, world))
