"""Data-parallel algebra of the dynamics step on one GPU, without collectives.

The gradient of the global batch equals the SUM of the per-rank gradients. Each rank trains its
batch shard, draws its own mask shard by Philox skip-ahead, and normalises its masked CE by the
GLOBAL mask count, which every rank recomputes from the full global mask (dp.py).

Here the two "ranks" run one after the other on the same device, with no inter-rank dependency
and no NCCL. Their gradients are summed on the host side of the test and compared with a single
process on the global batch: losses add up exactly, and gradients agree to fp32 summation-order
rounding. The NCCL all-reduce itself is covered by the gloo two-rank test (test_host.py).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

B_GLOBAL, WORLD, T, N, K = 4, 2, 16, 256, 1024


def _setup():
    from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
    from paper_2510_27002_b200.rng import stream
    from paper_2510_27002_b200.tensor import Tensor
    cfg = DynamicsConfig(model_dim=512, heads=8, ffn_dim=2048, blocks=2, token_codes=K, action_latent_dim=32,
                         patches_per_frame=N, max_frames=T)
    model = DynamicsModel(cfg, seed=0)
    tokens = torch.as_tensor(stream(1, "dp-tokens").integers(0, K, size=(B_GLOBAL, T, N)), device="cuda")
    cb = stream(2, "dp-cb").uniform(-1 / 6, 1 / 6, size=(6, 32)).astype(np.float32)
    lat = torch.as_tensor(cb[stream(2, "dp-acts").integers(0, 6, size=(B_GLOBAL, T - 1))], device="cuda")
    return model, tokens, lat, Tensor


def _grads(model):
    torch.cuda.synchronize()
    return model._store.grad_flat.clone()


def test_sharded_ranks_sum_to_the_global_step():
    from paper_2510_27002_b200 import kernels as Kn
    from paper_2510_27002_b200.dp import shard
    from paper_2510_27002_b200.rng import consume, stream
    model, tokens, lat, Tensor = _setup()
    cfg = model.cfg
    store = model._store
    store.grads()

    # single process on the global batch (the reference's run_stage step, trainer.py:168-176)
    store.grad_flat.zero_()
    loss_full, _ = model.loss(tokens, Tensor(lat), stream(0, "dynamics", "step", 3))
    loss_full.backward()
    g_full = _grads(model)
    lf = float(loss_full.data)

    # two ranks, one after the other (DynamicsTrainStep.step with world = 2, minus the all-reduce)
    g_sum = torch.zeros_like(g_full)
    l_sum = 0.0
    masks = []
    for rank in range(WORLD):
        rng = stream(0, "dynamics", "step", 3)
        st = consume(rng, B_GLOBAL + B_GLOBAL * T * N)
        b0, bl = shard(B_GLOBAL, rank, WORLD)
        mask = torch.empty(bl, T, N, dtype=torch.uint8, device="cuda")
        cnt_local = torch.zeros((), dtype=torch.int32, device="cuda")
        Kn.philox_mask(st, B_GLOBAL, b0, bl, T, N, cfg.mask_limit, mask, cnt_local)
        full = torch.empty(B_GLOBAL, T, N, dtype=torch.uint8, device="cuda")
        count = torch.zeros((), dtype=torch.int32, device="cuda")
        Kn.philox_mask(st, B_GLOBAL, 0, B_GLOBAL, T, N, cfg.mask_limit, full, count)
        assert torch.equal(full[b0:b0 + bl], mask)  # the shard is the global mask's slice
        masks.append(mask)
        store.grad_flat.zero_()
        loss_r, _ = model.loss(tokens[b0:b0 + bl], Tensor(lat[b0:b0 + bl]), None, mask=mask, _count=count)
        loss_r.backward()
        g_sum += _grads(model)
        l_sum += float(loss_r.data)

    # the union of the shards is the single-process mask (same Philox stream, dynamics.py:52-62)
    from paper_2510_27002_b200.dynamics import sample_masks_device
    m_full, _ = sample_masks_device(stream(0, "dynamics", "step", 3), B_GLOBAL, T, N)
    assert torch.equal(torch.cat(masks, 0).bool(), m_full.bool())
    assert abs(l_sum - lf) <= 1e-5 * abs(lf), (l_sum, lf)
    rel = float((g_sum - g_full).norm() / g_full.norm())
    assert rel < 1e-4, rel
