"""Device checkpoint / resume and the device data path."""
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
DKW = dict(model_dim=128, heads=2, ffn_dim=512, blocks=2, token_codes=256, action_latent_dim=32,
           patches_per_frame=256, max_frames=4)


def _inputs():
    from oracle import rng as OR
    from paper_2510_27002_b200.tensor import Tensor
    tokens = torch.as_tensor(OR.stream(3, "ck-tok").integers(0, 256, size=(2, 4, 256))).cuda()
    lat = Tensor(torch.as_tensor(OR.stream(3, "ck-lat").normal(size=(2, 3, 32)).astype(np.float32)).cuda() * 0.3)
    return tokens, lat


def _trainer(seed=0):
    from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
    from paper_2510_27002_b200.optim import WsdSchedule
    from paper_2510_27002_b200.trainer import DynamicsTrainStep
    m = DynamicsModel(DynamicsConfig(**DKW), seed=seed)
    return DynamicsTrainStep(m, WsdSchedule(peak_lr=1e-3, total_steps=100, warmup_steps=2), seed=7)


def test_resume_is_bitwise_identical(tmp_path):
    """3 uninterrupted steps == 1 step, save, restore into a fresh model, 2 more steps (bitwise)."""
    from paper_2510_27002_b200.checkpoint import load_checkpoint, save_checkpoint
    tokens, lat = _inputs()
    a = _trainer()
    for k in range(3):
        a.step(k, tokens, lat)
    b = _trainer()
    b.step(0, tokens, lat)
    save_checkpoint(b.pack(1, config={"test": True}), tmp_path / "s1.jasckpt")
    c = _trainer(seed=123)  # different init: everything must come from the checkpoint
    ls, step = c.restore(load_checkpoint(tmp_path / "s1.jasckpt"))
    assert step == 1 and c.opt.t == 1 and ls["seed"] == 7
    for k in range(step, 3):
        c.step(k, tokens, lat)
    torch.cuda.synchronize()
    assert torch.equal(a.model._store.flat, c.model._store.flat)
    assert torch.equal(a.opt.m_flat, c.opt.m_flat) and torch.equal(a.opt.v_flat, c.opt.v_flat)


def test_pack_matches_live_views():
    """Grouped (strided) q/k/v views are packed as the reference's contiguous per-name arrays."""
    t = _trainer()
    b = t.pack(0)
    for name, p in t.model.params.items():
        np.testing.assert_array_equal(b.arrays[f"param.{name}"], p.data.cpu().numpy(), err_msg=name)
        assert b.arrays[f"param.{name}"].flags["C_CONTIGUOUS"]
    assert b.meta["stage"] == "dynamics" and b.meta["adam"]["t"] == 0


def test_device_loader_matches_host_batches():
    from paper_2510_27002_b200.records import DatasetIndex, DeviceBatchLoader, LoaderState, shuffled_batches
    index = DatasetIndex.load(GOLD / "jasrec_ref")
    host = shuffled_batches(index, LoaderState(seed=11), batch_size=3, seq_len=5)
    dev = DeviceBatchLoader(index, LoaderState(seed=11), batch_size=3, seq_len=5, depth=2)
    try:
        for _ in range(9):  # more batches than slots: ring reuse + epoch rollover
            hf, ha, hs = next(host)
            df, da, ds = next(dev)
            assert df.is_cuda and df.dtype == torch.uint8
            np.testing.assert_array_equal(df.cpu().numpy(), hf)
            np.testing.assert_array_equal(da.cpu().numpy(), ha)
            assert ds == hs
    finally:
        dev.close()
