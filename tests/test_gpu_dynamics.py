"""Device parity of the MaskGIT dynamics training step against the oracle (same weights/inputs).

Tolerances: fidelity_threshold.json["parity"].
"""
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import model as OM
from oracle import rng as OR

pytestmark = pytest.mark.gpu
TOL = json.loads((Path(__file__).resolve().parent.parent / "fidelity_threshold.json").read_text())["parity"]


def _rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def _cos(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    na, nb = np.linalg.norm(a), np.linalg.norm(b)
    if na == 0 and nb == 0:
        return 1.0
    return float(a @ b / max(na * nb, 1e-30))


@pytest.fixture(scope="module")
def jasmine_case():
    from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
    B, T, N = 2, 16, 256
    blocks = 2
    cfg = DynamicsConfig(model_dim=512, heads=8, ffn_dim=2048, blocks=blocks, token_codes=1024,
                         action_latent_dim=32, patches_per_frame=N, max_frames=16)
    model = DynamicsModel(cfg, seed=0)
    tokens = OR.stream(1, "bench-tokens").integers(0, 1024, size=(B, T, N))
    lam_cb = OR.stream(2, "golden-lam-cb").uniform(-1 / 6, 1 / 6, size=(6, 32)).astype(np.float32)
    acts = OR.stream(2, "bench-actions").integers(0, 6, size=(B, T - 1))
    lat = lam_cb[acts]
    ocfg = OM.DynCfg(model_dim=512, heads=8, ffn_dim=2048, blocks=blocks, token_codes=1024, action_latent_dim=32,
                     patches_per_frame=N, max_frames=16)
    P = OM.params_to_torch(OM.init_dynamics(ocfg, seed=0))
    mask = OR.sample_masks(OR.PhiloxState.fresh(OR.fold_key(0, "dynamics", "step", 0)), B, T, N)
    torch.set_num_threads(8)
    loss_ref, _ = OM.dyn_loss(P, ocfg, tokens, torch.tensor(lat), mask)
    loss_ref.backward()
    with torch.no_grad():
        logits_ref = OM.dyn_logits(P, ocfg, tokens, torch.tensor(lat), mask).numpy()
    return dict(model=model, tokens=tokens, lat=lat, mask=mask, P=P, loss_ref=float(loss_ref),
                logits_ref=logits_ref, B=B, T=T, N=N)


def test_weights_identical_to_oracle(jasmine_case):
    c = jasmine_case
    for k, p in c["model"].params.items():
        np.testing.assert_array_equal(p.data.cpu().numpy(), c["P"][k].detach().numpy(), err_msg=k)


def test_device_masks_bit_exact():
    from paper_2510_27002_b200 import rng as R
    from paper_2510_27002_b200.dynamics import sample_masks_device
    for (B, T, N, key) in [(2, 16, 256, (0, "dynamics", "step", 0)), (36, 16, 256, (0, "dynamics", "step", 7)),
                           (5, 3, 17, ("x", 3))]:
        g = R.stream(*key)
        m, cnt = sample_masks_device(g, B, T, N)
        ref_g = R.stream(*key)
        ref = OR.sample_masks(OR.PhiloxState.of(ref_g), B, T, N)
        np.testing.assert_array_equal(m.cpu().numpy().astype(bool), ref)
        assert int(cnt) == int(ref.sum())
        # the host generator was advanced exactly past the mask draws
        ref_g.random(B + B * T * N)
        assert g.random() == ref_g.random()


def test_device_mask_sharding_skip_ahead():
    from paper_2510_27002_b200 import rng as R
    from paper_2510_27002_b200.dynamics import sample_masks_device
    full, _ = sample_masks_device(R.stream(0, "dynamics", "step", 3), 288, 16, 256)
    for b0, bl in [(0, 36), (36, 36), (252, 36), (144, 144)]:
        part, _ = sample_masks_device(R.stream(0, "dynamics", "step", 3), 288, 16, 256, shard=(b0, bl))
        assert torch.equal(part, full[b0:b0 + bl])


def test_logits_match_oracle(jasmine_case):
    c = jasmine_case
    from paper_2510_27002_b200.tensor import Tensor
    got = c["model"].logits(c["tokens"], Tensor(c["lat"]), mask=c["mask"]).numpy()
    assert _rel(got, c["logits_ref"]) < TOL["bf16_logits_rel_l2"]


def test_loss_and_grads_match_oracle(jasmine_case):
    c = jasmine_case
    from paper_2510_27002_b200.tensor import Tensor
    model = c["model"]
    loss, stats = model.loss(c["tokens"], Tensor(c["lat"]), None, mask=c["mask"])
    assert abs(float(loss.data) - c["loss_ref"]) < TOL["bf16_loss_abs"]
    assert stats["empty_mask"] == 0
    assert stats["masked_fraction"] == pytest.approx(float(np.mean(c["mask"])))
    loss.backward()
    bad = []
    for k, p in model.params.items():
        ref = c["P"][k].grad.numpy()
        got = p.grad.cpu().numpy()
        if k.endswith(".k.b"):
            # softmax is shift-invariant per query row, so dL/d(key bias) is exactly 0;
            # both sides only carry rounding noise -> bound it against the value-bias gradient
            scale = np.linalg.norm(c["P"][k[:-3] + "v.b"].grad.numpy())
            if np.linalg.norm(got) > 1e-2 * scale:
                bad.append((k, "nonzero", np.linalg.norm(got), scale))
            continue
        cs = _cos(got, ref)
        if cs < TOL["bf16_grad_cosine_min"] or _rel(got, ref) > TOL["bf16_grad_rel_l2"]:
            bad.append((k, cs, _rel(got, ref)))
    assert not bad, bad


def test_loss_draws_masks_from_rng(jasmine_case):
    """loss(rng=stream(seed,'dynamics','step',k)) uses the device Philox masks = oracle masks."""
    c = jasmine_case
    from paper_2510_27002_b200 import rng as R
    from paper_2510_27002_b200.tensor import Tensor
    loss, _ = c["model"].loss(c["tokens"], Tensor(c["lat"]), R.stream(0, "dynamics", "step", 0))
    assert abs(float(loss.data) - c["loss_ref"]) < TOL["bf16_loss_abs"]


def test_empty_mask_is_zero(jasmine_case):
    c = jasmine_case
    from paper_2510_27002_b200.tensor import Tensor
    mask = np.zeros_like(c["mask"])
    loss, stats = c["model"].loss(c["tokens"], Tensor(c["lat"]), None, mask=mask)
    assert float(loss.data) == 0.0 and stats["empty_mask"] == 1


def test_uniform_logits_loss_is_log_k(jasmine_case):
    c = jasmine_case
    from paper_2510_27002_b200.tensor import Tensor
    m = c["model"]
    saved = {k: m.params[k].data.clone() for k in ("to_logits.w", "to_logits.b")}
    try:
        for k in saved:
            m.params[k].data.zero_()
        loss, _ = m.loss(c["tokens"], Tensor(c["lat"]), None, mask=c["mask"])
        assert float(loss.data) == pytest.approx(np.log(1024), abs=1e-5)
    finally:
        for k, v in saved.items():
            m.params[k].data.copy_(v)


def test_token_id_out_of_range_raises(jasmine_case):
    c = jasmine_case
    from paper_2510_27002_b200.tensor import Tensor
    bad = c["tokens"].copy()
    bad[0, 0, 0] = 1024
    with pytest.raises(IndexError):
        c["model"].loss(bad, Tensor(c["lat"]), None, mask=c["mask"])
    with pytest.raises(ValueError):
        c["model"].loss(c["tokens"], Tensor(c["lat"][:, :-1]), None, mask=c["mask"])


@pytest.mark.parametrize("fused_bwd", [True, False])
def test_grads_with_and_without_layernorm_fusion(jasmine_case, fused_bwd):
    """The LayerNorm-fused GEMM epilogues (forward: attention output projections; backward: every
    LayerNorm-fed dX GEMM when enabled) keep every gradient within the stated tolerance; the
    standalone-kernel path (JZ_LN_FUSION=0) too."""
    from paper_2510_27002_b200 import kernels as Kn
    from paper_2510_27002_b200.tensor import Tensor
    c = jasmine_case
    saved = (Kn.LN_FUSION, Kn.LN_FUSION_BWD)
    Kn.LN_FUSION, Kn.LN_FUSION_BWD = fused_bwd, fused_bwd
    try:
        loss, _ = c["model"].loss(c["tokens"], Tensor(c["lat"]), None, mask=c["mask"])
        assert abs(float(loss.data) - c["loss_ref"]) < TOL["bf16_loss_abs"]
        loss.backward()
        bad = []
        for k, p in c["model"].params.items():
            if k.endswith(".k.b"):
                continue
            ref = c["P"][k].grad.numpy()
            got = p.grad.cpu().numpy()
            if _cos(got, ref) < TOL["bf16_grad_cosine_min"] or _rel(got, ref) > TOL["bf16_grad_rel_l2"]:
                bad.append((k, _cos(got, ref), _rel(got, ref)))
        assert not bad, bad
    finally:
        Kn.LN_FUSION, Kn.LN_FUSION_BWD = saved
