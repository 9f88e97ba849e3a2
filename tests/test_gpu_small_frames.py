"""Device parity at the reference's patch-16 geometry (64x64 frames -> 16 patches per frame).

The reference's own defaults (`TokenizerConfig.patch = 16`, `LamConfig.patch = 16`,
`DynamicsConfig.patches_per_frame = 16`; tokenizer.py:21-46, lam.py:22-47, dynamics.py:33-49)
put S = 16 (tokenizer, LAM encoder) and S = 17 (LAM decoder and dynamics, the prepended action
token) into spatial attention; those run on the register-tile kernel (K3s), not the S = 256/257
tcgen05 kernel. Full-width blocks (model_dim 512, 8 heads) as the jasmine-base stacks.
Tolerances: fidelity_threshold.json["parity"], as the S = 256/257 tests.
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
WIDE = dict(model_dim=512, heads=8, ffn_dim=2048, blocks=2)


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


def _grad_mismatches(params, P, cos_min, rel_max=None):
    bad = []
    for k, p in params.items():
        ref = P[k].grad.numpy()
        got = p.grad.cpu().numpy()
        if k.endswith(".k.b") or np.linalg.norm(ref) < 1e-9:
            continue  # .k.b: exactly zero in exact arithmetic (softmax shift invariance)
        cs = _cos(got, ref)
        if cs < cos_min or (rel_max is not None and _rel(got, ref) > rel_max):
            bad.append((k, cs, _rel(got, ref)))
    return bad


@pytest.fixture(scope="module")
def frames():
    return OR.stream(41, "patch16-frames").integers(0, 256, size=(3, 16, 64, 64, 3)).astype(np.uint8)


def test_dynamics_patch16_loss_and_grads():
    """S = 17 spatial attention, T = 16 causal temporal attention, full MaskGIT loss + backward."""
    from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
    from paper_2510_27002_b200.tensor import Tensor
    B, T, N = 4, 16, 16
    kw = dict(WIDE, token_codes=1024, action_latent_dim=32, patches_per_frame=N, max_frames=16)
    model = DynamicsModel(DynamicsConfig(**kw), seed=0)
    ocfg = OM.DynCfg(**kw)
    P = OM.params_to_torch(OM.init_dynamics(ocfg, seed=0))
    tokens = OR.stream(1, "p16-tokens").integers(0, 1024, size=(B, T, N))
    lat = (OR.stream(2, "p16-lat").normal(size=(B, T - 1, 32)) * 0.1).astype(np.float32)
    mask = OR.sample_masks(OR.PhiloxState.fresh(OR.fold_key(0, "dynamics", "step", 0)), B, T, N)
    loss_ref, _ = OM.dyn_loss(P, ocfg, tokens, torch.tensor(lat), mask)
    loss_ref.backward()
    with torch.no_grad():
        logits_ref = OM.dyn_logits(P, ocfg, tokens, torch.tensor(lat), mask).numpy()
    got = model.logits(tokens, Tensor(lat), mask=mask).numpy()
    assert _rel(got, logits_ref) < TOL["bf16_logits_rel_l2"]
    loss, stats = model.loss(tokens, Tensor(lat), None, mask=mask)
    assert abs(float(loss.data) - float(loss_ref)) < TOL["bf16_loss_abs"]
    loss.backward()
    bad = _grad_mismatches(model.params, P, TOL["bf16_grad_cosine_min"], TOL["bf16_grad_rel_l2"])
    assert not bad, bad


def test_tokenizer_patch16_forward_backward(frames):
    """S = 16 encoder/decoder stacks; losses and every parameter gradient on the same code indices."""
    from paper_2510_27002_b200.tokenizer import TokenizerConfig, VideoTokenizer
    kw = dict(WIDE, codes=1024, latent_dim=32, patch=16, height=64, width=64, max_frames=16)
    tok = VideoTokenizer(TokenizerConfig(**kw), seed=3)
    ocfg = OM.TokCfg(**kw)
    P = OM.params_to_torch(OM.init_tokenizer(ocfg, seed=3))
    unit = OM.frames_to_unit(frames)
    recon, idx, losses = tok.forward(unit)
    _, i2, _ = OM.tok_forward(P, ocfg, torch.tensor(unit))
    assert (idx == np.asarray(i2)).mean() >= TOL["vq_index_agreement_bf16_encoder"]  # bf16 encoder: only near-tie codes may flip
    u = torch.tensor(unit)
    z_e = OM.tok_encode_latent(P, ocfg, u)
    z_q = P["codebook"][torch.as_tensor(idx)]
    cb, commit = OM.mse(z_q, z_e.detach()), OM.mse(z_e, z_q.detach())
    r2 = OM.tok_decode_latent(P, ocfg, z_e + (z_q - z_e).detach())
    rec = OM.mse(r2, u)
    l2 = {"recon": rec, "codebook": cb, "commitment": commit, "total": rec + cb + ocfg.commitment_beta * commit}
    assert _rel(recon.numpy(), r2.detach().numpy()) < TOL["bf16_logits_rel_l2"]
    for k in ("recon", "codebook", "commitment", "total"):
        assert abs(float(losses[k].data) - float(l2[k])) < max(TOL["bf16_loss_abs"], TOL["bf16_loss_rel"] * float(l2[k])), k
    losses["total"].backward()
    l2["total"].backward()
    bad = _grad_mismatches(tok.params, P, TOL["bf16_grad_cosine_min_vq_models"])
    assert not bad, bad


def test_lam_patch16_forward_backward(frames):
    """S = 16 encoder, S = 17 decoder (action token prepended), K = 6 codebook."""
    from paper_2510_27002_b200.lam import LamConfig, LatentActionModel
    kw = dict(WIDE, codes=6, latent_dim=32, patch=16, height=64, width=64, max_frames=16)
    lam = LatentActionModel(LamConfig(**kw), seed=5)
    ocfg = OM.LamCfg(**kw)
    P = OM.params_to_torch(OM.init_lam(ocfg, seed=5))
    unit = OM.frames_to_unit(frames)
    recon, idx, losses = lam.forward(unit)
    _, i2, _ = OM.lam_forward(P, ocfg, torch.tensor(unit))
    # bf16 encoder: a code may flip only where the latent error explains it (6-code near-ties);
    # the oracle step then runs on the device's codes (a flipped code moves a whole action)
    with torch.no_grad():
        z_ref = OM.lam_encode_pre_vq(P, ocfg, torch.tensor(unit)).numpy()
    z_dev = lam._encode_pre_vq(unit).numpy()
    assert OM.vq_mismatch_explained(z_dev, z_ref, P["codebook"].detach().numpy(), idx, i2) == 0
    assert (np.asarray(idx) == np.asarray(i2)).mean() >= TOL["lam_code_agreement_bf16_encoder"]
    r2, _, l2 = OM.lam_forward_with_indices(P, ocfg, torch.tensor(unit), idx)
    assert _rel(recon.numpy(), r2.detach().numpy()) < TOL["bf16_logits_rel_l2"]
    for k in ("recon", "codebook", "commitment", "total"):
        assert abs(float(losses[k].data) - float(l2[k])) < max(TOL["bf16_loss_abs"], TOL["bf16_loss_rel"] * float(l2[k])), k
    losses["total"].backward()
    l2["total"].backward()
    bad = _grad_mismatches(lam.params, P, TOL["bf16_grad_cosine_min_vq_models"])
    assert not bad, bad


def test_envelope_errors():
    from paper_2510_27002_b200.st import StConfig, check_supported
    check_supported(StConfig(512, 8, 2048, 1), 18, 32)
    with pytest.raises(ValueError):
        check_supported(StConfig(512, 8, 2048, 1), 33, 16)
    check_supported(StConfig(1024, 16, 4096, 1), 17, 16)
    with pytest.raises(ValueError):
        check_supported(StConfig(512, 8, 2048, 1), 257, 33)
