"""Device ST-DiT (paper_2510_27002_b200.diffusion) against the oracle restatement of diffusion.py,
which tests/test_oracle_golden.py pins to the reference. Full-width blocks (model_dim 512, 8 heads)
at the reference's 16-patch default (S = N + 2 = 18). Tolerances: fidelity_threshold.json["parity"].
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
KW = dict(model_dim=512, heads=8, ffn_dim=2048, blocks=2, latent_dim=32, action_latent_dim=32, action_vocab=7,
          patches_per_frame=16, max_frames=16)


def _rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def _cos(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(a @ b / max(np.linalg.norm(a) * np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def case():
    from paper_2510_27002_b200.diffusion import DitConfig, DitDynamics
    dit = DitDynamics(DitConfig(**KW), seed=4)
    P = OM.params_to_torch(OM.init_dit(OM.DitCfg(**KW), seed=4))
    g = OR.stream(7, "dit-gpu-case")
    B, T, N = 3, 8, 16
    latents = np.tanh(g.normal(size=(B, T, N, 32))).astype(np.float32)
    act = (g.normal(size=(B, T - 1, 32)) * 0.1).astype(np.float32)
    return dict(dit=dit, P=P, latents=latents, act=act, B=B, T=T)


def test_weights_identical_to_oracle(case):
    for k, p in case["dit"].params.items():
        np.testing.assert_array_equal(p.data.cpu().numpy(), case["P"][k].detach().numpy(), err_msg=k)


def test_predict_clean_matches_oracle(case):
    g = OR.stream(8, "dit-tau")
    tau = g.uniform(0, 1, size=(case["B"], case["T"]))
    noised = OM.forcing_corrupt(case["latents"], tau, g)
    got = case["dit"].predict_clean(noised, tau, case["act"]).numpy()
    with torch.no_grad():
        ref = OM.dit_predict_clean(case["P"], OM.DitCfg(**KW), noised, tau, torch.tensor(case["act"])).numpy()
    assert got.shape == ref.shape
    assert _rel(got, ref) < TOL["bf16_logits_rel_l2"]


def test_loss_and_grads_match_oracle(case):
    from paper_2510_27002_b200 import rng as R
    dit, P = case["dit"], case["P"]
    loss = dit.loss(case["latents"], case["act"], R.stream(9, "dit-loss"))
    ref = OM.dit_loss(P, OM.DitCfg(**KW), case["latents"], torch.tensor(case["act"]), OR.stream(9, "dit-loss"))
    assert abs(float(loss.data) - float(ref)) < max(TOL["bf16_loss_abs"], TOL["bf16_loss_rel"] * float(ref))
    loss.backward()
    ref.backward()
    bad = []
    for k, p in dit.params.items():
        r = P[k].grad
        got = p.grad.cpu().numpy()
        if r is None or k.endswith(".k.b"):  # gt_action_embed: no gradient; .k.b: exactly 0 (shift invariance)
            if r is None:
                assert float(np.abs(got).max()) == 0.0, k
            continue
        r = r.numpy()
        if _cos(got, r) < TOL["bf16_grad_cosine_min"]:
            bad.append((k, _cos(got, r), _rel(got, r)))
    assert not bad, bad


def test_sample_frame_matches_oracle(case):
    from paper_2510_27002_b200 import rng as R
    ctx = case["latents"][:, :4]
    act = case["act"][:, :4]
    z = case["dit"].sample_frame(ctx, act, steps=4, rng=R.stream(10, "dit-sample"))
    zr = OM.dit_sample_frame(case["P"], OM.DitCfg(**KW), ctx, torch.tensor(act), steps=4,
                             gen=OR.stream(10, "dit-sample"))
    assert z.shape == (case["B"], 16, 32)
    assert _rel(z, zr) < TOL["bf16_logits_rel_l2"]


def test_errors(case):
    dit = case["dit"]
    with pytest.raises(ValueError):
        dit.predict_clean(case["latents"], np.zeros((case["B"], case["T"])), case["act"][:, :2])
    with pytest.raises(ValueError):
        dit.sample_frame(case["latents"][:, :2], case["act"][:, :2], steps=0)


MAEKW = dict(model_dim=512, heads=8, ffn_dim=2048, blocks=2, latent_dim=32, patch=16, height=64, width=64,
             max_frames=16)


@pytest.fixture(scope="module")
def mae_case():
    from paper_2510_27002_b200.diffusion import MaeConfig, MaeTokenizer
    mae = MaeTokenizer(MaeConfig(**MAEKW), seed=6)
    P = OM.params_to_torch(OM.init_mae(OM.MaeCfg(**MAEKW), seed=6))
    frames = OR.stream(11, "mae-frames").integers(0, 256, size=(3, 6, 64, 64, 3)).astype(np.uint8)
    return dict(mae=mae, P=P, frames=frames, unit=OM.frames_to_unit(frames))


def test_mae_encode_decode_match_oracle(mae_case):
    mae, P, unit = mae_case["mae"], mae_case["P"], mae_case["unit"]
    for k, p in mae.params.items():
        np.testing.assert_array_equal(p.data.cpu().numpy(), P[k].detach().numpy(), err_msg=k)
    cfg = OM.MaeCfg(**MAEKW)
    lat = mae.encode(mae_case["frames"]).numpy()  # uint8 in: unit conversion on device
    with torch.no_grad():
        lat_ref = OM.mae_encode(P, cfg, torch.tensor(unit)).numpy()
        mask = OR.stream(12, "m").random((3, 6, 16)) < 0.5
        lat_m_ref = OM.mae_encode(P, cfg, torch.tensor(unit), mask).numpy()
        rec_ref = OM.mae_decode(P, cfg, torch.tensor(lat_ref)).numpy()
    assert lat.shape == (3, 6, 16, 32)
    assert _rel(lat, lat_ref) < TOL["bf16_logits_rel_l2"]
    assert _rel(mae.encode(unit, mask=mask).numpy(), lat_m_ref) < TOL["bf16_logits_rel_l2"]
    assert _rel(mae.decode(lat_ref).numpy(), rec_ref) < TOL["bf16_logits_rel_l2"]


def test_mae_forward_backward_match_oracle(mae_case):
    from paper_2510_27002_b200 import rng as R
    mae, P = mae_case["mae"], mae_case["P"]
    recon, lat, loss = mae.forward(mae_case["unit"], R.stream(13, "mae-step"))
    r2, l2, loss2 = OM.mae_forward(P, OM.MaeCfg(**MAEKW), torch.tensor(mae_case["unit"]), OR.stream(13, "mae-step"))
    assert _rel(lat.numpy(), l2.detach().numpy()) < TOL["bf16_logits_rel_l2"]
    assert _rel(recon.numpy(), r2.detach().numpy()) < TOL["bf16_logits_rel_l2"]
    assert abs(float(loss.data) - float(loss2)) < max(TOL["bf16_loss_abs"], TOL["bf16_loss_rel"] * float(loss2))
    loss.backward()
    loss2.backward()
    bad = []
    for k, p in mae.params.items():
        if k.endswith(".k.b"):
            continue
        ref, got = P[k].grad.numpy(), p.grad.cpu().numpy()
        if _cos(got, ref) < TOL["bf16_grad_cosine_min_vq_models"]:
            bad.append((k, _cos(got, ref), _rel(got, ref)))
    assert not bad, bad


def test_diffusion_rollout_matches_oracle_composition(case, mae_case):
    """diffusion_rollout (diffusion.py:217-251): MAE encode -> per-frame DiT Euler sampling with
    ground-truth action ids -> clip -> MAE decode, against the same pipeline from oracle pieces."""
    from paper_2510_27002_b200 import rng as R
    from paper_2510_27002_b200.diffusion import diffusion_rollout
    mae, dit = mae_case["mae"], case["dit"]
    cond = mae_case["frames"][:2, :3]
    actions = [np.array([1, 4]), np.array([6, 0])]
    out = diffusion_rollout(mae, dit, cond, actions, horizon=2, steps=3, rng=R.stream(14, "roll"))
    assert out.shape == (2, 5, 64, 64, 3) and out.dtype == np.uint8
    Pm, Pd = mae_case["P"], case["P"]
    g = OR.stream(14, "roll")
    with torch.no_grad():
        lat = OM.mae_encode(Pm, OM.MaeCfg(**MAEKW), torch.tensor(OM.frames_to_unit(cond))).numpy()
        hist = Pd["null_action"].detach().reshape(1, 1, 32) + torch.zeros(2, 2, 32)
        for a in actions:
            hist = torch.cat([hist, Pd["gt_action_embed"].detach()[torch.as_tensor(a)].reshape(2, 1, 32)], 1)
            nxt = OM.dit_sample_frame(Pd, OM.DitCfg(**KW), lat, hist, steps=3, gen=g)
            lat = np.concatenate([lat, nxt[:, None]], axis=1)
        lat = np.clip(lat, -1.0 + 1e-6, 1.0 - 1e-6)
        ref = OM.unit_to_frames(OM.mae_decode(Pm, OM.MaeCfg(**MAEKW), torch.tensor(lat)).numpy())
    diff = np.abs(out.astype(np.int16) - ref.astype(np.int16))
    assert diff[:, :3].mean() < 1.0  # re-decoded conditioning frames
    assert diff.mean() < 2.0         # generated frames: bf16 chains through 2 x 3 model calls
