"""Device parity of the VQ kernel, tokenizer and latent action model against the oracle."""
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
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _cos(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    na, nb = np.linalg.norm(a), np.linalg.norm(b)
    return 1.0 if na == 0 and nb == 0 else float(a @ b / max(na * nb, 1e-30))


def _near_tie_ok(z, cb, got, ref):
    """Index mismatches allowed only where the fp64 distance gap is within the stated epsilon."""
    z = np.asarray(z, dtype=np.float64)
    cb = np.asarray(cb, dtype=np.float64)
    bad = np.nonzero(np.asarray(got) != np.asarray(ref))[0]
    for r in bad:
        d = ((z[r] - cb) ** 2).sum(-1)
        scale = (z[r] ** 2).sum() + (cb ** 2).sum(-1).max()
        if abs(d[got[r]] - d[ref[r]]) > TOL["vq_index_mismatch_rel_gap"] * scale:
            return False
    return True


class TestVqKernel:
    def test_matches_reference_golden(self, golden):
        from paper_2510_27002_b200 import kernels as K
        g = golden("vq_golden")
        z = torch.tensor(g["f32.z"]).cuda()
        cb = torch.tensor(g["f32.cb"]).cuda()
        idx, zq, sq = K.vq_fwd(z, cb)
        idx = idx.cpu().numpy()
        assert _near_tie_ok(g["f32.z"], g["f32.cb"], idx, g["f32.idx"])
        np.testing.assert_array_equal(idx, g["f32.idx"])
        np.testing.assert_allclose(zq.cpu().numpy(), g["f32.zq"], rtol=0, atol=1e-6)
        loss = float(K.sum_scaled(sq, 1.0 / z.numel()))
        np.testing.assert_allclose(loss, g["f32.cbl"], rtol=1e-5)
        # backward of cbl + 0.25*commit + sum(z_q_st^2)
        n = z.numel()
        dz = torch.empty_like(z)
        dcb = torch.empty_like(cb)
        K.vq_bwd(z, cb, torch.tensor(idx).cuda(), 2.0 * zq, commit_coef=0.25 * 2.0 / n, cb_coef=2.0 / n,
                 dz_out=dz, dcodebook=dcb)
        np.testing.assert_allclose(dz.cpu().numpy(), g["f32.gz"], rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(dcb.cpu().numpy(), g["f32.gcb"], rtol=1e-4, atol=1e-7)

    def test_k6_and_exact_hit(self, golden):
        from paper_2510_27002_b200 import kernels as K
        g = golden("vq_golden")
        idx, _, _ = K.vq_fwd(torch.tensor(g["k6.z"]).cuda(), torch.tensor(g["k6.cb"]).cuda())
        np.testing.assert_array_equal(idx.cpu().numpy(), g["k6.idx"])
        cb = torch.randn(1024, 32).cuda()
        z = cb[[5, 1000, 0]].clone()
        idx, zq, sq = K.vq_fwd(z, cb)
        assert idx.tolist() == [5, 1000, 0] and float(sq.abs().max()) == 0.0

    def test_random_1000_vs_bruteforce(self):
        """test_acceptance.py:214-229 at K=1024, dz=32 on identical fp32 inputs."""
        from paper_2510_27002_b200 import kernels as K
        rs = np.random.default_rng(0)
        z = (rs.normal(size=(1000, 32)) * 0.3).astype(np.float32)
        cb = (rs.normal(size=(1024, 32)) * 0.3).astype(np.float32)
        idx, _, _ = K.vq_fwd(torch.tensor(z).cuda(), torch.tensor(cb).cuda())
        ref = np.argmin(((z[:, None, :].astype(np.float64) - cb[None]) ** 2).sum(-1), axis=1)
        assert _near_tie_ok(z, cb, idx.cpu().numpy(), ref)


    @pytest.mark.parametrize("rows", [80000, 140000])
    def test_multi_row_kernel_bit_identical(self, rows):
        """Above 148 x 512 rows jz_vq_fwd runs two rows per thread, above ~148 x 896 four; both must
        equal the one-row kernel (used for fewer rows) bit for bit: indices, z_q and squared errors."""
        from paper_2510_27002_b200 import kernels as K
        g = torch.Generator(device="cuda").manual_seed(11)
        cb = torch.randn(1024, 32, device="cuda", generator=g) * 0.3
        z = torch.randn(rows, 32, device="cuda", generator=g) * 0.3
        for h, c in enumerate((513, 2, 1023, 0)):  # exact hits in every row slot of a thread
            z[7 + 256 * h] = cb[c]
        big = K.vq_fwd(z, cb)
        parts = [K.vq_fwd(z[a:a + 40000].contiguous(), cb) for a in range(0, rows, 40000)]
        for k in range(3):
            got, ref = big[k], torch.cat([p[k] for p in parts])
            assert torch.equal(got, ref), k
        assert [big[0][7 + 256 * h].item() for h in range(4)] == [513, 2, 1023, 0]


TOKKW = dict(model_dim=128, heads=2, ffn_dim=512, blocks=1, codes=64, latent_dim=32, patch=4, height=64, width=64,
             max_frames=4)


@pytest.fixture(scope="module")
def frames():
    return OR.stream(31, "video-frames").integers(0, 256, size=(2, 3, 64, 64, 3)).astype(np.uint8)


class TestTokenizer:
    def test_weights_and_encode(self, frames):
        from paper_2510_27002_b200.tokenizer import TokenizerConfig, VideoTokenizer
        tok = VideoTokenizer(TokenizerConfig(**TOKKW), seed=3)
        ocfg = OM.TokCfg(**TOKKW)
        P = OM.params_to_torch(OM.init_tokenizer(ocfg, seed=3), requires_grad=False)
        for k, p in tok.params.items():
            np.testing.assert_array_equal(p.data.cpu().numpy(), P[k].numpy(), err_msg=k)
        z = tok.encode_latent(frames).numpy()
        with torch.no_grad():
            zr = OM.tok_encode_latent(P, ocfg, torch.tensor(OM.frames_to_unit(frames))).numpy()
        assert _rel(z, zr) < TOL["bf16_logits_rel_l2"]
        idx = tok.encode(frames)
        ref = OM.tok_encode(P, ocfg, frames)
        # encoder runs in bf16: indices may legitimately flip where codes are nearly equidistant
        assert (idx == ref).mean() >= TOL["vq_index_agreement_small_encoder"]

    def test_decode_and_forward(self, frames):
        from paper_2510_27002_b200.tokenizer import TokenizerConfig, VideoTokenizer
        tok = VideoTokenizer(TokenizerConfig(**TOKKW), seed=3)
        ocfg = OM.TokCfg(**TOKKW)
        P = OM.params_to_torch(OM.init_tokenizer(ocfg, seed=3), requires_grad=False)
        tokens = OR.stream(32, "tok").integers(0, 64, size=(2, 3, 256))
        got = tok.decode(tokens)
        ref = OM.tok_decode(P, ocfg, tokens)
        assert _rel(got, ref) < TOL["bf16_logits_rel_l2"]
        with pytest.raises(IndexError):
            tok.decode(tokens + 64)
        unit = OM.frames_to_unit(frames)
        recon, idx, losses = tok.forward(unit)
        with torch.no_grad():
            r2, i2, l2 = OM.tok_forward(P, ocfg, torch.tensor(unit))
        for k in ("recon", "codebook", "commitment", "total"):
            assert abs(float(losses[k].data) - float(l2[k])) < max(TOL["bf16_loss_abs"], TOL["bf16_loss_rel"] * float(l2[k])), k

    def test_forward_backward_vs_oracle(self, frames):
        """Tokenizer training step (trainer.py:211-223): losses and every parameter gradient."""
        from paper_2510_27002_b200.tokenizer import TokenizerConfig, VideoTokenizer
        tok = VideoTokenizer(TokenizerConfig(**TOKKW), seed=3)
        ocfg = OM.TokCfg(**TOKKW)
        P = OM.params_to_torch(OM.init_tokenizer(ocfg, seed=3))
        unit = OM.frames_to_unit(frames)
        recon, idx, losses = tok.forward(unit)
        _, i2, _ = OM.tok_forward(P, ocfg, torch.tensor(unit))
        assert (idx == np.asarray(i2)).mean() >= TOL["vq_index_agreement_bf16_encoder"]  # bf16 encoder: only near-tie codes may flip
        # oracle step on OUR code indices (a flipped code moves a whole patch): tokenizer.py:58-79, 134-143
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
        bad = []
        for k, p in tok.params.items():
            ref = P[k].grad.numpy()
            got = p.grad.cpu().numpy()
            if k.endswith(".k.b") or np.linalg.norm(ref) < 1e-9:
                continue  # .k.b: exactly zero in exact arithmetic (softmax shift invariance)
            if _cos(got, ref) < TOL["bf16_grad_cosine_min_vq_models"]:
                bad.append((k, _cos(got, ref), _rel(got, ref)))
        assert not bad, bad

    def test_geometry_errors(self):
        from paper_2510_27002_b200.tokenizer import TokenizerConfig, VideoTokenizer
        tok = VideoTokenizer(TokenizerConfig(**TOKKW), seed=3)
        with pytest.raises(ValueError):
            tok.encode(np.zeros((1, 2, 32, 32, 3), dtype=np.uint8))
        with pytest.raises(ValueError):
            tok.encode(np.zeros((1, 5, 64, 64, 3), dtype=np.uint8))


LAMKW = dict(TOKKW, codes=6)


class TestLam:
    def test_forward_backward_vs_oracle(self, frames):
        from paper_2510_27002_b200.lam import LamConfig, LatentActionModel
        lam = LatentActionModel(LamConfig(**LAMKW), seed=5)
        ocfg = OM.LamCfg(**LAMKW)
        P = OM.params_to_torch(OM.init_lam(ocfg, seed=5))
        unit = OM.frames_to_unit(frames)
        recon, idx, losses = lam.forward(unit)
        r2, i2, l2 = OM.lam_forward(P, ocfg, torch.tensor(unit))
        np.testing.assert_array_equal(idx, i2)
        assert _rel(recon.numpy(), r2.detach().numpy()) < TOL["bf16_logits_rel_l2"]
        for k in ("recon", "codebook", "commitment", "total"):
            assert abs(float(losses[k].data) - float(l2[k])) < max(TOL["bf16_loss_abs"], TOL["bf16_loss_rel"] * float(l2[k])), k
        losses["total"].backward()
        l2["total"].backward()
        bad = []
        for k, p in lam.params.items():
            ref = P[k].grad.numpy()
            got = p.grad.cpu().numpy()
            if k.endswith(".k.b"):
                continue  # exactly zero in exact arithmetic (softmax shift invariance)
            if np.linalg.norm(ref) < 1e-9:
                continue
            if _cos(got, ref) < TOL["bf16_grad_cosine_min_vq_models"]:
                bad.append((k, _cos(got, ref), _rel(got, ref)))
        assert not bad, bad

    def test_infer_actions_and_latents(self, frames):
        from paper_2510_27002_b200.lam import LamConfig, LatentActionModel
        lam = LatentActionModel(LamConfig(**LAMKW), seed=5)
        ocfg = OM.LamCfg(**LAMKW)
        P = OM.params_to_torch(OM.init_lam(ocfg, seed=5), requires_grad=False)
        idx = lam.infer_actions(frames)
        with torch.no_grad():
            ref, _, _, _ = OM.lam_encoder_only(P, ocfg, torch.tensor(OM.frames_to_unit(frames)))
        np.testing.assert_array_equal(idx, ref)
        assert idx.shape == (2, 2) and idx.max() < 6
        lat = lam.action_latents(idx)
        np.testing.assert_array_equal(lat.numpy(), P["codebook"].numpy()[idx])
        with pytest.raises(ValueError):
            lam.infer_actions(frames[:, :1])


class TestCotrain:
    def test_cotrain_loss_and_grads_vs_oracle(self, frames):
        """trainer.py:306-309 cotrain: ce(dynamics | z_q_st of the LAM encoder) + cb + beta * commit.

        Gradients reach the dynamics model, and through the straight-through estimator, the LAM
        encoder (to_latent, stack, embeddings) and codebook; the LAM decoder takes no gradient."""
        from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
        from paper_2510_27002_b200.lam import LamConfig, LatentActionModel
        lam = LatentActionModel(LamConfig(**LAMKW), seed=5)
        dkw = dict(model_dim=128, heads=2, ffn_dim=512, blocks=1, token_codes=256, action_latent_dim=32,
                   patches_per_frame=256, max_frames=4)
        dyn = DynamicsModel(DynamicsConfig(**dkw), seed=9)
        Pl = OM.params_to_torch(OM.init_lam(OM.LamCfg(**LAMKW), seed=5))
        Pd = OM.params_to_torch(OM.init_dynamics(OM.DynCfg(**dkw), seed=9))
        unit = OM.frames_to_unit(frames)
        B, T = unit.shape[0], unit.shape[1]
        tokens = OR.stream(41, "cotrain-tokens").integers(0, 256, size=(B, T, 256))
        mask = OR.sample_masks(OR.PhiloxState.fresh(OR.fold_key(3, "cotrain")), B, T, 256)
        beta = lam.cfg.commitment_beta
        idx, zq, cb, commit = lam.encoder_only(unit)
        ce, _ = dyn.loss(tokens, zq, None, mask=mask)
        total = ce + cb + beta * commit
        i2, zq2, cb2, commit2 = OM.lam_encoder_only(Pl, OM.LamCfg(**LAMKW), torch.tensor(unit))
        ce2, _ = OM.dyn_loss(Pd, OM.DynCfg(**dkw), tokens, zq2, mask)
        total2 = ce2 + cb2 + beta * commit2
        np.testing.assert_array_equal(idx, np.asarray(i2))
        assert abs(float(total.data) - float(total2)) < max(TOL["bf16_loss_abs"], TOL["bf16_loss_rel"] * float(total2))
        total.backward()
        total2.backward()
        bad = []
        for model, P in ((dyn, Pd), (lam, Pl)):
            for k, p in model.params.items():
                got = p.grad.cpu().numpy() if p.grad is not None else np.zeros(p.shape)
                ref = P[k].grad.numpy() if P[k].grad is not None else np.zeros(p.shape)
                if k.endswith(".k.b") or np.linalg.norm(ref) < 1e-9:
                    if k.startswith("dec") and model is lam:
                        assert np.linalg.norm(got) == 0, k  # decoder is not in the cotrain graph
                    continue
                if _cos(got, ref) < TOL["bf16_grad_cosine_min_cotrain"]:
                    bad.append((k, _cos(got, ref), _rel(got, ref)))
        assert not bad, bad
        with pytest.raises(NotImplementedError):
            (2.0 * dyn.loss(tokens, zq.detach(), None, mask=mask)[0]).backward()
