"""Pin the oracle against golden vectors produced by the UNMODIFIED reference
(tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest
import torch

from oracle import model as M
from oracle import rng as R

torch.set_num_threads(max(1, torch.get_num_threads()))


def _key_parts(s):
    out = []
    for p in s.split("|"):
        try:
            out.append(int(p))
        except ValueError:
            out.append(p)
    return tuple(out)


class TestRng:
    def test_fold_key(self, golden):
        g = golden("rng_golden")
        for s, k in zip(g["key_strs"], g["folded"]):
            assert R.fold_key(*_key_parts(str(s))) == int(k)

    def test_philox_words_and_doubles(self, golden):
        g = golden("rng_golden")
        st = R.PhiloxState.fresh(R.fold_key(0, "dynamics", "step", 0))
        np.testing.assert_array_equal(st.words(64), g["words"])
        np.testing.assert_array_equal(R.words_to_doubles(st.words(64)), g["doubles"])

    def test_known_answer_vector(self):
        # SURVEY Appendix B
        st = R.PhiloxState.fresh(0xB44FA4F924E95B03)
        w = st.words(4)
        assert [int(x) for x in w] == [0x01E3F82C9EDD0D2A, 0xB6B2EB63775E7B15,
                                       0x00AAC7024F0DB0CA, 0x8E67613C237BA85C]
        d = R.words_to_doubles(w[:3])
        assert d.tolist() == [0.007384787458125541, 0.7136675947034464, 0.0026058560024952993]

    def test_masks_bit_exact(self, golden):
        g = golden("rng_golden")
        m, p = R.sample_masks(R.PhiloxState.fresh(R.fold_key(1, "m")), 3, 4, 16, return_p=True)
        np.testing.assert_array_equal(m, g["m_small"])
        np.testing.assert_array_equal(p, g["p_small"])
        st = R.PhiloxState.fresh(R.fold_key(0, "dynamics", "step", 5))
        m, p = R.sample_masks(st, 2, 16, 256, return_p=True)
        np.testing.assert_array_equal(m, g["m_full"])
        np.testing.assert_array_equal(p, g["p_full"])
        after = st.advanced(2 + 2 * 16 * 256)
        assert after.counter + [after.buffer_pos] == [int(x) for x in g["after_full"]]

    def test_state_continuation(self, golden):
        g = golden("rng_golden")
        gen = R.stream(9, "cont")
        gen.random(7)
        st = R.PhiloxState.of(gen)
        np.testing.assert_array_equal(R.words_to_doubles(st.words(15)).reshape(3, 5, 1), g["cont"])

    def test_skip_ahead_matches_global_mask(self):
        key = R.fold_key(0, "dynamics", "step", 0)
        m = R.sample_masks(R.PhiloxState.fresh(key), 8, 16, 32)
        rs = np.random.default_rng(0)
        for _ in range(20):
            b, t, n = int(rs.integers(8)), int(rs.integers(16)), int(rs.integers(32))
            assert R.mask_element(key, 8, 16, 32, b, t, n) == bool(m[b, t, n])

    def test_keep_schedule(self):
        assert R.keep_schedule(256, 25) == [1, 3, 5, 9, 13, 18, 25, 32, 40, 49, 59, 70, 81, 93, 106,
                                            119, 133, 148, 162, 177, 193, 209, 224, 240, 256]


class TestVq:
    @pytest.mark.parametrize("tag", ["f32", "f64"])
    def test_vq_matches_reference(self, golden, tag):
        g = golden("vq_golden")
        dt = torch.float32 if tag == "f32" else torch.float64
        z = torch.tensor(g[f"{tag}.z"], dtype=dt, requires_grad=True)
        cb = torch.tensor(g[f"{tag}.cb"], dtype=dt, requires_grad=True)
        idx, z_q, cbl, com = M.vq_quantize(z, cb)
        np.testing.assert_array_equal(idx, g[f"{tag}.idx"])
        np.testing.assert_array_equal(z_q.detach().numpy(), g[f"{tag}.zq"])
        (cbl + 0.25 * com + (z_q * z_q).sum()).backward()
        rtol = 1e-6 if tag == "f32" else 1e-12
        np.testing.assert_allclose(float(cbl), g[f"{tag}.cbl"], rtol=rtol)
        np.testing.assert_allclose(float(com), g[f"{tag}.com"], rtol=rtol)
        np.testing.assert_allclose(z.grad.numpy(), g[f"{tag}.gz"], rtol=rtol, atol=1e-7 if tag == "f32" else 1e-14)
        np.testing.assert_allclose(cb.grad.numpy(), g[f"{tag}.gcb"], rtol=rtol, atol=1e-7 if tag == "f32" else 1e-14)

    def test_vq_k6(self, golden):
        g = golden("vq_golden")
        idx, _, _, _ = M.vq_quantize(torch.tensor(g["k6.z"]), torch.tensor(g["k6.cb"]))
        np.testing.assert_array_equal(idx, g["k6.idx"])


def _check_grads(P, g, rtol=1e-9, atol=1e-12):
    for k, p in P.items():
        ref = g.get(f"grad.{k}")
        if ref is None:
            assert p.grad is None or float(p.grad.abs().max()) == 0.0, k
            continue
        np.testing.assert_allclose(p.grad.numpy(), ref, rtol=rtol, atol=atol, err_msg=k)


class TestModelsF64:
    @pytest.mark.parametrize("mode", ["prepend", "additive"])
    def test_dynamics_logits_loss_grads(self, golden, mode):
        g = golden(f"dynamics_{mode}_golden")
        cfg = M.DynCfg(model_dim=64, heads=2, ffn_dim=256, blocks=2, token_codes=64,
                       action_latent_dim=16, patches_per_frame=16, max_frames=4, mode=mode)
        init = M.init_dynamics(cfg, seed=3, dtype=np.float64)
        for k, v in init.items():
            np.testing.assert_array_equal(v, g[f"param.{k}"], err_msg=k)
        P = M.params_to_torch(init)
        lat = torch.tensor(g["latents"], requires_grad=True)
        logits = M.dyn_logits(P, cfg, g["tokens"], lat, g["mask"])
        np.testing.assert_allclose(logits.detach().numpy(), g["logits"], rtol=1e-10, atol=1e-12)
        loss, _ = M.dyn_loss(P, cfg, g["tokens"], lat, g["mask"])
        np.testing.assert_allclose(float(loss), float(g["loss"]), rtol=1e-12)
        loss.backward()
        _check_grads(P, g)
        np.testing.assert_allclose(lat.grad.numpy(), g["grad_latents"], rtol=1e-9, atol=1e-12)

    def test_tokenizer_forward_grads(self, golden):
        g = golden("tokenizer_golden")
        cfg = M.TokCfg(model_dim=32, heads=2, ffn_dim=128, blocks=1, codes=16, latent_dim=8,
                       patch=4, height=8, width=8, max_frames=3)
        init = M.init_tokenizer(cfg, seed=5, dtype=np.float64)
        for k, v in init.items():
            np.testing.assert_array_equal(v, g[f"param.{k}"], err_msg=k)
        P = M.params_to_torch(init)
        recon, idx, losses = M.tok_forward(P, cfg, torch.tensor(g["unit"]))
        np.testing.assert_array_equal(idx, g["idx"])
        np.testing.assert_allclose(recon.detach().numpy(), g["recon"], rtol=1e-10, atol=1e-12)
        for k in ("recon", "codebook", "commitment", "total"):
            np.testing.assert_allclose(float(losses[k]), float(g[f"loss.{k}"]), rtol=1e-11)
        losses["total"].backward()
        _check_grads(P, g)
        P32 = M.params_to_torch(M.init_tokenizer(cfg, seed=5), requires_grad=False)
        enc = M.tok_encode(P32, cfg, g["frames_u8"])
        np.testing.assert_array_equal(enc, g["enc32"])
        np.testing.assert_allclose(M.tok_decode(P32, cfg, enc), g["dec32"], rtol=1e-5, atol=1e-6)

    def test_lam_forward_grads(self, golden):
        g = golden("lam_golden")
        cfg = M.LamCfg(model_dim=32, heads=2, ffn_dim=128, blocks=1, codes=6, latent_dim=8,
                       patch=4, height=8, width=8, max_frames=3)
        init = M.init_lam(cfg, seed=6, dtype=np.float64)
        for k, v in init.items():
            np.testing.assert_array_equal(v, g[f"param.{k}"], err_msg=k)
        P = M.params_to_torch(init)
        recon, idx, losses = M.lam_forward(P, cfg, torch.tensor(g["unit"]))
        np.testing.assert_array_equal(idx, g["idx"])
        np.testing.assert_allclose(recon.detach().numpy(), g["recon"], rtol=1e-10, atol=1e-12)
        losses["total"].backward()
        _check_grads(P, g)


class TestSampling:
    @pytest.mark.parametrize("temp", [1.0, 0.7, 0.0])
    def test_sample_with_confidence(self, golden, temp):
        g = golden("sampling_golden")
        s, c = M.sample_with_confidence(g["logits"], temp, R.stream(16, "swc", str(temp)))
        np.testing.assert_array_equal(s, g[f"sampled.{temp}"])
        np.testing.assert_array_equal(c, g[f"conf.{temp}"])

    @pytest.mark.parametrize("tag", ["f32", "f64"])
    def test_decode_frame(self, golden, tag):
        g = golden("sampling_golden")
        dt = np.float32 if tag == "f32" else np.float64
        cfg = M.DynCfg(model_dim=64, heads=2, ffn_dim=256, blocks=2, token_codes=64,
                       action_latent_dim=16, patches_per_frame=16, max_frames=4)
        P = M.params_to_torch(M.init_dynamics(cfg, seed=4, dtype=dt), requires_grad=False)

        def logits_fn(tk, lat, mask):
            with torch.no_grad():
                return M.dyn_logits(P, cfg, tk, lat, mask).numpy()

        dec = M.decode_frame(logits_fn, g[f"{tag}.prev"], torch.tensor(g[f"{tag}.lat"]), steps=5,
                             gen=R.stream(18, "dec", tag))
        np.testing.assert_array_equal(dec, g[f"{tag}.decoded"])

    def test_rollout(self, golden):
        g = golden("sampling_golden")
        tcfg = M.TokCfg(model_dim=64, heads=2, ffn_dim=256, blocks=1, codes=64, latent_dim=16,
                        patch=4, height=16, width=16, max_frames=6)
        dcfg = M.DynCfg(model_dim=64, heads=2, ffn_dim=256, blocks=2, token_codes=64,
                        action_latent_dim=16, patches_per_frame=16, max_frames=6,
                        mode="ground_truth_embedding")
        tP = M.params_to_torch(M.init_tokenizer(tcfg, seed=6), requires_grad=False)
        dP = M.params_to_torch(M.init_dynamics(dcfg, seed=7), requires_grad=False)
        out = M.rollout(tP, tcfg, dP, dcfg, g["roll.frames"], [np.array([1, 3]), np.array([2, 0])],
                        horizon=2, steps=3, gen=R.stream(9, "roll"))
        # uint8 frames: allow the odd 1-LSB rounding flip from BLAS-order differences
        diff = np.abs(out.astype(int) - g["roll.out"].astype(int))
        assert diff.max() <= 1 and (diff > 0).mean() < 1e-3


def test_adamw_bit_exact(golden):
    g = golden("adamw_golden")
    params = {n: g[f"init.{n}"].copy() for n in ("a", "b", "c")}
    st = M.adamw_init(params)
    for step in range(3):
        grads = {n: g[f"grad{step}.{n}"] for n in params}
        M.adamw_step(params, grads, st, lr=3e-4 * (step + 1))
    for n in params:
        np.testing.assert_array_equal(params[n], g[f"final.{n}"])
        np.testing.assert_array_equal(st.m[n], g[f"m.{n}"])
        np.testing.assert_array_equal(st.v[n], g[f"v.{n}"])


def test_wsd_lr_endpoints():
    assert M.wsd_lr(1.0, 100, 10, 0.1, 0) == 0.0
    assert M.wsd_lr(1.0, 100, 10, 0.1, 5) == 0.5
    assert M.wsd_lr(1.0, 100, 10, 0.1, 50) == 1.0
    assert M.wsd_lr(1.0, 100, 10, 0.1, 95) == pytest.approx(0.5)
    assert M.wsd_lr(1.0, 100, 10, 0.1, 100) == 0.0


@pytest.mark.slow
def test_jasmine_b1_fp32(golden):
    """Full jasmine-base dims (patch 4), B=1, fp32: oracle vs reference loss / logits / grad norms."""
    g = golden("jasmine_b1_golden")
    cfg = M.DynCfg(patches_per_frame=256, max_frames=16)
    P = M.params_to_torch(M.init_dynamics(cfg, seed=0))
    lat = torch.tensor(g["lam_cb"][g["acts"]])
    loss, _ = M.dyn_loss(P, cfg, g["tokens"], lat, g["mask"])
    np.testing.assert_allclose(float(loss), float(g["loss"]), rtol=2e-6)
    loss.backward()
    for k, p in P.items():
        ref = float(g[f"gnorm.{k}"])
        got = float(p.grad.double().norm())
        assert got == pytest.approx(ref, rel=2e-4, abs=1e-9), k


def test_dit_predict_loss_grads_sample(golden):
    """ST-DiT oracle (diffusion.py:131-215) against the reference's f64 run: init draw order,
    x-prediction, ramp-weighted forcing loss with every gradient, and the Euler sampler."""
    g = golden("dit_golden")
    cfg = M.DitCfg(model_dim=32, heads=2, ffn_dim=128, blocks=1, latent_dim=8, action_latent_dim=8, action_vocab=7,
                   patches_per_frame=4, max_frames=4)
    init = M.init_dit(cfg, seed=3, dtype=np.float64)
    for k, v in init.items():
        np.testing.assert_array_equal(v, g[f"param.{k}"], err_msg=k)
    P = M.params_to_torch(init)
    act = torch.tensor(g["act"])
    pred = M.dit_predict_clean(P, cfg, g["latents"], g["tau"], act)
    np.testing.assert_allclose(pred.detach().numpy(), g["pred"], rtol=1e-10, atol=1e-12)
    loss = M.dit_loss(P, cfg, g["latents"], act, R.stream(22, "dit-loss"))
    np.testing.assert_allclose(float(loss), float(g["loss"]), rtol=1e-11)
    loss.backward()
    _check_grads(P, g)
    z = M.dit_sample_frame(P, cfg, g["latents"][:, :2], act, steps=3, gen=R.stream(23, "dit-sample"))
    np.testing.assert_allclose(z, g["sample"], rtol=1e-10, atol=1e-12)


def test_mae_forward_grads(golden):
    """MAE tokenizer oracle (diffusion.py:50-103) against the reference's f64 masked forward."""
    g = golden("mae_golden")
    cfg = M.MaeCfg(model_dim=32, heads=2, ffn_dim=128, blocks=1, latent_dim=8, patch=4, height=8, width=8,
                   max_frames=3)
    init = M.init_mae(cfg, seed=5, dtype=np.float64)
    for k, v in init.items():
        np.testing.assert_array_equal(v, g[f"param.{k}"], err_msg=k)
    P = M.params_to_torch(init)
    recon, latents, loss = M.mae_forward(P, cfg, torch.tensor(g["unit"]), R.stream(25, "mae-mask"))
    np.testing.assert_allclose(latents.detach().numpy(), g["latents"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(recon.detach().numpy(), g["recon"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(float(loss), float(g["loss"]), rtol=1e-11)
    loss.backward()
    _check_grads(P, g)
