"""Device parity at the BASELINE configurations (jasmine-base: D=512, 8 heads, F=2048, patch 4,
T=16, N=256; 6 dynamics blocks, 4 tokenizer / LAM blocks, 1024 / 6 codes), against the oracle
port and the reference's own golden runs.  Every tolerance comes from fidelity_threshold.json
["parity"] (the "_why" block there says what each one is calibrated on).

  C3  dynamics step, all 6 blocks, B=1: vs jasmine_b1_golden (the reference's fp32 run: loss,
      logits slice, every gradient norm) and vs the oracle port (every gradient)
  C1  tokenizer forward + quantize, B=2: losses, reconstruction; VQ indices exact on the oracle's
      fp32 z_e (near-ties within the stated epsilon excepted)
  C2  LAM forward + backward, B=1: losses and every gradient
  C5  decode_frame at jasmine-base dims (peaked logits), B=1, 25 MaskGIT steps
  AdamW: jz_adamw_step bit-exact against adamw_golden (the reference's optim.adamw_step)
  rollout: device rollout vs the reference's rollout (device_rollout_golden), ground-truth and
      additive conditioning; the reference's one-hot MaskGIT oracle (test_acceptance.py:236-266)
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
REPORT = {}

JB = dict(model_dim=512, heads=8, ffn_dim=2048)


def _rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _cos(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    na, nb = np.linalg.norm(a), np.linalg.norm(b)
    return 1.0 if na == 0 and nb == 0 else float(a @ b / max(na * nb, 1e-30))


def _report(name, **kv):
    REPORT.setdefault(name, {}).update({k: (float(v) if np.isscalar(v) else v) for k, v in kv.items()})
    out = Path(__file__).resolve().parent.parent / "gpurun_out"
    if out.is_dir():
        (out / "parity_report.json").write_text(json.dumps(REPORT, indent=1, default=str))


def _grad_check(model_params, ref_params, cos_min, rel_max=None, tag=""):
    """Every gradient against the reference; key biases (exactly 0 by softmax shift invariance)
    are bounded by the value-bias gradient instead.  Returns the worst cosine."""
    bad, worst = [], 1.0
    for k, p in model_params.items():
        ref = ref_params[k].grad
        got = p.grad.cpu().numpy() if p.grad is not None else np.zeros(p.shape, np.float32)
        if ref is None:
            continue
        ref = ref.numpy()
        if k.endswith(".k.b"):
            scale = np.linalg.norm(ref_params[k[:-3] + "v.b"].grad.numpy())
            if np.linalg.norm(got) > 1e-2 * max(scale, 1e-12):
                bad.append((k, "key-bias gradient not ~0", float(np.linalg.norm(got)), float(scale)))
            continue
        if np.linalg.norm(ref) < 1e-12 and np.linalg.norm(got) < 1e-12:
            continue
        c = _cos(got, ref)
        worst = min(worst, c)
        if c < cos_min or (rel_max is not None and _rel(got, ref) > rel_max):
            bad.append((k, c, _rel(got, ref)))
    _report(tag, worst_grad_cosine=worst)
    assert not bad, bad
    return worst


# ------------------------------------------------------------------------------------------------
# C3: dynamics train step, jasmine-base, all 6 blocks, B = 1
# ------------------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c3(golden):
    from paper_2510_27002_b200.configs import get_preset
    from paper_2510_27002_b200.dynamics import DynamicsModel
    import dataclasses
    g = golden("jasmine_b1_golden")
    cfg = dataclasses.replace(get_preset("jasmine-base"), patch=4, mode="pretrain_lam").dynamics_cfg()
    assert cfg.blocks == 6 and cfg.patches_per_frame == 256
    model = DynamicsModel(cfg, seed=0)
    ocfg = OM.DynCfg(**{k: getattr(cfg, k) for k in ("model_dim", "heads", "ffn_dim", "blocks", "token_codes",
                                                     "action_latent_dim", "patches_per_frame", "max_frames")})
    P = OM.params_to_torch(OM.init_dynamics(ocfg, seed=0))
    lat = g["lam_cb"][g["acts"]]
    torch.set_num_threads(max(1, min(16, torch.get_num_threads())))
    loss_ref, _ = OM.dyn_loss(P, ocfg, g["tokens"], torch.tensor(lat), g["mask"])
    loss_ref.backward()
    return dict(model=model, P=P, g=g, lat=lat, loss_ref=float(loss_ref))


def test_c3_six_blocks_vs_reference_golden(c3):
    """Loss, logits slice and every gradient norm against the reference's own fp32 run."""
    from paper_2510_27002_b200 import rng as R
    from paper_2510_27002_b200.tensor import Tensor
    model, g = c3["model"], c3["g"]
    # the reference drew the mask from stream(0, "dynamics", "step", 0): the device Philox must agree
    loss, stats = model.loss(g["tokens"], Tensor(c3["lat"]), R.stream(0, "dynamics", "step", 0))
    assert stats["masked_fraction"] == pytest.approx(float(g["mask"].mean()))
    dl = abs(float(loss.data) - float(g["loss"]))
    _report("c3", loss=float(loss.data), loss_ref=float(g["loss"]), loss_abs_diff=dl)
    assert dl < TOL["bf16_loss_abs"]
    loss.backward()
    worst_norm = 0.0
    for k, p in model.params.items():
        if k.endswith(".k.b"):
            continue
        ref = float(g[f"gnorm.{k}"])
        got = float(torch.linalg.vector_norm(p.grad.double()))
        if ref > 0:
            worst_norm = max(worst_norm, abs(got - ref) / ref)
    _report("c3", worst_grad_norm_rel=worst_norm)
    assert worst_norm < TOL["bf16_grad_rel_l2"]
    lg = model.logits(g["tokens"], Tensor(c3["lat"]), mask=g["mask"]).data
    sl = lg[0, :, :8, :16].cpu().numpy()
    r = _rel(sl, g["logits_slice"])
    rs = _rel(lg.sum(-1)[0].cpu().numpy(), g["logits_rowsum"])
    _report("c3", logits_slice_rel=r, logits_rowsum_rel=rs)
    assert r < TOL["bf16_logits_rel_l2"] and rs < TOL["bf16_logits_rel_l2"]


def test_c3_six_blocks_every_gradient_vs_oracle(c3):
    from paper_2510_27002_b200.tensor import Tensor
    model, g = c3["model"], c3["g"]
    loss, _ = model.loss(g["tokens"], Tensor(c3["lat"]), None, mask=g["mask"])
    # the port itself agrees with the reference's golden loss (fp32 summation-order noise only)
    assert abs(c3["loss_ref"] - float(g["loss"])) < 1e-4
    assert abs(float(loss.data) - c3["loss_ref"]) < TOL["bf16_loss_abs"]
    loss.backward()
    _grad_check(model.params, c3["P"], TOL["bf16_grad_cosine_min"], TOL["bf16_grad_rel_l2"], tag="c3")


# ------------------------------------------------------------------------------------------------
# C1: tokenizer forward + quantize at jasmine-base, B = 2
# ------------------------------------------------------------------------------------------------
TOK = dict(JB, blocks=4, codes=1024, latent_dim=32, patch=4, height=64, width=64, max_frames=16)


def _near_tie_ok(z, cb, got, ref):
    z = np.asarray(z, dtype=np.float64)
    cb = np.asarray(cb, dtype=np.float64)
    for r in np.nonzero(np.asarray(got) != np.asarray(ref))[0]:
        d = ((z[r] - cb) ** 2).sum(-1)
        scale = (z[r] ** 2).sum() + (cb ** 2).sum(-1).max()
        if abs(d[got[r]] - d[ref[r]]) > TOL["vq_index_mismatch_rel_gap"] * scale:
            return False
    return True


@pytest.fixture(scope="module")
def c1():
    from paper_2510_27002_b200.tokenizer import TokenizerConfig, VideoTokenizer
    tok = VideoTokenizer(TokenizerConfig(**TOK), seed=0)
    ocfg = OM.TokCfg(**TOK)
    P = OM.params_to_torch(OM.init_tokenizer(ocfg, seed=0), requires_grad=False)
    frames = OR.stream(0, "bench-frames").integers(0, 256, size=(2, 16, 64, 64, 3)).astype(np.uint8)
    unit = OM.frames_to_unit(frames)
    with torch.no_grad():
        z_e = OM.tok_encode_latent(P, ocfg, torch.tensor(unit))
        recon, idx, losses = OM.tok_forward(P, ocfg, torch.tensor(unit))
    return dict(tok=tok, P=P, frames=frames, unit=unit, z_e=z_e.numpy(), recon=recon.numpy(), idx=np.asarray(idx),
                losses={k: float(v) for k, v in losses.items()})


def test_c1_vq_indices_exact_on_oracle_latents(c1):
    """The fused VQ kernel on the oracle's own fp32 z_e: indices equal the reference argmin
    (dz=32, K=1024, 8,192 rows) except fp32 near-ties within the stated epsilon."""
    from paper_2510_27002_b200 import kernels as K
    z = c1["z_e"].reshape(-1, 32)
    cb = c1["P"]["codebook"].numpy()
    idx, zq, _ = K.vq_fwd(torch.tensor(z).cuda(), torch.tensor(cb).cuda())
    got = idx.cpu().numpy()
    ref = OM.vq_quantize(torch.tensor(c1["z_e"]), torch.tensor(cb))[0]
    ref = np.asarray(ref).reshape(-1)
    mism = int((got != ref).sum())
    _report("c1", vq_mismatches_on_oracle_latents=mism, rows=int(got.size))
    assert _near_tie_ok(z, cb, got, ref)
    # straight-through value z + (z_q - z) in f32 (tokenizer.py:78), not z_q itself
    np.testing.assert_array_equal(zq.cpu().numpy(), z + (cb[got] - z))


def test_c1_tokenizer_forward_vs_oracle(c1):
    tok = c1["tok"]
    z = tok.encode_latent(c1["frames"]).numpy()
    rz = _rel(z, c1["z_e"])
    recon, idx, losses = tok.forward(c1["unit"])
    agree = float((np.asarray(idx) == c1["idx"]).mean())
    rr = _rel(recon.numpy(), c1["recon"])
    diffs = {k: abs(float(losses[k].data) - c1["losses"][k]) / max(abs(c1["losses"][k]), 1e-12)
             for k in ("recon", "codebook", "commitment", "total")}
    _report("c1", z_e_rel=rz, index_agreement=agree, recon_rel=rr, **{f"loss_rel_{k}": v for k, v in diffs.items()})
    assert rz < TOL["bf16_logits_rel_l2"]
    # every code that differs from the oracle's must be explained by the bf16 encoder's latent
    # error: with z' = z + e, |z'-c|^2 - |z-c|^2 = 2 e.(z - c) + |e|^2, so a flip from the oracle's
    # code c_r to c_o needs gap = |z-c_o|^2 - |z-c_r|^2 <= 2 |e| (|z-c_o| + |z-c_r|) + 2 |e|^2
    zo = z.reshape(-1, 32).astype(np.float64)
    zr = c1["z_e"].reshape(-1, 32).astype(np.float64)
    cbk = c1["P"]["codebook"].numpy().astype(np.float64)
    io, ir = np.asarray(idx).reshape(-1), c1["idx"].reshape(-1)
    unexplained = 0
    for rrow in np.nonzero(io != ir)[0]:
        e = np.linalg.norm(zo[rrow] - zr[rrow])
        do, dr = np.linalg.norm(zr[rrow] - cbk[io[rrow]]), np.linalg.norm(zr[rrow] - cbk[ir[rrow]])
        if do ** 2 - dr ** 2 > 2 * e * (do + dr) + 2 * e ** 2:
            unexplained += 1
    _report("c1", mismatches=int((io != ir).sum()), unexplained_mismatches=unexplained)
    assert unexplained == 0
    assert agree >= TOL["vq_index_agreement_bf16_encoder"]
    assert rr < TOL["bf16_logits_rel_l2"]
    for k, v in diffs.items():
        assert v < TOL["bf16_loss_rel"], (k, v)


# ------------------------------------------------------------------------------------------------
# C2: LAM train step at jasmine-base (6 codes), B = 1
# ------------------------------------------------------------------------------------------------
def test_c2_lam_forward_backward_vs_oracle():
    from paper_2510_27002_b200.lam import LamConfig, LatentActionModel
    kw = dict(TOK, codes=6)
    lam = LatentActionModel(LamConfig(**kw), seed=0)
    ocfg = OM.LamCfg(**kw)
    P = OM.params_to_torch(OM.init_lam(ocfg, seed=0))
    frames = OR.stream(0, "bench-frames").integers(0, 256, size=(1, 16, 64, 64, 3)).astype(np.uint8)
    unit = OM.frames_to_unit(frames)
    recon, idx, losses = lam.forward(unit)
    r2, i2, l2 = OM.lam_forward(P, ocfg, torch.tensor(unit))
    np.testing.assert_array_equal(idx, np.asarray(i2))
    rr = _rel(recon.numpy(), r2.detach().numpy())
    diffs = {k: abs(float(losses[k].data) - float(l2[k])) / max(abs(float(l2[k])), 1e-12)
             for k in ("recon", "codebook", "commitment", "total")}
    _report("c2", recon_rel=rr, **{f"loss_rel_{k}": v for k, v in diffs.items()})
    assert rr < TOL["bf16_logits_rel_l2"]
    for k, v in diffs.items():
        assert v < TOL["bf16_loss_rel"], (k, v)
    losses["total"].backward()
    l2["total"].backward()
    _grad_check(lam.params, P, TOL["bf16_grad_cosine_min_vq_models"], tag="c2")


# ------------------------------------------------------------------------------------------------
# C5: decode_frame at jasmine-base dims
# ------------------------------------------------------------------------------------------------
def test_c5_decode_frame_jasmine_dims_vs_oracle():
    """One MaskGIT frame (25 steps, t = 4 context frames) at the C5 model dims, to_logits scaled so
    the picks are decided by clear margins.

    Per step (teacher-forced on the oracle's trajectory): the device logits of the same clip state
    pick the same token as the oracle's under the same uniform draws.  Whole chain: the device
    decode_frame (KV cache + device sampler) consumes exactly the oracle's draws, and its tokens
    agree with the oracle's; one early near-tie pick changes the context of every later step, so
    the chain agreement floor is lower than the per-step one."""
    import copy

    from paper_2510_27002_b200 import rng as R
    from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
    from paper_2510_27002_b200.tensor import Tensor
    kw = dict(JB, blocks=6, token_codes=1024, action_latent_dim=32, patches_per_frame=256, max_frames=16)
    m = DynamicsModel(DynamicsConfig(**kw), seed=0)
    m.params["to_logits.w"].data.mul_(60.0)
    ocfg = OM.DynCfg(**kw)
    P = OM.params_to_torch(OM.init_dynamics(ocfg, seed=0), requires_grad=False)
    P["to_logits.w"].mul_(60.0)
    prev = OR.stream(5, "c5-prev").integers(0, 1024, size=(1, 4, 256))
    lat = (OR.stream(5, "c5-lat").normal(size=(1, 4, 32)) * 0.1).astype(np.float32)
    og = OR.stream(5, "c5-rng")
    step_hits = [0, 0]

    def logits_fn(tk, la, mask):
        with torch.no_grad():
            ref = OM.dyn_logits(P, ocfg, tk, torch.tensor(la), mask).numpy()
        dev = m.logits(tk, Tensor(la), mask=mask).numpy()
        s_ref, _ = OM.sample_with_confidence(ref[:, -1], 1.0, copy.deepcopy(og))
        s_dev, _ = OM.sample_with_confidence(dev[:, -1], 1.0, copy.deepcopy(og))
        live = mask[:, -1]
        step_hits[0] += int((s_ref == s_dev)[live].sum())
        step_hits[1] += int(live.sum())
        return ref

    ref = OM.decode_frame(logits_fn, prev, lat, steps=25, gen=og)
    g = R.stream(5, "c5-rng")
    got = m.decode_frame(prev, lat, steps=25, rng=g)
    og2 = OR.stream(5, "c5-rng")
    OM.decode_frame(lambda tk, la, mask: np.zeros((1, tk.shape[1], 256, 1024), np.float32), prev, lat, steps=25,
                    gen=og2)
    step_agree = step_hits[0] / max(step_hits[1], 1)
    chain = float((got == ref).mean())
    _report("c5", step_agreement=step_agree, chain_token_agreement=chain)
    assert step_agree >= TOL["decode_step_agreement_peaked"]
    assert chain >= TOL["decode_token_agreement_jasmine_chain"]
    assert g.random() == og2.random()  # the device decode consumed exactly the reference's draws


# ------------------------------------------------------------------------------------------------
# AdamW bit-exact against the reference (optim.py:34-62)
# ------------------------------------------------------------------------------------------------
def test_adamw_kernel_bit_exact_vs_reference_golden(golden):
    from paper_2510_27002_b200.optim import adamw_init, adamw_step
    from paper_2510_27002_b200.tensor import Tensor
    g = golden("adamw_golden")
    names = ("b", "a", "c")
    params = {n: Tensor(g[f"init.{n}"].copy(), requires_grad=True) for n in names}
    st = adamw_init(params)
    for step in range(3):
        grads = {n: torch.tensor(g[f"grad{step}.{n}"]).cuda() for n in names}
        adamw_step(params, grads, st, lr=3e-4 * (step + 1))
    for n in names:
        np.testing.assert_array_equal(params[n].data.cpu().numpy(), g[f"final.{n}"], err_msg=n)
        np.testing.assert_array_equal(st.m[n].cpu().numpy(), g[f"m.{n}"], err_msg=n)
        np.testing.assert_array_equal(st.v[n].cpu().numpy(), g[f"v.{n}"], err_msg=n)


def test_adamw_flat_store_bit_exact_vs_reference_golden(golden):
    """The same three steps through ONE flat-buffer launch (ParamStore), as the trainers run it."""
    from collections import OrderedDict

    from paper_2510_27002_b200.optim import adamw_init, adamw_step
    from paper_2510_27002_b200.tensor import ParamStore
    g = golden("adamw_golden")
    names = ("b", "a", "c")
    store = ParamStore(OrderedDict((n, g[f"init.{n}"].copy()) for n in names))
    params = store.params
    st = adamw_init(params)
    grads = store.grads()
    for step in range(3):
        for n in names:
            grads[n].copy_(torch.tensor(g[f"grad{step}.{n}"]))
        adamw_step(params, grads, st, lr=3e-4 * (step + 1))
    for n in names:
        np.testing.assert_array_equal(params[n].data.cpu().numpy(), g[f"final.{n}"], err_msg=n)
        np.testing.assert_array_equal(st.m[n].cpu().numpy(), g[f"m.{n}"], err_msg=n)


def test_adamw_merged_params_with_strided_qkv_members():
    """cotrain merges dynamics params with LAM encoder params (trainer.py:290-293): the per-param
    path must update the strided q/k/v members of fused blocks exactly like the flat launch."""
    from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
    from paper_2510_27002_b200.optim import adamw_init, adamw_step
    from paper_2510_27002_b200.tensor import Tensor
    kw = dict(model_dim=128, heads=2, ffn_dim=512, blocks=1, token_codes=64, action_latent_dim=32,
              patches_per_frame=16, max_frames=4)
    a, b = DynamicsModel(DynamicsConfig(**kw), seed=1), DynamicsModel(DynamicsConfig(**kw), seed=1)
    gen = torch.Generator(device="cuda").manual_seed(0)
    ga = a._store.grads()
    for n, v in ga.items():
        v.copy_(torch.randn(v.shape, device="cuda", generator=gen) * 1e-2)
    merged = dict(b.params)
    merged["extra.w"] = Tensor(np.ones((3, 4), np.float32), requires_grad=True)
    gm = {n: ga[n].clone() for n in b.params}
    gm["extra.w"] = torch.full((3, 4), 0.5, device="cuda")
    sa, sb = adamw_init(a.params), adamw_init(merged)
    assert sa.store is not None and sb.store is None  # flat launch vs per-parameter fallback
    for step in range(2):
        adamw_step(a.params, ga, sa, 1e-3)
        adamw_step(merged, gm, sb, 1e-3)
    for n in a.params:
        assert torch.equal(a.params[n].data, b.params[n].data), n
    assert not torch.equal(merged["extra.w"].data, torch.ones(3, 4, device="cuda"))


# ------------------------------------------------------------------------------------------------
# rollout vs the reference, and the reference's one-hot MaskGIT oracle
# ------------------------------------------------------------------------------------------------
DEVROLL_TOK = dict(model_dim=128, heads=2, ffn_dim=512, blocks=1, codes=64, latent_dim=32, patch=16, height=64,
                   width=64, max_frames=6)
DEVROLL_DYN = dict(model_dim=128, heads=2, ffn_dim=512, blocks=1, token_codes=64, action_latent_dim=32,
                   patches_per_frame=16, max_frames=6)


@pytest.mark.parametrize("mode", ["ground_truth_embedding", "additive"])
def test_rollout_vs_reference_rollout(golden, mode):
    """dynamics.rollout through a real tokenizer against the reference's rollout output
    (device_rollout_golden; to_logits scaled x40 in both so picks have clear margins)."""
    from paper_2510_27002_b200 import rng as R
    from paper_2510_27002_b200 import sampling as SP
    from paper_2510_27002_b200.dynamics import ConditioningMode, DynamicsConfig, DynamicsModel, rollout
    from paper_2510_27002_b200.tensor import Tensor
    from paper_2510_27002_b200.tokenizer import TokenizerConfig, VideoTokenizer
    g = golden("device_rollout_golden")
    tok = VideoTokenizer(TokenizerConfig(**DEVROLL_TOK), seed=6)
    dyn = DynamicsModel(DynamicsConfig(**DEVROLL_DYN, mode=ConditioningMode(mode)), seed=7)
    dyn.params["to_logits.w"].data.mul_(40.0)
    np.testing.assert_array_equal(tok.encode(g["frames"]), g["tokens"])
    actions = list(g[f"{mode}.actions"])
    cb = Tensor(g[f"{mode}.codebook"]) if f"{mode}.codebook" in g else None
    out = rollout(tok, dyn, g["frames"], actions, horizon=2, steps=5, rng=R.stream(9, "dev-roll", mode),
                  source_codebook=cb)
    ref = g[f"{mode}.out"]
    assert out.shape == ref.shape and out.dtype == np.uint8
    # generated tokens: re-encode is not exact, so compare through the token path the rollout used
    if mode == "ground_truth_embedding":
        _, toks = SP.rollout_device(tok, dyn, g["frames"], actions, 2, steps=5, rng=R.stream(9, "dev-roll", mode),
                                    return_tokens=True)
        toks = toks.cpu().numpy()
    else:
        toks = None
    ref_tok = g[f"{mode}.out_tokens"]
    frame_diff = np.abs(out.astype(int) - ref.astype(int))
    rep = dict(frames_mean_abs=float(frame_diff.mean()), frames_max_abs=int(frame_diff.max()))
    if toks is not None:
        rep["token_agreement"] = float((toks == ref_tok).mean())
        assert rep["token_agreement"] >= TOL["decode_token_agreement_peaked"]
    _report(f"rollout.{mode}", **rep)
    assert rep["frames_mean_abs"] <= TOL["uint8_frames_mean_abs"]


def test_maskgit_one_hot_oracle_exact():
    """test_acceptance.py:236-266: a stand-in whose logits are +30 on the true token and -30
    elsewhere; decode_frame (device sampler) must return the truth exactly for steps 1, 5, 25."""
    from paper_2510_27002_b200 import rng as R
    from paper_2510_27002_b200.dynamics import ConditioningMode, DynamicsConfig, DynamicsModel
    from paper_2510_27002_b200.tensor import Tensor
    cfg = DynamicsConfig(model_dim=8, heads=2, ffn_dim=8, blocks=1, token_codes=8, action_latent_dim=4,
                         action_vocab=5, patches_per_frame=16, max_frames=6, mode=ConditioningMode.PREPEND)
    real = DynamicsModel(cfg, seed=15, dtype=np.float64)
    truth = R.stream(11, "acc-truth").integers(0, 8, size=(2, 4, 16))

    class Oracle:
        cfg = real.cfg
        params = real.params
        dtype = real.dtype

        def logits(self, tokens, action_latents, mask=None):
            b, t, n = tokens.shape
            out = np.full((b, t, n, 8), -30.0)
            grid = truth[:, :t]
            out[tuple(np.indices(grid.shape)) + (grid,)] = 30.0
            return out

    lat = Tensor(R.stream(12, "acc-lat").normal(size=(2, 3, 4)))
    for steps in (1, 5, 25):
        decoded = DynamicsModel.decode_frame(Oracle(), truth[:, :3], lat, steps=steps, rng=R.stream(13, "d", steps))
        np.testing.assert_array_equal(decoded, truth[:, 3], err_msg=f"steps={steps}")


# ------------------------------------------------------------------------------------------------
# gradients that flow through learned action tables
# ------------------------------------------------------------------------------------------------
def test_ground_truth_mode_trains_gt_action_embed():
    """GROUND_TRUTH conditioning: action ids go through embedding(gt_action_embed) (dynamics.py:95-96),
    so the table's gradient must match the oracle's (and every other gradient too)."""
    from paper_2510_27002_b200.dynamics import ConditioningMode, DynamicsConfig, DynamicsModel
    kw = dict(model_dim=128, heads=2, ffn_dim=512, blocks=1, token_codes=256, action_latent_dim=32,
              patches_per_frame=256, max_frames=4)
    m = DynamicsModel(DynamicsConfig(**kw, mode=ConditioningMode.GROUND_TRUTH), seed=3)
    ocfg = OM.DynCfg(**kw, mode="ground_truth_embedding")
    P = OM.params_to_torch(OM.init_dynamics(ocfg, seed=3))
    tokens = OR.stream(1, "gt-tokens").integers(0, 256, size=(2, 4, 256))
    acts = OR.stream(2, "gt-acts").integers(0, 7, size=(2, 3))
    mask = OR.sample_masks(OR.PhiloxState.fresh(OR.fold_key(0, "gt")), 2, 4, 256)
    loss, _ = m.loss(tokens, acts, None, mask=mask)
    ref, _ = OM.dyn_loss(P, ocfg, tokens, P["gt_action_embed"][torch.as_tensor(acts)], mask)
    assert abs(float(loss.data) - float(ref)) < TOL["bf16_loss_abs"]
    loss.backward()
    ref.backward()
    assert float(m.params["gt_action_embed"].grad.abs().max()) > 0
    _grad_check(m.params, P, TOL["bf16_grad_cosine_min"], tag="gt_mode")


def test_dit_trains_gt_action_embed_through_embedding():
    """train_diffusion's dit_loss (trainer.py:354-360): act = embedding(gt_action_embed, ids)."""
    from paper_2510_27002_b200 import rng as R
    from paper_2510_27002_b200.diffusion import DitConfig, DitDynamics
    from paper_2510_27002_b200.tensor import embedding
    kw = dict(model_dim=512, heads=8, ffn_dim=2048, blocks=1, latent_dim=32, action_latent_dim=32, action_vocab=7,
              patches_per_frame=16, max_frames=16)
    dit = DitDynamics(DitConfig(**kw), seed=4)
    P = OM.params_to_torch(OM.init_dit(OM.DitCfg(**kw), seed=4))
    g = OR.stream(7, "dit-gt")
    latents = np.tanh(g.normal(size=(2, 6, 16, 32))).astype(np.float32)
    ids = g.integers(0, 7, size=(2, 5))
    loss = dit.loss(latents, embedding(dit.params["gt_action_embed"], ids), R.stream(9, "dit-gt-loss"))
    ref = OM.dit_loss(P, OM.DitCfg(**kw), latents, P["gt_action_embed"][torch.as_tensor(ids)],
                      OR.stream(9, "dit-gt-loss"))
    assert abs(float(loss.data) - float(ref)) < max(TOL["bf16_loss_abs"], TOL["bf16_loss_rel"] * float(ref))
    loss.backward()
    ref.backward()
    got = dit.params["gt_action_embed"].grad.cpu().numpy()
    c = _cos(got, P["gt_action_embed"].grad.numpy())
    _report("dit_gt", gt_embed_cos=c)
    assert c >= TOL["bf16_grad_cosine_min"]
