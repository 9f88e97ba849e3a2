"""Generate the golden fixtures that pin the oracle to the UNMODIFIED reference.

Run in the build container (the reference is mounted read-only there; it does
not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes small .npz files next to this script.  Every array is produced by calling
deskworld (the reference) through its public API; nothing here re-implements it.
"""
from __future__ import annotations

import dataclasses
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = os.environ.get("DESKWORLD_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from deskworld import rng as R  # noqa: E402
from deskworld.autodiff import Tensor  # noqa: E402
from deskworld.dynamics import (ConditioningMode, DynamicsConfig, DynamicsModel,  # noqa: E402
                                _sample_with_confidence, rollout, sample_masks)
from deskworld.lam import LamConfig, LatentActionModel  # noqa: E402
from deskworld.optim import adamw_init, adamw_step  # noqa: E402
from deskworld.tokenizer import TokenizerConfig, VideoTokenizer, vq_quantize  # noqa: E402

OUT = Path(__file__).resolve().parent


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"wrote {name}.npz ({sum(a.nbytes for a in map(np.asarray, arrays.values()))} B raw)")


def grads_of(params, loss):
    loss.backward()
    return {f"grad.{k}": np.asarray(p.grad) for k, p in params.items() if p.grad is not None}


def gen_rng():
    keys = [(0,), (0, "dynamics", "step", 0), (7, "tokenizer-init"), (0, "dynamics", "step", 123456),
            (2**63 + 5, "x"), ("a", "b", 3)]
    folded = np.array([R.fold_key(*k) for k in keys], dtype=np.uint64)
    g = R.stream(0, "dynamics", "step", 0)
    words = g.integers(0, 2**64, size=64, dtype=np.uint64)
    g = R.stream(0, "dynamics", "step", 0)
    doubles = g.random(64)
    m_small, p_small = sample_masks(R.stream(1, "m"), 3, 4, 16, return_p=True)
    g = R.stream(0, "dynamics", "step", 5)
    m_full, p_full = sample_masks(g, 2, 16, 256, return_p=True)
    st = g.bit_generator.state
    after = np.array([int(x) for x in st["state"]["counter"]] + [int(st["buffer_pos"])], dtype=np.uint64)
    # a partially consumed generator (state continuation contract used by the sampler)
    g = R.stream(9, "cont")
    g.random(7)
    cont = g.random((3, 5, 1))
    save("rng_golden", folded=folded, words=words, doubles=doubles, m_small=m_small, p_small=p_small,
         m_full=m_full, p_full=p_full, after_full=after, cont=cont,
         key_strs=np.array(["|".join(map(str, k)) for k in keys]))


def gen_vq():
    out = {}
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        g = R.stream(3, "vq", tag)
        z = g.normal(size=(300, 8)).astype(dt) * 0.5
        cb = g.normal(size=(32, 8)).astype(dt) * 0.5
        z[5] = cb[7]                     # exact hit
        cb_t = Tensor(cb, requires_grad=True)
        z_t = Tensor(z, requires_grad=True)
        idx, z_q, cbl, com = vq_quantize(z_t, cb_t)
        (cbl + 0.25 * com + (z_q * z_q).sum()).backward()
        out.update({f"{tag}.z": z, f"{tag}.cb": cb, f"{tag}.idx": idx, f"{tag}.zq": z_q.data,
                    f"{tag}.cbl": np.asarray(cbl.data), f"{tag}.com": np.asarray(com.data),
                    f"{tag}.gz": z_t.grad, f"{tag}.gcb": cb_t.grad})
    # LAM-sized codebook (K=6) in f32
    g = R.stream(4, "vq6")
    z = g.normal(size=(45, 32)).astype(np.float32) * 0.1
    cb = g.uniform(-1 / 6, 1 / 6, size=(6, 32)).astype(np.float32)
    idx, _, _, _ = vq_quantize(Tensor(z), Tensor(cb))
    out.update({"k6.z": z, "k6.cb": cb, "k6.idx": idx})
    save("vq_golden", **out)


DYN_SMALL = dict(model_dim=64, heads=2, ffn_dim=256, blocks=2, token_codes=64,
                 action_latent_dim=16, patches_per_frame=16, max_frames=4)


def gen_dynamics():
    for mode in ("prepend", "additive"):
        cfg = DynamicsConfig(**DYN_SMALL, mode=ConditioningMode(mode))
        model = DynamicsModel(cfg, seed=3, dtype=np.float64)
        g = R.stream(11, "dyn-golden", mode)
        tokens = g.integers(0, 64, size=(2, 4, 16))
        lat = Tensor(g.normal(size=(2, 3, 16)) * 0.5, requires_grad=True)
        mask = sample_masks(R.stream(12, "dyn-mask", mode), 2, 4, 16)
        logits = model.logits(tokens, lat, mask=mask)
        loss, stats = model.loss(tokens, lat, R.stream(0, "unused"), mask=mask)
        grads = grads_of(model.params, loss)
        arrays = {f"param.{k}": v.data for k, v in model.params.items()}
        save(f"dynamics_{mode}_golden", tokens=tokens, latents=lat.data, mask=mask, logits=logits.data,
             loss=np.asarray(loss.data), grad_latents=lat.grad, **arrays, **grads)


TOK_SMALL = dict(model_dim=32, heads=2, ffn_dim=128, blocks=1, codes=16, latent_dim=8,
                 patch=4, height=8, width=8, max_frames=3)


def gen_tokenizer_lam():
    cfg = TokenizerConfig(**TOK_SMALL)
    tok = VideoTokenizer(cfg, seed=5, dtype=np.float64)
    g = R.stream(13, "tok-golden")
    unit = g.uniform(-1, 1, size=(2, 3, 8, 8, 3))
    recon, idx, losses = tok.forward(Tensor(unit))
    grads = grads_of(tok.params, losses["total"])
    frames_u8 = g.integers(0, 256, size=(2, 3, 8, 8, 3)).astype(np.uint8)
    tok32 = VideoTokenizer(cfg, seed=5)
    enc = tok32.encode(frames_u8)
    dec = tok32.decode(enc)
    save("tokenizer_golden", unit=unit, recon=recon.data, idx=idx,
         **{f"loss.{k}": np.asarray(v.data) for k, v in losses.items()},
         **{f"param.{k}": v.data for k, v in tok.params.items()}, **grads,
         frames_u8=frames_u8, enc32=enc, dec32=dec)

    lcfg = LamConfig(**{**TOK_SMALL, "codes": 6})
    lam = LatentActionModel(lcfg, seed=6, dtype=np.float64)
    unit = R.stream(14, "lam-golden").uniform(-1, 1, size=(2, 3, 8, 8, 3))
    recon, idx, losses = lam.forward(Tensor(unit))
    grads = grads_of(lam.params, losses["total"])
    save("lam_golden", unit=unit, recon=recon.data, idx=idx,
         **{f"loss.{k}": np.asarray(v.data) for k, v in losses.items()},
         **{f"param.{k}": v.data for k, v in lam.params.items()}, **grads)


def gen_sampling():
    g = R.stream(15, "swc")
    logits = (g.normal(size=(3, 16, 64)) * 2.0).astype(np.float32)
    out = {"logits": logits}
    for temp in (1.0, 0.7, 0.0):
        s, c = _sample_with_confidence(logits, temp, R.stream(16, "swc", str(temp)))
        out[f"sampled.{temp}"] = s
        out[f"conf.{temp}"] = c
    cfg = DynamicsConfig(**DYN_SMALL, mode=ConditioningMode.PREPEND)
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        model = DynamicsModel(cfg, seed=4, dtype=dt)
        gg = R.stream(17, "dec", tag)
        prev = gg.integers(0, 64, size=(2, 2, 16))
        lat = Tensor((gg.normal(size=(2, 2, 16)) * 0.5).astype(dt))
        dec = model.decode_frame(prev, lat, steps=5, rng=R.stream(18, "dec", tag))
        out.update({f"{tag}.prev": prev, f"{tag}.lat": lat.data, f"{tag}.decoded": dec})
    # rollout through a real tokenizer (ground-truth action table), as test_dynamics.py:203-222
    tcfg = TokenizerConfig(model_dim=64, heads=2, ffn_dim=256, blocks=1, codes=64, latent_dim=16,
                           patch=4, height=16, width=16, max_frames=6)
    tok = VideoTokenizer(tcfg, seed=6)
    dcfg = DynamicsConfig(**{**DYN_SMALL, "max_frames": 6}, mode=ConditioningMode.GROUND_TRUTH)
    dyn = DynamicsModel(dcfg, seed=7)
    frames = R.stream(23, "f").integers(0, 256, size=(2, 4, 16, 16, 3)).astype(np.uint8)
    actions = [np.array([1, 3]), np.array([2, 0])]
    roll = rollout(tok, dyn, frames, actions, horizon=2, steps=3, rng=R.stream(9, "roll"))
    out.update({"roll.frames": frames, "roll.out": roll})
    save("sampling_golden", **out)


def gen_adamw():
    g = R.stream(19, "adam")
    params = {n: Tensor(g.normal(size=s).astype(np.float32), requires_grad=True)
              for n, s in (("b", (7,)), ("a", (3, 5)), ("c", (64,)))}
    st = adamw_init(params)
    init = {f"init.{n}": p.data.copy() for n, p in params.items()}
    grads_all = {}
    for step in range(3):
        grads = {n: (g.normal(size=p.data.shape) * 10.0 ** (-step)).astype(np.float32) for n, p in params.items()}
        for n, v in grads.items():
            grads_all[f"grad{step}.{n}"] = v
        adamw_step(params, grads, st, lr=3e-4 * (step + 1))
    save("adamw_golden", **init, **grads_all, **{f"final.{n}": p.data for n, p in params.items()},
         **{f"m.{n}": st.m[n] for n in params}, **{f"v.{n}": st.v[n] for n in params})


def gen_jasmine_summary():
    """Full jasmine-base dims (patch 4), B=1, fp32: loss, logits slice and gradient norms."""
    from deskworld.configs import get_preset
    cfg = dataclasses.replace(get_preset("jasmine-base"), patch=4, mode="pretrain_lam")
    dcfg = cfg.dynamics_cfg()
    t0 = time.time()
    model = DynamicsModel(dcfg, seed=0)
    tokens = R.stream(1, "bench-tokens").integers(0, 1024, size=(1, 16, 256))
    lam_cb = R.stream(2, "golden-lam-cb").uniform(-1 / 6, 1 / 6, size=(6, 32)).astype(np.float32)
    acts = R.stream(2, "bench-actions").integers(0, 6, size=(1, 15))
    lat = Tensor(lam_cb[acts])
    loss, stats = model.loss(tokens, lat, R.stream(0, "dynamics", "step", 0))
    mask = sample_masks(R.stream(0, "dynamics", "step", 0), 1, 16, 256)
    logits = model.logits(tokens, lat, mask=mask)
    grads = grads_of(model.params, loss)
    norms = {f"gnorm.{k[5:]}": np.float64(np.linalg.norm(v.astype(np.float64))) for k, v in grads.items()}
    heads = {f"ghead.{k[5:]}": v.reshape(-1)[:16].copy() for k, v in grads.items()}
    save("jasmine_b1_golden", tokens=tokens, acts=acts, lam_cb=lam_cb, mask=mask,
         loss=np.asarray(loss.data), logits_slice=logits.data[0, :, :8, :16].copy(),
         logits_rowsum=logits.data.sum(axis=-1)[0], **norms, **heads)
    print(f"jasmine summary in {time.time() - t0:.1f}s")


def gen_checkpoint():
    """A JASCKPT1 bundle written by the reference's save_checkpoint (checkpoint.py:40-66)."""
    from deskworld.checkpoint import CheckpointBundle, save_checkpoint
    g = R.stream(7, "ckpt-golden")
    arrays = {"param.w": g.normal(size=(3, 5)).astype(np.float32),
              "param.b": g.normal(size=(5,)).astype(np.float32),
              "adam.m.w": np.zeros((3, 5), np.float32),
              "counts": np.arange(6, dtype=np.int64).reshape(2, 3),
              "scalar": np.array(2.5, dtype=np.float64)}
    bundle = CheckpointBundle(step=42, config={"preset": "tiny", "lr": 3e-5, "dims": [4, 8]}, arrays=arrays,
                              loader_state={"seed": 3, "epoch": 1, "cursor": 8, "prefetch_depth": 2},
                              rng_state={"seed": 3, "stage": "dynamics"},
                              meta={"stage": "dynamics", "seed": 3,
                                    "adam": {"t": 5, "beta1": 0.9, "beta2": 0.999, "eps": 1e-8, "weight_decay": 0.0}})
    save_checkpoint(bundle, OUT / "ckpt_ref.jasckpt")
    print("wrote ckpt_ref.jasckpt")


def gen_records():
    """A tiny JASREC dataset (records.py:120-169) and the reference loader's first batches."""
    import shutil

    from deskworld.env import Episode
    from deskworld.records import Chunking, LoaderState, shuffled_batches, write_dataset
    root = OUT / "jasrec_ref"
    shutil.rmtree(root, ignore_errors=True)
    g = R.stream(8, "jasrec-golden")
    eps = []
    for s in range(7):
        n = int(g.integers(10, 30))
        eps.append(Episode(seed=100 + s, frames=g.integers(0, 256, size=(n, 8, 8, 3), dtype=np.uint8),
                           actions=g.integers(0, 6, size=(n,)).astype(np.uint8)))
    index = write_dataset(iter(eps), Chunking(frames_per_record=8, records_per_file=4), root)
    it = shuffled_batches(index, LoaderState(seed=11), batch_size=3, seq_len=5)
    out = {}
    for k in range(5):
        fr, ac, st = next(it)
        out[f"frames{k}"] = fr
        out[f"actions{k}"] = ac
        out[f"state{k}"] = np.array([st.seed, st.epoch, st.cursor, st.prefetch_depth], dtype=np.int64)
    save("records", **out)


def gen_dit():
    """ST-DiT (diffusion.py:131-215): init, predict_clean, ramp-weighted loss + grads, sample_frame."""
    from deskworld.diffusion import DitConfig, DitDynamics
    kw = dict(model_dim=32, heads=2, ffn_dim=128, blocks=1, latent_dim=8, action_latent_dim=8, action_vocab=7,
              patches_per_frame=4, max_frames=4)
    dit = DitDynamics(DitConfig(**kw), seed=3, dtype=np.float64)
    g = R.stream(21, "dit-golden")
    latents = g.uniform(-1, 1, size=(2, 3, 4, 8))
    act = g.normal(size=(2, 2, 8)) * 0.1
    tau = g.uniform(0, 1, size=(2, 3))
    pred = dit.predict_clean(latents, tau, Tensor(act)).data
    loss = dit.loss(latents, Tensor(act), R.stream(22, "dit-loss"))
    grads = grads_of(dit.params, loss)
    z = dit.sample_frame(latents[:, :2], Tensor(act), steps=3, rng=R.stream(23, "dit-sample"))
    save("dit_golden", latents=latents, act=act, tau=tau, pred=pred, loss=np.asarray(loss.data), sample=z,
         **{f"param.{k}": v.data for k, v in dit.params.items()}, **grads)


def gen_mae():
    """MAE tokenizer (diffusion.py:50-103): init, masked forward (recon, latents, loss) + grads, decode."""
    from deskworld.diffusion import MaeConfig, MaeTokenizer
    kw = dict(model_dim=32, heads=2, ffn_dim=128, blocks=1, latent_dim=8, patch=4, height=8, width=8, max_frames=3)
    mae = MaeTokenizer(MaeConfig(**kw), seed=5, dtype=np.float64)
    unit = R.stream(24, "mae-golden").uniform(-1, 1, size=(2, 3, 8, 8, 3))
    recon, latents, loss = mae.forward(Tensor(unit), R.stream(25, "mae-mask"))
    grads = grads_of(mae.params, loss)
    save("mae_golden", unit=unit, recon=recon.data, latents=latents.data, loss=np.asarray(loss.data),
         **{f"param.{k}": v.data for k, v in mae.params.items()}, **grads)


def gen_device_rollout():
    """rollout (dynamics.py:220-260) through a real tokenizer at dims the device path runs
    (model_dim 128, 2 heads of 64, patch 16 on 64x64 frames: N = 16), ground-truth and additive
    conditioning.  to_logits.w is scaled by 40 so the MaskGIT picks are decided by clear margins
    (bf16 vs fp32 logits then pick the same tokens); the scaling is part of the fixture."""
    tcfg = TokenizerConfig(model_dim=128, heads=2, ffn_dim=512, blocks=1, codes=64, latent_dim=32,
                           patch=16, height=64, width=64, max_frames=6)
    tok = VideoTokenizer(tcfg, seed=6)
    frames = R.stream(23, "dev-roll").integers(0, 256, size=(2, 4, 64, 64, 3)).astype(np.uint8)
    out = {"frames": frames, "tokens": tok.encode(frames)}
    base = dict(model_dim=128, heads=2, ffn_dim=512, blocks=1, token_codes=64, action_latent_dim=32,
                patches_per_frame=16, max_frames=6)
    for mode in (ConditioningMode.GROUND_TRUTH, ConditioningMode.ADDITIVE):
        dyn = DynamicsModel(DynamicsConfig(**base, mode=mode), seed=7)
        dyn.params["to_logits.w"].data *= np.float32(40.0)
        if mode is ConditioningMode.GROUND_TRUTH:
            actions, cb = [np.array([1, 3]), np.array([2, 0])], None
        else:
            cb = Tensor(R.stream(24, "dev-roll-cb").uniform(-0.5, 0.5, size=(6, 32)).astype(np.float32))
            actions = [np.array([4, 1]), np.array([0, 5])]
        roll = rollout(tok, dyn, frames, actions, horizon=2, steps=5, rng=R.stream(9, "dev-roll", mode.value),
                       source_codebook=cb)
        # the generated tokens, through the same public calls rollout makes (dynamics.py:243-258)
        g = R.stream(9, "dev-roll", mode.value)
        tokens = tok.encode(frames)
        hist = Tensor(np.broadcast_to(dyn.params["null_action"].data, (2, 3, 32)).copy())
        for a in actions:
            lat = dyn.action_latents_for(a.reshape(2, 1), cb)
            hist = Tensor(np.concatenate([hist.data, lat.data], axis=1))
            nxt = dyn.decode_frame(tokens, hist, steps=5, rng=g)
            tokens = np.concatenate([tokens, nxt[:, None]], axis=1)
        from deskworld.tokenizer import unit_to_frames
        assert np.array_equal(unit_to_frames(tok.decode(tokens)), roll)
        out[f"{mode.value}.out"] = roll
        out[f"{mode.value}.out_tokens"] = tokens
        out[f"{mode.value}.actions"] = np.stack(actions)
        if cb is not None:
            out[f"{mode.value}.codebook"] = cb.data
    save("device_rollout_golden", **out)


def gen_configs():
    """configs.py presets and the model configs derived from them (JSON)."""
    import json
    from deskworld.configs import PRESETS
    res = {}
    for name, cfg in PRESETS.items():
        d = {"train": cfg.to_dict(), "tokenizer": dataclasses.asdict(cfg.tokenizer_cfg),
             "lam": dataclasses.asdict(cfg.lam_cfg), "mae": dataclasses.asdict(cfg.mae_cfg),
             "dit": dataclasses.asdict(cfg.dit_cfg)}
        for cond in (None, "additive", "prepend"):
            dc = dataclasses.asdict(cfg.dynamics_cfg(cond))
            dc["mode"] = cfg.dynamics_cfg(cond).mode.value
            d[f"dynamics.{cond}"] = dc
        res[name] = d
    (OUT / "configs_golden.json").write_text(json.dumps(res, indent=1, sort_keys=True))
    print("wrote configs_golden.json")


if __name__ == "__main__":
    which = sys.argv[1:] or ["rng", "vq", "dynamics", "toklam", "sampling", "adamw", "jasmine", "checkpoint",
                             "records"]
    fns = {"rng": gen_rng, "vq": gen_vq, "dynamics": gen_dynamics, "toklam": gen_tokenizer_lam,
           "sampling": gen_sampling, "adamw": gen_adamw, "jasmine": gen_jasmine_summary,
           "checkpoint": gen_checkpoint, "records": gen_records, "dit": gen_dit, "mae": gen_mae,
           "device_rollout": gen_device_rollout, "configs": gen_configs}
    for w in which:
        fns[w]()
