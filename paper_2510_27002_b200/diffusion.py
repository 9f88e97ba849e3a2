"""ST-DiT diffusion-forcing dynamics on the device (diffusion.py:114-215).

Same config fields, parameter names/shapes/init draws and public methods as the reference's
`DitConfig` / `DitDynamics`, so it drops in for it (the second model family on
the same ST kernels):
- `predict_clean(noised, tau, action_latents)`: x-prediction. The frame's tokens are
  [action token, noise-level token, N latent tokens] (S = N + 2 = 18 at the reference's
  16-patch default), so spatial attention runs on the small-frame register-tile kernel (K3s),
  temporal attention on K4, the projections on K1 and the fp32 small-width linears.
- `loss(latents, action_latents, rng)`: ramp-weighted (w(tau) = tau) x-prediction MSE under
  linear-interpolation corruption; `.backward()` writes every parameter gradient.
- `sample_frame(...)`: the Euler walk toward the predicted clean latent, context re-corrupted
  at every model call.

The noise levels tau and the Gaussian draws come from the caller's numpy generator in the
reference's draw order (they are copied to the device as inputs, as the reference consumes
them on the host); the sinusoidal noise embedding is formed from those host taus exactly as
nn.py:134-142 does. The model itself runs in libjz kernels. The per-frame weighted MSE over the
(B, T, N, latent_dim) prediction (a few thousand elements) uses torch device arithmetic.
"""
from __future__ import annotations

import math
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import kernels as K
from .rng import stream
from .st import StConfig, init_st_stack_arrays, st_backward, st_forward, st_param_groups
from .tensor import ParamStore, Tensor, as_device, grad_buffers
from .tokenizer import frames_to_unit, unit_to_frames


def sinusoidal_embedding(values, dim: int) -> np.ndarray:
    """nn.py:134-142: sin/cos embedding of scalars in [0, 1] (float32), (..., dim)."""
    half = dim // 2
    freqs = np.exp(-math.log(10000.0) * np.arange(half, dtype=np.float32) / max(half - 1, 1))
    angles = np.asarray(values, dtype=np.float32)[..., None] * freqs * 1000.0
    emb = np.concatenate([np.sin(angles), np.cos(angles)], axis=-1)
    if dim % 2:
        emb = np.concatenate([emb, np.zeros(emb.shape[:-1] + (1,), dtype=np.float32)], axis=-1)
    return emb


def forcing_corrupt(latents: np.ndarray, tau: np.ndarray, rng: np.random.Generator) -> np.ndarray:
    """diffusion.py:106-111: z_tau = (1 - tau) z + tau eps, eps ~ N(0, 1), tau per (batch, frame)."""
    tau = np.asarray(tau, dtype=latents.dtype)[..., None, None]
    eps = rng.standard_normal(latents.shape).astype(latents.dtype)
    return (1.0 - tau) * latents + tau * eps


@dataclass(frozen=True)
class DitConfig:
    """diffusion.py:114-128."""
    model_dim: int = 512
    heads: int = 8
    ffn_dim: int = 2048
    blocks: int = 6
    latent_dim: int = 32
    action_latent_dim: int = 32
    action_vocab: int = 7
    patches_per_frame: int = 16
    max_frames: int = 16

    @property
    def st(self) -> StConfig:
        return StConfig(self.model_dim, self.heads, self.ffn_dim, self.blocks)


class DitDynamics:
    """ST-DiT over MAE latents with prepended action + noise-level tokens (diffusion.py:131-215)."""

    def __init__(self, cfg: DitConfig = DitConfig(), seed: int = 0, dtype=np.float32):
        self.cfg = cfg
        self.dtype = dtype
        rng = stream(seed, "dit-init")
        d = cfg.model_dim
        p: "OrderedDict[str, np.ndarray]" = OrderedDict()
        p["latent_embed.w"] = rng.normal(0, 0.02, (cfg.latent_dim, d)).astype(dtype)
        p["latent_embed.b"] = np.zeros(d, dtype=dtype)
        p["action_proj.w"] = rng.normal(0, 0.02, (cfg.action_latent_dim, d)).astype(dtype)
        p["action_proj.b"] = np.zeros(d, dtype=dtype)
        p["null_action"] = rng.normal(0, 0.02, (cfg.action_latent_dim,)).astype(dtype)
        p["gt_action_embed"] = rng.normal(0, 0.02, (cfg.action_vocab, cfg.action_latent_dim)).astype(dtype)
        p["noise_proj.w"] = rng.normal(0, 0.02, (d, d)).astype(dtype)
        p["noise_proj.b"] = np.zeros(d, dtype=dtype)
        p["pos_spatial"] = rng.normal(0, 0.02, (cfg.patches_per_frame + 2, d)).astype(dtype)
        p["pos_temporal"] = rng.normal(0, 0.02, (cfg.max_frames, d)).astype(dtype)
        p.update(init_st_stack_arrays(rng, cfg.st, prefix="dit", dtype=dtype))
        p["to_latent.w"] = rng.normal(0, 0.02, (d, cfg.latent_dim)).astype(dtype)
        p["to_latent.b"] = np.zeros(cfg.latent_dim, dtype=dtype)
        self._store = ParamStore(p, groups=st_param_groups(cfg.st, "dit"))
        self.params = self._store.params

    # -----------------------------------------------------------------------------------------
    def _cond(self, action_latents, frames: int, B: int) -> torch.Tensor:
        """_conditioning (diffusion.py:156-162): [null_action, a_0 .. a_{T-2}] -> (B*T, dl_a) f32."""
        lat = as_device(action_latents, torch.float32)
        if lat.shape[1] != frames - 1:
            raise ValueError(f"need {frames - 1} actions for {frames} frames")
        dla = self.cfg.action_latent_dim
        null = self.params["null_action"].data.view(1, 1, dla).expand(B, 1, dla)
        return torch.cat([null, lat.view(B, frames - 1, dla)], dim=1).reshape(B * frames, dla).contiguous()

    def _forward(self, noised: torch.Tensor, tau: np.ndarray, action_latents, save: bool):
        cfg, P = self.cfg, self.params
        B, T, N, dl = noised.shape
        if N != cfg.patches_per_frame or dl != cfg.latent_dim:
            raise ValueError(f"latent grid {(N, dl)} does not match config")
        if T > cfg.max_frames:
            raise ValueError(f"clip length {T} exceeds max_frames {cfg.max_frames}")
        D, S = cfg.model_dim, N + 2
        z = noised.reshape(B * T * N, dl).contiguous()
        x_lat = K.linear_f32(z, P["latent_embed.w"].data, P["latent_embed.b"].data)
        cond = self._cond(action_latents, T, B)
        act = K.linear_f32(cond, P["action_proj.w"].data, P["action_proj.b"].data)
        nemb = as_device(sinusoidal_embedding(tau, D).astype(np.float32).reshape(B * T, D))
        ntok = K.linear_f32(nemb, P["noise_proj.w"].data, P["noise_proj.b"].data)
        # tokens 1..N+1 of every frame = [noise-level token, latents]; token 0 (the action) is
        # prepended by the assembly kernel with (e + pos_spatial[s]) + pos_temporal[t]
        emb = torch.cat([ntok.view(B, T, 1, D), x_lat.view(B, T, N, D)], dim=2).reshape(B * T * (N + 1), D)
        x = K.assemble_fwd(emb, act, P["pos_spatial"].data, P["pos_temporal"].data, B=B, T=T, N=N + 1, D=D,
                           prepend=True)
        (_, y32), ctx = st_forward(x, P, cfg.st, "dit", B=B, T=T, S=S, save=save, final_f32=True,
                                   final_bf16=False)
        y_lat = y32.view(B, T, S, D)[:, :, 2:].reshape(B * T * N, D).contiguous()
        pred = K.linear_f32(y_lat, P["to_latent.w"].data, P["to_latent.b"].data)
        saved = dict(ctx=ctx, z=z, cond=cond, nemb=nemb, y_lat=y_lat, B=B, T=T, N=N) if save else None
        return pred.view(B, T, N, dl), saved

    def predict_clean(self, noised, tau, action_latents) -> Tensor:
        """diffusion.py:164-180: estimate the clean latents, (B, T, N, latent_dim)."""
        tau = np.asarray(tau)
        pred, _ = self._forward(as_device(np.asarray(noised, dtype=np.float32) if not isinstance(noised, torch.Tensor)
                                          else noised, torch.float32), tau, action_latents, save=False)
        return Tensor(pred)

    def loss(self, latents: np.ndarray, action_latents, rng: np.random.Generator) -> Tensor:
        """diffusion.py:182-192: ramp-weighted x-prediction loss, per-frame tau ~ U(0, 1).
        `.backward()` writes the gradients of every parameter; gt_action_embed's comes through
        `action_latents` when it is `embedding(params["gt_action_embed"], ids)` (trainer.py:358-359)."""
        cfg, P = self.cfg, self.params
        latents = np.asarray(latents, dtype=np.float32)
        b, t = latents.shape[:2]
        tau = rng.uniform(0.0, 1.0, size=(b, t))
        noised = forcing_corrupt(latents, tau, rng)
        pred, sv = self._forward(as_device(noised), tau, action_latents, save=True)
        lat = as_device(latents)
        tau_d = as_device(tau.astype(np.float32))
        err = pred - lat
        per_frame = (err * err).mean(dim=(2, 3))
        loss = (per_frame * tau_d).mean()
        store = self._store
        N, dl, D = sv["N"], cfg.latent_dim, cfg.model_dim
        S = N + 2

        def backward():
            G = grad_buffers(P, store)
            # d loss / d pred = 2 err tau_bt / (N dl B T)
            d_pred = (err * (tau_d * (2.0 / (N * dl * b * t))).view(b, t, 1, 1)).reshape(b * t * N, dl).contiguous()
            d_ylat = torch.empty(b * t * N, D, dtype=K.F32, device=pred.device)
            K.linear_f32_bwd(sv["y_lat"], d_pred, P["to_latent.w"].data, dx=d_ylat, dW=G["to_latent.w"],
                             db=G["to_latent.b"])
            dy = torch.zeros(b, t, S, D, dtype=K.F32, device=pred.device)
            dy[:, :, 2:] = d_ylat.view(b, t, N, D)
            dx = st_backward(sv["ctx"], dy.view(b * t * S, D), P, G, cfg.st, "dit")
            K.assemble_bwd(dx, B=b, T=t, N=N + 1, D=D, prepend=True, d_ps=G["pos_spatial"],
                           d_pt=G["pos_temporal"][:t])
            if t < cfg.max_frames:
                G["pos_temporal"][t:].zero_()
            dxv = dx.view(b, t, S, D)
            d_act = dxv[:, :, 0].reshape(b * t, D).contiguous()
            d_ntok = dxv[:, :, 1].reshape(b * t, D).contiguous()
            d_xlat = dxv[:, :, 2:].reshape(b * t * N, D).contiguous()
            d_cond = torch.empty(b * t, cfg.action_latent_dim, dtype=K.F32, device=pred.device)
            K.linear_f32_bwd(sv["cond"], d_act, P["action_proj.w"].data, dx=d_cond, dW=G["action_proj.w"],
                             db=G["action_proj.b"])
            G["null_action"].copy_(d_cond.view(b, t, -1)[:, 0].sum(0))
            K.linear_f32_bwd(sv["nemb"], d_ntok, P["noise_proj.w"].data, dW=G["noise_proj.w"],
                             db=G["noise_proj.b"])
            K.linear_f32_bwd(sv["z"], d_xlat, P["latent_embed.w"].data, dW=G["latent_embed.w"],
                             db=G["latent_embed.b"])
            G["gt_action_embed"].zero_()
            if isinstance(action_latents, Tensor) and action_latents._backward is not None:
                # embedding(dit.params["gt_action_embed"], actions) (trainer.py:358-359): frames 1..T-1
                # of the conditioning are the action latents; the table gets their scatter
                action_latents.grad = d_cond.view(b, t, -1)[:, 1:].contiguous()
                action_latents.backward()

        return Tensor(loss, _backward=backward)

    def sample_frame(self, context_latents, action_latents, steps: int = 25, context_noise: float = 0.1,
                     rng: np.random.Generator | None = None) -> np.ndarray:
        """diffusion.py:194-215: the next frame's latents (B, N, latent_dim). One full-clip model call
        per Euler step, the context re-corrupted with fresh host draws each call; z stays on device."""
        if steps < 1:
            raise ValueError("steps must be >= 1")
        if rng is None:
            rng = stream(0, "diffusion-sample")
        context = np.asarray(context_latents, dtype=np.float32)
        b, t_prev, n, dl = context.shape
        z = as_device(rng.standard_normal((b, 1, n, dl)).astype(np.float32))
        full = torch.empty(b, t_prev + 1, n, dl, dtype=torch.float32, device=z.device)
        for k in range(steps, 0, -1):
            tau_k = k / steps
            tau_prev = (k - 1) / steps
            full[:, :t_prev] = as_device(forcing_corrupt(context, np.full((b, t_prev), context_noise), rng))
            full[:, t_prev:] = z
            tau = np.concatenate([np.full((b, t_prev), context_noise), np.full((b, 1), tau_k)], axis=1)
            pred, _ = self._forward(full, tau, action_latents, save=False)
            z = z + (tau_k - tau_prev) * (pred[:, -1:] - z) / tau_k
        return z[:, 0].cpu().numpy()


@dataclass(frozen=True)
class MaeConfig:
    """diffusion.py:23-47."""
    model_dim: int = 512
    heads: int = 8
    ffn_dim: int = 2048
    blocks: int = 4
    latent_dim: int = 32
    patch: int = 16
    height: int = 64
    width: int = 64
    channels: int = 3
    max_frames: int = 16
    mask_prob_max: float = 0.9

    @property
    def patches_per_frame(self) -> int:
        return (self.height // self.patch) * (self.width // self.patch)

    @property
    def patch_dim(self) -> int:
        return self.patch * self.patch * self.channels

    @property
    def st(self) -> StConfig:
        return StConfig(self.model_dim, self.heads, self.ffn_dim, self.blocks)


class MaeTokenizer:
    """MAE tokenizer with tanh-bounded continuous latents (diffusion.py:50-103): K9 patchify, K1
    patch embedding, mask-token select, ST encoder / decoder stacks (S = 16 at patch 16: the
    small-frame attention kernel), fp32 latent projections, K1 pixel head."""

    def __init__(self, cfg: MaeConfig = MaeConfig(), seed: int = 0, dtype=np.float32):
        self.cfg = cfg
        self.dtype = dtype
        rng = stream(seed, "mae-init")
        d = cfg.model_dim
        p: "OrderedDict[str, np.ndarray]" = OrderedDict()
        p["patch_embed.w"] = rng.normal(0, 0.02, (cfg.patch_dim, d)).astype(dtype)
        p["patch_embed.b"] = np.zeros(d, dtype=dtype)
        p["mask_token"] = rng.normal(0, 0.02, (d,)).astype(dtype)
        p["pos_spatial"] = rng.normal(0, 0.02, (cfg.patches_per_frame, d)).astype(dtype)
        p["pos_temporal"] = rng.normal(0, 0.02, (cfg.max_frames, d)).astype(dtype)
        p.update(init_st_stack_arrays(rng, cfg.st, prefix="enc", dtype=dtype))
        p["to_latent.w"] = rng.normal(0, 0.02, (d, cfg.latent_dim)).astype(dtype)
        p["to_latent.b"] = np.zeros(cfg.latent_dim, dtype=dtype)
        p["from_latent.w"] = rng.normal(0, 0.02, (cfg.latent_dim, d)).astype(dtype)
        p["from_latent.b"] = np.zeros(d, dtype=dtype)
        p.update(init_st_stack_arrays(rng, cfg.st, prefix="dec", dtype=dtype))
        p["to_pixels.w"] = rng.normal(0, 0.02, (d, cfg.patch_dim)).astype(dtype)
        p["to_pixels.b"] = np.zeros(cfg.patch_dim, dtype=dtype)
        self._store = ParamStore(p, groups=st_param_groups(cfg.st, "enc") + st_param_groups(cfg.st, "dec"))
        self.params = self._store.params

    def _frames(self, frames) -> torch.Tensor:
        fr = as_device(frames)
        if fr.dtype != torch.uint8:
            fr = fr.float()
        b, t, h, w, c = fr.shape
        if (h, w, c) != (self.cfg.height, self.cfg.width, self.cfg.channels):
            raise ValueError(f"frame geometry {(h, w, c)} does not match config")
        if t > self.cfg.max_frames:
            raise ValueError(f"clip length {t} exceeds max_frames {self.cfg.max_frames}")
        return fr.contiguous()

    def _encode(self, fr: torch.Tensor, mask, save: bool):
        cfg, P = self.cfg, self.params
        B, T = fr.shape[0], fr.shape[1]
        N, D = cfg.patches_per_frame, cfg.model_dim
        p16, p32 = K.patchify(fr.reshape(B * T, cfg.height, cfg.width, cfg.channels), cfg.patch, f32=save)
        emb = K.linear_fwd(p16, K.cast_bf16(P["patch_embed.w"].data), P["patch_embed.b"].data, epilogue=L.EPI_F32)
        m = None
        if mask is not None:  # diffusion.py:76-77: where(mask, mask_token, x)
            m = as_device(np.asarray(mask, dtype=bool).reshape(B * T * N))
            emb = torch.where(m[:, None], P["mask_token"].data.view(1, D), emb)
        x = K.assemble_fwd(emb, None, P["pos_spatial"].data, P["pos_temporal"].data, B=B, T=T, N=N, D=D,
                           prepend=False)
        (_, y32), ctx = st_forward(x, P, cfg.st, "enc", B=B, T=T, S=N, save=save, final_f32=True,
                                   final_bf16=False)
        lat = torch.tanh(K.linear_f32(y32, P["to_latent.w"].data, P["to_latent.b"].data))
        return lat, dict(ctx=ctx, y32=y32, p16=p16, p32=p32, m=m, B=B, T=T) if save else None

    def encode(self, frames, mask=None) -> Tensor:
        """diffusion.py:82-86: tanh-bounded latents (B, T, N, latent_dim); frames uint8 or unit f32."""
        fr = self._frames(frames.data if isinstance(frames, Tensor) else frames)
        lat, _ = self._encode(fr, mask, save=False)
        return Tensor(lat.view(fr.shape[0], fr.shape[1], self.cfg.patches_per_frame, self.cfg.latent_dim))

    def _decode(self, lat: torch.Tensor, B: int, T: int, save: bool):
        cfg, P = self.cfg, self.params
        x = K.linear_f32(lat, P["from_latent.w"].data, P["from_latent.b"].data)
        y, ctx = st_forward(x, P, cfg.st, "dec", B=B, T=T, S=cfg.patches_per_frame, save=save)
        w_tp = K.cast_bf16(P["to_pixels.w"].data)
        rp = K.linear_fwd(y, w_tp, P["to_pixels.b"].data, epilogue=L.EPI_F32)
        return rp, dict(ctx=ctx, y=y, w_tp=w_tp) if save else None

    def decode(self, latents) -> Tensor:
        """diffusion.py:88-92: unit-range frames (B, T, H, W, C)."""
        cfg = self.cfg
        lat = as_device(latents, torch.float32)
        B, T = lat.shape[0], lat.shape[1]
        rp, _ = self._decode(lat.reshape(-1, cfg.latent_dim).contiguous(), B, T, save=False)
        unit, _ = K.unpatchify(rp, B * T, cfg.height, cfg.width, cfg.channels, cfg.patch)
        return Tensor(unit.view(B, T, cfg.height, cfg.width, cfg.channels))

    def forward(self, frames, rng: np.random.Generator):
        """diffusion.py:94-103: masked-autoencoder pass -> (recon, latents, loss); loss.backward() trains."""
        cfg, P = self.cfg, self.params
        fr = self._frames(frames.data if isinstance(frames, Tensor) else frames)
        B, T = fr.shape[0], fr.shape[1]
        N, D, dl = cfg.patches_per_frame, cfg.model_dim, cfg.latent_dim
        p = rng.uniform(0.0, cfg.mask_prob_max, size=(B, T))
        mask = rng.random((B, T, N)) < p[:, :, None]
        lat, enc = self._encode(fr, mask, save=True)
        rp, dec = self._decode(lat, B, T, save=True)
        loss, _, g16 = K.mse(rp, enc["p32"], grad16=True)
        recon, _ = K.unpatchify(rp, B * T, cfg.height, cfg.width, cfg.channels, cfg.patch)
        store = self._store

        def backward():
            G = grad_buffers(P, store)
            K.colsum_bf16(g16, G["to_pixels.b"])
            K.linear_dw(dec["y"], g16, G["to_pixels.w"])
            dy = K.linear_dx(g16, dec["w_tp"], epilogue=L.EPI_F32)
            dxd = st_backward(dec["ctx"], dy, P, G, cfg.st, "dec")
            d_lat = torch.empty(B * T * N, dl, dtype=K.F32, device=dxd.device)
            K.linear_f32_bwd(lat, dxd, P["from_latent.w"].data, dx=d_lat, dW=G["from_latent.w"],
                             db=G["from_latent.b"])
            d_pre = d_lat * (1.0 - lat * lat)  # tanh'
            d_y = torch.empty(B * T * N, D, dtype=K.F32, device=dxd.device)
            K.linear_f32_bwd(enc["y32"], d_pre, P["to_latent.w"].data, dx=d_y, dW=G["to_latent.w"],
                             db=G["to_latent.b"])
            dxe = st_backward(enc["ctx"], d_y, P, G, cfg.st, "enc")
            d_emb = torch.empty(B * T * N, D, dtype=K.BF16, device=dxd.device)
            K.assemble_bwd(dxe, B=B, T=T, N=N, D=D, prepend=False, d_emb=d_emb, d_ps=G["pos_spatial"],
                           d_pt=G["pos_temporal"][:T])
            if T < cfg.max_frames:
                G["pos_temporal"][T:].zero_()
            m = enc["m"]
            G["mask_token"].copy_((dxe * m[:, None]).sum(0))  # masked rows feed the mask token
            d_emb.masked_fill_(m[:, None], 0)                  # ... and not the patch embedding
            K.colsum_bf16(d_emb, G["patch_embed.b"])
            K.linear_dw(enc["p16"], d_emb, G["patch_embed.w"])

        return (Tensor(recon.view(B, T, cfg.height, cfg.width, cfg.channels)),
                Tensor(lat.view(B, T, N, dl)), Tensor(loss, _backward=backward))


def diffusion_rollout(mae: MaeTokenizer, dit: DitDynamics, conditioning_frames: np.ndarray, actions, horizon: int,
                      steps: int = 25, context_noise: float = 0.1, rng: np.random.Generator | None = None,
                      prefix_action_latents=None) -> np.ndarray:
    """diffusion.py:217-251: encode the conditioning frames, generate `horizon` frames one at a time
    (sample_frame), clip to the tanh bottleneck and decode through the MAE -> uint8 frames."""
    if len(actions) < horizon:
        raise ValueError(f"need {horizon} actions, got {len(actions)}")
    if rng is None:
        rng = stream(0, "diffusion-rollout")
    b, n_cond = conditioning_frames.shape[:2]
    unit = frames_to_unit(conditioning_frames) if conditioning_frames.dtype == np.uint8 else conditioning_frames
    latents = mae.encode(np.asarray(unit, dtype=np.float32)).numpy()
    dlat = dit.cfg.action_latent_dim
    if prefix_action_latents is not None:
        history = as_device(prefix_action_latents, torch.float32)
    else:
        null = dit.params["null_action"].data.view(1, 1, dlat)
        history = torch.zeros(b, n_cond - 1, dlat, dtype=torch.float32, device=null.device) + null
    table = dit.params["gt_action_embed"].data
    for step in range(horizon):
        action = actions[step]
        if isinstance(action, (Tensor, torch.Tensor)):
            lat = as_device(action, torch.float32).reshape(b, 1, dlat)
        else:
            ids = as_device(np.asarray(action, dtype=np.int64).reshape(b))
            if int(ids.min()) < 0 or int(ids.max()) >= table.shape[0]:
                raise IndexError("action id out of range")
            lat = table[ids].view(b, 1, dlat)
        history = torch.cat([history, lat], dim=1)
        nxt = dit.sample_frame(latents, history, steps=steps, context_noise=context_noise, rng=rng)
        latents = np.concatenate([latents, nxt[:, None]], axis=1)
    latents = np.clip(latents, -1.0 + 1e-6, 1.0 - 1e-6)  # bottleneck contract
    return unit_to_frames(mae.decode(latents.astype(np.float32)).numpy())
