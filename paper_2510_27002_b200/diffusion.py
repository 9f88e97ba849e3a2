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

from . import kernels as K
from .rng import stream
from .st import StConfig, init_st_stack_arrays, st_backward, st_forward, st_param_groups
from .tensor import ParamStore, Tensor, as_device, grad_buffers


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
        `.backward()` writes the gradients of every parameter (gt_action_embed: zero)."""
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
            G["gt_action_embed"].zero_()  # rollout-only table: no gradient from the loss

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
