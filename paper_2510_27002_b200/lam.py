"""Latent action model on B200 (mirror of deskworld/lam.py), forward AND training backward.

Encoder (lam.py:79-94): patchify -> patch_embed GEMM -> positions -> ST stack ->
final LN (fp32) -> K10 mean-pool over patches -> frames 1..T-1 -> fp32 to_latent ->
K8 VQ (K = 6).  Decoder (lam.py:104-118): dec_embed GEMM on frames 0..T-2, fp32
action_proj of the quantised latent prepended as spatial token 0, dec positions,
ST stack (S = 257, T-1 frames) -> final LN dropping s=0 -> to_pixels GEMM ->
recon.  `forward(frames)` returns losses whose `total.backward()` runs the full
hand-scheduled backward (straight-through VQ, deterministic reductions) and
fills `p.grad` for every parameter — the C2 training step.
"""
from __future__ import annotations

from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import kernels as K
from .rng import stream
from .st import StConfig, init_st_stack_arrays, st_backward, st_forward, st_param_groups
from .tensor import ParamStore, Tensor, as_device, grad_buffers
from .tokenizer import _check_geometry, _vq


@dataclass(frozen=True)
class LamConfig:
    """lam.py:22-47."""
    model_dim: int = 512
    heads: int = 8
    ffn_dim: int = 2048
    blocks: int = 4
    codes: int = 6
    latent_dim: int = 32
    patch: int = 16
    height: int = 64
    width: int = 64
    channels: int = 3
    max_frames: int = 16
    commitment_beta: float = 0.25

    @property
    def patches_per_frame(self) -> int:
        return (self.height // self.patch) * (self.width // self.patch)

    @property
    def patch_dim(self) -> int:
        return self.patch * self.patch * self.channels

    @property
    def st(self) -> StConfig:
        return StConfig(self.model_dim, self.heads, self.ffn_dim, self.blocks)


class LatentActionModel:
    def __init__(self, cfg: LamConfig = LamConfig(), seed: int = 0, dtype=np.float32):
        self.cfg = cfg
        self.dtype = dtype
        rng = stream(seed, "lam-init")
        d = cfg.model_dim
        p: "OrderedDict[str, np.ndarray]" = OrderedDict()
        p["patch_embed.w"] = rng.normal(0, 0.02, (cfg.patch_dim, d)).astype(dtype)
        p["patch_embed.b"] = np.zeros(d, dtype=dtype)
        p["pos_spatial"] = rng.normal(0, 0.02, (cfg.patches_per_frame, d)).astype(dtype)
        p["pos_temporal"] = rng.normal(0, 0.02, (cfg.max_frames, d)).astype(dtype)
        p.update(init_st_stack_arrays(rng, cfg.st, prefix="enc", dtype=dtype))
        p["to_latent.w"] = rng.normal(0, 0.02, (d, cfg.latent_dim)).astype(dtype)
        p["to_latent.b"] = np.zeros(cfg.latent_dim, dtype=dtype)
        bound = 1.0 / cfg.codes
        p["codebook"] = rng.uniform(-bound, bound, (cfg.codes, cfg.latent_dim)).astype(dtype)
        p["dec_embed.w"] = rng.normal(0, 0.02, (cfg.patch_dim, d)).astype(dtype)
        p["dec_embed.b"] = np.zeros(d, dtype=dtype)
        p["action_proj.w"] = rng.normal(0, 0.02, (cfg.latent_dim, d)).astype(dtype)
        p["action_proj.b"] = np.zeros(d, dtype=dtype)
        p["dec_pos_spatial"] = rng.normal(0, 0.02, (cfg.patches_per_frame + 1, d)).astype(dtype)
        p["dec_pos_temporal"] = rng.normal(0, 0.02, (cfg.max_frames, d)).astype(dtype)
        p.update(init_st_stack_arrays(rng, cfg.st, prefix="dec", dtype=dtype))
        p["to_pixels.w"] = rng.normal(0, 0.02, (d, cfg.patch_dim)).astype(dtype)
        p["to_pixels.b"] = np.zeros(cfg.patch_dim, dtype=dtype)
        self._store = ParamStore(p, groups=st_param_groups(cfg.st, "enc") + st_param_groups(cfg.st, "dec"))
        self.params = self._store.params

    # -- helpers -----------------------------------------------------------------
    def _frames_device(self, frames) -> torch.Tensor:
        if isinstance(frames, Tensor):
            frames = frames.data
        if isinstance(frames, torch.Tensor):
            t = frames.to(torch.device("cuda", torch.cuda.current_device()))
            return t.contiguous() if t.dtype == torch.uint8 else t.float().contiguous()
        arr = np.asarray(frames)
        return as_device(arr if arr.dtype == np.uint8 else arr.astype(np.float32))

    def _check(self, fr):
        b, t = fr.shape[0], fr.shape[1]
        if t < 2:
            raise ValueError("need at least 2 frames to infer actions")
        _check_geometry(self.cfg, tuple(fr.shape))

    def _encoder(self, fr, save: bool):
        cfg, P = self.cfg, self.params
        B, T = fr.shape[0], fr.shape[1]
        N, D = cfg.patches_per_frame, cfg.model_dim
        p16, p32 = K.patchify(fr.reshape(B * T, cfg.height, cfg.width, cfg.channels), cfg.patch, f32=save)
        w_pe = K.cast_bf16(P["patch_embed.w"].data)
        emb = K.linear_fwd(p16, w_pe, P["patch_embed.b"].data, epilogue=L.EPI_F32)
        x = K.assemble_fwd(emb, None, P["pos_spatial"].data, P["pos_temporal"].data, B=B, T=T, N=N, D=D,
                           prepend=False)
        (_, y32), ctx = st_forward(x, P, cfg.st, "enc", B=B, T=T, S=N, save=save, final_f32=True, final_bf16=False)
        pooled = K.mean_pool(y32, B * T, N, D)
        trans = pooled.view(B, T, D)[:, 1:].contiguous().view(B * (T - 1), D)
        z_e = K.linear_f32(trans, P["to_latent.w"].data, P["to_latent.b"].data)
        return dict(p16=p16, p32=p32, ctx=ctx, trans=trans, z_e=z_e, B=B, T=T)

    # -- encoder (lam.py:79-101, 131-144) -----------------------------------------
    def _encode_pre_vq(self, frames) -> Tensor:
        fr = self._frames_device(frames)
        self._check(fr)
        e = self._encoder(fr, save=False)
        return Tensor(e["z_e"].view(e["B"], e["T"] - 1, self.cfg.latent_dim))

    def encoder_only(self, frames):
        """lam.py:96-101: (indices (B, T-1), z_q_st Tensor, codebook_loss, commitment_loss).

        The three tensors share one encoder graph (cotrain, trainer.py:306-309): the dynamics
        backward hands d(z_q_st) to z_q_st.backward(), the losses contribute their coefficients
        (codebook -> codebook rows, beta * commitment -> z_e), and the encoder backward runs once
        into p.grad (encoder parameters and codebook; decoder gradients are zero)."""
        cfg, P = self.cfg, self.params
        fr = self._frames_device(frames)
        self._check(fr)
        e = self._encoder(fr, save=True)
        B, T = e["B"], e["T"]
        Tm, D, N, dl = T - 1, cfg.model_dim, cfg.patches_per_frame, cfg.latent_dim
        z_e = e["z_e"]
        idx, zq, sq = _vq(z_e, P["codebook"].data)
        numel_z = z_e.numel()
        loss = K.sum_scaled(sq, 1.0 / numel_z)
        store = self._store
        graph = {"cb": 0.0, "commit": 0.0, "done": False}
        zq_t = Tensor(zq.view(B, Tm, dl), requires_grad=True)

        def run(d_zq):
            if graph["done"]:
                return
            graph["done"] = True
            G = grad_buffers(P, store)
            if store is not None and store.grad_flat is not None and store.grads_are_views(G):
                store.grad_flat.zero_()  # decoder parameters take no part in this graph
            else:
                for g in G.values():
                    g.zero_()
            dz = d_zq.reshape(B * Tm, dl).float().contiguous() if d_zq is not None else torch.zeros_like(z_e)
            d_ze = torch.empty_like(z_e)
            K.vq_bwd(z_e, P["codebook"].data, idx, dz, commit_coef=graph["commit"] * 2.0 / numel_z,
                     cb_coef=graph["cb"] * 2.0 / numel_z, dz_out=d_ze, dcodebook=G["codebook"])
            d_trans = torch.empty(B * Tm, D, dtype=K.F32, device=z_e.device)
            K.linear_f32_bwd(e["trans"], d_ze, P["to_latent.w"].data, dx=d_trans, dW=G["to_latent.w"],
                             db=G["to_latent.b"])
            d_pool = torch.zeros(B, T, D, dtype=K.F32, device=z_e.device)
            d_pool[:, 1:] = d_trans.view(B, Tm, D)
            d_y = K.mean_pool_bwd(d_pool.view(B * T, D), B * T, N, D)
            dx_e = st_backward(e["ctx"], d_y, P, G, cfg.st, "enc")
            d_emb = torch.empty(B * T * N, D, dtype=K.BF16, device=z_e.device)
            K.assemble_bwd(dx_e, B=B, T=T, N=N, D=D, prepend=False, d_emb=d_emb, d_ps=G["pos_spatial"],
                           d_pt=G["pos_temporal"][:T])
            K.colsum_bf16(d_emb, G["patch_embed.b"])
            K.linear_dw(e["p16"], d_emb, G["patch_embed.w"])

        zq_t._backward = lambda: run(zq_t.grad)

        def hook(role):
            def add(c):
                graph[role] += c
            return add

        cb_t = Tensor(loss, _backward=lambda: run(None), _coef_hook=hook("cb"))
        commit_t = Tensor(loss.clone(), _backward=lambda: run(None), _coef_hook=hook("commit"))
        return idx.view(B, Tm).cpu().numpy(), zq_t, cb_t, commit_t

    def infer_actions_device(self, frames) -> torch.Tensor:
        z_e = self._encode_pre_vq(frames)
        idx, _, _ = _vq(z_e.data.view(-1, self.cfg.latent_dim), self.params["codebook"].data)
        return idx.view(tuple(z_e.shape[:-1]))

    def infer_actions(self, frames) -> np.ndarray:
        """lam.py:131-136: latent action indices (B, T-1)."""
        return self.infer_actions_device(frames).cpu().numpy()

    def infer_action(self, frame_t, frame_t1) -> int:
        clip = np.stack([np.asarray(frame_t), np.asarray(frame_t1)])[None]
        return int(self.infer_actions(clip)[0, 0])

    def action_latents(self, indices) -> Tensor:
        """lam.py:143-144: codebook rows for action indices."""
        arr = indices.cpu().numpy() if isinstance(indices, torch.Tensor) else np.asarray(indices)
        if arr.size and (arr.min() < 0 or arr.max() >= self.cfg.codes):
            raise IndexError(f"embedding ids out of range [0, {self.cfg.codes})")
        return Tensor(self.params["codebook"].data[as_device(arr.astype(np.int64))])

    # -- full forward + backward (lam.py:104-129) ---------------------------------
    def forward(self, frames, _indices_on_device: bool = False):
        """(recon of frames 1..T-1, action indices (B, T-1), losses); losses["total"].backward() trains.
        `_indices_on_device` (internal, training stages): indices stay on device (no host sync)."""
        cfg, P = self.cfg, self.params
        fr = self._frames_device(frames)
        self._check(fr)
        B, T = fr.shape[0], fr.shape[1]
        N, D, dl, PD = cfg.patches_per_frame, cfg.model_dim, cfg.latent_dim, cfg.patch_dim
        Tm = T - 1
        enc = self._encoder(fr, save=True)
        z_e = enc["z_e"]
        idx, zq_st, sq = _vq(z_e, P["codebook"].data)
        numel_z = z_e.numel()
        vq_loss = K.sum_scaled(sq, 1.0 / numel_z)
        # decoder on frames 0..T-2 with the quantised action latent prepended as token 0
        p16 = enc["p16"].view(B, T, N, PD)
        past16 = p16[:, :-1].contiguous().view(B * Tm * N, PD)
        target32 = enc["p32"].view(B, T, N, PD)[:, 1:].contiguous().view(B * Tm * N, PD)
        w_de = K.cast_bf16(P["dec_embed.w"].data)
        emb = K.linear_fwd(past16, w_de, P["dec_embed.b"].data, epilogue=L.EPI_F32)
        act = K.linear_f32(zq_st, P["action_proj.w"].data, P["action_proj.b"].data)
        x = K.assemble_fwd(emb, act, P["dec_pos_spatial"].data, P["dec_pos_temporal"].data, B=B, T=Tm, N=N, D=D,
                           prepend=True)
        y, dctx = st_forward(x, P, cfg.st, "dec", B=B, T=Tm, S=N + 1, final_skip=True, save=True)
        w_tp = K.cast_bf16(P["to_pixels.w"].data)
        rp = K.linear_fwd(y, w_tp, P["to_pixels.b"].data, epilogue=L.EPI_F32)
        rec_loss, _, g16 = K.mse(rp, target32, grad16=True)
        total = rec_loss + vq_loss + cfg.commitment_beta * vq_loss
        recon, _ = K.unpatchify(rp, B * Tm, cfg.height, cfg.width, cfg.channels, cfg.patch)
        store = self._store

        def backward():
            G = grad_buffers(P, store)
            # to_pixels
            K.colsum_bf16(g16, G["to_pixels.b"])
            K.linear_dw(y, g16, G["to_pixels.w"])
            dy = K.linear_dx(g16, w_tp, epilogue=L.EPI_F32)
            dx = st_backward(dctx, dy, P, G, cfg.st, "dec")
            d_emb = torch.empty(B * Tm * N, D, dtype=K.BF16, device=dx.device)
            d_act = torch.empty(B * Tm, D, dtype=K.F32, device=dx.device)
            K.assemble_bwd(dx, B=B, T=Tm, N=N, D=D, prepend=True, d_emb=d_emb, d_act=d_act,
                           d_ps=G["dec_pos_spatial"], d_pt=G["dec_pos_temporal"][:Tm])
            if Tm < cfg.max_frames:
                G["dec_pos_temporal"][Tm:].zero_()
            K.colsum_bf16(d_emb, G["dec_embed.b"])
            K.linear_dw(past16, d_emb, G["dec_embed.w"])
            d_zq = torch.empty(B * Tm, dl, dtype=K.F32, device=dx.device)
            K.linear_f32_bwd(zq_st, d_act, P["action_proj.w"].data, dx=d_zq, dW=G["action_proj.w"],
                             db=G["action_proj.b"])
            # VQ: straight-through to z_e, commitment (beta) and codebook terms (lam.py:126)
            d_ze = torch.empty_like(z_e)
            K.vq_bwd(z_e, P["codebook"].data, idx, d_zq, commit_coef=cfg.commitment_beta * 2.0 / numel_z,
                     cb_coef=2.0 / numel_z, dz_out=d_ze, dcodebook=G["codebook"])
            d_trans = torch.empty(B * Tm, D, dtype=K.F32, device=dx.device)
            K.linear_f32_bwd(enc["trans"], d_ze, P["to_latent.w"].data, dx=d_trans, dW=G["to_latent.w"],
                             db=G["to_latent.b"])
            d_pool = torch.zeros(B, T, D, dtype=K.F32, device=dx.device)
            d_pool[:, 1:] = d_trans.view(B, Tm, D)
            d_y = K.mean_pool_bwd(d_pool.view(B * T, D), B * T, N, D)
            dx_e = st_backward(enc["ctx"], d_y, P, G, cfg.st, "enc")
            d_emb_e = torch.empty(B * T * N, D, dtype=K.BF16, device=dx.device)
            K.assemble_bwd(dx_e, B=B, T=T, N=N, D=D, prepend=False, d_emb=d_emb_e, d_ps=G["pos_spatial"],
                           d_pt=G["pos_temporal"][:T])
            if T < cfg.max_frames:
                G["pos_temporal"][T:].zero_()
            K.colsum_bf16(d_emb_e, G["patch_embed.b"])
            K.linear_dw(enc["p16"], d_emb_e, G["patch_embed.w"])

        losses = {"recon": Tensor(rec_loss), "codebook": Tensor(vq_loss), "commitment": Tensor(vq_loss.clone()),
                  "total": Tensor(total, _backward=backward)}
        return (Tensor(recon.view(B, Tm, cfg.height, cfg.width, cfg.channels)),
                (idx.view(B, Tm) if _indices_on_device else idx.view(B, Tm).cpu().numpy()), losses)
