"""VQ-VAE video tokenizer on B200 (mirror of deskworld/tokenizer.py).

Encoder: K9 patchify -> K1 patch_embed GEMM -> (+ spatial/temporal positions) ->
ST stack -> final LN (fp32) -> fp32 to_latent -> K8 VQ (fp32 distances, argmin).
Decoder: fp32 from_latent -> ST stack (no positions, tokenizer.py:128-132) ->
K1 to_pixels GEMM -> unpatchify.  Same config fields, parameter names/shapes and
init draw order as the reference.

The latent projections (512 <-> 32) run as fp32 CUDA-core kernels because their
outputs decide VQ argmins; everything 512-wide runs on tcgen05 in bf16.
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


@dataclass(frozen=True)
class TokenizerConfig:
    """tokenizer.py:21-46."""
    model_dim: int = 512
    heads: int = 8
    ffn_dim: int = 2048
    blocks: int = 4
    codes: int = 1024
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


def frames_to_unit(frames: np.ndarray) -> np.ndarray:
    """uint8 pixels -> f32 in [-1, 1] (tokenizer.py:49-51; host helper)."""
    return (frames.astype(np.float32) / 127.5) - 1.0


def unit_to_frames(unit) -> np.ndarray:
    """tokenizer.py:54-55 (round half-even)."""
    if isinstance(unit, torch.Tensor):
        unit = unit.detach().cpu().numpy()
    return np.clip((unit + 1.0) * 127.5, 0.0, 255.0).round().astype(np.uint8)


# --------------------------------------------------------------------------
# K8 vector quantization (tokenizer.py:58-79)
# --------------------------------------------------------------------------
def vq_quantize(z_e: Tensor, codebook: Tensor):
    """Returns (indices int64 ndarray, z_q_st Tensor, codebook_loss Tensor, commitment_loss Tensor).

    Ties break toward the lowest code index.  Both losses are mean((z_q - z_e)^2); their
    gradients differ (codebook vs encoder) and are produced by vq_backward.
    """
    if codebook.shape[0] == 0:
        raise ValueError("empty codebook")
    if z_e.shape[-1] != codebook.shape[-1]:
        raise ValueError("latent dim mismatch with codebook")
    idx, zq_st, sq = _vq(z_e.data, codebook.data)
    loss = K.sum_scaled(sq, 1.0 / max(z_e.data.numel(), 1))
    lead = tuple(z_e.shape[:-1])
    return (idx.view(lead).cpu().numpy(), Tensor(zq_st.view(z_e.shape)), Tensor(loss), Tensor(loss.clone()))


def _vq(z: torch.Tensor, codebook: torch.Tensor):
    dz = z.shape[-1]
    return K.vq_fwd(z.reshape(-1, dz).contiguous().float(), codebook.contiguous().float())


class _Linear:
    """Weight shadows for the reference's (din, dout) linear layers."""

    @staticmethod
    def bf16(P, name):
        return K.cast_bf16(P[f"{name}.w"].data)


def _check_geometry(cfg, frames_shape):
    b, t, h, w, c = frames_shape
    if (h, w, c) != (cfg.height, cfg.width, cfg.channels):
        raise ValueError(f"frame geometry {(h, w, c)} does not match config")
    if t > cfg.max_frames:
        raise ValueError(f"clip length {t} exceeds max_frames {cfg.max_frames}")


def encoder_forward(P: dict, cfg, frames: torch.Tensor, *, prefix="enc", save=False, final_f32=True,
                    pos=("pos_spatial", "pos_temporal"), embed="patch_embed"):
    """Shared tokenizer/LAM encoder: frames (B,T,H,W,C) u8 or unit f32 -> final-LN output.

    Returns (y, ctx, patches_bf16).  y is (bf16|None, f32) when final_f32.
    """
    B, T = frames.shape[0], frames.shape[1]
    N, D = cfg.patches_per_frame, cfg.model_dim
    p16, _ = K.patchify(frames.reshape(B * T, cfg.height, cfg.width, cfg.channels), cfg.patch)
    emb = K.linear_fwd(p16, _Linear.bf16(P, embed), P[f"{embed}.b"].data, epilogue=L.EPI_F32)
    x = K.assemble_fwd(emb, None, P[pos[0]].data, P[pos[1]].data, B=B, T=T, N=N, D=D, prepend=False)
    y, ctx = st_forward(x, P, cfg.st, prefix, B=B, T=T, S=N, save=save, final_f32=final_f32,
                        final_bf16=not final_f32 or save)
    return y, ctx, p16


class VideoTokenizer:
    def __init__(self, cfg: TokenizerConfig = TokenizerConfig(), seed: int = 0, dtype=np.float32):
        self.cfg = cfg
        self.dtype = dtype
        rng = stream(seed, "tokenizer-init")
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
        p["from_latent.w"] = rng.normal(0, 0.02, (cfg.latent_dim, d)).astype(dtype)
        p["from_latent.b"] = np.zeros(d, dtype=dtype)
        p.update(init_st_stack_arrays(rng, cfg.st, prefix="dec", dtype=dtype))
        p["to_pixels.w"] = rng.normal(0, 0.02, (d, cfg.patch_dim)).astype(dtype)
        p["to_pixels.b"] = np.zeros(cfg.patch_dim, dtype=dtype)
        self._store = ParamStore(p, groups=st_param_groups(cfg.st, "enc") + st_param_groups(cfg.st, "dec"))
        self.params = self._store.params

    # -- device building blocks ---------------------------------------------
    def _frames_device(self, frames) -> torch.Tensor:
        if isinstance(frames, Tensor):
            frames = frames.data
        if isinstance(frames, torch.Tensor):
            t = frames.to(torch.device("cuda", torch.cuda.current_device()))
            return t.contiguous() if t.dtype == torch.uint8 else t.float().contiguous()
        arr = np.asarray(frames)
        return as_device(arr if arr.dtype == np.uint8 else arr.astype(np.float32))

    def encode_latent(self, frames) -> Tensor:
        """tokenizer.py:121-126: z_e (B, T, N, latent_dim)."""
        fr = self._frames_device(frames)
        _check_geometry(self.cfg, tuple(fr.shape))
        B, T = fr.shape[0], fr.shape[1]
        (_, y32), _, _ = encoder_forward(self.params, self.cfg, fr)
        z = K.linear_f32(y32, self.params["to_latent.w"].data, self.params["to_latent.b"].data)
        return Tensor(z.view(B, T, self.cfg.patches_per_frame, self.cfg.latent_dim))

    def decode_latent(self, z_q: Tensor) -> Tensor:
        """tokenizer.py:128-132 (no positional embeddings in the decoder)."""
        cfg = self.cfg
        zq = z_q.data if isinstance(z_q, Tensor) else z_q
        B, T, N = zq.shape[0], zq.shape[1], zq.shape[2]
        P = self.params
        x = K.linear_f32(zq.reshape(-1, cfg.latent_dim).float().contiguous(), P["from_latent.w"].data,
                         P["from_latent.b"].data)
        y, _ = st_forward(x, P, cfg.st, "dec", B=B, T=T, S=N, save=False)
        rp = K.linear_fwd(y, _Linear.bf16(P, "to_pixels"), P["to_pixels.b"].data, epilogue=L.EPI_F32)
        unit, _ = K.unpatchify(rp, B * T, cfg.height, cfg.width, cfg.channels, cfg.patch)
        return Tensor(unit.view(B, T, cfg.height, cfg.width, cfg.channels))

    def forward(self, frames, _indices_on_device: bool = False):
        """tokenizer.py:134-143: (recon, indices, {"recon","codebook","commitment","total"}).

        `_indices_on_device` (internal, training stages): indices stay a device tensor, so the step
        has no host synchronisation (the reference API returns a numpy array).

        losses["total"].backward() runs the full training backward (trainer.py:211-223): recon MSE
        through to_pixels and the decoder stack, from_latent, the VQ straight-through estimator
        plus the commitment (beta) and codebook terms, to_latent, the encoder stack and the
        patch / positional embeddings; gradients land in p.grad.
        """
        cfg, P = self.cfg, self.params
        fr = self._frames_device(frames)
        _check_geometry(cfg, tuple(fr.shape))
        B, T = fr.shape[0], fr.shape[1]
        N, D, dl = cfg.patches_per_frame, cfg.model_dim, cfg.latent_dim
        # encoder (tokenizer.py:113-126)
        p16, p32 = K.patchify(fr.reshape(B * T, cfg.height, cfg.width, cfg.channels), cfg.patch, f32=True)
        w_pe = K.cast_bf16(P["patch_embed.w"].data)
        emb = K.linear_fwd(p16, w_pe, P["patch_embed.b"].data, epilogue=L.EPI_F32)
        x = K.assemble_fwd(emb, None, P["pos_spatial"].data, P["pos_temporal"].data, B=B, T=T, N=N, D=D,
                           prepend=False)
        (_, y32), ectx = st_forward(x, P, cfg.st, "enc", B=B, T=T, S=N, save=True, final_f32=True, final_bf16=False)
        z_e = K.linear_f32(y32, P["to_latent.w"].data, P["to_latent.b"].data)
        # VQ (tokenizer.py:58-79)
        idx, zq_st, sq = _vq(z_e, P["codebook"].data)
        numel_z = z_e.numel()
        vq_loss = K.sum_scaled(sq, 1.0 / numel_z)
        # decoder (tokenizer.py:128-132, no positional embeddings)
        xd = K.linear_f32(zq_st, P["from_latent.w"].data, P["from_latent.b"].data)
        yd, dctx = st_forward(xd, P, cfg.st, "dec", B=B, T=T, S=N, save=True)
        w_tp = K.cast_bf16(P["to_pixels.w"].data)
        rp = K.linear_fwd(yd, w_tp, P["to_pixels.b"].data, epilogue=L.EPI_F32)
        rec_loss, _, g16 = K.mse(rp, p32, grad16=True)
        total = rec_loss + vq_loss + cfg.commitment_beta * vq_loss
        recon, _ = K.unpatchify(rp, B * T, cfg.height, cfg.width, cfg.channels, cfg.patch)
        store = self._store

        def backward():
            G = grad_buffers(P, store)
            K.colsum_bf16(g16, G["to_pixels.b"])
            K.linear_dw(yd, g16, G["to_pixels.w"])
            dy = K.linear_dx(g16, w_tp, epilogue=L.EPI_F32)
            dxd = st_backward(dctx, dy, P, G, cfg.st, "dec")
            d_zq = torch.empty(B * T * N, dl, dtype=K.F32, device=dxd.device)
            K.linear_f32_bwd(zq_st, dxd, P["from_latent.w"].data, dx=d_zq, dW=G["from_latent.w"],
                             db=G["from_latent.b"])
            # straight-through to z_e, + beta * d commitment; codebook term into the codebook
            d_ze = torch.empty_like(z_e)
            K.vq_bwd(z_e, P["codebook"].data, idx, d_zq, commit_coef=cfg.commitment_beta * 2.0 / numel_z,
                     cb_coef=2.0 / numel_z, dz_out=d_ze, dcodebook=G["codebook"])
            d_y = torch.empty(B * T * N, D, dtype=K.F32, device=dxd.device)
            K.linear_f32_bwd(y32, d_ze, P["to_latent.w"].data, dx=d_y, dW=G["to_latent.w"], db=G["to_latent.b"])
            dxe = st_backward(ectx, d_y, P, G, cfg.st, "enc")
            d_emb = torch.empty(B * T * N, D, dtype=K.BF16, device=dxd.device)
            K.assemble_bwd(dxe, B=B, T=T, N=N, D=D, prepend=False, d_emb=d_emb, d_ps=G["pos_spatial"],
                           d_pt=G["pos_temporal"][:T])
            if T < cfg.max_frames:
                G["pos_temporal"][T:].zero_()
            K.colsum_bf16(d_emb, G["patch_embed.b"])
            K.linear_dw(p16, d_emb, G["patch_embed.w"])

        losses = {"recon": Tensor(rec_loss), "codebook": Tensor(vq_loss), "commitment": Tensor(vq_loss.clone()),
                  "total": Tensor(total, _backward=backward)}
        idx_out = idx.view(B, T, N) if _indices_on_device else idx.view(B, T, N).cpu().numpy()
        return (Tensor(recon.view(B, T, cfg.height, cfg.width, cfg.channels)), idx_out,
                losses)

    def encode_device(self, frames) -> torch.Tensor:
        """(B, T, N) int64 token grid in HBM."""
        z = self.encode_latent(frames)
        idx, _, _ = _vq(z.data, self.params["codebook"].data)
        return idx.view(tuple(z.shape[:-1]))

    def encode(self, frames) -> np.ndarray:
        """tokenizer.py:145-150: uint8 or unit-range frames -> (B, T, N) token grid (numpy)."""
        return self.encode_device(frames).cpu().numpy()

    def decode_device(self, tokens: torch.Tensor) -> torch.Tensor:
        z_q = self.params["codebook"].data[tokens.long()]
        return self.decode_latent(Tensor(z_q)).data

    def decode(self, tokens) -> np.ndarray:
        """tokenizer.py:152-158: (B, T, N) tokens -> unit-range frames (numpy)."""
        arr = tokens.cpu().numpy() if isinstance(tokens, torch.Tensor) else np.asarray(tokens)
        if arr.max(initial=0) >= self.cfg.codes or arr.min(initial=0) < 0:
            raise IndexError(f"token index outside [0, {self.cfg.codes})")
        return self.decode_device(as_device(arr.astype(np.int64))).cpu().numpy()
