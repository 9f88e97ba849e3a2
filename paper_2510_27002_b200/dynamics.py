"""Decoder-only MaskGIT dynamics model on B200 (mirror of deskworld/dynamics.py).

Same class/function names, config fields, parameter names/shapes and init draw
order as the reference, so weights are identical for the same seed.  The
training loss (dynamics.py:139-153) runs as:

  K6 device Philox masks (bit-exact, host generator advanced past the draws)
  K5 embed + mask token + prepended action token + positions
  ST stack (st.py) -> final LN dropping s=0 -> K1 to_logits GEMM -> K7 masked CE
  and `loss.backward()` replays the hand-scheduled backward.

`decode_frame` / `rollout` keep the reference's MaskGIT semantics (dynamics.py:
156-260); the device sampler lives in sampling.py.
"""
from __future__ import annotations

import enum
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import kernels as K
from .rng import PhiloxState, consume, stream
from .st import StConfig, init_st_stack_arrays, st_backward, st_forward, st_param_groups
from .tensor import ParamStore, Tensor, as_device, embedding, grad_buffers


class ConditioningMode(str, enum.Enum):
    ADDITIVE = "additive"
    PREPEND = "prepend"
    GROUND_TRUTH = "ground_truth_embedding"


@dataclass(frozen=True)
class DynamicsConfig:
    """dynamics.py:33-49."""
    model_dim: int = 512
    heads: int = 8
    ffn_dim: int = 2048
    blocks: int = 6
    token_codes: int = 1024
    action_latent_dim: int = 32
    action_vocab: int = 7
    patches_per_frame: int = 16
    max_frames: int = 16
    mode: ConditioningMode = ConditioningMode.PREPEND
    mask_limit: float = 0.5

    @property
    def st(self) -> StConfig:
        return StConfig(self.model_dim, self.heads, self.ffn_dim, self.blocks)


def sample_masks(rng: np.random.Generator, batch: int, frames: int, patches: int, mask_limit: float = 0.5,
                 return_p: bool = False):
    """Host version, identical to dynamics.py:52-62 (used by callers that want numpy masks)."""
    p = rng.uniform(mask_limit, 1.0, size=batch)
    mask = rng.random((batch, frames, patches)) < p[:, None, None]
    mask[:, 0] = False
    return (mask, p) if return_p else mask


def sample_masks_device(rng: np.random.Generator, batch: int, frames: int, patches: int, mask_limit: float = 0.5,
                        *, shard: tuple[int, int] | None = None):
    """K6: the same masks drawn on the device; `rng` is advanced exactly as sample_masks would.

    shard=(b0, b_local) draws only samples [b0, b0+b_local) of the global batch by
    counter skip-ahead (data parallel).  Returns (mask u8 [b_local, T, N], count int32 device scalar).
    """
    b0, bl = shard if shard is not None else (0, batch)
    st = consume(rng, batch + batch * frames * patches)
    dev = torch.device("cuda", torch.cuda.current_device())
    mask = torch.empty(bl, frames, patches, dtype=torch.uint8, device=dev)
    count = torch.zeros((), dtype=torch.int32, device=dev)
    K.philox_mask(st, batch, b0, bl, frames, patches, mask_limit, mask, count)
    return mask, count


class _LazyStats(dict):
    """{"masked_fraction", "empty_mask"} computed from the device mask on first access."""

    def __init__(self, mask: torch.Tensor, count: torch.Tensor):
        super().__init__()
        self._mask, self._count, self._done = mask, count, False

    def _fill(self):
        if not self._done:
            c = int(self._count)
            super().__setitem__("masked_fraction", c / max(self._mask.numel(), 1))
            super().__setitem__("empty_mask", int(c == 0))
            self._done = True

    def __getitem__(self, k):
        self._fill()
        return super().__getitem__(k)

    def __iter__(self):
        self._fill()
        return super().__iter__()

    def keys(self):
        self._fill()
        return super().keys()

    def items(self):
        self._fill()
        return super().items()

    def get(self, k, default=None):
        self._fill()
        return super().get(k, default)

    def __len__(self):
        return 2


class DynamicsModel:
    def __init__(self, cfg: DynamicsConfig = DynamicsConfig(), seed: int = 0, dtype=np.float32):
        self.cfg = cfg
        self.dtype = dtype
        rng = stream(seed, "dynamics-init")
        d = cfg.model_dim
        p: "OrderedDict[str, np.ndarray]" = OrderedDict()
        p["token_embed"] = rng.normal(0, 0.02, (cfg.token_codes, d)).astype(dtype)
        p["mask_token"] = rng.normal(0, 0.02, (d,)).astype(dtype)
        p["null_action"] = rng.normal(0, 0.02, (cfg.action_latent_dim,)).astype(dtype)
        p["action_proj.w"] = rng.normal(0, 0.02, (cfg.action_latent_dim, d)).astype(dtype)
        p["action_proj.b"] = np.zeros(d, dtype=dtype)
        if cfg.mode is ConditioningMode.GROUND_TRUTH:
            p["gt_action_embed"] = rng.normal(0, 0.02, (cfg.action_vocab, cfg.action_latent_dim)).astype(dtype)
        spatial = cfg.patches_per_frame + (0 if cfg.mode is ConditioningMode.ADDITIVE else 1)
        p["pos_spatial"] = rng.normal(0, 0.02, (spatial, d)).astype(dtype)
        p["pos_temporal"] = rng.normal(0, 0.02, (cfg.max_frames, d)).astype(dtype)
        p.update(init_st_stack_arrays(rng, cfg.st, prefix="dyn", dtype=dtype))
        p["to_logits.w"] = rng.normal(0, 0.02, (d, cfg.token_codes)).astype(dtype)
        p["to_logits.b"] = np.zeros(cfg.token_codes, dtype=dtype)
        self._store = ParamStore(p, groups=st_param_groups(cfg.st, "dyn"))
        self.params = self._store.params

    # -- conditioning (dynamics.py:90-99) -----------------------------------
    def action_latents_for(self, actions, source_codebook=None) -> Tensor:
        if isinstance(actions, Tensor):
            return actions
        if isinstance(actions, torch.Tensor) and actions.is_floating_point():
            return Tensor(actions)
        acts = np.asarray(actions.cpu() if isinstance(actions, torch.Tensor) else actions)
        if self.cfg.mode is ConditioningMode.GROUND_TRUTH:
            table = self.params["gt_action_embed"]
        else:
            if source_codebook is None:
                raise ValueError("latent action indices need the LAM codebook")
            table = source_codebook if isinstance(source_codebook, Tensor) else Tensor(source_codebook)
        if self.cfg.mode is ConditioningMode.GROUND_TRUTH:
            return embedding(table, acts)  # differentiable: trains gt_action_embed (dynamics.py:95-96)
        if acts.size and (acts.min() < 0 or acts.max() >= table.shape[0]):
            raise IndexError(f"embedding ids out of range [0, {table.shape[0]})")
        idx = torch.as_tensor(acts.astype(np.int64), device=table.data.device)
        return Tensor(table.data[idx])

    @property
    def _prepend(self) -> bool:
        return self.cfg.mode is not ConditioningMode.ADDITIVE

    # -- forward -------------------------------------------------------------
    def _check_tokens(self, tokens):
        if isinstance(tokens, torch.Tensor):
            t = tokens.to(torch.device("cuda", torch.cuda.current_device()))
            if t.dtype != torch.int64:
                t = t.long()
            return t.contiguous()
        arr = np.asarray(tokens)
        if arr.ndim != 3:
            raise ValueError(f"tokens must be (B, T, N), got {arr.shape}")
        if arr.size and (arr.min() < 0 or arr.max() >= self.cfg.token_codes):
            raise IndexError(f"embedding ids out of range [0, {self.cfg.token_codes})")
        return as_device(arr.astype(np.int64))

    def _forward(self, tokens, latents: Tensor, mask_d, save: bool):
        cfg = self.cfg
        b, t, n = tuple(tokens.shape)
        if n != cfg.patches_per_frame:
            raise ValueError("token grid width does not match config")
        if latents.shape[1] != t - 1:
            raise ValueError(f"need {t - 1} actions for {t} frames, got {latents.shape[1]}")
        if t > cfg.max_frames:
            raise ValueError(f"clip length {t} exceeds max_frames {cfg.max_frames}")
        P = self.params
        Pd = {k: v for k, v in P.items()}
        tok_d = self._check_tokens(tokens)
        lat_d = latents.data.to(torch.float32).contiguous()
        err = torch.zeros((), dtype=torch.int32, device=tok_d.device)
        prepend = self._prepend
        S = n + (1 if prepend else 0)
        x = K.dyn_embed_fwd(tok_d, mask_d, lat_d, {k: v.data for k, v in Pd.items()}, B=b, T=t, N=n,
                            D=cfg.model_dim, dl=cfg.action_latent_dim, K=cfg.token_codes, prepend=prepend, err=err)
        y, ctx = st_forward(x, P, cfg.st, "dyn", B=b, T=t, S=S, final_skip=prepend, save=save)
        wl = K.cast_bf16(P["to_logits.w"].data)
        logits = K.linear_fwd(y, wl, P["to_logits.b"].data, epilogue=L.EPI_F32)
        return dict(tok=tok_d, lat=lat_d, y=y, ctx=ctx, wl=wl, logits=logits, B=b, T=t, N=n, S=S)

    def logits(self, tokens, action_latents, mask=None) -> Tensor:
        """dynamics.py:121-137 -> Tensor (B, T, N, K) fp32 in HBM."""
        lat = action_latents if isinstance(action_latents, Tensor) else Tensor(action_latents)
        mask_d = None
        if mask is not None:
            mask_d = as_device(np.asarray(mask, dtype=np.uint8)) if not isinstance(mask, torch.Tensor) \
                else mask.to(torch.uint8).contiguous()
        f = self._forward(tokens, lat, mask_d, save=False)
        return Tensor(f["logits"].view(f["B"], f["T"], f["N"], self.cfg.token_codes))

    def loss(self, tokens, actions, rng: np.random.Generator, source_codebook=None, mask=None, *,
             _count=None, _on_grads_done=None):
        """dynamics.py:139-153: (loss Tensor with .backward(), stats).

        Internal keywords (data parallel, dp.py): `_count` overrides the masked-position count
        used for normalisation (the GLOBAL count); `_on_grads_done(name)` is called as each
        gradient bucket ("head", "block{i}", "embed") becomes final during backward.
        """
        cfg = self.cfg
        b, t, n = tuple(np.shape(tokens)) if not isinstance(tokens, torch.Tensor) else tuple(tokens.shape)
        latents = self.action_latents_for(actions, source_codebook)
        if mask is None:
            mask_d, count = sample_masks_device(rng, b, t, n, cfg.mask_limit)
        else:
            if isinstance(mask, torch.Tensor):
                mask_d = mask.to(torch.uint8).contiguous()
            else:
                mask_d = as_device(np.asarray(mask, dtype=np.uint8))
            count = _count if _count is not None else mask_d.sum(dtype=torch.int32)
        if _count is not None:
            count = _count
        stats = _LazyStats(mask_d, count)
        f = self._forward(tokens, latents, mask_d, save=True)
        loss, dlogits = K.ce_fwd_bwd(f["logits"], f["tok"].view(-1), mask_d.view(-1), count)
        f["logits"] = None  # consumed
        P = self.params
        need_lat_grad = latents.requires_grad or latents._backward is not None

        def backward():
            G = grad_buffers(P, self._store)
            K.colsum_bf16(dlogits, G["to_logits.b"])
            K.linear_dw(f["y"], dlogits, G["to_logits.w"])
            dy = K.linear_dx(dlogits, f["wl"], epilogue=L.EPI_F32)
            hook = None
            if _on_grads_done is not None:
                def hook(name):
                    _on_grads_done("head" if name == "head_ln" else name)
            dx = st_backward(f["ctx"], dy, P, G, cfg.st, "dyn", on_done=hook)
            d_lat = torch.empty_like(f["lat"]) if need_lat_grad else None
            K.dyn_embed_bwd(dx, f["tok"], mask_d, f["lat"], {k: v.data for k, v in P.items()}, G,
                            B=f["B"], T=f["T"], N=f["N"], D=cfg.model_dim, dl=cfg.action_latent_dim,
                            K=cfg.token_codes, prepend=self._prepend, d_latents=d_lat)
            if need_lat_grad:
                latents.grad = d_lat.view_as(latents.data)
                if latents._backward is not None:
                    latents.backward()  # e.g. the gt_action_embed scatter (dynamics.py:95-96)
            if _on_grads_done is not None:  # after every write into this model's gradient buffer
                _on_grads_done("embed")

        return Tensor(loss, _backward=backward), stats

    # -- sampling (dynamics.py:156-194) --------------------------------------
    def decode_frame(self, prev_tokens, action_latents, steps: int = 25, temperature: float = 1.0,
                     rng: np.random.Generator | None = None) -> np.ndarray:
        from .sampling import decode_frame
        return decode_frame(self, prev_tokens, action_latents, steps=steps, temperature=temperature, rng=rng)


def rollout(tokenizer, dynamics: DynamicsModel, conditioning_frames, actions, horizon: int, steps: int = 25,
            temperature: float = 1.0, rng=None, source_codebook=None, prefix_action_latents=None):
    """dynamics.py:220-260."""
    from .sampling import rollout as _rollout
    return _rollout(tokenizer, dynamics, conditioning_frames, actions, horizon, steps=steps,
                    temperature=temperature, rng=rng, source_codebook=source_codebook,
                    prefix_action_latents=prefix_action_latents)
