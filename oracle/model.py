"""ORACLE (test infrastructure only) — torch-CPU restatement of the deskworld models.

Every function cites the reference file:line it restates.  Parameters are
dict[str, torch.Tensor] with the reference's names and shapes;
gradients come from torch.autograd, in the dtype of the parameters (float64 to
pin against the reference's golden vectors, float32 as the parity oracle of the
B200 product).  Initialisation consumes the reference's numpy Philox streams in
the reference's draw order, so weights are identical by construction.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import rng as orng

# --------------------------------------------------------------------------
# configs (same fields/defaults as the reference dataclasses)
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class StCfg:  # st.py:20-31
    model_dim: int = 512
    heads: int = 8
    ffn_dim: int = 2048
    blocks: int = 4


@dataclass(frozen=True)
class TokCfg:  # tokenizer.py:21-46
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
    def patches_per_frame(self):
        return (self.height // self.patch) * (self.width // self.patch)

    @property
    def patch_dim(self):
        return self.patch * self.patch * self.channels

    @property
    def st(self):
        return StCfg(self.model_dim, self.heads, self.ffn_dim, self.blocks)


LamCfg = TokCfg  # lam.py:22-47 has the same fields (codes default 6)


@dataclass(frozen=True)
class DynCfg:  # dynamics.py:33-49
    model_dim: int = 512
    heads: int = 8
    ffn_dim: int = 2048
    blocks: int = 6
    token_codes: int = 1024
    action_latent_dim: int = 32
    action_vocab: int = 7
    patches_per_frame: int = 16
    max_frames: int = 16
    mode: str = "prepend"
    mask_limit: float = 0.5

    @property
    def st(self):
        return StCfg(self.model_dim, self.heads, self.ffn_dim, self.blocks)


# --------------------------------------------------------------------------
# nn ops (deskworld/nn.py)
# --------------------------------------------------------------------------

def softmax(x, dim=-1):  # nn.py:17-20 (max detached)
    shifted = x - x.detach().amax(dim=dim, keepdim=True)
    e = shifted.exp()
    return e / e.sum(dim=dim, keepdim=True)


def log_softmax(x, dim=-1):  # nn.py:23-25
    shifted = x - x.detach().amax(dim=dim, keepdim=True)
    return shifted - shifted.exp().sum(dim=dim, keepdim=True).log()


def gelu(x):  # nn.py:28-32 (tanh approximation)
    c = math.sqrt(2.0 / math.pi)
    inner = (x + 0.044715 * (x * x * x)) * c
    return 0.5 * (x * (1.0 + inner.tanh()))


def layer_norm(x, g, b, eps=1e-5):  # nn.py:35-40 (biased var, two-pass)
    mu = x.mean(dim=-1, keepdim=True)
    c = x - mu
    var = (c * c).mean(dim=-1, keepdim=True)
    return c / (var + eps).sqrt() * g + b


def linear(x, w, b=None):  # nn.py:43-47, W is (din, dout)
    y = x @ w
    return y if b is None else y + b


def mse(pred, target):  # nn.py:50-53
    d = pred - target
    return (d * d).mean()


def softmax_cross_entropy(logits, targets, weights=None):  # nn.py:56-77
    k = logits.shape[-1]
    if k < 2:
        raise ValueError("need at least 2 classes")
    t = torch.as_tensor(np.asarray(targets), dtype=torch.long)
    if t.numel() and int(t.max()) >= k:
        raise IndexError(f"target id >= number of classes ({k})")
    logp = log_softmax(logits)
    nll = -logp.gather(-1, t[..., None])[..., 0]
    if weights is None:
        return nll.mean()
    w = torch.as_tensor(np.asarray(weights), dtype=logits.dtype)
    total = float(w.sum())
    if total == 0.0:
        return torch.zeros((), dtype=logits.dtype)
    return (nll * w).sum() / total


def multi_head_attention(q, k, v, heads, causal=False):  # nn.py:80-110
    *lead, L, D = q.shape
    hd = D // heads

    def split(x):
        return x.reshape(*lead, L, heads, hd).transpose(-3, -2)

    qh, kh, vh = split(q), split(k), split(v)
    s = (qh @ kh.transpose(-1, -2)) * (1.0 / math.sqrt(hd))
    if causal:
        m = torch.triu(torch.ones(L, L, dtype=torch.bool), diagonal=1)
        s = s + torch.where(m, torch.tensor(-1e9, dtype=s.dtype), torch.tensor(0.0, dtype=s.dtype))
    out = softmax(s) @ vh
    return out.transpose(-3, -2).reshape(*lead, L, D)


def patchify(frames, patch):  # nn.py:113-121, order (gh, gw, ph, pw, c)
    b, t, h, w, c = frames.shape
    gh, gw = h // patch, w // patch
    x = frames.reshape(b, t, gh, patch, gw, patch, c).permute(0, 1, 2, 4, 3, 5, 6)
    return x.reshape(b, t, gh * gw, patch * patch * c)


def unpatchify(p, patch, h, w, c=3):  # nn.py:124-131
    b, t, n, d = p.shape
    gh, gw = h // patch, w // patch
    x = p.reshape(b, t, gh, gw, patch, patch, c).permute(0, 1, 2, 4, 3, 5, 6)
    return x.reshape(b, t, h, w, c)


def frames_to_unit(frames: np.ndarray) -> np.ndarray:  # tokenizer.py:49-51
    return (frames.astype(np.float32) / 127.5) - 1.0


def unit_to_frames(unit: np.ndarray) -> np.ndarray:  # tokenizer.py:54-55 (round half-even)
    return np.clip((unit + 1.0) * 127.5, 0.0, 255.0).round().astype(np.uint8)


# --------------------------------------------------------------------------
# ST backbone (deskworld/st.py)
# --------------------------------------------------------------------------

def init_st_stack(gen, cfg: StCfg, prefix: str, dtype=np.float32) -> dict:  # st.py:44-57
    p = {}
    d, f = cfg.model_dim, cfg.ffn_dim

    def lin(name, din, dout):
        p[f"{name}.w"] = gen.normal(0.0, 0.02, size=(din, dout)).astype(dtype)
        p[f"{name}.b"] = np.zeros(dout, dtype=dtype)

    def ln(name, dim):
        p[f"{name}.g"] = np.ones(dim, dtype=dtype)
        p[f"{name}.b"] = np.zeros(dim, dtype=dtype)

    for i in range(cfg.blocks):
        base = f"{prefix}.block{i}"
        for sub in ("spatial", "temporal"):
            ln(f"{base}.{sub}.ln", d)
            for proj in ("q", "k", "v", "o"):
                lin(f"{base}.{sub}.{proj}", d, d)
        ln(f"{base}.ffn.ln", d)
        lin(f"{base}.ffn.up", d, f)
        lin(f"{base}.ffn.down", f, d)
    ln(f"{prefix}.final_ln", d)
    return p


def _attend(x, P, base, heads, causal):  # st.py:60-66
    n = layer_norm(x, P[f"{base}.ln.g"], P[f"{base}.ln.b"])
    q = linear(n, P[f"{base}.q.w"], P[f"{base}.q.b"])
    k = linear(n, P[f"{base}.k.w"], P[f"{base}.k.b"])
    v = linear(n, P[f"{base}.v.w"], P[f"{base}.v.b"])
    return linear(multi_head_attention(q, k, v, heads, causal), P[f"{base}.o.w"], P[f"{base}.o.b"])


def st_block(x, P, cfg: StCfg, i: int, prefix: str):  # st.py:69-79
    if x.ndim != 4:
        raise ValueError(f"expected (B, T, S, D), got shape {tuple(x.shape)}")
    base = f"{prefix}.block{i}"
    x = x + _attend(x, P, f"{base}.spatial", cfg.heads, False)
    xt = x.transpose(1, 2)
    xt = xt + _attend(xt, P, f"{base}.temporal", cfg.heads, True)
    x = xt.transpose(1, 2)
    n = layer_norm(x, P[f"{base}.ffn.ln.g"], P[f"{base}.ffn.ln.b"])
    h = gelu(linear(n, P[f"{base}.ffn.up.w"], P[f"{base}.ffn.up.b"]))
    return x + linear(h, P[f"{base}.ffn.down.w"], P[f"{base}.ffn.down.b"])


def st_stack(x, P, cfg: StCfg, prefix: str):  # st.py:82-85
    for i in range(cfg.blocks):
        x = st_block(x, P, cfg, i, prefix)
    return layer_norm(x, P[f"{prefix}.final_ln.g"], P[f"{prefix}.final_ln.b"])


# --------------------------------------------------------------------------
# VQ (tokenizer.py:58-79)
# --------------------------------------------------------------------------

def vq_distances(flat: np.ndarray, codebook: np.ndarray) -> np.ndarray:
    """d2 = (|z|^2 - (2z).C^T) + |c|^2 in the array dtype (tokenizer.py:69-71)."""
    return (np.sum(flat ** 2, axis=1, keepdims=True) - 2.0 * flat @ codebook.T
            + np.sum(codebook ** 2, axis=1))


def vq_quantize(z_e, codebook):
    """Returns (indices int64 ndarray, z_q_st, codebook_loss, commitment_loss)."""
    if codebook.shape[0] == 0:
        raise ValueError("empty codebook")
    if z_e.shape[-1] != codebook.shape[-1]:
        raise ValueError("latent dim mismatch with codebook")
    flat = z_e.detach().reshape(-1, z_e.shape[-1]).numpy()
    d2 = vq_distances(flat, codebook.detach().numpy())
    idx = np.argmin(d2, axis=1).reshape(tuple(z_e.shape[:-1]))
    z_q = codebook[torch.as_tensor(idx)]
    cb = mse(z_q, z_e.detach())
    commit = mse(z_e, z_q.detach())
    z_q_st = z_e + (z_q.detach() - z_e.detach())
    return idx, z_q_st, cb, commit


# --------------------------------------------------------------------------
# models
# --------------------------------------------------------------------------

def _as_params(np_params: dict, requires_grad=True) -> dict:
    return {k: torch.tensor(v, requires_grad=requires_grad) for k, v in np_params.items()}


def init_tokenizer(cfg: TokCfg, seed=0, dtype=np.float32) -> dict:  # tokenizer.py:83-104
    g = orng.stream(seed, "tokenizer-init")
    d = cfg.model_dim
    p = {}
    p["patch_embed.w"] = g.normal(0, 0.02, (cfg.patch_dim, d)).astype(dtype)
    p["patch_embed.b"] = np.zeros(d, dtype=dtype)
    p["pos_spatial"] = g.normal(0, 0.02, (cfg.patches_per_frame, d)).astype(dtype)
    p["pos_temporal"] = g.normal(0, 0.02, (cfg.max_frames, d)).astype(dtype)
    p.update(init_st_stack(g, cfg.st, "enc", dtype))
    p["to_latent.w"] = g.normal(0, 0.02, (d, cfg.latent_dim)).astype(dtype)
    p["to_latent.b"] = np.zeros(cfg.latent_dim, dtype=dtype)
    bound = 1.0 / cfg.codes
    p["codebook"] = g.uniform(-bound, bound, (cfg.codes, cfg.latent_dim)).astype(dtype)
    p["from_latent.w"] = g.normal(0, 0.02, (cfg.latent_dim, d)).astype(dtype)
    p["from_latent.b"] = np.zeros(d, dtype=dtype)
    p.update(init_st_stack(g, cfg.st, "dec", dtype))
    p["to_pixels.w"] = g.normal(0, 0.02, (d, cfg.patch_dim)).astype(dtype)
    p["to_pixels.b"] = np.zeros(cfg.patch_dim, dtype=dtype)
    return p


def tok_encode_latent(P, cfg: TokCfg, unit):  # tokenizer.py:113-126
    t = unit.shape[1]
    x = linear(patchify(unit, cfg.patch), P["patch_embed.w"], P["patch_embed.b"])
    x = x + P["pos_spatial"]
    x = x + P["pos_temporal"][:t].reshape(1, t, 1, cfg.model_dim)
    x = st_stack(x, P, cfg.st, "enc")
    return linear(x, P["to_latent.w"], P["to_latent.b"])


def tok_decode_latent(P, cfg: TokCfg, z_q):  # tokenizer.py:128-132 (no positions)
    x = linear(z_q, P["from_latent.w"], P["from_latent.b"])
    x = st_stack(x, P, cfg.st, "dec")
    x = linear(x, P["to_pixels.w"], P["to_pixels.b"])
    return unpatchify(x, cfg.patch, cfg.height, cfg.width, cfg.channels)


def tok_forward(P, cfg: TokCfg, unit):  # tokenizer.py:134-143
    z_e = tok_encode_latent(P, cfg, unit)
    idx, z_q, cb, commit = vq_quantize(z_e, P["codebook"])
    recon = tok_decode_latent(P, cfg, z_q)
    rec = mse(recon, unit.detach())
    total = rec + cb + cfg.commitment_beta * commit
    return recon, idx, {"recon": rec, "codebook": cb, "commitment": commit, "total": total}


def tok_encode(P, cfg: TokCfg, frames: np.ndarray, dtype=torch.float32) -> np.ndarray:  # :145-150
    unit = frames_to_unit(frames) if frames.dtype == np.uint8 else frames
    with torch.no_grad():
        z_e = tok_encode_latent(P, cfg, torch.as_tensor(np.asarray(unit)).to(dtype))
        idx, _, _, _ = vq_quantize(z_e, P["codebook"])
    return idx


def tok_decode(P, cfg: TokCfg, tokens: np.ndarray) -> np.ndarray:  # :152-158
    if tokens.max(initial=0) >= cfg.codes or tokens.min(initial=0) < 0:
        raise IndexError(f"token index outside [0, {cfg.codes})")
    with torch.no_grad():
        z_q = P["codebook"][torch.as_tensor(tokens)]
        return tok_decode_latent(P, cfg, z_q).numpy()


def init_lam(cfg: LamCfg, seed=0, dtype=np.float32) -> dict:  # lam.py:50-76
    g = orng.stream(seed, "lam-init")
    d = cfg.model_dim
    p = {}
    p["patch_embed.w"] = g.normal(0, 0.02, (cfg.patch_dim, d)).astype(dtype)
    p["patch_embed.b"] = np.zeros(d, dtype=dtype)
    p["pos_spatial"] = g.normal(0, 0.02, (cfg.patches_per_frame, d)).astype(dtype)
    p["pos_temporal"] = g.normal(0, 0.02, (cfg.max_frames, d)).astype(dtype)
    p.update(init_st_stack(g, cfg.st, "enc", dtype))
    p["to_latent.w"] = g.normal(0, 0.02, (d, cfg.latent_dim)).astype(dtype)
    p["to_latent.b"] = np.zeros(cfg.latent_dim, dtype=dtype)
    bound = 1.0 / cfg.codes
    p["codebook"] = g.uniform(-bound, bound, (cfg.codes, cfg.latent_dim)).astype(dtype)
    p["dec_embed.w"] = g.normal(0, 0.02, (cfg.patch_dim, d)).astype(dtype)
    p["dec_embed.b"] = np.zeros(d, dtype=dtype)
    p["action_proj.w"] = g.normal(0, 0.02, (cfg.latent_dim, d)).astype(dtype)
    p["action_proj.b"] = np.zeros(d, dtype=dtype)
    p["dec_pos_spatial"] = g.normal(0, 0.02, (cfg.patches_per_frame + 1, d)).astype(dtype)
    p["dec_pos_temporal"] = g.normal(0, 0.02, (cfg.max_frames, d)).astype(dtype)
    p.update(init_st_stack(g, cfg.st, "dec", dtype))
    p["to_pixels.w"] = g.normal(0, 0.02, (d, cfg.patch_dim)).astype(dtype)
    p["to_pixels.b"] = np.zeros(cfg.patch_dim, dtype=dtype)
    return p


def lam_encode_pre_vq(P, cfg: LamCfg, unit):  # lam.py:79-94
    b, t = unit.shape[0], unit.shape[1]
    if t < 2:
        raise ValueError("need at least 2 frames to infer actions")
    d = cfg.model_dim
    x = linear(patchify(unit, cfg.patch), P["patch_embed.w"], P["patch_embed.b"])
    x = x + P["pos_spatial"]
    x = x + P["pos_temporal"][:t].reshape(1, t, 1, d)
    x = st_stack(x, P, cfg.st, "enc")
    pooled = x.mean(dim=2)
    return linear(pooled[:, 1:], P["to_latent.w"], P["to_latent.b"])


def lam_encoder_only(P, cfg: LamCfg, unit):  # lam.py:96-101
    return vq_quantize(lam_encode_pre_vq(P, cfg, unit), P["codebook"])


def lam_decode(P, cfg: LamCfg, past, latents):  # lam.py:104-118
    b, tm1 = past.shape[0], past.shape[1]
    d = cfg.model_dim
    x = linear(patchify(past, cfg.patch), P["dec_embed.w"], P["dec_embed.b"])
    act = linear(latents, P["action_proj.w"], P["action_proj.b"])
    x = torch.cat([act.reshape(b, tm1, 1, d), x], dim=2)
    x = x + P["dec_pos_spatial"]
    x = x + P["dec_pos_temporal"][:tm1].reshape(1, tm1, 1, d)
    x = st_stack(x, P, cfg.st, "dec")
    x = linear(x[:, :, 1:], P["to_pixels.w"], P["to_pixels.b"])
    return unpatchify(x, cfg.patch, cfg.height, cfg.width, cfg.channels)


def lam_forward(P, cfg: LamCfg, unit):  # lam.py:120-129
    idx, z_q, cb, commit = lam_encoder_only(P, cfg, unit)
    recon = lam_decode(P, cfg, unit[:, :-1], z_q)
    rec = mse(recon, unit.detach()[:, 1:])
    total = rec + cb + cfg.commitment_beta * commit
    return recon, idx, {"recon": rec, "codebook": cb, "commitment": commit, "total": total}


def lam_forward_with_indices(P, cfg: LamCfg, unit, idx):
    """lam.py:120-129 with the code indices given (the VQ argmin replaced by `idx`; the losses and
    the straight-through estimator exactly as vq_quantize forms them, tokenizer.py:58-79)."""
    z_e = lam_encode_pre_vq(P, cfg, unit)
    z_q = P["codebook"][torch.as_tensor(np.asarray(idx))]
    cb, commit = mse(z_q, z_e.detach()), mse(z_e, z_q.detach())
    z_q_st = z_e + (z_q.detach() - z_e.detach())
    recon = lam_decode(P, cfg, unit[:, :-1], z_q_st)
    rec = mse(recon, unit.detach()[:, 1:])
    total = rec + cb + cfg.commitment_beta * commit
    return recon, z_e, {"recon": rec, "codebook": cb, "commitment": commit, "total": total}


def vq_mismatch_explained(z_dev, z_ref, codebook, idx_dev, idx_ref) -> int:
    """Number of code mismatches NOT explained by the latent difference: with z' = z + e,
    |z'-c|^2 - |z-c|^2 = 2 e.(z - c) + |e|^2, so a flip from c_r to c_o needs
    |z-c_o|^2 - |z-c_r|^2 <= 2 |e| (|z-c_o| + |z-c_r|) + 2 |e|^2."""
    zd = np.asarray(z_dev, dtype=np.float64).reshape(-1, np.shape(codebook)[-1])
    zr = np.asarray(z_ref, dtype=np.float64).reshape(zd.shape)
    cb = np.asarray(codebook, dtype=np.float64)
    io, ir = np.asarray(idx_dev).reshape(-1), np.asarray(idx_ref).reshape(-1)
    bad = 0
    for r in np.nonzero(io != ir)[0]:
        e = np.linalg.norm(zd[r] - zr[r])
        do, dr = np.linalg.norm(zr[r] - cb[io[r]]), np.linalg.norm(zr[r] - cb[ir[r]])
        if do ** 2 - dr ** 2 > 2 * e * (do + dr) + 2 * e ** 2:
            bad += 1
    return bad


def init_dynamics(cfg: DynCfg, seed=0, dtype=np.float32) -> dict:  # dynamics.py:66-87
    g = orng.stream(seed, "dynamics-init")
    d = cfg.model_dim
    p = {}
    p["token_embed"] = g.normal(0, 0.02, (cfg.token_codes, d)).astype(dtype)
    p["mask_token"] = g.normal(0, 0.02, (d,)).astype(dtype)
    p["null_action"] = g.normal(0, 0.02, (cfg.action_latent_dim,)).astype(dtype)
    p["action_proj.w"] = g.normal(0, 0.02, (cfg.action_latent_dim, d)).astype(dtype)
    p["action_proj.b"] = np.zeros(d, dtype=dtype)
    if cfg.mode == "ground_truth_embedding":
        p["gt_action_embed"] = g.normal(0, 0.02, (cfg.action_vocab, cfg.action_latent_dim)).astype(dtype)
    spatial = cfg.patches_per_frame + (0 if cfg.mode == "additive" else 1)
    p["pos_spatial"] = g.normal(0, 0.02, (spatial, d)).astype(dtype)
    p["pos_temporal"] = g.normal(0, 0.02, (cfg.max_frames, d)).astype(dtype)
    p.update(init_st_stack(g, cfg.st, "dyn", dtype))
    p["to_logits.w"] = g.normal(0, 0.02, (d, cfg.token_codes)).astype(dtype)
    p["to_logits.b"] = np.zeros(cfg.token_codes, dtype=dtype)
    return p


def dyn_embed_actions(P, cfg: DynCfg, latents, x):  # dynamics.py:101-118
    b, t, n, d = x.shape
    if latents.shape[1] != t - 1:
        raise ValueError(f"need {t - 1} actions for {t} frames, got {latents.shape[1]}")
    null = P["null_action"].reshape(1, 1, -1).expand(b, 1, -1)
    cond = torch.cat([null, latents], dim=1)
    act = linear(cond, P["action_proj.w"], P["action_proj.b"])
    if cfg.mode == "additive":
        return x + act.reshape(b, t, 1, d)
    return torch.cat([act.reshape(b, t, 1, d), x], dim=2)


def dyn_logits(P, cfg: DynCfg, tokens: np.ndarray, latents, mask=None):  # dynamics.py:121-137
    b, t, n = tokens.shape
    if n != cfg.patches_per_frame:
        raise ValueError("token grid width does not match config")
    tok = torch.as_tensor(np.asarray(tokens), dtype=torch.long)
    if tok.numel() and (int(tok.min()) < 0 or int(tok.max()) >= cfg.token_codes):
        raise IndexError("embedding ids out of range")
    d = cfg.model_dim
    x = P["token_embed"][tok]
    if mask is not None:
        m = torch.as_tensor(np.asarray(mask, dtype=bool))[..., None]
        x = torch.where(m, P["mask_token"].expand_as(x), x)
    x = dyn_embed_actions(P, cfg, latents, x)
    x = x + P["pos_spatial"][: x.shape[2]]
    x = x + P["pos_temporal"][:t].reshape(1, t, 1, d)
    x = st_stack(x, P, cfg.st, "dyn")
    if cfg.mode != "additive":
        x = x[:, :, 1:]
    return linear(x, P["to_logits.w"], P["to_logits.b"])


def dyn_loss(P, cfg: DynCfg, tokens, latents, mask):  # dynamics.py:139-153 (mask given)
    stats = {"masked_fraction": float(np.mean(mask)), "empty_mask": int(np.sum(mask) == 0)}
    if np.sum(mask) == 0:
        return torch.zeros((), dtype=P["token_embed"].dtype), stats
    logits = dyn_logits(P, cfg, tokens, latents, mask)
    return softmax_cross_entropy(logits, tokens, weights=np.asarray(mask, dtype=np.float64)), stats


# --------------------------------------------------------------------------
# MaskGIT sampling (dynamics.py:156-217) and rollout (dynamics.py:220-260)
# --------------------------------------------------------------------------

def sample_with_confidence(logits: np.ndarray, temperature: float, gen: np.random.Generator):
    """dynamics.py:198-217 (numpy, dtype of `logits`)."""
    scaled = logits / max(temperature, 1e-8)
    scaled = scaled - scaled.max(axis=-1, keepdims=True)
    probs = np.exp(scaled)
    probs /= probs.sum(axis=-1, keepdims=True)
    if temperature < 1e-6:
        sampled = np.argmax(logits, axis=-1)
    else:
        cdf = np.cumsum(probs, axis=-1)
        u = gen.random(logits.shape[:-1] + (1,))
        sampled = (u > cdf).sum(axis=-1)
        sampled = np.minimum(sampled, logits.shape[-1] - 1)
    conf = np.take_along_axis(probs, sampled[..., None], axis=-1)[..., 0]
    return sampled.astype(np.int64), conf


def decode_frame(logits_fn, prev_tokens: np.ndarray, latents, steps=25, temperature=1.0, gen=None):
    """dynamics.py:156-194; logits_fn(tokens, latents, mask) -> (B,T,N,K) ndarray."""
    if steps < 1:
        raise ValueError("steps must be >= 1")
    if gen is None:
        gen = orng.stream(0, "maskgit-decode")
    b, t_prev, n = prev_tokens.shape
    if latents.shape[1] != t_prev:
        raise ValueError(f"need {t_prev} action latents, got {latents.shape[1]}")
    tokens = np.concatenate([prev_tokens, np.zeros((b, 1, n), dtype=prev_tokens.dtype)], axis=1)
    known = np.zeros((b, n), dtype=bool)
    cur = np.zeros((b, n), dtype=prev_tokens.dtype)
    for s in range(1, steps + 1):
        frac = np.cos(np.pi / 2 * s / steps)
        n_keep = n if s == steps else min(n, int(np.ceil(n * (1.0 - frac))))
        n_keep = max(n_keep, int(known[0].sum()))
        tokens[:, -1] = cur
        mask = np.zeros_like(tokens, dtype=bool)
        mask[:, -1] = ~known
        logits = logits_fn(tokens, latents, mask)[:, -1]
        sampled, conf = sample_with_confidence(logits, temperature, gen)
        cur = np.where(known, cur, sampled)
        conf = np.where(known, np.inf, conf)
        order = np.lexsort((np.broadcast_to(np.arange(n), conf.shape), -conf), axis=-1)
        new_known = np.zeros_like(known)
        np.put_along_axis(new_known, order[:, :n_keep], True, axis=-1)
        known = new_known
    return cur


def rollout(tok_P, tok_cfg, dyn_P, dyn_cfg, cond_frames, actions, horizon, steps=25,
            temperature=1.0, gen=None, source_codebook=None, dtype=torch.float32):
    """dynamics.py:220-260 with index actions through `source_codebook` (or gt table)."""
    if len(actions) < horizon:
        raise ValueError(f"need {horizon} actions, got {len(actions)}")
    n_cond = cond_frames.shape[1]
    if n_cond + horizon > dyn_cfg.max_frames:
        raise ValueError("horizon exceeds the model's maximum clip length")
    if gen is None:
        gen = orng.stream(0, "rollout")
    tokens = tok_encode(tok_P, tok_cfg, cond_frames, dtype)
    b = tokens.shape[0]
    dlat = dyn_cfg.action_latent_dim
    with torch.no_grad():
        null = dyn_P["null_action"].detach().reshape(1, 1, dlat)
        history = torch.zeros((b, n_cond - 1, dlat), dtype=dyn_P["null_action"].dtype) + null

        def logits_fn(tk, lat, mask):
            return dyn_logits(dyn_P, dyn_cfg, tk, lat, mask).numpy()

        for step in range(horizon):
            a = np.asarray(actions[step]).reshape(b, 1)
            table = dyn_P["gt_action_embed"] if dyn_cfg.mode == "ground_truth_embedding" else source_codebook
            lat = table[torch.as_tensor(a)]
            history = torch.cat([history, lat], dim=1)
            nxt = decode_frame(logits_fn, tokens, history, steps, temperature, gen)
            tokens = np.concatenate([tokens, nxt[:, None, :]], axis=1)
    return unit_to_frames(tok_decode(tok_P, tok_cfg, tokens))


# --------------------------------------------------------------------------
# optimizer (optim.py)
# --------------------------------------------------------------------------

@dataclass
class AdamState:  # optim.py:14-22
    m: dict = field(default_factory=dict)
    v: dict = field(default_factory=dict)
    t: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0


def adamw_init(params: dict) -> AdamState:  # optim.py:25-31
    st = AdamState()
    for n, p in params.items():
        st.m[n] = np.zeros_like(p)
        st.v[n] = np.zeros_like(p)
    return st


def adamw_step(params: dict, grads: dict, st: AdamState, lr: float) -> None:  # optim.py:34-62
    """numpy arrays, updated in place, sorted-name order, NEP-50 scalar casting."""
    st.t += 1
    t = st.t
    b1, b2 = st.beta1, st.beta2
    for name in sorted(params):
        p, g = params[name], grads[name]
        if g is None:
            continue
        if not np.all(np.isfinite(g)):
            raise FloatingPointError(f"non-finite gradient in parameter {name!r}")
        m, v = st.m[name], st.v[name]
        m *= b1
        m += (1.0 - b1) * g
        v *= b2
        v += (1.0 - b2) * (g * g)
        m_hat = m / (1.0 - b1 ** t)
        v_hat = v / (1.0 - b2 ** t)
        p -= (lr * (m_hat / (np.sqrt(v_hat) + st.eps))).astype(p.dtype)
        if st.weight_decay:
            p -= (lr * st.weight_decay) * p


def wsd_lr(peak_lr, total_steps, warmup_steps, decay_fraction, step) -> float:  # optim.py:76-89
    decay_steps = int(round(decay_fraction * total_steps))
    decay_start = total_steps - decay_steps
    if step <= 0 or step >= total_steps:
        return 0.0
    if step < warmup_steps:
        return peak_lr * step / warmup_steps
    if step <= decay_start or decay_steps == 0:
        return peak_lr
    return peak_lr * (total_steps - step) / decay_steps


def params_to_torch(np_params: dict, requires_grad=True) -> dict:
    return _as_params(np_params, requires_grad)


# --------------------------------------------------------------------------
# ST-DiT diffusion-forcing dynamics (diffusion.py:114-215): test oracle only
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class DitCfg:  # diffusion.py:114-128
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
    def st(self) -> StCfg:
        return StCfg(self.model_dim, self.heads, self.ffn_dim, self.blocks)


def sinusoidal_embedding(values, dim: int) -> np.ndarray:  # nn.py:134-142 (float32 throughout)
    half = dim // 2
    freqs = np.exp(-math.log(10000.0) * np.arange(half, dtype=np.float32) / max(half - 1, 1))
    angles = np.asarray(values, dtype=np.float32)[..., None] * freqs * 1000.0
    emb = np.concatenate([np.sin(angles), np.cos(angles)], axis=-1)
    if dim % 2:
        emb = np.concatenate([emb, np.zeros(emb.shape[:-1] + (1,), dtype=np.float32)], axis=-1)
    return emb


def init_dit(cfg: DitCfg, seed=0, dtype=np.float32) -> dict:  # diffusion.py:134-154 (draw order)
    g = orng.stream(seed, "dit-init")
    d = cfg.model_dim
    p = {}
    p["latent_embed.w"] = g.normal(0, 0.02, (cfg.latent_dim, d)).astype(dtype)
    p["latent_embed.b"] = np.zeros(d, dtype=dtype)
    p["action_proj.w"] = g.normal(0, 0.02, (cfg.action_latent_dim, d)).astype(dtype)
    p["action_proj.b"] = np.zeros(d, dtype=dtype)
    p["null_action"] = g.normal(0, 0.02, (cfg.action_latent_dim,)).astype(dtype)
    p["gt_action_embed"] = g.normal(0, 0.02, (cfg.action_vocab, cfg.action_latent_dim)).astype(dtype)
    p["noise_proj.w"] = g.normal(0, 0.02, (d, d)).astype(dtype)
    p["noise_proj.b"] = np.zeros(d, dtype=dtype)
    p["pos_spatial"] = g.normal(0, 0.02, (cfg.patches_per_frame + 2, d)).astype(dtype)
    p["pos_temporal"] = g.normal(0, 0.02, (cfg.max_frames, d)).astype(dtype)
    p.update(init_st_stack(g, cfg.st, "dit", dtype))
    p["to_latent.w"] = g.normal(0, 0.02, (d, cfg.latent_dim)).astype(dtype)
    p["to_latent.b"] = np.zeros(cfg.latent_dim, dtype=dtype)
    return p


def forcing_corrupt(latents: np.ndarray, tau, gen: np.random.Generator) -> np.ndarray:  # diffusion.py:106-111
    tau = np.asarray(tau, dtype=latents.dtype)[..., None, None]
    eps = gen.standard_normal(latents.shape).astype(latents.dtype)
    return (1.0 - tau) * latents + tau * eps


def dit_predict_clean(P, cfg: DitCfg, noised: np.ndarray, tau, action_latents):  # diffusion.py:164-180
    b, t, n, _ = noised.shape
    d = cfg.model_dim
    dtype = P["latent_embed.w"].dtype
    if action_latents.shape[1] != t - 1:  # _conditioning, diffusion.py:156-162
        raise ValueError(f"need {t - 1} actions for {t} frames")
    x = linear(torch.as_tensor(noised).to(dtype), P["latent_embed.w"], P["latent_embed.b"])
    null = P["null_action"].reshape(1, 1, -1) + torch.zeros(b, 1, cfg.action_latent_dim, dtype=dtype)
    act = linear(torch.cat([null, action_latents], dim=1), P["action_proj.w"], P["action_proj.b"])
    noise_emb = torch.as_tensor(sinusoidal_embedding(tau, d)).to(dtype)
    noise_tok = linear(noise_emb, P["noise_proj.w"], P["noise_proj.b"])
    x = torch.cat([act.reshape(b, t, 1, d), noise_tok.reshape(b, t, 1, d), x], dim=2)
    x = x + P["pos_spatial"]
    x = x + P["pos_temporal"][:t].reshape(1, t, 1, d)
    x = st_stack(x, P, cfg.st, "dit")
    return linear(x[:, :, 2:], P["to_latent.w"], P["to_latent.b"])


def dit_loss(P, cfg: DitCfg, latents: np.ndarray, action_latents, gen: np.random.Generator):  # :182-192
    b, t = latents.shape[:2]
    tau = gen.uniform(0.0, 1.0, size=(b, t))
    noised = forcing_corrupt(latents, tau, gen)
    pred = dit_predict_clean(P, cfg, noised, tau, action_latents)
    err = pred - torch.as_tensor(latents).to(pred.dtype)
    per_frame = (err * err).mean(dim=(2, 3))
    return (per_frame * torch.as_tensor(tau).to(pred.dtype)).mean()


def dit_sample_frame(P, cfg: DitCfg, context: np.ndarray, action_latents, steps=25, context_noise=0.1,
                     gen: np.random.Generator | None = None) -> np.ndarray:  # diffusion.py:194-215
    if steps < 1:
        raise ValueError("steps must be >= 1")
    if gen is None:
        gen = orng.stream(0, "diffusion-sample")
    b, t_prev, n, dl = context.shape
    z = gen.standard_normal((b, 1, n, dl)).astype(context.dtype)
    with torch.no_grad():
        for k in range(steps, 0, -1):
            tau_k, tau_prev = k / steps, (k - 1) / steps
            ctx = forcing_corrupt(context, np.full((b, t_prev), context_noise), gen)
            full = np.concatenate([ctx, z], axis=1)
            tau = np.concatenate([np.full((b, t_prev), context_noise), np.full((b, 1), tau_k)], axis=1)
            pred = dit_predict_clean(P, cfg, full, tau, action_latents).numpy()[:, -1:]
            z = z + (tau_k - tau_prev) * (pred - z) / tau_k
    return z[:, 0]


@dataclass(frozen=True)
class MaeCfg:  # diffusion.py:23-47
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
    def st(self) -> StCfg:
        return StCfg(self.model_dim, self.heads, self.ffn_dim, self.blocks)


def init_mae(cfg: MaeCfg, seed=0, dtype=np.float32) -> dict:  # diffusion.py:51-70 (draw order)
    g = orng.stream(seed, "mae-init")
    d = cfg.model_dim
    p = {}
    p["patch_embed.w"] = g.normal(0, 0.02, (cfg.patch_dim, d)).astype(dtype)
    p["patch_embed.b"] = np.zeros(d, dtype=dtype)
    p["mask_token"] = g.normal(0, 0.02, (d,)).astype(dtype)
    p["pos_spatial"] = g.normal(0, 0.02, (cfg.patches_per_frame, d)).astype(dtype)
    p["pos_temporal"] = g.normal(0, 0.02, (cfg.max_frames, d)).astype(dtype)
    p.update(init_st_stack(g, cfg.st, "enc", dtype))
    p["to_latent.w"] = g.normal(0, 0.02, (d, cfg.latent_dim)).astype(dtype)
    p["to_latent.b"] = np.zeros(cfg.latent_dim, dtype=dtype)
    p["from_latent.w"] = g.normal(0, 0.02, (cfg.latent_dim, d)).astype(dtype)
    p["from_latent.b"] = np.zeros(d, dtype=dtype)
    p.update(init_st_stack(g, cfg.st, "dec", dtype))
    p["to_pixels.w"] = g.normal(0, 0.02, (d, cfg.patch_dim)).astype(dtype)
    p["to_pixels.b"] = np.zeros(cfg.patch_dim, dtype=dtype)
    return p


def mae_encode(P, cfg: MaeCfg, unit, mask=None):  # diffusion.py:72-86
    t, d = unit.shape[1], cfg.model_dim
    x = linear(patchify(unit, cfg.patch), P["patch_embed.w"], P["patch_embed.b"])
    if mask is not None:
        m = torch.as_tensor(np.asarray(mask, dtype=bool))[..., None]
        x = torch.where(m, P["mask_token"].expand_as(x), x)
    x = x + P["pos_spatial"]
    x = x + P["pos_temporal"][:t].reshape(1, t, 1, d)
    x = st_stack(x, P, cfg.st, "enc")
    return torch.tanh(linear(x, P["to_latent.w"], P["to_latent.b"]))


def mae_decode(P, cfg: MaeCfg, latents):  # diffusion.py:88-92
    x = linear(latents, P["from_latent.w"], P["from_latent.b"])
    x = st_stack(x, P, cfg.st, "dec")
    x = linear(x, P["to_pixels.w"], P["to_pixels.b"])
    return unpatchify(x, cfg.patch, cfg.height, cfg.width, cfg.channels)


def mae_mask(cfg: MaeCfg, b: int, t: int, gen: np.random.Generator) -> np.ndarray:  # diffusion.py:97-99
    p = gen.uniform(0.0, cfg.mask_prob_max, size=(b, t))
    return gen.random((b, t, cfg.patches_per_frame)) < p[:, :, None]


def mae_forward(P, cfg: MaeCfg, unit, gen: np.random.Generator):  # diffusion.py:94-103
    mask = mae_mask(cfg, unit.shape[0], unit.shape[1], gen)
    latents = mae_encode(P, cfg, unit, mask)
    recon = mae_decode(P, cfg, latents)
    return recon, latents, mse(recon, unit.detach())
