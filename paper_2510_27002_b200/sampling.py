"""MaskGIT decoding and autoregressive rollout (dynamics.py:156-260).

`decode_frame` follows the reference loop exactly: cosine keep schedule with the
known-count floor, temperature softmax, inverse-CDF sampling with f64 uniforms
drawn from the caller's numpy Philox generator, confidence of the sampled token,
stable (confidence desc, position asc) top-n_keep.  Logits come from the model's
`logits` (device forward for DynamicsModel; any duck-typed stand-in with the
reference's signature also works, test_dynamics.py:143-170).
"""
from __future__ import annotations

import numpy as np
import torch

from .rng import stream
from .tensor import Tensor


def _np_logits(model, tokens, latents, mask) -> np.ndarray:
    out = model.logits(tokens, latents, mask=mask)
    data = out.data if hasattr(out, "data") else out
    if isinstance(data, torch.Tensor):
        data = data.detach().cpu().numpy()
    return np.asarray(data)


def _sample_with_confidence(logits: np.ndarray, temperature: float, rng: np.random.Generator):
    """dynamics.py:198-217."""
    scaled = logits / max(temperature, 1e-8)
    scaled = scaled - scaled.max(axis=-1, keepdims=True)
    probs = np.exp(scaled)
    probs /= probs.sum(axis=-1, keepdims=True)
    if temperature < 1e-6:
        sampled = np.argmax(logits, axis=-1)
    else:
        cdf = np.cumsum(probs, axis=-1)
        u = rng.random(logits.shape[:-1] + (1,))
        sampled = (u > cdf).sum(axis=-1)
        sampled = np.minimum(sampled, logits.shape[-1] - 1)
    conf = np.take_along_axis(probs, sampled[..., None], axis=-1)[..., 0]
    return sampled.astype(np.int64), conf


def decode_frame(model, prev_tokens, action_latents, steps: int = 25, temperature: float = 1.0,
                 rng: np.random.Generator | None = None) -> np.ndarray:
    if steps < 1:
        raise ValueError("steps must be >= 1")
    if rng is None:
        rng = stream(0, "maskgit-decode")
    prev_tokens = np.asarray(prev_tokens)
    b, t_prev, n = prev_tokens.shape
    if action_latents.shape[1] != t_prev:
        raise ValueError(f"need {t_prev} action latents, got {action_latents.shape[1]}")
    tokens = np.concatenate([prev_tokens, np.zeros((b, 1, n), dtype=prev_tokens.dtype)], axis=1)
    known = np.zeros((b, n), dtype=bool)
    cur = np.zeros((b, n), dtype=prev_tokens.dtype)
    for s in range(1, steps + 1):
        frac_masked = np.cos(np.pi / 2 * s / steps)
        n_keep = n if s == steps else min(n, int(np.ceil(n * (1.0 - frac_masked))))
        n_keep = max(n_keep, int(known[0].sum()))
        tokens[:, -1] = cur
        mask = np.zeros_like(tokens, dtype=bool)
        mask[:, -1] = ~known
        logits = _np_logits(model, tokens, action_latents, mask)[:, -1]
        sampled, conf = _sample_with_confidence(logits, temperature, rng)
        cur = np.where(known, cur, sampled)
        conf = np.where(known, np.inf, conf)
        order = np.lexsort((np.broadcast_to(np.arange(n), conf.shape), -conf), axis=-1)
        new_known = np.zeros_like(known)
        np.put_along_axis(new_known, order[:, :n_keep], True, axis=-1)
        known = new_known
    assert known.all(), "decode must leave zero masked positions"
    return cur


def rollout(tokenizer, dynamics, conditioning_frames, actions, horizon: int, steps: int = 25,
            temperature: float = 1.0, rng=None, source_codebook=None, prefix_action_latents=None):
    from .tokenizer import unit_to_frames
    if len(actions) < horizon:
        raise ValueError(f"need {horizon} actions, got {len(actions)}")
    n_cond = conditioning_frames.shape[1]
    if n_cond + horizon > dynamics.cfg.max_frames:
        raise ValueError("horizon exceeds the model's maximum clip length")
    if rng is None:
        rng = stream(0, "rollout")
    tokens = np.asarray(tokenizer.encode(conditioning_frames))
    b = tokens.shape[0]
    dlat = dynamics.cfg.action_latent_dim
    if prefix_action_latents is not None:
        history = prefix_action_latents.data if isinstance(prefix_action_latents, Tensor) else \
            torch.as_tensor(np.asarray(prefix_action_latents)).cuda()
    else:
        null = dynamics.params["null_action"].data.detach().reshape(1, 1, dlat)
        history = torch.zeros((b, n_cond - 1, dlat), dtype=torch.float32, device=null.device) + null
    for step in range(horizon):
        action = actions[step]
        if isinstance(action, Tensor):
            lat = action.data.reshape(b, 1, dlat)
        else:
            lat = dynamics.action_latents_for(np.asarray(action).reshape(b, 1), source_codebook).data
        history = torch.cat([history, lat.to(history.device)], dim=1)
        nxt = dynamics.decode_frame(tokens, Tensor(history), steps=steps, temperature=temperature, rng=rng)
        tokens = np.concatenate([tokens, np.asarray(nxt)[:, None, :]], axis=1)
    unit = tokenizer.decode(tokens)
    return unit_to_frames(unit)
