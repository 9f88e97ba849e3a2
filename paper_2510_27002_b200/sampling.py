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


def _is_device_model(model) -> bool:
    from .dynamics import DynamicsModel
    return isinstance(model, DynamicsModel)


def decode_frame(model, prev_tokens, action_latents, steps: int = 25, temperature: float = 1.0,
                 rng: np.random.Generator | None = None) -> np.ndarray:
    """dynamics.py:156-194.  A DynamicsModel with a prepended action token decodes on the KV-cached
    device path; any other model (additive conditioning, or a duck-typed stand-in with the
    reference's cfg/params/logits surface, test_dynamics.py:143-170) runs the same device sampler
    over full-clip logits (decode_frame_stepwise)."""
    if _is_device_model(model) and model.cfg.mode.value != "additive":
        return decode_frame_device(model, prev_tokens, action_latents, steps, temperature, rng).cpu().numpy()
    return decode_frame_stepwise(model, prev_tokens, action_latents, steps, temperature, rng).cpu().numpy()


def decode_frame_stepwise(model, prev_tokens, action_latents, steps: int = 25, temperature: float = 1.0,
                          rng: np.random.Generator | None = None) -> torch.Tensor:
    """MaskGIT loop of dynamics.py:164-194 with K11 (jz_maskgit_step) doing the sampling, the
    confidence and the top-n_keep reveal on the device every step; the logits of each step are a
    full-clip forward of `model.logits` (device forward for a DynamicsModel; a duck-typed model's
    host logits are copied in).  Draws: B*N uniforms per step from `rng` (none when greedy), in
    the reference's order.  Returns cur (B, N) int64 in HBM."""
    if steps < 1:
        raise ValueError("steps must be >= 1")
    if rng is None:
        rng = stream(0, "maskgit-decode")
    on_dev = _is_device_model(model)
    dev = torch.device("cuda", torch.cuda.current_device())
    prev = prev_tokens.cpu().numpy() if isinstance(prev_tokens, torch.Tensor) else np.asarray(prev_tokens)
    b, t_prev, n = prev.shape
    if action_latents.shape[1] != t_prev:
        raise ValueError(f"need {t_prev} action latents, got {action_latents.shape[1]}")
    K = int(model.cfg.token_codes)
    tokens = np.concatenate([prev, np.zeros((b, 1, n), dtype=prev.dtype)], axis=1)
    cur = torch.zeros(b, n, dtype=torch.int64, device=dev)
    known = torch.zeros(b, n, dtype=torch.uint8, device=dev)
    conf = torch.empty(b, n, dtype=torch.float32, device=dev)
    if on_dev:
        tok_d = torch.as_tensor(tokens).to(dev, torch.int64)
        lat = action_latents if isinstance(action_latents, Tensor) else Tensor(np.asarray(action_latents))
    greedy = temperature < 1e-6
    for s, n_keep in enumerate(keep_counts(n, steps)):
        if on_dev:
            tok_d[:, -1] = cur
            mask = torch.zeros(b, t_prev + 1, n, dtype=torch.uint8, device=dev)
            mask[:, -1] = 1 - known
            lg = model.logits(tok_d, lat, mask=mask).data[:, -1]
        else:  # duck-typed stand-in: numpy in, its logits copied to the device sampler
            tokens[:, -1] = cur.cpu().numpy()
            mask = np.zeros(tokens.shape, dtype=bool)
            mask[:, -1] = known.cpu().numpy() == 0
            out = model.logits(tokens, action_latents, mask=mask)
            lg = out.data if hasattr(out, "data") else out
            lg = torch.as_tensor(np.asarray(lg.cpu() if isinstance(lg, torch.Tensor) else lg)[:, -1])
        lg = lg.to(dev, torch.float32).contiguous()
        z = (_C.c_uint64 * 4)()
        if greedy:
            _L.call("jz_maskgit_step", lg.data_ptr(), b, n, K, float(temperature), _C.addressof(z), _C.addressof(z),
                    _C.addressof(z), 4, 0, n_keep, None, cur.data_ptr(), known.data_ptr(), conf.data_ptr(),
                    _L.stream_ptr())
        else:
            st = _consume(rng, b * n)
            ctr = (_C.c_uint64 * 4)(*st.counter)
            key = (_C.c_uint64 * 2)(*st.key)
            buf = (_C.c_uint64 * 4)(*st.buffer)
            _L.call("jz_maskgit_step", lg.data_ptr(), b, n, K, float(temperature), _C.addressof(ctr),
                    _C.addressof(key), _C.addressof(buf), int(st.buffer_pos), 0, n_keep, None, cur.data_ptr(),
                    known.data_ptr(), conf.data_ptr(), _L.stream_ptr())
    return cur


def rollout(tokenizer, dynamics, conditioning_frames, actions, horizon: int, steps: int = 25,
            temperature: float = 1.0, rng=None, source_codebook=None, prefix_action_latents=None):
    """dynamics.py:220-260.  Device models with a prepended action token run rollout_device (KV
    cache, graph-captured refinement steps); other models decode each frame with decode_frame's
    device sampler."""
    from .dynamics import DynamicsModel
    from .tokenizer import VideoTokenizer, unit_to_frames
    if isinstance(dynamics, DynamicsModel) and isinstance(tokenizer, VideoTokenizer) \
            and dynamics.cfg.mode.value != "additive":
        return rollout_device(tokenizer, dynamics, conditioning_frames, actions, horizon, steps, temperature, rng,
                              source_codebook, prefix_action_latents).cpu().numpy()
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
        history = torch.cat([history, lat.to(history.device, history.dtype)], dim=1)
        nxt = decode_frame(dynamics, tokens, Tensor(history), steps=steps, temperature=temperature, rng=rng)
        tokens = np.concatenate([tokens, np.asarray(nxt)[:, None, :]], axis=1)
    unit = tokenizer.decode(tokens)
    return unit_to_frames(unit)


# ==========================================================================
# Device path: KV-cached MaskGIT decoding (K11 + K12)
# ==========================================================================
import ctypes as _C

from . import _lib as _L
from . import kernels as _K
from .rng import PhiloxState as _PS
from .rng import consume as _consume
from .st import _shadows, check_supported


def keep_counts(n: int, steps: int) -> list[int]:
    """n_keep per step (dynamics.py:177-179), floor-maxed with the previous count (known grows)."""
    out, prev = [], 0
    for s in range(1, steps + 1):
        frac = np.cos(np.pi / 2 * s / steps)
        k = n if s == steps else min(n, int(np.ceil(n * (1.0 - frac))))
        k = max(k, prev)
        out.append(k)
        prev = k
    return out


class FrameDecoder:
    """Per-layer temporal K/V cache + single-frame forward of a DynamicsModel (prepend mode)."""

    def __init__(self, model, B: int, t_max: int | None = None):
        cfg = model.cfg
        if cfg.mode.value == "additive":
            raise ValueError("device MaskGIT decoding supports the prepended action token (prepend / ground-truth modes)")
        self.model, self.cfg, self.B = model, cfg, B
        self.N, self.D, self.H = cfg.patches_per_frame, cfg.model_dim, cfg.heads
        self.S = self.N + 1
        self.t_max = t_max or cfg.max_frames
        check_supported(cfg.st, self.S, self.t_max)
        if self.t_max > 16:
            raise ValueError(f"KV-cached decoding supports up to 16 frames (got t_max={self.t_max})")
        dev = model.params["token_embed"].data.device
        self.cache = [torch.empty(B, self.t_max, self.S, 2 * self.D, dtype=torch.bfloat16, device=dev)
                      for _ in range(cfg.blocks)]
        P = model.params
        self.P = P
        # private copies: the captured graph holds these addresses, and the store's shared shadow
        # is recast by every forward of the model
        self.sh = [{k: v.clone() for k, v in blk.items()} for blk in _shadows(P, cfg.st, "dyn")]
        self.wl = _K.cast_bf16(P["to_logits.w"].data)
        self.t = 0  # frames cached

    def prefill(self, tokens: torch.Tensor, latents: torch.Tensor) -> None:
        """Cache frames 0..t0-1 (tokens (B,t0,N) int64, latents (B,t0-1,dl)) — the full-clip forward of those frames."""
        cfg, P = self.cfg, self.P
        self._refresh_weights()
        B, t0, N = tokens.shape
        err = torch.zeros((), dtype=torch.int32, device=tokens.device)
        x = _K.dyn_embed_fwd(tokens, None, latents.contiguous(), {k: v.data for k, v in P.items()}, B=B, T=t0, N=N,
                             D=self.D, dl=cfg.action_latent_dim, K=cfg.token_codes, prepend=True, err=err)
        for i in range(cfg.blocks):
            x = self._block(i, x, B=B, T=t0, temporal=("full", None))
        self.t = t0

    def _refresh_weights(self):
        """Re-cast the bf16 weight shadows IN PLACE (graph-captured kernels hold their addresses)."""
        fresh = _shadows(self.P, self.cfg.st, "dyn")
        for old, new in zip(self.sh, fresh):
            for k in old:
                old[k].copy_(new[k])
        _K.cast_bf16(self.P["to_logits.w"].data, self.wl)

    def _block(self, i, x, *, B, T, temporal):
        P, w, base = self.P, self.sh[i], f"dyn.block{i}"
        H, S = self.H, self.S
        xn, _, _ = _K.layernorm_fwd(x, P[f"{base}.spatial.ln.g"].data, P[f"{base}.spatial.ln.b"].data)
        qkv = _K.linear_fwd(xn, w["spatial.wqkv"], w["spatial.bqkv"])
        ao, _, _ = _K.attn_spatial_fwd(qkv, B * T, S, H, keep_lo=False)
        # the attention output projections emit the next LayerNorm from their epilogue, as in training
        fuse = _K.ln_fusable(B * T * S, self.D, K=self.D)
        if fuse:
            x1, xn2, _, _ = _K.linear_fwd_ln(ao, w["spatial.wo"], P[f"{base}.spatial.o.b"].data, x,
                                             P[f"{base}.temporal.ln.g"].data, P[f"{base}.temporal.ln.b"].data)
        else:
            x1 = _K.linear_fwd(ao, w["spatial.wo"], P[f"{base}.spatial.o.b"].data, epilogue=_L.EPI_RESID, aux=x)
            xn2, _, _ = _K.layernorm_fwd(x1, P[f"{base}.temporal.ln.g"].data, P[f"{base}.temporal.ln.b"].data)
        qkv2 = _K.linear_fwd(xn2, w["temporal.wqkv"], w["temporal.bqkv"])
        mode, arg = temporal
        if mode == "full":
            ao2, _ = _K.attn_temporal_fwd(qkv2, B, T, S, H)
            _L.call("jz_kv_fill", qkv2.data_ptr(), self.cache[i].data_ptr(), B, T, 0, self.t_max, S, self.D,
                    _L.stream_ptr())
        else:
            t, append, dev_t = arg
            ao2 = torch.empty(B * S, self.D, dtype=torch.bfloat16, device=x.device)
            _L.call("jz_attn_temporal_decode", qkv2.data_ptr(), self.cache[i].data_ptr(), B, t,
                    None if dev_t is None else dev_t.data_ptr(), self.t_max, S, H, int(append), ao2.data_ptr(),
                    _L.stream_ptr())
        if fuse:
            x2, xn3, _, _ = _K.linear_fwd_ln(ao2, w["temporal.wo"], P[f"{base}.temporal.o.b"].data, x1,
                                             P[f"{base}.ffn.ln.g"].data, P[f"{base}.ffn.ln.b"].data)
        else:
            x2 = _K.linear_fwd(ao2, w["temporal.wo"], P[f"{base}.temporal.o.b"].data, epilogue=_L.EPI_RESID, aux=x1)
            xn3, _, _ = _K.layernorm_fwd(x2, P[f"{base}.ffn.ln.g"].data, P[f"{base}.ffn.ln.b"].data)
        h = _K.linear_fwd(xn3, w["ffn.wup"], P[f"{base}.ffn.up.b"].data, epilogue=_L.EPI_GELU)
        return _K.linear_fwd(h, w["ffn.wdown"], P[f"{base}.ffn.down.b"].data, epilogue=_L.EPI_RESID, aux=x2)

    def frame(self, tokens: torch.Tensor, known: torch.Tensor | None, cond: torch.Tensor, *, append: bool,
              logits: bool = True, dev_t: torch.Tensor | None = None):
        """Forward one frame ((B,N) tokens; known (B,N) u8 or None=all known) over the cache.

        The frame index is self.t, or the device scalar dev_t (graph-captured path)."""
        cfg, P = self.cfg, self.P
        B, N, D, t = self.B, self.N, self.D, self.t
        x = torch.empty(B * self.S, D, dtype=torch.float32, device=tokens.device)
        pt = P["pos_temporal"].data
        pt_row = pt if dev_t is not None else pt[t]
        _L.call("jz_dyn_embed_frame", tokens.data_ptr(), None if known is None else known.data_ptr(),
                cond.data_ptr(), P["token_embed"].data.data_ptr(), P["mask_token"].data.data_ptr(),
                P["action_proj.w"].data.data_ptr(), P["action_proj.b"].data.data_ptr(),
                P["pos_spatial"].data.data_ptr(), pt_row.data_ptr(), None if dev_t is None else dev_t.data_ptr(),
                B, N, D, cfg.action_latent_dim, cfg.token_codes, x.data_ptr(), _L.stream_ptr())
        for i in range(cfg.blocks):
            x = self._block(i, x, B=B, T=1, temporal=("decode", (t, append, dev_t)))
        if append and dev_t is None:
            self.t = t + 1
        if not logits:
            return None
        y, _, _ = _K.layernorm_fwd(x, P["dyn.final_ln.g"].data, P["dyn.final_ln.b"].data, skip_period=self.S)
        return _K.linear_fwd(y, self.wl, P["to_logits.b"].data, epilogue=_L.EPI_F32)

    # -- graph-captured decoding ------------------------------------------------
    def _static(self, dev):
        if getattr(self, "_cur", None) is None:
            B, N = self.B, self.N
            self._cur = torch.zeros(B, N, dtype=torch.int64, device=dev)
            self._known = torch.zeros(B, N, dtype=torch.uint8, device=dev)
            self._conf = torch.empty(B, N, dtype=torch.float32, device=dev)
            self._cond = torch.empty(B, self.cfg.action_latent_dim, dtype=torch.float32, device=dev)
            self._dev_t = torch.zeros((), dtype=torch.int32, device=dev)
            self._params = torch.zeros(13, dtype=torch.int64, device=dev)
            self._graphs: dict = {}

    def _step(self, temperature: float):
        logits = self.frame(self._cur, self._known, self._cond, append=False, dev_t=self._dev_t)
        z = (_C.c_uint64 * 4)()
        _L.call("jz_maskgit_step", logits.data_ptr(), self.B, self.N, self.cfg.token_codes, float(temperature),
                _C.addressof(z), _C.addressof(z), _C.addressof(z), 4, 0, 0, self._params.data_ptr(),
                self._cur.data_ptr(), self._known.data_ptr(), self._conf.data_ptr(), _L.stream_ptr())

    def _append(self):
        self.frame(self._cur, None, self._cond, append=True, logits=False, dev_t=self._dev_t)

    def decode(self, cond: torch.Tensor, steps: int, temperature: float, rng: np.random.Generator,
               graph: bool = True) -> torch.Tensor:
        """MaskGIT-decode frame self.t; returns cur (B, N) int64 in HBM and appends it to the cache.

        The refinement step (single-frame forward over the cache + sampler) and the cache
        append are each captured ONCE per decoder in a CUDA graph; the frame index, the
        step's draw offset / n_keep and the Philox state live in device memory and are
        refreshed by one small H2D copy before each replay.
        """
        dev = cond.device
        self._static(dev)
        B, N = self.B, self.N
        greedy = temperature < 1e-6
        st = _consume(rng, steps * B * N) if not greedy else None
        rows = []
        for s, k in enumerate(keep_counts(N, steps)):
            if st is None:
                rows.append([0, k] + [0] * 10 + [-1])
            else:
                rows.append([s * B * N, k] + st.counter + list(st.key) + st.buffer + [st.buffer_pos])
        mask64 = (1 << 64) - 1
        vals = torch.from_numpy(np.array([[v & mask64 for v in r] for r in rows], dtype=np.uint64).view(np.int64))
        # persistent pinned staging (freeing pinned blocks records CUDA events, which must never
        # happen while a graph is being captured)
        if getattr(self, "_host_rows", None) is None or self._host_rows.shape[0] < steps:
            torch.cuda.synchronize()
            self._host_rows = torch.empty((max(steps, 32), 13), dtype=torch.int64).pin_memory()
            self._host_t = torch.empty((), dtype=torch.int32).pin_memory()
        torch.cuda.current_stream().synchronize()  # previous H2D copies out of the staging are done
        host = self._host_rows
        host[:steps].copy_(vals)
        host_t = self._host_t
        host_t.fill_(self.t)
        self._cond.copy_(cond)
        self._cur.zero_()
        self._known.zero_()
        self._dev_t.copy_(host_t, non_blocking=True)
        key = ("step", float(temperature))
        g = self._graphs.get(key) if graph else None
        s0 = 0
        if graph and g is None:
            self._params.copy_(host[0], non_blocking=True)
            self._step(temperature)  # eager first step: loads every kernel before capture
            s0 = 1
            g = torch.cuda.CUDAGraph()
            with _no_gc(), torch.cuda.graph(g):
                self._step(temperature)
            self._graphs[key] = g
        for s in range(s0, steps):
            self._params.copy_(host[s], non_blocking=True)
            if g is not None:
                g.replay()
            else:
                self._step(temperature)
        ga = self._graphs.get("append") if graph else None
        if graph and ga is None:
            ga = torch.cuda.CUDAGraph()
            with _no_gc(), torch.cuda.graph(ga):
                self._append()
            self._graphs["append"] = ga
        if ga is not None:
            ga.replay()
        else:
            self._append()
        self.t += 1
        return self._cur.clone()


class _no_gc:
    """No Python garbage collection while a CUDA graph is captured: collecting an unrelated
    pinned tensor frees a host block and records a CUDA event, invalidating the capture."""

    def __enter__(self):
        import gc
        gc.collect()
        self._was = gc.isenabled()
        gc.disable()

    def __exit__(self, *exc):
        import gc
        if self._was:
            gc.enable()
        return False


def decoder_for(model, B: int, t_max: int) -> "FrameDecoder":
    """A FrameDecoder (KV cache + captured graphs) reused across calls for the same model/batch.

    The weight shadows are re-derived on every prefill (callers may update or swap params)."""
    cache = model.__dict__.setdefault("_frame_decoders", {})
    key = (B, t_max, id(model.params))
    dec = cache.get(key)
    if dec is None:
        cache.clear()  # keep one decoder (its KV cache is large)
        dec = FrameDecoder(model, B, t_max)
        cache[key] = dec
    return dec


def _dev_latents(model, action_latents) -> torch.Tensor:
    lat = action_latents.data if isinstance(action_latents, Tensor) else action_latents
    if not isinstance(lat, torch.Tensor):
        lat = torch.as_tensor(np.asarray(lat, dtype=np.float32))
    return lat.to(model.params["token_embed"].data.device, torch.float32).contiguous()


def decode_frame_device(model, prev_tokens, action_latents, steps: int = 25, temperature: float = 1.0,
                        rng: np.random.Generator | None = None) -> torch.Tensor:
    """dynamics.py:156-194 on device: prefill frames 0..t-1, then 'steps' KV-cached refinements."""
    if steps < 1:
        raise ValueError("steps must be >= 1")
    if rng is None:
        rng = stream(0, "maskgit-decode")
    tok = prev_tokens if isinstance(prev_tokens, torch.Tensor) else torch.as_tensor(np.asarray(prev_tokens))
    dev = model.params["token_embed"].data.device
    tok = tok.to(dev, torch.int64).contiguous()
    b, t_prev, n = tok.shape
    lat = _dev_latents(model, action_latents)
    if lat.shape[1] != t_prev:
        raise ValueError(f"need {t_prev} action latents, got {lat.shape[1]}")
    dec = decoder_for(model, b, max(model.cfg.max_frames, t_prev + 1))
    dec.prefill(tok, lat[:, : t_prev - 1])
    return dec.decode(lat[:, t_prev - 1].contiguous(), steps, temperature, rng)


def rollout_device(tokenizer, dynamics, conditioning_frames, actions, horizon: int, steps: int = 25,
                   temperature: float = 1.0, rng=None, source_codebook=None, prefix_action_latents=None,
                   return_tokens: bool = False):
    """dynamics.py:220-260 fully on device; returns uint8 frames (B, n_cond+horizon, H, W, C) in HBM."""
    if len(actions) < horizon:
        raise ValueError(f"need {horizon} actions, got {len(actions)}")
    n_cond = conditioning_frames.shape[1]
    if n_cond + horizon > dynamics.cfg.max_frames:
        raise ValueError("horizon exceeds the model's maximum clip length")
    if rng is None:
        rng = stream(0, "rollout")
    tokens = tokenizer.encode_device(conditioning_frames)
    b = tokens.shape[0]
    dlat = dynamics.cfg.action_latent_dim
    dev = tokens.device
    if prefix_action_latents is not None:
        history = _dev_latents(dynamics, prefix_action_latents)
    else:
        null = dynamics.params["null_action"].data.reshape(1, 1, dlat)
        history = torch.zeros((b, n_cond - 1, dlat), dtype=torch.float32, device=dev) + null
    dec = decoder_for(dynamics, b, dynamics.cfg.max_frames)
    dec.prefill(tokens, history)
    frames_tok = [tokens]
    for step in range(horizon):
        action = actions[step]
        if isinstance(action, Tensor):
            lat = action.data.reshape(b, dlat).float()
        else:
            lat = dynamics.action_latents_for(np.asarray(action).reshape(b, 1), source_codebook).data.reshape(b, dlat)
        nxt = dec.decode(lat.contiguous(), steps, temperature, rng)
        frames_tok.append(nxt[:, None, :])
    all_tok = torch.cat(frames_tok, dim=1)
    unit = tokenizer.decode_device(all_tok)
    cfg = tokenizer.cfg
    B, T = all_tok.shape[0], all_tok.shape[1]
    _, p32 = _K.patchify(unit.view(B * T, cfg.height, cfg.width, cfg.channels), cfg.patch, bf16=False, f32=True)
    _, u8 = _K.unpatchify(p32, B * T, cfg.height, cfg.width, cfg.channels, cfg.patch, unit=False, u8=True)
    out = u8.view(B, T, cfg.height, cfg.width, cfg.channels)
    return (out, all_tok) if return_tokens else out
