"""Spatio-temporal transformer backbone on B200 (mirror of deskworld/st.py).

`st_forward` / `st_backward` run one ST stack (st.py:69-85) as a fixed schedule
of libjz kernels on rows ordered (b, t, s):

  per block:  LN -> QKV GEMM(+bias) -> tcgen05 spatial attention -> O GEMM(+bias+residual)
              LN -> QKV GEMM(+bias) -> causal temporal attention  -> O GEMM(+bias+residual)
              LN -> up GEMM(+bias, GELU fused) -> down GEMM(+bias+residual)
  final LN (optionally dropping the s=0 action-token rows, dynamics.py:135-136)

The (B, T, S, D) -> (B, S, T, D) transpose of the reference's temporal sub-layer
(st.py:74-76) never materialises: the temporal kernel gathers rows with stride S.
The residual stream stays fp32; GEMM operands are bf16 with fp32 TMEM accumulation.
The backward is the exact reverse schedule with deterministic reductions.
"""
from __future__ import annotations

from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import kernels as K
from .tensor import Tensor, param_count, store_for  # noqa: F401  (re-export, st.py:97-98)


@dataclass(frozen=True)
class StConfig:
    """st.py:20-31 (same fields, defaults and validation)."""
    model_dim: int = 512
    heads: int = 8
    ffn_dim: int = 2048
    blocks: int = 4

    def __post_init__(self):
        if self.model_dim % self.heads != 0:
            raise ValueError("model_dim must divide by heads")
        if self.ffn_dim % self.model_dim != 0 or self.ffn_dim // self.model_dim not in (1, 4):
            raise ValueError("ffn expansion factor must be 1 or 4")


def init_st_stack_arrays(rng, cfg: StConfig, prefix: str = "st", dtype=np.float32) -> "OrderedDict[str, np.ndarray]":
    """Host init in the reference's exact draw order (st.py:34-57)."""
    p: "OrderedDict[str, np.ndarray]" = OrderedDict()
    d, f = cfg.model_dim, cfg.ffn_dim

    def lin(name, din, dout):
        p[f"{name}.w"] = rng.normal(0.0, 0.02, size=(din, dout)).astype(dtype)
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


def st_param_groups(cfg: StConfig, prefix: str) -> list:
    """ParamStore groups: each attention sub-layer's q/k/v weights (and biases) side by side,
    so the fused QKV projection reads one (d, 3d) bf16 view and writes one (d, 3d) gradient."""
    out = []
    for i in range(cfg.blocks):
        for sub in ("spatial", "temporal"):
            base = f"{prefix}.block{i}.{sub}"
            out.append(tuple(f"{base}.{p}.w" for p in "qkv"))
            out.append(tuple(f"{base}.{p}.b" for p in "qkv"))
    return out


def init_st_stack(rng, cfg: StConfig, prefix: str = "st", dtype=np.float32) -> dict:
    """st.py:44-57: returns device parameters."""
    return {k: Tensor(v, requires_grad=True) for k, v in init_st_stack_arrays(rng, cfg, prefix, dtype).items()}


def st_stack_param_count(cfg: StConfig) -> int:
    """st.py:88-94."""
    d, f = cfg.model_dim, cfg.ffn_dim
    per_attn = 4 * (d * d + d) + 2 * d
    per_ffn = d * f + f + f * d + d + 2 * d
    return cfg.blocks * (2 * per_attn + per_ffn) + 2 * d


def check_supported(cfg: StConfig, S: int, T: int) -> None:
    """The device path's shape envelope (raises ValueError outside it; no CPU fallback)."""
    if cfg.model_dim // cfg.heads != 64:
        raise ValueError(f"device ST stack needs head_dim 64 (got {cfg.model_dim // cfg.heads})")
    if cfg.model_dim % 128 or cfg.model_dim > 1024:
        raise ValueError(f"device ST stack needs model_dim % 128 == 0 and <= 1024 (got {cfg.model_dim})")
    if S not in (256, 257) and not 1 <= S <= 32:
        raise ValueError(f"device spatial attention supports S in (256, 257) or S <= 32, got {S}")
    if T > 32:
        raise ValueError(f"device temporal attention supports T <= 32, got {T}")


# --------------------------------------------------------------------------
# weight shadows (re-derived every call: callers may swap `params` wholesale)
# --------------------------------------------------------------------------
def _shadows(P: dict, cfg: StConfig, prefix: str) -> list:
    """bf16 GEMM operands of every block. With the model's grouped ParamStore this is ONE flat
    cast of all parameters (views into the shadow; qkv weights/biases are already fused blocks);
    otherwise (caller-assembled params) per-tensor casts."""
    st = store_for(P)
    if st is not None and st.block_of(st.flat, f"{prefix}.block0.spatial.q.w") is not None:
        sh = st.shadow()
        K.cast_bf16(st.flat, sh)
        out = []
        for i in range(cfg.blocks):
            base = f"{prefix}.block{i}"
            blk = {}
            for sub in ("spatial", "temporal"):
                blk[f"{sub}.wqkv"] = st.block_of(sh, f"{base}.{sub}.q.w")
                blk[f"{sub}.bqkv"] = st.block_of(st.flat, f"{base}.{sub}.q.b")
                blk[f"{sub}.wo"] = st.view_of(sh, f"{base}.{sub}.o.w")
            blk["ffn.wup"] = st.view_of(sh, f"{base}.ffn.up.w")
            blk["ffn.wdown"] = st.view_of(sh, f"{base}.ffn.down.w")
            out.append(blk)
        return out
    d, f = cfg.model_dim, cfg.ffn_dim
    dev = P[f"{prefix}.final_ln.g"].data.device
    out = []
    for i in range(cfg.blocks):
        base = f"{prefix}.block{i}"
        blk = {}
        for sub in ("spatial", "temporal"):
            w = torch.empty(d, 3 * d, dtype=K.BF16, device=dev)
            for j, proj in enumerate("qkv"):
                K.cast_bf16(P[f"{base}.{sub}.{proj}.w"].data, w[:, j * d:(j + 1) * d])
            blk[f"{sub}.wqkv"] = w
            blk[f"{sub}.bqkv"] = torch.cat([P[f"{base}.{sub}.{p}.b"].data for p in "qkv"])
            blk[f"{sub}.wo"] = K.cast_bf16(P[f"{base}.{sub}.o.w"].data)
        blk["ffn.wup"] = K.cast_bf16(P[f"{base}.ffn.up.w"].data)
        blk["ffn.wdown"] = K.cast_bf16(P[f"{base}.ffn.down.w"].data)
        out.append(blk)
    return out


def st_forward(x: torch.Tensor, P: dict, cfg: StConfig, prefix: str, *, B: int, T: int, S: int,
               final_skip: bool = False, save: bool = True, final_f32: bool = False, final_bf16: bool = True):
    """x f32 [B*T*S, D] (consumed as the residual stream).

    Returns (y, ctx): y is the final-LN output, bf16 [rows, D] (or (bf16|None, f32) when
    final_f32); rows drop the s=0 action-token rows when final_skip.
    """
    check_supported(cfg, S, T)
    H = cfg.heads
    frames = B * T
    sh = _shadows(P, cfg, prefix)
    rows = x.shape[0]
    # LayerNorm fused into the residual projections' epilogues (jz_gemm_bf16_ln_fwd): a residual
    # GEMM also emits the NEXT sub-layer's LayerNorm output.  kernels.ln_fusable holds the measured
    # policy (the attention output projections fuse; the K = 2048 FFN down-projection does not)
    fuse = K.ln_fusable(rows, cfg.model_dim, K=cfg.model_dim)           # after the attention projections
    fuse_ffn = K.ln_fusable(rows, cfg.model_dim, K=cfg.ffn_dim)         # after the FFN down-projection
    fuse_final = fuse_ffn and not final_f32
    blocks_ctx = []
    nxt = None  # (xn, mean, rstd) of this block's spatial LayerNorm, from the previous block's epilogue
    y = mf = rf = None
    for i in range(cfg.blocks):
        base = f"{prefix}.block{i}"
        w = sh[i]
        c = {"x_in": x}
        # spatial sub-layer (st.py:73)
        if nxt is None:
            xn, m1, r1 = K.layernorm_fwd(x, P[f"{base}.spatial.ln.g"].data, P[f"{base}.spatial.ln.b"].data)
        else:
            xn, m1, r1 = nxt
        qkv = K.linear_fwd(xn, w["spatial.wqkv"], w["spatial.bqkv"])
        ao, ao_lo, lse_s = K.attn_spatial_fwd(qkv, frames, S, H, keep_lo=save)
        if fuse:
            x1, xn2, m2, r2 = K.linear_fwd_ln(ao, w["spatial.wo"], P[f"{base}.spatial.o.b"].data, x,
                                               P[f"{base}.temporal.ln.g"].data, P[f"{base}.temporal.ln.b"].data)
        else:
            x1 = K.linear_fwd(ao, w["spatial.wo"], P[f"{base}.spatial.o.b"].data, epilogue=L.EPI_RESID, aux=x)
            xn2, m2, r2 = K.layernorm_fwd(x1, P[f"{base}.temporal.ln.g"].data, P[f"{base}.temporal.ln.b"].data)
        # temporal sub-layer (st.py:74-76)
        qkv2 = K.linear_fwd(xn2, w["temporal.wqkv"], w["temporal.bqkv"])
        ao2, lse_t = K.attn_temporal_fwd(qkv2, B, T, S, H)
        if fuse:
            x2, xn3, m3, r3 = K.linear_fwd_ln(ao2, w["temporal.wo"], P[f"{base}.temporal.o.b"].data, x1,
                                               P[f"{base}.ffn.ln.g"].data, P[f"{base}.ffn.ln.b"].data)
        else:
            x2 = K.linear_fwd(ao2, w["temporal.wo"], P[f"{base}.temporal.o.b"].data, epilogue=L.EPI_RESID, aux=x1)
            xn3, m3, r3 = K.layernorm_fwd(x2, P[f"{base}.ffn.ln.g"].data, P[f"{base}.ffn.ln.b"].data)
        # FFN (st.py:77-79)
        # training saves gelu'(pre-activation) (f16) from the same tanh, so the backward epilogue
        # only multiplies; inference skips it
        hpre = torch.empty(xn3.shape[0], cfg.ffn_dim, dtype=torch.float16, device=x.device) if save else None
        h = K.linear_fwd(xn3, w["ffn.wup"], P[f"{base}.ffn.up.b"].data,
                         epilogue=L.EPI_GELU_DG if save else L.EPI_GELU, out2=hpre)
        last = i == cfg.blocks - 1
        nxt = None
        if fuse_ffn and (not last or fuse_final):
            lnp = f"{prefix}.block{i + 1}.spatial.ln" if not last else f"{prefix}.final_ln"
            g_ln, b_ln = P[f"{lnp}.g"].data, P[f"{lnp}.b"].data
            x3, xn_n, m_n, r_n = K.linear_fwd_ln(h, w["ffn.wdown"], P[f"{base}.ffn.down.b"].data, x2, g_ln, b_ln,
                                                 skip_period=S if (last and final_skip) else 0)
            if last:
                y, mf, rf = xn_n, m_n, r_n
            else:
                nxt = (xn_n, m_n, r_n)
        else:
            x3 = K.linear_fwd(h, w["ffn.wdown"], P[f"{base}.ffn.down.b"].data, epilogue=L.EPI_RESID, aux=x2)
        if save:
            c.update(xn=xn, m1=m1, r1=r1, qkv=qkv, ao=ao, ao_lo=ao_lo, lse_s=lse_s, x1=x1, xn2=xn2, m2=m2, r2=r2, qkv2=qkv2,
                     ao2=ao2, lse_t=lse_t, x2=x2, xn3=xn3, m3=m3, r3=r3, h=h, hpre=hpre)
            blocks_ctx.append(c)
        x = x3
    if y is not None:  # the final LayerNorm came out of the last FFN-down GEMM's epilogue
        assert not final_f32
    elif final_f32:
        y16, y32, mf, rf = K.layernorm_fwd(x, P[f"{prefix}.final_ln.g"].data, P[f"{prefix}.final_ln.b"].data,
                                           skip_period=S if final_skip else 0, out_f32=True, out_bf16=final_bf16)
        y = (y16, y32)
    else:
        y, mf, rf = K.layernorm_fwd(x, P[f"{prefix}.final_ln.g"].data, P[f"{prefix}.final_ln.b"].data,
                                    skip_period=S if final_skip else 0)
    ctx = None
    if save:
        ctx = dict(blocks=blocks_ctx, shadows=sh, x_final=x, mf=mf, rf=rf, B=B, T=T, S=S,
                   final_skip=final_skip)
    return y, ctx


def st_backward(ctx: dict, dy: torch.Tensor, P: dict, G: dict, cfg: StConfig, prefix: str,
                on_done=None, want_dx_bf16: bool = False):
    """dy: f32 gradient of the final-LN output (compacted like y).  Writes G[...]; returns dx f32 [rows, D].

    on_done(name) is called (stream-ordered) as soon as a parameter group's gradients are final:
    "head_ln" after the final LN, then "block{i}" for i = n-1 .. 0 (data-parallel bucket hooks).
    """
    B, T, S = ctx["B"], ctx["T"], ctx["S"]
    H = cfg.heads
    frames = B * T
    d = cfg.model_dim
    x_final = ctx["x_final"]
    rows = x_final.shape[0]
    st = store_for(P)  # grouped-store gradients: the fused qkv blocks are written in place
    gst = st if (st is not None and st.grad_flat is not None and st.grads_are_views(G)
                 and st.block_of(st.grad_flat, f"{prefix}.block0.spatial.q.w") is not None) else None
    dev = x_final.device
    dres = torch.empty(rows, d, dtype=K.F32, device=dev)
    dres_b = torch.empty(rows, d, dtype=K.BF16, device=dev)
    nb = cfg.blocks
    # final LN; its dbias partial is the last block's down-projection bias gradient
    K.layernorm_bwd(x_final, ctx["mf"], ctx["rf"], P[f"{prefix}.final_ln.g"].data, dy, dres, accumulate=False,
                    dres_bf16=dres_b, dgamma=G[f"{prefix}.final_ln.g"], dbeta=G[f"{prefix}.final_ln.b"],
                    dbias=G[f"{prefix}.block{nb - 1}.ffn.down.b"], skip_period=S if ctx["final_skip"] else 0)
    if on_done is not None:
        on_done("head_ln")
    # LN-backward inputs in bf16: the dX GEMMs write half the bytes and the HBM-bound LN pass reads half
    fuse = K.ln_fusable(rows, d, backward=True)  # LayerNorm backward inside the dX GEMMs' epilogues
    dtmp = None if fuse else torch.empty(rows, d, dtype=K.BF16, device=dev)
    dh = torch.empty(rows, cfg.ffn_dim, dtype=K.BF16, device=dev)
    dao = torch.empty(rows, d, dtype=K.BF16, device=dev)
    for i in reversed(range(nb)):
        base = f"{prefix}.block{i}"
        c = ctx["blocks"][i]
        w = ctx["shadows"][i]
        # ---- FFN: x3 = x2 + gelu(LN(x2) Wup + bup) Wdown + bdown
        K.linear_dw(c["h"], dres_b, G[f"{base}.ffn.down.w"])
        K.linear_dx(dres_b, w["ffn.wdown"], epilogue=L.EPI_MUL_F16, out=dh, aux=c["hpre"],
                    colsum=G[f"{base}.ffn.up.b"])  # up-bias gradient from the epilogue's column sums
        K.linear_dw(c["xn3"], dh, G[f"{base}.ffn.up.w"])
        _dx_layernorm(dh, w["ffn.wup"], c["x2"], c["m3"], c["r3"], P[f"{base}.ffn.ln.g"].data, dres, dtmp,
                      dres_b, G[f"{base}.ffn.ln.g"], G[f"{base}.ffn.ln.b"], G[f"{base}.temporal.o.b"], fuse)
        # ---- temporal: x2 = x1 + attn_t(LN(x1)) Wo + bo
        K.linear_dw(c["ao2"], dres_b, G[f"{base}.temporal.o.w"])
        K.linear_dx(dres_b, w["temporal.wo"], epilogue=L.EPI_BF16, out=dao)
        gbt = gst.block_of(gst.grad_flat, f"{base}.temporal.q.b") if gst is not None else None
        dqkv = K.attn_temporal_bwd(c["qkv2"], c["ao2"], dao, c["lse_t"], B, T, S, H, colsum=gbt)
        _qkv_param_grads(dqkv, c["xn2"], G, f"{base}.temporal", d, gst, bias_done=gbt is not None)
        _dx_layernorm(dqkv, w["temporal.wqkv"], c["x1"], c["m2"], c["r2"], P[f"{base}.temporal.ln.g"].data, dres,
                      dtmp, dres_b, G[f"{base}.temporal.ln.g"], G[f"{base}.temporal.ln.b"], G[f"{base}.spatial.o.b"],
                      fuse)
        # ---- spatial: x1 = x + attn_s(LN(x)) Wo + bo
        K.linear_dw(c["ao"], dres_b, G[f"{base}.spatial.o.w"])
        gbs = gst.block_of(gst.grad_flat, f"{base}.spatial.q.b") if gst is not None else None
        K.linear_dx(dres_b, w["spatial.wo"], epilogue=L.EPI_BF16, out=dao)
        # the QKV bias gradient from the attention backward's own column-sum partials of dqkv (one
        # fused pass; measured 54 us per block faster than the dO-GEMM column sums + a q pass)
        dqkv = K.attn_spatial_bwd(c["qkv"], c["ao"], dao, c["lse_s"], frames, S, H, dqkv=dqkv, colsum=gbs,
                                  out_lo=c["ao_lo"])
        _qkv_param_grads(dqkv, c["xn"], G, f"{base}.spatial", d, gst, bias_done=gbs is not None)
        prev_bias = G[f"{prefix}.block{i - 1}.ffn.down.b"] if i > 0 else None
        _dx_layernorm(dqkv, w["spatial.wqkv"], c["x_in"], c["m1"], c["r1"], P[f"{base}.spatial.ln.g"].data, dres,
                      dtmp, dres_b if (i > 0 or want_dx_bf16) else None, G[f"{base}.spatial.ln.g"],
                      G[f"{base}.spatial.ln.b"], prev_bias, fuse)
        if on_done is not None:
            on_done(f"block{i}")
    if want_dx_bf16:
        return dres, dres_b
    return dres


def _dx_layernorm(dy, w, x, mean, rstd, gamma, dres, dtmp, dres_b, dgamma, dbeta, dbias, fuse: bool) -> None:
    """dres += LN_bwd(dy @ W^T) (nn.py:35-40 backward through the layer W feeds): one LN-fused GEMM,
    or the dX GEMM then the standalone LayerNorm backward."""
    if fuse:
        K.linear_dx_ln(dy, w, x=x, mean=mean, rstd=rstd, gamma=gamma, dres=dres, accumulate=True, dres_bf16=dres_b,
                       dgamma=dgamma, dbeta=dbeta, dbias=dbias)
        return
    K.linear_dx(dy, w, epilogue=L.EPI_BF16, out=dtmp)
    K.layernorm_bwd(x, mean, rstd, gamma, dtmp, dres, accumulate=True, dres_bf16=dres_b, dgamma=dgamma, dbeta=dbeta,
                    dbias=dbias)


def _qkv_param_grads(dqkv: torch.Tensor, xn: torch.Tensor, G: dict, base: str, d: int, st=None,
                     bias_done: bool = False) -> None:
    """bias_done: the attention backward already wrote the fused bias gradient (its colsum partials)."""
    if st is not None:
        gw = st.block_of(st.grad_flat, f"{base}.q.w")
        gb = st.block_of(st.grad_flat, f"{base}.q.b")
        if gw is not None and gb is not None:  # one (d, 3d) dW GEMM, bias sums straight into place
            if not bias_done:
                K.colsum_bf16(dqkv, gb)
            K.linear_dw(xn, dqkv, gw)
            return
    bq = torch.empty(3 * d, dtype=K.F32, device=dqkv.device)
    K.colsum_bf16(dqkv, bq)
    for j, proj in enumerate("qkv"):
        G[f"{base}.{proj}.b"].copy_(bq[j * d:(j + 1) * d])
        K.linear_dw(xn, dqkv[:, j * d:(j + 1) * d], G[f"{base}.{proj}.w"], n_cols=d)
