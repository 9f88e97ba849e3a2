"""Thin torch-facing wrappers over the libjz C ABI (include/jz.h).

Every function here takes device torch tensors, validates shapes/dtypes on the
host, and issues exactly one C-ABI call (or a fixed small sequence) on the
current CUDA stream.  torch is used only for device memory and streams; all
arithmetic happens in libjz's sm_100a kernels.  There is no fallback path.
"""
from __future__ import annotations

import os
import threading

import torch

from . import _lib as L

BF16 = torch.bfloat16
F32 = torch.float32


def _s() -> int:
    return L.stream_ptr()


def _p(t):
    return None if t is None else t.data_ptr()


# --------------------------------------------------------------------------
# scratch buffers (stream-ordered reuse; one set per device)
# --------------------------------------------------------------------------
class _Scratch(threading.local):
    def __init__(self):
        self.bufs: dict = {}


_scratch = _Scratch()


def scratch(name: str, numel: int, dtype=F32, device=None) -> torch.Tensor:
    """A reusable device buffer of at least `numel` elements (contents undefined)."""
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = (name, dtype, dev)
    buf = _scratch.bufs.get(key)
    if buf is None or buf.numel() < numel:
        buf = torch.empty(max(numel, 1), dtype=dtype, device=dev)
        _scratch.bufs[key] = buf
    return buf[:numel]


def release_scratch() -> None:
    """Drop every cached scratch buffer of this thread (they are re-created on demand)."""
    _scratch.bufs.clear()


def num_sms() -> int:
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


# --------------------------------------------------------------------------
# K1 GEMM
# --------------------------------------------------------------------------
class KernelTimer:
    """CUDA-event timing of every GEMM launch while active (roofline evidence for bench.py), plus
    per-family event pairs with algorithmic FLOPs and bytes for the attention kernels."""

    def __init__(self):
        self.active = False
        self.events: list = []
        self.flops = 0
        self.launches = 0
        self.families: dict = {}  # name -> {"events": [(e0, e1)], "flops": int, "bytes": int}

    def ms(self) -> float:
        return sum(a.elapsed_time(b) for a, b in self.events)

    def family_ms(self, name: str) -> float:
        return sum(a.elapsed_time(b) for a, b in self.families[name]["events"])


TIMER: KernelTimer | None = None
# LayerNorm fused into the GEMM epilogues where the shapes allow (JZ_LN_FUSION=0 runs the standalone
# LayerNorm kernels instead: A/B comparisons and the parity tests of both paths)
LN_FUSION = os.environ.get("JZ_LN_FUSION", "1") != "0"


def _fam_begin():
    if TIMER is None or not TIMER.active:
        return None
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    return e0


def _fam_end(e0, name: str, flops: int, nbytes: int) -> None:
    if e0 is None:
        return
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record()
    f = TIMER.families.setdefault(name, {"events": [], "flops": 0, "bytes": 0})
    f["events"].append((e0, e1))
    f["flops"] += int(flops)
    f["bytes"] += int(nbytes)


def gemm(A: torch.Tensor, B: torch.Tensor, *, M: int, N: int, K: int, a_kmajor: bool, b_kmajor: bool,
         out: torch.Tensor, epilogue: int, bias: torch.Tensor | None = None, aux: torch.Tensor | None = None,
         out2: torch.Tensor | None = None, split_k: int = 1, lda: int | None = None, ldb: int | None = None,
         ldd: int | None = None, ldaux: int | None = None, ldd2: int | None = None,
         colsum: torch.Tensor | None = None, colsum_accumulate: bool = False) -> torch.Tensor:
    """out = epilogue(A . B); see include/jz.h for operand layouts.

    colsum (fp32 [N]): also the column sums of the bf16 output (bias gradient of its consumer),
    reduced from per-32-row partials the epilogue writes (jz_gemm_bf16_colsum)."""
    assert A.dtype == BF16 and B.dtype == BF16, "GEMM operands must be bf16"
    lda = lda if lda is not None else A.stride(0)
    ldb = ldb if ldb is not None else B.stride(0)
    ldd = ldd if ldd is not None else out.stride(0)
    ws = None
    if split_k > 1:
        nbytes = L.load().jz_gemm_workspace_bytes(M, N, split_k)
        ws = scratch("gemm_splitk", nbytes // 4 + 1)
    timed = TIMER is not None and TIMER.active
    if timed:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
    la = ldaux if ldaux is not None else (aux.stride(0) if aux is not None else 0)
    l2 = ldd2 if ldd2 is not None else (out2.stride(0) if out2 is not None else 0)
    if colsum is not None:
        nparts = L.load().jz_gemm_colsum_parts(M)
        part = scratch("gemm_colsum", nparts * N)
        L.call("jz_gemm_bf16_colsum", A.data_ptr(), lda, int(a_kmajor), B.data_ptr(), ldb, int(b_kmajor),
               out.data_ptr(), ldd, M, N, K, epilogue, _p(bias), _p(aux), la, _p(out2), l2, part.data_ptr(), _s())
    else:
        L.call("jz_gemm_bf16", A.data_ptr(), lda, int(a_kmajor), B.data_ptr(), ldb, int(b_kmajor), out.data_ptr(),
               ldd, M, N, K, epilogue, _p(bias), _p(aux), la, _p(out2), l2, split_k, _p(ws), _s())
    if timed:
        e1.record()
        TIMER.events.append((e0, e1))
        TIMER.flops += 2 * M * N * K
        TIMER.launches += 1
    if colsum is not None:
        reduce_partials(part, nparts, N, colsum, colsum_accumulate)
    return out


def splitk_for(m_out: int, n_out: int, k: int) -> int:
    """Split-K for long-K GEMMs (dW): the smallest split whose work units fill the persistent grid's
    waves to >= 85% (fewer splits = fewer fp32 partials and longer pipelined K runs; measured: one
    86%-full wave beats two 97%-full ones).  Mirrors the kernel's tiling: CTA pairs with 256 x 256 tiles when N > 128 and
    M > 128 (num_sms / 2 workers), otherwise single CTAs with 128-row tiles."""
    bn = 256 if n_out > 128 else (128 if n_out > 64 else 64)
    pair = bn == 256 and m_out > 128
    tm = 256 if pair else 128
    workers = num_sms() // 2 if pair else num_sms()
    tiles = -(-m_out // tm) * -(-n_out // bn)
    kb = -(-k // 64)
    best, best_eff = 1, 0.0
    for sp in range(1, min(kb, 64) + 1):
        units = tiles * sp
        waves = -(-units // workers)
        eff = units / (waves * workers)
        if kb // sp < 8:  # keep >= 8 k-blocks per unit (pipeline fill)
            break
        if eff >= 0.85:
            return sp
        if eff > best_eff + 1e-9:
            best, best_eff = sp, eff
    return best


def linear_fwd(x_bf16: torch.Tensor, w_bf16: torch.Tensor, bias: torch.Tensor | None, *, epilogue=L.EPI_BF16,
               out=None, aux=None, out2=None) -> torch.Tensor:
    """y = x @ W (+b), W stored (din, dout) as the reference (nn.py:43-47)."""
    M, K = x_bf16.shape
    N = w_bf16.shape[1]
    if out is None:
        dt = BF16 if epilogue in (L.EPI_BF16, L.EPI_GELU, L.EPI_GELU_BWD, L.EPI_GELU_DG, L.EPI_MUL_F16) else F32
        out = torch.empty(M, N, dtype=dt, device=x_bf16.device)
    return gemm(x_bf16, w_bf16, M=M, N=N, K=K, a_kmajor=True, b_kmajor=False, out=out, epilogue=epilogue,
                bias=bias, aux=aux, out2=out2)


def linear_dx(dy_bf16: torch.Tensor, w_bf16: torch.Tensor, *, epilogue=L.EPI_F32, out=None, aux=None,
              out2=None, colsum=None) -> torch.Tensor:
    """dx = dy @ W^T  (W (din, dout) row-major is K-major for this product)."""
    M, N = dy_bf16.shape
    K_in = w_bf16.shape[0]
    if out is None:
        dt = BF16 if epilogue in (L.EPI_BF16, L.EPI_GELU_BWD, L.EPI_MUL_F16) else F32
        out = torch.empty(M, K_in, dtype=dt, device=dy_bf16.device)
    return gemm(dy_bf16, w_bf16, M=M, N=K_in, K=N, a_kmajor=True, b_kmajor=True, out=out, epilogue=epilogue,
                aux=aux, out2=out2, ldb=w_bf16.stride(0), colsum=colsum)


def _timed_call(name: str, flops: int, *args) -> None:
    timed = TIMER is not None and TIMER.active
    if timed:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
    L.call(name, *args)
    if timed:
        e1.record()
        TIMER.events.append((e0, e1))
        TIMER.flops += flops
        TIMER.launches += 1


LN_FUSED_N = 512  # the LayerNorm-fused GEMM epilogues own 512-wide rows (two 256-column pair tiles)
# Measured policy (tools/check_ln_fused.py, M = 148032): the fused forward wins where the GEMM itself
# is short (K = 512 residual projections: 176 vs 209 us per launch) and loses at K = 2048 (373 vs
# 330 us: the epilogue's staging tiles leave four operand stages and half of its work exposed);
# the fused backward loses at K = 1536 / 2048 (481 / 548 vs 404 / 452 us), so it runs only when
# JZ_LN_FUSION_BWD=1.
LN_FUSED_FWD_MAX_K = 512
LN_FUSION_BWD = os.environ.get("JZ_LN_FUSION_BWD", "0") == "1"


def ln_fusable(M: int, N: int, K: int | None = None, backward: bool = False) -> bool:
    if not (LN_FUSION and N == LN_FUSED_N and M > 128):
        return False
    if backward:
        return LN_FUSION_BWD
    return K is None or K <= LN_FUSED_FWD_MAX_K


def linear_fwd_ln(x_bf16: torch.Tensor, w_bf16: torch.Tensor, bias: torch.Tensor, resid: torch.Tensor,
                  gamma: torch.Tensor, beta: torch.Tensor, *, eps: float = 1e-5, skip_period: int = 0):
    """Residual projection + the next LayerNorm in one GEMM (jz_gemm_bf16_ln_fwd, N = 512):
    -> (x f32 = resid + x_bf16 @ W + b, LN(x) bf16 (rows compacted by skip_period), mean, rstd)."""
    M, K = x_bf16.shape
    N = w_bf16.shape[1]
    dev = x_bf16.device
    out = torch.empty(M, N, dtype=F32, device=dev)
    out_rows = M - (M // skip_period if skip_period else 0)
    xn = torch.empty(out_rows, N, dtype=BF16, device=dev)
    mean = torch.empty(M, dtype=F32, device=dev)
    rstd = torch.empty(M, dtype=F32, device=dev)
    _timed_call("jz_gemm_bf16_ln_fwd", 2 * M * N * K, x_bf16.data_ptr(), x_bf16.stride(0), 1, w_bf16.data_ptr(),
                w_bf16.stride(0), 0, out.data_ptr(), N, M, N, K, bias.data_ptr(), resid.data_ptr(), resid.stride(0),
                gamma.data_ptr(), beta.data_ptr(), eps, xn.data_ptr(), mean.data_ptr(), rstd.data_ptr(), skip_period,
                _s())
    return out, xn, mean, rstd


def linear_dx_ln(dy_bf16: torch.Tensor, w_bf16: torch.Tensor, *, x: torch.Tensor, mean: torch.Tensor,
                 rstd: torch.Tensor, gamma: torch.Tensor, dres: torch.Tensor, accumulate: bool = True,
                 dres_bf16: torch.Tensor | None = None, dgamma=None, dbeta=None, dbias=None) -> None:
    """Input gradient of a LayerNorm-fed layer + the LayerNorm backward in one GEMM
    (jz_gemm_bf16_ln_bwd): dres (+)= LN_bwd(dy_bf16 @ W^T); dgamma / dbeta / dbias (colsum of dres)."""
    M, Nout = dy_bf16.shape
    K_in = w_bf16.shape[0]
    nparts = L.load().jz_gemm_ln_bwd_parts(M)
    part = scratch("ln_gemm_part", 3 * nparts * K_in)
    _timed_call("jz_gemm_bf16_ln_bwd", 2 * M * K_in * Nout, dy_bf16.data_ptr(), dy_bf16.stride(0), 1,
                w_bf16.data_ptr(), w_bf16.stride(0), 1, M, K_in, Nout, x.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                gamma.data_ptr(), dres.data_ptr(), int(accumulate), _p(dres_bf16), part.data_ptr(), nparts,
                _p(dgamma), _p(dbeta), _p(dbias), _s())


def linear_dw(x_bf16: torch.Tensor, dy_bf16: torch.Tensor, out_f32: torch.Tensor, *, accumulate=False,
              n_cols: int | None = None) -> torch.Tensor:
    """dW = x^T @ dy  -> out_f32 (din, dout); dy may be a column slice (n_cols, row pitch = stride)."""
    Mtok, K_in = x_bf16.shape
    N = n_cols if n_cols is not None else dy_bf16.shape[1]
    split = splitk_for(K_in, N, Mtok)
    return gemm(x_bf16, dy_bf16, M=K_in, N=N, K=Mtok, a_kmajor=False, b_kmajor=False, out=out_f32,
                epilogue=L.EPI_F32_ACC if accumulate else L.EPI_F32, split_k=split, lda=x_bf16.stride(0),
                ldb=dy_bf16.stride(0), ldd=out_f32.stride(0))


# --------------------------------------------------------------------------
# reductions / casts
# --------------------------------------------------------------------------
def row_partials(rows: int) -> int:
    return L.load().jz_row_partials(rows)


def colsum_bf16(x: torch.Tensor, out: torch.Tensor, *, cols: int | None = None, accumulate=False) -> torch.Tensor:
    rows = x.shape[0]
    cols = cols if cols is not None else x.shape[1]
    npart = row_partials(rows)
    part = scratch("colsum_part", npart * cols)
    L.call("jz_colsum_bf16", x.data_ptr(), rows, cols, x.stride(0), part.data_ptr(), npart, _s())
    L.call("jz_reduce_partials", part.data_ptr(), npart, cols, out.data_ptr(), int(accumulate), _s())
    return out


def reduce_partials(part: torch.Tensor, nparts: int, D: int, out: torch.Tensor, accumulate=False) -> None:
    L.call("jz_reduce_partials", part.data_ptr(), nparts, D, out.data_ptr(), int(accumulate), _s())


def cast_bf16(src: torch.Tensor, dst: torch.Tensor | None = None) -> torch.Tensor:
    """2-D (or 1-D) fp32 -> bf16; dst may be a column slice of a wider matrix."""
    if src.dim() == 1:
        src2 = src.view(1, -1)
    else:
        src2 = src
    rows, cols = src2.shape
    if dst is None:
        dst = torch.empty(rows, cols, dtype=BF16, device=src.device)
    dst2 = dst.view(1, -1) if dst.dim() == 1 else dst
    L.call("jz_cast_f32_bf16_2d", src2.data_ptr(), src2.stride(0), dst2.data_ptr(), dst2.stride(0), rows, cols, _s())
    return dst


# --------------------------------------------------------------------------
# K2 LayerNorm
# --------------------------------------------------------------------------
def layernorm_fwd(x: torch.Tensor, g: torch.Tensor, b: torch.Tensor, *, skip_period: int = 0, eps: float = 1e-5,
                  out_f32: bool = False, out_bf16: bool = True):
    """-> (y_bf16 or None, mean, rstd) or (y_bf16, y_f32, mean, rstd) when out_f32."""
    rows, D = x.shape
    out_rows = rows - (rows // skip_period if skip_period else 0)
    y = torch.empty(out_rows, D, dtype=BF16, device=x.device) if out_bf16 else None
    y32 = torch.empty(out_rows, D, dtype=F32, device=x.device) if out_f32 else None
    mean = torch.empty(rows, dtype=F32, device=x.device)
    rstd = torch.empty(rows, dtype=F32, device=x.device)
    L.call("jz_layernorm_fwd", x.data_ptr(), rows, D, g.data_ptr(), b.data_ptr(), eps, _p(y), _p(y32),
           mean.data_ptr(), rstd.data_ptr(), skip_period, _s())
    if out_f32:
        return y, y32, mean, rstd
    return y, mean, rstd


def layernorm_bwd(x, mean, rstd, g, dy, dres, *, accumulate: bool, dres_bf16=None, dgamma=None, dbeta=None,
                  dbias=None, skip_period: int = 0, acc_params: bool = False):
    """dres = (accumulate ? dres : 0) + LN'(dy); reduces dgamma/dbeta/dbias(=colsum dres) into the given outs."""
    rows, D = x.shape
    npart = row_partials(rows)
    part = scratch("ln_part", 3 * npart * D)
    pg = part[: npart * D] if dgamma is not None else None
    pb = part[npart * D: 2 * npart * D] if dbeta is not None else None
    pz = part[2 * npart * D:] if dbias is not None else None
    L.call("jz_layernorm_bwd_bf16dy" if dy.dtype == BF16 else "jz_layernorm_bwd", x.data_ptr(), mean.data_ptr(),
           rstd.data_ptr(), g.data_ptr(), dy.data_ptr(),
           dres.data_ptr(), int(accumulate), _p(dres_bf16), _p(pg), _p(pb), _p(pz), npart, rows, D, skip_period,
           _s())
    if dgamma is not None or dbeta is not None or dbias is not None:  # one launch for the three reductions
        L.call("jz_reduce_partials3", _p(pg), _p(pb), _p(pz), npart, D, _p(dgamma), _p(dbeta), _p(dbias),
               int(acc_params), _s())


# --------------------------------------------------------------------------
# attention
# --------------------------------------------------------------------------
SMALL_S = 32  # spatial sequence lengths served by the register-tile kernel (K3s)


def attn_spatial_fwd(qkv: torch.Tensor, frames: int, S: int, H: int, keep_lo: bool = True):
    """-> (out bf16, out_lo bf16 or None, lse).  out_lo = O - bf16(O), the rounding residual of the fp32
    output (out + out_lo carries O to ~16 mantissa bits for the backward's Delta).  S <= 32 runs the
    register-tile kernel (K3s), whose backward forms Delta from its in-register P and dP: no residual."""
    D = H * 64
    out = torch.empty(frames * S, D, dtype=BF16, device=qkv.device)
    if S <= SMALL_S:
        lse = torch.empty(frames, H, S, dtype=F32, device=qkv.device)
        e0 = _fam_begin()
        L.call("jz_attn_spatial_small_fwd", qkv.data_ptr(), frames, S, H, 64, out.data_ptr(), lse.data_ptr(), _s())
        _fam_end(e0, "spatial_small_fwd", 4 * frames * H * S * S * 64, frames * S * (3 * D * 2 + D * 2 + H * 4))
        return out, None, lse
    out_lo = torch.empty(frames * S, D, dtype=BF16, device=qkv.device) if keep_lo else None
    lse = torch.empty(frames, H, S, dtype=F32, device=qkv.device)
    e0 = _fam_begin()
    L.call("jz_attn_spatial_fwd", qkv.data_ptr(), frames, S, H, 64, out.data_ptr(), _p(out_lo), lse.data_ptr(), _s())
    # algorithmic work: QK^T and PV over S x S per (frame, head); qkv in, O bf16 (+ residual) and lse out
    _fam_end(e0, "spatial_fwd", 4 * frames * H * S * S * 64,
             frames * S * (3 * D * 2 + D * 2 + (D * 2 if keep_lo else 0) + H * 4))
    return out, out_lo, lse


def attn_spatial_bwd(qkv, out, dout, lse, frames: int, S: int, H: int, dqkv=None, colsum=None, out_lo=None):
    """colsum (fp32 [3*H*64], optional): also the column sums of dqkv (QKV bias gradient).
    out: the forward's bf16 output; out_lo: its residual (required for S in {256, 257})."""
    if dqkv is None:
        dqkv = torch.empty_like(qkv)
    if S <= SMALL_S:
        if out.dtype != BF16:
            raise ValueError("small-frame spatial attention backward takes the bf16 forward output")
        part, nparts = None, 0
        if colsum is not None:
            nparts = frames
            part = scratch("attn_colsum", nparts * 3 * H * 64)
        e0 = _fam_begin()
        L.call("jz_attn_spatial_small_bwd", qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), frames,
               S, H, 64, dqkv.data_ptr(), _p(part), _s())
        D = H * 64
        _fam_end(e0, "spatial_small_bwd", 10 * frames * H * S * S * 64, frames * S * (3 * D * 2 + D * 2 + 3 * D * 2))
        if colsum is not None:
            reduce_partials(part, nparts, 3 * H * 64, colsum)
        return dqkv
    if out_lo is None:
        raise ValueError("spatial attention backward needs the forward's residual (attn_spatial_fwd(keep_lo=True))")
    ws = scratch("attn_uvb", L.load().jz_attn_spatial_bwd_workspace_bytes(frames, S, H) // 4)
    part, nparts = None, 0
    if colsum is not None:
        nparts = L.load().jz_attn_spatial_colsum_parts(frames)
        part = scratch("attn_colsum", nparts * 3 * H * 64)
    e0 = _fam_begin()
    L.call("jz_attn_spatial_bwd", qkv.data_ptr(), out.data_ptr(), out_lo.data_ptr(), dout.data_ptr(), lse.data_ptr(),
           frames, S, H, 64, dqkv.data_ptr(), ws.data_ptr(), _p(part), _s())
    # 2.5x the forward FLOPs (S, dP, dV, dK, dQ); bytes: qkv, dO (twice: Delta pass + MMAs), O + residual in, dqkv out
    D = H * 64
    _fam_end(e0, "spatial_bwd", 10 * frames * H * S * S * 64, frames * S * (3 * D * 2 + 2 * D * 2 + 2 * D * 2 + 3 * D * 2))
    if colsum is not None:
        reduce_partials(part, nparts, 3 * H * 64, colsum)
    return dqkv


def attn_temporal_fwd(qkv: torch.Tensor, B: int, T: int, S: int, H: int):
    D = H * 64
    out = torch.empty(B * T * S, D, dtype=BF16, device=qkv.device)
    lse = torch.empty(B * S, H, T, dtype=F32, device=qkv.device)
    e0 = _fam_begin()
    L.call("jz_attn_temporal_fwd", qkv.data_ptr(), B, T, S, H, 64, out.data_ptr(), lse.data_ptr(), _s())
    # causal pairs only: QK^T and PV over T (T + 1) / 2 pairs per (b, s, head)
    _fam_end(e0, "temporal_fwd", 2 * 2 * 64 * B * S * H * (T * (T + 1) // 2), B * T * S * (3 * D * 2 + D * 2 + H * 4))
    return out, lse


def attn_temporal_bwd(qkv, out, dout, lse, B: int, T: int, S: int, H: int, dqkv=None, colsum=None):
    """colsum (fp32 [3*H*64], optional): also the column sums of dqkv (QKV bias gradient)."""
    if dqkv is None:
        dqkv = torch.empty_like(qkv)
    part, nparts = None, 0
    if colsum is not None:
        nparts = L.load().jz_attn_temporal_colsum_parts_t(B, S, T, H)
        part = scratch("attn_colsum", nparts * 3 * H * 64)
    e0 = _fam_begin()
    L.call("jz_attn_temporal_bwd", qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), B, T, S, H, 64,
           dqkv.data_ptr(), _p(part), _s())
    D = H * 64
    # bytes: qkv and dO in, dqkv out (Delta comes from the in-register P and dP: O is not read)
    _fam_end(e0, "temporal_bwd", 10 * 64 * B * S * H * (T * (T + 1) // 2),
             B * T * S * (3 * D * 2 + D * 2 + 3 * D * 2))
    if colsum is not None:
        reduce_partials(part, nparts, 3 * H * 64, colsum)
    return dqkv


# --------------------------------------------------------------------------
# dynamics input side, masks, CE, AdamW
# --------------------------------------------------------------------------
# (philox state int64[11], AdamW scalars f32[9]) device buffers while a training step is being
# captured into a CUDA graph: the mask and optimizer launches then read the step's values from
# device memory, which the graph's owner refreshes before every replay (trainer.GraphedTrainStep)
DEVSTATE: tuple | None = None


def philox_mask(state, B_global: int, b0: int, B_local: int, T: int, N: int, mask_limit: float,
                mask_out: torch.Tensor, count_out: torch.Tensor) -> None:
    """state: rng.PhiloxState (host).  count_out must be zeroed (int32 device scalar)."""
    import ctypes as C
    if DEVSTATE is not None:
        L.call("jz_philox_mask_dev", DEVSTATE[0].data_ptr(), B_global, b0, B_local, T, N, float(mask_limit),
               mask_out.data_ptr(), count_out.data_ptr(), _s())
        return
    ctr = (C.c_uint64 * 4)(*state.counter)
    key = (C.c_uint64 * 2)(*state.key)
    buf = (C.c_uint64 * 4)(*state.buffer)
    L.call("jz_philox_mask", C.addressof(ctr), C.addressof(key), C.addressof(buf), state.buffer_pos, B_global, b0,
           B_local, T, N, float(mask_limit), mask_out.data_ptr(), count_out.data_ptr(), _s())


def dyn_embed_fwd(tokens, mask, latents, P: dict, *, B, T, N, D, dl, K, prepend, err):
    S = N + (1 if prepend else 0)
    x = torch.empty(B * T * S, D, dtype=F32, device=tokens.device)
    L.call("jz_dyn_embed_fwd", tokens.data_ptr(), _p(mask), _p(latents), P["token_embed"].data_ptr(),
           P["mask_token"].data_ptr(), P["null_action"].data_ptr(), P["action_proj.w"].data_ptr(),
           P["action_proj.b"].data_ptr(), P["pos_spatial"].data_ptr(), P["pos_temporal"].data_ptr(), B, T, N, D,
           dl, K, int(prepend), x.data_ptr(), err.data_ptr(), _s())
    return x


def dyn_embed_bwd(dx, tokens, mask, latents, P: dict, G: dict, *, B, T, N, D, dl, K, prepend, d_latents=None):
    nws = L.load().jz_dyn_embed_bwd_workspace(B, T, N, D, dl, int(prepend), K)
    ws = scratch("embed_ws", nws)
    L.call("jz_dyn_embed_bwd", dx.data_ptr(), tokens.data_ptr(), _p(mask), _p(latents),
           P["null_action"].data_ptr(), P["action_proj.w"].data_ptr(), B, T, N, D, dl, K, int(prepend),
           G["token_embed"].data_ptr(), G["mask_token"].data_ptr(), G["null_action"].data_ptr(),
           G["action_proj.w"].data_ptr(), G["action_proj.b"].data_ptr(), G["pos_spatial"].data_ptr(),
           G["pos_temporal"].data_ptr(), _p(d_latents), ws.data_ptr(), _s())


def embedding_table_bwd(dout: torch.Tensor, ids: torch.Tensor, dtable: torch.Tensor, accumulate: bool = False,
                        err: torch.Tensor | None = None) -> None:
    """dtable[k] (=|+=) sum_{ids[i]==k} dout[i] in index order (autodiff.py:344-364 embedding backward)."""
    Kt, D = dtable.shape
    if not dtable.is_contiguous():
        raise ValueError("embedding_table_bwd: the table gradient must be contiguous")
    ids = ids.reshape(-1).to(torch.int64).contiguous()
    dout = dout.reshape(ids.numel(), D).to(F32).contiguous()
    L.call("jz_embedding_table_bwd", dout.data_ptr(), ids.data_ptr(), ids.numel(), Kt, D, dtable.data_ptr(),
           int(accumulate), _p(err), _s())


def ce_fwd_bwd(logits: torch.Tensor, targets: torch.Tensor, mask: torch.Tensor | None, count: torch.Tensor,
               grad_scale: float = 1.0):
    rows, K = logits.shape
    dlogits = torch.empty(rows, K, dtype=BF16, device=logits.device)
    row_loss = scratch("ce_rowloss", rows)
    loss = torch.empty((), dtype=F32, device=logits.device)
    L.call("jz_ce_fwd_bwd", logits.data_ptr(), rows, K, targets.data_ptr(), _p(mask), count.data_ptr(),
           float(grad_scale), dlogits.data_ptr(), row_loss.data_ptr(), loss.data_ptr(), _s())
    return loss, dlogits


def finite_check(g: torch.Tensor, flag: torch.Tensor) -> None:
    L.call("jz_finite_check", g.data_ptr(), g.numel(), flag.data_ptr(), _s())


def adamw(p, g, m, v, *, lr, b1, b2, omb1, omb2, bc1, bc2, eps, lrwd, flag=None) -> None:
    """K13 over p[0..numel): every operand must be one dense contiguous block."""
    for name, t in (("param", p), ("grad", g), ("m", m), ("v", v)):
        if not t.is_contiguous() or t.numel() != p.numel():
            raise ValueError(f"adamw: {name} must be contiguous with {p.numel()} elements")
    if DEVSTATE is not None:
        L.call("jz_adamw_step_dev", p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), p.numel(),
               DEVSTATE[1].data_ptr(), _p(flag), _s())
        return
    L.call("jz_adamw_step", p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), p.numel(), lr, b1, b2, omb1,
           omb2, bc1, bc2, eps, lrwd, _p(flag), _s())


# --------------------------------------------------------------------------
# tokenizer / LAM side
# --------------------------------------------------------------------------
def patchify(frames: torch.Tensor, P: int, *, bf16=True, f32=False):
    """frames uint8 or fp32 (BT, H, W, C) -> (patches bf16 [BT*N, P*P*C] or None, fp32 or None)."""
    BT, H, W, C = frames.shape
    N, PD = (H // P) * (W // P), P * P * C
    o16 = torch.empty(BT * N, PD, dtype=BF16, device=frames.device) if bf16 else None
    o32 = torch.empty(BT * N, PD, dtype=F32, device=frames.device) if f32 else None
    L.call("jz_patchify", frames.data_ptr(), int(frames.dtype == torch.uint8), BT, H, W, C, P, _p(o16), _p(o32), _s())
    return o16, o32


def unpatchify(patches: torch.Tensor, BT: int, H: int, W: int, C: int, P: int, *, unit=True, u8=False):
    un = torch.empty(BT, H, W, C, dtype=F32, device=patches.device) if unit else None
    fr = torch.empty(BT, H, W, C, dtype=torch.uint8, device=patches.device) if u8 else None
    L.call("jz_unpatchify", patches.data_ptr(), BT, H, W, C, P, _p(un), _p(fr), _s())
    return un, fr


def assemble_fwd(emb, act, ps, pt, *, B, T, N, D, prepend):
    S = N + (1 if prepend else 0)
    x = torch.empty(B * T * S, D, dtype=F32, device=ps.device)
    L.call("jz_assemble_fwd", emb.data_ptr(), _p(act), ps.data_ptr(), pt.data_ptr(), B, T, N, D, int(prepend),
           x.data_ptr(), _s())
    return x


def assemble_bwd(dx, *, B, T, N, D, prepend, d_emb=None, d_act=None, d_ps=None, d_pt=None):
    nws = L.load().jz_assemble_bwd_workspace(B, T, N, D, int(prepend))
    ws = scratch("assemble_ws", nws)
    L.call("jz_assemble_bwd", dx.data_ptr(), B, T, N, D, int(prepend), _p(d_emb), _p(d_act), _p(d_ps), _p(d_pt),
           ws.data_ptr(), _s())


def mean_pool(x, BT, N, D):
    out = torch.empty(BT, D, dtype=F32, device=x.device)
    L.call("jz_mean_pool", x.data_ptr(), BT, N, D, out.data_ptr(), _s())
    return out


def mean_pool_bwd(dpool, BT, N, D):
    dx = torch.empty(BT * N, D, dtype=F32, device=dpool.device)
    L.call("jz_mean_pool_bwd", dpool.data_ptr(), BT, N, D, dx.data_ptr(), _s())
    return dx


def mse(pred, target, *, grad_scale=1.0, grad32=False, grad16=False):
    n = pred.numel()
    loss = torch.empty((), dtype=F32, device=pred.device)
    g32 = torch.empty_like(pred) if grad32 else None
    g16 = torch.empty(pred.shape, dtype=BF16, device=pred.device) if grad16 else None
    ws = scratch("mse_ws", 4 * num_sms(), dtype=torch.float64)
    L.call("jz_mse", pred.data_ptr(), target.data_ptr(), n, float(grad_scale), loss.data_ptr(), _p(g32), _p(g16),
           ws.data_ptr(), _s())
    return loss, g32, g16


def linear_f32(x, W, b=None, out=None, accumulate=False):
    R, Kd = x.shape
    N = W.shape[1]
    if out is None:
        out = torch.empty(R, N, dtype=F32, device=x.device)
    L.call("jz_linear_f32", x.data_ptr(), R, Kd, W.data_ptr(), N, _p(b), out.data_ptr(), int(accumulate), _s())
    return out


def linear_f32_bwd(x, dy, W, *, dx=None, dW=None, db=None, accumulate=False):
    R, Kd = x.shape
    N = W.shape[1]
    need = L.load().jz_linear_f32_bwd_workspace(R, Kd, N)
    ws = scratch("linear_f32_bwd", need) if need > 0 else None
    L.call("jz_linear_f32_bwd_ws", x.data_ptr(), dy.data_ptr(), R, Kd, N, W.data_ptr(), _p(dx), _p(dW), _p(db),
           int(accumulate), _p(ws), need, _s())


def vq_fwd(z: torch.Tensor, codebook: torch.Tensor):
    """z f32 [rows, dz] -> (idx int64 [rows], zq_st f32 [rows, dz], row_sq f32 [rows])."""
    rows, dz = z.shape
    idx = torch.empty(rows, dtype=torch.int64, device=z.device)
    zq = torch.empty_like(z)
    sq = torch.empty(rows, dtype=F32, device=z.device)
    L.call("jz_vq_fwd", z.data_ptr(), rows, dz, codebook.data_ptr(), codebook.shape[0], idx.data_ptr(),
           zq.data_ptr(), sq.data_ptr(), _s())
    return idx, zq, sq


def vq_bwd(z, codebook, idx, g_zq_st, *, commit_coef, cb_coef, dz_out=None, dcodebook=None):
    rows, dz = z.shape
    L.call("jz_vq_bwd", z.data_ptr(), codebook.data_ptr(), idx.data_ptr(), _p(g_zq_st), rows, dz, codebook.shape[0],
           float(commit_coef), float(cb_coef), _p(dz_out), _p(dcodebook), _s())


def sum_scaled(x: torch.Tensor, scale: float) -> torch.Tensor:
    """Deterministic fp64-accumulated scale * sum(x) of a device fp32 tensor -> fp32 device scalar."""
    out = torch.empty((), dtype=F32, device=x.device)
    ws = scratch("sum_ws", 4 * num_sms(), dtype=torch.float64)
    L.call("jz_sum", x.data_ptr(), x.numel(), float(scale), out.data_ptr(), ws.data_ptr(), _s())
    return out
