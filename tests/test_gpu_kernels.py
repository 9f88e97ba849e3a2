"""Kernel-level parity of the hand-written sm_100a kernels against plain torch fp32 references.

These are the floating-point kernels of the dynamics step: the tcgen05 GEMM with
every epilogue the model uses, LayerNorm fwd/bwd, spatial (S = 256/257, bidirectional) and temporal
(causal) attention fwd/bwd.  Tolerances are relative Frobenius errors; bf16 operands with fp32
accumulation put GEMM fp32 outputs at ~1e-6 of the fp32 product of the SAME bf16 operands, so the
GEMM bounds are tight, while attention goes through bf16 P/dS tiles (2e-2, as fidelity_threshold.json).
"""
import json
from pathlib import Path
import math

import pytest
import torch

from paper_2510_27002_b200 import _lib as L
from paper_2510_27002_b200 import kernels as Kn

pytestmark = pytest.mark.gpu
TOL = json.loads((Path(__file__).resolve().parent.parent / "fidelity_threshold.json").read_text())["parity"]
dev = "cuda"


def rel(a, b):
    a, b = a.float(), b.float()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def _operands(M, N, K, a_kmajor, b_kmajor, seed):
    g = torch.Generator(device=dev).manual_seed(seed)
    X = torch.randn(M, K, device=dev, generator=g).bfloat16()
    W = torch.randn(K, N, device=dev, generator=g).bfloat16()
    A = X.contiguous() if a_kmajor else X.t().contiguous()
    B = W.t().contiguous() if b_kmajor else W.contiguous()
    return X, W, A, B


@pytest.mark.parametrize("a_kmajor", [1, 0])
@pytest.mark.parametrize("b_kmajor", [0, 1])
@pytest.mark.parametrize("M,N,K", [(256, 256, 128), (296, 200, 192), (128, 64, 64), (1000, 1536, 512), (333, 48, 512)])
def test_gemm_majors_f32(M, N, K, a_kmajor, b_kmajor):
    if (not b_kmajor and N % 8) or (not a_kmajor and M % 8):
        pytest.skip("MN-major operand pitch must be a multiple of 8 elements")
    X, W, A, B = _operands(M, N, K, a_kmajor, b_kmajor, M + N + K)
    bias = torch.randn(N, device=dev)
    ref = X.float() @ W.float() + bias
    D = torch.full((M, N), float("nan"), device=dev)
    Kn.gemm(A, B, M=M, N=N, K=K, a_kmajor=a_kmajor, b_kmajor=b_kmajor, out=D, epilogue=L.EPI_F32, bias=bias,
            lda=K if a_kmajor else M, ldb=K if b_kmajor else N)
    assert rel(D, ref) < 1e-5


@pytest.mark.parametrize("M,N,K,split", [(512, 512, 4096, 4), (504, 296, 2048, 3), (1000, 1536, 2048, 2),
                                         (512, 1536, 20000, 6)])
@pytest.mark.parametrize("acc", [False, True])
def test_gemm_splitk_dw(M, N, K, split, acc):
    """dW = x^T dy form (both operands MN-major), split-K partials + reduction, optional accumulate."""
    X, W, A, B = _operands(M, N, K, 0, 0, K)
    prev = torch.randn(M, N, device=dev)
    D = prev.clone()
    Kn.gemm(A, B, M=M, N=N, K=K, a_kmajor=False, b_kmajor=False, out=D,
            epilogue=L.EPI_F32_ACC if acc else L.EPI_F32, split_k=split, lda=M, ldb=N)
    ref = X.float() @ W.float() + (prev if acc else 0)
    assert rel(D, ref) < 1e-5


@pytest.mark.parametrize("M", [1000, 4096 + 77])
def test_gemm_epilogues(M):
    N, K = 512, 256
    X, W, A, B = _operands(M, N, K, 1, 0, M)
    acc = X.float() @ W.float()
    bias = torch.randn(N, device=dev)
    aux = torch.randn(M, N, device=dev)
    # BF16: y = acc + b, rounded once
    y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    Kn.gemm(A, B, M=M, N=N, K=K, a_kmajor=1, b_kmajor=0, out=y, epilogue=L.EPI_BF16, bias=bias)
    assert rel(y, acc + bias) < 4e-3
    # RESID: out = aux + acc + b (fp32 residual stream)
    r = torch.empty(M, N, device=dev)
    Kn.gemm(A, B, M=M, N=N, K=K, a_kmajor=1, b_kmajor=0, out=r, epilogue=L.EPI_RESID, bias=bias, aux=aux)
    assert rel(r, aux + acc + bias) < 1e-5
    # F32_ACC: out += acc
    r2 = aux.clone()
    Kn.gemm(A, B, M=M, N=N, K=K, a_kmajor=1, b_kmajor=0, out=r2, epilogue=L.EPI_F32_ACC)
    assert rel(r2, aux + acc) < 1e-5
    # GELU: D = gelu(acc + b) bf16, D2 = pre-activation bf16 (tanh form, as nn.gelu); D2 optional
    g = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    pre = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    Kn.gemm(A, B, M=M, N=N, K=K, a_kmajor=1, b_kmajor=0, out=g, epilogue=L.EPI_GELU, bias=bias, out2=pre)
    assert rel(pre, acc + bias) < 4e-3
    assert rel(g, torch.nn.functional.gelu(acc + bias, approximate="tanh")) < TOL["bf16_epilogue_rel"]
    g2 = torch.empty_like(g)
    Kn.gemm(A, B, M=M, N=N, K=K, a_kmajor=1, b_kmajor=0, out=g2, epilogue=L.EPI_GELU, bias=bias)
    assert torch.equal(g2, g)
    # GELU_BWD: D = acc * gelu'(aux_pre) bf16
    pre_aux = (torch.randn(M, N, device=dev) * 2).bfloat16()
    gb = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    Kn.gemm(A, B, M=M, N=N, K=K, a_kmajor=1, b_kmajor=0, out=gb, epilogue=L.EPI_GELU_BWD, aux=pre_aux)
    xp = pre_aux.float().requires_grad_(True)
    torch.nn.functional.gelu(xp, approximate="tanh").backward(acc)
    assert rel(gb, xp.grad) < TOL["bf16_epilogue_rel"]


@pytest.mark.parametrize("M,N", [(1000, 512), (4096 + 77, 2048), (300, 48)])
def test_gemm_gelu_dg_and_mul_epilogues(M, N):
    """GELU_DG: D = gelu(acc + b) bf16 and D2 = gelu'(acc + b) f16 (the training forward);
    MUL_F16: D = acc * aux_f16 (its backward). N = 48 runs the direct (unstaged) epilogue."""
    K = 256
    X, W, A, B = _operands(M, N, K, 1, 0, 7 * M + N)
    # pre-activation 0.25 acc + b (std ~4 plus a +-12 ramp: both clamp sides and the centre)
    A4 = (A.float() * 0.25).bfloat16()  # exact: power-of-two scale
    bias = torch.linspace(-12, 12, N, device=dev)
    pre = (X.float() * 0.25) @ W.float() + bias
    g = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    dg = torch.empty(M, N, device=dev, dtype=torch.float16)
    Kn.gemm(A4, B, M=M, N=N, K=K, a_kmajor=1, b_kmajor=0, out=g, epilogue=L.EPI_GELU_DG, bias=bias, out2=dg)
    xp = pre.clone().requires_grad_(True)
    y = torch.nn.functional.gelu(xp, approximate="tanh")
    y.backward(torch.ones_like(y))
    assert rel(g, y.detach()) < TOL["bf16_epilogue_rel"]
    assert rel(dg, xp.grad) < 4e-3  # f16 tanh.approx: ~2^-11 absolute
    assert (dg.float() - xp.grad).abs().max() < 1.5e-2  # 1 - t^2 from a tanh.approx t near +-1
    # MUL_F16 with the saved derivative: D = acc2 * gelu'
    X2, W2, A2, B2 = _operands(M, N, K, 1, 0, 11 * M + N)
    acc2 = X2.float() @ W2.float()
    gb = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    Kn.gemm(A2, B2, M=M, N=N, K=K, a_kmajor=1, b_kmajor=0, out=gb, epilogue=L.EPI_MUL_F16, aux=dg)
    assert rel(gb, acc2 * dg.float()) < 4e-3


@pytest.mark.parametrize("M,N", [(4096 + 77, 2048), (1000, 512), (96, 1536)])
def test_gemm_colsum_epilogue(M, N):
    """Column sums of the bf16 output (bias gradient of the consumer) from the epilogue partials."""
    K = 256
    X, W, A, B = _operands(M, N, K, 1, 1, M + N)
    pre = (torch.randn(M, N, device=dev) * 2).bfloat16()
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    cs = torch.full((N,), float("nan"), device=dev)
    Kn.gemm(A, B, M=M, N=N, K=K, a_kmajor=1, b_kmajor=1, out=out, epilogue=L.EPI_GELU_BWD, aux=pre, colsum=cs)
    ref = torch.empty_like(cs)
    Kn.colsum_bf16(out, ref)
    assert rel(cs, ref) < 1e-6
    out2 = torch.empty_like(out)
    Kn.gemm(A, B, M=M, N=N, K=K, a_kmajor=1, b_kmajor=1, out=out2, epilogue=L.EPI_GELU_BWD, aux=pre)
    assert torch.equal(out, out2)


def test_gemm_rejects_bad_shapes():
    A = torch.zeros(64, 64, device=dev, dtype=torch.bfloat16)
    D = torch.zeros(64, 64, device=dev)
    with pytest.raises(ValueError):
        Kn.gemm(A, A, M=64, N=64, K=0, a_kmajor=1, b_kmajor=0, out=D, epilogue=L.EPI_F32)


@pytest.mark.parametrize("rows,D,skip", [(4096, 512, 0), (257 * 6, 512, 257), (1000, 256, 0)])
def test_layernorm_fwd_bwd(rows, D, skip):
    g = torch.Generator(device=dev).manual_seed(rows)
    x = torch.randn(rows, D, device=dev, generator=g) * 3 + 1
    gamma = torch.randn(D, device=dev, generator=g)
    beta = torch.randn(D, device=dev, generator=g)
    y, y32, mean, rstd = Kn.layernorm_fwd(x, gamma, beta, skip_period=skip, out_f32=True)
    keep = torch.ones(rows, dtype=torch.bool, device=dev)
    if skip:
        keep[::skip] = False  # skip_period drops row 0 of every period from the outputs
    xr = x.clone().requires_grad_(True)
    ref = torch.nn.functional.layer_norm(xr, (D,), gamma, beta, eps=1e-5)
    assert rel(y32, ref[keep]) < 1e-5
    assert rel(y, ref[keep]) < 4e-3
    dy = torch.randn(int(keep.sum()), D, device=dev, generator=g)
    full_dy = torch.zeros(rows, D, device=dev)
    full_dy[keep] = dy
    ref.backward(full_dy)
    dres = torch.randn(rows, D, device=dev, generator=g)
    dres0 = dres.clone()
    dg, db = torch.zeros(D, device=dev), torch.zeros(D, device=dev)
    Kn.layernorm_bwd(x, mean, rstd, gamma, dy, dres, accumulate=True, dgamma=dg, dbeta=db, skip_period=skip)
    assert rel(dres - dres0, xr.grad) < 1e-5
    gp = torch.nn.functional.layer_norm(x, (D,), eps=1e-5)
    assert rel(dg, (full_dy * gp).sum(0)) < 1e-5
    assert rel(db, full_dy.sum(0)) < 1e-5


def _ref_attn(qkv, lead, L_, H, causal):
    x = qkv.float().reshape(*lead, L_, 3, H, 64)
    q, k, v = (x[..., i, :, :].transpose(-3, -2) for i in range(3))
    s = q @ k.transpose(-1, -2) / math.sqrt(64)
    if causal:
        s = s.masked_fill(torch.triu(torch.ones(L_, L_, dtype=torch.bool, device=dev), 1), float("-inf"))
    o = (torch.softmax(s, -1) @ v).transpose(-3, -2).reshape(*lead, L_, H * 64)
    return o, torch.logsumexp(s, -1)


@pytest.mark.parametrize("S,frames", [(257, 13), (256, 13), (257, 40), (256, 40)])
def test_attn_spatial_fwd_bwd(S, frames):
    """frames = 40: 320 (frame, head) units on 148 CTAs, so every CTA pipelines 2-3 units through the
    backward's staged input release and its per-unit barrier phases."""
    H = 8
    D = H * 64
    g = torch.Generator(device=dev).manual_seed(S)
    qkv = (torch.randn(frames * S, 3 * D, device=dev, generator=g) * 1.5).bfloat16()
    out, out_lo, lse = Kn.attn_spatial_fwd(qkv, frames, S, H, keep_lo=True)
    qf = qkv.float().requires_grad_(True)
    o_ref, lse_ref = _ref_attn(qf.reshape(frames, S, 3 * D), (frames,), S, H, False)
    assert rel(out.reshape(frames, S, D), o_ref) < TOL["attn_out_rel_l2"]
    o_full = (out.float() + out_lo.float()).reshape(frames, S, D)  # the residual carries O past bf16
    assert rel(o_full, o_ref) < TOL["attn_out_rel_l2"]
    assert float((out_lo.float().abs() - out.float().abs() * 2.0 ** -8).clamp_min(0).max()) == 0.0
    assert rel(out.reshape(frames, S, D)[:, -1], o_ref[:, -1]) < TOL["attn_out_rel_l2"]  # the CUDA-core 257th row
    assert rel(lse, lse_ref) < TOL["attn_lse_rel"]
    go = torch.randn(o_ref.shape, device=dev, generator=g)
    o_ref.backward(go)
    dqkv = torch.full_like(qkv, float("nan"))
    cs = torch.full((3 * D,), float("nan"), device=dev)
    Kn.attn_spatial_bwd(qkv, out, go.reshape(frames * S, D).bfloat16().contiguous(), lse, frames, S, H, dqkv=dqkv,
                        colsum=cs, out_lo=out_lo)
    assert torch.isfinite(dqkv.float()).all()
    cs_ref = torch.empty_like(cs)
    Kn.colsum_bf16(dqkv, cs_ref)  # fused bias-gradient column sums == a pass over the written dqkv
    # q / v: the column sums of the written dq / dv; k: exactly 0 (every dS row sums to 0 over the
    # S keys, so a bias shared by all keys has no gradient), the summed written dk is rounding noise
    assert rel(cs[:D], cs_ref[:D]) < TOL["fp32_kernel_rel_l2"] and rel(cs[2 * D:], cs_ref[2 * D:]) < TOL["fp32_kernel_rel_l2"]
    assert float(cs[D:2 * D].abs().max()) == 0.0
    assert float(cs_ref[D:2 * D].norm()) < 1e-2 * float(cs_ref[2 * D:].norm()) + 1e-3
    for i in range(3):
        got, ref = dqkv[:, i * D:(i + 1) * D], qf.grad[:, i * D:(i + 1) * D]
        assert rel(got, ref) < TOL["attn_grad_rel_l2"], "qkv"[i]
        assert rel(got.reshape(frames, S, D)[:, -1], ref.reshape(frames, S, D)[:, -1]) < TOL["attn_grad_rel_l2"], "qkv"[i]


@pytest.mark.parametrize("S,frames", [(257, 1), (256, 1), (257, 19), (257, 37), (256, 149)])
def test_attn_spatial_unit_counts(S, frames):
    """Unit counts around the CTA grid (8 heads: 8 .. 1192 units on 148 CTAs, so CTAs run 0 to 9
    units and the K / V slots, the alternating tile epilogues and the tail warps wrap several
    times): forward (with and without the residual) and backward against torch fp32."""
    H = 8
    D = H * 64
    g = torch.Generator(device=dev).manual_seed(S * 1000 + frames)
    qkv = (torch.randn(frames * S, 3 * D, device=dev, generator=g) * 1.5).bfloat16()
    out, out_lo, lse = Kn.attn_spatial_fwd(qkv, frames, S, H, keep_lo=True)
    out2, _, lse2 = Kn.attn_spatial_fwd(qkv, frames, S, H, keep_lo=False)
    assert torch.equal(out, out2) and torch.equal(lse, lse2)
    qf = qkv.float().requires_grad_(True)
    o_ref, lse_ref = _ref_attn(qf.reshape(frames, S, 3 * D), (frames,), S, H, False)
    assert rel(out.reshape(frames, S, D), o_ref) < TOL["attn_out_rel_l2"]
    assert rel(lse, lse_ref) < TOL["attn_lse_rel"]
    go = torch.randn(o_ref.shape, device=dev, generator=g)
    o_ref.backward(go)
    dqkv = torch.full_like(qkv, float("nan"))
    Kn.attn_spatial_bwd(qkv, out, go.reshape(frames * S, D).bfloat16().contiguous(), lse, frames, S, H, dqkv=dqkv,
                        out_lo=out_lo)
    assert torch.isfinite(dqkv.float()).all()
    for i in range(3):
        assert rel(dqkv[:, i * D:(i + 1) * D], qf.grad[:, i * D:(i + 1) * D]) < TOL["attn_grad_rel_l2"], "qkv"[i]


@pytest.mark.parametrize("S", [257, 256])
def test_attn_spatial_run_to_run_bitwise(S):
    """Spatial attention forward (O, its residual, lse) and backward (dq/dk/dv, bias column sums) are
    bitwise identical across repeated launches with 2-3 units per CTA (no races in the warp-
    specialised pipelines, no float atomics)."""
    H, frames = 8, 40
    D = H * 64
    g = torch.Generator(device=dev).manual_seed(S + 1)
    qkv = (torch.randn(frames * S, 3 * D, device=dev, generator=g) * 1.5).bfloat16()
    dO = torch.randn(frames * S, D, device=dev, generator=g).bfloat16()
    res = []
    for _ in range(3):
        out, olo, lse = Kn.attn_spatial_fwd(qkv, frames, S, H, keep_lo=True)
        dq = torch.empty_like(qkv)
        cs = torch.empty(3 * D, device=dev)
        Kn.attn_spatial_bwd(qkv, out, dO, lse, frames, S, H, dqkv=dq, colsum=cs, out_lo=olo)
        res.append((out.clone(), olo.clone(), lse.clone(), dq.clone(), cs.clone()))
    for r in res[1:]:
        for a_, b_ in zip(res[0], r):
            assert torch.equal(a_, b_)


@pytest.mark.parametrize("S", [257, 256])
def test_attn_spatial_fwd_score_spread(S):
    """Rows whose dominant key lies in a later 64-key chunk, by far more than 2^32 in probability
    (the one-pass forward softmax rescales the probabilities it already wrote), and for S = 257 rows
    dominated by key 256."""
    H, frames = 8, 4
    D = H * 64
    g = torch.Generator(device=dev).manual_seed(7 + S)
    x = torch.randn(frames * S, 3 * D, device=dev, generator=g)
    q = x[:, :D].view(frames, S, H, 64)
    k = x[:, D:2 * D].view(frames, S, H, 64)
    q[0, 0:32, 0] = 4.0   # key 200 (chunk 3) against queries 0..31: scores 128 above the rest
    k[0, 200, 0] = 4.0
    q[1, 100:140, 3] = -3.0  # key 70 (chunk 1) against queries across both query tiles
    k[1, 70, 3] = -3.0
    if S == 257:
        q[2, 5:9, 1] = 4.0  # key 256 (CUDA cores + the PV MMA's 17th K-step)
        k[2, 256, 1] = 4.0
    qkv = x.bfloat16()
    out, out_lo, lse = Kn.attn_spatial_fwd(qkv, frames, S, H, keep_lo=True)
    o_ref, lse_ref = _ref_attn(qkv.float().reshape(frames, S, 3 * D), (frames,), S, H, False)
    assert torch.isfinite(out.float()).all() and torch.isfinite(lse).all()
    assert rel(out.reshape(frames, S, D), o_ref) < TOL["attn_out_rel_l2"]
    assert rel((out.float() + out_lo.float()).reshape(frames, S, D), o_ref) < TOL["attn_out_rel_l2"]
    assert rel(lse, lse_ref) < TOL["attn_lse_rel"]
    for f, rows, h in ((0, slice(0, 32), 0), (1, slice(100, 140), 3)) + (((2, slice(5, 9), 1),) if S == 257 else ()):
        o = out.reshape(frames, S, H, 64)[f, rows, h].float()
        assert rel(o, o_ref.reshape(frames, S, H, 64)[f, rows, h]) < TOL["attn_out_rel_l2"]


@pytest.mark.parametrize("T", [16, 5, 1])
def test_attn_temporal_fwd_bwd(T):
    B, S, H = 2, 257, 8
    D = H * 64
    g = torch.Generator(device=dev).manual_seed(T)
    qkv = (torch.randn(B * T * S, 3 * D, device=dev, generator=g) * 1.5).bfloat16()
    out, lse = Kn.attn_temporal_fwd(qkv, B, T, S, H)
    qf = qkv.float().requires_grad_(True)
    x = qf.reshape(B, T, S, 3 * D).transpose(1, 2)
    o_ref, lse_ref = _ref_attn(x, (B, S), T, H, True)
    assert rel(out.reshape(B, T, S, D).transpose(1, 2), o_ref) < TOL["attn_out_rel_l2"]
    assert rel(lse.reshape(B, S, H, T), lse_ref) < TOL["attn_lse_rel"]
    go = torch.randn(o_ref.shape, device=dev, generator=g)
    o_ref.backward(go)
    dout = go.transpose(1, 2).reshape(B * T * S, D).bfloat16().contiguous()
    cs = torch.full((3 * D,), float("nan"), device=dev)
    dqkv = Kn.attn_temporal_bwd(qkv, out, dout, lse, B, T, S, H, colsum=cs)
    cs_ref = torch.empty_like(cs)
    Kn.colsum_bf16(dqkv, cs_ref)
    # q / v bias gradients are the column sums of the written dq / dv; the key-bias gradient is
    # exactly zero (a bias shared by every key shifts each softmax row by a constant): the tcgen05
    # kernel writes 0 there, and the summed written dk is zero up to bf16 rounding noise
    assert rel(cs[:D], cs_ref[:D]) < TOL["fp32_kernel_rel_l2"] and rel(cs[2 * D:], cs_ref[2 * D:]) < TOL["fp32_kernel_rel_l2"]
    assert float(cs[D:2 * D].abs().max()) == 0.0
    assert float(cs_ref[D:2 * D].norm()) < 1e-2 * float(cs_ref[2 * D:].norm()) + 1e-3
    scale = float(qf.grad[:, 2 * D:].norm())
    for i in range(3):
        got, ref = dqkv[:, i * D:(i + 1) * D].float(), qf.grad[:, i * D:(i + 1) * D]
        if T == 1 and i < 2:  # one key: softmax has no gradient, dq = dk = 0 exactly
            assert float(got.norm()) < 1e-3 * scale, "qkv"[i]
        else:
            assert rel(got, ref) < TOL["attn_grad_rel_l2"], "qkv"[i]


@pytest.mark.parametrize("T", [17, 24, 32])
def test_attn_temporal_long_clip(T):
    """16 < T <= 32: two 16-row register tiles, the diagonal-crossing key tile masked."""
    B, S, H = 2, 17, 8
    D = H * 64
    g = torch.Generator(device=dev).manual_seed(100 + T)
    qkv = (torch.randn(B * T * S, 3 * D, device=dev, generator=g) * 1.5).bfloat16()
    out, lse = Kn.attn_temporal_fwd(qkv, B, T, S, H)
    qf = qkv.float().requires_grad_(True)
    o_ref, lse_ref = _ref_attn(qf.reshape(B, T, S, 3 * D).transpose(1, 2), (B, S), T, H, True)
    assert rel(out.reshape(B, T, S, D).transpose(1, 2), o_ref) < TOL["attn_out_rel_l2"]
    assert rel(lse.reshape(B, S, H, T), lse_ref) < TOL["attn_lse_rel"]
    go = torch.randn(o_ref.shape, device=dev, generator=g)
    o_ref.backward(go)
    dout = go.transpose(1, 2).reshape(B * T * S, D).bfloat16().contiguous()
    cs = torch.full((3 * D,), float("nan"), device=dev)
    dqkv = Kn.attn_temporal_bwd(qkv, out, dout, lse, B, T, S, H, colsum=cs)
    cs_ref = torch.empty_like(cs)
    Kn.colsum_bf16(dqkv, cs_ref)
    assert rel(cs, cs_ref) < TOL["fp32_kernel_rel_l2"]
    for i in range(3):
        assert rel(dqkv[:, i * D:(i + 1) * D].float(), qf.grad[:, i * D:(i + 1) * D]) < TOL["attn_grad_rel_l2"], "qkv"[i]


@pytest.mark.parametrize("S,H", [(16, 8), (17, 8), (18, 8), (32, 8), (5, 2), (1, 4), (24, 16), (18, 6), (9, 3)])
def test_attn_spatial_small_fwd_bwd(S, H):
    """S <= 32 (patch-16 presets, MAE S = 16, ST-DiT S = 18): the register-tile kernel, non-causal."""
    frames = 37
    D = H * 64
    g = torch.Generator(device=dev).manual_seed(S * 31 + H)
    qkv = (torch.randn(frames * S, 3 * D, device=dev, generator=g) * 1.5).bfloat16()
    out, out_lo, lse = Kn.attn_spatial_fwd(qkv, frames, S, H, keep_lo=True)
    assert out_lo is None  # the small kernel's backward reads the bf16 output
    qf = qkv.float().requires_grad_(True)
    o_ref, lse_ref = _ref_attn(qf.reshape(frames, S, 3 * D), (frames,), S, H, False)
    assert rel(out.reshape(frames, S, D), o_ref) < TOL["attn_out_rel_l2"]
    assert rel(lse, lse_ref) < TOL["attn_lse_rel"]
    go = torch.randn(o_ref.shape, device=dev, generator=g)
    o_ref.backward(go)
    dqkv = torch.full_like(qkv, float("nan"))
    cs = torch.full((3 * D,), float("nan"), device=dev)
    Kn.attn_spatial_bwd(qkv, out, go.reshape(frames * S, D).bfloat16().contiguous(), lse, frames, S, H, dqkv=dqkv,
                        colsum=cs)
    assert torch.isfinite(dqkv.float()).all()
    cs_ref = torch.empty_like(cs)
    Kn.colsum_bf16(dqkv, cs_ref)
    assert rel(cs, cs_ref) < TOL["fp32_kernel_rel_l2"]
    vscale = float(qf.grad[:, 2 * D:].norm())
    for i in range(3):
        got, ref = dqkv[:, i * D:(i + 1) * D].float(), qf.grad[:, i * D:(i + 1) * D]
        if S == 1 and i < 2:
            assert float(got.norm()) < 1e-3 * vscale, "qkv"[i]
        else:
            assert rel(got, ref) < TOL["attn_grad_rel_l2"], "qkv"[i]


# ---------------------------------------------------------------------------------------------
# column sums / partial-row reductions (bias and LayerNorm parameter gradients): every thread
# layout the kernels pick (row groups for cols/8 < 256, a column loop above), ragged row counts,
# padded leading dimensions, the two-stage path above 512 partials; deterministic run to run.
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("rows,cols,ld", [(1, 8, 8), (5, 64, 72), (296 * 3 + 7, 512, 1536), (5000, 1536, 1536),
                                          (777, 2056, 2064), (40000, 512, 3 * 512)])
def test_colsum_bf16_layouts(rows, cols, ld):
    g = torch.Generator(device=dev).manual_seed(rows + cols)
    x = torch.randn(rows, ld, device=dev, generator=g).bfloat16()
    out = torch.full((cols,), float("nan"), device=dev)
    Kn.colsum_bf16(x, out, cols=cols)
    ref = x[:, :cols].double().sum(0)
    assert float((out.double() - ref).abs().max()) <= 1e-5 * max(1.0, float(ref.abs().max())) + 1e-4
    again = torch.empty_like(out)
    Kn.colsum_bf16(x, again, cols=cols)
    assert torch.equal(out, again)


@pytest.mark.parametrize("nparts", [1, 7, 63, 64, 65, 296, 513, 1100, 9252])
@pytest.mark.parametrize("D", [1, 33, 512])
def test_reduce_partials(nparts, D):
    g = torch.Generator(device=dev).manual_seed(nparts * 7 + D)
    part = torch.randn(nparts, D, device=dev, generator=g)
    ref = part.double().sum(0)
    base = torch.randn(D, device=dev, generator=g)
    for acc in (False, True):
        out = base.clone()
        Kn.reduce_partials(part.clone(), nparts, D, out, accumulate=acc)  # two-stage path overwrites its input
        want = ref + (base.double() if acc else 0.0)
        assert float((out.double() - want).abs().max()) < 1e-5 * math.sqrt(nparts) + 1e-6
        again = base.clone()
        Kn.reduce_partials(part.clone(), nparts, D, again, accumulate=acc)
        assert torch.equal(out, again)


# ---------------------------------------------------------------------------------------------
# dynamics input embedding (K5 forward): both conditioning modes, masked positions, latent widths
# above one warp (dl > 32 takes the second shuffle register), and the bad-token error flag.
# ---------------------------------------------------------------------------------------------
def _embed_ref(tokens, mask, lat, P, B, T, N, D, dl, prepend):
    E, mt = P["token_embed"].double(), P["mask_token"].double()
    sel = E[tokens.long()]
    if mask is not None:
        sel = torch.where(mask.bool()[..., None], mt.expand_as(sel), sel)
    cond = torch.cat([P["null_action"].double().expand(B, 1, dl), lat.double()], 1)  # (B, T, dl)
    act = cond @ P["action_proj.w"].double() + P["action_proj.b"].double()        # (B, T, D)
    if prepend:
        x = torch.cat([act[:, :, None], sel], 2)
    else:
        x = sel + act[:, :, None]
    S = x.shape[2]
    return x + P["pos_spatial"].double()[:S] + P["pos_temporal"].double()[:T, None]


@pytest.mark.parametrize("prepend", [True, False])
@pytest.mark.parametrize("D,dl", [(512, 32), (256, 48), (96, 7)])
def test_dyn_embed_fwd_modes(prepend, D, dl):
    B, T, N, K = 3, 5, 19, 37
    g = torch.Generator(device=dev).manual_seed(D + dl + prepend)
    P = {"token_embed": torch.randn(K, D, device=dev, generator=g),
         "mask_token": torch.randn(D, device=dev, generator=g),
         "null_action": torch.randn(dl, device=dev, generator=g),
         "action_proj.w": torch.randn(dl, D, device=dev, generator=g),
         "action_proj.b": torch.randn(D, device=dev, generator=g),
         "pos_spatial": torch.randn(N + 1, D, device=dev, generator=g),
         "pos_temporal": torch.randn(T, D, device=dev, generator=g)}
    tokens = torch.randint(0, K, (B, T, N), device=dev, generator=g)
    mask = (torch.rand(B, T, N, device=dev, generator=g) < 0.3).to(torch.uint8)
    lat = torch.randn(B, T - 1, dl, device=dev, generator=g)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    x = Kn.dyn_embed_fwd(tokens, mask, lat, P, B=B, T=T, N=N, D=D, dl=dl, K=K, prepend=prepend, err=err)
    S = N + (1 if prepend else 0)
    ref = _embed_ref(tokens, mask, lat, P, B, T, N, D, dl, prepend).reshape(B * T * S, D)
    assert float((x.double() - ref).abs().max()) < 1e-4 * max(1.0, math.sqrt(dl))
    assert int(err.item()) == 0
    tokens[1, 2, 3] = K  # out of range: flagged (and read as token 0), never an out-of-bounds read
    Kn.dyn_embed_fwd(tokens, None, lat, P, B=B, T=T, N=N, D=D, dl=dl, K=K, prepend=prepend, err=err)
    assert int(err.item()) == 1


@pytest.mark.parametrize("R", [147456, 9000])
@pytest.mark.parametrize("accumulate", [0, 1])
def test_linear_f32_n32_rows_kernel_bit_identical(R, accumulate):
    """The 512 -> 32 fp32 latent projection: the two-rows-per-lane kernel and the thread-per-output
    kernel (reached through a 4-byte-misaligned x) both sum over k in order with fmaf, so their
    outputs are bit-identical."""
    K = 512
    g = torch.Generator(device=dev).manual_seed(R + accumulate)
    x = torch.randn(R, K, device=dev, generator=g)
    W = torch.randn(K, 32, device=dev, generator=g)
    b = torch.randn(32, device=dev, generator=g)
    base = torch.randn(R, 32, device=dev, generator=g)
    outs = []
    for mode in ("fast", "scalar"):
        y = base.clone()
        xm = x
        if mode == "scalar":
            mis = torch.empty(R * K + 1, device=dev)
            mis[1:].copy_(x.flatten())
            xm = mis[1:].view(R, K)  # 4-byte aligned only: the thread-per-output kernel
        Kn.linear_f32(xm, W, b, out=y, accumulate=bool(accumulate))
        outs.append(y)
    assert torch.equal(outs[0], outs[1])
    ref = x.double() @ W.double() + b.double() + (base.double() if accumulate else 0)
    assert rel(outs[0].double(), ref) < 1e-6


@pytest.mark.parametrize("K,N", [(512, 32), (32, 512), (48, 32)])
@pytest.mark.parametrize("accumulate", [0, 1])
def test_linear_f32_bwd_parallel_vs_reference_kernel(K, N, accumulate):
    """jz_linear_f32_bwd_ws (the latent projections' backward: parallel dW partials folded in order,
    dx from W in shared memory) against the thread-per-output jz_linear_f32_bwd: dx bit-identical
    (same summation order), dW / db within fp32 reassociation."""
    R = 5000 + 77
    g = torch.Generator(device=dev).manual_seed(K * N + accumulate)
    x = torch.randn(R, K, device=dev, generator=g)
    dy = torch.randn(R, N, device=dev, generator=g)
    W = torch.randn(K, N, device=dev, generator=g)
    outs = []
    for fast in (False, True):
        dx = torch.randn(R, K, device=dev, generator=torch.Generator(device=dev).manual_seed(1))
        dW = torch.randn(K, N, device=dev, generator=torch.Generator(device=dev).manual_seed(2))
        db = torch.randn(N, device=dev, generator=torch.Generator(device=dev).manual_seed(3))
        if fast:
            Kn.linear_f32_bwd(x, dy, W, dx=dx, dW=dW, db=db, accumulate=bool(accumulate))
        else:
            L.call("jz_linear_f32_bwd", x.data_ptr(), dy.data_ptr(), R, K, N, W.data_ptr(), dx.data_ptr(),
                   dW.data_ptr(), db.data_ptr(), accumulate, L.stream_ptr())
        outs.append((dx, dW, db))
    (dx0, dW0, db0), (dx1, dW1, db1) = outs
    assert torch.equal(dx0, dx1)
    assert rel(dW1, dW0) < 1e-5 and rel(db1, db0) < 1e-5
    ref = x.double().t() @ dy.double()
    base = torch.randn(K, N, device=dev, generator=torch.Generator(device=dev).manual_seed(2)).double()
    assert rel(dW1.double(), ref + (base if accumulate else 0)) < 1e-5


@pytest.mark.parametrize("M", [148032, 1000, 300])
def test_ln_fused_gemm_forward_matches_gemm_then_layernorm(M):
    """jz_gemm_bf16_ln_fwd (residual projection + next LayerNorm in the epilogue) against the
    separate RESID GEMM + LayerNorm kernels on the same bf16 operands (nn.py:35-40)."""
    from paper_2510_27002_b200 import _lib as L
    from paper_2510_27002_b200 import kernels as K
    g = torch.Generator(device="cuda").manual_seed(M)
    a = (torch.randn(M, 512, device="cuda", generator=g) * 0.5).bfloat16()
    w = (torch.randn(512, 512, device="cuda", generator=g) * 0.05).bfloat16()
    b = torch.randn(512, device="cuda", generator=g) * 0.1
    res = torch.randn(M, 512, device="cuda", generator=g)
    gm = 1 + 0.1 * torch.randn(512, device="cuda", generator=g)
    be = 0.1 * torch.randn(512, device="cuda", generator=g)
    x1, xn, mu, rs = K.linear_fwd_ln(a, w, b, res, gm, be)
    ref_x = K.linear_fwd(a, w, b, epilogue=L.EPI_RESID, aux=res)
    ref_xn, ref_mu, ref_rs = K.layernorm_fwd(ref_x, gm, be)
    assert torch.equal(x1, ref_x)
    assert float((mu - ref_mu).abs().max()) < 1e-6
    assert float(((rs - ref_rs) / ref_rs).abs().max()) < 1e-5
    assert float((xn.float() - ref_xn.float()).abs().max()) <= 2 ** -6 * float(ref_xn.float().abs().max())
    if M % 257 == 0:  # compacted output (final LayerNorm dropping the action-token rows)
        _, xs, _, _ = K.linear_fwd_ln(a, w, b, res, gm, be, skip_period=257)
        ref_s, _, _ = K.layernorm_fwd(ref_x, gm, be, skip_period=257)
        assert xs.shape == ref_s.shape
        assert float((xs.float() - ref_s.float()).abs().max()) <= 2 ** -6 * float(ref_s.float().abs().max())


@pytest.mark.parametrize("M,Kd", [(148032, 1536), (1000, 2048), (300, 512)])
def test_ln_fused_gemm_backward_matches_fp32_reference(M, Kd):
    """jz_gemm_bf16_ln_bwd (dX GEMM + LayerNorm backward in the epilogue) against a torch fp32
    LayerNorm backward of the same GEMM output (autodiff of nn.py:35-40)."""
    from paper_2510_27002_b200 import kernels as K
    g = torch.Generator(device="cuda").manual_seed(M + Kd)
    dy = (torch.randn(M, Kd, device="cuda", generator=g) * 0.1).bfloat16()
    w = (torch.randn(512, Kd, device="cuda", generator=g) * 0.05).bfloat16()
    x = torch.randn(M, 512, device="cuda", generator=g) * 2 + 0.3
    gm = 1 + 0.1 * torch.randn(512, device="cuda", generator=g)
    mean = x.mean(1)
    rstd = 1 / torch.sqrt(x.var(1, unbiased=False) + 1e-5)
    dres0 = torch.randn(M, 512, device="cuda", generator=g)
    dres = dres0.clone()
    dres_b = torch.empty(M, 512, device="cuda", dtype=torch.bfloat16)
    dgam, dbet, dbias = (torch.empty(512, device="cuda") for _ in range(3))
    K.linear_dx_ln(dy, w, x=x, mean=mean, rstd=rstd, gamma=gm, dres=dres, dres_bf16=dres_b, dgamma=dgam, dbeta=dbet,
                   dbias=dbias)
    gout = dy.float() @ w.float().t()  # gradient of the LayerNorm output
    xr = x.clone().requires_grad_(True)
    gr = gm.clone().requires_grad_(True)
    br = torch.zeros(512, device="cuda", requires_grad=True)
    torch.nn.functional.layer_norm(xr, (512,), gr, br, eps=1e-5).backward(gout)
    ref = dres0 + xr.grad
    rel = lambda p, q: float((p - q).norm() / q.norm())
    assert rel(dres - dres0, xr.grad) < TOL["fp32_kernel_rel_l2"] * 100  # fp32 accumulation-order level
    assert torch.equal(dres_b, dres.bfloat16())
    assert rel(dgam, gr.grad) < 1e-4 and rel(dbet, br.grad) < 1e-4
    assert rel(dbias, ref.sum(0)) < 1e-4
