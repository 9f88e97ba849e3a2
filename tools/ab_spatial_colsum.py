import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Spatial QKV-bias gradient: (a) v from the O-projection dX GEMM's column sums + a q pass over dqkv
vs (b) the attention backward's own column-sum partials.  C3 shape."""
import torch

from paper_2510_27002_b200 import _lib as L
from paper_2510_27002_b200 import kernels as K

L.ensure_device()
frames, S, H = 576, 257, 8
D = H * 64
M = frames * S
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn(M, 3 * D, device="cuda", generator=g).bfloat16()
o, olo, lse = K.attn_spatial_fwd(qkv, frames, S, H)
dres_b = (torch.randn(M, D, device="cuda", generator=g) * 0.1).bfloat16()
wo = (torch.randn(D, D, device="cuda", generator=g) * 0.05).bfloat16()
dao = torch.empty(M, D, device="cuda", dtype=torch.bfloat16)
dq = torch.empty_like(qkv)
gb = torch.empty(3 * D, device="cuda")


def a():
    K.linear_dx(dres_b, wo, epilogue=L.EPI_BF16, out=dao, colsum=gb[2 * D:])
    K.attn_spatial_bwd(qkv, o, dao, lse, frames, S, H, dqkv=dq, out_lo=olo)
    gb[D:2 * D].zero_()
    K.colsum_bf16(dq, gb[:D], cols=D)


def b():
    K.linear_dx(dres_b, wo, epilogue=L.EPI_BF16, out=dao)
    K.attn_spatial_bwd(qkv, o, dao, lse, frames, S, H, dqkv=dq, colsum=gb, out_lo=olo)


def t(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for _ in range(2):
    print(f"(a) GEMM colsum + q pass: {t(a):.1f} us   (b) attention colsum: {t(b):.1f} us")
