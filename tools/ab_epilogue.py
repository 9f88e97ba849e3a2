import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""A/B timing of the K1 GEMM launches of the dynamics step WITH their real epilogues, at the
training M (148032 rows) and the C5 decode M (16448 rows).

usage: python tools/ab_epilogue.py [LIB]   (LIB defaults to the in-tree build)"""
import torch

from paper_2510_27002_b200 import _lib as L

if len(sys.argv) > 1:
    L.LIB_PATH = pathlib.Path(sys.argv[1])
from paper_2510_27002_b200 import kernels as Kn  # noqa: E402

L.ensure_device()
d, f = 512, 2048
g = torch.Generator(device="cuda").manual_seed(0)


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


for M in (148032, 16448):
    xn = torch.randn(M, d, device="cuda", generator=g).bfloat16()
    h = torch.randn(M, f, device="cuda", generator=g).bfloat16()
    res = torch.randn(M, d, device="cuda", generator=g)
    wqkv = (torch.randn(d, 3 * d, device="cuda", generator=g) * 0.02).bfloat16()
    wo = (torch.randn(d, d, device="cuda", generator=g) * 0.02).bfloat16()
    wup = (torch.randn(d, f, device="cuda", generator=g) * 0.02).bfloat16()
    wdn = (torch.randn(f, d, device="cuda", generator=g) * 0.02).bfloat16()
    bq, bd, bf_ = (torch.randn(n, device="cuda", generator=g) * 0.1 for n in (3 * d, d, f))
    qkv = torch.empty(M, 3 * d, device="cuda", dtype=torch.bfloat16)
    xo = torch.empty(M, d, device="cuda")
    hh = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
    hp = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
    hd = torch.rand(M, f, device="cuda", generator=g).half()
    dy = torch.randn(M, d, device="cuda", generator=g).bfloat16()
    cases = {
        "QKV bf16+bias   N=1536 K=512": (lambda: Kn.linear_fwd(xn, wqkv, bq, out=qkv), 3 * d * d),
        "O   RESID       N=512  K=512": (lambda: Kn.linear_fwd(xn, wo, bd, epilogue=L.EPI_RESID, aux=res, out=xo), d * d),
        "up  GELU+D2     N=2048 K=512": (lambda: Kn.linear_fwd(xn, wup, bf_, epilogue=L.EPI_GELU, out2=hp, out=hh), d * f),
        "up  GELU        N=2048 K=512": (lambda: Kn.linear_fwd(xn, wup, bf_, epilogue=L.EPI_GELU, out=hh), d * f),
        "down RESID      N=512  K=2048": (lambda: Kn.linear_fwd(h, wdn, bd, epilogue=L.EPI_RESID, aux=res, out=xo), d * f),
        "dX GELU_BWD     N=2048 K=512": (lambda: Kn.linear_dx(dy, wdn, epilogue=L.EPI_GELU_BWD, out=hh, aux=hp), d * f),
        "up  GELU_DG     N=2048 K=512": (lambda: Kn.linear_fwd(xn, wup, bf_, epilogue=L.EPI_GELU_DG, out2=hd, out=hh), d * f),
        "dX MUL_F16      N=2048 K=512": (lambda: Kn.linear_dx(dy, wdn, epilogue=L.EPI_MUL_F16, out=hh, aux=hd), d * f),
        "dX bf16         N=512  K=2048": (lambda: Kn.linear_dx(h, wup, epilogue=L.EPI_BF16, out=dy), d * f),
    }
    tot = 0.0
    for name, (fn, macs_per_row) in cases.items():
        us = timeit(fn)
        tot += us
        print(f"M={M:6d} {name}: {us:8.1f} us  {2 * macs_per_row * M / us / 1e6:7.0f} TFLOP/s", flush=True)
    print(f"M={M:6d} total {tot:.1f} us", flush=True)
