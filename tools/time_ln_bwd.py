import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Event-timed LayerNorm backward at the C3 step shape (148032 x 512, bf16 dy, accumulate into the fp32
residual gradient, dgamma/dbeta/dbias partials), with and without the bf16 copy of the output."""
import torch

from paper_2510_27002_b200 import _lib as L
from paper_2510_27002_b200 import kernels as Kn

L.ensure_device()
M, D = 148032, 512
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(M, D, device="cuda", generator=g)
mean = x.mean(1)
rstd = torch.rsqrt(x.var(1, unbiased=False) + 1e-5)
gam = torch.randn(D, device="cuda", generator=g)
dy = torch.randn(M, D, device="cuda", generator=g).bfloat16()
dres = torch.randn(M, D, device="cuda", generator=g)
yb = torch.empty(M, D, device="cuda", dtype=torch.bfloat16)
dg, db, dz = (torch.zeros(D, device="cuda") for _ in range(3))


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


for name, yb_, nbytes in (("no bf16 copy", None, M * D * (4 + 2 + 4 + 4)), ("with bf16 copy", yb, M * D * (4 + 2 + 4 + 4 + 2))):
    us = timeit(lambda: Kn.layernorm_bwd(x, mean, rstd, gam, dy, dres, accumulate=True, dres_bf16=yb_, dgamma=dg,
                                         dbeta=db, dbias=dz))
    print(f"LN bwd {name}: {us:.1f} us  {nbytes / us / 1e3:.0f} GB/s", flush=True)
