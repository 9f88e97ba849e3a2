import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Event-timed A/B of every distinct K1 GEMM of the C3 step (M = 148032 tokens) against an
alternative libjz.so: python tools/ab_step_gemms.py [LIB]"""
import torch

from paper_2510_27002_b200 import _lib as L

if len(sys.argv) > 1:
    L.LIB_PATH = pathlib.Path(sys.argv[1])
from paper_2510_27002_b200 import kernels as Kn  # noqa: E402

L.ensure_device()
M, d, f = 148032, 512, 2048
g = torch.Generator(device="cuda").manual_seed(0)
r = lambda *s: (torch.randn(*s, device="cuda", generator=g) * 0.05).bfloat16()
x512, x1536, x2048 = r(M, d), r(M, 3 * d), r(M, f)
w_qkv, w_o, w_up, w_dn, w_lg = r(d, 3 * d), r(d, d), r(d, f), r(f, d), r(d, 1024)
b3, b1, bf = (torch.zeros(n, device="cuda") for n in (3 * d, d, f))
res = torch.randn(M, d, device="cuda", generator=g)
hd = torch.rand(M, f, device="cuda", generator=g).half()
o_bf_3, o_bf_f, o_bf_d = (torch.empty(M, n, device="cuda", dtype=torch.bfloat16) for n in (3 * d, f, d))
o_f_d, o_f_lg = torch.empty(M, d, device="cuda"), torch.empty(M, 1024, device="cuda")
dw_qkv, dw_up, dw_dn, dw_o = (torch.empty(*s, device="cuda") for s in ((d, 3 * d), (d, f), (f, d), (d, d)))
cs_f, cs_d = torch.empty(f, device="cuda"), torch.empty(d, device="cuda")
E = L
cases = {
    "QKV fwd      N=1536 K=512 ": (lambda: Kn.linear_fwd(x512, w_qkv, b3, out=o_bf_3), M * 3 * d * d),
    "up fwd GELU_DG N=2048 K=512": (lambda: Kn.linear_fwd(x512, w_up, bf, epilogue=E.EPI_GELU_DG, out2=hd, out=o_bf_f), M * f * d),
    "down fwd RESID N=512 K=2048": (lambda: Kn.linear_fwd(x2048, w_dn, b1, epilogue=E.EPI_RESID, aux=res, out=o_f_d), M * d * f),
    "O fwd RESID  N=512 K=512  ": (lambda: Kn.linear_fwd(x512, w_o, b1, epilogue=E.EPI_RESID, aux=res, out=o_f_d), M * d * d),
    "down dX MUL_F16+cs N=2048 ": (lambda: Kn.linear_dx(x512, w_dn, epilogue=E.EPI_MUL_F16, out=o_bf_f, aux=hd, colsum=cs_f), M * f * d),
    "up dX        N=512 K=2048 ": (lambda: Kn.linear_dx(x2048, w_up, epilogue=E.EPI_BF16, out=o_bf_d), M * d * f),
    "qkv dX       N=512 K=1536 ": (lambda: Kn.linear_dx(x1536, w_qkv, epilogue=E.EPI_BF16, out=o_bf_d), M * d * 3 * d),
    "O dX +cs     N=512 K=512  ": (lambda: Kn.linear_dx(x512, w_o, epilogue=E.EPI_BF16, out=o_bf_d, colsum=cs_d), M * d * d),
    "dW qkv 512x1536 K=M       ": (lambda: Kn.linear_dw(x512, x1536, dw_qkv), d * 3 * d * M),
    "dW up 512x2048 K=M        ": (lambda: Kn.linear_dw(x512, x2048, dw_up), d * f * M),
    "dW down 2048x512 K=M      ": (lambda: Kn.linear_dw(x2048, x512, dw_dn), d * f * M),
    "dW o 512x512 K=M          ": (lambda: Kn.linear_dw(x512, x512, dw_o), d * d * M),
    "logits fwd F32 N=1024     ": (lambda: Kn.linear_fwd(x512, w_lg, torch.zeros(1024, device="cuda"), epilogue=E.EPI_F32, out=o_f_lg), M * 1024 * d),
}


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


tot = 0.0
for name, (fn, macs) in cases.items():
    us = timeit(fn)
    tot += us
    print(f"{name}: {us:8.1f} us  {2 * macs / us / 1e6:7.0f} TFLOP/s", flush=True)
print(f"sum {tot:.1f} us")
