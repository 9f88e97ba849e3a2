import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""One K1 launch of a named step shape (ncu target): python tools/one_gemm.py {gelu_bwd|gelu_d2|resid|qkv} [M]"""
import torch

from paper_2510_27002_b200 import _lib as L
from paper_2510_27002_b200 import kernels as Kn

L.ensure_device()
which = sys.argv[1]
M = int(sys.argv[2]) if len(sys.argv) > 2 else 148032
d, f = 512, 2048
xn = torch.randn(M, d, device="cuda").bfloat16()
res = torch.randn(M, d, device="cuda")
hp = torch.randn(M, f, device="cuda").bfloat16()
hh = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
hd = torch.rand(M, f, device="cuda").half()
w = (torch.randn(f, d, device="cuda") * 0.02).bfloat16()
wup = (torch.randn(d, f, device="cuda") * 0.02).bfloat16()
wo = (torch.randn(d, d, device="cuda") * 0.02).bfloat16()
wqkv = (torch.randn(d, 3 * d, device="cuda") * 0.02).bfloat16()
bf_, bd, bq = torch.zeros(f, device="cuda"), torch.zeros(d, device="cuda"), torch.zeros(3 * d, device="cuda")
xo = torch.empty(M, d, device="cuda")
qkv = torch.empty(M, 3 * d, device="cuda", dtype=torch.bfloat16)
fn = {
    "gelu_bwd": lambda: Kn.linear_dx(xn, w, epilogue=L.EPI_GELU_BWD, out=hh, aux=hp),
    "gelu_dg": lambda: Kn.linear_fwd(xn, wup, bf_, epilogue=L.EPI_GELU_DG, out2=hd, out=hh),
    "mul_f16": lambda: Kn.linear_dx(xn, w, epilogue=L.EPI_MUL_F16, out=hh, aux=hd),
    "gelu_d2": lambda: Kn.linear_fwd(xn, wup, bf_, epilogue=L.EPI_GELU, out2=hp, out=hh),
    "resid": lambda: Kn.linear_fwd(xn, wo, bd, epilogue=L.EPI_RESID, aux=res, out=xo),
    "qkv": lambda: Kn.linear_fwd(xn, wqkv, bq, out=qkv),
}[which]
fn()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
fn()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
