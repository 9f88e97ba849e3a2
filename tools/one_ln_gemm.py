import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""One LN-fused GEMM launch at the step's shape (ncu target).  usage: one_ln_gemm.py fwd|bwd K"""
import torch

from paper_2510_27002_b200 import kernels as K, _lib as L

L.ensure_device()
mode, Kd = sys.argv[1], int(sys.argv[2])
M = 148032
torch.manual_seed(0)
if mode == "fwd":
    a = (torch.randn(M, Kd, device="cuda") * 0.5).bfloat16(); w = (torch.randn(Kd, 512, device="cuda") * 0.05).bfloat16()
    b = torch.zeros(512, device="cuda"); res = torch.randn(M, 512, device="cuda"); g = torch.ones(512, device="cuda")
    for _ in range(3):
        K.linear_fwd_ln(a, w, b, res, g, b)
else:
    dy = (torch.randn(M, Kd, device="cuda") * 0.1).bfloat16(); wq = (torch.randn(512, Kd, device="cuda") * 0.05).bfloat16()
    x = torch.randn(M, 512, device="cuda"); mean = x.mean(1); rstd = 1 / torch.sqrt(x.var(1, unbiased=False) + 1e-5)
    dres = torch.randn(M, 512, device="cuda"); dres_b = torch.empty(M, 512, device="cuda", dtype=torch.bfloat16)
    dg = torch.empty(512, device="cuda"); g = torch.ones(512, device="cuda")
    for _ in range(3):
        K.linear_dx_ln(dy, wq, x=x, mean=mean, rstd=rstd, gamma=g, dres=dres, dres_bf16=dres_b, dgamma=dg, dbeta=dg, dbias=dg)
torch.cuda.synchronize()
