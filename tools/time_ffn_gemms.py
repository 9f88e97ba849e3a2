import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Event-timed FFN GEMMs of the C3 step (M=148032): up-projection GELU_DG and the down dX MUL_F16
(+ column sums, as the step runs it).  A/B with JZ_GEMM_DB=0/1."""
import torch

from paper_2510_27002_b200 import _lib as L
if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    L.LIB_PATH = pathlib.Path(sys.argv[1]).resolve()
from paper_2510_27002_b200 import kernels as Kn  # noqa: E402

L.ensure_device()
M, d, f = 148032, 512, 2048
g = torch.Generator(device="cuda").manual_seed(0)
xn = torch.randn(M, d, device="cuda", generator=g).bfloat16()
wup = (torch.randn(d, f, device="cuda", generator=g) * 0.02).bfloat16()
wdn = (torch.randn(f, d, device="cuda", generator=g) * 0.02).bfloat16()
bf_ = torch.randn(f, device="cuda", generator=g) * 0.1
hh = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
hd = torch.empty(M, f, device="cuda", dtype=torch.float16)
dres = torch.randn(M, d, device="cuda", generator=g).bfloat16()
dh = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
cs = torch.empty(f, device="cuda")


def t(fn, n=20):
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


up = t(lambda: Kn.linear_fwd(xn, wup, bf_, epilogue=L.EPI_GELU_DG, out2=hd, out=hh))
dn = t(lambda: Kn.linear_dx(dres, wdn, epilogue=L.EPI_MUL_F16, out=dh, aux=hd))
dnc = t(lambda: Kn.linear_dx(dres, wdn, epilogue=L.EPI_MUL_F16, out=dh, aux=hd, colsum=cs))
print(f"GELU_DG up {up:.1f} us | MUL_F16 dX {dn:.1f} us | MUL_F16 dX + colsum {dnc:.1f} us "
      f"({pathlib.Path(sys.argv[1]).name if len(sys.argv) > 1 else 'default'})")
