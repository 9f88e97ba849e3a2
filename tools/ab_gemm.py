import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""A/B timing of K1 GEMM shapes of the dynamics step against an alternative libjz.so.

usage: python tools/ab_gemm.py [LIB]   (LIB defaults to the in-tree build)
Prints us per launch and TFLOP/s for the step's main GEMM shapes (M = 148032 tokens)."""
import torch

from paper_2510_27002_b200 import _lib as L

if len(sys.argv) > 1:
    L.LIB_PATH = pathlib.Path(sys.argv[1])
from paper_2510_27002_b200 import kernels as Kn  # noqa: E402

L.ensure_device()
M, d, f = 148032, 512, 2048
x = torch.randn(M, f, device="cuda").bfloat16()
w = torch.randn(f, 3 * d, device="cuda").bfloat16() * 0.02
out = torch.empty(M, 3 * d, device="cuda", dtype=torch.bfloat16)
outf = torch.empty(M, d, device="cuda")
wout = torch.empty(f, 3 * d, device="cuda")


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


cases = {
    "fwd QKV  N=1536 K=512": (lambda: Kn.gemm(x, w, M=M, N=3 * d, K=d, a_kmajor=True, b_kmajor=False, out=out,
                                             epilogue=L.EPI_BF16, lda=f), M * 3 * d * d),
    "fwd down N=512 K=2048": (lambda: Kn.gemm(x, w, M=M, N=d, K=f, a_kmajor=True, b_kmajor=False, out=out,
                                             epilogue=L.EPI_BF16, ldb=3 * d, ldd=3 * d), M * d * f),
    "dW  (512x1536) K=M": (lambda: Kn.gemm(x, x, M=d, N=3 * d, K=M, a_kmajor=False, b_kmajor=False, out=wout,
                                          epilogue=L.EPI_F32, lda=f, ldb=f, ldd=3 * d,
                                          split_k=Kn.splitk_for(d, 3 * d, M)), d * 3 * d * M),
}
for name, (fn, macs) in cases.items():
    us = timeit(fn)
    print(f"{name}: {us:8.1f} us  {2 * macs / us / 1e6:7.0f} TFLOP/s", flush=True)
