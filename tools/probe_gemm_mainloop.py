import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
import torch
from paper_2510_27002_b200 import _lib as L
L.ensure_device()
dev = "cuda"
def bench(M, N, K, epi, n=30):
    A = torch.randn(M, K, device=dev).bfloat16(); B = torch.randn(K, N, device=dev).bfloat16()
    D = torch.empty(M, N, device=dev, dtype=torch.float32)
    args = (A.data_ptr(), K, 1, B.data_ptr(), N, 0, D.data_ptr(), N, M, N, K, epi, None, None, 0, None, 0, 1, None, L.stream_ptr())
    for _ in range(3): L.call("jz_gemm_bf16", *args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): L.call("jz_gemm_bf16", *args)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1e3
    print(f"M={M} N={N} K={K} epi={epi}: {us:.1f} us {2*M*N*K/us/1e6:.0f} TF/s", flush=True)
for K in (512, 1024, 2048, 4096):
    bench(148032, 1536, K, 7)
bench(148032, 1536, 512, 1)
bench(148032, 512, 512, 7)
bench(148032, 2048, 512, 7)
bench(16384, 16384, 4096, 7)
