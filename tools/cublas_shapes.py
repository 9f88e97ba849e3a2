"""Reference point: cuBLAS (torch.matmul / addmm) on the dynamics-step GEMM shapes."""
import torch

dev = "cuda"


def t(fn, n=20):
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


M = 148032
for (m, n, k, trans) in [(M, 1536, 512, ""), (M, 512, 512, ""), (M, 2048, 512, ""), (M, 512, 2048, ""),
                         (M, 512, 1536, "bt"), (512, 1536, M, "at"), (2048, 512, M, "at")]:
    A = torch.randn(k, m, device=dev).bfloat16().t() if trans == "at" else torch.randn(m, k, device=dev).bfloat16()
    B = torch.randn(n, k, device=dev).bfloat16().t() if trans == "bt" else torch.randn(k, n, device=dev).bfloat16()
    bias = torch.randn(n, device=dev).bfloat16()
    out = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    us = t(lambda: torch.matmul(A, B, out=out))
    us2 = t(lambda: torch.addmm(bias, A, B, out=out))
    out32 = torch.empty(m, n, device=dev, dtype=torch.float32)
    print(f"cuBLAS M={m} N={n} K={k} {trans}: mm bf16 {us:.1f} us {2*m*n*k/us/1e6:.0f} TF/s | addmm {us2:.1f} us {2*m*n*k/us2/1e6:.0f} TF/s", flush=True)
