import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Scratch GPU check of the tcgen05 GEMM against torch fp32 (all majors/epilogues)."""
import sys
import time

import torch

from paper_2510_27002_b200 import _lib as L

L.ensure_device()
torch.manual_seed(0)
dev = "cuda"
ok = True


def run(M, N, K, a_kmajor, b_kmajor, epi=L.EPI_F32, split=1, bias=True):
    global ok
    X = torch.randn(M, K, device=dev).bfloat16()
    W = torch.randn(K, N, device=dev).bfloat16()
    ref = X.float() @ W.float()
    A = X.contiguous() if a_kmajor else X.t().contiguous()  # (m,k) at k*lda+m  => store [K][M]
    lda = K if a_kmajor else M
    B = W.t().contiguous() if b_kmajor else W.contiguous()
    if not b_kmajor and N % 8: return
    ldb = K if b_kmajor else N
    b = torch.randn(N, device=dev) if bias else None
    if b is not None:
        ref = ref + b
    D = torch.zeros(M, N, device=dev, dtype=torch.bfloat16 if epi == L.EPI_BF16 else torch.float32)
    ws = None
    if split > 1:
        ws = torch.empty(L.load().jz_gemm_workspace_bytes(M, N, split) // 4 + 1, device=dev)
    L.call("jz_gemm_bf16", A.data_ptr(), lda, a_kmajor, B.data_ptr(), ldb, b_kmajor, D.data_ptr(), N,
           M, N, K, epi, L.ptr(b), None, 0, None, 0, split, L.ptr(ws), L.stream_ptr())
    torch.cuda.synchronize()
    err = (D.float() - ref).norm() / ref.norm()
    good = err.item() < (1e-2 if epi == L.EPI_BF16 else 1e-4)
    ok &= good
    print(f"M={M} N={N} K={K} akm={a_kmajor} bkm={b_kmajor} epi={epi} split={split} relerr={err.item():.3e} {'OK' if good else 'FAIL'}", flush=True)


for akm in (1, 0):
    for bkm in (0, 1):
        run(256, 256, 128, akm, bkm)
        run(296 if akm == 0 else 300, 200 if bkm == 1 else 200, 192, akm, bkm)
        run(128, 64, 64, akm, bkm)
        run(1000, 1536, 512, akm, bkm, epi=L.EPI_BF16)
run(512, 512, 4096, 0, 0, split=4)
run(500, 300, 2048, 0, 0, split=3)
run(1000, 1536, 2048, 0, 0, split=2)
run(333, 48, 512, 1, 0)
run(333, 512, 48, 1, 0)
run(333, 32, 512, 1, 0)

# timing of the big forward shapes
def bench(M, N, K, akm=1, bkm=0, epi=L.EPI_BF16, split=1, aux=False):
    A = torch.randn(M, K, device=dev).bfloat16() if akm else torch.randn(K, M, device=dev).bfloat16()
    B = torch.randn(K, N, device=dev).bfloat16() if not bkm else torch.randn(N, K, device=dev).bfloat16()
    D = torch.empty(M, N, device=dev, dtype=torch.bfloat16 if epi == L.EPI_BF16 else torch.float32)
    lda = K if akm else M
    ldb = N if not bkm else K
    ws = None
    if split > 1:
        ws = torch.empty(L.load().jz_gemm_workspace_bytes(M, N, split) // 4 + 1, device=dev)
    bias = torch.randn(N, device=dev) if split == 1 and epi != L.EPI_GELU_BWD else None
    AUX = torch.randn(M, N, device=dev) if epi == L.EPI_RESID else None
    if epi == L.EPI_GELU_BWD:
        AUX = torch.randn(M, N, device=dev).bfloat16()
        D = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    D2 = torch.empty(M, N, device=dev, dtype=torch.bfloat16) if epi == L.EPI_GELU else None
    if epi == L.EPI_GELU:
        D = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    args = (A.data_ptr(), lda, akm, B.data_ptr(), ldb, bkm, D.data_ptr(), N, M, N, K, epi, L.ptr(bias), L.ptr(AUX), N,
            L.ptr(D2), N, split, L.ptr(ws), L.stream_ptr())
    for _ in range(3):
        L.call("jz_gemm_bf16", *args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 20
    for _ in range(n):
        L.call("jz_gemm_bf16", *args)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    tf = 2 * M * N * K / ms / 1e9
    Ab = A.float() if False else None
    print(f"bench M={M} N={N} K={K} akm={akm} bkm={bkm} epi={epi} split={split}: {ms*1e3:.1f} us  {tf:.0f} TFLOP/s", flush=True)


M = 148032
bench(M, 1536, 512)
bench(M, 512, 512, epi=L.EPI_RESID)
bench(M, 2048, 512, epi=L.EPI_GELU)
bench(M, 512, 2048, epi=L.EPI_RESID)
bench(M, 512, 1536, akm=1, bkm=1, epi=L.EPI_F32)
bench(M, 2048, 512, akm=1, bkm=1, epi=L.EPI_GELU_BWD)
bench(512, 1536, M, akm=0, bkm=0, epi=L.EPI_F32, split=6)
bench(2048, 512, M, akm=0, bkm=0, epi=L.EPI_F32, split=4)
from paper_2510_27002_b200.kernels import splitk_for
for (mm, nn) in ((512, 2048), (2048, 512), (512, 1536), (512, 512)):
    bench(mm, nn, M, akm=0, bkm=0, epi=L.EPI_F32, split=splitk_for(mm, nn, M))
print("ALL OK" if ok else "SOME FAILED")
sys.exit(0 if ok else 1)
