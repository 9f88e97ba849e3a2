import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Time jz_maskgit_step (sampler + selection) at the C5 shape: 64 x 256 rows of 1024 logits."""
import ctypes as C
import torch

from paper_2510_27002_b200 import _lib as L

if len(sys.argv) > 1:
    L.LIB_PATH = pathlib.Path(sys.argv[1])
L.ensure_device()
B, N, K = 64, 256, 1024
logits = torch.randn(B * N, K, device="cuda") * 3
cur = torch.zeros(B, N, dtype=torch.int64, device="cuda")
known = torch.zeros(B, N, dtype=torch.uint8, device="cuda")
conf = torch.empty(B, N, device="cuda")
z = (C.c_uint64 * 4)(1, 2, 3, 4)
k = (C.c_uint64 * 4)(5, 6)
flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
ts = []
for it in range(12):
    flush.zero_()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    L.call("jz_maskgit_step", logits.data_ptr(), B, N, K, 1.0, C.addressof(z), C.addressof(k), C.addressof(z), 4, 0, 9,
           None, cur.data_ptr(), known.data_ptr(), conf.data_ptr(), L.stream_ptr())
    b.record()
    torch.cuda.synchronize()
    if it >= 2:
        ts.append(a.elapsed_time(b) * 1e3)
us = sorted(ts)[len(ts) // 2]
print(f"maskgit step: {us:.1f} us  {B * N * K * 4 / us / 1e3:.0f} GB/s  cur checksum {int(cur.sum())}", flush=True)
