import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Time jz_attn_temporal_decode at the C5 shape (B=64, S=257, D=512) for frame indices 4/9/15."""
import torch

from paper_2510_27002_b200 import _lib as L

if len(sys.argv) > 1:
    L.LIB_PATH = pathlib.Path(sys.argv[1])
L.ensure_device()
B, S, Tmax, D = 64, 257, 16, 512
qkv = torch.randn(B * S, 3 * D, device="cuda").bfloat16()
cache = torch.randn(B, Tmax, S, 2 * D, device="cuda").bfloat16()
out = torch.empty(B * S, D, device="cuda", dtype=torch.bfloat16)
flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
for t in (4, 9, 15):
    ts = []
    for it in range(12):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        L.call("jz_attn_temporal_decode", qkv.data_ptr(), cache.data_ptr(), B, t, None, Tmax, S, D // 64, 0,
               out.data_ptr(), L.stream_ptr())
        b.record()
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(a.elapsed_time(b) * 1e3)
    us = sorted(ts)[len(ts) // 2]
    nbytes = B * S * (t * 2 * D * 2 + 3 * D * 2 + D * 2)
    print(f"t={t:2d}: {us:7.1f} us  {nbytes / us / 1e3:7.0f} GB/s", flush=True)
