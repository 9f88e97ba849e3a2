import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Spatial attention fwd/bwd timing at B=36 (576 frames x 8 heads), S = 256 and 257."""
import torch

from paper_2510_27002_b200 import _lib as L

L.ensure_device()
dev = "cuda"


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


for S in (256, 257):
    frames, H = 576, 8
    D = H * 64
    qkv = torch.randn(frames * S, 3 * D, device=dev).bfloat16()
    out = torch.empty(frames * S, D, device=dev, dtype=torch.bfloat16)
    olo = torch.empty(frames * S, D, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(frames, H, S, device=dev)
    dq = torch.empty_like(qkv)
    WS = torch.empty(frames * H * 780, device='cuda')
    f = lambda: L.call("jz_attn_spatial_fwd", qkv.data_ptr(), frames, S, H, 64, out.data_ptr(), olo.data_ptr(), lse.data_ptr(), L.stream_ptr())
    f2 = lambda: L.call("jz_attn_spatial_fwd", qkv.data_ptr(), frames, S, H, 64, out.data_ptr(), None, lse.data_ptr(), L.stream_ptr())
    bw = lambda: L.call("jz_attn_spatial_bwd", qkv.data_ptr(), out.data_ptr(), olo.data_ptr(), out.data_ptr(), lse.data_ptr(), frames, S, H, 64, dq.data_ptr(), WS.data_ptr(), None, L.stream_ptr())
    fl = 4 * frames * H * S * S * 64
    for name, fn, mult in (("fwd+residual", f, 1), ("fwd", f2, 1), ("bwd", bw, 2.5)):
        us = timeit(fn)
        print(f"S={S} {name}: {us:.1f} us  {mult * fl / us / 1e6:.0f} TFLOP/s", flush=True)
