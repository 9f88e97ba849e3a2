import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Spatial attention bwd timing (B=36, S=257/256) against the libjz.so given in argv[1]."""
import torch

from paper_2510_27002_b200 import _lib as L
if len(sys.argv) > 1:
    L.LIB_PATH = pathlib.Path(sys.argv[1]).resolve()
from paper_2510_27002_b200 import kernels as Kn  # noqa: E402

L.ensure_device()
for S in (257, 256):
    frames, H, D = 576, 8, 512
    qkv = torch.randn(frames * S, 3 * D, device="cuda").bfloat16()
    out, olo, lse = Kn.attn_spatial_fwd(qkv, frames, S, H, keep_lo=True)
    dO = torch.randn(frames * S, D, device="cuda").bfloat16()
    dq = torch.empty_like(qkv)
    cs = torch.empty(3 * D, device="cuda")
    fn = lambda: Kn.attn_spatial_bwd(qkv, out, dO, lse, frames, S, H, dqkv=dq, colsum=cs, out_lo=olo)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(f"S={S} bwd {a.elapsed_time(b) / 20 * 1e3:.1f} us ({sys.argv[1] if len(sys.argv) > 1 else 'default'})", flush=True)
