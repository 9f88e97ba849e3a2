import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Spatial attention fwd timing (B=36, S=257/256, with / without the fp32 O copy) against the libjz.so in argv[1]."""
import torch

from paper_2510_27002_b200 import _lib as L
if len(sys.argv) > 1:
    L.LIB_PATH = pathlib.Path(sys.argv[1]).resolve()
from paper_2510_27002_b200 import kernels as Kn  # noqa: E402

L.ensure_device()
for S in (257, 256):
    frames, H, D = 576, 8, 512
    qkv = torch.randn(frames * S, 3 * D, device="cuda").bfloat16()
    for keep in (True, False):
        fn = lambda: Kn.attn_spatial_fwd(qkv, frames, S, H, keep_lo=keep)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            fn()
        b.record()
        torch.cuda.synchronize()
        print(f"S={S} fwd keep_lo={keep}: {a.elapsed_time(b) / 20 * 1e3:.1f} us ({pathlib.Path(sys.argv[1]).name if len(sys.argv) > 1 else 'default'})", flush=True)
