import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Run the v3 spatial backward from the debug build (bounded barrier waits) at frames from argv."""
import torch

from paper_2510_27002_b200 import _lib as L
L.LIB_PATH = pathlib.Path(__file__).resolve().parent.parent / "paper_2510_27002_b200/lib/dbg/libjz.so"
from paper_2510_27002_b200 import kernels as Kn

L.ensure_device()
frames = int(sys.argv[1]) if len(sys.argv) > 1 else 40
S = int(sys.argv[2]) if len(sys.argv) > 2 else 257
H, D = 8, 512
qkv = torch.randn(frames * S, 3 * D, device="cuda").bfloat16()
out, olo, lse = Kn.attn_spatial_fwd(qkv, frames, S, H, keep_lo=True)
dO = torch.randn(frames * S, D, device="cuda").bfloat16()
dq = torch.full_like(qkv, float("nan"))
cs = torch.empty(3 * D, device="cuda")
Kn.attn_spatial_bwd(qkv, out, dO, lse, frames, S, H, dqkv=dq, colsum=cs, out_lo=olo)
torch.cuda.synchronize()
print("ok", frames, S, bool(torch.isfinite(dq.float()).all()))
