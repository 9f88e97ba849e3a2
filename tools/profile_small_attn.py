"""Small-frame spatial attention (K3s) at the ST-DiT bench shape: 576 frames x S = 18, 8 heads.
Runs fwd + bwd a few times (for ncu: -k regex:rowtile)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2510_27002_b200 import kernels as Kn  # noqa: E402

frames, S, H, D = 576, int(sys.argv[1]) if len(sys.argv) > 1 else 18, 8, 512
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn(frames * S, 3 * D, device="cuda", generator=g).bfloat16()
do = torch.randn(frames * S, D, device="cuda", generator=g).bfloat16()
dq = torch.empty_like(qkv)
for _ in range(3):
    o, _, lse = Kn.attn_spatial_fwd(qkv, frames, S, H)
    Kn.attn_spatial_bwd(qkv, o, do, lse, frames, S, H, dqkv=dq)
torch.cuda.synchronize()
print("ok")
