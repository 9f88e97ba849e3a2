import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""One spatial attention fwd + bwd launch pair at B=36 (576 frames x 8 heads), S from argv (257)."""
import torch

from paper_2510_27002_b200 import _lib as L

L.ensure_device()
S = int(sys.argv[1]) if len(sys.argv) > 1 else 257
frames, H = 576, 8
D = H * 64
qkv = torch.randn(frames * S, 3 * D, device="cuda").bfloat16()
out = torch.empty(frames * S, D, device="cuda", dtype=torch.bfloat16)
olo = torch.empty(frames * S, D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(frames, H, S, device="cuda")
dq = torch.empty_like(qkv)
ws = torch.empty(frames * H * 780, device="cuda")
for _ in range(2):
    L.call("jz_attn_spatial_fwd", qkv.data_ptr(), frames, S, H, 64, out.data_ptr(), olo.data_ptr(), lse.data_ptr(), L.stream_ptr())
    L.call("jz_attn_spatial_bwd", qkv.data_ptr(), out.data_ptr(), olo.data_ptr(), out.data_ptr(), lse.data_ptr(), frames, S, H, 64,
           dq.data_ptr(), ws.data_ptr(), None, L.stream_ptr())
torch.cuda.synchronize()
