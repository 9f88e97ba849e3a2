import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""C3-stage tokenizer encode (B=36 clips: patchify, 4 ST blocks, to_latent, VQ against 1024 codes)
between cudaProfilerStart/Stop: ncu target for the VQ and elementwise kernels."""
import numpy as np
import torch

from paper_2510_27002_b200.rng import stream
from paper_2510_27002_b200.tokenizer import TokenizerConfig, VideoTokenizer

tok = VideoTokenizer(TokenizerConfig(patch=4, codes=1024, latent_dim=32), seed=0)
frames = torch.as_tensor(stream(0, "f").integers(0, 256, size=(36, 16, 64, 64, 3)).astype(np.uint8), device="cuda")
tok.encode_device(frames)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
tok.encode_device(frames)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
