"""Kernel breakdown of the C5 rollout (bench 'sample' line)."""
import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity

from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
from paper_2510_27002_b200.rng import stream
from paper_2510_27002_b200.sampling import rollout_device
from paper_2510_27002_b200.tokenizer import TokenizerConfig, VideoTokenizer

dev = torch.device("cuda")
tok = VideoTokenizer(TokenizerConfig(patch=4, codes=1024, latent_dim=32), seed=0)
dyn = DynamicsModel(DynamicsConfig(patches_per_frame=256, max_frames=16), seed=0)
cb = torch.rand(6, 32, device=dev) * 0.3
B = 64
cond = torch.as_tensor(stream(5, "c").integers(0, 256, size=(B, 4, 64, 64, 3)).astype(np.uint8), device=dev)
acts = [stream(5, "acts", i).integers(0, 6, size=(B,)) for i in range(12)]
rollout_device(tok, dyn, cond, acts, horizon=1, steps=2, rng=stream(0, "w"), source_codebook=cb)
for rep in range(2):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    rollout_device(tok, dyn, cond, acts, horizon=12, steps=25, rng=stream(0, "r"), source_codebook=cb)
    b.record()
    torch.cuda.synchronize()
    print("rollout ms", a.elapsed_time(b), flush=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rollout_device(tok, dyn, cond, acts, horizon=12, steps=25, rng=stream(0, "r"), source_codebook=cb)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14, max_name_column_width=60))
