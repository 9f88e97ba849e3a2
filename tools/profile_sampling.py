import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
import time
import numpy as np
import torch
from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
from paper_2510_27002_b200.rng import stream
from paper_2510_27002_b200.sampling import FrameDecoder, rollout_device
from paper_2510_27002_b200.tokenizer import TokenizerConfig, VideoTokenizer
dev = torch.device("cuda")
tok = VideoTokenizer(TokenizerConfig(patch=4), seed=0)
dyn = DynamicsModel(DynamicsConfig(patches_per_frame=256, max_frames=16), seed=0)
cb = torch.rand(6, 32, device=dev) * 0.3
B = 64
cond = torch.as_tensor(stream(5, "c").integers(0, 256, size=(B, 4, 64, 64, 3)).astype(np.uint8), device=dev)
acts = [np.zeros(B, dtype=np.int64) for _ in range(12)]
def ev(fn, n=1):
    torch.cuda.synchronize(); t0 = time.time()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True); a.record()
    for _ in range(n): r = fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n, (time.time() - t0) * 1e3 / n, r
rollout_device(tok, dyn, cond, acts, horizon=1, steps=2, rng=stream(0, "w"), source_codebook=cb)
print("encode", ev(lambda: tok.encode_device(cond))[:2])
tokens = tok.encode_device(cond)
all_tok = torch.randint(0, 1024, (B, 16, 256), device=dev)
print("tok decode 16 frames", ev(lambda: tok.decode_device(all_tok))[:2])
lat = torch.zeros(B, 15, 32, device=dev)
dec = FrameDecoder(dyn, B, 16)
print("prefill 4", ev(lambda: dec.prefill(tokens, lat[:, :3]))[:2])
g = stream(0, "x")
print("decode frame (first, captures)", ev(lambda: dec.decode(lat[:, 3], 25, 1.0, g))[:2])
print("decode frame (graph)", ev(lambda: dec.decode(lat[:, 3], 25, 1.0, g))[:2])
print("single eager step", ev(lambda: dec._step(1.0), 5)[:2])
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    dec._step(1.0); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
