"""One eager MaskGIT refinement step of the C5 decoder (B=64, frame index 8) between
cudaProfilerStart/Stop: target for `ncu --profile-from-start off` launch lists."""
import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
import torch

from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
from paper_2510_27002_b200.rng import stream
from paper_2510_27002_b200.sampling import FrameDecoder

dev = torch.device("cuda")
dyn = DynamicsModel(DynamicsConfig(patches_per_frame=256, max_frames=16), seed=0)
B, t0 = 64, int(sys.argv[1]) if len(sys.argv) > 1 else 8
tokens = torch.as_tensor(stream(1, "t").integers(0, 1024, size=(B, t0, 256)), device=dev)
lat = torch.randn(B, 15, 32, device=dev) * 0.1
dec = FrameDecoder(dyn, B, 16)
dec.prefill(tokens, lat[:, :t0 - 1])
dec.decode(lat[:, t0 - 1], 2, 1.0, stream(0, "x"))  # captures graphs, appends frame t0
dec._static(dev)
dec._dev_t.fill_(dec.t)
for _ in range(3):
    dec._step(1.0)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
dec._step(1.0)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok t =", dec.t)
