import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""DiT train step time (bench.py's dit_train line) for A/B of kernel switches."""
import bench
import torch

r = bench._dit_train(torch.device("cuda", 0))
print(r["value"], r["ms_per_step"])
