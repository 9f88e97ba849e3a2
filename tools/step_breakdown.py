import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Per-call device-time breakdown of the dynamics train step (B=36, jasmine-base, patch 4).

Wraps every libjz entry point with CUDA events (warm caches, real clocks: not a profiler
replay), runs 3 warm-up + N recorded eager steps and prints the time per (entry point, shape
signature) and its share of the step.  usage: python tools/step_breakdown.py [N] [--json out]
"""
import json
import sys
from collections import defaultdict

import torch

from paper_2510_27002_b200 import _lib as L
from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
from paper_2510_27002_b200.optim import WsdSchedule
from paper_2510_27002_b200.rng import stream
from paper_2510_27002_b200.tensor import Tensor
from paper_2510_27002_b200.trainer import DynamicsTrainStep

n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 3
B = 36
m = DynamicsModel(DynamicsConfig(patches_per_frame=256, max_frames=16), seed=0)
tr = DynamicsTrainStep(m, WsdSchedule(3e-5, 200000, 1000))
tok = torch.as_tensor(stream(1, "bench-tokens").integers(0, 1024, size=(B, 16, 256))).cuda()
lat = Tensor(torch.randn(B, 15, 32, device="cuda") * 0.1)
for k in range(3):
    tr.step(k, tok, lat)
torch.cuda.synchronize()

rec = []
orig = L.call


def sig(name, args):
    ints = [a for a in args if isinstance(a, int) and not isinstance(a, bool) and abs(a) < (1 << 40)]
    if name.startswith("jz_gemm"):
        # A, lda, a_kmajor, B, ldb, b_kmajor, D, ldd, M, N, K, epi, ...
        return f"{name} M={args[8]} N={args[9]} K={args[10]} ak={args[2]} bk={args[5]} epi={args[11]}"
    return f"{name} {tuple(ints[:6])}"


def wrapped(name, *args):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    orig(name, *args)
    b.record()
    rec.append((sig(name, args), a, b))


L.call = wrapped
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(n):
    tr.step(3 + k, tok, lat)
e1.record()
torch.cuda.synchronize()
L.call = orig
step_ms = e0.elapsed_time(e1) / n
agg = defaultdict(lambda: [0.0, 0])
for s, a, b in rec:
    agg[s][0] += a.elapsed_time(b) / n
    agg[s][1] += 1
rows = sorted(agg.items(), key=lambda kv: -kv[1][0])
tot = sum(v[0] for v in agg.values())
print(f"step {step_ms:.3f} ms (with per-call events); sum of calls {tot:.3f} ms")
for s, (ms, c) in rows:
    print(f"{ms * 1e3:9.1f} us  {100 * ms / step_ms:5.1f}%  x{c // n:<3d} {s}")
if "--json" in sys.argv:
    out = sys.argv[sys.argv.index("--json") + 1]
    pathlib.Path(out).write_text(json.dumps({"step_ms": step_ms, "calls": [
        {"sig": s, "us": ms * 1e3, "per_step": c // n} for s, (ms, c) in rows]}, indent=1))
