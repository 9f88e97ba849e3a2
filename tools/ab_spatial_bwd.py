import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Spatial attention backward: accuracy against torch fp32 at frames=40 (several units per CTA) and
event timing at B=36 (576 frames x 8 heads), S = 256 and 257, for the default library and any
alternative builds given as JZ_LIB_PATH values.
usage: python tools/ab_spatial_bwd.py [LIB ...]          (spawns one process per library)"""
import json
import math
import os
import subprocess

if len(sys.argv) == 1 or sys.argv[1] != "run":
    for lib in [""] + sys.argv[1:]:
        env = dict(os.environ, JZ_LIB_PATH=lib) if lib else dict(os.environ)
        out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True)
        print(f"--- {lib or 'default library'}", out.returncode)
        print(out.stdout[-3000:], out.stderr[-3000:])
    sys.exit(0)

import torch

from paper_2510_27002_b200 import _lib as L
from paper_2510_27002_b200 import kernels as Kn

L.ensure_device()
dev = "cuda"


def rel(a, b):
    a, b = a.float(), b.float()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def ref_attn(qkv, frames, S, H):
    x = qkv.float().reshape(frames, S, 3, H, 64)
    q, k, v = (x[..., i, :, :].transpose(-3, -2) for i in range(3))
    s = q @ k.transpose(-1, -2) / math.sqrt(64)
    return (torch.softmax(s, -1) @ v).transpose(-3, -2).reshape(frames, S, H * 64)


res = {}
for S in (257, 256):
    frames, H = 40, 8
    D = H * 64
    g = torch.Generator(device=dev).manual_seed(S)
    qkv = (torch.randn(frames * S, 3 * D, device=dev, generator=g) * 1.5).bfloat16()
    out, olo, lse = Kn.attn_spatial_fwd(qkv, frames, S, H, keep_lo=True)
    qf = qkv.float().requires_grad_(True)
    o = ref_attn(qf, frames, S, H)
    go = torch.randn(o.shape, device=dev, generator=g)
    o.backward(go)
    dqkv = torch.full_like(qkv, float("nan"))
    cs = torch.full((3 * D,), float("nan"), device=dev)
    Kn.attn_spatial_bwd(qkv, out, go.reshape(frames * S, D).bfloat16().contiguous(), lse, frames, S, H, dqkv=dqkv,
                        colsum=cs, out_lo=olo)
    torch.cuda.synchronize()
    cs_ref = torch.empty_like(cs)
    Kn.colsum_bf16(dqkv, cs_ref)
    r = {"finite": bool(torch.isfinite(dqkv.float()).all()), "colsum_rel": rel(cs, cs_ref)}
    for i in range(3):
        got, ref = dqkv[:, i * D:(i + 1) * D], qf.grad[:, i * D:(i + 1) * D]
        r["qkv"[i]] = rel(got, ref)
        if S == 257:
            r["qkv"[i] + "256"] = rel(got.reshape(frames, S, D)[:, -1], ref.reshape(frames, S, D)[:, -1])
    # timing at B = 36
    frames = 576
    qkv = torch.randn(frames * S, 3 * D, device=dev).bfloat16()
    out, olo, lse = Kn.attn_spatial_fwd(qkv, frames, S, H, keep_lo=True)
    dO = torch.randn(frames * S, D, device=dev).bfloat16()
    dq = torch.empty_like(qkv)
    cs = torch.empty(3 * D, device=dev)
    fn = lambda: Kn.attn_spatial_bwd(qkv, out, dO, lse, frames, S, H, dqkv=dq, colsum=cs, out_lo=olo)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        fn()
    b.record()
    torch.cuda.synchronize()
    r["us_b36_incl_uvb_and_colsum_reduce"] = a.elapsed_time(b) / 20 * 1e3
    res[S] = r
print(json.dumps(res, indent=1))
