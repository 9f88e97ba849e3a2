import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Scratch GPU check of attention kernels vs torch fp32."""
import math
import sys
import time

import torch

from paper_2510_27002_b200 import _lib as L

L.ensure_device()
torch.manual_seed(0)
dev = "cuda"
ok = True


def ref_attn(qkv, lead, L_, H, causal):
    D = H * 64
    x = qkv.float().reshape(*lead, L_, 3, H, 64)
    q, k, v = x[..., 0, :, :], x[..., 1, :, :], x[..., 2, :, :]  # (..., L, H, 64)
    q, k, v = q.transpose(-3, -2), k.transpose(-3, -2), v.transpose(-3, -2)
    s = q @ k.transpose(-1, -2) / 8.0
    if causal:
        m = torch.triu(torch.ones(L_, L_, dtype=torch.bool, device=dev), 1)
        s = s.masked_fill(m, -1e9)
    p = torch.softmax(s, -1)
    o = (p @ v).transpose(-3, -2).reshape(*lead, L_, D)
    lse = torch.logsumexp(s, -1)
    return o, lse


def check(name, got, ref, tol):
    global ok
    err = ((got.float() - ref.float()).norm() / ref.float().norm()).item()
    good = err < tol
    ok &= good
    print(f"{name}: relerr={err:.3e} {'OK' if good else 'FAIL'}", flush=True)


for S in (257, 256):
    frames, H = 37, 8
    D = H * 64
    qkv = (torch.randn(frames * S, 3 * D, device=dev) * 1.5).bfloat16()
    out = torch.empty(frames * S, D, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(frames, H, S, device=dev)
    L.call("jz_attn_spatial_fwd", qkv.data_ptr(), frames, S, H, 64, out.data_ptr(), None, lse.data_ptr(), L.stream_ptr())
    torch.cuda.synchronize()
    o_ref, lse_ref = ref_attn(qkv.reshape(frames, S, 3 * D), (frames,), S, H, False)
    check(f"spatial fwd S={S} out", out.reshape(frames, S, D), o_ref, 1e-2)
    check(f"spatial fwd S={S} out row256" if S == 257 else "spatial fwd last", out.reshape(frames, S, D)[:, -1], o_ref[:, -1], 1e-2)
    check(f"spatial fwd S={S} lse", lse, lse_ref, 1e-4)

# temporal
B, T, S, H = 3, 16, 257, 8
D = H * 64
qkv = (torch.randn(B * T * S, 3 * D, device=dev) * 1.5).bfloat16()
out = torch.empty(B * T * S, D, device=dev, dtype=torch.bfloat16)
lse = torch.empty(B * S, H, T, device=dev)
L.call("jz_attn_temporal_fwd", qkv.data_ptr(), B, T, S, H, 64, out.data_ptr(), lse.data_ptr(), L.stream_ptr())
torch.cuda.synchronize()
x = qkv.reshape(B, T, S, 3 * D).transpose(1, 2)  # (B,S,T,3D)
o_ref, lse_ref = ref_attn(x, (B, S), T, H, True)
check("temporal fwd out", out.reshape(B, T, S, D).transpose(1, 2), o_ref, 1e-2)
check("temporal fwd lse", lse.reshape(B, S, H, T), lse_ref, 1e-4)

# temporal bwd
qkv_f = qkv.float().requires_grad_(True)
x = qkv_f.reshape(B, T, S, 3 * D).transpose(1, 2)
o_r, _ = ref_attn(x, (B, S), T, H, True)
go = torch.randn_like(o_r)
o_r.backward(go)
dref = qkv_f.grad.reshape(B * T * S, 3 * D)
dout = go.transpose(1, 2).reshape(B * T * S, D).bfloat16().contiguous()
dqkv = torch.empty_like(qkv)
L.call("jz_attn_temporal_bwd", qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), B, T, S, H, 64,
       dqkv.data_ptr(), None, L.stream_ptr())
torch.cuda.synchronize()
for i, nm in enumerate("qkv"):
    check(f"temporal bwd d{nm}", dqkv[:, i * D:(i + 1) * D], dref[:, i * D:(i + 1) * D], 2e-2)

if "spatial_bwd" in sys.argv:
    for S in (257, 256):
        frames, H = 37, 8
        D = H * 64
        qkv = (torch.randn(frames * S, 3 * D, device=dev) * 1.5).bfloat16()
        out = torch.empty(frames * S, D, device=dev, dtype=torch.bfloat16)
        lse = torch.empty(frames, H, S, device=dev)
        olo = torch.empty(frames * S, D, device=dev, dtype=torch.bfloat16)
        L.call("jz_attn_spatial_fwd", qkv.data_ptr(), frames, S, H, 64, out.data_ptr(), olo.data_ptr(), lse.data_ptr(), L.stream_ptr())
        qkv_f = qkv.float().requires_grad_(True)
        o_r, _ = ref_attn(qkv_f.reshape(frames, S, 3 * D), (frames,), S, H, False)
        go = torch.randn_like(o_r)
        o_r.backward(go)
        dref = qkv_f.grad
        dout = go.reshape(frames * S, D).bfloat16().contiguous()
        dqkv = torch.full_like(qkv, float("nan"))
        L.call("jz_attn_spatial_bwd", qkv.data_ptr(), out.data_ptr(), olo.data_ptr(), dout.data_ptr(), lse.data_ptr(), frames, S, H,
               64, dqkv.data_ptr(), torch.empty(frames * H * 780, device=dev).data_ptr(), None, L.stream_ptr())
        torch.cuda.synchronize()
        for i, nm in enumerate("qkv"):
            check(f"spatial bwd S={S} d{nm}", dqkv[:, i * D:(i + 1) * D], dref[:, i * D:(i + 1) * D], 2e-2)
            check(f"spatial bwd S={S} d{nm} last row", dqkv.reshape(frames, S, 3 * D)[:, -1, i * D:(i + 1) * D],
                  dref.reshape(frames, S, 3 * D)[:, -1, i * D:(i + 1) * D], 2e-2)


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


frames, S, H = 576, 257, 8
D = H * 64
qkv = torch.randn(frames * S, 3 * D, device=dev).bfloat16()
out = torch.empty(frames * S, D, device=dev, dtype=torch.bfloat16)
lse = torch.empty(frames, H, S, device=dev)
olo = torch.empty(frames * S, D, device=dev, dtype=torch.bfloat16)
us = timeit(lambda: L.call("jz_attn_spatial_fwd", qkv.data_ptr(), frames, S, H, 64, out.data_ptr(), olo.data_ptr(), lse.data_ptr(), L.stream_ptr()))
fl = 4 * frames * H * S * S * 64
print(f"spatial fwd B36: {us:.1f} us  {fl / us / 1e6:.0f} TFLOP/s", flush=True)
lse_t = torch.empty(36 * S, H, 16, device=dev)
us = timeit(lambda: L.call("jz_attn_temporal_fwd", qkv.data_ptr(), 36, 16, S, H, 64, out.data_ptr(), lse_t.data_ptr(), L.stream_ptr()))
print(f"temporal fwd B36: {us:.1f} us  {(qkv.numel() * 2 + out.numel() * 2) / us / 1e3:.0f} GB/s", flush=True)
dq = torch.empty_like(qkv)
WS = torch.empty(frames * H * 780, device='cuda')
us = timeit(lambda: L.call("jz_attn_temporal_bwd", qkv.data_ptr(), out.data_ptr(), out.data_ptr(), lse_t.data_ptr(), 36, 16, S, H, 64, dq.data_ptr(), None, L.stream_ptr()))
print(f"temporal bwd B36: {us:.1f} us  {(qkv.numel() * 4 + out.numel() * 4) / us / 1e3:.0f} GB/s", flush=True)
if "spatial_bwd" in sys.argv:
    us = timeit(lambda: L.call("jz_attn_spatial_bwd", qkv.data_ptr(), out.data_ptr(), olo.data_ptr(), out.data_ptr(), lse.data_ptr(), frames, S, H, 64, dq.data_ptr(), WS.data_ptr(), None, L.stream_ptr()))
    print(f"spatial bwd B36: {us:.1f} us  {2.5 * fl / us / 1e6:.0f} TFLOP/s", flush=True)
print("ALL OK" if ok else "SOME FAILED")
sys.exit(0 if ok else 1)
