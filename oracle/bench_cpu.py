"""ORACLE (test infrastructure only) — timing of the CPU restatement for bench.py.

Used solely by bench.py's `cpu_baseline` legs and its `--impl reference` arm: it
times the oracle port of each BASELINE configuration on the host cores at a
bounded batch -- the dynamics training step (dynamics.py:139-153 loss, autodiff
backward, optim.adamw_step), the tokenizer forward + quantize (tokenizer.py:134-143),
the LAM training step (lam.py:120-129 + backward + AdamW) and one MaskGIT frame
decode (dynamics.py:156-194).  The
real deskworld package cannot travel to the GPU box (/root/reference is only in
the build container), so the port is the reference arm there; SURVEY §6 lists
the reference's own numbers measured in the build container for comparison.
"""
from __future__ import annotations

import os
import time

import numpy as np
import torch

from . import model as M
from . import rng as R


def time_dynamics_step(batch: int = 1, steps: int = 2, warmup: int = 1, threads: int | None = None,
                       blocks: int = 6) -> dict:
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    cfg = M.DynCfg(model_dim=512, heads=8, ffn_dim=2048, blocks=blocks, token_codes=1024, action_latent_dim=32,
                   patches_per_frame=256, max_frames=16)
    init = M.init_dynamics(cfg, seed=0)
    P = M.params_to_torch(init)
    adam = M.adamw_init({k: v for k, v in init.items()})
    tokens = R.stream(1, "bench-tokens").integers(0, 1024, size=(batch, 16, 256))
    lam_cb = R.stream(2, "golden-lam-cb").uniform(-1 / 6, 1 / 6, size=(6, 32)).astype(np.float32)
    lat = torch.tensor(lam_cb[R.stream(2, "bench-actions").integers(0, 6, size=(batch, 15))])
    times = []
    for k in range(warmup + steps):
        t0 = time.perf_counter()
        mask = R.sample_masks(R.PhiloxState.fresh(R.fold_key(0, "dynamics", "step", k)), batch, 16, 256)
        loss, _ = M.dyn_loss(P, cfg, tokens, lat, mask)
        for p in P.values():
            p.grad = None
        loss.backward()
        np_params = {n: p.detach().numpy() for n, p in P.items()}
        M.adamw_step(np_params, {n: p.grad.numpy() for n, p in P.items()}, adam, 3e-5)
        if k >= warmup:
            times.append(time.perf_counter() - t0)
    s = float(np.mean(times))
    return {"seconds_per_step": s, "frames_per_s": batch * 16 / s, "threads": threads, "batch": batch,
            "steps": steps}


def host_info() -> dict:
    """CPU model, logical cores and the BLAS / intra-op thread counts the timings ran with."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": d.get("internal_api"), "threads": d.get("num_threads")} for d in threadpool_info()]
    except Exception:
        pass
    return {"cpu_model": model, "logical_cores": os.cpu_count(), "torch_threads": torch.get_num_threads(),
            "blas": blas}


JB = dict(model_dim=512, heads=8, ffn_dim=2048)


def _frames(batch: int, t: int = 16) -> np.ndarray:
    return R.stream(0, "bench-frames").integers(0, 256, size=(batch, t, 64, 64, 3)).astype(np.uint8)


def time_tokenizer_fwd(batch: int = 2, steps: int = 1, warmup: int = 1, threads: int | None = None) -> dict:
    """C1: tokenizer forward (encode, VQ, decode, losses) at jasmine-base dims, patch 4."""
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    cfg = M.TokCfg(**JB, blocks=4, codes=1024, latent_dim=32, patch=4, height=64, width=64, max_frames=16)
    P = M.params_to_torch(M.init_tokenizer(cfg, seed=0), requires_grad=False)
    unit = torch.tensor(M.frames_to_unit(_frames(batch)))
    times = []
    with torch.no_grad():
        for k in range(warmup + steps):
            t0 = time.perf_counter()
            M.tok_forward(P, cfg, unit)
            if k >= warmup:
                times.append(time.perf_counter() - t0)
    s = float(np.mean(times))
    return {"seconds_per_step": s, "frames_per_s": batch * 16 / s, "threads": threads, "batch": batch}


def time_lam_step(batch: int = 1, steps: int = 1, warmup: int = 1, threads: int | None = None) -> dict:
    """C2: LAM train step (forward, backward, AdamW) at jasmine-base dims, 6 codes."""
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    cfg = M.LamCfg(**JB, blocks=4, codes=6, latent_dim=32, patch=4, height=64, width=64, max_frames=16)
    init = M.init_lam(cfg, seed=0)
    P = M.params_to_torch(init)
    adam = M.adamw_init({k: v for k, v in init.items()})
    unit = torch.tensor(M.frames_to_unit(_frames(batch)))
    times = []
    for k in range(warmup + steps):
        t0 = time.perf_counter()
        for p in P.values():
            p.grad = None
        _, _, losses = M.lam_forward(P, cfg, unit)
        losses["total"].backward()
        np_params = {n: p.detach().numpy() for n, p in P.items()}
        M.adamw_step(np_params, {n: (p.grad.numpy() if p.grad is not None else None) for n, p in P.items()},
                     adam, 3e-5)
        if k >= warmup:
            times.append(time.perf_counter() - t0)
    s = float(np.mean(times))
    return {"seconds_per_step": s, "frames_per_s": batch * 16 / s, "threads": threads, "batch": batch}


def time_decode_frame(batch: int = 1, context: int = 10, steps: int = 25, threads: int | None = None) -> dict:
    """C5 sample: one generated frame (25 MaskGIT refinements, each a full-clip forward as the
    reference runs it) at `context` frames of history -- the middle of the 4 -> 16 rollout."""
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    cfg = M.DynCfg(**JB, blocks=6, token_codes=1024, action_latent_dim=32, patches_per_frame=256, max_frames=16)
    P = M.params_to_torch(M.init_dynamics(cfg, seed=0), requires_grad=False)
    prev = R.stream(5, "cpu-dec-prev").integers(0, 1024, size=(batch, context, 256))
    lat = (R.stream(5, "cpu-dec-lat").normal(size=(batch, context, 32)) * 0.1).astype(np.float32)

    def logits_fn(tk, la, mask):
        with torch.no_grad():
            return M.dyn_logits(P, cfg, tk, torch.tensor(la), mask).numpy()

    t0 = time.perf_counter()
    M.decode_frame(logits_fn, prev, lat, steps=steps, gen=R.stream(0, "cpu-dec"))
    s = time.perf_counter() - t0
    return {"seconds_per_frame": s, "frames_per_s": batch / s, "threads": threads, "batch": batch,
            "context": context, "maskgit_steps": steps}
