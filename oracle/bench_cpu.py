"""ORACLE (test infrastructure only) — timing of the CPU restatement for bench.py.

Used solely by bench.py's `cpu_baseline` leg and its `--impl reference` arm: it
times the oracle port of the dynamics training step (dynamics.py:139-153 loss,
autodiff backward, optim.adamw_step) on the host cores at a bounded batch.  The
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
