#!/usr/bin/env python
"""Benchmark: MaskGIT dynamics training frames/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload: jasmine-base dynamics (D=512, 8 heads, FFN 2048,
6 ST blocks, 1024 token codes, 32-d latent actions, prepend conditioning) on
CoinRun-shaped clips (T=16 frames of 64x64x3 at patch 4 -> 16x256 tokens).
One step = device Philox masks + forward + masked CE + backward (+ NCCL
all-reduce when N>1) + AdamW, on synthetic tokens/latents with random-init
weights.  Per-GPU batch is 36 (weak scaling: the 8-GPU run is C4's global 288).

Prints ONE JSON line on rank 0.  `value` is device-resident throughput (CUDA
events, max over ranks); `e2e` adds the per-step H2D copy of the step's tokens
and latents from pinned host memory and the D2H read of the loss through the
public API.  `--impl reference` times the CPU oracle port of the same step on the
host cores instead (the deskworld reference itself cannot travel to the GPU box).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FRAMES_T, PATCHES, CODES, DLAT = 16, 256, 1024, 32
METRIC = "dynamics train frames/sec"
UNIT = "frames/s"


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"bf16_tflops": d.get("bf16_tflops", 1590.0), "bf16_sustained": d.get("bf16_tflops_sustained", 1400.0),
                "hbm_gbs": d.get("hbm_gbs", 6650.0), "source": "MEASURED_PEAKS.json"}
    return {"bf16_tflops": 1590.0, "bf16_sustained": 1400.0, "hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while active."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=1)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(steps: int = 2) -> dict:
    from oracle.bench_cpu import host_info, time_dynamics_step
    r = time_dynamics_step(batch=1, steps=steps, warmup=1)
    return {"value": round(r["frames_per_s"], 4), "unit": UNIT, "cores": r["threads"], "kind": "port",
            "sample": f"oracle port (torch-CPU fp32 restatement of deskworld) dynamics train step, jasmine-base dims, "
                      f"B=1 (16 frames), {steps} timed steps after 1 warm-up, {r['seconds_per_step']:.2f} s/step",
            "host": host_info()}


def cpu_baseline_secondary() -> dict:
    """SURVEY §8d CPU timing plan for the other BASELINE configs (oracle port, all host cores):
    C1 tokenizer forward at B=2, C2 LAM train step at B=1, C5 one generated frame at B=1."""
    from oracle.bench_cpu import time_decode_frame, time_lam_step, time_tokenizer_fwd
    out = {}
    r = time_tokenizer_fwd(batch=2, steps=1, warmup=1)
    out["tokenizer_fwd"] = {"value": round(r["frames_per_s"], 3), "unit": "frames/s", "cores": r["threads"],
                            "kind": "port", "sample": f"C1 tokenizer forward + quantize, B=2 (32 frames), 1 timed "
                                                      f"step after 1 warm-up, {r['seconds_per_step']:.2f} s"}
    r = time_lam_step(batch=1, steps=1, warmup=1)
    out["lam_train"] = {"value": round(r["frames_per_s"], 3), "unit": "frames/s", "cores": r["threads"],
                        "kind": "port", "sample": f"C2 LAM forward + backward + AdamW, B=1 (16 frames), 1 timed "
                                                  f"step after 1 warm-up, {r['seconds_per_step']:.2f} s"}
    r = time_decode_frame(batch=1, context=10, steps=25)
    out["sample"] = {"value": round(r["frames_per_s"], 4), "unit": "frames/s", "cores": r["threads"],
                     "kind": "port", "sample": f"C5 one generated frame at B=1: 25 MaskGIT refinements, each the "
                                               f"reference's full-clip forward over 10 context frames (mid-rollout), "
                                               f"{r['seconds_per_frame']:.2f} s"}
    return out


def _events_ms(fn, reps: int = 1) -> float:
    import torch
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def secondary_configs(dev) -> dict:
    """BASELINE configs other than the headline: C5 sampling (generated frames/s), C2 LAM train
    step and C1 tokenizer forward (frames/s), jasmine-base dims at patch 4, synthetic data."""
    import numpy as np
    import torch

    from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
    from paper_2510_27002_b200.lam import LamConfig, LatentActionModel
    from paper_2510_27002_b200.rng import stream
    from paper_2510_27002_b200.sampling import rollout_device
    from paper_2510_27002_b200.tokenizer import TokenizerConfig, VideoTokenizer

    out = {}
    tok = VideoTokenizer(TokenizerConfig(patch=4, codes=1024, latent_dim=32), seed=0)
    dyn = DynamicsModel(DynamicsConfig(patches_per_frame=PATCHES, max_frames=FRAMES_T), seed=0)
    lam_cb = torch.as_tensor(stream(2, "bench-lam-codebook").uniform(-1 / 6, 1 / 6, size=(6, DLAT)).astype(np.float32),
                             device=dev)
    # C5: batch 64, 4 conditioning frames -> 12 generated, 25 MaskGIT steps, temperature 1
    B5 = 64
    cond = torch.as_tensor(stream(5, "cond-frames").integers(0, 256, size=(B5, 4, 64, 64, 3)).astype(np.uint8),
                           device=dev)
    acts = [stream(5, "acts", i).integers(0, 6, size=(B5,)) for i in range(12)]
    rollout_device(tok, dyn, cond, acts, horizon=1, steps=2, rng=stream(0, "roll-warm"), source_codebook=lam_cb)
    runs = [_events_ms(lambda: rollout_device(tok, dyn, cond, acts, horizon=12, steps=25, rng=stream(0, "roll"),
                                              source_codebook=lam_cb)) for _ in range(2)]
    ms = min(runs)
    gen = B5 * 12
    out["sample"] = {"metric": "sample frames/sec (generated)", "value": round(gen / (ms / 1e3), 1),
                     "unit": "frames/s", "ms_per_rollout": round(ms, 1), "rollouts_ms": [round(r, 1) for r in runs],
                     "config": "C5: batch 64, 4 cond -> 12 generated frames, 25 MaskGIT steps, T=1, KV-cached "
                               "last-frame forward, tokenizer encode+decode included",
                     "algorithmic_tflops": round(351.2e9 * gen / (ms / 1e3) / 1e12, 1),
                     "roofline": _frac_line(351.2e9 * gen / (ms / 1e3),
                                            "SURVEY §8d: 351.2 GFLOP per generated frame (KV-cached dynamics)")}
    # C2: LAM train step (forward, backward and AdamW: run_stage's step body), B=8, T=16
    from paper_2510_27002_b200.optim import WsdSchedule
    from paper_2510_27002_b200.trainer import lam_stage, tokenizer_stage
    lam = LatentActionModel(LamConfig(patch=4, codes=6, latent_dim=32), seed=0)
    fr8 = torch.as_tensor(stream(0, "bench-frames").integers(0, 256, size=(8, FRAMES_T, 64, 64, 3)).astype(np.uint8),
                          device=dev)
    lam_tr = lam_stage(lam, WsdSchedule(peak_lr=3e-5, total_steps=200_000), seed=0)
    lam_run = _graphed(lam_tr, fr8)
    lam_k = [1]

    def lam_step():
        lam_run.step(lam_k[0], fr8)
        lam_k[0] += 1

    lam_step()
    ms2 = _events_ms(lam_step, reps=3)
    lam_tr.opt.raise_if_nonfinite()
    out["lam_train"] = {"metric": "LAM train frames/sec", "value": round(8 * FRAMES_T / (ms2 / 1e3), 1),
                        "unit": "frames/s", "ms_per_step": round(ms2, 2),
                        "config": "C2: B=8, T=16, 6 codes; forward + backward + AdamW (trainer.lam_stage), "
                                  f"replayed as {'a CUDA graph' if lam_run is not lam_tr else 'eager steps'}",
                        "model_tflops": round(53.37e9 * 8 * FRAMES_T / (ms2 / 1e3) / 1e12, 1),
                        "roofline": _frac_line(53.37e9 * 8 * FRAMES_T / (ms2 / 1e3),
                                               "SURVEY §8d: 53.37 GFLOP per trained frame (3x forward)")}
    # C1: tokenizer forward (encode + VQ + decode + losses), B=2; static shapes, so the forward is
    # captured once as a CUDA graph (indices stay on device) and replayed
    fr2 = fr8[:2].clone()
    tok.forward(fr2)
    ms1_eager = _events_ms(lambda: tok.forward(fr2), reps=5)
    ms1, c1_mode = ms1_eager, "eager (indices copied to the host, as the reference API returns them)"
    try:
        from paper_2510_27002_b200.sampling import _no_gc
        tok.forward(fr2, _indices_on_device=True)
        torch.cuda.synchronize()
        g1 = torch.cuda.CUDAGraph()
        with _no_gc(), torch.cuda.graph(g1):
            tok.forward(fr2, _indices_on_device=True)
        g1.replay()
        ms1 = _events_ms(g1.replay, reps=10)
        c1_mode = "CUDA graph replay (indices on device)"
    except Exception as exc:
        c1_mode += f"; graph capture failed: {type(exc).__name__}"
        torch.cuda.synchronize()
    out["tokenizer_fwd"] = {"metric": "tokenizer fwd+quantize frames/sec", "value": round(2 * FRAMES_T / (ms1 / 1e3), 1),
                            "unit": "frames/s", "ms_per_step": round(ms1, 2),
                            "eager_ms_per_step": round(ms1_eager, 2),
                            "config": f"C1: B=2, T=16, 1024 codes; {c1_mode}",
                            "roofline": _frac_line(18.35e9 * 2 * FRAMES_T / (ms1 / 1e3),
                                                   "SURVEY §8d: 18.35 GFLOP per frame (encoder + decoder)")}

    # tokenizer training step: forward + full backward + AdamW, B=8
    tok_tr = tokenizer_stage(tok, WsdSchedule(peak_lr=3e-5, total_steps=200_000), seed=0)
    tok_run = _graphed(tok_tr, fr8)
    tok_k = [1]

    def tok_step():
        tok_run.step(tok_k[0], fr8)
        tok_k[0] += 1

    tok_step()
    ms3 = _events_ms(tok_step, reps=3)
    tok_tr.opt.raise_if_nonfinite()
    out["tokenizer_train"] = {"metric": "tokenizer train frames/sec", "value": round(8 * FRAMES_T / (ms3 / 1e3), 1),
                              "unit": "frames/s", "ms_per_step": round(ms3, 2),
                              "config": "B=8, T=16, 1024 codes, recon + VQ losses, full backward + AdamW "
                                        "(trainer.tokenizer_stage)"}
    out["tokenizer_fwd"]["fp32_kernels"] = _fp32_kernels(dev)
    out["pretrain_lam_stage"] = _pretrain_lam_stage(tok, lam, dev)
    out["play_act"] = _play_act(tok, lam, dev)
    out["dit_train"] = _dit_train(dev)
    return out


def _ffma_peak() -> tuple:
    p = ROOT / "profiles" / "r02" / "ffma_peak.json"
    if p.exists():
        return float(json.loads(p.read_text())["ffma_tflops"]), "profiles/r02/ffma_peak.json (tools/ffma_peak.cu)"
    return 72.3, "fallback: 148 SM x 128 FFMA x 2 x 1.965 GHz measured 72.3"


def _fp32_kernels(dev) -> dict:
    """The fp32 (CUDA-core FFMA) kernels of the tokenizer / LAM path at the pretrain_lam stage shape
    (R = 36 x 16 x 256 latent rows): the fused VQ distance + argmin + gather (K = 1024 codes, dz = 32)
    and the 512 -> 32 latent projection, event-timed, against the measured FFMA peak."""
    import torch

    from paper_2510_27002_b200 import kernels as Kn
    R = 36 * FRAMES_T * PATCHES
    g = torch.Generator(device=dev).manual_seed(0)
    z = torch.randn(R, 32, device=dev, generator=g)
    cb = torch.randn(1024, 32, device=dev, generator=g)
    x = torch.randn(R, 512, device=dev, generator=g)
    w = torch.randn(512, 32, device=dev, generator=g) * 0.05
    b = torch.zeros(32, device=dev)
    peak, src = _ffma_peak()
    out = {}
    for name, fn, flops in (("vq_fwd", lambda: Kn.vq_fwd(z, cb), 2.0 * R * 1024 * 32),
                            ("latent_projection_512x32", lambda: Kn.linear_f32(x, w, b), 2.0 * R * 512 * 32)):
        fn()
        us = 1e3 * _events_ms(fn, reps=10)
        tf = flops / us / 1e6
        out[name] = {"us_per_launch": round(us, 1), "tflops": round(tf, 1), "frac_ffma_peak": round(tf / peak, 3)}
    out["ffma_peak_tflops"] = peak
    out["peak_source"] = src
    out["shape"] = f"R = {R} latent rows (B=36 clips)"
    return out


def _frac_line(flops_per_s: float, basis: str) -> dict:
    """Whole-model throughput against the bf16 tensor peak (these steps are GEMM-dominated)."""
    pk = _peaks()
    tf = flops_per_s / 1e12
    return {"bound": "tensor", "achieved": round(tf, 1), "peak": pk["bf16_sustained"], "unit": "TFLOP/s",
            "frac": round(tf / pk["bf16_sustained"], 4), "basis": basis,
            "peak_source": f"{pk['source']} bf16_tflops_sustained"}


def _dit_train(dev) -> dict:
    """ST-DiT diffusion-forcing train step at the reference's DitConfig defaults
    (512 wide, 6 blocks, 16 latent patches -> S = 18, T = 16), B = 36: host tau / eps draws and
    their H2D copy, forward, ramp-weighted loss, full backward, AdamW. Plus the small-frame
    spatial attention kernels (K3s) alone at that shape, against their HBM roofline."""
    import numpy as np
    import torch

    from paper_2510_27002_b200 import kernels as Kn
    from paper_2510_27002_b200.diffusion import DitConfig, DitDynamics
    from paper_2510_27002_b200.optim import adamw_init, adamw_step
    from paper_2510_27002_b200.rng import stream

    B, T, N = 36, FRAMES_T, 16
    dit = DitDynamics(DitConfig(), seed=0)
    lat = np.tanh(stream(3, "dit-bench").normal(size=(B, T, N, 32))).astype(np.float32)
    act = (stream(4, "dit-bench").normal(size=(B, T - 1, 32)) * 0.1).astype(np.float32)
    opt = adamw_init(dit.params)
    k = [0]

    def step():
        loss = dit.loss(lat, act, stream(0, "dit", "step", k[0]))
        loss.backward()
        adamw_step(dit.params, {n: p.grad for n, p in dit.params.items()}, opt, 1e-4)
        k[0] += 1

    for _ in range(3):
        step()
    ms = _events_ms(step, reps=10)
    frames, S, H, D = B * T, N + 2, 8, 512
    g = torch.Generator(device=dev).manual_seed(0)
    qkv = torch.randn(frames * S, 3 * D, device=dev, generator=g).bfloat16()
    o, _, lse = Kn.attn_spatial_fwd(qkv, frames, S, H)
    do = torch.randn(frames * S, D, device=dev, generator=g).bfloat16()
    dq = torch.empty_like(qkv)
    fwd_us = 1e3 * _events_ms(lambda: Kn.attn_spatial_fwd(qkv, frames, S, H), reps=20)
    bwd_us = 1e3 * _events_ms(lambda: Kn.attn_spatial_bwd(qkv, o, do, lse, frames, S, H, dqkv=dq), reps=20)
    hbm = _peaks()["hbm_gbs"]
    fwd_b = frames * S * (3 * D * 2 + D * 2 + H * 4)
    bwd_b = frames * S * (3 * D * 2 + D * 2 + H * 4 + 3 * D * 2)
    return {"metric": "DiT train frames/sec", "value": round(B * T / (ms / 1e3), 1), "unit": "frames/s",
            "ms_per_step": round(ms, 2),
            "config": "ST-DiT at DitConfig defaults (512 wide, 8 heads, 6 blocks, 16 latent patches, S = 18), "
                      "B=36, T=16; host tau/eps draws + H2D, forward, loss, full backward, AdamW (eager; 10 steps "
                      "after 3 warm-up)",
            "attention_small": {"S": S, "frames": frames,
                                "fwd_us": round(fwd_us, 1), "fwd_gbs": round(fwd_b / fwd_us / 1e3, 1),
                                "fwd_frac_hbm": round(fwd_b / fwd_us / 1e3 / hbm, 3),
                                "bwd_us": round(bwd_us, 1), "bwd_gbs": round(bwd_b / bwd_us / 1e3, 1),
                                "bwd_frac_hbm": round(bwd_b / bwd_us / 1e3 / hbm, 3),
                                "bytes": "fwd: qkv in, O + lse out; bwd: qkv, dO, lse in, dqkv out"}}


def _play_act(tok, lam, dev) -> dict:
    """one interactive play session (B=1, jasmine-base dims, 25 MaskGIT steps) on
    the device sampler; latency of an 'act' (next frame decoded over the session's KV cache,
    tokenizer-decoded, PNG-encoded), including the window slide once the clip reaches 16 frames."""
    import time

    import numpy as np
    import torch

    from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
    from paper_2510_27002_b200.play import PlayService
    from paper_2510_27002_b200.rng import stream

    dyn = DynamicsModel(DynamicsConfig(patches_per_frame=PATCHES, max_frames=FRAMES_T), seed=0)
    svc = PlayService(tok, dyn, lam=lam,
                      episode_fn=lambda seed, n: stream(4, "play-episode", seed).integers(0, 256, size=(n, 64, 64, 3))
                      .astype(np.uint8))
    sid = svc.handle({"type": "reset", "seed": 1})["session"]
    for a in range(3):  # graph capture and first-use costs
        svc.handle({"type": "act", "session": sid, "action": a % 6})
    torch.cuda.synchronize()
    lat = []
    for a in range(20):  # crosses the 16-frame window (slides re-prefill the cache)
        t0 = time.perf_counter()
        r = svc.handle({"type": "act", "session": sid, "action": a % 6})
        lat.append((time.perf_counter() - t0) * 1e3)
        assert r["type"] == "frames"
    lat.sort()
    return {"metric": "play act latency (ms, median)", "value": round(lat[len(lat) // 2], 2), "unit": "ms",
            "higher_is_better": False, "p90_ms": round(lat[int(0.9 * (len(lat) - 1))], 2),
            "config": "PlayService session, B=1, jasmine-base dynamics + tokenizer, 25 MaskGIT steps, KV-cached "
                      "decode, PNG frame out; 20 acts after 3 warm-up, host wall clock per act"}


def _graphed(stage, frames):
    """A stage step replayed as a CUDA graph (trainer.GraphedStageStep) after one eager step; the
    eager step object if capture fails."""
    import torch

    from paper_2510_27002_b200.trainer import GraphedStageStep
    stage.step(0, frames)
    try:
        g = GraphedStageStep(stage)
        g.step(1, frames)
        torch.cuda.synchronize()
        return g
    except Exception:
        torch.cuda.synchronize()
        return stage


def _pretrain_lam_stage(tok, lam, dev) -> dict:
    """SURVEY §8d 'C3 full pretrain_lam stage step' from disk: JASREC records (synthetic frames
    written to a temp dir) -> DeviceBatchLoader (pinned ring, H2D u8) -> frozen tokenizer encode +
    LAM action inference -> dynamics train step, B=36, jasmine-base dims."""
    import tempfile

    import numpy as np

    from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
    from paper_2510_27002_b200.optim import WsdSchedule
    from paper_2510_27002_b200.records import Chunking, DeviceBatchLoader, LoaderState, write_dataset
    from paper_2510_27002_b200.rng import stream
    from paper_2510_27002_b200.trainer import PretrainLamStep

    B = 36

    class _Ep:
        def __init__(self, seed, frames, actions):
            self.seed, self.frames, self.actions = seed, frames, actions

    g = stream(9, "bench-records")
    with tempfile.TemporaryDirectory() as root:
        eps = (_Ep(i, g.integers(0, 256, size=(32, 64, 64, 3), dtype=np.uint8), np.zeros(32, np.uint8))
               for i in range(2 * B))
        index = write_dataset(eps, Chunking(frames_per_record=32, records_per_file=16), root)
        dyn = DynamicsModel(DynamicsConfig(patches_per_frame=PATCHES, max_frames=FRAMES_T), seed=0)
        step = PretrainLamStep(tok, lam, dyn, WsdSchedule(peak_lr=3e-5, total_steps=200_000), seed=0)
        loader = DeviceBatchLoader(index, LoaderState(seed=1), batch_size=B, seq_len=FRAMES_T, depth=2)
        try:
            for k in range(2):
                frames, _, _ = next(loader)
                step.step(k, frames)
            n = 4
            ms = _events_ms(lambda: step.step(2, next(loader)[0]), reps=n)
        finally:
            loader.close()
    return {"metric": "pretrain_lam stage frames/sec", "value": round(B * FRAMES_T / (ms / 1e3), 1), "unit": "frames/s",
            "ms_per_step": round(ms, 2),
            "config": "B=36, T=16 from JASREC on local disk via the device loader; tokenizer encode + LAM infer + "
                      "dynamics step (SURVEY §8d: ~60.5 GFLOP/frame)"}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps = max(1, min(args.steps, 3))
    warm = 1
    from oracle.bench_cpu import time_dynamics_step
    r = time_dynamics_step(batch=1, steps=steps, warmup=warm)
    v = round(r["frames_per_s"], 4)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus, "steps": steps,
            "warmup": warm, "ms_per_step": round(r["seconds_per_step"] * 1e3, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C3 dynamics train step (bounded CPU sample: B=1 of the B=36 workload)",
                       "global_batch": 1, "seq_len": FRAMES_T, "tokens_per_frame": PATCHES},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": r["threads"], "kind": "port",
                             "sample": f"B=1 (16 frames) per step, {steps} steps after {warm} warm-up"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=36, help="per-GPU batch (clips of 16 frames)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the C1/C2/C5 secondary measurements")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2510_27002_b200 import _lib
    from paper_2510_27002_b200 import kernels as K
    from paper_2510_27002_b200.dp import init_from_env
    from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
    from paper_2510_27002_b200.optim import WsdSchedule
    from paper_2510_27002_b200.rng import stream
    from paper_2510_27002_b200.tensor import Tensor
    from paper_2510_27002_b200.trainer import DynamicsTrainStep

    rank, world, local = init_from_env()
    torch.cuda.set_device(local)
    _lib.ensure_device()
    dev = torch.device("cuda", local)
    B = args.batch
    cfg = DynamicsConfig(model_dim=512, heads=8, ffn_dim=2048, blocks=6, token_codes=CODES, action_latent_dim=DLAT,
                         patches_per_frame=PATCHES, max_frames=FRAMES_T)
    model = DynamicsModel(cfg, seed=0)
    sched = WsdSchedule(peak_lr=3e-5, total_steps=200_000, warmup_steps=1000, decay_fraction=0.10)
    trainer = DynamicsTrainStep(model, sched, seed=0, rank=rank, world=world)
    g = stream(1, "bench-tokens", rank)
    tokens_h = torch.from_numpy(g.integers(0, CODES, size=(B, FRAMES_T, PATCHES))).pin_memory()
    lam_cb = stream(2, "bench-lam-codebook").uniform(-1 / 6, 1 / 6, size=(6, DLAT)).astype(np.float32)
    lat_h = torch.from_numpy(lam_cb[stream(2, "bench-actions", rank).integers(0, 6, size=(B, FRAMES_T - 1))]).pin_memory()
    tokens_d = tokens_h.to(dev)
    lat_d = Tensor(lat_h.to(dev))

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    step = 0
    for _ in range(args.warmup):
        trainer.step(step, tokens_d, lat_d)
        step += 1
    trainer.opt.raise_if_nonfinite()
    # single process: the step is replayed as one CUDA graph (trainer.GraphedTrainStep, bit-identical
    # to the eager step); data parallel: eager, with the NCCL buckets launched from backward hooks
    runner = trainer
    step_mode = "eager"
    if world == 1:
        from paper_2510_27002_b200.trainer import GraphedTrainStep
        try:
            g_runner = GraphedTrainStep(trainer)
            g_runner.step(step, tokens_d, lat_d)  # capture + first replay (untimed)
            torch.cuda.synchronize()
            runner, step_mode = g_runner, "cuda_graph"
        except Exception as exc:  # never sink the headline line: time the eager step instead
            step_mode = f"eager (graph capture failed: {type(exc).__name__}: {str(exc)[:120]})"
            torch.cuda.synchronize()
        step += 1
    # kernel-level evidence (GEMM roofline, attention families, launch count): an eager pass with
    # per-launch CUDA events, separate from the timed region
    sync_all()
    K.TIMER = K.KernelTimer()
    K.TIMER.active = True
    n0 = _lib.launch_count()
    prof_steps = min(args.steps, 5)
    for _ in range(prof_steps):
        trainer.step(step, tokens_d, lat_d)
        step += 1
    sync_all()
    K.TIMER.active = False
    launches = (_lib.launch_count() - n0) // prof_steps

    # ---- timed region: device-resident inputs ------------------------------
    sync_all()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        loss = runner.step(step, tokens_d, lat_d)
        step += 1
    e1.record()
    sync_all()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    gemm_ms = K.TIMER.ms()
    gemm_flops = K.TIMER.flops
    gemm_launches = K.TIMER.launches
    families = {name: (K.TIMER.family_ms(name), f["flops"], f["bytes"], len(f["events"]))
                for name, f in K.TIMER.families.items()}
    K.TIMER = None
    trainer.opt.raise_if_nonfinite()
    frames_per_step = B * FRAMES_T * world
    value = frames_per_step / (ms / 1e3)
    loss_val = float(loss.data)

    # ---- e2e: host buffers through the public API --------------------------
    loss_h = torch.empty((), dtype=torch.float32).pin_memory()
    sync_all()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    for _ in range(args.steps):
        tok_step = tokens_h.to(dev, non_blocking=True)
        lat_step = Tensor(lat_h.to(dev, non_blocking=True))
        loss = runner.step(step, tok_step, lat_step)
        loss_h.copy_(loss.data, non_blocking=True)
        step += 1
    e3.record()
    sync_all()
    ms_e2e = max_over_ranks(e2.elapsed_time(e3)) / args.steps
    e2e_value = frames_per_step / (ms_e2e / 1e3)
    h2d = tokens_h.numel() * tokens_h.element_size() + lat_h.numel() * lat_h.element_size()
    # the device-resident loop once more, after the e2e loop: on a power-capped box the clock drifts
    # between back-to-back loops, and |value - value_repeat| is that run-to-run spread (it can exceed
    # the ~1.25 MB / step H2D cost the e2e loop adds)
    sync_all()
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e4.record()
    for _ in range(args.steps):
        runner.step(step, tokens_d, lat_d)
        step += 1
    e5.record()
    sync_all()
    value_repeat = frames_per_step / (max_over_ranks(e4.elapsed_time(e5)) / args.steps / 1e3)

    # ---- secondary BASELINE configs (rank 0, N=1): C5 sampling, C2 LAM step, C1 tokenizer fwd ----
    extra = {}
    peak_gb = torch.cuda.max_memory_allocated(dev) / 2**30
    if rank == 0 and world == 1 and not args.no_extra:
        # independent workloads: release the training state (weights, AdamW moments, activation
        # scratch) so they run on a clean allocator, as they would in their own process
        del trainer, model, loss, tokens_d, lat_d
        import gc
        gc.collect()
        K.release_scratch()
        torch.cuda.empty_cache()
        try:
            extra = secondary_configs(dev)
        except Exception as exc:  # never sink the headline line
            extra = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
        if not args.no_cpu_baseline:
            try:
                for k, v in cpu_baseline_secondary().items():
                    if isinstance(extra.get(k), dict):
                        extra[k]["cpu_baseline"] = v
            except Exception as exc:
                extra["cpu_baseline_error"] = f"{type(exc).__name__}: {str(exc)[:200]}"

    peaks = _peaks()
    achieved = gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else 0.0
    traffic, traffic_note = None, None
    tf = ROOT / "profiles" / "roofline_traffic.json"
    if tf.exists():
        try:
            tj = json.loads(tf.read_text())
            traffic = tj.get("gemm_dram_bytes_per_launch")
            traffic_note = {"kernel": tj.get("kernel"), "algorithmic_bytes": tj.get("algorithmic_bytes"),
                            "source": tj.get("source")}
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "kernel": "jz::gemm_bf16_kernel (all K1 GEMM launches of the step)",
                "achieved": round(achieved, 1), "peak": peaks["bf16_sustained"], "unit": "TFLOP/s",
                "frac": round(achieved / peaks["bf16_sustained"], 4), "traffic": traffic,
                "peak_source": f"{peaks['source']} bf16_tflops_sustained",
                "gemm_share_of_step": round(gemm_ms / prof_steps / ms, 4), "gemm_launches_per_step": gemm_launches // prof_steps,
                "algorithmic_flops_per_step": gemm_flops // prof_steps, "traffic_launch": traffic_note,
                "measured_over": f"{prof_steps} eager steps with per-launch CUDA events (the timed steps are graph replays)"}
    # attention kernels (north_star: tensor-pipe utilisation against the bf16 peak): event-timed like
    # the GEMMs, algorithmic FLOPs and bytes per launch from kernels.py; the binding bound is the
    # roof the kernel's arithmetic intensity puts under it
    attention = {}
    for name, (fms, ffl, fby, fn) in sorted(families.items()):
        if fms <= 0:
            continue
        tfl = ffl / (fms / 1e3) / 1e12
        gbs = fby / (fms / 1e3) / 1e9
        t_tensor = ffl / (peaks["bf16_sustained"] * 1e12)
        t_hbm = fby / (peaks["hbm_gbs"] * 1e9)
        attention[name] = {"us_per_launch": round(fms * 1e3 / fn, 1), "launches_per_step": fn // prof_steps,
                           "tflops": round(tfl, 1), "frac_bf16_peak": round(tfl / peaks["bf16_sustained"], 4),
                           "gbs": round(gbs, 1), "frac_hbm_peak": round(gbs / peaks["hbm_gbs"], 4),
                           "bound": "hbm" if t_hbm > t_tensor else "tensor",
                           "frac_of_bound": round(max(t_tensor, t_hbm) / (fms / 1e3), 4)}
    step_flops = 42.13e9 * frames_per_step / world  # SURVEY §8d algorithmic FLOPs per GPU-step
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline()
            except Exception as exc:  # the baseline must never sink the bench line
                cpu = {"value": None, "error": str(exc)[:200]}
        line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": "C3/C4 MaskGIT dynamics train step, prepended latent actions, "
                                       "jasmine-base dims, T=16, 64x64x3 patch 4 (16x256 tokens), 1024 codes",
                           "global_batch": B * world, "per_gpu_batch": B, "seq_len": FRAMES_T,
                           "tokens_per_frame": PATCHES, "parallelism": f"dp{world}",
                           "l2": "working set ~20 GB per step >> 126 MB L2 (no flush needed)"},
                "e2e": {"value": round(e2e_value, 1), "unit": UNIT, "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": 4},
                "value_repeat": round(value_repeat, 1),
                "run_to_run_spread_pct": round(100 * abs(value - value_repeat) / value, 2),
                "gpu_launches": int(launches),
                "roofline": roofline,
                "model_tflops": round(step_flops / (ms / 1e3) / 1e12, 1),
                "model_flops_frac": round(step_flops / (ms / 1e3) / 1e12 / peaks["bf16_sustained"], 4),
                "cpu_baseline": cpu, "clocks": clk, "loss": round(loss_val, 5),
            "hbm_peak_gb": round(peak_gb, 1), "step_mode": step_mode, "attention": attention, **extra}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
