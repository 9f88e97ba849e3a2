"""The data-parallel dynamics step run for real: two processes (one rank each) on the box's GPU.

NCCL refuses two ranks on one device, so the ranks talk over gloo (dp.init_from_env's shared-GPU
mode: gloo all-reduces the CUDA gradient buckets through host memory).  Everything else is the
production DP path: per-rank Philox mask shards by skip-ahead, the global mask count, bucket
all-reduces launched from the backward hooks on the side stream, AdamW after the last bucket.

Checked against a single-process run of the global batch (SURVEY §8e parity):
  - step-0 summed gradients equal the single-process gradients (fp32 summation order only);
  - the parameter updates after 3 AdamW steps point the same way as the single-process ones,
    and the two replicas stay bitwise identical.
"""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
TOL = json.loads((ROOT / "fidelity_threshold.json").read_text())["parity"]

KW = dict(model_dim=128, heads=2, ffn_dim=512, blocks=2, token_codes=256, action_latent_dim=32,
          patches_per_frame=256, max_frames=4)
GB, T, N, STEPS = 4, 4, 256, 3


def _inputs():
    from oracle import rng as OR
    tokens = OR.stream(1, "dp-mp-tokens").integers(0, 256, size=(GB, T, N))
    lat = (OR.stream(2, "dp-mp-lat").normal(size=(GB, T - 1, 32)) * 0.1).astype(np.float32)
    return tokens, lat


def _run(rank: int, world: int, out_dir: str) -> None:
    """One rank: STEPS DynamicsTrainStep steps on its shard; saves step-0 grads and final params."""
    sys.path.insert(0, str(ROOT))
    from paper_2510_27002_b200.dp import init_from_env, shard
    from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
    from paper_2510_27002_b200.optim import WsdSchedule
    from paper_2510_27002_b200.tensor import Tensor
    from paper_2510_27002_b200.trainer import DynamicsTrainStep
    if world > 1:
        r, w, dev = init_from_env()
        assert (r, w) == (rank, world)
    else:
        dev = 0
        torch.cuda.set_device(0)
    model = DynamicsModel(DynamicsConfig(**KW), seed=0)
    tr = DynamicsTrainStep(model, WsdSchedule(peak_lr=1e-3, total_steps=100, warmup_steps=0), seed=0,
                           rank=rank, world=world)
    tokens, lat = _inputs()
    b0, bl = shard(GB, rank, world)
    tok_d = torch.as_tensor(tokens[b0:b0 + bl]).cuda()
    lat_d = Tensor(torch.as_tensor(lat[b0:b0 + bl]).cuda())
    losses = []
    for step in range(STEPS):
        loss = tr.step(step, tok_d, lat_d, global_batch=GB)
        losses.append(float(loss.data))
        if step == 0:
            g0 = {k: p.grad.detach().cpu().numpy().copy() for k, p in model.params.items()}
    tr.opt.raise_if_nonfinite()
    np.savez(os.path.join(out_dir, f"rank{rank}_of{world}.npz"), losses=np.array(losses),
             **{f"g0.{k}": v for k, v in g0.items()},
             **{f"p.{k}": p.data.cpu().numpy() for k, p in model.params.items()})
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def _init_params() -> dict:
    from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
    m = DynamicsModel(DynamicsConfig(**KW), seed=0)
    return {f"p.{k}": p.data.cpu().numpy() for k, p in m.params.items()}


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_process_dp_step_equals_single_process(tmp_path):
    port = _free_port()
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r); "
            "from test_gpu_dp_multiprocess import _run; _run(int(sys.argv[1]), 2, sys.argv[2])"
            % (str(ROOT), str(ROOT / "tests")))
    procs = []
    for rank in range(2):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2",
                   LOCAL_RANK=str(rank), JZ_DP_SHARED_GPU="1")
        procs.append(subprocess.Popen([sys.executable, "-c", code, str(rank), str(tmp_path)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=600)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-3000:]
    _run(0, 1, str(tmp_path))
    single = np.load(tmp_path / "rank0_of1.npz")
    r0, r1 = np.load(tmp_path / "rank0_of2.npz"), np.load(tmp_path / "rank1_of2.npz")
    # each rank's loss is its share of the global-count-normalised loss: the shares add up
    np.testing.assert_allclose(r0["losses"][0] + r1["losses"][0], single["losses"][0], rtol=1e-5)
    worst_g, worst_p = 0.0, 1.0
    init = _init_params()
    for key in single.files:
        if key.startswith("g0.") and not key.endswith(".k.b"):
            ref = single[key]
            for r in (r0, r1):  # after the all-reduce both ranks hold the global-batch gradient
                d = np.linalg.norm(r[key] - ref) / max(np.linalg.norm(ref), 1e-30)
                worst_g = max(worst_g, d)
        if key.startswith("p."):
            np.testing.assert_array_equal(r0[key], r1[key], err_msg=key)  # replicas stay identical
            if not key.endswith(".k.b"):
                # Adam's first steps are ~lr * sign(g): compare the update directions (cosine of the
                # parameter deltas), since entries whose gradient is at rounding-noise level flip sign
                d_dp = (r0[key] - init[key]).astype(np.float64).ravel()
                d_1 = (single[key] - init[key]).astype(np.float64).ravel()
                c = float(d_dp @ d_1 / max(np.linalg.norm(d_dp) * np.linalg.norm(d_1), 1e-30))
                worst_p = min(worst_p, c)
    assert worst_g < TOL["dp_grad_rel_l2"], worst_g
    assert worst_p >= TOL["dp_update_cosine_min"], worst_p
