"""Device training step for the dynamics stage (mirror of trainer.run_stage's step body).

run_stage (trainer.py:165-191) per step:
    rng = stream(seed, stage, "step", step)
    loss = loss_fn(frames, actions, rng); backward
    adamw_step(params, grads, adam, wsd_lr(schedule, step + 1)); grads reset

DynamicsTrainStep does the same for the dynamics model on device-resident tokens
and action latents (the frozen tokenizer/LAM labels), optionally data-parallel:
rank r draws its shard of the global Philox mask, normalises by the global mask
count and all-reduces gradient buckets (dp.py) overlapped with the backward.
"""
from __future__ import annotations

import torch

from . import kernels as K
from .dp import GradAllReduce, block_buckets, shard
from .dynamics import DynamicsModel
from .optim import WsdSchedule, adamw_init, adamw_step, wsd_lr
from .rng import consume, stream
from .tensor import Tensor


class DynamicsTrainStep:
    def __init__(self, model: DynamicsModel, schedule: WsdSchedule, *, seed: int = 0, stage: str = "dynamics",
                 rank: int = 0, world: int = 1, group=None):
        self.model = model
        self.schedule = schedule
        self.seed = seed
        self.stage = stage
        self.rank, self.world = rank, world
        self.opt = adamw_init(model.params)
        self.reducer = None
        if world > 1:
            store = model._store
            store.grads()  # allocate the flat gradient buffer
            buckets = block_buckets(store.extents, "dyn", model.cfg.blocks, store.flat.numel())
            self.reducer = GradAllReduce(store.grad_flat, buckets, group=group)

    def step(self, step: int, tokens: torch.Tensor, latents: Tensor, global_batch: int | None = None):
        """One training step on this rank's slice; returns the (rank-local share of the) loss tensor."""
        m = self.model
        cfg = m.cfg
        B, T, N = tokens.shape
        gb = global_batch if global_batch is not None else B * self.world
        rng = stream(self.seed, self.stage, "step", step)
        st = consume(rng, gb + gb * T * N)
        dev = tokens.device
        b0, bl = shard(gb, self.rank, self.world)
        mask = torch.empty(bl, T, N, dtype=torch.uint8, device=dev)
        count_local = torch.zeros((), dtype=torch.int32, device=dev)
        K.philox_mask(st, gb, b0, bl, T, N, cfg.mask_limit, mask, count_local)
        count = count_local
        if self.world > 1:
            full = K.scratch("dp_full_mask", gb * T * N, dtype=torch.uint8).view(gb, T, N)
            count = torch.zeros((), dtype=torch.int32, device=dev)
            K.philox_mask(st, gb, 0, gb, T, N, cfg.mask_limit, full, count)
        hook = self.reducer.ready if self.reducer is not None else None
        loss, _ = m.loss(tokens, latents, None, mask=mask, _count=count, _on_grads_done=hook)
        loss.backward()
        if self.reducer is not None:
            self.reducer.finish()
        adamw_step(m.params, {n: p.grad for n, p in m.params.items()}, self.opt, wsd_lr(self.schedule, step + 1),
                   check="deferred")
        return loss

    # -- checkpoint / resume (trainer.py:91-115, 442-473) ------------------------------
    def pack(self, step: int, config: dict | None = None, loader_state=None):
        """JASCKPT1 bundle of this stage (params + AdamW moments + loader state), deskworld layout."""
        from .checkpoint import pack_stage
        from .records import LoaderState
        ls = loader_state if loader_state is not None else LoaderState(seed=self.seed)
        return pack_stage(self.stage, config or {}, self.model.params, self.opt, ls, step, self.seed)

    def restore(self, bundle) -> tuple:
        """Load a bundle into the live device tensors; returns (loader_state dict, step)."""
        from .checkpoint import restore_stage
        _, ls, step = restore_stage(bundle, self.model.params, self.opt)
        return ls, step


class PretrainLamStep:
    """The pretrain_lam dynamics-stage step from raw frames (trainer.py:297-305): frozen tokenizer
    tokens + frozen LAM action latents (codebook rows of the inferred actions) -> dynamics step.

    frames: device uint8 (B, T, H, W, C), e.g. straight from records.DeviceBatchLoader."""

    def __init__(self, tokenizer, lam, dynamics: DynamicsModel, schedule: WsdSchedule, **kw):
        self.tokenizer, self.lam = tokenizer, lam
        self.inner = DynamicsTrainStep(dynamics, schedule, **kw)

    def step(self, step: int, frames: torch.Tensor):
        tokens = self.tokenizer.encode_device(frames)
        idx = self.lam.infer_actions_device(frames)
        latents = Tensor(self.lam.params["codebook"].data[idx])
        return self.inner.step(step, tokens, latents)


class StageTrainStep:
    """run_stage's per-step body (trainer.py:165-182) for any model stage on device:
    rng = stream(seed, stage, "step", step); loss = loss_fn(frames, actions, rng); backward;
    AdamW at wsd_lr(schedule, step + 1); gradients start from zero every step (the reference
    resets p.grad to None, trainer.py:181-183).  The finiteness check is deferred to the
    optimizer's device flag (`opt.raise_if_nonfinite()`), not a per-step host sync."""

    def __init__(self, params: dict, loss_fn, schedule: WsdSchedule, *, seed: int = 0, stage: str = "stage"):
        from .tensor import store_for
        self.params = params
        self.loss_fn = loss_fn
        self.schedule = schedule
        self.seed = seed
        self.stage = stage
        self.opt = adamw_init(params)
        self._store = store_for(params)

    def _zero_grads(self) -> None:
        st = self._store
        if st is not None and st.grad_flat is not None:
            st.grad_flat.zero_()
            return
        for p in self.params.values():
            if p.grad is not None:
                p.grad.zero_()

    def step(self, step: int, frames, actions=None):
        self._zero_grads()
        rng = stream(self.seed, self.stage, "step", step)
        loss = self.loss_fn(frames, actions, rng)
        loss.backward()
        adamw_step(self.params, {n: p.grad for n, p in self.params.items()}, self.opt,
                   wsd_lr(self.schedule, step + 1), check="deferred")
        return loss


def tokenizer_stage(tokenizer, schedule: WsdSchedule, *, seed: int = 0) -> StageTrainStep:
    """train_tokenizer's loss_fn (trainer.py:220-223): the tokenizer forward's total loss
    (reconstruction MSE + codebook + 0.25 commitment) on uint8 frames."""
    return StageTrainStep(tokenizer.params, lambda frames, actions, rng: tokenizer.forward(frames)[2]["total"],
                          schedule, seed=seed, stage="tokenizer")


def lam_stage(lam, schedule: WsdSchedule, *, seed: int = 0) -> StageTrainStep:
    """train_lam's loss_fn (trainer.py:254-257): the LAM forward's total loss."""
    return StageTrainStep(lam.params, lambda frames, actions, rng: lam.forward(frames)[2]["total"],
                          schedule, seed=seed, stage="lam")
