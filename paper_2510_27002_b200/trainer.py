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
        B, T, N = tokens.shape
        gb = global_batch if global_batch is not None else B * self.world
        rng = stream(self.seed, self.stage, "step", step)
        st = consume(rng, gb + gb * T * N)
        return self._device_step(tokens, latents, st, wsd_lr(self.schedule, step + 1), gb)

    def _device_step(self, tokens: torch.Tensor, latents: Tensor, st, lr: float, gb: int):
        """The step's device work for mask stream state `st` and learning rate `lr` (both ignored,
        read from device memory instead, while a GraphedTrainStep captures it)."""
        m = self.model
        cfg = m.cfg
        B, T, N = tokens.shape
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
        adamw_step(m.params, {n: p.grad for n, p in m.params.items()}, self.opt, lr, check="deferred")
        return loss

    # -- checkpoint / resume (trainer.py:91-115, 442-473) ------------------------------
    def pack(self, step: int, config: dict | None = None, loader_state=None):
        """JASCKPT1 bundle of this stage (params + AdamW moments + loader state), deskworld layout."""
        from .checkpoint import pack_stage
        from .records import LoaderState
        self.opt.raise_if_nonfinite()  # never checkpoint past a skipped (non-finite) update
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
        rng = stream(self.seed, self.stage, "step", step)
        return self._device_step(frames, actions, rng, wsd_lr(self.schedule, step + 1))

    def _device_step(self, frames, actions, rng, lr: float):
        """The step's device work (lr is read from device memory while a GraphedStageStep captures it)."""
        self._zero_grads()
        loss = self.loss_fn(frames, actions, rng)
        loss.backward()
        adamw_step(self.params, {n: p.grad for n, p in self.params.items()}, self.opt, lr, check="deferred")
        return loss


def tokenizer_stage(tokenizer, schedule: WsdSchedule, *, seed: int = 0) -> StageTrainStep:
    """train_tokenizer's loss_fn (trainer.py:220-223): the tokenizer forward's total loss
    (reconstruction MSE + codebook + 0.25 commitment) on uint8 frames."""
    return StageTrainStep(tokenizer.params, lambda frames, actions, rng: tokenizer.forward(frames, _indices_on_device=True)[2]["total"],
                          schedule, seed=seed, stage="tokenizer")


def lam_stage(lam, schedule: WsdSchedule, *, seed: int = 0) -> StageTrainStep:
    """train_lam's loss_fn (trainer.py:254-257): the LAM forward's total loss."""
    return StageTrainStep(lam.params, lambda frames, actions, rng: lam.forward(frames, _indices_on_device=True)[2]["total"],
                          schedule, seed=seed, stage="lam")


class GraphedTrainStep:
    """A single-process DynamicsTrainStep replayed as ONE CUDA graph per step.

    Everything that changes from step to step is refreshed in device memory before the replay by
    two small pinned H2D copies:
    - the step's Philox mask-stream state;
    - the AdamW scalars (learning rate, bias corrections; `opt.t` advances on the host as in
      adamw_step).

    The step's tokens and latents are copied into the graph's static inputs. Kernels, launch order
    and arithmetic are the eager step's, so replays are bit-identical to `trainer.step`
    (tests/test_gpu_fullsize.py). The data-parallel step stays eager: its NCCL buckets are
    launched from backward hooks on a side stream.
    """

    RING = 4  # pinned staging slots in flight (a slot is reused only after its copy has run)

    def __init__(self, trainer: DynamicsTrainStep):
        if trainer.world != 1:
            raise ValueError("graph replay is single-process; the data-parallel step runs eagerly")
        self.tr = trainer
        self.graph = None
        self.loss = None
        dev = trainer.model.params["token_embed"].data.device
        self.state_d = torch.zeros(11, dtype=torch.int64, device=dev)
        self.sc_d = torch.zeros(9, dtype=torch.float32, device=dev)
        self._state_h = [torch.zeros(11, dtype=torch.int64).pin_memory() for _ in range(self.RING)]
        self._sc_h = [torch.zeros(9, dtype=torch.float32).pin_memory() for _ in range(self.RING)]
        self._ev = [None] * self.RING
        self._k = 0

    def _capture(self, tokens: torch.Tensor, latents: Tensor) -> None:
        from .sampling import _no_gc
        tr = self.tr
        self.tok_buf = tokens.clone()
        self.lat_buf = latents.data.clone()
        t_saved = tr.opt.t
        K.DEVSTATE = (self.state_d, self.sc_d)
        try:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            B, T, N = tokens.shape
            with _no_gc(), torch.cuda.graph(g):
                self.loss = tr._device_step(self.tok_buf, Tensor(self.lat_buf), None, 0.0, B)
        finally:
            K.DEVSTATE = None
            tr.opt.t = t_saved  # the capture ran adamw_step's host bookkeeping once without a real step
        self.graph = g

    def step(self, step: int, tokens: torch.Tensor, latents: Tensor):
        import numpy as np
        from .optim import _scalars
        tr = self.tr
        B, T, N = tokens.shape
        st = consume(stream(tr.seed, tr.stage, "step", step), B + B * T * N)
        tr.opt.t += 1
        sc = _scalars(tr.opt, wsd_lr(tr.schedule, step + 1))
        slot = self._k % self.RING
        self._k += 1
        if self._ev[slot] is not None:
            self._ev[slot].synchronize()
        sh, hh = self._state_h[slot], self._sc_h[slot]
        vals = list(st.counter) + list(st.key) + list(st.buffer) + [st.buffer_pos]
        sh.numpy()[:] = np.array([v & ((1 << 64) - 1) for v in vals], dtype=np.uint64).view(np.int64)
        hh.numpy()[:] = [sc["lr"], sc["b1"], sc["b2"], sc["omb1"], sc["omb2"], sc["bc1"], sc["bc2"], sc["eps"],
                         sc["lrwd"]]
        self.state_d.copy_(sh, non_blocking=True)
        self.sc_d.copy_(hh, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._ev[slot] = ev
        if self.graph is None:
            self._capture(tokens, latents)
        if tokens.data_ptr() != self.tok_buf.data_ptr():
            self.tok_buf.copy_(tokens, non_blocking=True)
        lat = latents.data
        if lat.data_ptr() != self.lat_buf.data_ptr():
            self.lat_buf.copy_(lat, non_blocking=True)
        self.graph.replay()
        return self.loss


class GraphedStageStep:
    """A StageTrainStep (tokenizer / LAM) replayed as one CUDA graph per step. The per-step inputs
    are the frames, copied into the graph's static buffer, and the AdamW scalars, refreshed in device
    memory. The stage loss functions do not draw from the step generator (trainer.py:220-223,
    254-257), so nothing else changes. Replays are bit-identical to `stage.step`
    (tests/test_gpu_stages.py)."""

    RING = 4

    def __init__(self, stage: StageTrainStep):
        self.tr = stage
        self.graph = None
        self.loss = None
        dev = next(iter(stage.params.values())).data.device
        self.sc_d = torch.zeros(9, dtype=torch.float32, device=dev)
        self._unused_state = torch.zeros(11, dtype=torch.int64, device=dev)
        self._sc_h = [torch.zeros(9, dtype=torch.float32).pin_memory() for _ in range(self.RING)]
        self._ev = [None] * self.RING
        self._k = 0

    def step(self, step: int, frames, actions=None):
        from .optim import _scalars
        from .sampling import _no_gc
        tr = self.tr
        tr.opt.t += 1
        sc = _scalars(tr.opt, wsd_lr(tr.schedule, step + 1))
        slot = self._k % self.RING
        self._k += 1
        if self._ev[slot] is not None:
            self._ev[slot].synchronize()
        hh = self._sc_h[slot]
        hh.numpy()[:] = [sc["lr"], sc["b1"], sc["b2"], sc["omb1"], sc["omb2"], sc["bc1"], sc["bc2"], sc["eps"],
                         sc["lrwd"]]
        self.sc_d.copy_(hh, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._ev[slot] = ev
        if self.graph is None:
            self.frames_buf = frames.clone()
            t_saved = tr.opt.t
            K.DEVSTATE = (self._unused_state, self.sc_d)
            try:
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with _no_gc(), torch.cuda.graph(g):
                    self.loss = tr._device_step(self.frames_buf, None, None, 0.0)
            finally:
                K.DEVSTATE = None
                tr.opt.t = t_saved
            self.graph = g
        if frames.data_ptr() != self.frames_buf.data_ptr():
            self.frames_buf.copy_(frames, non_blocking=True)
        self.graph.replay()
        return self.loss
