"""AdamW + warmup-stable-decay schedule (mirror of deskworld/optim.py).

adamw_step runs K13 (jz_adamw_step): f32 arithmetic in the reference's exact
operation order with numpy/NEP-50 scalar casting and no FMA contraction, so a
step is bit-identical to the reference on identical inputs.  When the model's
parameters live in one flat buffer the whole update is a single launch.

Non-finite gradients: the reference raises NonFiniteGradient mid-loop after
having updated the params that sort before the offending one (optim.py:43-49).
Here a device flag is computed over ALL gradients first and the update kernel
leaves EVERY parameter untouched when it is set; `adamw_step(..., check="sync")`
(default) then raises NonFiniteGradient like the reference, `check="deferred"`
keeps the host asynchronous and `state.raise_if_nonfinite()` raises later.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels as K
from .tensor import store_for
from ._lib import NonFiniteGradient  # noqa: F401  (re-export, optim.py:10-11)


@dataclass
class AdamWState:
    m: dict = field(default_factory=dict)
    v: dict = field(default_factory=dict)
    t: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    flag: torch.Tensor | None = None
    m_flat: torch.Tensor | None = None
    v_flat: torch.Tensor | None = None
    store: object = None
    first_bad: torch.Tensor | None = None  # optimizer step (t) at which the flag first tripped, 0 = never

    def raise_if_nonfinite(self) -> None:
        """Raise NonFiniteGradient if any deferred check tripped (the reference raises at the first
        non-finite gradient, optim.py:48-49; every later update was skipped, trainer.py:170-180)."""
        if self.flag is not None and int(self.flag) != 0:
            at = int(self.first_bad) if self.first_bad is not None else 0
            self.flag.zero_()
            if self.first_bad is not None:
                self.first_bad.zero_()
            where = f" at optimizer step {at}" if at else ""
            raise NonFiniteGradient(f"non-finite gradient{where} (that update and every later one skipped)")


def adamw_init(params: dict, weight_decay: float = 0.0, beta1: float = 0.9, beta2: float = 0.999,
               eps: float = 1e-8, store=None) -> AdamWState:
    """optim.py:25-31 (moments zero-initialised in HBM)."""
    st = AdamWState(beta1=beta1, beta2=beta2, eps=eps, weight_decay=weight_decay)
    dev = next(iter(params.values())).data.device
    st.flag = torch.zeros((), dtype=torch.int32, device=dev)
    st.first_bad = torch.zeros((), dtype=torch.int32, device=dev)
    if store is None:
        store = store_for(params)
    if store is not None and store.owns(params):
        st.store = store
        st.m_flat = torch.zeros_like(store.flat)
        st.v_flat = torch.zeros_like(store.flat)
        for name in store.layout:
            st.m[name] = store.view_of(st.m_flat, name)
            st.v[name] = store.view_of(st.v_flat, name)
    else:
        for name, p in params.items():
            # contiguous moments even when p is a strided member of a fused block
            st.m[name] = torch.zeros(p.data.shape, dtype=p.data.dtype, device=p.data.device)
            st.v[name] = torch.zeros(p.data.shape, dtype=p.data.dtype, device=p.data.device)
    return st


def _scalars(state: AdamWState, lr: float):
    t = state.t
    b1, b2 = state.beta1, state.beta2
    f = np.float32
    return dict(lr=float(f(lr)), b1=float(f(b1)), b2=float(f(b2)), omb1=float(f(1.0 - b1)), omb2=float(f(1.0 - b2)),
                bc1=float(f(1.0 - b1 ** t)), bc2=float(f(1.0 - b2 ** t)), eps=float(f(state.eps)),
                lrwd=float(f(lr * state.weight_decay)) if state.weight_decay else 0.0)


def adamw_step(params: dict, grads: dict, state: AdamWState, lr: float, check: str = "sync") -> None:
    """optim.py:34-62.  `grads` maps names to device tensors (p.grad) or None."""
    state.t += 1
    sc = _scalars(state, lr)
    flat_ok = (state.store is not None and state.store.owns(params) and state.store.grads_are_views(grads))
    if flat_ok:
        g = state.store.grad_flat
        K.finite_check(g, state.flag)
        K.adamw(state.store.flat, g, state.m_flat, state.v_flat, flag=state.flag, **sc)
    else:
        names = [n for n in sorted(params) if grads.get(n) is not None]
        for n in names:
            g = grads[n]
            if tuple(g.shape) != tuple(params[n].data.shape):
                raise ValueError(f"gradient shape {tuple(g.shape)} != param shape {tuple(params[n].data.shape)} for {n!r}")
            K.finite_check(g.contiguous(), state.flag)
        for n in names:
            p = params[n].data
            if p.is_contiguous():
                K.adamw(p, grads[n].contiguous(), state.m[n], state.v[n], flag=state.flag, **sc)
            else:  # strided member of a fused q/k/v block: update a dense copy, write it back
                pc = p.contiguous()
                K.adamw(pc, grads[n].contiguous(), state.m[n], state.v[n], flag=state.flag, **sc)
                p.copy_(pc)
    if state.first_bad is not None and not torch.cuda.is_current_stream_capturing():
        # remember the first step whose gradients tripped the flag (device-side, no host sync)
        torch.where((state.flag != 0) & (state.first_bad == 0), torch.full_like(state.first_bad, state.t),
                    state.first_bad, out=state.first_bad)
    if check == "sync":
        state.raise_if_nonfinite()


@dataclass(frozen=True)
class WsdSchedule:
    """optim.py:65-73."""
    peak_lr: float
    total_steps: int
    warmup_steps: int = 1000
    decay_fraction: float = 0.10

    def __post_init__(self):
        if self.warmup_steps < 0 or self.total_steps <= 0:
            raise ValueError("invalid schedule bounds")


def wsd_lr(schedule: WsdSchedule, step: int) -> float:
    """optim.py:76-89 (host scalar)."""
    decay_steps = int(round(schedule.decay_fraction * schedule.total_steps))
    decay_start = schedule.total_steps - decay_steps
    if step <= 0 or step >= schedule.total_steps:
        return 0.0
    if step < schedule.warmup_steps:
        return schedule.peak_lr * step / schedule.warmup_steps
    if step <= decay_start or decay_steps == 0:
        return schedule.peak_lr
    return schedule.peak_lr * (schedule.total_steps - step) / decay_steps
