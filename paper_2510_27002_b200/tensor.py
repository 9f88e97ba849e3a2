"""Device-resident mirror of deskworld.autodiff's public surface.

deskworld.autodiff.Tensor (autodiff.py:35-103) is a numpy array plus a closure
graph.  Here `.data` is a torch tensor in HBM and `.backward()` runs the
explicit backward kernels of whatever op produced the value (there is no
generic tape: the hot path's backward is hand-scheduled, see st.py /
dynamics.py).  Parameters of one model live in one flat fp32 buffer (and their
gradients in another) so the fused AdamW kernel updates everything with a
single launch.
"""
from __future__ import annotations

import weakref
from collections import OrderedDict

import numpy as np
import torch

from . import _lib


def device() -> torch.device:
    _lib.ensure_device()
    return torch.device("cuda", torch.cuda.current_device())


class Tensor:
    __slots__ = ("data", "grad", "requires_grad", "_backward", "__weakref__")

    def __init__(self, data, requires_grad: bool = False, _backward=None):
        if not isinstance(data, torch.Tensor):
            arr = np.asarray(data)
            if arr.dtype == np.float64:
                arr = arr.astype(np.float32)
            data = torch.as_tensor(arr).to(device())
        self.data = data
        self.grad = None
        self.requires_grad = requires_grad
        self._backward = _backward

    # -- array-like ---------------------------------------------------------
    @property
    def shape(self):
        return tuple(self.data.shape)

    @property
    def ndim(self):
        return self.data.dim()

    @property
    def dtype(self):
        return self.data.dtype

    def numpy(self) -> np.ndarray:
        return self.data.detach().cpu().numpy()

    def __float__(self):
        return float(self.data)

    def __repr__(self):
        return f"Tensor(shape={self.shape}, dtype={self.dtype}, device={self.data.device})"

    def detach(self) -> "Tensor":
        return Tensor(self.data)

    def backward(self) -> None:
        """Run the hand-scheduled backward of the op that produced this scalar."""
        if self._backward is None:
            raise RuntimeError("backward() on a tensor that does not require grad")
        fn, self._backward = self._backward, None
        fn()


def parameter(data) -> Tensor:
    return Tensor(data, requires_grad=True)


def tensor(data, dtype=np.float32, requires_grad=False) -> Tensor:
    return Tensor(np.asarray(data, dtype=dtype), requires_grad=requires_grad)


class ParamStore:
    """Flat fp32 storage for a model's parameters (+ lazily a flat gradient buffer).

    `params` is an OrderedDict name -> Tensor whose `.data` are views into `flat`.
    """

    def __init__(self, arrays: "OrderedDict[str, np.ndarray]"):
        dev = device()
        total = sum(int(a.size) for a in arrays.values())
        host = np.empty(total, dtype=np.float32)
        self.offsets: dict[str, tuple[int, tuple]] = {}
        off = 0
        for name, a in arrays.items():
            n = int(a.size)
            host[off:off + n] = a.reshape(-1).astype(np.float32)
            self.offsets[name] = (off, tuple(a.shape))
            off += n
        self.flat = torch.from_numpy(host).to(dev)
        self.grad_flat: torch.Tensor | None = None
        self.params: "OrderedDict[str, Tensor]" = OrderedDict()
        for name, (o, shp) in self.offsets.items():
            n = int(np.prod(shp)) if shp else 1
            self.params[name] = Tensor(self.flat[o:o + n].view(shp), requires_grad=True)
        _STORES[id(self.params)] = self

    def grads_are_views(self, grads: dict) -> bool:
        if self.grad_flat is None:
            return False
        base = self.grad_flat.data_ptr()
        for name, (o, _) in self.offsets.items():
            g = grads.get(name)
            if g is None or g.data_ptr() != base + 4 * o:
                return False
        return True

    def grads(self) -> dict:
        """Gradient views (allocated on first use) keyed by name; also sets p.grad."""
        if self.grad_flat is None:
            self.grad_flat = torch.zeros_like(self.flat)
        out = {}
        for name, (o, shp) in self.offsets.items():
            n = int(np.prod(shp)) if shp else 1
            out[name] = self.grad_flat[o:o + n].view(shp)
        return out

    def owns(self, params: dict) -> bool:
        """True when `params` are still exactly this store's views (not swapped by a caller)."""
        if params.keys() != self.params.keys():
            return False
        return all(params[k] is self.params[k] for k in params)


_STORES: "weakref.WeakValueDictionary[int, ParamStore]" = weakref.WeakValueDictionary()


def store_for(params: dict):
    """The ParamStore whose `params` dict is exactly `params` (None if swapped / merged)."""
    st = _STORES.get(id(params))
    return st if st is not None and st.owns(params) else None


def grad_buffers(params: dict, store: ParamStore | None) -> dict:
    """Gradient destination per parameter name: store views when possible, else fresh buffers."""
    if store is not None and store.owns(params):
        g = store.grads()
        for k, p in params.items():
            p.grad = g[k]
        return g
    out = {}
    for k, p in params.items():
        if p.grad is None or p.grad.shape != p.data.shape:
            p.grad = torch.zeros_like(p.data)
        out[k] = p.grad
    return out


def as_device(x, dtype=None) -> torch.Tensor:
    """numpy / Tensor / torch -> contiguous device torch tensor."""
    if isinstance(x, Tensor):
        t = x.data
    elif isinstance(x, torch.Tensor):
        t = x
    else:
        arr = np.asarray(x)
        t = torch.from_numpy(np.ascontiguousarray(arr))
    t = t.to(device(), non_blocking=True)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def param_count(params: dict) -> int:
    """deskworld/st.py:97-98."""
    return sum(int(np.prod(p.shape)) if p.shape else 1 for p in params.values())
