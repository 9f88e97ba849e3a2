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
    """A device array with the reference's Tensor surface (autodiff.py:22-103), narrowed to what
    the hot path needs: a loss carries its hand-scheduled backward, and scalar losses combine
    linearly (`ce + cb + beta * commit`, trainer.py:306-309) with the coefficients routed to
    each leaf's backward."""
    __slots__ = ("data", "grad", "requires_grad", "_backward", "_terms", "_coef_hook", "__weakref__")

    def __init__(self, data, requires_grad: bool = False, _backward=None, _terms=None, _coef_hook=None):
        if not isinstance(data, torch.Tensor):
            arr = np.asarray(data)
            if arr.dtype == np.float64:
                arr = arr.astype(np.float32)
            data = torch.as_tensor(arr).to(device())
        self.data = data
        self.grad = None
        self.requires_grad = requires_grad
        self._backward = _backward
        self._terms = _terms          # linear combination of leaf losses: [(leaf, coef)]
        self._coef_hook = _coef_hook  # leaf whose backward needs its total coefficient up front

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

    # -- linear combinations of scalar losses ----------------------------------
    def _leaf_terms(self, c: float):
        if self._terms is None:
            return [(self, c)]
        return [(t, cc * c) for t, cc in self._terms]

    def _combine(self, other, ca: float, cb: float) -> "Tensor":
        if isinstance(other, Tensor):
            return Tensor(self.data * ca + other.data * cb, _terms=self._leaf_terms(ca) + other._leaf_terms(cb))
        if isinstance(other, (int, float, np.floating, np.integer)):
            return Tensor(self.data * ca + float(other) * cb, _terms=self._leaf_terms(ca))
        return NotImplemented

    def __add__(self, other):
        return self._combine(other, 1.0, 1.0)

    def __radd__(self, other):
        return self._combine(other, 1.0, 1.0)

    def __sub__(self, other):
        return self._combine(other, 1.0, -1.0)

    def __rsub__(self, other):
        return self._combine(other, -1.0, 1.0)

    def __mul__(self, k):
        if isinstance(k, (int, float, np.floating, np.integer)):
            return Tensor(self.data * float(k), _terms=self._leaf_terms(float(k)))
        return NotImplemented

    __rmul__ = __mul__

    def __neg__(self):
        return self * -1.0

    def backward(self) -> None:
        """Run the hand-scheduled backward of the op(s) that produced this scalar.

        Leaves with a coefficient hook (VQ losses of an encoder graph) learn their total
        coefficient first, then ordinary leaves run (only with coefficient 1: their backward
        kernels are normalised for the loss itself), then hook leaves finish their graphs."""
        if self._terms is None and self._coef_hook is None:
            if self._backward is None:
                raise RuntimeError("backward() on a tensor that does not require grad")
            fn, self._backward = self._backward, None
            fn()
            return
        acc: dict = {}
        for t, c in self._leaf_terms(1.0):
            acc.setdefault(id(t), [t, 0.0])[1] += c
        leaves = list(acc.values())
        if all(t._backward is None and t._coef_hook is None for t, _ in leaves):
            raise RuntimeError("backward() on a tensor that does not require grad")
        for t, c in leaves:
            if t._coef_hook is not None:
                t._coef_hook(c)
        for t, c in leaves:
            if t._coef_hook is None and t._backward is not None:
                if abs(c - 1.0) > 1e-12:
                    raise NotImplementedError(f"scaled backward (coefficient {c}) of a fused loss")
                fn, t._backward = t._backward, None
                fn()
        for t, _ in leaves:
            if t._coef_hook is not None and t._backward is not None:
                fn, t._backward = t._backward, None
                fn()


def embedding(table: Tensor, ids) -> Tensor:
    """autodiff.embedding (autodiff.py:350-364): row lookup `table[ids]`; the output's backward
    scatters `out.grad` into `table.grad` with a deterministic owner-computes kernel. Gradients
    here are per-step buffers, so the scatter overwrites (the reference accumulates into a fresh
    p.grad = None each step, trainer.py:181-183)."""
    from . import kernels as K
    if isinstance(ids, torch.Tensor):
        idx = ids.to(table.data.device, torch.int64)
        if idx.numel():
            lo, hi = int(idx.min()), int(idx.max())
            if lo < 0 or hi >= table.shape[0]:
                raise IndexError(f"embedding ids out of range [0, {table.shape[0]})")
    else:
        arr = np.asarray(ids)
        if arr.size and (arr.min() < 0 or arr.max() >= table.shape[0]):
            raise IndexError(f"embedding ids out of range [0, {table.shape[0]})")
        idx = torch.as_tensor(arr.astype(np.int64)).to(table.data.device)
    out = Tensor(table.data[idx])
    if not table.requires_grad:
        return out

    def bw():
        if out.grad is None:
            return
        if table.grad is None or tuple(table.grad.shape) != tuple(table.data.shape):
            table.grad = torch.zeros_like(table.data)
        K.embedding_table_bwd(out.grad, idx, table.grad)

    out._backward = bw
    return out


def parameter(data) -> Tensor:
    return Tensor(data, requires_grad=True)


def tensor(data, dtype=np.float32, requires_grad=False) -> Tensor:
    return Tensor(np.asarray(data, dtype=dtype), requires_grad=requires_grad)


class ParamStore:
    """Flat fp32 storage for a model's parameters (+ lazily a flat gradient buffer).

    `params` is an OrderedDict name -> Tensor whose `.data` are views into `flat`.
    `groups` lists tuples of names laid out side by side as the column blocks of one matrix
    (2-D members with equal rows) or one vector (1-D members): an attention sub-layer's
    q/k/v weights become one (d, 3d) block, so its bf16 shadow and its weight gradient are
    plain contiguous views (one GEMM operand, one dW GEMM). Members are strided views.
    """

    def __init__(self, arrays: "OrderedDict[str, np.ndarray]", groups=()):
        dev = device()
        total = sum(int(a.size) for a in arrays.values())
        host = np.empty(total, dtype=np.float32)
        group_of = {}
        for g in groups:
            for n in g:
                group_of[n] = tuple(g)
        # name -> (storage offset, shape, strides); extents -> (first, last+1) storage element
        self.layout: dict[str, tuple[int, tuple, tuple]] = {}
        self.extents: dict[str, tuple[int, int]] = {}
        self.blocks: dict[tuple, tuple[int, tuple]] = {}  # group -> (offset, block shape)
        off = 0
        for name, a in arrays.items():
            if name in self.layout:
                continue
            g = group_of.get(name)
            if g is None:
                n = int(a.size)
                host[off:off + n] = a.reshape(-1).astype(np.float32)
                shp = tuple(a.shape)
                self.layout[name] = (off, shp, _contig_strides(shp))
                self.extents[name] = (off, off + max(n, 1))
                off += n
                continue
            mem = [arrays[m] for m in g]
            if any(x.ndim != mem[0].ndim for x in mem) or mem[0].ndim not in (1, 2):
                raise ValueError(f"parameter group {g}: members must all be 1-D or all 2-D")
            if mem[0].ndim == 2:
                rows = mem[0].shape[0]
                if any(x.shape[0] != rows for x in mem):
                    raise ValueError(f"parameter group {g}: 2-D members need equal row counts")
                cols = sum(x.shape[1] for x in mem)
                block = np.concatenate([x.astype(np.float32) for x in mem], axis=1)
                bshape = (rows, cols)
                c0 = 0
                for m, x in zip(g, mem):
                    self.layout[m] = (off + c0, tuple(x.shape), (cols, 1))
                    self.extents[m] = (off + c0, off + (rows - 1) * cols + c0 + x.shape[1])
                    c0 += x.shape[1]
            else:
                block = np.concatenate([x.astype(np.float32) for x in mem])
                bshape = (block.size,)
                c0 = 0
                for m, x in zip(g, mem):
                    self.layout[m] = (off + c0, tuple(x.shape), (1,))
                    self.extents[m] = (off + c0, off + c0 + x.size)
                    c0 += x.size
            host[off:off + block.size] = block.reshape(-1)
            self.blocks[tuple(g)] = (off, bshape)
            off += block.size
        # offsets (name -> (offset, shape)) kept for callers that only need the first element
        self.offsets = {n: (o, shp) for n, (o, shp, _) in self.layout.items()}
        self.flat = torch.from_numpy(host).to(dev)
        self.grad_flat: torch.Tensor | None = None
        self.params: "OrderedDict[str, Tensor]" = OrderedDict()
        for name in arrays:
            self.params[name] = Tensor(self.view_of(self.flat, name), requires_grad=True)
        _STORES[id(self.params)] = self

    def view_of(self, buf: torch.Tensor, name: str) -> torch.Tensor:
        """`name`'s view into a flat buffer laid out like `flat` (params, grads, moments, shadows)."""
        o, shp, st = self.layout[name]
        return buf.as_strided(shp, st, buf.storage_offset() + o)

    def block_of(self, buf: torch.Tensor, first: str) -> torch.Tensor | None:
        """The whole group block starting with member `first` as a contiguous view, or None."""
        for g, (o, bshape) in self.blocks.items():
            if g[0] == first:
                n = int(np.prod(bshape))
                return buf[o:o + n].view(bshape)
        return None

    def grads_are_views(self, grads: dict) -> bool:
        if self.grad_flat is None:
            return False
        for name, (o, shp, st) in self.layout.items():
            g = grads.get(name)
            if (g is None or g.data_ptr() != self.grad_flat.data_ptr() + 4 * o or tuple(g.shape) != shp
                    or (g.numel() > 1 and tuple(g.stride()) != st)):
                return False
        return True

    def grads(self) -> dict:
        """Gradient views (allocated on first use) keyed by name."""
        if self.grad_flat is None:
            self.grad_flat = torch.zeros_like(self.flat)
        return {name: self.view_of(self.grad_flat, name) for name in self.layout}

    def shadow(self) -> torch.Tensor:
        """bf16 copy of `flat` (same layout), refreshed by the caller with one cast per use."""
        if getattr(self, "_shadow", None) is None:
            self._shadow = torch.empty(self.flat.numel(), dtype=torch.bfloat16, device=self.flat.device)
        return self._shadow

    def owns(self, params: dict) -> bool:
        """True when `params` are still exactly this store's views (not swapped by a caller)."""
        if params.keys() != self.params.keys():
            return False
        return all(params[k] is self.params[k] for k in params)


def _contig_strides(shp: tuple) -> tuple:
    st, acc = [], 1
    for s in reversed(shp):
        st.append(acc)
        acc *= s
    return tuple(reversed(st))


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
