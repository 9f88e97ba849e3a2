"""JASCKPT1 checkpoint bundles, interoperable with deskworld (checkpoint.py:1-93, trainer.py:91-115).

The file format is the reference's, byte for byte:

    b"JASCKPT1" | u64 LE meta length | meta JSON (sort_keys, default separators) |
    raw array bytes in sorted-name order | sha256(everything before)

so a bundle written here loads in deskworld and vice versa (tests/golden/ckpt_ref.jasckpt is a
file the unmodified reference wrote).  Writes are atomic (temp file + fsync + rename); readers
verify the digest before deserialising anything.

The device side packs a training stage straight from the model's flat parameter store and the
AdamW moments (one device->host copy per flat buffer) and restores IN PLACE into the live
device tensors, so the flat-buffer views (grouped q/k/v blocks, moments, shadows) stay valid and
a resumed run is bitwise identical to an uninterrupted one (tests/test_gpu_checkpoint.py).
"""
from __future__ import annotations

import hashlib
import json
import os
import struct
from dataclasses import asdict, dataclass, field
from pathlib import Path

import numpy as np
import torch

MAGIC = b"JASCKPT1"
VERSION = 1
_LEN = struct.Struct("<Q")
_DIGEST = 32


class CheckpointError(Exception):
    """Unreadable, truncated, tampered or version-incompatible checkpoint (checkpoint.py:25-26)."""


@dataclass
class CheckpointBundle:
    step: int
    config: dict
    arrays: dict                      # name -> ndarray (params, optimizer moments)
    loader_state: dict = field(default_factory=dict)
    rng_state: dict = field(default_factory=dict)
    meta: dict = field(default_factory=dict)
    version: int = VERSION


def _meta_json(bundle: CheckpointBundle, manifest: list) -> bytes:
    meta = {"version": bundle.version, "step": bundle.step, "config": bundle.config,
            "loader_state": bundle.loader_state, "rng_state": bundle.rng_state, "meta": bundle.meta,
            "manifest": manifest}
    return json.dumps(meta, sort_keys=True).encode("utf-8")


def encode_checkpoint(bundle: CheckpointBundle) -> bytes:
    """The complete file contents of `bundle` (body + sha256 trailer)."""
    names = sorted(bundle.arrays)
    parts = []
    manifest = []
    for name in names:
        arr = np.ascontiguousarray(bundle.arrays[name])
        manifest.append({"name": name, "dtype": arr.dtype.str, "shape": list(arr.shape)})
        parts.append(arr.tobytes())
    meta = _meta_json(bundle, manifest)
    h = hashlib.sha256()
    chunks = [MAGIC, _LEN.pack(len(meta)), meta] + parts
    for c in chunks:
        h.update(c)
    return b"".join(chunks) + h.digest()


def save_checkpoint(bundle: CheckpointBundle, path) -> None:
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    data = encode_checkpoint(bundle)
    tmp = path.with_suffix(path.suffix + ".tmp")
    with open(tmp, "wb") as fh:
        fh.write(data)
        fh.flush()
        os.fsync(fh.fileno())
    os.replace(tmp, path)


def decode_checkpoint(raw: bytes, where: str = "<bytes>") -> CheckpointBundle:
    head = len(MAGIC) + _LEN.size
    if len(raw) < head + _DIGEST or raw[:len(MAGIC)] != MAGIC:
        raise CheckpointError(f"{where}: not a checkpoint file")
    body = memoryview(raw)[:-_DIGEST]
    if hashlib.sha256(body).digest() != raw[-_DIGEST:]:
        raise CheckpointError(f"{where}: digest mismatch (truncated or corrupt)")
    (meta_len,) = _LEN.unpack_from(raw, len(MAGIC))
    try:
        meta = json.loads(bytes(body[head:head + meta_len]).decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise CheckpointError(f"{where}: unreadable meta block") from exc
    if meta.get("version") != VERSION:
        raise CheckpointError(f"{where}: version {meta.get('version')} not supported")
    arrays = {}
    pos = head + meta_len
    for e in meta["manifest"]:
        dt = np.dtype(e["dtype"])
        shape = tuple(e["shape"])
        n = dt.itemsize * (int(np.prod(shape)) if shape else 1)
        if pos + n > len(body):
            raise CheckpointError(f"{where}: array {e['name']!r} runs past the end of the file")
        arrays[e["name"]] = np.frombuffer(body[pos:pos + n], dtype=dt).reshape(shape).copy()
        pos += n
    return CheckpointBundle(step=meta["step"], config=meta["config"], arrays=arrays,
                            loader_state=meta["loader_state"], rng_state=meta["rng_state"], meta=meta["meta"],
                            version=meta["version"])


def load_checkpoint(path) -> CheckpointBundle:
    path = Path(path)
    return decode_checkpoint(path.read_bytes(), str(path))


# ---------------------------------------------------------------------------
# stage packing (trainer.py:91-115) from / into device tensors
# ---------------------------------------------------------------------------
def _host_views(params: dict, buf_of) -> dict:
    """name -> contiguous numpy copy of each parameter's view into a flat device buffer.

    One device->host copy per distinct flat buffer; strided (grouped) views are materialised
    row-major on the host, exactly the array the reference would hold."""
    hosts: dict = {}
    out = {}
    for name, p in params.items():
        t = buf_of(name, p)
        base = t if t._base is None else t._base
        key = (base.data_ptr(), base.numel())
        if key not in hosts:
            hosts[key] = (base.detach().cpu(), base)
        hb, db = hosts[key]
        view = hb.as_strided(t.shape, t.stride(), t.storage_offset() - db.storage_offset())
        out[name] = np.ascontiguousarray(view.numpy())
    return out


def pack_stage(stage: str, config: dict, params: dict, adam, loader_state, step: int, seed: int) -> CheckpointBundle:
    """The reference's _pack (trainer.py:91-102): param.* / adam.m.* / adam.v.* arrays + AdamW meta."""
    pv = _host_views(params, lambda n, p: p.data)
    mv = _host_views(params, lambda n, p: adam.m[n])
    vv = _host_views(params, lambda n, p: adam.v[n])
    arrays = {}
    for name in sorted(params):
        arrays[f"param.{name}"] = pv[name]
        arrays[f"adam.m.{name}"] = mv[name]
        arrays[f"adam.v.{name}"] = vv[name]
    meta = {"stage": stage, "seed": seed,
            "adam": {"t": adam.t, "beta1": adam.beta1, "beta2": adam.beta2, "eps": adam.eps,
                     "weight_decay": adam.weight_decay}}
    ls = asdict(loader_state) if not isinstance(loader_state, dict) else dict(loader_state)
    return CheckpointBundle(step=step, config=config, arrays=arrays, loader_state=ls,
                            rng_state={"seed": seed, "stage": stage}, meta=meta)


def restore_stage(bundle: CheckpointBundle, params: dict, adam=None):
    """trainer.py:105-115: copy a packed stage back into the LIVE device tensors.

    Returns (adam_state, loader_state_dict, step).  `adam` (an AdamWState from adamw_init on the
    same params) is restored in place when given; otherwise a fresh state is built."""
    from .optim import adamw_init
    am = bundle.meta["adam"]
    if adam is None:
        adam = adamw_init(params, weight_decay=am["weight_decay"], beta1=am["beta1"], beta2=am["beta2"],
                          eps=am["eps"])
    missing = [n for n in params if f"param.{n}" not in bundle.arrays]
    if missing:
        raise CheckpointError(f"checkpoint lacks parameters {missing[:5]}")
    for name, p in params.items():
        for dst, key in ((p.data, f"param.{name}"), (adam.m[name], f"adam.m.{name}"), (adam.v[name], f"adam.v.{name}")):
            src = bundle.arrays[key]
            if tuple(src.shape) != tuple(dst.shape):
                raise CheckpointError(f"{key}: shape {tuple(src.shape)} != live {tuple(dst.shape)}")
            dst.copy_(torch.from_numpy(np.ascontiguousarray(src, dtype=np.float32)))
    adam.t = am["t"]
    adam.beta1, adam.beta2, adam.eps, adam.weight_decay = am["beta1"], am["beta2"], am["eps"], am["weight_decay"]
    return adam, dict(bundle.loader_state), bundle.step
