"""JASREC record store + deterministic loader (records.py:1-410), with a device data path.

File layout (little-endian, records.py:7-16), interoperable with deskworld both ways:

    b"JASREC\\x01\\x00" | u32 version | u32 count | u32 frames_per_record | u16 h, w, c |
    u64 absolute payload offset per record | per record: frames bytes + one u8 action per frame

`shuffled_batches` yields the reference's batches bit for bit (the epoch permutation is
stream(seed, "perm", epoch).permutation(total) and each record's subsequence start is
fold_key(seed, "subseq", epoch, record) % span, both on the numpy Philox mirror in rng.py), but
reads only the subsequence's bytes instead of the whole record.

`DeviceBatchLoader` is the B200 side: a worker thread assembles batches straight
into a ring of pinned host slots, each batch goes up as one uint8 H2D copy on a side stream, and
the consumer receives device uint8 frames (B, T, H, W, C) ready for the fused unit/patchify
kernel (jz_patchify) — 12 KB per 64x64x3 frame, so even 100k frames/s is 1.2 GB/s of PCIe.
"""
from __future__ import annotations

import hashlib
import json
import os
import queue
import struct
import threading
from dataclasses import dataclass, replace
from pathlib import Path

import numpy as np
import torch

from .rng import fold_key, stream

MAGIC = b"JASREC\x01\x00"
VERSION = 1
_FIXED = struct.Struct("<IIIHHH")  # version, count, frames_per_record, h, w, c


class RecordFormatError(Exception):
    """Corrupt or incompatible record file (records.py:40-41)."""


@dataclass(frozen=True)
class Chunking:
    frames_per_record: int = 160
    records_per_file: int = 100


@dataclass(frozen=True)
class LoaderState:
    seed: int
    epoch: int = 0
    cursor: int = 0
    prefetch_depth: int = 1


@dataclass
class DatasetIndex:
    root: Path
    files: list
    frames_per_record: int
    records_per_file: int
    geometry: tuple
    record_seeds: list

    @property
    def total_records(self) -> int:
        return sum(f["records"] for f in self.files)

    def save(self) -> None:
        (Path(self.root) / "index.json").write_text(json.dumps({
            "files": self.files, "frames_per_record": self.frames_per_record,
            "records_per_file": self.records_per_file, "geometry": list(self.geometry),
            "record_seeds": self.record_seeds}))

    @classmethod
    def load(cls, root) -> "DatasetIndex":
        root = Path(root)
        d = json.loads((root / "index.json").read_text())
        return cls(root=root, files=d["files"], frames_per_record=d["frames_per_record"],
                   records_per_file=d["records_per_file"], geometry=tuple(d["geometry"]),
                   record_seeds=d["record_seeds"])


def _frame_bytes(geometry) -> int:
    h, w, c = geometry
    return h * w * c


def _file_image(records: list, fpr: int, geometry) -> np.ndarray:
    """The whole JASREC file (records.py:7-16) as one uint8 array: header, absolute payload
    offsets, then each record's frames followed by its per-frame actions."""
    h, w, c = geometry
    n = len(records)
    head = MAGIC + _FIXED.pack(VERSION, n, fpr, h, w, c)
    rec_bytes = fpr * _frame_bytes(geometry) + fpr
    base = len(head) + 8 * n
    img = np.empty(base + n * rec_bytes, dtype=np.uint8)
    img[:len(head)] = np.frombuffer(head, dtype=np.uint8)
    offsets = base + rec_bytes * np.arange(n, dtype="<u8")
    img[len(head):base] = offsets.view(np.uint8)
    body = img[base:].reshape(n, rec_bytes) if n else img[base:].reshape(0, rec_bytes)
    nfb = fpr * _frame_bytes(geometry)
    for row, (frames, actions) in zip(body, records):
        row[:nfb] = np.asarray(frames, dtype=np.uint8).reshape(-1)
        row[nfb:] = np.asarray(actions, dtype=np.uint8).reshape(-1)
    return img


def _atomic_write(path: Path, data: np.ndarray) -> None:
    """Write through a sibling temp file and rename: a reader never sees a partial file."""
    tmp = path.with_suffix(".tmp")
    try:
        data.tofile(tmp)
        os.replace(tmp, path)
    finally:
        if tmp.exists():
            tmp.unlink()


def _full_records(episodes, fpr: int):
    """(seed, geometry, frames, actions) of every whole frames_per_record chunk of every episode;
    shorter episodes and ragged tails yield nothing (records.py:120-169 chunking rule)."""
    for ep in episodes:
        frames = np.asarray(ep.frames)
        for k in range(len(frames) // fpr):
            sl = slice(k * fpr, (k + 1) * fpr)
            yield int(ep.seed), tuple(int(g) for g in frames.shape[1:]), frames[sl], np.asarray(ep.actions)[sl]


def write_dataset(episodes, chunking: Chunking, out_dir) -> DatasetIndex:
    """records.py:120-169: fixed-size records grouped records_per_file to a file
    (records-00000.bin, ...), plus index.json.  Byte-identical to the reference's files."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    fpr, rpf = chunking.frames_per_record, chunking.records_per_file
    files, seeds, group, geometry = [], [], [], None

    def emit():
        name = f"records-{len(files):05d}.bin"
        _atomic_write(out / name, _file_image(group, fpr, geometry))
        files.append({"name": name, "records": len(group)})
        group.clear()

    for seed, geo, frames, actions in _full_records(episodes, fpr):
        geometry = geometry or geo
        group.append((frames, actions))
        seeds.append(seed)
        if len(group) == rpf:
            emit()
    if group:
        emit()
    if geometry is None:
        raise ValueError("no episodes long enough to produce a record")
    index = DatasetIndex(root=out, files=files, frames_per_record=fpr, records_per_file=rpf, geometry=geometry,
                         record_seeds=seeds)
    index.save()
    return index


class RecordReader:
    """One record file: header checked once, O(1) positioned reads (os.pread, thread-safe)."""

    def __init__(self, path):
        self.path = Path(path)
        self._fd = os.open(self.path, os.O_RDONLY)
        head = os.pread(self._fd, len(MAGIC) + _FIXED.size, 0)
        if len(head) < len(MAGIC) + _FIXED.size or head[:len(MAGIC)] != MAGIC:
            os.close(self._fd)
            raise RecordFormatError(f"{self.path}: bad magic")
        version, self.count, self.frames_per_record, h, w, c = _FIXED.unpack(head[len(MAGIC):])
        if version != VERSION:
            os.close(self._fd)
            raise RecordFormatError(f"{self.path}: unsupported version {version}")
        self.geometry = (h, w, c)
        raw = os.pread(self._fd, 8 * self.count, len(MAGIC) + _FIXED.size)
        if len(raw) != 8 * self.count:
            os.close(self._fd)
            raise RecordFormatError(f"{self.path}: truncated offset table")
        self._offsets = struct.unpack(f"<{self.count}Q", raw)
        self._fb = _frame_bytes(self.geometry)

    def _check(self, i: int) -> int:
        if not 0 <= i < self.count:
            raise IndexError(f"record {i} outside [0, {self.count})")
        return self._offsets[i]

    def read(self, i: int):
        """records.py:198-210: (frames (fpr, h, w, c) u8, actions (fpr,) u8)."""
        off = self._check(i)
        n = self.frames_per_record * (self._fb + 1)
        blob = os.pread(self._fd, n, off)
        if len(blob) != n:
            raise RecordFormatError(f"{self.path}: truncated record {i}")
        nfb = self.frames_per_record * self._fb
        frames = np.frombuffer(blob[:nfb], dtype=np.uint8).reshape((self.frames_per_record,) + self.geometry)
        return frames, np.frombuffer(blob[nfb:], dtype=np.uint8)

    def read_span_into(self, i: int, start: int, length: int, frames_out: np.ndarray, actions_out: np.ndarray):
        """Frames [start, start+length) of record i written straight into caller buffers."""
        off = self._check(i)
        n = length * self._fb
        got = os.preadv(self._fd, [memoryview(frames_out.reshape(-1))[:n]], off + start * self._fb)
        a = os.pread(self._fd, length, off + self.frames_per_record * self._fb + start)
        if got != n or len(a) != length:
            raise RecordFormatError(f"{self.path}: truncated record {i}")
        actions_out[:] = np.frombuffer(a, dtype=np.uint8)

    def close(self):
        if self._fd >= 0:
            os.close(self._fd)
            self._fd = -1


class DatasetReader:
    """records.py:213-242: random access over every file of an index."""

    def __init__(self, index: DatasetIndex):
        self.index = index
        self._readers: dict = {}
        self._starts = np.cumsum([0] + [f["records"] for f in index.files])
        self.total = int(self._starts[-1])

    def _locate(self, i: int):
        if not 0 <= i < self.total:
            raise IndexError(f"record {i} outside [0, {self.total})")
        fid = int(np.searchsorted(self._starts, i, side="right") - 1)
        if fid not in self._readers:
            self._readers[fid] = RecordReader(Path(self.index.root) / self.index.files[fid]["name"])
        return self._readers[fid], i - int(self._starts[fid])

    def read_record(self, i: int):
        r, j = self._locate(i)
        return r.read(j)

    def read_span_into(self, i: int, start: int, length: int, frames_out, actions_out):
        r, j = self._locate(i)
        r.read_span_into(j, start, length, frames_out, actions_out)

    def close(self):
        for r in self._readers.values():
            r.close()
        self._readers.clear()


def read_record(index: DatasetIndex, i: int):
    reader = DatasetReader(index)
    try:
        return reader.read_record(i)
    finally:
        reader.close()


def subsequence_start(seed: int, epoch: int, record_id: int, fpr: int, seq_len: int) -> int:
    """records.py:253-256."""
    return fold_key(seed, "subseq", epoch, record_id) % (fpr - seq_len + 1)


def _epoch_batches(seed: int, epoch: int, first: int, total: int, batch_size: int):
    """Record ids of the batches of one epoch from cursor `first`: consecutive windows of the
    epoch's permutation stream(seed, "perm", epoch) (records.py:273-294)."""
    order = stream(seed, "perm", epoch).permutation(total)
    return [order[c:c + batch_size] for c in range(first, total - batch_size + 1, batch_size)]


def _batch_plan(index: DatasetIndex, state: LoaderState, batch_size: int, seq_len: int):
    """(record ids, subsequence starts, loader state after the batch) of every batch, in the
    reference's order.  The state after a batch points at the next batch: the same epoch at the
    next cursor, or cursor 0 of the next epoch when no full batch is left."""
    if seq_len > index.frames_per_record:
        raise ValueError("seq_len exceeds frames_per_record")
    total = index.total_records
    if batch_size > total:
        raise ValueError(f"batch_size {batch_size} > total records {total}")
    fpr = index.frames_per_record
    epoch, cursor = state.epoch, state.cursor
    while True:
        for ids in _epoch_batches(state.seed, epoch, cursor, total, batch_size):
            cursor += batch_size
            after = (epoch, cursor) if cursor + batch_size <= total else (epoch + 1, 0)
            rids = [int(r) for r in ids]
            yield (rids, [subsequence_start(state.seed, epoch, r, fpr, seq_len) for r in rids],
                   replace(state, epoch=after[0], cursor=after[1]))
        epoch, cursor = epoch + 1, 0


def shuffled_batches(index: DatasetIndex, state: LoaderState, batch_size: int, seq_len: int = 16):
    """records.py:259-292: endless (frames (B,T,H,W,C) u8, actions (B,T) u8, next_state) stream;
    only each record's subsequence bytes are read."""
    reader = DatasetReader(index)
    shape = (batch_size, seq_len) + tuple(index.geometry)
    try:
        for ids, starts, nxt in _batch_plan(index, state, batch_size, seq_len):
            frames = np.empty(shape, dtype=np.uint8)
            actions = np.empty(shape[:2], dtype=np.uint8)
            for j, rid in enumerate(ids):
                reader.read_span_into(rid, starts[j], seq_len, frames[j], actions[j])
            yield frames, actions, nxt
    finally:
        reader.close()


_END = object()


def prefetch(iterator, depth: int):
    """records.py:295-322 semantics (same items in the same order, produced ahead by a background
    thread; a producer error re-raises at the consumer): `depth` next() calls are kept in flight
    on a single worker thread."""
    if depth < 1:
        raise ValueError("depth must be >= 1")
    import collections
    from concurrent.futures import ThreadPoolExecutor
    source = iter(iterator)
    pool = ThreadPoolExecutor(max_workers=1, thread_name_prefix="jasrec-prefetch")
    try:
        ahead = collections.deque(pool.submit(next, source, _END) for _ in range(depth))
        while True:
            item = ahead.popleft().result()
            if item is _END:
                return
            ahead.append(pool.submit(next, source, _END))
            yield item
    finally:
        pool.shutdown(wait=False, cancel_futures=True)


def detect_duplicates(index: DatasetIndex) -> dict:
    """records.py:329-378 (byte-confirmed exact duplicate frames): {"groups": [[(rec, frame), ...], ...]}."""
    reader = DatasetReader(index)
    try:
        seen: dict = {}
        for r in range(index.total_records):
            frames, _ = reader.read_record(r)
            for k, f in enumerate(frames):
                key = hashlib.blake2b(f.tobytes(), digest_size=16).digest()
                seen.setdefault(key, []).append((r, k, f.copy()))
        groups = []
        for items in seen.values():
            if len(items) > 1:
                first = items[0][2]
                same = [(r, k) for r, k, f in items if np.array_equal(f, first)]
                if len(same) > 1:
                    groups.append(same)
        return {"groups": groups}
    finally:
        reader.close()


class DeviceBatchLoader:
    """Deterministic batches delivered to the GPU: (frames u8 (B,T,H,W,C), actions u8 (B,T), next_state).

    A worker thread fills a ring of `depth + 1` pinned slots (positioned reads straight into the
    slot); each batch is one non-blocking H2D copy on a side stream, and a slot is refilled only
    after its copy event completed.  The consumer's current stream waits on the copy event, so
    the device tensors are safe to use immediately.  Same batch sequence as shuffled_batches.
    """

    def __init__(self, index: DatasetIndex, state: LoaderState, batch_size: int, seq_len: int = 16, *,
                 depth: int = 2, device=None):
        self.index, self.B, self.T = index, batch_size, seq_len
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        geo = tuple(index.geometry)
        nslots = depth + 1
        self._frames = [torch.empty((batch_size, seq_len) + geo, dtype=torch.uint8).pin_memory() for _ in range(nslots)]
        self._actions = [torch.empty((batch_size, seq_len), dtype=torch.uint8).pin_memory() for _ in range(nslots)]
        self._copied = [None] * nslots          # CUDA event of the last H2D out of each slot
        self._free: queue.Queue = queue.Queue()
        for k in range(nslots):
            self._free.put(k)
        self._ready: queue.Queue = queue.Queue()
        self._stream = torch.cuda.Stream(device=self.device)
        self._stop = threading.Event()
        self._plan = _batch_plan(index, state, batch_size, seq_len)
        self._thread = threading.Thread(target=self._work, daemon=True)
        self._thread.start()

    def _work(self):
        reader = DatasetReader(self.index)
        try:
            for ids, starts, nxt in self._plan:
                k = self._free.get()
                if k is None or self._stop.is_set():
                    return
                if self._copied[k] is not None:
                    self._copied[k].synchronize()   # the previous batch left this slot
                fr, ac = self._frames[k].numpy(), self._actions[k].numpy()
                for j, (rid, st) in enumerate(zip(ids, starts)):
                    reader.read_span_into(rid, st, self.T, fr[j], ac[j])
                self._ready.put((k, nxt))
        except BaseException as exc:  # surfaced to the consumer
            self._ready.put(exc)
        finally:
            reader.close()

    def __iter__(self):
        return self

    def __next__(self):
        item = self._ready.get()
        if isinstance(item, BaseException):
            raise item
        k, nxt = item
        with torch.cuda.stream(self._stream):
            frames = self._frames[k].to(self.device, non_blocking=True)
            actions = self._actions[k].to(self.device, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self._stream)
        self._copied[k] = ev
        torch.cuda.current_stream(self.device).wait_event(ev)
        frames.record_stream(torch.cuda.current_stream(self.device))
        actions.record_stream(torch.cuda.current_stream(self.device))
        self._free.put(k)
        return frames, actions, nxt

    def close(self):
        self._stop.set()
        self._free.put(None)
        self._thread.join(timeout=5)
