"""Deterministic random streams (mirror of deskworld/rng.py) + device Philox hand-off.

`splitmix64`, `fold_key` and `stream` are the reference's host API (rng.py:17-44).
`PhiloxState` snapshots a numpy Philox bit generator so the device kernel
(jz_philox_mask, csrc/philox.cuh) can draw the SAME numbers the host generator
would, and `consume(gen, n)` advances the host generator past the draws the device
used — so host and device draws interleave exactly like the reference's.
"""
from __future__ import annotations

import numpy as np

_MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def fold_key(*parts) -> int:
    acc = 0x243F6A8885A308D3
    for part in parts:
        if isinstance(part, str):
            for byte in part.encode("utf-8"):
                acc = splitmix64(acc ^ byte)
        else:
            acc = splitmix64(acc ^ (int(part) & _MASK64))
    return acc


def stream(*parts) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=fold_key(*parts)))


def _philox_block(counter: list[int], key: tuple[int, int]) -> list[int]:
    c0, c1, c2, c3 = counter
    k0, k1 = key
    for r in range(10):
        if r:
            k0 = (k0 + 0x9E3779B97F4A7C15) & _MASK64
            k1 = (k1 + 0xBB67AE8584CAA73B) & _MASK64
        p0 = 0xD2E7470EE14C6C93 * c0
        p1 = 0xCA5A826395121157 * c2
        hi0, lo0 = p0 >> 64, p0 & _MASK64
        hi1, lo1 = p1 >> 64, p1 & _MASK64
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return [c0, c1, c2, c3]


class PhiloxState:
    __slots__ = ("counter", "key", "buffer", "buffer_pos")

    def __init__(self, counter, key, buffer, buffer_pos):
        self.counter = [int(x) for x in counter]
        self.key = (int(key[0]), int(key[1]))
        self.buffer = [int(x) for x in buffer]
        self.buffer_pos = int(buffer_pos)

    @classmethod
    def of(cls, gen: np.random.Generator) -> "PhiloxState":
        st = gen.bit_generator.state
        if st.get("bit_generator") != "Philox":
            raise ValueError("device sampling needs a Philox generator (deskworld.rng.stream)")
        return cls(st["state"]["counter"], st["state"]["key"], st["buffer"], st["buffer_pos"])

    def advanced(self, n: int) -> "PhiloxState":
        avail = 4 - self.buffer_pos
        if n <= avail:
            return PhiloxState(self.counter, self.key, self.buffer, self.buffer_pos + n)
        rest = n - avail
        nblocks = (rest + 3) // 4
        v = sum(w << (64 * i) for i, w in enumerate(self.counter)) + nblocks
        v &= (1 << 256) - 1
        counter = [(v >> (64 * i)) & _MASK64 for i in range(4)]
        return PhiloxState(counter, self.key, _philox_block(counter, self.key), rest - 4 * (nblocks - 1))

    def apply_to(self, gen: np.random.Generator) -> None:
        st = gen.bit_generator.state
        st["state"]["counter"] = np.array(self.counter, dtype=np.uint64)
        st["state"]["key"] = np.array(self.key, dtype=np.uint64)
        st["buffer"] = np.array(self.buffer, dtype=np.uint64)
        st["buffer_pos"] = self.buffer_pos
        gen.bit_generator.state = st


def consume(gen: np.random.Generator, n: int) -> PhiloxState:
    """Snapshot `gen`, advance it by n uint64 draws (as if the host had drawn them); return the snapshot."""
    st = PhiloxState.of(gen)
    st.advanced(n).apply_to(gen)
    return st
