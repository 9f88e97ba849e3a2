"""ORACLE (test infrastructure only) — deterministic RNG restatement.

Restates deskworld/rng.py (splitmix64 :17-23, fold_key :26-35, stream :38-44) and
the numpy Philox4x64-10 bit generator that `stream` wraps (numpy is the
reference's unpinned third-party dependency, pyproject.toml:11; here numpy 2.3).
numpy's published algorithm (numpy/random/src/philox/philox.h):

  * state: 256-bit counter c[4] (starts 0), 128-bit key k[2] = (key & 2^64-1, key >> 64)
  * next_uint64: if buffer exhausted -> counter += 1 (with carry), buffer =
    Philox4x64_10(counter, key), return buffer[0]; else return buffer[pos++]
  * Philox4x64 round: (hi0,lo0)=M0*c0, (hi1,lo1)=M1*c2,
    c = [hi1^c1^k0, lo1, hi0^c3^k1, lo0]; key += (W0, W1) between rounds
  * next_double = (u64 >> 11) * 2^-53;  uniform(a,b) = a + (b-a)*next_double

so draw i of a fresh stream is word i%4 of the block at counter 1 + i//4.
Pinned by tests/golden/rng_golden.npz (raw words + doubles + masks produced by
the reference) and the known-answer vector of SURVEY Appendix B.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
PHILOX_M0 = 0xD2E7470EE14C6C93
PHILOX_M1 = 0xCA5A826395121157
PHILOX_W0 = 0x9E3779B97F4A7C15
PHILOX_W1 = 0xBB67AE8584CAA73B


def splitmix64(x: int) -> int:
    """deskworld/rng.py:17-23."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def fold_key(*parts) -> int:
    """deskworld/rng.py:26-35: strings fold byte-wise (utf-8), ints as 64-bit words."""
    acc = 0x243F6A8885A308D3
    for part in parts:
        if isinstance(part, str):
            for byte in part.encode("utf-8"):
                acc = splitmix64(acc ^ byte)
        else:
            acc = splitmix64(acc ^ (int(part) & MASK64))
    return acc


def stream(*parts) -> np.random.Generator:
    """deskworld/rng.py:38-44 (numpy Generator over Philox keyed by fold_key)."""
    return np.random.Generator(np.random.Philox(key=fold_key(*parts)))


# --------------------------------------------------------------------------
# Philox4x64-10, vectorised over counters (exact uint64 arithmetic)
# --------------------------------------------------------------------------
_M32 = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def _mulhilo(a: int, b: np.ndarray):
    a_lo, a_hi = np.uint64(a & 0xFFFFFFFF), np.uint64(a >> 32)
    b_lo, b_hi = b & _M32, b >> _S32
    with np.errstate(over="ignore"):
        lo = np.uint64(a) * b
        t = a_lo * b_lo
        m1 = a_hi * b_lo
        m2 = a_lo * b_hi
        carry = ((t >> _S32) + (m1 & _M32) + (m2 & _M32)) >> _S32
        hi = a_hi * b_hi + (m1 >> _S32) + (m2 >> _S32) + carry
    return hi, lo


def philox4x64_10(counters: np.ndarray, key: tuple[int, int]) -> np.ndarray:
    """counters: (n, 4) uint64 -> (n, 4) uint64 output words."""
    c = [counters[:, i].astype(np.uint64) for i in range(4)]
    k0, k1 = key[0] & MASK64, key[1] & MASK64
    for r in range(10):
        if r:
            k0 = (k0 + PHILOX_W0) & MASK64
            k1 = (k1 + PHILOX_W1) & MASK64
        hi0, lo0 = _mulhilo(PHILOX_M0, c[0])
        hi1, lo1 = _mulhilo(PHILOX_M1, c[2])
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
    return np.stack(c, axis=1)


def _add_counter(counter: list[int], n: int) -> list[int]:
    v = sum(int(w) << (64 * i) for i, w in enumerate(counter)) + n
    v &= (1 << 256) - 1
    return [(v >> (64 * i)) & MASK64 for i in range(4)]


class PhiloxState:
    """A snapshot of numpy's Philox bit-generator state (counter, key, buffer, pos)."""

    def __init__(self, counter, key, buffer, buffer_pos):
        self.counter = [int(x) for x in counter]
        self.key = (int(key[0]), int(key[1]))
        self.buffer = [int(x) for x in buffer]
        self.buffer_pos = int(buffer_pos)

    @classmethod
    def fresh(cls, key: int) -> "PhiloxState":
        return cls([0, 0, 0, 0], (key & MASK64, key >> 64), [0, 0, 0, 0], 4)

    @classmethod
    def of(cls, gen: np.random.Generator) -> "PhiloxState":
        st = gen.bit_generator.state
        if st["bit_generator"] != "Philox":
            raise ValueError("only Philox generators are supported")
        return cls(st["state"]["counter"], st["state"]["key"], st["buffer"], st["buffer_pos"])

    def words(self, n: int) -> np.ndarray:
        """The next n uint64 draws (does not mutate)."""
        out = np.empty(n, dtype=np.uint64)
        avail = 4 - self.buffer_pos
        take = min(avail, n)
        if take > 0:
            out[:take] = np.array(self.buffer[self.buffer_pos:self.buffer_pos + take], dtype=np.uint64)
        rest = n - take
        if rest > 0:
            nblocks = (rest + 3) // 4
            base = sum(int(w) << (64 * i) for i, w in enumerate(self.counter))
            ctrs = np.zeros((nblocks, 4), dtype=np.uint64)
            idx = np.arange(1, nblocks + 1, dtype=object) + base
            if (base + nblocks) >> 64:
                for i in range(4):
                    ctrs[:, i] = np.array([(int(v) >> (64 * i)) & MASK64 for v in idx], dtype=np.uint64)
            else:
                ctrs[:, 0] = np.arange(1, nblocks + 1, dtype=np.uint64) + np.uint64(base)
            blocks = philox4x64_10(ctrs, self.key).reshape(-1)
            out[take:] = blocks[:rest]
        return out

    def advanced(self, n: int) -> "PhiloxState":
        """State after n uint64 draws."""
        avail = 4 - self.buffer_pos
        if n <= avail:
            return PhiloxState(self.counter, self.key, self.buffer, self.buffer_pos + n)
        rest = n - avail
        nblocks = (rest + 3) // 4
        counter = _add_counter(self.counter, nblocks)
        blk = philox4x64_10(np.array([counter], dtype=np.uint64), self.key)[0]
        pos = rest - 4 * (nblocks - 1)
        return PhiloxState(counter, self.key, [int(x) for x in blk], pos)

    def apply_to(self, gen: np.random.Generator) -> None:
        st = gen.bit_generator.state
        st["state"]["counter"] = np.array(self.counter, dtype=np.uint64)
        st["state"]["key"] = np.array(self.key, dtype=np.uint64)
        st["buffer"] = np.array(self.buffer, dtype=np.uint64)
        st["buffer_pos"] = self.buffer_pos
        gen.bit_generator.state = st


def words_to_doubles(w: np.ndarray) -> np.ndarray:
    """numpy next_double: (u64 >> 11) * 2^-53."""
    return (w >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def sample_masks(state: PhiloxState, batch: int, frames: int, patches: int,
                 mask_limit: float = 0.5, return_p: bool = False):
    """deskworld/dynamics.py:52-62 via the stream layout above.

    p = uniform(mask_limit, 1, B)  (draws 0..B-1);  mask = random((B,T,N)) < p[:,None,None]
    (draws B..B+BTN-1, C order);  mask[:, 0] = False (its draws are still consumed).
    """
    n = batch + batch * frames * patches
    u = words_to_doubles(state.words(n))
    p = mask_limit + (1.0 - mask_limit) * u[:batch]
    mask = u[batch:].reshape(batch, frames, patches) < p[:, None, None]
    mask[:, 0] = False
    return (mask, p) if return_p else mask


def mask_element(key: int, batch_global: int, frames: int, patches: int, b: int, t: int, n: int,
                 mask_limit: float = 0.5) -> bool:
    """Single mask element by counter skip-ahead (DP sharding contract)."""
    st = PhiloxState.fresh(key)
    u_b = words_to_doubles(_word_at(st, b))[0]
    idx = batch_global + (b * frames + t) * patches + n
    u = words_to_doubles(_word_at(st, idx))[0]
    p = mask_limit + (1.0 - mask_limit) * u_b
    return bool(t != 0 and u < p)


def _word_at(state: PhiloxState, i: int) -> np.ndarray:
    blk = philox4x64_10(np.array([_add_counter(state.counter, 1 + i // 4)], dtype=np.uint64), state.key)
    return blk[:, i % 4]


def keep_schedule(n: int, steps: int) -> list[int]:
    """MaskGIT keep counts per step, deskworld/dynamics.py:177-179 (before the known-count max)."""
    out = []
    for s in range(1, steps + 1):
        frac = np.cos(np.pi / 2 * s / steps)
        out.append(n if s == steps else min(n, int(np.ceil(n * (1.0 - frac)))))
    return out
