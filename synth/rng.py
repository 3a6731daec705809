"""Counter-based splitmix64 random streams (numpy, vectorised).

This module is shared by the oracle side (tests) and the CUDA side (bench,
tests): it produces *inputs only* and holds none of the ICP method's
arithmetic. Every draw is a pure function of (seed, stream, counter), so a
config is bit-reproducible regardless of numpy version for the integer part;
transcendental post-processing (Box-Muller log/cos) goes through numpy's libm
and may differ in the last ulp between hosts.

Seeds follow SURVEY.md §8(d): 0x1801_0984_7000 + 16*config_id + stream_id.
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
SEED_BASE = 0x1801_0984_7000


def config_seed(config_id: int, stream_id: int) -> int:
    return (SEED_BASE + 16 * int(config_id) + int(stream_id)) & 0xFFFFFFFFFFFFFFFF


def splitmix64(seed: int, counter: np.ndarray) -> np.ndarray:
    """splitmix64 output for state = seed + (counter+1)*golden (mod 2^64)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (counter.astype(np.uint64) + np.uint64(1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


class Stream:
    """A sequential view over one counter-based stream."""

    def __init__(self, seed: int):
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self.pos = 0

    def u64(self, n: int) -> np.ndarray:
        c = np.arange(self.pos, self.pos + n, dtype=np.uint64)
        self.pos += n
        return splitmix64(self.seed, c)

    def uniform(self, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        """fp64 uniform in [lo, hi): top 53 bits of each draw."""
        u = (self.u64(n) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
        return lo + (hi - lo) * u

    def normal(self, n: int) -> np.ndarray:
        """Standard normal via Box-Muller (two uniforms per variate, cos branch)."""
        u1 = self.uniform(n)
        u2 = self.uniform(n)
        return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)

    def integers(self, n: int, hi: int) -> np.ndarray:
        """Integers in [0, hi) (multiply-shift on the top 32 bits)."""
        top = self.u64(n) >> np.uint64(32)
        return ((top * np.uint64(hi)) >> np.uint64(32)).astype(np.int64)

    def unit_vectors(self, n: int) -> np.ndarray:
        v = np.stack([self.normal(n), self.normal(n), self.normal(n)], axis=1)
        return v / np.linalg.norm(v, axis=1, keepdims=True)
