"""Seeded synthetic inputs shared by the tests, smoke() and bench.py's CPU legs.

Holds none of the decoder's arithmetic: it draws random information bits and channel
noise and applies the channel model the paper names (BPSK over AWGN with random
codewords).  Codewords are computed by the caller (tests use ``oracle.encode_*``).

Recipe (readings C6/C7):
  * generator: Philox4x32-10 (numpy ``Philox``) keyed by (seed, global frame index), so a
    frame's content does not depend on batching or on the number of ranks;
  * per frame: K information bits, then N standard normals;
  * BPSK 0 -> +1, 1 -> -1; y = s + sigma n, sigma^2 = 1 / (2 R 10^(EbN0/10)), R = K/N;
  * channel LLR = 2 y / sigma^2 rounded to float32;
  * int8 profile: q = clamp(rint_half_even(4 * LLR), -127, 127)   (2 fractional bits).
"""
from __future__ import annotations

import numpy as np

DEFAULT_SEED = 1504000353
Q_SCALE = 4.0


def sigma2(ebn0_db: float, K: int, N: int) -> float:
    R = K / N
    return 1.0 / (2.0 * R * 10.0 ** (ebn0_db / 10.0))


def _rng(seed: int, frame: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=np.array([seed, frame], dtype=np.uint64)))


def draw(seed: int, first_frame: int, n_frames: int, K: int, N: int):
    """(info bits uint8[n, K], standard normals float64[n, N]) for frames
    first_frame .. first_frame + n_frames - 1."""
    bits = np.empty((n_frames, K), np.uint8)
    noise = np.empty((n_frames, N), np.float64)
    for r in range(n_frames):
        g = _rng(seed, first_frame + r)
        bits[r] = g.integers(0, 2, size=K, dtype=np.uint8)
        noise[r] = g.standard_normal(N)
    return bits, noise


def bpsk_awgn_llr(codewords: np.ndarray, noise: np.ndarray, ebn0_db: float, K: int) -> np.ndarray:
    """Channel LLRs (float32) for codewords uint8[n, N] and unit normals float64[n, N]."""
    N = codewords.shape[-1]
    s2 = sigma2(ebn0_db, K, N)
    y = (1.0 - 2.0 * codewords.astype(np.float64)) + np.sqrt(s2) * noise
    return (2.0 * y / s2).astype(np.float32)


def quantize_i8(llr: np.ndarray, scale: float = Q_SCALE) -> np.ndarray:
    q = np.rint(np.asarray(llr, np.float64) * scale)
    return np.clip(q, -127, 127).astype(np.int8)


def random_llr_f32(seed: int, shape, scale: float = 4.0) -> np.ndarray:
    """Plain Gaussian LLRs (no codeword) for decoder edge/stress tests."""
    g = np.random.Generator(np.random.Philox(key=np.array([seed, 0xF32], dtype=np.uint64)))
    return (g.standard_normal(shape) * scale).astype(np.float32)


def random_llr_i8(seed: int, shape, lo: int = -128, hi: int = 127) -> np.ndarray:
    g = np.random.Generator(np.random.Philox(key=np.array([seed, 0x18], dtype=np.uint64)))
    return g.integers(lo, hi + 1, size=shape, dtype=np.int64).astype(np.int8)


def random_mask(seed: int, N: int, K: int) -> np.ndarray:
    """A uniformly random frozen set with N-K frozen positions (not a construction)."""
    g = np.random.Generator(np.random.Philox(key=np.array([seed, 0x3A5C], dtype=np.uint64)))
    m = np.zeros(N, np.uint8)
    m[g.permutation(N)[: N - K]] = 1
    return m
