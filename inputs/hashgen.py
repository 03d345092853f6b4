"""Counter-based input generator (SURVEY.md §8(c) "Inputs").

x_r[i] = f(splitmix64(key(seed, collId, rank, i)))

A counter-based generator lets a test compute the input value of ANY element
(rank r, index i) without materialising whole buffers, which is what the
sampled parity checks at full BASELINE sizes (8 ranks x 1 GiB) need.

Value maps (chosen so that every value is EXACTLY representable in its dtype,
so no rounding happens during generation and the GPU generator in
``paper_2303_06324_b200/csrc/testgen.cu`` reproduces it bit for bit):

* ``f32`` : m = u >> 40 (24 bits), e = (u >> 32) & 7,
            x = (m - 2^23) * 2^(-23 - e)          in [-1, 1), varied exponents
            so that ring partial sums round (order-sensitive, see tests).
* ``bf16``: m = u >> 56 (8 bits),  e = (u >> 32) & 7,
            x = (m - 128) * 2^(-7 - e)            exact in bf16 (<= 8 sig. bits);
            returned as uint16 bit patterns (numpy has no bfloat16).
* ``f16`` : m = u >> 53 (11 bits), e = (u >> 32) & 7,
            x = (m - 1024) * 2^(-10 - e)          exact in IEEE binary16 (11 sig. bits,
            2^-17 >= the smallest normal's ulp range); stored as numpy float16.
* ``i32`` : low 32 bits of u, as two's-complement int32.
* ``i64`` : all 64 bits of u, as two's-complement int64.
* ``f64`` : m = u >> 11 (53 bits), e = (u >> 32) & 7,
            x = (m - 2^52) * 2^(-52 - e)          exact in binary64.

This module holds no arithmetic of the collective method.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1

DTYPES = ("i32", "f32", "bf16", "f16", "i64", "f64")
ITEMSIZE = {"i32": 4, "f32": 4, "bf16": 2, "f16": 2, "i64": 8, "f64": 8}
NP_STORAGE = {"i32": np.int32, "f32": np.float32, "bf16": np.uint16, "f16": np.float16, "i64": np.int64,
              "f64": np.float64}


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def keys(seed: int, coll: int, rank: int, idx: np.ndarray) -> np.ndarray:
    """key = seed ^ (coll << 40) ^ (rank << 32) ^ i   (i < 2^32)."""
    base = (int(seed) ^ (int(coll) << 40) ^ (int(rank) << 32)) & MASK64
    return np.asarray(idx, dtype=np.uint64) ^ np.uint64(base)


def values(dtype: str, seed: int, coll: int, rank: int, idx) -> np.ndarray:
    """Values x_rank[idx] for collective ``coll`` (storage dtype, see module doc)."""
    with np.errstate(over="ignore"):
        u = splitmix64(keys(seed, coll, rank, np.asarray(idx, dtype=np.uint64)))
    if dtype == "i32":
        return (u & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)
    if dtype == "i64":
        return u.view(np.int64)
    e = ((u >> np.uint64(32)) & np.uint64(7)).astype(np.int64)
    if dtype == "f32":
        m = (u >> np.uint64(40)).astype(np.int64) - (1 << 23)
        return np.ldexp(m.astype(np.float64), -23 - e).astype(np.float32)
    if dtype == "bf16":
        m = (u >> np.uint64(56)).astype(np.int64) - 128
        f = np.ldexp(m.astype(np.float64), -7 - e).astype(np.float32)
        return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    if dtype == "f16":
        m = (u >> np.uint64(53)).astype(np.int64) - 1024
        return np.ldexp(m.astype(np.float64), -10 - e).astype(np.float16)
    if dtype == "f64":
        m = (u >> np.uint64(11)).astype(np.int64) - (1 << 52)
        return np.ldexp(m.astype(np.float64), -52 - e)
    raise ValueError(f"unknown dtype {dtype!r}")


def buffer(dtype: str, seed: int, coll: int, rank: int, count: int, offset: int = 0) -> np.ndarray:
    """Contiguous x_rank[offset : offset + count]."""
    return values(dtype, seed, coll, rank, np.arange(offset, offset + count, dtype=np.uint64))


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """Widen bf16 bit patterns to float32 (exact; a bit shift, no arithmetic)."""
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)
