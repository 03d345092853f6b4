"""Seeded inputs that mix IEEE-754 special values (test infrastructure).

The counter-based generator (inputs.hashgen) only produces finite normal values.
The special-value parity tests need the cases where a reducing function's
definition has edges: signed zeros (-0 + -0 = -0, -0 + +0 = +0 under
round-to-nearest; max/min with -0 < +0), subnormal operands and results
(gradual underflow, no flush-to-zero), and +-Inf (Inf + -Inf = NaN).

Each element draws one category; bit patterns are built per storage format:

  category   p      pattern
  +0 / -0    .20/.20  sign only
  subnormal  .30    exponent 0, random non-zero mantissa, random sign
  tiny       .12    the smallest normal exponent (or the next), random mantissa / sign
  normal     .15    exponent near 1.0, random mantissa / sign
  +Inf/-Inf  .015/.015

This module holds no arithmetic of the collective method.
"""
from __future__ import annotations

import numpy as np

# storage bits: (total bits, exponent bits, mantissa bits)
FORMATS = {"f32": (32, 8, 23), "bf16": (16, 8, 7), "f16": (16, 5, 10)}
_CUM = np.cumsum([0.20, 0.20, 0.30, 0.12, 0.15, 0.015, 0.015])


def special_bits(dtype: str, seed: int, rank: int, count: int) -> np.ndarray:
    """Unsigned bit patterns (uint32 for f32, uint16 for bf16 / f16)."""
    tot, eb, mb = FORMATS[dtype]
    rng = np.random.default_rng([int(seed), int(rank), tot, eb])
    cat = np.searchsorted(_CUM, rng.random(count) * _CUM[-1], side="right")
    sign = rng.integers(0, 2, count, dtype=np.uint64) << np.uint64(tot - 1)
    mant = rng.integers(1, 1 << mb, count, dtype=np.uint64)
    bias = (1 << (eb - 1)) - 1
    exp_inf = np.uint64((1 << eb) - 1)
    out = np.zeros(count, dtype=np.uint64)
    e = np.zeros(count, dtype=np.uint64)
    m = np.zeros(count, dtype=np.uint64)
    s = np.zeros(count, dtype=np.uint64)
    s[cat == 1] = np.uint64(1) << np.uint64(tot - 1)            # -0 (cat 0: +0)
    sub = cat == 2
    m[sub], s[sub] = mant[sub], sign[sub]
    tiny = cat == 3
    e[tiny] = 1 + rng.integers(0, 2, int(tiny.sum()), dtype=np.uint64)
    m[tiny], s[tiny] = mant[tiny] - 1, sign[tiny]
    nrm = cat == 4
    e[nrm] = bias - 2 + rng.integers(0, 4, int(nrm.sum()), dtype=np.uint64)
    m[nrm], s[nrm] = mant[nrm] - 1, sign[nrm]
    e[cat == 5] = exp_inf                                       # +Inf
    e[cat == 6] = exp_inf
    s[cat == 6] = np.uint64(1) << np.uint64(tot - 1)            # -Inf
    out = s | (e << np.uint64(mb)) | m
    return out.astype(np.uint32 if tot == 32 else np.uint16)


def special_buffer(dtype: str, seed: int, rank: int, count: int) -> np.ndarray:
    """Values in the oracle's storage dtype (float32 / uint16 bf16 bits / float16)."""
    b = special_bits(dtype, seed, rank, count)
    if dtype == "f32":
        return b.view(np.float32)
    if dtype == "f16":
        return b.view(np.float16)
    return b
