"""O1 -- closed-form collective results in the ring's reduction order.  TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module.  Shares no code with paper_2303_06324_b200/.

What the method computes (§2.3 "The Preemption Opportunity"):
the commonly used collectives (all-reduce, all-gather, reduce-scatter, broadcast)
are executed as per-rank *primitive sequences* of the NCCL Ring algorithm with the
Simple protocol (§5 "Benchmarks").  The result of each collective is
its textbook definition; in floating point the reduction ORDER is the ring's:

  AR  out[i]        = ((x_{c+1}[i] (+) x_{c+2}[i]) (+) ... (+) x_{c-1}[i]) (+) x_c[i],
                      c = owner(i) = floor(i / L),  L = ceil(ceil(N/n)/A)*A,
                      A = 16 / sizeof(T) (one 128-bit vector)  [DESIGN.md reading R6]
  RS  out_r[j]      = the same fold with c = r over x_q[r*N + j]
  AG  out[q*N + j]  = x_q[j]
  BC  out           = x_root
  RED out_root      = ((x_{root+1} (+) x_{root+2}) (+) ...) (+) x_root   (recv buffers of the
                      other ranks are not written; NCCL's ring Reduce chain)
  n = 1             => copy

Indices are mod n.  (+) is the collective's reducing function (PAPER.md:306
"a specified reducing function"): sum (default), prod, max or min, per dtype
(readings R7 / R22):
  i32  : (a + b) mod 2^32, (a * b) mod 2^32, signed max / min
  f32  : IEEE-754 binary32 add / multiply, round-to-nearest-even (numpy float32)
  bf16 : RNE_bf16(float32(a) op float32(b))  (= the correctly rounded bf16 result:
         a bf16 product is exact in f32, and for sums double rounding is innocuous
         since 24 >= 2*8 + 2)
  f16  : RNE_f16(float32(a) op float32(b))   (same argument, 24 >= 2*11 + 2)
  i64  : two's-complement wrap (sum, prod), signed max / min
  f64  : IEEE-754 binary64, round-to-nearest-even (numpy float64)
  max / min are exact (no rounding); -0 < +0 (IEEE 754-2019 maximum / minimum,
  reading R24); their inputs carry no NaN.  Sums may meet +-Inf and produce
  NaN (Inf + -Inf); NaN payloads are unspecified by IEEE 754, so tests compare
  NaN results by class, every other result bit for bit.

Where the paper is silent (segment map, operand order, bf16 partial precision)
the readings are SURVEY.md §8(c) Q6/Q7, listed in DESIGN.md.
"""
from __future__ import annotations

import numpy as np

from inputs import hashgen

KINDS = ("allreduce", "allgather", "reducescatter", "broadcast")
ALL_KINDS = KINDS + ("reduce",)
ITEMSIZE = {"i32": 4, "f32": 4, "bf16": 2, "f16": 2, "i64": 8, "f64": 8}
OPS = ("sum", "prod", "max", "min")


# ----------------------------------------------------------------------------- (+) per dtype
def bf16_rne(f32: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit pattern, round to nearest even (finite inputs)."""
    u = np.asarray(f32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    return ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)


def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def ieee_max(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """IEEE 754-2019 maximum of non-NaN operands (reading R24): the
    larger value, where -0 compares less than +0 (so max(-0, +0) = +0 in either
    operand order; numpy's np.maximum returns its first operand on ties)."""
    x, y = np.asarray(x), np.asarray(y)
    r = np.where(x > y, x, y)
    z = (x == 0) & (y == 0)
    return np.where(z, np.where(np.signbit(x) & np.signbit(y), x, np.abs(x)), r)


def ieee_min(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """IEEE 754-2019 minimum of non-NaN operands (reading R24): -0 < +0."""
    x, y = np.asarray(x), np.asarray(y)
    r = np.where(x < y, x, y)
    z = (x == 0) & (y == 0)
    return np.where(z, np.where(np.signbit(x) | np.signbit(y), -np.abs(x), np.abs(x)), r)


def _f32_op(x: np.ndarray, y: np.ndarray, op: str) -> np.ndarray:
    """The reducing function on float32 operands (IEEE, round to nearest even)."""
    if op == "sum":
        return (x + y).astype(np.float32)
    if op == "prod":
        return (x * y).astype(np.float32)
    if op == "max":
        return ieee_max(x, y)
    if op == "min":
        return ieee_min(x, y)
    raise ValueError(op)


def add(a: np.ndarray, b: np.ndarray, dtype: str, op: str = "sum") -> np.ndarray:
    """Elementwise reducing function (+) ("reduces data ... with a
    specified reducing function"): sum, prod, max or min."""
    if dtype == "i32":
        ua, ub = np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32)
        if op == "sum":
            return (ua + ub).view(np.int32)
        if op == "prod":
            return (ua * ub).view(np.int32)            # mod 2^32 (two's complement product)
        ia, ib = np.asarray(a).view(np.int32), np.asarray(b).view(np.int32)
        if op == "max":
            return np.maximum(ia, ib)
        if op == "min":
            return np.minimum(ia, ib)
        raise ValueError(op)
    if dtype == "f32":
        return _f32_op(np.asarray(a, dtype=np.float32), np.asarray(b, dtype=np.float32), op)
    if dtype == "bf16":
        return bf16_rne(_f32_op(bf16_to_f32(a), bf16_to_f32(b), op))
    if dtype == "f16":
        return _f32_op(np.asarray(a, dtype=np.float16).astype(np.float32),
                       np.asarray(b, dtype=np.float16).astype(np.float32), op).astype(np.float16)
    if dtype == "i64":
        ua, ub = np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64)
        if op == "sum":
            return (ua + ub).view(np.int64)            # mod 2^64
        if op == "prod":
            return (ua * ub).view(np.int64)
        ia, ib = np.asarray(a).view(np.int64), np.asarray(b).view(np.int64)
        return np.maximum(ia, ib) if op == "max" else np.minimum(ia, ib)
    if dtype == "f64":
        x, y = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
        if op == "sum":
            return x + y
        if op == "prod":
            return x * y
        return ieee_max(x, y) if op == "max" else ieee_min(x, y)
    raise ValueError(dtype)


def ring_fold(parts_in_ring_order, dtype: str, op: str = "sum") -> np.ndarray:
    """Left fold: ((p0 (+) p1) (+) p2) ... -- p0 = x_{c+1}, ..., last = x_c."""
    acc = np.array(parts_in_ring_order[0], copy=True)
    for p in parts_in_ring_order[1:]:
        acc = add(acc, p, dtype, op)
    return acc


def fold_order(c: int, n: int):
    """Ranks whose inputs are folded for a segment owned by c: c+1, c+2, ..., c-1, c."""
    return [(c + k) % n for k in range(1, n)] + [c % n]


# ----------------------------------------------------------------------------- segment map
def vec_elems(dtype: str) -> int:
    return 16 // ITEMSIZE[dtype]


def ar_segment_len(count: int, n: int, dtype: str) -> int:
    """L = ceil(ceil(N/n)/A)*A (segment-first map, reading R6)."""
    a = vec_elems(dtype)
    per = -(-count // n)
    return -(-per // a) * a


def ar_owner(i, count: int, n: int, dtype: str):
    """owner(i) = floor(i / L)."""
    return np.asarray(i) // ar_segment_len(count, n, dtype)


# ----------------------------------------------------------------------------- full results
def allreduce(xs, dtype: str, op: str = "sum") -> np.ndarray:
    """AR result (identical on every rank) for per-rank inputs xs[r] (length N each)."""
    n = len(xs)
    count = len(xs[0])
    if n == 1:
        return np.array(xs[0], copy=True)
    L = ar_segment_len(count, n, dtype)
    out = np.empty_like(np.asarray(xs[0]))
    for c in range(n):
        lo, hi = min(c * L, count), min((c + 1) * L, count)
        if lo >= hi:
            continue
        out[lo:hi] = ring_fold([xs[q][lo:hi] for q in fold_order(c, n)], dtype, op)
    return out


def reduce_scatter(xs, dtype: str, op: str = "sum"):
    """RS: xs[r] has n*N elements; returns [out_0, ..., out_{n-1}], out_r has N."""
    n = len(xs)
    N = len(xs[0]) // n
    if n == 1:
        return [np.array(xs[0][:N], copy=True)]
    return [ring_fold([xs[q][r * N:(r + 1) * N] for q in fold_order(r, n)], dtype, op) for r in range(n)]


def all_gather(xs) -> np.ndarray:
    """AG: out[q*N + j] = x_q[j] (identical on every rank)."""
    return np.concatenate([np.asarray(x) for x in xs])


def broadcast(xs, root: int) -> np.ndarray:
    return np.array(xs[root], copy=True)


def reduce(xs, dtype: str, root: int, op: str = "sum") -> np.ndarray:
    """Reduce to root: the chain root+1 -> root+2 -> ... -> root, folded in that order."""
    n = len(xs)
    if n == 1:
        return np.array(xs[0], copy=True)
    return ring_fold([xs[q] for q in fold_order(root, n)], dtype, op)


# ----------------------------------------------------------------------------- sampled results
def expected_at(kind: str, dtype: str, n: int, count: int, seed: int, coll: int,
                idx, rank: int = 0, root: int = 0, op: str = "sum") -> np.ndarray:
    """Expected output values at output indices ``idx`` of rank ``rank``, computing
    only the needed inputs from the counter-based generator (inputs.hashgen).

    count: AR/BC elements per rank; AG sendcount (output has n*count); RS recvcount.
    """
    idx = np.asarray(idx, dtype=np.int64)
    val = lambda q, ii: hashgen.values(dtype, seed, coll, q, ii.astype(np.uint64))
    if kind == "allgather":
        q = idx // count
        out = np.empty(idx.shape, dtype=hashgen.NP_STORAGE[dtype])
        for src in range(n):
            m = q == src
            out[m] = val(src, idx[m] - src * count)
        return out
    if kind == "reduce" and n > 1:
        return ring_fold([val(q, idx) for q in fold_order(root, n)], dtype, op)
    if kind in ("broadcast", "reduce") or n == 1:
        if kind == "reducescatter":
            return val(0, idx)
        return val(root if kind == "broadcast" else 0, idx)
    if kind == "allreduce":
        owner = ar_owner(idx, count, n, dtype)
        out = np.empty(idx.shape, dtype=hashgen.NP_STORAGE[dtype])
        for c in range(n):
            m = owner == c
            if m.any():
                out[m] = ring_fold([val(q, idx[m]) for q in fold_order(c, n)], dtype, op)
        return out
    if kind == "reducescatter":
        src = rank * count + idx
        return ring_fold([val(q, src) for q in fold_order(rank, n)], dtype, op)
    raise ValueError(kind)


def inputs_full(kind: str, dtype: str, n: int, count: int, seed: int, coll: int):
    """Materialised per-rank inputs for a collective (input length per nccl conventions)."""
    inlen = count * n if kind == "reducescatter" else count
    return [hashgen.buffer(dtype, seed, coll, r, inlen) for r in range(n)]


def result_full(kind: str, dtype: str, xs, root: int = 0, op: str = "sum"):
    """Per-rank expected outputs for materialised inputs xs."""
    n = len(xs)
    if kind == "allreduce":
        o = allreduce(xs, dtype, op)
        return [o] * n
    if kind == "reducescatter":
        return reduce_scatter(xs, dtype, op)
    if kind == "allgather":
        o = all_gather(xs)
        return [o] * n
    if kind == "broadcast":
        o = broadcast(xs, root)
        return [o] * n
    if kind == "reduce":
        return [reduce(xs, dtype, root, op) if r == root else None for r in range(n)]   # root only
    raise ValueError(kind)


# ----------------------------------------------------------------------------- ring sequences
# Primitive vocabulary (§2.3).  Each primitive is the
# fused action set: (recv, reduce, copy-to-recvbuf, send).
PRIMS = {
    "Send":               (False, False, False, True),
    "Recv":               (True,  False, True,  False),
    "CopySend":           (False, False, True,  True),
    "RecvCopySend":       (True,  False, True,  True),
    "RecvReduceSend":     (True,  True,  False, True),
    "RecvReduceCopy":     (True,  True,  True,  False),
    "RecvReduceCopySend": (True,  True,  True,  True),
    "Copy":               (False, False, True,  False),   # n == 1 local copy (reading R18)
}


def ring_sequence(kind: str, n: int, r: int, root: int = 0, inplace: bool = False):
    """Per-rank primitive sequence of one loop, as (primitive, segment) pairs.

    NCCL Ring/Simple sequences; segment
    selectors are the reading of SURVEY.md §8(c) (R5).  Ring: rank r
    sends to (r+1) mod n and receives from (r-1) mod n.
    """
    if n == 1:
        return [("Copy", 0)]
    m = lambda x: x % n
    if kind == "allreduce":
        seq = [("Send", m(r - 1))]
        seq += [("RecvReduceSend", m(r - 1 - j)) for j in range(1, n - 1)]
        seq += [("RecvReduceCopySend", m(r))]
        seq += [("RecvCopySend", m(r - (j - n + 1))) for j in range(n, 2 * n - 2)]
        seq += [("Recv", m(r + 1))]
        return seq
    if kind == "reducescatter":
        seq = [("Send", m(r - 1))]
        seq += [("RecvReduceSend", m(r - 1 - j)) for j in range(1, n - 1)]
        seq += [("RecvReduceCopy", m(r))]
        return seq
    if kind == "allgather":
        seq = [("CopySend", m(r))]
        seq += [("RecvCopySend", m(r - j)) for j in range(1, n - 1)]
        seq += [("Recv", m(r + 1))]
        return seq
    if kind == "broadcast":
        pos = m(r - root)
        if pos == 0:
            return [("Send" if inplace else "CopySend", 0)]
        if pos == n - 1:
            return [("Recv", 0)]
        return [("RecvCopySend", 0)]
    if kind == "reduce":
        # chain root+1 -> ... -> root (NCCL ring Reduce); one segment
        pos = m(r - root - 1)
        if pos == 0:
            return [("Send", 0)]
        if pos == n - 1:
            return [("RecvReduceCopy", 0)]
        return [("RecvReduceSend", 0)]
    raise ValueError(kind)
