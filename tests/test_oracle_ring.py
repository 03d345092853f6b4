"""Pins for O1 (oracle/ring.py) against things other than itself (-m "not gpu").

Each pin would fail under a plausible mistake: a dropped rank, a wrong segment
owner, a reversed fold, wrong bf16 rounding, an off-by-one in the sequences.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

from inputs import hashgen
from oracle import dfce, ring

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
NS = [1, 2, 3, 4, 8]
COUNTS = [1, 7, 256, 1000, 65536]


def _bits(a):
    a = np.asarray(a)
    return a.view({8: np.uint64, 4: np.uint32, 2: np.uint16}[a.dtype.itemsize])


# ------------------------------------------------------------------ SPEC / paper examples
@pytest.mark.parametrize("ex", GOLDEN["results"], ids=lambda e: e["kind"])
def test_spec_result_examples(ex):
    xs = [np.array(v, dtype=np.int32) for v in ex["inputs"]]
    outs = ring.result_full(ex["kind"], ex["dtype"], xs)
    exp = ex["expected"]
    if len(exp) == 1:
        exp = exp * len(xs)
    for r, o in enumerate(outs):
        assert o.tolist() == exp[r], ex["cite"]


def test_spec_sequences():
    for ex in GOLDEN["sequences"]:
        if "per_rank" in ex:
            for r, prims in enumerate(ex["per_rank"]):
                got = [p for p, _ in ring.ring_sequence(ex["kind"], ex["n"], r, ex["root"], ex["inplace"])]
                assert got == prims, ex["cite"]
        else:
            got = [p for p, _ in ring.ring_sequence(ex["kind"], ex["n"], ex["rank"], ex["root"], ex["inplace"])]
            assert got == ex["prims"], ex["cite"]


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8])
def test_sequence_lengths_and_coverage(n):
    """AR 2n-1 steps, AG/RS n steps, BC 1 step; every primitive has
    a send or a recv; AR reduces every segment exactly once per rank
    and writes every segment exactly once per rank."""
    for r in range(n):
        ar = ring.ring_sequence("allreduce", n, r)
        assert len(ar) == 2 * n - 1
        assert len(ring.ring_sequence("allgather", n, r)) == n
        assert len(ring.ring_sequence("reducescatter", n, r)) == n
        assert len(ring.ring_sequence("broadcast", n, r, root=n - 1)) == 1
        for p, _ in ar:
            rv, _, _, sd = ring.PRIMS[p]
            assert rv or sd
        reduced = [q for p, q in ar if ring.PRIMS[p][1]] + [q for p, q in ar if p == "Send"]
        assert sorted(reduced) == list(range(n))
        written = [q for p, q in ar if ring.PRIMS[p][2]]
        assert sorted(written) == list(range(n))
    # neighbour consistency: what rank r sends at step j, rank r+1 receives at step j+1
    for kind in ("allreduce", "allgather", "reducescatter"):
        for r in range(n):
            s = ring.ring_sequence(kind, n, r)
            d = ring.ring_sequence(kind, n, (r + 1) % n)
            for j in range(len(s) - 1):
                if ring.PRIMS[s[j][0]][3]:
                    assert ring.PRIMS[d[j + 1][0]][0] and d[j + 1][1] == s[j][1]


# ------------------------------------------------------------------ closed forms (integers)
@pytest.mark.parametrize("n", NS)
@pytest.mark.parametrize("count", COUNTS)
def test_int_closed_form_allreduce(n, count):
    """x_r[i] = (r+1)*(i mod 97 + 1) => AR = n(n+1)/2 * (i mod 97 + 1), order-free."""
    i = np.arange(count)
    xs = [((r + 1) * (i % 97 + 1)).astype(np.int32) for r in range(n)]
    out = ring.allreduce(xs, "i32")
    assert np.array_equal(out, (n * (n + 1) // 2 * (i % 97 + 1)).astype(np.int32))


@pytest.mark.parametrize("n", NS)
def test_int_closed_form_rs_ag_bc(n):
    N = 37
    xs = [np.array([1000 * q + j for j in range(n * N)], dtype=np.int32) for q in range(n)]
    for r, o in enumerate(ring.reduce_scatter(xs, "i32")):
        j = np.arange(N)
        assert np.array_equal(o, sum(1000 * q + r * N + j for q in range(n)).astype(np.int32))
    ys = [np.array([1000 * q + j for j in range(N)], dtype=np.int32) for q in range(n)]
    ag = ring.all_gather(ys)
    assert ag.tolist() == [1000 * q + j for q in range(n) for j in range(N)]
    for root in range(n):
        assert ring.broadcast(ys, root).tolist() == [1000 * root + j for j in range(N)]


def test_int32_wraparound():
    xs = [np.array([2**31 - 1, -2**31], dtype=np.int32), np.array([1, -1], dtype=np.int32)]
    assert ring.allreduce(xs, "i32").tolist() == [-2**31, 2**31 - 1]


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_fp32_exact_small_integer_sums(n):
    """x_r[i] = r*1024 + i is exact in fp32 and so is every partial sum => order-free."""
    count = 4099
    i = np.arange(count)
    xs = [(r * 1024 + i).astype(np.float32) for r in range(n)]
    out = ring.allreduce(xs, "f32")
    assert np.array_equal(out, (sum(r * 1024 for r in range(n)) + n * i).astype(np.float32))


# ------------------------------------------------------------------ order pins (floating point)
def test_fp32_n2_is_order_free_sum():
    xs = ring.inputs_full("allreduce", "f32", 2, 5000, 11, 0)
    assert np.array_equal(_bits(ring.allreduce(xs, "f32")), _bits(xs[0] + xs[1]))


@pytest.mark.parametrize("n", [3, 4, 8])
def test_fp32_order_is_observable(n):
    """Discrimination: the ring order differs from a naive rank-0-first fold on some
    elements of random fp32 inputs, so parity tests can see a wrong order."""
    xs = ring.inputs_full("allreduce", "f32", n, 1 << 14, 5, 3)
    o = ring.allreduce(xs, "f32")
    naive = xs[0].copy()
    for q in range(1, n):
        naive = naive + xs[q]
    assert (_bits(o) != _bits(naive)).any()
    # and the ring order for segment c really starts at rank c+1 and ends at c
    L = ring.ar_segment_len(len(xs[0]), n, "f32")
    for c in range(n):
        seg = slice(c * L, (c + 1) * L)
        ref = xs[(c + 1) % n][seg].copy()
        for k in range(2, n):
            ref = ref + xs[(c + k) % n][seg]
        ref = ref + xs[c][seg]
        assert np.array_equal(_bits(o[seg]), _bits(ref))


def test_rs_equals_ar_segment_when_aligned():
    """RS_r == AR[r*N:(r+1)*N] when N is a multiple of the vector unit (the AR owner
    map then coincides with the RS segments) -- two different code paths."""
    for dtype in ("f32", "bf16", "i32"):
        n, N = 4, 1024
        xs = ring.inputs_full("reducescatter", dtype, n, N, 9, 1)
        ar = ring.allreduce(xs, dtype)
        for r, o in enumerate(ring.reduce_scatter(xs, dtype)):
            assert np.array_equal(_bits(o), _bits(ar[r * N:(r + 1) * N]))


# ------------------------------------------------------------------ bf16 arithmetic pins
def _bf16_correctly_rounded(a_bits, b_bits):
    """Independent: exact rational sum, then round to 8 significant bits, ties-to-even."""
    out = []
    for a, b in zip(a_bits.tolist(), b_bits.tolist()):
        fa = Fraction(float(np.array([a], dtype=np.uint16).astype(np.uint32).__lshift__(16).view(np.float32)[0]))
        fb = Fraction(float(np.array([b], dtype=np.uint16).astype(np.uint32).__lshift__(16).view(np.float32)[0]))
        s = fa + fb
        if s == 0:
            out.append(0.0)
            continue
        sign = -1 if s < 0 else 1
        s = abs(s)
        e = 0
        while s >= 2:
            s /= 2
            e += 1
        while s < 1:
            s *= 2
            e -= 1
        m = s * 128                       # 8 significant bits: 1.xxxxxxx
        fl = m.numerator // m.denominator
        rem = m - fl
        if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
            fl += 1
        out.append(sign * float(Fraction(fl, 128) * Fraction(2) ** e))
    return np.array(out, dtype=np.float32)


def test_bf16_add_is_correctly_rounded():
    a = hashgen.values("bf16", 1, 0, 0, np.arange(3000))
    b = hashgen.values("bf16", 1, 0, 1, np.arange(3000))
    got = ring.bf16_to_f32(ring.add(a, b, "bf16"))
    assert np.array_equal(got, _bf16_correctly_rounded(a, b))
    exact = ring.bf16_to_f32(a).astype(np.float64) + ring.bf16_to_f32(b).astype(np.float64)
    assert (exact != got.astype(np.float64)).sum() > 100      # rounding really exercised


@pytest.mark.parametrize("n", [2, 3, 8])
def test_bf16_fold_matches_torch(n):
    """Library pin: torch CPU bfloat16 addition in the same ring order."""
    xs = ring.inputs_full("allreduce", "bf16", n, 4096, 2, 2)
    o = ring.allreduce(xs, "bf16")
    ts = [torch.from_numpy(x.astype(np.int16)).view(torch.bfloat16) for x in xs]
    L = ring.ar_segment_len(4096, n, "bf16")
    ref = torch.empty_like(ts[0])
    for c in range(n):
        seg = slice(c * L, (c + 1) * L)
        acc = ts[(c + 1) % n][seg].clone()
        for k in range(2, n):
            acc = acc + ts[(c + k) % n][seg]
        ref[seg] = acc + ts[c][seg]
    assert np.array_equal(ref.view(torch.int16).numpy().view(np.uint16), o)


def test_fp32_add_matches_torch():
    xs = ring.inputs_full("allreduce", "f32", 3, 4096, 4, 4)
    o = ring.allreduce(xs, "f32")
    ts = [torch.from_numpy(x) for x in xs]
    L = ring.ar_segment_len(4096, 3, "f32")
    ref = torch.empty_like(ts[0])
    for c in range(3):
        seg = slice(c * L, (c + 1) * L)
        ref[seg] = (ts[(c + 1) % 3][seg] + ts[(c + 2) % 3][seg]) + ts[c][seg]
    assert np.array_equal(ref.numpy().view(np.uint32), o.view(np.uint32))


# ------------------------------------------------------------------ segment map
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
@pytest.mark.parametrize("n", [2, 3, 8])
def test_segment_map_cover_and_alignment(dtype, n):
    A = 16 // ring.ITEMSIZE[dtype]
    for count in (1, 7, 8, 9, 63, 1000, 65537):
        L = ring.ar_segment_len(count, n, dtype)
        assert L % A == 0 and L * n >= count and (L - A) * n < count + n * A
        owner = ring.ar_owner(np.arange(count), count, n, dtype)
        assert owner.min() >= 0 and owner.max() < n
        assert np.all(np.diff(owner) >= 0)


# ------------------------------------------------------------------ sampled == full
@pytest.mark.parametrize("kind", ring.KINDS)
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
def test_expected_at_matches_full(kind, dtype):
    n, count, seed, coll = 4, 777, 13, 5
    xs = ring.inputs_full(kind, dtype, n, count, seed, coll)
    full = ring.result_full(kind, dtype, xs, root=2)
    rng = np.random.default_rng(0)
    for r in range(n):
        idx = rng.integers(0, len(full[r]), 200)
        got = ring.expected_at(kind, dtype, n, count, seed, coll, idx, rank=r, root=2)
        assert np.array_equal(_bits(got), _bits(full[r][idx]))


# ------------------------------------------------------------------ O1 == O2 (two derivations)
@pytest.mark.parametrize("kind", ring.KINDS)
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_o1_equals_o2_execution(kind, dtype, n):
    """O2 executes the ring primitive sequences over connectors; its outputs must equal
    O1's closed-form fold bit-exactly."""
    for count, lanes, inplace in ((1, 1, False), (7, 2, False), (1000, 3, False), (2053, 2, True)):
        m = dfce.CollMeta(0, kind, dtype, count, root=min(1, n - 1), nblocks=lanes, inplace=inplace)
        cfg = dfce.SimConfig(lanes=lanes, K=3, slice_elems=16, slices_per_chunk=2,
                             spin_base=8, spin_step=1, spin_min=1, spin_cap=32, seed=n)
        sim, bufs = dfce.run_orders([m], [[0]] * n, cfg, seed=17)
        xs = ring.inputs_full(kind, dtype, n, count, 17, 0)
        exp = ring.result_full(kind, dtype, xs, root=m.root)
        for r in range(n):
            got = sim.results[(r, 0, 0)]
            assert np.array_equal(_bits(got), _bits(exp[r])), (kind, dtype, n, count, r)


# ------------------------------------------------------------------ reducing functions and f16
def _round_to_sig_bits(x: Fraction, bits: int, emin: int):
    """Exact rational -> nearest binary float with `bits` significand bits (ties to
    even), subnormals below 2^emin (IEEE gradual underflow)."""
    if x == 0:
        return Fraction(0)
    sign = -1 if x < 0 else 1
    s = abs(x)
    e = 0
    while s >= 2:
        s /= 2
        e += 1
    while s < 1:
        s *= 2
        e -= 1
    e = max(e, emin)                     # subnormal: fixed exponent, fewer bits
    q = abs(x) / Fraction(2) ** e * 2 ** (bits - 1)
    fl = q.numerator // q.denominator
    rem = q - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return sign * Fraction(fl, 2 ** (bits - 1)) * Fraction(2) ** e


@pytest.mark.parametrize("op", ["sum", "prod"])
def test_f16_ops_correctly_rounded(op):
    """f16 sum / product equal the exact rational result rounded to binary16
    (11 significant bits, subnormals below 2^-14) -- an independent derivation."""
    a = hashgen.values("f16", 3, 0, 0, np.arange(2000))
    b = hashgen.values("f16", 3, 0, 1, np.arange(2000))
    got = ring.add(a, b, "f16", op)
    for x, y, g in zip(a.tolist(), b.tolist(), got.tolist()):
        fx, fy = Fraction(x), Fraction(y)
        exact = fx + fy if op == "sum" else fx * fy
        assert Fraction(g) == _round_to_sig_bits(exact, 11, -14), (x, y, g)


def test_bf16_prod_correctly_rounded():
    a = hashgen.values("bf16", 5, 0, 0, np.arange(2000))
    b = hashgen.values("bf16", 5, 0, 1, np.arange(2000))
    got = ring.bf16_to_f32(ring.add(a, b, "bf16", "prod"))
    for x, y, g in zip(ring.bf16_to_f32(a).tolist(), ring.bf16_to_f32(b).tolist(), got.tolist()):
        assert Fraction(g) == _round_to_sig_bits(Fraction(x) * Fraction(y), 8, -126)


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16", "i32"])
@pytest.mark.parametrize("n", [2, 3, 8])
def test_max_min_are_elementwise_extrema(dtype, n):
    """max / min need no rounding: the all-reduce equals numpy's element-wise
    extremum over ranks (order-free), and reduce-scatter its segments."""
    xs = ring.inputs_full("allreduce", dtype, n, 3001, 8, 2)
    conv = (lambda v: ring.bf16_to_f32(v)) if dtype == "bf16" else (lambda v: v)
    for op, f in (("max", np.maximum.reduce), ("min", np.minimum.reduce)):
        got = conv(ring.allreduce(xs, dtype, op))
        assert np.array_equal(got, f([conv(x) for x in xs])), op


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_int_prod_closed_form(n):
    """i32 prod with rank-constant inputs r+1: n! (mod 2^32); wraps at n = 13+."""
    xs = [np.full(777, r + 1, dtype=np.int32) for r in range(n)]
    import math
    assert np.all(ring.allreduce(xs, "i32", "prod") == math.factorial(n))
    big = [np.full(5, 1 << 20, dtype=np.int32) for _ in range(2)]
    assert np.all(ring.allreduce(big, "i32", "prod") == 0)          # 2^40 mod 2^32


@pytest.mark.parametrize("n", [3, 8])
def test_fp32_prod_order_is_observable(n):
    """The ring's fold order matters for products too (rounding): the O1 result
    differs from a rank-0-first fold on some elements of random inputs."""
    xs = ring.inputs_full("allreduce", "f32", n, 4096, 6, 6)
    o = ring.allreduce(xs, "f32", "prod")
    naive = xs[0].copy()
    for x in xs[1:]:
        naive = (naive * x).astype(np.float32)
    assert (o.view(np.uint32) != naive.view(np.uint32)).sum() > 0
    assert np.allclose(o, naive, rtol=1e-5, atol=0)


@pytest.mark.parametrize("op", ["sum", "prod", "max", "min"])
@pytest.mark.parametrize("dtype", ["f32", "f16", "i32"])
def test_o1_equals_o2_execution_ops(op, dtype):
    """O2 executes the primitive sequences with the same reducing function; its
    outputs equal O1's closed form bit for bit (AR and RS, n = 3)."""
    n = 3
    for kind in ("allreduce", "reducescatter"):
        meta = dfce.CollMeta(0, kind, dtype, 70, nblocks=2, op=op)
        cfg = dfce.SimConfig(lanes=2, K=3, slice_elems=8, slices_per_chunk=2, seed=1)
        sim, bufs = dfce.run_orders([meta], [[0]] * n, cfg, seed=4)
        xs = [bufs[(r, 0, 0)][0] for r in range(n)]
        exp = ring.result_full(kind, dtype, xs, op=op)
        for r in range(n):
            assert np.array_equal(_bits(sim.results[(r, 0, 0)]), _bits(exp[r])), (kind, r)


def test_f16_generator_exact():
    """f16 inputs are exactly (m - 1024) * 2^(-10-e): no rounding in generation."""
    v = hashgen.values("f16", 1, 2, 3, np.arange(5000)).astype(np.float64)
    scaled = [Fraction(x) for x in v.tolist()]
    for x in scaled:
        assert x == 0 or any((x * 2 ** (10 + e)).denominator == 1 and abs(x * 2 ** (10 + e)) <= 1024
                             for e in range(8))


# ------------------------------------------------------------------ Reduce (ring chain to root)
@pytest.mark.parametrize("n", [1, 2, 3, 8])
def test_reduce_int_closed_form_and_root_only(n):
    xs = [np.full(1001, r + 1, dtype=np.int32) for r in range(n)]
    for root in range(n):
        out = ring.result_full("reduce", "i32", xs, root=root)
        assert np.all(out[root] == n * (n + 1) // 2)
        assert all(o is None for r, o in enumerate(out) if r != root)     # only the root is written


@pytest.mark.parametrize("n", [3, 8])
def test_reduce_fold_matches_torch_chain(n):
    """Library pin: torch float32 additions in the chain order root+1, ..., root."""
    xs = ring.inputs_full("allreduce", "f32", n, 3000, 12, 4)
    ts = [torch.from_numpy(x) for x in xs]
    seen = set()
    for root in range(n):
        acc = ts[(root + 1) % n].clone()
        for k in range(2, n + 1):
            acc = acc + ts[(root + k) % n]
        got = ring.reduce(xs, "f32", root)
        assert np.array_equal(acc.numpy().view(np.uint32), got.view(np.uint32))
        seen.add(got.tobytes())
    assert len(seen) > 1                     # the root (fold order) is observable in fp32


@pytest.mark.parametrize("op", ["sum", "prod", "max", "min"])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16", "i32"])
def test_reduce_o1_equals_o2(op, dtype):
    n = 4
    for root in (0, 3):
        meta = dfce.CollMeta(0, "reduce", dtype, 50, root=root, nblocks=2, op=op)
        cfg = dfce.SimConfig(lanes=2, K=3, slice_elems=8, slices_per_chunk=2, seed=2)
        sim, bufs = dfce.run_orders([meta], [[0]] * n, cfg, seed=5)
        xs = [bufs[(r, 0, 0)][0] for r in range(n)]
        exp = ring.reduce(xs, dtype, root, op)
        assert np.array_equal(_bits(sim.results[(root, 0, 0)]), _bits(exp))
        idx = np.arange(50)
        assert np.array_equal(_bits(ring.expected_at("reduce", dtype, n, 50, 5, 0, idx, root=root, op=op)), _bits(exp))


def test_reduce_in_random_orders_completes():
    """A reduce among all-reduces in every per-rank order (n = 2, k = 3): all
    complete, root result exact (the liveness argument covers chain primitives)."""
    metas = [dfce.CollMeta(0, "allreduce", "f32", 40), dfce.CollMeta(1, "reduce", "f32", 33, root=1),
             dfce.CollMeta(2, "allreduce", "i32", 17)]
    import itertools
    for si, orders in enumerate(itertools.product(itertools.permutations(range(3)), repeat=2)):
        cfg = dfce.SimConfig(spin_base=3, spin_step=1, spin_min=1, spin_cap=12, K=3, slice_elems=8,
                             slices_per_chunk=2, seed=si)
        sim, bufs = dfce.run_orders(metas, [list(o) for o in orders], cfg, seed=si)
        xs = [bufs[(r, 1, 0)][0] for r in range(2)]
        assert np.array_equal(_bits(sim.results[(1, 1, 0)]), _bits(ring.reduce(xs, "f32", 1)))


# ------------------------------------------------------------------ 64-bit types
def test_64bit_generators_exact_and_ops():
    """i64 wraps mod 2^64 (closed form on rank-constant inputs), f64 inputs are
    exact (m - 2^52) * 2^(-52-e) and fold in the ring order like f32."""
    n = 4
    xs = [np.full(300, (1 << 62) + r, dtype=np.int64) for r in range(n)]
    s = ring.allreduce(xs, "i64")
    assert np.all(s == np.int64(((4 << 62) + 6) % (1 << 64)))              # 2^64 wraps to 0, + 0+1+2+3
    assert np.all(ring.allreduce(xs, "i64", "max") == (1 << 62) + 3)
    v = hashgen.values("f64", 9, 1, 2, np.arange(4000))
    for x in v[:500].tolist():
        f = Fraction(x)
        assert any((f * 2 ** (52 + e)).denominator == 1 for e in range(8))
    xs = ring.inputs_full("allreduce", "f64", 8, 4096, 3, 3)
    o = ring.allreduce(xs, "f64")
    naive = xs[0].copy()
    for x in xs[1:]:
        naive = naive + x
    assert (o.view(np.uint64) != naive.view(np.uint64)).any()               # order observable
    assert np.allclose(o, naive, rtol=1e-12, atol=1e-18)


@pytest.mark.parametrize("op", ["sum", "prod", "max", "min"])
@pytest.mark.parametrize("dtype", ["i64", "f64"])
def test_o1_equals_o2_execution_64bit(op, dtype):
    n = 3
    for kind in ("allreduce", "reducescatter", "reduce"):
        meta = dfce.CollMeta(0, kind, dtype, 37, nblocks=2, op=op, root=1)
        cfg = dfce.SimConfig(lanes=2, K=3, slice_elems=4, slices_per_chunk=2, seed=1)
        sim, bufs = dfce.run_orders([meta], [[0]] * n, cfg, seed=7)
        xs = [bufs[(r, 0, 0)][0] for r in range(n)]
        exp = ring.result_full(kind, dtype, xs, root=1, op=op)
        for r in range(n):
            if exp[r] is not None:
                assert np.array_equal(_bits(sim.results[(r, 0, 0)]), _bits(exp[r])), (kind, r)


# ----------------------------------------------------------------------------- R24: signed zeros, specials
def test_ieee_max_min_signed_zero_closed_form():
    """IEEE 754-2019 maximum / minimum (reading R24): -0 < +0, in either operand
    order (numpy's np.maximum returns its FIRST operand on a tie, so it is not
    the definition)."""
    pz, nz = np.float32(0.0), np.float32(-0.0)
    for a, b in ((pz, nz), (nz, pz)):
        assert not np.signbit(ring.ieee_max(a, b)) and ring.ieee_max(a, b) == 0
        assert np.signbit(ring.ieee_min(a, b)) and ring.ieee_min(a, b) == 0
    assert np.signbit(ring.ieee_max(nz, nz)) and not np.signbit(ring.ieee_min(pz, pz))
    inf = np.float32(np.inf)
    assert ring.ieee_max(-inf, nz) == 0 and np.signbit(ring.ieee_max(-inf, nz))
    assert ring.ieee_min(inf, -inf) == -inf


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("n", [2, 3, 8])
def test_signed_zero_folds_are_order_free(dtype, n):
    """Every ring order gives the same max / min of signed zeros: +0 iff some rank
    holds +0 (max), -0 iff some rank holds -0 (min) -- checked against that
    closed form for all 2^n sign patterns; and a sum of zeros is -0 iff every
    operand is -0 (round to nearest, IEEE 754 §6.3)."""
    pats = np.array([[(m >> r) & 1 for r in range(n)] for m in range(1 << n)], dtype=bool)   # True = -0
    if dtype == "f32":
        mk = lambda neg: np.where(neg, np.float32(-0.0), np.float32(0.0)).astype(np.float32)
        sign = np.signbit
    elif dtype == "f16":
        mk = lambda neg: np.where(neg, np.float16(-0.0), np.float16(0.0)).astype(np.float16)
        sign = np.signbit
    else:
        mk = lambda neg: np.where(neg, np.uint16(0x8000), np.uint16(0)).astype(np.uint16)
        sign = lambda v: (np.asarray(v) & 0x8000) != 0
    xs = [mk(pats[:, r]) for r in range(n)]
    assert np.array_equal(sign(ring.allreduce(xs, dtype, "max")), pats.all(axis=1))
    assert np.array_equal(sign(ring.allreduce(xs, dtype, "min")), pats.any(axis=1))
    assert np.array_equal(sign(ring.allreduce(xs, dtype, "sum")), pats.all(axis=1))


def test_special_generator_covers_every_category():
    from inputs import special
    for dtype, (tot, eb, mb) in special.FORMATS.items():
        b = special.special_bits(dtype, 1, 0, 200_000).astype(np.uint64)
        e = (b >> np.uint64(mb)) & np.uint64((1 << eb) - 1)
        m = b & np.uint64((1 << mb) - 1)
        s = b >> np.uint64(tot - 1)
        top = np.uint64((1 << eb) - 1)
        assert ((e == 0) & (m == 0) & (s == 0)).any() and ((e == 0) & (m == 0) & (s == 1)).any()   # +0, -0
        assert ((e == 0) & (m != 0)).any()                                                     # subnormal
        assert ((e == top) & (m == 0) & (s == 0)).any() and ((e == top) & (m == 0) & (s == 1)).any()   # +-Inf
        assert not ((e == top) & (m != 0)).any()                                              # no NaN input
        assert np.array_equal(b, special.special_bits(dtype, 1, 0, 200_000).astype(np.uint64))  # seeded


def test_subnormal_sums_are_exact_gradual_underflow():
    """Two f32 subnormals add exactly (their sum has at most 25 significant bits
    at the subnormal exponent, so it is representable or overflows into the
    normal range exactly): the oracle does not flush to zero."""
    a = np.array([1, 0x007FFFFF, 0x00400000], dtype=np.uint32).view(np.float32)
    b = np.array([1, 1, 0x00400000], dtype=np.uint32).view(np.float32)
    got = ring.add(a, b, "f32").view(np.uint32)
    assert got.tolist() == [2, 0x00800000, 0x00800000]
    # bf16: subnormal 0x0001 + 0x0001 = 0x0002 (exact), through the f32 widening
    assert ring.add(np.array([1], np.uint16), np.array([1], np.uint16), "bf16").tolist() == [2]
