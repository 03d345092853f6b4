"""Helpers for the -m gpu parity tests: device buffers from the seeded generator,
expected values from the CPU oracle (O1), element-by-element comparison."""
from __future__ import annotations

import numpy as np
import torch

from inputs import hashgen
from oracle import ring
from paper_2303_06324_b200 import occl

TORCH_DT = {"f32": torch.float32, "bf16": torch.bfloat16, "i32": torch.int32, "f16": torch.float16,
            "i64": torch.int64, "f64": torch.float64}
WAIT_S = 60.0


def bits(a):
    a = np.asarray(a)
    return a.view({8: np.uint64, 4: np.uint32, 2: np.uint16}[a.dtype.itemsize])


def to_np_bits(t: torch.Tensor) -> np.ndarray:
    t = t.detach().cpu()
    if t.dtype in (torch.bfloat16, torch.float16):
        return t.view(torch.int16).numpy().view(np.uint16)
    if t.dtype in (torch.int64, torch.float64):
        return t.numpy().view(np.uint64)
    return t.numpy().view(np.uint32)


def in_len(kind, n, count):
    return count * n if kind == "reducescatter" else count


def out_len(kind, n, count):
    return count * n if kind == "allgather" else count


def make_bufs(kind, dtype, n, count, seed, coll, device=0, inplace=False):
    """Per-rank (send, recv) device tensors; send filled by the GPU generator."""
    sends, recvs = [], []
    for r in range(n):
        if inplace:
            if kind in ("allreduce", "broadcast"):
                buf = torch.empty(count, dtype=TORCH_DT[dtype], device=device)
                occl.test_fill(buf, dtype, seed, coll, r)
                sends.append(buf)
                recvs.append(buf)
            elif kind == "allgather":
                buf = torch.full((count * n,), 0, dtype=TORCH_DT[dtype], device=device)
                s = buf[r * count:(r + 1) * count]
                occl.test_fill(s, dtype, seed, coll, r)
                sends.append(s)
                recvs.append(buf)
            else:  # reducescatter: recv == send + rank*recvcount
                buf = torch.empty(count * n, dtype=TORCH_DT[dtype], device=device)
                occl.test_fill(buf, dtype, seed, coll, r)
                sends.append(buf)
                recvs.append(buf[r * count:(r + 1) * count])
        else:
            s = torch.empty(in_len(kind, n, count), dtype=TORCH_DT[dtype], device=device)
            occl.test_fill(s, dtype, seed, coll, r)
            rv = torch.full((out_len(kind, n, count),), -7, dtype=TORCH_DT[dtype], device=device) \
                if dtype not in ("bf16", "f16") else torch.zeros(out_len(kind, n, count), dtype=TORCH_DT[dtype],
                                                                device=device)
            sends.append(s)
            recvs.append(rv)
    # inputs complete before submission (occl.h conventions): sync torch's stream
    # only -- a device-wide sync would wait for a running persistent daemon
    # (Fig. 1(c); it returns only once the daemon quits voluntarily)
    torch.cuda.current_stream(device).synchronize()
    return sends, recvs


def expected_full(kind, dtype, n, count, seed, coll, root=0, op="sum"):
    xs = ring.inputs_full(kind, dtype, n, count, seed, coll)
    return [bits(o) for o in ring.result_full(kind, dtype, xs, root=root, op=op)]


def check_full(kind, dtype, n, count, seed, coll, recvs, root=0, op="sum"):
    exp = expected_full(kind, dtype, n, count, seed, coll, root, op)
    for r in range(n):
        got = to_np_bits(recvs[r])
        if not np.array_equal(got, exp[r]):
            bad = np.nonzero(got != exp[r])[0]
            raise AssertionError(f"{kind} {dtype} n={n} count={count} rank {r}: {len(bad)} mismatches, "
                                 f"first at {bad[:8].tolist()} got {got[bad[:4]].tolist()} exp {exp[r][bad[:4]].tolist()}")


def check_sampled(kind, dtype, n, count, seed, coll, recvs, root=0, nsamples=4096, boundaries=(), op="sum"):
    """Sampled comparison at full sizes: random indices + segment/block boundaries."""
    rng = np.random.default_rng(seed ^ coll)
    for r in range(n):
        L = out_len(kind, n, count)
        idx = np.concatenate([rng.integers(0, L, nsamples), np.array([0, L - 1], dtype=np.int64),
                              np.array([b for b in boundaries if 0 <= b < L], dtype=np.int64)])
        idx = np.unique(idx)
        got = to_np_bits(recvs[r][torch.from_numpy(idx).to(recvs[r].device)])
        exp = bits(ring.expected_at(kind, dtype, n, count, seed, coll, idx, rank=r, root=root, op=op))
        if not np.array_equal(got, exp):
            bad = np.nonzero(got != exp)[0]
            raise AssertionError(f"{kind} {dtype} n={n} count={count} rank {r}: {len(bad)} sampled mismatches "
                                 f"at {idx[bad[:8]].tolist()}")


def run_collective(comms, kind, sends, recvs, coll, count, dtype, root=0, order=None, op="sum"):
    order = order if order is not None else range(len(comms))
    for r in order:
        comms[r].submit(kind, sends[r], recvs[r], coll, count, dtype, root, op=op)
    for c in comms:
        c.wait(coll, WAIT_S)
