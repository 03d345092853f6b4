"""Workload recipes for BASELINE.json configs C1..C4.

Pure data + seeded permutations; no arithmetic of the method lives here.

* C1: 2 ranks, 2 fp32 all-reduces of 1024 elements, opposite per-rank orders.
* C2: single-collective size sweep 4 KiB .. 1 GiB (nccl-tests conventions).
* C3: 64 mixed collectives (AR/AG/RS/BC, fp32/bf16, 1-64 MiB log-uniform),
      independent random per-rank orders.
* C4: data-parallel gradient buckets shaped like ResNet-50 / BERT-large
      (25 MiB buckets) and the paper's 161 per-tensor ResNet-50 all-reduces
      ("161 all-reduces ... between 256B and 9MB").
* Deadlock campaign: k all-reduces of 256 B .. 1 MiB in
  independent random per-rank orders.
"""
from __future__ import annotations

import math
import random
from dataclasses import dataclass

MiB = 1 << 20

# torchvision resnet50() parameter element counts in registration order
# (161 tensors, 25,557,032 parameters; 256 B .. 9 MiB as fp32).
RESNET50_PARAM_NUMEL = [
    9408, 64, 64, 4096, 64, 64, 36864, 64, 64, 16384, 256, 256, 16384, 256, 256, 16384, 64, 64,
    36864, 64, 64, 16384, 256, 256, 16384, 64, 64, 36864, 64, 64, 16384, 256, 256, 32768, 128,
    128, 147456, 128, 128, 65536, 512, 512, 131072, 512, 512, 65536, 128, 128, 147456, 128, 128,
    65536, 512, 512, 65536, 128, 128, 147456, 128, 128, 65536, 512, 512, 65536, 128, 128, 147456,
    128, 128, 65536, 512, 512, 131072, 256, 256, 589824, 256, 256, 262144, 1024, 1024, 524288,
    1024, 1024, 262144, 256, 256, 589824, 256, 256, 262144, 1024, 1024, 262144, 256, 256, 589824,
    256, 256, 262144, 1024, 1024, 262144, 256, 256, 589824, 256, 256, 262144, 1024, 1024, 262144,
    256, 256, 589824, 256, 256, 262144, 1024, 1024, 262144, 256, 256, 589824, 256, 256, 262144,
    1024, 1024, 524288, 512, 512, 2359296, 512, 512, 1048576, 2048, 2048, 2097152, 2048, 2048,
    1048576, 512, 512, 2359296, 512, 512, 1048576, 2048, 2048, 1048576, 512, 512, 2359296, 512,
    512, 1048576, 2048, 2048, 2048000, 1000,
]
RESNET50_PARAMS = 25_557_032
BERT_LARGE_PARAMS = 335_141_888
BUCKET_BYTES = 25 * MiB


@dataclass(frozen=True)
class Coll:
    """One registered collective of a workload (identical on every rank)."""
    coll_id: int
    kind: str          # "allreduce" | "allgather" | "reducescatter" | "broadcast"
    dtype: str         # "f32" | "bf16" | "i32"
    count: int         # AR/BC: elements per rank; AG: sendcount; RS: recvcount
    root: int = 0


def c1():
    """C1: 2 ranks, 2 fp32 ARs of 1024 elements, rank 0 order [0,1], rank 1 [1,0]."""
    colls = [Coll(0, "allreduce", "f32", 1024), Coll(1, "allreduce", "f32", 1024)]
    return colls, [[0, 1], [1, 0]]


def c2_sizes(min_bytes: int = 4096, max_bytes: int = 1 << 30):
    """C2: nccl-tests sweep, factor 2 (19 points for 4 KiB .. 1 GiB)."""
    out, s = [], min_bytes
    while s <= max_bytes:
        out.append(s)
        s *= 2
    return out


def c3(nranks: int = 8, ncoll: int = 64, seed: int = 0, scale: int = 1,
       min_bytes: int = 1 * MiB, max_bytes: int = 64 * MiB):
    """C3: mixed collectives, sizes log-uniform in [min,max] rounded to 4 KiB (÷scale),
    kind uniform over AR/AG/RS/BC, dtype 50/50 fp32/bf16; per-rank independent
    permutations seeded with seed ^ rank."""
    rng = random.Random(seed)
    kinds = ["allreduce", "allgather", "reducescatter", "broadcast"]
    colls = []
    for cid in range(ncoll):
        kind = rng.choice(kinds)
        dtype = rng.choice(["f32", "bf16"])
        nbytes = math.exp(rng.uniform(math.log(min_bytes), math.log(max_bytes)))
        nbytes = max(4096, int(nbytes) // 4096 * 4096) // scale
        item = 4 if dtype == "f32" else 2
        total = max(item * nranks, nbytes)
        if kind in ("allgather", "reducescatter"):
            count = max(1, total // item // nranks)   # nccl-tests: S = total output/input
        else:
            count = max(1, total // item)
        root = rng.randrange(nranks) if kind == "broadcast" else 0
        colls.append(Coll(cid, kind, dtype, count, root))
    orders = []
    for r in range(nranks):
        o = list(range(ncoll))
        random.Random(seed ^ (0x9E3779B9 * (r + 1))).shuffle(o)
        orders.append(o)
    return colls, orders


def resnet50_buckets(bucket_bytes: int = BUCKET_BYTES):
    """C4: ResNet-50 fp32 gradients grouped into 25 MiB buckets (reverse layer order,
    as DDP does) -> list of element counts."""
    return _bucketize(list(reversed(RESNET50_PARAM_NUMEL)), bucket_bytes)


def bert_large_buckets(bucket_bytes: int = BUCKET_BYTES):
    """C4: BERT-large 335,141,888 fp32 params as 25 MiB buckets (51 x 25 MiB + tail)."""
    per = bucket_bytes // 4
    full, tail = divmod(BERT_LARGE_PARAMS, per)
    return [per] * full + ([tail] if tail else [])


def _bucketize(numels, bucket_bytes):
    out, cur = [], 0
    for n in numels:
        cur += n
        if cur * 4 >= bucket_bytes:
            out.append(cur)
            cur = 0
    if cur:
        out.append(cur)
    return out


def c4(model: str = "resnet50", nranks: int = 8, seed: int = 0, per_tensor: bool = False):
    """C4: one DP iteration's gradient all-reduces; per-rank randomized arrival order."""
    if model == "resnet50":
        counts = list(reversed(RESNET50_PARAM_NUMEL)) if per_tensor else resnet50_buckets()
    elif model == "bert-large":
        counts = bert_large_buckets()
    else:
        raise ValueError(model)
    colls = [Coll(i, "allreduce", "f32", c) for i, c in enumerate(counts)]
    orders = []
    for r in range(nranks):
        o = list(range(len(colls)))
        random.Random((seed << 8) ^ r).shuffle(o)
        orders.append(o)
    return colls, orders


def deadlock_trial(nranks: int = 8, k: int = 8, seed: int = 0,
                   min_bytes: int = 256, max_bytes: int = 1 * MiB):
    """Deadlock campaign trial: k fp32 ARs of 256 B .. 1 MiB (log-uniform),
    independent random permutation per rank."""
    rng = random.Random(seed)
    colls = []
    for cid in range(k):
        nbytes = math.exp(rng.uniform(math.log(min_bytes), math.log(max_bytes)))
        colls.append(Coll(cid, "allreduce", "f32", max(1, int(nbytes) // 4)))
    orders = []
    for r in range(nranks):
        o = list(range(k))
        rng.shuffle(o)
        orders.append(o)
    return colls, orders


def pairwise_reversed_orders(nranks: int, k: int):
    """PAPER.md:737 'different orders pairwise' read as adjacent rank pairs reversed
    (SPEC.md:548): even ranks ascending, odd ranks descending."""
    return [list(range(k)) if r % 2 == 0 else list(reversed(range(k))) for r in range(nranks)]


def arrival_delays(nranks: int, nitems: int, mean_s: float, seed: int):
    """Per-rank inter-arrival gaps (seconds) ~ Exp(mean_s), independent per rank:
    rank r waits delays[r][k] before its k-th submission (C3 / C4 live arrival,
    VERDICT r01 next #2).  Seeded; pure data."""
    out = []
    for r in range(nranks):
        rng = random.Random((seed * 1_000_003) ^ (0x5DEECE66D * (r + 1)))
        out.append([rng.expovariate(1.0 / mean_s) if mean_s > 0 else 0.0 for _ in range(nitems)])
    return out


def iteration_orders(nranks: int, nitems: int, seed: int, iteration: int):
    """Independent random per-rank permutation for one DP iteration (C4)."""
    orders = []
    for r in range(nranks):
        o = list(range(nitems))
        random.Random((seed << 20) ^ (iteration << 8) ^ r).shuffle(o)
        orders.append(o)
    return orders
