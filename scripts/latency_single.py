"""Single-collective device latency: ONE all-reduce per daemon launch (CUDA events
around the launch: includes the launch, SQE fetch, the ring's 2(n-1) hops and the
CQE), median of 30, LL protocol vs Simple, 8 virtual ranks."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2303_06324_b200 import harness, occl  # noqa: E402

n = 8
out = []
for llmax in (64 << 10, 0):
    comms = harness.ring(n, 0, gridBlocks=18, maxColl=16, autoLaunch=0, llMaxBytes=llmax)
    for S in (4096, 65536, 262144, 1 << 20):
        count = S // 4
        bufs = harness.buffers("allreduce", "f32", n, count, comms)
        job = [(0, "allreduce", "f32", count, 0, bufs)]
        ts = sorted(harness.timed_batch(comms, job) for _ in range(30))
        row = {"proto": "ll" if llmax else "simple", "bytes": S, "median_us": ts[15] * 1e3, "p10_us": ts[3] * 1e3}
        out.append(row)
        print(json.dumps(row), flush=True)
    occl.destroy_group(comms)
