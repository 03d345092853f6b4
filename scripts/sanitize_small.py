#!/usr/bin/env python
"""Small end-to-end run of the daemon for compute-sanitizer (memcheck /
synccheck / racecheck): every kind, Simple and LL (with and without LL
speculation, and as LL runs), direct mode on and off, a sub-communicator, the TMA SQ fetch and
the readiness board, checked bit-exactly against the oracle.  Sizes are tiny so
the instrumented persistent kernel finishes in minutes.

  compute-sanitizer --tool memcheck python scripts/sanitize_small.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import gpu_util as U  # noqa: E402
from paper_2303_06324_b200 import occl  # noqa: E402


def main():
    torch.cuda.set_device(0)
    U.WAIT_S = 600.0
    n = 4
    runs = 0
    # (direct mode, LL limit, LL speculation): Simple + LL with direct mode, Simple-only
    # connector path, LL with speculation (abortable data-warp polling); the default
    # priority policy with the readiness board throughout
    # (and LL runs, llSpeculate = 2: data warps walking a whole slice schedule with
    # a named barrier per slice)
    for direct, llmax, spec in [(1, 64 << 10, 0), (0, 0, 0), (1, 64 << 10, 1), (1, 64 << 10, 2)]:
        comms = occl.local_group(n, 0, gridBlocks=2, maxColl=8, sliceBytes=16 << 10, stagingTiles=2,
                                 directMode=direct, llMaxBytes=llmax, llSpeculate=spec, quitIdleNs=500_000)
        try:
            for ci, (kind, dtype, count) in enumerate([("allreduce", "f32", 20_003), ("allreduce", "bf16", 3_001),
                                                       ("allgather", "i32", 5_001), ("reducescatter", "f32", 4_099),
                                                       ("broadcast", "f16", 7_777), ("allreduce", "f64", 2_049)]):
                sends, recvs = U.make_bufs(kind, dtype, n, count, 70 + ci, ci)
                U.run_collective(comms, kind, sends, recvs, ci, count, dtype, root=ci % n)
                U.check_full(kind, dtype, n, count, 70 + ci, ci, recvs, root=ci % n)
                runs += 1
            kids = [c.split([0, 2]) for c in comms[0::2]]
            sends, recvs = U.make_bufs("allreduce", "f32", 2, 10_001, 5, 7)
            for i, k in enumerate(kids):
                k.submit("allreduce", sends[i], recvs[i], 7, 10_001, "f32")
            for k in kids:
                k.wait(7, 600)
            U.check_full("allreduce", "f32", 2, 10_001, 5, 7, recvs)
            runs += 1
            for k in kids:
                k.destroy()
        finally:
            occl.destroy_group(comms)
    print(f"sanitize_small: {runs} collectives bit-exact", flush=True)


if __name__ == "__main__":
    main()
