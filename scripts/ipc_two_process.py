#!/usr/bin/env python
"""Cross-process ring on ONE B200: P processes, each with R/P fused virtual ranks,
connected through CUDA IPC (occlCommGetHandle / Connect over a gloo process
group).  This exercises the multi-process path the N-GPU bench uses -- IPC-opened
peer arenas, system-scope fences, connector-only edges between processes (direct
mode is off across processes) -- on the single GPU available here.  The daemons
of the processes are separate kernels in separate CUDA contexts, time-sliced by
the GPU, so this checks correctness, not speed.

Every collective is checked bit-exactly against the oracle; exits non-zero on a
mismatch or a timeout."""
import argparse
import os
import socket
import sys
import time

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(prank, world, ranks, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=prank, world_size=world)
    torch.cuda.set_device(0)
    import gpu_util as U
    from paper_2303_06324_b200 import harness, occl
    V = ranks // world
    ok, msg = True, ""
    try:
        comms = harness.ring(ranks, 0, dist=dist, world=world, prank=prank, gridBlocks=2, maxColl=16,
                             sliceBytes=65536, quitIdleNs=200_000)
        for ci, (kind, dtype, count) in enumerate([("allreduce", "f32", 1000), ("allreduce", "bf16", 300_001),
                                                   ("allgather", "i32", 50_001), ("reducescatter", "f32", 20_003),
                                                   ("broadcast", "f32", 100_000), ("allreduce", "f32", 7)]):
            # every process builds all ranks' inputs (seeded) and submits its own ranks'
            sends, recvs = U.make_bufs(kind, dtype, ranks, count, 50 + ci, ci)
            for i, c in enumerate(comms):
                r = prank * V + i
                c.submit(kind, sends[r], recvs[r], ci, count, dtype, 1)
            t0 = time.time()
            for c in comms:
                c.wait(ci, 120)
            exp = U.expected_full(kind, dtype, ranks, count, 50 + ci, ci, root=1)
            for i in range(V):
                r = prank * V + i
                if not np.array_equal(U.to_np_bits(recvs[r]), exp[r]):
                    ok, msg = False, f"{kind} {dtype} rank {r} mismatch"
            msg += f" {kind}:{time.time() - t0:.2f}s"
        # sub-communicators across processes: groups of non-neighbouring parent
        # ranks (even / odd ranks), whose ring edges are IPC-opened on demand
        groups = [list(range(0, ranks, 2)), list(range(1, ranks, 2))]
        kids = []
        for i, c in enumerate(comms):
            r = prank * V + i
            g = groups[r % 2]
            kids.append((r, g, c.split(g)))
        count = 30_001
        xs = {}
        for r, g, k in kids:
            sends, recvs = U.make_bufs("allreduce", "f32", len(g), count, 99 + r % 2, 12)
            xs[r] = (sends, recvs, g)
            k.submit("allreduce", sends[g.index(r)], recvs[g.index(r)], 12, count, "f32")
        for r, g, k in kids:
            k.wait(12, 120)
        for r, (sends, recvs, g) in xs.items():
            exp = U.expected_full("allreduce", "f32", len(g), count, 99 + r % 2, 12)
            if not np.array_equal(U.to_np_bits(recvs[g.index(r)]), exp[g.index(r)]):
                ok, msg = False, f"split allreduce rank {r} mismatch"
        msg += " split:ok"
        dist.barrier()
        for _, _, k in kids:
            k.destroy()
        st = comms[0].stats()
        msg += f" launches={st['launches']} quits={st['quits']}"
        dist.barrier()
        occl.destroy_group(comms)
    except Exception as e:  # noqa: BLE001
        ok, msg = False, f"{type(e).__name__}: {e}"
    q.put((prank, ok, msg))
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--ranks", type=int, default=4)
    a = ap.parse_args()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=worker, args=(r, a.world, a.ranks, port, q)) for r in range(a.world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for r in sorted(res):
        print(r, flush=True)
    sys.exit(0 if all(ok for _, ok, _ in res) else 1)


if __name__ == "__main__":
    main()
