#!/usr/bin/env python
"""occlCommInit across processes (tests/test_gpu_hazards.py): `world` processes,
one rank each, bootstrap all-gather = torch.distributed (gloo) all_gather_object
called from inside occlCommInit; every collective kind checked bit-exactly
against the oracle.  All processes share GPU 0 (CUDA IPC between them)."""
import argparse
import os
import socket
import sys

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


def worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import gpu_util as U
    from paper_2303_06324_b200 import occl
    ok, msg = True, ""
    try:
        comm = occl.process_group(device=0, gridBlocks=2, maxColl=8, sliceBytes=65536, quitIdleNs=200_000)
        for ci, (kind, dtype, count) in enumerate([("allreduce", "f32", 100_003), ("allgather", "bf16", 5_001),
                                                   ("reducescatter", "i32", 20_003), ("broadcast", "f32", 9_999)]):
            sends, recvs = U.make_bufs(kind, dtype, world, count, 30 + ci, ci)
            comm.submit(kind, sends[rank], recvs[rank], ci, count, dtype, 1 % world)
            comm.wait(ci, 120)
            exp = U.expected_full(kind, dtype, world, count, 30 + ci, ci, root=1 % world)
            if not np.array_equal(U.to_np_bits(recvs[rank]), exp[rank]):
                ok, msg = False, f"{kind} mismatch"
        dist.barrier()
        comm.destroy()
    except Exception as e:  # noqa: BLE001
        ok, msg = False, f"{type(e).__name__}: {e}"
    q.put((rank, ok, msg))
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    a = ap.parse_args()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=worker, args=(r, a.world, port, q)) for r in range(a.world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=280) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for r, ok, msg in sorted(res):
        print("INIT_OK" if ok else "INIT_FAIL", r, msg, flush=True)
    sys.exit(0 if all(ok for _, ok, _ in res) else 1)


if __name__ == "__main__":
    main()
