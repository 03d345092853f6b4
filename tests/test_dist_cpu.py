"""N>1 host-side logic on CPU (gloo, world_size 2): the ring of R ranks spread over
processes (R/world consecutive ranks per process) exchanges handles with
torch.distributed and every process connects its communicators with the full
rank-ordered handle list.  The C-ABI calls are replaced by recorders (no GPU)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, ranks_total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2303_06324_b200 import harness, occl
    created, connected, fused = [], [], []
    occl.occlConfigDefault = lambda **kw: dict(kw)
    occl.occlCommCreate = lambda n, r, dev, cfg: ("comm", n, r)
    occl.occlCommGetHandle = lambda h: f"handle-of-rank-{h[2]}".encode()
    occl.occlCommConnect = lambda h, handles: connected.append((h[2], list(handles)))
    occl.occlCommFuse = lambda comms: fused.append([c.rank for c in comms])
    comms = harness.ring(ranks_total, 0, dist=dist, world=world, prank=rank)
    q.put((rank, [c.rank for c in comms], connected, fused))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ranks_total", [2, 8])
def test_ring_handle_exchange_gloo(ranks_total):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ranks_total, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(world):
        r, ranks, connected, fused = q.get(timeout=120)
        res[r] = (ranks, connected, fused)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    V = ranks_total // world
    expect = [f"handle-of-rank-{i}".encode() for i in range(ranks_total)]
    for r in range(world):
        ranks, connected, fused = res[r]
        assert ranks == list(range(r * V, (r + 1) * V))
        assert [c[0] for c in connected] == ranks
        for _, handles in connected:
            assert handles == expect                      # full ring, rank order
        assert fused == ([ranks] if V > 1 else [])
