"""GPU parity: the CUDA daemon path (through the C-ABI) vs the CPU oracle O1,
element by element, bit-exact for i32 / f32 / bf16 (the ring
order is reproduced, so no tolerance is needed).  Virtual ranks: several
communicators in one process on one B200, each with its own daemon kernel."""
import numpy as np
import pytest
import torch

from inputs import hashgen
from oracle import ring

pytestmark = pytest.mark.gpu

import gpu_util as U  # noqa: E402

SMALL = dict(maxColl=16, gridBlocks=4, connSlots=3, slicesPerChunk=2, sliceBytes=4096,
             minBlockBytes=8192, quitIdleNs=50_000_000)


@pytest.fixture(scope="module")
def occl_mod():
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    from paper_2303_06324_b200 import occl
    occl._lib()
    return occl


_groups = {}


def group(occl_mod, n, **kw):
    key = (n, tuple(sorted(kw.items())))
    if key not in _groups:
        cfg = dict(SMALL)
        cfg.update(kw)
        _groups[key] = occl_mod.local_group(n, 0, **cfg)
    return _groups[key]


@pytest.fixture(scope="module", autouse=True)
def _teardown():
    yield
    for comms in _groups.values():
        for c in comms:
            c.destroy()
    _groups.clear()


def test_generator_matches_numpy(occl_mod):
    for dtype in ("f32", "bf16", "i32"):
        t = torch.empty(100_003, dtype=U.TORCH_DT[dtype], device=0)
        occl_mod.test_fill(t, dtype, 0x1234567, 7, 3, offset=11)
        torch.cuda.synchronize()
        exp = U.bits(hashgen.values(dtype, 0x1234567, 7, 3, np.arange(11, 11 + 100_003)))
        assert np.array_equal(U.to_np_bits(t), exp), dtype


@pytest.mark.parametrize("kind", ring.KINDS)
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("proto", ["ll", "ll-spec", "ll-run", "simple"])
def test_parity_small(occl_mod, kind, dtype, n, proto):
    """LL (flags inside 16-B lines) for small per-block parts -- with the data
    warps polling the lines themselves (ll-spec, cfg.llSpeculate = 1), after the
    control lane saw the slice's last line (ll, 0), or walking the whole slice
    schedule as an LL run (ll-run, 2, the default) -- and Simple (head / credit
    flags + release fence) when LL is disabled."""
    mode = {"ll": 0, "ll-spec": 1, "ll-run": 2, "simple": 2}[proto]
    comms = group(occl_mod, n, llMaxBytes=0 if proto == "simple" else (64 << 10), llSpeculate=mode)
    for ci, count in enumerate([1, 7, 256, 1000, 4099, 65536]):
        root = (ci + 1) % n
        seed = 1000 + ci
        coll = ci
        sends, recvs = U.make_bufs(kind, dtype, n, count, seed, coll)
        U.run_collective(comms, kind, sends, recvs, coll, count, dtype, root)
        U.check_full(kind, dtype, n, count, seed, coll, recvs, root)


@pytest.mark.parametrize("kind", ring.KINDS)
@pytest.mark.parametrize("n", [2, 3, 8])
def test_parity_inplace(occl_mod, kind, n):
    comms = group(occl_mod, n)
    for ci, count in enumerate([5, 1000, 70_001]):
        dtype = ["f32", "bf16", "i32"][ci]
        sends, recvs = U.make_bufs(kind, dtype, n, count, 77 + ci, 9, inplace=True)
        U.run_collective(comms, kind, sends, recvs, 9, count, dtype, root=n - 1)
        U.check_full(kind, dtype, n, count, 77 + ci, 9, recvs, root=n - 1)


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("llmax,spec", [(0, 0), (1 << 20, 0), (1 << 20, 1), (1 << 20, 2)])
def test_parity_1mib_multiblock(occl_mod, n, llmax, spec):
    """1 Mi elements: many loops and slices per block, ragged tail, all blocks;
    Simple, and LL forced for every size (many LL slices and loops), with and
    without LL speculation."""
    comms = group(occl_mod, n, llMaxBytes=llmax, llSpeculate=spec)
    for kind in ring.KINDS:
        count = (1 << 20) + 13
        sends, recvs = U.make_bufs(kind, "f32", n, count, 5, 3)
        U.run_collective(comms, kind, sends, recvs, 3, count, "f32", root=1 % n)
        U.check_full(kind, "f32", n, count, 5, 3, recvs, root=1 % n)


def test_resubmission_same_id_new_buffers(occl_mod):
    """An id is resubmitted with new buffers / sizes after completing;
    connector sequence numbers carry over."""
    comms = group(occl_mod, 4)
    for it, (kind, count) in enumerate([("allreduce", 5000), ("allgather", 333), ("allreduce", 77),
                                        ("reducescatter", 1024), ("broadcast", 9999)] * 2):
        sends, recvs = U.make_bufs(kind, "f32", 4, count, 300 + it, 11)
        U.run_collective(comms, kind, sends, recvs, 11, count, "f32", root=it % 4)
        U.check_full(kind, "f32", 4, count, 300 + it, 11, recvs, root=it % 4)


def test_count_zero_completes_immediately(occl_mod):
    comms = group(occl_mod, 2)
    x = torch.zeros(4, device=0)
    for c in comms:
        c.all_reduce(x, x, 12, count=0)
        assert c.test(12)


def test_errors(occl_mod):
    comms = group(occl_mod, 2)
    x = torch.zeros(1 << 16, device=0)
    with pytest.raises(occl_mod.OcclError) as e:
        comms[0].all_reduce(x, x, 10_000)
    assert e.value.code == occl_mod.occlRegistryFull
    with pytest.raises(occl_mod.OcclError) as e:
        comms[0].broadcast(x, x, 5, 1)
    assert e.value.code == occl_mod.occlInvalidArgument
    with pytest.raises(occl_mod.OcclError) as e:
        comms[0].wait(13)
    assert e.value.code == occl_mod.occlUnknownId
    # duplicate submission of an in-flight id
    comms[0].all_reduce(x, x, 14)
    with pytest.raises(occl_mod.OcclError) as e:
        comms[0].all_reduce(x, x, 14)
    assert e.value.code == occl_mod.occlDuplicateSubmit
    comms[1].all_reduce(x, x, 14)
    for c in comms:
        c.wait(14, U.WAIT_S)
