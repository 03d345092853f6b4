"""GPU parity for the reducing functions (sum / prod / max / min)
and fp16, through the C-ABI, bit-exact against the oracle O1 on the same seeded
inputs: the register path and LL (small configuration) and the TMA staging path
with direct mode (bench configuration)."""
import numpy as np
import pytest
import torch

from inputs import hashgen

pytestmark = pytest.mark.gpu

import gpu_util as U  # noqa: E402

OPS = ["sum", "prod", "max", "min"]
DTYPES = ["f32", "bf16", "f16", "i32", "i64", "f64"]


@pytest.fixture(scope="module")
def occl_mod():
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    from paper_2303_06324_b200 import occl
    occl._lib()
    return occl


@pytest.fixture(scope="module")
def rings(occl_mod):
    made = {}

    def get(n, big):
        key = (n, big)
        if key not in made:
            cfg = dict(gridBlocks=18, sliceBytes=192 << 10, stagingTiles=5, maxColl=64) if big else \
                dict(gridBlocks=4, sliceBytes=8192, connSlots=3, slicesPerChunk=2, minBlockBytes=16384, maxColl=64)
            made[key] = occl_mod.local_group(n, 0, **cfg)
        return made[key]
    yield get
    for comms in made.values():
        occl_mod.destroy_group(comms)


@pytest.mark.parametrize("dtype", ["f16", "i64", "f64"])
def test_new_dtype_generators_match_numpy(occl_mod, dtype):
    t = torch.empty(70_001, dtype=U.TORCH_DT[dtype], device=0)
    occl_mod.test_fill(t, dtype, 0x55, 3, 2, offset=9)
    torch.cuda.synchronize()
    assert np.array_equal(U.to_np_bits(t), U.bits(hashgen.values(dtype, 0x55, 3, 2, np.arange(9, 9 + 70_001))))


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("n", [2, 3, 8])
def test_ops_small(rings, op, dtype, n):
    comms = rings(n, False)
    for ci, (kind, count) in enumerate([("allreduce", 1), ("allreduce", 1003), ("allreduce", 70_001),
                                        ("reducescatter", 777), ("reducescatter", 20_003)]):
        cid = ci
        seed = 900 + ci + 10 * OPS.index(op)
        sends, recvs = U.make_bufs(kind, dtype, n, count, seed, cid)
        U.run_collective(comms, kind, sends, recvs, cid, count, dtype, op=op)
        U.check_full(kind, dtype, n, count, seed, cid, recvs, op=op)


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("dtype", DTYPES)
def test_ops_bench_config(rings, op, dtype):
    """TMA staging path (192 KiB slices), 8 ranks, ragged sizes."""
    comms = rings(8, True)
    for ci, (kind, count) in enumerate([("allreduce", 1_500_007), ("reducescatter", 200_003)]):
        seed = 1900 + ci + 10 * OPS.index(op)
        sends, recvs = U.make_bufs(kind, dtype, 8, count, seed, 20 + ci)
        U.run_collective(comms, kind, sends, recvs, 20 + ci, count, dtype, op=op)
        U.check_full(kind, dtype, 8, count, seed, 20 + ci, recvs, op=op)


@pytest.mark.parametrize("kind", ["allgather", "broadcast"])
def test_f16_copies(rings, kind):
    for big in (False, True):
        comms = rings(8, big)
        count = 300_001 if big else 5_003
        sends, recvs = U.make_bufs(kind, "f16", 8, count, 77, 30)
        U.run_collective(comms, kind, sends, recvs, 30, count, "f16", root=5)
        U.check_full(kind, "f16", 8, count, 77, 30, recvs, root=5)


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("n", [1, 2, 3, 8])
def test_reduce_to_root(rings, op, dtype, n):
    """Reduce (NCCL ring chain root+1 -> ... -> root): the root's output is the
    oracle's fold in chain order, bit-exact; other ranks' recv buffers untouched."""
    from oracle import ring
    for big in (False, True):
        if big and n != 8:
            continue
        comms = rings(n, big)
        for ci, count in enumerate([1, 5_003, 300_001] if big else [1, 5_003]):
            root = (ci + 1) % n
            cid = 40 + ci
            seed = 3000 + ci + 10 * OPS.index(op)
            sends, recvs = U.make_bufs("allreduce", dtype, n, count, seed, cid)   # same buffer shapes
            before = [U.to_np_bits(r) for r in recvs]
            U.run_collective(comms, "reduce", sends, recvs, cid, count, dtype, root=root, op=op)
            xs = ring.inputs_full("allreduce", dtype, n, count, seed, cid)
            exp = U.bits(ring.reduce(xs, dtype, root, op))
            for r in range(n):
                got = U.to_np_bits(recvs[r])
                assert np.array_equal(got, exp if r == root else before[r]), (r, root, count)
