"""GPU parity cases that round 1 left open:

* send-buffer reuse / resubmission right after local completion, with direct
  read on (tests/hazard_driver.py runs the deterministic scenario in a
  subprocess under a hard timeout, because a broken build deadlocks);
* in-place collectives of every kind in the bench launch configuration (TMA
  staging ring, 192 KiB slices, direct mode + direct read);
* IEEE special values (+-0, subnormals, +-Inf) for sum / max / min in f32 /
  bf16 / f16 on both the register / LL path and the TMA path -- bit-exact,
  NaN results (Inf + -Inf) compared by class;
* occlCommInit, the bootstrap entry the north star names, through a Python
  all-gather callback (threads in one process, and one rank per process over
  torch.distributed).
"""
import os
import subprocess
import sys
import threading

import numpy as np
import pytest
import torch

from inputs import special
from oracle import ring

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

import gpu_util as U  # noqa: E402

BENCH = dict(gridBlocks=18, sliceBytes=192 << 10, connSlots=5, slicesPerChunk=2, blockThreads=608, pipeDepth=4,
             stagingTiles=6, maxColl=16)
SMALL = dict(maxColl=16, gridBlocks=4, connSlots=3, slicesPerChunk=2, sliceBytes=4096, minBlockBytes=8192)


@pytest.fixture(scope="module")
def occl_mod():
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    from paper_2303_06324_b200 import occl
    occl._lib()
    return occl


# --------------------------------------------------------------------------- hazards
# RS: a rank's completion never depends on its downstream reading its send
# buffer when its last loop's sends fit in the connector, (n-2)*spc <= K
# (here spc = 2, K = 5: n = 2, 3, 4).  AR n = 3 / 4 with spc = 1 parts: the
# final Recv passes through the downstream, so AR is safe -- kept as a check.
HAZARDS = [("reducescatter", 2, 200_000), ("reducescatter", 3, 200_000), ("reducescatter", 4, 200_000),
           ("allreduce", 2, 200_000), ("allreduce", 3, 300_000), ("allreduce", 4, 400_000)]


@pytest.mark.parametrize("mode", ["scribble", "resubmit"])
@pytest.mark.parametrize("kind,n,count", HAZARDS)
def test_send_buffer_reuse_after_wait(kind, n, count, mode):
    cmd = [sys.executable, os.path.join(ROOT, "tests", "hazard_driver.py"), "--kind", kind, "--n", str(n),
           "--count", str(count), "--mode", mode]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=90, cwd=ROOT)
    except subprocess.TimeoutExpired as e:
        pytest.fail(f"hazard scenario hung (deadlock): {kind} n={n} {mode}\n{(e.stdout or '')[-2000:]}")
    assert "HAZARD_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


# --------------------------------------------------------------------------- in place, TMA path
@pytest.mark.parametrize("n", [2, 3, 8])
def test_inplace_bench_config_all_kinds(occl_mod, n):
    """In-place (NCCL conventions) on the bench data path: parts of ~100 KiB..1.5 MiB
    per block go through the TMA staging ring, with direct mode and direct read."""
    comms = occl_mod.local_group(n, 0, **BENCH)
    try:
        for ci, (kind, dtype, count) in enumerate([("allreduce", "f32", 3_000_017), ("allreduce", "bf16", 2_000_003),
                                                   ("allgather", "f32", 400_009), ("reducescatter", "f32", 500_007),
                                                   ("reducescatter", "bf16", 300_001), ("broadcast", "f32", 2_000_001),
                                                   ("allreduce", "i32", 1_048_576)]):
            root = (ci + 1) % n
            sends, recvs = U.make_bufs(kind, dtype, n, count, 60 + ci, ci, inplace=True)
            U.run_collective(comms, kind, sends, recvs, ci, count, dtype, root)
            U.check_full(kind, dtype, n, count, 60 + ci, ci, recvs, root)
            del sends, recvs
    finally:
        occl_mod.destroy_group(comms)


# --------------------------------------------------------------------------- special values
TDT = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}


def _to_dev(arr, dtype):
    b = special.FORMATS[dtype]
    if dtype == "f32":
        return torch.from_numpy(np.ascontiguousarray(arr)).to(0)
    bits = np.ascontiguousarray(arr).view(np.int16)
    return torch.from_numpy(bits).to(0).view(TDT[dtype])


def _same(got, exp, dtype):
    """Bit-exact, except that NaN matches NaN (IEEE leaves NaN payloads open)."""
    tot = special.FORMATS[dtype][0]
    e = np.asarray(exp).view(np.uint32 if tot == 32 else np.uint16)
    ex_bits, mb = (8, 23) if dtype == "f32" else ((8, 7) if dtype == "bf16" else (5, 10))
    emask = ((1 << ex_bits) - 1) << mb
    mmask = (1 << mb) - 1
    nan_e = ((e & emask) == emask) & ((e & mmask) != 0)
    nan_g = ((got & emask) == emask) & ((got & mmask) != 0)
    ok = (got == e) | (nan_e & nan_g)
    return ok


@pytest.mark.parametrize("cfg", ["small", "bench"])
@pytest.mark.parametrize("op", ["sum", "max", "min"])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
def test_special_values(occl_mod, cfg, op, dtype):
    n = 8 if cfg == "bench" else 3
    comms = occl_mod.local_group(n, 0, **(BENCH if cfg == "bench" else SMALL))
    try:
        for ci, (kind, count) in enumerate([("allreduce", 1_000_003 if cfg == "bench" else 20_011),
                                            ("reducescatter", 200_003 if cfg == "bench" else 5_003)]):
            inl = count * n if kind == "reducescatter" else count
            xs = [special.special_buffer(dtype, 900 + ci, r, inl) for r in range(n)]
            if op in ("max", "min"):
                # max / min inputs carry no NaN by construction; Inf is kept
                pass
            sends = [_to_dev(x, dtype) for x in xs]
            recvs = [torch.zeros(count, dtype=TDT[dtype], device=0) for _ in range(n)]
            torch.cuda.current_stream().synchronize()
            for r in range(n):
                comms[r].submit(kind, sends[r], recvs[r], ci, count, dtype, op=op)
            for c in comms:
                c.wait(ci, U.WAIT_S)
            exp = ring.result_full(kind, dtype, xs, op=op)
            for r in range(n):
                got = U.to_np_bits(recvs[r])
                ok = _same(got, exp[r], dtype)
                if not ok.all():
                    bad = np.nonzero(~ok)[0]
                    xin = [U.bits(x)[bad[:4]].tolist() for x in xs] if kind == "allreduce" else None
                    raise AssertionError(f"{kind} {dtype} {op} n={n} rank {r}: {len(bad)} mismatches at "
                                         f"{bad[:4].tolist()} got {got[bad[:4]].tolist()} exp "
                                         f"{U.bits(exp[r])[bad[:4]].tolist()} inputs {xin}")
    finally:
        occl_mod.destroy_group(comms)


# --------------------------------------------------------------------------- occlCommInit
def test_comm_init_with_allgather_callback(occl_mod):
    """occlCommInit = Create + GetHandle + the caller's all-gather + Connect
    (PAPER.md:373-375): 4 ranks, one host thread each, a Python all-gather
    over a barrier as the bootstrap transport."""
    import ctypes as C
    n = 4
    slots = [None] * n
    bar = threading.Barrier(n)
    errors = []

    def ag(inp, out, nbytes, ctx):
        r = int(ctx or 0)
        slots[r] = C.string_at(inp, nbytes)
        bar.wait()
        C.memmove(out, b"".join(slots), nbytes * n)
        bar.wait()
        return 0

    cb = occl_mod.ALLGATHER(ag)
    cfg = occl_mod.occlConfigDefault(**SMALL)
    handles = [None] * n

    def init(r):
        try:
            h = C.c_void_p()
            occl_mod.check(occl_mod._lib().occlCommInit(C.byref(h), n, r, 0, cb, C.c_void_p(r), C.byref(cfg)),
                           "occlCommInit")
            handles[r] = h.value
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            bar.abort()

    ts = [threading.Thread(target=init, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    assert not errors, errors
    comms = [occl_mod.Comm(h, n, r, 0, cfg) for r, h in enumerate(handles)]
    try:
        for ci, (kind, count) in enumerate([("allreduce", 30_011), ("allgather", 1_001), ("reducescatter", 7_003)]):
            sends, recvs = U.make_bufs(kind, "f32", n, count, 70 + ci, ci)
            U.run_collective(comms, kind, sends, recvs, ci, count, "f32", order=[2, 0, 3, 1])
            U.check_full(kind, "f32", n, count, 70 + ci, ci, recvs)
    finally:
        occl_mod.destroy_group(comms)


def test_comm_init_process_group():
    """occlCommInit over torch.distributed (one rank per process, CUDA IPC between
    processes): occl.process_group() passes a dist.all_gather_object callback."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "init_driver.py"), "--world", "2"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0 and r.stdout.count("INIT_OK") == 2, r.stdout[-3000:] + r.stderr[-3000:]
