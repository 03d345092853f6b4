"""Thin ctypes binding of include/occl.h (argument marshalling only).

Every step of the collective path runs inside libocclb200.so (host runtime +
sm_100a daemon kernel).  There is no fallback: importing this module on a box
without the built library raises, and every call checks its occlResult_t.

Names mirror the C-ABI (occlCommCreate, occlAllReduce, occlWait, ...); a small
``Comm`` convenience class accepts torch tensors (or raw device pointers) and
``local_group`` / ``process_group`` build rings of virtual ranks in one process
or one rank per process over torch.distributed.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OCCL_LIB_PATH") or os.path.join(_HERE, "lib", "libocclb200.so")
GEN_PATH = os.path.join(_HERE, "lib", "libocclgen.so")

# ---------------------------------------------------------------- enums (occl.h)
occlSuccess, occlInvalidArgument, occlInvalidUsage, occlRegistryFull, occlQueueFull, \
    occlDuplicateSubmit, occlUnknownId, occlCudaError, occlSystemError, occlTimeout, \
    occlInProgress, occlInternalError = range(12)
occlInt32, occlFloat32, occlBfloat16, occlFloat16, occlInt64, occlFloat64 = 0, 1, 2, 3, 4, 5
occlSum, occlProd, occlMax, occlMin = 0, 1, 2, 3
OPS = {"sum": occlSum, "prod": occlProd, "max": occlMax, "min": occlMin}
occlOrderFifo, occlOrderPriority = 0, 1
KIND = {"allreduce": 0, "allgather": 1, "reducescatter": 2, "broadcast": 3, "reduce": 4}
DTYPE = {"i32": occlInt32, "f32": occlFloat32, "bf16": occlBfloat16, "f16": occlFloat16, "i64": occlInt64,
         "f64": occlFloat64}
OCCL_HANDLE_BYTES = 256

EXPORTED = [
    "occlGetErrorString", "occlConfigDefault", "occlCommCreate", "occlCommGetHandle", "occlCommConnect",
    "occlCommInit", "occlCommDestroy", "occlAllReduce", "occlAllGather", "occlReduceScatter",
    "occlBroadcast", "occlWait", "occlTest", "occlSetCallback", "occlGetStats", "occlGetCollStats",
    "occlCommExit", "occlCommLaunch", "occlCommSetAutoLaunch", "occlCommQuiesce", "occlCommGetStream",
    "occlCollBlocks", "occlCommFuse", "occlGetProbes", "occlSetPriority", "occlGetTrace", "occlTraceReset",
    "occlCommSplit", "occlReduce", "occlGetFootprint",
]
TRACE_EVENTS = {1: "fetch", 2: "switch_in", 3: "issue", 4: "publish", 5: "preempt", 6: "done", 7: "cqe",
                8: "quit", 9: "exit", 10: "sdone", 11: "start", 12: "mark"}


class occlConfig_t(C.Structure):
    _fields_ = [
        ("maxColl", C.c_int), ("gridBlocks", C.c_int), ("blockThreads", C.c_int), ("connSlots", C.c_int),
        ("slicesPerChunk", C.c_int), ("sliceBytes", C.c_size_t), ("minBlockBytes", C.c_size_t),
        ("sqDepth", C.c_int), ("orderPolicy", C.c_int), ("priorityCadence", C.c_int), ("stickiness", C.c_int),
        ("spinBase", C.c_uint32), ("spinStep", C.c_uint32), ("spinMin", C.c_uint32), ("spinBoost", C.c_uint32),
        ("spinCap", C.c_uint32), ("stallLimit", C.c_uint32), ("quitEnabled", C.c_int),
        ("quitIdleNs", C.c_uint64), ("idleSleepNs", C.c_uint32), ("autoLaunch", C.c_int), ("cacheWays", C.c_int),
        ("pipeDepth", C.c_int), ("prefetchSlices", C.c_int), ("discardConsumed", C.c_int), ("l2Hints", C.c_int),
        ("directMode", C.c_int), ("stagingTiles", C.c_int), ("blocksPerSM", C.c_int), ("traceCap", C.c_uint32),
        ("llSliceBytes", C.c_uint32), ("llMaxBytes", C.c_uint32), ("spinNs", C.c_uint32),
        ("bulkStores", C.c_int), ("directRead", C.c_int), ("stallNs", C.c_uint64),
        ("forceSysScope", C.c_int), ("cqMode", C.c_int), ("sqYieldNs", C.c_uint64),
        ("llSpeculate", C.c_int), ("readyFirst", C.c_int),
    ]


class occlStats_t(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("launches", "quits", "exits", "preemptions", "ctxLoads", "ctxSaves",
                                          "slices", "sqeFetched", "cqeWritten")] + [("lastLaunchMs", C.c_float)]


class occlCollStats_t(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("preemptions", "ctxLoads", "ctxSaves", "slices", "completions")]


class occlTraceRec_t(C.Structure):
    _fields_ = [("t", C.c_uint64), ("tag", C.c_uint32), ("arg", C.c_uint32)]


class occlFootprint_t(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("device", "connectorData", "connectorFlags", "llLines", "contexts",
                                          "other", "pinnedHost")] + [("perBlockPerColl", C.c_double)]


class occlProbes_t(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("cycRun", "cycPoll", "cycAcqFence", "cycRelFence", "cycData",
                                          "cycDataWait", "nData", "nCommit", "nFence", "cycCtxLoad",
                                          "nCtxLoad", "cycCtxSave", "nCtxSave", "cycCqe", "nCqe")]


CALLBACK = C.CFUNCTYPE(None, C.c_int, C.c_void_p)
ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class OcclError(RuntimeError):
    def __init__(self, code, what=""):
        self.code = code
        super().__init__(f"{what}: occl error {code} ({_lib().occlGetErrorString(code).decode()})")


_LIB = None
_GEN = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i, sz, i64 = C.c_void_p, C.c_int, C.c_size_t, C.c_int64
        L.occlGetErrorString.restype = C.c_char_p
        L.occlGetErrorString.argtypes = [i]
        for name, args in {
            "occlConfigDefault": [C.POINTER(occlConfig_t)],
            "occlCommCreate": [C.POINTER(vp), i, i, i, C.POINTER(occlConfig_t)],
            "occlCommGetHandle": [vp, vp, C.POINTER(sz)],
            "occlCommConnect": [vp, vp, sz],
            "occlCommInit": [C.POINTER(vp), i, i, i, ALLGATHER, vp, C.POINTER(occlConfig_t)],
            "occlCommDestroy": [vp],
            "occlAllReduce": [vp, vp, sz, i, i, i, vp],
            "occlAllGather": [vp, vp, sz, i, i, vp],
            "occlReduceScatter": [vp, vp, sz, i, i, i, vp],
            "occlBroadcast": [vp, vp, sz, i, i, i, vp],
            "occlReduce": [vp, vp, sz, i, i, i, i, vp],
            "occlGetFootprint": [vp, C.POINTER(occlFootprint_t)],
            "occlWait": [vp, i, i64],
            "occlTest": [vp, i, C.POINTER(i)],
            "occlSetCallback": [vp, i, CALLBACK, vp],
            "occlGetStats": [vp, C.POINTER(occlStats_t)],
            "occlGetCollStats": [vp, i, C.POINTER(occlCollStats_t)],
            "occlCommExit": [vp],
            "occlCommLaunch": [vp],
            "occlCommSetAutoLaunch": [vp, i],
            "occlCommQuiesce": [vp, i64],
            "occlCommGetStream": [vp, C.POINTER(vp)],
            "occlCollBlocks": [vp, i, sz, i, C.POINTER(i)],
            "occlCommFuse": [C.POINTER(vp), i],
            "occlGetProbes": [vp, C.POINTER(occlProbes_t)],
            "occlSetPriority": [vp, i, C.c_int32],
            "occlGetTrace": [vp, i, C.POINTER(occlTraceRec_t), sz, C.POINTER(sz)],
            "occlTraceReset": [vp],
            "occlCommSplit": [vp, i, C.POINTER(i), C.POINTER(vp)],
        }.items():
            f = getattr(L, name, None)
            if f is None:
                if os.environ.get("OCCL_LIB_PATH"):
                    continue                     # diagnostics against an older build
                raise ImportError(f"{LIB_PATH}: missing symbol {name}")
            f.restype = C.c_int
            f.argtypes = args
        _LIB = L
    return _LIB


def gen_lib():
    """Test/bench-only GPU input generator (libocclgen.so)."""
    global _GEN
    if _GEN is None:
        if not os.path.exists(GEN_PATH):
            raise ImportError(f"{GEN_PATH} missing")
        G = C.CDLL(GEN_PATH)
        G.occlTestFill.restype = C.c_int
        G.occlTestFill.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.c_uint32, C.c_uint32,
                                   C.c_uint64, C.c_void_p]
        _GEN = G
    return _GEN


def check(code, what=""):
    if code != occlSuccess:
        raise OcclError(code, what)
    return code


# ---------------------------------------------------------------- same-name wrappers
def occlGetErrorString(code):
    return _lib().occlGetErrorString(code).decode()


def occlConfigDefault(**overrides) -> occlConfig_t:
    cfg = occlConfig_t()
    check(_lib().occlConfigDefault(C.byref(cfg)), "occlConfigDefault")
    for k, v in overrides.items():
        if not hasattr(cfg, k):
            raise KeyError(k)
        setattr(cfg, k, v)
    return cfg


def occlCommCreate(nranks, rank, dev, cfg=None):
    h = C.c_void_p()
    check(_lib().occlCommCreate(C.byref(h), nranks, rank, dev, C.byref(cfg) if cfg is not None else None),
          "occlCommCreate")
    return h


def occlCommGetHandle(comm) -> bytes:
    buf = C.create_string_buffer(OCCL_HANDLE_BYTES)
    n = C.c_size_t(OCCL_HANDLE_BYTES)
    check(_lib().occlCommGetHandle(comm, buf, C.byref(n)), "occlCommGetHandle")
    return buf.raw[:OCCL_HANDLE_BYTES]


def occlCommConnect(comm, handles):
    blob = b"".join(h.ljust(OCCL_HANDLE_BYTES, b"\0") for h in handles)
    check(_lib().occlCommConnect(comm, blob, OCCL_HANDLE_BYTES), "occlCommConnect")


def occlCommDestroy(comm):
    check(_lib().occlCommDestroy(comm), "occlCommDestroy")


def occlAllReduce(send, recv, count, dtype, op, coll_id, comm):
    return _lib().occlAllReduce(send, recv, count, dtype, op, coll_id, comm)


def occlAllGather(send, recv, sendcount, dtype, coll_id, comm):
    return _lib().occlAllGather(send, recv, sendcount, dtype, coll_id, comm)


def occlReduceScatter(send, recv, recvcount, dtype, op, coll_id, comm):
    return _lib().occlReduceScatter(send, recv, recvcount, dtype, op, coll_id, comm)


def occlBroadcast(send, recv, count, dtype, root, coll_id, comm):
    return _lib().occlBroadcast(send, recv, count, dtype, root, coll_id, comm)


def occlWait(comm, coll_id, timeout_ns=-1):
    return _lib().occlWait(comm, coll_id, timeout_ns)


def occlTest(comm, coll_id):
    d = C.c_int(0)
    check(_lib().occlTest(comm, coll_id, C.byref(d)), "occlTest")
    return bool(d.value)


def occlGetStats(comm) -> dict:
    s = occlStats_t()
    check(_lib().occlGetStats(comm, C.byref(s)), "occlGetStats")
    return {k: getattr(s, k) for k, _ in occlStats_t._fields_}


def occlGetCollStats(comm, coll_id) -> dict:
    s = occlCollStats_t()
    check(_lib().occlGetCollStats(comm, coll_id, C.byref(s)), "occlGetCollStats")
    return {k: getattr(s, k) for k, _ in occlCollStats_t._fields_}


# ---------------------------------------------------------------- convenience
def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


class Comm:
    """One rank.  Buffers are torch CUDA tensors (or raw device pointers)."""

    def __init__(self, handle, nranks, rank, dev, cfg):
        self.h, self.nranks, self.rank, self.dev, self.cfg = handle, nranks, rank, dev, cfg
        self._callbacks = {}

    # submission (asynchronous) -------------------------------------------------
    def all_reduce(self, send, recv, coll_id, count=None, dtype=None, op="sum"):
        count = send.numel() if count is None else count
        dtype = _dt(send) if dtype is None else dtype
        check(occlAllReduce(_ptr(send), _ptr(recv), count, dtype, OPS.get(op, op), coll_id, self.h), "occlAllReduce")

    def all_gather(self, send, recv, coll_id, count=None, dtype=None):
        count = send.numel() if count is None else count
        dtype = _dt(send) if dtype is None else dtype
        check(occlAllGather(_ptr(send), _ptr(recv), count, dtype, coll_id, self.h), "occlAllGather")

    def reduce_scatter(self, send, recv, coll_id, count=None, dtype=None, op="sum"):
        count = recv.numel() if count is None else count
        dtype = _dt(recv) if dtype is None else dtype
        check(occlReduceScatter(_ptr(send), _ptr(recv), count, dtype, OPS.get(op, op), coll_id, self.h),
              "occlReduceScatter")

    def broadcast(self, send, recv, root, coll_id, count=None, dtype=None):
        count = recv.numel() if count is None else count
        dtype = _dt(recv) if dtype is None else dtype
        check(occlBroadcast(_ptr(send), _ptr(recv), count, dtype, root, coll_id, self.h), "occlBroadcast")

    def reduce(self, send, recv, root, coll_id, count=None, dtype=None, op="sum"):
        count = send.numel() if count is None else count
        dtype = _dt(send) if dtype is None else dtype
        check(_lib().occlReduce(_ptr(send), _ptr(recv), count, dtype, OPS.get(op, op), root, coll_id, self.h),
              "occlReduce")

    def submit(self, kind, send, recv, coll_id, count, dtype, root=0, op="sum"):
        k = KIND[kind] if isinstance(kind, str) else kind
        d = DTYPE[dtype] if isinstance(dtype, str) else dtype
        o = OPS[op] if isinstance(op, str) else op
        if k == 0:
            r = occlAllReduce(_ptr(send), _ptr(recv), count, d, o, coll_id, self.h)
        elif k == 1:
            r = occlAllGather(_ptr(send), _ptr(recv), count, d, coll_id, self.h)
        elif k == 2:
            r = occlReduceScatter(_ptr(send), _ptr(recv), count, d, o, coll_id, self.h)
        elif k == 3:
            r = occlBroadcast(_ptr(send), _ptr(recv), count, d, root, coll_id, self.h)
        else:
            r = _lib().occlReduce(_ptr(send), _ptr(recv), count, d, o, root, coll_id, self.h)
        check(r, f"submit {kind}")

    # completion ------------------------------------------------------------------
    def wait(self, coll_id, timeout_s=None):
        t = -1 if timeout_s is None else int(timeout_s * 1e9)
        check(occlWait(self.h, coll_id, t), f"occlWait({coll_id})")

    def test(self, coll_id):
        return occlTest(self.h, coll_id)

    def set_callback(self, coll_id, fn):
        if fn is None:
            cb = CALLBACK()
            self._callbacks.pop(coll_id, None)
        else:
            cb = CALLBACK(lambda cid, arg: fn(cid))
            self._callbacks[coll_id] = cb
        check(_lib().occlSetCallback(self.h, coll_id, cb, None), "occlSetCallback")

    # daemon control -----------------------------------------------------------------
    def exit(self):
        check(_lib().occlCommExit(self.h), "occlCommExit")

    def launch(self):
        check(_lib().occlCommLaunch(self.h), "occlCommLaunch")

    def set_auto_launch(self, on):
        check(_lib().occlCommSetAutoLaunch(self.h, 1 if on else 0), "occlCommSetAutoLaunch")

    def quiesce(self, timeout_s=None):
        t = -1 if timeout_s is None else int(timeout_s * 1e9)
        check(_lib().occlCommQuiesce(self.h, t), "occlCommQuiesce")

    def stream(self) -> int:
        s = C.c_void_p()
        check(_lib().occlCommGetStream(self.h, C.byref(s)), "occlCommGetStream")
        return s.value or 0

    def coll_blocks(self, kind, count, dtype) -> int:
        nb = C.c_int()
        check(_lib().occlCollBlocks(self.h, KIND[kind], count, DTYPE[dtype], C.byref(nb)), "occlCollBlocks")
        return nb.value

    def stats(self):
        return occlGetStats(self.h)

    def coll_stats(self, coll_id):
        return occlGetCollStats(self.h, coll_id)

    def set_priority(self, coll_id, priority):
        check(_lib().occlSetPriority(self.h, coll_id, priority), "occlSetPriority")

    def footprint(self) -> dict:
        f = occlFootprint_t()
        check(_lib().occlGetFootprint(self.h, C.byref(f)), "occlGetFootprint")
        return {k: getattr(f, k) for k, _ in occlFootprint_t._fields_}

    def probes(self) -> dict:
        s = occlProbes_t()
        check(_lib().occlGetProbes(self.h, C.byref(s)), "occlGetProbes")
        return {k: getattr(s, k) for k, _ in occlProbes_t._fields_}

    def split(self, members):
        """Sub-communicator over parent ranks `members` (in the new ring's order);
        shares this communicator's daemon (occlCommSplit)."""
        arr = (C.c_int * len(members))(*members)
        h = C.c_void_p()
        check(_lib().occlCommSplit(self.h, len(members), arr, C.byref(h)), "occlCommSplit")
        return Comm(h.value, len(members), list(members).index(self.rank), self.dev, self.cfg)

    def trace(self, block):
        """Device event trace of one daemon block: list of (t_ns, event, coll, arg), oldest first."""
        cap = max(1, int(self.cfg.traceCap))
        buf = (occlTraceRec_t * cap)()
        n = C.c_size_t()
        check(_lib().occlGetTrace(self.h, block, buf, cap, C.byref(n)), "occlGetTrace")
        return [(buf[k].t, TRACE_EVENTS.get(buf[k].tag >> 24, "?"), buf[k].tag & 0xffff, buf[k].arg)
                for k in range(n.value)]

    def trace_reset(self):
        check(_lib().occlTraceReset(self.h), "occlTraceReset")

    def destroy(self):
        if self.h:
            occlCommDestroy(self.h)
            self.h = None


def _dt(t):
    import torch
    return {torch.float32: occlFloat32, torch.bfloat16: occlBfloat16, torch.int32: occlInt32,
            torch.float16: occlFloat16, torch.int64: occlInt64, torch.float64: occlFloat64}[t.dtype]


def occlCommFuse(comms):
    arr = (C.c_void_p * len(comms))(*[c.h if isinstance(c, Comm) else c for c in comms])
    check(_lib().occlCommFuse(arr, len(comms)), "occlCommFuse")


def local_group(nranks, device=0, cfg=None, fuse=True, **overrides):
    """A ring of `nranks` virtual ranks in this process on one device.  Each rank is
    its own communicator (SQ, CQ, contexts, connectors in plain HBM); with
    fuse=True one daemon kernel launch serves all of them (occlCommFuse)."""
    cfg = cfg if cfg is not None else occlConfigDefault(**overrides)
    hs = [occlCommCreate(nranks, r, device, cfg) for r in range(nranks)]
    handles = [occlCommGetHandle(h) for h in hs]
    for h in hs:
        occlCommConnect(h, handles)
    comms = [Comm(h, nranks, r, device, cfg) for r, h in enumerate(hs)]
    if fuse and nranks > 1:
        occlCommFuse(comms)
    return comms


def occlCommInit(nranks, rank, dev, allgather, cfg=None):
    """occlCommInit with a Python bootstrap all-gather: ``allgather(mine: bytes)
    -> list[bytes]`` (rank-major) is called once, from inside the C call."""
    failure = []

    def ag(inp, out, nbytes, ctx):
        try:
            parts = allgather(C.string_at(inp, nbytes))
            blob = b"".join(bytes(p).ljust(nbytes, b"\0")[:nbytes] for p in parts)
            if len(blob) != nbytes * nranks:
                return 1
            C.memmove(out, blob, len(blob))
            return 0
        except Exception as e:  # noqa: BLE001 -- reported after the C call returns
            failure.append(e)
            return 1

    cb = ALLGATHER(ag)
    h = C.c_void_p()
    code = _lib().occlCommInit(C.byref(h), nranks, rank, dev, cb, None, C.byref(cfg) if cfg is not None else None)
    if failure:
        raise failure[0]
    check(code, "occlCommInit")
    return h


def process_group(pg=None, device=None, cfg=None, **overrides):
    """One rank per process over torch.distributed: occlCommInit with
    dist.all_gather_object as the bootstrap all-gather; connectors are opened
    through CUDA IPC / peer access."""
    import torch
    import torch.distributed as dist
    rank, n = dist.get_rank(pg), dist.get_world_size(pg)
    device = torch.cuda.current_device() if device is None else device
    cfg = cfg if cfg is not None else occlConfigDefault(**overrides)

    def allgather(mine):
        allh = [None] * n
        dist.all_gather_object(allh, mine, group=pg)
        return allh

    h = occlCommInit(n, rank, device, allgather, cfg)
    return Comm(h, n, rank, device, cfg)


def split_group(comms, groups):
    """Split every rank of a local group into the sub-communicator of the group
    (list of parent ranks) it belongs to; returns {group index: [child comms in
    child-rank order]}."""
    out = {}
    for gi, g in enumerate(groups):
        out[gi] = [comms[q].split(g) for q in g]
    return out


def destroy_group(comms):
    for c in comms:
        c.destroy()


def test_fill(t, dtype: str, seed: int, coll: int, rank: int, offset: int = 0, stream: int = 0):
    """Fill tensor `t` with the seeded generator values x_rank[offset + i] (GPU)."""
    r = gen_lib().occlTestFill(t.data_ptr(), t.numel(), DTYPE[dtype], seed & ((1 << 64) - 1), coll, rank,
                               offset, stream)
    if r != 0:
        raise RuntimeError(f"occlTestFill failed: cuda error {r}")
