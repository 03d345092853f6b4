"""O2 -- slow deterministic multi-rank simulator of OCCL's DFCE framework.  TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module.  Shares no code with paper_2303_06324_b200/.

It follows the paper's algorithm step by step (§3 "Design", §4
"Implementation and Optimizations"), in the paper's vocabulary:

* every rank ("GPU") runs a *daemon* made of ``lanes`` independent blocks
  ("the block with a high index can execute a different
  collective"); each block keeps a *task queue* and traverses it,
  executing *primitive sequences* in a two-phase blocking manner:
  spin on the connector up to a *spin threshold*, then preempt;
* a collective's *context* = static (meta, plan, buffers, connectors) + dynamic
  (chunk/loop id, primitive/step id, slice id); the
  dynamic context is saved to the "global" context buffer only when the collective
  made progress before preemption (lazy save) and loaded through a
  direct-mapped context cache;
* connectors are bounded FIFOs dedicated to one (collective, block, edge)
  (PAPER.md:301-303, :377, :581); committed pushes stay visible after preemption
  (PAPER.md:317-319);
* SQ: one host writer, every block reads every SQE; a block
  executes a collective only if blockIdx < its block count (reading Q11);
  Exiting SQE;
* CQ + per-collective completion counter: the block whose increment reaches the
  collective's block count posts the CQE; the host poller fires
  the callback bound at submission;
* voluntary quit when the queue is empty or every entry is stuck and no SQE came
  for a while, event-driven relaunch when SQEs are pending or
  #CQE < #SQE;
* stickiness: FIFO or priority-front ordering; initial spin
  threshold decremented by queue position, raised on each successful primitive
  (PAPER.md:449-452); optionally the readiness-board extension of the priority
  policy (ready_first, reading R29 -- not in the paper, labelled): at
  switch-in the first entry every member of its ring admitted runs, and only a
  ready front is boosted;
* "baseline" mode is the NCCL-like negative control: infinite
  threshold, no quit, a fixed number of resident slots ("streams", Fig. 1(b)),
  strictly in submission order.

A seeded scheduler picks one actor (a rank's block, or a rank's host program) per
global tick and runs one micro-step.  PASS = every host program finished and every
submission completed; DEADLOCK = no progress event for a long window.

Parity unpinned (timing-dependent, reported only): preemption counts, queue-length
traces, stickiness speed-ups.
"""
from __future__ import annotations

import random
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from . import ring

INF = float("inf")


@dataclass
class SimConfig:
    lanes: int = 1                 # daemon grid size G (blocks per rank)
    K: int = 8                     # connector slots
    slice_elems: int = 256         # elements per connector slot
    slices_per_chunk: int = 4
    order_policy: str = "fifo"     # "fifo" | "priority"
    priority_cadence: int = 4      # priority policy: check SQ every R lane ticks
    ready_first: int = 0           # priority policy extension (reading R29): at switch-in run
                                   # the highest-priority entry (among the first ready_scan) every member admitted;
                                   # 2 = a lane whose whole queue is scanned and has no ready entry runs
                                   # nothing (waits; counts as stuck for the quit rule)
    ready_scan: int = 64           # R29 scan window (the daemon's kReadyScan)
    stickiness: bool = True        # paper's spin-threshold policy; False = constant T
    spin_base: int = 4096          # SPEC.md:421 desk-scale defaults
    spin_step: int = 256
    spin_min: int = 64
    spin_boost: int = 2
    spin_cap: int = 16384
    stall_limit: int = 2           # "cannot progress for a long time" (reading Q3)
    quit_enabled: bool = True
    quit_idle: int = 256           # lane ticks without a fetch (reading Q4)
    cache_ways: int = 4            # direct-mapped context cache
    baseline: bool = False         # NCCL-like negative control
    baseline_slots: int = 1        # resident collectives ("streams", Fig. 1(b))
    scheduler: str = "random"      # "random" | "roundrobin"
    seed: int = 0
    max_ticks: int = 50_000_000
    stuck_window: int = 0          # 0 = derived from thresholds


@dataclass
class CollMeta:
    """A collective invocation (identical on every rank except buffers)."""
    coll_id: int
    kind: str
    dtype: str
    count: int
    root: int = 0
    nblocks: int = 1
    inplace: bool = False
    priority: int | None = None    # priority policy: globally agreed, lower first (default coll_id)
    members: tuple | None = None   # sub-communicator ring (parent ranks in ring order); None = all
    op: str = "sum"                # reducing function
                                   # (the static context carries nranks / rank)


@dataclass
class _Sqe:
    meta: CollMeta | None          # None = Exiting SQE
    sendbuf: np.ndarray | None = None
    recvbuf: np.ndarray | None = None
    sub_index: int = 0


@dataclass
class _Dyn:
    loop: int = 0                  # chunk (loop) id
    step: int = 0                  # primitive id in the sequence
    slc: int = 0                   # slice id inside the chunk
    progressed: bool = False

    def copy(self):
        return _Dyn(self.loop, self.step, self.slc, self.progressed)


@dataclass
class _Static:
    meta: CollMeta
    rank: int
    n: int
    seq: list
    segs: list                     # per segment: (send_base | None, recv_base | None, length)
    part: int                      # lane part length per segment (Pb)
    lane: int
    nloops: int
    sendbuf: np.ndarray
    recvbuf: np.ndarray
    sub_index: int
    members: tuple = ()            # the collective's ring (parent ranks)


class _Connector:
    """Bounded FIFO (PAPER.md:301 'lock-free ring buffers'); sequence-number audited."""
    __slots__ = ("cap", "q", "pushed", "popped", "tag")

    def __init__(self, cap, tag):
        self.cap, self.q, self.pushed, self.popped, self.tag = cap, deque(), 0, 0, tag

    def can_push(self):
        return len(self.q) < self.cap

    def can_pop(self):
        return len(self.q) > 0

    def push(self, payload, coll_id):
        assert len(self.q) < self.cap, "connector occupancy exceeded"
        self.q.append((self.pushed, np.array(payload, copy=True), coll_id))
        self.pushed += 1

    def pop(self, coll_id):
        seq, payload, tag = self.q.popleft()
        assert seq == self.popped, "connector FIFO order violated"
        assert tag == coll_id, "connector shared between collectives"
        self.popped += 1
        return payload


@dataclass
class _Lane:
    alive: bool = False
    cursor: int = 0
    queue: list = field(default_factory=list)
    pos: int = 0
    T: float | None = None         # live spin threshold of the current visit
    boost_ok: bool = True          # ready_first: the current visit may be boosted
    waiting: bool = False          # ready_first = 2: nothing in the queue is ready
    spins: int = 0
    stall: dict = field(default_factory=dict)
    clock: int = 0
    last_fetch: int = 0
    exiting: bool = False
    cache: dict = field(default_factory=dict)   # way -> (coll_id, _Dyn)


@dataclass
class _Rank:
    sq: list = field(default_factory=list)
    lanes: list = field(default_factory=list)
    alive: bool = False
    submitted: int = 0
    completed: int = 0
    cq: list = field(default_factory=list)
    cnt: dict = field(default_factory=dict)       # completion counters
    static: dict = field(default_factory=dict)    # (coll, lane) -> _Static
    dyn_global: dict = field(default_factory=dict)  # (coll, lane) -> _Dyn (context buffer)
    outstanding: dict = field(default_factory=dict)  # coll -> submission count in flight
    adm: dict = field(default_factory=dict)       # (coll, lane) -> admissions so far (readiness board, R29)
    program: list = field(default_factory=list)
    pc: int = 0
    delay_until: int = 0
    sync_gen: int | None = None


class Deadlock(Exception):
    pass



# ============================================================================ pure pieces
def apply_action_set(prim: str, incoming, local, dtype: str, op: str = "sum"):
    """Fused actions of one primitive on one slice:
    recv grabs ``incoming`` from the recv connector, reduce combines it with the
    send-buffer slice ``local``, copy puts the value into the recv buffer, send pushes
    it to the send connector.  Returns (to_recv_buf | None, to_send_conn | None)."""
    recv, reduce_, copy, send = ring.PRIMS[prim]
    if recv and reduce_:
        val = ring.add(incoming, local, dtype, op)
    elif recv:
        val = incoming
    else:
        val = local
    return (val if copy else None), (val if send else None)


def initial_threshold(pos: int, cfg: "SimConfig") -> float:
    """Initial spin threshold by task-queue position:
    max(min, base - pos*step); constant base when stickiness is off."""
    if cfg.baseline:
        return INF
    if not cfg.stickiness:
        return cfg.spin_base
    return max(cfg.spin_min, cfg.spin_base - pos * cfg.spin_step)


def boosted_threshold(T: float, cfg: "SimConfig") -> float:
    """Raise the threshold after a successful primitive, capped."""
    if cfg.baseline or not cfg.stickiness:
        return T
    return min(cfg.spin_cap, T * cfg.spin_boost)

# ============================================================================ geometry
def lane_geometry(meta: CollMeta, n: int, rank: int, cfg: SimConfig):
    """Segments + lane-part + loop count.  AR uses the segment-first owner map of O1's
    reading (R6); RS/AG segments are fixed by the API; BC is one segment."""
    A = 16 // ring.ITEMSIZE[meta.dtype]
    N = meta.count
    if meta.kind == "allreduce":
        per = -(-N // n)
        L = -(-per // A) * A
        segs = [(q * L, q * L, max(0, min(N, (q + 1) * L) - q * L)) for q in range(n)]
        seglen = L
    elif meta.kind == "reducescatter":
        segs = [(q * N, 0 if q == rank else None, N) for q in range(n)]
        seglen = N
    elif meta.kind == "allgather":
        segs = [(0 if q == rank else None, q * N, N) for q in range(n)]
        seglen = N
    elif meta.kind in ("broadcast", "reduce"):
        segs = [(0, 0, N)]
        seglen = N
    else:
        raise ValueError(meta.kind)
    if n == 1:
        segs = [(0, 0, N)]
        seglen = N
    B = meta.nblocks
    part = -(-(-(-seglen // B)) // A) * A
    chunk = cfg.slices_per_chunk * cfg.slice_elems
    nloops = max(1, -(-part // chunk))
    return segs, part, nloops


def ring_members(meta: CollMeta, nranks: int) -> tuple:
    """Parent ranks of the collective's ring, in ring order."""
    return tuple(meta.members) if meta.members is not None else tuple(range(nranks))


def slice_range(st: _Static, q: int, loop: int, slc: int, cfg: SimConfig):
    """Element range [lo, lo+len) inside segment q for (lane, loop, slice)."""
    seglen = st.segs[q][2]
    lane_lo = st.lane * st.part
    lane_hi = min(seglen, (st.lane + 1) * st.part)
    lo = lane_lo + loop * cfg.slices_per_chunk * cfg.slice_elems + slc * cfg.slice_elems
    hi = min(lane_hi, lo + cfg.slice_elems)
    return lo, max(0, hi - lo)


# ============================================================================ simulator
class Simulator:
    def __init__(self, nranks: int, cfg: SimConfig | None = None):
        self.n = nranks
        self.cfg = cfg or SimConfig()
        if self.cfg.K <= self.cfg.slices_per_chunk:
            # A fused recv+send primitive pops and pushes one slice at a time; the first
            # Send step pushes a whole chunk.  If K == slices_per_chunk every connector of
            # the ring can be full while every rank waits to push: circular wait.  K must
            # exceed the slices in flight per step (DESIGN.md invariant I7).
            raise ValueError("connector slots K must exceed slices_per_chunk")
        self.rng = random.Random(self.cfg.seed)
        self.ranks = [_Rank(lanes=[_Lane() for _ in range(self.cfg.lanes)]) for _ in range(nranks)]
        self.conn = {}                 # (coll, lane, src_rank) -> _Connector
        self.tick = 0
        self.last_progress = 0
        # statistics (reported, not asserted: parity unpinned)
        self.preempt = {}              # (rank, coll, lane) -> count
        self.ready_picks_behind_front = 0   # R29 switch-ins that ran a ready entry behind the queue front
        self.ready_waits = 0                # R29 wait mode: lane ticks with nothing ready to run
        self.loads = 0
        self.saves = 0
        self.launches = [0] * nranks
        self.quits = [0] * nranks
        self.queue_len_at_fetch = [[] for _ in range(nranks)]
        self.transfers = {}            # (rank, coll, sub, lane, step) -> slices moved
        self.callbacks = {}            # (rank, coll) -> count
        self.results = {}              # (rank, coll, sub) -> recvbuf
        self._sub_counter = {}

    # ------------------------------------------------------------------ host side
    def set_program(self, rank: int, ops):
        """ops: list of ("submit", CollMeta, sendbuf, recvbuf) | ("sync",) |
        ("wait", coll_id) | ("delay", ticks)."""
        self.ranks[rank].program = list(ops)

    def _host_step(self, r: int) -> bool:
        R = self.ranks[r]
        if R.pc >= len(R.program) or self.tick < R.delay_until:
            return False
        op = R.program[R.pc]
        if op[0] == "submit":
            meta, sendbuf, recvbuf = op[1], op[2], op[3]
            assert R.outstanding.get(meta.coll_id, 0) == 0, "duplicate submit (reading Q10)"
            sub = self._sub_counter.get((r, meta.coll_id), 0)
            self._sub_counter[(r, meta.coll_id)] = sub + 1
            if meta.count == 0:           # completes at submission (reading Q18)
                self.callbacks[(r, meta.coll_id)] = self.callbacks.get((r, meta.coll_id), 0) + 1
                self.results[(r, meta.coll_id, sub)] = recvbuf
            else:
                R.sq.append(_Sqe(meta, sendbuf, recvbuf, sub))
                R.submitted += 1
                R.outstanding[meta.coll_id] = 1
        elif op[0] == "exit":
            R.sq.append(_Sqe(None))
        elif op[0] == "sync":
            # device synchronisation blocks until the daemon instance running when the
            # sync was issued has exited (Fig. 1(c)); a relaunch by
            # the supervisor after that exit is work issued after the sync.
            if R.sync_gen is None:
                R.sync_gen = self.launches[r]
            if R.alive and self.launches[r] == R.sync_gen:
                return False
            R.sync_gen = None
        elif op[0] == "wait":
            if R.outstanding.get(op[1], 0):
                return False
        elif op[0] == "delay":
            R.delay_until = self.tick + op[1]
        else:
            raise ValueError(op)
        R.pc += 1
        return True

    def _supervisor(self, r: int) -> bool:
        """Event-driven (re)start."""
        R = self.ranks[r]
        if R.alive:
            return False
        pending = any(L.cursor < len(R.sq) for L in R.lanes) or R.submitted > R.completed
        if not pending:
            return False
        R.alive = True
        self.launches[r] += 1
        for L in R.lanes:
            L.alive = True
            L.last_fetch = L.clock
            L.T = None
            L.spins = 0
            L.cache = {}          # shared memory does not survive a relaunch
        return True

    # ------------------------------------------------------------------ daemon side
    def _T_init(self, pos: int) -> float:
        return initial_threshold(pos, self.cfg)

    def _can_fetch(self, L: _Lane) -> bool:
        c = self.cfg
        if L.exiting:
            return False
        if c.baseline:
            return len(L.queue) < c.baseline_slots
        if not L.queue:
            return True
        if c.order_policy == "priority":
            return L.clock % c.priority_cadence == 0
        return all(L.stall.get(i, 0) >= c.stall_limit for i in L.queue)

    def _load_ctx(self, r: int, b: int, coll: int) -> _Dyn:
        """Direct-mapped context cache: hit => no load."""
        R, L = self.ranks[r], self.ranks[r].lanes[b]
        way = coll % self.cfg.cache_ways
        ent = L.cache.get(way)
        if ent is not None and ent[0] == coll:
            return ent[1]
        if ent is not None and ent[1].progressed:
            # the way holds another collective's context that progressed since its
            # last save: it is switched out here, so the lazy save happens now
            # (PAPER.md:513-514).  Reached when an admission under the priority
            # policy moves the lane's position between two micro-steps of a run.
            self._save_ctx(r, b, ent[0], ent[1])
        d = R.dyn_global[(coll, b)].copy()
        self.loads += 1
        L.cache[way] = (coll, d)
        return d

    def _save_ctx(self, r: int, b: int, coll: int, d: _Dyn):
        """Lazy save: only a dynamic context that progressed."""
        if d.progressed:
            d.progressed = False
            self.ranks[r].dyn_global[(coll, b)] = d.copy()
            self.saves += 1

    def _admit(self, r: int, b: int, sqe: _Sqe):
        R, L = self.ranks[r], self.ranks[r].lanes[b]
        m = sqe.meta
        members = ring_members(m, self.n)
        n, rr = len(members), members.index(r)          # the collective's own ring size / rank
        segs, part, nloops = lane_geometry(m, n, rr, self.cfg)
        seq = ring.ring_sequence(m.kind, n, rr, m.root, m.inplace)
        R.static[(m.coll_id, b)] = _Static(m, rr, n, seq, segs, part, b, nloops,
                                           sqe.sendbuf, sqe.recvbuf, sqe.sub_index, members)
        R.dyn_global[(m.coll_id, b)] = _Dyn()
        R.adm[(m.coll_id, b)] = R.adm.get((m.coll_id, b), 0) + 1
        way = m.coll_id % self.cfg.cache_ways
        if way in L.cache and L.cache[way][0] == m.coll_id:
            del L.cache[way]
        self.queue_len_at_fetch[r].append(len(L.queue))
        if self.cfg.order_policy == "priority" and not self.cfg.baseline:
            # priority-based ordering, reading R10: the
            # queue is kept sorted by the user-defined priority (ties: arrival) and
            # the traversal restarts at the front
            prio = lambda cid: R.static[(cid, b)].meta.priority if R.static[(cid, b)].meta.priority is not None \
                else cid
            at = len(L.queue)
            while at > 0 and prio(L.queue[at - 1]) > prio(m.coll_id):
                at -= 1
            L.queue.insert(at, m.coll_id)
            L.pos = 0
            L.T = None
        else:
            L.queue.append(m.coll_id)
        L.stall[m.coll_id] = 0

    def _connector(self, coll: int, lane: int, src: int) -> _Connector:
        key = (coll, lane, src)
        c = self.conn.get(key)
        if c is None:
            c = self.conn[key] = _Connector(self.cfg.K, key)
        return c

    def _try_slice(self, r: int, b: int, st: _Static, d: _Dyn) -> bool:
        """One attempt at the current slice: True if it executed."""
        prim, q = st.seq[d.step]
        recv, reduce_, copy, send = ring.PRIMS[prim]
        m = st.meta
        n, mem = st.n, st.members
        # connector (coll, lane, writer): written by the ring predecessor, a parent rank
        cin = self._connector(m.coll_id, b, mem[(st.rank - 1) % n]) if recv else None
        cout = self._connector(m.coll_id, b, r) if send else None
        if recv and not cin.can_pop():
            return False
        if send and not cout.can_push():
            return False
        lo, ln = slice_range(st, q, d.loop, d.slc, self.cfg)
        send_base, recv_base, _ = st.segs[q]
        incoming = cin.pop(m.coll_id) if recv else None
        if incoming is not None:
            assert len(incoming) == ln, "slice length mismatch across ranks"
        local = None
        if (reduce_ or not recv) and prim != "Recv":
            local = st.sendbuf[send_base + lo: send_base + lo + ln]
        to_recv, to_send = apply_action_set(prim, incoming, local, m.dtype, m.op)
        if to_recv is not None:
            st.recvbuf[recv_base + lo: recv_base + lo + ln] = to_recv
        if to_send is not None:
            cout.push(to_send, m.coll_id)
        key = (r, m.coll_id, st.sub_index, b, d.step)
        self.transfers[key] = self.transfers.get(key, 0) + 1
        return True

    def _advance(self, st: _Static, d: _Dyn) -> bool:
        """slice -> step -> loop; True when the lane's part is done."""
        d.slc += 1
        if d.slc == self.cfg.slices_per_chunk:
            d.slc = 0
            d.step += 1
            if d.step == len(st.seq):
                d.step = 0
                d.loop += 1
        d.progressed = True
        return d.loop >= st.nloops

    def _complete(self, r: int, b: int, coll: int):
        """Completion counter; last block posts the CQE."""
        R, L = self.ranks[r], self.ranks[r].lanes[b]
        st = R.static[(coll, b)]
        R.cnt[coll] = R.cnt.get(coll, 0) + 1
        idx = L.queue.index(coll)
        L.queue.pop(idx)
        L.stall.pop(coll, None)
        if L.queue:
            if idx < L.pos:
                L.pos -= 1
            L.pos %= len(L.queue)
        else:
            L.pos = 0
        L.T = None
        L.spins = 0
        way = coll % self.cfg.cache_ways
        if way in L.cache and L.cache[way][0] == coll:
            del L.cache[way]
        if R.cnt[coll] == st.meta.nblocks:
            R.cnt[coll] = 0
            R.cq.append(coll)
            R.completed += 1
            R.outstanding[coll] = 0
            self.callbacks[(r, coll)] = self.callbacks.get((r, coll), 0) + 1
            self.results[(r, coll, st.sub_index)] = st.recvbuf

    def _lane_step(self, r: int, b: int) -> bool:
        """One micro-step of block b of rank r's daemon.  Returns True on progress."""
        R, L, c = self.ranks[r], self.ranks[r].lanes[b], self.cfg
        if not L.alive:
            return False
        L.clock += 1
        # (1) fetch an SQE, policy-gated
        if self._can_fetch(L) and L.cursor < len(R.sq):
            sqe = R.sq[L.cursor]
            L.cursor += 1
            L.last_fetch = L.clock
            if sqe.meta is None:
                L.exiting = True
            elif b < sqe.meta.nblocks:          # reading Q11
                self._admit(r, b, sqe)
            return True
        # (2) execute the entry at the current position
        if L.queue:
            ready_first = c.ready_first and c.order_policy == "priority" and not c.baseline
            if L.T is None and ready_first:
                # switch-in under the readiness board (R29): the first entry every
                # member of its ring admitted wins and, if it is the front, runs with
                # the full boostable threshold; otherwise the entry at pos waits
                # at most spin_min
                pick = None
                for i, cid in enumerate(L.queue[:c.ready_scan]):
                    need = R.adm[(cid, b)]
                    if all(self.ranks[q].adm.get((cid, b), 0) >= need for q in R.static[(cid, b)].members):
                        pick = i
                        break
                L.waiting = pick is None and c.ready_first >= 2 and len(L.queue) <= c.ready_scan
                if L.waiting:                     # none can complete: run nothing (R29, wait mode)
                    self.ready_waits += 1
                    self._quit_check(r, b)
                    return False
                if pick is not None:
                    L.pos = pick
                    if pick > 0:
                        self.ready_picks_behind_front += 1
                L.boost_ok = pick == 0
                L.T = c.spin_base if L.boost_ok else c.spin_min
            coll = L.queue[L.pos]
            st = R.static[(coll, b)]
            d = self._load_ctx(r, b, coll)
            if L.T is None:
                L.T = self._T_init(L.pos)
            if self._try_slice(r, b, st, d):
                L.spins = 0
                L.stall[coll] = 0
                if not ready_first or L.boost_ok:
                    L.T = boosted_threshold(L.T, c)
                if self._advance(st, d):
                    self._complete(r, b, coll)
                return True
            L.spins += 1
            if c.baseline:
                if len(L.queue) > 1:          # independent resident "streams" interleave
                    L.pos = (L.pos + 1) % len(L.queue)
                return False
            if L.spins > L.T:                 # preempt
                self._save_ctx(r, b, coll, d)
                k = (r, coll, b)
                self.preempt[k] = self.preempt.get(k, 0) + 1
                L.stall[coll] = L.stall.get(coll, 0) + 1
                L.pos = (L.pos + 1) % len(L.queue)
                L.T = None                    # recomputed from position at switch-in (Q12)
                L.spins = 0
            self._quit_check(r, b)            # all entries stuck and no new SQE
            return False
        # (3) empty queue: exit after Exiting SQE, or voluntary quit
        if L.exiting:
            L.alive = False
            L.exiting = False
            self._maybe_dead(r)
            return False
        self._quit_check(r, b)
        return False

    def _quit_check(self, r: int, b: int):
        R, L, c = self.ranks[r], self.ranks[r].lanes[b], self.cfg
        if not c.quit_enabled or c.baseline:
            return
        stuck = (not L.queue) or all(L.stall.get(i, 0) >= c.stall_limit for i in L.queue) or L.waiting
        if stuck and L.clock - L.last_fetch >= c.quit_idle:
            for coll in L.queue:              # contexts already saved at preemption
                way = coll % c.cache_ways
                ent = L.cache.get(way)
                if ent is not None and ent[0] == coll:
                    self._save_ctx(r, b, coll, ent[1])
            L.alive = False
            self.quits[r] += 1
            self._maybe_dead(r)

    def _maybe_dead(self, r):
        R = self.ranks[r]
        if not any(L.alive for L in R.lanes):
            R.alive = False

    # ------------------------------------------------------------------ driver
    def done(self) -> bool:
        return all(R.pc >= len(R.program) and R.completed == R.submitted for R in self.ranks)

    def _window(self) -> int:
        c = self.cfg
        if c.stuck_window:
            return c.stuck_window
        actors = self.n * (c.lanes + 1)
        spin = 2 if c.baseline else c.spin_cap + 2
        return 64 * actors * (spin + c.quit_idle + 4)

    def run(self):
        """Run until PASS; raise Deadlock if no progress for a full window."""
        actors = [("host", r, 0) for r in range(self.n)]
        actors += [("lane", r, b) for r in range(self.n) for b in range(self.cfg.lanes)]
        window = self._window()
        rr = 0
        while not self.done():
            self.tick += 1
            if self.tick > self.cfg.max_ticks:
                raise Deadlock("tick budget exhausted")
            for r in range(self.n):
                if self._supervisor(r):
                    self.last_progress = self.tick
            if self.cfg.scheduler == "random":
                kind, r, b = actors[self.rng.randrange(len(actors))]
            else:
                kind, r, b = actors[rr % len(actors)]
                rr += 1
            prog = self._host_step(r) if kind == "host" else self._lane_step(r, b)
            if prog:
                self.last_progress = self.tick
            elif self.tick - self.last_progress > window:
                raise Deadlock(f"no progress for {window} ticks at tick {self.tick}")
        return self

    def total_preemptions(self) -> int:
        return sum(self.preempt.values())


# ============================================================================ helpers
def plan_transfers(meta: CollMeta, n: int, cfg: SimConfig):
    """Planned slice transfers per (lane, step) for one submission: nloops * slices."""
    out = {}
    members = ring_members(meta, n)
    for r in members:
        rr, ns = members.index(r), len(members)
        for b in range(meta.nblocks):
            _, _, nloops = lane_geometry(meta, ns, rr, cfg)
            seq = ring.ring_sequence(meta.kind, ns, rr, meta.root, meta.inplace)
            for j in range(len(seq)):
                out[(r, b, j)] = nloops * cfg.slices_per_chunk
    return out


def make_buffers(meta: CollMeta, n: int, seed: int):
    """Per-rank (sendbuf, recvbuf) from the shared generator (nccl-tests conventions);
    for a sub-communicator, n is its ring size and index r its ring rank."""
    from inputs import hashgen
    xs = ring.inputs_full(meta.kind, meta.dtype, n, meta.count, seed, meta.coll_id)
    outs = []
    for r in range(n):
        if meta.kind == "allgather":
            rlen = meta.count * n
        else:
            rlen = meta.count
        rb = np.zeros(rlen, dtype=hashgen.NP_STORAGE[meta.dtype])
        if meta.inplace:
            if meta.kind in ("allreduce", "broadcast"):
                rb = xs[r]
            elif meta.kind == "allgather":
                rb[r * meta.count:(r + 1) * meta.count] = xs[r]
                xs[r] = rb[r * meta.count:(r + 1) * meta.count]
        outs.append(rb)
    return xs, outs


def run_orders(metas, orders, cfg: SimConfig, seed: int = 1, iterations: int = 1,
               sync_after_first: bool = False):
    """Every rank r submits metas in orders[r] (per iteration), then waits for all.
    Returns (sim, expected, buffers) -- caller checks results against O1."""
    n = len(orders)
    sim = Simulator(n, cfg)
    bufs = {}
    programs = [[] for _ in range(n)]
    for it in range(iterations):
        for m in metas:
            mem = ring_members(m, n)
            xs, outs = make_buffers(m, len(mem), seed + it)
            for k, r in enumerate(mem):
                bufs[(r, m.coll_id, it)] = (xs[k], outs[k])
        for r in range(n):
            for k, cid in enumerate(orders[r]):
                m = metas[cid]
                programs[r].append(("submit", m, *bufs[(r, cid, it)]))
                if sync_after_first and k == 0:
                    programs[r].append(("sync",))
            for cid in orders[r]:
                programs[r].append(("wait", cid))
    for r in range(n):
        sim.set_program(r, programs[r])
    sim.run()
    return sim, bufs
