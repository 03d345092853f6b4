"""CPU oracle for the OCCL hot path (arXiv 2303.06324).  TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The product
path (``paper_2303_06324_b200``) never imports it and shares no code with it.

Two independent halves:

* :mod:`oracle.ring` (O1) -- the plain definition of each collective's result,
  written as the ring's left fold in the ring's reduction order, per dtype.
* :mod:`oracle.dfce` (O2) -- a slow, deterministic multi-rank simulator of the
  paper's deadlock-free collective execution framework (daemon, task queue,
  spin thresholds, context save/restore, SQ/CQ, voluntary quit, event-driven
  restart, stickiness), which *executes* the primitive sequences over bounded
  connectors.  O1 == O2 bit-exactly is one of the pins.

Parity pins live in ``tests/test_oracle_*.py`` (``-m "not gpu"``).
Parity unpinned (timing-dependent, reported only): preemption counts,
task-queue-length traces and stickiness speed-ups produced by O2.
"""
