"""Seeded synthetic input generators shared by the oracle side and the GPU side.

This package holds NO arithmetic of the method (no reduction, no ring order,
no geometry).  It only produces deterministic inputs and workload recipes:

* :mod:`inputs.hashgen`   -- counter-based per-element values x_r[i]
                            (splitmix64 of a key; SURVEY.md §8(c) "Inputs").
* :mod:`inputs.workloads` -- the C1..C4 workload recipes of BASELINE.json
                            (sizes, per-rank submission orders).

Both ``oracle/`` and the CUDA-side test/bench harness import from here; the
CUDA side also has its own implementation of the same generator
(``paper_2303_06324_b200/csrc/testgen.cu``) so that full-size inputs can be
produced in HBM without a host round trip.
"""
