"""oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the Winograd hot
path computes, written from PAPER.md (arxiv 1611.06565).  It exists to prove
the CUDA path right; it is not part of the product:

* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import, call, link or
  execute anything in this directory.
* It shares no code, header, table, constant generator or helper with
  ``paper_1611_06565_b200/`` and neither imports the other.  Seeded inputs
  come from ``paper_1611_06565_b200/workloads.py`` via the *tests*, which
  pass plain arrays in; the oracle itself never imports the product.

Modules
-------
direct     float64 direct N-D cross-correlation, Eq. (2) (C + OpenMP), and a
           pure-Python brute force for tiny inputs.
toomcook   exact-rational Toom-Cook / CRT synthesis of (A, B, C) (Sec. 2.1-2.2,
           Eq. (1), Algorithm 1, Theorem 1) and the exact identity check.
winograd   the N-D Winograd algorithm of Eq. (3)-(5) step by step (tiling,
           n-mode products, per-point matmul, inverse transform, stitch), in
           exact Fractions or float64: stage-level references.

Parity pins of every function are in tests/test_oracle_*.py; none is
"parity unpinned" ("Oracle and pins").
"""
