"""CPU FP64 oracle for arXiv 1912.05508 (recursive Gram-Schmidt QR + R-preconditioned CGLS).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything under ``oracle/``. The product
path (``paper_1912_05508_b200``) never imports it and shares no code with it.

Plain, slow, obviously-correct numpy in float64. Every function cites the PAPER.md passage
it follows; readings of silent/garbled passages are the R-A* entries of DESIGN.md §3.

Modules
-------
fp16         IEEE binary16 rounding and the per-column power-of-two range guard (R-A3, R-A4).
qr           Alg. 4 MGS, Eq. (6) CAQR panel, Alg. 2 recursive Gram-Schmidt (RGS).
householder  brute-force Householder QR / LS in loops (cross-check for tiny inputs).
cgls         corrected Alg. 5 (R-preconditioned CGLS) with the stop/restart rule (R-A10..A12).
metrics      backward error, orthogonality, R error, LLS optimality, flop conventions.
dist         the row-partitioned (P ranks) decomposition of the same algorithm, over an
             abstract communicator (used by the gloo world_size-2 tests).

Parity pins: every function is checked by ``tests/test_oracle_*.py`` against closed forms,
the paper's stated facts, brute force or invariants; none is "parity unpinned" except the
items listed in DESIGN.md §3.4 (tensor-core accumulation bits, MAGMA streams, cluster2).
"""
