"""MLfabric CPU oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct implementation of what the MLfabric hot path
computes (arXiv 1907.00434, /root/reference/PAPER.md cited as P:line), written
from the paper before any kernel.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product path (``paper_1907_00434_b200``) never imports, calls or links it;
the two share no code.  The only shared module is ``synthgen`` (seeded input
generation, none of the method's arithmetic).

Modules
  netmodel     O1/O2  network model, t_en water-filling (Fig. 5b), NetUp (Fig. 5c)
  ordering     O3     deadlines + Alg. 1 ShrtUp + Alg. 2 look-ahead drops; App. B.2
  aggregation  O4     Alg. 3 DetAgg + enumeration over n
  replication  O5     §5.3 tentative replica plan, T_last, divergence bound, freeze/punt/delay
  plan         -      the full per-batch pipeline -> integer plan (mirror of mlf_plan)
  numerics     O6     ordered commit w <- w - lr*x, in-group left fold, mirror backup
  checks       O7     delay invariant, plan well-formedness
  bruteforce   O8     exhaustive orderings / partitions for <= 5 updates (App. B.1 objectives)

Readings of silent / ambiguous passages (R1-R20) are listed in DESIGN.md §3 and
cited at the point of use.  Parity status per function is in each module
header; "parity unpinned" items are repeated in DESIGN.md.
"""
