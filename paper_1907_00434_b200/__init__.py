"""paper_1907_00434_b200 — B200-native MLfabric plan-execution hot path (arXiv 1907.00434).

The product: libmlfabric.so (include/mlfabric.h) — host C++ planner (Alg. 1-3,
App. B.2, §5.3) and sm_100a kernels (fused ordered commit, tree_reduce, mirror
store) — plus the thin ctypes binding in ``mlfabric``.  No CPU fallback: importing
``paper_1907_00434_b200.mlfabric`` without the built library raises ImportError.
"""
