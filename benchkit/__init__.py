"""bench.py's harness (timing legs, denominators, clocks).  Not product code: the product is
paper_1907_00434_b200/ (the C-ABI library and its binding); nothing in the package imports this."""
