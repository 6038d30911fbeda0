"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation of what the AlphaSparse hot path
computes (arXiv 2212.10432, /root/reference/PAPER.md = "P:<line>").  It shares no code
with the CUDA path (`paper_2212_10432_b200/`) and neither imports the other.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import, call, link or execute anything under `oracle/`.
The product path never routes through it.

Modules
  graph_ref   operator-graph DSL parser, canonical printer, dependency validator
              (P:36 draft §Operator, §IV-B; readings A16/A37 in DESIGN.md)
  builder_ref reference Matrix-Metadata-Set builder: converting / mapping /
              implementing operators executed in order
  spmv_ref.c  long-double CSR SpMV  y = alpha*A*x + beta*y  with per-row error bound
              ("y=Ax"; north_star tolerances)  — loaded by `spmv`
  spmv        ctypes loader + acceptance check
  mtx_ref     Matrix Market parser, COO canonicaliser, row statistics (P:2)

Parity status per function is listed in DESIGN.md §Oracle; functions with no external
pin say "parity unpinned" in their docstring.
"""
