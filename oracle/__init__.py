"""CPU oracle for PHIKS — TEST INFRASTRUCTURE ONLY.

Plain, slow, fp64/complex128 numpy implementation of what the paper's method
computes, written from PAPER.md.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import it.  The
product path (`paper_2210_07667_b200`) never imports, calls or links anything
here, and this package never imports the product path (only the seeded input
generators in `paper_2210_07667_b200.workloads`, which hold no method
arithmetic).
"""
from .phiks_oracle import *  # noqa: F401,F403
