"""CPU oracle for the BDDC-preconditioned CG of arXiv 2304.09770 (3D divergence-free VEM Stokes).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this package.
The product path (`paper_2304_09770_b200/`, `csrc/`) never imports, links or
executes anything here, and this package never imports the product path; both
read their inputs from `synthetic/` only.

Plain, slow, fp64 NumPy/SciPy, written from PAPER.md in the paper's order and
notation.  `P:n` = /root/reference/PAPER.md line n.  Every function cites the
passage it follows.  Readings of silent/garbled passages are SURVEY.md §8(c)
A1-A23 and are listed in DESIGN.md.

Parity status: every function is pinned by tests/test_oracle_*.py except the
D-recipe constant and the DOF normalisations, which the paper does not state
("parity unpinned", DESIGN.md §Readings A13/A14).
"""
