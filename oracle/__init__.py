"""Oracle: plain, slow, obviously-correct fp64 CPU implementation of the method.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import anything
under `oracle/`.  The product path (`paper_2204_05988_b200/`) never imports it
and shares no code with it; the two meet only in `sginputs/` (plain problem
data + seeded random inputs).

Every function cites the PAPER.md passage it follows (line numbers refer to
/root/reference/PAPER.md, the LaTeX of arXiv:2204.05988).  Readings of
ambiguous/garbled passages are listed in DESIGN.md ("Readings R1..").

Modules
  mesh      nested structured P1 meshes + embedding E (sec. 2 l.64-67, sec. 4.2 l.506)
  fem       exact factor matrices (eq. (14) l.450-461, l.486-504), quadrature loads
  problem   time basis (l.441-448), Kronecker expansion of A^(delta) (l.462-477)
  sgrid     sparse-grid blocks, cross-level blocks (l.506-516), Richardson +
            combination preconditioner (sec. 4.3 l.540-566), time stepping (eq. (4))

Parity status: every function is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py; none is "parity unpinned".
"""
