"""CPU oracle for the p-multigrid hot path of arXiv 1808.03595 (Huismann, Stiller, Froehlich).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything from this package.  The
CUDA product path (``paper_1808_03595_b200``) never imports it and shares no code with it.

The oracle is deliberately plain and slow: dense element matrices built from Kronecker
products, dense Schur complements, dense LU inverses of every star block, explicit
interpolation matrices and their explicit transposes.  Every function cites the passage of
``PAPER.md`` (P:line) that defines it; where the paper is silent or garbled the reading is
the one listed in ``DESIGN.md`` ("Readings").  All arithmetic is float64.

Vectors are stored on the global tensor-product GLL grid (index [i3, i2, i1], x1 fastest,
N_d = k_d p + 1 points per direction, boundary included).  A condensed ("hat") vector is a
grid vector that is non-zero only on free skeleton points (element-boundary points that are
not on the Dirichlet boundary).

Parity status: every public function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` against closed forms, brute force or the paper's printed numbers;
none is "parity unpinned" except the iteration counts of BASELINE configs the paper never
ran.
"""
from . import gll, mesh, condensed, smoother, transfer, mg  # noqa: F401
