"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation (Python + NumPy, fp64 for
reals, Python ints for hashing) of what the B200 hot path computes: the paper's
count-sketch (CS) and higher-order count-sketch (HCS) LSH hashers, the dense
E2LSH/SRP projection they replace, the (m, L) table keys, and the grouping of
points into the buckets of every table.

Citations: ``P:<line>`` = /root/reference/PAPER.md line (LaTeX source of
arXiv 2503.06737), ``S:<line>`` = SPEC.md line, ``B<k>`` = the reading listed in
DESIGN.md §"Readings of the paper" (same numbering as SURVEY.md §8(c)-B).

Rules this package obeys:
  * It shares no code, header, table or constant generator with the CUDA path
    (``paper_2503_06737_b200/``) and never imports it.
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import it.  The product path
    must never route through it.
  * Every function cites the passage it follows; where the paper is silent the
    DESIGN.md reading is cited instead.

Parity pins (tests/test_oracle_*.py, run with ``-m "not gpu"``) tie every
function to something other than itself: the paper's / SPEC's worked examples,
closed forms, exact enumeration, brute force (Kronecker products, dense
matrices), published test vectors of the named generators, and Monte-Carlo
checks of the collision laws.  Functions without such a pin are marked
"parity unpinned" below; there are none at present.
"""

from . import rng, lsh, theory  # noqa: F401
