"""CPU oracle for CPA singular-value shrinkage (arXiv 1705.07112).

TEST INFRASTRUCTURE ONLY.  This package is the plain, slow, fp64 reference
that the CUDA path is checked against.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
(``paper_1705_07112_b200``) never imports it and shares no code with it.

Every function cites the PAPER.md passage it follows (``PAPER.md:<line>``,
with the equation label of the LaTeX source).  Where the paper is silent the
reading taken is the one listed in DESIGN.md §"Readings of the paper".

Pins: every function here is pinned by ``tests/test_oracle_pins.py``
(closed forms, invariants, brute force, library special cases).  The paper
prints no worked example of the coefficients, of Lambda_max or of any
shrinkage output, so no pin is a printed paper value.
"""

from .cpa_oracle import *  # noqa: F401,F403
