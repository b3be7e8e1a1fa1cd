"""Float64 CPU oracle for the Flash PD-SSM hot path (arXiv 2605.19150).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import anything
under ``oracle/``.  The product path (``paper_2605_19150_b200`` and its CUDA
library) never imports, links or executes this package, and this package never
imports the product path: the two share no code.

Every function is a plain, slow, obviously-correct transcription of a passage of
PAPER.md (cited in its docstring as ``PAPER.md:<line>``) in the scatter
(column-one-hot) convention adopted in DESIGN.md (reading R1).

Parity pins: every public function is pinned by ``tests/test_oracle_pins.py``
(dense-matrix products, closed forms, FSA emulation, S_5 group products via
sympy, finite differences, brute-force argmax).  No function is "parity
unpinned".
"""
from .pdssm_oracle import *  # noqa: F401,F403
from . import fsa  # noqa: F401
