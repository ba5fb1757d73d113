"""CPU oracle for RedSync RGC (arXiv 1808.04357).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_1808_04357_b200`` and never imports
it.  See ``rgc_oracle.c`` for the citations (PAPER.md line numbers).
"""
from .oracle import *  # noqa: F401,F403
