"""fp64 CPU oracle for the B-KFAC hot path.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2210_08494_b200``) never imports it and shares no code with it.
"""
from .bkfac_oracle import *  # noqa: F401,F403
