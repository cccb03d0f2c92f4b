"""CPU oracle of the PSP-GMRES hot path (arXiv 1308.5626).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this package.
It never imports the product package ``paper_1308_5626_b200``.
"""
from .oracle import *  # noqa: F401,F403
