"""CPU oracle for Kronecker-sparse matmul -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2405_15013_b200``) never imports it and shares no code
with it.  See ``oracle/ks_oracle.py`` for what each function follows.
"""
from .ks_oracle import *  # noqa: F401,F403
