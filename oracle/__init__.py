"""Brute-force CPU oracle for the GRCA hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with ``paper_2605_10457_b200`` (neither imports the other).

See ``oracle/grca_oracle.c`` for the definition it implements (PAPER.md
Eq. 1 at 150-157, Eq. ray_dir at 418-423, Moller-Trumbore at 756) and
``oracle/compare.py`` for the parity contract (SURVEY 8c comparator).
"""
from .oracle import (  # noqa: F401
    build_oracle,
    cast,
    lib_path,
    mt,
    n_rays,
    near_edge_count,
    ray_table,
    ray_tri,
)
from .compare import compare  # noqa: F401
