"""TEST INFRASTRUCTURE — the CPU float64 checker for the DUFWI physics step.

Nothing in ``paper_2603_04070_b200`` imports this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it, and only as the thing results are
checked against or the CPU baseline that is timed — never as a product path.

Parity is PINNED: ``oracle/make_golden.py`` imports the reference package
(``fwilab`` from ``/root/reference/pkg/src``) in the build container, runs it on
seeded inputs and writes the fixtures under ``tests/golden/``; the CPU test
suite asserts the restatement here reproduces those fixtures bit for bit.
"""

from .dufwi_oracle import *  # noqa: F401,F403
