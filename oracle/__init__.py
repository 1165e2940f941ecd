"""CPU checkers for the chunked backward-Euler path. TEST INFRASTRUCTURE ONLY.

Two implementations share one calling convention (the flat C types of
include/chunkode_b200.h):

* ``port``: the plain-C restatement ``oracle/src/cko_oracle.c`` built into
  ``oracle/_build/libcko_oracle.so`` (always available once built);
* ``ref``: the unmodified reference sources compiled into
  ``oracle/_ref/libchunkode_ref.so`` (built where /root/reference exists;
  the built file travels with the repo snapshot).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this package, and only as the checker or the
CPU baseline.
"""
from .bind import Oracle, load_port, load_ref, ref_available, build  # noqa: F401
