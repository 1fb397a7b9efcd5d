"""TEST INFRASTRUCTURE — the CPU oracle. Not product code.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker / the CPU
baseline. Two interchangeable backends with the same API:

  * ``Oracle("ref")``  — oracle/_ref/libprrtc_ref.so: the UNMODIFIED reference
    sources (/root/reference/proj/src) compiled by oracle/Makefile behind the
    extern "C" wrapper oracle/ref_capi.cpp.
  * ``Oracle("port")`` — oracle/liboracle.so: the C restatement
    oracle/prrtc_oracle.c (pinned against the reference build and the golden
    fixtures in tests/golden/).
"""
from .binding import Oracle, available  # noqa: F401
