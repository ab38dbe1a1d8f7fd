"""fp64 CPU oracle for the PVR SR iteration — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package. The product package (paper_1611_07289_b200) never
imports it and shares no code with it. See oracle/pvro.h for what it computes and
which PAPER.md passages each function restates.
"""
from .pvro import Oracle, build, lib  # noqa: F401
