"""fp64 CPU oracle of the DTS-Gate MoE layer -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
may import this package.  It shares no code with paper_2112_14397_b200/.
"""
from . import dts_moe  # noqa: F401
