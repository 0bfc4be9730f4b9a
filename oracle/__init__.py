"""CPU oracle for the cascaded-columnar decode hot path -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this package.  It shares no code with paper_2602_08190_b200 (the product path never imports it).
See cdm_oracle.c's header for the paper passages each function follows and what pins it.
"""
from .oracle import decode_chunk, decode_many, OracleError, build, checksum  # noqa: F401
from .johnson import johnson_order, flow_shop_makespan, brute_force_best  # noqa: F401
