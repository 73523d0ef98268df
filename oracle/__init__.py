"""ParoQuant fp64 CPU oracle -- TEST INFRASTRUCTURE, not product code.

May be imported only by tests/, __graft_entry__.smoke() and bench.py (cpu_baseline
and --impl reference legs).  Shares no code with paper_2511_10645_b200/.
See oracle/paro_oracle.py for the per-function paper citations.
"""
from .paro_oracle import (  # noqa: F401
    OracleError, validate_transform, givens_coefficients, apply_independent_rotations, fold,
    transform_activations, rtn_groups, dequantize, oracle_pack, oracle_linear, linear_fp,
    materialize, normwise_error, FP16_MIN_SUBNORMAL,
)
