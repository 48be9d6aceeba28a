"""Seeded synthetic-input generators (shared by the oracle tests, the CUDA-path tests and bench.py).

This package holds NONE of the method's arithmetic (no attention, no paging rules). It only turns
(seed, stream ids, element counters) into bf16 bit patterns with a counter-based integer hash, so that
any sub-range of any tensor can be regenerated independently on the host (numpy) or on the device
(torch) with bit-identical results. See DESIGN.md "Input recipe".
"""
from .gen import (  # noqa: F401
    stream_key,
    normal_bf16_np,
    normal_bf16_torch,
    uniform_u32_np,
    exp1_scores_np,
)
