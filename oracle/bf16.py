"""bf16 helpers for the oracle (rule R12): K/V/Q are bf16 bit patterns; the output is
the bf16 round-to-nearest-even of the exact result.

Pinned by: tests/test_oracle_pins.py::test_bf16_roundtrip_and_rne (every bf16 bit pattern round-trips;
RNE agrees with torch's float32->bfloat16 cast on ties and non-ties).
"""
from __future__ import annotations

import numpy as np


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    """uint16 bf16 bit patterns -> float64 (exact: bf16 is the top half of an fp32)."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32).astype(np.float64)


def f64_to_bf16_rne(x: np.ndarray) -> np.ndarray:
    """float64 -> bf16 bits, rounding to nearest even directly from the float64 value.

    Written from the definition: the two bf16 neighbours of x are found from its fp32-truncation and the
    nearer one is taken, ties to the even mantissa. (Rounding fp64->fp32->bf16 would double-round.)"""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty(x.shape, dtype=np.uint16)
    flat_x = x.reshape(-1)
    flat_o = out.reshape(-1)
    for i, v in enumerate(flat_x):
        if v != v:
            flat_o[i] = 0x7FC0
            continue
        # candidate below/above |v| in bf16 (sign handled separately)
        s = 0x8000 if (v < 0 or (v == 0 and np.signbit(v))) else 0
        a = abs(v)
        # truncate to bf16 toward zero: largest bf16 <= a
        f32 = np.float32(a)
        if float(f32) > a:  # fp32 rounding went up; step down one fp32 ulp
            f32 = np.nextafter(f32, np.float32(0))
        lo_bits = int(np.array(f32, dtype=np.float32).view(np.uint32)) >> 16
        lo = float(bf16_to_f64(np.array([lo_bits], dtype=np.uint16))[0])
        if lo == a:
            flat_o[i] = s | lo_bits
            continue
        hi_bits = lo_bits + 1
        hi = float(bf16_to_f64(np.array([hi_bits], dtype=np.uint16))[0])
        if a - lo < hi - a:
            pick = lo_bits
        elif a - lo > hi - a:
            pick = hi_bits
        else:
            pick = lo_bits if (lo_bits & 1) == 0 else hi_bits
        flat_o[i] = s | pick
    return out
