"""Tensor-level wrappers over the counter-based generator (still no method arithmetic).

Every synthetic tensor of the workloads is addressed by (seed, tag, layer, owner, serial):
  * K / V rows of a file: owner = file id, serial = the token's append serial number, element
    counter = serial * Hkv * D + g * D + d  -> any token range is regenerated independently;
  * Q rows of a pred step: owner = file id, serial = (step, row) flattened by the caller.
"""
from __future__ import annotations

import numpy as np

from .gen import normal_bf16_np, normal_bf16_torch, stream_key

TAG_K, TAG_V, TAG_Q = 1, 2, 3


def rows_np(seed: int, tag: int, layer: int, owner: int, s0: int, s1: int, width: int,
            std: float = 1.0) -> np.ndarray:
    """uint16 bf16 bits [s1 - s0][width] for serials s0 .. s1-1."""
    key = stream_key(seed, tag, layer, owner)
    return normal_bf16_np(key, s0 * width, (s1 - s0) * width, std).reshape(s1 - s0, width)


def outlier_channels(bits: np.ndarray, D: int, channels, e: int) -> np.ndarray:
    """Outlier-channel inputs (real K caches carry a few channels of much larger magnitude, and Q follows
    them): multiply channels `channels` of every D-wide head of bf16 bit patterns [..][H*D] by 2^e, EXACTLY,
    by adding e to the exponent field of the nonzero values (the generator's values are normal and bounded,
    so nothing overflows or goes subnormal for |e| <= 30).  A power of two is used so both sides see the
    same bits without any rounding; no method arithmetic here."""
    b = np.array(bits, dtype=np.uint16, copy=True)
    w = b.shape[-1]
    cols = np.array([h * D + c for h in range(w // D) for c in channels], dtype=np.int64)
    sub = b[..., cols].astype(np.int32)
    nz = (sub & 0x7FFF) != 0
    ex = (sub >> 7) & 0xFF
    assert ((ex[nz] + e) > 0).all() and ((ex[nz] + e) < 255).all(), "outlier scaling leaves the normal range"
    sub = np.where(nz, (sub & ~(0xFF << 7)) | ((ex + e) << 7), sub)
    b[..., cols] = sub.astype(np.uint16)
    return b


def rows_torch(seed: int, tag: int, layer: int, owner: int, s0: int, s1: int, width: int,
               std: float = 1.0, device="cpu", out=None):
    """Same bits as rows_np as a torch.bfloat16 tensor [s1 - s0][width] (or written into `out`)."""
    key = stream_key(seed, tag, layer, owner)
    t = normal_bf16_torch(key, s0 * width, (s1 - s0) * width, std, device=device,
                          out=None if out is None else out.reshape(-1))
    return t.view(s1 - s0, width) if out is None else out


# ------------------------------------------------------------------ cfg5(ii) LIP eviction policy (inputs)
# a heavy-hitter-like replacement policy evicts the `drop` lowest-score tokens of a
# file, protecting the first `sink` and the last `recent` ones, ties to the lower index.  The scores are
# either synthetic (Exp(1), seeded) or a decode step's H2O scores; choosing the ranges from them is the LIP's
# policy (an INPUT to kvfs_evict), not KVFS arithmetic.
TAG_SCORE = 4


def lowest_score_ranges(scores, drop: int, sink: int = 4, recent: int = 1024) -> np.ndarray:
    """Sorted disjoint half-open logical ranges [a, b) covering the `drop` lowest scores (int64 [n][2])."""
    sc = np.array(scores, dtype=np.float64, copy=True)
    n = sc.shape[0]
    sc[:sink] = np.inf
    sc[max(0, n - recent):] = np.inf
    idx = np.sort(np.argsort(sc, kind="stable")[:drop])
    brk = np.nonzero(np.diff(idx) != 1)[0]
    starts = np.concatenate([[idx[0]], idx[brk + 1]])
    ends = np.concatenate([idx[brk], [idx[-1]]]) + 1
    return np.stack([starts, ends], axis=1).astype(np.int64)


def heavy_hitter_ranges(seed: int, f: int, n: int, drop: int, sink: int = 4, recent: int = 1024) -> np.ndarray:
    """cfg5(ii) with synthetic scores: Exp(1) per token of file f (stream (seed, TAG_SCORE, 0, f))."""
    from .gen import exp1_scores_np

    return lowest_score_ranges(exp1_scores_np(stream_key(seed, TAG_SCORE, 0, f), 0, n), drop, sink, recent)
