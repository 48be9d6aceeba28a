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


def rows_torch(seed: int, tag: int, layer: int, owner: int, s0: int, s1: int, width: int,
               std: float = 1.0, device="cpu", out=None):
    """Same bits as rows_np as a torch.bfloat16 tensor [s1 - s0][width] (or written into `out`)."""
    key = stream_key(seed, tag, layer, owner)
    t = normal_bf16_torch(key, s0 * width, (s1 - s0) * width, std, device=device,
                          out=None if out is None else out.reshape(-1))
    return t.view(s1 - s0, width) if out is None else out
