"""Counter-based synthetic input generator: bf16 bit patterns, bit-identical on numpy and torch.

Recipe:
  key      = stream_key(seed, tag, layer, file, ...)            (32-bit, hashed)
  h_j(c)   = H(key ^ H(2c + j)),  j in {0, 1}                    (H = 32-bit integer avalanche hash)
  s(c)     = sum of the four 16-bit halves of h_0(c), h_1(c)  -  2*65535   (Irwin-Hall(4), exact int)
  x(c)     = fp32(s(c)) * fp32(std / sigma_IH)                   (one IEEE fp32 multiply, RNE)
  bits(c)  = bf16 round-to-nearest-even of x(c), done with integer ops on the fp32 bits
where sigma_IH = sqrt(4 * (65536^2 - 1) / 12) is the standard deviation of s.  x is an
approximately N(0, std^2) variate bounded at +-3.46 std.  Every step is integer arithmetic or a
single IEEE fp32 multiply, so numpy (host) and torch (CPU or CUDA) produce the same bits.

No attention / paging arithmetic lives here.
"""
from __future__ import annotations

import math

import numpy as np

M32 = 0xFFFFFFFF
_C1 = 0x7FEB352D
_C2 = 0x846CA68B
_SIGMA_IH = math.sqrt(4.0 * (65536.0 ** 2 - 1.0) / 12.0)


def _scale_f32(std: float) -> np.float32:
    return np.float32(std / _SIGMA_IH)


# ----------------------------------------------------------------------------------- numpy (host)
def _mul32_np(x: np.ndarray, c: int) -> np.ndarray:
    lo, hi = c & 0xFFFF, c >> 16
    return (x * np.uint64(lo) + (((x * np.uint64(hi)) & np.uint64(0xFFFF)) << np.uint64(16))) & np.uint64(M32)


def _hash_np(x: np.ndarray) -> np.ndarray:
    x = x & np.uint64(M32)
    x ^= x >> np.uint64(16)
    x = _mul32_np(x, _C1)
    x ^= x >> np.uint64(15)
    x = _mul32_np(x, _C2)
    x ^= x >> np.uint64(16)
    return x


def _hash_int(v: int) -> int:
    return int(_hash_np(np.array([v & M32], dtype=np.uint64))[0])


def stream_key(seed: int, *ids: int) -> int:
    """32-bit stream key from a seed and a tuple of non-negative integer ids."""
    k = _hash_int(seed & M32)
    for i in ids:
        k = _hash_int(k ^ _hash_int(int(i) & M32))
    return k


def uniform_u32_np(key: int, start: int, count: int) -> np.ndarray:
    """count uniform 32-bit integers (as uint64) for counters start .. start+count-1."""
    c = np.arange(start, start + count, dtype=np.uint64)
    return _hash_np(np.uint64(key) ^ _hash_np(c))


def normal_bf16_np(key: int, start: int, count: int, std: float = 1.0) -> np.ndarray:
    """bf16 bit patterns (uint16) of approx N(0, std^2) variates for counters start..start+count-1."""
    assert 0 <= start and start + count <= (1 << 30), "counter range exceeds 2^30"
    c = np.arange(start, start + count, dtype=np.uint64)
    key64 = np.uint64(key)
    h0 = _hash_np(key64 ^ _hash_np(c * np.uint64(2)))
    h1 = _hash_np(key64 ^ _hash_np(c * np.uint64(2) + np.uint64(1)))
    m16 = np.uint64(0xFFFF)
    s = ((h0 & m16) + (h0 >> np.uint64(16)) + (h1 & m16) + (h1 >> np.uint64(16))).astype(np.int64) - 131070
    x = s.astype(np.float32) * _scale_f32(std)
    b = x.view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return (r & m16).astype(np.uint16)


def exp1_scores_np(key: int, start: int, count: int) -> np.ndarray:
    """Exp(1) synthetic 'importance' scores (float64) for heavy-hitter-like eviction policies."""
    u = (uniform_u32_np(key, start, count).astype(np.float64) + 0.5) / 4294967296.0
    return -np.log(u)


# ----------------------------------------------------------------------------------- torch (device)
def _mul32_t(x, c: int):
    lo, hi = c & 0xFFFF, c >> 16
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & M32


def _hash_t(x):
    x = x & M32
    x = x ^ (x >> 16)
    x = _mul32_t(x, _C1)
    x = x ^ (x >> 15)
    x = _mul32_t(x, _C2)
    x = x ^ (x >> 16)
    return x


def normal_bf16_torch(key: int, start: int, count: int, std: float = 1.0, device="cpu", out=None,
                      chunk: int = 1 << 24):
    """Same bits as normal_bf16_np, produced by torch integer ops (CPU or CUDA).

    Returns a torch.bfloat16 tensor of shape [count] (or fills `out`, a contiguous bf16 tensor)."""
    import torch

    assert 0 <= start and start + count <= (1 << 30), "counter range exceeds 2^30"
    if out is None:
        out = torch.empty(count, dtype=torch.bfloat16, device=device)
    flat = out.view(-1).view(torch.int16)
    assert flat.numel() == count
    scale = torch.tensor(float(_scale_f32(std)), dtype=torch.float32, device=flat.device)
    for b in range(0, count, chunk):
        n = min(chunk, count - b)
        c = torch.arange(start + b, start + b + n, dtype=torch.int64, device=flat.device)
        h0 = _hash_t(key ^ _hash_t(c * 2))
        h1 = _hash_t(key ^ _hash_t(c * 2 + 1))
        s = (h0 & 0xFFFF) + (h0 >> 16) + (h1 & 0xFFFF) + (h1 >> 16) - 131070
        x = s.to(torch.float32) * scale
        bits = x.view(torch.int32).to(torch.int64) & M32
        r = ((bits + 0x7FFF + ((bits >> 16) & 1)) >> 16) & 0xFFFF
        r = r - ((r >> 15) << 16)  # to signed 16-bit range without relying on narrowing casts
        flat[b:b + n] = r.to(torch.int16)
    return out
