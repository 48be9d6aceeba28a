"""Rule R10: attention of a `pred` over a KVFS file, in float64.

PAPER.md §4.1: pred(kv, tokens, positions) updates the file "with new tensors corresponding to
the provided tokens" and returns a result "for each input token"; §2.1: a token's K/V "depend solely
on preceding tokens in causal Transformers"; §4.2: pruned tokens are removed from the file.
Reading (Z3-Z5): after the append the file holds `len` retained tokens in logical order, the
n_q new ones last; query row i (0-based) sees logical keys 0 .. len - n_q + i (bottom-right-aligned
causal), head h uses KV head g = floor(h / (Hq / Hkv)) (GQA), and

    s_k      = scale * <Q[i,h,:], K[k,g,:]>
    out[i,h] = sum_k softmax_k(s)_k * V[k,g,:]        lse[i,h] = log(sum_k exp(s_k))

Pinned by tests/test_oracle_pins.py: torch SDPA (fp64, explicit bottom-right mask, enable_gqa) on random
inputs; closed forms (single key => out = V, lse = s; Q = 0 => lse = ln|vis|, out = mean V);
brute-force pure-Python loops on tiny inputs; evict/truncate equivalence (tests/test_oracle_kvfs.py).
"""
from __future__ import annotations

import numpy as np

from .bf16 import bf16_to_f64


def gqa_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float):
    """q [n_q][Hq][D], k/v [len][Hkv][D] (float64, the file's retained tokens in logical order, the
    n_q query tokens being the last n_q keys). Returns out [n_q][Hq][D] float64, lse [n_q][Hq] float64."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    n_q, hq, d = q.shape
    length, hkv, d2 = k.shape
    assert d == d2 and v.shape == k.shape and hq % hkv == 0 and n_q <= length
    group = hq // hkv
    out = np.zeros((n_q, hq, d), dtype=np.float64)
    lse = np.zeros((n_q, hq), dtype=np.float64)
    for i in range(n_q):
        n_vis = length - n_q + i + 1  # keys 0 .. len - n_q + i
        for h in range(hq):
            g = h // group
            s = scale * (k[:n_vis, g, :] @ q[i, h, :])
            m = s.max()
            p = np.exp(s - m)
            l_sum = p.sum()
            out[i, h, :] = (p / l_sum) @ v[:n_vis, g, :]
            lse[i, h] = m + np.log(l_sum)
    return out, lse


def attention_scores(q: np.ndarray, k: np.ndarray, scale: float) -> np.ndarray:
    """NEXT-2 (H2O, §6): per retained key k (logical order) the softmax weight of R10 summed
    over the query rows i and the Hq heads (0 where row i cannot see k).  q [n_q][Hq][D], k [len][Hkv][D]
    float64.  Pinned by tests/test_oracle_pins.py: Q = 0 closed form (uniform weights 1/|vis(i)|), the
    total = n_q * Hq, and torch.softmax over an explicitly masked dense score matrix."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    n_q, hq, d = q.shape
    length, hkv, _ = k.shape
    group = hq // hkv
    acc = np.zeros(length, dtype=np.float64)
    for i in range(n_q):
        n_vis = length - n_q + i + 1
        for h in range(hq):
            s = scale * (k[:n_vis, h // group, :] @ q[i, h, :])
            p = np.exp(s - s.max())
            acc[:n_vis] += p / p.sum()
    return acc


def attention_over_file(q_bits: np.ndarray, k_bits: np.ndarray, v_bits: np.ndarray, scale: float):
    """Same as gqa_attention on bf16 bit-pattern inputs (uint16)."""
    return gqa_attention(bf16_to_f64(q_bits), bf16_to_f64(k_bits), bf16_to_f64(v_bits), scale)


def brute_force_attention(q, k, v, scale):
    """Pure-Python loops (no NumPy reductions) for tiny inputs; an independent re-derivation of R10."""
    import math

    n_q, hq, d = len(q), len(q[0]), len(q[0][0])
    length, hkv = len(k), len(k[0])
    group = hq // hkv
    out = [[[0.0] * d for _ in range(hq)] for _ in range(n_q)]
    lse = [[0.0] * hq for _ in range(n_q)]
    for i in range(n_q):
        for h in range(hq):
            g = h // group
            scores = []
            for key in range(length - n_q + i + 1):
                acc = 0.0
                for j in range(d):
                    acc += float(q[i][h][j]) * float(k[key][g][j])
                scores.append(scale * acc)
            mx = max(scores)
            w = [math.exp(s - mx) for s in scores]
            tot = sum(w)
            for j in range(d):
                out[i][h][j] = sum(w[key] * float(v[key][g][j]) for key in range(len(w))) / tot
            lse[i][h] = mx + math.log(tot)
    return out, lse
