"""Pins of the oracle's attention (rule R10) and bf16 helpers (R12) against things other than itself:
a library routine (torch SDPA, fp64, explicit bottom-right mask, enable_gqa), closed forms, pure-Python
brute force on tiny inputs. CPU only."""
import math

import numpy as np
import pytest
import torch

from oracle.attention import brute_force_attention, gqa_attention
from oracle.bf16 import bf16_to_f64, f64_to_bf16_rne
from synth.workloads import TAG_K, TAG_Q, TAG_V, rows_np


def _sdpa(q, k, v, scale):
    """torch SDPA reference: q [n_q][Hq][D], k/v [len][Hkv][D] float64 -> out, lse."""
    n_q, hq, d = q.shape
    length, hkv, _ = k.shape
    tq = torch.from_numpy(q).permute(1, 0, 2)[None]  # [1][Hq][n_q][D]
    tk = torch.from_numpy(k).permute(1, 0, 2)[None]
    tv = torch.from_numpy(v).permute(1, 0, 2)[None]
    i = torch.arange(n_q)[:, None]
    j = torch.arange(length)[None, :]
    mask = j <= (length - n_q + i)  # bottom-right aligned causal (SURVEY §8(c) C4 gotcha)
    out = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, attn_mask=mask, scale=scale,
                                                           enable_gqa=True)
    # lse from the definition with torch ops (independent of the oracle's numpy path)
    rep = hq // hkv
    kk = tk.repeat_interleave(rep, dim=1)
    s = (tq @ kk.transpose(-1, -2)) * scale
    s = s.masked_fill(~mask, float("-inf"))
    lse = torch.logsumexp(s, dim=-1)
    return out[0].permute(1, 0, 2).numpy(), lse[0].permute(1, 0).numpy()


def _rand(seed, n_q, length, hq, hkv, d, qstd=1.0):
    q = bf16_to_f64(rows_np(seed, TAG_Q, 0, 0, 0, n_q, hq * d, qstd)).reshape(n_q, hq, d)
    k = bf16_to_f64(rows_np(seed, TAG_K, 0, 0, 0, length, hkv * d)).reshape(length, hkv, d)
    v = bf16_to_f64(rows_np(seed, TAG_V, 0, 0, 0, length, hkv * d)).reshape(length, hkv, d)
    return q, k, v


@pytest.mark.parametrize("n_q,length,hq,hkv,d,qstd", [
    (1, 1, 8, 2, 64, 1.0), (1, 37, 8, 2, 64, 1.0), (5, 40, 8, 2, 64, 4.0), (16, 16, 4, 4, 32, 1.0),
    (3, 300, 32, 8, 128, 1.0), (7, 129, 6, 3, 16, 4.0), (2, 50, 8, 1, 64, 1.0)])
def test_attention_matches_torch_sdpa(n_q, length, hq, hkv, d, qstd):
    q, k, v = _rand(11 + n_q + length, n_q, length, hq, hkv, d, qstd)
    scale = 1.0 / math.sqrt(d)
    out, lse = gqa_attention(q, k, v, scale)
    ref_out, ref_lse = _sdpa(q, k, v, scale)
    np.testing.assert_allclose(out, ref_out, rtol=0, atol=1e-12)
    np.testing.assert_allclose(lse, ref_lse, rtol=0, atol=1e-12)


def test_gqa_head_mapping_is_floor_division():
    """Distinct KV heads: head h must use KV head h // (Hq/Hkv) (repeat_interleave), not h % Hkv."""
    n_q, length, hq, hkv, d = 1, 5, 4, 2, 8
    q = np.ones((n_q, hq, d))
    k = np.zeros((length, hkv, d))
    v = np.zeros((length, hkv, d))
    v[:, 0, :] = 1.0
    v[:, 1, :] = 2.0
    out, _ = gqa_attention(q, k, v, 1.0)
    assert np.allclose(out[0, 0], 1.0) and np.allclose(out[0, 1], 1.0)
    assert np.allclose(out[0, 2], 2.0) and np.allclose(out[0, 3], 2.0)


def test_closed_form_single_key():
    """A fresh file plus one pred: softmax over one key is 1 => out = V_new exactly, lse = scale*<q,k>."""
    q, k, v = _rand(5, 1, 1, 8, 2, 64)
    out, lse = gqa_attention(q, k, v, 0.125)
    for h in range(8):
        g = h // 4
        assert np.array_equal(out[0, h], v[0, g])
        assert lse[0, h] == pytest.approx(0.125 * float(q[0, h] @ k[0, g]), abs=1e-12)


def test_closed_form_zero_query_counts_visible_keys():
    """Q = 0 => all visible scores are 0 => lse = ln|vis|, out = mean of the visible V rows."""
    n_q, length = 4, 23
    _, k, v = _rand(6, n_q, length, 8, 2, 64)
    q = np.zeros((n_q, 8, 64))
    out, lse = gqa_attention(q, k, v, 0.3)
    for i in range(n_q):
        n_vis = length - n_q + i + 1
        assert np.allclose(lse[i], math.log(n_vis), atol=1e-13, rtol=0)
        for h in range(8):
            assert np.allclose(out[i, h], v[:n_vis, h // 4].mean(axis=0), atol=1e-13, rtol=0)


def test_brute_force_tiny():
    q, k, v = _rand(7, 3, 6, 4, 2, 4, 4.0)
    out, lse = gqa_attention(q, k, v, 0.7)
    bo, bl = brute_force_attention(q.tolist(), k.tolist(), v.tolist(), 0.7)
    np.testing.assert_allclose(out, np.array(bo), atol=1e-12, rtol=0)
    np.testing.assert_allclose(lse, np.array(bl), atol=1e-12, rtol=0)


def test_bf16_roundtrip_and_rne():
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    f = bf16_to_f64(bits)
    finite = np.isfinite(f)
    back = f64_to_bf16_rne(f[finite][::97])
    np.testing.assert_array_equal(back, bits[finite][::97])
    # RNE against torch's float32 -> bfloat16 cast (exactly representable fp32 inputs, incl. ties)
    rng = np.random.default_rng(0)
    x32 = (rng.standard_normal(4000) * 3).astype(np.float32)
    ties = (bf16_to_f64(np.array([0x3F80, 0x3F81, 0x4000, 0xC001], np.uint16)).astype(np.float32)
            + np.float32(2.0 ** -8) * np.array([1, 1, 2, -2], np.float32))  # exact midpoints
    x32 = np.concatenate([x32, ties])
    ref = torch.from_numpy(x32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(f64_to_bf16_rne(x32.astype(np.float64)), ref)


# ------------------------------------------------------------------ NEXT-2 attention-score accumulation
from oracle.attention import attention_scores  # noqa: E402


def test_scores_zero_query_closed_form():
    """Q = 0: every visible key of row i has weight 1/|vis(i)| in each of the Hq heads."""
    n_q, length, hq, hkv, d = 3, 11, 4, 2, 8
    k = np.random.default_rng(0).normal(size=(length, hkv, d))
    sc = attention_scores(np.zeros((n_q, hq, d)), k, 0.3)
    ref = np.zeros(length)
    for i in range(n_q):
        nv = length - n_q + i + 1
        ref[:nv] += hq / nv
    assert np.allclose(sc, ref, rtol=0, atol=1e-14)


@pytest.mark.parametrize("n_q,length,hq,hkv", [(1, 50, 8, 2), (4, 33, 4, 4), (7, 64, 8, 1)])
def test_scores_match_torch_softmax_of_masked_matrix(n_q, length, hq, hkv):
    rng = np.random.default_rng(n_q * 100 + length)
    d = 16
    q = rng.normal(size=(n_q, hq, d))
    k = rng.normal(size=(length, hkv, d))
    scale = d ** -0.5
    qt = torch.from_numpy(q).permute(1, 0, 2)                      # [Hq][n_q][D]
    kt = torch.from_numpy(k).permute(1, 0, 2).repeat_interleave(hq // hkv, dim=0)  # [Hq][len][D]
    s = scale * qt @ kt.transpose(1, 2)                             # [Hq][n_q][len]
    mask = torch.ones(n_q, length, dtype=torch.bool).tril(diagonal=length - n_q)  # bottom-right causal
    w = torch.softmax(s.masked_fill(~mask, float("-inf")), dim=-1)
    ref = w.sum(dim=(0, 1)).numpy()
    sc = attention_scores(q, k, scale)
    assert np.allclose(sc, ref, rtol=0, atol=1e-12)
    assert math.isclose(sc.sum(), n_q * hq, rel_tol=1e-12)         # every (row, head) distribution sums to 1
