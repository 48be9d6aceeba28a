"""Pins of the oracle's extract (R13) and merge (R14): PAPER.md §4.2 P:225 "create new files from existing
ones by extracting specific token indices with extract, or merging existing files into one with merge";
SPEC S:90-106 worked examples (each cited below), page arithmetic, atomic failure, source isolation, and
attention over the new file = dense attention over the selected / merged token list (R10). CPU only."""
import random

import numpy as np
import pytest
import torch

from oracle import EBADF, EBUSY, EEXIST, EINVAL, ENOSPC, EPOS, ERANGE, KvfsError, Oracle
from oracle.bf16 import bf16_to_f64
from synth.workloads import TAG_K, TAG_Q, TAG_V, rows_np


def _kv(seed, s0, n, hkv=2, d=8):
    k = rows_np(seed, TAG_K, 0, 0, s0, s0 + n, hkv * d).reshape(1, n, hkv, d)
    v = rows_np(seed, TAG_V, 0, 0, s0, s0 + n, hkv * d).reshape(1, n, hkv, d)
    return k, v


def _file(o, name, pos, seed=1, s0=0):
    fd = o.open(name)
    k, v = _kv(seed, s0, len(pos))
    o.append(fd, pos, k, v)
    return fd, k[0], v[0]


def test_spec_s97_extract_all_is_identical_copy_without_sharing():
    o = Oracle(40, 16, 1, 2, 8)
    a, k, v = _file(o, "a", list(range(0, 100, 3)))  # 34 tokens, positions with gaps
    n = o.stat(a)[0]
    b = o.extract(a, list(range(n)), "b")
    assert o.positions(b) == o.positions(a)
    kb, vb = o.read(b, 0, 0, n)
    assert np.array_equal(kb, k) and np.array_equal(vb, v)
    pa = {p for p, _ in o.table(a)}
    pb = {p for p, _ in o.table(b)}
    assert not (pa & pb)  # pages rebuilt: no sharing
    assert all(o.refcnt[p] == 1 for p in pa | pb)
    o.audit()


def test_spec_s98_extract_empty():
    o = Oracle(8, 16, 1, 2, 8)
    a, _, _ = _file(o, "a", list(range(20)))
    free = o.free_count()
    b = o.extract(a, [], "b")
    assert o.stat(b) == (0, 0, -1) and o.table(b) == [] and o.free_count() == free


def test_spec_s99_extract_even_indices_of_10():
    o = Oracle(8, 16, 1, 2, 8)
    pos = [3, 4, 8, 11, 12, 20, 21, 22, 30, 41]
    a, k, v = _file(o, "a", pos)
    b = o.extract(a, [0, 2, 4, 6, 8], "b")
    assert o.positions(b) == [3, 8, 12, 21, 30]
    kb, vb = o.read(b, 0, 0, 5)
    assert np.array_equal(kb, k[0::2]) and np.array_equal(vb, v[0::2])
    assert o.table(b) == [(o.table(b)[0][0], 0x1F)]  # 5 tokens, one fresh page, slots 0..4


def test_extract_page_arithmetic_s62_and_r1():
    """3000 tokens -> ceil(3000/16) = 188 pages (S:62 arithmetic), smallest-free ids in logical order (R1)."""
    o = Oracle(400, 16, store_data=False)
    a = o.open("a")
    o.append(a, list(range(3000)))
    assert len(o.table(a)) == 188
    o.evict(a, [(100, 200)])  # tokens 112..191 were pages 7..11: freed
    b = o.extract(a, list(range(2900)), "b")
    t = o.table(b)
    # 2900 -> 182 pages, smallest free first: the 5 freed ids, then 188, 189, ...
    assert [p for p, _ in t] == [7, 8, 9, 10, 11] + list(range(188, 188 + 177))
    assert all(m == 0xFFFF for _, m in t[:-1]) and t[-1][1] == (1 << (2900 - 181 * 16)) - 1


def test_spec_s104_merge_disjoint():
    o = Oracle(8, 16, 1, 2, 8)
    a, ka, va = _file(o, "A", list(range(10)), s0=0)
    b, kb, vb = _file(o, "B", list(range(10, 20)), s0=100)
    m = o.merge([a, b], "M")
    assert o.positions(m) == list(range(20))
    km, vm = o.read(m, 0, 0, 20)
    assert np.array_equal(km, np.concatenate([ka, kb])) and np.array_equal(vm, np.concatenate([va, vb]))


def test_spec_s105_merge_overlap_rejected_atomically():
    o = Oracle(8, 16, 1, 2, 8)
    a, _, _ = _file(o, "A", [1, 5, 9])
    b, _, _ = _file(o, "B", [2, 5])
    snap = (list(o.refcnt), o.free_count())
    with pytest.raises(KvfsError) as e:
        o.merge([a, b], "M")
    assert e.value.code == EPOS
    assert (list(o.refcnt), o.free_count()) == snap and "M" not in o.names


def test_spec_s106_merge_order_independent_and_interleaved():
    o = Oracle(16, 16, 1, 2, 8)
    a, ka, _ = _file(o, "A", [0, 2, 4, 6, 40], s0=0)
    b, kb, _ = _file(o, "B", [1, 3, 5, 39], s0=50)
    m1 = o.merge([a, b], "M1")
    m2 = o.merge([b, a], "M2")
    assert o.positions(m1) == o.positions(m2) == [0, 1, 2, 3, 4, 5, 6, 39, 40]
    k1, v1 = o.read(m1, 0, 0, 9)
    k2, v2 = o.read(m2, 0, 0, 9)
    assert np.array_equal(k1, k2) and np.array_equal(v1, v2)
    order = [ka[0], kb[0], ka[1], kb[1], ka[2], kb[2], ka[3], kb[3], ka[4]]
    assert np.array_equal(k1, np.stack(order))


def test_extract_merge_errors():
    o = Oracle(4, 16, store_data=False)
    a = o.open("a")
    o.append(a, list(range(40)))  # 3 pages, 1 free
    for idx, code in (([3, 3], EINVAL), ([5, 2], EINVAL), ([0, 40], ERANGE), ([-1], ERANGE)):
        with pytest.raises(KvfsError) as e:
            o.extract(a, idx, "x")
        assert e.value.code == code
    with pytest.raises(KvfsError) as e:
        o.extract(a, [0], "a")
    assert e.value.code == EEXIST
    with pytest.raises(KvfsError) as e:
        o.extract(a, list(range(17)), "x")  # needs 2 pages, 1 free
    assert e.value.code == ENOSPC
    with pytest.raises(KvfsError) as e:
        o.merge([a, 77], "x")
    assert e.value.code == EBADF
    with pytest.raises(KvfsError) as e:
        o.merge([a, a], "x")
    assert e.value.code == EBUSY
    assert o.free_count() == 1 and "x" not in o.names
    o.audit()


def test_extract_merge_source_isolation():
    """The sources keep their tables, positions and bits; later ops on the new file never touch them."""
    o = Oracle(32, 16, 1, 2, 8)
    a, k, v = _file(o, "a", list(range(50)))
    b = o.fork(a, "b")
    t_a, t_b = o.table(a), o.table(b)
    x = o.extract(b, list(range(10, 30)), "x")
    o.evict(x, [(0, 5)])
    k2, v2 = _kv(9, 1000, 3)
    o.append(x, [100, 101, 102], k2, v2)
    assert o.table(a) == t_a and o.table(b) == t_b
    ka, va = o.read(a, 0, 0, 50)
    assert np.array_equal(ka, k) and np.array_equal(va, v)


@pytest.mark.parametrize("seed", range(6))
def test_attention_over_extracted_and_merged_equals_dense(seed):
    """R10 over the new file = torch SDPA (fp64) over the selected / merged token list, q after the last."""
    rnd = random.Random(seed)
    Hq, Hkv, D = 4, 2, 8
    o = Oracle(64, 16, 1, Hkv, D)
    pos_a = sorted(rnd.sample(range(0, 300), 60))
    pos_b = sorted(rnd.sample([p for p in range(0, 300) if p not in pos_a], 40))
    a, ka, va = _file(o, "a", pos_a, seed)
    b, kb, vb = _file(o, "b", pos_b, seed, s0=500)
    sel = sorted(rnd.sample(range(60), 25))
    x = o.extract(a, sel, "x")
    m = o.merge([a, b], "m")
    k_all = np.concatenate([ka, kb])
    v_all = np.concatenate([va, vb])
    p_all = np.array(pos_a + pos_b)
    order = np.argsort(p_all, kind="stable")
    for fd, keys, vals in ((x, ka[sel], va[sel]), (m, k_all[order], v_all[order])):
        q = rows_np(seed, TAG_Q, 0, 7, 0, 1, Hq * D).reshape(1, 1, Hq, D)
        k1, v1 = _kv(seed + 1, 900, 1, Hkv, D)
        st, out, lse = o.pred_batch([(fd, 1)], [400], q, k1, v1, D ** -0.5)
        assert st == [0]
        kk = np.concatenate([keys, k1[0]])
        vv = np.concatenate([vals, v1[0]])
        qt = torch.from_numpy(bf16_to_f64(q[0, 0])).reshape(1, Hq, 1, D)
        kt = torch.from_numpy(bf16_to_f64(kk)).permute(1, 0, 2).reshape(1, Hkv, -1, D)
        vt = torch.from_numpy(bf16_to_f64(vv)).permute(1, 0, 2).reshape(1, Hkv, -1, D)
        ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, scale=D ** -0.5, enable_gqa=True)
        assert np.allclose(out[0, 0], ref[0, :, 0].numpy(), atol=1e-12)
