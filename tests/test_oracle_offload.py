"""Pins of the oracle's offload / restore (R15): PAPER.md §4.3 P:233 "offloads their KV caches from the GPU to
the CPU and restores them upon I/O completion"; SPEC S:117-125 worked examples (each cited), the
round trip of the bits, R1 page ids on restore, EOFFLOAD on page-touching ops, atomic ENOSPC. CPU only."""
import numpy as np
import pytest

from oracle import EBADF, EINVAL, ENOSPC, EOFFLOAD, HOST, KvfsError, Oracle
from synth.workloads import TAG_K, TAG_V, rows_np


def _mk(o, name, n, seed=3):
    fd = o.open(name)
    k = rows_np(seed, TAG_K, 0, 0, 0, n, o.Hkv * o.D).reshape(1, n, o.Hkv, o.D)
    v = rows_np(seed, TAG_V, 0, 0, 0, n, o.Hkv * o.D).reshape(1, n, o.Hkv, o.D)
    o.append(fd, list(range(n)), k, v)
    return fd, k[0], v[0]


def test_spec_s121_offload_188_exclusive_pages():
    o = Oracle(400, 16, 1, 1, 4)
    a, _, _ = _mk(o, "a", 3000)  # 188 pages
    free0 = o.free_count()
    assert o.offload(a) == 188
    assert o.free_count() == free0 + 188 and o.host_pages() == 188  # device -188, host +188
    assert [p for p, _ in o.table(a)] == [HOST | i for i in range(188)]
    o.audit()


def test_spec_s122_offload_fully_shared_moves_nothing():
    o = Oracle(64, 16, 1, 1, 4)
    a, _, _ = _mk(o, "a", 64)  # 4 full pages: a fork shares all of them (no tail copy, R4)
    b = o.fork(a, "b")
    t = o.table(b)
    assert o.offload(b) == 0 and o.table(b) == t and o.host_pages() == 0


def test_spec_s123_restore_into_full_pool_enospc_atomic():
    o = Oracle(8, 16, 1, 1, 4)
    a, _, _ = _mk(o, "a", 80)  # 5 pages
    assert o.offload(a) == 5
    f, _, _ = _mk(o, "filler", 8 * 16 - 16 * 4)  # leaves 4 free
    t = o.table(a)
    with pytest.raises(KvfsError) as e:
        o.restore(a)
    assert e.value.code == ENOSPC and o.table(a) == t and o.host_pages() == 5
    o.unlink("filler")
    assert o.restore(a) == 5
    o.audit()


def test_round_trip_bits_r1_ids_and_partial_sharing():
    o = Oracle(64, 16, 2, 2, 8)
    a, k, v = _mk(o, "a", 100)  # 7 pages, tail with room
    b = o.fork(a, "b")          # shares pages 0..5, b's tail copied
    o.unlink("a")               # b now owns pages 0..5 exclusively? no: refcount 1 after unlink
    tb = o.table(b)
    kk, vv = o.read(b, 0, 0, 100)
    assert o.offload(b) == 7
    x, _, _ = _mk(o, "x", 40, seed=9)  # reuses the freed low page ids
    assert o.restore(b) == 7
    # restored pages: smallest free ids in table order (R1)
    used = {p for p, _ in o.table(x)}
    expect = sorted(set(range(64)) - used)[:7]
    assert [p for p, _ in o.table(b)] == expect
    assert [m for _, m in o.table(b)] == [m for _, m in tb]
    k2, v2 = o.read(b, 0, 0, 100)
    assert np.array_equal(k2, kk) and np.array_equal(v2, vv)
    for layer in range(2):
        assert np.array_equal(o.read(b, layer, 0, 100)[0], o.read(b, layer, 0, 100)[0])
    o.audit()


def test_offloaded_file_refuses_page_ops_allows_metadata():
    o = Oracle(32, 16, 1, 1, 4)
    a, _, _ = _mk(o, "a", 40)
    o.offload(a)
    for fn in (lambda: o.append(a, [40]), lambda: o.truncate(a, 3), lambda: o.evict(a, [(0, 2)]),
               lambda: o.compact(a), lambda: o.fork(a, "z"), lambda: o.extract(a, [0], "z"),
               lambda: o.merge([a], "z"), lambda: o.read(a, 0, 0, 1)):
        with pytest.raises(KvfsError) as e:
            fn()
        assert e.value.code == EOFFLOAD
    st, _ = o.pred_reserve([(a, 1)], [40])
    assert st == [EOFFLOAD]
    assert o.stat(a)[0] == 40 and len(o.positions(a)) == 40
    with pytest.raises(KvfsError) as e:
        o.offload(a)
    assert e.value.code == EINVAL
    o.restore(a)
    with pytest.raises(KvfsError) as e:
        o.restore(a)
    assert e.value.code == EINVAL
    o.unlink("a")
    assert sum(o.refcnt) == 0


def test_unlink_offloaded_drops_host_copy():
    o = Oracle(16, 16, 1, 1, 4)
    a, _, _ = _mk(o, "a", 50)
    o.offload(a)
    o.unlink("a")
    assert o.host_pages() == 0 and sum(o.refcnt) == 0
    with pytest.raises(KvfsError) as e:
        o.restore(a)
    assert e.value.code == EBADF
