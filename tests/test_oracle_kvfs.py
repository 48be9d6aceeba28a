"""Pins of the oracle's KVFS model (rules R1-R9, R11) and of attention-over-a-file (R10):
SPEC.md worked examples, the hand-derived golden trace (tests/golden/c7_trace.json),
a deep-copy shadow model on random op sequences, invariants after every op,
and evict/truncate equivalence against torch SDPA on the dense sequence (north star). CPU only."""
import json
import math
import os
import random

import numpy as np
import pytest
import torch

from oracle import (EBADF, EBUSY, EEXIST, EINVAL, ENOENT, ENOSPC, EPOS, ERANGE, EVICT_COMPACT, O_CREAT,
                    O_EXCL, KvfsError, Oracle)
from oracle.bf16 import bf16_to_f64
from synth.workloads import TAG_K, TAG_Q, TAG_V, rows_np

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "c7_trace.json")


def kv(seed, owner, s0, s1, hkv, d, layers=1):
    k = np.stack([rows_np(seed, TAG_K, l, owner, s0, s1, hkv * d).reshape(s1 - s0, hkv, d) for l in range(layers)])
    v = np.stack([rows_np(seed, TAG_V, l, owner, s0, s1, hkv * d).reshape(s1 - s0, hkv, d) for l in range(layers)])
    return k, v


def expand(table_spec):
    out = []
    for a, b, m in table_spec:
        out.extend([p, m] for p in range(a, b + 1))
    return out


# ------------------------------------------------------------------ SPEC worked examples
def test_spec_s62_3000_tokens_188_pages():
    o = Oracle(400, 16, store_data=False)
    fd = o.open("doc")
    o.append(fd, list(range(3000)))
    assert len(o.table(fd)) == 188 and o.free_count() == 400 - 188  # ceil(3000/16)
    o.audit()


def test_spec_s78_fork_3000_one_new_page_187_increments():
    o = Oracle(400, 16, store_data=False)
    fd = o.open("doc")
    o.append(fd, list(range(3000)))
    before = list(o.refcnt)
    c = o.fork(fd, "child")
    after = o.refcnt
    incremented = [p for p in range(400) if after[p] == before[p] + 1 and before[p] > 0]
    new = [p for p in range(400) if before[p] == 0 and after[p] == 1]
    assert len(incremented) == 187 and len(new) == 1
    assert o.table(c)[:187] == o.table(fd)[:187] and o.table(c)[187][0] == new[0]
    o.audit()


def test_spec_s79_fork_empty():
    o = Oracle(8, 16, store_data=False)
    fd = o.open("e")
    c = o.fork(fd, "e2")
    assert o.table(c) == [] and o.free_count() == 8


def test_spec_s70_remove_once_forked_frees_nothing():
    o = Oracle(64, 16, store_data=False)
    fd = o.open("a")
    o.append(fd, list(range(64)))  # 4 full pages -> fork shares all
    o.fork(fd, "b")
    free_before = o.free_count()
    o.unlink("a")
    assert o.free_count() == free_before
    o.audit()


def test_spec_s87_append_to_shared_tail_copies():
    o = Oracle(16, 16, store_data=False)
    a = o.open("a")
    o.append(a, list(range(32)))
    b = o.fork(a, "b")  # full tail: everything shared
    o.truncate(b, 24)   # b's tail page (mask 0x00ff) is shared with a (refcount 2)
    tail = o.table(b)[-1][0]
    assert o.refcnt[tail] == 2
    o.append(b, [24])
    assert o.table(b)[-1][0] != tail and o.refcnt[tail] == 1 and o.refcnt[o.table(b)[-1][0]] == 1
    assert o.copies == [(tail, o.table(b)[-1][0])]
    o.audit()


def test_spec_s88_position_conflict():
    o = Oracle(8, 16, store_data=False)
    fd = o.open("a")
    o.append(fd, [0, 1, 2])
    for bad in ([2], [1], [5, 5], [7, 6]):
        with pytest.raises(KvfsError) as e:
            o.append(fd, bad)
        assert e.value.code == EPOS
    assert o.positions(fd) == [0, 1, 2]


def test_spec_s89_8_plus_16():
    o = Oracle(8, 16, store_data=False)
    fd = o.open("a")
    o.append(fd, list(range(8)))
    o.append(fd, list(range(8, 24)))
    t = o.table(fd)
    assert [bin(m).count("1") for _, m in t] == [16, 8]


def test_spec_s608_32_siblings_32_tail_copies():
    hkv, d = 2, 8
    o = Oracle(400, 16, 1, hkv, d)
    root = o.open("prefix")
    k, v = kv(7, 0, 0, 3000, hkv, d)
    o.append(root, list(range(3000)), k, v)
    o.copies.clear()
    sibs = [o.fork(root, f"s{i}") for i in range(32)]
    assert len(o.copies) == 32  # exactly 32 tail copies, 0 full-page copies
    assert all(o.refcnt[p] == 33 for p, _ in o.table(root)[:187])
    snap = {fd: o.read(fd, 0, 0, o.stat(fd)[0]) for fd in [root] + sibs}
    for i, fd in enumerate(sibs):
        kk, vv = kv(7, 100 + i, 0, 64, hkv, d)
        o.append(fd, list(range(3000, 3064)), kk, vv)
        for other in [root] + sibs:
            if other != fd:
                r = o.read(other, 0, 0, o.stat(other)[0])
                n = snap[other][0].shape[0]
                assert np.array_equal(r[0][:n], snap[other][0]) and np.array_equal(r[1][:n], snap[other][1])
        o.audit()


def test_errors():
    o = Oracle(4, 16, store_data=False)
    a = o.open("a")
    with pytest.raises(KvfsError) as e:
        o.open("a", O_CREAT | O_EXCL)
    assert e.value.code == EEXIST
    with pytest.raises(KvfsError) as e:
        o.open("zz", 0)
    assert e.value.code == ENOENT
    with pytest.raises(KvfsError) as e:
        o.truncate(99, 0)
    assert e.value.code == EBADF
    o.append(a, list(range(20)))
    with pytest.raises(KvfsError) as e:
        o.truncate(a, 21)
    assert e.value.code == ERANGE
    for bad, code in ([[(3, 3)], EINVAL], [[(5, 8), (6, 9)], EINVAL], [[(0, 21)], ERANGE], [[(-1, 2)], ERANGE]):
        with pytest.raises(KvfsError) as e:
            o.evict(a, bad)
        assert e.value.code == code
    with pytest.raises(KvfsError) as e:
        o.append(a, list(range(20, 20 + 16 * 3 + 1)))  # needs 4 pages, only 2 free
    assert e.value.code == ENOSPC
    assert o.stat(a) == (20, 2, 19)
    o.audit()


# ------------------------------------------------------------------ golden trace
def _check_tables(o, fds, tables):
    for name, spec in tables.items():
        assert [list(e) for e in o.table(fds[name])] == expand(spec), name


def _dense_sdpa(qrows, ks, vs, scale):
    """torch SDPA reference on an explicitly built dense K/V sequence (float64)."""
    n_q = qrows.shape[0]
    length = ks.shape[0]
    tq = torch.from_numpy(qrows).permute(1, 0, 2)[None]
    tk = torch.from_numpy(ks).permute(1, 0, 2)[None]
    tv = torch.from_numpy(vs).permute(1, 0, 2)[None]
    mask = torch.arange(length)[None, :] <= (length - n_q + torch.arange(n_q)[:, None])
    o = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, attn_mask=mask, scale=scale,
                                                         enable_gqa=True)
    return o[0].permute(1, 0, 2).numpy()


def test_golden_trace_c7():
    g = json.load(open(GOLDEN))
    c = g["config"]
    hq, hkv, d, P = c["n_q_heads"], c["n_kv_heads"], c["head_dim"], c["page_size"]
    seed = 1001
    o = Oracle(c["n_pages"], P, 1, hkv, d)
    fds = {}
    serial = {}
    dense = {}  # name -> list of (pos, k row, v row) built directly from the generator

    def app(name, positions):
        s0 = serial.get(name, 0)
        owner = int(name[1:])
        k, v = kv(seed, owner, s0, s0 + len(positions), hkv, d)
        serial[name] = s0 + len(positions)
        return k, v

    steps = {s["op"]: s for s in g["steps"]}
    for i in range(4):
        fds[f"f{i}"] = o.open(f"f{i}")
    for i in range(4):
        k, v = app(f"f{i}", range(256))
        o.append(fds[f"f{i}"], list(range(256)), k, v)
        dense[f"f{i}"] = [(p, k[0, p], v[0, p]) for p in range(256)]
    _check_tables(o, fds, steps["0"]["tables"])
    assert o.free_count() == 32 and o.refcnt[64:] == [0] * 32

    fds["f4"] = o.fork(fds["f0"], "f4")
    dense["f4"] = list(dense["f0"])
    _check_tables(o, fds, steps["A"]["tables"])
    assert o.refcnt[:16] == [2] * 16 and o.free_count() == 32

    o.evict(fds["f1"], [(100, 132)])
    dense["f1"] = dense["f1"][:100] + dense["f1"][132:]
    _check_tables(o, fds, steps["B"]["tables"])
    assert o.stat(fds["f1"])[0] == 224 and o.refcnt[23] == 0

    scale = 1.0 / math.sqrt(d)
    qstep = 0

    def pred(rows):  # rows: list of (name, positions)
        nonlocal qstep
        qstep += 1
        descs, pos, ks, vs, qs = [], [], [], [], []
        for name, ps in rows:
            descs.append((fds[name], len(ps)))
            pos.extend(ps)
            k, v = app(name, ps)
            ks.append(k)
            vs.append(v)
            q = rows_np(seed, TAG_Q, 0, int(name[1:]) + 16 * qstep, 0, len(ps), hq * d, 4.0)
            qs.append(q.reshape(1, len(ps), hq, d))
        k = np.concatenate(ks, axis=1)
        v = np.concatenate(vs, axis=1)
        q = np.concatenate(qs, axis=1)
        st, out, lse = o.pred_batch(descs, pos, q, k, v, scale)
        assert st == [0] * len(rows)
        r = 0
        for name, ps in rows:
            for j, p in enumerate(ps):
                dense[name].append((p, k[0, r + j], v[0, r + j]))
            # attention = dense SDPA over the explicitly tracked retained sequence
            kd = bf16_to_f64(np.stack([e[1] for e in dense[name]]))
            vd = bf16_to_f64(np.stack([e[2] for e in dense[name]]))
            ref = _dense_sdpa(bf16_to_f64(q[0, r:r + len(ps)]), kd, vd, scale)
            np.testing.assert_allclose(out[0, r:r + len(ps)], ref, atol=1e-12, rtol=0)
            assert o.positions(fds[name]) == [e[0] for e in dense[name]]
            r += len(ps)

    pred([(f"f{i}", [256]) for i in range(5)])
    for name, (page, mask) in steps["C"]["new_tail"].items():
        assert list(o.table(fds[name])[-1]) == [page, mask], name
    assert o.positions(fds["f1"]) == list(range(100)) + list(range(132, 257))

    o.truncate(fds["f4"], 200)
    dense["f4"] = dense["f4"][:200]
    _check_tables(o, fds, steps["D"]["tables"])
    assert o.refcnt[13:16] == [1, 1, 1] and o.refcnt[67] == 0

    pred([(f"f{i}", [257]) for i in range(4)] + [("f4", [200, 201, 202, 203])])
    _check_tables(o, fds, steps["E"]["tables"])
    for name, (page, mask) in steps["E"]["new_tail"].items():
        assert list(o.table(fds[name])[-1]) == [page, mask], name
    assert o.refcnt[12] == 1

    o.compact(fds["f1"])
    _check_tables(o, fds, steps["F"]["tables"])
    assert all(o.refcnt[p] == 0 for p in list(range(16, 23)) + list(range(24, 32)) + [64])

    pred([(f"f{i}", [258]) for i in range(4)] + [("f4", [204])])
    for name, (page, mask) in steps["G"]["new_tail"].items():
        assert list(o.table(fds[name])[-1]) == [page, mask], name

    fds["f5"] = o.fork(fds["f4"], "f5")
    _check_tables(o, fds, steps["H"]["tables"])
    assert o.refcnt[:12] == [3] * 12

    expect = [0] * c["n_pages"]
    for rng, cnt in steps["end"]["refcnt"].items():
        a, b = map(int, rng.split(".."))
        for p in range(a, b + 1):
            expect[p] = cnt
    assert o.refcnt == expect
    assert sum(1 for x in o.refcnt if x) == steps["end"]["allocated"]
    o.audit()
    # the data of every file equals the explicitly tracked dense sequence
    for name, fd in fds.items():
        if name == "f5":
            continue
        kk, vv = o.read(fd, 0, 0, o.stat(fd)[0])
        assert np.array_equal(kk, np.stack([e[1] for e in dense[name]]))
        assert np.array_equal(vv, np.stack([e[2] for e in dense[name]]))


# ------------------------------------------------------------------ evict / truncate equivalence
def test_evict_equivalence_all_subsets_of_8():
    """evict(E) then decode == dense attention over the 8-token sequence with E removed (2^8 subsets)."""
    hq, hkv, d, P = 4, 2, 16, 16
    seed = 77
    k0, v0 = kv(seed, 0, 0, 9, hkv, d)
    q = rows_np(seed, TAG_Q, 0, 0, 0, 1, hq * d, 4.0).reshape(1, 1, hq, d)
    for subset in range(256):
        o = Oracle(8, P, 1, hkv, d)
        fd = o.open("f")
        o.append(fd, list(range(8)), k0[:, :8], v0[:, :8])
        ev = [i for i in range(8) if subset >> i & 1]
        ranges = []
        for i in ev:
            if ranges and ranges[-1][1] == i:
                ranges[-1][1] = i + 1
            else:
                ranges.append([i, i + 1])
        o.evict(fd, [tuple(r) for r in ranges])
        keep = [i for i in range(8) if not subset >> i & 1]
        assert o.positions(fd) == keep
        st, out, _ = o.pred_batch([(fd, 1)], [8], q, k0[:, 8:9], v0[:, 8:9], 0.25)
        idx = keep + [8]
        ref = _dense_sdpa(bf16_to_f64(q[0]), bf16_to_f64(k0[0, idx]), bf16_to_f64(v0[0, idx]), 0.25)
        np.testing.assert_allclose(out[0], ref, atol=1e-12, rtol=0)
        o.audit()


def test_truncate_equivalence_all_points():
    hq, hkv, d, P = 4, 2, 16, 16
    seed = 78
    k0, v0 = kv(seed, 0, 0, 41, hkv, d)
    q = rows_np(seed, TAG_Q, 0, 0, 0, 1, hq * d, 4.0).reshape(1, 1, hq, d)
    for n in range(41):
        o = Oracle(8, P, 1, hkv, d)
        fd = o.open("f")
        o.append(fd, list(range(40)), k0[:, :40], v0[:, :40])
        o.truncate(fd, n)
        st, out, _ = o.pred_batch([(fd, 1)], [n], q, k0[:, 40:41], v0[:, 40:41], 0.25)
        idx = list(range(n)) + [40]
        ref = _dense_sdpa(bf16_to_f64(q[0]), bf16_to_f64(k0[0, idx]), bf16_to_f64(v0[0, idx]), 0.25)
        np.testing.assert_allclose(out[0], ref, atol=1e-12, rtol=0)
        assert len(o.table(fd)) == math.ceil((n + 1) / P)


def test_partition_invariance():
    """n tokens in one pred == n successive decode preds, up to fp64 rounding."""
    hq, hkv, d, P = 4, 2, 16, 16
    seed = 79
    k0, v0 = kv(seed, 0, 0, 70, hkv, d)
    q = rows_np(seed, TAG_Q, 0, 0, 0, 30, hq * d).reshape(1, 30, hq, d)
    a = Oracle(16, P, 1, hkv, d)
    fa = a.open("f")
    a.append(fa, list(range(40)), k0[:, :40], v0[:, :40])
    _, out_a, lse_a = a.pred_batch([(fa, 30)], list(range(40, 70)), q, k0[:, 40:], v0[:, 40:], 0.25)
    b = Oracle(16, P, 1, hkv, d)
    fb = b.open("f")
    b.append(fb, list(range(40)), k0[:, :40], v0[:, :40])
    for i in range(30):
        _, o1, l1 = b.pred_batch([(fb, 1)], [40 + i], q[:, i:i + 1], k0[:, 40 + i:41 + i], v0[:, 40 + i:41 + i], 0.25)
        np.testing.assert_allclose(o1[0, 0], out_a[0, i], atol=1e-12, rtol=0)
        np.testing.assert_allclose(l1[0, 0], lse_a[0, i], atol=1e-12, rtol=0)
    assert a.table(fa) == b.table(fb)


def test_batch_rules():
    o = Oracle(8, 16, 1, 1, 4)
    a = o.open("a")
    a2 = o.open("a")  # second fd to the same file
    b = o.open("b")
    z = np.zeros((1, 4, 2, 4), np.uint16)
    zk = np.zeros((1, 4, 1, 4), np.uint16)
    st, out, _ = o.pred_batch([(a, 1), (a2, 1), (99, 1), (b, 1)], [0, 1, 0, 0], z, zk, zk, 1.0)
    assert st == [0, EBUSY, EBADF, 0]
    assert np.isnan(out[0, 1]).all() and np.isnan(out[0, 2]).all() and not np.isnan(out[0, 3]).any()
    st, _, _ = o.pred_batch([(a, 1), (b, 0)], [0], z[:, :1], zk[:, :1], zk[:, :1], 1.0)
    assert st == [EPOS, 0]
    with pytest.raises(KvfsError) as e:
        o.pred_reserve([(a, 2)], [5])
    assert e.value.code == EINVAL


# ------------------------------------------------------------------ deep-copy shadow model
class Shadow:
    """Each file is a plain list of (pos, k row, v row), deep-copied on fork. No pages."""

    def __init__(self):
        self.files = {}

    def length(self, name):
        return len(self.files[name])


def _ranges_from(idx):
    out = []
    for i in idx:
        if out and out[-1][1] == i:
            out[-1][1] = i + 1
        else:
            out.append([i, i + 1])
    return [tuple(r) for r in out]


@pytest.mark.parametrize("seed", range(40))
def test_shadow_model_random_ops(seed):
    rnd = random.Random(seed)
    hkv, d, P = 1, 4, 16
    n_pages = rnd.choice([6, 12, 40])
    o = Oracle(n_pages, P, 1, hkv, d)
    sh = Shadow()
    fds = {}
    serial = 0
    for step in range(200):
        names = list(sh.files)
        op = rnd.choice(["open", "append", "append", "append", "fork", "truncate", "evict", "evictc",
                         "compact", "unlink", "pred", "extract", "merge"])
        snap = (list(o.refcnt), {n: o.table(fds[n]) for n in names})
        err = None
        expect = None
        try:
            if op == "open" or not names:
                name = f"n{step}"
                fds[name] = o.open(name)
                sh.files[name] = []
            elif op in ("append", "pred"):
                name = rnd.choice(names)
                n = rnd.choice([1, 1, 2, 5, 16, 17, 40])
                last = sh.files[name][-1][0] if sh.files[name] else -1
                start = last + rnd.choice([1, 1, 3]) if rnd.random() > 0.05 else last  # 5%: EPOS
                expect = EPOS if start <= last else None
                pos = list(range(start, start + n))
                k = rows_np(seed, TAG_K, 0, 0, serial, serial + n, hkv * d).reshape(1, n, hkv, d)
                v = rows_np(seed, TAG_V, 0, 0, serial, serial + n, hkv * d).reshape(1, n, hkv, d)
                serial += n
                if op == "append":
                    o.append(fds[name], pos, k, v)
                else:
                    q = np.zeros((1, n, 2, d), np.uint16)
                    st, _, _ = o.pred_batch([(fds[name], n)], pos, q, k, v, 1.0)
                    if st[0] != 0:
                        raise KvfsError(st[0])
                sh.files[name].extend((p, k[0, i], v[0, i]) for i, p in enumerate(pos))
            elif op == "fork":
                src = rnd.choice(names)
                name = f"n{step}"
                fds[name] = o.fork(fds[src], name)
                sh.files[name] = list(sh.files[src])
            elif op == "truncate":
                name = rnd.choice(names)
                n = rnd.randint(0, sh.length(name) + 1)
                expect = ERANGE if n > sh.length(name) else None
                o.truncate(fds[name], n)
                sh.files[name] = sh.files[name][:n]
            elif op in ("evict", "evictc"):
                name = rnd.choice(names)
                ln = sh.length(name)
                idx = sorted(rnd.sample(range(ln), rnd.randint(0, min(ln, 20)))) if ln else []
                if rnd.random() < 0.1 and ln:
                    idx = list(range(rnd.randint(0, ln - 1), ln))
                o.evict(fds[name], _ranges_from(idx), EVICT_COMPACT if op == "evictc" else 0)
                drop = set(idx)
                sh.files[name] = [e for i, e in enumerate(sh.files[name]) if i not in drop]
            elif op == "compact":
                name = rnd.choice(names)
                o.compact(fds[name])
            elif op == "extract":  # R13: the selected entries, positions kept
                src = rnd.choice(names)
                ln = sh.length(src)
                idx = sorted(rnd.sample(range(ln), rnd.randint(0, min(ln, 40)))) if ln else []
                name = f"n{step}"
                fds[name] = o.extract(fds[src], idx, name)
                sh.files[name] = [sh.files[src][i] for i in idx]
            elif op == "merge":  # R14: union sorted by position; duplicates -> EPOS
                parts = rnd.sample(names, min(len(names), rnd.randint(1, 3)))
                toks = sorted((e for p in parts for e in sh.files[p]), key=lambda e: e[0])
                dup = any(a[0] == b[0] for a, b in zip(toks, toks[1:]))
                expect = EPOS if dup else None
                name = f"n{step}"
                fds[name] = o.merge([fds[p] for p in parts], name)
                sh.files[name] = toks
            elif op == "unlink":
                name = rnd.choice(names)
                o.unlink(name)
                o.close(fds.pop(name))
                del sh.files[name]
        except KvfsError as e:
            err = e.code
        if expect is not None:
            assert err == expect, (op, err, expect)
        if err is not None:
            assert err == expect or err == ENOSPC, (op, err)
            # atomic failure: nothing changed
            assert o.refcnt == snap[0]
            assert {n: o.table(fds[n]) for n in names} == snap[1]
        o.audit()
        for name, ent in sh.files.items():
            fd = fds[name]
            assert o.positions(fd) == [e[0] for e in ent]
            kk, vv = o.read(fd, 0, 0, len(ent))
            if ent:
                assert np.array_equal(kk, np.stack([e[1] for e in ent]))
                assert np.array_equal(vv, np.stack([e[2] for e in ent]))
    for name in list(sh.files):
        o.unlink(name)
    o.audit()
    assert sum(o.refcnt) == 0  # I5: no leaks
