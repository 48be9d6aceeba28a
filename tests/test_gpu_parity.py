"""CUDA path (libkvfs.so through the C ABI) vs the oracle on the same seeded inputs.
Metadata and K/V bits: bit-exact. Attention: max-abs <= 2e-2, mean-abs <= 2e-3 (north star)."""
import math
import random

import numpy as np
import pytest
import torch

from oracle.bf16 import bf16_to_f64

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes only with -m gpu
    pytest.skip("needs a GPU", allow_module_level=True)

from gpu_harness import Harness, assert_close, to_bits, to_dev  # noqa: E402


def test_golden_trace_c7_gpu():
    """Config 1: tables/refcounts bit-exact, K/V read-back bit-exact, attention at C, E, G."""
    h = Harness(96, 16, 8, 2, 64, seed=1001)
    for i in range(4):
        h.open(f"f{i}")
    for i in range(4):
        h.append(f"f{i}", list(range(256)))
    h.fork("f0", "f4")
    h.evict("f1", [(100, 132)])
    h.check_meta()
    h.pred([(f"f{i}", [256]) for i in range(5)], qstd=4.0)
    h.truncate("f4", 200)
    h.pred([(f"f{i}", [257]) for i in range(4)] + [("f4", [200, 201, 202, 203])], qstd=4.0)
    h.compact("f1")
    h.check_data()
    h.pred([(f"f{i}", [258]) for i in range(4)] + [("f4", [204])], qstd=4.0)
    h.fork("f4", "f5")
    h.check_meta()
    h.check_data()
    assert h.c.table(h.fds["f1"][0]) == [(p, 0xFFFF) for p in range(68, 82)] + [(82, 0x7)]


@pytest.mark.parametrize("P,Hq,Hkv,D", [(16, 8, 2, 64), (16, 32, 8, 128), (32, 4, 4, 64), (64, 16, 2, 128),
                                        (16, 8, 1, 128), (16, 16, 2, 128), (32, 8, 8, 64)])
def test_random_ops_with_attention(P, Hq, Hkv, D):
    rnd = random.Random(P * 1000 + Hq * 10 + D)
    h = Harness(600, P, Hq, Hkv, D, seed=P + Hq + D)
    names = []
    for step in range(60):
        op = rnd.choice(["open", "append", "fork", "truncate", "evict", "evictc", "compact", "pred", "pred", "pred"])
        if op == "open" or len(names) < 2:
            name = f"n{step}"
            h.open(name)
            names.append(name)
            h.append(name, list(range(rnd.randint(1, 5 * P))))
        elif op == "append":
            name = rnd.choice(names)
            last = h.o.stat(h.fds[name][1])[2]
            h.append(name, list(range(last + 1, last + 1 + rnd.randint(1, 3 * P))))
        elif op == "fork":
            name = f"n{step}"
            h.fork(rnd.choice(names), name)
            names.append(name)
        elif op == "truncate":
            name = rnd.choice(names)
            h.truncate(name, rnd.randint(0, h.o.stat(h.fds[name][1])[0]))
        elif op in ("evict", "evictc"):
            name = rnd.choice(names)
            n = h.o.stat(h.fds[name][1])[0]
            if n < 2:
                continue
            a = rnd.randint(0, n - 2)
            b = rnd.randint(a + 1, min(n, a + 2 * P))
            rg = [(a, b)]
            if b + 3 < n:
                rg.append((b + 1, b + 3))
            h.evict(name, rg, compact=(op == "evictc"))
        elif op == "compact":
            h.compact(rnd.choice(names))
        else:
            chosen = rnd.sample(names, min(len(names), rnd.randint(1, 5)))
            rows = []
            for name in chosen:
                last = h.o.stat(h.fds[name][1])[2]
                nq = rnd.choice([1, 1, 1, 2, 3, P + 1])
                rows.append((name, list(range(last + 1, last + 1 + nq))))
            h.pred(rows, qstd=rnd.choice([1.0, 4.0]))
        h.check_meta()
    h.check_data()


def test_closed_forms():
    """Fresh file + one pred: out == V_new bitwise, lse == scale*<q,k>. Q = 0: lse = ln|vis|, out = mean V."""
    h = Harness(64, 16, 8, 2, 64, seed=5)
    h.open("a")
    st, ob, lb, out_o, lse_o = h.pred([("a", [0])])
    v_new = h.o.read(h.fds["a"][1], 0, 0, 1)[1][0]  # oracle's stored bits (from the generator)
    for hh in range(8):
        assert np.array_equal(ob[0, hh], v_new[hh // 4])
    np.testing.assert_allclose(lb[0], lse_o[0], atol=1e-5, rtol=0)
    # Q = 0 membership probe through the C ABI
    h.open("b")
    h.append("b", list(range(100)))
    h.evict("b", [(10, 30), (50, 51)])
    k, v = h._kv(1)
    q = torch.zeros((1, 8, 64), dtype=torch.bfloat16, device="cuda")
    out = torch.empty((1, 8, 64), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((1, 8), dtype=torch.float32, device="cuda")
    st = h.c.pred_attn_batch([(h.fds["b"][0], 1)], [100], q, to_dev(k[0]), to_dev(v[0]), out, lse)
    torch.cuda.synchronize()
    assert st == [0]
    np.testing.assert_allclose(lse.cpu().numpy(), math.log(80), atol=2e-6, rtol=0)
    h.o.pred_batch([(h.fds["b"][1], 1)], [100], np.zeros((1, 1, 8, 64), np.uint16), k, v, 0.125)
    vo = bf16_to_f64(h.o.read(h.fds["b"][1], 0, 0, 80)[1])
    ref = np.stack([vo[:, hh // 4].mean(axis=0) for hh in range(8)])
    assert_close(to_bits(out)[0], ref, "mean V")


@pytest.mark.parametrize("ctas,chunks", [(1, 0), (2, 0), (7, 0), (148, 0), (592, 0), (2048, 0),
                                         (0, 1), (0, 5), (0, 600), (0, 2048)])
def test_split_invariance_and_determinism(ctas, chunks):
    """Forced grid sizes (split counts) agree within tolerance with the oracle; each is bitwise repeatable.
    chunks > 0: dynamic scheduling (KVFS_OPT_DECODE_CHUNKS): rings take the chunks from a device counter in
    whatever order they finish; the merge of a unit's pieces is still in chunk order, so the result is
    bitwise repeatable too, and the counter resets itself between launches (second batch below)."""
    h = Harness(2000, 16, 32, 8, 128, seed=9)
    rows = []
    for i in range(12):
        h.open(f"f{i}")
        h.append(f"f{i}", list(range(50 + 97 * i)))
    h.evict("f3", [(5, 200)])
    h.c.set_option(1, ctas)  # KVFS_OPT_DECODE_CTAS
    h.c.set_option(8, chunks)  # KVFS_OPT_DECODE_CHUNKS
    for i in range(12):
        last = h.o.stat(h.fds[f"f{i}"][1])[2]
        rows.append((f"f{i}", [last + 1] if i % 3 else [last + 1, last + 2, last + 3]))
    _, ob1, lb1, _, _ = h.pred(rows, qstd=4.0)
    # replay the identical batch on a fresh harness with the same seed: bitwise equal
    h2 = Harness(2000, 16, 32, 8, 128, seed=9)
    for i in range(12):
        h2.open(f"f{i}")
        h2.append(f"f{i}", list(range(50 + 97 * i)))
    h2.evict("f3", [(5, 200)])
    h2.c.set_option(1, ctas)
    h2.c.set_option(8, chunks)
    _, ob2, lb2, _, _ = h2.pred(rows, qstd=4.0)
    assert np.array_equal(ob1, ob2) and np.array_equal(lb1, lb2)
    # a second batch on each (the dynamic counters were reset by the first launch)
    rows2 = [(n, [p[-1] + 1]) for n, p in rows]
    _, ob3, lb3, _, _ = h.pred(rows2, qstd=4.0)
    _, ob4, lb4, _, _ = h2.pred(rows2, qstd=4.0)
    assert np.array_equal(ob3, ob4) and np.array_equal(lb3, lb4)


def test_fork_isolation_bitwise():
    h = Harness(400, 16, 8, 2, 64, seed=11)
    h.open("p")
    h.append("p", list(range(1000)))
    kp0, vp0 = [to_bits(t) for t in h.c.read(h.fds["p"][0], 0, 0, 1000)]
    for i in range(6):
        h.fork("p", f"c{i}")
    for i in range(6):
        h.pred([(f"c{i}", [1000 + j for j in range(i + 1)])])
    h.truncate("c1", 500)
    h.evict("c2", [(0, 900)], compact=True)
    h.compact("c3")
    h.pred([("c1", [500, 501])])
    kp1, vp1 = [to_bits(t) for t in h.c.read(h.fds["p"][0], 0, 0, 1000)]
    assert np.array_equal(kp0, kp1) and np.array_equal(vp0, vp1)
    h.check_meta()
    h.check_data()


def test_partial_batch_and_edge_cases():
    h = Harness(20, 16, 8, 2, 64, seed=13)
    h.open("a")
    h.open("b")
    h.append("a", list(range(10)))
    # EBUSY (same file twice), EPOS, EBADF, n_q = 0, success: rows of failures untouched
    st, *_ = h.pred([("a", [10]), ("a", [11]), ("b", [3, 2]), ("zz", [0]), ("b", [])])
    assert st == [0, -16, -1001, -9, -16]
    # ENOSPC isolates the descriptor
    h.open("big")
    st, *_ = h.pred([("big", list(range(16 * 30))), ("b", [0])])
    assert st == [-28, 0]
    # empty batch
    st, *_ = h.pred([])
    assert st == []
    h.check_meta()
    h.check_data()


@pytest.mark.parametrize("P,Hq,Hkv", [(16, 32, 8), (16, 8, 8), (32, 16, 8), (64, 16, 2), (16, 16, 8)])
def test_chunk_tcgen05_kernel(P, Hq, Hkv):
    """K2 (tcgen05) for descriptors with n_q >= cutover, mixed with K1 rows in the same batch; holes from
    eviction, truncation + re-append (autocompletion), a fresh file, several 128-row M-tiles."""
    D = 128
    h = Harness(3000, P, Hq, Hkv, D, seed=P + Hq + 7)
    h.c.set_option(2, 8)  # KVFS_OPT_CHUNK_CUTOVER 8: rows with n_q < 8 on K1 (the default is 2)
    lens = [300, 1000, 77, 513, 0, 2048]
    for i, n in enumerate(lens):
        h.open(f"f{i}")
        if n:
            h.append(f"f{i}", list(range(n)))
    h.evict("f1", [(10, 200), (500, 517)])
    h.truncate("f5", 2000)
    rows = []
    for i, nq in enumerate([64, 17, 8, 100, 40, 48]):
        last = h.o.stat(h.fds[f"f{i}"][1])[2]
        rows.append((f"f{i}", list(range(last + 1, last + 1 + nq))))
    rows.append(("f0", [999]))  # EBUSY: repeated file
    h.open("d")
    h.append("d", list(range(50)))
    rows.append(("d", [50, 51]))  # K1 row in the same batch
    st, *_ = h.pred(rows, qstd=4.0)
    assert st[:6] == [0] * 6 and st[6] == -16 and st[7] == 0
    G = Hq // Hkv
    assert h.c.counter(5) == Hkv * sum(((nq * G + 127) // 128 + 1) // 2 for nq in [64, 17, 8, 100, 40, 48])  # K2 CTAs
    # second step: decode + another chunk on the grown files
    rows = []
    for i, nq in enumerate([1, 64, 1, 16, 3, 64]):
        last = h.o.stat(h.fds[f"f{i}"][1])[2]
        rows.append((f"f{i}", list(range(last + 1, last + 1 + nq))))
    h.pred(rows)
    h.check_meta()
    h.check_data()


def test_chunk_autocompletion_shape():
    """Config-4 shape in miniature: 8 LIPs x 1024 tokens, truncate-to-cursor then a 64-token re-append."""
    h = Harness(1200, 16, 32, 8, 128, seed=1004)
    h.c.set_option(2, 8)
    for i in range(8):
        h.open(f"f{i}")
        h.append(f"f{i}", list(range(1024)))
    import random as _r
    rnd = _r.Random(1004)
    for step in range(3):
        rows = []
        for i in range(8):
            r = rnd.randint(1, 64) if step else 64
            n = h.o.stat(h.fds[f"f{i}"][1])[0]
            h.truncate(f"f{i}", n - r)
            last = h.o.stat(h.fds[f"f{i}"][1])[2]
            rows.append((f"f{i}", list(range(last + 1, last + 65))))
        h.pred(rows, qstd=1.0)
    h.check_meta()


def test_migration_pack_unpack_two_ctx():
    """§8(e) data path with two ctxs on one GPU (the NCCL transport replaced by the buffer itself): the
    moved files' K/V bits, masks and positions survive; decode on the destination matches the oracle."""
    from paper_2510_25412_b200 import kvfs as K

    h = Harness(600, 16, 32, 8, 128, seed=21)
    h.open("base")
    h.append("base", list(range(300)))
    h.fork("base", "child")
    h.pred([("child", [300, 301, 302])])
    h.evict("base", [(10, 40)])
    h.open("other")
    h.append("other", list(range(77)))
    names = ["base", "child", "other"]
    hdr, buf = h.c.pack([h.fds[n][0] for n in names])
    dst = K.KVFS(1, 32, 8, 128, 16, 500, device=0)
    dst.open("pre-existing")  # the destination allocates smallest-free pages around its own state
    free0 = dst.free_pages()
    with pytest.raises(K.KvfsError) as e:  # a truncated transfer: EINVAL, nothing created, nothing read
        dst.unpack(hdr, buf[:buf.numel() - 4096], names)
    assert e.value.code == K.EINVAL and dst.free_pages() == free0
    fds = dst.unpack(hdr, buf, names)
    torch.cuda.synchronize()
    dst.audit()
    for n, fd in zip(names, fds):
        ofd = h.fds[n][1]
        assert [m for _, m in dst.table(fd)] == [m for _, m in h.o.table(ofd)]
        assert dst.positions(fd) == h.o.positions(ofd)
        ln = h.o.stat(ofd)[0]
        k, v = dst.read(fd, 0, 0, ln)
        ko, vo = h.o.read(ofd, 0, 0, ln)
        assert np.array_equal(to_bits(k), ko) and np.array_equal(to_bits(v), vo)
    shared = {p for p, _ in dst.table(fds[0])} & {p for p, _ in dst.table(fds[1])}
    rc = dst.refcounts()
    assert shared and all(rc[p] == 2 for p in shared)  # CoW sharing preserved
    # a decode step on the destination == the oracle (source state) on the same inputs
    rows = [(n, [h.o.stat(h.fds[n][1])[2] + 1]) for n in names]
    k_new, v_new = h._kv(3)
    q = h._q(3, 4.0)
    out = torch.empty((3, 32, 128), dtype=torch.bfloat16, device="cuda")
    st = dst.pred_attn_batch([(fd, 1) for fd in fds], [r[1][0] for r in rows], to_dev(q[0]), to_dev(k_new[0]),
                             to_dev(v_new[0]), out)
    torch.cuda.synchronize()
    assert st == [0, 0, 0]
    _, ref, _ = h.o.pred_batch([(h.fds[n][1], 1) for n in names], [r[1][0] for r in rows], q, k_new, v_new,
                               128 ** -0.5)
    assert_close(to_bits(out), ref[0], "migrated decode")


def test_compact_files_batched():
    """kvfs_compact_files = kvfs_compact of each file in order (pages, tables, positions; K/V bit-exact),
    including forks sharing pages and a two-layer pool."""
    from paper_2510_25412_b200 import kvfs as K
    rnd = random.Random(77)
    h = Harness(3000, 16, 8, 2, 128, seed=77, L=2)
    names = []
    for i in range(6):
        nm = f"f{i}"
        h.open(nm)
        h.append(nm, list(range(rnd.randint(40, 500))))
        names.append(nm)
    h.fork("f0", "g0")
    h.fork("f3", "g3")
    names += ["g0", "g3"]
    for nm in names:
        ln = h.o.stat(h.fds[nm][1])[0]
        a = rnd.randint(0, ln // 2)
        h.evict(nm, [(a, a + rnd.randint(1, ln // 3))])
    sel = ["f3", "g0", "f0", "f5", "g3", "f1"]
    done = h.c.compact_files([h.fds[nm][0] for nm in sel])
    assert done == len(sel)
    for nm in sel:
        h.o.compact(h.fds[nm][1])
    h.check_meta()
    h.check_data()
    with pytest.raises(K.KvfsError) as e:
        h.c.compact_files([h.fds["f1"][0], h.fds["f1"][0]])
    assert e.value.code == K.EBUSY


@pytest.mark.parametrize("gather", [1, 0])
@pytest.mark.parametrize("P,Hq,Hkv,D", [(16, 32, 8, 128), (32, 8, 2, 64), (64, 16, 2, 128)])
def test_heavy_eviction_gather(P, Hq, Hkv, D, gather):
    """Lazy eviction leaving sparse pages (KVFS_OPT_HOLES_GATHER): most pages keep 1-4 of P slots spread over
    their span, so the decode kernel fetches their retained rows with TMA gather4 into packed stage rows
    (gather = 1) or copies the whole spans (0).  Outputs, lse and the fused H2O scores (whose logit index
    follows the packed rows) equal the oracle's."""
    import torch

    from gpu_harness import scores_rtol

    from paper_2510_25412_b200 import kvfs as K

    h = Harness(3000, P, Hq, Hkv, D, seed=31 + P + D)
    h.c.set_option(K.OPT_HOLES_GATHER, gather)
    h.c.set_option(K.OPT_CASCADE_MIN_ENTRIES, 0)
    logits = torch.empty(4 << 20, dtype=torch.float32, device="cuda")
    h.c.set_logits_buffer(logits)
    rng = random.Random(P * D + gather)
    for f in range(3):
        name = f"h{f}"
        h.open(name)
        n = 700 + 300 * f
        h.append(name, list(range(n)))
        keep = set(rng.sample(range(n), n // 8)) | {0, n - 1}
        ranges, a = [], None
        for t in range(n + 1):
            if t < n and t not in keep:
                a = t if a is None else a
            elif a is not None:
                ranges.append((a, t))
                a = None
        h.evict(name, ranges)
    names = ["h0", "h1", "h2"]
    rows = []
    for name in names:
        last = h.o.stat(h.fds[name][1])[2]
        rows.append((name, [last + 1]))
    descs_c = [(h.fds[n][0], 1) for n in names]
    descs_o = [(h.fds[n][1], 1) for n in names]
    pos = [p[0] for _, p in rows]
    k, v = h._kv(3)
    q = h._q(3, 2.0)
    scale = D ** -0.5
    out = torch.empty((3, Hq, D), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((3, Hq), dtype=torch.float32, device="cuda")
    lens = [h.c.stat(fd)[0] + 1 for fd, _ in descs_c]
    step, st = h.c.pred_step_begin(descs_c, pos)
    qd = to_dev(q[0])
    h.c.pred_attn_layer(step, 0, qd, to_dev(k[0]), to_dev(v[0]), out, lse, scale)
    off = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    sc = torch.full((int(sum(lens)),), float("nan"), dtype=torch.float32, device="cuda")
    h.c.pred_attn_scores(step, 0, qd, lse, sc, off, scale)
    h.c.pred_step_end(step)
    torch.cuda.synchronize()
    assert st == [0, 0, 0]
    assert h.c.counter(K.CTR_LAST_FUSED_SCORES) == 3
    st_o, out_o, lse_o, sc_o = h.o.pred_batch(descs_o, pos, q, k, v, scale, scores=True)
    assert st_o == [0, 0, 0]
    assert_close(to_bits(out), out_o[0], "heavy eviction")
    lg = lse.cpu().numpy()
    np.testing.assert_allclose(lg, lse_o[0], atol=2e-3, rtol=0)
    got = sc.cpu().numpy().astype(np.float64)
    for i, name in enumerate(names):
        kk = bf16_to_f64(h.o.read(h.fds[name][1], 0, 0, lens[i])[0])
        ref = sc_o[i]
        rtol = scores_rtol(bf16_to_f64(q[0, i:i + 1]), kk, lg[i:i + 1], lse_o[0, i:i + 1], scale)
        g = got[off[i]:off[i] + lens[i]]
        assert g.shape == ref.shape
        assert (np.abs(g - ref) <= rtol * ref + 1e-30).all(), (name, rtol)
    h.check_meta()
    h.check_data()
