"""The C-ABI library on a CPU box: it loads, exports every symbol include/kvfs.h declares, and its C++ host
control plane (host-only ctx, no CUDA calls) reproduces the oracle's metadata bit-exactly: page tables,
masks, positions, refcounts, allocation order, fds and error codes (rules R1-R9, R11)."""
import json
import os
import random
import re

import pytest

from oracle import EVICT_COMPACT, KvfsError as OErr, Oracle
from oracle.kvfs import EOFFLOAD
from paper_2510_25412_b200 import kvfs as K

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "kvfs.h")).read()
    declared = set(re.findall(r"^\s*(?:int|size_t|const char \*)\s*\*?\s*(\w+)\s*\(", hdr, re.M))
    assert declared == set(K.EXPORTS), declared ^ set(K.EXPORTS)
    lib = K.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert K.strerror(K.ENOSPC) == "page pool exhausted"


def test_host_only_ctx_refuses_data_ops():
    k = K.KVFS(1, 8, 2, 64, 16, 32, device=-1)
    fd = k.open("a")
    k.append(fd, [0, 1, 2])
    with pytest.raises(K.KvfsError) as e:
        k.pred_attn_batch([(fd, 1)], [3], None, None, None, None, stream=0)
    assert e.value.code == K.ENOSYS


def test_invalid_configs():
    for args in [(1, 8, 3, 64, 16, 32), (1, 8, 2, 96, 16, 32), (1, 8, 2, 64, 8, 32), (1, 24, 2, 64, 16, 32)]:
        with pytest.raises(K.KvfsError) as e:
            K.KVFS(*args, device=-1)
        assert e.value.code == K.EINVAL


class Pair:
    """Drives the C++ host-only ctx and the oracle with the same ops and compares them after each op."""

    def __init__(self, n_pages, P=16):
        self.c = K.KVFS(1, 4, 1, 64, P, n_pages, max_batch_rows=512, max_batch_descs=64, device=-1)
        self.o = Oracle(n_pages, P, store_data=False)
        self.fds = {}

    def both(self, fc, fo):
        ec = eo = None
        rc = ro = None
        try:
            rc = fc()
        except K.KvfsError as e:
            ec = e.code
        try:
            ro = fo()
        except OErr as e:
            eo = e.code
        assert ec == eo, (ec, eo)
        return rc, ro, ec

    def check(self):
        assert self.c.refcounts() == self.o.refcnt
        assert self.c.free_pages() == self.o.free_count()
        for name, (cfd, ofd) in self.fds.items():
            assert self.c.table(cfd) == self.o.table(ofd), name
            assert self.c.positions(cfd) == self.o.positions(ofd), name
            assert self.c.stat(cfd) == self.o.stat(ofd), name
        self.c.audit()
        self.o.audit()


def test_options_validate():
    """kvfs_set_option: every knob accepts its documented range and rejects the rest (include/kvfs.h)."""
    k = K.KVFS(1, 8, 2, 64, 16, 32, device=-1)
    for opt, good, bad in ((K.OPT_DECODE_CTAS, [0, 1, 4096], [-1, 4097]),
                           (K.OPT_CHUNK_CUTOVER, [0, 8, 1 << 20], [-1]),
                           (K.OPT_CASCADE_MIN_ENTRIES, [0, 16], [-1]),
                           (K.OPT_PREFIX_SPLITS, [0, 1, 8, 16], [-1, 17])):
        for v in good:
            k.set_option(opt, v)
        for v in bad:
            with pytest.raises(K.KvfsError):
                k.set_option(opt, v)
    with pytest.raises(K.KvfsError):
        k.set_option(99, 0)


def test_compact_files_errors():
    """kvfs_compact_files: a file twice is EBUSY and a bad fd EBADF with nothing done; ENOSPC stops at the
    first file whose pages are not free, the earlier files compacted (include/kvfs.h)."""
    P = 16
    c = K.KVFS(1, 8, 2, 64, P, 10, device=-1)
    o = Oracle(10, P, store_data=False)
    fds = {}
    for nm in ("a", "c"):
        fds[nm] = (c.open(nm), o.open(nm))
        c.append(fds[nm][0], list(range(40)))
        o.append(fds[nm][1], list(range(40)))
    fds["b"] = (c.fork(fds["a"][0], "b"), o.fork(fds["a"][1], "b"))  # shares a's two full pages
    for fc, fo in fds.values():
        c.evict(fc, [(1, 3)])
        o.evict(fo, [(1, 3)], 0)
    for bad, code in (([fds["a"][0], fds["a"][0]], K.EBUSY), ([fds["a"][0], 999], K.EBADF)):
        with pytest.raises(K.KvfsError) as e:
            c.compact_files(bad)
        assert e.value.code == code
    assert c.table(fds["a"][0]) == o.table(fds["a"][1])  # nothing done
    # 7 of 10 pages in use: a fits (3 new pages) but frees only its own tail page (b still holds the two
    # shared ones), so b (3 pages) hits ENOSPC; c is not reached
    with pytest.raises(K.KvfsError) as e:
        c.compact_files([fds[nm][0] for nm in ("a", "b", "c")])
    assert e.value.code == K.ENOSPC
    o.compact(fds["a"][1])
    with pytest.raises(OErr):
        o.compact(fds["b"][1])
    for fc, fo in fds.values():
        assert c.table(fc) == o.table(fo)
        assert c.positions(fc) == o.positions(fo)
    assert c.refcounts() == o.refcnt


def test_golden_trace_c7_host_plane():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "c7_trace.json")))
    c = K.KVFS(1, 8, 2, 64, 16, 96, device=-1)
    fds = [c.open(f"f{i}") for i in range(4)]
    for fd in fds:
        c.append(fd, list(range(256)))
    fds.append(c.fork(fds[0], "f4"))
    c.evict(fds[1], [(100, 132)])
    step, st = c.pred_step_begin([(fd, 1) for fd in fds], [256] * 5)
    c.pred_step_end(step)
    assert st == [0] * 5
    c.truncate(fds[4], 200)
    step, st = c.pred_step_begin([(fd, 1) for fd in fds[:4]] + [(fds[4], 4)], [257] * 4 + [200, 201, 202, 203])
    c.pred_step_end(step)
    c.compact(fds[1])
    step, st = c.pred_step_begin([(fd, 1) for fd in fds], [258] * 4 + [204])
    c.pred_step_end(step)
    fds.append(c.fork(fds[4], "f5"))
    end = {s["op"]: s for s in g["steps"]}
    expect = [0] * 96
    for rng, cnt in end["end"]["refcnt"].items():
        a, b = map(int, rng.split(".."))
        for p in range(a, b + 1):
            expect[p] = cnt
    assert c.refcounts() == expect
    assert c.table(fds[5]) == [(p, 0xFFFF) for p in range(12)] + [(16, 0x1FFF)]
    assert c.table(fds[1]) == [(p, 0xFFFF) for p in range(68, 82)] + [(82, 0x7)]
    assert c.table(fds[4]) == [(p, 0xFFFF) for p in range(12)] + [(67, 0x1FFF)]
    c.audit()


def _ranges(idx):
    out = []
    for i in idx:
        if out and out[-1][1] == i:
            out[-1][1] = i + 1
        else:
            out.append([i, i + 1])
    return [tuple(r) for r in out]


def run_random(seed, n_ops=200):
    rnd = random.Random(seed)
    P = rnd.choice([16, 16, 32, 64])
    pr = Pair(rnd.choice([5, 12, 40, 200]), P)
    c, o = pr.c, pr.o
    serial = 0
    for step in range(n_ops):
        names = list(pr.fds)
        op = rnd.choice(["open", "append", "append", "fork", "truncate", "evict", "evictc", "compact", "compact_files",
                         "unlink",
                         "pred", "pred", "close_reopen", "bad", "extract", "merge", "offload", "restore"])
        if op == "open" or not names:
            name = f"n{step}"
            rc, ro, e = pr.both(lambda: c.open(name), lambda: o.open(name))
            assert rc == ro
            pr.fds[name] = (rc, ro)
        elif op == "append":
            name = rnd.choice(names)
            cfd, ofd = pr.fds[name]
            n = rnd.choice([1, 2, 7, P - 1, P, P + 1, 3 * P + 5])
            last = o.stat(ofd)[2]
            start = last + 1 + rnd.choice([0, 0, 4]) - (2 if rnd.random() < 0.05 else 0)
            pos = list(range(start, start + n))
            pr.both(lambda: c.append(cfd, pos), lambda: o.append(ofd, pos))
        elif op == "pred":
            k = rnd.randint(1, min(6, len(names)))
            chosen = [rnd.choice(names) for _ in range(k)]
            descs, pos = [], []
            for name in chosen:
                cfd, ofd = pr.fds[name]
                nq = rnd.choice([0, 1, 1, 2, 5, P + 3])
                last = o.stat(ofd)[2]
                start = last + 1 if rnd.random() > 0.05 else last
                descs.append((cfd, ofd, nq))
                pos.extend(range(start, start + nq))
            step_h, st_c = c.pred_step_begin([(a, n) for a, _, n in descs], pos)
            c.pred_step_end(step_h)
            st_o, _ = o.pred_reserve([(b, n) for _, b, n in descs], pos)
            assert st_c == st_o, (st_c, st_o)
        elif op == "fork":
            src = rnd.choice(names)
            name = f"n{step}"
            rc, ro, e = pr.both(lambda: c.fork(pr.fds[src][0], name), lambda: o.fork(pr.fds[src][1], name))
            if e is None:
                assert rc == ro
                pr.fds[name] = (rc, ro)
        elif op == "truncate":
            name = rnd.choice(names)
            cfd, ofd = pr.fds[name]
            n = rnd.randint(0, o.stat(ofd)[0] + 1)
            pr.both(lambda: c.truncate(cfd, n), lambda: o.truncate(ofd, n))
        elif op in ("evict", "evictc"):
            name = rnd.choice(names)
            cfd, ofd = pr.fds[name]
            ln = o.stat(ofd)[0]
            idx = sorted(rnd.sample(range(ln), rnd.randint(0, min(ln, 3 * P)))) if ln else []
            if rnd.random() < 0.2 and ln:
                a = rnd.randint(0, ln - 1)
                idx = list(range(a, rnd.randint(a + 1, ln)))
            rg = _ranges(idx)
            if rnd.random() < 0.05:
                rg = rg[::-1] + [(0, 0)]  # malformed
            fl = EVICT_COMPACT if op == "evictc" else 0
            pr.both(lambda: c.evict(cfd, rg, compact=bool(fl)), lambda: o.evict(ofd, rg, fl))
        elif op == "compact":
            name = rnd.choice(names)
            cfd, ofd = pr.fds[name]
            pr.both(lambda: c.compact(cfd), lambda: o.compact(ofd))
        elif op == "compact_files":
            # kvfs_compact_files == kvfs_compact of each file in order, stopping at the first failure
            sel = rnd.sample(names, rnd.randint(1, len(names)))
            cfds = [pr.fds[nm][0] for nm in sel]

            def oracle_seq():
                # include/kvfs.h: an offloaded file fails the whole call before anything is done
                for nm in sel:
                    if o._file(pr.fds[nm][1]).host is not None:
                        raise OErr(EOFFLOAD, "offloaded")
                for nm in sel:
                    o.compact(pr.fds[nm][1])
                return len(sel)
            pr.both(lambda: c.compact_files(cfds), oracle_seq)
        elif op == "extract":
            src = rnd.choice(names)
            cfd, ofd = pr.fds[src]
            ln = o.stat(ofd)[0]
            idx = sorted(rnd.sample(range(ln), rnd.randint(0, min(ln, 3 * P)))) if ln else []
            if rnd.random() < 0.1 and len(idx) > 1:
                idx = idx[::-1]  # EINVAL
            elif rnd.random() < 0.05:
                idx = idx + [ln]  # ERANGE
            name = f"n{step}" if rnd.random() > 0.05 else src  # EEXIST
            rc, ro, e = pr.both(lambda: c.extract(cfd, idx, name), lambda: o.extract(ofd, idx, name))
            if e is None:
                assert rc == ro
                pr.fds[name] = (rc, ro)
        elif op in ("offload", "restore"):  # R15 (metadata on a host-only ctx)
            name = rnd.choice(names)
            cfd, ofd = pr.fds[name]
            if op == "offload":
                rc, ro, e = pr.both(lambda: c.offload(cfd), lambda: o.offload(ofd))
            else:
                rc, ro, e = pr.both(lambda: c.restore(cfd), lambda: o.restore(ofd))
            if e is None:
                assert rc == ro
            assert c.counter(K.CTR_HOST_PAGES) == o.host_pages()
        elif op == "merge":
            parts = [rnd.choice(names) for _ in range(rnd.randint(1, 3))]  # repeats -> EBUSY
            name = f"n{step}"
            rc, ro, e = pr.both(lambda: c.merge([pr.fds[p][0] for p in parts], name),
                                lambda: o.merge([pr.fds[p][1] for p in parts], name))
            if e is None:
                assert rc == ro
                pr.fds[name] = (rc, ro)
        elif op == "unlink":
            name = rnd.choice(names)
            cfd, ofd = pr.fds.pop(name)
            pr.both(lambda: c.unlink(name), lambda: o.unlink(name))
            pr.both(lambda: c.truncate(cfd, 0), lambda: o.truncate(ofd, 0))  # EBADF on both
            pr.both(lambda: c.close(cfd), lambda: o.close(ofd))
        elif op == "close_reopen":
            name = rnd.choice(names)
            cfd, ofd = pr.fds[name]
            pr.both(lambda: c.close(cfd), lambda: o.close(ofd))
            rc, ro, e = pr.both(lambda: c.open(name, 0), lambda: o.open(name, 0))
            assert rc == ro
            pr.fds[name] = (rc, ro)
        elif op == "bad":
            pr.both(lambda: c.open(names[0], K.O_CREAT | K.O_EXCL), lambda: o.open(names[0], 3))
            pr.both(lambda: c.open("missing", 0), lambda: o.open("missing", 0))
            pr.both(lambda: c.truncate(987, 0), lambda: o.truncate(987, 0))
        pr.check()
    for name in list(pr.fds):
        c.unlink(name)
        o.unlink(name)
    pr.fds.clear()
    pr.check()
    assert c.free_pages() == o.n_pages


@pytest.mark.parametrize("seed", range(60))
def test_host_plane_matches_oracle_random(seed):
    run_random(seed)


@pytest.mark.slow
@pytest.mark.parametrize("block", range(20))
def test_host_plane_matches_oracle_random_many(block):
    for seed in range(1000 + block * 500, 1000 + (block + 1) * 500):
        run_random(seed, n_ops=100)


def test_no_exception_crosses_the_abi():
    """include/kvfs.h: "No C++ exception crosses this ABI".  KVFS_OPT_FAULT_INJECT makes a std::bad_alloc
    fly from inside the library (mid-way through a pred reservation, after the first descriptor committed;
    in fork; in open): the call returns KVFS_ENOMEM instead of terminating the process, the possibly
    half-applied ctx is BROKEN (every later call KVFS_EIO), and kvfs_destroy still frees it."""
    for where in ("pred", "fork", "open"):
        c = K.KVFS(1, 8, 2, 64, 16, 64, device=-1)
        a = c.open("a")
        b = c.open("b")
        c.append(a, list(range(20)))
        c.append(b, list(range(20)))
        c.set_option(K.OPT_FAULT_INJECT, 1)
        with pytest.raises(K.KvfsError) as e:
            if where == "pred":
                c.pred_step_begin([(a, 1), (b, 1)], [20, 20])
            elif where == "fork":
                c.fork(a, "a2")
            else:
                c.open("z")
        assert e.value.code == K.ENOMEM, where
        for call in (lambda: c.open("q"), lambda: c.stat(a), lambda: c.truncate(a, 3), lambda: c.audit(),
                     lambda: c.pred_step_begin([(a, 1)], [99]), lambda: c.set_option(K.OPT_FAULT_INJECT, 0)):
            with pytest.raises(K.KvfsError) as e:
                call()
            assert e.value.code == K.EIO, where
        c.close_ctx()  # kvfs_destroy of a broken ctx
    # countdown: the injection fires on the n-th pass only; earlier calls are unaffected
    c = K.KVFS(1, 8, 2, 64, 16, 64, device=-1)
    c.set_option(K.OPT_FAULT_INJECT, 3)
    c.open("x")
    c.open("y")
    with pytest.raises(K.KvfsError) as e:
        c.open("w")
    assert e.value.code == K.ENOMEM


def test_unpack_checks_the_header_on_a_host_ctx():
    """kvfs_unpack takes the received buffer size; on a host-only ctx only the header matters, and a
    truncated or foreign header is EINVAL with nothing created (atomic)."""
    c = K.KVFS(1, 8, 2, 64, 16, 64, device=-1)
    a = c.open("a")
    c.append(a, list(range(40)))
    hdr, buf = c.pack([a])
    assert buf is None
    d = K.KVFS(1, 8, 2, 64, 16, 64, device=-1)
    for bad in (hdr[:10], hdr[:-4], b"\0" * len(hdr)):
        with pytest.raises(K.KvfsError) as e:
            d.unpack(bad, None, ["a"])
        assert e.value.code == K.EINVAL
    assert d.free_pages() == 64
    (fd,) = d.unpack(hdr, None, ["a"])
    assert d.table(fd) == c.table(a) and d.positions(fd) == c.positions(a)
