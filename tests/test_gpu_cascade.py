"""Shared-prefix ("cascade") decode for CoW fork families (§4.2: fork
shares pages without duplicating tensors, `fig:example` P:177 forks a generation into branches).

The leading run of (page, mask) entries a fork family shares is attended once per batch by the tcgen05
kernel in prefix mode and merged (log-sum-exp) into each member's decode result.  The results must equal
the oracle's dense attention over every file's retained tokens (rule R10), exactly as without the cascade;
the counters prove the cascade path actually ran."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from gpu_harness import Harness  # noqa: E402

from paper_2510_25412_b200 import kvfs as K  # noqa: E402


def _family(h, root, n_root, kids, tail_lens, evict_root=None):
    h.open(root)
    h.append(root, list(range(n_root)))
    if evict_root:
        h.evict(root, evict_root)
    for i, (kid, n) in enumerate(zip(kids, tail_lens)):
        h.fork(root, kid)
        last = h.o.stat(h.fds[kid][1])[2]
        if n:
            h.append(kid, list(range(last + 1, last + 1 + n)))


def _decode_rows(h, names, nq=None):
    rows = []
    for i, name in enumerate(names):
        n = 1 if nq is None else nq[i]
        last = h.o.stat(h.fds[name][1])[2]
        rows.append((name, list(range(last + 1, last + 1 + n))))
    return rows


@pytest.mark.parametrize("P,Hq,Hkv,cutover", [(16, 32, 8, 8), (32, 16, 8, 8), (64, 16, 2, 8), (16, 8, 8, 8),
                                               (16, 32, 8, 2), (64, 16, 2, 2)])
def test_cascade_fork_family_decode(P, Hq, Hkv, cutover):
    """cutover 8: the draft rows (n_q 3, 7) stay on the decode path and join the family's cascade; cutover 2
    (the default): they go to the tcgen05 chunk kernel in the same batch, the n_q = 1 members cascade."""
    h = Harness(4000, P, Hq, Hkv, 128, seed=P * 7 + Hq)
    h.c.set_option(K.OPT_CASCADE_MIN_ENTRIES, 4)
    h.c.set_option(K.OPT_CHUNK_CUTOVER, cutover)
    kids = [f"k{i}" for i in range(9)]
    # root of 1500 tokens with holes (evicted before the fork: the shared masks carry them), 9 branches
    _family(h, "root", 1500, kids, [0, 5, 40, 300, 1, 17, 160, 64, 2], evict_root=[(3, 9), (700, 760)])
    h.evict("k3", [(1600, 1650)])            # a hole in a private suffix
    h.open("solo")
    h.append("solo", list(range(333)))
    for step in range(3):
        names = kids + ["root", "solo"]
        nq = [1] * len(names)
        if step == 1:
            nq[2], nq[5] = 3, 7              # short speculative drafts
        st, *_ = h.pred(_decode_rows(h, names, nq), qstd=4.0 if step == 2 else 1.0)
        assert st == [0] * len(names)
        assert h.c.counter(K.CTR_LAST_PREFIX_GROUPS) == 1
        assert h.c.counter(K.CTR_LAST_PREFIX_UNITS) > 0
    h.check_meta()
    h.check_data()


def test_cascade_equals_no_cascade_and_two_families():
    """Two families + a member truncated back into the shared run (the family's common run shrinks to it);
    the same batch with the cascade disabled gives the same attention (both within tolerance of the oracle,
    and within 2 bf16 ulps-ish of each other)."""
    h = Harness(3000, 16, 32, 8, 128, seed=11)
    h.c.set_option(K.OPT_CASCADE_MIN_ENTRIES, 2)
    _family(h, "A", 900, ["a0", "a1", "a2", "a3"], [10, 0, 33, 120])
    _family(h, "B", 2048, ["b0", "b1"], [16, 1])
    h.truncate("a2", 500)                   # shares only 500 tokens (31 full entries) with the others
    names = ["a0", "a1", "a2", "a3", "b0", "b1", "A"]
    st, ob_on, *_ = h.pred(_decode_rows(h, names))
    assert st == [0] * len(names)
    assert h.c.counter(K.CTR_LAST_PREFIX_GROUPS) == 2
    # same step once more with the cascade off: compare with the oracle again (independent path)
    h.c.set_option(K.OPT_CASCADE_MIN_ENTRIES, 0)
    st, *_ = h.pred(_decode_rows(h, names))
    assert st == [0] * len(names)
    assert h.c.counter(K.CTR_LAST_PREFIX_UNITS) == 0
    h.check_meta()


def test_cascade_random_families():
    """Random families, random tails, random evictions in branches, several steps; every result vs oracle."""
    rnd = random.Random(2510)
    h = Harness(6000, 16, 32, 8, 128, seed=5)
    h.c.set_option(K.OPT_CASCADE_MIN_ENTRIES, 3)
    names = []
    for f in range(3):
        kids = [f"f{f}k{i}" for i in range(rnd.randint(2, 12))]
        _family(h, f"f{f}", rnd.randint(100, 1200), kids, [rnd.randint(0, 200) for _ in kids])
        names += kids
    for step in range(4):
        for n in rnd.sample(names, 3):
            ln = h.o.stat(h.fds[n][1])[0]
            if ln > 40:
                a = rnd.randint(ln // 2, ln - 20)
                h.evict(n, [(a, a + 5)])
        batch = rnd.sample(names, max(2, len(names) - 2))
        st, *_ = h.pred(_decode_rows(h, batch))
        assert st == [0] * len(batch)
    h.check_meta()
    h.check_data()


@pytest.mark.parametrize("splits,n_root", [(1, 1300), (3, 1300), (8, 1300), (16, 1300), (13, 2400), (16, 4200)])
def test_cascade_forced_splits(splits, n_root):
    """KVFS_OPT_PREFIX_SPLITS: any split count of the shared run gives the oracle's attention."""
    h = Harness(3000, 16, 32, 8, 128, seed=40 + splits)
    h.c.set_option(K.OPT_CASCADE_MIN_ENTRIES, 4)
    h.c.set_option(K.OPT_PREFIX_SPLITS, splits)
    with pytest.raises(Exception):
        h.c.set_option(K.OPT_PREFIX_SPLITS, 17)
    kids = [f"k{i}" for i in range(6)]
    _family(h, "root", n_root, kids, [0, 3, 30, 129, 1, 64], evict_root=[(100, 117)])
    st, *_ = h.pred(_decode_rows(h, kids + ["root"]))
    assert st == [0] * 7
    assert h.c.counter(K.CTR_LAST_PREFIX_GROUPS) == 1
    h.check_meta()


@pytest.mark.parametrize("chunks", [64, 700])
def test_cascade_dynamic_decode(chunks):
    """The cascade with the dynamic decode scheduling (KVFS_OPT_DECODE_CHUNKS): chunks merge with the
    shared-prefix partials exactly as the static grid."""
    h = Harness(3000, 16, 32, 8, 128, seed=60 + chunks)
    h.c.set_option(K.OPT_CASCADE_MIN_ENTRIES, 4)
    h.c.set_option(K.OPT_DECODE_CHUNKS, chunks)
    kids = [f"k{i}" for i in range(9)]
    _family(h, "root", 1500, kids, [0, 3, 30, 129, 1, 64, 300, 2, 17], evict_root=[(10, 33)])
    for _ in range(2):
        st, *_ = h.pred(_decode_rows(h, kids + ["root"]))
        assert st == [0] * 10
        assert h.c.counter(K.CTR_LAST_PREFIX_GROUPS) == 1
    h.check_meta()
    h.check_data()


def test_cascade_pipelined_steps_with_changing_splits():
    """Regression: consecutive steps issued WITHOUT a host synchronisation while the key-split count changes
    from step to step (a different packet layout every step).  The shared-prefix kernel is a programmatic
    dependent launch after the step prologue that uploads the step's packet; it read its unit records before
    waiting for that upload and so picked up the previous step's records (illegal address on B200 when the
    layout changed).  Every step's output must equal the oracle's."""
    import torch

    from gpu_harness import assert_close, to_bits, to_dev

    h = Harness(4000, 16, 32, 8, 128, seed=5)
    h.c.set_option(K.OPT_CASCADE_MIN_ENTRIES, 4)
    kids = [f"k{i}" for i in range(24)]
    _family(h, "root", 1200, kids, [3 + 5 * i for i in range(24)])
    splits = [2, 1, 3, 1, 2, 4, 1, 2]
    outs, refs = [], []
    for step, sp in enumerate(splits):
        h.c.set_option(K.OPT_PREFIX_SPLITS, sp)
        rows = _decode_rows(h, kids)
        descs_c = [(h.fds[n][0], len(p)) for n, p in rows]
        descs_o = [(h.fds[n][1], len(p)) for n, p in rows]
        pos = [x for _, p in rows for x in p]
        T = len(pos)
        k, v = h._kv(T)
        q = h._q(T)
        out = torch.full((T, h.Hq, h.D), float("nan"), dtype=torch.bfloat16, device="cuda")
        lse = torch.empty((T, h.Hq), dtype=torch.float32, device="cuda")
        st = h.c.pred_attn_batch(descs_c, pos, to_dev(q[0]), to_dev(k[0]), to_dev(v[0]), out, lse)  # no sync
        assert st == [0] * T
        assert h.c.counter(K.CTR_LAST_PREFIX_GROUPS) == 1
        st_o, out_o, lse_o = h.o.pred_batch(descs_o, pos, q, k, v, h.D ** -0.5)
        outs.append((out, lse))
        refs.append((out_o[0], lse_o[0]))
    torch.cuda.synchronize()
    for step, ((out, lse), (ro, rl)) in enumerate(zip(outs, refs)):
        assert_close(to_bits(out), ro, f"step {step}")
        np.testing.assert_allclose(lse.cpu().numpy(), rl, atol=2e-3, rtol=0)
    h.check_meta()
    h.check_data()


@pytest.mark.parametrize("P,Hq,Hkv,n_root,nq", [(16, 32, 8, 1300, None), (16, 32, 8, 4200, None), (32, 16, 8, 700, None),
                                                  (16, 32, 8, 1300, [1, 2, 1, 3, 1, 1, 1, 1]), (16, 16, 2, 2500, None),
                                                  (16, 8, 8, 1500, None)])
def test_cascade_paired_partition(P, Hq, Hkv, n_root, nq):
    """KVFS_OPT_PREFIX_PAIRED = 2: lanes in pairs, 3 key pieces each, one CTA per pair running two pieces of
    different kv heads in turn (barriers re-armed between them); the decode kernel folds the 3 records."""
    h = Harness(3000, P, Hq, Hkv, 128, seed=90 + n_root + Hkv)
    h.c.set_option(K.OPT_CASCADE_MIN_ENTRIES, 4)
    h.c.set_option(K.OPT_PREFIX_PAIRED, 2)
    with pytest.raises(Exception):
        h.c.set_option(K.OPT_PREFIX_PAIRED, 3)
    kids = [f"k{i}" for i in range(7)]
    _family(h, "root", n_root, kids, [0, 3, 30, 129, 1, 64, 5], evict_root=[(100, 117)])
    for _ in range(3):
        st, *_ = h.pred(_decode_rows(h, kids + ["root"], nq))
        assert st == [0] * 8
        assert h.c.counter(K.CTR_LAST_PREFIX_GROUPS) == 1
        # 3 pieces per lane, 5 CTAs per lane pair: 3 * Hkv units
        assert h.c.counter(K.CTR_LAST_PREFIX_UNITS) == 3 * Hkv
    h.check_meta()
    h.check_data()


def test_cascade_paired_two_families_and_holes():
    """The paired partition over two families of different run lengths (one truncated member shrinks family A's
    run), holes in the shared run, several steps: every result vs the oracle."""
    h = Harness(3000, 16, 32, 8, 128, seed=12)
    h.c.set_option(K.OPT_CASCADE_MIN_ENTRIES, 2)
    h.c.set_option(K.OPT_PREFIX_PAIRED, 2)
    _family(h, "A", 900, ["a0", "a1", "a2", "a3"], [10, 0, 33, 120], evict_root=[(40, 77), (300, 301)])
    _family(h, "B", 2048, ["b0", "b1"], [16, 1])
    h.truncate("a2", 500)
    names = ["a0", "a1", "a2", "a3", "b0", "b1", "A"]
    for _ in range(3):
        st, *_ = h.pred(_decode_rows(h, names))
        assert st == [0] * len(names)
        assert h.c.counter(K.CTR_LAST_PREFIX_GROUPS) == 2
        assert h.c.counter(K.CTR_LAST_PREFIX_UNITS) == 2 * 3 * 8
    h.check_meta()
    h.check_data()
