"""Offload / restore (R15; §4.3) on the GPU path: the exclusively owned pages
go to the pinned host tier and come back bit-exact into the pages rule R1 picks; shared pages never move;
EOFFLOAD while offloaded; decode after restore matches the oracle; metadata bit-exact throughout."""
import pytest
import torch

pytestmark = pytest.mark.gpu

from gpu_harness import Harness  # noqa: E402

from paper_2510_25412_b200 import kvfs as K  # noqa: E402


@pytest.mark.parametrize("P,Hq,Hkv,D,L", [(16, 32, 8, 128, 1), (32, 8, 2, 64, 1)])
def test_offload_restore_gpu(P, Hq, Hkv, D, L):
    h = Harness(2000, P, Hq, Hkv, D, L=L, seed=P + D)
    h.open("a")
    h.append("a", list(range(900)))
    h.fork("a", "b")                    # b shares a's full pages
    last = h.o.stat(h.fds["b"][1])[2]
    h.append("b", list(range(last + 1, last + 301)))
    h.evict("b", [(950, 980)])
    h.open("c")
    h.append("c", list(range(333)))
    moved = {}
    for name in ("b", "c"):
        cfd, ofd = h.fds[name]
        mc, mo = h.c.offload(cfd), h.o.offload(ofd)
        assert mc == mo
        moved[name] = mc
    torch.cuda.synchronize()
    assert moved["c"] == len(h.o.table(h.fds["c"][1]))          # all exclusive
    assert 0 < moved["b"] < len(h.o.table(h.fds["b"][1]))       # shared pages stayed
    assert h.c.counter(K.CTR_HOST_PAGES) == h.o.host_pages() == moved["b"] + moved["c"]
    h.check_meta()
    with pytest.raises(K.KvfsError) as e:
        h.c.truncate(h.fds["c"][0], 3)
    assert e.value.code == K.EOFFLOAD
    st, *_ = h.pred([("b", [5000]), ("a", [901])])
    assert st == [K.EOFFLOAD, 0]
    # reuse the freed pages, then restore both (new pages by R1)
    h.open("d")
    h.append("d", list(range(200)))
    for name in ("c", "b"):
        cfd, ofd = h.fds[name]
        assert h.c.restore(cfd) == h.o.restore(ofd)
    assert h.c.counter(K.CTR_HOST_PAGES) == 0
    h.check_meta()
    h.check_data()
    rows = []
    for name in ("a", "b", "c", "d"):
        last = h.o.stat(h.fds[name][1])[2]
        rows.append((name, [last + 1]))
    st, *_ = h.pred(rows, qstd=3.0)
    assert st == [0, 0, 0, 0]
    h.check_meta()
    h.check_data()
    # unlink while offloaded releases everything
    h.c.offload(h.fds["d"][0])
    h.o.offload(h.fds["d"][1])
    h.unlink("d")
    assert h.c.counter(K.CTR_HOST_PAGES) == 0
    h.check_meta()
