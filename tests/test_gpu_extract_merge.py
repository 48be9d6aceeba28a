"""extract (R13) / merge (R14) on the GPU path (§4.2): the new file's K/V
bits (kvfs_read) equal the oracle's bit for bit, metadata is bit-exact, and decode / chunk attention over
the new files matches the oracle (dense attention over the selected / merged tokens)."""
import random

import pytest

pytestmark = pytest.mark.gpu

from gpu_harness import Harness  # noqa: E402


@pytest.mark.parametrize("P,Hq,Hkv,D", [(16, 32, 8, 128), (32, 8, 2, 64), (64, 16, 2, 128)])
def test_extract_merge_gpu(P, Hq, Hkv, D):
    rnd = random.Random(P + D)
    h = Harness(3000, P, Hq, Hkv, D, seed=P * 3 + D)
    h.open("a")
    h.append("a", list(range(0, 1400, 2)))        # even positions
    h.open("b")
    h.append("b", list(range(1, 700, 2)))         # odd positions
    h.evict("a", [(30, 90)])
    h.fork("a", "a2")

    def ext(src, idx, name):
        cfd, ofd = h.fds[src]
        h.fds[name] = (h.c.extract(cfd, idx, name), h.o.extract(ofd, idx, name))

    def mrg(parts, name):
        h.fds[name] = (h.c.merge([h.fds[p][0] for p in parts], name), h.o.merge([h.fds[p][1] for p in parts], name))

    n = h.o.stat(h.fds["a"][1])[0]
    ext("a", sorted(rnd.sample(range(n), 300)), "x")   # sparse selection
    ext("a2", list(range(n)), "full")                   # identity selection of a fork
    ext("b", [], "empty")
    mrg(["x", "b"], "m")                                 # interleaved positions
    h.check_meta()
    h.check_data()
    for step in range(2):
        rows = []
        for name, nq in (("x", 1), ("full", 1), ("m", 9 if D == 128 else 3), ("empty", 2)):
            last = h.o.stat(h.fds[name][1])[2]
            rows.append((name, list(range(last + 1, last + 1 + nq))))
        st, *_ = h.pred(rows, qstd=4.0)
        assert st == [0, 0, 0, 0]
    h.check_meta()
    h.check_data()
