"""pred_attn_batch_host (include/kvfs.h): the batched pred with HOST buffers -- the library stages the step's
inputs into its device slots, runs the pred and copies the results back -- against the oracle, single steps
(decode, chunk rows through the tcgen05 kernel, a fork family through the cascade, a failed descriptor whose
rows must stay untouched) and a pipeline of steps issued back to back with no host synchronisation."""
import numpy as np
import pytest
import torch

from oracle.bf16 import bf16_to_f64

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from gpu_harness import Harness, assert_close, to_bits, to_host_pinned  # noqa: E402


def test_host_io_single_steps():
    h = Harness(2400, 16, 32, 8, 128, seed=71)
    for i in range(6):
        h.open(f"f{i}")
        h.append(f"f{i}", list(range(300 + 37 * i)))
    h.fork("f0", "c0")
    h.fork("f0", "c1")
    h.evict("f2", [(40, 90)])
    # decode rows, a failed descriptor (bad fd: its rows stay NaN), a draft descriptor (n_q = 5)
    h.pred([(f"f{i}", [400 + i]) for i in range(6)] + [("nofile", [1, 2])], host_io=True)
    h.pred([("f1", [500, 501, 502, 503, 504]), ("f3", [600])], host_io=True)
    # the fork family (cascade path) and chunk rows
    h.pred([("f0", [900]), ("c0", [900]), ("c1", [900])], host_io=True)
    h.pred([("f4", list(range(700, 764)))], host_io=True)
    h.check_meta()
    h.check_data()


def test_host_io_pipelined_steps():
    """Eight steps issued back to back (the input copy of step i+1 and the output copy of step i-1 overlap
    step i), each with its own pinned output buffer; checked against the oracle after one fence + sync."""
    h = Harness(1200, 16, 8, 2, 64, seed=72)
    names = [f"f{i}" for i in range(5)]
    for i, nm in enumerate(names):
        h.open(nm)
        h.append(nm, list(range(200 + 50 * i)))
    pos0 = 10_000
    pending = []
    keep = []
    for step in range(8):
        rows = [(nm, [pos0 + step * 10 + j for j in range(1 + (step + i) % 3)]) for i, nm in enumerate(names)]
        descs_c = [(h.fds[nm][0], len(ps)) for nm, ps in rows]
        descs_o = [(h.fds[nm][1], len(ps)) for nm, ps in rows]
        pos = [p for _, ps in rows for p in ps]
        T = len(pos)
        k, v = h._kv(T)
        q = h._q(T, 2.0)
        qh, kh, vh = (to_host_pinned(x[0]) for x in (q, k, v))
        out = torch.full((T, h.Hq, h.D), float("nan"), dtype=torch.bfloat16).pin_memory()
        lse = torch.full((T, h.Hq), float("nan"), dtype=torch.float32).pin_memory()
        st = h.c.pred_attn_batch_host(descs_c, pos, qh, kh, vh, out, lse)
        keep.append((qh, kh, vh))  # inputs must outlive their copies
        st_o, out_o, lse_o = h.o.pred_batch(descs_o, pos, q, k, v, h.D ** -0.5)
        assert st == st_o == [0] * len(rows)
        pending.append((out, lse, out_o[0], lse_o[0]))
    h.c.pred_host_fence()
    torch.cuda.synchronize()
    for i, (out, lse, out_o, lse_o) in enumerate(pending):
        assert_close(to_bits(out), out_o, f"step {i}")
        np.testing.assert_allclose(lse.numpy(), lse_o, atol=2e-3, rtol=0)
    h.check_meta()
    h.check_data()


def test_host_io_failed_rows_untouched_and_errors():
    h = Harness(300, 16, 8, 2, 64, seed=73)
    h.open("a")
    h.append("a", list(range(100)))
    st, ob, _, _, _ = h.pred([("nofile", [5, 6]), ("a", [200])], host_io=True)
    assert st[0] != 0 and st[1] == 0
    assert np.isnan(bf16_to_f64(ob[:2])).all()
    # call-level error (negative n_q): nothing runs, nothing is copied
    out = torch.full((1, h.Hq, h.D), float("nan"), dtype=torch.bfloat16).pin_memory()
    with pytest.raises(Exception):
        h.c.pred_attn_batch_host([(h.fds["a"][0], -1)], [], None, None, None, out)
    h.c.pred_host_fence()
    torch.cuda.synchronize()
    assert torch.isnan(out.float()).all()


def test_host_io_packed_buffers_one_copy_layout():
    """Q / K_new / V_new (and out / lse) as views of one pinned buffer at 256-byte aligned offsets (how a serving
    loop packs a step) give the oracle's results."""
    h = Harness(800, 16, 8, 2, 64, seed=74)
    for i in range(3):
        h.open(f"p{i}")
        h.append(f"p{i}", list(range(120 + 40 * i)))
    descs_c = [(h.fds[f"p{i}"][0], 1 + i) for i in range(3)]
    descs_o = [(h.fds[f"p{i}"][1], 1 + i) for i in range(3)]
    pos = [p for i in range(3) for p in range(1000, 1001 + i)]
    T = len(pos)
    k, v = h._kv(T)
    q = h._q(T, 2.0)

    def packed(arrays):
        sizes = [a.nbytes for a in arrays]
        offs = np.concatenate([[0], np.cumsum([(z + 255) // 256 * 256 for z in sizes])]).astype(int)
        buf = torch.full((int(offs[-1]),), 0x7F, dtype=torch.uint8).pin_memory()
        views = []
        for a, o, z in zip(arrays, offs, sizes):
            t = buf[o:o + z]
            t.copy_(torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1)))
            views.append(t)
        return buf, views

    _, (qb, kb, vb) = packed([q[0], k[0], v[0]])
    qh, kh, vh = (x.view(torch.bfloat16) for x in (qb, kb, vb))
    outbuf, (ob, lb) = packed([np.zeros((T, h.Hq, h.D), np.uint16), np.zeros((T, h.Hq), np.float32)])
    out, lse = ob.view(torch.bfloat16).view(T, h.Hq, h.D), lb.view(torch.float32).view(T, h.Hq)
    st = h.c.pred_attn_batch_host(descs_c, pos, qh, kh, vh, out, lse)
    h.c.pred_host_fence()
    torch.cuda.synchronize()
    st_o, out_o, lse_o = h.o.pred_batch(descs_o, pos, q, k, v, h.D ** -0.5)
    assert st == st_o == [0, 0, 0]
    assert_close(to_bits(out), out_o[0], "packed host buffers")
    np.testing.assert_allclose(lse.numpy(), lse_o[0], atol=2e-3, rtol=0)
    h.check_meta()
    h.check_data()
