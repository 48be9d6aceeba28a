"""NEXT-2 attention-score accumulation (H2O; §6) on the GPU path: pred_attn_scores after
pred_attn_layer equals the oracle's per-token softmax weight summed over query rows and heads, for decode,
drafts and chunk descriptors, files with holes, forks sharing a prefix (cascade on), a failed descriptor."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from gpu_harness import Harness, assert_close, scores_rtol, to_bits, to_dev  # noqa: E402

from oracle.attention import attention_scores  # noqa: E402
from oracle.bf16 import bf16_to_f64  # noqa: E402

from paper_2510_25412_b200 import kvfs as K  # noqa: E402


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("P,Hq,Hkv,D", [(16, 32, 8, 128), (32, 8, 2, 64), (64, 16, 2, 128), (16, 8, 8, 128),
                                        (16, 16, 8, 64), (32, 8, 1, 128)])
def test_scores_match_oracle(P, Hq, Hkv, D, fused):
    """fused: the decode kernel writes its logits (kvfs_set_logits_buffer) and the decode descriptors' scores
    come from them (K10); chunk descriptors and cascade members still go through K9 in the same call."""
    _scores_case(P, Hq, Hkv, D, fused)


@pytest.mark.parametrize("fused", [False, True])
def test_scores_paired_cascade(fused):
    """The same batch with the cascade's paired partition forced (KVFS_OPT_PREFIX_PAIRED = 2): the members'
    attention folds 3 prefix records, their scores (K9) and the others' are unchanged."""
    _scores_case(16, 32, 8, 128, fused, paired=2)


def _scores_case(P, Hq, Hkv, D, fused, paired=0):
    h = Harness(4000, P, Hq, Hkv, D, seed=P + Hq + D)
    h.c.set_option(K.OPT_CASCADE_MIN_ENTRIES, 2)
    h.c.set_option(K.OPT_PREFIX_PAIRED, paired)
    if fused:
        logits = torch.empty(16 << 20, dtype=torch.float32, device="cuda")
        h.c.set_logits_buffer(logits)
    h.open("r")
    h.append("r", list(range(700)))
    h.evict("r", [(5, 40), (300, 333)])
    for i in range(3):
        h.fork("r", f"k{i}")
        last = h.o.stat(h.fds[f"k{i}"][1])[2]
        h.append(f"k{i}", list(range(last + 1, last + 1 + 50 * i + 3)))
    h.open("big")
    h.append("big", list(range(2000)))
    h.open("solo")
    h.append("solo", list(range(333)))
    h.evict("solo", [(30, 41)])
    rows = []
    for name, nq in (("k0", 1), ("k1", 1), ("k2", 3), ("big", 20 if D == 128 else 5), ("r", 1), ("solo", 1)):
        last = h.o.stat(h.fds[name][1])[2]
        rows.append((name, list(range(last + 1, last + 1 + nq))))
    rows.append(("k0", [99999]))  # EBUSY: ignored by the scores
    descs_c = [(h.fds[n][0], len(p)) for n, p in rows]
    descs_o = [(h.fds[n][1], len(p)) for n, p in rows]
    pos = [x for _, p in rows for x in p]
    T = len(pos)
    k, v = h._kv(T)
    q = h._q(T, 2.0)
    scale = D ** -0.5
    out = torch.empty((T, Hq, D), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((T, Hq), dtype=torch.float32, device="cuda")
    lens = [h.c.stat(fd)[0] + n for fd, n in descs_c]  # length after the append (stat is refused mid-step)
    lens[-1] = 0                                        # the EBUSY descriptor: no scores
    step, st = h.c.pred_step_begin(descs_c, pos)
    qd = to_dev(q[0])
    h.c.pred_attn_layer(step, 0, qd, to_dev(k[0]), to_dev(v[0]), out, lse, scale)
    off = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    scores = torch.full((int(sum(lens)),), float("nan"), dtype=torch.float32, device="cuda")
    h.c.pred_attn_scores(step, 0, qd, lse, scores, off, scale)
    h.c.pred_step_end(step)
    torch.cuda.synchronize()
    if paired:
        assert h.c.counter(K.CTR_LAST_PREFIX_UNITS) == 3 * Hkv  # the paired partition ran
    n_fused = h.c.counter(K.CTR_LAST_FUSED_SCORES)
    assert (n_fused > 0) == fused, n_fused  # "solo" (and for D 64 every descriptor) is a plain decode descriptor
    if fused and D == 64:
        assert n_fused == 6
    st_o, out_o, lse_o, sc_o = h.o.pred_batch(descs_o, pos, q, k, v, scale, scores=True)
    assert st == st_o and st[-1] == -16
    sc = scores.cpu().numpy()
    r = 0
    for i, ((name, p), s) in enumerate(zip(rows, st)):
        if s == 0:
            assert_close(to_bits(out)[r:r + len(p)], out_o[0, r:r + len(p)], name)
            got = sc[off[i]:off[i] + lens[i]]
            ref = sc_o[i]
            assert got.shape == ref.shape
            kk = bf16_to_f64(h.o.read(h.fds[name][1], 0, 0, lens[i])[0])
            rtol = scores_rtol(bf16_to_f64(q[0, r:r + len(p)]), kk, lse.cpu().numpy()[r:r + len(p)],
                               lse_o[0, r:r + len(p)], scale)
            assert rtol < 5e-3, (name, rtol)
            assert (np.abs(got - ref) <= rtol * ref + 1e-30).all(), (name, rtol, np.abs(got - ref).max())
            assert abs(got.sum() - len(p) * Hq) <= 1e-3 * len(p) * Hq, name  # weights of each row-head sum to 1
        r += len(p)
    assert len(sc) == off[-1]  # nothing was written past the successful descriptors' ranges


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("P,Hq,Hkv,D", [(16, 32, 8, 128), (32, 8, 2, 64)])
def test_scores_between_layers(P, Hq, Hkv, D, fused):
    """pred_attn_scores after layer l of an OPEN multi-layer step, then pred_attn_layer for
    layer l + 1 (the per-layer H2O order).  The scores packet must not overwrite the step's uploaded plan
    (descriptors, destination slots): every layer's output, lse, scores and pool bits equal the oracle's."""
    L = 3
    h = Harness(3000, P, Hq, Hkv, D, L=L, seed=11 + P + D)
    h.c.set_option(K.OPT_CASCADE_MIN_ENTRIES, 2)
    if fused:  # each layer's logits overwrite the previous layer's; scores follow every layer
        logits = torch.empty(8 << 20, dtype=torch.float32, device="cuda")
        h.c.set_logits_buffer(logits)
    h.open("r")
    h.append("r", list(range(500)))
    h.evict("r", [(7, 29)])
    for i in range(2):
        h.fork("r", f"k{i}")
    h.open("big")
    h.append("big", list(range(700)))
    rows = []
    for name, nq in (("k0", 1), ("big", 24 if D == 128 else 5), ("k1", 3), ("r", 1)):
        last = h.o.stat(h.fds[name][1])[2]
        rows.append((name, list(range(last + 1, last + 1 + nq))))
    descs_c = [(h.fds[n][0], len(p)) for n, p in rows]
    descs_o = [(h.fds[n][1], len(p)) for n, p in rows]
    pos = [x for _, p in rows for x in p]
    T = len(pos)
    k, v = h._kv(T)
    q = h._q(T, 2.0)
    scale = D ** -0.5
    lens = [h.c.stat(fd)[0] + n for fd, n in descs_c]
    off = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    step, st = h.c.pred_step_begin(descs_c, pos)
    res = []
    for layer in range(L):
        qd = to_dev(q[layer])
        out = torch.full((T, Hq, D), float("nan"), dtype=torch.bfloat16, device="cuda")
        lse = torch.full((T, Hq), float("nan"), dtype=torch.float32, device="cuda")
        h.c.pred_attn_layer(step, layer, qd, to_dev(k[layer]), to_dev(v[layer]), out, lse, scale)
        sc = torch.full((int(sum(lens)),), float("nan"), dtype=torch.float32, device="cuda")
        h.c.pred_attn_scores(step, layer, qd, lse, sc, off, scale)
        res.append((out, lse, sc))
    h.c.pred_step_end(step)
    torch.cuda.synchronize()
    st_o, out_o, lse_o = h.o.pred_batch(descs_o, pos, q, k, v, scale)
    assert st == st_o == [0] * len(rows)
    for layer, (out, lse, sc) in enumerate(res):
        assert_close(to_bits(out), out_o[layer], f"layer {layer}")
        lg = lse.cpu().numpy()
        np.testing.assert_allclose(lg, lse_o[layer], atol=2e-3, rtol=0)
        scn = sc.cpu().numpy()
        r = 0
        for i, (name, p) in enumerate(rows):
            n = len(p)
            kk = bf16_to_f64(h.o.read(h.fds[name][1], layer, 0, lens[i])[0])
            qq = bf16_to_f64(q[layer, r:r + n])
            ref = attention_scores(qq, kk, scale)
            rtol = scores_rtol(qq, kk, lg[r:r + n], lse_o[layer, r:r + n], scale)
            got = scn[off[i]:off[i] + lens[i]]
            assert (np.abs(got - ref) <= rtol * ref + 1e-30).all(), (layer, name, rtol)
            r += n
    h.check_meta()
    h.check_data()  # every layer's appended K/V bits landed in the reserved slots
