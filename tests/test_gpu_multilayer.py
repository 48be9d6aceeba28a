"""Multi-layer steps (include/kvfs.h pred_step_begin / pred_attn_layer / pred_step_end): one
reservation per step, one attention call per layer; every layer's output equals the oracle's, every layer's
pool holds exactly the appended bits, and copy-on-write / fork tail copies cover all layers."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from gpu_harness import Harness, assert_close, to_bits, to_dev  # noqa: E402

from paper_2510_25412_b200 import kvfs as K  # noqa: E402


@pytest.mark.parametrize("P,Hq,Hkv,D", [(16, 32, 8, 128), (32, 8, 2, 64)])
def test_multilayer_step(P, Hq, Hkv, D):
    L = 3
    h = Harness(3000, P, Hq, Hkv, D, L=L, seed=7 + P + D)
    h.c.set_option(K.OPT_CASCADE_MIN_ENTRIES, 2)
    h.open("r")
    h.append("r", list(range(600)))
    h.evict("r", [(10, 30)])
    for i in range(3):
        h.fork("r", f"k{i}")                       # fork tail copies: every layer
    h.open("big")
    h.append("big", list(range(900)))
    h.truncate("big", 850)
    for step in range(2):
        rows = []
        for name, nq in (("k0", 1), ("k1", 2), ("k2", 1), ("big", 24 if D == 128 else 5), ("r", 1)):
            last = h.o.stat(h.fds[name][1])[2]
            rows.append((name, list(range(last + 1, last + 1 + nq))))
        descs_c = [(h.fds[n][0], len(p)) for n, p in rows]
        descs_o = [(h.fds[n][1], len(p)) for n, p in rows]
        pos = [x for _, p in rows for x in p]
        T = len(pos)
        k, v = h._kv(T)
        q = h._q(T, 2.0)
        scale = D ** -0.5
        step_h, st = h.c.pred_step_begin(descs_c, pos)
        outs = []
        for layer in range(L):
            out = torch.full((T, Hq, D), float("nan"), dtype=torch.bfloat16, device="cuda")
            lse = torch.full((T, Hq), float("nan"), dtype=torch.float32, device="cuda")
            h.c.pred_attn_layer(step_h, layer, to_dev(q[layer]), to_dev(k[layer]), to_dev(v[layer]), out, lse, scale)
            outs.append((out, lse))
        h.c.pred_step_end(step_h)
        torch.cuda.synchronize()
        st_o, out_o, lse_o = h.o.pred_batch(descs_o, pos, q, k, v, scale)
        assert st == st_o == [0] * len(rows)
        for layer in range(L):
            assert_close(to_bits(outs[layer][0]), out_o[layer], f"layer {layer}")
            np.testing.assert_allclose(outs[layer][1].cpu().numpy(), lse_o[layer], atol=2e-3, rtol=0)
    h.check_meta()
    h.check_data()  # every layer's K/V bits (kvfs_read per layer)
