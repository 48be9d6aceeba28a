"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (default grid, cfg2:
256 LIPs x 2048-token files, Hq 32 / Hkv 8 / D 128 / P 16): sampled descriptors recomputed one by one by the
oracle from the generator (no input or expected value read back from the CUDA path)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from gpu_harness import assert_close, to_bits  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_2510_25412_b200.workloads import CONFIGS, STEP_OWNER, DecodeWorkload  # noqa: E402
from synth.workloads import TAG_K, TAG_Q, TAG_V, rows_np  # noqa: E402


def oracle_for_lip(cfg, f, n_steps):
    """The oracle's output for LIP f at decode step n_steps-1 (files built exactly as DecodeWorkload does)."""
    s = cfg["shape"]
    L0 = cfg["file_len"]
    o = Oracle((L0 + n_steps) // s.P + 4, s.P, 1, s.Hkv, s.D)
    fd = o.open("f")
    k = rows_np(cfg["seed"], TAG_K, 0, f, 0, L0, s.Hkv * s.D).reshape(1, L0, s.Hkv, s.D)
    v = rows_np(cfg["seed"], TAG_V, 0, f, 0, L0, s.Hkv * s.D).reshape(1, L0, s.Hkv, s.D)
    o.append(fd, list(range(L0)), k, v)
    out = lse = None
    for st in range(n_steps):
        own = STEP_OWNER + st
        q = rows_np(cfg["seed"], TAG_Q, 0, own, f, f + 1, s.Hq * s.D).reshape(1, 1, s.Hq, s.D)
        kn = rows_np(cfg["seed"], TAG_K, 0, own, f, f + 1, s.Hkv * s.D).reshape(1, 1, s.Hkv, s.D)
        vn = rows_np(cfg["seed"], TAG_V, 0, own, f, f + 1, s.Hkv * s.D).reshape(1, 1, s.Hkv, s.D)
        _, out, lse = o.pred_batch([(fd, 1)], [L0 + st], q, kn, vn, s.D ** -0.5)
    return out[0, 0], lse[0, 0]


def test_cfg2_full_size_sampled_parity():
    cfg = CONFIGS["cfg2"]
    n_steps = 3
    wl = DecodeWorkload("cfg2", steps_total=n_steps + 1)
    s = wl.shape
    T = wl.n_files
    out = torch.empty((T, s.Hq, s.D), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((T, s.Hq), dtype=torch.float32, device="cuda")
    for st in range(n_steps):
        q, k, v = wl.make_inputs(st)
        descs, pos = wl.descs_and_pos()
        status = wl.kv.pred_attn_batch(descs, pos, q, k, v, out, lse)
        assert status == [0] * T
        wl.advance()
    torch.cuda.synchronize()
    ob = to_bits(out)
    lb = lse.cpu().numpy()
    assert np.isfinite(lb).all()
    for f in [0, 1, 37, 127, 128, 200, 254, 255]:
        ref_out, ref_lse = oracle_for_lip(cfg, f, n_steps)
        assert_close(ob[f], ref_out, f"cfg2 LIP {f}")
        np.testing.assert_allclose(lb[f], ref_lse, atol=2e-3, rtol=0)
    # every LIP's file holds exactly its 2048 + 3 positions
    for f in [0, 255]:
        assert wl.kv.positions(wl.fds[f]) == list(range(cfg["file_len"] + n_steps))
    wl.kv.audit()
