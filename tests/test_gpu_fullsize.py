"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (default grids, the
workloads' own per-step LIP policies): cfg2 (256 x 2048 decode), cfg3 (64 forks of a 4096-token CoW
prefix), cfg4 (128 x 8192, truncate-to-cursor + 64-token re-append through the tcgen05 kernel), cfg5
(128 x 32768 with sink + window eviction).  Sampled LIPs are recomputed one by one by the oracle from the
generator (oracle/workload.py); nothing is read back from the CUDA path to build the expectation."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from gpu_harness import assert_close, to_bits  # noqa: E402
from oracle.workload import OracleWorkload  # noqa: E402
from paper_2510_25412_b200.workloads import DecodeWorkload  # noqa: E402


@pytest.mark.parametrize("cfg,steps,lips,cutover", [
    ("cfg2", 3, [0, 1, 37, 127, 128, 200, 254, 255], None),
    ("cfg2d", 3, [0, 99, 255], None),   # drafts (n_q = 4) through K1
    ("cfg2d", 3, [0, 99, 255], 2),      # ... and through the tcgen05 chunk kernel (cut-over 2)
    ("cfg3", 3, [0, 31, 63], None),
    ("cfg4", 2, [0, 77, 127], None),
    ("cfg5", 2, [5], None),
])
def test_full_size_sampled_parity(cfg, steps, lips, cutover):
    from paper_2510_25412_b200 import kvfs as K

    wl = DecodeWorkload(cfg, steps_total=steps + 1)
    if cutover is not None:
        wl.kv.set_option(K.OPT_CHUNK_CUTOVER, cutover)
    s = wl.shape
    T = wl.n_files * wl.n_q
    out = torch.empty((T, s.Hq, s.D), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((T, s.Hq), dtype=torch.float32, device="cuda")
    for st in range(steps):
        q, k, v = wl.make_inputs(st)
        wl.pre_step()
        status = wl.kv.pred_attn_batch(wl.descs, wl.positions(), q, k, v, out, lse)
        assert status == [0] * wl.n_files
        wl.advance()
    torch.cuda.synchronize()
    ob = to_bits(out).reshape(wl.n_files, wl.n_q, s.Hq, s.D)
    lb = lse.cpu().numpy().reshape(wl.n_files, wl.n_q, s.Hq)
    assert np.isfinite(lb).all()
    ow = OracleWorkload(cfg, lips, max_steps=steps + 1)
    for _ in range(steps):
        st, ref_out, ref_lse = ow.run_step()
        assert st == [0] * len(lips)
    for i, f in enumerate(lips):
        assert_close(ob[f], ref_out[i], f"{cfg} LIP {f}")
        np.testing.assert_allclose(lb[f], ref_lse[i], atol=2e-3, rtol=0)
        assert wl.kv.positions(wl.fds[f]) == ow.o.positions(ow.fds[i])
    if cfg == "cfg3":  # the fan-out shares the prefix: 256 pages referenced by the prefix + 64 forks
        tab = wl.kv.table(wl.fds[0])
        rc = wl.kv.refcounts()
        assert all(rc[p] == 65 for p, _ in tab[:256])
    wl.kv.audit()
