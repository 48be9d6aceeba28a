"""Development tool: per-tile pipeline timeline of the K2 chunk kernel (cfg4 workload).

    python -c 'from paper_2510_25412_b200 import build as b; b.build(defines=("KVFS_K2_TRACE",),
               lib="build_var/trace/libkvfs.so", out_dir="build_var/trace")'
    KVFS_LIB_PATH=build_var/trace/libkvfs.so python tools/k2_trace.py

Prints, for two CTAs, the median over tiles of every event's time relative to softmax 0's S-ready of the
same tile, and the median tile period."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_25412_b200 import kvfs  # noqa: E402
from paper_2510_25412_b200.workloads import DecodeWorkload  # noqa: E402

NAMES_EXTRA = {29: "S0:JF waited"}
NAMES = ["K:empty", "K:issued", "V:empty", "V:issued", "M:K(t+1)", "M:SE0", "M:S0 iss", "M:SE1", "M:S1 iss",
         "M:V(t)", "M:PF0", "M:PV0 iss", "M:PF1", "M:PV1 iss"] + \
        [f"S{m}:{e}" for m in range(2) for e in ("S rdy", "S read", "max", "PE/resc", "exp done", "PF arr")]


def main():
    wl = DecodeWorkload(os.environ.get("CFG", "cfg4"), steps_total=4)
    kv = wl.kv
    T = wl.n_files * wl.n_q
    s = wl.shape
    out = torch.empty((T, s.Hq, s.D), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((T, s.Hq), dtype=torch.float32, device="cuda")
    for i in range(2):
        q, k, v = wl.make_inputs(i)
        wl.pre_step()
        kv.pred_attn_batch(wl.descs, wl.positions(), q, k, v, out, lse)
        wl.advance()
    torch.cuda.synchronize()
    buf = np.zeros((2, 32, 512), dtype=np.uint64)
    fn = kvfs.lib().kvfs_debug_k2_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    assert fn(buf.ctypes.data, buf.nbytes) == 0
    t0 = buf[0, 24, 0].astype(np.int64)
    if t0:
        print("CTA 0 one-off events (clk from kernel start): Q ready %d, first S ready %d, last O %d, end %d"
              % tuple(int(buf[0, e, 0]) - t0 if buf[0, e, 0] else -1 for e in (25, 14, 26, 27)))
    if t0:
        print("epilogue stamps (clk from start):", [int(buf[0, 28, c]) - t0 for c in range(5)])
        if buf[0, 30, 0]:
            print("  prefix epilogue per chunk: TMEM data ready", [int(buf[0, 30, c]) - t0 for c in range(4)],
                  "staged", [int(buf[0, 31, c]) - t0 for c in range(4)])
    st, en, sm = buf[1, 30].astype(np.int64), buf[1, 31].astype(np.int64), buf[1, 29].astype(np.int64)
    nb = int((en > 0).sum())
    if nb and os.environ.get("CTA_TIMES"):
        t0 = st[:nb].min()
        print("per-CTA start/end (us from the first start), sm:")
        for b in range(nb):
            print(f"  cta {b:4d} sm {sm[b]:3d} start {(st[b] - t0) / 1e3:8.2f} end {(en[b] - t0) / 1e3:8.2f} dur {(en[b] - st[b]) / 1e3:7.2f}")
        return
    for c in range(2):
        tr = buf[c].astype(np.int64)
        n = int((tr[14] > 0).sum())
        ref = tr[14, :n]
        print(f"--- CTA {'0' if c == 0 else '296'}: {n} tiles, median period {np.median(np.diff(ref[5:n - 5])):.0f} clk")
        for e, name in list(enumerate(NAMES)) + list(NAMES_EXTRA.items()):
            d = tr[e, 5:n - 5] - ref[5:n - 5]
            if (tr[e, 5:n - 5] == 0).all():
                continue
            print(f"  {name:12s} {np.median(d):8.0f}  p10 {np.percentile(d, 10):8.0f}  p90 {np.percentile(d, 90):8.0f}")


if __name__ == "__main__":
    main()
