"""Development tool: globaltimer timeline of one cascade step (cfg3): the shared-prefix K2 kernel's CTAs and the
decode kernel's rings (start, first data, end of streaming, end of output), to see how the two kernels share
the SMs.

    python -c 'from paper_2510_25412_b200 import build as b; b.build(defines=("KVFS_K1_TRACE", "KVFS_K2_TRACE"),
               lib="build_var/trace/libkvfs.so", out_dir="build_var/trace")'
    KVFS_LIB_PATH=build_var/trace/libkvfs.so python tools/cascade_trace.py [extra bench-like options via env]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_25412_b200 import kvfs  # noqa: E402
from paper_2510_25412_b200.workloads import DecodeWorkload  # noqa: E402


def main():
    wl = DecodeWorkload(os.environ.get("CFG", "cfg3"), steps_total=8)
    kv = wl.kv
    for k, opt in (("SPLITS", kvfs.OPT_PREFIX_SPLITS), ("CHUNKS", kvfs.OPT_DECODE_CHUNKS),
                   ("CTAS", kvfs.OPT_DECODE_CTAS)):
        if os.environ.get(k) and int(os.environ[k]) > 0:
            kv.set_option(opt, int(os.environ[k]))
    T = wl.n_files * wl.n_q
    s = wl.shape
    out = torch.empty((T, s.Hq, s.D), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((T, s.Hq), dtype=torch.float32, device="cuda")
    for i in range(4):
        q, k, v = wl.make_inputs(i)
        wl.pre_step()
        kv.pred_attn_batch(wl.descs, wl.positions(), q, k, v, out, lse)
        wl.advance()
    torch.cuda.synchronize()
    t2 = np.zeros((2, 32, 512), dtype=np.uint64)
    t1 = np.zeros((8, 2048), dtype=np.uint64)
    L = kvfs.lib()
    for name, buf in (("kvfs_debug_k2_trace", t2), ("kvfs_debug_k1_trace", t1)):
        fn = getattr(L, name)
        fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
        assert fn(buf.ctypes.data, buf.nbytes) == 0
    ps, pe = t2[1, 30].astype(np.int64), t2[1, 31].astype(np.int64)
    n_p = int((pe > 0).sum())
    nr = int((t1[4] > 0).sum())
    t0 = min(ps[:n_p].min() if n_p else 1 << 62, t1[0, :nr].astype(np.int64).min())
    us = lambda x: (x.astype(np.int64) - t0) / 1e3  # noqa: E731
    if n_p:
        d = (pe[:n_p] - ps[:n_p]) / 1e3
        print(f"prefix kernel: {n_p} CTAs, start {us(ps[:n_p]).min():.2f}..{us(ps[:n_p]).max():.2f} us, "
              f"end {us(pe[:n_p]).min():.2f}..{us(pe[:n_p]).max():.2f} us, duration median {np.median(d):.2f} us")
        smp = set(t2[1, 29, :n_p].tolist())
        gw, of = t2[1, 26, :n_p].astype(np.int64), t2[1, 27, :n_p].astype(np.int64)
        if (gw > 0).all() and (of > 0).all():
            qg, s0, k0 = (t2[1, j, :n_p].astype(np.int64) for j in (20, 21, 22))
            if (qg > 0).all() and (s0 > 0).all() and (k0 > 0).all():
                print(f"  prefix start -> Q gathered {np.median(qg - ps[:n_p]) / 1e3:.2f} us, -> first K tile "
                      f"{np.median(k0 - ps[:n_p]) / 1e3:.2f} us, -> first S ready {np.median(s0 - ps[:n_p]) / 1e3:.2f} us "
                      f"(medians)")
            g0, rr, ql = (t2[1, j, :n_p].astype(np.int64) for j in (18, 23, 19))
            if (g0 > 0).all() and (rr > 0).all() and (ql > 0).all():
                print(f"  gather: softmax start {np.median(g0 - ps[:n_p]) / 1e3:.2f} us, row record "
                      f"{np.median(rr - ps[:n_p]) / 1e3:.2f} us, Q loads {np.median(ql - ps[:n_p]) / 1e3:.2f} us")
            sw, mg = (t2[1, j, :n_p].astype(np.int64) for j in (16, 17))
            if (sw > 0).all() and (mg > 0).all():
                print(f"  split merge: group complete {np.median(sw - pe[:n_p]) / 1e3:.2f} us after the CTA's own end "
                      f"(max {np.max(sw - pe[:n_p]) / 1e3:.2f}), merge {np.median(mg - sw) / 1e3:.2f} us, "
                      f"last merged at {us(mg).max():.2f} us")
            e1, e2, e3 = (t2[1, j, :n_p].astype(np.int64) for j in (10, 11, 12))
            if (e1 > 0).all() and (e2 > 0).all() and (e3 > 0).all():
                print(f"  epilogue (medians): other M-tile's O {np.median(e1 - of) / 1e3:.2f} us, staging "
                      f"{np.median(e2 - e1) / 1e3:.2f} us, record stores {np.median(e3 - e2) / 1e3:.2f} us, to CTA end "
                      f"{np.median(pe[:n_p] - e3) / 1e3:.2f} us")
            dn = t2[1, 25, :n_p].astype(np.int64)
            if (dn > 0).all():
                print(f"  prefix CTAs done at {us(dn).min():.2f}..{us(dn).max():.2f} us")
            print(f"  prefix CTA phases (medians): griddepcontrol.wait {np.median(gw - ps[:n_p]) / 1e3:.2f} us, "
                  f"Q + tiles {np.median(of - gw) / 1e3:.2f} us, epilogue {np.median(pe[:n_p] - of) / 1e3:.2f} us")
    else:
        smp = set()
    st, tma, fd, se, en, sm = (t1[i, :nr] for i in range(6))
    print(f"decode kernel: {nr} rings; start {us(st).min():.2f}..{us(st).max():.2f}; first TMA median "
          f"{np.median(us(tma) - us(st)):.2f} us after start; first data median {np.median(us(fd) - us(st)):.2f}; "
          f"streaming ends {us(se).min():.2f}..{us(se).max():.2f}; output ends {us(en).min():.2f}..{us(en).max():.2f} us")
    on_p = np.array([int(x) in smp for x in sm])
    if on_p.any():
        print(f"  rings on SMs that ran a prefix CTA: {on_p.sum()}, start median {np.median(us(st[on_p])):.2f} us; "
              f"others start median {np.median(us(st[~on_p])):.2f} us")
    dur = us(en) - us(st)
    cb, gw = t1[6, :nr], t1[7, :nr]
    print(f"  after streaming: combine {np.median(us(cb) - us(se)):.2f} us, griddepcontrol.wait "
          f"{np.median(us(gw) - us(cb)):.2f} us, merge + output {np.median(us(en) - us(gw)):.2f} us (medians)")
    print(f"  ring duration median {np.median(dur):.2f} p10 {np.percentile(dur, 10):.2f} p90 {np.percentile(dur, 90):.2f} us; "
          f"merge part median {np.median(us(en) - us(se)):.2f} us")


if __name__ == "__main__":
    main()
