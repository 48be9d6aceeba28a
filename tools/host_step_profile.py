"""Development tool: host-side cost of one bench decode step, call by call (perf_counter stamps, no device
sync inside the loop), to see whether a workload's step is host-bound.   CFG=cfg3 python tools/host_step_profile.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_25412_b200.workloads import DecodeWorkload  # noqa: E402


def main():
    cfg = os.environ.get("CFG", "cfg3")
    n = int(os.environ.get("STEPS", "200"))
    wl = DecodeWorkload(cfg, steps_total=2 * n + 40)
    kv, s = wl.kv, wl.shape
    T = wl.n_files * wl.n_q
    out = torch.empty((T, s.Hq, s.D), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((T, s.Hq), dtype=torch.float32, device="cuda")
    inputs = [wl.make_inputs(i) for i in range(4)]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    names = ["pre_step", "positions", "begin", "ev0", "layer", "ev1", "end", "advance"]
    acc = np.zeros(len(names))
    for it in range(n + 20):
        q, k, v = inputs[it % 4]
        t = [time.perf_counter()]
        wl.pre_step(); t.append(time.perf_counter())
        pos = wl.positions(); t.append(time.perf_counter())
        step, st = kv.pred_step_begin(wl.descs, pos); t.append(time.perf_counter())
        assert not any(st), st
        ev[0].record(); t.append(time.perf_counter())
        kv.pred_attn_layer(step, 0, q, k, v, out, lse); t.append(time.perf_counter())
        ev[1].record(); t.append(time.perf_counter())
        kv.pred_step_end(step); t.append(time.perf_counter())
        wl.advance(); t.append(time.perf_counter())
        if it >= 20:
            acc += np.diff(t)
    torch.cuda.synchronize()
    acc = acc / n * 1e6
    from paper_2510_25412_b200 import kvfs as K
    ph = {nm: kv.counter(c) / 1e3 / (n + 20) for nm, c in (("reserve", K.CTR_HOST_RESERVE_NS),
                                                           ("split+cascade", K.CTR_HOST_SPLIT_NS),
                                                           ("upload+prologue", K.CTR_HOST_UPLOAD_NS),
                                                           ("layer launches", K.CTR_HOST_LAUNCH_NS))}
    print(cfg, "library host us per step:", " ".join(f"{a}={b:.1f}" for a, b in ph.items()))
    print(cfg, "host us per step:", " ".join(f"{a}={b:.1f}" for a, b in zip(names, acc)), f"total={acc.sum():.1f}")
    # the same with one pred_attn_batch call per step
    from paper_2510_25412_b200 import kvfs as K
    ctrs = (("reserve", K.CTR_HOST_RESERVE_NS), ("split+cascade", K.CTR_HOST_SPLIT_NS),
            ("upload+prologue", K.CTR_HOST_UPLOAD_NS), ("layer launches", K.CTR_HOST_LAUNCH_NS))
    before = {nm: kv.counter(c) for nm, c in ctrs}
    t0 = time.perf_counter()
    for it in range(n):
        q, k, v = inputs[it % 4]
        wl.pre_step()
        st = kv.pred_attn_batch(wl.descs, wl.positions(), q, k, v, out, lse)
        assert not any(st), st
        wl.advance()
    host = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    dev = (time.perf_counter() - t0) / n * 1e6
    print(cfg, f"pred_attn_batch loop: host {host:.1f} us per step, wall incl. drain {dev:.1f}")
    print(cfg, "  library host us per step in that loop:",
          " ".join(f"{nm}={(kv.counter(c) - before[nm]) / 1e3 / n:.1f}" for nm, c in ctrs))


if __name__ == "__main__":
    main()
