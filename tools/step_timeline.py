"""Development tool: GPU timeline of a few decode steps (torch.profiler / CUPTI kernel + memcpy activity):
per step, every kernel's start and duration relative to the step's first activity, and the gaps.
    CFG=cfg3 python tools/step_timeline.py"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_25412_b200.workloads import DecodeWorkload  # noqa: E402


def main():
    cfg = os.environ.get("CFG", "cfg3")
    n = int(os.environ.get("STEPS", "30"))
    wl = DecodeWorkload(cfg, steps_total=n + 40)
    kv, s = wl.kv, wl.shape
    T = wl.n_files * wl.n_q
    out = torch.empty((T, s.Hq, s.D), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((T, s.Hq), dtype=torch.float32, device="cuda")
    inputs = [wl.make_inputs(i) for i in range(4)]

    def step(i):
        q, k, v = inputs[i % 4]
        wl.pre_step()
        st = kv.pred_attn_batch(wl.descs, wl.positions(), q, k, v, out, lse)
        assert not any(st)
        wl.advance()

    for i in range(20):
        step(i)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(n):
            step(i)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    rows = [(e.time_range.start, e.time_range.end, e.name[:60]) for e in evs]
    t0 = rows[0][0]
    # steps start at the upload of the step packet (a memcpy or the upload kernel)
    starts = [i for i, r in enumerate(rows) if "Memcpy" in r[2] or "upload" in r[2] or "step_prologue" in r[2]]
    print(f"{len(rows)} device activities over {(rows[-1][1] - t0):.1f} us for {n} steps: "
          f"{(rows[-1][1] - t0) / n:.1f} us per step")
    for si in range(min(4, len(starts) - 1)):
        a, b = starts[si + n // 2 if si + n // 2 < len(starts) - 1 else si], None
        a = starts[len(starts) // 2 + si]
        b = starts[len(starts) // 2 + si + 1] if len(starts) // 2 + si + 1 < len(starts) else len(rows)
        base = rows[a][0]
        print(f"-- step (next step starts at +{rows[b][0] - base:.1f} us)" if b < len(rows) else "-- step")
        prev_end = base
        for r in rows[a:b]:
            print(f"   +{r[0] - base:7.1f} us  dur {r[1] - r[0]:7.1f}  gap {r[0] - prev_end:6.1f}  {r[2]}")
            prev_end = max(prev_end, r[1])


if __name__ == "__main__":
    main()
