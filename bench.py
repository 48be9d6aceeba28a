#!/usr/bin/env python
"""Benchmark of the batched `pred` hot path (BASELINE.json metric: pred decode tokens/s at the Llama-3-8B
attention shape and KV-attention HBM GB/s vs peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

One step = one batched pred over the workload's batch: batch assembly + validate/reserve
(host C++), one metadata H2D copy, the table-delta/copy-on-write prologue kernel, and the fused
append + split-KV decode attention kernel, through the C ABI.  N > 1: one process per GPU (torchrun),
each rank runs its own LIPs (weak scaling, no collective on the step); the time is the max over ranks.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pred decode tokens/s (8B-attn shape) and KV-attn HBM GB/s vs peak at 1/2/4/8 GPU"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="bounded oracle sample for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--real-scores", action="store_true",
                    help="cfg5hh: pick the evicted tokens by the H2O scores of a decode step (pred_attn_scores) "
                         "instead of synthetic Exp(1) scores")
    ap.add_argument("--prefix-splits", type=int, default=0,
                    help="cascade tuning: key splits per shared run (KVFS_OPT_PREFIX_SPLITS; 0 = auto)")
    ap.add_argument("--cutover", type=int, default=-1,
                    help="tuning: n_q at or above which the tcgen05 chunk kernel runs (KVFS_OPT_CHUNK_CUTOVER; "
                         "-1 = library default 8)")
    ap.add_argument("--decode-chunks", type=int, default=-1,
                    help="tuning: dynamic decode scheduling with this many chunks (KVFS_OPT_DECODE_CHUNKS; 0 = static; "
                         "-1 = library default)")
    ap.add_argument("--decode-ctas", type=int, default=0,
                    help="tuning: decode-kernel ring count (KVFS_OPT_DECODE_CTAS; 0 = auto)")
    ap.add_argument("--hh-drop", type=float, default=0.0,
                    help="cfg5hh tuning: fraction of each file evicted (default 0.5, the SURVEY workload)")
    ap.add_argument("--holes-gather", type=int, default=-1,
                    help="tuning: KVFS_OPT_HOLES_GATHER (1 = TMA gather4 of retained rows in holey pages; -1 = default)")
    ap.add_argument("--fused-scores", action="store_true",
                    help="with --scores / --real-scores: the decode kernel writes its logits into a registered buffer "
                         "(kvfs_set_logits_buffer) and the score pass reads them (K10) instead of K (K9)")
    ap.add_argument("--scores", action="store_true",
                    help="also run pred_attn_scores (NEXT-2, H2O score accumulation) every timed step")
    ap.add_argument("--migrate", action="store_true",
                    help="cfg5 at N > 1: skewed 160/96 LIP placement on even/odd ranks, one rebalance round "
                         "(kvfs_pack -> NCCL send/recv -> kvfs_unpack), then the timed decode steps")
    ap.add_argument("--sched", action="store_true",
                    help="cfg2 LIPs driven by the inference scheduler (kvfs_sched_*) in an event loop: wall-clock "
                         "tokens/s with scheduler-formed batches")
    ap.add_argument("--think-us", type=float, default=200.0, help="--sched: mean LIP think time between preds (us)")
    ap.add_argument("--w-max-us", type=float, default=1000.0, help="--sched: scheduler W_max (us)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="functional multi-process run on ONE GPU (every rank on cuda:0, gloo with host staging); "
                         "not a measurement")
    return ap.parse_args()


def relaunch_distributed(args) -> int:
    """`bench.py --gpus N` started without torchrun: re-execute this script under torch.distributed.run with
    N processes (one per GPU, rendezvous on 127.0.0.1) and return its exit code.  Rank 0 prints the line."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "4")
    print(f"[bench] relaunching under torch.distributed.run: {args.gpus} ranks", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def tensor_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), \
            "measured (MEASURED_PEAKS.json bf16_tflops_sustained: cuBLAS bf16 GEMM, 4 s back to back)"
    return 1400.0, "fallback (B200_PROFILING.md sustained bf16)"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: copy bandwidth)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md recipe)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _one(self):
        try:
            r = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
            if r.returncode == 0 and r.stdout.strip():
                self.samples.append([x.strip() for x in r.stdout.strip().split(",")])
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._one()
            self._stop.wait(0.1)

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join()
        if not self.samples:
            self._one()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def dist_setup(args):
    """One process per GPU (torchrun env).  NCCL for N > 1; --share-gpu: every rank on cuda:0 over gloo."""
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if world != args.gpus:
        print(f"[bench] warning: --gpus {args.gpus} but WORLD_SIZE={world}; using {world}", file=sys.stderr)
    devi = 0 if args.share_gpu else local
    torch.cuda.set_device(devi)
    if world > 1:
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", devi))
    return world, rank, local, devi


def all_max(x: float, world: int) -> float:
    """Max over ranks (CPU tensor under gloo, device tensor under NCCL)."""
    if world == 1:
        return float(x)
    import torch
    import torch.distributed as dist

    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rank_info(world: int, info: dict):
    if world == 1:
        return [info]
    import torch.distributed as dist

    out = [None] * world
    dist.all_gather_object(out, info)
    return out


NVLINK_GBS = 900.0  # NVLink 5 per direction per GPU (B200_PROFILING.md / SURVEY §8(e))


def migration_summary(per_rank):
    """Per pair of the rebalance: bytes moved, device-timed pack (K6 gather) / transfer / unpack (K6 scatter)
    and their GB/s (pack / unpack: read + write of the page bytes against the HBM peak; transfer against
    NVLink 5's ~900 GB/s per direction)."""
    peak, _ = peaks()
    pairs = []
    by_rank = {x["rank"]: x for x in per_rank}
    for x in per_rank:
        if x.get("role") != "send":
            continue
        r = by_rank.get(x.get("peer"), {})
        b = x.get("buf_bytes") or 0
        xfer = max(v for v in (x.get("send_ms"), r.get("recv_ms"), 1e-9) if v is not None)
        p = {"src": x["rank"], "dst": x.get("peer"), "files": x.get("files"), "moved": x.get("moved"),
             "bytes": b, "pack_ms": x.get("pack_ms"), "pack_host_ms": x.get("pack_host_ms"),
             "send_ms": x.get("send_ms"), "recv_ms": r.get("recv_ms"), "unpack_ms": r.get("unpack_ms"),
             "unpack_host_ms": r.get("unpack_host_ms")}
        if b and x.get("pack_ms"):
            p["pack_gbs"] = 2 * b / (x["pack_ms"] / 1000) / 1e9
            p["pack_frac_hbm"] = p["pack_gbs"] / peak
        if b:
            p["xfer_gbs"] = b / (xfer / 1000) / 1e9
            p["xfer_frac_nvlink"] = p["xfer_gbs"] / NVLINK_GBS
        if b and r.get("unpack_ms"):
            p["unpack_gbs"] = 2 * b / (r["unpack_ms"] / 1000) / 1e9
            p["unpack_frac_hbm"] = p["unpack_gbs"] / peak
        pairs.append(p)
    return {"pairs": pairs, "per_rank": per_rank, "nvlink_gbs_ref": NVLINK_GBS,
            "note": "device-timed (CUDA events; the host part of kvfs_pack / kvfs_unpack is reported separately as "
                    "*_host_ms); transfer = max(sender send, receiver recv) event time of the page buffer"}


def pci_bus_id(devi: int):
    try:
        import torch

        return torch.cuda.get_device_properties(devi).pci_bus_id
    except Exception:
        return None


# ------------------------------------------------------------------------------------------ CPU oracle
def host_op_costs(wl, reps: int = 200):
    """SURVEY §8(d) host-op cost: microseconds per KVFS host operation and per pred planning call, measured
    on a host-only ctx (the C++ control plane alone, through the C ABI) holding the workload's file shape:
    n_files x file_len tokens.  The device-side cost of the same calls is inside the timed step."""
    import numpy as np

    from paper_2510_25412_b200 import kvfs as K

    s = wl.shape
    n_files = min(wl.n_files, 256)
    L0 = wl.file_len + wl.prefix_len
    per = -(-L0 // s.P) + 8
    c = K.KVFS(1, s.Hq, s.Hkv, s.D, s.P, n_files * per + 4 * per + 64, max_batch_rows=max(16, n_files * wl.n_q),
               max_batch_descs=max(16, n_files), device=-1)
    pos = np.arange(L0, dtype=np.int32)
    fds = []
    for f in range(n_files):
        fd = c.open(f"h{f}")
        c.append(fd, pos)
        fds.append(fd)
    out = {}

    def timed(fn, n):
        t0 = time.perf_counter()
        for i in range(n):
            fn(i)
        return 1e6 * (time.perf_counter() - t0) / n

    descs = np.array([[fd, wl.n_q] for fd in fds], dtype=np.int32)
    nxt = np.full(n_files, L0, dtype=np.int64)
    offs = np.arange(wl.n_q, dtype=np.int64)

    def plan(i):
        step, _ = c.pred_step_begin(descs, (nxt[:, None] + offs[None, :]).reshape(-1).astype(np.int32))
        c.pred_step_end(step)
        nxt[:] += wl.n_q

    out["pred_planning_per_step"] = timed(plan, reps)
    out["pred_planning_per_descriptor"] = out["pred_planning_per_step"] / n_files
    out["truncate"] = timed(lambda i: c.truncate(fds[i % n_files], int(L0 - 1 - (i // n_files))), reps)
    out["evict_1_token_at_4"] = timed(lambda i: c.evict(fds[i % n_files], [(4, 5)]), reps)
    out["fork"] = timed(lambda i: c.fork(fds[i % n_files], f"fk{i}"), min(reps, 64))
    out["offload_meta"] = timed(lambda i: c.offload(fds[i]), min(reps, n_files // 2))
    out["restore_meta"] = timed(lambda i: c.restore(fds[i]), min(reps, n_files // 2))
    sch = K.Scheduler(w_max=0.01, b_max=64)
    out["sched_enqueue"] = timed(lambda i: sch.enqueue(fds[i % n_files], [i], 1e-5 * i), reps)
    out["sched_form"] = timed(lambda i: sch.form(1.0 + i), 20)
    return {"unit": "us", "ctx": f"host-only, {n_files} files x {L0} tokens, n_q {wl.n_q}",
            **{k: round(v, 2) for k, v in out.items()}}


def oracle_sample(cfg_name: str, seconds: float, max_steps: int = None, n_sample: int = 8):
    """Time the oracle (as it stands) on a bounded sample of the workload: n_sample of the LIPs with their
    full files and per-step policies, one pred per step, repeated until `seconds` elapse (or max_steps)."""
    from oracle.workload import OracleWorkload
    from synth.configs import CONFIGS

    c = CONFIGS[cfg_name]
    n_sample = min(n_sample, c["n_files"])
    cap = max_steps if max_steps is not None else 10 ** 9
    ow = OracleWorkload(cfg_name, range(n_sample), max_steps=min(cap, 256))
    try:
        from threadpoolctl import threadpool_info
        blas_threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        blas_threads = None
    cores = len(os.sched_getaffinity(0))
    rows = steps = 0
    t0 = time.perf_counter()
    while steps < cap and (max_steps is not None or time.perf_counter() - t0 < seconds or steps == 0):
        st, _, _ = ow.run_step()
        assert all(x == 0 for x in st), st
        rows += n_sample * c["n_q"]
        steps += 1
    el = time.perf_counter() - t0
    return {"value": rows / el, "unit": "tokens/s", "cores": cores, "blas_threads": blas_threads,
            "kind": "oracle",
            "sample": f"{n_sample} of {c['n_files']} LIPs (full files, n_q={c['n_q']}, same per-step policy), "
                      f"{steps} preds in {el:.1f} s via oracle.Oracle.pred_batch (numpy fp64)",
            "steps": steps, "seconds": el}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from synth.configs import CONFIGS

    c = CONFIGS[args.config]
    # warm-up steps are run untimed, then exactly K timed steps (each a bounded 4-LIP sample)
    oracle_sample(args.config, 0.0, max_steps=args.warmup, n_sample=4)
    cb = oracle_sample(args.config, 0.0, max_steps=args.steps, n_sample=4)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * cb["seconds"] / cb["steps"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (counter-based generator, DESIGN.md input recipe)",
        "config": {"workload": c["workload"], "reference_sample": cb["sample"]},
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------ ours
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2510_25412_b200 import kvfs as K
    from paper_2510_25412_b200.workloads import DecodeWorkload

    world, rank, local, devi = dist_setup(args)
    W, Kst = args.warmup, args.steps
    n_e2e = 0 if args.no_e2e else Kst
    # rank r holds its own LIPs (generator owners r * n_files ...) and its own step inputs: weak scaling
    n_files0 = DecodeWorkload.config_files(args.config)
    migration = None
    if args.migrate and world > 1:
        # SURVEY §8(d) cfg5 "Migration": skewed placement, n + n/4 LIPs on even ranks and n - n/4 on odd ranks
        # (160 / 96 at cfg5's 128 per GPU; an odd last rank keeps n), then one rebalance round moves n/4
        # files even -> odd over NCCL (kvfs_pack -> send / recv -> kvfs_unpack, ACKed); the timed steps run
        # on the balanced placement
        skew = n_files0 // 4
        odd_last = world % 2 == 1 and rank == world - 1
        n_mine = n_files0 if odd_last else (n_files0 + skew if rank % 2 == 0 else n_files0 - skew)
        wl = DecodeWorkload(args.config, steps_total=W + Kst + n_e2e + 3, device=devi, n_files=n_mine,
                            owner_base=rank * (n_files0 + skew), room_files=0 if rank % 2 == 0 else skew + 2,
                            step_owner_base=rank * 100_000)
        from paper_2510_25412_b200.parallel import rebalance

        torch.cuda.synchronize()
        dist.barrier()
        mstats = {}
        files = rebalance(wl.kv, wl.file_map(), stats=mstats)
        torch.cuda.synchronize()
        wl.set_files(files)
        mstats["lips_after"] = wl.n_files
        mstats["moved_files"] = len(mstats.get("moved_files", []))
        migration = gather_rank_info(world, dict(mstats, rank=rank, lips_before=n_mine))
    else:
        wl = DecodeWorkload(args.config, steps_total=W + Kst + n_e2e + 3, device=devi, owner_base=rank * n_files0,
                            step_owner_base=rank * 100_000)
    if args.prefix_splits:
        wl.kv.set_option(K.OPT_PREFIX_SPLITS, args.prefix_splits)
    if args.decode_ctas:
        wl.kv.set_option(K.OPT_DECODE_CTAS, args.decode_ctas)
    if args.cutover >= 0:
        wl.kv.set_option(K.OPT_CHUNK_CUTOVER, args.cutover)
    if args.decode_chunks >= 0:
        wl.kv.set_option(K.OPT_DECODE_CHUNKS, args.decode_chunks)
    if args.holes_gather >= 0:
        wl.kv.set_option(K.OPT_HOLES_GATHER, args.holes_gather)
    s = wl.shape
    kv = wl.kv
    T = wl.n_files * wl.n_q
    inputs = [wl.make_inputs(i) for i in range(W + Kst)]
    out = torch.empty((T, s.Hq, s.D), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((T, s.Hq), dtype=torch.float32, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()

    for i in range(W):
        q, k, v = inputs[i]
        wl.pre_step()
        st = kv.pred_attn_batch(wl.descs, wl.positions(), q, k, v, out, lse)
        assert all(x == 0 for x in st), st
        wl.advance()
    torch.cuda.synchronize()
    barrier()
    launches0 = kv.counter(K.CTR_KERNEL_LAUNCHES)
    h2d0 = kv.counter(K.CTR_H2D_BYTES)
    sampler = ClockSampler(devi)
    sampler.start()
    torch.cuda.synchronize()
    barrier()
    # The attention layer's device time (first to last kernel of pred_attn_layer: chunk / shared-prefix /
    # decode) comes from CUDA events the library records on the launching stream around its own launches
    # (KVFS_OPT_TIMING) inside the timed loop, on every `every`-th step only: two event records cost ~16 us of
    # host time and break the programmatic-launch chain of the step, which on a short step (cfg3) made a fully
    # instrumented loop host-bound (0.059 instead of 0.050 ms per step).  ~20 sampled steps per run; with
    # --scores every step is instrumented (the score pass is timed by Python events around its call).
    every = 1 if args.scores else max(1, Kst // 20)
    kv.set_option(K.OPT_TIMING, every)
    kv.counter(K.CTR_LAYER_DEVICE_NS)  # start a new sum (the warm-up steps were not timed)
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(Kst)] if args.scores else None
    ev2 = [torch.cuda.Event(enable_timing=True) for _ in range(Kst)] if args.scores else None
    scores_buf = None
    if args.scores:
        scores_buf = torch.empty(int((wl.lens + wl.n_q).sum()) + T + 16, dtype=torch.float32, device="cuda")
        if args.fused_scores:
            kv.set_logits_buffer(logits_buffer(wl, Kst))
    alg_bytes, alg_flops, logical = [], [], []
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    lens_seen = []  # per-step retained lengths; the byte / flop accounting is computed after the timed loop
    host_t0 = time.perf_counter()
    t_start.record()
    for i in range(Kst):
        q, k, v = inputs[W + i]
        wl.pre_step()
        lens_seen.append(wl.lens.copy())
        if args.scores:
            step, st = kv.pred_step_begin(wl.descs, wl.positions())
            kv.pred_attn_layer(step, 0, q, k, v, out, lse)
            ev1[i].record()
            la = wl.lens + wl.n_q
            kv.pred_attn_scores(step, 0, q, lse, scores_buf, np.concatenate([[0], np.cumsum(la)[:-1]]))
            ev2[i].record()
            kv.pred_step_end(step)
        else:
            kv.pred_attn_batch(wl.descs, wl.positions(), q, k, v, out, lse)
        wl.advance()
    t_end.record()
    host_s = time.perf_counter() - host_t0
    for ln in lens_seen:
        alg_bytes.append(wl.algorithmic_bytes(ln))
        alg_flops.append(wl.flops(ln))
        logical.append(wl.logical_kv_bytes(ln))
    torch.cuda.synchronize()
    barrier()
    sampler.stop()
    ms_total = t_start.elapsed_time(t_end)
    launches = kv.counter(K.CTR_KERNEL_LAUNCHES) - launches0
    h2d = kv.counter(K.CTR_H2D_BYTES) - h2d0
    # the sampled steps' own byte / flop counts (the files grow by n_q per step)
    kernel_bytes = [b for i, b in enumerate(alg_bytes) if i % every == 0]
    kernel_flops = [f for i, f in enumerate(alg_flops) if i % every == 0]
    layer_ns = kv.counter(K.CTR_LAYER_DEVICE_NS)
    n_timed = len(kernel_bytes)
    assert kv.counter(K.CTR_LAYER_TIMED) == n_timed, (kv.counter(K.CTR_LAYER_TIMED), n_timed)
    kv.set_option(K.OPT_TIMING, 0)
    kernel_ms = [layer_ns / 1e6 / n_timed] * n_timed
    ms_max = all_max(ms_total, world)
    ms_step = ms_max / Kst
    value = world * T * Kst / (ms_max / 1000.0)

    # ---- end to end: host (pinned) inputs -> device -> pred -> host outputs, every step, through the C ABI's
    # host-buffer call pred_attn_batch_host (include/kvfs.h): the library copies each step's Q / K_new / V_new
    # into one of its two device slots on its own copy stream, runs the pred on the compute stream and copies
    # out + lse back on a second copy stream, so consecutive steps overlap (the input copy of step i+1 and the
    # output copy of step i-1 run beside the pred of step i).  Every step moves its full inputs in and its
    # full result out inside the timed region; the region ends after pred_host_fence (all output copies).
    e2e = None
    if n_e2e:
        def pinned(shapes_dtypes):
            # one pinned buffer per step, the tensors at 256-byte aligned offsets (as a serving loop packs a step)
            sizes = [int(np.prod(sh)) * torch.empty((), dtype=dt).element_size() for sh, dt in shapes_dtypes]
            offs = np.concatenate([[0], np.cumsum([(z + 255) // 256 * 256 for z in sizes])]).astype(int)
            buf = torch.empty(int(offs[-1]), dtype=torch.uint8).pin_memory()
            return [buf[o:o + z].view(dt).view(sh) for (sh, dt), o, z in zip(shapes_dtypes, offs, sizes)]

        in_sd = [(tuple(x.shape), x.dtype) for x in inputs[0]]
        out_sd = [(tuple(out.shape), out.dtype), (tuple(lse.shape), lse.dtype)]
        ring_h = []
        for i in range(4):
            views = pinned(in_sd)
            for dst, src in zip(views, inputs[i % len(inputs)]):
                dst.copy_(src.cpu())
            ring_h.append(views)
        host_out = [pinned(out_sd) for _ in range(2)]
        cs = torch.cuda.current_stream()
        for i in range(2):  # untimed: the library sizes its two device slots on first use
            wl.pre_step()
            kv.pred_attn_batch_host(wl.descs, wl.positions(), *ring_h[i], *host_out[i])
            wl.advance()
        kv.pred_host_fence()
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        for i in range(n_e2e):
            qh, kh, vh = ring_h[i % 4]
            oh, lh = host_out[i % 2]
            wl.pre_step()
            kv.pred_attn_batch_host(wl.descs, wl.positions(), qh, kh, vh, oh, lh)
            wl.advance()
        kv.pred_host_fence()
        e1.record(cs)
        torch.cuda.synchronize()
        et = all_max(e0.elapsed_time(e1), world)
        h2d_b = int(sum(x.numel() * x.element_size() for x in ring_h[0]))
        d2h_b = int(sum(x.numel() * x.element_size() for x in host_out[0]))
        e2e = {"value": world * T * n_e2e / (et / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b, "steps": n_e2e,
               "note": "pred_attn_batch_host through the C ABI with pinned host Q/K_new/V_new and out/lse: the "
                       "library's H2D copy stream, the pred on the compute stream, its D2H copy stream; steps "
                       "pipelined over two device slots; the timed region ends after pred_host_fence"}

    ranks = gather_rank_info(world, {
        "rank": rank, "device": devi, "pci_bus_id": pci_bus_id(devi), "lips": wl.n_files, "ms_total": ms_total,
        "kernel_ms_mean": statistics.mean(kernel_ms), "clocks": sampler.summary(),
        "e2e_value": None if e2e is None else e2e["value"]})
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    tc_peak, tc_src = tensor_peak()
    k_ms = statistics.mean(kernel_ms)
    achieved = statistics.mean(kernel_bytes) / (k_ms / 1000.0) / 1e9
    flops_mean = statistics.mean(kernel_flops)
    t_bytes = statistics.mean(kernel_bytes) / (peak * 1e9)
    t_flops = flops_mean / (tc_peak * 1e12)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak}
    if t_flops > 0.5 * t_bytes:
        # chunk workloads sit at the ridge: report the binding roof (the larger ideal time)
        ach_tf = flops_mean / (k_ms / 1000.0) / 1e12
        if t_flops >= t_bytes:
            roof = {"bound": "tensor", "achieved": ach_tf, "peak": tc_peak, "unit": "TFLOP/s", "frac": ach_tf / tc_peak}
            peak_src = tc_src
        roof["ridge"] = {"ideal_ms_hbm": 1000 * t_bytes, "ideal_ms_tensor": 1000 * t_flops,
                         "frac_of_max_ideal": max(t_bytes, t_flops) / (k_ms / 1000.0),
                         "achieved_gbs": achieved, "achieved_tflops": ach_tf}
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "decode_traffic.json")
    if os.path.exists(tp):
        try:
            t = json.load(open(tp)).get(args.config)
            traffic, traffic_src = t["traffic_bytes_per_launch"], t["source"]
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": Kst, "warmup": W,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (counter-based generator seed %d, DESIGN.md input recipe)" % wl.seed,
        "config": {"workload": wl.desc, "lips_per_gpu": wl.n_files, "file_len_start": wl.file_len + wl.prefix_len,
                   "n_q": wl.n_q, "n_q_heads": s.Hq, "n_kv_heads": s.Hkv, "head_dim": s.D, "page_size": s.P,
                   "layers_per_step": 1,
                   "parallelism": f"dp{world} (LIPs partitioned by process, no collective)"
                   + (" [--share-gpu: every rank on cuda:0, functional run, not a measurement]" if args.share_gpu else ""),
                   "l2": ("inputs larger than L2 (K/V read per step %.2f GB > 126 MB L2)" % (logical[0] / 1e9)
                          if logical[0] > 126e6 * 4 else
                          "unique K/V %.0f MB per step; the CoW-shared prefix is L2-resident by design" % (alg_bytes[0] / 1e6))},
        "roofline": dict(roof, traffic=traffic, traffic_source=traffic_src, kernel=wl.dominant_kernel(args.cutover if args.cutover >= 0 else 8),
                         kernel_ms_mean=k_ms, peak_source=peak_src,
                         kernel_timing="CUDA events the library records on the launching stream before the first "
                                       "and after the last kernel of each pred_attn_layer (KVFS_OPT_TIMING, "
                                       "KVFS_CTR_LAYER_DEVICE_NS), mean over every %d-th step of the timed loop "
                                       "(%d steps; algorithmic bytes of those steps)" % (every, len(kernel_bytes)),
                         algorithmic_bytes_per_launch=statistics.mean(kernel_bytes),
                         algorithmic_flops_per_launch=flops_mean),
        "gpu_launches": launches,
        "clocks": sampler.summary(),
        "ranks": ranks if world > 1 else None,
        "extra": {"kv_attn_gbs_step": statistics.mean(alg_bytes) / (ms_step / 1000.0) / 1e9,
                  "logical_kv_bytes_per_step": statistics.mean(logical),
                  "logical_gbs_kernel": statistics.mean(logical) / (k_ms / 1000.0) / 1e9,
                  "tok_s_32_layer_equiv": value / 32.0, "host_s_per_step": host_s / Kst,
                  "h2d_metadata_bytes_per_step": h2d / Kst,
                  "decode_ctas": kv.counter(K.CTR_LAST_DECODE_CTAS),
                  "host_ops_us": host_op_costs(wl)},
    }
    if migration is not None:
        line["migration"] = migration_summary(migration)
        line["config"]["workload"] += (" | migration: skewed %d/%d LIPs on even/odd ranks, one rebalance round "
                                       "(kvfs_pack, NCCL send/recv, kvfs_unpack) before the timed steps"
                                       % (n_files0 + n_files0 // 4, n_files0 - n_files0 // 4))
    if args.scores:
        sc_ms = statistics.mean(a.elapsed_time(b) for a, b in zip(ev1, ev2))
        k_bytes = statistics.mean(logical) / 2
        if args.fused_scores:
            # K10 reads the logits (Hq fp32 per key and row) and the lse; K1 wrote them during the attention
            n_fused = kv.counter(K.CTR_LAST_FUSED_SCORES)
            lg_bytes = int(statistics.mean(float((ln + wl.n_q).sum()) for ln in lens_seen)) * wl.n_q * s.Hq * 4
            line["extra"]["scores"] = {
                "kernel": "logit_scores_kernel (K10, fused H2O scores from the decode kernel's logits)",
                "fused_descriptors": n_fused, "ms_mean": sc_ms, "logit_bytes_per_step": lg_bytes,
                "gbs": lg_bytes / (sc_ms / 1000.0) / 1e9, "frac_of_peak": lg_bytes / (sc_ms / 1000.0) / 1e9 / peak,
                "overhead_vs_attention": sc_ms / k_ms,
                "note": "the attention kernel time (roofline.kernel_ms_mean) includes writing the logits"}
        else:
            line["extra"]["scores"] = {
                "kernel": "scores_kernel (K9, H2O attention-score accumulation, second pass over K)",
                "ms_mean": sc_ms, "k_bytes_per_step": k_bytes, "gbs": k_bytes / (sc_ms / 1000.0) / 1e9,
                "frac_of_peak": k_bytes / (sc_ms / 1000.0) / 1e9 / peak,
                "overhead_vs_attention": sc_ms / k_ms}
    if e2e:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = oracle_sample(args.config, args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def logits_buffer(wl, steps: int):
    """Device buffer for the fused scores (include/kvfs.h kvfs_set_logits_buffer): 4 Hq P n_q (entries + ceil(n_q / P))
    bytes per descriptor, sized for the longest files of the run (`steps` more tokens per file)."""
    import torch

    s = wl.shape
    ent = (wl.lens + steps * wl.n_q + s.P - 1) // s.P + 1 + (wl.n_q + s.P - 1) // s.P
    floats = int((ent * s.P).sum()) * wl.n_q * s.Hq + 32 * len(ent)  # + 128-byte alignment per descriptor
    return torch.empty(floats + 64, dtype=torch.float32, device="cuda")


def evict_ranges_heavy_hitter(seed: int, f: int, n: int, drop: int, sink: int = 4, recent: int = 1024):
    """cfg5(ii) policy: evict the `drop` lowest Exp(1) synthetic scores of file f, protecting
    the first `sink` and last `recent` tokens; ties -> lower index. Returns sorted disjoint [a, b) ranges."""
    from synth.workloads import heavy_hitter_ranges

    return heavy_hitter_ranges(seed, f, n, drop, sink, recent)


def run_heavy_hitter(args):
    """cfg5(ii): 128 LIPs x 65536 tokens, evict the 32768 lowest-score tokens (lazy holes, ~50%-dense pages),
    time decode, compact every file (K5 gather), time decode again.  One JSON line."""
    import numpy as np
    import torch

    from paper_2510_25412_b200 import kvfs as K
    from paper_2510_25412_b200.workloads import STEP_OWNER
    from synth.configs import Shape
    from synth.workloads import TAG_K, TAG_Q, TAG_V, rows_torch

    torch.cuda.set_device(0)
    s, n_files, L0, seed = Shape(32, 8, 128, 16), 128, 65536, 1005
    W, Kst = args.warmup, args.steps
    n_pages = n_files * (L0 // 16 + 4) + n_files * (L0 // 32 + 8)
    kv = K.KVFS(1, s.Hq, s.Hkv, s.D, s.P, n_pages, max_batch_rows=n_files, max_batch_descs=n_files, device=0)
    if args.holes_gather >= 0:
        kv.set_option(K.OPT_HOLES_GATHER, args.holes_gather)
    dev = torch.device("cuda", 0)
    fds = []
    for f in range(n_files):
        fd = kv.open(f"hh{f}")
        k = rows_torch(seed, TAG_K, 0, f, 0, L0, s.Hkv * s.D, device=dev).view(1, L0, s.Hkv, s.D)
        v = rows_torch(seed, TAG_V, 0, f, 0, L0, s.Hkv * s.D, device=dev).view(1, L0, s.Hkv, s.D)
        kv.append(fd, list(range(L0)), k, v)
        fds.append(fd)
        del k, v
    torch.cuda.synchronize()
    descs = np.array([[fd, 1] for fd in fds], dtype=np.int32)
    scores_info = None
    if args.real_scores:
        # NEXT-2 in use: one decode step with H2O score accumulation (pred_attn_scores), then evict the L0 / 2
        # lowest-score tokens of every file (first 4 and last 1024 protected; ties -> lower index)
        own = STEP_OWNER + 10 ** 6
        q, k1, v1 = (rows_torch(seed, t, 0, own, 0, n_files, w, device=dev).view(n_files, -1, s.D)
                     for t, w in ((TAG_Q, s.Hq * s.D), (TAG_K, s.Hkv * s.D), (TAG_V, s.Hkv * s.D)))
        out0 = torch.empty((n_files, s.Hq, s.D), dtype=torch.bfloat16, device=dev)
        lse0 = torch.empty((n_files, s.Hq), dtype=torch.float32, device=dev)
        n1 = L0 + 1
        sc = torch.empty(n_files * n1, dtype=torch.float32, device=dev)
        if args.fused_scores:  # K1 writes the logits, K10 sums them (kvfs_set_logits_buffer)
            kv.set_logits_buffer(torch.empty(n_files * ((L0 // s.P + 2) * s.P * s.Hq + 32) + 64, dtype=torch.float32,
                                             device=dev))
        step, st = kv.pred_step_begin(descs, np.full(n_files, L0, dtype=np.int32))
        assert st == [0] * n_files
        kv.pred_attn_layer(step, 0, q, k1, v1, out0, lse0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        kv.pred_attn_scores(step, 0, q, lse0, sc, np.arange(n_files, dtype=np.int64) * n1)
        e1.record()
        kv.pred_step_end(step)
        torch.cuda.synchronize()
        scores_ms = e0.elapsed_time(e1)
        n_fused = kv.counter(K.CTR_LAST_FUSED_SCORES)
        kv.set_logits_buffer(None)
        sch = sc.view(n_files, n1).cpu().numpy().astype(np.float64)
        t0 = time.perf_counter()
        from synth.workloads import lowest_score_ranges

        for f, fd in enumerate(fds):
            kv.evict(fd, lowest_score_ranges(sch[f], L0 // 2))
        host_sel_s = time.perf_counter() - t0
        scores_info = {"kernel": ("logit_scores_kernel (K10, fused: the decode kernel's logits)" if n_fused else
                                  "scores_kernel (K9)") + " over 128 x 65537 tokens", "scores_ms": scores_ms,
                       "fused_descriptors": n_fused,
                       "k_gbs": n_files * n1 * s.Hkv * s.D * 2 / (scores_ms / 1000) / 1e9,
                       "host_select_and_evict_s": host_sel_s,
                       "score_sum_check": float(sch.sum() / (n_files * s.Hq))}  # = 1 (softmax weights)
        next_pos = np.full(n_files, L0 + 1, dtype=np.int64)
        lens = np.full(n_files, L0 + 1 - L0 // 2, dtype=np.int64)
    else:
        drop = int(L0 * args.hh_drop) if args.hh_drop > 0 else L0 // 2
        for f, fd in enumerate(fds):
            kv.evict(fd, evict_ranges_heavy_hitter(seed, f, L0, drop))
        next_pos = np.full(n_files, L0, dtype=np.int64)
        lens = np.full(n_files, L0 - drop, dtype=np.int64)
    out = torch.empty((n_files, s.Hq, s.D), dtype=torch.bfloat16, device=dev)
    row_kv = s.Hkv * s.D * 2

    def decode(steps, step0):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ins = []
        for i in range(steps):
            own = STEP_OWNER + step0 + i
            ins.append(tuple(rows_torch(seed, t, 0, own, 0, n_files, w, device=dev).view(n_files, -1, s.D)
                             for t, w in ((TAG_Q, s.Hq * s.D), (TAG_K, s.Hkv * s.D), (TAG_V, s.Hkv * s.D))))
        torch.cuda.synchronize()
        e0.record()
        for q, k, v in ins:
            st = kv.pred_attn_batch(descs, next_pos.astype(np.int32), q, k, v, out)
            assert st == [0] * n_files
            next_pos[:] += 1
            lens[:] += 1
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    sampler = ClockSampler(0)
    sampler.start()
    decode(W, 0)
    alg_before = 2 * int(lens.sum()) * row_kv
    ms_before = decode(Kst, W)
    retained = int(lens.sum())
    # kvfs_compact_files of all files: (1) as the caller sees it (CUDA events around the call: the host R1 /
    # table work and the device gathers, overlapped by file groups) and (2) the device work alone (the
    # library's own events around each group's upload + K5 launches, KVFS_OPT_TIMING)
    kv.set_option(K.OPT_TIMING, 1)
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_host0 = time.perf_counter()
    c0.record()
    kv.compact_files(fds)  # one call: page / table work in order, host position passes on worker threads
    c1.record()
    host_ms = 1000 * (time.perf_counter() - t_host0)
    torch.cuda.synchronize()
    ms_call = c0.elapsed_time(c1)
    ms_compact = kv.counter(K.CTR_COMPACT_DEVICE_NS) / 1e6
    kv.set_option(K.OPT_TIMING, 0)
    compact_bytes = 2 * 2 * retained * row_kv  # K and V of every retained token: read + write
    decode(W, W + Kst)
    alg_after = 2 * int(lens.sum()) * row_kv
    ms_after = decode(Kst, 2 * W + Kst)
    sampler.stop()
    peak, peak_src = peaks()
    traffic = None
    tp = os.path.join(ROOT, "profiles", "decode_traffic.json")
    tinfo = {}
    if os.path.exists(tp):
        try:
            tinfo = json.load(open(tp)).get("cfg5hh", {})
            traffic = tinfo.get("k5_traffic_bytes_per_file")
        except Exception:
            tinfo = {}
    line = {
        "metric": METRIC, "value": n_files / (ms_after / 1000.0), "unit": "tokens/s", "n_gpus": 1, "steps": Kst,
        "warmup": W, "ms_per_step": ms_after, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (counter-based generator seed 1005, Exp(1) scores; DESIGN.md)",
        "config": {"workload": "cfg5(ii): 128 LIPs x 65536-token files, heavy-hitter-like eviction of the 32768 "
                               "lowest Exp(1) scores (first 4 and last 1024 protected), decode before / after "
                               "kvfs_compact", "l2": "inputs larger than L2"},
        "roofline": {"bound": "hbm", "achieved": compact_bytes / (ms_compact / 1000.0) / 1e9, "peak": peak,
                     "unit": "GB/s", "frac": compact_bytes / (ms_compact / 1000.0) / 1e9 / peak,
                     "kernel": "compact_kernel (K5, evict-compact gather, all 128 files, device time only)",
                     "peak_source": peak_src, "traffic": traffic, "traffic_source": tinfo.get("source"),
                     "algorithmic_bytes_per_launch": compact_bytes / n_files},
        "clocks": sampler.summary(),
        "extra": {"decode_ms_holes": ms_before, "decode_gbs_holes": alg_before / (ms_before / 1000.0) / 1e9,
                  "decode_holes_traffic_ratio": tinfo.get("holes_decode_traffic_over_algorithmic"),
                  "decode_ms_compacted": ms_after, "decode_gbs_compacted": alg_after / (ms_after / 1000.0) / 1e9,
                  "compact_ms_device": ms_compact, "compact_ms_call": ms_call, "compact_call_host_ms": host_ms,
                  "compact_bytes": compact_bytes,
                  "retained_tokens": retained, "h2o_scores": scores_info},
    }
    if args.real_scores:
        line["config"]["workload"] = line["config"]["workload"].replace(
            "lowest Exp(1) scores", "lowest H2O scores of a decode step (pred_attn_scores)")
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = oracle_compaction_sample(s, seed)
    print(json.dumps(line), flush=True)


def oracle_compaction_sample(s, seed: int):
    """cpu_baseline for cfg5(ii): the oracle's R7 compaction (oracle.Oracle.compact, NumPy) of ONE 65536-token
    file with the same Exp(1) eviction, timed on the host cores; reported in the K5 roofline's unit (GB/s of
    algorithmic compaction bytes)."""
    import numpy as np

    from oracle import Oracle
    from synth.workloads import TAG_K, TAG_V, heavy_hitter_ranges, rows_np

    L0, w = 65536, s.Hkv * s.D
    o = Oracle(L0 // 16 * 2 + 64, s.P, 1, s.Hkv, s.D)
    fd = o.open("x")
    o.append(fd, list(range(L0)), rows_np(seed, TAG_K, 0, 0, 0, L0, w).reshape(1, L0, s.Hkv, s.D),
             rows_np(seed, TAG_V, 0, 0, 0, L0, w).reshape(1, L0, s.Hkv, s.D))
    o.evict(fd, [tuple(r) for r in heavy_hitter_ranges(seed, 0, L0, L0 // 2).tolist()])
    t0 = time.perf_counter()
    o.compact(fd)
    el = time.perf_counter() - t0
    nbytes = 2 * 2 * (L0 // 2) * w * 2
    return {"value": nbytes / el / 1e9, "unit": "GB/s", "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
            "sample": f"oracle.Oracle.compact of 1 of 128 files (32768 retained tokens, 50% random holes) in {el:.2f} s"}


def run_sched(args):
    """Scheduler-formed batches in the measured loop (§4.4; VERDICT r1 "missing" #5): the
    cfg2 LIPs are driven by an event loop on the host clock.  A LIP whose pred completed (CUDA event) thinks
    for Exp(--think-us) and then enqueues its next decode request (kvfs_sched_enqueue); every iteration asks
    the inference scheduler for a due batch (kvfs_sched_form: Poisson-rate-sized B*, FIFO, one request per
    file, W_max deadline) and runs it with pred_attn_batch.  Wall-clock tokens/s of the whole loop (host
    dispatch, scheduling and GPU), the batch-size distribution and the queueing delay are reported."""
    import heapq

    import numpy as np
    import torch

    from paper_2510_25412_b200 import kvfs as K
    from paper_2510_25412_b200.workloads import DecodeWorkload

    torch.cuda.set_device(0)
    W, Kst = args.warmup, args.steps
    n_batches = max(50, Kst * 20)
    wl = DecodeWorkload("cfg2", steps_total=n_batches + W * 20 + 8, device=0)
    s = wl.shape
    kv = wl.kv
    T = wl.n_files
    q0, k0, v0 = wl.make_inputs(0)
    out = torch.empty((T, s.Hq, s.D), dtype=torch.bfloat16, device="cuda")
    w_max, think = args.w_max_us * 1e-6, args.think_us * 1e-6
    sch = K.Scheduler(w_max=w_max, b_max=T)
    idx = {int(fd): i for i, fd in enumerate(wl.fds)}
    rng = np.random.default_rng(7)
    arrivals = []  # (time, fd)
    t0 = time.perf_counter()
    for fd in wl.fds:
        heapq.heappush(arrivals, (t0 + rng.exponential(think) if think > 0 else t0, int(fd)))
    inflight = []  # (event, [fd])
    stats = {"batches": 0, "rows": 0, "sizes": [], "qdelay": []}
    enq_t = {}

    def loop(n):
        done = 0
        while done < n:
            now = time.perf_counter()
            while inflight and inflight[0][0].query():
                ev, fds = inflight.pop(0)
                t = time.perf_counter()
                for fd in fds:
                    heapq.heappush(arrivals, (t + (rng.exponential(think) if think > 0 else 0.0), fd))
            while arrivals and arrivals[0][0] <= now:
                t, fd = heapq.heappop(arrivals)
                i = idx[fd]
                sch.enqueue(fd, [int(wl.next_pos[i])], t)
                enq_t[fd] = t
            b = sch.form(now)
            if b is None:
                continue
            descs, pos = b
            n_b = len(descs)
            st = kv.pred_attn_batch(descs, pos, q0[:n_b], k0[:n_b], v0[:n_b], out[:n_b])
            assert all(x == 0 for x in st), st
            ev = torch.cuda.Event()
            ev.record()
            fds = [fd for fd, _ in descs]
            for fd in fds:
                i = idx[fd]
                wl.next_pos[i] += 1
                wl.lens[i] += 1
                stats["qdelay"].append(now - enq_t[fd])
            inflight.append((ev, fds))
            stats["batches"] += 1
            stats["rows"] += n_b
            stats["sizes"].append(n_b)
            done += 1

    loop(W * 20)
    torch.cuda.synchronize()
    for k in ("batches", "rows"):
        stats[k] = 0
    stats["sizes"], stats["qdelay"] = [], []
    sampler = ClockSampler(0)
    sampler.start()
    l0 = kv.counter(K.CTR_KERNEL_LAUNCHES)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_a = time.perf_counter()
    e0.record()
    loop(n_batches)
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_a
    sampler.stop()
    sz = np.array(stats["sizes"])
    qd = np.array(stats["qdelay"]) * 1e6
    line = {
        "metric": "pred decode tokens/s with scheduler-formed batches (kvfs_sched, PAPER.md §4.4), wall clock",
        "value": stats["rows"] / wall, "unit": "tokens/s", "n_gpus": 1, "steps": stats["batches"], "warmup": W * 20,
        "ms_per_step": 1000 * wall / stats["batches"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (cfg2 LIPs, seed 1002)",
        "config": {"workload": "cfg2 LIPs (256 x 2048-token files) as a closed population: each LIP thinks Exp(%g us) "
                               "after its pred completes, then enqueues; kvfs_sched_form batches (W_max %g us, "
                               "B_max 256)" % (args.think_us, args.w_max_us)},
        "gpu_launches": kv.counter(K.CTR_KERNEL_LAUNCHES) - l0,
        "device_ms_total": e0.elapsed_time(e1), "wall_s": wall,
        "clocks": sampler.summary(),
        "extra": {"batch_size_mean": float(sz.mean()), "batch_size_p10_p50_p90": [float(x) for x in np.percentile(sz, [10, 50, 90])],
                  "queue_delay_us_p50_p90_p99": [float(x) for x in np.percentile(qd, [50, 90, 99])],
                  "device_busy_frac": e0.elapsed_time(e1) / 1000 / wall,
                  "lambda_target_waiting": list(sch.state())},
    }
    print(json.dumps(line), flush=True)


def run_offload(args):
    """NEXT-3 host tier (R15): offload then restore 32 LIPs x 8192-token files of the 8B
    attention shape (32 MiB of K+V each, exclusively owned), through the C ABI.  One JSON line: GB/s each way."""
    import numpy as np
    import torch

    from paper_2510_25412_b200 import kvfs as K
    from synth.configs import Shape
    from synth.workloads import TAG_K, TAG_V, rows_torch

    torch.cuda.set_device(0)
    s, n_files, n, seed = Shape(32, 8, 128, 16), 32, 8192, 1006
    kv = K.KVFS(1, s.Hq, s.Hkv, s.D, s.P, n_files * (n // 16) + 64, device=0)
    dev = torch.device("cuda", 0)
    fds = []
    for f in range(n_files):
        fd = kv.open(f"o{f}")
        k = rows_torch(seed, TAG_K, 0, f, 0, n, s.Hkv * s.D, device=dev).view(1, n, s.Hkv, s.D)
        v = rows_torch(seed, TAG_V, 0, f, 0, n, s.Hkv * s.D, device=dev).view(1, n, s.Hkv, s.D)
        kv.append(fd, list(range(n)), k, v)
        fds.append(fd)
    torch.cuda.synchronize()
    nbytes = n_files * n * s.Hkv * s.D * 2 * 2
    res = {"offload": [], "restore": []}
    kdev = {"offload": [], "restore": []}
    kv.set_option(K.OPT_TIMING, 1)
    sampler = ClockSampler(0)
    sampler.start()
    for it in range(args.warmup + max(1, min(args.steps, 5))):
        for what in ("offload", "restore"):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            kv.counter(K.CTR_COPY_DEVICE_NS)  # new sum
            t0 = time.perf_counter()
            e0.record()
            for fd in fds:
                getattr(kv, what)(fd)
            e1.record()
            torch.cuda.synchronize()
            if it >= args.warmup:
                res[what].append((e0.elapsed_time(e1), 1000 * (time.perf_counter() - t0)))
                kdev[what].append(kv.counter(K.CTR_COPY_DEVICE_NS) / 1e6)
    sampler.stop()
    off_ms = statistics.median(a for a, _ in res["offload"])
    res_ms = statistics.median(max(a, b) for a, b in res["restore"])  # restore syncs its stream
    k_off, k_res = statistics.median(kdev["offload"]), statistics.median(kdev["restore"])
    pcie = 63.0  # PCIe Gen5 x16 per direction, nominal (no measured PCIe peak in MEASURED_PEAKS.json)
    line = {"metric": "KVFS host-tier offload / restore GB/s (PAPER.md P:233)", "value": nbytes / (off_ms / 1000) / 1e9,
            "unit": "GB/s", "n_gpus": 1, "steps": len(res["offload"]), "warmup": args.warmup, "higher_is_better": True,
            "dtype": "bf16", "data": "synthetic (seed 1006)",
            "config": {"workload": "32 files x 8192 tokens (8B attention shape, 32 MiB K+V each), kvfs_offload then "
                                   "kvfs_restore of every file", "bytes_each_way": nbytes},
            "roofline": {"bound": "pcie", "achieved": nbytes / (k_off / 1000) / 1e9, "peak": pcie, "unit": "GB/s",
                         "frac": nbytes / (k_off / 1000) / 1e9 / pcie, "kernel": "pack_kernel (K6) over mapped host memory",
                         "peak_source": "nominal PCIe Gen5 x16 per direction (no measured PCIe peak)",
                         "traffic": None, "kernel_ms": k_off},
            "clocks": sampler.summary(),
            "extra": {"offload_ms": off_ms, "offload_gbs": nbytes / (off_ms / 1000) / 1e9,
                      "restore_ms": res_ms, "restore_gbs": nbytes / (res_ms / 1000) / 1e9,
                      "offload_kernel_ms": k_off, "restore_kernel_ms": k_res,
                      "offload_kernel_gbs": nbytes / (k_off / 1000) / 1e9,
                      "restore_kernel_gbs": nbytes / (k_res / 1000) / 1e9,
                      "timing": "call time: CUDA events around the kvfs_offload / kvfs_restore calls (host work "
                                "included); kernel: events the library records around its K6 launches "
                                "(KVFS_OPT_TIMING, KVFS_CTR_COPY_DEVICE_NS)",
                      "cpu_baseline": "not meaningful (a host memcpy, not the method's arithmetic)",
                      "path": "page-pack kernel writing / reading pinned host memory through its mapped device address"}}
    print(json.dumps(line), flush=True)


def run_migrate(args):
    """SURVEY §8(e) migration data path on one GPU: kvfs_pack of 32 files x 32768 tokens (8B attention shape,
    128 MiB of K+V each, the cfg5 file size) into one contiguous device buffer (K6 gather), then kvfs_unpack
    into a second ctx (K6 scatter into R1 pages).  The NVLink send/recv between the two (NCCL over NVSwitch)
    needs two GPUs and is not measured here.  One JSON line: pack / unpack GB/s against the HBM peak."""
    import numpy as np
    import torch

    from paper_2510_25412_b200 import kvfs as K
    from synth.configs import Shape
    from synth.workloads import TAG_K, TAG_V, rows_torch

    torch.cuda.set_device(0)
    s, n_files, n, seed = Shape(32, 8, 128, 16), 32, 32768, 1007
    n_pages = n_files * (n // 16) + 64
    src = K.KVFS(1, s.Hq, s.Hkv, s.D, s.P, n_pages, device=0)
    dst = K.KVFS(1, s.Hq, s.Hkv, s.D, s.P, n_pages, device=0)
    dev = torch.device("cuda", 0)
    fds = []
    for f in range(n_files):
        fd = src.open(f"m{f}")
        k = rows_torch(seed, TAG_K, 0, f, 0, n, s.Hkv * s.D, device=dev).view(1, n, s.Hkv, s.D)
        v = rows_torch(seed, TAG_V, 0, f, 0, n, s.Hkv * s.D, device=dev).view(1, n, s.Hkv, s.D)
        src.append(fd, np.arange(n, dtype=np.int32), k, v)
        fds.append(fd)
        del k, v
    torch.cuda.synchronize()
    nbytes = n_files * n * s.Hkv * s.D * 2 * 2
    pk, up, kpk, kup = [], [], [], []
    src.set_option(K.OPT_TIMING, 1)
    dst.set_option(K.OPT_TIMING, 1)
    sampler = ClockSampler(0)
    sampler.start()
    for it in range(args.warmup + max(1, min(args.steps, 5))):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        src.counter(K.CTR_COPY_DEVICE_NS)
        dst.counter(K.CTR_COPY_DEVICE_NS)
        e[0].record()
        hdr, buf = src.pack(fds)
        e[1].record()
        new = dst.unpack(hdr, buf, [f"r{it}_{f}" for f in range(n_files)])
        e[2].record()
        torch.cuda.synchronize()
        if it >= args.warmup:
            kpk.append(src.counter(K.CTR_COPY_DEVICE_NS) / 1e6)
            kup.append(dst.counter(K.CTR_COPY_DEVICE_NS) / 1e6)
        for nm in [f"r{it}_{f}" for f in range(n_files)]:
            dst.unlink(nm)
        for fd in new:
            dst.close(fd)
        del buf
        if it >= args.warmup:
            pk.append(e[0].elapsed_time(e[1]))
            up.append(e[1].elapsed_time(e[2]))
    sampler.stop()
    peak, peak_src = peaks()
    pk_ms, up_ms = statistics.median(pk), statistics.median(up)
    kpk_ms, kup_ms = statistics.median(kpk), statistics.median(kup)
    gbs = lambda ms: 2 * nbytes / (ms / 1000) / 1e9  # read + write
    line = {"metric": "KV-file migration pack / unpack GB/s (SURVEY 8(e); one GPU, NVLink leg not measured)",
            "value": gbs(kpk_ms), "unit": "GB/s", "n_gpus": 1, "steps": len(pk), "warmup": args.warmup,
            "higher_is_better": True, "dtype": "bf16", "data": "synthetic (seed 1007)",
            "config": {"workload": "32 files x 32768 tokens (128 MiB K+V each, 4 GiB total): kvfs_pack into one "
                                   "device buffer, kvfs_unpack into a second ctx", "bytes_moved_each": nbytes},
            "roofline": {"bound": "hbm", "achieved": gbs(kpk_ms), "peak": peak, "unit": "GB/s",
                         "frac": gbs(kpk_ms) / peak, "kernel": "pack_kernel (K6), device time only",
                         "peak_source": peak_src, "algorithmic_bytes_per_launch": 2 * nbytes, "traffic": None,
                         "kernel_ms": kpk_ms},
            "clocks": sampler.summary(),
            "extra": {"pack_kernel_ms": kpk_ms, "unpack_kernel_ms": kup_ms, "pack_kernel_gbs": gbs(kpk_ms),
                      "unpack_kernel_gbs": gbs(kup_ms), "pack_call_ms": pk_ms, "unpack_call_ms": up_ms,
                      "pack_call_gbs": gbs(pk_ms), "unpack_call_gbs": gbs(up_ms),
                      "timing": "kernel: events the library records around its K6 launch (KVFS_OPT_TIMING, "
                                "KVFS_CTR_COPY_DEVICE_NS); call: events around kvfs_pack / kvfs_unpack, host side "
                                "(page lists, R1 allocation, header) included",
                      "cpu_baseline": "not meaningful (a memcpy, not the method's arithmetic)"}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args))
    if args.impl == "reference":
        run_reference(args)
    elif args.sched:
        run_sched(args)
    elif args.config == "cfg5hh":
        run_heavy_hitter(args)
    elif args.config == "offload":
        run_offload(args)
    elif args.config == "migrate" or (args.migrate and args.gpus == 1):
        run_migrate(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
