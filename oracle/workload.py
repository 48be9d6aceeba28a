"""The BASELINE.json workloads driven through the oracle for a sample of LIPs (TEST INFRASTRUCTURE ONLY:
used by tests/ for full-size sampled parity and by bench.py's cpu_baseline / --impl reference legs).

Builds, for the sampled LIPs only, exactly the files the CUDA-path workloads build (same synth/ recipe,
synth/configs.py shapes, same per-step LIP policies), so the oracle's outputs for those LIPs are the
expected values of the batched CUDA run."""
from __future__ import annotations

import math
from typing import List, Sequence

import numpy as np

from synth.configs import CONFIGS, PREFIX_OWNER, STEP_OWNER
from synth.workloads import TAG_K, TAG_Q, TAG_V, rows_np

from .kvfs import Oracle


class OracleWorkload:
    def __init__(self, name: str, lips: Sequence[int], max_steps: int = 64):
        c = CONFIGS[name]
        self.c = c
        self.s = c["shape"]
        self.lips = list(lips)
        self.n_q = c["n_q"]
        s = self.s
        prefix = c.get("prefix_len", 0)
        grow = max_steps * max(0, self.n_q - c.get("rewind", 0))
        per_file = math.ceil((c["file_len"] + grow + s.P) / s.P) + 2
        self.o = Oracle(len(self.lips) * per_file + math.ceil(prefix / s.P) + 8, s.P, 1, s.Hkv, s.D)
        w = s.Hkv * s.D
        pfd = None
        if prefix:
            pfd = self.o.open("prefix")
            self.o.append(pfd, list(range(prefix)),
                          rows_np(c["seed"], TAG_K, 0, PREFIX_OWNER, 0, prefix, w).reshape(1, prefix, s.Hkv, s.D),
                          rows_np(c["seed"], TAG_V, 0, PREFIX_OWNER, 0, prefix, w).reshape(1, prefix, s.Hkv, s.D))
        self.fds: List[int] = []
        L = c["file_len"]
        for f in self.lips:
            fd = self.o.fork(pfd, f"lip{f}") if pfd is not None else self.o.open(f"lip{f}")
            self.o.append(fd, list(range(prefix, prefix + L)),
                          rows_np(c["seed"], TAG_K, 0, f, 0, L, w).reshape(1, L, s.Hkv, s.D),
                          rows_np(c["seed"], TAG_V, 0, f, 0, L, w).reshape(1, L, s.Hkv, s.D))
            self.fds.append(fd)
        self.next_pos = [prefix + L] * len(self.lips)
        self.step = 0

    def run_step(self):
        """One step for the sampled LIPs: the LIP policy, then one oracle pred (rows of LIP f of the batched
        CUDA run = rows f*n_q .. f*n_q + n_q - 1 of step `step`). Returns (status, out [n][n_q][Hq][D], lse)."""
        c, s, n = self.c, self.s, self.n_q
        if c.get("rewind"):
            r = c["rewind"]
            self.next_pos = [p - r for p in self.next_pos]
            for fd in self.fds:
                self.o.truncate(fd, self.o.stat(fd)[0] - r)
        if c.get("evict_sink") and self.step > 0:
            e = c["evict_sink"]
            for fd in self.fds:
                self.o.evict(fd, [(e, e + 1)])
        own = STEP_OWNER + self.step
        qs, ks, vs, pos = [], [], [], []
        for f, p0 in zip(self.lips, self.next_pos):
            qs.append(rows_np(c["seed"], TAG_Q, 0, own, f * n, f * n + n, s.Hq * s.D).reshape(n, s.Hq, s.D))
            ks.append(rows_np(c["seed"], TAG_K, 0, own, f * n, f * n + n, s.Hkv * s.D).reshape(n, s.Hkv, s.D))
            vs.append(rows_np(c["seed"], TAG_V, 0, own, f * n, f * n + n, s.Hkv * s.D).reshape(n, s.Hkv, s.D))
            pos.extend(range(p0, p0 + n))
        q = np.concatenate(qs)[None]
        k = np.concatenate(ks)[None]
        v = np.concatenate(vs)[None]
        st, out, lse = self.o.pred_batch([(fd, n) for fd in self.fds], pos, q, k, v, s.D ** -0.5)
        self.next_pos = [p + n for p in self.next_pos]
        self.step += 1
        return st, out[0].reshape(len(self.lips), n, s.Hq, s.D), lse[0].reshape(len(self.lips), n, s.Hq)
