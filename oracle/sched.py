"""Inference-scheduler batch formation oracle (§4.4). TEST INFRASTRUCTURE ONLY.

P:242: "Executing the batch prematurely can result in underutilized GPU resources ... whereas delaying it
excessively can increase wait times"; Symphony "dynamically adjusts batch size according to the
average frequency of system calls, leveraging models like Poisson process."  The paper gives no formula;
the reading (reading S1) is:

  enqueue(now)   lam <- 1 / dt_default on the first enqueue, else lam <- (1 - alpha) lam + alpha / dt with
                 dt = max(now - t_prev, eps), eps = 1e-9 (Poisson rate estimate by an EWMA of 1/dt)
  form(now)      B* = clamp(round(lam * W_max), 1, B_max) (expected arrivals within W_max); dispatch when
                 the pool holds >= B* requests or the oldest has waited >= W_max; the batch is the pool's
                 requests in FIFO enqueue order (P:241 aggregation), at most B_max, skipping a
                 request whose file is already in the batch (it stays queued, in order: one pred per file per
                 batch, rule R11 EBUSY)
round() is round-half-to-even (Python's round, C's nearbyint in the default rounding mode).
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

EPS = 1e-9


class Dispatcher:
    def __init__(self, w_max: float = 0.010, b_max: int = 64, alpha: float = 0.2, dt_default: float = 0.1):
        self.w_max, self.b_max, self.alpha, self.dt_default = w_max, b_max, alpha, dt_default
        self.lam: Optional[float] = None
        self.t_prev: Optional[float] = None
        self.pool: List[Tuple[int, List[int], float]] = []  # (fd, positions, enqueue time), FIFO

    def enqueue(self, fd: int, pos: Sequence[int], now: float) -> None:
        if self.lam is None:
            self.lam = 1.0 / self.dt_default
        else:
            dt = max(now - self.t_prev, EPS)
            self.lam = (1.0 - self.alpha) * self.lam + self.alpha / dt
        self.t_prev = now
        self.pool.append((fd, list(pos), now))

    def target(self) -> int:
        lam = self.lam if self.lam is not None else 1.0 / self.dt_default
        return max(1, min(self.b_max, round(lam * self.w_max)))

    def form(self, now: float):
        """None if the batch is not due yet, else (descs [(fd, n_q)], positions) in FIFO order."""
        if not self.pool:
            return None
        if len(self.pool) < self.target() and now - self.pool[0][2] < self.w_max:
            return None
        taken, rest, seen = [], [], set()
        for req in self.pool:
            if len(taken) < self.b_max and req[0] not in seen:
                taken.append(req)
                seen.add(req[0])
            else:
                rest.append(req)
        self.pool = rest
        return [(fd, len(p)) for fd, p, _ in taken], [x for _, p, _ in taken for x in p]
