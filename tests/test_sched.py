"""Inference-scheduler batch formation (§4.4; reading S1 in DESIGN.md).

Oracle pins: the SPEC worked examples (EWMA fixed point, initialisation, the eps floor, B* = 32 at 3200/s
and 10 ms, saturation at B_max, the deadline path) and FIFO / one-pred-per-file order; then the native
kvfs_sched_* (C ABI) equals the oracle decision for decision on random arrival traces.  CPU only."""
import math
import random

import pytest

from oracle.sched import EPS, Dispatcher
from paper_2510_25412_b200 import kvfs as K


def test_s385_ewma_fixed_point_10_per_s():
    d = Dispatcher(alpha=0.2, dt_default=1.0)
    for i in range(200):
        d.enqueue(i, [0], 0.1 * i)
    assert abs(d.lam - 10.0) < 1e-9  # fixed point of lam = (1-a) lam + a / 0.1


def test_s386_first_enqueue_initialises_and_s387_eps_floor():
    d = Dispatcher(alpha=0.5, dt_default=0.25)
    d.enqueue(0, [0], 5.0)
    assert d.lam == 4.0  # 1 / dt_default
    d.enqueue(1, [0], 5.0)  # identical virtual time: dt floored at eps
    assert d.lam == 0.5 * 4.0 + 0.5 / EPS


def test_s393_b_star_32_at_3200_per_s():
    d = Dispatcher(w_max=0.010, b_max=64, alpha=1.0, dt_default=1 / 3200)
    d.enqueue(0, [0], 0.0)
    assert d.target() == 32
    for i in range(1, 31):
        d.enqueue(i, [0], i / 3200)
    assert d.form(30 / 3200) is None  # 31 waiting < 32 and the oldest waited < 10 ms
    d.enqueue(31, [0], 31 / 3200)
    descs, pos = d.form(31 / 3200)
    assert [fd for fd, _ in descs] == list(range(32)) and not d.pool


def test_s391_saturation_64_of_64():
    d = Dispatcher(w_max=0.010, b_max=64, alpha=1.0, dt_default=1e-6)
    for i in range(70):
        d.enqueue(i, [i, i + 1], 0.0)
    assert d.target() == 64
    descs, pos = d.form(0.0)
    assert len(descs) == 64 and pos[:4] == [0, 1, 1, 2] and len(d.pool) == 6


def test_s392_deadline_path_single_request():
    d = Dispatcher(w_max=0.010, b_max=64, alpha=0.2, dt_default=10.0)  # lam = 0.1/s -> B* = 1
    d2 = Dispatcher(w_max=0.010, b_max=64, alpha=1.0, dt_default=1e-4)  # lam = 1e4/s -> B* = 64
    d.enqueue(3, [7], 1.0)
    assert d.form(1.0) is not None  # B* = 1: due at once
    d2.enqueue(3, [7], 1.0)
    assert d2.form(1.005) is None
    assert d2.form(1.010) == ([(3, 1)], [7])  # oldest waited W_max


def test_fifo_and_one_pred_per_file():
    d = Dispatcher(w_max=0.001, b_max=8, alpha=1.0, dt_default=1.0)
    for fd in [5, 6, 5, 7, 6, 8]:
        d.enqueue(fd, [fd], 0.0)
    descs, pos = d.form(1.0)
    assert descs == [(5, 1), (6, 1), (7, 1), (8, 1)] and pos == [5, 6, 7, 8]
    assert [r[0] for r in d.pool] == [5, 6]  # repeats stay queued, in order
    assert d.form(1.0)[0] == [(5, 1), (6, 1)]


@pytest.mark.parametrize("seed", range(20))
def test_native_scheduler_matches_oracle(seed):
    rnd = random.Random(seed)
    cfg = dict(w_max=rnd.choice([0.002, 0.01, 0.05]), b_max=rnd.choice([1, 4, 16, 64]),
               alpha=rnd.choice([0.1, 0.2, 1.0]), dt_default=rnd.choice([0.001, 0.1]))
    o = Dispatcher(**cfg)
    c = K.Scheduler(**cfg)
    t = 0.0
    for step in range(400):
        if rnd.random() < 0.6:
            t += rnd.expovariate(rnd.choice([50.0, 500.0, 5000.0])) if rnd.random() > 0.05 else 0.0
            fd = rnd.randint(0, 30)
            pos = list(range(rnd.randint(0, 1000), rnd.randint(0, 1000) + rnd.randint(1, 3)))
            o.enqueue(fd, pos, t)
            c.enqueue(fd, pos, t)
        else:
            t += rnd.random() * 0.004
            assert c.form(t) == o.form(t)
        lam, tgt, n = c.state()
        assert math.isclose(lam, o.lam if o.lam is not None else 1 / cfg["dt_default"], rel_tol=1e-12)
        assert tgt == o.target() and n == len(o.pool)
