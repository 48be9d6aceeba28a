"""N > 1 path on CPU: two processes (gloo, world_size 2, 127.0.0.1) each own a host-only KVFS ctx with an
uneven LIP load; one rebalance round moves files by ascending fd from the heavier rank over
torch.distributed; the receiving ctx rebuilds the moved files' per-entry masks and positions exactly (pages
renumbered smallest-free), CoW sharing inside the moved set is preserved, and the sender unlinks its files
only after the receiver's ACK (a receiver without room keeps nothing and the sender keeps everything)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_25412_b200.parallel import choose_files, plan_rebalance


def test_plan_rebalance_deterministic():
    assert plan_rebalance([100, 10]) == [(0, 1, 45)]
    assert plan_rebalance([5, 50, 20, 30]) == [(1, 0, 22), (3, 2, 5)]
    assert plan_rebalance([7, 7]) == []
    files = [(3, "c", 10), (1, "a", 10), (2, "b", 30)]
    assert [f[1] for f in choose_files(files, 25)] == ["a"]
    assert [f[1] for f in choose_files(files, 45)] == ["a", "b"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, recv_pages=400):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_25412_b200 import kvfs as K
    from paper_2510_25412_b200.parallel import rebalance

    kv = K.KVFS(1, 8, 2, 64, 16, 400 if rank == 0 else recv_pages, device=-1)
    files = {}
    if rank == 0:  # heavy: 6 LIPs, two of them forks sharing a prefix
        base = kv.open("r0_base")
        kv.append(base, list(range(64)))
        files["r0_base"] = base
        for i in range(2):
            fd = kv.fork(base, f"r0_fork{i}")
            kv.append(fd, list(range(64, 64 + 10 * (i + 1))))
            files[f"r0_fork{i}"] = fd
        for i in range(3):
            fd = kv.open(f"r0_lip{i}")
            kv.append(fd, list(range(200 + 50 * i)))
            files[f"r0_lip{i}"] = fd
    else:
        fd = kv.open("r1_lip0")
        kv.append(fd, list(range(30)))
        files["r1_lip0"] = fd
    before = {n: (kv.table(fd), kv.positions(fd)) for n, fd in files.items()}
    stats = {}
    files = rebalance(kv, files, stats=stats)
    kv.audit()
    after = {n: (kv.table(fd), kv.positions(fd)) for n, fd in files.items()}
    q.put((rank, before, after, kv.refcounts(), stats))
    dist.destroy_process_group()


def _run(recv_pages):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, recv_pages)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, before, after, refc, stats = q.get(timeout=120)
        res[r] = (before, after, refc, stats)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_rebalance_refused_keeps_the_files():
    """the receiver cannot unpack (ENOSPC: 3 free pages) -> it ACKs the error, creates
    nothing, and the sender keeps every file (nothing is lost)."""
    res = _run(recv_pages=3)
    b0, a0, _, s0 = res[0]
    b1, a1, _, s1 = res[1]
    assert s0["role"] == "send" and s0["ack"] == -28 and not s0["moved"]
    assert s1["role"] == "recv" and s1["status"] == -28
    assert a0 == b0 and a1 == b1


def test_rebalance_two_ranks_gloo():
    res = _run(recv_pages=400)
    b0, a0, rc0, _ = res[0]
    b1, a1, rc1, _ = res[1]
    moved = sorted(set(b0) - set(a0))
    assert moved and set(moved) <= set(a1)  # what left rank 0 arrived at rank 1
    load0 = sum(len(p) for _, p in a0.values())
    load1 = sum(len(p) for _, p in a1.values())
    total = sum(len(p) for _, p in b0.values()) + sum(len(p) for _, p in b1.values())
    assert load0 + load1 == total and load0 >= load1
    for n in moved:  # positions and per-entry masks survive; pages are renumbered smallest-free
        assert a1[n][1] == b0[n][1]
        assert [m for _, m in a1[n][0]] == [m for _, m in b0[n][0]]
    # CoW sharing inside the moved set is preserved: shared prefix pages have refcount = sharers
    if "r0_base" in moved and "r0_fork0" in moved:
        shared = {p for p, _ in a1["r0_base"][0]} & {p for p, _ in a1["r0_fork0"][0]}
        assert shared and all(rc1[p] >= 2 for p in shared)
