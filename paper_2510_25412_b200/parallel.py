"""Multi-GPU plumbing: one process per GPU, each with its own KVFS ctx and its own LIPs.
The decode step runs no collective (the path partitions: a `pred` touches only its own file).
The only exchange is KV-file migration when the scheduler rebalances:

  1. all_gather of every rank's retained-token load (int64),
  2. a deterministic plan: ranks sorted by load (desc, rank asc); the i-th heaviest sends to the i-th
     lightest; the sender moves its files in ascending fd order while the move keeps it at or above the
     pair's mean (so the imbalance ends below one file),
  3. sender: kvfs_pack (K6 gather of the set's distinct pages, CoW sharing inside the set preserved) ->
     torch.distributed send of a size record, the header, the names and the page buffer (NCCL over
     NVLink for device buffers; with gloo, device tensors are staged through host memory),
  4. receiver: recv -> kvfs_unpack (smallest-free pages in packed order, K6 scatter) -> an ACK with
     kvfs_unpack's status back to the sender,
  5. sender: kvfs_unlink of the moved files ONLY if the ACK says the receiver created them (EEXIST /
     ENOSPC / EINVAL on the receiver: the files stay where they are, nothing is lost).
"""
from __future__ import annotations

import time
from typing import Dict, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from .kvfs import OK, KVFS, KvfsError


def plan_rebalance(loads: Sequence[int]) -> List[Tuple[int, int, int]]:
    """Pairs (src, dst, amount): heaviest with lightest; amount = half the pair's load difference."""
    order = sorted(range(len(loads)), key=lambda r: (-loads[r], r))
    plan = []
    for i in range(len(order) // 2):
        src, dst = order[i], order[len(order) - 1 - i]
        diff = loads[src] - loads[dst]
        if diff > 0:
            plan.append((src, dst, diff // 2))
    return plan


def choose_files(file_loads: Sequence[Tuple[int, str, int]], amount: int) -> List[Tuple[int, str, int]]:
    """Files (fd, name, load) in ascending fd order while the cumulative moved load stays <= amount."""
    out, moved = [], 0
    for fd, name, ld in sorted(file_loads):
        if moved + ld > amount:
            break
        out.append((fd, name, ld))
        moved += ld
    return out


def _gloo(group) -> bool:
    return dist.get_backend(group) == "gloo"


def _ctl_dev(kv: KVFS, group):
    """Device of the small control tensors: the ctx's GPU for NCCL, host memory for gloo."""
    if kv.device >= 0 and not _gloo(group):
        return kv.k_pool[0].device
    return torch.device("cpu")


def _send(t: torch.Tensor, dst: int, group) -> None:
    if t.is_cuda and _gloo(group):  # gloo moves host tensors: stage device buffers through host memory
        t = t.cpu()
    dist.send(t, dst, group=group)


def _recv(t: torch.Tensor, src: int, group) -> None:
    if t.is_cuda and _gloo(group):
        h = torch.empty(t.shape, dtype=t.dtype)
        dist.recv(h, src, group=group)
        t.copy_(h)
    else:
        dist.recv(t, src, group=group)


class _DevTimer:
    """Device time of work enqueued on the current stream, excluding the host time spent enqueueing it: the
    stream is first held busy by a spin kernel longer than that host time, so the start event fires only
    after the host has enqueued everything that follows (B200_PROFILING.md: CUDA events on the launching
    stream)."""

    def __init__(self, enabled: bool, hold_ms: float = 30.0):
        self.enabled = enabled
        self.hold_ms = hold_ms

    def __enter__(self):
        if self.enabled:
            torch.cuda._sleep(int(self.hold_ms * 2.0e6))  # ~hold_ms at <= 2 GHz
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e1 = torch.cuda.Event(enable_timing=True)
            self.e0.record()
            self.t0 = time.perf_counter()
        return self

    def __exit__(self, *exc):
        if self.enabled:
            self.host_ms = 1000 * (time.perf_counter() - self.t0)
            self.e1.record()
            self.e1.synchronize()
            self.ms = self.e0.elapsed_time(self.e1)
        return False


def send_files(kv: KVFS, files: Sequence[Tuple[int, str]], dst: int, group=None,
               stats: Optional[dict] = None) -> Tuple[bool, int]:
    """Pack and send (fd, name) files to rank dst; unlink them locally once the receiver ACKs that it
    created them.  Returns (moved, bytes sent).  `stats` (optional) receives device-timed pack / send
    times (ms) and the bytes."""
    dev = _ctl_dev(kv, group)
    timed = stats is not None and kv.device >= 0
    if not files:  # nothing fits the plan's amount: tell the receiver (it is waiting for a size record)
        _send(torch.zeros(3, dtype=torch.int64, device=dev), dst, group)
        ack = torch.zeros(1, dtype=torch.int64, device=dev)
        _recv(ack, dst, group)
        return False, 0
    with _DevTimer(timed) as tp:
        hdr, buf = kv.pack([fd for fd, _ in files])
    names = "\0".join(n for _, n in files).encode()
    nbuf = 0 if buf is None else buf.numel()
    if kv.device >= 0:
        torch.cuda.current_stream().synchronize()  # the K6 gather is done before the transfer starts
    _send(torch.tensor([len(hdr), len(names), nbuf], dtype=torch.int64, device=dev), dst, group)
    _send(torch.frombuffer(bytearray(hdr), dtype=torch.uint8).to(dev), dst, group)
    if names:
        _send(torch.frombuffer(bytearray(names), dtype=torch.uint8).to(dev), dst, group)
    t_send = None
    if nbuf:
        if timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        _send(buf, dst, group)
        if timed:
            e1.record()
            e1.synchronize()
            t_send = e0.elapsed_time(e1)
    ack = torch.zeros(1, dtype=torch.int64, device=dev)
    _recv(ack, dst, group)
    code = int(ack.item())
    if stats is not None:
        stats.update(pack_ms=getattr(tp, "ms", None), pack_host_ms=getattr(tp, "host_ms", None),
                     send_ms=t_send, buf_bytes=nbuf, hdr_bytes=len(hdr), files=len(files), ack=code)
    if code != OK:  # the receiver did not create the files: keep them here
        return False, len(hdr) + len(names) + nbuf
    for fd, name in files:
        kv.unlink(name)
        kv.close(fd)
    return True, len(hdr) + len(names) + nbuf


def recv_files(kv: KVFS, src: int, group=None, stats: Optional[dict] = None) -> List[Tuple[int, str]]:
    """Receive a packed file set from rank src, create its files (kvfs_unpack) and ACK the status.
    Returns [(fd, name)] (empty if kvfs_unpack refused the set)."""
    dev = _ctl_dev(kv, group)
    bdev = kv.k_pool[0].device if kv.device >= 0 else torch.device("cpu")
    timed = stats is not None and kv.device >= 0
    sizes = torch.empty(3, dtype=torch.int64, device=dev)
    _recv(sizes, src, group)
    nh, nn, nb = (int(x) for x in sizes.tolist())
    if nh == 0:  # empty set
        _send(torch.tensor([OK], dtype=torch.int64, device=dev), src, group)
        return []
    hdr = torch.empty(nh, dtype=torch.uint8, device=dev)
    _recv(hdr, src, group)
    names: List[str] = []
    if nn:
        nm = torch.empty(nn, dtype=torch.uint8, device=dev)
        _recv(nm, src, group)
        names = bytes(nm.cpu().numpy().tobytes()).decode().split("\0")
    buf = None
    t_recv = None
    if nb:
        buf = torch.empty(nb, dtype=torch.uint8, device=bdev)
        if timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        _recv(buf, src, group)
        if timed:
            e1.record()
            e1.synchronize()
            t_recv = e0.elapsed_time(e1)
    code, fds = OK, []
    try:
        with _DevTimer(timed) as tu:
            fds = kv.unpack(hdr.cpu().numpy().tobytes(), buf, names)
    except KvfsError as e:
        code = e.code
    if kv.device >= 0:
        torch.cuda.current_stream().synchronize()
    _send(torch.tensor([code], dtype=torch.int64, device=dev), src, group)
    if stats is not None:
        stats.update(recv_ms=t_recv, unpack_ms=getattr(tu, "ms", None), unpack_host_ms=getattr(tu, "host_ms", None),
                     buf_bytes=nb, files=len(names), status=code)
    return list(zip(fds, names)) if code == OK else []


def rebalance(kv: KVFS, files: Dict[str, int], group=None, stats: Optional[dict] = None) -> Dict[str, int]:
    """One rebalance round over the group. `files` maps this rank's LIP file names to fds; returns the
    updated map. Every rank must call it.  `stats` (optional) receives this rank's role, the loads and the
    device-timed pack / transfer / unpack of its transfer."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _ctl_dev(kv, group)
    mine = [(fd, name, kv.stat(fd)[0]) for name, fd in files.items()]
    load = torch.tensor([sum(x[2] for x in mine)], dtype=torch.int64, device=dev)
    loads = [torch.zeros_like(load) for _ in range(world)]
    dist.all_gather(loads, load, group=group)
    loads_i = [int(x.item()) for x in loads]
    files = dict(files)
    if stats is not None:
        stats.update(loads_before=loads_i, role="idle")
    for src, dst, amount in plan_rebalance(loads_i):
        if rank == src:
            moving = choose_files(mine, amount)
            ok, _ = send_files(kv, [(fd, name) for fd, name, _ in moving], dst, group, stats)
            if ok:
                for _, name, _ in moving:
                    files.pop(name)
            if stats is not None:
                stats.update(role="send", peer=dst, moved=ok, moved_files=[n for _, n, _ in moving],
                             moved_tokens=sum(x[2] for x in moving))
        elif rank == dst:
            got = recv_files(kv, src, group, stats)
            for fd, name in got:
                files[name] = fd
            if stats is not None:
                stats.update(role="recv", peer=src, moved_files=[n for _, n in got])
    return files
