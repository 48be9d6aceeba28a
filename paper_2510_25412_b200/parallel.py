"""Multi-GPU plumbing: one process per GPU, each with its own KVFS ctx and its own LIPs.
The decode step runs no collective (the path partitions: a `pred` touches only its own file).
The only exchange is KV-file migration when the scheduler rebalances:

  1. all_gather of every rank's retained-token load (int64),
  2. a deterministic plan: ranks sorted by load (desc, rank asc); the i-th heaviest sends to the i-th
     lightest; the sender moves its files in ascending fd order while the move keeps it at or above the
     pair's mean (so the imbalance ends below one file),
  3. sender: kvfs_pack (K6 gather of the set's distinct pages, CoW sharing inside the set preserved) ->
     torch.distributed send of a size record, the header, the names and the page buffer (NCCL over
     NVLink for device buffers, gloo for host-only ctxs) -> kvfs_unlink of the moved files,
  4. receiver: recv -> kvfs_unpack (smallest-free pages in packed order, K6 scatter).
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import torch
import torch.distributed as dist

from .kvfs import KVFS


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


def _dev(kv: KVFS):
    return kv.k_pool[0].device if kv.device >= 0 else torch.device("cpu")


def send_files(kv: KVFS, files: Sequence[Tuple[int, str]], dst: int, group=None) -> int:
    """Pack and send (fd, name) files to rank dst; unlink them locally. Returns bytes sent."""
    dev = _dev(kv)
    hdr, buf = kv.pack([fd for fd, _ in files])
    names = "\0".join(n for _, n in files).encode()
    nbuf = 0 if buf is None else buf.numel()
    sizes = torch.tensor([len(hdr), len(names), nbuf], dtype=torch.int64, device=dev)
    dist.send(sizes, dst, group=group)
    dist.send(torch.frombuffer(bytearray(hdr), dtype=torch.uint8).to(dev), dst, group=group)
    if names:
        dist.send(torch.frombuffer(bytearray(names), dtype=torch.uint8).to(dev), dst, group=group)
    if nbuf:
        dist.send(buf, dst, group=group)
    if kv.device >= 0:
        torch.cuda.current_stream().synchronize()
    for fd, name in files:
        kv.unlink(name)
        kv.close(fd)
    return len(hdr) + len(names) + nbuf


def recv_files(kv: KVFS, src: int, group=None) -> List[Tuple[int, str]]:
    dev = _dev(kv)
    sizes = torch.empty(3, dtype=torch.int64, device=dev)
    dist.recv(sizes, src, group=group)
    nh, nn, nb = (int(x) for x in sizes.tolist())
    hdr = torch.empty(nh, dtype=torch.uint8, device=dev)
    dist.recv(hdr, src, group=group)
    names: List[str] = []
    if nn:
        nm = torch.empty(nn, dtype=torch.uint8, device=dev)
        dist.recv(nm, src, group=group)
        names = bytes(nm.cpu().tolist()).decode().split("\0")
    buf = None
    if nb:
        buf = torch.empty(nb, dtype=torch.uint8, device=dev)
        dist.recv(buf, src, group=group)
    fds = kv.unpack(bytes(hdr.cpu().tolist()), buf, names)
    return list(zip(fds, names))


def rebalance(kv: KVFS, files: Dict[str, int], group=None) -> Dict[str, int]:
    """One rebalance round over the group. `files` maps this rank's LIP file names to fds; returns the
    updated map. Every rank must call it."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _dev(kv)
    mine = [(fd, name, kv.stat(fd)[0]) for name, fd in files.items()]
    load = torch.tensor([sum(x[2] for x in mine)], dtype=torch.int64, device=dev)
    loads = [torch.zeros_like(load) for _ in range(world)]
    dist.all_gather(loads, load, group=group)
    loads_i = [int(x.item()) for x in loads]
    files = dict(files)
    for src, dst, amount in plan_rebalance(loads_i):
        if rank == src:
            moving = choose_files(mine, amount)
            send_files(kv, [(fd, name) for fd, name, _ in moving], dst, group)
            for _, name, _ in moving:
                files.pop(name)
        elif rank == dst:
            for fd, name in recv_files(kv, src, group):
                files[name] = fd
    return files
