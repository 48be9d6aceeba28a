"""Synthetic workloads of BASELINE.json's configs, built on the device through the public API.

Inputs follow DESIGN.md "Input recipe" (synth/, counter-based, bit-identical on host and device):
  * initial K/V of file f, token serial t:  rows(seed, TAG_K|TAG_V, layer, owner=f, serial=t)
  * the shared prefix (cfg3):              rows(seed, TAG_K|TAG_V, layer, owner=PREFIX_OWNER, serial=t)
  * new K/V of step s, row r:              rows(seed, TAG_K|TAG_V, layer, owner=STEP_OWNER+s, serial=r)
  * Q of step s, row r:                    rows(seed, TAG_Q, layer, owner=STEP_OWNER+s, serial=r)
so a test can regenerate any file's or step's inputs on the host for the oracle.
"""
from __future__ import annotations

import math
from typing import Tuple

import numpy as np
import torch

from synth.workloads import TAG_K, TAG_Q, TAG_V, rows_torch

from .kvfs import KVFS

from synth.configs import CONFIGS, PREFIX_OWNER, STEP_OWNER, Shape  # noqa: F401


class DecodeWorkload:
    """n_files LIPs, each owning one file; every step is one batched pred with n_q rows per LIP.

    Per-step LIP policies (host, through the C ABI): `rewind` truncates every file by r tokens before the
    step (autocompletion); `evict_sink` evicts logical [sink, sink+1) (attention sink + sliding
    window); `prefix_len` builds every file as a fork of one shared prefix."""

    @staticmethod
    def config_files(name: str) -> int:
        return CONFIGS[name]["n_files"]

    def __init__(self, name: str, steps_total: int, device: int = 0, n_files: int = None, owner_base: int = 0,
                 room_files: int = 0, step_owner_base: int = 0):
        """owner_base: the first file's generator owner id (and name "lip<owner>"), so the ranks of a multi-GPU
        run hold distinct LIPs; room_files: pool room for that many more files (migration targets);
        step_owner_base: offset of the per-step input owners (distinct inputs per rank)."""
        c = CONFIGS[name]
        self.name = name
        self.desc = c["workload"]
        self.shape: Shape = c["shape"]
        self.seed = c["seed"]
        self.n_files = n_files or c["n_files"]
        self.file_len = c["file_len"]
        self.n_q = c["n_q"]
        self.rewind = c.get("rewind", 0)
        self.prefix_len = c.get("prefix_len", 0)
        self.evict_sink = c.get("evict_sink", 0)
        self.steps_total = steps_total
        s = self.shape
        self.dev = torch.device("cuda", device)
        grow = steps_total * max(0, self.n_q - self.rewind)  # net growth per step (drafts: n_q - rewind)
        per_file = math.ceil((self.file_len + grow + s.P) / s.P) + 2
        self.n_pages = (self.n_files + room_files) * per_file + math.ceil(self.prefix_len / s.P) + 64
        self.step_owner_base = step_owner_base
        self.per_file_pages = per_file
        rows = (self.n_files + room_files) * self.n_q
        self.kv = KVFS(1, s.Hq, s.Hkv, s.D, s.P, self.n_pages, max_batch_rows=max(rows, 16),
                       max_batch_descs=max(self.n_files + room_files, 16), device=device)
        width = s.Hkv * s.D
        fds = []
        self.prefix_fd = None
        if self.prefix_len:
            self.prefix_fd = self.kv.open("prefix")
            k = rows_torch(self.seed, TAG_K, 0, PREFIX_OWNER, 0, self.prefix_len, width, device=self.dev)
            v = rows_torch(self.seed, TAG_V, 0, PREFIX_OWNER, 0, self.prefix_len, width, device=self.dev)
            self.kv.append(self.prefix_fd, list(range(self.prefix_len)), k.view(1, -1, s.Hkv, s.D),
                           v.view(1, -1, s.Hkv, s.D))
        self.names = []
        for f in range(owner_base, owner_base + self.n_files):
            fd = self.kv.fork(self.prefix_fd, f"lip{f}") if self.prefix_fd is not None else self.kv.open(f"lip{f}")
            self.names.append(f"lip{f}")
            k = rows_torch(self.seed, TAG_K, 0, f, 0, self.file_len, width, device=self.dev)
            v = rows_torch(self.seed, TAG_V, 0, f, 0, self.file_len, width, device=self.dev)
            p0 = self.prefix_len
            self.kv.append(fd, list(range(p0, p0 + self.file_len)), k.view(1, self.file_len, s.Hkv, s.D),
                           v.view(1, self.file_len, s.Hkv, s.D))
            fds.append(fd)
        torch.cuda.synchronize(self.dev)
        self.fds = fds
        self.descs = np.array([[fd, self.n_q] for fd in fds], dtype=np.int32)
        self.lens = np.full(self.n_files, self.prefix_len + self.file_len, dtype=np.int64)  # retained tokens
        self.next_pos = self.lens.copy()  # next absolute position of every LIP
        self._offs = np.arange(self.n_q, dtype=np.int64)
        self.step = 0

    # ------------------------------------------------------------------ migration (parallel.rebalance)
    def file_map(self):
        return dict(zip(self.names, self.fds))

    def set_files(self, files) -> None:
        """Adopt the file set after a rebalance ({name: fd}; moved-in files continue at their own last
        retained position; files are kept in name order so the batch is deterministic)."""
        items = sorted(files.items(), key=lambda x: (len(x[0]), x[0]))
        self.names = [n for n, _ in items]
        self.fds = [fd for _, fd in items]
        st = [self.kv.stat(fd) for fd in self.fds]
        self.n_files = len(self.fds)
        self.lens = np.array([x[0] for x in st], dtype=np.int64)
        self.next_pos = np.array([x[2] + 1 for x in st], dtype=np.int64)
        self.descs = np.array([[fd, self.n_q] for fd in self.fds], dtype=np.int32)

    # ------------------------------------------------------------------ per step
    def make_inputs(self, step: int) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
        """Device Q [T][Hq][D], K_new/V_new [T][Hkv][D] of step `step`."""
        s = self.shape
        T = self.n_files * self.n_q
        owner = STEP_OWNER + self.step_owner_base + step
        q = rows_torch(self.seed, TAG_Q, 0, owner, 0, T, s.Hq * s.D, device=self.dev).view(T, s.Hq, s.D)
        k = rows_torch(self.seed, TAG_K, 0, owner, 0, T, s.Hkv * s.D, device=self.dev).view(T, s.Hkv, s.D)
        v = rows_torch(self.seed, TAG_V, 0, owner, 0, T, s.Hkv * s.D, device=self.dev).view(T, s.Hkv, s.D)
        return q, k, v

    def pre_step(self) -> None:
        """Host-side LIP policy before a step (through the C ABI)."""
        if self.rewind:
            self.lens -= self.rewind
            self.next_pos -= self.rewind
            for fd, ln in zip(self.fds, self.lens.tolist()):
                self.kv.truncate(fd, ln)
        if self.evict_sink and self.step > 0:
            e = self.evict_sink
            for fd in self.fds:
                self.kv.evict(fd, [(e, e + 1)])
            self.lens -= 1

    def positions(self) -> np.ndarray:
        return (self.next_pos[:, None] + self._offs[None, :]).reshape(-1).astype(np.int32)

    def descs_and_pos(self):
        return [(int(a), int(b)) for a, b in self.descs], self.positions().tolist()

    def advance(self) -> None:
        self.lens += self.n_q
        self.next_pos += self.n_q
        self.step += 1

    # ------------------------------------------------------------------ accounting
    def logical_kv_bytes(self, lens=None) -> int:
        s = self.shape
        lens = self.lens if lens is None else lens
        return int(2 * lens.sum() * s.Hkv * s.D * 2)

    def unique_kv_bytes(self, lens=None) -> int:
        """K/V bytes of the distinct retained rows the batch reads (a CoW-shared prefix counted once)."""
        s = self.shape
        lens = self.lens if lens is None else lens
        row_kv = s.Hkv * s.D * 2
        if not self.prefix_len:
            return int(2 * lens.sum() * row_kv)
        return int(2 * (self.prefix_len + (lens - self.prefix_len).sum()) * row_kv)

    def algorithmic_bytes(self, lens=None) -> int:
        """Bytes one pred step must move: every unique retained K/V row read once (the old tokens; the new
        rows come from K_new), Q read, out + lse written, new K/V read once and written once."""
        s = self.shape
        row_kv = s.Hkv * s.D * 2
        T = self.n_files * self.n_q
        return (self.unique_kv_bytes(lens) + T * s.Hq * s.D * 2 + T * s.Hq * s.D * 2 + T * s.Hq * 4
                + 2 * 2 * T * row_kv)

    def flops(self, lens=None) -> int:
        s = self.shape
        n = self.n_q
        lens = self.lens if lens is None else lens
        return int(4 * s.Hq * s.D * (n * int(lens.sum()) + self.n_files * (n * (n + 1) // 2)))

    def dominant_kernel(self, cutover: int = 8) -> str:
        if cutover > 0 and self.n_q >= cutover:
            return "chunk_attn_tc_kernel (K2, tcgen05 QK^T / PV with TMEM accumulators)"
        if self.prefix_len:
            return ("chunk_attn_tc_kernel<G, prefix> (shared prefix once per batch, tcgen05) + decode_attn_kernel "
                    "(K1, private suffixes + log-sum-exp merge); time = both launches of the step")
        return "decode_attn_kernel (K1, fused append + split-KV attention)"
