"""Synthetic workloads of BASELINE.json's configs, built on the device through the public API.

Inputs follow DESIGN.md "Input recipe" (synth/, counter-based, bit-identical on host and device):
  * initial K/V of file f, token serial t:  rows(seed, TAG_K|TAG_V, layer, owner=f, serial=t)
  * new K/V of decode step s, row r:       rows(seed, TAG_K|TAG_V, layer, owner=STEP_OWNER+s, serial=r)
  * Q of decode step s, row r:             rows(seed, TAG_Q, layer, owner=STEP_OWNER+s, serial=r)
so a test can regenerate any file's or step's inputs on the host for the oracle.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Tuple

import torch

from synth.workloads import TAG_K, TAG_Q, TAG_V, rows_torch

from .kvfs import KVFS

STEP_OWNER = 1_000_000


@dataclass
class Shape:
    Hq: int = 32
    Hkv: int = 8
    D: int = 128
    P: int = 16


CONFIGS: Dict[str, dict] = {
    # BASELINE.json configs[1]: Llama-3-8B attention shape, 256 LIPs decoding from 2k-token files
    "cfg2": dict(workload="cfg2: Llama-3-8B attn (32q/8kv, hd128, bf16, P=16), 256 LIPs decode (n_q=1) "
                          "from 2048-token KVFS files, 1 layer per step",
                 shape=Shape(32, 8, 128, 16), n_files=256, file_len=2048, n_q=1, seed=1002, rewind=0),
    # BASELINE.json configs[3]: live code autocompletion, truncate-to-cursor (r = 64) + 64-token re-append
    "cfg4": dict(workload="cfg4: autocompletion, 128 LIPs x 8192-token files (32q/8kv, hd128, P=16); each step "
                          "truncates every file to 8192-64 and re-appends 64 tokens (n_q=64, tcgen05 chunk kernel)",
                 shape=Shape(32, 8, 128, 16), n_files=128, file_len=8192, n_q=64, seed=1004, rewind=64),
}


class DecodeWorkload:
    """n_files LIPs, each owning one file of file_len tokens; every step is one batched pred with n_q rows
    per LIP (positions continue the file)."""

    def __init__(self, name: str, steps_total: int, device: int = 0, n_files: int = None):
        c = CONFIGS[name]
        self.name = name
        self.desc = c["workload"]
        self.shape: Shape = c["shape"]
        self.seed = c["seed"]
        self.n_files = n_files or c["n_files"]
        self.file_len = c["file_len"]
        self.n_q = c["n_q"]
        self.rewind = c.get("rewind", 0)  # truncate-to-cursor before every step (autocompletion)
        self.steps_total = steps_total
        s = self.shape
        self.dev = torch.device("cuda", device)
        grow = 0 if self.rewind else steps_total * self.n_q
        per_file = math.ceil((self.file_len + grow + s.P) / s.P) + 1
        self.n_pages = self.n_files * per_file + 64
        rows = self.n_files * self.n_q
        self.kv = KVFS(1, s.Hq, s.Hkv, s.D, s.P, self.n_pages, max_batch_rows=max(rows, 16),
                       max_batch_descs=max(self.n_files, 16), device=device)
        self.fds: List[int] = []
        self.lens: List[int] = []
        width = s.Hkv * s.D
        for f in range(self.n_files):
            fd = self.kv.open(f"lip{f}")
            k = rows_torch(self.seed, TAG_K, 0, f, 0, self.file_len, width, device=self.dev)
            v = rows_torch(self.seed, TAG_V, 0, f, 0, self.file_len, width, device=self.dev)
            self.kv.append(fd, list(range(self.file_len)), k.view(1, self.file_len, s.Hkv, s.D),
                           v.view(1, self.file_len, s.Hkv, s.D))
            self.fds.append(fd)
            self.lens.append(self.file_len)
        torch.cuda.synchronize(self.dev)
        self.step = 0

    def make_inputs(self, step: int) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
        """Device Q [T][Hq][D], K_new/V_new [T][Hkv][D] of decode step `step`."""
        s = self.shape
        T = self.n_files * self.n_q
        owner = STEP_OWNER + step
        q = rows_torch(self.seed, TAG_Q, 0, owner, 0, T, s.Hq * s.D, device=self.dev).view(T, s.Hq, s.D)
        k = rows_torch(self.seed, TAG_K, 0, owner, 0, T, s.Hkv * s.D, device=self.dev).view(T, s.Hkv, s.D)
        v = rows_torch(self.seed, TAG_V, 0, owner, 0, T, s.Hkv * s.D, device=self.dev).view(T, s.Hkv, s.D)
        return q, k, v

    def pre_step(self) -> None:
        """Host-side LIP policy before a step: truncate-to-cursor for the autocompletion workload."""
        if self.rewind:
            for i, fd in enumerate(self.fds):
                self.lens[i] -= self.rewind
                self.kv.truncate(fd, self.lens[i])

    def descs_and_pos(self) -> Tuple[List[Tuple[int, int]], List[int]]:
        descs, pos = [], []
        for fd, ln in zip(self.fds, self.lens):
            descs.append((fd, self.n_q))
            pos.extend(range(ln, ln + self.n_q))
        return descs, pos

    def advance(self) -> None:
        self.lens = [ln + self.n_q for ln in self.lens]
        self.step += 1

    def algorithmic_bytes(self) -> int:
        """Bytes one pred step must move: every retained K/V row read once (the old tokens;
        the new rows are read from K_new), Q read, out + lse written, new K/V read once and written once."""
        s = self.shape
        row_kv = s.Hkv * s.D * 2  # one token's K (or V) bytes
        T = self.n_files * self.n_q
        old = sum(self.lens)  # retained tokens before this step's append
        return (2 * old * row_kv            # K and V of the retained tokens
                + T * s.Hq * s.D * 2        # Q
                + T * s.Hq * s.D * 2        # out
                + T * s.Hq * 4              # lse
                + 2 * 2 * T * row_kv)       # K_new, V_new: read + written into the pool

    def flops(self) -> int:
        s = self.shape
        n = self.n_q
        return sum(4 * s.Hq * s.D * (n * ln + n * (n + 1) // 2) for ln in self.lens)

    def dominant_kernel(self) -> str:
        return ("chunk_attn_tc_kernel (K2, tcgen05 QK^T / PV with TMEM accumulators)" if self.n_q >= 8
                else "decode_attn_kernel (K1, fused append + split-KV attention)")
