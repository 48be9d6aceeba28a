"""Workload shapes of BASELINE.json's configs (sizes, seeds, per-step LIP policies).

Pure data: no method arithmetic.  Shared by the CUDA-path workloads (paper_2510_25412_b200/workloads.py)
and the oracle-side drivers (oracle/workload.py) so both build the same synthetic workloads.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict

STEP_OWNER = 1_000_000
PREFIX_OWNER = 999_999


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
                 shape=Shape(32, 8, 128, 16), n_files=256, file_len=2048, n_q=1, seed=1002),
    # PAPER.md §4.1 P:217 speculative drafts on the cfg2 shape: every step a LIP appends 4 draft tokens
    # (n_q = 4: 2 <= n_q < the chunk cut-over), the verifier keeps the first, the rest is truncated before
    # the next step (rewind 3): files grow by one token per step
    "cfg2d": dict(workload="cfg2d: speculative drafts on the cfg2 shape, 256 LIPs x 2048-token files (32q/8kv, hd128, "
                           "P=16), each step truncates the 3 rejected drafts of the previous step and appends 4 draft "
                           "tokens (n_q=4)",
                  shape=Shape(32, 8, 128, 16), n_files=256, file_len=2048, n_q=4, seed=1012, rewind=3),
    # BASELINE.json configs[2]: tree-of-thought fan-out, 64 forks of a 4096-token CoW prefix + 512-token branches
    "cfg3": dict(workload="cfg3: ToT fan-out, 64 LIPs forked from one 4096-token prefix file (CoW, 0 tail copies) "
                          "+ 512-token private branches, decode n_q=1 (32q/8kv, hd128, P=16)",
                 shape=Shape(32, 8, 128, 16), n_files=64, file_len=512, prefix_len=4096, n_q=1, seed=1003),
    # BASELINE.json configs[3]: live code autocompletion, truncate-to-cursor (r = 64) + 64-token re-append
    "cfg4": dict(workload="cfg4: autocompletion, 128 LIPs x 8192-token files (32q/8kv, hd128, P=16); each step "
                          "truncates every file to 8192-64 and re-appends 64 tokens (n_q=64, tcgen05 chunk kernel)",
                 shape=Shape(32, 8, 128, 16), n_files=128, file_len=8192, n_q=64, seed=1004, rewind=64),
    # BASELINE.json configs[4] (per GPU): long-context custom eviction, attention sink (4) + sliding window:
    # every step evicts logical [4, 5) and appends 1 token, files stay at 32768 tokens
    "cfg5": dict(workload="cfg5: long-context sink+window eviction, 128 LIPs/GPU x 32768-token files, each step "
                          "evicts logical [4,5) and appends 1 token (32q/8kv, hd128, P=16)",
                 shape=Shape(32, 8, 128, 16), n_files=128, file_len=32768, n_q=1, seed=1005, evict_sink=4),
}


