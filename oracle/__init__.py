"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously correct CPU model of what the batched `pred` path computes (§4.1
P:210-217, §4.2) under the readings fixed in SURVEY.md §8(c) / DESIGN.md "Readings":
  * oracle.kvfs      — KVFS page pool, refcounts, files, open/fork/truncate/evict/compact/append and the
                       batched pred reserve (rules R1-R9, R11), pure Python, with an optional physical
                       bf16 page store;
  * oracle.attention — attention of a pred over a file = dense softmax attention over the file's
                       retained-token list (rule R10), NumPy fp64;
  * oracle.bf16      — bf16 <-> float conversions and round-to-nearest-even (rule R12);
  * oracle.sched     — the inference scheduler's Poisson-sized batch formation (§4.4).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this package. It imports nothing from the CUDA path (paper_2510_25412_b200) and the CUDA path never
imports it. Parity status of each function is stated in its docstring ("pinned by: ..."); see also
DESIGN.md "Oracle pins". Nothing here is parity-unpinned.
"""
from .kvfs import (  # noqa: F401
    Oracle,
    KvfsError,
    OK, ENOENT, EBADF, EBUSY, EEXIST, EINVAL, ENOSPC, ERANGE, EPOS, EPARTIAL, EIO, EOFFLOAD, HOST,
    O_CREAT, O_EXCL, EVICT_COMPACT,
)
from .attention import gqa_attention, attention_over_file  # noqa: F401
from .bf16 import bf16_to_f64, f64_to_bf16_rne  # noqa: F401
from .sched import Dispatcher  # noqa: F401
