"""B200-native KVFS + batched `pred` attention (arXiv 2510.25412, Symphony): the C-ABI library
libkvfs.so (csrc/) and its thin ctypes binding (kvfs.py)."""
from .kvfs import KVFS, KvfsError, lib  # noqa: F401
