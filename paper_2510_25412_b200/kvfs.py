"""Thin ctypes binding of include/kvfs.h (argument marshalling only: every step of the path runs in
libkvfs.so).  PyTorch provides the device memory (pools, workspace, Q/K/V/out) and streams.

The CUDA extension is mandatory for every data operation: if libkvfs.so is missing this module raises
at load time; there is no fallback of any kind.  A host-only ctx (device=-1) exists to test the C++
control plane on a machine without a GPU; its data calls fail with KVFS_ENOSYS.
"""
from __future__ import annotations

import ctypes
import os
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# KVFS_LIB_PATH: an alternative in-tree build (tuning experiments); the default is the product library
LIB_PATH = os.environ.get("KVFS_LIB_PATH") or os.path.join(_HERE, "libkvfs.so")

OK, ENOENT, EIO, EBADF, ENOMEM, EBUSY, EEXIST, EINVAL, ENOSPC, ERANGE, ENOSYS = \
    0, -2, -5, -9, -12, -16, -17, -22, -28, -34, -38
EPOS, EPARTIAL, EOFFLOAD = -1001, -1002, -1003
HOST_PAGE = 0x80000000
O_CREAT, O_EXCL = 1, 2
EVICT_COMPACT = 1
OPT_DECODE_CTAS, OPT_CHUNK_CUTOVER, OPT_DETERMINISTIC, OPT_CASCADE_MIN_ENTRIES, OPT_PREFIX_SPLITS = 1, 2, 3, 4, 5
OPT_FAULT_INJECT, OPT_TIMING, OPT_DECODE_CHUNKS, OPT_HOLES_GATHER, OPT_PREFIX_PAIRED = 6, 7, 8, 9, 10
CTR_KERNEL_LAUNCHES, CTR_H2D_BYTES, CTR_PAGE_COPIES, CTR_LAST_DECODE_CTAS, CTR_LAST_CHUNK_UNITS = 1, 2, 3, 4, 5
CTR_LAST_PREFIX_UNITS, CTR_LAST_PREFIX_GROUPS, CTR_HOST_PAGES, CTR_COMPACT_DEVICE_NS = 6, 7, 8, 9
CTR_LAYER_DEVICE_NS, CTR_LAYER_TIMED = 10, 11
CTR_HOST_RESERVE_NS, CTR_HOST_SPLIT_NS, CTR_HOST_UPLOAD_NS, CTR_HOST_LAUNCH_NS = 12, 13, 14, 15
CTR_COPY_DEVICE_NS, CTR_LAST_FUSED_SCORES = 16, 17

# every symbol include/kvfs.h declares (tests check the library exports all of them)
EXPORTS = [
    "kvfs_workspace_bytes", "kvfs_init", "kvfs_destroy", "kvfs_strerror", "kvfs_open", "kvfs_close",
    "kvfs_unlink", "kvfs_fork", "kvfs_truncate", "kvfs_evict", "kvfs_compact", "kvfs_compact_files",
    "kvfs_append",
    "pred_attn_batch", "pred_attn_batch_host", "pred_host_fence", "pred_step_begin", "pred_attn_layer", "pred_step_end", "kvfs_stat",
    "kvfs_get_table", "kvfs_get_positions", "kvfs_get_refcounts", "kvfs_free_pages", "kvfs_read",
    "kvfs_audit", "kvfs_set_option", "kvfs_get_counter", "kvfs_pack", "kvfs_unpack", "kvfs_extract",
    "kvfs_merge", "kvfs_sched_create", "kvfs_sched_destroy", "kvfs_sched_enqueue", "kvfs_sched_state",
    "kvfs_sched_form", "pred_attn_scores", "kvfs_offload", "kvfs_restore", "kvfs_set_logits_buffer",
]


class SchedConfig(ctypes.Structure):
    _fields_ = [("w_max", ctypes.c_double), ("b_max", ctypes.c_int), ("alpha", ctypes.c_double),
                ("dt_default", ctypes.c_double)]


class KvfsConfig(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int), ("n_layers", ctypes.c_int), ("n_q_heads", ctypes.c_int),
        ("n_kv_heads", ctypes.c_int), ("head_dim", ctypes.c_int), ("page_size", ctypes.c_int),
        ("n_pages", ctypes.c_int64), ("k_pool", ctypes.POINTER(ctypes.c_void_p)),
        ("v_pool", ctypes.POINTER(ctypes.c_void_p)), ("max_batch_rows", ctypes.c_int32),
        ("max_batch_descs", ctypes.c_int32), ("table_capacity", ctypes.c_int64),
        ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
    ]


class PredDesc(ctypes.Structure):
    _fields_ = [("fd", ctypes.c_int32), ("n_q", ctypes.c_int32)]


class KvfsStat(ctypes.Structure):
    _fields_ = [("len", ctypes.c_int64), ("n_entries", ctypes.c_int64), ("last_pos", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


_lib = None


def lib():
    """Load libkvfs.so (built by paper_2510_25412_b200.build / __graft_entry__.build()). Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2510_25412_b200.build` "
                               "(there is no fallback implementation)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, cint = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int
        P = ctypes.POINTER
        sigs = {
            "kvfs_workspace_bytes": (ctypes.c_size_t, [P(KvfsConfig)]),
            "kvfs_init": (cint, [P(KvfsConfig), P(vp)]),
            "kvfs_destroy": (cint, [vp]),
            "kvfs_strerror": (ctypes.c_char_p, [cint]),
            "kvfs_open": (cint, [vp, ctypes.c_char_p, cint, P(cint)]),
            "kvfs_close": (cint, [vp, cint]),
            "kvfs_unlink": (cint, [vp, ctypes.c_char_p]),
            "kvfs_fork": (cint, [vp, cint, ctypes.c_char_p, P(cint), vp]),
            "kvfs_truncate": (cint, [vp, cint, i64]),
            "kvfs_evict": (cint, [vp, cint, P(i64), cint, cint, vp]),
            "kvfs_compact": (cint, [vp, cint, vp]),
            "kvfs_compact_files": (cint, [vp, P(cint), cint, P(cint), vp]),
            "kvfs_extract": (cint, [vp, cint, P(ctypes.c_int64), i64, ctypes.c_char_p, P(cint), vp]),
            "kvfs_merge": (cint, [vp, P(cint), cint, ctypes.c_char_p, P(cint), vp]),
            "kvfs_sched_create": (cint, [P(SchedConfig), P(vp)]),
            "pred_attn_scores": (cint, [vp, vp, cint, vp, vp, ctypes.c_float, vp, P(i64), vp]),
            "kvfs_offload": (cint, [vp, cint, P(i64), vp]),
            "kvfs_restore": (cint, [vp, cint, P(i64), vp]),
            "kvfs_sched_destroy": (cint, [vp]),
            "kvfs_sched_enqueue": (cint, [vp, cint, cint, P(i32), ctypes.c_double]),
            "kvfs_sched_state": (cint, [vp, P(ctypes.c_double), P(cint), P(cint)]),
            "kvfs_sched_form": (cint, [vp, ctypes.c_double, vp, cint, P(i32), i64, P(cint), P(i64)]),
            "kvfs_append": (cint, [vp, cint, i64, P(i32), vp, vp, vp]),
            # the per-step calls take plain addresses (ints) for every array: no ctypes pointer objects
            "pred_attn_batch": (cint, [vp, vp, cint, vp, vp, vp, vp, vp, vp, ctypes.c_float, vp, vp]),
            "pred_attn_batch_host": (cint, [vp, vp, cint, vp, vp, vp, vp, vp, vp, ctypes.c_float, vp, vp]),
            "pred_host_fence": (cint, [vp, vp]),
            "pred_step_begin": (cint, [vp, vp, cint, vp, vp, P(vp), vp]),
            "pred_attn_layer": (cint, [vp, vp, cint, vp, vp, vp, vp, vp, ctypes.c_float, vp]),
            "pred_step_end": (cint, [vp, vp]),
            "kvfs_set_logits_buffer": (cint, [vp, vp, ctypes.c_size_t]),
            "kvfs_stat": (cint, [vp, cint, P(KvfsStat)]),
            "kvfs_get_table": (cint, [vp, cint, P(ctypes.c_uint32), P(ctypes.c_uint64), i64, P(i64)]),
            "kvfs_get_positions": (cint, [vp, cint, P(i32), i64, P(i64)]),
            "kvfs_get_refcounts": (cint, [vp, P(ctypes.c_uint32), i64]),
            "kvfs_free_pages": (cint, [vp, P(i64)]),
            "kvfs_read": (cint, [vp, cint, cint, i64, i64, vp, vp, vp]),
            "kvfs_audit": (cint, [vp]),
            "kvfs_set_option": (cint, [vp, cint, i64]),
            "kvfs_get_counter": (cint, [vp, cint, P(i64)]),
            "kvfs_pack": (cint, [vp, P(cint), cint, vp, ctypes.c_size_t, P(ctypes.c_size_t), vp, ctypes.c_size_t,
                                 P(ctypes.c_size_t), vp]),
            "kvfs_unpack": (cint, [vp, vp, ctypes.c_size_t, vp, ctypes.c_size_t, P(ctypes.c_char_p), P(cint), vp]),
        }
        for name, (res, args) in sigs.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def strerror(code: int) -> str:
    return lib().kvfs_strerror(code).decode()


class KvfsError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        super().__init__(f"{what}: {strerror(code)} ({code})")
        self.code = code


def _check(rc: int, what: str) -> int:
    if rc != OK:
        raise KvfsError(rc, what)
    return rc


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _stream(stream, device: int = -1):
    if stream is None:
        import torch
        if device >= 0:  # the raw handle of the device's current stream, without a Stream object
            return torch._C._cuda_getCurrentRawStream(device)
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _dptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _daddr(t):
    return None if t is None else t.data_ptr()


class KVFS:
    """One KVFS context (one page pool) on one device, or a host-only metadata context (device=-1)."""

    def __init__(self, n_layers: int, n_q_heads: int, n_kv_heads: int, head_dim: int, page_size: int,
                 n_pages: int, max_batch_rows: int = 4096, max_batch_descs: int = 1024, device: int = 0,
                 table_capacity: int = 0):
        self.L, self.Hq, self.Hkv, self.D, self.P = n_layers, n_q_heads, n_kv_heads, head_dim, page_size
        self.n_pages = n_pages
        self.device = device
        self.k_pool: List = []
        self.v_pool: List = []
        self.workspace = None
        cfg = KvfsConfig(device=device, n_layers=n_layers, n_q_heads=n_q_heads, n_kv_heads=n_kv_heads,
                         head_dim=head_dim, page_size=page_size, n_pages=n_pages,
                         max_batch_rows=max_batch_rows, max_batch_descs=max_batch_descs,
                         table_capacity=table_capacity)
        self._ptr_arrays = None
        if device >= 0:
            import torch

            dev = torch.device("cuda", device)
            for _ in range(n_layers):
                self.k_pool.append(torch.empty((n_pages, n_kv_heads, page_size, head_dim), dtype=torch.bfloat16,
                                               device=dev))
                self.v_pool.append(torch.empty((n_pages, n_kv_heads, page_size, head_dim), dtype=torch.bfloat16,
                                               device=dev))
            kp = (ctypes.c_void_p * n_layers)(*[t.data_ptr() for t in self.k_pool])
            vp = (ctypes.c_void_p * n_layers)(*[t.data_ptr() for t in self.v_pool])
            self._ptr_arrays = (kp, vp)
            cfg.k_pool = ctypes.cast(kp, ctypes.POINTER(ctypes.c_void_p))
            cfg.v_pool = ctypes.cast(vp, ctypes.POINTER(ctypes.c_void_p))
            nbytes = lib().kvfs_workspace_bytes(ctypes.byref(cfg))
            if nbytes == 0:
                raise KvfsError(EINVAL, "kvfs_workspace_bytes")
            self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=dev)
            base = self.workspace.data_ptr()
            cfg.workspace = ctypes.c_void_p((base + 255) & ~255)
            cfg.workspace_bytes = nbytes
        self._cfg = cfg
        h = ctypes.c_void_p()
        _check(lib().kvfs_init(ctypes.byref(cfg), ctypes.byref(h)), "kvfs_init")
        self._h = h

    # ------------------------------------------------------------------ lifecycle
    def close_ctx(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().kvfs_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close_ctx()
        except Exception:
            pass

    # ------------------------------------------------------------------ files
    def open(self, name: str, flags: int = O_CREAT) -> int:
        fd = ctypes.c_int()
        _check(lib().kvfs_open(self._h, name.encode(), flags, ctypes.byref(fd)), f"open {name}")
        return fd.value

    def close(self, fd: int) -> None:
        _check(lib().kvfs_close(self._h, fd), "close")

    def unlink(self, name: str) -> None:
        _check(lib().kvfs_unlink(self._h, name.encode()), f"unlink {name}")

    def fork(self, src_fd: int, dst_name: str, stream=None) -> int:
        fd = ctypes.c_int()
        st = _stream(stream) if self.device >= 0 else None
        _check(lib().kvfs_fork(self._h, src_fd, dst_name.encode(), ctypes.byref(fd), st), "fork")
        return fd.value

    def truncate(self, fd: int, n: int) -> None:
        _check(lib().kvfs_truncate(self._h, fd, n), "truncate")

    def evict(self, fd: int, ranges: Sequence[Tuple[int, int]], compact: bool = False, stream=None) -> None:
        arr = np.ascontiguousarray(np.asarray(ranges, dtype=np.int64).reshape(-1, 2))
        st = _stream(stream) if self.device >= 0 else None
        _check(lib().kvfs_evict(self._h, fd, _ptr(arr, ctypes.c_int64), arr.shape[0],
                                EVICT_COMPACT if compact else 0, st), "evict")

    def compact(self, fd: int, stream=None) -> None:
        st = _stream(stream) if self.device >= 0 else None
        _check(lib().kvfs_compact(self._h, fd, st), "compact")

    def compact_files(self, fds, stream=None) -> int:
        """kvfs_compact of every fd in order (one call; host position passes on worker threads).  Returns
        the number of files compacted; raises on an error (files before the failing one stay compacted)."""
        a = np.ascontiguousarray(np.asarray(list(fds), dtype=np.int32))
        done = ctypes.c_int(0)
        st = _stream(stream) if self.device >= 0 else None
        rc = lib().kvfs_compact_files(self._h, _ptr(a, ctypes.c_int), a.shape[0], ctypes.byref(done), st)
        if rc != OK:
            raise KvfsError(rc, f"compact_files ({done.value} done)")
        return done.value

    def extract(self, src_fd: int, indices, name: str, stream=None) -> int:
        """New file `name` with the logical tokens `indices` of src (kvfs_extract)."""
        idx = np.ascontiguousarray(np.asarray(list(indices), dtype=np.int64))
        fd = ctypes.c_int()
        st = _stream(stream) if self.device >= 0 else None
        _check(lib().kvfs_extract(self._h, src_fd, _ptr(idx, ctypes.c_int64), idx.shape[0], name.encode(),
                                  ctypes.byref(fd), st), f"extract {name}")
        return fd.value

    def merge(self, fds, name: str, stream=None) -> int:
        """New file `name` with every part's tokens sorted by position (kvfs_merge)."""
        arr = np.ascontiguousarray(np.asarray(list(fds), dtype=np.int32))
        fd = ctypes.c_int()
        st = _stream(stream) if self.device >= 0 else None
        _check(lib().kvfs_merge(self._h, _ptr(arr, ctypes.c_int32), arr.shape[0], name.encode(),
                                ctypes.byref(fd), st), f"merge {name}")
        return fd.value

    def offload(self, fd: int, stream=None) -> int:
        """Move the file's exclusively owned pages to the host tier (R15). Returns pages moved."""
        n = ctypes.c_int64()
        st = _stream(stream) if self.device >= 0 else None
        _check(lib().kvfs_offload(self._h, fd, ctypes.byref(n), st), "offload")
        return n.value

    def restore(self, fd: int, stream=None) -> int:
        """Bring an offloaded file's host pages back into fresh device pages (R15). Returns pages moved."""
        n = ctypes.c_int64()
        st = _stream(stream) if self.device >= 0 else None
        _check(lib().kvfs_restore(self._h, fd, ctypes.byref(n), st), "restore")
        return n.value

    def append(self, fd: int, pos, k=None, v=None, stream=None) -> None:
        """pos: host int sequence; k, v: device bf16 tensors [L][n][Hkv][D] (None on a host-only ctx)."""
        p = _i32(pos)
        st = _stream(stream) if self.device >= 0 else None
        _check(lib().kvfs_append(self._h, fd, p.shape[0], _ptr(p, ctypes.c_int32), _dptr(k), _dptr(v), st),
               "append")

    # ------------------------------------------------------------------ pred
    @staticmethod
    def _descs(descs):
        """descs: list of (fd, n_q) or an int32 numpy array [n][2] (fast path, no per-item Python work).
        Returns (address of the pred_desc array, n, the array to keep alive)."""
        if isinstance(descs, np.ndarray):
            a = np.ascontiguousarray(descs, dtype=np.int32).reshape(-1, 2)
        else:
            a = np.array(list(descs), dtype=np.int32).reshape(-1, 2)
        return (a.ctypes.data if a.shape[0] else None), a.shape[0], a

    def pred_attn_batch(self, descs, pos, q, k_new, v_new, out, lse=None, scale: Optional[float] = None,
                        stream=None) -> List[int]:
        """Batched pred (one layer). Returns the per-descriptor status list; raises on call-level errors."""
        arr, n, _keep = self._descs(descs)
        p = _i32(pos)
        status = np.empty(max(1, n), np.int32)
        scale = float(scale if scale is not None else self.D ** -0.5)
        rc = _lib.pred_attn_batch(self._h, arr, n, p.ctypes.data, _daddr(q), _daddr(k_new), _daddr(v_new),
                                  _daddr(out), _daddr(lse), scale, status.ctypes.data, _stream(stream, self.device))
        if rc not in (OK, EPARTIAL):
            raise KvfsError(rc, "pred_attn_batch")
        return status[:n].tolist()

    def pred_attn_batch_host(self, descs, pos, q, k_new, v_new, out, lse=None, scale: Optional[float] = None,
                             stream=None) -> List[int]:
        """Batched pred with HOST buffers (include/kvfs.h pred_attn_batch_host): q / k_new / v_new / out / lse are
        pinned CPU tensors; the library stages them through its device slots.  out / lse are complete after
        pred_host_fence(stream) and a synchronisation of that stream."""
        arr, n, _keep = self._descs(descs)
        p = _i32(pos)
        status = np.empty(max(1, n), np.int32)
        scale = float(scale if scale is not None else self.D ** -0.5)
        rc = _lib.pred_attn_batch_host(self._h, arr, n, p.ctypes.data, _daddr(q), _daddr(k_new), _daddr(v_new),
                                       _daddr(out), _daddr(lse), scale, status.ctypes.data,
                                       _stream(stream, self.device))
        if rc not in (OK, EPARTIAL):
            raise KvfsError(rc, "pred_attn_batch_host")
        return status[:n].tolist()

    def pred_host_fence(self, stream=None) -> None:
        _check(_lib.pred_host_fence(self._h, _stream(stream, self.device)), "pred_host_fence")

    def pred_step_begin(self, descs, pos, stream=None):
        arr, n, _keep = self._descs(descs)
        p = _i32(pos)
        status = np.empty(max(1, n), np.int32)
        step = ctypes.c_void_p()
        st = _stream(stream, self.device) if self.device >= 0 else None
        rc = _lib.pred_step_begin(self._h, arr, n, p.ctypes.data, status.ctypes.data, ctypes.byref(step), st)
        if rc not in (OK, EPARTIAL):
            raise KvfsError(rc, "pred_step_begin")
        return step, status[:n].tolist()

    def pred_attn_layer(self, step, layer, q, k_new, v_new, out, lse=None, scale=None, stream=None) -> None:
        scale = float(scale if scale is not None else self.D ** -0.5)
        rc = _lib.pred_attn_layer(self._h, step, layer, _daddr(q), _daddr(k_new), _daddr(v_new), _daddr(out),
                                  _daddr(lse), scale, _stream(stream, self.device))
        if rc != OK:
            raise KvfsError(rc, "pred_attn_layer")

    def pred_step_end(self, step) -> None:
        _check(lib().pred_step_end(self._h, step), "pred_step_end")

    def set_logits_buffer(self, buf) -> None:
        """Fused scores (include/kvfs.h kvfs_set_logits_buffer): a device tensor the decode kernel writes its
        logits into (None = off).  Keep it alive while registered."""
        self._logits = buf
        _check(_lib.kvfs_set_logits_buffer(self._h, None if buf is None else buf.data_ptr(),
                                           0 if buf is None else buf.numel() * buf.element_size()),
               "set_logits_buffer")

    def pred_attn_scores(self, step, layer, q, lse, scores, score_off, scale=None, stream=None) -> None:
        """Accumulated softmax weight per retained token (H2O; include/kvfs.h pred_attn_scores): after
        pred_attn_layer of the same step with the same q and the lse it wrote."""
        scale = float(scale if scale is not None else self.D ** -0.5)
        off = np.ascontiguousarray(np.asarray(score_off, dtype=np.int64))
        _check(lib().pred_attn_scores(self._h, step, layer, _dptr(q), _dptr(lse), scale, _dptr(scores),
                                      _ptr(off, ctypes.c_int64), _stream(stream)), "pred_attn_scores")

    # ------------------------------------------------------------------ introspection
    def stat(self, fd: int) -> Tuple[int, int, int]:
        s = KvfsStat()
        _check(lib().kvfs_stat(self._h, fd, ctypes.byref(s)), "stat")
        return s.len, s.n_entries, s.last_pos

    def table(self, fd: int) -> List[Tuple[int, int]]:
        n = ctypes.c_int64()
        _check(lib().kvfs_get_table(self._h, fd, None, None, 0, ctypes.byref(n)), "get_table")
        pg = np.zeros(max(1, n.value), np.uint32)
        mk = np.zeros(max(1, n.value), np.uint64)
        _check(lib().kvfs_get_table(self._h, fd, _ptr(pg, ctypes.c_uint32), _ptr(mk, ctypes.c_uint64), n.value,
                                    ctypes.byref(n)), "get_table")
        return [(int(a), int(b)) for a, b in zip(pg[:n.value], mk[:n.value])]

    def positions(self, fd: int) -> List[int]:
        n = ctypes.c_int64()
        _check(lib().kvfs_get_positions(self._h, fd, None, 0, ctypes.byref(n)), "get_positions")
        out = np.zeros(max(1, n.value), np.int32)
        _check(lib().kvfs_get_positions(self._h, fd, _ptr(out, ctypes.c_int32), n.value, ctypes.byref(n)),
               "get_positions")
        return out[:n.value].tolist()

    def refcounts(self) -> List[int]:
        out = np.zeros(self.n_pages, np.uint32)
        _check(lib().kvfs_get_refcounts(self._h, _ptr(out, ctypes.c_uint32), self.n_pages), "get_refcounts")
        return out.tolist()

    def free_pages(self) -> int:
        n = ctypes.c_int64()
        _check(lib().kvfs_free_pages(self._h, ctypes.byref(n)), "free_pages")
        return n.value

    def read(self, fd: int, layer: int, begin: int, end: int, stream=None):
        import torch

        n = end - begin
        k = torch.empty((n, self.Hkv, self.D), dtype=torch.bfloat16, device=self.k_pool[0].device)
        v = torch.empty_like(k)
        _check(lib().kvfs_read(self._h, fd, layer, begin, end, _dptr(k), _dptr(v), _stream(stream)), "read")
        return k, v

    def audit(self) -> None:
        _check(lib().kvfs_audit(self._h), "audit")

    def set_option(self, option: int, value: int) -> None:
        _check(lib().kvfs_set_option(self._h, option, value), "set_option")

    # ------------------------------------------------------------------ migration
    def pack(self, fds: Sequence[int], stream=None):
        """Pack a file set: returns (header bytes, device uint8 buffer or None on a host-only ctx)."""
        arr = (ctypes.c_int * max(1, len(fds)))(*fds)
        bu, hu = ctypes.c_size_t(), ctypes.c_size_t()
        st = _stream(stream) if self.device >= 0 else None
        rc = lib().kvfs_pack(self._h, arr, len(fds), None, 0, ctypes.byref(bu), None, 0, ctypes.byref(hu), st)
        if rc not in (OK, ENOMEM):
            raise KvfsError(rc, "pack")
        hdr = ctypes.create_string_buffer(max(1, hu.value))
        buf = None
        if self.device >= 0:
            import torch
            buf = torch.empty(max(16, bu.value), dtype=torch.uint8, device=self.k_pool[0].device)
        _check(lib().kvfs_pack(self._h, arr, len(fds), _dptr(buf), 0 if buf is None else buf.numel(),
                               ctypes.byref(bu), hdr, len(hdr), ctypes.byref(hu), st), "pack")
        return hdr.raw[:hu.value], buf

    def unpack(self, hdr: bytes, buf, names: Sequence[str], stream=None) -> List[int]:
        n = len(names)
        nm = (ctypes.c_char_p * max(1, n))(*[x.encode() for x in names])
        fds = (ctypes.c_int * max(1, n))()
        st = _stream(stream) if self.device >= 0 else None
        nbuf = 0 if buf is None else buf.numel() * buf.element_size()
        _check(lib().kvfs_unpack(self._h, _dptr(buf), nbuf, hdr, len(hdr), nm, fds, st), "unpack")
        return list(fds[:n])

    def counter(self, which: int) -> int:
        v = ctypes.c_int64()
        _check(lib().kvfs_get_counter(self._h, which, ctypes.byref(v)), "get_counter")
        return v.value


class Scheduler:
    """Inference scheduler batch formation (kvfs_sched_*, §4.4): Poisson-rate-sized
    FIFO batches of pred requests.  Host only."""

    def __init__(self, w_max: float = 0.010, b_max: int = 64, alpha: float = 0.2, dt_default: float = 0.1):
        cfg = SchedConfig(w_max, b_max, alpha, dt_default)
        h = ctypes.c_void_p()
        _check(lib().kvfs_sched_create(ctypes.byref(cfg), ctypes.byref(h)), "sched_create")
        self._h = h
        self.b_max = b_max

    def __del__(self):
        if getattr(self, "_h", None):
            lib().kvfs_sched_destroy(self._h)
            self._h = None

    def enqueue(self, fd: int, pos, now: float) -> None:
        p = _i32(pos)
        _check(lib().kvfs_sched_enqueue(self._h, fd, p.shape[0], _ptr(p, ctypes.c_int32), now), "sched_enqueue")

    def state(self):
        lam, tgt, n = ctypes.c_double(), ctypes.c_int(), ctypes.c_int()
        _check(lib().kvfs_sched_state(self._h, ctypes.byref(lam), ctypes.byref(tgt), ctypes.byref(n)), "sched_state")
        return lam.value, tgt.value, n.value

    def form(self, now: float, pos_cap: int = 1 << 16):
        """None if no batch is due, else ([(fd, n_q)], positions)."""
        descs = (PredDesc * self.b_max)()
        pos = np.zeros(pos_cap, dtype=np.int32)
        nd, nr = ctypes.c_int(), ctypes.c_int64()
        rc = lib().kvfs_sched_form(self._h, now, ctypes.cast(descs, ctypes.c_void_p), self.b_max,
                                   _ptr(pos, ctypes.c_int32), pos_cap, ctypes.byref(nd), ctypes.byref(nr))
        if rc == 0:
            return None
        _check(rc if rc < 0 else 0, "sched_form")
        return [(descs[i].fd, descs[i].n_q) for i in range(nd.value)], pos[:nr.value].tolist()
