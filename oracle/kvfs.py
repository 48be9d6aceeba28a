"""KVFS oracle: page pool + refcounts + files (§4.2) and the batched pred reserve
(§4.1, §4.4). TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

State: refcnt[page] (free <=> 0); files: name -> {table: [[page, mask]], pos: [int]};
optionally the physical bf16 pages K[l][page][g][slot][:], V[...] (uint16 bit patterns).
Derived: len = sum popcount(mask); logical token k = k-th set bit scanning entries in order, slots
ascending; hi(entry) = highest set slot; the tail = the last entry.

Rules (readings of a silent paper; numbers as in SURVEY.md §8(c) C3):
  R1 allocation  smallest free page id, one page at a time, in logical / descriptor order
  R2 open        P:223 "creating an empty file"; EEXIST with O_EXCL, ENOENT without O_CREAT
  R3 append      P:215 file "updated with new tensors"; CoW of a shared tail with room
  R4 fork        P:177, "without duplicating the actual tensors": full pages shared, a tail with
                 room deep-copied into a fresh page
  R5 truncate    keep logical [0, n); positions truncated (rollback)
  R6 evict       P:225 "removing invalid or unimportant tokens": clear mask bits, drop empty entries,
                 retained positions unchanged
  R7 compact     gather the retained tokens in logical order into ceil(len/P) fresh pages allocated
                 while the old ones are still held, then release the old entries
  R8 evict+COMPACT  R6 then R7 as one atomic op
  R9 unlink/close   unlink releases every entry and the name; close releases the fd
  R11 batch      descriptors in order; per descriptor EBADF / EBUSY (file repeated) / EPOS / ENOSPC,
                 isolated failures, EPARTIAL overall
  R13 extract    P:225 "create new files from existing ones by extracting specific token indices": a new
                 file holding the selected logical tokens (strictly increasing indices, EINVAL; < len,
                 ERANGE) in order with their original positions, in ceil(k/P) fresh pages allocated by R1
                 in logical order (pages rebuilt, no sharing); the source is unchanged
  R15 offload    P:233 "offloads their KV caches from the GPU to the CPU and restores them upon I/O
                 completion": offload moves every EXCLUSIVELY owned page (refcount 1) of the file to the
                 host tier (entry page := HOST | host slot, in table order) and frees it on the device;
                 shared pages stay.  restore allocates device pages by R1 in table order
                 for the host entries (ENOSPC atomic) and copies the bits back.  While offloaded, every op
                 touching the file's pages (append / pred / fork / truncate / evict / compact / extract /
                 merge / read) is EOFFLOAD; stat, tables, close and unlink are allowed
  R14 merge      P:225 "merging existing files into one": a new file holding every part's retained tokens
                 sorted by position (duplicate positions: EPOS), pages rebuilt as in R13;
                 a part listed twice is EBUSY; the parts are unchanged
Pinned by tests/test_oracle_kvfs.py: SPEC worked examples S:62, S:70, S:78, S:79, S:87, S:88, S:89,
S:608; the golden trace tests/golden/c7_trace.json; a deep-copy shadow model on
random op sequences; invariants I1-I5 after every op.
"""
from __future__ import annotations

import heapq
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .attention import attention_scores, gqa_attention
from .bf16 import bf16_to_f64

OK = 0
ENOENT = -2
EIO = -5
EBADF = -9
EBUSY = -16
EEXIST = -17
EINVAL = -22
ENOSPC = -28
ERANGE = -34
EPOS = -1001
EPARTIAL = -1002
EOFFLOAD = -1003  # the file's exclusive pages are in the host tier (R15): restore it first
HOST = 1 << 31    # table page field of an entry whose page lives in the host tier: HOST | host slot

O_CREAT = 1
O_EXCL = 2
EVICT_COMPACT = 1


class KvfsError(Exception):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"kvfs error {code}: {msg}")
        self.code = code


def _popcount(mask: int) -> int:
    return bin(mask).count("1")


def _hi(mask: int) -> int:
    return mask.bit_length() - 1


class _File:
    __slots__ = ("name", "table", "pos", "alive", "host")

    def __init__(self, name: str):
        self.name = name
        self.table: List[List[int]] = []  # [[page, mask], ...]
        self.pos: List[int] = []
        self.alive = True
        self.host = None  # R15: list of saved (K, V) page bits per host slot while offloaded

    def length(self) -> int:
        return sum(_popcount(m) for _, m in self.table)

    def logical(self) -> List[Tuple[int, int]]:
        """(page, slot) of every retained token in logical order."""
        out = []
        for page, mask in self.table:
            for slot in range(mask.bit_length()):
                if mask >> slot & 1:
                    out.append((page, slot))
        return out


class Oracle:
    def __init__(self, n_pages: int, page_size: int = 16, n_layers: int = 1, n_kv_heads: int = 1,
                 head_dim: int = 64, store_data: bool = True):
        assert page_size in (16, 32, 64)
        self.n_pages = n_pages
        self.P = page_size
        self.L = n_layers
        self.Hkv = n_kv_heads
        self.D = head_dim
        self.refcnt = [0] * n_pages
        self._free = list(range(n_pages))  # min-heap of free page ids (R1)
        heapq.heapify(self._free)
        self.names: Dict[str, _File] = {}
        self.fds: Dict[int, _File] = {}
        self.copies: List[Tuple[int, int]] = []  # every whole-page copy (src, dst): CoW and fork tails
        self.store = store_data
        if store_data:
            shape = (n_layers, n_pages, n_kv_heads, page_size, head_dim)
            self.K = np.zeros(shape, dtype=np.uint16)
            self.V = np.zeros(shape, dtype=np.uint16)

    # ------------------------------------------------------------------ pool (R1)
    def free_count(self) -> int:
        return len(self._free)

    def _alloc(self) -> int:
        p = heapq.heappop(self._free)  # smallest free id
        assert self.refcnt[p] == 0
        self.refcnt[p] = 1
        return p

    def _release(self, page: int) -> None:
        assert self.refcnt[page] > 0
        self.refcnt[page] -= 1
        if self.refcnt[page] == 0:
            heapq.heappush(self._free, page)

    def _copy_slots(self, src: int, dst: int, mask: int) -> None:
        self.copies.append((src, dst))
        if self.store:
            for slot in range(self.P):
                if mask >> slot & 1:
                    self.K[:, dst, :, slot, :] = self.K[:, src, :, slot, :]
                    self.V[:, dst, :, slot, :] = self.V[:, src, :, slot, :]

    # ------------------------------------------------------------------ names / fds (R2, R9)
    def _file(self, fd: int) -> _File:
        f = self.fds.get(fd)
        if f is None or not f.alive:
            raise KvfsError(EBADF, f"bad fd {fd}")
        return f

    def _live(self, fd: int) -> _File:
        """A file whose pages are on the device (R15)."""
        f = self._file(fd)
        if f.host is not None:
            raise KvfsError(EOFFLOAD, "offloaded")
        return f

    def _new_fd(self, f: _File) -> int:
        fd = 0
        while fd in self.fds:
            fd += 1
        self.fds[fd] = f
        return fd

    def open(self, name: str, flags: int = O_CREAT) -> int:
        if not name:
            raise KvfsError(EINVAL, "empty name")
        f = self.names.get(name)
        if f is not None:
            if (flags & O_CREAT) and (flags & O_EXCL):
                raise KvfsError(EEXIST, name)
            return self._new_fd(f)
        if not (flags & O_CREAT):
            raise KvfsError(ENOENT, name)
        f = _File(name)
        self.names[name] = f
        return self._new_fd(f)

    def close(self, fd: int) -> None:
        if fd not in self.fds:
            raise KvfsError(EBADF, f"bad fd {fd}")
        del self.fds[fd]

    def unlink(self, name: str) -> None:
        f = self.names.get(name)
        if f is None:
            raise KvfsError(ENOENT, name)
        for page, _ in f.table:
            if not page & HOST:
                self._release(page)
        f.table = []
        f.pos = []
        f.host = None
        f.alive = False
        del self.names[name]

    # ------------------------------------------------------------------ introspection
    def table(self, fd: int) -> List[Tuple[int, int]]:
        return [(p, m) for p, m in self._file(fd).table]

    def positions(self, fd: int) -> List[int]:
        return list(self._file(fd).pos)

    def stat(self, fd: int) -> Tuple[int, int, int]:
        f = self._file(fd)
        return f.length(), len(f.table), (f.pos[-1] if f.pos else -1)

    def read(self, fd: int, layer: int, begin: int, end: int):
        """bf16 bits of logical tokens [begin, end): k, v of shape [n][Hkv][D]."""
        f = self._live(fd)
        assert self.store
        if not (0 <= begin <= end <= f.length()):
            raise KvfsError(ERANGE, "read range")
        lg = f.logical()[begin:end]
        if not lg:
            z = np.zeros((0, self.Hkv, self.D), np.uint16)
            return z, z.copy()
        pages = np.array([p for p, _ in lg])
        sl = np.array([x for _, x in lg])
        return self.K[layer, pages, :, sl, :], self.V[layer, pages, :, sl, :]

    def audit(self) -> None:
        """Invariants I1-I5. Raises AssertionError on violation."""
        count = [0] * self.n_pages
        for f in self.names.values():
            seen = set()
            for page, mask in f.table:
                assert mask != 0, "I1: empty entry"
                assert mask < (1 << self.P)
                assert page not in seen, "I2: page twice in one file"
                seen.add(page)
                if page & HOST:
                    assert f.host is not None and (page & ~HOST) < len(f.host), "host entry of a live file"
                    continue
                count[page] += 1
            assert len(f.pos) == f.length(), "positions vs length"
            assert all(a < b for a, b in zip(f.pos, f.pos[1:])), "I4: positions not increasing"
        assert count == self.refcnt, "I3: refcount != number of referencing files"
        assert sorted(self._free) == [p for p in range(self.n_pages) if self.refcnt[p] == 0]
        if not self.names:
            assert sum(self.refcnt) == 0, "I5: leak"

    # ------------------------------------------------------------------ R3 append
    def _append_plan(self, f: _File, pos: Sequence[int]) -> int:
        """Validate (EPOS) and return the page need of appending len(pos) tokens (raises ENOSPC)."""
        n = len(pos)
        last = f.pos[-1] if f.pos else -1
        if pos[0] <= last or any(b <= a for a, b in zip(pos, pos[1:])):
            raise KvfsError(EPOS, "positions must be strictly increasing and > last retained")
        room, cow = 0, False
        if f.table:
            page, mask = f.table[-1]
            room = self.P - 1 - _hi(mask)
            cow = room > 0 and self.refcnt[page] > 1
        need = (1 if cow else 0) + -(-max(0, n - room) // self.P)
        if need > self.free_count():
            raise KvfsError(ENOSPC, f"need {need} pages")
        return need

    def _append_commit(self, f: _File, pos: Sequence[int]) -> List[Tuple[int, int]]:
        """Apply R3 after _append_plan succeeded. Returns the (page, slot) of each new token."""
        n = len(pos)
        slots: List[Tuple[int, int]] = []
        if f.table:
            entry = f.table[-1]
            page, mask = entry
            hi = _hi(mask)
            room = self.P - 1 - hi
            if room > 0 and self.refcnt[page] > 1:  # copy-on-write of the shared tail
                q = self._alloc()
                self._copy_slots(page, q, mask)
                self._release(page)
                entry[0] = q
            take = min(n, room)
            for i in range(take):
                entry[1] |= 1 << (hi + 1 + i)
                slots.append((entry[0], hi + 1 + i))
        i = len(slots)
        while i < n:
            q = self._alloc()
            take = min(self.P, n - i)
            f.table.append([q, (1 << take) - 1])
            slots.extend((q, s) for s in range(take))
            i += take
        f.pos.extend(int(p) for p in pos)
        return slots

    def _write_rows(self, slots, k_rows, v_rows) -> None:
        """k_rows / v_rows: [L][n][Hkv][D] bf16 bits."""
        if not self.store or not slots:
            return
        pages = np.array([p for p, _ in slots])
        sl = np.array([x for _, x in slots])
        # advanced indices split by a slice put the row axis first: [n][L][Hkv][D]
        self.K[:, pages, :, sl, :] = np.asarray(k_rows).transpose(1, 0, 2, 3)
        self.V[:, pages, :, sl, :] = np.asarray(v_rows).transpose(1, 0, 2, 3)

    def append(self, fd: int, pos: Sequence[int], k_rows=None, v_rows=None) -> None:
        f = self._live(fd)
        if len(pos) == 0:
            return
        self._append_plan(f, pos)
        slots = self._append_commit(f, pos)
        if self.store:
            self._write_rows(slots, np.asarray(k_rows), np.asarray(v_rows))

    # ------------------------------------------------------------------ R4 fork
    def fork(self, src_fd: int, dst_name: str) -> int:
        src = self._live(src_fd)
        if not dst_name:
            raise KvfsError(EINVAL, "empty name")
        if dst_name in self.names:
            raise KvfsError(EEXIST, dst_name)
        copy_tail = bool(src.table) and _hi(src.table[-1][1]) < self.P - 1
        if copy_tail and self.free_count() < 1:
            raise KvfsError(ENOSPC, "fork tail copy")
        dst = _File(dst_name)
        dst.table = [[p, m] for p, m in src.table]
        dst.pos = list(src.pos)
        for p, _ in dst.table:
            self.refcnt[p] += 1
        if copy_tail:
            page, mask = dst.table[-1]
            q = self._alloc()
            self._copy_slots(page, q, mask)
            self._release(page)  # restore the parent tail's count
            dst.table[-1][0] = q
        self.names[dst_name] = dst
        return self._new_fd(dst)

    # ------------------------------------------------------------------ R5 truncate
    def truncate(self, fd: int, n: int) -> None:
        f = self._live(fd)
        length = f.length()
        if n < 0 or n > length:
            raise KvfsError(ERANGE, "truncate length")
        keep: List[List[int]] = []
        acc = 0
        for entry in f.table:
            page, mask = entry
            c = _popcount(mask)
            if acc >= n:
                self._release(page)
                continue
            if acc + c > n:  # keep only the lowest (n - acc) set bits
                need, new = n - acc, 0
                for slot in range(self.P):
                    if need == 0:
                        break
                    if mask >> slot & 1:
                        new |= 1 << slot
                        need -= 1
                mask = new
            keep.append([page, mask])
            acc += _popcount(mask)
        f.table = keep
        f.pos = f.pos[:n]

    # ------------------------------------------------------------------ R6/R7/R8 evict, compact
    def _check_ranges(self, f: _File, ranges: Sequence[Tuple[int, int]]) -> None:
        length = f.length()
        prev_b = None
        for a, b in ranges:
            if a >= b:
                raise KvfsError(EINVAL, "empty range")
            if prev_b is not None and a < prev_b:
                raise KvfsError(EINVAL, "ranges not sorted/disjoint")
            if a < 0 or b > length:
                raise KvfsError(ERANGE, "range outside file")
            prev_b = b

    def evict(self, fd: int, ranges: Sequence[Tuple[int, int]], flags: int = 0) -> None:
        f = self._live(fd)
        self._check_ranges(f, ranges)
        drop = set()
        for a, b in ranges:
            drop.update(range(a, b))
        # accounting after R6: pages whose every reference disappears become free
        new_table, released = [], []
        idx = 0
        new_pos = []
        for page, mask in f.table:
            new = mask
            for slot in range(self.P):
                if mask >> slot & 1:
                    if idx in drop:
                        new &= ~(1 << slot)
                    else:
                        new_pos.append(f.pos[idx])
                    idx += 1
            if new:
                new_table.append([page, new])
            else:
                released.append(page)
        if flags & EVICT_COMPACT:
            length = len(new_pos)
            k = -(-length // self.P)
            freed = sum(1 for p in released if self.refcnt[p] == 1)
            if k > self.free_count() + freed:
                raise KvfsError(ENOSPC, "compact after evict")
        for p in released:
            self._release(p)
        f.table = new_table
        f.pos = new_pos
        if flags & EVICT_COMPACT:
            self._compact_commit(f)

    def compact(self, fd: int) -> None:
        f = self._live(fd)
        length = f.length()
        if length == 0:
            return
        if -(-length // self.P) > self.free_count():
            raise KvfsError(ENOSPC, "compact")
        self._compact_commit(f)

    def _compact_commit(self, f: _File) -> None:
        length = f.length()
        if length == 0:
            return
        k = -(-length // self.P)
        new_pages = [self._alloc() for _ in range(k)]  # old pages are still held: never destinations
        src = f.logical()
        if self.store:
            for i, (page, slot) in enumerate(src):
                dp, ds = new_pages[i // self.P], i % self.P
                self.K[:, dp, :, ds, :] = self.K[:, page, :, slot, :]
                self.V[:, dp, :, ds, :] = self.V[:, page, :, slot, :]
        old = f.table
        full = (1 << self.P) - 1
        f.table = [[p, full] for p in new_pages[:-1]]
        f.table.append([new_pages[-1], (1 << (length - (k - 1) * self.P)) - 1])
        for page, _ in old:
            self._release(page)

    # ------------------------------------------------------------------ R15 offload / restore
    def host_pages(self) -> int:
        return sum(len(f.host) for f in self.names.values() if f.host is not None)

    def offload(self, fd: int) -> int:
        """Returns the number of pages moved to the host tier."""
        f = self._file(fd)
        if f.host is not None:
            raise KvfsError(EINVAL, "already offloaded")
        f.host = []
        for e in f.table:
            page = e[0]
            if self.refcnt[page] == 1:
                f.host.append((self.K[:, page].copy(), self.V[:, page].copy()) if self.store else None)
                e[0] = HOST | (len(f.host) - 1)
                self._release(page)
        return len(f.host)

    def restore(self, fd: int) -> int:
        f = self._file(fd)
        if f.host is None:
            raise KvfsError(EINVAL, "not offloaded")
        n = sum(1 for page, _ in f.table if page & HOST)
        if n > self.free_count():
            raise KvfsError(ENOSPC, "restore")
        for e in f.table:
            if e[0] & HOST:
                q = self._alloc()
                if self.store:
                    kk, vv = f.host[e[0] & ~HOST]
                    self.K[:, q] = kk
                    self.V[:, q] = vv
                e[0] = q
        f.host = None
        return n

    # ------------------------------------------------------------------ R13 extract, R14 merge
    def _build(self, name: str, src: List[Tuple[int, int]], pos: List[int]) -> int:
        """New file `name` whose token i is a copy of pool slot src[i] = (page, slot), position pos[i]:
        ceil(k/P) fresh pages allocated one at a time (R1), token i -> (new[i // P], i % P)."""
        if name in self.names:
            raise KvfsError(EEXIST, name)
        k = len(src)
        n_new = -(-k // self.P)
        if n_new > self.free_count():
            raise KvfsError(ENOSPC, "extract/merge")
        new_pages = [self._alloc() for _ in range(n_new)]
        if self.store:
            for i, (page, slot) in enumerate(src):
                dp, ds = new_pages[i // self.P], i % self.P
                self.K[:, dp, :, ds, :] = self.K[:, page, :, slot, :]
                self.V[:, dp, :, ds, :] = self.V[:, page, :, slot, :]
        f = _File(name)
        full = (1 << self.P) - 1
        for j, p in enumerate(new_pages):
            cnt = min(self.P, k - j * self.P)
            f.table.append([p, full if cnt == self.P else (1 << cnt) - 1])
        f.pos = list(pos)
        self.names[name] = f
        return self._new_fd(f)

    def extract(self, src_fd: int, indices: Sequence[int], name: str) -> int:
        f = self._live(src_fd)
        idx = list(indices)
        if any(b <= a for a, b in zip(idx, idx[1:])):
            raise KvfsError(EINVAL, "indices not strictly increasing")
        if idx and (idx[0] < 0 or idx[-1] >= f.length()):
            raise KvfsError(ERANGE, "index out of range")
        lg = f.logical()
        return self._build(name, [lg[i] for i in idx], [f.pos[i] for i in idx])

    def merge(self, fds: Sequence[int], name: str) -> int:
        files = [self._live(fd) for fd in fds]
        if len(set(map(id, files))) != len(files):
            raise KvfsError(EBUSY, "a part appears twice")
        toks = []
        for f in files:
            toks.extend(zip(f.pos, f.logical()))
        toks.sort(key=lambda t: t[0])
        if any(a[0] == b[0] for a, b in zip(toks, toks[1:])):
            raise KvfsError(EPOS, "duplicate position across parts")
        return self._build(name, [t[1] for t in toks], [t[0] for t in toks])

    # ------------------------------------------------------------------ R11 batched pred (+ R10)
    def pred_reserve(self, descs: Sequence[Tuple[int, int]], pos: Sequence[int]):
        """Reserve-only form of pred_batch (no data). Returns (status list, per-desc slot lists)."""
        T = len(pos)
        if any(nq < 0 for _, nq in descs) or sum(nq for _, nq in descs) != T:
            raise KvfsError(EINVAL, "descriptor row counts")
        status, slot_lists = [], []
        seen = set()
        row = 0
        for fd, nq in descs:
            rows = list(pos[row:row + nq])
            row += nq
            f = self.fds.get(fd)
            if f is None or not f.alive:
                status.append(EBADF)
                slot_lists.append(None)
                continue
            if id(f) in seen:
                status.append(EBUSY)
                slot_lists.append(None)
                continue
            seen.add(id(f))
            if f.host is not None:
                status.append(EOFFLOAD)
                slot_lists.append(None)
                continue
            if nq == 0:
                status.append(OK)
                slot_lists.append([])
                continue
            try:
                self._append_plan(f, rows)
            except KvfsError as e:
                status.append(e.code)
                slot_lists.append(None)
                continue
            slot_lists.append(self._append_commit(f, rows))
            status.append(OK)
        return status, slot_lists

    def pred_batch(self, descs: Sequence[Tuple[int, int]], pos: Sequence[int], q, k_new, v_new,
                   scale: float, scores: bool = False):
        """Batched pred: q [L][T][Hq][D], k_new/v_new [L][T][Hkv][D] bf16 bits (rows packed in descriptor
        order). Returns (status, out [L][T][Hq][D] float64 (NaN rows for failed descriptors), lse)."""
        q = np.asarray(q)
        k_new = np.asarray(k_new)
        v_new = np.asarray(v_new)
        L, T, Hq, D = q.shape
        status, slot_lists = self.pred_reserve(descs, pos)
        out = np.full((L, T, Hq, D), np.nan)
        lse = np.full((L, T, Hq), np.nan)
        row = 0
        fd_of = []
        for (fd, nq), st, slots in zip(descs, status, slot_lists):
            fd_of.append((fd, row, nq, st, slots))
            row += nq
        for fd, r0, nq, st, slots in fd_of:
            if st != OK or nq == 0:
                continue
            self._write_rows(slots, k_new[:, r0:r0 + nq], v_new[:, r0:r0 + nq])
        for fd, r0, nq, st, slots in fd_of:
            if st != OK or nq == 0:
                continue
            f = self.fds[fd]
            length = f.length()
            for layer in range(L):
                kk, vv = self.read(fd, layer, 0, length)
                o, s = gqa_attention(bf16_to_f64(q[layer, r0:r0 + nq]), bf16_to_f64(kk),
                                     bf16_to_f64(vv), scale)
                out[layer, r0:r0 + nq] = o
                lse[layer, r0:r0 + nq] = s
        if scores:  # per descriptor (None if failed / n_q = 0): layer-0 accumulated weights (NEXT-2)
            sc = []
            for fd, r0, nq, st, slots in fd_of:
                if st != OK or nq == 0:
                    sc.append(None)
                    continue
                kk, _ = self.read(fd, 0, 0, self.fds[fd].length())
                sc.append(attention_scores(bf16_to_f64(q[0, r0:r0 + nq]), bf16_to_f64(kk), scale))
            return status, out, lse, sc
        return status, out, lse
