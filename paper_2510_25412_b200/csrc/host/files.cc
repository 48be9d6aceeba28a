// KVFS file operations (§4.2) on host metadata.  Each function validates first and
// mutates only after every check passed (atomic failure).  Rule numbers refer to
// SURVEY.md §8(c) C3 (restated in DESIGN.md "Readings").
#include <algorithm>
#include <cstring>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include "kvfs_impl.h"

namespace kvfs {

namespace {

inline int popc(uint64_t m) { return __builtin_popcountll(m); }
inline int hi_slot(uint64_t m) { return 63 - __builtin_clzll(m); }  // m != 0
// Slot of the r-th (0-based) set bit of m (precondition: popc(m) > r).
inline int select_bit(uint64_t m, int r) {
  for (; r > 0; --r) m &= m - 1;
  return __builtin_ctzll(m);
}

// Mask keeping only the set bits of m whose rank (0-based, ascending slots) is in [r0, r1).
uint64_t rank_range_bits(uint64_t m, int r0, int r1) {
  uint64_t out = 0;
  int r = 0;
  while (m) {
    const int s = __builtin_ctzll(m);
    if (r >= r0 && r < r1) out |= 1ull << s;
    m &= m - 1;
    if (++r >= r1) break;
  }
  return out;
}

int64_t new_fd(Ctx &c, const FilePtr &f) {
  for (size_t i = 0; i < c.fds.size(); ++i)
    if (!c.fds[i]) {
      c.fds[i] = f;
      return static_cast<int64_t>(i);
    }
  c.fds.push_back(f);
  return static_cast<int64_t>(c.fds.size() - 1);
}

// Entries at indices >= i moved or are new: the device copy of the whole suffix is stale.
void mark_dirty_from(File &f, size_t i) { f.dirty_from = std::min(f.dirty_from, i); }
// Entry i's page or mask changed in place.
void mark_dirty_pt(File &f, size_t i) {
  if (i < f.dirty_from) f.dirty_pts.push_back(static_cast<uint32_t>(i));
}

}  // namespace

// ------------------------------------------------------------------------------------------ slab
bool Slab::alloc(int64_t n, int64_t *off, int64_t *cap) {
  int cls = 6;
  while ((int64_t{1} << cls) < n) ++cls;
  if (cls >= static_cast<int>(free_.size())) return false;
  const int64_t size = int64_t{1} << cls;
  if (!free_[cls].empty()) {
    *off = free_[cls].back();
    free_[cls].pop_back();
  } else if (top_ + size <= cap_) {
    *off = top_;
    top_ += size;
  } else {
    return false;
  }
  *cap = size;
  return true;
}

void Slab::free(int64_t off, int64_t cap) {
  int cls = 0;
  while ((int64_t{1} << cls) < cap) ++cls;
  free_[cls].push_back(off);
}

void release_file_slab(Ctx &c, File &f) {
  if (f.slab_off >= 0) c.slab.free(f.slab_off, f.slab_cap);
  f.slab_off = -1;
  f.slab_cap = 0;
  f.dirty_from = 0;
  f.dirty_pts.clear();
}

int32_t last_pos(const Ctx &c, const File &f) {
  if (f.table.empty()) return -1;
  const Entry &t = f.table.back();
  return f.spos[(f.table.size() - 1) * c.cfg.page_size + hi_slot(t.mask)];
}

void file_positions(const Ctx &c, const File &f, std::vector<int32_t> *out) {
  const int P = c.cfg.page_size;
  out->clear();
  out->reserve(static_cast<size_t>(f.len));
  for (size_t e = 0; e < f.table.size(); ++e)
    for (uint64_t m = f.table[e].mask; m; m &= m - 1) out->push_back(f.spos[e * P + __builtin_ctzll(m)]);
}

// ------------------------------------------------------------------------------------------ helpers
void recompute_lstart(File &f, size_t from) {
  int64_t acc = 0;
  if (from > 0 && from <= f.table.size()) acc = f.table[from - 1].lstart + popc(f.table[from - 1].mask);
  if (from > f.table.size()) from = f.table.size();
  for (size_t i = from; i < f.table.size(); ++i) {
    f.table[i].lstart = static_cast<int32_t>(acc);
    acc += popc(f.table[i].mask);
  }
  f.len = f.table.empty() ? 0 : f.table.back().lstart + popc(f.table.back().mask);
}

// lstart of entries [from, to) from entry from - 1 (len is not touched)
static void recompute_lstart_span(File &f, size_t from, size_t to) {
  int64_t acc = from > 0 ? f.table[from - 1].lstart + popc(f.table[from - 1].mask) : 0;
  for (size_t i = from; i < to; ++i) {
    f.table[i].lstart = static_cast<int32_t>(acc);
    acc += popc(f.table[i].mask);
  }
}

File *get_file(Ctx &c, int fd) {
  if (fd < 0 || static_cast<size_t>(fd) >= c.fds.size() || !c.fds[fd] || !c.fds[fd]->alive) return nullptr;
  return c.fds[fd].get();
}

// ------------------------------------------------------------------------------------------ R2, R9
int open_file(Ctx &c, const char *name, int flags, int *fd) {
  if (!name || !*name || !fd) return KVFS_EINVAL;
  auto it = c.names.find(name);
  if (it != c.names.end()) {
    if ((flags & KVFS_O_CREAT) && (flags & KVFS_O_EXCL)) return KVFS_EEXIST;
    *fd = static_cast<int>(new_fd(c, it->second));
    return KVFS_OK;
  }
  if (!(flags & KVFS_O_CREAT)) return KVFS_ENOENT;
  auto f = std::make_shared<File>();
  f->name = name;
  c.names.emplace(f->name, f);
  *fd = static_cast<int>(new_fd(c, f));
  return KVFS_OK;
}

int close_file(Ctx &c, int fd) {
  if (fd < 0 || static_cast<size_t>(fd) >= c.fds.size() || !c.fds[fd]) return KVFS_EBADF;
  c.fds[fd].reset();
  return KVFS_OK;
}

int unlink_file(Ctx &c, const char *name) {
  if (!name || !*name) return KVFS_EINVAL;
  auto it = c.names.find(name);
  if (it == c.names.end()) return KVFS_ENOENT;
  File &f = *it->second;
  for (const Entry &e : f.table)
    if (!(e.page & KVFS_HOST_PAGE)) c.pool->release(e.page);
  if (f.offloaded) {
    c.ctr.host_pages -= f.n_host;
    if (c.dev && f.host_buf) {
      c.dev->sync();  // an offload copy may still be writing the buffer
      c.dev->host_free(f.host_buf);
    }
    f.host_buf = f.host_dev = nullptr;
    f.offloaded = false;
    f.n_host = 0;
  }
  f.table.clear();
  f.spos.clear();
  f.len = 0;
  f.alive = false;
  release_file_slab(c, f);
  c.names.erase(it);
  return KVFS_OK;
}

// ------------------------------------------------------------------------------------------ R3
int append_plan(const Ctx &c, const File &f, int64_t n, const int32_t *pos, int64_t *need, int64_t *new_entries) {
  const int P = c.cfg.page_size;
  const int64_t last = last_pos(c, f);
  if (pos[0] <= last) return KVFS_EPOS;
  for (int64_t i = 1; i < n; ++i)
    if (pos[i] <= pos[i - 1]) return KVFS_EPOS;
  int64_t room = 0;
  bool cow = false;
  if (!f.table.empty()) {
    const Entry &t = f.table.back();
    room = P - 1 - hi_slot(t.mask);
    cow = room > 0 && c.pool->refcnt(t.page) > 1;
  }
  const int64_t over = std::max<int64_t>(0, n - room);
  *need = (cow ? 1 : 0) + (over + P - 1) / P;
  if (new_entries) *new_entries = (over + P - 1) / P;
  if (*need > c.pool->n_free()) return KVFS_ENOSPC;
  return KVFS_OK;
}

void append_commit(Ctx &c, File &f, int64_t n, const int32_t *pos, std::vector<int32_t> *dst,
                   std::vector<PageCopy> *copies) {
  const int P = c.cfg.page_size;
  int64_t i = 0;
  size_t first_changed = f.table.size();
  if (!f.table.empty()) {
    const size_t ti = f.table.size() - 1;
    Entry &t = f.table[ti];
    const int hi = hi_slot(t.mask);
    const int room = P - 1 - hi;
    if (room > 0) {
      if (c.pool->refcnt(t.page) > 1) {  // copy-on-write of the shared tail
        const uint32_t q = c.pool->alloc();
        copies->push_back({t.page, q});
        c.pool->release(t.page);
        t.page = q;
        f.tver = next_tver();
      }
      const int take = static_cast<int>(std::min<int64_t>(n, room));
      for (int s = 0; s < take; ++s) {
        t.mask |= 1ull << (hi + 1 + s);
        f.spos[ti * P + hi + 1 + s] = pos[s];
        if (dst) dst->push_back(static_cast<int32_t>(t.page) * P + hi + 1 + s);
      }
      i = take;
      first_changed = ti;
      mark_dirty_pt(f, ti);
    }
  }
  mark_dirty_from(f, f.table.size());
  while (i < n) {
    const uint32_t q = c.pool->alloc();
    const int take = static_cast<int>(std::min<int64_t>(P, n - i));
    Entry e{q, 0, take == 64 ? ~0ull : ((1ull << take) - 1)};
    f.table.push_back(e);
    f.spos.resize(f.table.size() * P, 0);
    for (int s = 0; s < take; ++s) {
      f.spos[(f.table.size() - 1) * P + s] = pos[i + s];
      if (dst) dst->push_back(static_cast<int32_t>(q) * P + s);
    }
    i += take;
  }
  recompute_lstart(f, first_changed);
}

// ------------------------------------------------------------------------------------------ R4
int fork_file(Ctx &c, File &src, const char *dst_name, int *dst_fd, std::vector<PageCopy> *copies) {
  const int P = c.cfg.page_size;
  if (!dst_name || !*dst_name || !dst_fd) return KVFS_EINVAL;
  if (c.names.count(dst_name)) return KVFS_EEXIST;
  const bool copy_tail = !src.table.empty() && hi_slot(src.table.back().mask) < P - 1;
  if (copy_tail && c.pool->n_free() < 1) return KVFS_ENOSPC;
  auto f = std::make_shared<File>();
  f->name = dst_name;
  f->table = src.table;
  f->spos = src.spos;
  f->len = src.len;
  for (const Entry &e : f->table) c.pool->incref(e.page);
  if (copy_tail) {
    Entry &t = f->table.back();
    const uint32_t q = c.pool->alloc();
    copies->push_back({t.page, q});
    c.pool->release(t.page);  // restore the parent tail's count
    t.page = q;
  }
  c.names.emplace(f->name, f);
  *dst_fd = static_cast<int>(new_fd(c, f));
  return KVFS_OK;
}

// ------------------------------------------------------------------------------------------ R5
int truncate_file(Ctx &c, File &f, int64_t n) {
  const int P = c.cfg.page_size;
  if (n < 0 || n > f.len) return KVFS_ERANGE;
  if (n == f.len) return KVFS_OK;
  f.tver = next_tver();
  if (n == 0) {
    for (const Entry &e : f.table) c.pool->release(e.page);
    f.table.clear();
    f.spos.clear();
    f.len = 0;
    return KVFS_OK;
  }
  // entry holding logical token n-1
  size_t i = 0;
  while (f.table[i].lstart + popc(f.table[i].mask) < n) ++i;
  Entry &e = f.table[i];
  const uint64_t m = rank_range_bits(e.mask, 0, static_cast<int>(n - e.lstart));
  if (m != e.mask) {
    e.mask = m;
    mark_dirty_pt(f, i);
  }
  for (size_t j = i + 1; j < f.table.size(); ++j) c.pool->release(f.table[j].page);
  f.table.resize(i + 1);
  f.spos.resize((i + 1) * P);
  f.len = n;
  return KVFS_OK;
}

// ------------------------------------------------------------------------------------------ R6-R8
// Compacts the retained slots of a partial mask m (P slots at sp + r) to sp + w, w <= r.  Group by group:
// the group is loaded before anything is stored, and a store never reaches past the group being read.
static size_t compress_slots_scalar(int32_t *sp, size_t w, size_t r, uint64_t m, int P) {
  for (uint64_t b = m; b; b &= b - 1) sp[w++] = sp[r + static_cast<size_t>(__builtin_ctzll(b))];
  return w;
}

#if defined(__x86_64__)
__attribute__((target("avx512f"))) static size_t compress_slots_avx512(int32_t *sp, size_t w, size_t r, uint64_t m,
                                                                         int P) {
  for (int g = 0; g < P; g += 16) {
    const __mmask16 k = static_cast<__mmask16>(m >> g);
    if (!k) continue;
    const __m512i v = _mm512_loadu_si512(sp + r + g);
    _mm512_storeu_si512(sp + w, _mm512_maskz_compress_epi32(k, v));
    w += static_cast<size_t>(__builtin_popcount(k));
  }
  return w;
}
static const bool kHaveAvx512 = __builtin_cpu_supports("avx512f");
#endif

static size_t compress_slots(int32_t *sp, size_t w, size_t r, uint64_t m, int P) {
#if defined(__x86_64__)
  if (kHaveAvx512) return compress_slots_avx512(sp, w, r, m, P);
#endif
  return compress_slots_scalar(sp, w, r, m, P);
}

// R7 metadata except the positions: ceil(len/P) fresh pages (smallest free first, while the old pages are
// still held), the new table, the old entries released.  f.spos still follows `old` afterwards.
static void compact_tables(Ctx &c, File &f, std::vector<Entry> *old, std::vector<uint32_t> *np) {
  const int P = c.cfg.page_size;
  const int64_t len = f.len;
  const int64_t k = (len + P - 1) / P;
  np->resize(static_cast<size_t>(k));
  c.pool->alloc_n(k, np->data());  // old pages still held: never destinations
  const uint64_t full = P == 64 ? ~0ull : ((1ull << P) - 1);
  old->clear();
  old->swap(f.table);
  f.tver = next_tver();
  f.table.resize(static_cast<size_t>(k));
  for (int64_t j = 0; j < k; ++j) {
    const int64_t cnt = std::min<int64_t>(P, len - j * P);
    f.table[j] = {(*np)[j], static_cast<int32_t>(j * P), cnt == P ? full : ((1ull << cnt) - 1)};
  }
  for (const Entry &e : *old) c.pool->release(e.page);
  mark_dirty_from(f, 0);
}

// The positions of a compaction: token i -> slot (new[i/P], i%P), compacted in place from the layout of
// `old` (the write cursor, retained tokens before a slot, never passes the slot being read).
void compact_positions(File &f, const std::vector<Entry> &old, int P) {
  const int64_t k = (f.len + P - 1) / P;
  const uint64_t full = P == 64 ? ~0ull : ((1ull << P) - 1);
  int32_t *sp = f.spos.data();
  size_t w = 0;
  for (size_t e = 0; e < old.size(); ++e) {
    const uint64_t m = old[e].mask;
    const size_t r = e * static_cast<size_t>(P);
    if (m == full) {
      if (w != r) std::memmove(sp + w, sp + r, sizeof(int32_t) * static_cast<size_t>(P));
      w += static_cast<size_t>(P);
    } else {
      w = compress_slots(sp, w, r, m, P);
    }
  }
  f.spos.resize(static_cast<size_t>(k) * P);
  std::fill(f.spos.begin() + static_cast<std::ptrdiff_t>(w), f.spos.end(), 0);
}

static void compact_commit(Ctx &c, File &f, std::vector<Entry> *old_table, std::vector<uint32_t> *new_pages) {
  if (f.len == 0) return;
  std::vector<Entry> old;
  std::vector<uint32_t> np;
  compact_tables(c, f, &old, &np);
  compact_positions(f, old, c.cfg.page_size);
  if (old_table) old_table->swap(old);
  if (new_pages) new_pages->swap(np);
}

int evict_file(Ctx &c, File &f, const int64_t *ranges, int n_ranges, int flags, std::vector<Entry> *old_table,
               std::vector<uint32_t> *new_pages) {
  const int P = c.cfg.page_size;
  if (n_ranges < 0 || (n_ranges > 0 && !ranges)) return KVFS_EINVAL;
  for (int r = 0; r < n_ranges; ++r) {
    const int64_t a = ranges[2 * r], b = ranges[2 * r + 1];
    if (a >= b) return KVFS_EINVAL;
    if (r > 0 && a < ranges[2 * r - 1]) return KVFS_EINVAL;
    if (a < 0 || b > f.len) return KVFS_ERANGE;
  }
  // new masks of the touched entries (not yet committed)
  std::vector<std::pair<size_t, uint64_t>> touched;
  int64_t evicted = 0;
  size_t ei = 0;
  for (int r = 0; r < n_ranges; ++r) {
    const int64_t a = ranges[2 * r], b = ranges[2 * r + 1];
    evicted += b - a;
    // first entry ending after a (entry ends are non-decreasing in table order): galloping search from
    // the previous range's entry, O(log distance)
    {
      auto before = [&](size_t i) { return f.table[i].lstart + popc(f.table[i].mask) <= a; };
      size_t lo = ei, step = 1;
      while (lo + step < f.table.size() && before(lo + step)) {
        lo += step;
        step <<= 1;
      }
      const size_t hi = std::min(f.table.size(), lo + step);
      ei = static_cast<size_t>(
          std::partition_point(f.table.begin() + static_cast<std::ptrdiff_t>(lo), f.table.begin() + static_cast<std::ptrdiff_t>(hi),
                               [a](const Entry &e) { return e.lstart + popc(e.mask) <= a; }) -
          f.table.begin());
    }
    for (size_t i = ei; i < f.table.size() && f.table[i].lstart < b; ++i) {
      const int64_t ls = f.table[i].lstart;
      const int r0 = static_cast<int>(std::max<int64_t>(0, a - ls));
      const int r1 = static_cast<int>(std::min<int64_t>(popc(f.table[i].mask), b - ls));
      if (r0 >= r1) continue;
      const uint64_t clear = rank_range_bits(f.table[i].mask, r0, r1);
      if (!touched.empty() && touched.back().first == i) touched.back().second &= ~clear;
      else touched.push_back({i, f.table[i].mask & ~clear});
    }
  }
  const bool compact = (flags & KVFS_EVICT_COMPACT) != 0;
  if (compact) {
    const int64_t new_len = f.len - evicted;
    const int64_t k = (new_len + P - 1) / P;
    int64_t freed = 0;
    for (const auto &t : touched)
      if (t.second == 0 && c.pool->refcnt(f.table[t.first].page) == 1) ++freed;
    if (k > c.pool->n_free() + freed) return KVFS_ENOSPC;
  }
  if (!touched.empty()) {
    bool removed = false;
    f.tver = next_tver();
    for (const auto &t : touched) {
      f.table[t.first].mask = t.second;
      if (t.second == 0) {
        c.pool->release(f.table[t.first].page);
        removed = true;
      } else {
        mark_dirty_pt(f, t.first);
      }
    }
    if (removed) {  // drop emptied entries (and their position slots) in place
      size_t w = touched.front().first;
      for (size_t i = w; i < f.table.size(); ++i) {
        if (f.table[i].mask == 0) continue;
        if (w != i) {
          f.table[w] = f.table[i];
          std::copy(f.spos.begin() + static_cast<long>(i * P), f.spos.begin() + static_cast<long>((i + 1) * P),
                    f.spos.begin() + static_cast<long>(w * P));
        }
        ++w;
      }
      mark_dirty_from(f, touched.front().first);
      f.table.resize(w);
      f.spos.resize(w * P);
      recompute_lstart(f, touched.front().first);
    } else {
      // offsets change inside the touched span; every later entry moves down by the evicted count
      const size_t last = touched.back().first;
      recompute_lstart_span(f, touched.front().first, last + 1);
      const int32_t ev = static_cast<int32_t>(evicted);
      for (size_t i = last + 1; i < f.table.size(); ++i) f.table[i].lstart -= ev;
      f.len -= evicted;
    }
  }
  if (compact) compact_commit(c, f, old_table, new_pages);
  return KVFS_OK;
}

// R13 / R14 common tail: a new file `name` whose token i copies pool slot src[i] (page * P + slot), at
// position pos[i]; ceil(k/P) fresh pages allocated one at a time (R1), token i -> (new[i/P], i % P).
static int build_file(Ctx &c, const char *name, const std::vector<int32_t> &src, const std::vector<int32_t> &pos,
                      int *fd, std::vector<uint32_t> *new_pages) {
  const int P = c.cfg.page_size;
  if (!name || !*name || !fd) return KVFS_EINVAL;
  if (c.names.count(name)) return KVFS_EEXIST;
  const int64_t k = static_cast<int64_t>(src.size());
  const int64_t np = (k + P - 1) / P;
  if (np > c.pool->n_free()) return KVFS_ENOSPC;
  auto f = std::make_shared<File>();
  f->name = name;
  const uint64_t full = P == 64 ? ~0ull : ((1ull << P) - 1);
  new_pages->resize(static_cast<size_t>(np));
  f->table.resize(static_cast<size_t>(np));
  f->spos.assign(static_cast<size_t>(np) * P, 0);
  for (int64_t j = 0; j < np; ++j) {
    (*new_pages)[j] = c.pool->alloc();
    const int64_t cnt = std::min<int64_t>(P, k - j * P);
    f->table[j] = {(*new_pages)[j], static_cast<int32_t>(j * P), cnt == P ? full : ((1ull << cnt) - 1)};
  }
  std::copy(pos.begin(), pos.end(), f->spos.begin());
  f->len = k;
  c.names.emplace(f->name, f);
  *fd = static_cast<int>(new_fd(c, f));
  return KVFS_OK;
}

int extract_file(Ctx &c, File &src, const int64_t *idx, int64_t n, const char *name, int *fd,
                 std::vector<int32_t> *src_slots, std::vector<uint32_t> *new_pages) {
  const int P = c.cfg.page_size;
  if (n < 0 || (n > 0 && !idx)) return KVFS_EINVAL;
  for (int64_t i = 1; i < n; ++i)
    if (idx[i] <= idx[i - 1]) return KVFS_EINVAL;
  if (n > 0 && (idx[0] < 0 || idx[n - 1] >= src.len)) return KVFS_ERANGE;
  std::vector<int32_t> pos(static_cast<size_t>(n));
  src_slots->resize(static_cast<size_t>(n));
  // walk the table once: logical index -> (entry, slot)
  size_t e = 0;
  for (int64_t i = 0; i < n; ++i) {
    while (src.table[e].lstart + popc(src.table[e].mask) <= idx[i]) ++e;
    const int slot = select_bit(src.table[e].mask, static_cast<int>(idx[i] - src.table[e].lstart));
    (*src_slots)[i] = static_cast<int32_t>(src.table[e].page) * P + slot;
    pos[i] = src.spos[e * P + slot];
  }
  return build_file(c, name, *src_slots, pos, fd, new_pages);
}

int merge_files(Ctx &c, const int *fds, int n, const char *name, int *fd, std::vector<int32_t> *src_slots,
                std::vector<uint32_t> *new_pages) {
  const int P = c.cfg.page_size;
  if (n < 0 || (n > 0 && !fds)) return KVFS_EINVAL;
  std::vector<File *> parts;
  for (int i = 0; i < n; ++i) {
    File *f = get_file(c, fds[i]);
    if (!f) return KVFS_EBADF;
    if (f->offloaded) return KVFS_EOFFLOAD;
    parts.push_back(f);
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j)
      if (parts[i] == parts[j]) return KVFS_EBUSY;
  std::vector<std::pair<int32_t, int32_t>> toks;  // (position, pool slot)
  for (File *f : parts)
    for (size_t e = 0; e < f->table.size(); ++e)
      for (uint64_t m = f->table[e].mask; m; m &= m - 1) {
        const int slot = __builtin_ctzll(m);
        toks.emplace_back(f->spos[e * P + slot], static_cast<int32_t>(f->table[e].page) * P + slot);
      }
  std::stable_sort(toks.begin(), toks.end(),
                   [](const std::pair<int32_t, int32_t> &a, const std::pair<int32_t, int32_t> &b) {
                     return a.first < b.first;
                   });
  for (size_t i = 1; i < toks.size(); ++i)
    if (toks[i].first == toks[i - 1].first) return KVFS_EPOS;
  std::vector<int32_t> pos(toks.size());
  src_slots->resize(toks.size());
  for (size_t i = 0; i < toks.size(); ++i) {
    pos[i] = toks[i].first;
    (*src_slots)[i] = toks[i].second;
  }
  return build_file(c, name, *src_slots, pos, fd, new_pages);
}

int offload_file(Ctx &c, File &f, std::vector<uint32_t> *pages) {
  if (f.offloaded) return KVFS_EINVAL;
  pages->clear();
  f.tver = next_tver();
  for (Entry &e : f.table) {
    if (c.pool->refcnt(e.page) != 1) continue;
    pages->push_back(e.page);
    c.pool->release(e.page);
    e.page = KVFS_HOST_PAGE | static_cast<uint32_t>(pages->size() - 1);
  }
  f.offloaded = true;
  f.n_host = static_cast<int64_t>(pages->size());
  c.ctr.host_pages += f.n_host;
  mark_dirty_from(f, 0);
  return KVFS_OK;
}

int restore_file(Ctx &c, File &f, std::vector<uint32_t> *new_pages) {
  if (!f.offloaded) return KVFS_EINVAL;
  if (f.n_host > c.pool->n_free()) return KVFS_ENOSPC;
  new_pages->assign(static_cast<size_t>(f.n_host), 0u);
  f.tver = next_tver();
  for (Entry &e : f.table) {
    if (!(e.page & KVFS_HOST_PAGE)) continue;
    const uint32_t slot = e.page & ~KVFS_HOST_PAGE;
    const uint32_t q = c.pool->alloc();
    (*new_pages)[slot] = q;
    e.page = q;
  }
  c.ctr.host_pages -= f.n_host;
  f.offloaded = false;
  f.n_host = 0;
  mark_dirty_from(f, 0);
  return KVFS_OK;
}

int compact_file(Ctx &c, File &f, std::vector<Entry> *old_table, std::vector<uint32_t> *new_pages) {
  const int P = c.cfg.page_size;
  if (f.len == 0) return KVFS_OK;
  if ((f.len + P - 1) / P > c.pool->n_free()) return KVFS_ENOSPC;
  compact_commit(c, f, old_table, new_pages);
  return KVFS_OK;
}

int compact_file_tables(Ctx &c, File &f, std::vector<Entry> *old_table, std::vector<uint32_t> *new_pages) {
  const int P = c.cfg.page_size;
  old_table->clear();
  new_pages->clear();
  if (f.len == 0) return KVFS_OK;
  if ((f.len + P - 1) / P > c.pool->n_free()) return KVFS_ENOSPC;
  compact_tables(c, f, old_table, new_pages);
  return KVFS_OK;
}

// ------------------------------------------------------------------------------------------ audit
int audit(Ctx &c) {
  const int P = c.cfg.page_size;
  const uint64_t lim = P == 64 ? ~0ull : ((1ull << P) - 1);
  std::vector<uint32_t> cnt(static_cast<size_t>(c.pool->n_pages()), 0u);
  for (const auto &kv : c.names) {
    const File &f = *kv.second;
    std::vector<uint32_t> pages;
    int64_t acc = 0;
    for (const Entry &e : f.table) {
      if (e.mask == 0 || (e.mask & ~lim)) return KVFS_EINVAL;  // I1
      if (e.lstart != acc) return KVFS_EINVAL;
      acc += popc(e.mask);
      pages.push_back(e.page);
      if (e.page & KVFS_HOST_PAGE) {
        if (!f.offloaded || static_cast<int64_t>(e.page & ~KVFS_HOST_PAGE) >= f.n_host) return KVFS_EINVAL;
        continue;
      }
      if (e.page >= static_cast<uint32_t>(c.pool->n_pages())) return KVFS_EINVAL;
      ++cnt[e.page];
    }
    std::sort(pages.begin(), pages.end());
    if (std::adjacent_find(pages.begin(), pages.end()) != pages.end()) return KVFS_EINVAL;  // I2
    if (acc != f.len || f.spos.size() != f.table.size() * static_cast<size_t>(P)) return KVFS_EINVAL;
    std::vector<int32_t> lp;
    file_positions(c, f, &lp);
    for (size_t i = 1; i < lp.size(); ++i)
      if (lp[i] <= lp[i - 1]) return KVFS_EINVAL;  // I4
  }
  int64_t n_free = 0;
  for (int64_t p = 0; p < c.pool->n_pages(); ++p) {
    if (cnt[p] != c.pool->refcnt(static_cast<uint32_t>(p))) return KVFS_EINVAL;  // I3
    if (cnt[p] == 0) ++n_free;
  }
  if (n_free != c.pool->n_free()) return KVFS_EINVAL;
  if (c.names.empty() && n_free != c.pool->n_pages()) return KVFS_EINVAL;  // I5
  return KVFS_OK;
}

}  // namespace kvfs
