// KVFS file operations (§4.2) on host metadata.  Each function validates first and
// mutates only after every check passed (atomic failure).  Rule numbers refer to
// SURVEY.md §8(c) C3 (restated in DESIGN.md "Readings").
#include <algorithm>
#include <cstring>

#include "kvfs_impl.h"

namespace kvfs {

namespace {

inline int popc(uint64_t m) { return __builtin_popcountll(m); }
inline int hi_slot(uint64_t m) { return 63 - __builtin_clzll(m); }  // m != 0

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

void mark_dirty(File &f, size_t i) { f.dirty_from = std::min(f.dirty_from, i); }

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
  for (const Entry &e : f.table) c.pool->release(e.page);
  f.table.clear();
  f.pos.clear();
  f.len = 0;
  f.alive = false;
  release_file_slab(c, f);
  c.names.erase(it);
  return KVFS_OK;
}

// ------------------------------------------------------------------------------------------ R3
int append_plan(const Ctx &c, const File &f, int64_t n, const int32_t *pos, int64_t *need, int64_t *new_entries) {
  const int P = c.cfg.page_size;
  int64_t last = f.pos.empty() ? -1 : f.pos.back();
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
    Entry &t = f.table.back();
    const int hi = hi_slot(t.mask);
    const int room = P - 1 - hi;
    if (room > 0) {
      if (c.pool->refcnt(t.page) > 1) {  // copy-on-write of the shared tail
        const uint32_t q = c.pool->alloc();
        copies->push_back({t.page, q});
        c.pool->release(t.page);
        t.page = q;
      }
      const int take = static_cast<int>(std::min<int64_t>(n, room));
      for (int s = 0; s < take; ++s) {
        t.mask |= 1ull << (hi + 1 + s);
        if (dst) dst->push_back(static_cast<int32_t>(t.page) * P + hi + 1 + s);
      }
      i = take;
      first_changed = f.table.size() - 1;
    }
  }
  while (i < n) {
    const uint32_t q = c.pool->alloc();
    const int take = static_cast<int>(std::min<int64_t>(P, n - i));
    Entry e{q, 0, take == 64 ? ~0ull : ((1ull << take) - 1)};
    f.table.push_back(e);
    if (dst)
      for (int s = 0; s < take; ++s) dst->push_back(static_cast<int32_t>(q) * P + s);
    i += take;
  }
  f.pos.insert(f.pos.end(), pos, pos + n);
  mark_dirty(f, first_changed);
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
  f->pos = src.pos;
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
  if (n < 0 || n > f.len) return KVFS_ERANGE;
  if (n == f.len) return KVFS_OK;
  if (n == 0) {
    for (const Entry &e : f.table) c.pool->release(e.page);
    f.table.clear();
    f.pos.clear();
    f.len = 0;
    f.dirty_from = 0;
    return KVFS_OK;
  }
  // entry holding logical token n-1
  size_t i = 0;
  while (f.table[i].lstart + popc(f.table[i].mask) < n) ++i;
  Entry &e = f.table[i];
  e.mask = rank_range_bits(e.mask, 0, static_cast<int>(n - e.lstart));
  for (size_t j = i + 1; j < f.table.size(); ++j) c.pool->release(f.table[j].page);
  f.table.resize(i + 1);
  f.pos.resize(static_cast<size_t>(n));
  f.len = n;
  mark_dirty(f, i);
  return KVFS_OK;
}

// ------------------------------------------------------------------------------------------ R6-R8
static void compact_commit(Ctx &c, File &f, std::vector<Entry> *old_table, std::vector<uint32_t> *new_pages) {
  const int P = c.cfg.page_size;
  const int64_t len = f.len;
  if (len == 0) return;
  const int64_t k = (len + P - 1) / P;
  std::vector<uint32_t> np(static_cast<size_t>(k));
  for (int64_t j = 0; j < k; ++j) np[j] = c.pool->alloc();  // old pages still held: never destinations
  std::vector<Entry> old;
  old.swap(f.table);
  const uint64_t full = P == 64 ? ~0ull : ((1ull << P) - 1);
  f.table.reserve(static_cast<size_t>(k));
  for (int64_t j = 0; j < k; ++j) {
    const int64_t cnt = std::min<int64_t>(P, len - j * P);
    f.table.push_back({np[j], static_cast<int32_t>(j * P), cnt == 64 ? ~0ull : (cnt == P ? full : ((1ull << cnt) - 1))});
  }
  for (const Entry &e : old) c.pool->release(e.page);
  f.dirty_from = 0;
  recompute_lstart(f, 0);
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
  // new masks (not yet committed)
  std::vector<uint64_t> masks(f.table.size());
  for (size_t i = 0; i < f.table.size(); ++i) masks[i] = f.table[i].mask;
  size_t first_changed = f.table.size();
  int64_t evicted = 0;
  size_t ei = 0;
  for (int r = 0; r < n_ranges; ++r) {
    const int64_t a = ranges[2 * r], b = ranges[2 * r + 1];
    evicted += b - a;
    while (ei < f.table.size() && f.table[ei].lstart + popc(f.table[ei].mask) <= a) ++ei;
    for (size_t i = ei; i < f.table.size() && f.table[i].lstart < b; ++i) {
      const int64_t ls = f.table[i].lstart;
      const int r0 = static_cast<int>(std::max<int64_t>(0, a - ls));
      const int r1 = static_cast<int>(std::min<int64_t>(popc(f.table[i].mask), b - ls));
      if (r0 < r1) {
        masks[i] &= ~rank_range_bits(f.table[i].mask, r0, r1);
        first_changed = std::min(first_changed, i);
      }
    }
  }
  const bool compact = (flags & KVFS_EVICT_COMPACT) != 0;
  if (compact) {
    const int64_t new_len = f.len - evicted;
    const int64_t k = (new_len + P - 1) / P;
    int64_t freed = 0;
    for (size_t i = 0; i < masks.size(); ++i)
      if (masks[i] == 0 && c.pool->refcnt(f.table[i].page) == 1) ++freed;
    if (k > c.pool->n_free() + freed) return KVFS_ENOSPC;
  }
  if (n_ranges > 0) {
    // positions: drop the evicted logical indices
    std::vector<int32_t> np;
    np.reserve(static_cast<size_t>(f.len - evicted));
    int64_t idx = 0;
    for (int r = 0; r < n_ranges; ++r) {
      for (; idx < ranges[2 * r]; ++idx) np.push_back(f.pos[idx]);
      idx = ranges[2 * r + 1];
    }
    for (; idx < f.len; ++idx) np.push_back(f.pos[idx]);
    f.pos.swap(np);
    std::vector<Entry> nt;
    nt.reserve(f.table.size());
    for (size_t i = 0; i < f.table.size(); ++i) {
      if (masks[i]) {
        Entry e = f.table[i];
        e.mask = masks[i];
        nt.push_back(e);
      } else {
        c.pool->release(f.table[i].page);
      }
    }
    f.table.swap(nt);
    mark_dirty(f, first_changed);
    recompute_lstart(f, first_changed);
  }
  if (compact) compact_commit(c, f, old_table, new_pages);
  return KVFS_OK;
}

int compact_file(Ctx &c, File &f, std::vector<Entry> *old_table, std::vector<uint32_t> *new_pages) {
  const int P = c.cfg.page_size;
  if (f.len == 0) return KVFS_OK;
  if ((f.len + P - 1) / P > c.pool->n_free()) return KVFS_ENOSPC;
  compact_commit(c, f, old_table, new_pages);
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
      ++cnt[e.page];
    }
    std::sort(pages.begin(), pages.end());
    if (std::adjacent_find(pages.begin(), pages.end()) != pages.end()) return KVFS_EINVAL;  // I2
    if (acc != f.len || static_cast<int64_t>(f.pos.size()) != f.len) return KVFS_EINVAL;
    for (size_t i = 1; i < f.pos.size(); ++i)
      if (f.pos[i] <= f.pos[i - 1]) return KVFS_EINVAL;  // I4
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
