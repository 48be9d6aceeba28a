// KV-file migration between contexts: pack a file set into (distinct pages, header) and
// rebuild it in another ctx.  Host metadata only; the page gather / scatter is the device's (K6).
#include <algorithm>
#include <cstring>
#include <map>
#include <set>
#include <string>

#include "kvfs_impl.h"

namespace kvfs {

namespace {

constexpr uint32_t kMagic = 0x3150564Bu;  // "KVP1" little-endian

template <class T>
void put(std::vector<uint8_t> *b, T v) {
  const size_t o = b->size();
  b->resize(o + sizeof(T));
  std::memcpy(b->data() + o, &v, sizeof(T));
}

struct Reader {
  const uint8_t *p;
  size_t n, off = 0;
  template <class T>
  bool get(T *v) {
    if (off + sizeof(T) > n) return false;
    std::memcpy(v, p + off, sizeof(T));
    off += sizeof(T);
    return true;
  }
};

}  // namespace

int pack_files(Ctx &c, const int *fds, int n, std::vector<uint32_t> *pages, std::vector<uint8_t> *hdr) {
  if (n < 0 || (n > 0 && !fds)) return KVFS_EINVAL;
  std::vector<File *> files;
  std::set<File *> seen;
  for (int i = 0; i < n; ++i) {
    File *f = get_file(c, fds[i]);
    if (!f) return KVFS_EBADF;
    if (f->offloaded) return KVFS_EOFFLOAD;
    if (!seen.insert(f).second) return KVFS_EBUSY;
    files.push_back(f);
  }
  // distinct pages of the set, ascending source page id (vector sort + unique; O(pages log pages))
  pages->clear();
  for (File *f : files)
    for (const Entry &e : f->table) pages->push_back(e.page);
  std::sort(pages->begin(), pages->end());
  pages->erase(std::unique(pages->begin(), pages->end()), pages->end());
  std::vector<uint32_t> local(static_cast<size_t>(c.pool->n_pages()), 0u);
  for (size_t j = 0; j < pages->size(); ++j) local[(*pages)[j]] = static_cast<uint32_t>(j);
  const kvfs_config &cfg = c.cfg;
  // header size first, then one pass of bulk writes
  size_t bytes = 8 * 4 + 8;
  for (File *f : files) bytes += 8 + f->table.size() * 16 + static_cast<size_t>(f->len) * 4;
  hdr->clear();
  hdr->reserve(bytes);
  put<uint32_t>(hdr, kMagic);
  put<uint32_t>(hdr, 1);
  put<uint32_t>(hdr, static_cast<uint32_t>(n));
  put<uint32_t>(hdr, static_cast<uint32_t>(pages->size()));
  put<uint32_t>(hdr, static_cast<uint32_t>(cfg.page_size));
  put<uint32_t>(hdr, static_cast<uint32_t>(cfg.n_layers));
  put<uint32_t>(hdr, static_cast<uint32_t>(cfg.n_kv_heads));
  put<uint32_t>(hdr, static_cast<uint32_t>(cfg.head_dim));
  put<uint64_t>(hdr, static_cast<uint64_t>(cfg.n_kv_heads) * cfg.page_size * cfg.head_dim * 2);
  std::vector<int32_t> lp;
  std::vector<uint8_t> ent;
  for (File *f : files) {
    file_positions(c, *f, &lp);
    put<uint32_t>(hdr, static_cast<uint32_t>(f->table.size()));
    put<uint32_t>(hdr, static_cast<uint32_t>(lp.size()));
    ent.resize(f->table.size() * 16);
    for (size_t e = 0; e < f->table.size(); ++e) {
      const uint32_t loc = local[f->table[e].page], pad = 0;
      std::memcpy(ent.data() + e * 16, &loc, 4);
      std::memcpy(ent.data() + e * 16 + 4, &pad, 4);
      std::memcpy(ent.data() + e * 16 + 8, &f->table[e].mask, 8);
    }
    hdr->insert(hdr->end(), ent.begin(), ent.end());
    const uint8_t *pb = reinterpret_cast<const uint8_t *>(lp.data());
    hdr->insert(hdr->end(), pb, pb + lp.size() * 4);
  }
  return KVFS_OK;
}

int unpack_files(Ctx &c, const void *hdr_v, size_t hdr_bytes, const char *const *names, int *fds_out,
                 std::vector<uint32_t> *new_pages) {
  if (!hdr_v || !fds_out) return KVFS_EINVAL;
  const kvfs_config &cfg = c.cfg;
  const int P = cfg.page_size;
  const uint64_t lim = P == 64 ? ~0ull : ((1ull << P) - 1);
  Reader r{static_cast<const uint8_t *>(hdr_v), hdr_bytes};
  uint32_t magic, ver, n, nu, hp, hl, hh, hd;
  uint64_t pb;
  if (!r.get(&magic) || !r.get(&ver) || !r.get(&n) || !r.get(&nu) || !r.get(&hp) || !r.get(&hl) || !r.get(&hh) ||
      !r.get(&hd) || !r.get(&pb))
    return KVFS_EINVAL;
  if (magic != kMagic || ver != 1 || hp != static_cast<uint32_t>(P) || hl != static_cast<uint32_t>(cfg.n_layers) ||
      hh != static_cast<uint32_t>(cfg.n_kv_heads) || hd != static_cast<uint32_t>(cfg.head_dim))
    return KVFS_EINVAL;
  if (n > 0 && !names) return KVFS_EINVAL;
  // parse + validate everything before changing any state (atomic failure)
  struct Parsed {
    std::vector<std::pair<uint32_t, uint64_t>> ent;
    std::vector<int32_t> pos;
  };
  std::vector<Parsed> files(n);
  std::set<std::string> nm;
  for (uint32_t i = 0; i < n; ++i) {
    if (!names[i] || !*names[i]) return KVFS_EINVAL;
    if (c.names.count(names[i]) || !nm.insert(names[i]).second) return KVFS_EEXIST;
    uint32_t ne, nt;
    if (!r.get(&ne) || !r.get(&nt)) return KVFS_EINVAL;
    uint64_t total = 0;
    for (uint32_t e = 0; e < ne; ++e) {
      uint32_t loc, pad;
      uint64_t mask;
      if (!r.get(&loc) || !r.get(&pad) || !r.get(&mask)) return KVFS_EINVAL;
      if (loc >= nu || mask == 0 || (mask & ~lim)) return KVFS_EINVAL;
      files[i].ent.push_back({loc, mask});
      total += static_cast<uint64_t>(__builtin_popcountll(mask));
    }
    if (total != nt) return KVFS_EINVAL;
    files[i].pos.resize(nt);
    for (uint32_t t = 0; t < nt; ++t)
      if (!r.get(&files[i].pos[t])) return KVFS_EINVAL;
    for (uint32_t t = 1; t < nt; ++t)
      if (files[i].pos[t] <= files[i].pos[t - 1]) return KVFS_EINVAL;
  }
  if (static_cast<int64_t>(nu) > c.pool->n_free()) return KVFS_ENOSPC;
  // allocate in packed order (R1), then build the files
  new_pages->resize(nu);
  for (uint32_t j = 0; j < nu; ++j) (*new_pages)[j] = c.pool->alloc();
  std::vector<uint32_t> refs(nu, 0);
  for (uint32_t i = 0; i < n; ++i)
    for (const auto &e : files[i].ent) ++refs[e.first];
  for (uint32_t j = 0; j < nu; ++j) {
    if (refs[j] == 0) {
      c.pool->release((*new_pages)[j]);  // never referenced (cannot happen for a well-formed pack)
      continue;
    }
    for (uint32_t k = 1; k < refs[j]; ++k) c.pool->incref((*new_pages)[j]);
  }
  for (uint32_t i = 0; i < n; ++i) {
    int fd = -1;
    open_file(c, names[i], KVFS_O_CREAT | KVFS_O_EXCL, &fd);
    File &f = *c.fds[fd];
    f.spos.assign(files[i].ent.size() * P, 0);
    size_t t = 0;
    for (size_t e = 0; e < files[i].ent.size(); ++e) {
      const uint64_t m = files[i].ent[e].second;
      f.table.push_back({(*new_pages)[files[i].ent[e].first], 0, m});
      for (uint64_t mm = m; mm; mm &= mm - 1) f.spos[e * P + __builtin_ctzll(mm)] = files[i].pos[t++];
    }
    recompute_lstart(f, 0);
    fds_out[i] = fd;
  }
  return KVFS_OK;
}

}  // namespace kvfs
