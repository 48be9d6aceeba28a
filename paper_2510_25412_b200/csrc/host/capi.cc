// extern "C" shims of include/kvfs.h: argument validation, the ctx mutex, error mapping, and the split
// between host metadata (this directory) and the device data plane (csrc/cuda).
#include <cstring>
#include <memory>
#include <new>

#include <thread>
#include <atomic>
#include <algorithm>
#include <chrono>
#include "kvfs_impl.h"

#ifndef KVFS_SCORE_UNIT_ENTRIES
#define KVFS_SCORE_UNIT_ENTRIES 32  // page entries per K9 CTA (<= 32: the kernel's accumulator rows)
#endif

using namespace kvfs;

namespace {

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

bool supported_shape(const kvfs_config &c) {
  if (c.n_layers < 1 || c.n_layers > 1024) return false;
  if (c.n_kv_heads < 1 || c.n_q_heads < c.n_kv_heads || c.n_q_heads % c.n_kv_heads) return false;
  const int G = c.n_q_heads / c.n_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8) return false;
  if (c.head_dim != 64 && c.head_dim != 128) return false;
  if (c.page_size != 16 && c.page_size != 32 && c.page_size != 64) return false;
  if (c.n_pages < 1 || c.n_pages >= (int64_t{1} << 25)) return false;
  if (static_cast<int64_t>(c.n_pages) * c.page_size >= (int64_t{1} << 31)) return false;
  if (c.max_batch_rows < 1 || c.max_batch_descs < 1) return false;
  return true;
}

int64_t default_table_capacity(const kvfs_config &c) {
  return c.table_capacity > 0 ? c.table_capacity : 2 * c.n_pages + 65536;
}

struct Lock {
  explicit Lock(kvfs_ctx *ctx) : c(reinterpret_cast<Ctx *>(ctx)), g(c->mu) {}
  Ctx *c;
  std::lock_guard<std::mutex> g;
};

// include/kvfs.h promises that no call throws across the C ABI.  Every extern "C" body runs inside this
// guard: a C++ exception (std::bad_alloc from a table / position / plan vector, std::system_error from a
// worker thread) becomes KVFS_ENOMEM / KVFS_EIO, and the ctx is marked broken, because the call may have
// been half-applied (its metadata can no longer be trusted); a broken ctx answers KVFS_EIO to every call
// but kvfs_destroy.
template <class F>
int guarded(kvfs_ctx *ctx, F &&f) noexcept {
  try {
    return f();
  } catch (const std::bad_alloc &) {
    if (ctx) reinterpret_cast<Ctx *>(ctx)->broken.store(true);
    return KVFS_ENOMEM;
  } catch (...) {
    if (ctx) reinterpret_cast<Ctx *>(ctx)->broken.store(true);
    return KVFS_EIO;
  }
}

}  // namespace

struct kvfs_ctx {};  // opaque; the real object is kvfs::Ctx
struct pred_step {};

extern "C" {

const char *kvfs_strerror(int err) {
  switch (err) {
    case KVFS_OK: return "ok";
    case KVFS_ENOENT: return "no such file";
    case KVFS_EIO: return "CUDA error (ctx poisoned)";
    case KVFS_EBADF: return "bad file descriptor";
    case KVFS_ENOMEM: return "out of memory (host, table slab or workspace)";
    case KVFS_EBUSY: return "busy (file repeated in a batch, or a pred step is open)";
    case KVFS_EEXIST: return "file exists";
    case KVFS_EINVAL: return "invalid argument";
    case KVFS_ENOSPC: return "page pool exhausted";
    case KVFS_ERANGE: return "out of range";
    case KVFS_ENOSYS: return "data operation on a host-only ctx";
    case KVFS_EPOS: return "position conflict";
    case KVFS_EPARTIAL: return "some batch descriptors failed";
    case KVFS_EOFFLOAD: return "file is offloaded to the host tier (restore it first)";
    default: return "unknown error";
  }
}

size_t kvfs_workspace_bytes(const kvfs_config *cfg) {
  try {
    if (!cfg || !supported_shape(*cfg) || cfg->device < 0) return 0;
    kvfs_config c = *cfg;
    c.table_capacity = default_table_capacity(c);
    return device_workspace_bytes(c);
  } catch (...) {
    return 0;
  }
}

int kvfs_init(const kvfs_config *cfg, kvfs_ctx **out) {
  return guarded(nullptr, [&]() -> int {
    if (!cfg || !out || !supported_shape(*cfg)) return KVFS_EINVAL;
    std::unique_ptr<Ctx> c(new Ctx());  // freed if anything below fails or throws
    c->cfg = *cfg;
    c->cfg.table_capacity = default_table_capacity(*cfg);
    c->pool.reset(new PagePool(cfg->n_pages));
    c->slab.init(c->cfg.table_capacity);
    if (cfg->device >= 0) {
      if (!cfg->k_pool || !cfg->v_pool || !cfg->workspace) return KVFS_EINVAL;
      for (int l = 0; l < cfg->n_layers; ++l) {
        if (!cfg->k_pool[l] || !cfg->v_pool[l]) return KVFS_EINVAL;
        c->kpool.push_back(cfg->k_pool[l]);
        c->vpool.push_back(cfg->v_pool[l]);
      }
      c->cfg.k_pool = c->kpool.data();
      c->cfg.v_pool = c->vpool.data();
      if (cfg->workspace_bytes < device_workspace_bytes(c->cfg)) return KVFS_ENOMEM;
      Device *d = nullptr;
      const int rc = create_device(*c, &d);
      if (rc != KVFS_OK) return rc;
      c->dev = d;
    } else {
      c->cfg.k_pool = nullptr;
      c->cfg.v_pool = nullptr;
    }
    *out = reinterpret_cast<kvfs_ctx *>(c.release());
    return KVFS_OK;
  });
}

int kvfs_destroy(kvfs_ctx *ctx) {
  return guarded(ctx, [&]() -> int {
    if (!ctx) return KVFS_EINVAL;
    Ctx *c = reinterpret_cast<Ctx *>(ctx);
    if (c->dev) {
      c->dev->sync();
      for (auto &kv : c->names)
        if (kv.second->host_buf) c->dev->host_free(kv.second->host_buf);
      delete c->dev;
    }
    delete c;
    return KVFS_OK;
  });
}

#define KVFS_LOCK_OR(ctx)                       \
  if (!(ctx)) return KVFS_EINVAL;               \
  Lock lk_(ctx);                                \
  Ctx &c = *lk_.c;                              \
  if (c.broken) return KVFS_EIO;                \
  if (c.step_open) return KVFS_EBUSY;

int kvfs_open(kvfs_ctx *ctx, const char *name, int flags, int *fd) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    fault_point(c);
    return open_file(c, name, flags, fd);
  });
}

int kvfs_close(kvfs_ctx *ctx, int fd) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    return close_file(c, fd);
  });
}

int kvfs_unlink(kvfs_ctx *ctx, const char *name) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    return unlink_file(c, name);
  });
}

int kvfs_fork(kvfs_ctx *ctx, int src_fd, const char *dst_name, int *dst_fd, kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (c.dev && c.poisoned) return KVFS_EIO;
    File *src = get_file(c, src_fd);
    if (!src) return KVFS_EBADF;
    if (src->offloaded) return KVFS_EOFFLOAD;
    std::vector<PageCopy> copies;
    fault_point(c);
    int rc = fork_file(c, *src, dst_name, dst_fd, &copies);
    if (rc != KVFS_OK) return rc;
    c.ctr.page_copies += static_cast<int64_t>(copies.size());
    if (c.dev && !copies.empty()) {
      rc = c.dev->copy_pages(copies, stream);
      if (rc != KVFS_OK) c.poisoned = true;
    }
    return rc;
  });
}

int kvfs_truncate(kvfs_ctx *ctx, int fd, int64_t new_len) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    File *f = get_file(c, fd);
    if (!f) return KVFS_EBADF;
    if (f->offloaded) return KVFS_EOFFLOAD;
    return truncate_file(c, *f, new_len);
  });
}

int kvfs_evict(kvfs_ctx *ctx, int fd, const int64_t *ranges, int n_ranges, int flags, kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (c.dev && c.poisoned) return KVFS_EIO;
    File *f = get_file(c, fd);
    if (!f) return KVFS_EBADF;
    if (f->offloaded) return KVFS_EOFFLOAD;
    if (flags & ~KVFS_EVICT_COMPACT) return KVFS_EINVAL;
    std::vector<Entry> old_table;
    std::vector<uint32_t> new_pages;
    int rc = evict_file(c, *f, ranges, n_ranges, flags, &old_table, &new_pages);
    if (rc != KVFS_OK) return rc;
    if (c.dev && !new_pages.empty()) {
      rc = c.dev->compact({CompactJob{&old_table, &new_pages, f->len}}, stream);
      if (rc != KVFS_OK) c.poisoned = true;
    }
    return rc;
  });
}

int kvfs_compact(kvfs_ctx *ctx, int fd, kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (c.dev && c.poisoned) return KVFS_EIO;
    File *f = get_file(c, fd);
    if (!f) return KVFS_EBADF;
    if (f->offloaded) return KVFS_EOFFLOAD;
    std::vector<Entry> old_table;
    std::vector<uint32_t> new_pages;
    int rc = compact_file(c, *f, &old_table, &new_pages);
    if (rc != KVFS_OK) return rc;
    if (c.dev && !new_pages.empty()) {
      rc = c.dev->compact({CompactJob{&old_table, &new_pages, f->len}}, stream);
      if (rc != KVFS_OK) c.poisoned = true;
    }
    return rc;
  });
}

int kvfs_compact_files(kvfs_ctx *ctx, const int *fds, int n, int *n_done, kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (n_done) *n_done = 0;
    if (n < 0 || (n > 0 && !fds)) return KVFS_EINVAL;
    if (c.dev && c.poisoned) return KVFS_EIO;
    std::vector<File *> files(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      File *f = get_file(c, fds[i]);
      if (!f) return KVFS_EBADF;
      if (f->offloaded) return KVFS_EOFFLOAD;
      files[i] = f;
    }
    {  // one file twice would race its deferred position pass
      std::vector<File *> u(files);
      std::sort(u.begin(), u.end());
      if (std::adjacent_find(u.begin(), u.end()) != u.end()) return KVFS_EBUSY;
    }
    std::vector<std::vector<Entry>> olds(static_cast<size_t>(n));
    std::vector<std::vector<uint32_t>> nps(static_cast<size_t>(n));
    int rc = KVFS_OK, done = 0;
    // Pages and tables in order (R1: each file's allocation sees the previous files' releases); the device
    // gathers are handed to the data plane in groups of files as the host goes, so the host table work of
    // the next group overlaps the GPU copying this one.  Inside a group the data plane chains the files
    // (a file's destinations may be the previous file's sources); consecutive groups are stream-ordered.
    constexpr int kGroup = 8;
    std::vector<CompactJob> jobs;
    auto flush = [&]() {
      if (jobs.empty() || !c.dev || rc == KVFS_EIO) return;
      const int drc = c.dev->compact(jobs, stream);
      jobs.clear();
      if (drc != KVFS_OK) {
        c.poisoned = true;
        rc = drc;
      }
    };
    for (int i = 0; i < n; ++i) {
      const int trc = compact_file_tables(c, *files[i], &olds[i], &nps[i]);
      if (trc != KVFS_OK) {
        rc = trc;
        break;
      }
      ++done;
      if (!nps[i].empty()) jobs.push_back({&olds[i], &nps[i], files[i]->len});
      if (static_cast<int>(jobs.size()) == kGroup) flush();
      if (rc != KVFS_OK) break;
    }
    {
      const int keep = rc;
      flush();  // the committed files' gathers (also after an ENOSPC stop)
      if (rc == KVFS_OK) rc = keep;
    }
    const int P = c.cfg.page_size;
    // Position passes: independent per file, on worker threads; a thread that cannot be started (resource
    // limits: std::system_error) leaves its share to the others and to this thread, so the tables that are
    // already committed (and the K5 gathers already enqueued) always get their positions.
    std::atomic<int> next{0};
    auto work = [&]() {
      for (int i = next++; i < done; i = next++)
        if (!olds[i].empty()) compact_positions(*files[i], olds[i], P);
    };
    const int nt = done < 4 ? 1 : static_cast<int>(std::min<unsigned>(8u, std::max(1u, std::thread::hardware_concurrency())));
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) {
      try {
        pool.emplace_back(work);
      } catch (...) {
        break;
      }
    }
    work();
    for (auto &t : pool) t.join();
    if (n_done) *n_done = done;
    if (c.dev && c.opt_timing) c.last_compact_device_ns = c.dev->take_device_ns();
    return rc;
  });
}

int kvfs_extract(kvfs_ctx *ctx, int src_fd, const int64_t *indices, int64_t n, const char *name, int *fd,
                 kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (c.dev && c.poisoned) return KVFS_EIO;
    File *f = get_file(c, src_fd);
    if (!f) return KVFS_EBADF;
    if (f->offloaded) return KVFS_EOFFLOAD;
    std::vector<int32_t> src;
    std::vector<uint32_t> pages;
    int rc = extract_file(c, *f, indices, n, name, fd, &src, &pages);
    if (rc != KVFS_OK) return rc;
    if (c.dev && !src.empty()) {
      rc = c.dev->gather(src, pages, stream);
      if (rc != KVFS_OK) c.poisoned = true;
    }
    return rc;
  });
}

int kvfs_offload(kvfs_ctx *ctx, int fd, int64_t *moved, kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (c.dev && c.poisoned) return KVFS_EIO;
    File *f = get_file(c, fd);
    if (!f) return KVFS_EBADF;
    if (f->offloaded) return KVFS_EINVAL;
    // host buffer first (nothing changes if it cannot be had)
    int64_t n_ex = 0;
    for (const Entry &e : f->table) n_ex += c.pool->refcnt(e.page) == 1;
    const size_t page_bytes = static_cast<size_t>(c.cfg.n_kv_heads) * c.cfg.page_size * c.cfg.head_dim * 2;
    void *hb = nullptr, *hd = nullptr;
    if (c.dev && n_ex > 0) {
      const int rc = c.dev->host_alloc(static_cast<size_t>(n_ex) * c.cfg.n_layers * 2 * page_bytes, &hb, &hd);
      if (rc != KVFS_OK) return rc;
    }
    std::vector<uint32_t> pages;
    int rc = offload_file(c, *f, &pages);
    if (rc != KVFS_OK) {
      if (hb) c.dev->host_free(hb);
      return rc;
    }
    f->host_buf = hb;
    f->host_dev = hd;
    if (moved) *moved = static_cast<int64_t>(pages.size());
    if (c.dev && !pages.empty()) {
      rc = c.dev->pack_pages(pages, hd, stream);  // device pages -> host tier (mapped pinned memory)
      if (rc != KVFS_OK) c.poisoned = true;
    }
    return rc;
  });
}

int kvfs_restore(kvfs_ctx *ctx, int fd, int64_t *moved, kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (c.dev && c.poisoned) return KVFS_EIO;
    File *f = get_file(c, fd);
    if (!f) return KVFS_EBADF;
    void *hb = f->host_buf, *hd = f->host_dev;
    std::vector<uint32_t> pages;
    int rc = restore_file(c, *f, &pages);
    if (rc != KVFS_OK) return rc;
    f->host_buf = f->host_dev = nullptr;
    if (moved) *moved = static_cast<int64_t>(pages.size());
    if (c.dev && !pages.empty()) {
      rc = c.dev->unpack_pages(pages, hd, stream);  // host tier -> fresh device pages
      if (rc != KVFS_OK) c.poisoned = true;
    }
    if (c.dev && hb) c.dev->host_release(hb, stream);  // recycled once the copy on `stream` is done
    return rc;
  });
}

int kvfs_merge(kvfs_ctx *ctx, const int *fds, int n_fds, const char *name, int *fd, kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (c.dev && c.poisoned) return KVFS_EIO;
    std::vector<int32_t> src;
    std::vector<uint32_t> pages;
    int rc = merge_files(c, fds, n_fds, name, fd, &src, &pages);
    if (rc != KVFS_OK) return rc;
    if (c.dev && !src.empty()) {
      rc = c.dev->gather(src, pages, stream);
      if (rc != KVFS_OK) c.poisoned = true;
    }
    return rc;
  });
}

int kvfs_append(kvfs_ctx *ctx, int fd, int64_t n, const int32_t *pos, const void *k, const void *v,
                kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (c.dev && c.poisoned) return KVFS_EIO;
    File *f = get_file(c, fd);
    if (!f) return KVFS_EBADF;
    if (f->offloaded) return KVFS_EOFFLOAD;
    if (n < 0 || (n > 0 && !pos)) return KVFS_EINVAL;
    if (n == 0) return KVFS_OK;
    if (n >= (int64_t{1} << 30)) return KVFS_EINVAL;
    if (c.dev && (!k || !v)) return KVFS_EINVAL;
    int64_t need = 0;
    int rc = append_plan(c, *f, n, pos, &need, nullptr);
    if (rc != KVFS_OK) return rc;
    std::vector<int32_t> dst;
    std::vector<PageCopy> copies;
    dst.reserve(static_cast<size_t>(n));
    append_commit(c, *f, n, pos, &dst, &copies);
    c.ctr.page_copies += static_cast<int64_t>(copies.size());
    if (c.dev) {
      if (!copies.empty()) rc = c.dev->copy_pages(copies, stream);
      if (rc == KVFS_OK) rc = c.dev->append_rows(dst, k, v, stream);
      if (rc != KVFS_OK) c.poisoned = true;
    }
    return rc;
  });
}

// ------------------------------------------------------------------------------------------ pred
int pred_step_begin(kvfs_ctx *ctx, const pred_desc *descs, int n_desc, const int32_t *pos, int *status,
                    pred_step **step, kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (!step) return KVFS_EINVAL;
    if (c.dev && c.poisoned) return KVFS_EIO;
    const int64_t t0 = now_ns();
    const int rc = pred_reserve(c, descs, n_desc, pos, status, &c.plan);
    const int64_t t1 = now_ns();
    c.ctr.host_reserve_ns += t1 - t0;
    if (rc != KVFS_OK && rc != KVFS_EPARTIAL) return rc;
    if (c.dev) {
      pred_split(c, c.opt_chunk_cutover, &c.plan);
      pred_cascade(c, c.opt_cascade_min_entries, c.opt_prefix_splits, c.opt_prefix_paired, c.dev->sms(), c.dev->prefix_partial_capacity(),
                   &c.plan);
      pred_logits(c, &c.plan);
      const int64_t t2 = now_ns();
      c.ctr.host_split_ns += t2 - t1;
      const int drc = c.dev->pred_begin(c.plan, stream);
      c.ctr.host_upload_ns += now_ns() - t2;
      if (drc != KVFS_OK) {
        c.poisoned = true;
        return drc;
      }
    }
    c.step_open = true;
    *step = reinterpret_cast<pred_step *>(&c.plan);
    return rc;
  });
}

int pred_attn_layer(kvfs_ctx *ctx, pred_step *step, int layer, const void *q, const void *k_new,
                    const void *v_new, void *out, float *lse, float scale, kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    if (!ctx) return KVFS_EINVAL;
    Lock lk(ctx);
    Ctx &c = *lk.c;
    if (c.broken) return KVFS_EIO;
    if (!c.step_open || step != reinterpret_cast<pred_step *>(&c.plan)) return KVFS_EINVAL;
    if (!c.dev) return KVFS_ENOSYS;
    if (c.poisoned) return KVFS_EIO;
    if (layer < 0 || layer >= c.cfg.n_layers || !(scale > 0.f)) return KVFS_EINVAL;
    if (c.plan.T > 0 && (!q || !k_new || !v_new || !out)) return KVFS_EINVAL;
    const int64_t t0 = now_ns();
    c.logits_layer = c.logits_buf ? layer : -1;  // the decode kernel (over)writes this layer's logits
    c.logits_gather = c.opt_holes_gather;         // ... at packed row positions in gathered stages
    const int rc = c.dev->pred_layer(c.plan, layer, q, k_new, v_new, out, lse, scale, stream);
    c.ctr.host_launch_ns += now_ns() - t0;
    if (rc != KVFS_OK) c.poisoned = true;
    return rc;
  });
}

int pred_attn_scores(kvfs_ctx *ctx, pred_step *step, int layer, const void *q, const float *lse, float scale,
                     float *scores, const int64_t *score_off, kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    if (!ctx) return KVFS_EINVAL;
    Lock lk(ctx);
    Ctx &c = *lk.c;
    if (c.broken) return KVFS_EIO;
    if (!c.step_open || step != reinterpret_cast<pred_step *>(&c.plan)) return KVFS_EINVAL;
    if (!c.dev) return KVFS_ENOSYS;
    if (c.poisoned) return KVFS_EIO;
    if (layer < 0 || layer >= c.cfg.n_layers || !(scale > 0.f)) return KVFS_EINVAL;
    if (c.plan.score_src.empty()) return KVFS_OK;
    if (!q || !lse || !scores || !score_off) return KVFS_EINVAL;
    std::vector<ScoreDesc> sd;
    std::vector<ScoreUnit> su, lu;
    std::vector<LogitDesc> ld;
    // descriptors whose keys the decode kernel scored for this layer: fused pass over its logits (K10);
    // the others (chunk descriptors, shared-prefix members, no buffer, another layer): K9 over K
    const bool fused = c.logits_buf && c.logits_layer == layer;
    for (const ScoreSrc &x : c.plan.score_src) {
      const File &f = *x.file;
      const int32_t ne = static_cast<int32_t>(f.table.size());
      if (fused && x.logit_off >= 0) {
        const int32_t di = static_cast<int32_t>(ld.size());
        ld.push_back({score_off[x.batch_idx], x.logit_off, x.slab_off, x.n_q, x.row0, x.n_old, x.n_old_entries,
                      x.stages_per_unit, c.logits_gather, 0});
        for (int32_t e0 = 0; e0 < ne; e0 += 32) lu.push_back({di, e0, std::min(ne, e0 + 32), f.table[e0].lstart});
        continue;
      }
      const int32_t di = static_cast<int32_t>(sd.size());
      sd.push_back({x.slab_off, x.n_q, x.row0, static_cast<int32_t>(f.len), score_off[x.batch_idx]});
      for (int32_t e0 = 0; e0 < ne; e0 += KVFS_SCORE_UNIT_ENTRIES)
        su.push_back({di, e0, std::min(ne, e0 + KVFS_SCORE_UNIT_ENTRIES), f.table[e0].lstart});
    }
    int rc = KVFS_OK;
    c.ctr.last_fused_scores = static_cast<int64_t>(ld.size());
    if (!ld.empty()) rc = c.dev->logit_scores(ld, lu, lse, scores, stream);
    if (rc == KVFS_OK && !sd.empty()) rc = c.dev->scores(sd, su, layer, q, lse, scale, scores, stream);
    if (rc != KVFS_OK) c.poisoned = true;
    return rc;
  });
}

int pred_step_end(kvfs_ctx *ctx, pred_step *step) {
  return guarded(ctx, [&]() -> int {
    if (!ctx) return KVFS_EINVAL;
    Lock lk(ctx);
    Ctx &c = *lk.c;
    if (c.broken) return KVFS_EIO;
    if (!c.step_open || step != reinterpret_cast<pred_step *>(&c.plan)) return KVFS_EINVAL;
    c.step_open = false;
    return KVFS_OK;
  });
}

int pred_attn_batch(kvfs_ctx *ctx, const pred_desc *descs, int n_desc, const int32_t *pos, const void *q,
                    const void *k_new, const void *v_new, void *out, float *lse, float scale, int *status,
                    kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    if (!ctx) return KVFS_EINVAL;
    {
      Lock lk(ctx);
      Ctx &c = *lk.c;
      if (c.broken) return KVFS_EIO;
      if (c.step_open) return KVFS_EBUSY;
      if (!c.dev) return KVFS_ENOSYS;
      if (c.poisoned) return KVFS_EIO;
      if (c.cfg.n_layers != 1 || !(scale > 0.f)) return KVFS_EINVAL;
      int64_t T = 0;
      for (int i = 0; descs && i < n_desc; ++i) T += descs[i].n_q > 0 ? descs[i].n_q : 0;
      if (T > 0 && (!q || !k_new || !v_new || !out)) return KVFS_EINVAL;
    }
    pred_step *st = nullptr;
    const int rc = pred_step_begin(ctx, descs, n_desc, pos, status, &st, stream);
    if (rc != KVFS_OK && rc != KVFS_EPARTIAL) return rc;
    const int lrc = pred_attn_layer(ctx, st, 0, q, k_new, v_new, out, lse, scale, stream);
    pred_step_end(ctx, st);
    return lrc != KVFS_OK ? lrc : rc;
  });
}

int pred_attn_batch_host(kvfs_ctx *ctx, const pred_desc *descs, int n_desc, const int32_t *pos, const void *q,
                         const void *k_new, const void *v_new, void *out, float *lse, float scale, int *status,
                         kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    if (!ctx) return KVFS_EINVAL;
    Device::HostIo io;
    int64_t T = 0;
    {
      Lock lk(ctx);
      Ctx &c = *lk.c;
      if (c.broken) return KVFS_EIO;
      if (c.step_open) return KVFS_EBUSY;
      if (!c.dev) return KVFS_ENOSYS;
      if (c.poisoned) return KVFS_EIO;
      if (c.cfg.n_layers != 1 || !(scale > 0.f) || n_desc < 0 || (n_desc > 0 && !descs)) return KVFS_EINVAL;
      for (int i = 0; i < n_desc; ++i) {
        if (descs[i].n_q < 0) return KVFS_EINVAL;
        T += descs[i].n_q;
      }
      if (T > c.cfg.max_batch_rows) return KVFS_EINVAL;
      if (T > 0 && (!q || !k_new || !v_new || !out)) return KVFS_EINVAL;
      if (T > 0) {
        const int rc = c.dev->io_begin(T, q, k_new, v_new, lse != nullptr, stream, &io);
        if (rc != KVFS_OK) return rc;
      }
    }
    std::vector<int> st_local;
    int *st = status;
    if (!st) {
      st_local.assign(static_cast<size_t>(std::max(1, n_desc)), 0);
      st = st_local.data();
    }
    const int rc = pred_attn_batch(ctx, descs, n_desc, pos, T ? io.q : nullptr, T ? io.k : nullptr,
                                   T ? io.v : nullptr, T ? io.out : nullptr, T ? io.lse : nullptr, scale, st, stream);
    if (T == 0) return rc;
    // copy out the rows of the descriptors that succeeded (failed descriptors' rows stay untouched); after a
    // call-level error nothing is copied
    std::vector<std::pair<int64_t, int64_t>> rows;
    if (rc == KVFS_OK || rc == KVFS_EPARTIAL) {
      int64_t r = 0;
      for (int i = 0; i < n_desc; ++i) {
        const int64_t n = descs[i].n_q;
        if (n > 0 && st[i] == KVFS_OK) {
          if (!rows.empty() && rows.back().second == r) rows.back().second = r + n;
          else rows.push_back({r, r + n});
        }
        r += n;
      }
    }
    Lock lk(ctx);
    const int erc = lk.c->dev->io_end(io, out, lse, rows, stream);
    return erc != KVFS_OK ? erc : rc;
  });
}

int pred_host_fence(kvfs_ctx *ctx, kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (!c.dev) return KVFS_ENOSYS;
    return c.dev->io_fence(stream);
  });
}

// ------------------------------------------------------------------------------------------ introspection
int kvfs_stat(kvfs_ctx *ctx, int fd, kvfs_stat_t *st) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    File *f = get_file(c, fd);
    if (!f) return KVFS_EBADF;
    if (!st) return KVFS_EINVAL;
    st->len = f->len;
    st->n_entries = static_cast<int64_t>(f->table.size());
    st->last_pos = last_pos(c, *f);
    st->reserved = 0;
    return KVFS_OK;
  });
}

int kvfs_get_table(kvfs_ctx *ctx, int fd, uint32_t *page, uint64_t *mask, int64_t cap, int64_t *n) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    File *f = get_file(c, fd);
    if (!f) return KVFS_EBADF;
    if (cap < 0 || (cap > 0 && (!page || !mask))) return KVFS_EINVAL;
    const int64_t m = static_cast<int64_t>(f->table.size());
    for (int64_t i = 0; i < m && i < cap; ++i) {
      page[i] = f->table[i].page;
      mask[i] = f->table[i].mask;
    }
    if (n) *n = m;
    return KVFS_OK;
  });
}

int kvfs_get_positions(kvfs_ctx *ctx, int fd, int32_t *pos, int64_t cap, int64_t *n) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    File *f = get_file(c, fd);
    if (!f) return KVFS_EBADF;
    if (cap < 0 || (cap > 0 && !pos)) return KVFS_EINVAL;
    std::vector<int32_t> lp;
    file_positions(c, *f, &lp);
    const int64_t m = static_cast<int64_t>(lp.size());
    if (m > 0 && cap > 0) std::memcpy(pos, lp.data(), sizeof(int32_t) * static_cast<size_t>(std::min(m, cap)));
    if (n) *n = m;
    return KVFS_OK;
  });
}

int kvfs_get_refcounts(kvfs_ctx *ctx, uint32_t *refcnt, int64_t n) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (n < 0 || (n > 0 && !refcnt)) return KVFS_EINVAL;
    for (int64_t p = 0; p < n && p < c.pool->n_pages(); ++p) refcnt[p] = c.pool->refcnt(static_cast<uint32_t>(p));
    return KVFS_OK;
  });
}

int kvfs_free_pages(kvfs_ctx *ctx, int64_t *n_free) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (!n_free) return KVFS_EINVAL;
    *n_free = c.pool->n_free();
    return KVFS_OK;
  });
}

int kvfs_read(kvfs_ctx *ctx, int fd, int layer, int64_t begin, int64_t end, void *k_out, void *v_out,
              kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    File *f = get_file(c, fd);
    if (!f) return KVFS_EBADF;
    if (f->offloaded) return KVFS_EOFFLOAD;
    if (!c.dev) return KVFS_ENOSYS;
    if (c.poisoned) return KVFS_EIO;
    if (layer < 0 || layer >= c.cfg.n_layers) return KVFS_EINVAL;
    if (begin < 0 || end < begin || end > f->len) return KVFS_ERANGE;
    if (end == begin) return KVFS_OK;
    if (!k_out || !v_out) return KVFS_EINVAL;
    const int rc = c.dev->read(f->table, layer, begin, end, k_out, v_out, stream);
    if (rc != KVFS_OK) c.poisoned = true;
    return rc;
  });
}

int kvfs_audit(kvfs_ctx *ctx) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    return audit(c);
  });
}

int kvfs_pack(kvfs_ctx *ctx, const int *fds, int n_fds, void *buf_dev, size_t buf_cap, size_t *buf_used, void *hdr,
              size_t hdr_cap, size_t *hdr_used, kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (c.dev && c.poisoned) return KVFS_EIO;
    std::vector<uint32_t> pages;
    std::vector<uint8_t> h;
    const int rc = pack_files(c, fds, n_fds, &pages, &h);
    if (rc != KVFS_OK) return rc;
    const size_t need = pages.size() * static_cast<size_t>(c.cfg.n_layers) * 2 * c.cfg.n_kv_heads * c.cfg.page_size *
                        c.cfg.head_dim * 2;
    if (buf_used) *buf_used = c.dev ? need : 0;
    if (hdr_used) *hdr_used = h.size();
    if (!hdr || hdr_cap < h.size()) return KVFS_ENOMEM;
    if (c.dev && need > 0 && (!buf_dev || buf_cap < need)) return KVFS_ENOMEM;
    std::memcpy(hdr, h.data(), h.size());
    if (c.dev && !pages.empty()) {
      const int drc = c.dev->pack_pages(pages, buf_dev, stream);
      if (drc != KVFS_OK) c.poisoned = true;
      return drc;
    }
    return KVFS_OK;
  });
}

int kvfs_unpack(kvfs_ctx *ctx, const void *buf_dev, size_t buf_bytes, const void *hdr, size_t hdr_bytes,
                const char *const *names, int *fds_out, kvfs_stream_t stream) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (c.dev && c.poisoned) return KVFS_EIO;
    if (c.dev && !buf_dev) return KVFS_EINVAL;
    std::vector<uint32_t> pages;
    if (c.dev) {  // the buffer must hold every packed page (a truncated transfer would be read out of bounds)
      uint32_t nu = 0;
      if (!hdr || hdr_bytes < 16) return KVFS_EINVAL;
      std::memcpy(&nu, static_cast<const char *>(hdr) + 12, 4);
      const size_t need = static_cast<size_t>(nu) * c.cfg.n_layers * 2 * c.cfg.n_kv_heads * c.cfg.page_size *
                          c.cfg.head_dim * 2;
      if (buf_bytes < need) return KVFS_EINVAL;
    }
    const int rc = unpack_files(c, hdr, hdr_bytes, names, fds_out, &pages);
    if (rc != KVFS_OK) return rc;
    if (c.dev && !pages.empty()) {
      const int drc = c.dev->unpack_pages(pages, buf_dev, stream);
      if (drc != KVFS_OK) c.poisoned = true;
      return drc;
    }
    return KVFS_OK;
  });
}

int kvfs_set_logits_buffer(kvfs_ctx *ctx, void *buf, size_t bytes) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    if (!c.dev) return KVFS_EINVAL;
    if (c.step_open) return KVFS_EBUSY;
    if (buf && (reinterpret_cast<uintptr_t>(buf) & 15)) return KVFS_EINVAL;
    c.logits_buf = (buf && bytes >= 16) ? static_cast<float *>(buf) : nullptr;
    c.logits_cap = c.logits_buf ? static_cast<int64_t>(bytes / 16) * 4 : 0;
    c.logits_layer = -1;
    return KVFS_OK;
  });
}

int kvfs_set_option(kvfs_ctx *ctx, int option, int64_t value) {
  return guarded(ctx, [&]() -> int {
    KVFS_LOCK_OR(ctx);
    switch (option) {
      case KVFS_OPT_DECODE_CTAS:
        if (value < 0 || value > 4096) return KVFS_EINVAL;
        c.opt_decode_ctas = value;
        return KVFS_OK;
      case KVFS_OPT_CHUNK_CUTOVER:
        if (value < 0) return KVFS_EINVAL;
        c.opt_chunk_cutover = value;
        return KVFS_OK;
      case KVFS_OPT_DETERMINISTIC:
        return KVFS_OK;
      case KVFS_OPT_CASCADE_MIN_ENTRIES:
        if (value < 0) return KVFS_EINVAL;
        c.opt_cascade_min_entries = value;
        return KVFS_OK;
      case KVFS_OPT_HOLES_GATHER:
        if (value < 0 || value > 1) return KVFS_EINVAL;
        c.opt_holes_gather = static_cast<int>(value);
        return KVFS_OK;
      case KVFS_OPT_PREFIX_SPLITS:
        if (value < 0 || value > kMaxPrefixSplits) return KVFS_EINVAL;
        c.opt_prefix_splits = static_cast<int>(value);
        return KVFS_OK;
      case KVFS_OPT_PREFIX_PAIRED:
        if (value < 0 || value > 2) return KVFS_EINVAL;
        c.opt_prefix_paired = static_cast<int>(value);
        return KVFS_OK;
      case KVFS_OPT_DECODE_CHUNKS:
        if (value < 0 || value > 2048) return KVFS_EINVAL;
        c.opt_decode_chunks = value;
        return KVFS_OK;
      case KVFS_OPT_TIMING:
        if (value < 0 || value > 1000000) return KVFS_EINVAL;
        c.opt_timing = value != 0;
        c.opt_timing_every = value > 1 ? value : 1;
        c.layer_calls = 0;
        return KVFS_OK;
      case KVFS_OPT_FAULT_INJECT:
        if (value < 0) return KVFS_EINVAL;
        c.fault_countdown = value;
        return KVFS_OK;
      default:
        return KVFS_EINVAL;
    }
  });
}

int kvfs_get_counter(kvfs_ctx *ctx, int counter, int64_t *value) {
  return guarded(ctx, [&]() -> int {
    if (!ctx || !value) return KVFS_EINVAL;
    Lock lk(ctx);
    Ctx &c = *lk.c;
    if (c.broken) return KVFS_EIO;
    switch (counter) {
      case KVFS_CTR_KERNEL_LAUNCHES: *value = c.ctr.launches; return KVFS_OK;
      case KVFS_CTR_H2D_BYTES: *value = c.ctr.h2d_bytes; return KVFS_OK;
      case KVFS_CTR_PAGE_COPIES: *value = c.ctr.page_copies; return KVFS_OK;
      case KVFS_CTR_LAST_DECODE_CTAS: *value = c.ctr.last_decode_ctas; return KVFS_OK;
      case KVFS_CTR_LAST_CHUNK_UNITS: *value = c.ctr.last_chunk_units; return KVFS_OK;
      case KVFS_CTR_LAST_PREFIX_UNITS: *value = c.ctr.last_prefix_units; return KVFS_OK;
      case KVFS_CTR_LAST_PREFIX_GROUPS: *value = c.ctr.last_prefix_groups; return KVFS_OK;
      case KVFS_CTR_HOST_PAGES: *value = c.ctr.host_pages; return KVFS_OK;
      case KVFS_CTR_COMPACT_DEVICE_NS: *value = c.last_compact_device_ns; return KVFS_OK;
      case KVFS_CTR_LAYER_DEVICE_NS: {
        int64_t n = 0;
        *value = c.dev ? c.dev->take_layer_ns(&n) : 0;
        c.last_layer_timed = n;
        return KVFS_OK;
      }
      case KVFS_CTR_LAYER_TIMED: *value = c.last_layer_timed; return KVFS_OK;
      case KVFS_CTR_COPY_DEVICE_NS: {
        int64_t n = 0;
        *value = c.dev ? c.dev->take_copy_ns(&n) : 0;
        return KVFS_OK;
      }
      case KVFS_CTR_LAST_FUSED_SCORES: *value = c.ctr.last_fused_scores; return KVFS_OK;
      case KVFS_CTR_HOST_RESERVE_NS: *value = c.ctr.host_reserve_ns; return KVFS_OK;
      case KVFS_CTR_HOST_SPLIT_NS: *value = c.ctr.host_split_ns; return KVFS_OK;
      case KVFS_CTR_HOST_UPLOAD_NS: *value = c.ctr.host_upload_ns; return KVFS_OK;
      case KVFS_CTR_HOST_LAUNCH_NS: *value = c.ctr.host_launch_ns; return KVFS_OK;
      default: return KVFS_EINVAL;
    }
  });
}

}  // extern "C"
