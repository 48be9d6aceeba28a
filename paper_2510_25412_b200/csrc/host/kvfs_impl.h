// Host control plane of KVFS (no CUDA dependency): files, page tables, the batched-pred reserve and
// the plan handed to the device data plane.  Rules R1-R11 as in SURVEY.md §8(c) C3 / DESIGN.md.
#pragma once
#include <atomic>
#include <cstdint>
#include <memory>
#include <new>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../../include/kvfs.h"
#include "pool.h"

namespace kvfs {

// One page-table entry.  Byte-identical to the device mirror entry (16 B): the slab is a plain copy.
struct Entry {
  uint32_t page;
  int32_t lstart;  // logical index of the entry's first retained token (prefix sum of popcounts)
  uint64_t mask;   // bit s = slot s retained
};
static_assert(sizeof(Entry) == 16, "Entry must be 16 bytes");

// Table version stamps: globally unique and increasing, so (file, stamp) identifies one state of a table.
inline uint64_t next_tver() {
  static std::atomic<uint64_t> clock{0};
  return ++clock;
}

struct File {
  std::string name;
  // Version of the table's existing entries: a new stamp whenever an entry is changed in place or removed
  // (truncate, evict, compaction, copy-on-write of the tail, offload / restore).  Appends that only add
  // entries or fill the slots of an unshared tail keep it (an entry identical to another file's entry
  // holds a shared page, and appending into a shared tail copies it first, i.e. gets a new stamp).
  uint64_t tver = next_tver();
  // Cascade planning cache (pred_cascade): the number of leading entries identical to those of file
  // run_lead, valid while both stamps are unchanged.
  const File *run_lead = nullptr;
  uint64_t run_lead_tver = 0, run_self_tver = 0;
  int64_t run_len = 0;
  bool alive = true;
  std::vector<Entry> table;
  std::vector<int32_t> spos;  // [n_entries * P]: absolute position of the token in (entry, slot)
  int64_t len = 0;
  // Device mirror of `table` (page and mask only; the kernels never read the device lstart): entries at
  // indices >= dirty_from and the indices in dirty_pts may be stale on the device.
  int64_t slab_off = -1;
  int64_t slab_cap = 0;
  size_t dirty_from = 0;
  std::vector<uint32_t> dirty_pts;
  int64_t batch_tag = -1;  // pred batch id that last used the file (EBUSY detection)
  int32_t score_slot = -1; // index of its ScoreSrc in the current pred plan (fused-scores bookkeeping)
  // R15 host tier: while offloaded, entries with page & KVFS_HOST_PAGE live in host_buf (pinned, mapped;
  // host_dev = its device address), slot order = table order
  bool offloaded = false;
  int64_t n_host = 0;
  void *host_buf = nullptr, *host_dev = nullptr;
};
using FilePtr = std::shared_ptr<File>;

struct PageCopy {
  uint32_t src, dst;
};

// Slab of device table entries: per-file blocks of power-of-two capacity (>= 64 entries) with per-class
// free lists.  Host bookkeeping only; a freed block is reused by later uploads, which are stream-ordered
// after every kernel that could still read it.
class Slab {
 public:
  void init(int64_t capacity) { cap_ = capacity; top_ = 0; free_.assign(40, {}); }
  bool alloc(int64_t n, int64_t *off, int64_t *cap);
  void free(int64_t off, int64_t cap);
  int64_t capacity() const { return cap_; }

 private:
  int64_t cap_ = 0, top_ = 0;
  std::vector<std::vector<int64_t>> free_;
};

// Per-descriptor record consumed by the decode kernel (layout shared with csrc/cuda/common.cuh).
struct DevDesc {
  int64_t cost_begin;        // first global stage index of this descriptor's units
  int32_t slab_off;          // entry base of the file's table in the slab
  int32_t n_old_entries;     // entries holding at least one token retained before this call
  int32_t n_old;             // retained tokens before this call's append
  int32_t n_q;               // new tokens (query rows)
  int32_t row0;              // first packed row of the descriptor
  int32_t unit_base;         // global unit index of (g=0, qi=0)
  int32_t stages_per_unit;   // n_old_entries + ceil(n_q / P)
  int32_t n_entries;         // entries after the append
  int32_t tail_lstart;       // logical index of the first token of entry n_old_entries - 1
  int32_t first_new_entry;   // entry holding logical token n_old (the first new token)
  int32_t first_new_lstart;  // logical index of that entry's first token
  int32_t skip;              // leading entries attended by the shared-prefix kernel (0: none)
  int32_t pref_splits;       // shared-prefix partials per unit (0: none)
  int32_t pref_base;         // first shared-prefix partial of unit (g = 0, qi = 0): unit (g, qi) split s is
                             // partial pref_base + (g * n_q + qi) * pref_splits + s (the cascade writes one
                             // merged partial per unit: pref_splits = 1)
  int64_t logit_off;         // >= 0: the decode kernel writes the scaled logits of this descriptor's keys for
                             // the fused scores (kvfs_set_logits_buffer); unit (g, qi), stage st, slot s, head h
                             // at logit_off + (((g * n_q + qi) * stages_per_unit + st) * P + s) * G + h.  -1: none
  int64_t pad;
};
static_assert(sizeof(DevDesc) == 80, "DevDesc must be 80 bytes");

struct SlabRun {
  int64_t dst;    // first slab entry written
  int32_t src;    // first entry in the uploaded run array
  int32_t count;  // entries
};
static_assert(sizeof(SlabRun) == 16, "SlabRun must be 16 bytes");

// K2 (tcgen05 chunk kernel) records (layouts shared with csrc/cuda/kernels.cuh)
struct ChunkDesc {
  int32_t slab_off, n_entries, n_old, n_q, row0, first_new_entry, first_new_lstart, pad;
};
struct ChunkUnit {
  int32_t desc, g, m;
  int32_t group;  // shared-prefix mode: the (family, kv head, M-tile pair) group whose splits merge together
};
constexpr int kMaxPrefixGroups = 4096;  // group counters in the workspace (a prefix grid with S > 1 is <= 1 CTA per SM)
constexpr int kMaxPrefixSplits = 16;  // key splits of one shared prefix (the decode merge folds them in groups)
// Up to this many key splits the decode kernel folds a unit's split records itself (no in-kernel group merge)
constexpr int kMaxFoldSplits = 4;
// Shared-prefix (cascade) work: one record per (fork family, key split); the family's query rows are
// listed in PrefixRow order (row0 .. row0 + n_rows - 1).
struct PrefixDesc {
  int32_t slab_off;   // slab index of the split's first entry (in the leader file's table)
  int32_t n_entries;  // entries of this split
  int32_t n_rows;     // query rows (tokens) of the family
  int32_t row0;       // first PrefixRow of the family
  int32_t split, n_splits;
  int32_t q_t0;       // >= 0: the family's query rows are the consecutive packed rows q_t0 .. q_t0 + n_rows - 1
                      // (Q tiles by TMA); -1: rows gathered through the PrefixRow records
  int32_t split_off;  // n_splits > 1: split partial s of merged record r is split_off + r * n_splits + s
};
// NEXT-2 attention-score accumulation (pred_attn_scores): every successful descriptor of the step, and
// the work units (descriptor, entry chunk of <= 32 entries, logical index of the chunk's first token).
struct ScoreDesc {
  int32_t slab_off, n_q, row0, len_after;
  int64_t out_off;  // caller's offset of the descriptor's scores
};
struct ScoreUnit {
  int32_t desc, e0, e1, l0;
};
struct ScoreSrc {
  int32_t batch_idx, slab_off, n_q, row0;
  File *file;
  // fused scores: the decode kernel's logits of this descriptor (logit_off >= 0), with the layout numbers
  int64_t logit_off = -1;
  int32_t n_old = 0, n_old_entries = 0, stages_per_unit = 0;
};
// Fused-scores pass (pred_attn_scores over the decode kernel's logits, include/kvfs.h kvfs_set_logits_buffer)
struct LogitDesc {
  int64_t out_off, logit_off;
  int32_t slab_off, n_q, row0, n_old, n_old_entries, stages_per_unit;
  int32_t gather, pad;
};
struct PrefixRow {
  int32_t t;          // packed row (Q row) of the query token
  int32_t pref_base;  // DevDesc::pref_base of its descriptor
  int32_t n_q;        // n_q of its descriptor
  int32_t qi;         // row within its descriptor
};

struct PredPlan {
  std::vector<DevDesc> descs;       // successful descriptors with n_q > 0, in order
  std::vector<int32_t> dst_slot;    // [T] page * P + slot of every appended row (-1: row not appended)
  std::vector<int64_t> run_dst;     // slab updates: slab index of each run_entries[j]
  std::vector<Entry> run_entries;
  std::vector<PageCopy> copies;     // copy-on-write copies
  int64_t total_cost = 0;
  int32_t n_units = 0;
  int32_t T = 0;
  int32_t max_nq = 0;
  // split by n_q (pred_split): descriptors with n_q >= cutover go to K2
  std::vector<ChunkDesc> chunk_descs;
  std::vector<ChunkUnit> chunk_units;
  std::vector<int32_t> chunk_dst;  // [T] dst slot of rows of K2 descriptors, -1 otherwise
  std::vector<File *> desc_files;   // file of every descriptor in `descs` (host only)
  // shared-prefix (cascade) plan (pred_cascade)
  std::vector<PrefixDesc> prefix_descs;
  std::vector<ChunkUnit> prefix_units;
  std::vector<PrefixRow> prefix_rows;
  std::vector<int32_t> prefix_cta_units;  // paired cascade: per CTA (first unit, count); empty: one unit per CTA
  int32_t prefix_partials = 0;  // partials the prefix kernel writes (PART floats each)
  std::vector<ScoreSrc> score_src;  // every successful descriptor with n_q > 0 (batch order)
  int32_t prefix_groups = 0;
  int32_t decode_sms = 0;  // cascade: SMs the decode kernel's rings take (the prefix CTAs hold the rest); 0: all
  int32_t prefix_fold = 0;  // cascade: 1 = the decode kernel folds the S split records (no in-kernel merge)
};

class Device;  // data plane (csrc/cuda), absent for a host-only ctx

// one file's compaction gather (R7): token i of old_table (logical order) -> (new_pages[i / P], i % P)
struct CompactJob {
  const std::vector<Entry> *old_table;
  const std::vector<uint32_t> *new_pages;
  int64_t len;
};

struct CtxCounters {
  int64_t launches = 0, h2d_bytes = 0, page_copies = 0, last_decode_ctas = 0, last_chunk_units = 0,
          last_prefix_units = 0, last_prefix_groups = 0, host_pages = 0;
  int64_t host_reserve_ns = 0, host_split_ns = 0, host_upload_ns = 0, host_launch_ns = 0;
  int64_t last_fused_scores = 0;
};

struct Ctx {
  std::mutex mu;
  kvfs_config cfg{};
  std::vector<void *> kpool, vpool;
  std::unique_ptr<PagePool> pool;
  std::unordered_map<std::string, FilePtr> names;
  std::vector<FilePtr> fds;  // index = fd
  Slab slab;
  Device *dev = nullptr;
  bool poisoned = false;
  std::atomic<bool> broken{false};  // a C++ exception escaped a call (capi.cc guarded): every call is EIO
  int64_t fault_countdown = 0;       // KVFS_OPT_FAULT_INJECT (tests)
  bool step_open = false;
  // Fused scores (kvfs_set_logits_buffer): caller-owned device buffer for the decode kernel's logits, and the
  // layer whose logits it holds (pred_attn_scores uses them only for that layer; else the K9 pass)
  float *logits_buf = nullptr;
  int64_t logits_cap = 0;  // floats
  int logits_layer = -1;
  int logits_gather = 1;  // KVFS_OPT_HOLES_GATHER in force when those logits were written
  int64_t batch_counter = 0;
  int64_t opt_decode_ctas = 0;
  int64_t opt_decode_chunks = 0;  // KVFS_OPT_DECODE_CHUNKS (0: static scheduling)
  int opt_holes_gather = 1;       // KVFS_OPT_HOLES_GATHER
  int64_t opt_chunk_cutover = 2;  // measured: cfg2d drafts (n_q 4) K1 1.29 ms / 4.0x HBM traffic, K2 0.44 ms / 1.0x
  int64_t opt_cascade_min_entries = 16;
  int opt_prefix_splits = 0;  // 0 = auto
  int opt_prefix_paired = 0;  // 0 = auto, 1 = off, 2 = on when possible
  bool opt_timing = false;    // KVFS_OPT_TIMING
  int64_t opt_timing_every = 1;  // KVFS_OPT_TIMING = n: every n-th pred_attn_layer call is timed
  int64_t layer_calls = 0;        // pred_attn_layer calls since KVFS_OPT_TIMING was set
  int64_t last_compact_device_ns = 0;
  int64_t last_layer_timed = 0;
  CtxCounters ctr;
  PredPlan plan;  // the open step's plan
  std::vector<int> step_status;
};

// KVFS_OPT_FAULT_INJECT: the n-th pass through an injection point throws (tests of the no-exception ABI)
inline void fault_point(Ctx &c) {
  if (c.fault_countdown > 0 && --c.fault_countdown == 0) throw std::bad_alloc();
}

// ---- host operations (files.cc); return kvfs_err codes, atomic on failure
int open_file(Ctx &c, const char *name, int flags, int *fd);
int close_file(Ctx &c, int fd);
int unlink_file(Ctx &c, const char *name);
File *get_file(Ctx &c, int fd);
int append_plan(const Ctx &c, const File &f, int64_t n, const int32_t *pos, int64_t *need, int64_t *new_entries);
// Commit R3; appends dst slots (page * P + slot) of the new tokens and any copy-on-write copy.
void append_commit(Ctx &c, File &f, int64_t n, const int32_t *pos, std::vector<int32_t> *dst,
                   std::vector<PageCopy> *copies);
int fork_file(Ctx &c, File &src, const char *dst_name, int *dst_fd, std::vector<PageCopy> *copies);
int truncate_file(Ctx &c, File &f, int64_t n);
int evict_file(Ctx &c, File &f, const int64_t *ranges, int n_ranges, int flags, std::vector<Entry> *old_table,
               std::vector<uint32_t> *new_pages);
int compact_file(Ctx &c, File &f, std::vector<Entry> *old_table, std::vector<uint32_t> *new_pages);
// Batched compaction, split in two: the page / table part (sequential: R1 allocation order), then the
// positions (per file, independent: may run on worker threads) with the old table it returned.
int compact_file_tables(Ctx &c, File &f, std::vector<Entry> *old_table, std::vector<uint32_t> *new_pages);
void compact_positions(File &f, const std::vector<Entry> &old, int P);
// R13 / R14: new file from selected tokens / from the union of parts; src_slots[i] = page * P + slot of the
// source of token i, new_pages = the file's pages (token i -> (new_pages[i / P], i % P)).  Atomic.
int extract_file(Ctx &c, File &src, const int64_t *idx, int64_t n, const char *name, int *fd,
                 std::vector<int32_t> *src_slots, std::vector<uint32_t> *new_pages);
int merge_files(Ctx &c, const int *fds, int n, const char *name, int *fd, std::vector<int32_t> *src_slots,
                std::vector<uint32_t> *new_pages);
void recompute_lstart(File &f, size_t from);
int32_t last_pos(const Ctx &c, const File &f);
void file_positions(const Ctx &c, const File &f, std::vector<int32_t> *out);
void release_file_slab(Ctx &c, File &f);
int audit(Ctx &c);
// R15: mark the file's exclusive entries as host entries (in table order), release their device pages;
// `pages` = the device pages to copy out, in host-slot order.  restore: allocate (R1, table order).
int offload_file(Ctx &c, File &f, std::vector<uint32_t> *pages);
int restore_file(Ctx &c, File &f, std::vector<uint32_t> *new_pages);

// ---- migration (migrate.cc)
int pack_files(Ctx &c, const int *fds, int n, std::vector<uint32_t> *pages, std::vector<uint8_t> *hdr);
int unpack_files(Ctx &c, const void *hdr, size_t hdr_bytes, const char *const *names, int *fds_out,
                 std::vector<uint32_t> *new_pages);

// ---- batched pred (batch.cc)
int pred_reserve(Ctx &c, const pred_desc *descs, int n_desc, const int32_t *pos, int *status, PredPlan *plan);
// Move descriptors with n_q >= cutover (0: none) from the K1 list to the K2 list (D = 128 only).
void pred_split(const Ctx &c, int64_t cutover, PredPlan *plan);
// Shared-prefix plan for the K1 list (KVFS_OPT_CASCADE_MIN_ENTRIES): groups descriptors whose files start
// with the same run of (page, mask) entries, sets their skip / pref_* fields and emits the prefix work.
// `sms` sizes the key splits, `max_partials` is the workspace capacity in partials.
// force_splits > 0: key splits per shared run (else chosen from the SM count)
// paired_mode: 0 = the cost model decides, 1 = never the paired partition, 2 = paired whenever possible
void pred_cascade(const Ctx &c, int64_t min_entries, int force_splits, int paired_mode, int sms, int64_t max_partials,
                  PredPlan *plan);
void pred_logits(Ctx &c, PredPlan *plan);

// ---- data plane interface (implemented in csrc/cuda/device.cu)
class Device {
 public:
  virtual ~Device() = default;
  virtual int copy_pages(const std::vector<PageCopy> &copies, kvfs_stream_t s) = 0;
  virtual int append_rows(const std::vector<int32_t> &dst, const void *k, const void *v, kvfs_stream_t s) = 0;
  // the files' gathers in order (a later file's destinations may be an earlier file's sources)
  virtual int compact(const std::vector<CompactJob> &jobs, kvfs_stream_t s) = 0;
  virtual int gather(const std::vector<int32_t> &src_slots, const std::vector<uint32_t> &new_pages,
                     kvfs_stream_t s) = 0;
  virtual int read(const std::vector<Entry> &table, int layer, int64_t begin, int64_t end, void *k_out,
                   void *v_out, kvfs_stream_t s) = 0;
  virtual int pred_begin(PredPlan &plan, kvfs_stream_t s) = 0;
  virtual int pred_layer(const PredPlan &plan, int layer, const void *q, const void *k_new, const void *v_new,
                         void *out, float *lse, float scale, kvfs_stream_t s) = 0;
  // fused scores (K10) of the descriptors whose logits the decode kernel wrote
  virtual int logit_scores(const std::vector<LogitDesc> &descs, const std::vector<ScoreUnit> &units,
                           const float *lse, float *out, kvfs_stream_t s) = 0;
  virtual int scores(const std::vector<ScoreDesc> &descs, const std::vector<ScoreUnit> &units, int layer,
                     const void *q, const float *lse, float scale, float *out, kvfs_stream_t s) = 0;
  // pinned, device-mapped host memory for the host tier (R15)
  virtual int host_alloc(size_t bytes, void **host, void **dev) = 0;
  virtual void host_free(void *host) = 0;
  // return a host buffer once the work queued on `s` (reading it) is done; no host wait
  virtual void host_release(void *host, kvfs_stream_t s) = 0;
  virtual int stream_sync(kvfs_stream_t s) = 0;
  virtual int pack_pages(const std::vector<uint32_t> &pages, void *buf, kvfs_stream_t s) = 0;
  virtual int unpack_pages(const std::vector<uint32_t> &pages, const void *buf, kvfs_stream_t s) = 0;
  virtual int sync() = 0;
  virtual int sms() const = 0;
  virtual int64_t prefix_partial_capacity() const = 0;
  // KVFS_OPT_TIMING: device time (ns) of the intervals recorded since the last call (waits for them)
  virtual int64_t take_device_ns() = 0;
  // KVFS_OPT_TIMING: summed device time of the pred layers recorded since the last call (waits for them);
  // *n = how many
  virtual int64_t take_layer_ns(int64_t *n) = 0;
  // KVFS_OPT_TIMING: summed device time of the page pack / unpack kernels (K6) since the last call
  virtual int64_t take_copy_ns(int64_t *n) = 0;
  // Host-buffer pred (pred_attn_batch_host): io_begin copies the step's inputs from host memory into one of
  // two device slots (library copy stream) and makes `s` wait for them (and for the slot's previous output
  // copy); io_end copies the slot's outputs to host memory once `s` has produced them (second copy stream);
  // io_fence makes `s2` wait for every output copy issued so far.
  struct HostIo {
    void *q = nullptr, *k = nullptr, *v = nullptr, *out = nullptr;
    float *lse = nullptr;
    int slot = -1;
    size_t q_bytes = 0, kv_bytes = 0, out_bytes = 0, lse_bytes = 0;
  };
  virtual int io_begin(int64_t T, const void *q, const void *k, const void *v, bool want_lse, kvfs_stream_t s,
                       HostIo *io) = 0;
  // rows: [begin, end) row ranges to copy out (the rows of the descriptors that succeeded)
  virtual int io_end(const HostIo &io, void *out, float *lse, const std::vector<std::pair<int64_t, int64_t>> &rows,
                     kvfs_stream_t s) = 0;
  virtual int io_fence(kvfs_stream_t s) = 0;
};

size_t device_workspace_bytes(const kvfs_config &cfg);
int create_device(Ctx &c, Device **out);

}  // namespace kvfs
