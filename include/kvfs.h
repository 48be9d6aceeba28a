/*
 * kvfs.h — C ABI of the B200-native KVFS + batched `pred` attention hot path
 * (arXiv 2510.25412, "Serve Programs, Not Prompts", Symphony).
 *
 * Citation key: P:n = PAPER.md line n, S:n = SPEC.md line n, §8 = SURVEY.md §8 (the scope table),
 * R1..R12 = the readings in SURVEY.md §8(c) C3 restated in DESIGN.md "Readings".
 *
 * What the calls compute
 *   pred (§4.1): "pred(kv: kv_file, tokens, positions) -> list[dist]"; the file is "updated
 *   with new tensors corresponding to the provided tokens" and a result is returned "for each input
 *   token".  This library implements the attention part of that system call for a batch of LIPs
 *   (§4.4 P:241 "aggregates multiple pred system calls into a single batch"): given the already
 *   projected Q / K_new / V_new rows of every LIP's new tokens it appends K_new / V_new into the LIP's
 *   file and returns, per query row and head, softmax attention over exactly the tokens the file
 *   retains (R10).  Tokens -> embeddings -> projections and the LM head / `dist` are outside (§2.1 M2/M3).
 *   KVFS (§4.2): the KV cache as files over fixed-size pages ("PagedAttention"), with
 *   open / fork ("clone the prefix file ... without duplicating the actual tensors") /
 *   remove, and pruning of "invalid or unimportant tokens" as in-place evict + compaction.
 *
 * Conventions (all functions)
 *   - Return KVFS_OK (0) or a negative kvfs_err.  Never throw, never abort, never print.
 *   - Atomic failure: a call that fails changes nothing.  pred_* is atomic per
 *     descriptor: failing descriptors get their own status and leave their output rows untouched, the
 *     others proceed, and the call returns KVFS_EPARTIAL.
 *   - Ownership: the caller owns every device buffer (pools, workspace, Q/K/V/out/lse), typically torch
 *     tensors, and keeps them alive until kvfs_destroy returns.  The ctx owns only host metadata, pinned
 *     staging buffers and CUDA events; it copies `name` strings.
 *   - Streams: host metadata changes take effect at call time.  Device work is enqueued on the given
 *     stream (NULL = legacy default stream).  All device work of one ctx must be issued on one stream
 *     (or the caller serialises streams): a page freed by evict/truncate may be reused by the next
 *     call's device work, and stream order is what keeps earlier readers safe.
 *   - Thread safety: calls on one ctx are serialised by an internal mutex.
 *   - Host-only ctx (cfg.device == -1): metadata only, for testing the control plane without a GPU.
 *     No CUDA call is ever made; calls that need data (pred_attn_batch, pred_attn_layer, kvfs_read)
 *     return KVFS_ENOSYS; kvfs_append / fork / evict / compact update metadata only.
 *   - A CUDA error poisons the ctx: that call and every later data call return KVFS_EIO.
 *   - No C++ exception crosses this ABI.  If one is raised inside a call (a host allocation failure:
 *     std::bad_alloc from a table, position or plan vector; std::system_error from a worker thread), the
 *     call returns KVFS_ENOMEM (allocation) or KVFS_EIO (anything else) and the ctx becomes BROKEN: the
 *     failed call may have been half-applied, so every later call on that ctx returns KVFS_EIO except
 *     kvfs_destroy, which still frees it.  (KVFS_OPT_FAULT_INJECT exercises this path in the tests.)
 *
 * Data layout (device)
 *   K and V pools, one pair per layer: [n_pages][n_kv_heads][page_size][head_dim] bf16 ("HND" pages):
 *   the (page, kv head) block is page_size*head_dim*2 contiguous bytes, which is the unit the decode
 *   kernel streams with 1-D TMA bulk copies.  One page id addresses the same page in every layer.
 *   Q rows [T][n_q_heads][head_dim] bf16, K_new/V_new rows [T][n_kv_heads][head_dim] bf16, out
 *   [T][n_q_heads][head_dim] bf16, lse [T][n_q_heads] fp32 (natural log), all row-major, rows packed in
 *   descriptor order (S:355 FIFO).  GQA: query head h reads KV head h / (n_q_heads / n_kv_heads).
 */
#ifndef KVFS_H_
#define KVFS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* cudaStream_t / CUstream without including CUDA headers. */
typedef struct CUstream_st *kvfs_stream_t;

typedef enum {
  KVFS_OK = 0,
  KVFS_ENOENT = -2,      /* name not found (open without O_CREAT, unlink) */
  KVFS_EIO = -5,         /* CUDA error; the ctx is poisoned */
  KVFS_EBADF = -9,       /* fd not open, or its file was unlinked */
  KVFS_ENOMEM = -12,     /* host allocation / device table slab / workspace too small */
  KVFS_EBUSY = -16,      /* pred batch: the descriptor's file already appeared earlier in the batch */
  KVFS_EEXIST = -17,     /* name exists (open O_CREAT|O_EXCL, fork destination) */
  KVFS_EINVAL = -22,     /* malformed arguments (NULL pointers, bad sizes, unsorted ranges, ...) */
  KVFS_ENOSPC = -28,     /* page pool exhausted (SPEC PoolExhausted) */
  KVFS_ERANGE = -34,     /* index / length out of range */
  KVFS_ENOSYS = -38,     /* data operation on a host-only ctx */
  KVFS_EPOS = -1001,     /* positions not strictly increasing / not > last retained (SPEC PositionConflict) */
  KVFS_EPARTIAL = -1002, /* pred batch: some descriptors failed, see status[] */
  KVFS_EOFFLOAD = -1003  /* the file is offloaded to the host tier (kvfs_offload): restore it first */
} kvfs_err;

enum { KVFS_O_CREAT = 1, KVFS_O_EXCL = 2 };   /* kvfs_open flags (R2) */
enum { KVFS_EVICT_COMPACT = 1 };              /* kvfs_evict flag (R8) */

typedef struct kvfs_ctx kvfs_ctx;
typedef struct pred_step pred_step;

typedef struct {
  int device;              /* CUDA device ordinal, or -1 for a host-only ctx */
  int n_layers;            /* >= 1 */
  int n_q_heads;           /* Hq, multiple of n_kv_heads */
  int n_kv_heads;          /* Hkv */
  int head_dim;            /* D: 64 or 128 */
  int page_size;           /* P: 16, 32 or 64 tokens (the per-entry slot mask is a u64) */
  int64_t n_pages;         /* pool size in pages, < 2^25 */
  void *const *k_pool;     /* [n_layers] device pointers (NULL for a host-only ctx) */
  void *const *v_pool;     /* [n_layers] device pointers */
  int32_t max_batch_rows;  /* max total query rows (sum of n_q) of one pred call */
  int32_t max_batch_descs; /* max descriptors of one pred call */
  int64_t table_capacity;  /* device table slab capacity in entries; 0 = 2*n_pages + 65536 */
  void *workspace;         /* device scratch, >= kvfs_workspace_bytes(cfg) bytes, 256-B aligned */
  size_t workspace_bytes;
} kvfs_config;

/* Bytes of device workspace kvfs_init needs for cfg (slab, upload area, split partials, counters). */
size_t kvfs_workspace_bytes(const kvfs_config *cfg);

/* Create a ctx over caller-owned pools (all pages free).  Validates shapes; ENOMEM if the workspace is
 * too small; EINVAL for unsupported shapes.  A device ctx zero-fills the pools once (synchronously), so
 * every pool slot always holds finite bf16 (the tensor-core kernel multiplies masked keys' V by P = 0). */
int kvfs_init(const kvfs_config *cfg, kvfs_ctx **out);

/* Synchronises the ctx's last stream use, frees host resources.  Device buffers stay the caller's. */
int kvfs_destroy(kvfs_ctx *ctx);

/* Human-readable name of an error code (static storage). */
const char *kvfs_strerror(int err);

/* ---------------------------------------------------------------- files (R2, R9) */
/* Open `name`, creating an empty file (no pages) with KVFS_O_CREAT; EEXIST with O_CREAT|O_EXCL if it
 * exists; ENOENT without O_CREAT if missing.  *fd is the smallest non-negative integer not open. */
int kvfs_open(kvfs_ctx *ctx, const char *name, int flags, int *fd);
/* Release the fd only (pages stay with the file).  EBADF if not open. */
int kvfs_close(kvfs_ctx *ctx, int fd);
/* kv_remove: drop every page reference of the file (refcount--, freed at 0) and remove
 * the name.  fds still open on it become EBADF for everything but kvfs_close. */
int kvfs_unlink(kvfs_ctx *ctx, const char *name);

/* kv_fork (R4): new file `dst_name` sharing every page of src (refcount++).  If src's tail
 * page has room, the child's tail is a fresh page (smallest free id, R1) holding a copy of the retained
 * slots (device copy of the whole page for every layer, K and V, enqueued on `stream`).  ENOSPC if that
 * page cannot be allocated, EEXIST if dst_name exists. */
int kvfs_fork(kvfs_ctx *ctx, int src_fd, const char *dst_name, int *dst_fd, kvfs_stream_t stream);

/* Keep logical tokens [0, new_len) (R5): later entries are dropped (refcount--), the last mask is trimmed,
 * positions are truncated.  ERANGE unless 0 <= new_len <= len.  Host only. */
int kvfs_truncate(kvfs_ctx *ctx, int fd, int64_t new_len);

/* Evict logical ranges (R6): ranges = [n_ranges][2] half-open [a, b), a < b, sorted, disjoint
 * (else EINVAL), within [0, len) (else ERANGE).  Clears mask bits, drops emptied entries; retained
 * positions are unchanged; no data moves.  With KVFS_EVICT_COMPACT the file is then
 * compacted (R7) in the same atomic call (R8), the page need being checked after the eviction. */
int kvfs_evict(kvfs_ctx *ctx, int fd, const int64_t *ranges, int n_ranges, int flags,
               kvfs_stream_t stream);

/* Compaction (R7): gather the retained tokens in logical order into ceil(len/P) fresh pages allocated
 * (smallest free first) while the old pages are still held, then release the old entries.  The device
 * gather (all layers, K and V) is enqueued on `stream`.  ENOSPC if the pages are not free.  No-op when
 * the file is empty. */
int kvfs_compact(kvfs_ctx *ctx, int fd, kvfs_stream_t stream);

/* Batched compaction (R7 for many files, e.g. a policy compacting every LIP after an eviction sweep,
 * P:225): kvfs_compact of fds[0..n) in that order (the same pages, tables and positions as n calls: R1
 * allocation sees each earlier file's releases), each file's device gather enqueued on `stream` in that
 * order (the next file's destinations may be the pages this one released), then the host position passes
 * on worker threads (on the calling thread if none can be started).  fds: host [n].  EBADF / EOFFLOAD
 * (nothing done) if an fd is invalid or offloaded, EBUSY if a file appears twice (as in a pred batch,
 * kvfs_merge and kvfs_pack); ENOSPC stops at the first file whose pages are not free, the files
 * before it being compacted.  *n_done (host, may be NULL) = files compacted. */
int kvfs_compact_files(kvfs_ctx *ctx, const int *fds, int n, int *n_done, kvfs_stream_t stream);

/* Append n tokens (R3) without attention (e.g. a prefilled prompt, "fills the file with the KV
 * cache").  pos: host [n] int32, strictly increasing and > the last retained position (else EPOS).
 * k, v: device [n_layers][n][n_kv_heads][head_dim] bf16 (may be NULL on a host-only ctx).
 * A shared tail page with room is copied first (copy-on-write). */
int kvfs_append(kvfs_ctx *ctx, int fd, int64_t n, const int32_t *pos, const void *k, const void *v,
                kvfs_stream_t stream);

/* ---------------------------------------------------------------- batched pred */
typedef struct {
  int32_t fd;   /* the LIP's KV file */
  int32_t n_q;  /* number of new tokens (query rows) of this LIP in the batch; 0 = no-op */
} pred_desc;

/* One layer (n_layers == 1) batched pred.  Descriptors are processed in order (R11): EBADF, EBUSY (the
 * file appeared in an earlier descriptor), EPOS, ENOSPC per descriptor; the others reserve their slots
 * (copy-on-write of a shared tail, smallest-free pages), append K_new/V_new and compute
 *   out[r][h] = sum_k softmax_k(scale * <q[r][h], K[k][g]>) V[k][g],   lse[r][h] = log sum_k exp(...)
 * over the file's retained tokens k with logical index <= len - n_q + i (row r = i-th row of the
 * descriptor, bottom-right-aligned causal; g = h / (Hq/Hkv)).
 *   pos    host [T] int32, T = sum of n_q (EINVAL if any n_q < 0 or T > max_batch_rows)
 *   q      device [T][Hq][D] bf16;  k_new, v_new device [T][Hkv][D] bf16
 *   out    device [T][Hq][D] bf16;  lse device [T][Hq] fp32 or NULL
 *   scale  > 0 (usually 1/sqrt(D))
 *   status host [n_desc] int, per-descriptor result (may be NULL)
 * Returns KVFS_OK, KVFS_EPARTIAL, or a call-level error (nothing changed). */
int pred_attn_batch(kvfs_ctx *ctx, const pred_desc *descs, int n_desc, const int32_t *pos,
                    const void *q, const void *k_new, const void *v_new, void *out, float *lse,
                    float scale, int *status, kvfs_stream_t stream);

/* pred_attn_batch with HOST buffers (the serving loop's end-to-end form: PAPER.md §4.4, the runtime
 * hands each batch's projected rows to the GPU and reads the attention output back).  Same arguments and
 * results as pred_attn_batch, except
 *   q, k_new, v_new  HOST [T][Hq][D] / [T][Hkv][D] bf16 (page-locked memory for asynchronous copies)
 *   out, lse         HOST [T][Hq][D] bf16 / [T][Hq] fp32 (lse may be NULL)
 * The library copies the inputs into one of two device slots on its own copy stream, runs the pred on
 * `stream` once they landed, and copies the rows of the descriptors that succeeded back on a second copy
 * stream (rows of failed descriptors are not written).  The call returns once this is enqueued: the host
 * may refill q / k_new / v_new only after the outputs of the same call are complete, and out / lse are
 * complete after pred_host_fence(ctx, s) followed by a synchronisation of s.  Consecutive calls overlap:
 * the input copy of call i+1 and the output copy of call i-1 run beside the pred of call i.
 * Errors: as pred_attn_batch; KVFS_ENOMEM if the device slots cannot grow; after a call-level error
 * nothing is copied out. */
int pred_attn_batch_host(kvfs_ctx *ctx, const pred_desc *descs, int n_desc, const int32_t *pos,
                         const void *q, const void *k_new, const void *v_new, void *out, float *lse,
                         float scale, int *status, kvfs_stream_t stream);
/* Make `stream` wait (no host wait) for every output copy pred_attn_batch_host issued so far. */
int pred_host_fence(kvfs_ctx *ctx, kvfs_stream_t stream);

/* Multi-layer form: pred_step_begin validates + reserves once (host metadata committed, device tables
 * and copy-on-write copies enqueued), then the caller issues pred_attn_layer for EVERY layer (append of
 * that layer's K_new/V_new fused with its attention), then pred_step_end.  Only one step may be open per
 * ctx; other calls on the ctx return EBUSY while it is open.  Same arguments as pred_attn_batch. */
int pred_step_begin(kvfs_ctx *ctx, const pred_desc *descs, int n_desc, const int32_t *pos, int *status,
                    pred_step **step, kvfs_stream_t stream);
int pred_attn_layer(kvfs_ctx *ctx, pred_step *step, int layer, const void *q, const void *k_new,
                    const void *v_new, void *out, float *lse, float scale, kvfs_stream_t stream);
int pred_step_end(kvfs_ctx *ctx, pred_step *step);
/* Attention-score accumulation for heavy-hitter (H2O-style) replacement policies (§6: the
 * key finer-grained interface is attention-level access, e.g. H2O; §4.2 P:225 the LIP then evicts the
 * "unimportant tokens").  After pred_attn_layer(step, layer, ... lse ...) of an open
 * step, for every successful descriptor d with n_q > 0 and every token k of its file after the append
 * (logical order, len_after = kvfs_stat len), writes
 *     scores[score_off[d] + k] = sum over the descriptor's query rows i and the Hq query heads h of
 *                                softmax_{i,h}(k)      (0 for a key row i cannot see; rule R10's weights)
 * i.e. exp(scale <q_ih, k_g(h)> - lse_ih) summed, from the SAME q and the lse that pred_attn_layer wrote.
 * q: device [T][Hq][D] bf16; lse: device [T][Hq] fp32 (as written by pred_attn_layer); scores: device fp32,
 * caller-owned; score_off: host [n_desc] (entries of failed or n_q = 0 descriptors are ignored).  Costs one
 * extra read of the files' K rows of that layer (HBM-bound, kernel K9).  EINVAL if lse or scores is NULL
 * or no step is open. */
int pred_attn_scores(kvfs_ctx *ctx, pred_step *step, int layer, const void *q, const float *lse, float scale,
                     float *scores, const int64_t *score_off, kvfs_stream_t stream);
/* Fused scores (same result as above, ~16x fewer bytes for decode descriptors).  Registers a caller-owned
 * device buffer (16-byte aligned; NULL or 0 bytes = off).  While registered, every pred_attn_layer's decode
 * kernel also writes the scaled logit of every key it attends, per head, for each descriptor it attends in
 * full (not chunk descriptors, not shared-prefix cascade members) that still fits in the buffer: a
 * descriptor takes 4 * Hq * P * n_q * (entries before the call + ceil(n_q / P)) bytes rounded up to 128, in
 * batch order.  The logits are written with an L2 evict-last policy and, when the buffer is 128-byte aligned
 * and P * Hq / Hkv is a multiple of 32, the score pass drops their L2 lines after reading them (no write-back):
 * with a buffer smaller than the L2 they need not reach DRAM at all.  A
 * pred_attn_scores for the most recent pred_attn_layer's layer then sums exp(logit - lse) from the buffer
 * for those descriptors (kernel K10) and falls back to the pass over K (K9) for the others.  The buffer must
 * stay valid until pred_step_end.  EBUSY while a step is open; EINVAL for a host-only ctx or a misaligned
 * buffer. */
int kvfs_set_logits_buffer(kvfs_ctx *ctx, void *buf, size_t bytes);

/* ---------------------------------------------------------------- introspection (tests, policies) */
typedef struct {
  int64_t len;        /* retained tokens */
  int64_t n_entries;  /* page entries */
  int32_t last_pos;   /* last retained position, -1 if empty */
  int32_t reserved;
} kvfs_stat_t;

int kvfs_stat(kvfs_ctx *ctx, int fd, kvfs_stat_t *st);
/* The file's page table: page ids and slot masks (bit s = slot s retained).  *n = n_entries; at most
 * cap are written. */
int kvfs_get_table(kvfs_ctx *ctx, int fd, uint32_t *page, uint64_t *mask, int64_t cap, int64_t *n);
int kvfs_get_positions(kvfs_ctx *ctx, int fd, int32_t *pos, int64_t cap, int64_t *n);
/* refcnt[p] for p < min(n, n_pages). */
int kvfs_get_refcounts(kvfs_ctx *ctx, uint32_t *refcnt, int64_t n);
int kvfs_free_pages(kvfs_ctx *ctx, int64_t *n_free);
/* Gather logical tokens [begin, end) of one layer into dense device k_out/v_out [end-begin][Hkv][D]. */
int kvfs_read(kvfs_ctx *ctx, int fd, int layer, int64_t begin, int64_t end, void *k_out, void *v_out,
              kvfs_stream_t stream);
/* Recompute refcounts from the tables and check invariants I1-I5 (§8(c) C2).  EIO-free: returns
 * KVFS_EINVAL (and leaves state as is) if an invariant is violated. */
int kvfs_audit(kvfs_ctx *ctx);

/* ---------------------------------------------------------------- migration */
/* Pack a file set for transfer to another ctx (another GPU): the set's distinct pages, in ascending
 * source page id (a page shared by several files of the set is packed once, so CoW sharing inside the
 * set survives the move; pages shared with files outside the set are duplicated), are gathered into
 * buf_dev as [n_layers][K, V][n_unique][n_kv_heads][page_size][head_dim] bf16 (device, K6 gather on
 * `stream`), and hdr (host) receives the tables relative to that order plus positions:
 *   u32 magic 'KVP1', u32 version 1, u32 n_files, u32 n_unique, u32 P, L, Hkv, D, u64 bytes per page
 *   per layer per K|V; then per file: u32 n_entries, u32 n_tokens, n_entries x {u32 local page, u32 0,
 *   u64 mask}, n_tokens x i32 positions (logical order).
 * The source files are not modified (the caller unlinks them after the transfer).  ENOMEM with
 * *buf_used / *hdr_used set to the sizes needed if a capacity is too small; EBADF for a bad fd; EBUSY
 * if a file appears twice.  A host-only ctx packs the header only (buf_dev may be NULL). */
int kvfs_pack(kvfs_ctx *ctx, const int *fds, int n_fds, void *buf_dev, size_t buf_cap, size_t *buf_used,
              void *hdr, size_t hdr_cap, size_t *hdr_used, kvfs_stream_t stream);
/* Create files names[i] from a packed set: n_unique pages are allocated smallest-free first in packed order
 * (R1), buf_dev is scattered into them (device, on `stream`), tables and positions are rebuilt and the
 * refcounts count the sharing within the set.  fds_out[i] receives the new fds.  buf_bytes = the size of
 * buf_dev as received (device ctx: EINVAL, nothing done, if it is smaller than the header's n_unique x
 * L x 2 x page bytes, e.g. a truncated transfer or a header from another pack; ignored by a host-only
 * ctx).  EINVAL for a malformed header or a shape mismatch, EEXIST if a name exists, ENOSPC if the
 * pages are not free (atomic). */
int kvfs_unpack(kvfs_ctx *ctx, const void *buf_dev, size_t buf_bytes, const void *hdr, size_t hdr_bytes,
                const char *const *names, int *fds_out, kvfs_stream_t stream);

/* ---------------------------------------------------------------- new files from existing ones
 * PAPER.md §4.2: LIPs "create new files from existing ones by extracting specific token indices with
 * extract, or merging existing files into one with merge".  Both build a NEW file whose
 * pages are rebuilt (no sharing: a selection or an interleaving breaks page alignment): k tokens go to
 * ceil(k/P) fresh pages allocated smallest-free first in the new file's logical order (rule R1), token i
 * at (page i / P, slot i % P), every retained token keeping its original absolute position.  The K/V bits
 * of every layer are gathered on `stream` (device; a host-only ctx builds the metadata only).  The sources
 * are unchanged.  Atomic: a failing call changes nothing.
 *
 * kvfs_extract: indices[n] = LOGICAL token indices of src, strictly increasing (EINVAL otherwise), each in
 *   [0, len) (ERANGE); n = 0 gives an empty file.  Errors: EBADF, EINVAL, ERANGE, EEXIST (name exists),
 *   ENOSPC (not enough free pages), in that order of checking.
 * kvfs_merge: the union of the parts' retained tokens sorted by position; two tokens with the same
 *   position (in one or in different parts) are EPOS (overlap semantics are undefined in the
 *   paper, so they are rejected); a part listed twice is EBUSY.  Errors: EBADF, EBUSY, EPOS, EEXIST, ENOSPC.
 * *fd receives the new file's fd (open, like kvfs_open). */
int kvfs_extract(kvfs_ctx *ctx, int src_fd, const int64_t *indices, int64_t n, const char *name, int *fd,
                 kvfs_stream_t stream);
int kvfs_merge(kvfs_ctx *ctx, const int *fds, int n_fds, const char *name, int *fd, kvfs_stream_t stream);

/* ---------------------------------------------------------------- host tier: offload / restore
 * PAPER.md §4.3: while a thread waits on I/O, Symphony "offloads their KV caches from the GPU to the
 * CPU and restores them upon I/O completion".  Rule R15: kvfs_offload moves every page the
 * file owns EXCLUSIVELY (refcount 1) to a pinned host buffer owned by the ctx (recycled between files) (bits of every layer, K and V,
 * copied by the page-pack kernel writing through the mapped host pointer on `stream`) and frees it on the
 * device; pages shared with other files stay (another file may need them).  In the table such an entry's
 * page reads KVFS_HOST_PAGE | host slot (slots in table order).  kvfs_restore allocates device pages
 * smallest-free first in table order for those entries (ENOSPC, atomic, if too few are free), copies the
 * bits back on `stream` (the host buffer is recycled once that copy is done; no host wait).  While offloaded the file is
 * EOFFLOAD for append / pred (per-descriptor status) / fork / truncate / evict / compact / extract / merge /
 * read / pack; stat, tables, positions, close and unlink work (unlink drops the host copy).  kvfs_offload of
 * an offloaded file, or kvfs_restore of one that is not, is EINVAL.  *moved (nullable) = pages moved. */
#define KVFS_HOST_PAGE 0x80000000u
int kvfs_offload(kvfs_ctx *ctx, int fd, int64_t *moved, kvfs_stream_t stream);
int kvfs_restore(kvfs_ctx *ctx, int fd, int64_t *moved, kvfs_stream_t stream);

/* ---------------------------------------------------------------- inference scheduler: batch formation
 * PAPER.md §4.4: the inference scheduler "aggregates multiple pred system calls into a single
 * batch"; executing too early under-uses the GPU, too late makes threads wait; Symphony "dynamically adjusts
 * batch size according to the average frequency of system calls, leveraging models like Poisson process".
 * Reading (S1): lam = EWMA of 1/dt over enqueue gaps (first enqueue: 1/dt_default;
 * dt floored at 1e-9); target B* = clamp(round(lam * w_max), 1, b_max) = expected arrivals within w_max;
 * a batch is due when >= B* requests wait or the oldest waited >= w_max; it is the waiting requests in FIFO
 * order, at most b_max, a request whose fd is already in the batch staying queued (one pred per file per
 * batch).  Times are caller-supplied seconds (any monotonic clock).  Host only; no device work. */
typedef struct kvfs_sched kvfs_sched;
typedef struct {
  double w_max;      /* max wait of the oldest request (s), > 0 */
  int b_max;         /* max batch size (descriptors), >= 1 */
  double alpha;      /* EWMA weight in (0, 1] */
  double dt_default; /* initial mean gap (s), > 0 */
} kvfs_sched_config;
int kvfs_sched_create(const kvfs_sched_config *cfg, kvfs_sched **out); /* EINVAL for a bad config */
int kvfs_sched_destroy(kvfs_sched *s);
/* Queue one pred request: fd, its n_q positions (host, copied). */
int kvfs_sched_enqueue(kvfs_sched *s, int fd, int n_q, const int32_t *pos, double now);
/* Current rate estimate lam (1/s) and target B*. */
int kvfs_sched_state(kvfs_sched *s, double *lambda, int *target, int *n_waiting);
/* If a batch is due at `now`: write its descriptors and packed positions (rows in descriptor order, the
 * layout pred_attn_batch takes), remove them from the queue and return 1; else return 0 and write nothing.
 * ENOMEM (nothing removed) if desc_cap / pos_cap are too small for the batch. */
int kvfs_sched_form(kvfs_sched *s, double now, pred_desc *descs, int desc_cap, int32_t *pos, int64_t pos_cap,
                    int *n_desc, int64_t *n_rows);

/* ---------------------------------------------------------------- knobs and counters */
typedef enum {
  KVFS_OPT_DECODE_CTAS = 1,     /* grid size of the decode kernel; 0 = auto (SM count x occupancy) */
  KVFS_OPT_CHUNK_CUTOVER = 2,   /* n_q at or above which the tcgen05 chunk kernel is used (head_dim 128);
                                   0 = never; default 2: the decode kernel streams a file once per query row
                                   (ncu, cfg2 shape with n_q = 4 drafts: 4.0x the K/V bytes, 1.29 ms), the chunk
                                   kernel once per (descriptor, kv head) (1.0x, 0.44 ms) */
  KVFS_OPT_DETERMINISTIC = 3,   /* reserved (the kernels are deterministic for a fixed grid) */
  KVFS_OPT_CASCADE_MIN_ENTRIES = 4 /* shared-prefix ("cascade") decode for CoW fork families (§4.2
                                   P:223 fork shares pages): decode descriptors (n_q
                                   below the chunk cut-over) whose files share a leading run of at least this
                                   many identical (page, mask) entries, all before their new tokens, have
                                   that run attended ONCE per batch by the tcgen05 kernel over all sharers'
                                   query rows, and the per-file rest by the decode kernel, merged exactly
                                   (log-sum-exp).  0 = off; default 16 (head_dim 128 only) */,
  KVFS_OPT_PREFIX_SPLITS = 5,   /* key splits of each shared run in the cascade (1..16); 0 = auto */
  KVFS_OPT_DECODE_CHUNKS = 8,   /* decode-kernel scheduling: 0 = static (ring r streams the r-th of
                                   KVFS_OPT_DECODE_CTAS equal contiguous stage ranges; default); n in 1..2048 =
                                   dynamic: the batch's stages are cut into n equal ranges that at most one
                                   wave of rings takes from a device counter as they finish (load balance when
                                   some SMs are busy, e.g. with the cascade's shared-prefix kernel) */
  KVFS_OPT_TIMING = 7,          /* 1: kvfs_compact_files records CUDA events around its device work (file
                                   groups: upload + gathers) and, before returning, waits for them and
                                   stores their summed device time in KVFS_CTR_COMPACT_DEVICE_NS (the host
                                   R1 / table work that overlaps it excluded); pred_attn_layer records
                                   events around its kernels (chunk, shared-prefix, decode), summed by
                                   KVFS_CTR_LAYER_DEVICE_NS; n > 1: only every n-th pred_attn_layer call
                                   (counted from this setting; the first is timed) records them
                                   (KVFS_CTR_LAYER_TIMED counts the timed calls); 0 = off (default) */
  KVFS_OPT_HOLES_GATHER = 9,    /* decode kernel, page entries whose retained slots fill less than 40% of
                                   their [lowest, highest] span (heavy lazy eviction): 1 = fetch only the
                                   retained rows with TMA gather4 (4 rows per copy, packed in shared memory;
                                   default), 0 = always copy the whole span (reads the holes too) */
  KVFS_OPT_PREFIX_PAIRED = 10,  /* cascade: 0 = the cost model may pick the paired partition (the (kv head,
                                   M-tile pair) lanes of a shared run taken in pairs, 3 key pieces each, 5
                                   prefix CTAs per pair, one of them running two short pieces in turn; the
                                   decode kernel folds the 3 records), 1 = never, 2 = whenever possible */
  KVFS_OPT_FAULT_INJECT = 6     /* tests only: value n > 0 makes the n-th following pass through an
                                   injection point (mid-way through a pred reservation, after the first
                                   descriptor is committed; fork; open) throw std::bad_alloc inside the
                                   library, to exercise the no-exception guarantee above; 0 = off */
} kvfs_option;
int kvfs_set_option(kvfs_ctx *ctx, int option, int64_t value);

typedef enum {
  KVFS_CTR_KERNEL_LAUNCHES = 1, /* CUDA kernels this ctx has launched */
  KVFS_CTR_H2D_BYTES = 2,       /* bytes of host->device metadata uploads */
  KVFS_CTR_PAGE_COPIES = 3,     /* whole-page copies (copy-on-write + fork tails), per page */
  KVFS_CTR_LAST_DECODE_CTAS = 4, /* grid (virtual CTAs = rings) of the last decode launch */
  KVFS_CTR_LAST_CHUNK_UNITS = 5, /* CTAs of the last tcgen05 chunk launch (0: none) */
  KVFS_CTR_LAST_PREFIX_UNITS = 6,  /* CTAs of the last shared-prefix (cascade) launch (0: none) */
  KVFS_CTR_LAST_PREFIX_GROUPS = 7, /* fork families (groups) the last pred batch attended as shared prefixes */
  KVFS_CTR_HOST_PAGES = 8,         /* pages currently in the host tier (kvfs_offload) */
  KVFS_CTR_COMPACT_DEVICE_NS = 9,  /* KVFS_OPT_TIMING: device time of the last kvfs_compact_files (ns) */
  KVFS_CTR_LAYER_DEVICE_NS = 10,   /* KVFS_OPT_TIMING: summed device time (ns) of the pred_attn_layer calls
                                      recorded since the previous read of this counter, from the event
                                      before a layer's first kernel to the event after its last (reading
                                      waits for them and starts a new sum) */
  KVFS_CTR_LAYER_TIMED = 11,       /* KVFS_OPT_TIMING: number of pred_attn_layer calls in the last
                                      KVFS_CTR_LAYER_DEVICE_NS sum */
  /* Host time (ns, summed since kvfs_init) of the phases of pred_step_begin / pred_attn_layer: the
     reservation and plan of the batch (R11), the chunk split + shared-prefix planning, the metadata upload
     + prologue launch, and pred_attn_layer's kernel launches.  Host-cost observability. */
  KVFS_CTR_HOST_RESERVE_NS = 12,
  KVFS_CTR_HOST_SPLIT_NS = 13,
  KVFS_CTR_HOST_UPLOAD_NS = 14,
  KVFS_CTR_HOST_LAUNCH_NS = 15,
  KVFS_CTR_COPY_DEVICE_NS = 16,    /* KVFS_OPT_TIMING: summed device time (ns) of the whole-page pack /
                                      unpack kernel launches (kvfs_pack, kvfs_unpack, kvfs_offload,
                                      kvfs_restore) since the previous read (reading waits for them) */
  KVFS_CTR_LAST_FUSED_SCORES = 17  /* descriptors the last pred_attn_scores served from the decode kernel's
                                      logits (K10); the rest went through K9 */
} kvfs_counter;
int kvfs_get_counter(kvfs_ctx *ctx, int counter, int64_t *value);

#ifdef __cplusplus
}
#endif
#endif /* KVFS_H_ */
