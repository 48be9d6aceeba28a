// Device data plane of KVFS: workspace layout, the per-call metadata upload (one pinned H2D copy per
// call), and the bandwidth-bound copy kernels (K4 copy-on-write / fork tail page copy, K5 evict-compact
// gather, K7 dense read-back, the kvfs_append scatter, the table-delta scatter).  The attention kernel
// lives in decode_attn.cu.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "../host/kvfs_impl.h"
#include "kernels.cuh"

namespace kvfs {

namespace {

constexpr int kMaxCtas = 2048;

size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

struct WsLayout {
  size_t slab = 0, upload = 0, counters = 0, partials = 0, ptrs = 0, prefix = 0, total = 0, upload_cap = 0;
  size_t scratch = 0, scratch_cap = 0;  // second upload area: packets sent while a pred step is open
  size_t work = 0;                      // [2] int: K1 dynamic-scheduling counters (self-resetting)
  size_t pgroup = 0;                    // [2][kMaxPrefixGroups] int: shared-prefix split-group counters
  int64_t prefix_cap = 0;  // shared-prefix partials (PART floats each)
};

WsLayout ws_layout(const kvfs_config &c) {
  WsLayout w;
  const int G = c.n_q_heads / c.n_kv_heads;
  const size_t part = static_cast<size_t>(dev::part_floats(G, c.head_dim)) * 4;
  size_t off = 0;
  w.slab = off;
  off = align256(off + static_cast<size_t>(c.table_capacity) * 16);
  w.upload = off;
  w.upload_cap = align256(static_cast<size_t>(c.table_capacity) * 16 + static_cast<size_t>(c.n_pages) * 24 +
                          static_cast<size_t>(c.max_batch_descs) * 96 + static_cast<size_t>(c.max_batch_rows) * 8 +
                          (1u << 20));
  off = align256(off + w.upload_cap);
  // The open step's plan (descriptors, destination slots, chunk / prefix records) stays in the upload area
  // until pred_step_end; the only call allowed between the layers of an open step that uploads anything is
  // pred_attn_scores (every other op is EBUSY), so its packet goes here instead: ScoreDesc (24 B) per
  // descriptor + one ScoreUnit (16 B) per <= 8..32 table entries of the batch's files (<= table_capacity).
  w.scratch = off;
  w.scratch_cap = align256(static_cast<size_t>(c.max_batch_descs) * 48 + static_cast<size_t>(c.table_capacity) * 2 +
                           (size_t{1} << 16));
  off = align256(off + w.scratch_cap);
  w.counters = off;
  off = align256(off + static_cast<size_t>(c.max_batch_rows) * c.n_kv_heads * 4);
  w.work = off;
  off = align256(off + 16);
  w.pgroup = off;
  off = align256(off + 2 * static_cast<size_t>(kMaxPrefixGroups) * 4);
  w.partials = off;
  off = align256(off + static_cast<size_t>(kMaxCtas) * dev::kDecodeRecSlots * part);
  w.ptrs = off;
  off = align256(off + static_cast<size_t>(c.n_layers) * 2 * sizeof(void *));
  // shared-prefix (cascade) partials: one merged partial per decode unit + up to kMaxPrefixSplits split
  // partials, capped at 16384 + the merged ones
  w.prefix_cap = c.head_dim == 128
                     ? std::min<int64_t>(static_cast<int64_t>(c.max_batch_rows) * c.n_kv_heads * (kMaxPrefixSplits + 1),
                                         16384 + static_cast<int64_t>(c.max_batch_rows) * c.n_kv_heads)
                     : 0;
  w.prefix = off;
  off = align256(off + static_cast<size_t>(w.prefix_cap) * part);
  w.total = off;
  return w;
}

// ------------------------------------------------------------------------------------------ kernels
using bf16 = __nv_bfloat16;

// The step's metadata packet from mapped pinned host memory into the device upload area, by SM loads over
// PCIe instead of a copy-engine DMA: the DMA would queue behind the caller's own (large) input copies on
// the copy engines and stall the compute stream (bytes a multiple of 16, both ends 16-byte aligned).
__global__ void upload_kernel(uint4 *dst, const uint4 *src, int64_t n16) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

// A pred step's metadata packet and its device-table work in ONE launch (replaces a DMA of the packet and
// a separate prologue launch: the copy engine's latency plus a kernel boundary, ~5 us per step on B200):
// every CTA copies a slice of the packet from mapped pinned host memory into the device upload area (the
// later kernels of the step read it there), and the table deltas / copy-on-write pages are applied from
// the HOST copy of the same packet (no dependency on the device copy inside this grid).
// Each table delta is (slab index, entry) read independently from host memory, so the deltas cost one
// PCIe round trip, in parallel with the packet copy (a run list first, then its entries, cost two).
__global__ void step_prologue_kernel(uint4 *dst, const uint4 *src, int64_t n16, const int64_t *delta_dst,
                                     int n_deltas, const dev::Entry *delta_entries, dev::Entry *slab,
                                     const dev::PageCopy *copies, int n_copies, bf16 *const *kp, bf16 *const *vp, int L,
                                     int64_t page_elems) {
  asm volatile("griddepcontrol.launch_dependents;");
  // Launched programmatically after the previous step's last kernel, whose trigger comes early: this grid's
  // launch and its host-memory reads (the packet and the deltas live in this step's pinned staging buffer,
  // which no running grid reads) overlap that kernel's tail; the stores into the upload area and the slab,
  // which it reads, wait for it (griddepcontrol.wait).
  const int delta_blocks = (n_deltas + 255) / 256;
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t ddst = -1;
  dev::Entry de{};
  if (static_cast<int>(blockIdx.x) < delta_blocks && j < n_deltas) {
    ddst = delta_dst[j];
    de = delta_entries[j];
  }
  constexpr int PRE = 4;  // packet vectors per thread loaded before the wait
  uint4 pv[PRE];
#pragma unroll
  for (int k = 0; k < PRE; ++k)
    if (j + k * stride < n16) pv[k] = src[j + k * stride];
  asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
  for (int k = 0; k < PRE; ++k)
    if (j + k * stride < n16) dst[j + k * stride] = pv[k];
  for (int64_t i = j + PRE * stride; i < n16; i += stride) dst[i] = src[i];
  if (static_cast<int>(blockIdx.x) < delta_blocks) {
    if (ddst >= 0) slab[ddst] = de;
    return;
  }
  const int b = blockIdx.x - delta_blocks;
  const int ci = b / (2 * L), rem = b % (2 * L), l = rem >> 1, isv = rem & 1;
  if (ci >= n_copies) return;
  const dev::PageCopy pc = copies[ci];
  const bf16 *pool = isv ? vp[l] : kp[l];
  const uint4 *ps = reinterpret_cast<const uint4 *>(pool + static_cast<int64_t>(pc.src) * page_elems);
  uint4 *pd = reinterpret_cast<uint4 *>(const_cast<bf16 *>(pool) + static_cast<int64_t>(pc.dst) * page_elems);
  const int64_t m16 = page_elems / 8;
  for (int64_t i = threadIdx.x; i < m16; i += blockDim.x) pd[i] = ps[i];
}

// Table deltas into the slab (one warp per run) and whole-page copies (one CTA per page, layer, K|V).
__global__ void prologue_kernel(const dev::SlabRun *runs, int n_runs, const dev::Entry *run_entries,
                                dev::Entry *slab, const dev::PageCopy *copies, int n_copies, bf16 *const *kp,
                                bf16 *const *vp, int L, int64_t page_elems) {
  // the next kernel (decode / shared-prefix, launched programmatically) may start its setup now; it waits
  // (griddepcontrol.wait) for this grid's completion before reading the tables
  asm volatile("griddepcontrol.launch_dependents;");
  const int run_blocks = (n_runs + 7) / 8;
  if (static_cast<int>(blockIdx.x) < run_blocks) {
    const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (r >= n_runs) return;
    const dev::SlabRun run = runs[r];
    for (int i = threadIdx.x & 31; i < run.count; i += 32) slab[run.dst + i] = run_entries[run.src + i];
    return;
  }
  const int b = blockIdx.x - run_blocks;
  const int ci = b / (2 * L), rem = b % (2 * L), l = rem >> 1, isv = rem & 1;
  if (ci >= n_copies) return;
  const bf16 *pool = isv ? vp[l] : kp[l];
  const uint4 *src = reinterpret_cast<const uint4 *>(pool + static_cast<int64_t>(copies[ci].src) * page_elems);
  uint4 *dst = reinterpret_cast<uint4 *>(const_cast<bf16 *>(pool) + static_cast<int64_t>(copies[ci].dst) * page_elems);
  const int64_t n16 = page_elems / 8;
  for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
}

// kvfs_append scatter: rows [row_base, row_base + n) of k/v [L][n_total][Hkv][D] -> pool slots
// dst[r] = page * P + slot.
__global__ void append_rows_kernel(const int32_t *dst, int64_t n, int64_t row_base, int64_t n_total, const bf16 *k,
                                   const bf16 *v, bf16 *const *kp, bf16 *const *vp, int L, int Hkv, int D, int P) {
  const int cpr = D / 8;
  const int64_t total = static_cast<int64_t>(L) * n * Hkv * cpr;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(idx % cpr);
    int64_t t = idx / cpr;
    const int g = static_cast<int>(t % Hkv);
    t /= Hkv;
    const int64_t r = t % n;
    const int l = static_cast<int>(t / n);
    const int32_t ds = dst[r];
    const int64_t so = ((static_cast<int64_t>(l) * n_total + row_base + r) * Hkv + g) * D + c * 8;
    const int64_t po = ((static_cast<int64_t>(ds / P) * Hkv + g) * P + ds % P) * D + c * 8;
    *reinterpret_cast<uint4 *>(kp[l] + po) = *reinterpret_cast<const uint4 *>(k + so);
    *reinterpret_cast<uint4 *>(vp[l] + po) = *reinterpret_cast<const uint4 *>(v + so);
  }
}

// extract / merge (R13, R14): token i of the new file <- pool slot src[i] (page * P + slot), into
// (new_pages[i / P], i % P), every layer, K and V.  One CTA per (destination page, layer), 16-byte vectors.
__global__ void __launch_bounds__(256) gather_kernel(const int32_t *src, int64_t n, const uint32_t *new_pages,
                                                     bf16 *const *kp, bf16 *const *vp, int Hkv, int D, int P) {
  const int j = blockIdx.x, l = blockIdx.y;
  const int64_t i0 = static_cast<int64_t>(j) * P;
  const int ntok = static_cast<int>(n - i0 < P ? n - i0 : static_cast<int64_t>(P));
  bf16 *kk = kp[l];
  bf16 *vv = vp[l];
  const int cpr = D / 8;
  const int total = Hkv * ntok * cpr;
  const int64_t dpage = new_pages[j];
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int c = idx % cpr, r = idx / cpr, t = r % ntok, g = r / ntok;
    const int32_t sl = src[i0 + t];
    const int64_t so = ((static_cast<int64_t>(sl / P) * Hkv + g) * P + sl % P) * D + c * 8;
    const int64_t po = ((dpage * Hkv + g) * P + t) * D + c * 8;
    const uint4 a = *reinterpret_cast<const uint4 *>(kk + so);
    const uint4 b = *reinterpret_cast<const uint4 *>(vv + so);
    *reinterpret_cast<uint4 *>(kk + po) = a;
    *reinterpret_cast<uint4 *>(vv + po) = b;
  }
}

__device__ __forceinline__ int find_entry(const dev::Entry *t, int n, int64_t i) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (t[mid].lstart <= i) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// K5: compaction gather (R7).  Token i of the old table (logical order) -> (new_pages[i / P], i % P), every
// layer, K and V.  The unit of work is a destination BLOCK = one (page, layer, K|V, kv head): P rows of D bf16,
// contiguous in the pool (P * D * 2 bytes, 4 KiB at the 8B shape).  Blocks are ordered (page, layer, K|V,
// head) and cut into 32 KiB stages; each CTA takes a contiguous range of stages (so a contiguous range of
// destination pages) and pipelines them through kK5Stages shared-memory buffers:
//   * sources: every row is a 256-byte (D = 128) scattered read (holes): the 256 threads issue 16-byte
//     cp.async (LDGSTS) copies straight into the stage buffer, laid out as the destination blocks -- the
//     bytes in flight live in shared memory, not in registers (the round-1 register-held copy kept only
//     ~128 B per thread in flight: 0.46 eligible warps per scheduler, 3.9 TB/s);
//   * destinations: one 1-D TMA bulk store (cp.async.bulk.global.shared::cta) per block, issued by one
//     lane per block of warp 0 -- whole 4 KiB contiguous writes.
// Source (page, slot) of every token of the CTA's pages is resolved once per chunk of pages into shared
// memory from `first_entry[j]` (host: the old entry holding token j * P), walking forward <= P entries.
// Programmatic dependent launch (kvfs_compact_files chains one launch per file, R1 order): the grid reads
// its own sources at once (a later file's sources were held while earlier files compacted, so no earlier
// grid writes them) and executes griddepcontrol.wait before its first store (its destinations may be the
// pages the previous file just released, i.e. the previous grid's sources).
constexpr int kK5Threads = 256;
constexpr int kK5StageBytes = 32768;
constexpr int kK5Stages = 3;
constexpr int kK5SrcCap = 1024;  // tokens whose sources are resolved at a time
constexpr int kK5MaxBps = 16;    // blocks per stage (block >= 2 KiB)
struct K5Block {                 // one destination block of a stage (shared memory)
  const bf16 *src_pool;          // the layer's K or V pool
  bf16 *dst;                     // destination block (page new_pages[j], kv head g, slot 0)
  int32_t gP;                    // g * P (row offset of the head inside a page)
  int32_t k0;                    // index of the block's first token in the resolved chunk
  int32_t ntok;                  // rows (P, or fewer on the last page; 0: past the end)
  int32_t pad;
};
constexpr int kK5Smem = kK5Stages * kK5StageBytes + kK5SrcCap * 8 + kK5Stages * kK5MaxBps * 32 + 128;

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}

__global__ void __launch_bounds__(kK5Threads, 2)
compact_kernel(const dev::Entry *old, int n_old, const uint32_t *new_pages, const int32_t *first_entry, int n_new,
               int64_t len, bf16 *const *kp, bf16 *const *vp, int L, int Hkv, int lgD, int lgP) {
  asm volatile("griddepcontrol.launch_dependents;");
  extern __shared__ __align__(128) unsigned char k5_smem[];
  unsigned char *stage_base = k5_smem;
  uint32_t *src_page = reinterpret_cast<uint32_t *>(k5_smem + kK5Stages * kK5StageBytes);
  int32_t *src_slot = reinterpret_cast<int32_t *>(src_page + kK5SrcCap);
  K5Block *blk = reinterpret_cast<K5Block *>(src_slot + kK5SrcCap);  // [kK5Stages][kK5MaxBps]
  const int tid = threadIdx.x;
  const int P = 1 << lgP, D = 1 << lgD;
  const int lg_cpr = lgD - 3;                            // 16-byte chunks per row: D / 8
  const int lg_blk_chunks = lgP + lg_cpr;                // chunks per block
  const int bps = kK5StageBytes >> (lg_blk_chunks + 4);  // blocks per stage
  const int bpp = L * 2 * Hkv;                           // blocks per destination page
  const int64_t nb = static_cast<int64_t>(n_new) * bpp;
  const int64_t n_stages = (nb + bps - 1) / bps;
  const int64_t q0 = n_stages * blockIdx.x / gridDim.x, q1 = n_stages * (blockIdx.x + 1) / gridDim.x;
  if (q0 >= q1) return;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(stage_base));
  const int chunk_pages = kK5SrcCap >> lgP;
  int64_t cj0 = -1;  // first page of the resolved chunk

  // resolve the sources of pages [j0, j0 + chunk_pages) into src_page / src_slot (all threads)
  auto resolve = [&](int64_t j0) {
    __syncthreads();  // every thread is done computing addresses from the previous chunk
    const int64_t i_begin = j0 << lgP;
    const int64_t i_end = min(len, i_begin + kK5SrcCap);
    for (int64_t i = i_begin + tid; i < i_end; i += kK5Threads) {
      int e = first_entry[i >> lgP];
      dev::Entry en = old[e];
      while (e + 1 < n_old && en.lstart + __popcll(en.mask) <= i) en = old[++e];
      src_page[i - i_begin] = en.page;
      src_slot[i - i_begin] = dev::select_bit64(en.mask, static_cast<int>(i - en.lstart));
    }
    cj0 = j0;
    __syncthreads();
  };
  // issue the cp.async copies of stage q into buffer `buf` (one commit group per call, possibly empty)
  auto issue = [&](int64_t q, int buf) {
    if (q < q1) {  // uniform
      const int64_t b0 = q * bps;
      const int64_t jf = b0 / bpp;
      const int r0 = static_cast<int>(b0 - jf * bpp);
      const int64_t jl = min(nb - 1, b0 + bps - 1) / bpp;  // last page of the stage
      if (cj0 < 0 || jl >= cj0 + chunk_pages) resolve(jf);
      K5Block *bd = blk + buf * kK5MaxBps;
      if (tid < bps) {  // the stage's block descriptors (also read by the stores, kK5Stages - 1 iterations later)
        const int rr = r0 + tid;
        const int64_t j = jf + rr / bpp;
        const int r = rr % bpp;
        const int g = r % Hkv, kv = (r / Hkv) & 1, l = r / (2 * Hkv);
        K5Block d{};
        if (b0 + tid < nb) {
          bf16 *pool = kv ? vp[l] : kp[l];
          d.src_pool = pool;
          d.dst = pool + ((static_cast<int64_t>(new_pages[j]) * Hkv + g) << (lgP + lgD));
          d.gP = g << lgP;
          d.k0 = static_cast<int32_t>((j - cj0) << lgP);
          d.ntok = static_cast<int32_t>(min(static_cast<int64_t>(P), len - (j << lgP)));
        }
        bd[tid] = d;
      }
      __syncthreads();
      const uint32_t sb = sbase + buf * kK5StageBytes;
      const int HkvP = Hkv << lgP;
      // kK5StageBytes / 16 chunks per stage = (block, row, 16-byte chunk), chunk fastest (coalesced rows)
#pragma unroll 4
      for (int x = tid; x < kK5StageBytes / 16; x += kK5Threads) {
        const K5Block &d = bd[x >> lg_blk_chunks];
        const int t = (x >> lg_cpr) & (P - 1);
        if (t >= d.ntok) continue;
        const int k = d.k0 + t;
        const int64_t row = static_cast<int64_t>(src_page[k]) * HkvP + d.gP + src_slot[k];
        cp_async16(sb + (x << 4), d.src_pool + (row << lgD) + ((x & ((1 << lg_cpr) - 1)) << 3));
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  for (int k = 0; k < kK5Stages - 1; ++k) issue(q0 + k, k);
  for (int64_t q = q0; q < q1; ++q) {
    const int buf = static_cast<int>((q - q0) % kK5Stages);
    asm volatile("cp.async.wait_group %0;" ::"n"(kK5Stages - 2) : "memory");  // this thread's part of stage q
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the async (TMA) proxy
    __syncthreads();
    if (tid < 32) {
      if (q == q0) asm volatile("griddepcontrol.wait;" ::: "memory");  // before the first write (see above)
      const K5Block &d = blk[buf * kK5MaxBps + (tid < bps ? tid : 0)];
      if (tid < bps && d.ntok > 0) {
        const uint32_t src = sbase + buf * kK5StageBytes + (tid << (lg_blk_chunks + 4));
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d.dst), "r"(src),
                     "r"(d.ntok << (lgD + 1))
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      // the buffer refilled next held stage q - 1: its bulk stores must have finished reading it
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    }
    __syncthreads();
    issue(q + kK5Stages - 1, static_cast<int>((q - q0 + kK5Stages - 1) % kK5Stages));
  }
  if (tid < 32) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // writes performed before exit
}

// K6: whole pages <-> a packed buffer [L][K, V][n][page_elems] (migration pack / unpack).
__global__ void pack_kernel(const uint32_t *pages, int n, bf16 *const *kp, bf16 *const *vp, int L, int64_t page_elems,
                            bf16 *buf, int unpack) {
  const int b = blockIdx.x;
  const int j = b % n, rem = b / n, isv = rem & 1, l = rem >> 1;
  bf16 *pool = isv ? vp[l] : kp[l];
  uint4 *pg = reinterpret_cast<uint4 *>(pool + static_cast<int64_t>(pages[j]) * page_elems);
  uint4 *bb = reinterpret_cast<uint4 *>(buf + ((static_cast<int64_t>(l) * 2 + isv) * n + j) * page_elems);
  const int64_t n16 = page_elems / 8;
  if (unpack) {
    for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) pg[i] = bb[i];
  } else {
    for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) bb[i] = pg[i];
  }
}

// K7: logical tokens [begin, end) of one layer -> dense [n][Hkv][D].
__global__ void read_kernel(const dev::Entry *t, int n_ent, int64_t begin, int64_t end, const bf16 *kpl,
                            const bf16 *vpl, bf16 *kout, bf16 *vout, int Hkv, int D, int P) {
  const int cpr = D / 8;
  const int64_t n = end - begin;
  const int64_t total = n * Hkv * cpr;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(idx % cpr);
    int64_t r = idx / cpr;
    const int g = static_cast<int>(r % Hkv);
    r /= Hkv;
    const int64_t i = begin + r;
    const dev::Entry e = t[find_entry(t, n_ent, i)];
    const int slot = dev::select_bit64(e.mask, static_cast<int>(i - e.lstart));
    const int64_t so = ((static_cast<int64_t>(e.page) * Hkv + g) * P + slot) * D + c * 8;
    const int64_t doff = (r * Hkv + g) * D + c * 8;
    *reinterpret_cast<uint4 *>(kout + doff) = *reinterpret_cast<const uint4 *>(kpl + so);
    *reinterpret_cast<uint4 *>(vout + doff) = *reinterpret_cast<const uint4 *>(vpl + so);
  }
}

// ------------------------------------------------------------------------------------------ device
#ifdef KVFS_HOST_PROFILE
// Development: host time of the launch-path pieces, printed every 200 layers (build variant only).
struct HostProf {
  double t[8] = {0};
  int64_t n = 0;
  static double now() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
};
static HostProf g_hprof;
#define HP_MARK(var) const double var = HostProf::now()
#define HP_ADD(i, a, b) g_hprof.t[i] += (b) - (a)
#else
#define HP_MARK(var)
#define HP_ADD(i, a, b)
#endif

class CudaDevice final : public Device {
 public:
  explicit CudaDevice(Ctx &c) : c_(c) {}
  ~CudaDevice() override {
    if (io_h2d_) {
      cudaStreamSynchronize(io_h2d_);
      cudaStreamSynchronize(io_d2h_);
      for (IoSlot &x : io_) {
        for (cudaEvent_t e : {x.in_ready, x.used, x.out_done})
          if (e) cudaEventDestroy(e);
        if (x.in) cudaFree(x.in);
        if (x.out) cudaFree(x.out);
      }
      cudaStreamDestroy(io_h2d_);
      cudaStreamDestroy(io_d2h_);
    }
    for (auto &s : stg_) {
      if (s.ev) cudaEventDestroy(s.ev);
      if (s.host) cudaFreeHost(s.host);
    }
    for (auto &b : host_cache_) {
      if (b.ev) cudaEventDestroy(b.ev);
      cudaFreeHost(b.host);
    }
    for (auto &kv : host_sizes_) cudaFreeHost(kv.first);
    for (auto *v : {&layer_timing_, &copy_timing_})
      for (auto &t : *v) {
        cudaEventDestroy(t.first);
        cudaEventDestroy(t.second);
      }
    for (cudaEvent_t e : ev_pool_) cudaEventDestroy(e);
  }

  int init() {
    const kvfs_config &cfg = c_.cfg;
    if (cudaSetDevice(cfg.device) != cudaSuccess) return KVFS_EINVAL;
    lay_ = ws_layout(cfg);
    char *ws = static_cast<char *>(cfg.workspace);
    if (reinterpret_cast<uintptr_t>(ws) % 256) return KVFS_EINVAL;
    slab_ = reinterpret_cast<dev::Entry *>(ws + lay_.slab);
    upload_ = ws + lay_.upload;
    counters_ = reinterpret_cast<int *>(ws + lay_.counters);
    partials_ = reinterpret_cast<float *>(ws + lay_.partials);
    ppart_ = reinterpret_cast<float *>(ws + lay_.prefix);
    kptrs_ = reinterpret_cast<bf16 **>(ws + lay_.ptrs);
    vptrs_ = kptrs_ + cfg.n_layers;
    std::vector<void *> ptrs(c_.kpool);
    ptrs.insert(ptrs.end(), c_.vpool.begin(), c_.vpool.end());
    if (cudaMemcpy(kptrs_, ptrs.data(), ptrs.size() * sizeof(void *), cudaMemcpyHostToDevice) != cudaSuccess)
      return KVFS_EIO;
    if (cudaMemset(counters_, 0, static_cast<size_t>(cfg.max_batch_rows) * cfg.n_kv_heads * 4) != cudaSuccess)
      return KVFS_EIO;
    work_ = reinterpret_cast<int *>(ws + lay_.work);
    if (cudaMemset(work_, 0, 16) != cudaSuccess) return KVFS_EIO;
    pgroup_ = reinterpret_cast<int *>(ws + lay_.pgroup);
    if (cudaMemset(pgroup_, 0, 2 * static_cast<size_t>(kMaxPrefixGroups) * 4) != cudaSuccess) return KVFS_EIO;
    // Zero-fill the pools once: every slot then always holds finite bf16 (only finite rows are ever
    // written), so the tensor-core kernel can multiply masked-out keys' V rows by P = 0 safely.
    const size_t pool_bytes = static_cast<size_t>(cfg.n_pages) * cfg.n_kv_heads * cfg.page_size * cfg.head_dim * 2;
    for (int l = 0; l < cfg.n_layers; ++l) {
      if (cudaMemset(c_.kpool[l], 0, pool_bytes) != cudaSuccess) return KVFS_EIO;
      if (cudaMemset(c_.vpool[l], 0, pool_bytes) != cudaSuccess) return KVFS_EIO;
    }
    {
      void *fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess || !fn)
        return KVFS_EIO;
      encode_ = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    if (cfg.head_dim == 128) {
      kmaps_.resize(cfg.n_layers);
      vmaps_.resize(cfg.n_layers);
      for (int l = 0; l < cfg.n_layers; ++l) {
        if (!pool_map(c_.kpool[l], &kmaps_[l], cfg.page_size) || !pool_map(c_.vpool[l], &vmaps_[l], cfg.page_size))
          return KVFS_EIO;
      }
    }
    if (cfg.head_dim == 64 || cfg.head_dim == 128) {  // K1 holes: single rows for TMA gather4
      gkmaps_.resize(cfg.n_layers);
      gvmaps_.resize(cfg.n_layers);
      for (int l = 0; l < cfg.n_layers; ++l)
        if (!row_map(c_.kpool[l], &gkmaps_[l]) || !row_map(c_.vpool[l], &gvmaps_[l])) return KVFS_EIO;
    }
    if (cfg.head_dim == 64 || cfg.head_dim == 128) {  // K9: 16-row tiles of the K pool
      smaps_.resize(cfg.n_layers);
      for (int l = 0; l < cfg.n_layers; ++l)
        if (!pool_map(c_.kpool[l], &smaps_[l], 16)) return KVFS_EIO;
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg.device);
    sms_ = sms > 0 ? sms : 148;
    for (auto &s : stg_) {
      if (cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming) != cudaSuccess) return KVFS_EIO;
      if (!grow(s, 1 << 20)) return KVFS_ENOMEM;
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return KVFS_EIO;
    return KVFS_OK;
  }

  int copy_pages(const std::vector<PageCopy> &copies, kvfs_stream_t s) override {
    begin_packet();
    const void *dc = push(copies.data(), copies.size() * sizeof(PageCopy));
    if (!dc) return KVFS_ENOMEM;
    if (!send(s)) return KVFS_EIO;
    return launch_prologue(nullptr, 0, nullptr, static_cast<const dev::PageCopy *>(dc),
                           static_cast<int>(copies.size()), s);
  }

  int append_rows(const std::vector<int32_t> &dst, const void *k, const void *v, kvfs_stream_t s) override {
    // the slot list is uploaded in pieces that fit the upload area
    const int64_t n = static_cast<int64_t>(dst.size());
    const int64_t piece = std::max<int64_t>(1, static_cast<int64_t>(lay_.upload_cap / 8));
    for (int64_t b = 0; b < n; b += piece) {
      const int rc = append_piece(dst.data() + b, std::min(piece, n - b), b, n, static_cast<const bf16 *>(k),
                                  static_cast<const bf16 *>(v), s);
      if (rc != KVFS_OK) return rc;
    }
    return KVFS_OK;
  }

  int compact(const std::vector<CompactJob> &jobs, kvfs_stream_t s) override {
    // one packet for every file (old tables, new pages, first entries), then one K5 launch per file in
    // order, each after the first a programmatic dependent launch of the previous one (see compact_kernel)
    const kvfs_config &cfg = c_.cfg;
    cudaEvent_t ev_end = nullptr;
    if (c_.opt_timing) {  // device time of this group: upload + gathers (KVFS_CTR_COMPACT_DEVICE_NS)
      cudaEvent_t e0 = nullptr;
      if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&ev_end) != cudaSuccess) return KVFS_EIO;
      cudaEventRecord(e0, cs(s));
      timing_.push_back({e0, ev_end});
    }
    const int P = cfg.page_size;
    std::vector<std::vector<int32_t>> fe(jobs.size());
    std::vector<const void *> dt(jobs.size()), dp(jobs.size()), df(jobs.size());
    begin_packet();
    for (size_t f = 0; f < jobs.size(); ++f) {
      const std::vector<Entry> &old = *jobs[f].old_table;
      const size_t n_new = jobs[f].new_pages->size();
      fe[f].resize(n_new);
      size_t e = 0;
      for (size_t j = 0; j < n_new; ++j) {  // the old entry holding logical token j * P
        const int64_t i = static_cast<int64_t>(j) * P;
        while (e + 1 < old.size() && old[e + 1].lstart <= i) ++e;
        fe[f][j] = static_cast<int32_t>(e);
      }
      dt[f] = push(old.data(), old.size() * sizeof(Entry));
      dp[f] = push(jobs[f].new_pages->data(), n_new * sizeof(uint32_t));
      df[f] = push(fe[f].data(), n_new * sizeof(int32_t));
      if (!dt[f] || !dp[f] || !df[f]) return KVFS_ENOMEM;
    }
    if (!send(s)) return KVFS_EIO;
    if (k5_grid_ == 0) {
      if (cudaFuncSetAttribute(compact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kK5Smem) != cudaSuccess)
        return KVFS_EIO;
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, compact_kernel, kK5Threads, kK5Smem);
      k5_grid_ = sms_ * std::max(1, per_sm);  // one wave of resident CTAs (2 per SM)
    }
    const int lgD = cfg.head_dim == 128 ? 7 : 6;
    const int lgP = __builtin_ctz(static_cast<unsigned>(P));
    for (size_t f = 0; f < jobs.size(); ++f) {
      const int64_t n_new = static_cast<int64_t>(jobs[f].new_pages->size());
      if (n_new == 0) continue;
      const int64_t stages = (n_new * cfg.n_layers * 2 * cfg.n_kv_heads * P * cfg.head_dim * 2 + kK5StageBytes - 1) /
                             kK5StageBytes;
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(k5_grid_, stages)));
      lc.blockDim = dim3(kK5Threads);
      lc.dynamicSmemBytes = kK5Smem;
      lc.stream = cs(s);
      cudaLaunchAttribute la[1];
      la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      la[0].val.programmaticStreamSerializationAllowed = f > 0 ? 1 : 0;  // the first waits for everything before
      lc.attrs = la;
      lc.numAttrs = 1;
      const cudaError_t e = cudaLaunchKernelEx(&lc, compact_kernel, static_cast<const dev::Entry *>(dt[f]),
                                               static_cast<int>(jobs[f].old_table->size()),
                                               static_cast<const uint32_t *>(dp[f]), static_cast<const int32_t *>(df[f]),
                                               static_cast<int>(n_new), jobs[f].len, kptrs_, vptrs_, cfg.n_layers,
                                               cfg.n_kv_heads, lgD, lgP);
      ++c_.ctr.launches;
      if (e != cudaSuccess) return KVFS_EIO;
    }
    if (ev_end) cudaEventRecord(ev_end, cs(s));
    return KVFS_OK;
  }

  // Sum of the recorded device intervals (each: a compact group's upload + gathers), then forget them.
  int64_t take_device_ns() override {
    double ms = 0;
    for (auto &t : timing_) {
      float x = 0.f;
      if (cudaEventSynchronize(t.second) == cudaSuccess && cudaEventElapsedTime(&x, t.first, t.second) == cudaSuccess)
        ms += x;
      cudaEventDestroy(t.first);
      cudaEventDestroy(t.second);
    }
    timing_.clear();
    return static_cast<int64_t>(ms * 1e6);
  }

  int logit_scores(const std::vector<LogitDesc> &descs, const std::vector<ScoreUnit> &units, const float *lse,
                   float *out, kvfs_stream_t s) override {
    begin_packet(/*scratch=*/true);
    const void *dd = push(descs.data(), descs.size() * sizeof(LogitDesc));
    const void *du = push(units.data(), units.size() * sizeof(ScoreUnit));
    if (!dd || !du) return KVFS_ENOMEM;
    if (!send(s)) return KVFS_EIO;
    const kvfs_config &cfg = c_.cfg;
    const cudaError_t e = dev::launch_logit_scores(static_cast<const dev::ScoreUnit *>(du), static_cast<int>(units.size()),
                                                   static_cast<const dev::LogitDesc *>(dd), slab_, c_.logits_buf, lse,
                                                   out, cfg.n_q_heads, cfg.n_kv_heads, cfg.page_size, cs(s));
    ++c_.ctr.launches;
    return e == cudaSuccess ? KVFS_OK : KVFS_EIO;
  }

  int scores(const std::vector<ScoreDesc> &descs, const std::vector<ScoreUnit> &units, int layer, const void *q,
             const float *lse, float scale, float *out, kvfs_stream_t s) override {
    begin_packet(/*scratch=*/true);  // the open step's plan in the upload area must survive (later layers)
    const void *dd = push(descs.data(), descs.size() * sizeof(ScoreDesc));
    const void *du = push(units.data(), units.size() * sizeof(ScoreUnit));
    if (!dd || !du) return KVFS_ENOMEM;
    if (!send(s)) return KVFS_EIO;
    const kvfs_config &cfg = c_.cfg;
    if (smaps_.empty()) return KVFS_EINVAL;
    const cudaError_t e = dev::launch_scores(
        smaps_[layer], static_cast<const dev::ScoreUnit *>(du), static_cast<int>(units.size()),
        static_cast<const dev::ScoreDesc *>(dd), slab_, static_cast<const bf16 *>(q), lse, scale * 1.4426950408889634f,
        out, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, cfg.page_size, cs(s));
    ++c_.ctr.launches;
    return e == cudaSuccess ? KVFS_OK : KVFS_EIO;
  }

  int gather(const std::vector<int32_t> &src_slots, const std::vector<uint32_t> &new_pages,
             kvfs_stream_t s) override {
    begin_packet();
    const void *ds = push(src_slots.data(), src_slots.size() * sizeof(int32_t));
    const void *dp = push(new_pages.data(), new_pages.size() * sizeof(uint32_t));
    if (!ds || !dp) return KVFS_ENOMEM;
    if (!send(s)) return KVFS_EIO;
    const kvfs_config &cfg = c_.cfg;
    const dim3 grid(static_cast<unsigned>(new_pages.size()), static_cast<unsigned>(cfg.n_layers));
    gather_kernel<<<grid, 256, 0, cs(s)>>>(static_cast<const int32_t *>(ds), static_cast<int64_t>(src_slots.size()),
                                           static_cast<const uint32_t *>(dp), kptrs_, vptrs_, cfg.n_kv_heads,
                                           cfg.head_dim, cfg.page_size);
    ++c_.ctr.launches;
    return cudaGetLastError() == cudaSuccess ? KVFS_OK : KVFS_EIO;
  }

  int read(const std::vector<Entry> &table, int layer, int64_t begin, int64_t end, void *k_out, void *v_out,
           kvfs_stream_t s) override {
    begin_packet();
    const void *dt = push(table.data(), table.size() * sizeof(Entry));
    if (!dt) return KVFS_ENOMEM;
    if (!send(s)) return KVFS_EIO;
    const kvfs_config &cfg = c_.cfg;
    const int64_t total = (end - begin) * cfg.n_kv_heads * (cfg.head_dim / 8);
    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, sms_ * 16));
    read_kernel<<<grid, 256, 0, cs(s)>>>(static_cast<const dev::Entry *>(dt), static_cast<int>(table.size()), begin,
                                         end, static_cast<const bf16 *>(c_.kpool[layer]),
                                         static_cast<const bf16 *>(c_.vpool[layer]), static_cast<bf16 *>(k_out),
                                         static_cast<bf16 *>(v_out), cfg.n_kv_heads, cfg.head_dim, cfg.page_size);
    ++c_.ctr.launches;
    return cudaGetLastError() == cudaSuccess ? KVFS_OK : KVFS_EIO;
  }

  int pred_begin(PredPlan &pl, kvfs_stream_t s) override {
    begin_packet();
    d_runs_ = push(pl.run_dst.data(), pl.run_dst.size() * sizeof(int64_t));
    d_run_entries_ = push(pl.run_entries.data(), pl.run_entries.size() * sizeof(Entry));
    d_copies_ = push(pl.copies.data(), pl.copies.size() * sizeof(PageCopy));
    const size_t off_runs = pending_[0].off, off_entries = pending_[1].off, off_copies = pending_[2].off;
    d_descs_ = push(pl.descs.data(), pl.descs.size() * sizeof(DevDesc));
    d_dst_ = push(pl.dst_slot.data(), pl.dst_slot.size() * sizeof(int32_t));
    d_cdescs_ = push(pl.chunk_descs.data(), pl.chunk_descs.size() * sizeof(ChunkDesc));
    d_cunits_ = push(pl.chunk_units.data(), pl.chunk_units.size() * sizeof(ChunkUnit));
    d_cdst_ = push(pl.chunk_dst.data(), pl.chunk_dst.size() * sizeof(int32_t));
    d_pdescs_ = push(pl.prefix_descs.data(), pl.prefix_descs.size() * sizeof(PrefixDesc));
    d_punits_ = push(pl.prefix_units.data(), pl.prefix_units.size() * sizeof(ChunkUnit));
    d_prows_ = push(pl.prefix_rows.data(), pl.prefix_rows.size() * sizeof(PrefixRow));
    d_pctas_ = push(pl.prefix_cta_units.data(), pl.prefix_cta_units.size() * sizeof(int32_t));
    if (!d_runs_ || !d_run_entries_ || !d_copies_ || !d_descs_ || !d_dst_ || !d_cdescs_ || !d_cunits_ || !d_cdst_ ||
        !d_pdescs_ || !d_punits_ || !d_prows_ || !d_pctas_)
      return KVFS_ENOMEM;
    // one launch: packet copy (SM loads over PCIe) + table deltas + copy-on-write pages (step_prologue_kernel)
    Staging &st = stg_[cur_];
    if (!gather(st)) return KVFS_EIO;
    const kvfs_config &cfg = c_.cfg;
    const int64_t n16 = static_cast<int64_t>((used_ + 15) / 16);
    const int n_deltas = static_cast<int>(pl.run_dst.size()), n_copies = static_cast<int>(pl.copies.size());
    const int work = (n_deltas + 255) / 256 + n_copies * 2 * cfg.n_layers;
    const int blocks = std::max<int>(work, static_cast<int>(std::min<int64_t>((n16 + 255) / 256, 64)));
    if (blocks == 0) return KVFS_OK;
    const int64_t page_elems = static_cast<int64_t>(cfg.n_kv_heads) * cfg.page_size * cfg.head_dim;
    {
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(static_cast<unsigned>(blocks));
      lc.blockDim = dim3(256);
      lc.stream = cs(s);
      cudaLaunchAttribute la[1];
      la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      la[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = la;
      lc.numAttrs = 1;
      if (cudaLaunchKernelEx(&lc, step_prologue_kernel, reinterpret_cast<uint4 *>(area_),
                             reinterpret_cast<const uint4 *>(st.dev), static_cast<int64_t>(n16),
                             reinterpret_cast<const int64_t *>(st.dev + off_runs), n_deltas,
                             reinterpret_cast<const dev::Entry *>(st.dev + off_entries), slab_,
                             reinterpret_cast<const dev::PageCopy *>(st.dev + off_copies), n_copies, kptrs_, vptrs_,
                             cfg.n_layers, page_elems) != cudaSuccess)
        return KVFS_EIO;
    }
    ++c_.ctr.launches;
    if (cudaEventRecord(st.ev, cs(s)) != cudaSuccess) return KVFS_EIO;
    st.pending = true;
    c_.ctr.h2d_bytes += static_cast<int64_t>(used_);
    return KVFS_OK;
  }

  // KVFS_OPT_TIMING: events on the stream before the layer's first kernel and after its last
  int pred_layer(const PredPlan &pl, int layer, const void *q, const void *k_new, const void *v_new, void *out,
                 float *lse, float scale, kvfs_stream_t s) override {
    if (!c_.opt_timing || (c_.layer_calls++ % c_.opt_timing_every) != 0)
      return pred_layer_kernels(pl, layer, q, k_new, v_new, out, lse, scale, s);
    cudaEvent_t e0 = pooled_event(), e1 = pooled_event();
    if (!e0 || !e1) return KVFS_EIO;
    cudaEventRecord(e0, cs(s));
    const int rc = pred_layer_kernels(pl, layer, q, k_new, v_new, out, lse, scale, s);
    cudaEventRecord(e1, cs(s));
    layer_timing_.push_back({e0, e1});
    return rc;
  }

  int64_t take_layer_ns(int64_t *n) override { return take_pairs(layer_timing_, n); }
  int64_t take_copy_ns(int64_t *n) override { return take_pairs(copy_timing_, n); }

  int64_t take_pairs(std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &v, int64_t *n) {
    double ms = 0;
    for (auto &t : v) {
      float x = 0.f;
      if (cudaEventSynchronize(t.second) == cudaSuccess && cudaEventElapsedTime(&x, t.first, t.second) == cudaSuccess)
        ms += x;
      ev_pool_.push_back(t.first);
      ev_pool_.push_back(t.second);
    }
    *n = static_cast<int64_t>(v.size());
    v.clear();
    return static_cast<int64_t>(ms * 1e6);
  }

  cudaEvent_t pooled_event() {
    if (!ev_pool_.empty()) {
      cudaEvent_t e = ev_pool_.back();
      ev_pool_.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    return cudaEventCreate(&e) == cudaSuccess ? e : nullptr;
  }

  int pred_layer_kernels(const PredPlan &pl, int layer, const void *q, const void *k_new, const void *v_new,
                         void *out, float *lse, float scale, kvfs_stream_t s) {
    c_.ctr.last_chunk_units = static_cast<int64_t>(pl.chunk_units.size());
    c_.ctr.last_prefix_units = static_cast<int64_t>(pl.prefix_units.size());
    c_.ctr.last_prefix_groups = pl.prefix_groups;
    if (!pl.chunk_units.empty()) {
      const int rc = chunk_layer(pl, layer, q, k_new, v_new, out, lse, scale, s);
      if (rc != KVFS_OK) return rc;
    }
    if (pl.descs.empty()) return KVFS_OK;
    if (!pl.prefix_units.empty()) {
      const int rc = prefix_layer(pl, layer, q, scale, s);
      if (rc != KVFS_OK) return rc;
    }
    const kvfs_config &cfg = c_.cfg;
    dev::DecodeParams p{};
    p.descs = static_cast<const dev::Desc *>(d_descs_);
    p.n_desc = static_cast<int>(pl.descs.size());
    p.total = pl.total_cost;
    if (per_sm_ == 0) per_sm_ = dev::decode_ctas_per_sm(cfg.head_dim, cfg.n_q_heads / cfg.n_kv_heads, cfg.page_size);
    int64_t ncta = c_.opt_decode_ctas > 0 ? c_.opt_decode_ctas : static_cast<int64_t>(sms_) * per_sm_;
    if (c_.opt_decode_ctas <= 0 && !pl.prefix_units.empty() && pl.decode_sms > 0) {
      // the shared-prefix grid (one CTA per SM, launched first) holds the other SMs for most of the step: the
      // decode rings go to the free ones, so none of them starts late (pred_cascade chose the split)
      ncta = static_cast<int64_t>(pl.decode_sms) * per_sm_;
    }
    if (c_.opt_decode_ctas <= 0 && pl.n_units > 0 && pl.n_units <= ncta) {
      // Few units (e.g. the short private suffixes of a fork family after the shared prefix went to the
      // cascade): one ring per unit when the units are about equally long, so no unit is cut by a range
      // boundary and none pays the cross-ring partial merge.
      int32_t spu_max = 0;
      for (const DevDesc &d : pl.descs) spu_max = std::max(spu_max, d.stages_per_unit);
      if (4 * static_cast<int64_t>(spu_max) * pl.n_units <= 5 * pl.total_cost) ncta = pl.n_units;
    }
    ncta = std::min<int64_t>(std::min<int64_t>(ncta, kMaxCtas), pl.total_cost);
    p.ncta = static_cast<int>(ncta);
    p.n_rings = p.ncta;
    p.dynamic = 0;
    p.work = work_;
    if (c_.opt_decode_chunks > 0) {
      // dynamic scheduling: opt_decode_chunks chunks taken from a counter by at most one wave of rings
      const int64_t chunks = std::min<int64_t>(std::min<int64_t>(c_.opt_decode_chunks, kMaxCtas), pl.total_cost);
      p.ncta = static_cast<int>(chunks);
      p.n_rings = static_cast<int>(std::min<int64_t>(chunks, static_cast<int64_t>(sms_) * per_sm_));
      p.dynamic = 1;
      ncta = chunks;
    }
    p.slab = slab_;
    p.dst_slot = static_cast<const int32_t *>(d_dst_);
    p.q = static_cast<const bf16 *>(q);
    p.k_new = static_cast<const bf16 *>(k_new);
    p.v_new = static_cast<const bf16 *>(v_new);
    p.out = static_cast<bf16 *>(out);
    p.lse = lse;
    p.kpool = static_cast<bf16 *>(c_.kpool[layer]);
    p.vpool = static_cast<bf16 *>(c_.vpool[layer]);
    p.scale_log2 = scale * 1.4426950408889634f;
    p.partials = partials_;
    p.ppart = ppart_;
    p.wait_at_start = pl.prefix_units.empty() ? 1 : 0;
    p.counters = counters_;
    p.logits = c_.logits_buf;
    p.Hq = cfg.n_q_heads;
    p.Hkv = cfg.n_kv_heads;
    p.gather = c_.opt_holes_gather && !gkmaps_.empty() ? 1 : 0;
    if (p.gather) {
      p.gk = gkmaps_[layer];
      p.gv = gvmaps_[layer];
    }
    // always a programmatic dependent launch: after the prologue (waits at start) or after the shared-prefix
    // kernel (which waited for the prologue itself; waits before merging)
    HP_MARK(d0);
    const cudaError_t e = dev::launch_decode(p, cfg.head_dim, cfg.n_q_heads / cfg.n_kv_heads, cfg.page_size, cs(s),
                                             true);
    HP_MARK(d1);
    HP_ADD(2, d0, d1);
#ifdef KVFS_HOST_PROFILE
    if (++g_hprof.n % 200 == 0) {
      fprintf(stderr, "[hprof] per layer us: qmap encode %.2f prefix launch %.2f decode launch %.2f\n",
              g_hprof.t[0] / 200, g_hprof.t[1] / 200, g_hprof.t[2] / 200);
      for (double &x : g_hprof.t) x = 0;
    }
#endif
    ++c_.ctr.launches;
    c_.ctr.last_decode_ctas = p.ncta;
    return e == cudaSuccess ? KVFS_OK : KVFS_EIO;
  }

  int sync() override { return cudaDeviceSynchronize() == cudaSuccess ? KVFS_OK : KVFS_EIO; }

  // ---- host-buffer pred: two device slots, an H2D and a D2H copy stream of the library
  int io_begin(int64_t T, const void *q, const void *k, const void *v, bool want_lse, kvfs_stream_t s,
               HostIo *io) override {
    const kvfs_config &cfg = c_.cfg;
    if (!io_h2d_) {
      if (cudaStreamCreateWithFlags(&io_h2d_, cudaStreamNonBlocking) != cudaSuccess ||
          cudaStreamCreateWithFlags(&io_d2h_, cudaStreamNonBlocking) != cudaSuccess)
        return KVFS_EIO;
      for (IoSlot &x : io_)
        for (cudaEvent_t *e : {&x.in_ready, &x.used, &x.out_done})
          if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return KVFS_EIO;
    }
    const int b = io_next_;
    io_next_ ^= 1;
    IoSlot &x = io_[b];
    auto al = [](size_t n) { return (n + 255) & ~static_cast<size_t>(255); };
    io->q_bytes = static_cast<size_t>(T) * cfg.n_q_heads * cfg.head_dim * 2;
    io->kv_bytes = static_cast<size_t>(T) * cfg.n_kv_heads * cfg.head_dim * 2;
    io->out_bytes = io->q_bytes;
    io->lse_bytes = want_lse ? static_cast<size_t>(T) * cfg.n_q_heads * 4 : 0;
    const size_t need_in = al(io->q_bytes) + 2 * al(io->kv_bytes), need_out = al(io->out_bytes) + al(io->lse_bytes);
    if (x.in_cap < need_in || x.out_cap < need_out) {
      // grow: the slot's previous use must be over (its input and output copies and the pred between them)
      if (x.live && (cudaEventSynchronize(x.used) != cudaSuccess || cudaEventSynchronize(x.out_done) != cudaSuccess))
        return KVFS_EIO;
      if (x.in_cap < need_in) {
        if (x.in) cudaFree(x.in);
        x.in = nullptr;
        x.in_cap = 0;
        if (cudaMalloc(&x.in, need_in) != cudaSuccess) return KVFS_ENOMEM;
        x.in_cap = need_in;
      }
      if (x.out_cap < need_out) {
        if (x.out) cudaFree(x.out);
        x.out = nullptr;
        x.out_cap = 0;
        if (cudaMalloc(&x.out, need_out) != cudaSuccess) return KVFS_ENOMEM;
        x.out_cap = need_out;
      }
    }
    char *in = static_cast<char *>(x.in), *out = static_cast<char *>(x.out);
    io->slot = b;
    io->q = in;
    io->k = in + al(io->q_bytes);
    io->v = in + al(io->q_bytes) + al(io->kv_bytes);
    io->out = out;
    io->lse = want_lse ? reinterpret_cast<float *>(out + al(io->out_bytes)) : nullptr;
    // inputs: after the pred that last read this slot
    if (x.live && cudaStreamWaitEvent(io_h2d_, x.used, 0) != cudaSuccess) return KVFS_EIO;
    if (cudaMemcpyAsync(io->q, q, io->q_bytes, cudaMemcpyHostToDevice, io_h2d_) != cudaSuccess ||
        cudaMemcpyAsync(io->k, k, io->kv_bytes, cudaMemcpyHostToDevice, io_h2d_) != cudaSuccess ||
        cudaMemcpyAsync(io->v, v, io->kv_bytes, cudaMemcpyHostToDevice, io_h2d_) != cudaSuccess ||
        cudaEventRecord(x.in_ready, io_h2d_) != cudaSuccess)
      return KVFS_EIO;
    // the pred: after its inputs landed and after the slot's previous outputs were copied out
    if (cudaStreamWaitEvent(cs(s), x.in_ready, 0) != cudaSuccess) return KVFS_EIO;
    if (x.live && cudaStreamWaitEvent(cs(s), x.out_done, 0) != cudaSuccess) return KVFS_EIO;
    return KVFS_OK;
  }

  int io_end(const HostIo &io, void *out, float *lse, const std::vector<std::pair<int64_t, int64_t>> &rows,
             kvfs_stream_t s) override {
    IoSlot &x = io_[io.slot];
    if (cudaEventRecord(x.used, cs(s)) != cudaSuccess || cudaStreamWaitEvent(io_d2h_, x.used, 0) != cudaSuccess)
      return KVFS_EIO;
    const size_t orow = static_cast<size_t>(c_.cfg.n_q_heads) * c_.cfg.head_dim * 2, lrow = c_.cfg.n_q_heads * 4;
    for (const auto &r : rows) {
      const size_t n = static_cast<size_t>(r.second - r.first);
      if (cudaMemcpyAsync(static_cast<char *>(out) + r.first * orow, static_cast<const char *>(io.out) + r.first * orow,
                          n * orow, cudaMemcpyDeviceToHost, io_d2h_) != cudaSuccess)
        return KVFS_EIO;
      if (lse && io.lse &&
          cudaMemcpyAsync(lse + r.first * c_.cfg.n_q_heads, io.lse + r.first * c_.cfg.n_q_heads, n * lrow,
                          cudaMemcpyDeviceToHost, io_d2h_) != cudaSuccess)
        return KVFS_EIO;
    }
    if (cudaEventRecord(x.out_done, io_d2h_) != cudaSuccess) return KVFS_EIO;
    x.live = true;
    return KVFS_OK;
  }

  int io_fence(kvfs_stream_t s) override {
    if (!io_d2h_) return KVFS_OK;
    for (IoSlot &x : io_)
      if (x.live && cudaStreamWaitEvent(cs(s), x.out_done, 0) != cudaSuccess) return KVFS_EIO;
    return KVFS_OK;
  }
  // Host tier buffers are recycled: a released buffer is cached with an event recorded on the releasing
  // stream (the restore that reads it may still be running) and handed out again, after that event, to an
  // offload needing between half and all of its size.  cudaHostAlloc of pinned memory costs milliseconds.
  int host_alloc(size_t bytes, void **host, void **dev) override {
    size_t best = host_cache_.size();
    for (size_t i = 0; i < host_cache_.size(); ++i) {
      const HostBuf &b = host_cache_[i];
      if (b.bytes >= bytes && b.bytes <= 2 * bytes && (best == host_cache_.size() || b.bytes < host_cache_[best].bytes))
        best = i;
    }
    if (best < host_cache_.size()) {
      HostBuf b = host_cache_[best];
      host_cache_.erase(host_cache_.begin() + static_cast<long>(best));
      if (b.ev) {
        cudaEventSynchronize(b.ev);
        cudaEventDestroy(b.ev);
      }
      cached_bytes_ -= b.bytes;
      *host = b.host;
      *dev = b.dev;
      host_sizes_[b.host] = b.bytes;
      return KVFS_OK;
    }
    if (cudaHostAlloc(host, bytes, cudaHostAllocMapped) != cudaSuccess) return KVFS_ENOMEM;
    if (cudaHostGetDevicePointer(dev, *host, 0) != cudaSuccess) {
      cudaFreeHost(*host);
      return KVFS_EIO;
    }
    host_sizes_[*host] = bytes;
    return KVFS_OK;
  }
  void host_free(void *host) override { host_release(host, nullptr); }
  void host_release(void *host, kvfs_stream_t s) override {
    auto it = host_sizes_.find(host);
    if (it == host_sizes_.end()) return;
    HostBuf b{host, nullptr, it->second, nullptr};
    host_sizes_.erase(it);
    cudaHostGetDevicePointer(&b.dev, host, 0);
    if (cached_bytes_ + b.bytes > (size_t{8} << 30)) {  // keep at most 8 GiB cached
      if (s) cudaStreamSynchronize(cs(s));
      cudaFreeHost(host);
      return;
    }
    if (s && cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming) == cudaSuccess) cudaEventRecord(b.ev, cs(s));
    cached_bytes_ += b.bytes;
    host_cache_.push_back(b);
  }
  int stream_sync(kvfs_stream_t s) override {
    return cudaStreamSynchronize(cs(s)) == cudaSuccess ? KVFS_OK : KVFS_EIO;
  }
  int sms() const override { return sms_; }
  int64_t prefix_partial_capacity() const override { return lay_.prefix_cap; }

  // Shared-prefix (cascade) attention of the fork families (tcgen05 kernel in prefix mode): partials
  // (O, m, l) per (member row, head, key split) into the workspace, merged by the decode kernel.
  int prefix_layer(const PredPlan &pl, int layer, const void *q, float scale, kvfs_stream_t s) {
    const kvfs_config &cfg = c_.cfg;
    const int G = cfg.n_q_heads / cfg.n_kv_heads;
    dev::ChunkParams p{};
    p.units = static_cast<const dev::ChunkUnit *>(d_punits_);
    p.descs = nullptr;
    p.slab = slab_;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.P = cfg.page_size;
    p.Hkv = cfg.n_kv_heads;
    p.Hq = cfg.n_q_heads;
    p.pool_rows = static_cast<int>(cfg.n_pages * cfg.n_kv_heads * cfg.page_size);
    p.pdescs = static_cast<const dev::PrefixDesc *>(d_pdescs_);
    p.prows = static_cast<const dev::PrefixRow *>(d_prows_);
    p.q = static_cast<const bf16 *>(q);
    p.ppart = ppart_;
    p.pgroup = pgroup_;
    p.pgroup_parity = static_cast<int>(prefix_launches_++ & 1);
    p.cta_units = pl.prefix_cta_units.empty() ? nullptr : static_cast<const int2 *>(d_pctas_);
    const int n_ctas = pl.prefix_cta_units.empty() ? static_cast<int>(pl.prefix_units.size())
                                                   : static_cast<int>(pl.prefix_cta_units.size() / 2);
    alignas(64) CUtensorMap qmap;
    HP_MARK(a0);
    if (!encode_q_map(&qmap, q, pl.T)) return KVFS_EINVAL;
    HP_MARK(a1);
    const cudaError_t e = dev::launch_prefix(kmaps_[layer], vmaps_[layer], qmap, p,
                                             n_ctas, G, cs(s));
    HP_MARK(a2);
    HP_ADD(0, a0, a1);
    HP_ADD(1, a1, a2);
    ++c_.ctr.launches;
    return e == cudaSuccess ? KVFS_OK : KVFS_EIO;
  }

  int pack_pages(const std::vector<uint32_t> &pages, void *buf, kvfs_stream_t s) override {
    return pack_impl(pages, buf, 0, s);
  }
  int unpack_pages(const std::vector<uint32_t> &pages, const void *buf, kvfs_stream_t s) override {
    return pack_impl(pages, const_cast<void *>(buf), 1, s);
  }
  int pack_impl(const std::vector<uint32_t> &pages, void *buf, int unpack, kvfs_stream_t s) {
    begin_packet();
    const void *dp = push(pages.data(), pages.size() * sizeof(uint32_t));
    if (!dp) return KVFS_ENOMEM;
    if (!send(s)) return KVFS_EIO;
    const kvfs_config &cfg = c_.cfg;
    const int64_t page_elems = static_cast<int64_t>(cfg.n_kv_heads) * cfg.page_size * cfg.head_dim;
    const int64_t blocks = static_cast<int64_t>(pages.size()) * cfg.n_layers * 2;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c_.opt_timing) {  // KVFS_CTR_COPY_DEVICE_NS: the K6 kernel alone (no host work, no packet upload)
      e0 = pooled_event();
      e1 = pooled_event();
      if (!e0 || !e1) return KVFS_EIO;
      cudaEventRecord(e0, cs(s));
    }
    pack_kernel<<<static_cast<unsigned>(blocks), 256, 0, cs(s)>>>(static_cast<const uint32_t *>(dp),
                                                                  static_cast<int>(pages.size()), kptrs_, vptrs_,
                                                                  cfg.n_layers, page_elems, static_cast<bf16 *>(buf),
                                                                  unpack);
    ++c_.ctr.launches;
    if (e1) {
      cudaEventRecord(e1, cs(s));
      copy_timing_.push_back({e0, e1});
    }
    return cudaGetLastError() == cudaSuccess ? KVFS_OK : KVFS_EIO;
  }

  // K2: scatter the chunk descriptors' new rows into the pool, then tcgen05 attention from the pool.
  // Q [T][Hq][D] as a 4-D tensor (D, G, Hkv, T), boxes of {64 dims, G heads, 1 kv head, 128 / G rows} with
  // 128-byte swizzle: one box = one 64-column half of a 128-row M-tile (rows = (token, head), head fastest)
  bool encode_q_map(CUtensorMap *qmap, const void *q, int64_t T) {
    const kvfs_config &cfg = c_.cfg;
    const int G = cfg.n_q_heads / cfg.n_kv_heads;
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(cfg.head_dim), static_cast<cuuint64_t>(G),
                                static_cast<cuuint64_t>(cfg.n_kv_heads), static_cast<cuuint64_t>(T)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(cfg.head_dim) * 2,
                                   static_cast<cuuint64_t>(G) * cfg.head_dim * 2,
                                   static_cast<cuuint64_t>(cfg.n_q_heads) * cfg.head_dim * 2};
    const cuuint32_t box[4] = {64, static_cast<cuuint32_t>(G), 1, static_cast<cuuint32_t>(128 / G)};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    return encode_(qmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(q), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }

  int chunk_layer(const PredPlan &pl, int layer, const void *q, const void *k_new, const void *v_new, void *out,
                  float *lse, float scale, kvfs_stream_t s) {
    const kvfs_config &cfg = c_.cfg;
    cudaError_t e = dev::launch_scatter_rows(static_cast<const int32_t *>(d_cdst_), pl.T,
                                             static_cast<const bf16 *>(k_new), static_cast<const bf16 *>(v_new),
                                             static_cast<bf16 *>(c_.kpool[layer]), static_cast<bf16 *>(c_.vpool[layer]),
                                             cfg.n_kv_heads, cfg.head_dim, cfg.page_size, sms_, cs(s));
    ++c_.ctr.launches;
    if (e != cudaSuccess) return KVFS_EIO;
    const int G = cfg.n_q_heads / cfg.n_kv_heads;
    alignas(64) CUtensorMap qmap;
    if (!encode_q_map(&qmap, q, pl.T)) return KVFS_EINVAL;
    dev::ChunkParams p{};
    p.units = static_cast<const dev::ChunkUnit *>(d_cunits_);
    p.descs = static_cast<const dev::ChunkDesc *>(d_cdescs_);
    p.slab = slab_;
    p.out = static_cast<bf16 *>(out);
    p.lse = lse;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.P = cfg.page_size;
    p.Hkv = cfg.n_kv_heads;
    p.Hq = cfg.n_q_heads;
    p.pool_rows = static_cast<int>(cfg.n_pages * cfg.n_kv_heads * cfg.page_size);
    e = dev::launch_chunk(kmaps_[layer], vmaps_[layer], qmap, p, static_cast<int>(pl.chunk_units.size()), G, cs(s));
    ++c_.ctr.launches;
    return e == cudaSuccess ? KVFS_OK : KVFS_EIO;
  }

 private:
  struct Staging {
    char *host = nullptr;
    char *dev = nullptr;  // device address of the mapped host buffer
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    bool pending = false;
  };

  static cudaStream_t cs(kvfs_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

  bool grow(Staging &s, size_t need) {
    if (s.cap >= need) return true;
    if (s.pending) {
      cudaEventSynchronize(s.ev);
      s.pending = false;
    }
    if (s.host) cudaFreeHost(s.host);
    s.host = s.dev = nullptr;
    size_t cap = std::max<size_t>(need, 2 * s.cap);
    if (cudaHostAlloc(reinterpret_cast<void **>(&s.host), cap, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void **>(&s.dev), s.host, 0) != cudaSuccess) {
      if (s.host) cudaFreeHost(s.host);
      s.host = s.dev = nullptr;
      s.cap = 0;
      return false;
    }
    s.cap = cap;
    return true;
  }

  // scratch: the packet goes to the second upload area (see WsLayout::scratch), leaving an open step's plan
  // in the first one intact
  void begin_packet(bool scratch = false) {
    area_ = scratch ? upload_ + (lay_.scratch - lay_.upload) : upload_;
    area_cap_ = scratch ? lay_.scratch_cap : lay_.upload_cap;
    cur_ = (cur_ + 1) % 4;
    Staging &s = stg_[cur_];
    if (s.pending) {
      cudaEventSynchronize(s.ev);  // the H2D copy that last used this buffer has finished
      s.pending = false;
    }
    used_ = 0;
    pending_.clear();
  }

  // Reserve bytes in the packet; returns the device address they will occupy.  Data is gathered into the
  // pinned buffer at send().
  const void *push(const void *data, size_t bytes) {
    const size_t off = (used_ + 15) & ~static_cast<size_t>(15);
    if (off + bytes > area_cap_) return nullptr;
    pending_.push_back({data, bytes, off});
    used_ = off + bytes;
    return area_ + off;
  }

  // the packet's pieces into the pinned staging buffer
  bool gather(Staging &st) {
    if (!grow(st, std::max<size_t>(used_, 16))) return false;
    for (const auto &p : pending_)
      if (p.bytes) std::memcpy(st.host + p.off, p.data, p.bytes);
    return true;
  }

  bool send(kvfs_stream_t s) {
    Staging &st = stg_[cur_];
    if (!gather(st)) return false;
    if (used_ == 0) return true;
    const size_t n16 = (used_ + 15) / 16;
    // packets of 16 KB .. 1 MB by SM loads (measured: cfg2 / cfg4 / cfg5 steps faster, e2e +10-17%); smaller
    // ones by DMA, whose fixed cost is lower (cfg3's 9 KB packet: the extra launch cost ~3 us per step)
    if (n16 * 16 <= st.cap && used_ >= (size_t{16} << 10) && used_ <= (size_t{1} << 20)) {
      const int grid = static_cast<int>(std::min<size_t>((n16 + 255) / 256, 64));
      upload_kernel<<<grid, 256, 0, cs(s)>>>(reinterpret_cast<uint4 *>(area_), reinterpret_cast<const uint4 *>(st.dev),
                                             static_cast<int64_t>(n16));
      ++c_.ctr.launches;
      if (cudaGetLastError() != cudaSuccess) return false;
    } else if (cudaMemcpyAsync(area_, st.host, used_, cudaMemcpyHostToDevice, cs(s)) != cudaSuccess) {
      return false;
    }
    if (cudaEventRecord(st.ev, cs(s)) != cudaSuccess) return false;
    st.pending = true;
    c_.ctr.h2d_bytes += static_cast<int64_t>(used_);
    return true;
  }

  int launch_prologue(const dev::SlabRun *runs, int n_runs, const dev::Entry *run_entries,
                      const dev::PageCopy *copies, int n_copies, kvfs_stream_t s) {
    const kvfs_config &cfg = c_.cfg;
    const int blocks = (n_runs + 7) / 8 + n_copies * 2 * cfg.n_layers;
    if (blocks == 0) return KVFS_OK;
    const int64_t page_elems = static_cast<int64_t>(cfg.n_kv_heads) * cfg.page_size * cfg.head_dim;
    prologue_kernel<<<blocks, 256, 0, cs(s)>>>(runs, n_runs, run_entries, slab_, copies, n_copies, kptrs_, vptrs_,
                                               cfg.n_layers, page_elems);
    ++c_.ctr.launches;
    return cudaGetLastError() == cudaSuccess ? KVFS_OK : KVFS_EIO;
  }

  int append_piece(const int32_t *dst, int64_t m, int64_t row_base, int64_t n_total, const bf16 *k, const bf16 *v,
                   kvfs_stream_t s) {
    begin_packet();
    const void *dd = push(dst, static_cast<size_t>(m) * sizeof(int32_t));
    if (!dd) return KVFS_ENOMEM;
    if (!send(s)) return KVFS_EIO;
    const kvfs_config &cfg = c_.cfg;
    const int64_t total = cfg.n_layers * m * cfg.n_kv_heads * (cfg.head_dim / 8);
    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, sms_ * 16));
    append_rows_kernel<<<grid, 256, 0, cs(s)>>>(static_cast<const int32_t *>(dd), m, row_base, n_total, k, v, kptrs_,
                                                vptrs_, cfg.n_layers, cfg.n_kv_heads, cfg.head_dim, cfg.page_size);
    ++c_.ctr.launches;
    return cudaGetLastError() == cudaSuccess ? KVFS_OK : KVFS_EIO;
  }

  // the pool as [n_pages * Hkv * P rows][D] bf16, box 64 dims x box_rows rows, 128-byte swizzle
  bool pool_map(void *pool, CUtensorMap *m, int box_rows) {
    const kvfs_config &cfg = c_.cfg;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cfg.head_dim),
                                static_cast<cuuint64_t>(cfg.n_pages) * cfg.n_kv_heads * cfg.page_size};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cfg.head_dim) * 2};
    const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t es[2] = {1, 1};
    return encode_(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pool, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }

  // the pool as [n_pages * Hkv * P rows][D] with one-row boxes of the whole head dim, no swizzle: the
  // decode kernel's tile::gather4 copies land rows packed in a [row][D] shared-memory stage
  bool row_map(void *pool, CUtensorMap *m) {
    const kvfs_config &cfg = c_.cfg;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cfg.head_dim),
                                static_cast<cuuint64_t>(cfg.n_pages) * cfg.n_kv_heads * cfg.page_size};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cfg.head_dim) * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(cfg.head_dim), 1};
    const cuuint32_t es[2] = {1, 1};
    return encode_(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pool, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }

  struct Pending {
    const void *data;
    size_t bytes, off;
  };
  struct HostBuf {
    void *host, *dev;
    size_t bytes;
    cudaEvent_t ev;
  };
  std::vector<HostBuf> host_cache_;
  std::unordered_map<void *, size_t> host_sizes_;
  size_t cached_bytes_ = 0;

  Ctx &c_;
  WsLayout lay_;
  dev::Entry *slab_ = nullptr;
  char *upload_ = nullptr;
  char *area_ = nullptr;  // upload area of the current packet (upload_ or the scratch area)
  size_t area_cap_ = 0;
  int *counters_ = nullptr;
  int *work_ = nullptr;
  int *pgroup_ = nullptr;
  uint64_t prefix_launches_ = 0;
  float *partials_ = nullptr;
  float *ppart_ = nullptr;
  bf16 **kptrs_ = nullptr, **vptrs_ = nullptr;
  int sms_ = 148;
  int per_sm_ = 0;
  struct IoSlot {  // host-buffer pred: one device slot (inputs, outputs) and its events
    void *in = nullptr, *out = nullptr;
    size_t in_cap = 0, out_cap = 0;
    cudaEvent_t in_ready = nullptr, used = nullptr, out_done = nullptr;
    bool live = false;  // used before (its events were recorded)
  };
  IoSlot io_[2];
  int io_next_ = 0;
  cudaStream_t io_h2d_ = nullptr, io_d2h_ = nullptr;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timing_;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> layer_timing_;  // KVFS_OPT_TIMING: per pred layer
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> copy_timing_;   // KVFS_OPT_TIMING: per K6 launch
  std::vector<cudaEvent_t> ev_pool_;
  int64_t k5_grid_ = 0;
  Staging stg_[4];
  int cur_ = 0;
  size_t used_ = 0;
  std::vector<Pending> pending_;
  const void *d_pctas_ = nullptr;
  const void *d_runs_ = nullptr, *d_run_entries_ = nullptr, *d_copies_ = nullptr, *d_descs_ = nullptr,
             *d_dst_ = nullptr, *d_cdescs_ = nullptr, *d_cunits_ = nullptr, *d_cdst_ = nullptr,
             *d_pdescs_ = nullptr, *d_punits_ = nullptr, *d_prows_ = nullptr;
  PFN_cuTensorMapEncodeTiled_v12000 encode_ = nullptr;
  std::vector<CUtensorMap> kmaps_, vmaps_, smaps_;  // smaps_: K pool in 16-row boxes (K9)
  std::vector<CUtensorMap> gkmaps_, gvmaps_;          // single-row boxes (K1 gather4 over holes)
};

}  // namespace

size_t device_workspace_bytes(const kvfs_config &cfg) { return ws_layout(cfg).total; }

int create_device(Ctx &c, Device **out) {
  auto *d = new (std::nothrow) CudaDevice(c);
  if (!d) return KVFS_ENOMEM;
  const int rc = d->init();
  if (rc != KVFS_OK) {
    delete d;
    return rc;
  }
  *out = d;
  return KVFS_OK;
}

}  // namespace kvfs
