// Device data plane of KVFS: workspace layout, the per-call metadata upload (one pinned H2D copy per
// call), and the bandwidth-bound copy kernels (K4 copy-on-write / fork tail page copy, K5 evict-compact
// gather, K7 dense read-back, the kvfs_append scatter, the table-delta scatter).  The attention kernel
// lives in decode_attn.cu.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
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
  int64_t prefix_cap = 0;  // shared-prefix partials (PART floats each)
};

WsLayout ws_layout(const kvfs_config &c) {
  WsLayout w;
  const int G = c.n_q_heads / c.n_kv_heads;
  const size_t part = static_cast<size_t>(G) * (c.head_dim + 2) * 4;
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
  w.partials = off;
  off = align256(off + static_cast<size_t>(kMaxCtas) * 2 * part);
  w.ptrs = off;
  off = align256(off + static_cast<size_t>(c.n_layers) * 2 * sizeof(void *));
  // shared-prefix (cascade) partials: up to kMaxPrefixSplits key splits per decode unit, capped at 16384
  w.prefix_cap = c.head_dim == 128
                     ? std::min<int64_t>(static_cast<int64_t>(c.max_batch_rows) * c.n_kv_heads * kMaxPrefixSplits, 16384)
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

#ifndef KVFS_K5_MINB
#define KVFS_K5_MINB 1  // resident CTAs per SM the register budget is sized for
#endif
#ifndef KVFS_K5_U
#define KVFS_K5_U 4  // 16-byte K and V loads in flight per thread
#endif

// K5: token i of the old table (logical order) -> (new_pages[i / P], i % P), every layer, K and V.
// A CTA per (destination page, layer), grid-stride over the pages: the P source (page, slot) pairs are
// resolved once into shared memory, then the CTA streams the page's Hkv x P rows of K and V with 16-byte vectors (4 loads in flight
// per thread before the stores).
__global__ void __launch_bounds__(256, KVFS_K5_MINB) compact_kernel(const dev::Entry *old, int n_old, const uint32_t *new_pages,
                                                      int n_new, int64_t len, bf16 *const *kp, bf16 *const *vp, int L,
                                                      int Hkv, int D, int P) {
  __shared__ uint32_t src_page[64];
  __shared__ int src_slot[64];
  const int l = blockIdx.y;
  for (int j = blockIdx.x; j < n_new; j += gridDim.x) {  // grid-stride over destination pages
  const int64_t i0 = static_cast<int64_t>(j) * P;
  const int ntok = static_cast<int>(len - i0 < P ? len - i0 : static_cast<int64_t>(P));
  if (threadIdx.x < ntok) {
    const int64_t i = i0 + threadIdx.x;
    const dev::Entry e = old[find_entry(old, n_old, i)];
    src_page[threadIdx.x] = e.page;
    src_slot[threadIdx.x] = dev::select_bit64(e.mask, static_cast<int>(i - e.lstart));
  }
  __syncthreads();
  const bf16 *ks = kp[l];
  const bf16 *vs = vp[l];
  bf16 *kd = kp[l];
  bf16 *vd = vp[l];
  const int cpr = D / 8;
  const int total = Hkv * ntok * cpr;
  const int64_t dpage = new_pages[j];
  constexpr int U = KVFS_K5_U;
  for (int base = threadIdx.x; base < total; base += U * blockDim.x) {
    uint4 kr[U], vr[U];
    int64_t po[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = base + u * blockDim.x;
      if (idx < total) {
        const int c = idx % cpr, r = idx / cpr, t = r % ntok, g = r / ntok;
        const int64_t so = ((static_cast<int64_t>(src_page[t]) * Hkv + g) * P + src_slot[t]) * D + c * 8;
        po[u] = ((dpage * Hkv + g) * P + t) * D + c * 8;
        kr[u] = *reinterpret_cast<const uint4 *>(ks + so);
        vr[u] = *reinterpret_cast<const uint4 *>(vs + so);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (base + u * static_cast<int>(blockDim.x) < total) {
        *reinterpret_cast<uint4 *>(kd + po[u]) = kr[u];
        *reinterpret_cast<uint4 *>(vd + po[u]) = vr[u];
      }
    }
  }
  __syncthreads();  // src_page / src_slot are rewritten for the next destination page
  }
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
class CudaDevice final : public Device {
 public:
  explicit CudaDevice(Ctx &c) : c_(c) {}
  ~CudaDevice() override {
    for (auto &s : stg_) {
      if (s.ev) cudaEventDestroy(s.ev);
      if (s.host) cudaFreeHost(s.host);
    }
    for (auto &b : host_cache_) {
      if (b.ev) cudaEventDestroy(b.ev);
      cudaFreeHost(b.host);
    }
    for (auto &kv : host_sizes_) cudaFreeHost(kv.first);
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

  int compact(const std::vector<Entry> &old_table, const std::vector<uint32_t> &new_pages, int64_t len,
              kvfs_stream_t s) override {
    begin_packet();
    const void *dt = push(old_table.data(), old_table.size() * sizeof(Entry));
    const void *dp = push(new_pages.data(), new_pages.size() * sizeof(uint32_t));
    if (!dt || !dp) return KVFS_ENOMEM;
    if (!send(s)) return KVFS_EIO;
    const kvfs_config &cfg = c_.cfg;
    // one wave: up to 8 resident CTAs per SM, each looping over destination pages (a file of ~2k pages
    // was 1.7 waves of one-page CTAs)
    const int64_t per_layer = std::max<int64_t>(1, static_cast<int64_t>(sms_) * 8 / cfg.n_layers);  // >= resident
    const dim3 grid(static_cast<unsigned>(std::min<int64_t>(static_cast<int64_t>(new_pages.size()), per_layer)),
                    static_cast<unsigned>(cfg.n_layers));
    compact_kernel<<<grid, 256, 0, cs(s)>>>(static_cast<const dev::Entry *>(dt), static_cast<int>(old_table.size()),
                                            static_cast<const uint32_t *>(dp), static_cast<int>(new_pages.size()), len,
                                            kptrs_, vptrs_, cfg.n_layers, cfg.n_kv_heads, cfg.head_dim, cfg.page_size);
    ++c_.ctr.launches;
    return cudaGetLastError() == cudaSuccess ? KVFS_OK : KVFS_EIO;
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
    d_runs_ = push(pl.runs.data(), pl.runs.size() * sizeof(SlabRun));
    d_run_entries_ = push(pl.run_entries.data(), pl.run_entries.size() * sizeof(Entry));
    d_copies_ = push(pl.copies.data(), pl.copies.size() * sizeof(PageCopy));
    d_descs_ = push(pl.descs.data(), pl.descs.size() * sizeof(DevDesc));
    d_dst_ = push(pl.dst_slot.data(), pl.dst_slot.size() * sizeof(int32_t));
    d_cdescs_ = push(pl.chunk_descs.data(), pl.chunk_descs.size() * sizeof(ChunkDesc));
    d_cunits_ = push(pl.chunk_units.data(), pl.chunk_units.size() * sizeof(ChunkUnit));
    d_cdst_ = push(pl.chunk_dst.data(), pl.chunk_dst.size() * sizeof(int32_t));
    d_pdescs_ = push(pl.prefix_descs.data(), pl.prefix_descs.size() * sizeof(PrefixDesc));
    d_punits_ = push(pl.prefix_units.data(), pl.prefix_units.size() * sizeof(ChunkUnit));
    d_prows_ = push(pl.prefix_rows.data(), pl.prefix_rows.size() * sizeof(PrefixRow));
    if (!d_runs_ || !d_run_entries_ || !d_copies_ || !d_descs_ || !d_dst_ || !d_cdescs_ || !d_cunits_ || !d_cdst_ ||
        !d_pdescs_ || !d_punits_ || !d_prows_)
      return KVFS_ENOMEM;
    if (!send(s)) return KVFS_EIO;
    if (pl.runs.empty() && pl.copies.empty()) return KVFS_OK;
    return launch_prologue(static_cast<const dev::SlabRun *>(d_runs_), static_cast<int>(pl.runs.size()),
                           static_cast<const dev::Entry *>(d_run_entries_),
                           static_cast<const dev::PageCopy *>(d_copies_), static_cast<int>(pl.copies.size()), s);
  }

  int pred_layer(const PredPlan &pl, int layer, const void *q, const void *k_new, const void *v_new, void *out,
                 float *lse, float scale, kvfs_stream_t s) override {
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
    p.Hq = cfg.n_q_heads;
    p.Hkv = cfg.n_kv_heads;
    // always a programmatic dependent launch: after the prologue (waits at start) or after the shared-prefix
    // kernel (which waited for the prologue itself; waits before merging)
    const cudaError_t e = dev::launch_decode(p, cfg.head_dim, cfg.n_q_heads / cfg.n_kv_heads, cfg.page_size, cs(s),
                                             true);
    ++c_.ctr.launches;
    c_.ctr.last_decode_ctas = ncta;
    return e == cudaSuccess ? KVFS_OK : KVFS_EIO;
  }

  int sync() override { return cudaDeviceSynchronize() == cudaSuccess ? KVFS_OK : KVFS_EIO; }
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
    const cudaError_t e = dev::launch_prefix(kmaps_[layer], vmaps_[layer], kmaps_[layer], p,
                                             static_cast<int>(pl.prefix_units.size()), G, cs(s));
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
    pack_kernel<<<static_cast<unsigned>(blocks), 256, 0, cs(s)>>>(static_cast<const uint32_t *>(dp),
                                                                  static_cast<int>(pages.size()), kptrs_, vptrs_,
                                                                  cfg.n_layers, page_elems, static_cast<bf16 *>(buf),
                                                                  unpack);
    ++c_.ctr.launches;
    return cudaGetLastError() == cudaSuccess ? KVFS_OK : KVFS_EIO;
  }

  // K2: scatter the chunk descriptors' new rows into the pool, then tcgen05 attention from the pool.
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
    {
      const cuuint64_t dims[4] = {static_cast<cuuint64_t>(cfg.head_dim), static_cast<cuuint64_t>(G),
                                  static_cast<cuuint64_t>(cfg.n_kv_heads), static_cast<cuuint64_t>(pl.T)};
      const cuuint64_t strides[3] = {static_cast<cuuint64_t>(cfg.head_dim) * 2,
                                     static_cast<cuuint64_t>(G) * cfg.head_dim * 2,
                                     static_cast<cuuint64_t>(cfg.n_q_heads) * cfg.head_dim * 2};
      const cuuint32_t box[4] = {64, static_cast<cuuint32_t>(G), 1, static_cast<cuuint32_t>(128 / G)};
      const cuuint32_t es[4] = {1, 1, 1, 1};
      if (encode_(&qmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(q), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return KVFS_EINVAL;
    }
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

  bool send(kvfs_stream_t s) {
    Staging &st = stg_[cur_];
    if (!grow(st, std::max<size_t>(used_, 16))) return false;
    for (const auto &p : pending_)
      if (p.bytes) std::memcpy(st.host + p.off, p.data, p.bytes);
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
  float *partials_ = nullptr;
  float *ppart_ = nullptr;
  bf16 **kptrs_ = nullptr, **vptrs_ = nullptr;
  int sms_ = 148;
  int per_sm_ = 0;
  Staging stg_[4];
  int cur_ = 0;
  size_t used_ = 0;
  std::vector<Pending> pending_;
  const void *d_runs_ = nullptr, *d_run_entries_ = nullptr, *d_copies_ = nullptr, *d_descs_ = nullptr,
             *d_dst_ = nullptr, *d_cdescs_ = nullptr, *d_cunits_ = nullptr, *d_cdst_ = nullptr,
             *d_pdescs_ = nullptr, *d_punits_ = nullptr, *d_prows_ = nullptr;
  PFN_cuTensorMapEncodeTiled_v12000 encode_ = nullptr;
  std::vector<CUtensorMap> kmaps_, vmaps_, smaps_;  // smaps_: K pool in 16-row boxes (K9)
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
