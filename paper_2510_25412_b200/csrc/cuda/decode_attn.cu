// K1: fused append + split-KV page-gathering GQA attention for the batched `pred` (§4.1
// P:210-215 semantics, rule R10 of SURVEY.md §8(c); HBM-bound, AI ~ 4 flop/B).
//
// Work decomposition ("stage" = one (page entry, kv head) block of K and V, or one block of up to P new
// rows of K_new/V_new):
//   unit  = (descriptor d, kv head g, query row qi): the G query heads of one new token against the
//           file's retained tokens;  units of d are ordered g-major so that consecutive units (same g,
//           consecutive qi) stream the same pages;
//   stages of a unit = its file's n_old_entries page entries, then ceil(n_q / P) "new-row" stages;
//   the batch's stages are concatenated in descriptor order and the grid splits that sequence into
//   equal contiguous ranges, one per CTA (split-KV at page granularity, exact load balance).
//   A unit cut by a range boundary is finished by whichever CTA completes its last piece: partial
//   (O, m, l) go to the workspace and that CTA merges them in range order (deterministic).
// Per CTA: one producer lane streams stages into a ring of NSTAGES shared-memory slots with 1-D TMA
// bulk copies (cp.async.bulk, completion on mbarriers, evict-first L2 policy); NW consumer warps take
// ring slots round-robin.  In a consumer warp, LPK lanes share one key (16 B bf16 vectors, DPL dims per
// lane), so a warp scores KG = 32/LPK keys per step with packed fp32x2 FMAs and an xor-shuffle
// reduction; softmax is online in the log2 domain with lazy rescaling (only when the running max grows
// by > 8); the new-row stage of unit qi = 0 also writes K_new/V_new into the file's reserved slots
// (the fused append).  Warps combine through shared memory at unit boundaries.
#include <cuda_bf16.h>
#include <math_constants.h>

#include <type_traits>

#include "kernels.cuh"

namespace kvfs {
namespace dev {

template <int D_, int G_, int P_>
struct DecodeCfg {
  static constexpr int D = D_, G = G_, P = P_;
  static constexpr int DPL = (G <= 4) ? 16 : 8;  // dims per lane
  static constexpr int LPK = D / DPL;            // lanes per key
  static constexpr int KG = 32 / LPK;            // keys per warp step
  static constexpr int CH = DPL / 8;             // 16-byte chunks per lane per row
  static constexpr int SUB = 16;                 // slots per softmax sub-block
  static constexpr int NIT = SUB / KG;           // warp steps per sub-block
  static constexpr int BLOCK_BYTES = P * D * 2;  // one (page, head) block of K or V
  static constexpr int STAGE_BYTES = 2 * BLOCK_BYTES;
  // One CTA per SM holding R independent rings; ring = 1 producer warp (1-D TMA) + NW consumer warps.
  // An SM's TMA bandwidth grows with the number of independent producer streams (tools/bw_probe.cu:
  // 1 stream/SM ~2.5 TB/s, 3-4 streams/SM ~6.4-6.9 TB/s), so the rings are what feeds HBM; one CTA of
  // 12 warps lets setmaxnreg move registers from the 4-warp producer warpgroup to the 8 consumers.
#ifndef KVFS_K1_NW
#define KVFS_K1_NW 2
#endif
  static constexpr int NW = KVFS_K1_NW;          // consumer warps per ring (8 / NW rings per CTA)
  static constexpr int NSTAGES_RAW = 49152 / 2 * NW / STAGE_BYTES;  // 48 KiB of stages per 2 consumer warps
  static constexpr int NSTAGES = NSTAGES_RAW < NW ? NW : (NSTAGES_RAW > 16 ? 16 : NSTAGES_RAW);
  // NW <= NSTAGES is required: a warp never waits on a ring slot more than one phase ahead (mbarrier
  // parity waits are ambiguous beyond that).
  static constexpr int THREADS = 12 * 32;        // producer warpgroup (4 warps) + 2 consumer warpgroups
  static constexpr int PRODUCER_REGS = 56, CONSUMER_REGS = 224;
  static constexpr int NQ = 4;                   // Q ring slots
  static constexpr int PART = part_floats(G, D);  // floats per partial (o, m, l per head, 16-byte padded)
  static constexpr int KDEF = kDecodeRecSlots;   // workspace records per range; deferred merges per ring
  static constexpr int SEGMETA_BYTES = 64;       // per Q slot: the producer's resolved segment (struct SegMeta)
  static constexpr int RING_BYTES_RAW = NSTAGES * STAGE_BYTES + NQ * G * D * 2 + NW * PART * 4 + NSTAGES * 16 +
                                        (2 * NSTAGES + 2 * NQ + 4) * 8 + 32 + KDEF * 32 + NQ * SEGMETA_BYTES;
  static constexpr int RING_BYTES = (RING_BYTES_RAW + 127) / 128 * 128;
  static constexpr int R_RAW = 232448 / RING_BYTES;  // 227 KB of dynamic shared memory per CTA
  static constexpr int R = R_RAW > 8 / NW ? 8 / NW : R_RAW;  // rings per CTA
  static_assert(LPK * KG == 32 && SUB % KG == 0 && P % SUB == 0 && NW <= NSTAGES && NW * R <= 8 && R >= 1, "layout");
  static_assert(!(D == 128 && G == 4 && P == 16 && NW == 2) || R == 4, "the 8B shape keeps 4 rings per CTA");
};

// A segment of a unit whose final merge waits for the shared-prefix grid (Desc::pref_splits != 0): its record
// is in the partials workspace, and the arrival count, the merge and the wait run only when the ring has
// streamed its range (flush_deferred), so the ring never stalls on the prefix kernel (or on a fence) between
// two of its segments.
struct Deferred {
  int64_t ubeg;   // global stage index of the unit's first stage
  int32_t d;      // descriptor
  int32_t unit;   // Desc::unit_base + g * n_q + qi
  int32_t rslot;  // >= 0: a whole unit, its record in slot rslot of the range; -1: a piece (slot 0 / 1)
  int32_t merge;  // flush: this ring merges the unit
  int32_t pad[2];
};

struct StageMeta {
  uint64_t mask;  // slots (or new rows) that are visible keys
  int32_t kind;   // 0 = page entry, 1 = new rows
  int32_t nrows;  // new-row stage: rows loaded
};



__device__ __forceinline__ int64_t cta_start(int64_t c, const DecodeParams &p) { return c * p.total / p.ncta; }

// chunk holding stage x
__device__ __forceinline__ int cta_of(int64_t x, const DecodeParams &p) {
  int64_t c = x * p.ncta / p.total;
  if (c >= p.ncta) c = p.ncta - 1;
  while (c + 1 < p.ncta && cta_start(c + 1, p) <= x) ++c;
  while (c > 0 && cta_start(c, p) > x) --c;
  return static_cast<int>(c);
}

// Largest d with descs[d].cost_begin <= x (cost_begin is nondecreasing, descs[0].cost_begin = 0).
// Warp-collective (all 32 lanes, uniform arguments): each round the lanes probe 32 evenly spaced
// descriptors in one load, so a batch of n descriptors takes ceil(log33 n) dependent loads (2 for 1024)
// instead of log2 n (a cold ring start used to spend ~3 us in the binary search).  hint >= 0: the caller
// knows d >= hint (the previous segment's descriptor); a short forward scan from it first.
__device__ __forceinline__ int find_desc(const Desc *descs, int n, int64_t x, int hint) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = n - 1;  // the answer is in [lo, hi]
  if (hint >= 0) {
    // lanes probe hint + 1 .. hint + 32: the answer is hint + (number of probes <= x), if not past them
    const int pos = hint + 1 + lane;
    const bool le = pos < n && descs[pos].cost_begin <= x;
    const unsigned m = __ballot_sync(0xffffffffu, le);
    if (m != 0xffffffffu) return hint + __popc(m);
    lo = hint + 32;
  }
  while (lo < hi) {
    const int64_t span = hi - lo;                                   // candidates lo + 1 .. hi
    const int pos = lo + 1 + static_cast<int>(span * lane / 32);   // nondecreasing in lane, <= hi
    const bool le = descs[pos].cost_begin <= x;
    const unsigned m = __ballot_sync(0xffffffffu, le);
    if (m == 0) return lo;  // pos(lane 0) = lo + 1 is already past x
    const int L = 31 - __clz(m);  // last lane whose probe is <= x (probes are monotone)
    const int newlo = lo + 1 + static_cast<int>(span * L / 32);
    const int newhi = (L < 31) ? lo + static_cast<int>(span * (L + 1) / 32) : hi;  // pos(L + 1) - 1
    lo = newlo;
    hi = newhi;
  }
  return lo;
}

struct Segment {
  int d;         // descriptor
  int g, qi;     // kv head, query row within the descriptor
  int st0, nst;  // first stage within the unit, number of stages
  int spu;       // stages per unit
  int64_t ubeg;  // global stage index of the unit's first stage
};

// Segment containing global stage x (x < total), clipped to [x, end).  Warp-collective (find_desc).
__device__ __forceinline__ Segment make_segment(const Desc *descs, int n_desc, int64_t x, int64_t end, int hint) {
  Segment s;
  s.d = find_desc(descs, n_desc, x, hint);
  const Desc &dd = descs[s.d];
  s.spu = dd.stages_per_unit;
  const int64_t rel = x - dd.cost_begin;
  const int u = static_cast<int>(rel / s.spu);
  s.st0 = static_cast<int>(rel - static_cast<int64_t>(u) * s.spu);
  s.g = u / dd.n_q;
  s.qi = u - s.g * dd.n_q;
  s.ubeg = dd.cost_begin + static_cast<int64_t>(u) * s.spu;
  const int64_t uend = s.ubeg + s.spu;
  s.nst = static_cast<int>((end < uend ? end : uend) - x);
  return s;
}

// A segment as the producer resolved it, handed to the ring's consumers with the segment's Q slot (written
// before the Q slot's arrive, which releases it): the consumers do not repeat the descriptor search and the
// descriptor load, two dependent global loads at every segment start.
// (64 bytes: the 4 rings of a CTA then still fit 227 KB of shared memory at the 8B shape)
struct SegMeta {
  int64_t ubeg, logit_off;
  int32_t d, g, qi, st0, nst, spu;
  int32_t n_os, n_q, row0, unit_base, pref_splits, pref_base;  // n_os = old-entry stages (n_old_entries - skip)
};
static_assert(sizeof(SegMeta) == 64, "SegMeta must be DecodeCfg::SEGMETA_BYTES");

// Final merge of a unit's output (whole unit, or the last piece of a unit cut by ring boundaries).  Each of
// the ring's NT = NW * 32 consumer threads owns one head h and DPT consecutive dims d0 .. d0 + DPT of it and
// folds (o, m, l) partial records into a running (M, L, acc) in the log2 domain.  Global records (other
// rings' pieces, shared-prefix key splits) are read in groups of SG with every load of a group in flight, so
// a merge of S prefix splits costs ceil(S / SG) L2 round trips (not one per element and split).
template <int D, int G, int NT>
struct MergeMap {
  static constexpr int TPH = NT / G > D ? D : NT / G;  // threads per head (threads past G TPH idle)
  static constexpr int DPT = D / TPH;  // dims per thread
  static constexpr int SG = DPT >= 16 ? 4 : (DPT >= 8 ? 8 : 16);
  static_assert(NT % G == 0 && D % TPH == 0 && DPT >= 1, "merge map");
};

template <int DPT>
__device__ __forceinline__ void ld_dims(const float *p, float (&x)[DPT]) {
  if constexpr (DPT % 2 == 0) {
#pragma unroll
    for (int i = 0; i < DPT / 2; ++i) {
      const float2 t = __ldcg(reinterpret_cast<const float2 *>(p) + i);
      x[2 * i] = t.x;
      x[2 * i + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < DPT; ++i) x[i] = __ldcg(p + i);
  }
}

// Fold n records rec(s) = base + s * stride (s < n) of one head: (o[D], m, l); the thread's dims at d0.
template <int D, int DPT, int SG>
__device__ __forceinline__ void fold_records(const float *base, int64_t stride, int n, int d0, float &M, float &L,
                                             float (&acc)[DPT]) {
  for (int s0 = 0; s0 < n; s0 += SG) {
    float2 ml[SG];
    float o[SG][DPT];
#pragma unroll
    for (int j = 0; j < SG; ++j) {
      ml[j] = make_float2(-CUDART_INF_F, 0.f);
#pragma unroll
      for (int i = 0; i < DPT; ++i) o[j][i] = 0.f;
      if (s0 + j < n) {
        const float *r = base + (s0 + j) * stride;
        ml[j] = __ldcg(reinterpret_cast<const float2 *>(r + D));
        ld_dims<DPT>(r + d0, o[j]);
      }
    }
    float Mg = M;
#pragma unroll
    for (int j = 0; j < SG; ++j) Mg = fmaxf(Mg, ml[j].x);
    if (Mg == -CUDART_INF_F) continue;
    const float a = (M == -CUDART_INF_F) ? 0.f : fast_exp2(M - Mg);
    L *= a;
#pragma unroll
    for (int i = 0; i < DPT; ++i) acc[i] *= a;
#pragma unroll
    for (int j = 0; j < SG; ++j) {
      const float f = (ml[j].x == -CUDART_INF_F) ? 0.f : fast_exp2(ml[j].x - Mg);
      L += ml[j].y * f;
#pragma unroll
      for (int i = 0; i < DPT; ++i) acc[i] += o[j][i] * f;
    }
    M = Mg;
  }
}

// Fold the n <= N records rec[j] (each (o[D], m, l) of one head; the thread's dims at d0) with every load in
// flight at once (one L2 round trip for a unit's pieces and shared-prefix splits together).
template <int D, int DPT, int N>
__device__ __forceinline__ void fold_ptrs(const float *const (&rec)[N], int n, int d0, float &M, float &L,
                                          float (&acc)[DPT]) {
  float2 ml[N];
  float o[N][DPT];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    ml[j] = make_float2(-CUDART_INF_F, 0.f);
#pragma unroll
    for (int i = 0; i < DPT; ++i) o[j][i] = 0.f;
    if (j < n) {
      ml[j] = __ldcg(reinterpret_cast<const float2 *>(rec[j] + D));
      ld_dims<DPT>(rec[j] + d0, o[j]);
    }
  }
  float Mg = M;
#pragma unroll
  for (int j = 0; j < N; ++j) Mg = fmaxf(Mg, ml[j].x);
  if (Mg == -CUDART_INF_F) return;
  const float a = (M == -CUDART_INF_F) ? 0.f : fast_exp2(M - Mg);
  L *= a;
#pragma unroll
  for (int i = 0; i < DPT; ++i) acc[i] *= a;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const float f = (ml[j].x == -CUDART_INF_F) ? 0.f : fast_exp2(ml[j].x - Mg);
    L += ml[j].y * f;
#pragma unroll
    for (int i = 0; i < DPT; ++i) acc[i] += o[j][i] * f;
  }
  M = Mg;
}

// The ring's warps' (o, m, l) of this segment from shared memory (comb), head h, dims d0..
template <int D, int DPT, int NW, int PART>
__device__ __forceinline__ void fold_comb(const float *comb, int h, int d0, float &M, float &L, float (&acc)[DPT]) {
  M = -CUDART_INF_F;
  L = 0.f;
#pragma unroll
  for (int i = 0; i < DPT; ++i) acc[i] = 0.f;
#pragma unroll
  for (int w = 0; w < NW; ++w) M = fmaxf(M, comb[w * PART + h * (D + 2) + D]);
  if (M == -CUDART_INF_F) return;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const float *cw = comb + w * PART + h * (D + 2);
    const float f = (cw[D] == -CUDART_INF_F) ? 0.f : fast_exp2(cw[D] - M);
    L += cw[D + 1] * f;
#pragma unroll
    for (int i = 0; i < DPT; ++i) acc[i] += cw[d0 + i] * f;
  }
}

// out[d0 .. d0 + DPT) = acc / L as bf16 (RNE), lse = (M + log2 L) ln 2 by the thread holding d0 = 0
template <int DPT>
__device__ __forceinline__ void store_out(__nv_bfloat16 *o, float *lse, int d0, float M, float L,
                                          const float (&acc)[DPT]) {
  const float inv = 1.f / L;
  if constexpr (DPT == 1) {
    o[0] = __float2bfloat16_rn(acc[0] * inv);
  } else {
    uint32_t w[DPT / 2];
#pragma unroll
    for (int i = 0; i < DPT / 2; ++i) {
      __nv_bfloat162 pr = __floats2bfloat162_rn(acc[2 * i] * inv, acc[2 * i + 1] * inv);
      w[i] = *reinterpret_cast<uint32_t *>(&pr);
    }
    if constexpr (DPT == 2) {
      *reinterpret_cast<uint32_t *>(o) = w[0];
    } else if constexpr (DPT == 4) {
      *reinterpret_cast<uint2 *>(o) = make_uint2(w[0], w[1]);
    } else {
#pragma unroll
      for (int i = 0; i < DPT / 8; ++i)
        reinterpret_cast<uint4 *>(o)[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
    }
  }
  if (d0 == 0 && lse) *lse = (M + __log2f(L)) * 0.69314718055994531f;
}

#ifdef KVFS_K1_TRACE
// Development trace (tools/cascade_trace.py): per physical ring, %globaltimer (ns) at kernel start, the
// producer's first TMA, the consumers' first full stage, the end of streaming and the end of the output.
__device__ unsigned long long g_k1_trace[8][2048];
__device__ __forceinline__ unsigned long long k1_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define K1T(ev, r)                                  \
  do {                                              \
    if ((r) < 2048) g_k1_trace[ev][r] = k1_now();   \
  } while (0)
extern "C" int kvfs_debug_k1_trace(void *host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, g_k1_trace, bytes < sizeof(g_k1_trace) ? bytes : sizeof(g_k1_trace)) ==
                 cudaSuccess ? 0 : -1;
}
#else
#define K1T(ev, r) \
  do {             \
  } while (0)
#endif

// Position of the k-th (0-based) set bit of a 16-bit mask (k < popc(m)): a 4-step popcount search.
__device__ __forceinline__ int kth_set_bit16(uint32_t m, int k) {
  int pos = 0;
  int c = __popc(m & 0xFFu);
  if (k >= c) { k -= c; pos += 8; m >>= 8; }
  c = __popc(m & 0xFu);
  if (k >= c) { k -= c; pos += 4; m >>= 4; }
  c = __popc(m & 0x3u);
  if (k >= c) { k -= c; pos += 2; m >>= 2; }
  if (k >= static_cast<int>(m & 1u)) pos += 1;
  return pos;
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1) decode_attn_kernel(const __grid_constant__ DecodeParams p) {
  constexpr int D = C::D, G = C::G, P = C::P, NW = C::NW, NSTAGES = C::NSTAGES;
  constexpr int LPK = C::LPK, KG = C::KG, CH = C::CH, DPL = C::DPL, NIT = C::NIT, SUB = C::SUB;
  extern __shared__ __align__(128) uint8_t smem_all[];
  const int warp_all = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool is_producer = warp_all < 4;
  const int ring = is_producer ? warp_all : (warp_all - 4) / NW;
  const int warp = is_producer ? NW : (warp_all - 4) % NW;  // consumer index in the ring (NW = producer)
  uint8_t *smem = smem_all + ring * C::RING_BYTES;
  uint8_t *stage_data = smem;                                                    // [NSTAGES][2][P][D] bf16
  __nv_bfloat16 *qring = reinterpret_cast<__nv_bfloat16 *>(smem + NSTAGES * C::STAGE_BYTES);  // [NQ][G][D]
  float *comb = reinterpret_cast<float *>(qring + C::NQ * G * D);                // [NW][PART]
  StageMeta *meta = reinterpret_cast<StageMeta *>(comb + NW * C::PART);          // [NSTAGES]
  uint64_t *bars = reinterpret_cast<uint64_t *>(meta + NSTAGES);  // full, empty, qfull, qempty, cfull, cempty
  int *flag = reinterpret_cast<int *>(bars + 2 * NSTAGES + 2 * C::NQ + 4);
  int *chunk_slot = flag + 4;                                        // [2] chunk ids (dynamic scheduling)
  SegMeta *segmeta = reinterpret_cast<SegMeta *>(reinterpret_cast<uint8_t *>(flag + 8) + C::KDEF * 32);  // [NQ]

  // Physical ring pr processes "chunks" = virtual CTAs (contiguous stage ranges, p.ncta of them): static
  // scheduling gives ring pr chunk pr; dynamic scheduling (p.dynamic) lets the ring's producer take chunk
  // after chunk from a global counter and hand each id to its consumers through a 2-slot chunk ring, so
  // rings whose SM frees up early (e.g. next to the shared-prefix kernel of a cascade) do more of the work.
  const int pr = blockIdx.x * C::R + ring;
  auto full_bar = [&](int s) { return smem_u32(bars + s); };
  auto empty_bar = [&](int s) { return smem_u32(bars + NSTAGES + s); };
  auto qfull_bar = [&](int s) { return smem_u32(bars + 2 * NSTAGES + s); };
  auto qempty_bar = [&](int s) { return smem_u32(bars + 2 * NSTAGES + C::NQ + s); };
  auto cfull_bar = [&](int s) { return smem_u32(bars + 2 * NSTAGES + 2 * C::NQ + s); };
  auto cempty_bar = [&](int s) { return smem_u32(bars + 2 * NSTAGES + 2 * C::NQ + 2 + s); };

  if (threadIdx.x < C::R) {  // thread r initialises ring r's barriers
    uint64_t *rb = reinterpret_cast<uint64_t *>(
        reinterpret_cast<uint8_t *>(bars) + (static_cast<int>(threadIdx.x) - ring) * C::RING_BYTES);
    for (int s = 0; s < NSTAGES; ++s) {
      mbar_init(smem_u32(rb + s), 1);
      mbar_init(smem_u32(rb + NSTAGES + s), 1);
    }
    for (int s = 0; s < C::NQ; ++s) {
      mbar_init(smem_u32(rb + 2 * NSTAGES + s), 1);
      mbar_init(smem_u32(rb + 2 * NSTAGES + C::NQ + s), NW);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(rb + 2 * NSTAGES + 2 * C::NQ + s), 1);
      mbar_init(smem_u32(rb + 2 * NSTAGES + 2 * C::NQ + 2 + s), NW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // launched programmatically after the table-delta prologue (no shared-prefix kernel in between): the
  // setup above overlapped its tail; wait for it before reading the page tables
  if (p.wait_at_start) asm volatile("griddepcontrol.wait;" ::: "memory");
  // The next step's prologue (a programmatic launch that waits for this grid before touching anything) may be
  // launched now: its launch latency then overlaps this kernel instead of following it.
  asm volatile("griddepcontrol.launch_dependents;");
  const bool ring_live = ring < C::R && pr < p.n_rings;
#ifdef KVFS_K1_TRACE
  if (is_producer && lane == 0 && ring_live) {
    K1T(0, pr);
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (pr < 2048) g_k1_trace[5][pr] = smid;
  }
#endif

  if (is_producer) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::PRODUCER_REGS));
    if (!ring_live) return;
    // ================================================================ producer warp
    // Lanes prepare up to 32 stages at once (one coalesced load of their page-table entries), then lane 0
    // issues them in order: wait for the ring slot, publish the stage meta, arm the barrier, 1-D TMA.
    const uint64_t pol = policy_evict_first();
    int local = 0, segi = 0;
    for (int k = 0;; ++k) {
    int cta = (k == 0) ? pr : p.ncta;  // static: one chunk per ring
    if (p.dynamic) {
      if (lane == 0) {
        cta = atomicAdd(p.work, 1);
        if (k >= 2) mbar_wait_sleep(cempty_bar(k & 1), ((k >> 1) & 1) ^ 1);
        chunk_slot[k & 1] = cta;
        mbar_arrive(cfull_bar(k & 1));  // release: the id is visible to the consumers
        // the last ring to run out of chunks resets the counters for the next launch (every ring's final
        // fetch happened before its increment of the second counter)
        if (cta >= p.ncta && atomicAdd(p.work + 1, 1) == p.n_rings - 1) {
          p.work[0] = 0;
          p.work[1] = 0;
        }
      }
      cta = __shfl_sync(0xffffffffu, cta, 0);
    }
    if (cta >= p.ncta) break;
    const int64_t beg = cta_start(cta, p), end = cta_start(cta + 1, p);
    int64_t x = beg;
    int dhint = -1;
    while (x < end) {
      const Segment sg = make_segment(p.descs, p.n_desc, x, end, dhint);
      dhint = sg.d;
      const Desc dd = p.descs[sg.d];
      if (lane == 0) {  // Q rows of this unit -> Q ring, with the resolved segment
        const int qs = segi % C::NQ;
        if (segi >= C::NQ) mbar_wait_sleep(qempty_bar(qs), ((segi / C::NQ) & 1) ^ 1);
        segmeta[qs] = SegMeta{sg.ubeg, dd.logit_off, sg.d, sg.g, sg.qi, sg.st0, sg.nst, sg.spu,
                              dd.n_old_entries - dd.skip, dd.n_q, dd.row0, dd.unit_base, dd.pref_splits, dd.pref_base};
        const __nv_bfloat16 *src = p.q + (static_cast<int64_t>(dd.row0 + sg.qi) * p.Hq + sg.g * G) * D;
        mbar_arrive_expect_tx(qfull_bar(qs), G * D * 2);
        bulk_g2s(smem_u32(qring + qs * G * D), src, G * D * 2, qfull_bar(qs), pol);
      }
      for (int base = 0; base < sg.nst; base += 32) {
        const int n = min(32, sg.nst - base);
        uint64_t mask = 0;
        int64_t off = 0;
        int lo = 0, nrows = 0;
        const int st = sg.st0 + base + lane;
        const int n_os = dd.n_old_entries - dd.skip;  // old-entry stages (the shared prefix is skipped)
        if (lane < n) {
          if (st < n_os) {
            const int ent = st + dd.skip;
            const Entry e = p.slab[dd.slab_off + ent];
            mask = e.mask;
            // only the last old entry can also hold new tokens (the device lstart is not maintained)
            if (ent == dd.n_old_entries - 1) mask = lowest_bits(mask, dd.n_old - dd.tail_lstart);
            lo = __ffsll(static_cast<long long>(mask)) - 1;
            const int hi = 63 - __clzll(static_cast<long long>(mask));
            nrows = hi - lo + 1;
            off = ((static_cast<int64_t>(e.page) * p.Hkv + sg.g) * P + lo) * D;
            // sparse span (lazy eviction left more than 60% of it as holes): fetch only the retained rows
            // (gather4), packed from stage row 0; nrows < 0 marks it (-popcount).  Measured on cfg5(ii)
            // (50% random holes, spans ~57% retained): gather4 of every holey span 7.7 ms = 2.2 TB/s of
            // retained bytes against 5.7 ms for the span copies (5.3 TB/s raw), so the break-even density is
            // ~0.42 (gather4 is bound by TMA operations of 4 x 256 B, not by bytes)
            if (p.gather && mask != 0 && 5 * __popcll(mask) < 2 * nrows) nrows = -__popcll(mask);
          } else {
            const int v0 = (st - n_os) * P;
            const int r_end = min(dd.n_q, v0 + P);
            const int vis_end = min(r_end, sg.qi + 1);  // causal: row qi sees new rows <= qi
            const int n_vis = vis_end > v0 ? vis_end - v0 : 0;
            mask = n_vis >= 64 ? ~0ull : ((1ull << n_vis) - 1);
            nrows = (sg.qi == 0) ? (r_end - v0) : n_vis;  // unit qi = 0 also writes the append
            lo = -1;                                        // marks a new-row stage
            off = static_cast<int64_t>(v0);
          }
        }
        for (int j = 0; j < n; ++j, ++local) {
          const uint64_t mj = __shfl_sync(0xffffffffu, mask, j);
          const int64_t offj = __shfl_sync(0xffffffffu, off, j);
          const int loj = __shfl_sync(0xffffffffu, lo, j);
          const int nrj = __shfl_sync(0xffffffffu, nrows, j);
          if (lane == 0) {
            if (local == 0) K1T(1, pr);
            const int slot = local % NSTAGES;
            if (local >= NSTAGES) mbar_wait_sleep(empty_bar(slot), ((local / NSTAGES) & 1) ^ 1);
            const uint32_t kdst = smem_u32(stage_data + slot * C::STAGE_BYTES);
            const uint32_t vdst = kdst + C::BLOCK_BYTES;
            StageMeta m;
            m.mask = mj;
            if (loj >= 0 && nrj < 0) {
              // gathered stage: the n retained rows of the page's span, in slot order, at stage rows 0 .. n-1
              // (the consumers see them as slots 0 .. n-1: attention over a set; the fused-scores logits use
              // the same packed index, K10 recomputes it); 4 rows per gather4, the last group padded by
              // repeating its last row
              const int n = -nrj;
              m.kind = 0;
              m.nrows = 0;
              m.mask = (1ull << n) - 1;  // n < P <= 64
              meta[slot] = m;
              const int rowb = static_cast<int>(offj / D) - loj;  // pool row of slot 0 of the (page, head)
              mbar_arrive_expect_tx(full_bar(slot), static_cast<uint32_t>((n + 3) / 4) * 4 * D * 2 * 2);
              uint64_t mm = mj;
              for (int gi = 0; gi < n; gi += 4) {
                int r[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                  if (mm) {
                    r[t] = rowb + __ffsll(static_cast<long long>(mm)) - 1;
                    mm &= mm - 1;
                  } else {
                    r[t] = r[t > 0 ? t - 1 : 0];
                  }
                }
                tma_gather4(kdst + gi * D * 2, &p.gk, 0, r[0], r[1], r[2], r[3], full_bar(slot), pol);
                tma_gather4(vdst + gi * D * 2, &p.gv, 0, r[0], r[1], r[2], r[3], full_bar(slot), pol);
              }
            } else if (loj >= 0) {
              m.kind = 0;
              m.nrows = 0;
              meta[slot] = m;
              const uint32_t nb = static_cast<uint32_t>(nrj) * D * 2;
              mbar_arrive_expect_tx(full_bar(slot), 2 * nb);
              bulk_g2s(kdst + loj * D * 2, p.kpool + offj, nb, full_bar(slot), pol);
              bulk_g2s(vdst + loj * D * 2, p.vpool + offj, nb, full_bar(slot), pol);
            } else {
              m.kind = 1;
              m.nrows = nrj;
              meta[slot] = m;
              if (nrj) {
                mbar_arrive_expect_tx(full_bar(slot), 2u * nrj * D * 2);
                for (int r = 0; r < nrj; ++r) {
                  const int64_t o = (static_cast<int64_t>(dd.row0 + offj + r) * p.Hkv + sg.g) * D;
                  bulk_g2s(kdst + r * D * 2, p.k_new + o, D * 2, full_bar(slot), pol);
                  bulk_g2s(vdst + r * D * 2, p.v_new + o, D * 2, full_bar(slot), pol);
                }
              } else {
                mbar_arrive(full_bar(slot));
              }
            }
          }
          __syncwarp();
        }
      }
      x += sg.nst;
      ++segi;
    }
    }
    return;
  }

  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::CONSUMER_REGS));
  if (!ring_live) return;
  // ================================================================ consumers
  // Lane (kg, sub): key group kg = lane / LPK scores key kg of every warp step; sub = lane % LPK owns
  // dims {(c*LPK + sub)*8 .. +8} for c < CH.  After the transposing xor-reduction of the G partial dot
  // products, lane holds the full score of head hm = sub / (LPK/G) (its "own" head): exp / max / l are
  // per own head, then the G probabilities of the key are gathered back with G shuffles for P.V.
  constexpr int LG = (G == 1) ? 0 : (G == 2 ? 1 : (G == 4 ? 2 : 3));
  constexpr int SPH = LPK / G;  // lanes per head within a key group
  const int kg = lane / LPK, sub = lane % LPK;
  const int hm = sub / SPH;
  int local0 = 0, segi = 0;
  // fused-scores logits stay in L2 (evict_last) until the score pass reads and discards them
  const uint64_t lpol = policy_evict_last();
  // merge map: consumer thread ctid owns head mh, dims md0 .. md0 + DPT of a unit's output
  const int ctid = warp * 32 + lane;
  using MM = MergeMap<D, G, NW * 32>;
  const int mh = ctid / MM::TPH, md0 = (ctid % MM::TPH) * MM::DPT;
  const bool mlive = mh < G;
  int *ndef = flag + 2, *ndw = flag + 3;  // deferred merges pending / of which whole-unit records
  Deferred *dlist = reinterpret_cast<Deferred *>(flag + 8);
  if (ctid == 0) {
    *ndef = 0;
    *ndw = 0;
  }
  named_bar_sync(1 + ring, NW * 32);
  for (int k = 0;; ++k) {
  int cta = (k == 0) ? pr : p.ncta;
  if (p.dynamic) {
    mbar_wait(cfull_bar(k & 1), (k >> 1) & 1);
    cta = chunk_slot[k & 1];
    __syncwarp();
    if (lane == 0) mbar_arrive(cempty_bar(k & 1));
  }
  if (cta >= p.ncta) break;
  const int64_t beg = cta_start(cta, p), end = cta_start(cta + 1, p);
  // Final output of one unit (threads with mlive): its record(s) in the workspace -- the whole unit's record
  // `wrec` (index), or else the pieces of the rings covering it in range order (deterministic) -- then the
  // shared-prefix record(s), if any.
  auto merge_unit = [&](int64_t ua, int spu, int64_t row, int g, int64_t wrec, const float *pref, int nsplit) {
    float M = -CUDART_INF_F, L = 0.f, acc[MM::DPT];
#pragma unroll
    for (int i = 0; i < MM::DPT; ++i) acc[i] = 0.f;
    // the unit's records (its whole-unit record, or the pieces of the rings covering it in range order) and
    // its shared-prefix split records: up to 8 folded with all loads in flight
    const int c0 = wrec >= 0 ? 0 : cta_of(ua, p), c1 = wrec >= 0 ? 0 : cta_of(ua + spu - 1, p);
    const int npref = pref ? nsplit : 0;
    if (c1 - c0 + 1 + npref <= 8) {
      const float *rec[8];
      int n = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) rec[j] = nullptr;
      if (wrec >= 0) {
        rec[n++] = p.partials + wrec * C::PART + mh * (D + 2);
      } else {
        for (int c = c0; c <= c1; ++c)
          rec[n++] = p.partials + (static_cast<int64_t>(c) * C::KDEF + ((cta_start(c, p) >= ua) ? 0 : 1)) * C::PART +
                     mh * (D + 2);
      }
      for (int sp = 0; sp < npref; ++sp) rec[n++] = pref + static_cast<int64_t>(sp) * C::PART + mh * (D + 2);
      fold_ptrs<D, MM::DPT, 8>(rec, n, md0, M, L, acc);
    } else {
      if (wrec >= 0) {
        fold_records<D, MM::DPT, 1>(p.partials + wrec * C::PART + mh * (D + 2), 0, 1, md0, M, L, acc);
      } else {
        for (int c = c0; c <= c1; ++c) {
          const int wh = (cta_start(c, p) >= ua) ? 0 : 1;
          fold_records<D, MM::DPT, 1>(p.partials + (static_cast<int64_t>(c) * C::KDEF + wh) * C::PART + mh * (D + 2),
                                      0, 1, md0, M, L, acc);
        }
      }
      if (pref) fold_records<D, MM::DPT, MM::SG>(pref + mh * (D + 2), C::PART, nsplit, md0, M, L, acc);
    }
    const int64_t orow = row * p.Hq + g * G + mh;
    store_out<MM::DPT>(p.out + orow * D + md0, p.lse ? p.lse + orow : nullptr, md0, M, L, acc);
  };
  // The deferred merges (units with a shared prefix): one griddepcontrol.wait for the prefix grid, then each
  // unit's records + its prefix record.  Called by every consumer thread of the ring (uniform).
  auto flush_deferred = [&]() {
    const int n = *ndef;
    if (n == 0) return;
    if (ctid == 0) K1T(6, pr);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (ctid == 0) K1T(7, pr);
    __threadfence();  // this ring's piece records before its arrivals
    named_bar_sync(1 + ring, NW * 32);
    if (ctid < n) {  // one thread per entry: the arrivals in parallel
      Deferred &df = dlist[ctid];
      df.merge = 1;
      if (df.rslot < 0) {  // a piece: the last of the unit's rings to arrive merges it
        const int spu = p.descs[df.d].stages_per_unit;
        const int c0 = cta_of(df.ubeg, p), c1 = cta_of(df.ubeg + spu - 1, p);
        const int prev = atomicAdd(p.counters + df.unit, 1);
        df.merge = (prev == c1 - c0) ? 1 : 0;
        if (df.merge) p.counters[df.unit] = 0;  // self-cleaning for the next launch
      }
      __threadfence();
    }
    named_bar_sync(1 + ring, NW * 32);
    for (int j = 0; j < n; ++j) {
      const Deferred df = dlist[j];
      if (!df.merge || !mlive) continue;
      const Desc &du = p.descs[df.d];
      const int ui = df.unit - du.unit_base, g = ui / du.n_q, qi = ui - g * du.n_q;
      const float *pref = p.ppart + (static_cast<int64_t>(du.pref_base) + static_cast<int64_t>(ui) * du.pref_splits) * C::PART;
      merge_unit(df.ubeg, du.stages_per_unit, du.row0 + qi, g,
                 df.rslot >= 0 ? static_cast<int64_t>(cta) * C::KDEF + df.rslot : -1, pref, du.pref_splits);
    }
    named_bar_sync(1 + ring, NW * 32);
    if (ctid == 0) {
      *ndef = 0;
      *ndw = 0;
    }
    named_bar_sync(1 + ring, NW * 32);
  };
  int64_t x = beg;
  bool first_seg = true;
  while (x < end) {
    // ---- the segment (resolved by the producer) and its Q (scaled into the log2 domain) from the Q ring
    float2 q2[G][DPL / 2];
    Segment sg;
    Desc dd;
    {
      const int qs = segi % C::NQ;
      mbar_wait(qfull_bar(qs), (segi / C::NQ) & 1);
      const SegMeta sm = segmeta[qs];
      sg = Segment{sm.d, sm.g, sm.qi, sm.st0, sm.nst, sm.spu, sm.ubeg};
      dd = Desc{};
      dd.logit_off = sm.logit_off;
      dd.n_old_entries = sm.n_os;  // (skip stays 0: n_old_entries - skip is what the consumers use)
      dd.n_q = sm.n_q;
      dd.row0 = sm.row0;
      dd.unit_base = sm.unit_base;
      dd.pref_splits = sm.pref_splits;
      dd.pref_base = sm.pref_base;
      dd.stages_per_unit = sm.spu;
#pragma unroll
      for (int h = 0; h < G; ++h)
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const uint4 w = *reinterpret_cast<const uint4 *>(qring + (qs * G + h) * D + (c * LPK + sub) * 8);
          const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float2 f = bf2_to_f2(ws[j]);
            q2[h][c * 4 + j] = make_float2(f.x * p.scale_log2, f.y * p.scale_log2);
          }
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(qempty_bar(qs));
    }
    float2 o2[G][DPL / 2];
    float m_own = -CUDART_INF_F, l_own = 0.f;  // running max / sum of the lane's own head
#pragma unroll
    for (int h = 0; h < G; ++h)
#pragma unroll
      for (int j = 0; j < DPL / 2; ++j) o2[h][j] = make_float2(0.f, 0.f);

    for (int i = warp; i < sg.nst; i += NW) {
      const int local = local0 + i;
      const int slot = local % NSTAGES;
      mbar_wait(full_bar(slot), (local / NSTAGES) & 1);
      if (local == 0 && warp == 0 && lane == 0) K1T(2, pr);
      const StageMeta m = meta[slot];
      const __nv_bfloat16 *ks = reinterpret_cast<const __nv_bfloat16 *>(stage_data + slot * C::STAGE_BYTES);
      const __nv_bfloat16 *vs = ks + P * D;
      // fused scores: this stage's scaled logits (log2 domain) of every visible key, per head, for the score
      // pass (pred_attn_scores reads them instead of re-reading K)
      float *lg = nullptr;
      if (p.logits != nullptr && dd.logit_off >= 0)
        lg = p.logits + dd.logit_off +
             (static_cast<int64_t>(sg.g * dd.n_q + sg.qi) * dd.stages_per_unit + (sg.st0 + i)) * (P * G);
      // one softmax sub-block of SUB slots; FULL = every slot is a visible key (the common case: no
      // per-key predicates or divergent branches)
      auto sub_block = [&](auto full_tag, const uint32_t sbm, const int sb) {
        constexpr bool FULL = decltype(full_tag)::value;
        // A partial sub-block (lazy-eviction holes, a gathered stage, the last page) walks its retained keys
        // packed: warp step `it` scores the (it KG + kg)-th set bit of the mask, and steps past the retained
        // count are skipped (warp-uniform), so a half-empty page costs about half the consumer work.
        const int nk = FULL ? SUB : __popc(sbm);
        int kslot[NIT];  // the lane's key slot per warp step (packed retained keys in a partial sub-block)
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
          const int kidx = it * KG + kg;
          kslot[it] = FULL ? kidx : (kidx < nk ? kth_set_bit16(sbm, kidx) : 0);
        }
        float s[NIT];
        float smax = -CUDART_INF_F;
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
          s[it] = -CUDART_INF_F;
          if (!FULL && it * KG >= nk) continue;  // warp-uniform
          const int kidx = it * KG + kg;
          const bool valid = FULL || kidx < nk;
          const int slot_k = sb * SUB + kslot[it];
          float2 acc[G];
#pragma unroll
          for (int h = 0; h < G; ++h) acc[h] = make_float2(0.f, 0.f);
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const uint4 w = *reinterpret_cast<const uint4 *>(ks + slot_k * D + (c * LPK + sub) * 8);
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float2 kf = bf2_to_f2(ws[j]);
#pragma unroll
              for (int h = 0; h < G; ++h) fma2(acc[h], q2[h][c * 4 + j], kf);
            }
          }
          float v[G];
#pragma unroll
          for (int h = 0; h < G; ++h) v[h] = acc[h].x + acc[h].y;
          // transposing reduction: each level halves the values a lane carries
#pragma unroll
          for (int lvl = 0, cnt = G; lvl < LG; ++lvl, cnt >>= 1) {
            const int o = LPK >> (lvl + 1);
            const bool up = (sub & o) != 0;
#pragma unroll
            for (int t = 0; t < cnt / 2; ++t) {
              const float send = up ? v[t] : v[t + cnt / 2];
              const float keep = up ? v[t + cnt / 2] : v[t];
              v[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
          float sc = v[0];
#pragma unroll
          for (int o = SPH / 2; o > 0; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
          if (lg != nullptr && valid && (sub % SPH) == 0) st_hint(lg + slot_k * G + hm, sc, lpol);
          s[it] = FULL ? sc : (valid ? sc : -CUDART_INF_F);
          smax = fmaxf(smax, s[it]);
        }
        // sub-block max of the own head over the warp's key groups
#pragma unroll
        for (int o = LPK; o < 32; o <<= 1) smax = fmaxf(smax, __shfl_xor_sync(0xffffffffu, smax, o));
        // lazy rescale: only when some running max would be exceeded by more than 2^8
        if (__any_sync(0xffffffffu, smax > m_own + 8.f)) {
          const float mn = fmaxf(m_own, smax);
          const float a = (m_own == -CUDART_INF_F) ? 0.f : fast_exp2(m_own - mn);
          m_own = mn;
          l_own *= a;
#pragma unroll
          for (int h = 0; h < G; ++h) {
            const float ah = __shfl_sync(0xffffffffu, a, h * SPH);
            const float2 a2 = make_float2(ah, ah);
#pragma unroll
            for (int j = 0; j < DPL / 2; ++j) o2[h][j] = mul2(o2[h][j], a2);
          }
        }
        // P.V
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
          if (!FULL && it * KG >= nk) continue;  // warp-uniform
          const int kidx = it * KG + kg;
          const bool valid = FULL || kidx < nk;
          const int slot_k = sb * SUB + kslot[it];
          const float pown = FULL ? fast_exp2(s[it] - m_own) : (valid ? fast_exp2(s[it] - m_own) : 0.f);
          l_own += pown;
          float pw[G];
#pragma unroll
          for (int h = 0; h < G; ++h) pw[h] = __shfl_sync(0xffffffffu, pown, kg * LPK + h * SPH);
          if (valid) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
              const uint4 w = *reinterpret_cast<const uint4 *>(vs + slot_k * D + (c * LPK + sub) * 8);
              const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float2 vf = bf2_to_f2(ws[j]);
#pragma unroll
                for (int h = 0; h < G; ++h) fma2(o2[h][c * 4 + j], make_float2(pw[h], pw[h]), vf);
              }
            }
          }
        }
      };
#pragma unroll 1
      for (int sb = 0; sb < P / SUB; ++sb) {
        const uint32_t sbm = static_cast<uint32_t>(m.mask >> (sb * SUB)) & ((1u << SUB) - 1);
        if (sbm == (1u << SUB) - 1) sub_block(std::true_type{}, sbm, sb);
        else if (sbm != 0) sub_block(std::false_type{}, sbm, sb);  // warp-uniform
      }
      // fused append: the new-row stage of unit qi = 0 writes K_new / V_new into the reserved slots
      if (m.kind == 1 && sg.qi == 0) {
        const int st = sg.st0 + i;
        const int v0 = (st - (dd.n_old_entries - dd.skip)) * P;
        constexpr int CPR = D / 8;  // 16-byte chunks per row
        for (int idx = lane; idx < m.nrows * CPR; idx += 32) {
          const int r = idx / CPR, cc = idx % CPR;
          const int32_t ds = p.dst_slot[dd.row0 + v0 + r];
          const int page = ds / P, sl = ds % P;
          const int64_t off = ((static_cast<int64_t>(page) * p.Hkv + sg.g) * P + sl) * D + cc * 8;
          *reinterpret_cast<uint4 *>(p.kpool + off) = *reinterpret_cast<const uint4 *>(ks + r * D + cc * 8);
          *reinterpret_cast<uint4 *>(p.vpool + off) = *reinterpret_cast<const uint4 *>(vs + r * D + cc * 8);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_bar(slot));
    }

    if (warp == 0 && lane == 0) K1T(3, pr);
    // ---- combine the warps' (m, l, O) of this segment
#pragma unroll
    for (int o = LPK; o < 32; o <<= 1) {
      l_own += __shfl_xor_sync(0xffffffffu, l_own, o);
#pragma unroll
      for (int h = 0; h < G; ++h)
#pragma unroll
        for (int j = 0; j < DPL / 2; ++j) {
          o2[h][j].x += __shfl_xor_sync(0xffffffffu, o2[h][j].x, o);
          o2[h][j].y += __shfl_xor_sync(0xffffffffu, o2[h][j].y, o);
        }
    }
    float *cw = comb + warp * C::PART;
    if (kg == 0) {
#pragma unroll
      for (int h = 0; h < G; ++h)
#pragma unroll
        for (int c = 0; c < CH; ++c)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int dim = (c * LPK + sub) * 8 + 2 * j;
            *reinterpret_cast<float2 *>(cw + h * (D + 2) + dim) = o2[h][c * 4 + j];
          }
      if (sub % SPH == 0) {
        cw[hm * (D + 2) + D] = m_own;
        cw[hm * (D + 2) + D + 1] = l_own;
      }
    }
    named_bar_sync(1 + ring, NW * 32);

    const bool whole = (sg.st0 == 0) && (sg.nst == sg.spu);
    const int tid = ctid;
    const int unit = dd.unit_base + sg.g * dd.n_q + sg.qi;
    // A unit with a shared-prefix partial (written by the prefix kernel launched before this one; with a
    // programmatic dependent launch this kernel runs alongside it) is merged only after griddepcontrol.wait.
    // Waiting here, between two segments, would stall the ring's streaming until the prefix grid completed,
    // so the unit's record goes to the workspace and its merge is deferred to the end of the ring's range.
    // (The range's last segment has nothing streaming behind it: it waits and merges in place.)
    const bool defer = dd.pref_splits != 0 && x + sg.nst < end;
    const float *pref = dd.pref_splits ? p.ppart + (static_cast<int64_t>(dd.pref_base) +
                                                    static_cast<int64_t>(sg.g * dd.n_q + sg.qi) * dd.pref_splits) *
                                                       C::PART
                                       : nullptr;
    if (whole && !defer) {
      if (pref) {
        if (ctid == 0) K1T(6, pr);
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (ctid == 0) K1T(7, pr);
      }
      float M, L, acc[MM::DPT];
      if (mlive) {
        fold_comb<D, MM::DPT, NW, C::PART>(comb, mh, md0, M, L, acc);
        if (pref) fold_records<D, MM::DPT, MM::SG>(pref + mh * (D + 2), C::PART, dd.pref_splits, md0, M, L, acc);
        const int64_t orow = (dd.row0 + sg.qi) * p.Hq + sg.g * G + mh;
        store_out<MM::DPT>(p.out + orow * D + md0, p.lse ? p.lse + orow : nullptr, md0, M, L, acc);
      }
      named_bar_sync(1 + ring, NW * 32);
    } else {
      // record of this segment: a piece of a unit cut by a range boundary (slot 0: the range's first segment,
      // slot 1: its last) or a whole deferred unit (slots 2 ..)
      int rslot = first_seg ? 0 : 1;
      if (whole) {
        if (*ndw == C::KDEF - 2) flush_deferred();  // no free slot: merge what is pending now
        rslot = 2 + *ndw;
      }
      float *part = p.partials + (static_cast<int64_t>(cta) * C::KDEF + rslot) * C::PART;
      for (int e = tid; e < G * (D + 2); e += NW * 32) {
        const int h = e / (D + 2), dim = e % (D + 2);
        float M = -CUDART_INF_F;
#pragma unroll
        for (int w = 0; w < NW; ++w) M = fmaxf(M, comb[w * C::PART + h * (D + 2) + D]);
        float acc = 0.f;
        if (dim == D) {
          acc = M;
        } else {
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const float *cwp = comb + w * C::PART + h * (D + 2);
            const float f = (cwp[D] == -CUDART_INF_F) ? 0.f : fast_exp2(cwp[D] - M);
            acc += (dim == D + 1 ? cwp[D + 1] : cwp[dim]) * f;
          }
        }
        part[e] = acc;
      }
      if (defer) {  // record only: arrival, wait and merge at the end of the range (flush_deferred)
        named_bar_sync(1 + ring, NW * 32);
        if (tid == 0) {
          Deferred &df = dlist[*ndef];
          df.ubeg = sg.ubeg;
          df.d = sg.d;
          df.unit = unit;
          df.rslot = whole ? rslot : -1;
          *ndef += 1;
          if (whole) *ndw += 1;
        }
        named_bar_sync(1 + ring, NW * 32);
      } else {  // a piece at the end of the range: the last of the unit's rings to arrive merges it now
        __threadfence();
        named_bar_sync(1 + ring, NW * 32);
        if (tid == 0) {
          const int64_t ua = sg.ubeg, ub = sg.ubeg + sg.spu;
          const int c0 = cta_of(ua, p), c1 = cta_of(ub - 1, p);
          const int prev = atomicAdd(p.counters + unit, 1);
          *flag = (prev == c1 - c0) ? 1 : 0;
          if (prev == c1 - c0) p.counters[unit] = 0;  // self-cleaning for the next launch
        }
        named_bar_sync(1 + ring, NW * 32);
        if (*flag) {
          if (pref) {
            if (ctid == 0) K1T(6, pr);
            asm volatile("griddepcontrol.wait;" ::: "memory");
            if (ctid == 0) K1T(7, pr);
          }
          __threadfence();
          if (mlive) merge_unit(sg.ubeg, sg.spu, dd.row0 + sg.qi, sg.g, -1, pref, dd.pref_splits);
        }
        named_bar_sync(1 + ring, NW * 32);
      }
      if (*ndef == C::KDEF) flush_deferred();
    }
    x += sg.nst;
    local0 += sg.nst;
    ++segi;
    first_seg = false;
  }
  flush_deferred();
  }
  if (warp == 0 && lane == 0) K1T(4, pr);
}

template <class C>
static size_t decode_smem_bytes() {
  static_assert(sizeof(StageMeta) == 16, "StageMeta");
  return static_cast<size_t>(C::R) * C::RING_BYTES;
}

template <int D, int G, int P>
static cudaError_t launch_decode_t(const DecodeParams &p, cudaStream_t s, int *per_sm, bool pdl) {
  using C = DecodeCfg<D, G, P>;
  const size_t smem = decode_smem_bytes<C>();
  static int occ = -1;
  if (occ < 0) {
    cudaError_t e = cudaFuncSetAttribute(decode_attn_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int o = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, decode_attn_kernel<C>, C::THREADS, smem);
    if (e != cudaSuccess) return e;
    occ = (o > 0 ? o : 1) * C::R;  // virtual CTAs (rings) per SM
  }
  if (per_sm) {
    *per_sm = occ;
    return cudaSuccess;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((p.n_rings + C::R - 1) / C::R);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, decode_attn_kernel<C>, p);
}

template <int D, int G>
static cudaError_t launch_decode_p(const DecodeParams &p, int P, cudaStream_t s, int *per_sm, bool pdl) {
  switch (P) {
    case 16: return launch_decode_t<D, G, 16>(p, s, per_sm, pdl);
    case 32: return launch_decode_t<D, G, 32>(p, s, per_sm, pdl);
    case 64: return launch_decode_t<D, G, 64>(p, s, per_sm, pdl);
    default: return cudaErrorInvalidValue;
  }
}

template <int D>
static cudaError_t launch_decode_g(const DecodeParams &p, int G, int P, cudaStream_t s, int *per_sm, bool pdl) {
  switch (G) {
    case 1: return launch_decode_p<D, 1>(p, P, s, per_sm, pdl);
    case 2: return launch_decode_p<D, 2>(p, P, s, per_sm, pdl);
    case 4: return launch_decode_p<D, 4>(p, P, s, per_sm, pdl);
    case 8: return launch_decode_p<D, 8>(p, P, s, per_sm, pdl);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_decode(const DecodeParams &p, int D, int G, int P, cudaStream_t s, bool pdl) {
  if (D == 64) return launch_decode_g<64>(p, G, P, s, nullptr, pdl);
  if (D == 128) return launch_decode_g<128>(p, G, P, s, nullptr, pdl);
  return cudaErrorInvalidValue;
}

int decode_ctas_per_sm(int D, int G, int P) {
  int o = 1;
  DecodeParams dummy{};
  if (D == 64) launch_decode_g<64>(dummy, G, P, nullptr, &o, false);
  if (D == 128) launch_decode_g<128>(dummy, G, P, nullptr, &o, false);
  return o;
}

}  // namespace dev
}  // namespace kvfs
