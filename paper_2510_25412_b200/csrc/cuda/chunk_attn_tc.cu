// K2: multi-token (chunked prefill / speculative draft / keystroke re-append) attention on the 5th-gen
// tensor cores: tcgen05.mma with TMEM accumulators, operands staged by TMA (§4.1 P:215-217;
// rule R10 of SURVEY.md §8(c): each of the n_q new tokens attends to the file's retained tokens with
// logical index <= len - n_q + i).
//
// Unit = (descriptor, kv head g, M-tile m): 128 query rows R = 128 m + r, row R <-> (qi = R / G, h = R % G),
// so Q of the unit is a [rows][D] K-major tile loaded by one 4-D TMA box per 64-column half.
// KV tiles = 128 keys = 128 / P consecutive page entries of the file (K and V blocks of the (page, g) pairs
// loaded with 2-D TMA boxes of {64 cols, P rows}, 128-byte swizzle); the new tokens were scattered into the
// pool by scatter_rows_kernel before this launch, so every key is read from the pool.
//   S  = Q K^T      tcgen05.mma kind::f16, M = 128, N = 128, K = 16 x 8, A = Q (smem, K-major),
//                   B = K tile (smem, K-major), D = S in TMEM (double-buffered: columns 0 / 128)
//   softmax         4 warps, thread = row: tcgen05.ld of the S row, masks (retained slots, causality from
//                   per-column "new-token index" metadata written by the TMA warp), online softmax in the
//                   log2 domain with lazy rescale of O (tcgen05.ld/st, only when the row max grows > 8),
//                   P -> bf16 into smem in the 128B-swizzled K-major layout
//   O += P V        M = 128, N = 128 (D), K = 16 x 8, A = P (smem, K-major), B = V tile (smem, MN-major),
//                   D = O in TMEM (columns 256..383)
// Warp roles: 0 = TMA producer, 1 = MMA issuer (one elected lane), 2 = TMEM allocator, 3 = idle,
// 4..7 = softmax / epilogue warpgroup.
#include <cuda.h>
#include <cuda_bf16.h>
#include <math_constants.h>

#include "kernels.cuh"

namespace kvfs {
namespace dev {

namespace tc {

constexpr int BM = 128;   // rows per M-tile
constexpr int HD = 128;   // head dim (K2 is specialised for D = 128)
#ifndef KVFS_EXP_EMU
#define KVFS_EXP_EMU 2
#endif
constexpr int EXP_EMU = KVFS_EXP_EMU;  // of every 8 exp2 pairs in the softmax, how many run as a polynomial on the FMA pipe
constexpr uint32_t TMEM_COLS = 512;
#ifndef KVFS_K2_ISSUERS
#define KVFS_K2_ISSUERS 2
#endif
constexpr int K2_ISSUERS = KVFS_K2_ISSUERS;  // MMA-issuing warps (1: warp 1 issues both M-tiles)

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version (Blackwell)
  d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// One elected lane of a converged warp (elect.sync): the issue region of the single-thread tcgen05 ops.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\telect.sync rx|px, 0xffffffff;\n\tselp.b32 %0, 1, 0, px;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31])));
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1, uint32_t bar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// A operand from TMEM (P aliasing the S columns): D[tmem] (+)= A[tmem] * B[smem]
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}


// S_m = Q_m K^T for one 64-key tile: 8 MMAs (K = 16 each) in one asm block.  a / b are the SW128 K-major
// descriptors of the Q tile (128 rows, halves 16 KiB apart) and the K tile (64 rows, halves 8 KiB apart);
// step k advances the start address by (k / 4) * half + (k % 4) * 32 bytes (in 16-byte units below).
__device__ __forceinline__ void mma_s_group(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .b64 a1, a2, a3, a4, a5, a6, a7, b1, b2, b3, b4, b5, b6, b7;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 b1, %2, 2;\n\t"
      "add.s64 a2, %1, 4;\n\tadd.s64 b2, %2, 4;\n\t"
      "add.s64 a3, %1, 6;\n\tadd.s64 b3, %2, 6;\n\t"
      "add.s64 a4, %1, 1024;\n\tadd.s64 b4, %2, 512;\n\t"
      "add.s64 a5, %1, 1026;\n\tadd.s64 b5, %2, 514;\n\t"
      "add.s64 a6, %1, 1028;\n\tadd.s64 b6, %2, 516;\n\t"
      "add.s64 a7, %1, 1030;\n\tadd.s64 b7, %2, 518;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a4, b4, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a5, b5, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a6, b6, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a7, b7, %3, 1;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc));
}

// O_m (+)= P_m V for one 64-key tile: 4 MMAs with A = P from TMEM (8 columns = 16 keys per step) and
// B = the V tile (MN-major SW128, 16 key rows = 2048 B = 128 units per step).
__device__ __forceinline__ void mma_pv_group(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 b1, b2, b3;\n\t.reg .b32 t1, t2, t3;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.s64 b1, %2, 128;\n\tadd.s64 b2, %2, 256;\n\tadd.s64 b3, %2, 384;\n\t"
      "add.s32 t1, %1, 8;\n\tadd.s32 t2, %1, 16;\n\tadd.s32 t3, %1, 24;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [t1], b1, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [t2], b2, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [t3], b3, %3, 1;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

}  // namespace tc

// v3 layout: one CTA = (descriptor, kv head, pair of 128-row M-tiles) sharing every K/V tile; KV tiles of
// 64 keys.  TMEM: S0 [0,64) S1 [64,128), P_m[b] at [128 + 32 (2m + b), +32) (double-buffered by tile
// parity b), O0 [256,384) O1 [384,512).  P has its own columns, so S_m(t+1) is issued as soon as softmax m
// has read S_m(t) into registers and runs on the tensor pipe while the softmax of tile t computes its
// exponentials; with two P buffers the softmax never waits for P.V(t-1) (only for P.V(t-2), long done,
// and for P.V(t-1) when it must rescale O).  No S -> P -> PV -> S dependency chain remains.
namespace tc3 {
constexpr int THREADS = 384;  // warps 0-3: K producer, MMA, TMEM alloc, V producer; 4-7, 8-11: softmax M-tiles
constexpr int BN = 64;        // keys per KV tile
constexpr int KVS = 4;        // K stages and V stages (independent rings)
constexpr int JR = 8;         // column-metadata ring (>= KVS + 2, see the producer)
constexpr int QT_BYTES = tc::BM * tc::HD * 2;       // one [128][128] Q tile (two SW128 halves of 16 KiB)
constexpr int QH_BYTES = QT_BYTES / 2;
constexpr int KT_BYTES = BN * tc::HD * 2;           // one [64][128] K or V tile (two SW128 halves of 8 KiB)
constexpr int KH_BYTES = KT_BYTES / 2;
constexpr uint32_t S_COL = 0, P_COL = 128, O_COL = 256;
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + 2 * QT_BYTES;
constexpr int OFF_V = OFF_K + KVS * KT_BYTES;
constexpr int OFF_JCOL = OFF_V + KVS * KT_BYTES;     // JR x BN int32 + JR tile flags
constexpr int OFF_BAR = OFF_JCOL + JR * BN * 4 + JR * 4;
constexpr int N_BARS = 1 + 4 * KVS + 12 + JR;
constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
constexpr int SMEM = OFF_TMEM + 16 + 1024;
static_assert(SMEM <= 232448, "shared memory");

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc(int n, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         ((static_cast<uint32_t>(n) >> 3) << 17) | ((static_cast<uint32_t>(tc::BM) >> 4) << 24);
}
}  // namespace tc3

// Development tracing (build with -DKVFS_K2_TRACE, read with tools/k2_trace.py): clock64() stamps of the
// pipeline events of two CTAs (block 0 and block 296, first and third wave) per KV tile.
#ifdef KVFS_K2_TRACE
__device__ unsigned long long g_k2_trace[2][32][512];
#define K2T(ev, t)                                                                  \
  do {                                                                              \
    if (trace_cta >= 0 && (t) < 512) g_k2_trace[trace_cta][ev][t] = clock64();      \
  } while (0)
#else
#define K2T(ev, t) \
  do {             \
  } while (0)
#endif

template <int G>
__global__ void __launch_bounds__(tc3::THREADS, 1)
    chunk_attn_tc_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                         const __grid_constant__ CUtensorMap qmap, const ChunkParams p) {
  using namespace tc;
  using namespace tc3;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
  auto bar = [&](int i) { return smem_u32(bars + i); };
  // barriers: Q; K full/empty, V full/empty rings; per M-tile S full (MMA commit), S consumed (softmax read
  // S into registers), P full (softmax wrote P); per (M-tile, P buffer) P consumed (PV done: that P buffer
  // free, O stable; index 2m + b); column metadata
  // P full is per (M-tile, tile parity) too: it counts one arrival per softmax warp, and a fast warp may
  // reach tile t+1 (S(t+1) is issued once every warp has READ S(t)) before a slow warp has written P(t);
  // with one barrier its early arrival would complete the phase of tile t.  Two tiles ahead is impossible
  // (S(t+2) waits for every warp to read S(t+1), i.e. to finish tile t).
  constexpr int B_Q = 0, B_KF = 1, B_KE = 1 + KVS, B_VF = 1 + 2 * KVS, B_VE = 1 + 3 * KVS, B_SF = 1 + 4 * KVS,
                B_SE = B_SF + 2, B_PF = B_SE + 2, B_PE = B_PF + 4, B_JF = B_PE + 4;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + OFF_TMEM);
  int32_t *jcol_all = reinterpret_cast<int32_t *>(smem + OFF_JCOL);
  int32_t *jflag = jcol_all + JR * BN;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef KVFS_K2_TRACE
  const int trace_cta = blockIdx.x == 0 ? 0 : (blockIdx.x == 296 ? 1 : -1);
#endif
  const ChunkUnit u = p.units[blockIdx.x];
  const ChunkDesc cd = p.descs[u.desc];
  const int epb = BN / p.P;  // page entries per KV tile
  const int n_tiles = (cd.n_entries + epb - 1) / epb;
  const int rows_total = cd.n_q * G;
  const int m0 = 2 * u.m;                                     // first M-tile of this CTA
  const int n_mt = min(2, (rows_total + BM - 1) / BM - m0);  // 1 or 2 M-tiles

  if (threadIdx.x == 0) {
    mbar_init(bar(B_Q), 1);
    for (int s = 0; s < KVS; ++s) {
      mbar_init(bar(B_KF + s), 1);
      mbar_init(bar(B_KE + s), K2_ISSUERS == 2 ? n_mt : 1);  // one commit per MMA issuer
      mbar_init(bar(B_VF + s), 1);
      mbar_init(bar(B_VE + s), K2_ISSUERS == 2 ? n_mt : 1);
    }
    for (int m = 0; m < 2; ++m) {
      mbar_init(bar(B_SF + m), 1);
      mbar_init(bar(B_SE + m), 4);
      mbar_init(bar(B_PF + 2 * m), 4);
      mbar_init(bar(B_PF + 2 * m + 1), 4);
      mbar_init(bar(B_PE + 2 * m), 1);
      mbar_init(bar(B_PE + 2 * m + 1), 1);
    }
    for (int j = 0; j < JR; ++j) mbar_init(bar(B_JF + j), 1);
    fence_mbar_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // The CTA owns all 512 TMEM columns (one CTA per SM), so the allocation starts at lane 0, column 0.  The
  // constant keeps every tcgen05 operand a compile-time uniform value (no R2UR waterfall per MMA).
  if (*tmem_slot != 0u) __trap();
  constexpr uint32_t tmem = 0;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (warp == 0) {
      // ============================================================ K producer (+ Q, + column metadata)
      const uint64_t pol = policy_evict_first();
      if (lane == 0) {
        mbar_arrive_expect_tx(bar(B_Q), n_mt * QT_BYTES);
        for (int m = 0; m < n_mt; ++m) {
          const int qrow = cd.row0 + ((m0 + m) * BM) / G;
          tma_load_4d(sbase + OFF_Q + m * QT_BYTES, &qmap, 0, 0, u.g, qrow, bar(B_Q));
          tma_load_4d(sbase + OFF_Q + m * QT_BYTES + QH_BYTES, &qmap, 64, 0, u.g, qrow, bar(B_Q));
        }
      }
      // Page-table entries are fetched 32 at a time with one coalesced load (lane i <-> entry 32 blk + i)
      // and handed to the tile's columns by shuffles: no dependent global load on the per-tile path.
      // jbase(e) = j of entry e's first retained token = first_new_lstart - n_old + sum of the popcounts
      // of the entries fne .. e-1 (entries at or after the first new entry hold new tokens).
      // Ring safety of jcol: the producer writes tile t after K(t - KVS) was released, i.e. after both
      // softmax groups read S(t - KVS - 1); they read jcol(t') right after S(t'), so slot t % JR (JR >= KVS + 2)
      // last held tile t - JR <= t - KVS - 2, already consumed.
      uint64_t emask = 0;
      int32_t erow = p.pool_rows, jbase = 0, carry = cd.first_new_lstart - cd.n_old;
      int cached = -1;
      for (int t = 0; t < n_tiles; ++t) {
        const int s = t % KVS;
        if (t >= KVS) mbar_wait_sleep(bar(B_KE + s), ((t / KVS) & 1) ^ 1);
        if (lane == 0) K2T(0, t);
        const int e0 = t * epb, blk = e0 >> 5;
        if (blk != cached) {
          const int e = blk * 32 + lane;
          emask = 0;
          erow = p.pool_rows;
          if (e < cd.n_entries) {
            const Entry en = p.slab[cd.slab_off + e];
            emask = en.mask;
            erow = (static_cast<int>(en.page) * p.Hkv + u.g) * p.P;
          }
          const int cnt = (e >= cd.first_new_entry) ? __popcll(emask) : 0;
          int incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          jbase = carry + incl - cnt;
          carry += __shfl_sync(0xffffffffu, incl, 31);
          cached = blk;
        }
        // column metadata of tile t: j = logical index - n_old (visible iff j <= qi), INT_MAX = no key;
        // jflag = 1 when every column is an old retained token (visible to every row: no masking)
        int32_t *jcol = jcol_all + (t % JR) * BN;
        bool vis_all = true;
#pragma unroll
        for (int k = 0; k < BN / 32; ++k) {
          const int c = k * 32 + lane;
          const int i = c / p.P, slot = c % p.P;
          const int src = (e0 & 31) + i;
          const uint64_t m = __shfl_sync(0xffffffffu, emask, src);
          const int32_t jb = __shfl_sync(0xffffffffu, jbase, src);
          const int e = e0 + i;
          int32_t j = 0x7fffffff;
          if (e < cd.n_entries && ((m >> slot) & 1ull))
            j = (e < cd.first_new_entry) ? -1 : jb + __popcll(m & ((1ull << slot) - 1ull));
          jcol[c] = j;
          vis_all &= (j < 0);
        }
        vis_all = __all_sync(0xffffffffu, vis_all);
        const int32_t row = __shfl_sync(0xffffffffu, erow, (e0 & 31) + (lane % epb));
        if (lane == 0) {
          jflag[t % JR] = vis_all ? 1 : 0;
          mbar_arrive(bar(B_JF + t % JR));
          mbar_arrive_expect_tx(bar(B_KF + s), KT_BYTES);
        }
        __syncwarp();
        if (lane < epb) {  // entry e0 + lane (rows past the table: out-of-bounds box, zero-filled)
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sbase + OFF_K + s * KT_BYTES + h * KH_BYTES + lane * p.P * 128, &kmap, h * 64, row,
                        bar(B_KF + s), pol);
        }
        if (lane == 0) K2T(1, t);
        __syncwarp();
      }
    } else if (warp == 3) {
      // ============================================================ V producer
      const uint64_t pol = policy_evict_first();
      int32_t erow = p.pool_rows;
      int cached = -1;
      for (int t = 0; t < n_tiles; ++t) {
        const int s = t % KVS;
        if (t >= KVS) mbar_wait_sleep(bar(B_VE + s), ((t / KVS) & 1) ^ 1);
        if (lane == 0) K2T(2, t);
        const int e0 = t * epb, blk = e0 >> 5;
        if (blk != cached) {
          const int e = blk * 32 + lane;
          erow = e < cd.n_entries ? (static_cast<int>(p.slab[cd.slab_off + e].page) * p.Hkv + u.g) * p.P : p.pool_rows;
          cached = blk;
        }
        const int32_t row = __shfl_sync(0xffffffffu, erow, (e0 & 31) + (lane % epb));
        if (lane == 0) mbar_arrive_expect_tx(bar(B_VF + s), KT_BYTES);
        __syncwarp();
        if (lane < epb) {
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sbase + OFF_V + s * KT_BYTES + h * KH_BYTES + lane * p.P * 128, &vmap, h * 64, row,
                        bar(B_VF + s), pol);
        }
        if (lane == 0) K2T(3, t);
        __syncwarp();
      }
    } else if (warp == 1 || (warp == 2 && K2_ISSUERS == 2)) {
      // ============================================================ MMA issuers
      // K2_ISSUERS == 2: warp 1 + m issues M-tile m; == 1: warp 1 issues both.
      // Per tile t: S_m(t+1) as soon as softmax m read S_m(t) (and K(t+1) landed), then PV_m(t) as soon as
      // P_m(t) is written (and V(t) landed).  The tensor pipe runs in order per issuer, so softmax m of
      // tile t+1 finds S_m(t+1) ready.  K / V stages are released by a commit of each issuer.
      constexpr uint32_t ID_S = idesc(BN, false), ID_O = idesc(HD, true);
      const int m_lo = K2_ISSUERS == 2 ? warp - 1 : 0;
      const int m_hi = K2_ISSUERS == 2 ? min(warp, n_mt) : n_mt;
      if (m_lo < m_hi) {
        const uint64_t qd = umma_desc(sbase + OFF_Q, 16, 1024);
        const uint64_t kd0 = umma_desc(sbase + OFF_K, 16, 1024);
        const uint64_t vd0 = umma_desc(sbase + OFF_V, KH_BYTES, 1024);
        constexpr uint64_t STAGE_UNITS = KT_BYTES >> 4, QT_UNITS = QT_BYTES >> 4;
        mbar_wait(bar(B_Q), 0);
        mbar_wait(bar(B_KF + 0), 0);
        tc_fence_after();
        if (elect_one()) {
          for (int m = m_lo; m < m_hi; ++m) {
            mma_s_group(tmem + S_COL + m * BN, qd + m * QT_UNITS, kd0, ID_S);
            mma_commit(bar(B_SF + m));
          }
          mma_commit(bar(B_KE + 0));
        }
        __syncwarp();
        for (int t = 0; t < n_tiles; ++t) {
#ifdef KVFS_K2_LOCKSTEP
          if (K2_ISSUERS == 2 && n_mt == 2) named_bar_sync(14, 64);
#endif
          if (t + 1 < n_tiles) {
            const int s1 = (t + 1) % KVS;
            mbar_wait(bar(B_KF + s1), ((t + 1) / KVS) & 1);
            for (int m = m_lo; m < m_hi; ++m) {
              mbar_wait(bar(B_SE + m), t & 1);  // softmax m holds S_m(t) in registers
              if (m == 0 && lane == 0) K2T(5, t);
              tc_fence_after();
              if (elect_one()) {
                mma_s_group(tmem + S_COL + m * BN, qd + m * QT_UNITS, kd0 + s1 * STAGE_UNITS, ID_S);
                mma_commit(bar(B_SF + m));
              }
              __syncwarp();
              if (m == 0 && lane == 0) K2T(6, t);
            }
            if (elect_one()) mma_commit(bar(B_KE + s1));
            __syncwarp();
          }
          const int s = t % KVS;
          mbar_wait(bar(B_VF + s), (t / KVS) & 1);
          for (int m = m_lo; m < m_hi; ++m) {
            mbar_wait(bar(B_PF + 2 * m + (t & 1)), (t >> 1) & 1);  // softmax m wrote P_m(t) (and corrected O)
            if (m == 0 && lane == 0) K2T(10, t);
            tc_fence_after();
            if (elect_one()) {
              mma_pv_group(tmem + O_COL + m * HD, tmem + P_COL + (2 * m + (t & 1)) * (BN / 2),
                           vd0 + s * STAGE_UNITS, ID_O, t > 0 ? 1u : 0u);
              mma_commit(bar(B_PE + 2 * m + (t & 1)));
            }
            __syncwarp();
            if (m == 0 && lane == 0) K2T(11, t);
          }
          if (elect_one()) mma_commit(bar(B_VE + s));
          __syncwarp();
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    // ============================================================ softmax warpgroups (thread = row)
    const int m = (warp - 4) >> 2;          // M-tile of this warpgroup
    const int wq = (warp - 4) & 3;          // TMEM lane quarter
    if (m < n_mt) {
      const int r = wq * 32 + lane;
      const int R = (m0 + m) * BM + r;
      const int qi = R / G, h = R % G;
      const bool live = qi < cd.n_q;
      const uint32_t lane_addr = static_cast<uint32_t>(wq * 32) << 16;
      const uint32_t s_col = tmem + lane_addr + S_COL + m * BN;
      const uint32_t p_col = tmem + lane_addr + P_COL + 2 * m * (BN / 2);  // + (t & 1) * (BN / 2)
      const uint32_t o_col = tmem + lane_addr + O_COL + m * HD;
      float m_run = -CUDART_INF_F, l_run = 0.f;
      for (int t = 0; t < n_tiles; ++t) {
        mbar_wait(bar(B_SF + m), t & 1);
        if (wq == 0 && lane == 0) K2T(14 + 6 * m, t);
        tc_fence_after();
        float x[BN];
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          float v[32];
          tmem_ld32(s_col + c * 32, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) x[c * 32 + i] = v[i];
        }
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(B_SE + m));  // S_m may now be overwritten by S_m(t+1)
        if (wq == 0 && lane == 0) K2T(15 + 6 * m, t);
        mbar_wait(bar(B_JF + t % JR), (t / JR) & 1);
        const int32_t *jcol = jcol_all + (t % JR) * BN;
        // raw-score max (scale > 0 commutes with max); masked columns -> -inf.  Four independent chains.
        float mx4[4] = {-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F};
        if (jflag[t % JR]) {
#pragma unroll
          for (int c = 0; c < BN; ++c) mx4[c & 3] = fmaxf(mx4[c & 3], x[c]);
        } else {
#pragma unroll
          for (int c = 0; c < BN; ++c) {
            if (jcol[c] > qi) x[c] = -CUDART_INF_F;
            mx4[c & 3] = fmaxf(mx4[c & 3], x[c]);
          }
        }
        float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
        mx = mx == -CUDART_INF_F ? mx : mx * p.scale_log2;
        if (wq == 0 && lane == 0) K2T(16 + 6 * m, t);
        // P buffer t & 1 was last read by P.V(t-2): phase (t-2)/2 of its barrier
        if (t >= 2) mbar_wait(bar(B_PE + 2 * m + (t & 1)), ((t - 2) >> 1) & 1);
        tc_fence_after();
        const bool need = mx > m_run + 8.f;
        if (__any_sync(0xffffffffu, need)) {
          if (t > 0) {  // O must be stable: P.V(t-1) done (phase (t-1)/2 of buffer (t-1) & 1)
            mbar_wait(bar(B_PE + 2 * m + ((t - 1) & 1)), ((t - 1) >> 1) & 1);
            tc_fence_after();
          }
          const float mn = need ? mx : m_run;
          const float a = (need && m_run != -CUDART_INF_F) ? fast_exp2(m_run - mn) : (need ? 0.f : 1.f);
          if (t > 0) {
#pragma unroll
            for (int c = 0; c < HD / 32; ++c) {
              float v[32];
              tmem_ld32(o_col + c * 32, v);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] *= a;
              tmem_st32(o_col + c * 32, v);
            }
          }
          l_run *= a;
          m_run = mn;
        }
        if (wq == 0 && lane == 0) K2T(17 + 6 * m, t);
        const float mref = m_run == -CUDART_INF_F ? 0.f : m_run;
        // P = exp2(x * scale_log2 - m) -> packed bf16 pairs into P_m (the A operand of P.V)
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        const float2 nm2 = make_float2(-mref, -mref);
        float2 ls2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        float w[BN / 2];
#pragma unroll
        for (int i = 0; i < BN / 2; ++i) {
          float2 a = nm2;
          fma2(a, make_float2(x[2 * i], x[2 * i + 1]), sc2);
          // EXP_EMU of every 8 pairs go to the FMA pipe (polynomial), the rest to MUFU
          const float2 pp = ((i & 7) >= 8 - EXP_EMU) ? exp2_poly2(a) : make_float2(fast_exp2(a.x), fast_exp2(a.y));
          ls2[i & 1] = add2(ls2[i & 1], pp);
          __nv_bfloat162 pr = __floats2bfloat162_rn(pp.x, pp.y);
          w[i] = __uint_as_float(*reinterpret_cast<uint32_t *>(&pr));
        }
        if (wq == 0 && lane == 0) K2T(18 + 6 * m, t);
        tmem_st32(p_col + (t & 1) * (BN / 2), w);
        const float2 lsum = add2(ls2[0], ls2[1]);
        l_run += lsum.x + lsum.y;
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(B_PF + 2 * m + (t & 1)));
        if (wq == 0 && lane == 0) K2T(19 + 6 * m, t);
      }
      // epilogue: O / l -> bf16 out, lse
      mbar_wait(bar(B_PE + 2 * m + ((n_tiles - 1) & 1)), ((n_tiles - 1) >> 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l_run;
      const int64_t orow = (static_cast<int64_t>(cd.row0 + qi) * p.Hq + u.g * G + h) * HD;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        float v[32];
        tmem_ld32(o_col + c * 32, v);
        tmem_wait_ld();
        if (live) {
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint32_t w4[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              __nv_bfloat162 pr = __floats2bfloat162_rn(v[i + 2 * j] * inv, v[i + 2 * j + 1] * inv);
              w4[j] = *reinterpret_cast<uint32_t *>(&pr);
            }
            *reinterpret_cast<uint4 *>(p.out + orow + c * 32 + i) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
          }
        }
      }
      if (live && p.lse)
        p.lse[static_cast<int64_t>(cd.row0 + qi) * p.Hq + u.g * G + h] =
            (m_run + __log2f(l_run)) * 0.69314718055994531f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// Scatter the new rows of the chunk descriptors into their reserved pool slots (K and V of one layer).
__global__ void scatter_rows_kernel(const int32_t *dst, int T, const __nv_bfloat16 *k, const __nv_bfloat16 *v,
                                    __nv_bfloat16 *kp, __nv_bfloat16 *vp, int Hkv, int D, int P) {
  const int cpr = D / 8;
  const int64_t total = static_cast<int64_t>(T) * Hkv * cpr;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(idx % cpr);
    const int64_t t = idx / cpr;
    const int g = static_cast<int>(t % Hkv);
    const int r = static_cast<int>(t / Hkv);
    const int32_t ds = dst[r];
    if (ds < 0) continue;
    const int64_t so = (static_cast<int64_t>(r) * Hkv + g) * D + c * 8;
    const int64_t po = ((static_cast<int64_t>(ds / P) * Hkv + g) * P + ds % P) * D + c * 8;
    *reinterpret_cast<uint4 *>(kp + po) = *reinterpret_cast<const uint4 *>(k + so);
    *reinterpret_cast<uint4 *>(vp + po) = *reinterpret_cast<const uint4 *>(v + so);
  }
}

cudaError_t launch_scatter_rows(const int32_t *dst, int T, const __nv_bfloat16 *k, const __nv_bfloat16 *v,
                                __nv_bfloat16 *kp, __nv_bfloat16 *vp, int Hkv, int D, int P, int sms,
                                cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(T) * Hkv * (D / 8);
  const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, static_cast<int64_t>(sms) * 16));
  if (grid <= 0) return cudaSuccess;
  scatter_rows_kernel<<<grid, 256, 0, s>>>(dst, T, k, v, kp, vp, Hkv, D, P);
  return cudaGetLastError();
}

int chunk_smem_bytes() { return tc3::SMEM; }

#ifdef KVFS_K2_TRACE
extern "C" int kvfs_debug_k2_trace(void *host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, g_k2_trace, bytes < sizeof(g_k2_trace) ? bytes : sizeof(g_k2_trace)) ==
                 cudaSuccess ? 0 : -1;
}
#endif

template <int G>
static cudaError_t launch_chunk_g(const CUtensorMap &km, const CUtensorMap &vm, const CUtensorMap &qm,
                                  const ChunkParams &p, int n_units, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(chunk_attn_tc_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         tc3::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  chunk_attn_tc_kernel<G><<<n_units, tc3::THREADS, tc3::SMEM, s>>>(km, vm, qm, p);
  return cudaGetLastError();
}

cudaError_t launch_chunk(const CUtensorMap &km, const CUtensorMap &vm, const CUtensorMap &qm, const ChunkParams &p,
                         int n_units, int G, cudaStream_t s) {
  switch (G) {
    case 1: return launch_chunk_g<1>(km, vm, qm, p, n_units, s);
    case 2: return launch_chunk_g<2>(km, vm, qm, p, n_units, s);
    case 4: return launch_chunk_g<4>(km, vm, qm, p, n_units, s);
    case 8: return launch_chunk_g<8>(km, vm, qm, p, n_units, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace dev
}  // namespace kvfs
