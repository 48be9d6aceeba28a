// K2: multi-token (chunked prefill / speculative draft / keystroke re-append) attention on the 5th-gen
// tensor cores: tcgen05.mma with TMEM accumulators, operands staged by TMA (§4.1 P:215-217;
// rule R10 of SURVEY.md §8(c): each of the n_q new tokens attends to the file's retained tokens with
// logical index <= len - n_q + i).
//
// CTA = (descriptor, kv head g, pair of 128-row M-tiles) sharing every K/V tile.  Rows R = 128 m + r,
// row R <-> (qi = R / G, h = R % G), so Q of an M-tile is a [rows][D] K-major tile loaded by one 4-D TMA box
// per 64-column half.  KV tiles = 128 keys = 128 / P consecutive page entries of the file (K and V blocks of
// the (page, g) pairs loaded with 2-D TMA boxes of {64 cols, P rows}, 128-byte swizzle); the new tokens were
// scattered into the pool by scatter_rows_kernel before this launch, so every key is read from the pool.
//   S  = Q K^T      tcgen05.mma kind::f16, M = 128, N = 128, K = 16 x 8, A = Q (smem, K-major),
//                   B = K tile (smem, K-major), D = S in TMEM (S0 / S1 at columns 0 / 128, one per M-tile)
//   softmax         one warpgroup per M-tile, thread = row: tcgen05.ld of the S row, masks (retained slots,
//                   causality from per-column "new-token index" metadata written by the K producer), online
//                   softmax in the log2 domain with lazy rescale of O (tcgen05.ld/st, only when the row max
//                   grows by > 8), P -> bf16 pairs written back into TMEM over the first 64 columns of S
//   O += P V        M = 128, N = 128 (D), K = 16 x 8, A = P (TMEM, the .kind::f16 [a_tmem] form), B = V tile
//                   (smem, MN-major), D = O in TMEM (O0 / O1 at columns 256 / 384), in two 64-key halves
// Warp roles: 0 = K producer (+ Q, column metadata), 1 = MMA issuer (elect.sync lane), 2 = TMEM allocator,
// 3 = V producer, 4..7 / 8..11 = softmax + epilogue of M-tile 0 / 1.
// Measured per-128-key-tile timeline (tools/k2_trace.py, cfg4): softmax ~1.65k clk (MUFU floor ~0.77k with
// EXP_EMU of 8 exp2 pairs on the FMA pipe), MMA-warp reaction ~0.26k, P.V(second half) + S(t+1) ~0.77k on
// the tensor pipe, wake-up ~0.3k: period ~3.1k clk, tensor pipe ~64% busy.  Variants measured slower and
// removed (git history): P in separate TMEM columns with 64-key tiles,
// softmax groups issuing their own MMAs, one MMA warp per M-tile, split-column softmax, suspend-hint waits.
#include <cuda.h>
#include <cuda_bf16.h>
#include <math_constants.h>

#include "kernels.cuh"

namespace kvfs {
namespace dev {

namespace tc {

constexpr int BM = 128;   // rows per M-tile
constexpr int BN = 128;   // keys per KV tile
constexpr int HD = 128;   // head dim (K2 is specialised for D = 128)
constexpr int HALF_BYTES = BM * 64 * 2;  // one 64-column half of a [128][64] bf16 SW128 tile = 16 KiB
constexpr int TILE_BYTES = 2 * HALF_BYTES;  // [128][128] bf16 = 32 KiB
#ifndef KVFS_EXP_EMU
#define KVFS_EXP_EMU 2
#endif
constexpr int EXP_EMU = KVFS_EXP_EMU;  // of every 8 exp2 pairs in the softmax, how many run as a polynomial on the FMA pipe
constexpr uint32_t TMEM_COLS = 512;
#define K2_WAIT(b, ph) mbar_wait(b, ph)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version (Blackwell)
  d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, M = 128, N = 128
__host__ __device__ constexpr uint32_t idesc_bf16(bool b_mn_major) {
  return (1u << 4)                                  // c_format = F32
         | (1u << 7)                                // a_format = BF16
         | (1u << 10)                               // b_format = BF16
         | (0u << 15)                               // a K-major
         | ((b_mn_major ? 1u : 0u) << 16)           // b major
         | ((static_cast<uint32_t>(BN) >> 3) << 17)  // N >> 3
         | ((static_cast<uint32_t>(BM) >> 4) << 24); // M >> 4
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

}  // namespace tc

// v2 layout: one CTA = (descriptor, kv head, pair of 128-row M-tiles) sharing every K/V tile.
// TMEM: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512); P_m aliases the first 64 columns of S_m.
namespace tc2 {
constexpr int THREADS = 384;  // warps 0-3: K producer, MMA, TMEM alloc, V producer; 4-7, 8-11: softmax M-tiles
// K and V stages (independent rings).  3 V stages (with JR = 3 to stay inside 227 KB) measured the same as 2:
// the MMA warp's wait for V(t) (tools/k2_trace.py) is where it arrives after issuing the previous M-tile's
// P.V and S MMAs, whose issue the tensor pipe throttles, not a late TMA.
constexpr int KS2 = 2;
constexpr int VS2 = 2;
constexpr int JR = 4;         // column-metadata ring
constexpr uint32_t O_COL2 = 256;
constexpr int OFF_Q2 = 0;                                   // 2 Q tiles
constexpr int OFF_K2 = OFF_Q2 + 2 * tc::TILE_BYTES;         // KS2 K tiles
constexpr int OFF_V2 = OFF_K2 + KS2 * tc::TILE_BYTES;       // VS2 V tiles
constexpr int OFF_JCOL2 = OFF_V2 + VS2 * tc::TILE_BYTES;    // JR x BN int32
constexpr int OFF_BAR2 = OFF_JCOL2 + JR * tc::BN * 4 + 64;  // + JR tile flags
constexpr int N_BARS2 = 1 + 2 * KS2 + 2 * VS2 + 8 + JR + 1;
constexpr int OFF_TMEM2 = OFF_BAR2 + N_BARS2 * 8;
constexpr int SMEM2 = OFF_TMEM2 + 16 + 1024;
static_assert(SMEM2 <= 232448, "227 KB of dynamic shared memory per CTA");
static_assert(256 * part_floats(1, 128) * 4 <= OFF_JCOL2, "prefix-mode record staging (256 rows, G = 1 worst case) overlays Q, K and V");
}  // namespace tc2

#ifdef KVFS_K2_TRACE
__device__ unsigned long long g_k2_trace[2][32][512];
#define K2T(ev, t)                                                                  \
  do {                                                                              \
    if (trace_cta >= 0 && (t) < 512) g_k2_trace[trace_cta][ev][t] = clock64();      \
  } while (0)
// per-CTA globaltimer stamps (prefix-mode phases; tools/cascade_trace.py), slots 20..23 of trace row 1
#define K2G(slot)                                                                   \
  do {                                                                              \
    if (blockIdx.x < 512) {                                                         \
      unsigned long long gt_;                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));                       \
      g_k2_trace[1][slot][blockIdx.x] = gt_;                                        \
    }                                                                               \
  } while (0)
#else
#define K2T(ev, t) \
  do {             \
  } while (0)
#define K2G(slot) \
  do {            \
  } while (0)
#endif

// PREFIX = shared-prefix (cascade) mode: a unit is (fork family + key split, kv head, M-tile pair); the
// rows are the family's query tokens x the G heads of the kv head (gathered from Q by the softmax warps
// into the 128B-swizzled layout), every key is an old retained token (no causal part), and the output is
// the unnormalised partial (O, m, l) per (row, head) that the decode kernel merges.
// MULTI (prefix mode with ChunkParams::cta_units): a CTA runs a list of units in turn.  A separate
// instantiation, so the one-unit kernels keep their per-unit values constant (no loop-carried state: the
// loop version measured ~6% slower per tile).
template <int G, bool PREFIX, bool MULTI = false>
__global__ void __launch_bounds__(tc2::THREADS, 1)
    chunk_attn_tc_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                         const __grid_constant__ CUtensorMap qmap, const ChunkParams p) {
  using namespace tc;
  using namespace tc2;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned (128B-swizzle atoms) by pointer arithmetic on the shared array itself, so the compiler
  // keeps the shared address space (LDS / STS, not generic LD / ST)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + OFF_BAR2);
  auto bar = [&](int i) { return smem_u32(bars + i); };
  // barrier indices
  constexpr int B_Q = 0, B_KF = 1, B_KE = 1 + KS2, B_VF = 1 + 2 * KS2, B_VE = 1 + 2 * KS2 + VS2,
                B_SF = 1 + 2 * KS2 + 2 * VS2,
                B_PF = B_SF + 2, B_OF = B_PF + 4, B_JF = B_OF + 2,  // B_PF + 2m + half
                B_X = B_JF + JR;  // prefix mode: the split-exchange loads
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + OFF_TMEM2);
  int32_t *jcol_all = reinterpret_cast<int32_t *>(smem + OFF_JCOL2);
  int32_t *jflag = jcol_all + JR * BN;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef KVFS_K2_TRACE
  const int trace_cta = blockIdx.x == 0 ? 0 : (blockIdx.x == 296 ? 1 : -1);
#endif
  // Prefix mode is a programmatic dependent launch after the step prologue, which copies this step's packet
  // (units, prefix descriptors and rows) into the upload area and applies the table deltas: wait for it
  // before the first read of either.  (Reading the units earlier returned the PREVIOUS step's records
  // whenever the packet layout changed between steps, e.g. with another split count.)
  if constexpr (PREFIX) asm volatile("griddepcontrol.wait;" ::: "memory");
  // The CTA's units: unit blockIdx.x, or in prefix mode with p.cta_units the list [first, first + count), run
  // one after the other (a balanced partition of the shared runs' key tiles over fewer CTAs than pieces).
  int u_first = blockIdx.x, n_my = 1;
  if constexpr (PREFIX && MULTI) {
    const int2 cr = p.cta_units[blockIdx.x];
    u_first = cr.x;
    n_my = cr.y;
  }
  ChunkUnit u;
  ChunkDesc cd;
  int q_t0 = -1;  // prefix mode: first packed Q row when the family's rows are consecutive (Q by TMA)
  int pd_split = 0, pd_nsplits = 1, pd_split_off = 0;  // prefix mode: the unit's key split (PrefixDesc)
  const int epb = BN / p.P;  // page entries per KV tile
  int n_tiles = 0, m0 = 0, n_mt = 0;
  auto load_unit = [&](int ui) {
    u = p.units[ui];
    if constexpr (PREFIX) {
      const PrefixDesc pd = p.pdescs[u.desc];
      cd = ChunkDesc{pd.slab_off, pd.n_entries, 0, pd.n_rows, pd.row0, pd.n_entries, 0, 0};
      q_t0 = pd.q_t0;
      pd_split = pd.split;
      pd_nsplits = pd.n_splits;
      pd_split_off = pd.split_off;
    } else {
      cd = p.descs[u.desc];
    }
    n_tiles = (cd.n_entries + epb - 1) / epb;
    const int rows_total = cd.n_q * G;
    m0 = 2 * u.m;                                     // first M-tile of this CTA
    n_mt = min(2, (rows_total + BM - 1) / BM - m0);  // 1 or 2 M-tiles
  };
  load_unit(u_first);

  if (threadIdx.x == 0) K2T(24, 0);
#ifdef KVFS_K2_TRACE
  unsigned long long gt0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
  if (threadIdx.x == 0 && blockIdx.x < 512) g_k2_trace[1][30][blockIdx.x] = gt0;
#endif
  auto init_bars = [&]() {
    // prefix mode with gathered rows: one arrival per softmax warp that gathers Q; else one TMA transaction
    mbar_init(bar(B_Q), (PREFIX && q_t0 < 0) ? 4 * n_mt : 1);
    for (int s = 0; s < KS2; ++s) {
      mbar_init(bar(B_KF + s), 1);
      mbar_init(bar(B_KE + s), 1);
    }
    for (int s = 0; s < VS2; ++s) {
      mbar_init(bar(B_VF + s), 1);
      mbar_init(bar(B_VE + s), 1);
    }
    for (int m = 0; m < 2; ++m) {
      mbar_init(bar(B_SF + m), 1);
      mbar_init(bar(B_PF + 2 * m), 4);      // P keys 0..63 written
      mbar_init(bar(B_PF + 2 * m + 1), 4);  // P keys 64..127 written
      mbar_init(bar(B_OF + m), 1);
    }
    for (int j = 0; j < JR; ++j) mbar_init(bar(B_JF + j), 1);
    mbar_init(bar(B_X), 1);
    fence_mbar_init();
  };
  if (threadIdx.x == 0) init_bars();
  // Between two units of the CTA: every role has finished the previous one (the MMA warp waited for its last
  // commits' arrivals, the epilogue's bulk stores have read their staging), so the barriers are invalidated
  // and re-armed for the next unit, whose phases start again at 0.
  auto next_unit = [&](int j) {
    tc_fence_before();
    named_bar_sync(1, THREADS);
    load_unit(u_first + j);
    if (threadIdx.x == 0) {
      for (int i = 0; i <= B_X; ++i) mbar_inval(bar(i));
      init_bars();
    }
    named_bar_sync(1, THREADS);
    tc_fence_after();
  };
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
  if constexpr (PREFIX) {
    // (waited for the step prologue at the top) let the decode kernel that merges these partials start: it
    // reads them only after its own griddepcontrol.wait, i.e. after this grid completed
    asm volatile("griddepcontrol.launch_dependents;");
#ifdef KVFS_K2_TRACE
    if (threadIdx.x == 0 && blockIdx.x < 512) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      g_k2_trace[1][26][blockIdx.x] = gt;  // prologue dependency satisfied
    }
#endif
  }
  constexpr uint32_t tmem = 0;

  // MMA issue helpers (one elected lane of the MMA warp)
  constexpr uint32_t ID_S = idesc_bf16(false), ID_O = idesc_bf16(true);
    auto issue_s = [&](int t, int m) {
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t koff = (k >> 2) * HALF_BYTES + (k & 3) * 32;
          mma_bf16(tmem + m * BN, umma_desc(sbase + OFF_Q2 + m * TILE_BYTES + koff, 16, 1024),
                   umma_desc(sbase + OFF_K2 + (t % KS2) * TILE_BYTES + koff, 16, 1024), ID_S, k > 0);
        }
        mma_commit(bar(B_SF + m));
      }
      __syncwarp();
    };
    // P.V in two halves of 64 keys: the first half runs on the tensor pipe while the softmax computes
    // the exponentials of the second
    auto issue_pv = [&](int t, int m, int half) {
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < BN / 32; ++kk) {
          const int k = half * (BN / 32) + kk;
          mma_bf16_ts(tmem + O_COL2 + m * HD, tmem + m * BN + k * 8,
                      umma_desc(sbase + OFF_V2 + (t % VS2) * TILE_BYTES + k * 2048, HALF_BYTES, 1024), ID_O,
                      (t > 0 || k > 0));
        }
        // O complete: one commit after the last tile's P.V only (the softmax waits for it once, in the
        // epilogue; a commit per tile left phases nobody waits on, which compute-sanitizer synccheck reports)
        if (half && t == n_tiles - 1) mma_commit(bar(B_OF + m));
      }
      __syncwarp();
    };
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    for (int j = 0; j < n_my; ++j) {
    if (j > 0) next_unit(j);
    if (warp == 0) {
      // ============================================================ K producer (+ Q, + column metadata)
      const uint64_t pol = policy_evict_first();
      if ((!PREFIX || q_t0 >= 0) && lane == 0) {
        mbar_arrive_expect_tx(bar(B_Q), n_mt * TILE_BYTES);
        for (int m = 0; m < n_mt; ++m) {
          const int qrow = (PREFIX ? q_t0 : cd.row0) + ((m0 + m) * BM) / G;
          tma_load_4d(sbase + OFF_Q2 + m * TILE_BYTES, &qmap, 0, 0, u.g, qrow, bar(B_Q));
          tma_load_4d(sbase + OFF_Q2 + m * TILE_BYTES + HALF_BYTES, &qmap, 64, 0, u.g, qrow, bar(B_Q));
        }
      }
      // Page-table entries are fetched 32 at a time with one coalesced load (lane i <-> entry 32 blk + i)
      // and handed to the tile's columns by shuffles: no dependent global load on the per-tile path.
      // jbase(e) = j of entry e's first retained token = first_new_lstart - n_old + sum of the popcounts
      // of the entries fne .. e-1 (entries at or after the first new entry hold new tokens).
      uint64_t emask = 0;
      int32_t erow = p.pool_rows, jbase = 0, carry = cd.first_new_lstart - cd.n_old;
      int cached = -1;
      for (int t = 0; t < n_tiles; ++t) {
        const int s = t % KS2;
        if (t >= KS2) mbar_wait_sleep(bar(B_KE + s), ((t / KS2) & 1) ^ 1);
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
          if constexpr (!PREFIX) {  // (prefix mode: every key is an old token, no logical index needed)
            const int cnt = (e >= cd.first_new_entry) ? __popcll(emask) : 0;
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int y = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += y;
            }
            jbase = carry + incl - cnt;
            carry += __shfl_sync(0xffffffffu, incl, 31);
          }
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
          const int e = e0 + i;
          int32_t j = 0x7fffffff;
          if constexpr (PREFIX) {
            if (e < cd.n_entries && ((m >> slot) & 1ull)) j = -1;
          } else {
            const int32_t jb = __shfl_sync(0xffffffffu, jbase, src);
            if (e < cd.n_entries && ((m >> slot) & 1ull))
              j = (e < cd.first_new_entry) ? -1 : jb + __popcll(m & ((1ull << slot) - 1ull));
          }
          jcol[c] = j;
          vis_all &= (j < 0);
        }
        vis_all = __all_sync(0xffffffffu, vis_all);
        const int32_t row = __shfl_sync(0xffffffffu, erow, (e0 & 31) + (lane % epb));
        if (lane == 0) {
          jflag[t % JR] = vis_all ? 1 : 0;
          mbar_arrive(bar(B_JF + t % JR));
          mbar_arrive_expect_tx(bar(B_KF + s), TILE_BYTES);
        }
        __syncwarp();
        if (lane < epb) {  // entry e0 + lane (rows past the table: out-of-bounds box, zero-filled)
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sbase + OFF_K2 + s * TILE_BYTES + h * HALF_BYTES + lane * p.P * 128, &kmap, h * 64, row,
                        bar(B_KF + s), pol);
        }
        __syncwarp();
      }
    } else if (warp == 3) {
      // ============================================================ V producer
      const uint64_t pol = policy_evict_first();
      int32_t erow = p.pool_rows;
      int cached = -1;
      for (int t = 0; t < n_tiles; ++t) {
        const int s = t % VS2;
        if (t >= VS2) mbar_wait_sleep(bar(B_VE + s), ((t / VS2) & 1) ^ 1);
        const int e0 = t * epb, blk = e0 >> 5;
        if (blk != cached) {
          const int e = blk * 32 + lane;
          erow = e < cd.n_entries ? (static_cast<int>(p.slab[cd.slab_off + e].page) * p.Hkv + u.g) * p.P : p.pool_rows;
          cached = blk;
        }
        const int32_t row = __shfl_sync(0xffffffffu, erow, (e0 & 31) + (lane % epb));
        if (lane == 0) mbar_arrive_expect_tx(bar(B_VF + s), TILE_BYTES);
        __syncwarp();
        if (lane < epb) {
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sbase + OFF_V2 + s * TILE_BYTES + h * HALF_BYTES + lane * p.P * 128, &vmap, h * 64, row,
                        bar(B_VF + s), pol);
        }
        __syncwarp();
      }
    } else if (warp == 1) {
      // ============================================================ MMA issuer
      mbar_wait(bar(B_Q), 0);
      if (lane == 0) K2T(25, 0);
      mbar_wait(bar(B_KF + 0), 0);
      if (lane == 0) K2G(22);  // first K tile landed
      for (int m = 0; m < n_mt; ++m) issue_s(0, m);
      if (elect_one()) mma_commit(bar(B_KE + 0));
      __syncwarp();
      for (int t = 0; t < n_tiles; ++t) {
        const int s = t % VS2;  // V stage of tile t
        const bool more = t + 1 < n_tiles;
        mbar_wait(bar(B_VF + s), (t / VS2) & 1);
        if (lane == 0) K2T(9, t);
        for (int m = 0; m < n_mt; ++m) {
          K2_WAIT(bar(B_PF + 2 * m), t & 1);  // softmax m wrote P(t) keys 0..63 (and corrected O)
          issue_pv(t, m, 0);
          K2_WAIT(bar(B_PF + 2 * m + 1), t & 1);  // keys 64..127
          if (lane == 0) K2T(10 + 2 * m, t);
          issue_pv(t, m, 1);
          if (more) {                       // in-order after PV(t): S(t+1) may overwrite P(t)'s columns
            if (m == 0) mbar_wait(bar(B_KF + (t + 1) % KS2), ((t + 1) / KS2) & 1);
            issue_s(t + 1, m);
          }
          if (lane == 0) K2T(11 + 2 * m, t);
        }
        if (elect_one()) {
          if (more) mma_commit(bar(B_KE + (t + 1) % KS2));
          mma_commit(bar(B_VE + s));
        }
        __syncwarp();
      }
      if (j + 1 < n_my) {
        // another unit follows: wait until the arrivals of the last K / V stage commits (nobody else waits
        // for them) have landed, so the barriers can be re-armed
        for (int t = max(0, n_tiles - KS2); t < n_tiles; ++t) mbar_wait(bar(B_KE + t % KS2), (t / KS2) & 1);
        for (int t = max(0, n_tiles - VS2); t < n_tiles; ++t) mbar_wait(bar(B_VE + t % VS2), (t / VS2) & 1);
      }
    }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    for (int j = 0; j < n_my; ++j) {
    if (j > 0) next_unit(j);
    // ============================================================ softmax warpgroups (thread = row)
    const int m = (warp - 4) >> 2;          // M-tile of this warpgroup
    const int wq = (warp - 4) & 3;          // TMEM lane quarter
    if (m < n_mt) {
      const int r = wq * 32 + lane;
      const int R = (m0 + m) * BM + r;
      const int qi = R / G, h = R % G;
      const bool live = qi < cd.n_q;
      const uint32_t lane_addr = static_cast<uint32_t>(wq * 32) << 16;
      const uint32_t s_col = tmem + lane_addr + m * BN;
      const uint32_t o_col = tmem + lane_addr + O_COL2 + m * HD;
      if (PREFIX && q_t0 < 0) {
        // thread r gathers its row (family token qi, head h) of Q into the K-major SW128 tile: 16-byte
        // chunk cc of row r of a 64-column half lands at chunk cc ^ (r % 8) of the row's 128-byte line
        uint8_t *qt = smem + OFF_Q2 + m * TILE_BYTES;
        uint4 v[16];
        if (m == 0 && wq == 0 && lane == 0) K2G(18);  // softmax warps start the gather
        if (live) {
          const PrefixRow pr = p.prows[cd.row0 + qi];
          if (m == 0 && wq == 0 && lane == 0) K2G(23);  // row record loaded
          const uint4 *src = reinterpret_cast<const uint4 *>(p.q + (static_cast<int64_t>(pr.t) * p.Hq + u.g * G + h) * HD);
#pragma unroll
          for (int c = 0; c < 16; ++c) v[c] = __ldg(src + c);
          if (m == 0 && wq == 0 && lane == 0 && v[15].w != 0x7fffffffu) K2G(19);  // Q loads returned
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c) v[c] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int c = 0; c < 16; ++c)
          *reinterpret_cast<uint4 *>(qt + (c >> 3) * HALF_BYTES + r * 128 + (((c & 7) ^ (r & 7)) << 4)) = v[c];
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(B_Q));
        if (m == 0 && wq == 0 && lane == 0) K2G(20);  // Q rows gathered
      }
      // prefix mode: lane j < 32 / G of the warp stores the record of the warp's j-th query token in the
      // epilogue; its destination is resolved now, off the epilogue's critical path
      int64_t rec_idx = -1;
      if (PREFIX && lane < 32 / G) {
        const int tq = ((m0 + m) * BM + wq * 32 + lane * G) / G;
        if (tq < cd.n_q) {
          const PrefixRow pr = p.prows[cd.row0 + tq];
          const int64_t uq = static_cast<int64_t>(u.g * pr.n_q + pr.qi);
          const int64_t rr = pr.pref_base + uq;
          // fold mode (split_off < 0): the decode kernel folds the S split records of its unit itself,
          // record pref_base + (g n_q + qi) S + split; else split records for the in-kernel group merge
          rec_idx = pd_split_off < 0 ? pr.pref_base + uq * pd_nsplits + pd_split
                                     : (pd_nsplits > 1 ? pd_split_off + rr * pd_nsplits + pd_split : rr);
        }
      }
      float m_run = -CUDART_INF_F, l_run = 0.f;
      for (int t = 0; t < n_tiles; ++t) {
        // The column metadata of tile t is ready long before S(t): its (~150 clk) barrier wait is taken
        // while the tensor pipe is still computing S(t), off the critical path.
        mbar_wait(bar(B_JF + t % JR), (t / JR) & 1);
        const int32_t *jcol = jcol_all + (t % JR) * BN;
        const bool vis_all = jflag[t % JR] != 0;
        K2_WAIT(bar(B_SF + m), t & 1);
        if (wq == 0 && lane == 0) K2T(14 + 6 * m, t);
        if (PREFIX && t == 0 && m == 0 && wq == 0 && lane == 0) K2G(21);  // first S ready
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
        if (wq == 0 && lane == 0) K2T(15 + 6 * m, t);
        if (m == 0 && wq == 0 && lane == 0) K2T(29, t);
        // raw-score max (scale > 0 commutes with max); masked columns -> -inf.  Four independent chains.
        float mx4[4] = {-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F};
        if (vis_all) {
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
        // O is stable here without waiting on B_OF: S(t) was committed after P.V(t-1) by the same thread, and a
        // tcgen05.commit arrives only when all of that thread's earlier tcgen05 ops are complete.
        const bool need = mx > m_run + 8.f;
        if (__any_sync(0xffffffffu, need)) {
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
        // P = exp2(x * scale_log2 - m) -> bf16 pairs into the first 64 columns of this tile's S (the A
        // operand of P.V); packed fp32x2 FMA for the argument and the row sum
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        const float2 nm2 = make_float2(-mref, -mref);
        float2 ls4[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float w[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float2 a = nm2;
            fma2(a, make_float2(x[c * 64 + 2 * i], x[c * 64 + 2 * i + 1]), sc2);
            // EXP_EMU of every 8 pairs go to the FMA pipe (polynomial), the rest to MUFU
            const float2 pp = ((i & 7) >= 8 - EXP_EMU) ? exp2_poly2(a) : make_float2(fast_exp2(a.x), fast_exp2(a.y));
            ls4[i & 1] = add2(ls4[i & 1], pp);
            __nv_bfloat162 pr = __floats2bfloat162_rn(pp.x, pp.y);
            w[i] = __uint_as_float(*reinterpret_cast<uint32_t *>(&pr));
          }
          tmem_st32(s_col + c * 32, w);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar(B_PF + 2 * m + c));
        }
        if (wq == 0 && lane == 0) K2T(18 + 6 * m, t);
        const float2 ls2 = add2(ls4[0], ls4[1]);
        const float ls = ls2.x + ls2.y;
        l_run += ls;
        if (wq == 0 && lane == 0) K2T(19 + 6 * m, t);
      }
      // epilogue: O / l -> bf16 out, lse   (prefix mode: the partial O, m, l of the split)
      mbar_wait(bar(B_OF + m), 0);
      if (m == 0 && wq == 0 && lane == 0) K2T(26, 0);
#ifdef KVFS_K2_TRACE
      if (m == 0 && wq == 0 && lane == 0 && blockIdx.x < 512) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        g_k2_trace[1][27][blockIdx.x] = gt;  // O complete (main loop done)
      }
#endif
      tc_fence_after();
      if constexpr (PREFIX) {
        // The partial (o, m, l) rows go out by 1-D TMA bulk stores from a shared-memory image of their global
        // layout: row R of the pair (qi = R / G, h = R % G) -> staging byte R * 4 (HD + 2), so the G rows of
        // one query token qi are one contiguous G (HD + 2)-float record, stored with one bulk copy.  The
        // staging overlays Q, K and V (256 rows x 520 B = 130 KiB).  Each M-tile stages as soon as its own O
        // is complete: M-tile 0's half (bytes 0 .. 66.5 KiB: Q and the first 2.5 KiB of K stage 0) is dead
        // then, because the tensor pipe runs in issue order and the MMA warp issued the last S of M-tile 1
        // before the last P.V of M-tile 0; M-tile 1's half (66.5 .. 133 KiB: K and the first 5 KiB of V stage
        // 0) is dead once its own last P.V, issued after M-tile 0's, completed.
        if (m == 0 && wq == 0 && lane == 0) K2G(10);  // this M-tile's O complete
        tc_fence_after();
        constexpr int PARTF = part_floats(G, HD);
        const int Rl = m * BM + r;  // row within the pair: token Rl / G, head Rl % G
        float *row = reinterpret_cast<float *>(smem + OFF_Q2) + (Rl / G) * PARTF + (Rl % G) * (HD + 2);
        float va[32], vb[32];
        tmem_ld32(o_col, va);
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
          float(&v)[32] = (c & 1) ? vb : va;
          float(&vn)[32] = (c & 1) ? va : vb;
          tmem_wait_ld();
          if (c + 1 < HD / 32) tmem_ld32(o_col + (c + 1) * 32, vn);
#pragma unroll
          for (int i = 0; i < 32; i += 2) *reinterpret_cast<float2 *>(row + c * 32 + i) = make_float2(v[i], v[i + 1]);
        }
        *reinterpret_cast<float2 *>(row + HD) = make_float2(m_run, l_run);
        fence_proxy_async();
        __syncwarp();
        if (m == 0 && wq == 0 && lane == 0) K2G(11);  // staging written
        // lane j < 32 / G stores the record of the warp's j-th query token
        if (lane < 32 / G) {
          if (rec_idx >= 0) {
            const uint32_t src = sbase + OFF_Q2 + static_cast<uint32_t>(((m * BM + wq * 32) / G + lane) * PARTF * 4);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p.ppart + rec_idx * PARTF),
                         "r"(src), "r"(static_cast<uint32_t>(PARTF * 4))
                         : "memory");
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          if (pd_split_off < 0) {
            // fold mode: only the next grid reads the records (after this grid completed): the staging must
            // just outlive the copies' shared-memory reads
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          } else {
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // performed: visible after the fences below
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
        }
        __syncwarp();
        if (m == 0 && wq == 0 && lane == 0) K2G(12);  // records stored
      } else {
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
            uint32_t w[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              __nv_bfloat162 pr = __floats2bfloat162_rn(v[i + 2 * j] * inv, v[i + 2 * j + 1] * inv);
              w[j] = *reinterpret_cast<uint32_t *>(&pr);
            }
            *reinterpret_cast<uint4 *>(p.out + orow + c * 32 + i) = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
      if (live && p.lse)
        p.lse[static_cast<int64_t>(cd.row0 + qi) * p.Hq + u.g * G + h] =
            (m_run + __log2f(l_run)) * 0.69314718055994531f;
      }
    }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) K2T(27, 0);
#ifdef KVFS_K2_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 512) {
    unsigned long long gt1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
    g_k2_trace[1][31][blockIdx.x] = gt1;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_k2_trace[1][29][blockIdx.x] = smid;
  }
#endif
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
  if constexpr (PREFIX) {
    // Split merge: the S CTAs of a (family, kv head, M-tile pair) group wait for each other (the host makes
    // such a grid at most one CTA per SM, so all are resident; the decode kernel cannot start before every
    // CTA of this grid has started), then CTA `split` folds the S split partials of its slice of the pair's
    // rows into the merged record: (o, m, l) with one (M, L) per row, all loads of up to 8 splits in flight.
    const PrefixDesc pd = p.pdescs[u.desc];
    const int S = pd.n_splits;
    // Arrival counters alternate between two arrays by launch parity: this launch counts in array `parity`
    // and clears the other one, which the previous launch used (it completed before this one started) and
    // the next launch will use.
    {
      int *clear = p.pgroup + (p.pgroup_parity ^ 1) * kMaxPrefixGroups;
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kMaxPrefixGroups; i += gridDim.x * blockDim.x) clear[i] = 0;
    }
    if (S > 1 && pd.split_off >= 0) {
      int *arrived = p.pgroup + p.pgroup_parity * kMaxPrefixGroups + u.group;
      __threadfence();  // this CTA's partial records (bulk stores waited for), before the group sees the arrival
      __syncthreads();
      if (threadIdx.x == 0) {
        atomicAdd(arrived, 1);
        while (ld_acquire_gpu(arrived) < S) {
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");  // the bulk loads below read what others stored
        K2G(16);  // the group's partials are all written
      }
      __syncthreads();
      // Owned slice: rows [r0, r1) of the pair = query tokens [t0, t1).  The S split records of token t are
      // contiguous in global memory (split_off + r * S + s): one bulk copy of S G (HD + 2) floats per token
      // into shared memory (over the staging area, whose stores were waited for), all in flight at once.
      constexpr int PARTF = part_floats(G, HD);
      const int rp = n_mt * BM;
      const int tpo = ((rp / G) + S - 1) / S;  // tokens per owner
      const int t0 = m0 * BM / G + pd.split * tpo, t1 = min(m0 * BM / G + rp / G, t0 + tpo);
      const int nt = max(0, min(t1, cd.n_q) - t0);
      float *stage = reinterpret_cast<float *>(smem + OFF_Q2);
      if (threadIdx.x < 32) {
        const uint32_t xb = bar(B_X);
        if (threadIdx.x == 0) mbar_arrive_expect_tx(xb, static_cast<uint32_t>(nt * S * PARTF * 4));
        __syncwarp();
        for (int j = threadIdx.x; j < nt; j += 32) {
          const PrefixRow pr = p.prows[cd.row0 + t0 + j];
          const int64_t rr = pr.pref_base + static_cast<int64_t>(u.g * pr.n_q + pr.qi);
          bulk_g2s(sbase + OFF_Q2 + static_cast<uint32_t>(j * S * PARTF * 4), p.ppart + (pd.split_off + rr * S) * PARTF,
                   static_cast<uint32_t>(S * PARTF * 4), xb, policy_evict_first());
        }
      }
      if (nt > 0) mbar_wait(bar(B_X), 0);
      // fold: item = (token j, head h, 8 dims), the softmax warps (the others run at 56 registers)
      for (int it = static_cast<int>(threadIdx.x) - 128; it >= 0 && it < nt * G * (HD / 8); it += 256) {
        const int j = it / (G * (HD / 8)), h = (it / (HD / 8)) % G, d0 = (it % (HD / 8)) * 8;
        const float *rec = stage + static_cast<int64_t>(j) * S * PARTF + h * (HD + 2);
        float M = -CUDART_INF_F;
        for (int sp = 0; sp < S; ++sp) M = fmaxf(M, rec[sp * PARTF + HD]);
        float L = 0.f, acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int sp = 0; sp < S; ++sp) {
          const float *x = rec + sp * PARTF;
          const float f = (x[HD] == -CUDART_INF_F) ? 0.f : fast_exp2(x[HD] - M);
          L += x[HD + 1] * f;
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            const float2 v = *reinterpret_cast<const float2 *>(x + d0 + i);
            acc[i] += v.x * f;
            acc[i + 1] += v.y * f;
          }
        }
        const PrefixRow pr = p.prows[cd.row0 + t0 + j];
        const int64_t rr = pr.pref_base + static_cast<int64_t>(u.g * pr.n_q + pr.qi);
        float *dst = p.ppart + rr * PARTF + h * (HD + 2);
#pragma unroll
        for (int i = 0; i < 8; i += 2) __stcg(reinterpret_cast<float2 *>(dst + d0 + i), make_float2(acc[i], acc[i + 1]));
        if (d0 == 0) __stcg(reinterpret_cast<float2 *>(dst + HD), make_float2(M, L));
      }
#ifdef KVFS_K2_TRACE
      __syncthreads();
      if (threadIdx.x == 0) K2G(17);  // merged
#endif
    }
#ifdef KVFS_K2_TRACE
    __syncthreads();
    if (threadIdx.x == 0) K2G(25);  // CTA done
#endif
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

int chunk_smem_bytes() { return tc2::SMEM2; }

#ifdef KVFS_K2_TRACE
extern "C" int kvfs_debug_k2_trace(void *host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, g_k2_trace, bytes < sizeof(g_k2_trace) ? bytes : sizeof(g_k2_trace)) ==
                 cudaSuccess ? 0 : -1;
}
#endif

template <int G, bool PREFIX, bool MULTI>
static cudaError_t launch_chunk_gm(const CUtensorMap &km, const CUtensorMap &vm, const CUtensorMap &qm,
                                   const ChunkParams &p, int n_units, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(chunk_attn_tc_kernel<G, PREFIX, MULTI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, tc2::SMEM2);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_units);
  cfg.blockDim = dim3(tc2::THREADS);
  cfg.dynamicSmemBytes = tc2::SMEM2;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = PREFIX ? 1 : 0;  // prefix mode waits in-kernel
  cfg.attrs = la;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, chunk_attn_tc_kernel<G, PREFIX, MULTI>, km, vm, qm, p);
}

template <int G, bool PREFIX>
static cudaError_t launch_chunk_g(const CUtensorMap &km, const CUtensorMap &vm, const CUtensorMap &qm,
                                  const ChunkParams &p, int n_units, cudaStream_t s) {
  if constexpr (PREFIX) {
    if (p.cta_units) return launch_chunk_gm<G, true, true>(km, vm, qm, p, n_units, s);
  }
  return launch_chunk_gm<G, PREFIX, false>(km, vm, qm, p, n_units, s);
}

template <bool PREFIX>
static cudaError_t launch_mode(const CUtensorMap &km, const CUtensorMap &vm, const CUtensorMap &qm,
                               const ChunkParams &p, int n_units, int G, cudaStream_t s) {
  switch (G) {
    case 1: return launch_chunk_g<1, PREFIX>(km, vm, qm, p, n_units, s);
    case 2: return launch_chunk_g<2, PREFIX>(km, vm, qm, p, n_units, s);
    case 4: return launch_chunk_g<4, PREFIX>(km, vm, qm, p, n_units, s);
    case 8: return launch_chunk_g<8, PREFIX>(km, vm, qm, p, n_units, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_chunk(const CUtensorMap &km, const CUtensorMap &vm, const CUtensorMap &qm, const ChunkParams &p,
                         int n_units, int G, cudaStream_t s) {
  return launch_mode<false>(km, vm, qm, p, n_units, G, s);
}

cudaError_t launch_prefix(const CUtensorMap &km, const CUtensorMap &vm, const CUtensorMap &qm, const ChunkParams &p,
                          int n_units, int G, cudaStream_t s) {
  return launch_mode<true>(km, vm, qm, p, n_units, G, s);
}

}  // namespace dev
}  // namespace kvfs
