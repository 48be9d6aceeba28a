// K9: attention-score accumulation for heavy-hitter replacement policies (§6, H2O;
// include/kvfs.h pred_attn_scores).  A second, HBM-bound pass over the K rows of the step's files:
//   scores[off_d + k] = sum_{rows i of d, heads h} exp2(scale_log2 <q_ih, K_k,g(h)> - lse_ih log2 e)
// for every retained token k visible to row i (logical k <= len_after - n_q + i), exactly the softmax
// weights of rule R10 given the lse the attention kernels wrote.
// One CTA per (descriptor, chunk of <= 32 page entries).  Tensor-core contraction of 16-key tiles (below).
#include <cuda_bf16.h>

#include "kernels.cuh"

namespace kvfs {
namespace dev {

// Layout per CTA (256 threads = 8 warps, two CTAs per SM): warp w takes kv head g = w % Hkv and every
// (8 / Hkv)-th 16-slot tile of the unit's entries that holds a retained slot.  Each warp streams its tiles
// through a private ring of NS stages with 2-D TMA (16 rows x 64 dims per box, 128-byte swizzle; lane 0
// issues, completion on the stage's mbarrier) and contracts them on the tensor cores: S^T = K_tile Q^T as
// mma.m16n8k16 (A = 16 keys x 16 dims from ldmatrix, B = 16 dims x 8 columns, a column = one (query row,
// head) pair of the descriptor, G <= 8 heads per kv head, n_q * G columns in tiles of 8).  The epilogue of a
// tile is exp2(s * scale_log2 - lse_col * log2 e) for the visible (key, row) pairs, summed over the lane's
// columns, reduced over the 4 lanes of a row, and added into the key's shared-memory accumulator.
// Holes of a partially retained tile are read (one TMA box) and masked out of the sums.
#ifndef KVFS_K9_NS
#define KVFS_K9_NS 2
#endif
#ifndef KVFS_K9_MINB
#define KVFS_K9_MINB 3
#endif
constexpr int kScoreStages = KVFS_K9_NS;  // ring stages per warp (2 x 4 KB x 8 warps: three CTAs per SM)

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &a0, uint32_t &a1, uint32_t &a2, uint32_t &a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr)
               : "memory");
}

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int D>
__global__ void __launch_bounds__(256, KVFS_K9_MINB)
    scores_kernel(const __grid_constant__ CUtensorMap kmap, const ScoreUnit *units, const ScoreDesc *descs,
                  const Entry *slab, const __nv_bfloat16 *q, const float *lse, float scale_log2, float *out, int Hkv,
                  int G, int P) {
  constexpr int NS = kScoreStages;
  constexpr int NB = D / 64;          // 64-dim TMA boxes per tile
  constexpr int TILE = 16 * D * 2;    // bytes of one 16-key tile
  constexpr int KS = D / 16;          // mma k-steps
  __shared__ float acc[32 * 64];      // [entry][slot]
  __shared__ uint64_t emask[32];
  __shared__ uint32_t epage[32];
  __shared__ int32_t elog[32];
  __shared__ __align__(8) uint64_t fullb[8][NS];
  extern __shared__ __align__(16) uint8_t dyn[];
  const uint32_t ring0 = (smem_u32(dyn) + 1023u) & ~1023u;
  const ScoreUnit u = units[blockIdx.x];
  const ScoreDesc d = descs[u.desc];
  const int ne = u.e1 - u.e0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    uint64_t m = 0;
    uint32_t pg = 0;
    if (lane < ne) {
      const Entry e = slab[d.slab_off + u.e0 + lane];
      m = e.mask;
      pg = e.page;
    }
    const int cnt = __popcll(m);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    emask[lane] = m;
    epage[lane] = pg;
    elog[lane] = incl - cnt;  // unit-relative logical index of the entry's first retained slot
  }
  if (lane < NS) mbar_init(smem_u32(&fullb[warp][lane]), 1);
  for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) acc[i] = 0.f;
  fence_mbar_init();
  __syncthreads();

  const int g = warp % Hkv, kset = warp / Hkv, nsets = 8 / Hkv;  // Hkv in {1, 2, 4, 8}
  const int tpe = P >> 4, ntiles = ne * tpe;
  const uint32_t ring = ring0 + static_cast<uint32_t>(warp * NS * TILE);
  const uint64_t pol = policy_evict_first();
  auto tmask = [&](int t) -> uint32_t { return static_cast<uint32_t>(emask[t / tpe] >> ((t % tpe) * 16)) & 0xffffu; };
  auto next = [&](int t) {
    while (t < ntiles && !tmask(t)) t += nsets;
    return t;
  };
  auto issue = [&](int t, int slot) {
    if (lane == 0) {
      const uint32_t bar = smem_u32(&fullb[warp][slot]);
      mbar_arrive_expect_tx(bar, TILE);
      const int row = (static_cast<int>(epage[t / tpe]) * Hkv + g) * P + (t % tpe) * 16;
#pragma unroll
      for (int b = 0; b < NB; ++b) tma_load_2d(ring + slot * TILE + b * 2048, &kmap, b * 64, row, bar, pol);
    }
  };
  int tiss = next(kset);
#pragma unroll
  for (int s2 = 0; s2 < NS; ++s2) {
    if (tiss < ntiles) {
      issue(tiss, s2);
      tiss = next(tiss + nsets);
    }
  }

  // columns: c = r * G + h (query row r of the descriptor, head h of kv head g)
  const int Hq = Hkv * G;
  const int ncols = d.n_q * G, nct = (ncols + 7) >> 3;
  const int base = d.len_after - d.n_q - u.l0;  // row r sees unit-relative keys <= base + r
  uint32_t bq[KS][2];
  float l2c[2];
  int lim[2];  // highest visible unit-relative key of the lane's two C columns (-1: padding column)
  auto load_cols = [&](int ct) {
    const int n = ct * 8 + (lane >> 2);
    if (n < ncols) {
      const uint32_t *qp = reinterpret_cast<const uint32_t *>(
          q + (static_cast<int64_t>(d.row0 + n / G) * Hq + g * G + n % G) * D);
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        bq[ks][0] = __ldg(qp + ks * 8 + (lane & 3));
        bq[ks][1] = __ldg(qp + ks * 8 + 4 + (lane & 3));
      }
    } else {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) bq[ks][0] = bq[ks][1] = 0u;
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int c = ct * 8 + (lane & 3) * 2 + j;
      if (c < ncols) {
        l2c[j] = lse[static_cast<int64_t>(d.row0 + c / G) * Hq + g * G + c % G] * 1.4426950408889634f;
        lim[j] = base + c / G;
      } else {
        l2c[j] = 0.f;
        lim[j] = -1;
      }
    }
  };
  if (nct == 1) load_cols(0);

  // ldmatrix addressing (128-byte swizzle: 16-byte chunk c of row r sits at chunk c ^ (r & 7))
  const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lhi = lane >> 4;
  const int r0 = lane >> 2, r1 = r0 + 8;
  int tcon = next(kset);
  for (int i = 0; tcon < ntiles; ++i) {
    const int slot = i % NS;
    mbar_wait(smem_u32(&fullb[warp][slot]), static_cast<uint32_t>((i / NS) & 1));
    const uint32_t st = ring + slot * TILE;
    uint32_t a[KS][4];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const uint32_t chunk = static_cast<uint32_t>(((ks & 3) * 2 + lhi) ^ (lrow & 7));
      ldsm_x4(st + (ks >> 2) * 2048 + lrow * 128 + (chunk << 4), a[ks][0], a[ks][1], a[ks][2], a[ks][3]);
    }
    __syncwarp();  // the stage is in registers: refill it
    if (tiss < ntiles) {
      issue(tiss, slot);
      tiss = next(tiss + nsets);
    }
    const int e = tcon / tpe, sub = tcon % tpe;
    const uint64_t em = emask[e];
    const int s0 = sub * 16 + r0, s1 = sub * 16 + r1;
    const int lg0 = elog[e] + __popcll(em & ((1ull << s0) - 1)), lg1 = elog[e] + __popcll(em & ((1ull << s1) - 1));
    float p0 = 0.f, p1 = 0.f;
    for (int ct = 0; ct < nct; ++ct) {
      if (nct > 1) load_cols(ct);
      float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) mma_bf16_16816(c, a[ks], bq[ks][0], bq[ks][1]);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (lg0 <= lim[j]) p0 += exp2f(fmaf(c[j], scale_log2, -l2c[j]));
        if (lg1 <= lim[j]) p1 += exp2f(fmaf(c[2 + j], scale_log2, -l2c[j]));
      }
    }
    p0 += __shfl_xor_sync(0xffffffffu, p0, 1);
    p1 += __shfl_xor_sync(0xffffffffu, p1, 1);
    p0 += __shfl_xor_sync(0xffffffffu, p0, 2);
    p1 += __shfl_xor_sync(0xffffffffu, p1, 2);
    if ((lane & 3) == 0) {
      if (em >> s0 & 1) atomicAdd(&acc[e * 64 + s0], p0);
      if (em >> s1 & 1) atomicAdd(&acc[e * 64 + s1], p1);
    }
    tcon = next(tcon + nsets);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ne * 64; i += blockDim.x) {
    const int e = i >> 6, s2 = i & 63;
    const uint64_t em = emask[e];
    if (s2 < P && (em >> s2 & 1))
      out[d.out_off + u.l0 + elog[e] + __popcll(em & ((1ull << s2) - 1))] = acc[i];
  }
}

template <int D>
static cudaError_t launch_scores_d(const CUtensorMap &kmap, const ScoreUnit *units, int n_units,
                                   const ScoreDesc *descs, const Entry *slab, const __nv_bfloat16 *q,
                                   const float *lse, float scale_log2, float *out, int G, int Hkv, int P,
                                   cudaStream_t s) {
  constexpr int smem = 8 * kScoreStages * 16 * D * 2 + 1024;  // 8 warps x NS tiles + alignment slack
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(scores_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  scores_kernel<D><<<n_units, 256, smem, s>>>(kmap, units, descs, slab, q, lse, scale_log2, out, Hkv, G, P);
  return cudaGetLastError();
}

cudaError_t launch_scores(const CUtensorMap &kmap, const ScoreUnit *units, int n_units, const ScoreDesc *descs,
                          const Entry *slab, const __nv_bfloat16 *q, const float *lse, float scale_log2, float *out,
                          int Hq, int Hkv, int D, int P, cudaStream_t s) {
  if (Hkv > 8 || 8 % Hkv || Hq % Hkv || Hq / Hkv > 8 || P % 16) return cudaErrorInvalidValue;
  if (D == 64) return launch_scores_d<64>(kmap, units, n_units, descs, slab, q, lse, scale_log2, out, Hq / Hkv, Hkv, P, s);
  if (D == 128) return launch_scores_d<128>(kmap, units, n_units, descs, slab, q, lse, scale_log2, out, Hq / Hkv, Hkv, P, s);
  return cudaErrorInvalidValue;
}

}  // namespace dev
}  // namespace kvfs

namespace kvfs {
namespace dev {

// K10: fused scores.  The decode kernel (K1) wrote, for every key it attended, the scaled logit s (log2
// domain) of each head (DevDesc::logit_off); the score of retained token k of descriptor d is then
//   sum_{rows qi of d that see k} sum_{kv heads g, heads h of g} exp2(s[g, qi][k][h] - lse[qi][g G + h] log2 e)
// (rule H1), reading Hq floats per (key, row) instead of the K row (Hkv D bf16): ~16x fewer bytes than K9.
// One CTA per (descriptor, <= 32 final-table entries); thread per (entry, slot).  The key's place in K1's
// stage layout: an old token (logical < n_old) sits at stage = its entry, slot = its slot; new row r at stage
// n_old_entries + r / P, slot r % P, visible to the rows qi >= r.
constexpr int kMaxLogitHeads = 1024;
__global__ void __launch_bounds__(256) logit_scores_kernel(const ScoreUnit *units, const LogitDesc *descs,
                                                           const Entry *slab, const float *logits, const float *lse,
                                                           float *out, int Hq, int Hkv, int P) {
  __shared__ uint64_t emask[32];
  __shared__ int32_t elog[32];
  const ScoreUnit u = units[blockIdx.x];
  const LogitDesc d = descs[u.desc];
  const int ne = u.e1 - u.e0, G = Hq / Hkv;
  if (threadIdx.x < 32) {
    const int e = threadIdx.x;
    const uint64_t m = e < ne ? slab[d.slab_off + u.e0 + e].mask : 0ull;
    const int pc = __popcll(m);
    int incl = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (e >= o) incl += y;
    }
    emask[e] = m;
    elog[e] = u.l0 + incl - pc;
  }
  constexpr float kLog2e = 1.4426950408889634f;
  // lse * log2(e) of the descriptor's rows in shared memory when they fit (decode descriptors: one row)
  __shared__ __align__(16) float lsh[kMaxLogitHeads];
  const bool lsm = d.n_q * Hq <= kMaxLogitHeads;
  if (lsm)
    for (int i = threadIdx.x; i < d.n_q * Hq; i += blockDim.x)
      lsh[i] = __ldg(lse + static_cast<int64_t>(d.row0) * Hq + i) * kLog2e;
  __syncthreads();
  for (int j = threadIdx.x; j < ne * P; j += blockDim.x) {
    const int e = j / P, sl = j % P;
    const uint64_t m = emask[e];
    if (!((m >> sl) & 1ull)) continue;
    const int k = elog[e] + __popcll(m & ((1ull << sl) - 1ull));
    int st, slot, q0;
    if (k < d.n_old) {
      st = u.e0 + e;
      slot = sl;
      q0 = 0;
      if (d.gather) {
        // the decode kernel's row of this key in the stage: a page whose retained slots (the old ones of the
        // last old entry) fill less than 40% of their span was gathered packed (DecodeParams::gather; the
        // same rule as decode_attn.cu)
        const uint64_t m1 = (st == d.n_old_entries - 1) ? lowest_bits(m, d.n_old - elog[e]) : m;
        const int lo = __ffsll(static_cast<long long>(m1)) - 1, hi = 63 - __clzll(static_cast<long long>(m1));
        if (5 * __popcll(m1) < 2 * (hi - lo + 1)) slot = __popcll(m1 & ((1ull << sl) - 1ull));
      }
    } else {
      const int r = k - d.n_old;
      st = d.n_old_entries + r / P;
      slot = r % P;
      q0 = r;
    }
    float acc = 0.f;
    // unit (g, qi) of the key: its G logits at lg0 + (g * n_q + qi) * ustride
    const int64_t ustride = static_cast<int64_t>(d.stages_per_unit) * P * G;
    const float *lg0 = logits + d.logit_off + (static_cast<int64_t>(st) * P + slot) * G;
    for (int qi = q0; qi < d.n_q; ++qi) {
      const float *ls = lse + static_cast<int64_t>(d.row0 + qi) * Hq;  // head g G + h of row qi (lsm: unscaled)
      const float *lss = lsh + qi * Hq;                                // (lsm: scaled)
      if ((G & 3) == 0) {
        // the row's Hq logits as Hq / 4 float4 (16-byte aligned: logit_off and every stride are multiples
        // of 4), 8 loads in flight per thread
        const int nv = Hq >> 2;
        for (int j0 = 0; j0 < nv; j0 += 8) {
          float4 x[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int jj = j0 + t, g = (4 * jj) / G, h = (4 * jj) - g * G;
            if (jj < nv) x[t] = __ldcs(reinterpret_cast<const float4 *>(lg0 + (g * d.n_q + qi) * ustride + h));
          }
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int jj = j0 + t;
            if (jj < nv) {
              float4 l;
              if (lsm) {
                l = *reinterpret_cast<const float4 *>(lss + 4 * jj);
              } else {
                l = make_float4(__ldg(ls + 4 * jj) * kLog2e, __ldg(ls + 4 * jj + 1) * kLog2e,
                                __ldg(ls + 4 * jj + 2) * kLog2e, __ldg(ls + 4 * jj + 3) * kLog2e);
              }
              acc += fast_exp2(x[t].x - l.x) + fast_exp2(x[t].y - l.y) + fast_exp2(x[t].z - l.z) +
                     fast_exp2(x[t].w - l.w);
            }
          }
        }
      } else {
        for (int g = 0; g < Hkv; ++g) {
          const float *lg = lg0 + (g * d.n_q + qi) * ustride;
          for (int h = 0; h < G; ++h)
            acc += fast_exp2(__ldcs(lg + h) - (lsm ? lss[g * G + h] : __ldg(ls + g * G + h) * kLog2e));
        }
      }
    }
    out[d.out_off + k] = acc;
  }
  // The logits are dead now: drop their L2 lines without a write-back (they were written with an evict_last
  // policy by K1, so they never reach DRAM).  Only the old-entry stages of this CTA's entries (each read by
  // this CTA alone); whole lines only: every unit-stage block is P G floats at a 128-byte aligned offset
  // (pred_logits aligns logit_off) when P G is a multiple of 32.
  if ((P * G) % 32 == 0 && (reinterpret_cast<uintptr_t>(logits) & 127) == 0) {
    __syncthreads();
    const int n_old_st = max(0, min(u.e1, d.n_old_entries) - u.e0);  // stages u.e0 .. of old entries
    const int lpb = P * G / 32;                                      // lines per unit-stage block
    const int n_units = Hkv * d.n_q;
    const int total = n_units * n_old_st * lpb;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const int ln = i % lpb, r = i / lpb, st = u.e0 + r % n_old_st, un = r / n_old_st;
      discard_l2(logits + d.logit_off + (static_cast<int64_t>(un) * d.stages_per_unit + st) * P * G + ln * 32);
    }
  }
}

cudaError_t launch_logit_scores(const ScoreUnit *units, int n_units, const LogitDesc *descs, const Entry *slab,
                                const float *logits, const float *lse, float *out, int Hq, int Hkv, int P,
                                cudaStream_t s) {
  if (n_units <= 0) return cudaSuccess;
  logit_scores_kernel<<<n_units, 256, 0, s>>>(units, descs, slab, logits, lse, out, Hq, Hkv, P);
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace kvfs
