// K9: attention-score accumulation for heavy-hitter replacement policies (§6, H2O;
// include/kvfs.h pred_attn_scores).  A second, HBM-bound pass over the K rows of the step's files:
//   scores[off_d + k] = sum_{rows i of d, heads h} exp2(scale_log2 <q_ih, K_k,g(h)> - lse_ih log2 e)
// for every retained token k visible to row i (logical k <= len_after - n_q + i), exactly the softmax
// weights of rule R10 given the lse the attention kernels wrote.
// One CTA per (descriptor, chunk of <= 32 page entries).
#include <cuda_bf16.h>

#include "kernels.cuh"

namespace kvfs {
namespace dev {

// Layout per CTA (256 threads = 8 warps): warp w takes kv head g = w % Hkv and every (8 / Hkv)-th group
// of 4 keys (Hkv < 8) of the unit's entries; in a warp, 8 lanes share a key (D / 8 dims each, loaded as
// 16-byte vectors: the 8 lanes read the key's contiguous row), 4 keys per step, UNR steps in flight.  The
// lane's slice of q (G heads of the current query row) stays in registers; the G partial dot products
// are reduced by xor-shuffles over the 8 lanes; lane 0 of the key adds sum_h exp2(s - lse2) into the
// key's shared-memory accumulator.  Query rows are processed one after another (decode: one row).
template <int D, int G>
__global__ void __launch_bounds__(256) scores_kernel(const ScoreUnit *units, const ScoreDesc *descs,
                                                     const Entry *slab, const __nv_bfloat16 *q, const float *lse,
                                                     const __nv_bfloat16 *kpool, float scale_log2, float *out,
                                                     int Hkv, int P) {
  constexpr int DPL = D / 8;   // dims per lane
  constexpr int CH = DPL / 8;  // 16-byte chunks per lane
  constexpr int NS = 8;        // ring stages per warp (4 key rows each)
  __shared__ float acc[32 * 64];  // [entry][slot]
  __shared__ uint64_t emask[32];
  __shared__ uint32_t epage[32];
  __shared__ int32_t elog[32];
  __shared__ int16_t kslot[32 * 64];  // retained keys of the unit: (entry << 8) | slot, logical order
  __shared__ int nkeys;
  extern __shared__ __align__(16) uint32_t ring_all[];  // [8 warps][NS][32 lanes][DPL bf16]
  const ScoreUnit u = units[blockIdx.x];
  const ScoreDesc d = descs[u.desc];
  const int ne = u.e1 - u.e0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *ring = ring_all + warp * NS * 32 * (DPL * 2 / 4);
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
    elog[lane] = incl - cnt;  // unit-relative
    int w = incl - cnt;
    for (uint64_t mm = m; mm; mm &= mm - 1) kslot[w++] = static_cast<int16_t>((lane << 8) | __ffsll(mm) - 1);
    if (lane == 31) nkeys = incl;
  }
  for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) acc[i] = 0.f;
  __syncthreads();
  const int n = nkeys;
  const int g = warp % Hkv, kset = warp / Hkv, nsets = 8 / Hkv;  // Hkv in {1, 2, 4, 8}
  const int kg = lane >> 3, sub = lane & 7;
  const int base = d.len_after - d.n_q - u.l0;  // row i sees unit-relative keys <= base + i
  for (int r = 0; r < d.n_q; ++r) {
    const int row = d.row0 + r;
    float2 qf[G][DPL / 2];
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const uint4 *qs = reinterpret_cast<const uint4 *>(q + (static_cast<int64_t>(row) * (Hkv * G) + g * G + h) * D) +
                        sub * CH;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const uint4 w = __ldg(qs + c);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = bf2_to_f2(ws[j]);
          qf[h][c * 4 + j] = make_float2(f.x * scale_log2, f.y * scale_log2);
        }
      }
    }
    float l2[G];
#pragma unroll
    for (int h = 0; h < G; ++h) l2[h] = lse[static_cast<int64_t>(row) * (Hkv * G) + g * G + h] * 1.4426950408889634f;
    const int vis = min(n, base + r + 1);  // unit-relative keys visible to this row
    // warp-private ring of NS stages of 4 key rows (cp.async, 16 B per lane per chunk): NS - 1 steps in
    // flight while one is computed
    const int n_steps = vis > kset * 4 ? (vis - kset * 4 + nsets * 4 - 1) / (nsets * 4) : 0;
    auto issue = [&](int step) {
      if (step < n_steps) {
        const int key = kset * 4 + step * nsets * 4 + kg;
        if (key < vis) {
          const int ks = kslot[key], e = ks >> 8, slot = ks & 255;
          const char *src = reinterpret_cast<const char *>(
              kpool + ((static_cast<int64_t>(epage[e]) * Hkv + g) * P + slot) * D + sub * DPL);
          const uint32_t dst = smem_u32(ring + ((step % NS) * 32 + lane) * (DPL * 2 / 4));
#pragma unroll
          for (int c = 0; c < CH; ++c)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + c * 16), "l"(src + c * 16) : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int st = 0; st < NS - 1; ++st) issue(st);
    // two steps per iteration (independent dot chains), packed fp32x2 FMAs
    for (int step = 0; step < n_steps; step += 2) {
      asm volatile("cp.async.wait_group %0;" ::"n"(NS - 3) : "memory");
      __syncwarp();
      float2 dot2[2][G];
      int keys[2];
#pragma unroll
      for (int u2 = 0; u2 < 2; ++u2) {
        keys[u2] = (step + u2 < n_steps) ? kset * 4 + (step + u2) * nsets * 4 + kg : vis;
#pragma unroll
        for (int h = 0; h < G; ++h) dot2[u2][h] = make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        uint4 w[2];
#pragma unroll
        for (int u2 = 0; u2 < 2; ++u2)
          w[u2] = keys[u2] < vis
                      ? reinterpret_cast<const uint4 *>(ring + (((step + u2) % NS) * 32 + lane) * (DPL * 2 / 4))[c]
                      : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
          for (int u2 = 0; u2 < 2; ++u2) {
            const uint32_t wv = j == 0 ? w[u2].x : (j == 1 ? w[u2].y : (j == 2 ? w[u2].z : w[u2].w));
            const float2 kf = bf2_to_f2(wv);
#pragma unroll
            for (int h = 0; h < G; ++h) fma2(dot2[u2][h], qf[h][c * 4 + j], kf);
          }
        }
      }
      __syncwarp();  // both stages are consumed: they may be refilled
      issue(step + NS - 1);
      issue(step + NS);
#pragma unroll
      for (int u2 = 0; u2 < 2; ++u2) {
        float dot[G];
#pragma unroll
        for (int h = 0; h < G; ++h) dot[h] = dot2[u2][h].x + dot2[u2][h].y;
#pragma unroll
        for (int h = 0; h < G; ++h)
#pragma unroll
          for (int o = 1; o < 8; o <<= 1) dot[h] += __shfl_xor_sync(0xffffffffu, dot[h], o);
        const int key = keys[u2];
        if (sub == 0 && key < vis) {
          float sum = 0.f;
#pragma unroll
          for (int h = 0; h < G; ++h) sum += exp2f(dot[h] - l2[h]);
          const int ks = kslot[key];
          atomicAdd(&acc[(ks >> 8) * 64 + (ks & 255)], sum);
        }
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const int ks = kslot[t];
    out[d.out_off + u.l0 + t] = acc[(ks >> 8) * 64 + (ks & 255)];
  }
  (void)elog;
}

template <int D, int G>
static cudaError_t launch_scores_t(const ScoreUnit *units, int n_units, const ScoreDesc *descs, const Entry *slab,
                                   const __nv_bfloat16 *q, const float *lse, const __nv_bfloat16 *kpool,
                                   float scale_log2, float *out, int Hkv, int P, cudaStream_t s) {
  constexpr int smem = 8 * 8 * 32 * (D / 8) * 2;  // 8 warps x NS stages x 32 lanes x DPL bf16
  static bool attr = false;
  if (!attr && smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(scores_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  scores_kernel<D, G><<<n_units, 256, smem, s>>>(units, descs, slab, q, lse, kpool, scale_log2, out, Hkv, P);
  return cudaGetLastError();
}

template <int D>
static cudaError_t launch_scores_d(const ScoreUnit *units, int n_units, const ScoreDesc *descs, const Entry *slab,
                                   const __nv_bfloat16 *q, const float *lse, const __nv_bfloat16 *kpool,
                                   float scale_log2, float *out, int G, int Hkv, int P, cudaStream_t s) {
  switch (G) {
    case 1: return launch_scores_t<D, 1>(units, n_units, descs, slab, q, lse, kpool, scale_log2, out, Hkv, P, s);
    case 2: return launch_scores_t<D, 2>(units, n_units, descs, slab, q, lse, kpool, scale_log2, out, Hkv, P, s);
    case 4: return launch_scores_t<D, 4>(units, n_units, descs, slab, q, lse, kpool, scale_log2, out, Hkv, P, s);
    case 8: return launch_scores_t<D, 8>(units, n_units, descs, slab, q, lse, kpool, scale_log2, out, Hkv, P, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_scores(const ScoreUnit *units, int n_units, const ScoreDesc *descs, const Entry *slab,
                          const __nv_bfloat16 *q, const float *lse, const __nv_bfloat16 *kpool, float scale_log2,
                          float *out, int Hq, int Hkv, int D, int P, cudaStream_t s) {
  if (Hkv > 8 || 8 % Hkv) return cudaErrorInvalidValue;
  if (D == 64) return launch_scores_d<64>(units, n_units, descs, slab, q, lse, kpool, scale_log2, out, Hq / Hkv, Hkv, P, s);
  if (D == 128) return launch_scores_d<128>(units, n_units, descs, slab, q, lse, kpool, scale_log2, out, Hq / Hkv, Hkv, P, s);
  return cudaErrorInvalidValue;
}

}  // namespace dev
}  // namespace kvfs
