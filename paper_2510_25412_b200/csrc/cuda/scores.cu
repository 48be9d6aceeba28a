// K9: attention-score accumulation for heavy-hitter replacement policies (§6, H2O;
// include/kvfs.h pred_attn_scores).  A second, HBM-bound pass over the K rows of the step's files:
//   scores[off_d + k] = sum_{rows i of d, heads h} exp2(scale_log2 <q_ih, K_k,g(h)> - lse_ih log2 e)
// for every retained token k visible to row i (logical k <= len_after - n_q + i), exactly the softmax
// weights of rule R10 given the lse the attention kernels wrote.
// One CTA per (descriptor, chunk of <= 32 page entries); thread = (entry, kv head, slot) with the slot
// fastest (a warp reads two contiguous (page, head) blocks); Q rows (bf16) and lse (log2 domain) of up to
// QB query rows staged in shared memory; per-key sums over heads in shared-memory atomics.
#include <cuda_bf16.h>

#include "kernels.cuh"

namespace kvfs {
namespace dev {

constexpr int QB = 8;  // query rows per pass over the chunk's keys

__global__ void __launch_bounds__(256) scores_kernel(const ScoreUnit *units, const ScoreDesc *descs,
                                                     const Entry *slab, const __nv_bfloat16 *q, const float *lse,
                                                     const __nv_bfloat16 *kpool, float scale_log2, float *out,
                                                     int Hq, int Hkv, int D, int P) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ float acc[32 * 64];      // [entry][slot]
  __shared__ uint64_t emask[32];
  __shared__ uint32_t epage[32];
  __shared__ int32_t elog[32];        // logical index of the entry's first retained token
  const ScoreUnit u = units[blockIdx.x];
  const ScoreDesc d = descs[u.desc];
  const int ne = u.e1 - u.e0;
  const int G = Hq / Hkv;
  __nv_bfloat16 *qs = reinterpret_cast<__nv_bfloat16 *>(sm);  // [QB][Hq][D]
  float *ls = reinterpret_cast<float *>(qs + QB * Hq * D);     // [QB][Hq]
  if (threadIdx.x < 32) {
    uint64_t m = 0;
    uint32_t pg = 0;
    if (static_cast<int>(threadIdx.x) < ne) {
      const Entry e = slab[d.slab_off + u.e0 + threadIdx.x];
      m = e.mask;
      pg = e.page;
    }
    int cnt = __popcll(m), incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (static_cast<int>(threadIdx.x) >= o) incl += y;
    }
    emask[threadIdx.x] = m;
    epage[threadIdx.x] = pg;
    elog[threadIdx.x] = u.l0 + incl - cnt;
  }
  for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) acc[i] = 0.f;
  const int base = d.len_after - d.n_q;  // row i sees logical keys <= base + i
  const int pairs = ne * Hkv * P;
  for (int qb = 0; qb < d.n_q; qb += QB) {
    const int nr = min(QB, d.n_q - qb);
    __syncthreads();
    for (int i = threadIdx.x; i < nr * Hq * D / 8; i += blockDim.x)
      reinterpret_cast<uint4 *>(qs)[i] =
          reinterpret_cast<const uint4 *>(q + static_cast<int64_t>(d.row0 + qb) * Hq * D)[i];
    for (int i = threadIdx.x; i < nr * Hq; i += blockDim.x)
      ls[i] = lse[static_cast<int64_t>(d.row0 + qb) * Hq + i] * 1.4426950408889634f;
    __syncthreads();
    for (int t = threadIdx.x; t < pairs; t += blockDim.x) {
      const int slot = t % P, g = (t / P) % Hkv, e = t / (P * Hkv);
      const uint64_t m = emask[e];
      if (!((m >> slot) & 1ull)) continue;
      const int key = elog[e] + __popcll(m & ((1ull << slot) - 1ull));
      if (key > base + qb + nr - 1) continue;  // no row of this block sees it
      const uint4 *kr = reinterpret_cast<const uint4 *>(
          kpool + ((static_cast<int64_t>(epage[e]) * Hkv + g) * P + slot) * D);
      float dot[QB][8];
#pragma unroll
      for (int r = 0; r < QB; ++r)
#pragma unroll
        for (int h = 0; h < 8; ++h) dot[r][h] = 0.f;
      for (int c = 0; c < D / 8; ++c) {
        const uint4 w = __ldg(kr + c);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        float kf[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = bf2_to_f2(ws[j]);
          kf[2 * j] = f.x;
          kf[2 * j + 1] = f.y;
        }
#pragma unroll
        for (int r = 0; r < QB; ++r) {
          if (r < nr) {
#pragma unroll
            for (int h = 0; h < 8; ++h) {
              if (h < G) {
                const uint4 qw = reinterpret_cast<const uint4 *>(qs + (r * Hq + g * G + h) * D)[c];
                const uint32_t qq[4] = {qw.x, qw.y, qw.z, qw.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float2 f = bf2_to_f2(qq[j]);
                  dot[r][h] = fmaf(f.x, kf[2 * j], fmaf(f.y, kf[2 * j + 1], dot[r][h]));
                }
              }
            }
          }
        }
      }
      float sum = 0.f;
#pragma unroll
      for (int r = 0; r < QB; ++r)
        if (r < nr && key <= base + qb + r)
#pragma unroll
          for (int h = 0; h < 8; ++h)
            if (h < G) sum += exp2f(dot[r][h] * scale_log2 - ls[r * Hq + g * G + h]);
      atomicAdd(&acc[e * 64 + slot], sum);
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ne * P; t += blockDim.x) {
    const int e = t / P, slot = t % P;
    const uint64_t m = emask[e];
    if ((m >> slot) & 1ull) out[d.out_off + elog[e] + __popcll(m & ((1ull << slot) - 1ull))] = acc[e * 64 + slot];
  }
}

size_t scores_smem_bytes(int Hq, int D) { return static_cast<size_t>(QB) * Hq * D * 2 + QB * Hq * 4; }

cudaError_t launch_scores(const ScoreUnit *units, int n_units, const ScoreDesc *descs, const Entry *slab,
                          const __nv_bfloat16 *q, const float *lse, const __nv_bfloat16 *kpool, float scale_log2,
                          float *out, int Hq, int Hkv, int D, int P, cudaStream_t s) {
  const size_t smem = scores_smem_bytes(Hq, D);
  static size_t attr = 0;
  if (smem > 48 * 1024 && attr < smem) {
    const cudaError_t e = cudaFuncSetAttribute(scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  scores_kernel<<<n_units, 256, smem, s>>>(units, descs, slab, q, lse, kpool, scale_log2, out, Hq, Hkv, D, P);
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace kvfs
