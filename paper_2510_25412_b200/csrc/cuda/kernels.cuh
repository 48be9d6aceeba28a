// Kernel parameter blocks and launchers shared by csrc/cuda/*.cu.
#pragma once
#include "common.cuh"

namespace kvfs {
namespace dev {

struct DecodeParams {
  const Desc *descs;
  int n_desc;
  int64_t total;  // total stages
  int ncta;
  const Entry *slab;
  const int32_t *dst_slot;
  const __nv_bfloat16 *q, *k_new, *v_new;
  __nv_bfloat16 *out;
  float *lse;
  __nv_bfloat16 *kpool, *vpool;
  float scale_log2;  // scale * log2(e)
  float *partials;   // [ncta][2][PART]
  int *counters;     // [n_units]
  int Hq, Hkv;
};

cudaError_t launch_decode(const DecodeParams &p, int D, int G, int P, cudaStream_t s);
// resident decode CTAs per SM for this shape (occupancy query; the default grid is SMs x this)
int decode_ctas_per_sm(int D, int G, int P);

}  // namespace dev
}  // namespace kvfs
