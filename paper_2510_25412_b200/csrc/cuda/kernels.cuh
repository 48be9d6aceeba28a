// Kernel parameter blocks and launchers shared by csrc/cuda/*.cu.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace kvfs {
namespace dev {

// K1 workspace records per ring range (DecodeCfg::KDEF): 2 cut-unit pieces + 2 deferred whole units
constexpr int kDecodeRecSlots = 4;

// Floats of one partial record (o, m, l) of a unit's G heads: G (D + 2) rounded up to 16 bytes, so records
// can be moved by 1-D TMA bulk copies (head h at h (D + 2))
__host__ __device__ constexpr int part_floats(int G, int D) { return (G * (D + 2) + 3) & ~3; }
constexpr int kMaxPrefixSplits = 16;  // == kvfs::kMaxPrefixSplits (key splits of a shared prefix)

struct DecodeParams {
  const Desc *descs;
  int n_desc;
  int64_t total;  // total stages
  int ncta;       // chunks (virtual CTAs: contiguous stage ranges)
  int n_rings;    // physical rings launched (== ncta unless dynamic)
  int dynamic;    // 1: rings take chunks from the counter `work` (else ring r takes chunk r)
  int *work;      // [2] self-resetting counters (next chunk, finished rings)
  const Entry *slab;
  const int32_t *dst_slot;
  const __nv_bfloat16 *q, *k_new, *v_new;
  __nv_bfloat16 *out;
  float *lse;
  __nv_bfloat16 *kpool, *vpool;
  float scale_log2;  // scale * log2(e)
  float *partials;   // [ncta][kDecodeRecSlots][PART] (K1 records: range pieces, deferred whole units)
  const float *ppart;  // shared-prefix partials [..][PART] (Desc::pref_*)
  int wait_at_start;   // 1: griddepcontrol.wait before reading the tables (programmatic launch after the prologue)
  int *counters;     // [n_units]
  float *logits;     // fused scores: descriptors with logit_off >= 0 get their logits written here (else null)
  int Hq, Hkv;
  int gather;        // 1: holey page spans are fetched row by row with TMA gather4 (packed stage rows)
  // the layer's K / V pools as 2-D maps [n_pages * Hkv * P rows][D], box {D, 1}, no swizzle (gather4)
  alignas(64) CUtensorMap gk;
  alignas(64) CUtensorMap gv;
};

// pdl: programmatic dependent launch after the shared-prefix kernel (the kernel waits for it before merging)
cudaError_t launch_decode(const DecodeParams &p, int D, int G, int P, cudaStream_t s, bool pdl = false);
// ---- K2 (tcgen05 chunk attention, D = 128)
struct ChunkDesc {  // == kvfs::ChunkDesc
  int32_t slab_off, n_entries, n_old, n_q, row0, first_new_entry, first_new_lstart, pad;
};
struct ChunkUnit {  // == kvfs::ChunkUnit
  int32_t desc, g, m, group;
};
constexpr int kMaxPrefixGroups = 4096;  // == kvfs::kMaxPrefixGroups
struct PrefixDesc {  // == kvfs::PrefixDesc
  int32_t slab_off, n_entries, n_rows, row0, split, n_splits, q_t0, split_off;
};
struct PrefixRow {  // == kvfs::PrefixRow
  int32_t t, pref_base, n_q, qi;
};
struct ScoreDesc {  // == kvfs::ScoreDesc
  int32_t slab_off, n_q, row0, len_after;
  int64_t out_off;
};
struct ScoreUnit {  // == kvfs::ScoreUnit
  int32_t desc, e0, e1, l0;
};
struct LogitDesc {  // == kvfs::LogitDesc
  int64_t out_off, logit_off;
  int32_t slab_off, n_q, row0, n_old, n_old_entries, stages_per_unit;
  int32_t gather, pad;  // gather: the decode kernel packed holey page spans (DecodeParams::gather)
};
// Fused scores (K10): scores of the descriptors whose keys the decode kernel scored, from its logits.
cudaError_t launch_logit_scores(const ScoreUnit *units, int n_units, const LogitDesc *descs, const Entry *slab,
                                const float *logits, const float *lse, float *out, int Hq, int Hkv, int P,
                                cudaStream_t s);
// kmap: the layer's K pool as a 2-D map [n_pages * Hkv * P rows][D], box 64 dims x 16 rows, 128-byte swizzle
cudaError_t launch_scores(const CUtensorMap &kmap, const ScoreUnit *units, int n_units, const ScoreDesc *descs,
                          const Entry *slab, const __nv_bfloat16 *q, const float *lse, float scale_log2, float *out,
                          int Hq, int Hkv, int D, int P, cudaStream_t s);
struct ChunkParams {
  const ChunkUnit *units;
  const ChunkDesc *descs;
  const Entry *slab;
  __nv_bfloat16 *out;
  float *lse;
  float scale_log2;
  int P, Hkv, Hq;
  int pool_rows;  // n_pages * Hkv * P: a row coordinate out of the pool tensor (zero-filled TMA box)
  // shared-prefix mode only: units index pdescs; Q rows gathered through prows; partials -> ppart
  const PrefixDesc *pdescs;
  const PrefixRow *prows;
  const __nv_bfloat16 *q;
  float *ppart;
  int *pgroup;         // [2][kMaxPrefixGroups] arrival counters of the split groups, by launch parity
  int pgroup_parity;   // 0 / 1: this launch's counter array (the other one is cleared)
  const int2 *cta_units;  // prefix mode: per CTA (first unit, count), units run in turn; null: unit = CTA
};
cudaError_t launch_chunk(const CUtensorMap &km, const CUtensorMap &vm, const CUtensorMap &qm, const ChunkParams &p,
                         int n_units, int G, cudaStream_t s);
cudaError_t launch_scatter_rows(const int32_t *dst, int T, const __nv_bfloat16 *k, const __nv_bfloat16 *v,
                                __nv_bfloat16 *kp, __nv_bfloat16 *vp, int Hkv, int D, int P, int sms, cudaStream_t s);
int chunk_smem_bytes();
// Shared-prefix (cascade) attention: same kernel in prefix mode (no causal part, partial (O, m, l) output).
cudaError_t launch_prefix(const CUtensorMap &km, const CUtensorMap &vm, const CUtensorMap &qm, const ChunkParams &p,
                          int n_units, int G, cudaStream_t s);

// resident decode CTAs per SM for this shape (occupancy query; the default grid is SMs x this)
int decode_ctas_per_sm(int D, int G, int P);

}  // namespace dev
}  // namespace kvfs
