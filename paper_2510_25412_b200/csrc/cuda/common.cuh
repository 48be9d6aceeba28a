// Shared device-side definitions: table entry / descriptor layouts (byte-identical to the host structs in
// csrc/host/kvfs_impl.h) and the sm_100a PTX helpers (mbarrier, 1-D TMA bulk copy, packed fp32x2 FMA).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace kvfs {
namespace dev {

struct Entry {  // == kvfs::Entry (the slab copy's lstart is not maintained: kernels must not read it)
  uint32_t page;
  int32_t lstart;
  uint64_t mask;
};

struct Desc {  // == kvfs::DevDesc
  int64_t cost_begin;
  int32_t slab_off;
  int32_t n_old_entries;
  int32_t n_old;
  int32_t n_q;
  int32_t row0;
  int32_t unit_base;
  int32_t stages_per_unit;
  int32_t n_entries;
  int32_t tail_lstart;
  int32_t first_new_entry;
  int32_t first_new_lstart;
  int32_t skip;         // leading entries attended by the shared-prefix kernel
  int32_t pref_splits;  // shared-prefix partials per unit (0: none)
  int32_t pref_base;    // partial of unit (g, qi), split s: pref_base + (g * n_q + qi) * pref_splits + s
  int64_t logit_off;    // >= 0: fused-scores logits of unit (g, qi), stage st, slot s, head h at
                        // logit_off + (((g * n_q + qi) * stages_per_unit + st) * P + s) * G + h; -1: none
  int64_t pad;
};

struct SlabRun {
  int64_t dst;
  int32_t src;
  int32_t count;
};

struct PageCopy {
  uint32_t src, dst;
};

// ------------------------------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_inval(uint32_t bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Same wait with a suspend-time hint (ns): the waiting thread sleeps in the barrier instead of
// re-issuing try_wait, which would steal issue slots from the warps sharing its SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITS_%=;\n\t}" ::"r"(bar),
      "r"(parity), "r"(1000000)
      : "memory");
}

// 1-D TMA: global -> shared, completion counted on an mbarrier (bytes multiple of 16, 16-B aligned).
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}

// 2-D tensor TMA: global -> shared (box of the map at coordinates (c0 innermost, c1)), L2 cache hint.
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void *map, int c0, int c1, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// TMA tile::gather4: rows r0..r3 (any order, repeats allowed) of a 2-D map with one-row boxes, columns from
// c0, into 4 consecutive box rows of shared memory; completion counted on the mbarrier
__device__ __forceinline__ void tma_gather4(uint32_t dst, const void *map, int c0, int r0, int r1, int r2, int r3,
                                            uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
      "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar), "l"(policy)
      : "memory");
}

// 4-byte global store with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void st_hint(float *a, float v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(policy) : "memory");
}

// Invalidate the 128-byte L2 line at a (128-byte aligned) WITHOUT writing it back: for dead data that was
// written and consumed inside L2 (the fused-scores logits), so it never costs DRAM write bandwidth.
__device__ __forceinline__ void discard_l2(const void *a) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// d += a * b on packed fp32 pairs (sm_100a FFMA2).
__device__ __forceinline__ void fma2(float2 &d, const float2 a, const float2 b) {
  unsigned long long dd = *reinterpret_cast<unsigned long long *>(&d);
  const unsigned long long aa = *reinterpret_cast<const unsigned long long *>(&a);
  const unsigned long long bb = *reinterpret_cast<const unsigned long long *>(&b);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dd) : "l"(aa), "l"(bb));
  d = *reinterpret_cast<float2 *>(&dd);
}

__device__ __forceinline__ float2 mul2(const float2 a, const float2 b) {
  unsigned long long dd;
  const unsigned long long aa = *reinterpret_cast<const unsigned long long *>(&a);
  const unsigned long long bb = *reinterpret_cast<const unsigned long long *>(&b);
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(dd) : "l"(aa), "l"(bb));
  return *reinterpret_cast<float2 *>(&dd);
}

__device__ __forceinline__ float2 add2(const float2 a, const float2 b) {
  unsigned long long dd;
  const unsigned long long aa = *reinterpret_cast<const unsigned long long *>(&a);
  const unsigned long long bb = *reinterpret_cast<const unsigned long long *>(&b);
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(dd) : "l"(aa), "l"(bb));
  return *reinterpret_cast<float2 *>(&dd);
}

__device__ __forceinline__ float2 sub2(const float2 a, const float2 b) {
  unsigned long long dd;
  const unsigned long long aa = *reinterpret_cast<const unsigned long long *>(&a);
  const unsigned long long bb = *reinterpret_cast<const unsigned long long *>(&b);
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dd) : "l"(aa), "l"(bb));
  return *reinterpret_cast<float2 *>(&dd);
}

// bf16 pair (little-endian u32: element 0 in the low half) -> fp32 pair, exact.
__device__ __forceinline__ float2 bf2_to_f2(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}

// acquire load at GPU scope (spin-waits on counters other CTAs release with __threadfence + atomics)
__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^a for a pair on the FMA/ALU pipes instead of MUFU (offloads the SFU in the tensor-core softmax):
// round-to-nearest split a = j + f (f in [-0.5, 0.5]) with the 1.5 * 2^23 trick, 2^f by a degree-3
// polynomial (relative error 7.7e-5, far below bf16's 2^-9 rounding of P), then j added to the exponent
// field: bits(r) << 23 == j << 23 (mod 2^32) because bits(1.5 * 2^23) << 23 == 0 (mod 2^32).
// Inputs are clamped at -126, so masked (-inf) columns give <= 2^-126 (not exactly 0; negligible).
__device__ __forceinline__ float2 exp2_poly2(float2 a) {
  a.x = fmaxf(a.x, -126.f);
  a.y = fmaxf(a.y, -126.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 r = add2(a, magic);
  const float2 f = sub2(a, sub2(r, magic));  // exact: r - magic is the integer j
  float2 q = make_float2(0.05508868f, 0.05508868f);
  float2 t = make_float2(0.24260405f, 0.24260405f);
  fma2(t, q, f);
  q = make_float2(0.6932762f, 0.6932762f);
  fma2(q, t, f);
  t = make_float2(0.99992895f, 0.99992895f);
  fma2(t, q, f);
  return make_float2(__uint_as_float((__float_as_uint(r.x) << 23) + __float_as_uint(t.x)),
                     __uint_as_float((__float_as_uint(r.y) << 23) + __float_as_uint(t.y)));
}

// Position of the r-th (0-based) set bit of m (precondition: popc(m) > r).
__device__ __forceinline__ int select_bit64(uint64_t m, int r) {
  const uint32_t lo = static_cast<uint32_t>(m);
  const int nlo = __popc(lo);
  if (r < nlo) return __fns(lo, 0, r + 1);
  return 32 + __fns(static_cast<uint32_t>(m >> 32), 0, r - nlo + 1);
}

// Keep the lowest k set bits of m.
__device__ __forceinline__ uint64_t lowest_bits(uint64_t m, int k) {
  if (k <= 0) return 0;
  if (k >= __popcll(m)) return m;
  const int s = select_bit64(m, k);  // position of the (k+1)-th set bit
  return m & ((1ull << s) - 1);
}

}  // namespace dev
}  // namespace kvfs
