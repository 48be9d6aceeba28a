// Read-bandwidth probe for the decode kernel's memory pipeline design (not part of the library).
// Streams a 2 GiB buffer in 4 KiB "page-head" blocks through (a) a 1-D TMA bulk-copy ring in shared
// memory with mbarriers (the K1 design) at several ring depths / CTA counts, (b) plain LDG.128 loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe tools/bw_probe.cu && ./bw_probe
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_spin(uint32_t bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\n\tS_%=:\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra S_%=;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// mode 0: 1-D TMA bulk copies issued by lane 0 of each of NPW producer warps (stage i -> warp i % NPW)
// mode 1: cp.async 16-B copies by all 32 lanes of the producer warps, completion via cp.async.mbarrier.arrive
template <int NW, int NPW>
__global__ void __launch_bounds__((NW + NPW) * 32) tma_ring(const uint8_t *buf, int64_t n_blocks, int blk, int nstages,
                                                            int per_copy, int *sink, int mode) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)nstages * blk);
  uint64_t *empty = full + nstages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t per = (n_blocks + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = min(n_blocks, b0 + per);
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstages; ++s) { mbar_init(smem_u32(full + s), mode ? 32 : 1); mbar_init(smem_u32(empty + s), 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t n = b1 - b0;
  if (warp >= NW) {
    const int pw = warp - NW;
    if (mode == 0 && lane) return;
    for (int64_t i = pw; i < n; i += NPW) {
      const int slot = i % nstages;
      if (i >= nstages) mbar_wait(smem_u32(empty + slot), ((i / nstages) & 1) ^ 1);
      const int64_t b = b0 + i;
      const int64_t pb = (b % 8) * (n_blocks / 8) + b / 8;
      if (mode == 0) {
        mbar_expect(smem_u32(full + slot), blk);
        for (int o = 0; o < blk; o += per_copy)
          bulk(smem_u32(sm + (size_t)slot * blk + o), buf + pb * blk + o, per_copy, smem_u32(full + slot));
      } else {
        const uint32_t d = smem_u32(sm + (size_t)slot * blk);
        const uint8_t *src = buf + pb * blk;
        for (int o = lane * 16; o < blk; o += 512)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + o), "l"(src + o) : "memory");
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full + slot)) : "memory");
      }
    }
    return;
  }
  int acc = 0;
  for (int64_t i = warp; i < n; i += NW) {
    const int slot = i % nstages;
    mbar_wait(smem_u32(full + slot), (i / nstages) & 1);
    acc += reinterpret_cast<const int *>(sm + (size_t)slot * blk)[lane];
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(empty + slot));
  }
  if (acc == 0x12345678) sink[0] = acc;
}


// R independent rings in ONE CTA: ring r = producer warp r (lane 0 issues 1-D TMA) + CPR consumer warps.
template <int R, int CPR>
__global__ void __launch_bounds__(R * (CPR + 1) * 32) multi_ring(const uint8_t *buf, int64_t n_blocks, int blk,
                                                                  int nstages, int *sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = warp < R ? warp : (warp - R) / CPR;          // ring of this warp
  const int cw = warp < R ? -1 : (warp - R) % CPR;           // consumer index within the ring
  uint8_t *ring = sm + (size_t)r * nstages * blk;
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)R * nstages * blk) + r * 2 * nstages;
  uint64_t *empty = full + nstages;
  const int64_t nstream = (int64_t)gridDim.x * R;
  const int64_t stream = (int64_t)blockIdx.x * R + r;
  const int64_t per = (n_blocks + nstream - 1) / nstream;
  const int64_t b0 = stream * per, b1 = min(n_blocks, b0 + per);
  if (threadIdx.x == 0) {
    uint64_t *b = reinterpret_cast<uint64_t *>(sm + (size_t)R * nstages * blk);
    for (int s = 0; s < 2 * R * nstages; ++s) mbar_init(smem_u32(b + s), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t n = b1 - b0;
  if (warp < R) {
    if (lane) return;
    for (int64_t i = 0; i < n; ++i) {
      const int slot = i % nstages;
      if (i >= nstages) mbar_wait(smem_u32(empty + slot), ((i / nstages) & 1) ^ 1);
      const int64_t b = b0 + i;
      const int64_t pb = (b % 8) * (n_blocks / 8) + b / 8;
      mbar_expect(smem_u32(full + slot), blk);
      for (int o = 0; o < blk; o += 4096)
        bulk(smem_u32(ring + (size_t)slot * blk + o), buf + pb * blk + o, 4096, smem_u32(full + slot));
    }
    return;
  }
  int acc = 0;
  for (int64_t i = cw; i < n; i += CPR) {
    const int slot = i % nstages;
    mbar_wait(smem_u32(full + slot), (i / nstages) & 1);
    acc += reinterpret_cast<const int *>(ring + (size_t)slot * blk)[lane];
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(empty + slot));
  }
  if (acc == 0x12345678) sink[0] = acc;
}


// One ring; each stage's copies split across NPW producer warps (lanes [0, NL) of each issue a part).
// Stage i is fully issued by all producers before the next (all wait the same empty barrier).
template <int NPW, int NL>
__global__ void __launch_bounds__((NPW + 7) * 32) split_ring(const uint8_t *buf, int64_t n_blocks, int blk, int nstages,
                                                             int *sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)nstages * blk);
  uint64_t *empty = full + nstages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t per = (n_blocks + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = min(n_blocks, b0 + per);
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstages; ++s) { mbar_init(smem_u32(full + s), NPW * NL); mbar_init(smem_u32(empty + s), 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t n = b1 - b0;
  constexpr int NW = 7;
  if (warp >= NW) {
    const int pw = warp - NW;
    if (lane >= NL) return;
    const int part = pw * NL + lane, nparts = NPW * NL;
    for (int64_t i = 0; i < n; ++i) {
      const int slot = i % nstages;
      if (i >= nstages) mbar_wait(smem_u32(empty + slot), ((i / nstages) & 1) ^ 1);
      const int64_t b = b0 + i;
      const int64_t pb = (b % 8) * (n_blocks / 8) + b / 8;
      const int chunk = blk / nparts;
      mbar_expect(smem_u32(full + slot), chunk);
      bulk(smem_u32(sm + (size_t)slot * blk + part * chunk), buf + pb * blk + part * chunk, chunk, smem_u32(full + slot));
    }
    return;
  }
  int acc = 0;
  for (int64_t i = warp; i < n; i += NW) {
    const int slot = i % nstages;
    mbar_wait(smem_u32(full + slot), (i / nstages) & 1);
    acc += reinterpret_cast<const int *>(sm + (size_t)slot * blk)[lane];
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(empty + slot));
  }
  if (acc == 0x12345678) sink[0] = acc;
}

__global__ void ldg_stream(const int4 *buf, int64_t n16, int *sink) {
  int acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    int4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(buf + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
  }
  for (; i < n16; i += stride) acc ^= __ldcs(buf + i).x;
  if (acc == 0x12345678) sink[0] = acc;
}

int main(int argc, char **argv) {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  const int64_t bytes = 2ll << 30;
  uint8_t *buf;
  int *sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return bytes * 5 / (ms / 1e3) / 1e9;
  };
  if (only < 0)
    printf("ldg_stream (LDG.128 x8 unroll, 148x1024 thr): %.0f GB/s\n",
           timeit([&] { ldg_stream<<<148 * 2, 1024>>>((const int4 *)buf, bytes / 16, sink); }));
  if (only >= 200) {
    const int k = only - 200;
    const size_t smem = (size_t)16 * 8192 + 2 * 16 * 8;
    const int64_t nb = bytes / 8192;
    double gbs = 0;
    const char *name = "";
#define SR(NPW_, NL_)                                                                                        \
  cudaFuncSetAttribute(split_ring<NPW_, NL_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
  gbs = timeit([&] { split_ring<NPW_, NL_><<<148, (NPW_ + 7) * 32, smem>>>(buf, nb, 8192, 16, sink); }); \
  name = #NPW_ " producer warps x " #NL_ " lanes";
    switch (k) { case 0: SR(1, 1) break; case 1: SR(1, 4) break; case 2: SR(4, 1) break; case 3: SR(2, 2) break; case 4: SR(1, 8) break; }
    cudaError_t e = cudaGetLastError();
    printf("split_ring 16 x 8 KiB, %s: %.0f GB/s %s\n", name, gbs, e ? cudaGetErrorString(e) : "");
    return 0;
  }
  if (only >= 100) {
    const int k = only - 100;
    struct M { int R, CPR, nst, ctas; } ms[] = {{2, 3, 8, 1}, {3, 2, 8, 1}, {4, 2, 6, 1}, {4, 1, 6, 1}, {1, 1, 6, 4}, {2, 1, 6, 2}};
    M m = ms[k];
    const size_t smem = (size_t)m.R * m.nst * 8192 + m.R * 2 * m.nst * 8;
    const int64_t nb = bytes / 8192;
    double gbs = 0;
#define MR(R_, C_)                                                                                          \
  cudaFuncSetAttribute(multi_ring<R_, C_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
  gbs = timeit([&] { multi_ring<R_, C_><<<148 * m.ctas, R_ * (C_ + 1) * 32, smem>>>(buf, nb, 8192, m.nst, sink); });
    if (m.R == 2 && m.CPR == 3) { MR(2, 3) } else if (m.R == 3 && m.CPR == 2) { MR(3, 2) }
    else if (m.R == 4 && m.CPR == 2) { MR(4, 2) } else if (m.R == 4 && m.CPR == 1) { MR(4, 1) }
    else if (m.R == 1 && m.CPR == 1) { MR(1, 1) } else if (m.R == 2 && m.CPR == 1) { MR(2, 1) }
    cudaError_t e = cudaGetLastError();
    printf("multi_ring rings/CTA=%d consumers/ring=%d stages=%d ctas/sm=%d (%zu KiB/CTA): %.0f GB/s %s\n", m.R, m.CPR,
           m.nst, m.ctas, smem / 1024, gbs, e ? cudaGetErrorString(e) : "");
    return 0;
  }
  struct Cfg { int kind, blk, nst, ctas_per_sm, per_copy, mode; };
  // kind: 0 = <7,1>, 1 = <7,2>, 2 = <6,4>(4 producer warps), 3 = <4,1>, 4 = <7,1> cp.async, 5 = <6,2> cp.async
  std::vector<Cfg> cfgs = {{0, 8192, 16, 1, 4096, 0}, {1, 8192, 16, 1, 4096, 0}, {2, 8192, 16, 1, 4096, 0},
                           {3, 8192, 12, 2, 4096, 0}, {3, 8192, 8, 3, 4096, 0}, {0, 8192, 16, 1, 8192, 0},
                           {4, 8192, 16, 1, 0, 1}, {5, 8192, 16, 1, 0, 1}, {5, 8192, 24, 1, 0, 1},
                           {1, 8192, 24, 1, 8192, 0}, {2, 8192, 24, 1, 8192, 0}, {3, 8192, 6, 4, 8192, 0}};
  for (size_t ci = 0; ci < cfgs.size(); ++ci) {
    if (only >= 0 && (int)ci != only) continue;
    if (only < 0) break;
    auto c = cfgs[ci];
    const size_t smem = (size_t)c.nst * c.blk + 2 * c.nst * 8;
    const int64_t nb = bytes / c.blk;
    const int grid = 148 * c.ctas_per_sm;
    double gbs = 0;
    switch (c.kind) {
#define RUN(NW_, NPW_)                                                                                  \
  cudaFuncSetAttribute(tma_ring<NW_, NPW_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
  gbs = timeit([&] { tma_ring<NW_, NPW_><<<grid, (NW_ + NPW_) * 32, smem>>>(buf, nb, c.blk, c.nst, c.per_copy, sink, c.mode); });
      case 0: RUN(7, 1); break;
      case 1: RUN(7, 2); break;
      case 2: RUN(6, 4); break;
      case 3: RUN(4, 1); break;
      case 4: RUN(7, 1); break;
      case 5: RUN(6, 2); break;
    }
    cudaError_t e = cudaGetLastError();
    printf("kind=%d blk=%5d stages=%2d ctas/sm=%d per_copy=%5d mode=%d (%3zu KiB/SM): %.0f GB/s %s\n", c.kind, c.blk,
           c.nst, c.ctas_per_sm, c.per_copy, c.mode, smem * c.ctas_per_sm / 1024, gbs, e ? cudaGetErrorString(e) : "");
    if (e) break;
  }
  return 0;
}
