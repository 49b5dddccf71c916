// tcgen05.mma issue/pipe throughput probe for the small-N shapes of hd-16 attention.
// Each CTA (or CTA pair for cta_group::2) issues R back-to-back MMAs from one elected lane of
// warp 0 into TMEM (zero operands), then commits once and waits.  Reported: MMA instructions per
// clock per SM (all CTAs on an SM together) and clocks per instruction per issuing CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2603_11441_b200/csrc
//        -o mma_pipe mma_pipe.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace dart;

__device__ __forceinline__ uint64_t dsw32(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;
  return d;
}

__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// CG 1 or 2; TS: A operand from TMEM; CEVERY: a tcgen05.commit after every CEVERY MMAs (0: none)
template <int CG, int N, bool TS, int CEVERY>
__global__ void __launch_bounds__(128) mma_probe(int R, long long* clk) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 32768 + 64);
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  if (threadIdx.x < 32) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(slot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc<256>(slot);
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  const uint32_t tmem = *slot;
  const bool issuer = CG == 1 || ctarank() == 0;
  if (threadIdx.x < 32 && issuer) {
    constexpr uint32_t idesc = umma_idesc_f16(128 * CG, N);
    const uint64_t da = dsw32(smem_u32(smem)), db = dsw32(smem_u32(smem + 8192));
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
      if constexpr (CG == 1) {
        if constexpr (TS)
          umma_f16_ts_w(tmem, tmem + 128, db, idesc, 1);
        else
          umma_f16_w(tmem, da, db, idesc, 1);
        if (CEVERY && (r % (CEVERY ? CEVERY : 1)) == 0) umma_commit_w(&bar[1]);
      } else {
        if constexpr (TS)
          asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                       "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(tmem),
                       "r"(tmem + 128), "l"(db), "r"(idesc));
        else
          asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                       "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 1;\n\t}" ::"r"(tmem),
                       "l"(da), "l"(db), "r"(idesc));
      }
    }
    if constexpr (CG == 1) {
      umma_commit_w(&bar[0]);
    } else {
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
                       smem_u32(&bar[0])),
                   "h"((uint16_t)3)
                   : "memory");
    }
    long long t1 = clock64();
    mbar_wait(&bar[0], 0);
    long long t2 = clock64();
    if (threadIdx.x == 0) {
      clk[blockIdx.x * 2] = t1 - t0;
      clk[blockIdx.x * 2 + 1] = t2 - t0;
    }
  }
  if (CG == 2 && !issuer && threadIdx.x == 0) mbar_wait(&bar[0], 0);
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) {
    tc_fence_after();
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
    else
      tmem_dealloc<256>(tmem);
  }
}

template <int CG, int N, bool TS, int CEVERY>
void run(const char* name, int ctas_per_sm, long long* dclk) {
  auto k = mma_probe<CG, N, TS, CEVERY>;
  // smem per CTA forces the residency: 1 CTA/SM -> 120 KB, 2 -> 100 KB
  const int smem = ctas_per_sm == 1 ? 120 * 1024 : 100 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = 148 * ctas_per_sm;
  const int R = 4096;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, 16, dclk);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, R, dclk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[2 * 296];
  cudaMemcpy(h, dclk, sizeof(long long) * 2 * grid, cudaMemcpyDeviceToHost);
  double issue = 0, total = 0;
  int n = 0;
  for (int i = 0; i < grid; ++i)
    if (h[2 * i + 1] > 0) {
      issue += h[2 * i];
      total += h[2 * i + 1];
      ++n;
    }
  issue /= n;
  total /= n;
  const double issuers_per_sm = (double)n / 148.0;
  printf("%-34s ctas/SM %d  issue %6.1f clk/instr  complete %6.1f clk/instr/issuer  -> %5.1f clk per instr per SM   (%.3f ms, err %s)\n",
         name, ctas_per_sm, issue / R, total / R, total / R / issuers_per_sm, ms, cudaGetErrorString(cudaGetLastError()));
  cudaMemset(dclk, 0, sizeof(long long) * 2 * 296);
}

int main() {
  long long* dclk;
  cudaMalloc(&dclk, sizeof(long long) * 2 * 296);
  cudaMemset(dclk, 0, sizeof(long long) * 2 * 296);
  run<1, 32, false, 0>("cg1 M128 N32 SS", 1, dclk);
  run<1, 32, false, 0>("cg1 M128 N32 SS", 2, dclk);
  run<1, 32, true, 0>("cg1 M128 N32 TS", 1, dclk);
  run<1, 32, true, 0>("cg1 M128 N32 TS", 2, dclk);
  run<1, 96, false, 0>("cg1 M128 N96 SS", 1, dclk);
  run<1, 96, false, 0>("cg1 M128 N96 SS", 2, dclk);
  run<1, 256, false, 0>("cg1 M128 N256 SS", 1, dclk);
  run<1, 256, false, 0>("cg1 M128 N256 SS", 2, dclk);
  run<1, 32, true, 1>("cg1 M128 N32 TS + commit each", 1, dclk);
  run<1, 32, true, 1>("cg1 M128 N32 TS + commit each", 2, dclk);
  run<1, 32, true, 4>("cg1 M128 N32 TS + commit /4", 2, dclk);
  run<2, 32, false, 0>("cg2 M256 N32 SS", 1, dclk);
  run<2, 32, false, 0>("cg2 M256 N32 SS", 2, dclk);
  run<2, 32, true, 0>("cg2 M256 N32 TS", 1, dclk);
  run<2, 32, true, 0>("cg2 M256 N32 TS", 2, dclk);
  run<2, 96, false, 0>("cg2 M256 N96 SS", 2, dclk);
  run<2, 256, false, 0>("cg2 M256 N256 SS", 1, dclk);
  return 0;
}
