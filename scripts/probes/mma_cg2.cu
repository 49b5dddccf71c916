// Probe: tcgen05.mma.cta_group::2 (M=256 over a CTA pair) cost per instruction vs N, against
// the cta_group::1 M=128 form: does one pair-instruction double the rows per issue at small N?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2603_11441_b200/csrc -o mma_cg2 mma_cg2.cu
#include <cstdio>
#include "common.cuh"
using namespace dart;

__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N, int REPS>
__global__ void __cluster_dims__(2, 1, 1) k_cg2(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  const uint32_t rank = ctarank();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    const uint32_t idesc = umma_idesc_f16(256, N);
    long long t0 = 0;
    for (int rep = 0; rep < 2; ++rep) {
      t0 = clock64();
      for (int i = 0; i < REPS; ++i) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(umma_desc_sw128(a)), "l"(umma_desc_sw128(b)), "r"(idesc));
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                       smem_u32(&bar)), "h"((uint16_t)3) : "memory");
      mbar_wait(&bar, rep & 1);
    }
    out[blockIdx.x / 2] = clock64() - t0;
  } else if (threadIdx.x == 0) {
    mbar_wait(&bar, 0);
    mbar_wait(&bar, 1);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

template <typename K>
void run(const char* name, K kern, int reps, int pairs) {
  long long* d;
  cudaMalloc(&d, 296 * sizeof(long long));
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  kern<<<2 * pairs, 128, 64 * 1024>>>(d);
  kern<<<2 * pairs, 128, 64 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, d, sizeof(long long) * pairs, cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < pairs; ++i) m += h[i];
  m /= pairs;
  printf("%-36s %8.1f clk per instruction  (%s)\n", name, m / reps, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run("cg2 M256 N32 (74 pairs)", k_cg2<32, 256>, 256, 74);
  run("cg2 M256 N64 (74 pairs)", k_cg2<64, 256>, 256, 74);
  run("cg2 M256 N96 (74 pairs)", k_cg2<96, 256>, 256, 74);
  run("cg2 M256 N128 (74 pairs)", k_cg2<128, 256>, 256, 74);
  run("cg2 M256 N256 (74 pairs)", k_cg2<256, 256>, 256, 74);
  run("cg2 M256 N32 (148 pairs, 2/SM)", k_cg2<32, 256>, 256, 148);
  return 0;
}
