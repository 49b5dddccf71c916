// Probe: latency of mbarrier waits on an ALREADY COMPLETED phase (try_wait with / without a
// suspend-time hint, test_wait), as seen by one thread (clock64 around each wait).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2603_11441_b200/csrc -o mbar_lat mbar_lat.cu
#include <cstdio>
#include "common.cuh"
using namespace dart;

__device__ __forceinline__ void wait_hint(uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); }
__device__ __forceinline__ void wait_nohint(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra W_%=;\n\t}" ::"r"(addr), "r"(parity) : "memory");
}
__device__ __forceinline__ void wait_test(uint64_t* bar, uint32_t parity) { mbar_spin(bar, parity); }

template <int MODE>
__global__ void k(long long* out) {
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    mbar_arrive(&bar);  // phase 0 complete
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int i = 0; i < 1000; ++i) {
      const long long t0 = clock64();
      if (MODE == 0) wait_hint(&bar, 0);
      if (MODE == 1) wait_nohint(&bar, 0);
      if (MODE == 2) wait_test(&bar, 0);
      const long long t1 = clock64();
      tot += t1 - t0;
    }
    out[blockIdx.x] = tot / 1000;
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  long long h[148];
  const char* names[3] = {"try_wait + suspend hint (mbar_wait)", "try_wait, no hint", "test_wait spin (mbar_spin)"};
  for (int m = 0; m < 3; ++m) {
    if (m == 0) k<0><<<148, 64>>>(d);
    if (m == 1) k<1><<<148, 64>>>(d);
    if (m == 2) k<2><<<148, 64>>>(d);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-40s %lld clk per completed-phase wait\n", names[m], h[0]);
  }
  return 0;
}
