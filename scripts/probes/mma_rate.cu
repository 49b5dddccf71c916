// Probe: tcgen05.mma issue-to-completion cost vs N (M=128, K=16, kind::f16), SS and TS forms,
// and the commit -> mbarrier -> thread -> mbarrier -> issuer round trip.  One CTA per SM;
// smem operands are zero-filled (values do not matter).  Reports clk per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2603_11441_b200/csrc -o mma_rate mma_rate.cu
#include <cstdio>
#include "common.cuh"
using namespace dart;

template <int N, bool TS, int REPS>
__global__ void k_mma(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    const uint32_t idesc = umma_idesc_f16(128, N);
    long long t0 = 0;
    for (int rep = 0; rep < 2; ++rep) {
      t0 = clock64();
      for (int i = 0; i < REPS; ++i) {
        if (TS)
          umma_f16_ts(tmem, tmem + 256, umma_desc_sw128(b), idesc, 1);
        else
          umma_f16(tmem, umma_desc_sw128(a), umma_desc_sw128(b), idesc, 1);
      }
      umma_commit(&bar);
      mbar_wait(&bar, rep & 1);
    }
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// round trip: issuer does one small MMA + commit(bar0); warp 1 waits bar0, arrives bar1;
// issuer waits bar1.  REPS iterations.
template <int REPS>
__global__ void k_roundtrip(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar0, bar1;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar0, 1);
    mbar_init(&bar1, 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    long long t0 = clock64();
    for (int i = 0; i < REPS; ++i) {
      umma_f16(tmem, umma_desc_sw128(a), umma_desc_sw128(b), umma_idesc_f16(128, 32), 1);
      umma_commit(&bar0);
      mbar_wait(&bar1, i & 1);
      tc_fence_after();
    }
    out[blockIdx.x] = clock64() - t0;
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < REPS; ++i) {
      mbar_wait(&bar0, i & 1);
      tc_fence_after();
      mbar_arrive(&bar1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <typename K>
void run(const char* name, K kern, int reps) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  kern<<<148, 128, 64 * 1024>>>(d);
  kern<<<148, 128, 64 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148; ++i) m += h[i];
  m /= 148;
  printf("%-34s %8.1f clk per op  (%s)\n", name, m / reps, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run("SS M128 N32  K16", k_mma<32, false, 256>, 256);
  run("SS M128 N64  K16", k_mma<64, false, 256>, 256);
  run("SS M128 N96  K16", k_mma<96, false, 256>, 256);
  run("SS M128 N128 K16", k_mma<128, false, 256>, 256);
  run("SS M128 N256 K16", k_mma<256, false, 256>, 256);
  run("TS M128 N32  K16", k_mma<32, true, 256>, 256);
  run("TS M128 N64  K16", k_mma<64, true, 256>, 256);
  run("TS M128 N96  K16", k_mma<96, true, 256>, 256);
  run("TS M128 N128 K16", k_mma<128, true, 256>, 256);
  run("TS M128 N256 K16", k_mma<256, true, 256>, 256);
  run("SS N32 x1 (latency incl commit)", k_mma<32, false, 1>, 1);
  run("SS N96 x8 (commit incl)", k_mma<96, false, 8>, 8);
  run("roundtrip mma+commit->wait->arrive", k_roundtrip<256>, 256);
  return 0;
}
