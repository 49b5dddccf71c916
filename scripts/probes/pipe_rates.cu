// Probe: per-SM issue rates of the softmax building blocks on this GPU (ex2.approx MUFU,
// FFMA2 packed, degree-3 exp2 polynomial on the FMA pipe, F2FP pack).  Reports
// results/clk/SM from clock64 deltas, 148 SMs x 8 warps/SMSP worth of threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rates pipe_rates.cu && ./pipe_rates
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

#define ITERS 4096
#define U 16

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint64_t pk(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__global__ void k_mufu(float* out, long long* cyc, float seed) {
  float v[U];
#pragma unroll
  for (int i = 0; i < U; ++i) v[i] = seed * (threadIdx.x + i) * -1e-3f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < U; ++i) v[i] = ex2(v[i]) - 1.0f;
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < U; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_mufu_only(float* out, long long* cyc, float seed) {
  // ex2 chain without the FADD: x -> ex2(x) -> ex2(...)  (values stay bounded in (0, 2])
  float v[U];
#pragma unroll
  for (int i = 0; i < U; ++i) v[i] = seed * (threadIdx.x + i) * -1e-3f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < U; ++i) v[i] = ex2(-v[i]);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < U; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma2(float* out, long long* cyc, float seed) {
  uint64_t v[U];
#pragma unroll
  for (int i = 0; i < U; ++i) v[i] = pk(seed + i, seed - i);
  const uint64_t a = pk(0.999f, 0.998f), b = pk(1e-3f, 2e-3f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < U; ++i) v[i] = ffma2(v[i], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < U; ++i) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(v[i]));
    s += x + y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma(float* out, long long* cyc, float seed) {
  float v[U];
#pragma unroll
  for (int i = 0; i < U; ++i) v[i] = seed + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < U; ++i) asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, 0f3A83126F;" : "+f"(v[i]));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < U; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_hfma2(float* out, long long* cyc, float seed) {
  __half2 v[U];
#pragma unroll
  for (int i = 0; i < U; ++i) v[i] = __floats2half2_rn(seed + i, seed - i);
  const __half2 a = __floats2half2_rn(0.999f, 0.998f), b = __floats2half2_rn(1e-3f, 2e-3f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < U; ++i) {
      uint32_t& r = reinterpret_cast<uint32_t&>(v[i]);
      asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(r) : "r"(reinterpret_cast<const uint32_t&>(a)),
                   "r"(reinterpret_cast<const uint32_t&>(b)));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < U; ++i) s += __low2float(v[i]) + __high2float(v[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_f2fp(float* out, long long* cyc, float seed) {
  float v[U];
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < U; ++i) v[i] = seed + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < U; i += 2) {
      uint32_t r;
      asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[i]), "f"(v[i + 1]));
      acc ^= r;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K>
void run(const char* name, K kern, double ops_per_iter_per_thread, int threads) {
  float* out;
  long long* cyc;
  const int blocks = 148;
  cudaMalloc(&out, blocks * threads * sizeof(float));
  cudaMalloc(&cyc, blocks * sizeof(long long));
  kern<<<blocks, threads>>>(out, cyc, 0.5f);
  kern<<<blocks, threads>>>(out, cyc, 0.5f);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < blocks; ++i) mean += h[i];
  mean /= blocks;
  const double ops = ops_per_iter_per_thread * ITERS * threads;
  printf("%-28s threads/SM %4d : %.2f results/clk/SM (%.0f clk)\n", name, threads, ops / mean, mean);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int t : {256, 512, 1024}) {
    run("ex2.approx.f32 + fadd", k_mufu, U, t);
    run("ex2.approx.f32 chain", k_mufu_only, U, t);
    run("fma.f32 (results)", k_ffma, U, t);
    run("fma.f32x2 (results=2/inst)", k_ffma2, 2 * U, t);
    run("fma.f16x2 (results=2/inst)", k_hfma2, 2 * U, t);
    run("cvt.f16x2.f32 (inst)", k_f2fp, U / 2, t);
  }
  return 0;
}
