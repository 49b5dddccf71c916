#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
__global__ void k16(const float* in, uint32_t* out, int n, int iters) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  float a = in[i & 1023], b = in[(i + 7) & 1023];
  uint32_t acc = 0;
  uint32_t x[8];
  for (int k = 0; k < 8; ++k) { __half2 h = __floats2half2_rn(a + k * 0.01f, b - k * 0.01f); x[k] = *(uint32_t*)&h; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x[k]));
  }
  for (int k = 0; k < 8; ++k) acc ^= x[k];
  out[i] = acc;
}
__global__ void k32(const float* in, uint32_t* out, int n, int iters) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  float x[8];
  for (int k = 0; k < 8; ++k) x[k] = in[(i + k) & 1023];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[k]));
  }
  uint32_t acc = 0;
  for (int k = 0; k < 8; ++k) acc ^= __float_as_uint(x[k]);
  out[i] = acc;
}
__global__ void kbf(const float* in, uint32_t* out, int n, int iters) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t x[8];
  for (int k = 0; k < 8; ++k) x[k] = __float_as_uint(in[(i + k) & 1023]);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x[k]));
  }
  uint32_t acc = 0;
  for (int k = 0; k < 8; ++k) acc ^= x[k];
  out[i] = acc;
}
// cvt f32x2 -> f16x2 + ex2 f16x2 (the realistic softmax sequence)
__global__ void kseq(const float* in, uint32_t* out, int n, int iters) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  float v[16];
  for (int k = 0; k < 16; ++k) v[k] = in[(i + k) & 1023];
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t h;
      float a = fmaf(v[2*k], 1.01f, -0.5f), b = fmaf(v[2*k+1], 1.01f, -0.5f);
      asm volatile("cvt.rn.f16x2.f32 %0, %2, %1;" : "=r"(h) : "f"(a), "f"(b));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h));
      acc += h;
      v[2*k] = a; v[2*k+1] = b;
    }
  }
  out[i] = acc;
}
int main() {
  float* in; uint32_t* out;
  cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096*4);
  int blocks = 148 * 8, threads = 256, iters = 4096;
  cudaMalloc(&out, blocks * threads * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  auto run = [&](const char* name, void (*k)(const float*, uint32_t*, int, int), double per_instr) {
    k<<<blocks, threads>>>(in, out, 0, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(in, out, 0, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double instr = (double)blocks * threads * iters * 8;
    double per_s = instr / (ms * 1e-3);
    printf("%-10s %.3f ms  %.3f Tinstr/s  %.3f Tresults/s  (%.2f instr/clk/SM at %d MHz nominal)\n", name, ms, per_s / 1e12,
           per_s * per_instr / 1e12, per_s / 148 / (clk * 1e3), clk / 1000);
  };
  run("ex2.f32", k32, 1); run("ex2.f16x2", k16, 2); run("ex2.bf16x2", kbf, 2); run("cvt+ex2h2", kseq, 2);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
