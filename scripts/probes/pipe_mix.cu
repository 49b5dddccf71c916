// Throughput of the softmax instruction classes alone and mixed (per SM per clock):
// MUFU.EX2, F2FP.F16.F32.PACK_AB (cvt.rn.f16x2.f32), FFMA2, and MUFU+F2FP / MUFU+FFMA2 mixes.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KIND>
__global__ void k(const float* in, uint32_t* out, int iters) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  float x[8];
  uint32_t h[8];
  uint64_t d[8];
  for (int j = 0; j < 8; ++j) {
    x[j] = in[(i + j) & 1023];
    h[j] = __float_as_uint(x[j]);
    d[j] = ((uint64_t)h[j] << 32) | h[j];
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (KIND == 0 || KIND == 3 || KIND == 4) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[j]));
      if (KIND == 1 || KIND == 3) asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h[j]) : "f"(x[j]), "f"(__uint_as_float(h[j])));
      if (KIND == 2 || KIND == 4) {
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(d[j]));
      }
    }
  }
  uint32_t acc = 0;
  for (int j = 0; j < 8; ++j) acc ^= __float_as_uint(x[j]) ^ h[j] ^ (uint32_t)d[j];
  out[i] = acc;
}

template <int KIND>
void run(const char* name, const float* in, uint32_t* out, int ninstr) {
  const int blocks = 148 * 8, threads = 256, iters = 2048;
  k<KIND><<<blocks, threads>>>(in, out, 8);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<KIND><<<blocks, threads>>>(in, out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warp_instr = (double)blocks * threads / 32 * iters * 8 * ninstr;
  const double clk = ms * 1e-3 * 1.965e9;  // nominal max clock
  printf("%-22s %.3f ms  %.3f warp-instr/clk/SM (x32 = %.1f thread-instr/clk/SM)\n", name, ms, warp_instr / clk / 148,
         32 * warp_instr / clk / 148);
}

int main() {
  float* in;
  uint32_t* out;
  cudaMalloc(&in, 4096 * 4);
  cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  run<0>("MUFU.EX2", in, out, 1);
  run<1>("F2FP pack", in, out, 1);
  run<2>("FFMA2", in, out, 1);
  run<3>("MUFU + F2FP (1:1)", in, out, 2);
  run<4>("MUFU + FFMA2 (1:1)", in, out, 2);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
