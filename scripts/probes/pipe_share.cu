// Which softmax instruction classes share an execution pipe on sm_100a: each kernel issues a
// fixed mix from 8 independent chains per thread at full occupancy; the rate (thread-instr /
// clk / SM, nominal 1.965 GHz) of a mix against its parts' rates alone tells whether they
// overlap (rate adds) or share a pipe (time adds).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_share pipe_share.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define OP_EX2(x) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x))
#define OP_F2FP(h, x) asm volatile("cvt.rn.f16x2.f32 %0, %1, %0;" : "+r"(h) : "f"(x))
#define OP_FFMA2(d) asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(d))
#define OP_FADD2(d) asm volatile("add.rn.f32x2 %0, %0, %0;" : "+l"(d))
#define OP_FFMA(x) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(x))
#define OP_FFMAS(x) asm volatile("fma.rn.sat.f32 %0, %0, %0, %0;" : "+f"(x))
#define OP_IMAD(u) asm volatile("mad.lo.u32 %0, %0, %0, %0;" : "+r"(u))
#define OP_IADD(u) asm volatile("add.u32 %0, %0, 7;" : "+r"(u))
#define OP_LEA(u, v) asm volatile("{.reg .u32 t; shl.b32 t, %1, 23; add.u32 %0, %0, t;}" : "+r"(u) : "r"(v))
#define OP_MAX3(x) asm volatile("max.f32 %0, %0, %0, %0;" : "+f"(x))
#define OP_HFMA2(u) asm volatile("fma.rn.f16x2 %0, %0, %0, %0;" : "+r"(u))
#define OP_PRMT(u, v) asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(u) : "r"(v))

// KIND bit flags: which ops one iteration of a chain issues
enum { EX2 = 1, F2FP = 2, FFMA2 = 4, FADD2 = 8, FFMA = 16, FFMAS = 32, IMAD = 64, IADD = 128, LEA = 256,
       MAX3 = 512, HFMA2 = 1024, PRMT = 2048, EX2x2 = 4096 };

template <int KIND>
__global__ void k(const float* in, uint32_t* out, int iters) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  float x[8], y[8], z[8];
  uint32_t h[8], u[8], w[8];
  uint64_t d[8], e[8];
  for (int j = 0; j < 8; ++j) {
    x[j] = in[(i + j) & 1023];
    y[j] = x[j] + 1.f;
    z[j] = x[j] + 2.f;
    h[j] = __float_as_uint(x[j]);
    u[j] = h[j] ^ 5;
    w[j] = h[j] ^ 9;
    d[j] = ((uint64_t)h[j] << 32) | h[j];
    e[j] = d[j] ^ 3;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (KIND & EX2) OP_EX2(x[j]);
      if (KIND & EX2x2) OP_EX2(z[j]);
      if (KIND & F2FP) OP_F2FP(h[j], y[j]);
      if (KIND & FFMA2) OP_FFMA2(d[j]);
      if (KIND & FADD2) OP_FADD2(e[j]);
      if (KIND & FFMA) OP_FFMA(y[j]);
      if (KIND & FFMAS) OP_FFMAS(z[j]);
      if (KIND & IMAD) OP_IMAD(u[j]);
      if (KIND & IADD) OP_IADD(w[j]);
      if (KIND & LEA) OP_LEA(w[j], u[j]);
      if (KIND & MAX3) OP_MAX3(y[j]);
      if (KIND & HFMA2) OP_HFMA2(u[j]);
      if (KIND & PRMT) OP_PRMT(h[j], w[j]);
    }
  }
  uint32_t acc = 0;
  for (int j = 0; j < 8; ++j)
    acc ^= __float_as_uint(x[j]) ^ __float_as_uint(y[j]) ^ __float_as_uint(z[j]) ^ h[j] ^ u[j] ^ w[j] ^
           (uint32_t)d[j] ^ (uint32_t)e[j];
  out[i] = acc;
}

template <int KIND>
void run(const char* name, const float* in, uint32_t* out) {
  const int ninstr = __builtin_popcount(KIND);
  const int blocks = 148 * 8, threads = 256, iters = 2048;
  k<KIND><<<blocks, threads>>>(in, out, 8);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k<KIND><<<blocks, threads>>>(in, out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double per_thread_iter = (double)blocks * threads * iters * 8;  // one chain step
  const double clk = best * 1e-3 * 1.965e9;
  printf("%-28s %7.3f ms  %6.1f chain-steps/clk/SM  %6.1f thread-instr/clk/SM\n", name, best,
         per_thread_iter / clk / 148, ninstr * per_thread_iter / clk / 148);
}

int main() {
  float* in;
  uint32_t* out;
  cudaMalloc(&in, 4096 * 4);
  cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  run<EX2>("MUFU.EX2", in, out);
  run<F2FP>("F2FP", in, out);
  run<FFMA2>("FFMA2", in, out);
  run<FADD2>("FADD2", in, out);
  run<FFMA>("FFMA", in, out);
  run<FFMAS>("FFMA.SAT", in, out);
  run<IMAD>("IMAD", in, out);
  run<IADD>("IADD", in, out);
  run<LEA>("SHL+ADD (LEA?)", in, out);
  run<MAX3>("FMNMX3", in, out);
  run<HFMA2>("HFMA2", in, out);
  run<PRMT>("PRMT", in, out);
  run<FFMA2 | F2FP>("FFMA2+F2FP", in, out);
  run<FFMA | F2FP>("FFMA+F2FP", in, out);
  run<FFMA2 | FFMA>("FFMA2+FFMA", in, out);
  run<FFMA2 | IMAD>("FFMA2+IMAD", in, out);
  run<FFMA2 | IADD>("FFMA2+IADD", in, out);
  run<FFMA2 | LEA>("FFMA2+LEA", in, out);
  run<FFMA | IADD>("FFMA+IADD", in, out);
  run<F2FP | IADD>("F2FP+IADD", in, out);
  run<F2FP | PRMT>("F2FP+PRMT", in, out);
  run<FFMA2 | HFMA2>("FFMA2+HFMA2", in, out);
  run<FFMA | HFMA2>("FFMA+HFMA2", in, out);
  run<F2FP | HFMA2>("F2FP+HFMA2", in, out);
  run<FFMA2 | MAX3>("FFMA2+FMNMX3", in, out);
  run<EX2 | FFMA2 | F2FP>("EX2+FFMA2+F2FP", in, out);
  run<EX2 | EX2x2 | FFMA2 | F2FP>("2EX2+FFMA2+F2FP", in, out);
  run<EX2 | FFMA2 | FADD2 | F2FP | IADD>("EX2+FFMA2+FADD2+F2FP+IADD", in, out);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
