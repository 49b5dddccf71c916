// Which blocks share an SM when a persistent kernel runs 2 CTAs per SM (grid = 2 x SMs)?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void place(int* out) {
  extern __shared__ char s[];
  unsigned smid, wid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  if (threadIdx.x % 32 == 0) out[blockIdx.x * 8 + threadIdx.x / 32] = (int)(smid * 100 + wid);
  s[threadIdx.x] = 0;
  long long t = clock64();
  while (clock64() - t < 200000) {}
}
int main() {
  int* d;
  const int grid = 296;
  cudaMalloc(&d, grid * 8 * 4);
  cudaFuncSetAttribute(place, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  place<<<grid, 192, 100 * 1024>>>(d);
  int h[296 * 8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  int same_half = 0, pairs = 0;
  for (int b = 0; b < grid; ++b)
    for (int c = b + 1; c < grid; ++c)
      if (h[b * 8] / 100 == h[c * 8] / 100) {
        ++pairs;
        same_half += (b * 2 >= grid) == (c * 2 >= grid);
        if (pairs <= 6) printf("blocks %d and %d share SM %d; warpids %d..%d and %d..%d\n", b, c, h[b * 8] / 100,
                               h[b * 8] % 100, h[b * 8 + 5] % 100, h[c * 8] % 100, h[c * 8 + 5] % 100);
      }
  printf("%d SM-sharing pairs, %d with both blocks in the same grid half (role swap ineffective for them)\n", pairs, same_half);
  return 0;
}
