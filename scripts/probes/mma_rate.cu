// Probe: tcgen05.mma issue-to-completion cost vs N (M=128, K=16, kind::f16), SS and TS forms,
// and the commit -> mbarrier -> thread -> mbarrier -> issuer round trip.  One CTA per SM;
// smem operands are zero-filled (values do not matter).  Reports clk per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2603_11441_b200/csrc -o mma_rate mma_rate.cu
#include <cstdio>
#include "common.cuh"
using namespace dart;

__device__ __forceinline__ uint64_t desc_sw32(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;
  return d;
}
// MODE 0: SW128 K-major (GEMM form); 1: SW32 K-major A and B (attention S = Q K^T form);
// 2: TS A from TMEM, B SW32 MN-major (attention P.V form, B = V with LBO = BKV*32)
template <int N, int MODE, int REPS>
__global__ void k_mma_attn(long long* out) {
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
    const uint32_t idesc = umma_idesc_f16(128, N) | (MODE == 2 ? (1u << 16) : 0u);
    long long t0 = 0;
    for (int rep = 0; rep < 2; ++rep) {
      t0 = clock64();
      for (int i = 0; i < REPS; ++i) {
        if (MODE == 0)
          umma_f16(tmem, umma_desc_sw128(a), umma_desc_sw128(b), idesc, 1);
        else if (MODE == 1)
          umma_f16(tmem, desc_sw32(a, 16, 256), desc_sw32(b, 16, 256), idesc, 1);
        else
          umma_f16_ts(tmem, tmem + 384, desc_sw32(b, 96 * 32, 256), idesc, 1);
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

// commit cost: every MMA followed by NC commits to (distinct) barriers nobody waits on
template <int N, int NC, int REPS>
__global__ void k_commit(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, sink[4];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&sink[i], 1 << 20);
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
        umma_f16(tmem, umma_desc_sw128(a), umma_desc_sw128(b), idesc, 1);
        for (int c = 0; c < NC; ++c) umma_commit(&sink[c]);
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

// attention tile pattern: NPV P.V-form MMAs (TS, N=32, B MN-major SW32) + 1 S-form (SS, N=96,
// SW32) per "tile", REPS tiles; TMEM 256 columns so two CTAs can share an SM.
template <int NPV, int REPS, int COMMITS>
__global__ void k_tile(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, sink[4];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&sink[i], 1 << 20);
    fence_barrier_init();
  }
  fence_proxy_async();
  if (threadIdx.x < 32) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    const uint32_t id_pv = umma_idesc_f16(128, 32) | (1u << 16), id_s = umma_idesc_f16(128, 96);
    long long t0 = 0;
    for (int rep = 0; rep < 2; ++rep) {
      t0 = clock64();
      for (int i = 0; i < REPS; ++i) {
        for (int k = 0; k < NPV; ++k) umma_f16_ts(tmem + 192, tmem + k * 8, desc_sw32(b, 96 * 32, 256), id_pv, 1);
        for (int c = 0; c < COMMITS / 2; ++c) umma_commit(&sink[c]);
        umma_f16(tmem + (i & 1) * 96, desc_sw32(a, 16, 256), desc_sw32(b, 16, 256), id_s, 0);
        for (int c = COMMITS / 2; c < COMMITS; ++c) umma_commit(&sink[c]);
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
    tmem_dealloc<256>(tmem);
  }
}

// k_tile plus the real kernel's per-tile overheads: WAITS mbarrier waits on already-completed
// barriers and FENCE tcgen05.fence::after_thread_sync before each MMA group
template <int REPS, int WAITS, int FENCE>
__global__ void k_tile_sync(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, done;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&done, 1);
    fence_barrier_init();
    mbar_arrive(&done);  // phase 0 complete
  }
  fence_proxy_async();
  if (threadIdx.x < 32) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    const uint32_t id_pv = umma_idesc_f16(128, 32) | (1u << 16), id_s = umma_idesc_f16(128, 96);
    long long t0 = 0;
    for (int rep = 0; rep < 2; ++rep) {
      t0 = clock64();
      for (int i = 0; i < REPS; ++i) {
        for (int w = 0; w < WAITS; ++w) mbar_wait(&done, 0);
        if (FENCE) tc_fence_after();
        for (int k = 0; k < 6; ++k) umma_f16_ts(tmem + 192, tmem + k * 8, desc_sw32(b, 96 * 32, 256), id_pv, 1);
        for (int w = 0; w < WAITS; ++w) mbar_wait(&done, 0);
        if (FENCE) tc_fence_after();
        umma_f16(tmem + (i & 1) * 96, desc_sw32(a, 16, 256), desc_sw32(b, 16, 256), id_s, 0);
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
    tmem_dealloc<256>(tmem);
  }
}

template <int N, bool TS, int REPS, int NACC = 1>
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
        const uint32_t d = tmem + (uint32_t)((i % NACC) * N);
        if (TS)
          umma_f16_ts(d, tmem + 384, umma_desc_sw128(b), idesc, 1);
        else
          umma_f16(d, umma_desc_sw128(a), umma_desc_sw128(b), idesc, 1);
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


// Latency of an mbarrier wait on an ALREADY COMPLETED phase issued right after NMMA async
// MMAs (+ NCOMMIT commits to another barrier): does pending tensor work slow the wait?
template <int NMMA, int NCOMMIT, int REPS>
__global__ void k_wait_after_mma(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, done, sink;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&done, 1);
    mbar_init(&sink, 1);
    fence_barrier_init();
    mbar_arrive(&done);  // phase 0 of `done` complete
  }
  fence_proxy_async();
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    const uint32_t idesc = umma_idesc_f16(128, 32);
    long long tot = 0;
    for (int i = 0; i < REPS; ++i) {
      for (int m = 0; m < NMMA; ++m) umma_f16(tmem, umma_desc_sw128(a), umma_desc_sw128(b), idesc, 1);
      for (int c = 0; c < NCOMMIT; ++c) umma_commit(&sink);
      const long long t0 = clock64();
      mbar_wait(&done, 0);
      tot += clock64() - t0;
      umma_commit(&bar);  // drain before the next round
      mbar_wait(&bar, i & 1);
    }
    out[blockIdx.x] = tot * 64 / REPS;  // run() divides by its reps argument (64)
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}


// The attention MMA-alone protocol in isolation (no TMA, no softmax math): warp 0 issues
// S(g) = 1 MMA (N=96) and P.V(g) = 6 TS MMAs (N=32) per tile with NS S buffers; NSOFT
// "softmax" warps wait S-ready, fence and arrive P-ready.  EXTRA extra commits per tile
// (the kernel's non-LEAN stage releases).  Reports clk per tile.
template <int NS, int NSOFT, int EXTRA, int TILES>
__global__ void k_pingpong(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t s_full[NS], p_full[NS], sink;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], NSOFT);
    }
    mbar_init(&sink, 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  if (threadIdx.x < 32) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    const uint32_t id_pv = umma_idesc_f16(128, 32) | (1u << 16), id_s = umma_idesc_f16(128, 96);
    const long long t0 = clock64();
    for (int g = 0; g < NS; ++g) {
      umma_f16_w(tmem + g * 96, desc_sw32(a, 16, 256), desc_sw32(b, 16, 256), id_s, 0);
      umma_commit_w(&s_full[g]);
    }
    for (int g = 0; g < TILES; ++g) {
      mbar_wait(&p_full[g % NS], (g / NS) & 1);
      tc_fence_after();
      for (int k = 0; k < 6; ++k)
        umma_f16_ts_w(tmem + NS * 96, tmem + (g % NS) * 96 + k * 8, desc_sw32(b, 96 * 32, 256), id_pv, 1);
      for (int c = 0; c < EXTRA; ++c) umma_commit_w(&sink);
      if (g + NS < TILES) {
        umma_f16_w(tmem + (g % NS) * 96, desc_sw32(a, 16, 256), desc_sw32(b, 16, 256), id_s, 0);
        umma_commit_w(&s_full[g % NS]);
      }
    }
    umma_commit_w(&sink);
    if (lane == 0) out[blockIdx.x] = (clock64() - t0) * 64 / TILES;  // run() divides by 64
  } else if (warp <= NSOFT) {
    for (int g = 0; g < TILES; ++g) {
      mbar_wait(&s_full[g % NS], (g / NS) & 1);
      tc_fence_after();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[g % NS]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

template <typename K>
void run(const char* name, K kern, int reps, int blocks = 148, int threads = 128) {
  long long* d;
  cudaMalloc(&d, 296 * sizeof(long long));
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  kern<<<blocks, threads, 64 * 1024>>>(d);
  kern<<<blocks, threads, 64 * 1024>>>(d);
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
  run("pingpong NS2 soft1 extra0 1CTA", k_pingpong<2, 1, 0, 256>, 64, 148, 64);
  run("pingpong NS2 soft4 extra0 1CTA", k_pingpong<2, 4, 0, 256>, 64, 148, 160);
  run("pingpong NS2 soft4 extra3 1CTA", k_pingpong<2, 4, 3, 256>, 64, 148, 160);
  run("pingpong NS2 soft4 extra3 2CTA", k_pingpong<2, 4, 3, 256>, 64, 296, 160);
  run("pingpong NS3 soft4 extra3 1CTA", k_pingpong<3, 4, 3, 256>, 64, 148, 160);
  run("wait(completed) after 0 MMA", k_wait_after_mma<0, 0, 64>, 64);
  run("wait(completed) after 1 MMA", k_wait_after_mma<1, 0, 64>, 64);
  run("wait(completed) after 6 MMA", k_wait_after_mma<6, 0, 64>, 64);
  run("wait(completed) after 1 MMA+1 commit", k_wait_after_mma<1, 1, 64>, 64);
  run("wait(completed) after 6 MMA+2 commits", k_wait_after_mma<6, 2, 64>, 64);
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
  run("tile+sync W0 F1 2CTA", k_tile_sync<64, 0, 1>, 64, 296);
  run("tile+sync W1 F0 2CTA", k_tile_sync<64, 1, 0>, 64, 296);
  run("tile+sync W1 F1 2CTA", k_tile_sync<64, 1, 1>, 64, 296);
  run("tile+sync W1 F1 1CTA", k_tile_sync<64, 1, 1>, 64, 148);
  run("tile+sync W2 F1 2CTA", k_tile_sync<64, 2, 1>, 64, 296);
  run("tile 6PV+1S, 1 CTA/SM", k_tile<6, 64, 0>, 64);
  run("tile 6PV+1S, 2 CTA/SM", k_tile<6, 64, 0>, 64, 296);
  run("tile 6PV+1S+4commits, 1 CTA/SM", k_tile<6, 64, 4>, 64);
  run("tile 6PV+1S+4commits, 2 CTA/SM", k_tile<6, 64, 4>, 64, 296);
  run("tile 6PV+1S+2commits, 2 CTA/SM", k_tile<6, 64, 2>, 64, 296);
  run("N32 MMA + 1 commit", k_commit<32, 1, 256>, 256);
  run("N32 MMA + 2 commits", k_commit<32, 2, 256>, 256);
  run("N32 MMA + 4 commits", k_commit<32, 4, 256>, 256);
  run("N256 MMA + 1 commit", k_commit<256, 1, 256>, 256);
  run("attn S form SW32 N96", k_mma_attn<96, 1, 256>, 256);
  run("attn S form SW32 N64", k_mma_attn<64, 1, 256>, 256);
  run("attn PV form TS SW32 MN N32", k_mma_attn<32, 2, 256>, 256);
  run("attn PV form TS SW32 MN N96", k_mma_attn<96, 2, 256>, 256);
  run("TS M128 N32 2 accumulators", k_mma<32, true, 256, 2>, 256);
  run("TS M128 N32 4 accumulators", k_mma<32, true, 256, 4>, 256);
  run("TS M128 N32 8 accumulators", k_mma<32, true, 256, 8>, 256);
  run("SS M128 N32 4 accumulators", k_mma<32, false, 256, 4>, 256);
  run("SS M128 N64 4 accumulators", k_mma<64, false, 256, 4>, 256);
  run("SS M128 N96 2 accumulators", k_mma<96, false, 256, 2>, 256);
  run("TS M128 N96 2 accumulators", k_mma<96, true, 256, 2>, 256);
  run("SS N32 x1 (latency incl commit)", k_mma<32, false, 1>, 1);
  run("SS N96 x8 (commit incl)", k_mma<96, false, 8>, 8);
  run("roundtrip mma+commit->wait->arrive", k_roundtrip<256>, 256);
  return 0;
}
