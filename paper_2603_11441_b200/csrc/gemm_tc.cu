// Persistent tcgen05 GEMM for sm_100a: D[M,N] = A[M,K] . W[N,K]^T (+ fused epilogue).
//
// Replaces every `_linear` on the DART hot path (reference model.py:356-358:
// y = x @ W + b with W stored [in, out]; here W is stored transposed [out, in] so
// both operands are K-major).  Warp roles (256 threads, 1 CTA per SM):
//   warp 0  TMA producer  (A 128x64 and W BNx64 fp16 tiles, 128B swizzle, STAGES-deep ring)
//   warp 1  MMA issuer    (one thread, tcgen05.mma.cta_group::1.kind::f16, fp32 accumulators in TMEM)
//   warp 2  TMEM allocator
//   warps 4-7 epilogue    (tcgen05.ld -> bias / ReLU / residual / RoPE -> global)
// Two TMEM accumulator buffers let the epilogue of tile i overlap the MMAs of tile i+1.
#include "common.cuh"
#include "kernels.h"

namespace dart {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 fp16 = 128 B = one swizzle atom row

template <int BN, int STAGES, bool RESID = false>
struct GemmSmem {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_OFF = STAGES * STAGE_BYTES;  // 4 epilogue staging buffers of 4 KB
  static constexpr int RES_OFF = EPI_OFF + 4 * 4096;    // residual tile (RESID epilogue only)
  static constexpr int BAR_OFF = RES_OFF + (RESID ? BM * BN * 4 : 0);
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;  // barriers + 1 KB alignment slack
  static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
};

__device__ __forceinline__ void store_f16x32(act_t* dst, const float* v) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    u.x = pack_half2(v[8 * q + 0], v[8 * q + 1]);
    u.y = pack_half2(v[8 * q + 2], v[8 * q + 3]);
    u.z = pack_half2(v[8 * q + 4], v[8 * q + 5]);
    u.w = pack_half2(v[8 * q + 6], v[8 * q + 7]);
    d[q] = u;
  }
}

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(float* v, int row, int col, const GemmEpi& e, int rope_tok) {
  if (e.bias != nullptr) {
    const float4* b4 = reinterpret_cast<const float4*>(e.bias + col);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 b = __ldg(b4 + q);
      v[4 * q + 0] += b.x;
      v[4 * q + 1] += b.y;
      v[4 * q + 2] += b.z;
      v[4 * q + 3] += b.w;
    }
  }
  if (EPI == EPI_F16_RELU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.0f);
  }
  if (EPI == EPI_QKV_ROPE) {
    if (col < e.rope_cols) {
      // rope_tok: this row's true token (computed once per tile row by the caller)
      const int half_hd = e.rope_hd >> 1;
      const float* ct = e.rope_cos + (size_t)rope_tok * half_hd;
      const float* st = e.rope_sin + (size_t)rope_tok * half_hd;
      int p = (col % e.rope_hd) >> 1;  // pair index within the head, wraps at half_hd
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float c = __ldg(ct + p), s = __ldg(st + p);
        const float ev = v[j], od = v[j + 1];
        v[j] = ev * c - od * s;
        v[j + 1] = ev * s + od * c;
        p = (p + 1 == half_hd) ? 0 : p + 1;
      }
    }
  }
}

// ---- coalesced chunk I/O through a per-warp staging buffer -----------------------------
// A warp owns a 32-row x 32-column chunk (thread = row after tcgen05.ld).  The chunk goes
// through 4 KB of shared memory whose 16-byte slots are XOR-swizzled by row, so both the
// row-per-thread accesses and the line-per-8-lanes global accesses run at 4 wavefronts per
// 128-bit instruction, and every global load/store moves full 128-byte lines.
__device__ __forceinline__ float4* slot32(float* buf, int r, int k) {  // fp32 row r, 16B slot k (0..7)
  return reinterpret_cast<float4*>(buf) + r * 8 + (k ^ (r & 7));
}
__device__ __forceinline__ uint4* slot16(float* buf, int r, int k) {  // fp16 row r, 16B slot k (0..3)
  return reinterpret_cast<uint4*>(buf) + r * 4 + (k ^ (r & 3));
}

// dst_row(r): global row for chunk row r (identity, or the FPN's window-major -> token scatter)
__device__ __forceinline__ int chunk_dst_row(int row, const GemmEpi& e) {
  if (e.wm_scatter) {
    const int T = e.wm_grid * e.wm_grid;
    return (row / T) * T + wm_to_token(row % T, e.wm_grid, e.wm_win);
  }
  return row;
}

// Write the warp's chunk of fp32 values (v = this lane's row) to out (+= residual if RESID).
template <bool RESID>
__device__ __forceinline__ void chunk_store_f32(float* buf, const float* v, float* out, int ldo, int row0, int col,
                                                int M, const GemmEpi& e) {
  const int lane = threadIdx.x & 31;
  const int sub = lane >> 3, k = lane & 7;  // coalesced phase: 4 rows x 8 slots per instruction
  if (RESID) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = i * 4 + sub;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row0 + r < M) x = *reinterpret_cast<const float4*>(out + (size_t)(row0 + r) * ldo + col + 4 * k);
      *slot32(buf, r, k) = x;
    }
    __syncwarp();
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    if (RESID) {
      const float4 x = *slot32(buf, lane, q);
      o.x += x.x;
      o.y += x.y;
      o.z += x.z;
      o.w += x.w;
    }
    *slot32(buf, lane, q) = o;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = i * 4 + sub;
    if (row0 + r < M)
      *reinterpret_cast<float4*>(out + (size_t)chunk_dst_row(row0 + r, e) * ldo + col + 4 * k) = *slot32(buf, r, k);
  }
  __syncwarp();
}

__device__ __forceinline__ void chunk_store_f16(float* buf, const float* v, act_t* out, int ldo, int row0, int col,
                                                int M, const GemmEpi& e) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    u.x = pack_half2(v[8 * q + 0], v[8 * q + 1]);
    u.y = pack_half2(v[8 * q + 2], v[8 * q + 3]);
    u.z = pack_half2(v[8 * q + 4], v[8 * q + 5]);
    u.w = pack_half2(v[8 * q + 6], v[8 * q + 7]);
    *slot16(buf, lane, q) = u;
  }
  __syncwarp();
  const int sub = lane >> 2, k = lane & 3;  // 8 rows x 4 slots (64 B rows) per instruction
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = i * 8 + sub;
    if (row0 + r < M)
      *reinterpret_cast<uint4*>(out + (size_t)chunk_dst_row(row0 + r, e) * ldo + col + 8 * k) = *slot16(buf, r, k);
  }
  __syncwarp();
}

template <int EPI>
__device__ __forceinline__ void epilogue_store(float* buf, const float* v, int row0, int col, int M,
                                               const GemmEpi& e) {
  if (EPI == EPI_F16 || EPI == EPI_F16_RELU || EPI == EPI_QKV_ROPE) {
    chunk_store_f16(buf, v, reinterpret_cast<act_t*>(e.out), e.ldo, row0, col, M, e);
  } else if (EPI == EPI_F32 || EPI == EPI_F32_F16) {
    chunk_store_f32<false>(buf, v, reinterpret_cast<float*>(e.out), e.ldo, row0, col, M, e);
    if (EPI == EPI_F32_F16) chunk_store_f16(buf, v, reinterpret_cast<act_t*>(e.out2), e.ldo2, row0, col, M, e);
  } else if (EPI == EPI_F32_RESID) {
    chunk_store_f32<true>(buf, v, reinterpret_cast<float*>(e.out), e.ldo, row0, col, M, e);
  }
}

// Residual epilogue (EPI_F32_RESID, BN <= 128): warp 3 TMA-loads the tile's fp32 residual
// [128 x BN] into smem (32x32 boxes, 128B swizzle == slot32 layout) while the MMAs run; each
// epilogue warp adds its accumulator chunk in place and TMA-stores the chunk back.
template <int EPI>
__device__ __forceinline__ void resid_chunk(float* buf, const float* v, const CUtensorMap* tmC, int row0, int col) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float4* s = slot32(buf, lane, q);
    float4 x = *s;
    x.x += v[4 * q];
    x.y += v[4 * q + 1];
    x.z += v[4 * q + 2];
    x.w += v[4 * q + 3];
    *s = x;
  }
  fence_proxy_async();  // generic-proxy smem writes -> visible to the TMA (async proxy) store
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tmC, buf, col, row0);
    tma_store_commit();
  }
}

template <int BN, int STAGES, int EPI>
__global__ void __launch_bounds__(256, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, int M, int N, int K, GemmEpi epi) {
  using L = GemmSmem<BN, STAGES, EPI == EPI_F32_RESID>;
  constexpr bool RESID = EPI == EPI_F32_RESID;
  constexpr int CPW = BN / 32;  // 32-column chunks per epilogue warp and tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;
  uint64_t* rempty = rfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rempty + 1);
  float* resid = reinterpret_cast<float*>(smem + L::RES_OFF);  // [4 warps][CPW chunks][32 x 32]

  const int warp = warp_id();
  const int lane = lane_id();
  const int num_m = (M + BM - 1) / BM;
  const int num_n = N / BN;
  const int num_tiles = num_m * num_n;
  const int nk = K / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    mbar_init(rfull, 1);
    mbar_init(rempty, 4);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<L::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m0 = (tile / num_n) * BM;
        const int n0 = (tile % num_n) * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::STAGE_BYTES;
          uint8_t* sb = sa + L::A_BYTES;
          mbar_arrive_expect_tx(&full[stage], L::STAGE_BYTES);
          tma_load_2d(sa, &tmA, &full[stage], kb * BK, m0);
          tma_load_2d(sb, &tmB, &full[stage], kb * BK, n0);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_f16(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * L::STAGE_BYTES);
          const uint32_t sb = sa + L::A_BYTES;
          const uint64_t da = umma_desc_sw128(sa);
          const uint64_t db = umma_desc_sw128(sb);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // advance 16 fp16 = 32 B along K inside the swizzle atom (encoded >> 4)
            umma_f16(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp == 3) {
    if (RESID && lane == 0) {  // residual prefetch, one tile ahead of the epilogue
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int m0 = (tile / num_n) * BM;
        const int n0 = (tile % num_n) * BN;
        mbar_wait(rempty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(rfull, BM * BN * 4);
        for (int q = 0; q < 4; ++q)
          for (int c = 0; c < CPW; ++c)
            tma_load_2d(resid + (q * CPW + c) * 1024, &tmC, rfull, n0 + 32 * c, m0 + 32 * q);
      }
    }
  } else if (warp >= 4) {
    const int quarter = warp & 3;
    float* stage_buf = reinterpret_cast<float*>(smem + L::EPI_OFF) + quarter * 1024;  // 4 KB per warp
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int m0 = (tile / num_n) * BM;
      const int n0 = (tile % num_n) * BN;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + quarter * 32 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
      int rope_tok = 0;
      if (EPI == EPI_QKV_ROPE) {
        rope_tok = row % epi.rope_T;
        if (epi.wm_grid > 0) rope_tok = wm_to_token(rope_tok, epi.wm_grid, epi.wm_win);
      }
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        float v[32];
        tmem_ld32(taddr + c, v);
        tmem_ld_wait();
        if (c + 32 >= BN) {
          // all accumulator columns of this buffer are in registers: hand TMEM back early
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        epilogue_chunk<EPI>(v, row, n0 + c, epi, rope_tok);
        if constexpr (RESID) {
          if (c == 0) mbar_wait(rfull, it & 1);
          resid_chunk<EPI>(resid + (quarter * CPW + c / 32) * 1024, v, &tmC, m0 + quarter * 32, n0 + c);
        } else {
          epilogue_store<EPI>(stage_buf, v, m0 + quarter * 32, n0 + c, M, epi);
        }
      }
      if constexpr (RESID) {  // residual buffer reusable once the TMA stores have read it
        if (lane == 0) {
          tma_store_wait_read0();
          mbar_arrive(rempty);
        }
      }
    }
    if constexpr (RESID) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // writes landed
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<L::TMEM_COLS>(tmem_base);
  }
}

template <int BN, int STAGES, int EPI>
int launch_gemm(const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tC, int M, int N, int K,
                const GemmEpi& epi, int num_sms, cudaStream_t stream) {
  using L = GemmSmem<BN, STAGES, EPI == EPI_F32_RESID>;
  auto kern = gemm_tc_kernel<BN, STAGES, EPI>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
    if (e != cudaSuccess) return (int)e;
    configured = true;
  }
  const int tiles = ((M + BM - 1) / BM) * (N / BN);
  const int grid = tiles < num_sms ? tiles : num_sms;
  kern<<<grid, 256, L::TOTAL, stream>>>(tA, tB, tC, M, N, K, epi);
  return (int)cudaGetLastError();
}

template <int BN, int STAGES>
int dispatch_epi(int epi_mode, const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tC, int M, int N,
                 int K, const GemmEpi& epi, int num_sms, cudaStream_t stream) {
  switch (epi_mode) {
    case EPI_F16: return launch_gemm<BN, STAGES, EPI_F16>(tA, tB, tC, M, N, K, epi, num_sms, stream);
    case EPI_F16_RELU: return launch_gemm<BN, STAGES, EPI_F16_RELU>(tA, tB, tC, M, N, K, epi, num_sms, stream);
    case EPI_F32: return launch_gemm<BN, STAGES, EPI_F32>(tA, tB, tC, M, N, K, epi, num_sms, stream);
    case EPI_QKV_ROPE: return launch_gemm<BN, STAGES, EPI_QKV_ROPE>(tA, tB, tC, M, N, K, epi, num_sms, stream);
    case EPI_F32_F16: return launch_gemm<BN, STAGES, EPI_F32_F16>(tA, tB, tC, M, N, K, epi, num_sms, stream);
  }
  return (int)cudaErrorInvalidValue;
}

}  // namespace

int gemm_bn_for(int N) {
  if (N % 256 == 0) return 256;
  if (N % 128 == 0) return 128;
  if (N % 64 == 0) return 64;
  return 0;
}

// Tile width minimising wave-quantised work: cost = waves(tiles / SMs) * (BN + 32), where the
// +32 charges per-tile fixed cost (epilogue drain, A re-reads).  E.g. M=5184, N=1280 picks 128
// (410 tiles = 2.8 waves) over 256 (205 tiles = 1.4 waves).
int gemm_pick_bn(int M, int N, int num_sms) {
  int best = 0;
  long long best_cost = 0;
  for (int bn = 256; bn >= 64; bn >>= 1) {
    if (N % bn) continue;
    const long long tiles = (long long)((M + BM - 1) / BM) * (N / bn);
    const long long waves = (tiles + num_sms - 1) / num_sms;
    const long long cost = waves * (bn + 32);
    if (best == 0 || cost < best_cost) {
      best = bn;
      best_cost = cost;
    }
  }
  return best;
}

int gemm_tc(const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap* tC, int M, int N, int K, int BN,
            int epi_mode, const GemmEpi& epi, int num_sms, cudaStream_t stream) {
  if (M <= 0) return 0;
  if (K % BK != 0 || N % BN != 0) return (int)cudaErrorInvalidValue;
  if (epi_mode == EPI_F32_RESID) {  // TMA residual epilogue: BN <= 128, fewer mainloop stages
    if (!tC) return (int)cudaErrorInvalidValue;
    if (BN == 128) return launch_gemm<128, 4, EPI_F32_RESID>(tA, tB, *tC, M, N, K, epi, num_sms, stream);
    if (BN == 64) return launch_gemm<64, 6, EPI_F32_RESID>(tA, tB, *tC, M, N, K, epi, num_sms, stream);
    return (int)cudaErrorInvalidValue;
  }
  switch (BN) {
    case 256: return dispatch_epi<256, 4>(epi_mode, tA, tB, tA, M, N, K, epi, num_sms, stream);
    case 128: return dispatch_epi<128, 6>(epi_mode, tA, tB, tA, M, N, K, epi, num_sms, stream);
    case 64: return dispatch_epi<64, 8>(epi_mode, tA, tB, tA, M, N, K, epi, num_sms, stream);
  }
  return (int)cudaErrorInvalidValue;
}

int gemm_resid_bn(int N) { return N % 128 == 0 ? 128 : (N % 64 == 0 ? 64 : 0); }

}  // namespace dart
