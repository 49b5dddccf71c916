// Persistent tcgen05 GEMM for sm_100a: D[M,N] = A[M,K] . W[N,K]^T (+ fused epilogue).
//
// Replaces every `_linear` on the DART hot path (reference model.py:356-358:
// y = x @ W + b with W stored [in, out]; here W is stored transposed [out, in] so
// both operands are K-major).  Warp roles (384 threads, 1 CTA per SM):
//   warp 0  TMA producer  (A 128x64 and W (BN/CG)x64 fp16 tiles, 128B swizzle, STAGES-deep ring)
//   warp 1  MMA issuer    (one thread, tcgen05.mma.cta_group::CG.kind::f16, fp32 accumulators in TMEM)
//   warp 2  TMEM allocator
//   warps 4-11 epilogue   (two per TMEM lane quarter, alternating 32-column chunks: tcgen05.ld ->
//                          bias / ReLU / RoPE / residual -> swizzled smem chunk -> TMA bulk store;
//                          the residual chunk is TMA-prefetched one chunk ahead)
// Two TMEM accumulator buffers let the epilogue of tile i overlap the MMAs of tile i+1.
//
// CG = 2 is the CTA-pair ("2-SM") form: a cluster of 2 CTAs on one TPC computes a 256 x BN
// tile with M=256 tcgen05.mma.cta_group::2 issued by the leader CTA.  Each CTA loads its own
// 128 rows of A and HALF of the BN rows of W, so the smem / L2 operand traffic per FLOP is
// 25-33% lower than the 1-SM form; both CTAs' TMA loads complete on the leader's full barrier,
// MMA completion is multicast to both CTAs' empty / accumulator-full barriers, and both CTAs'
// epilogue warps release the accumulator on the leader's barrier.
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace dart {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 fp16 = 128 B = one swizzle atom row
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;  // shared::cluster address of the leader CTA's copy
constexpr int ROPE_PAD = 21;                 // float2 row stride of the small RoPE tables (bank spread)
constexpr int ROPE_MAX_GRID = 72;
constexpr int ROPE_MAX_Q = 20;               // hd / 4

template <int BN, int STAGES, int EPI, int CG>
struct GemmSmem {
  static constexpr int B_ROWS = BN / CG;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr bool RESID = EPI == EPI_F32_RESID || EPI == EPI_F32_RESID_LN || EPI == EPI_F32_RESID_X16;
  static constexpr bool LNO = EPI == EPI_F32_RESID_LN;  // fused LayerNorm output of full rows
  static constexpr bool X16 = EPI == EPI_F32_RESID_X16;  // + fp16 copy and LN chunk statistics
  // staging buffers per epilogue warp; 4 for the residual epilogue (3 chunks prefetched) measured
  // slower: the extra 64 KB costs two operand stages (out-proj 24.8 -> 27.1 us, fc2 63.4 -> 80 us)
  static constexpr int NBUF = 2;
  // staging buffer per chunk: 32x32 fp32 (4 KB), or 32x32 fp16 (2 KB) for the fp16-only epilogues
  static constexpr int BUF_BYTES = (EPI == EPI_F16 || EPI == EPI_F16_RELU || EPI == EPI_QKV_ROPE) ? 2048 : 4096;
  static constexpr int EPI_OFF = STAGES * STAGE_BYTES;  // 8 warps x NBUF staging buffers
  // fused LN: 2 fp16 32x32 staging chunks per epilogue warp + the row-statistics exchange
  static constexpr int LN_OFF = EPI_OFF + 8 * NBUF * BUF_BYTES;
  // (X16: one fp16 32x32 staging chunk per epilogue warp for the fp16 copy of the new residual)
  static constexpr int LN_BYTES = LNO ? 8 * 2 * 2048 + 4 * 2 * 32 * 4 : X16 ? 8 * 2048 : 0;
  static constexpr int ROPE_OFF = LN_OFF + LN_BYTES;  // [2][grid][ROPE_PAD] float2 (QKV epilogue only)
  static constexpr int ROPE_BYTES = EPI == EPI_QKV_ROPE ? 2 * ROPE_MAX_GRID * ROPE_PAD * 8 : 0;
  static constexpr int BAR_OFF = ROPE_OFF + ROPE_BYTES;
  static constexpr int TOTAL = BAR_OFF + 512 + 1024;  // barriers + 1 KB alignment slack
  static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static_assert(TOTAL <= 227 * 1024, "shared memory budget");
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load whose completion is signalled on the LEADER CTA's barrier (CTA-pair form).
__device__ __forceinline__ void tma_load_2d_cg2(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & PEER_MASK), "r"(c0), "r"(c1)
      : "memory");
}
// Issued by the converged MMA warp: one elected lane (see umma_f16_w in common.cuh).
template <int CG>
__device__ __forceinline__ void umma_f16_cg(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  if constexpr (CG == 1) {
    umma_f16_w(tmem_d, a_desc, b_desc, idesc, accumulate);
  } else {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
  }
}
// MMA completion -> barrier at the same smem offset in every CTA of the pair (or the own CTA).
template <int CG>
__device__ __forceinline__ void umma_commit_cg(uint64_t* bar) {
  if constexpr (CG == 1) {
    umma_commit_w(bar);
  } else {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
  }
}
// Arrive on the leader CTA's copy of `bar` (rank 0 of the pair).
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
template <int NCOLS, int CG>
__device__ __forceinline__ void tmem_alloc_cg(uint32_t* smem_dst) {
  if constexpr (CG == 1) {
    tmem_alloc<NCOLS>(smem_dst);
  } else {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
                 "n"(NCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
}
template <int NCOLS, int CG>
__device__ __forceinline__ void tmem_dealloc_cg(uint32_t base) {
  if constexpr (CG == 1) {
    tmem_dealloc<NCOLS>(base);
  } else {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(NCOLS) : "memory");
  }
}

// 2-D RoPE (reference tensors.py:235-252, model.py:203-213) on a 32-column chunk of this
// lane's row: pair p of head-local columns (2p, 2p+1) rotates by the row-coordinate angle for
// p < hd/4 and by the column-coordinate angle otherwise.  `rt` / `ct` point at this token's
// row of the small per-coordinate tables [coord][ROPE_PAD] of (cos, sin).
__device__ __forceinline__ void rope_chunk(float* v, int col, int hd, const float2* rt, const float2* ct) {
  const int q = hd >> 2, half = hd >> 1;
  int p = (col % hd) >> 1;
#pragma unroll
  for (int j = 0; j < 32; j += 2) {
    const float2 cs = p < q ? rt[p] : ct[p - q];
    const float ev = v[j], od = v[j + 1];
    v[j] = ev * cs.x - od * cs.y;
    v[j + 1] = ev * cs.y + od * cs.x;
    p = (p + 1 == half) ? 0 : p + 1;
  }
}

// rope_chunk for hd 80 (ViT-H/14) with the chunk's first pair index P0 = (col % 80) / 2 known at
// compile time: the row / column angle choice and the wrap at 40 pairs fold away, and the tables
// are read with ld.shared (the generic-pointer form above costs ~300 extra instructions per chunk
// in index arithmetic and generic loads).  rt_s / ct_s: shared addresses of this token's rows.
__device__ __forceinline__ float2 lds_f2(uint32_t addr) {
  float2 r;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "r"(addr));
  return r;
}
template <int P0>
__device__ __forceinline__ void rope_chunk80(float* v, uint32_t rt_s, uint32_t ct_s) {
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int p = (P0 + j) % 40;
    const float2 cs = p < 20 ? lds_f2(rt_s + p * 8) : lds_f2(ct_s + (p - 20) * 8);
    const float ev = v[2 * j], od = v[2 * j + 1];
    v[2 * j] = ev * cs.x - od * cs.y;
    v[2 * j + 1] = ev * cs.y + od * cs.x;
  }
}
__device__ __forceinline__ void rope_chunk_hd80(float* v, int col, uint32_t rt_s, uint32_t ct_s) {
  switch ((col % 80) >> 1) {  // col is a multiple of 32
    case 0: rope_chunk80<0>(v, rt_s, ct_s); break;
    case 8: rope_chunk80<8>(v, rt_s, ct_s); break;
    case 16: rope_chunk80<16>(v, rt_s, ct_s); break;
    case 24: rope_chunk80<24>(v, rt_s, ct_s); break;
    default: rope_chunk80<32>(v, rt_s, ct_s); break;
  }
}

// fp16 storage rounding, saturating at +-65504 like the reference's half_round (tensors.py:99-109)
__device__ __forceinline__ float sat_f16(float x) { return fminf(fmaxf(x, -65504.0f), 65504.0f); }
__device__ __forceinline__ float round_f16(float x) { return __half2float(__float2half_rn(sat_f16(x))); }

// bias chunk of 32 columns, loaded ahead of the TMEM load so its latency overlaps it
__device__ __forceinline__ void bias_prefetch(float4 (&b)[8], int col, const float* bias) {
  if (bias != nullptr) {
    const float4* b4 = reinterpret_cast<const float4*>(bias + col);
#pragma unroll
    for (int q = 0; q < 8; ++q) b[q] = __ldg(b4 + q);
  }
}
template <int EPI>
__device__ __forceinline__ void epilogue_bias_act(float* v, const float4 (&b)[8], const float* bias) {
  if (bias != nullptr) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      v[4 * q + 0] += b[q].x;
      v[4 * q + 1] += b[q].y;
      v[4 * q + 2] += b[q].z;
      v[4 * q + 3] += b[q].w;
    }
  }
  if (EPI == EPI_F16_RELU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.0f);
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

// Write the warp's chunk of fp32 values (v = this lane's row) to out.
__device__ __forceinline__ void chunk_store_f32(float* buf, const float* v, float* out, int ldo, int row0, int col,
                                                int M, const GemmEpi& e) {
  const int lane = threadIdx.x & 31;
  const int sub = lane >> 3, k = lane & 7;  // coalesced phase: 4 rows x 8 slots per instruction
#pragma unroll
  for (int q = 0; q < 8; ++q) *slot32(buf, lane, q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
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

// fp16 32x32 chunk slot under the TMA 64-byte swizzle (64 B rows, 16 B slot k of row r at
// k ^ ((r >> 1) & 3)): conflict-free for the row-per-lane writes.
__device__ __forceinline__ uint4* slot16_sw64(float* buf, int r, int k) {
  return reinterpret_cast<uint4*>(buf) + r * 4 + (k ^ ((r >> 1) & 3));
}
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Fused LayerNorm epilogue over whole 256-column rows (the enc-dec's d = 256; reference
// tensors.py:215-227: two-pass mean / population variance, eps 1e-6, then * gamma + beta).
// Called by each of the 8 epilogue warps after it stashed its chunks of the NEW residual rows
// (columns half*32 + 64 i, i < 4, relative to `taddr`) back into TMEM and summed them into
// `row_sum`: the two warps of a lane quarter combine their partial sums through `red`
// ([4 quarters][2 halves][32] floats) in a fixed order, re-read the stash for the variance and
// the normalisation, and store the fp16 rows with TMA (tmOut, box 32x32, 64B swizzle) through
// two 2 KB staging chunks `lnbuf`, `stride` floats apart.  Every operation is pinned to an IEEE
// intrinsic, so the GEMM epilogue and the fused-MLP epilogue produce identical bits.
__device__ __forceinline__ void ln_rows_epilogue(uint32_t taddr, int quarter, int half, int lane, float row_sum,
                                                 const float* gamma, const float* beta, float* red, float* lnbuf,
                                                 int stride, const CUtensorMap* tmOut, int col0, int row0) {
  tmem_st_wait();  // the stash is in TMEM before any warp re-reads it
  float* r = red + quarter * 64;
  r[half * 32 + lane] = row_sum;
  named_bar_sync(2 + quarter, 64);
  const float mu = __fmul_rn(__fadd_rn(r[lane], r[32 + lane]), 1.0f / 256.0f);
  named_bar_sync(2 + quarter, 64);  // both partners have read the sums before `r` is reused
  float q = 0.f;
#pragma unroll 1
  for (int i = 0; i < 4; ++i) {
    float x[32];
    tmem_ld32(taddr + half * 32 + 64 * i, x);
    tmem_ld_wait();
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const float d = __fsub_rn(x[k], mu);
      q = __fmaf_rn(d, d, q);
    }
  }
  r[half * 32 + lane] = q;
  named_bar_sync(2 + quarter, 64);
  const float var = __fmul_rn(__fadd_rn(r[lane], r[32 + lane]), 1.0f / 256.0f);
  named_bar_sync(2 + quarter, 64);  // the variances are read before the next row block's sums land
  const float rstd = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-6f)));
#pragma unroll 1
  for (int i = 0; i < 4; ++i) {
    const int c = half * 32 + 64 * i;
    float x[32];
    tmem_ld32(taddr + c, x);
    tmem_ld_wait();
    const float4* g4 = reinterpret_cast<const float4*>(gamma + c);
    const float4* b4 = reinterpret_cast<const float4*>(beta + c);
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) {
      const float4 gg = __ldg(g4 + qq), bb = __ldg(b4 + qq);
      x[4 * qq] = __fmaf_rn(__fmul_rn(__fsub_rn(x[4 * qq], mu), rstd), gg.x, bb.x);
      x[4 * qq + 1] = __fmaf_rn(__fmul_rn(__fsub_rn(x[4 * qq + 1], mu), rstd), gg.y, bb.y);
      x[4 * qq + 2] = __fmaf_rn(__fmul_rn(__fsub_rn(x[4 * qq + 2], mu), rstd), gg.z, bb.z);
      x[4 * qq + 3] = __fmaf_rn(__fmul_rn(__fsub_rn(x[4 * qq + 3], mu), rstd), gg.w, bb.w);
    }
    float* lb = lnbuf + (i & 1) * stride;
    if (lane == 0) {  // the stores that last used this staging chunk have read it
      if (i == 0)
        bulk_wait_read0();
      else
        bulk_wait_read1();
    }
    __syncwarp();
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      uint4 u;
      u.x = pack_half2(x[8 * qq + 0], x[8 * qq + 1]);
      u.y = pack_half2(x[8 * qq + 2], x[8 * qq + 3]);
      u.z = pack_half2(x[8 * qq + 4], x[8 * qq + 5]);
      u.w = pack_half2(x[8 * qq + 6], x[8 * qq + 7]);
      *slot16_sw64(lb, lane, qq) = u;
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(tmOut, lb, col0 + c, row0);
      tma_store_commit();
    }
  }
}

// LayerNorm statistics of one 32-value chunk of a row (two-pass: mean, then the centred sum of
// squares), the producer half of the LN fold (GemmEpi::ln_stats_out)
__device__ __forceinline__ float2 chunk_ln_stats(const float* v) {
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) s += v[j];
  const float mu = s * (1.0f / 32.0f);
  float q = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float d = v[j] - mu;
    q = fmaf(d, d, q);
  }
  return make_float2(mu, q);
}
// Consumer half: the row's `parts` chunk statistics combined in order (Chan et al. pairwise
// update, equal chunk sizes), -> (mean, 1/sqrt(var + eps)) with population variance (reference
// tensors.py:215-227, eps 1e-6)
__device__ __forceinline__ float2 ln_row_stats(const float2* st, int parts) {
  // equal-size chunks: mean = mean of the chunk means; M2 = sum of the chunk M2 + 32 * the chunk
  // means' sum of squared deviations, taken about the first chunk's mean (shifted, one pass, so
  // every load is in flight at once; parts is even: E % 64 == 0, 16-byte loads, fixed order)
  const float4* st4 = reinterpret_cast<const float4*>(st);
  const float k0 = __ldcg(&st[0].x);
  float sm = 0.f, sq = 0.f, sd = 0.f;
  for (int i0 = 0; i0 < parts / 2; i0 += 10) {
    float4 b[10];
#pragma unroll
    for (int j = 0; j < 10; ++j) b[j] = i0 + j < parts / 2 ? __ldcg(st4 + i0 + j) : make_float4(k0, 0.f, k0, 0.f);
#pragma unroll
    for (int j = 0; j < 10; ++j) {
      sm += b[j].x + b[j].z;
      sq += b[j].y + b[j].w;
      const float d0 = b[j].x - k0, d1 = b[j].z - k0;
      sd = fmaf(d0, d0, fmaf(d1, d1, sd));
    }
  }
  const float n = (float)parts;
  const float mu = sm / n;
  const float dm = mu - k0;
  const float var = (sq + 32.f * fmaxf(sd - n * dm * dm, 0.f)) / (32.f * n);
  return make_float2(mu, 1.0f / sqrtf(var + 1e-6f));
}

constexpr int GEMM_THREADS = 384;
// fp32 residual epilogue through a TMA reduce-add (see RED in gemm_tc_kernel); -DDART_RESID_REDUCE=0
// builds the load-add-store epilogue instead (A/B)
#ifndef DART_RESID_REDUCE
#define DART_RESID_REDUCE 1
#endif
constexpr bool RESID_REDUCE = DART_RESID_REDUCE != 0;

// PREC: the precision-study variant (GemmEpi::acc_f16 / round_f16 honoured); the detection
// path's instantiations (PREC = false) carry none of that code.  SPLITK: two K halves per tile
// combined through a partial-accumulator workspace (GemmEpi::splitk); without it the split-K
// paths compile out.
// dart_gemm_trace: per-CTA globaltimer stamps of the first GEMM launch after it is set (timeline
// microbenchmarks; nullptr = off, one predicated global load per stamp site)
__device__ long long* g_gemm_trace = nullptr;
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define GEMM_STAMP(k)                                                   \
  do {                                                                  \
    long long* _tr = g_gemm_trace;                                      \
    if (_tr) _tr[blockIdx.x * 8 + (k)] = gtimer();                      \
  } while (0)
// per-unit stamps (first 8 units of a CTA) after the per-CTA block: [148 * 8][unit < 8][8]
#define GEMM_STAMP_U(u, k)                                                              \
  do {                                                                                  \
    long long* _tr = g_gemm_trace;                                                      \
    if (_tr && (u) < 8) _tr[148 * 8 + (blockIdx.x * 8 + (u)) * 8 + (k)] = gtimer();     \
  } while (0)

template <int BN, int STAGES, int EPI, int CG, bool PREC, bool SPLITK>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmC,
                   const __grid_constant__ CUtensorMap tmD, int M, int N, int K, GemmEpi epi) {
  // tmC: fp32 [M, N] output / residual map (box 32x32, 128B swizzle); tmD: fp16 [M, N] output map
  // (box 32x32, 64B swizzle).  Outputs leave through per-warp smem chunks and TMA bulk stores.
  using L = GemmSmem<BN, STAGES, EPI, CG>;
  // RED: the fp32 residual add x += acc + bias as a TMA reduce-add (cp.reduce.async.bulk.tensor
  // .add) -- the epilogue never loads x, the L2 adds on the way in.  Not for the fused-LN epilogue
  // (it needs the new row values) nor the fp16-storage study variant (it rounds the sum).
  constexpr bool RED = EPI == EPI_F32_RESID && !PREC && RESID_REDUCE;
  constexpr bool RESID = L::RESID && !RED;  // epilogues that load the residual chunk
  static_assert(BN % 32 == 0, "32-column epilogue chunks");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;  // [8 warps][NBUF buffers]: residual chunk landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rfull + 8 * L::NBUF);

  const int warp = warp_id();
  const int lane = lane_id();
  const int rank = CG == 2 ? (int)cluster_ctarank() : 0;
  const int cl = blockIdx.x / CG, ncl = gridDim.x / CG;
  const int num_m = (M + BM * CG - 1) / (BM * CG);
  const int num_n = N / BN;
  const int num_tiles = num_m * num_n;
  static_assert(!(SPLITK && L::LNO), "split-K is not combined with the full-row LayerNorm epilogue");
  constexpr int SK = SPLITK ? 2 : 1;      // K halves per tile (work unit = tile x half)
  const int TF = SPLITK ? 0 : epi.tail_full;  // tail halves: units >= TF are BN/2-wide halves of a tile
  const int num_units = TF > 0 ? TF + 2 * (num_tiles - TF) : num_tiles * SK;
  const int nk = K / BK / SK;             // k-blocks per unit
  // unit -> (tile, K half, n half or -1 for a full-width unit).  Split-K: units 2t and 2t+1 are
  // the two K halves of tile t, on neighbouring CTA pairs of the same wave, so a partial
  // accumulator is consumed microseconds after it is written and stays in L2 (halves a wave
  // apart keep ~a wave of partials in flight: 80 MB for the QKV shape, which spills to HBM)
  auto decode = [&](int u, int& tile, int& kh, int& nh) {
    if (TF > 0 && u >= TF) {
      tile = TF + ((u - TF) >> 1);
      nh = (u - TF) & 1;
      kh = 0;
    } else {
      tile = u / SK;
      kh = u % SK;
      nh = -1;
    }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (TF > 0) tma_prefetch_desc(&tmB2);
    if (RESID || RED || EPI == EPI_F32) tma_prefetch_desc(&tmC);
    if (EPI == EPI_F16 || EPI == EPI_F16_RELU || EPI == EPI_QKV_ROPE || EPI == EPI_F32_RESID_LN || EPI == EPI_F32_RESID_X16)
      tma_prefetch_desc(&tmD);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8 * CG);
    }
    for (int i = 0; i < 8 * L::NBUF; ++i) mbar_init(&rfull[i], 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_cg<L::TMEM_COLS, CG>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync_all();  // peer barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) GEMM_STAMP(0);
  // the previous kernel's outputs (our A / residual) are complete from here on -- or, in a
  // row-block dependency chain (GemmEpi::dep_wait), per 128-row block as the producer sees them
  if (!epi.skip_pdl_wait) pdl_wait();
  if (epi.early_trigger) pdl_launch_dependents();
  if (threadIdx.x == 0) GEMM_STAMP(1);

  if (warp == 0) {
    if (lane == 0) {
      // kernel parameters read inside the loops are hoisted: after every asm "memory" clobber
      // (barrier waits, TMA) a parameter is otherwise re-loaded from the constant bank
      const bool noload = epi.dbg_noload != 0;
      const int* const dep_wait = epi.dep_wait;
      const int dep_mult = epi.dep_mult, dep_per_row = epi.dep_per_row;
      int stage = 0;
      uint32_t phase = 0;
      for (int unit = cl; unit < num_units; unit += ncl) {
        int tile, kh, nh;
        decode(unit, tile, kh, nh);
        const int kb0 = kh * nk;
        const bool hu = nh >= 0;
        const int m0 = (tile / num_n) * BM * CG + rank * BM;
        if (dep_wait != nullptr && m0 < M) {  // dependency chain: this CTA's 128 A rows are complete
          const int rows_blk = M - m0 < BM ? M - m0 : BM;
          const int target = dep_mult * (dep_per_row ? rows_blk : 1);
          long long spins = 0;
          while (*reinterpret_cast<const volatile int*>(dep_wait + (m0 >> 7)) < target) {
            __nanosleep(256);
            if (++spins > (1ll << 25)) __trap();  // a broken chain fails loudly instead of hanging
          }
          __threadfence();
          asm volatile("fence.proxy.async.global;" ::: "memory");  // the TMA reads below see the rows
        }
        const int n0 = (tile % num_n) * BN + (hu ? nh * (BN / 2) + rank * (L::B_ROWS / 2) : rank * L::B_ROWS);
        const CUtensorMap* mb = hu ? &tmB2 : &tmB;
        const uint32_t bytes = hu ? L::A_BYTES + L::B_BYTES / 2 : L::STAGE_BYTES;
        for (int kb = kb0; kb < kb0 + nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::STAGE_BYTES;
          uint8_t* sb = sa + L::A_BYTES;
          if (noload && (unit != cl || kb >= STAGES)) {
            if (rank == 0) mbar_arrive(&full[stage]);
          } else if constexpr (CG == 1) {
            mbar_arrive_expect_tx(&full[stage], bytes);
            tma_load_2d(sa, &tmA, &full[stage], kb * BK, m0);
            tma_load_2d(sb, mb, &full[stage], kb * BK, n0);
          } else {
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * bytes);
            tma_load_2d_cg2(sa, &tmA, &full[stage], kb * BK, m0);
            tma_load_2d_cg2(sb, mb, &full[stage], kb * BK, n0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // the whole (converged) warp runs the issue loop; one elected lane issues
      const uint32_t dfmt = (PREC && epi.acc_f16) ? (1u << 4) : 0u;  // clear D = f32 -> f16 accumulator
      const uint32_t idesc_full = umma_idesc_f16(BM * CG, BN) ^ dfmt;
      const uint32_t idesc_half = umma_idesc_f16(BM * CG, BN / 2) ^ dfmt;
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int unit = cl; unit < num_units; unit += ncl, ++it) {
        const uint32_t idesc = (TF > 0 && unit >= TF) ? idesc_half : idesc_full;
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          if (it == 0 && kb == 0 && lane == 0) GEMM_STAMP(2);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * L::STAGE_BYTES);
          const uint32_t sb = sa + L::A_BYTES;
          const uint64_t da = umma_desc_sw128(sa);
          const uint64_t db = umma_desc_sw128(sb);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // advance 16 fp16 = 32 B along K inside the swizzle atom (encoded >> 4)
            umma_f16_cg<CG>(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          }
          umma_commit_cg<CG>(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_cg<CG>(&tfull[acc]);
        if (lane == 0) GEMM_STAMP(it == 0 ? 3 : 6);
        if (lane == 0) GEMM_STAMP_U(it, 0);  // unit's MMAs issued
      }
    }
  } else if (warp >= 4) {
    if constexpr (EPI == EPI_QKV_ROPE) {
      // small per-coordinate RoPE tables from the [T, hd/2] tables: row angles of token (c, 0)
      // (pairs < hd/4) and column angles of token (0, c) (pairs >= hd/4).  Filled by the
      // epilogue warps only, while the producer / MMA warps already run the first tile.
      float2* rs = reinterpret_cast<float2*>(smem + L::ROPE_OFF);
      const int g = epi.rope_grid, q = epi.rope_hd >> 2, hh = epi.rope_hd >> 1;
      for (int i = threadIdx.x - 128; i < 2 * g * q; i += GEMM_THREADS - 128) {
        const int which = i / (g * q), c = (i / q) % g, f = i % q;
        const size_t src = which == 0 ? (size_t)c * g * hh + f : (size_t)c * hh + q + f;
        rs[(which * ROPE_MAX_GRID + c) * ROPE_PAD + f] = make_float2(__ldg(epi.rope_cos + src), __ldg(epi.rope_sin + src));
      }
      named_bar_sync(1, GEMM_THREADS - 128);
    }
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    const float* const bias = epi.bias;  // hoisted kernel parameters (see the producer)
    [[maybe_unused]] const float2* const ln_stats = epi.ln_stats;
    [[maybe_unused]] const float* const ln_colsum = epi.ln_colsum;
    [[maybe_unused]] float2* const ln_stats_out = epi.ln_stats_out;
    [[maybe_unused]] const int ln_parts = epi.ln_parts;
    const int rope_cols = epi.rope_cols, rope_hd = epi.rope_hd;
    constexpr int NBUF = L::NBUF;
    constexpr int BUF_F = L::BUF_BYTES / 4;  // staging buffer size in floats
    float* bufs = reinterpret_cast<float*>(smem + L::EPI_OFF) + (warp - 4) * NBUF * BUF_F;
    uint64_t* rbar = rfull + (warp - 4) * NBUF;
    const float2* rope_s = reinterpret_cast<const float2*>(smem + L::ROPE_OFF);
    // residual chunk g of this warp -> smem buffer g % NBUF (lane 0 issues; NBUF-1 chunks ahead)
    // residual prefetch iterator: (unit, chunk) of the next chunk this warp will process
    // (split-K: no look-ahead across units -- only the half that combines reads the residual,
    // and which half that is is decided when its epilogue starts)
    int pf_u = SPLITK ? num_units : cl, pf_c = 0;
    auto resid_load = [&](int g) {  // prefetch the iterator's chunk into buffer g % NBUF, advance
      if (pf_u >= num_units) return;
      int t, kh, nh;
      decode(pf_u, t, kh, nh);
      const int bne = nh >= 0 ? BN / 2 : BN;
      const int rr = (t / num_n) * BM * CG + rank * BM + quarter * 32;
      const int cc = (t % num_n) * BN + (nh >= 0 ? nh * (BN / 2) : 0) + (pf_c * 2 + half) * 32;
      mbar_arrive_expect_tx(&rbar[g % NBUF], 32 * 32 * 4);
      tma_load_2d(bufs + (g % NBUF) * BUF_F, &tmC, &rbar[g % NBUF], cc, rr);
      if (++pf_c == (bne - half * 32 + 63) / 64) {
        pf_c = 0;
        pf_u = SPLITK ? num_units : pf_u + ncl;
      }
    };
    if (RESID && lane == 0)
      for (int i = 0; i < NBUF - 1; ++i) resid_load(i);
    int it = 0, g = 0;
    for (int unit = cl; unit < num_units; unit += ncl, ++it) {
      int tile, kh, nh;
      decode(unit, tile, kh, nh);
      const int bn_eff = nh >= 0 ? BN / 2 : BN;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int m0 = (tile / num_n) * BM * CG + rank * BM;
      const int n0 = (tile % num_n) * BN + (nh >= 0 ? nh * (BN / 2) : 0);
      const int row0 = m0 + quarter * 32;
      // LN fold consumer: this row's (mean, rstd), finalised by the producer; loaded while the
      // unit's main loop still runs
      [[maybe_unused]] float2 lnrs = make_float2(0.f, 1.f);
      if constexpr (EPI == EPI_QKV_ROPE || EPI == EPI_F16_RELU) {
        if (ln_stats != nullptr && row0 + lane < M) lnrs = __ldcg(ln_stats + row0 + lane);
      }
      mbar_wait(&tfull[acc], acc_phase);
      if (it == 0 && warp == 4 && lane == 0) GEMM_STAMP(4);
      if (warp == 4 && lane == 0) GEMM_STAMP_U(it, 1);  // accumulator ready
      tc_fence_after();
      const int row = row0 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
      [[maybe_unused]] int* sk_flag = nullptr;
      [[maybe_unused]] const float4* sk_part = nullptr;
      if constexpr (SPLITK) {
        // claim: the first of the two K halves of this (tile, CTA, warp) to get here publishes
        // its partial accumulator, the second combines (claim +1, publish +16)
        sk_flag = epi.tile_flags + ((size_t)tile * CG + rank) * 8 + (warp - 4);
        float4* part = reinterpret_cast<float4*>(epi.ws) + ((size_t)tile * CG + rank) * (BN / 32) * 4 * 256;
        int old = 0;
        if (lane == 0) old = atomicAdd(sk_flag, 1);
        old = __shfl_sync(0xffffffffu, old, 0);
        if ((old & 15) == 0) {
#pragma unroll 1
          for (int c = half * 32; c < bn_eff; c += 64) {
            float v[32];
            tmem_ld32(taddr + c, v);
            tmem_ld_wait();
            if (c + 64 >= bn_eff) {  // accumulator fully read: hand TMEM back
              tc_fence_before();
              __syncwarp();
              if (lane == 0) {
                if constexpr (CG == 1) {
                  mbar_arrive(&tempty[acc]);
                } else {
                  mbar_arrive_leader(&tempty[acc]);
                }
              }
            }
            // [chunk column][quarter][float4 q][lane]: coalesced 512-byte rows for both halves
            float4* p = part + ((c >> 5) * 4 + quarter) * 256 + lane;
#pragma unroll
            for (int q = 0; q < 8; ++q) __stcg(p + q * 32, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
          }
          if (warp == 4 && lane == 0) GEMM_STAMP_U(it, 2);  // partial stored
          __threadfence();
          __syncwarp();
          if (lane == 0) atomicAdd(sk_flag, 16);
          if (warp == 4 && lane == 0) GEMM_STAMP_U(it, 3);  // published
          continue;
        }
        if (RESID && lane == 0) {  // residual chunks of this unit only, from chunk 0
          bulk_wait_read0();
          pf_u = unit;
          pf_c = 0;
          for (int i = 0; i < NBUF - 1; ++i) resid_load(g + i);
        }
        if (warp == 4 && lane == 0) GEMM_STAMP_U(it, 4);  // combining: before the wait
        if (lane == 0 && old < 16)
          while (*reinterpret_cast<volatile int*>(sk_flag) < 16) __nanosleep(32);
        __syncwarp();
        __threadfence();
        if (warp == 4 && lane == 0) GEMM_STAMP_U(it, 5);  // partial visible
        sk_part = part + quarter * 256 + lane;
      }
      [[maybe_unused]] float ln_sum = 0.f;
      const float2 *rt = nullptr, *ct = nullptr;
      if (EPI == EPI_QKV_ROPE) {
        int tok = row % epi.rope_T;
        if (epi.wm_grid > 0) tok = wm_to_token(tok, epi.wm_grid, epi.wm_win);
        const int tr = tok / epi.rope_grid, tc = tok - tr * epi.rope_grid;
        rt = rope_s + tr * ROPE_PAD;
        ct = rope_s + (ROPE_MAX_GRID + tc) * ROPE_PAD;
      }
#pragma unroll 1
      for (int c = half * 32; c < bn_eff; c += 64, ++g) {
        float* buf = bufs + (g % NBUF) * BUF_F;
        if (lane == 0) {
          if (RESID) {
            bulk_wait_read0();  // store g-1 has read buffer (g-1) % NBUF = (g+NBUF-1) % NBUF
            resid_load(g + NBUF - 1);
          } else {
            bulk_wait_read1();  // store g-2 has read this buffer
          }
        }
        __syncwarp();
        float4 bq[8];  // (the RoPE epilogue loads its bias after the TMEM wait: register budget)
        if constexpr (EPI != EPI_QKV_ROPE) bias_prefetch(bq, n0 + c, bias);
        float v[32];
        tmem_ld32(taddr + c, v);
        if constexpr (SPLITK) {  // + the other K half's partial (commutative: same bits either way)
          float4 pp[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) pp[q] = __ldcg(sk_part + (c >> 5) * 4 * 256 + q * 32);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            v[4 * q] += pp[q].x;
            v[4 * q + 1] += pp[q].y;
            v[4 * q + 2] += pp[q].z;
            v[4 * q + 3] += pp[q].w;
          }
        } else {
          tmem_ld_wait();
        }
        if ((PREC && epi.acc_f16)) {  // f16 accumulator: one value per 32-bit TMEM cell, low half
#pragma unroll
          for (int j = 0; j < 32; ++j)
            v[j] = __half2float(__ushort_as_half((unsigned short)(__float_as_uint(v[j]) & 0xFFFFu)));
        }
        if (!L::LNO && c + 64 >= bn_eff) {
          // all of this warp's accumulator columns are in registers: hand TMEM back early
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 1) {
              mbar_arrive(&tempty[acc]);
            } else {
              mbar_arrive_leader(&tempty[acc]);
            }
          }
        }
        if constexpr (EPI == EPI_QKV_ROPE || EPI == EPI_F16_RELU) {
          if (ln_stats != nullptr) {  // LN fold: rstd * (x W' - mu * colsum(W'))
            const float4* cs4 = reinterpret_cast<const float4*>(ln_colsum + n0 + c);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 cs = __ldg(cs4 + q);
              v[4 * q] = fmaf(-lnrs.x, cs.x, v[4 * q]) * lnrs.y;
              v[4 * q + 1] = fmaf(-lnrs.x, cs.y, v[4 * q + 1]) * lnrs.y;
              v[4 * q + 2] = fmaf(-lnrs.x, cs.z, v[4 * q + 2]) * lnrs.y;
              v[4 * q + 3] = fmaf(-lnrs.x, cs.w, v[4 * q + 3]) * lnrs.y;
            }
          }
        }
        if constexpr (EPI == EPI_QKV_ROPE) bias_prefetch(bq, n0 + c, bias);
        epilogue_bias_act<EPI>(v, bq, bias);
        if (EPI == EPI_QKV_ROPE && n0 + c < rope_cols) {
          if (rope_hd == 80)  // ViT-H/14: compile-time pair indices, ld.shared
            rope_chunk_hd80(v, n0 + c, (uint32_t)__cvta_generic_to_shared(rt), (uint32_t)__cvta_generic_to_shared(ct));
          else
            rope_chunk(v, n0 + c, rope_hd, rt, ct);
        }
        if ((PREC && epi.round_f16)) {  // fp16 storage: fp32 outputs rounded, fp16 outputs saturated
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = (EPI == EPI_F32 || EPI == EPI_F32_F16) ? round_f16(v[j]) : sat_f16(v[j]);
        }
        if constexpr (EPI == EPI_F32_F16) {
          if (ln_stats_out != nullptr && row < M)
            __stcg(ln_stats_out + (size_t)row * ln_parts + ((n0 + c) >> 5), chunk_ln_stats(v));
        }
        if ((EPI == EPI_F32 && epi.wm_scatter) || EPI == EPI_F32_F16) {  // row scatter / 2 outputs: plain stores
          chunk_store_f32(buf, v, reinterpret_cast<float*>(epi.out), epi.ldo, row0, n0 + c, M, epi);
          if (EPI == EPI_F32_F16)
            chunk_store_f16(buf, v, reinterpret_cast<act_t*>(epi.out2), epi.ldo2, row0, n0 + c, M, epi);
          continue;
        }
        if constexpr (RED) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *slot32(buf, lane, q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else if constexpr (RESID) {
          mbar_wait(&rbar[g % NBUF], (g / NBUF) & 1);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float4* sp = slot32(buf, lane, q);
            float4 x = *sp;
            x.x += v[4 * q];
            x.y += v[4 * q + 1];
            x.z += v[4 * q + 2];
            x.w += v[4 * q + 3];
            if ((PREC && epi.round_f16)) x = make_float4(round_f16(x.x), round_f16(x.y), round_f16(x.z), round_f16(x.w));
            *sp = x;
            if constexpr (L::LNO || L::X16) {
              v[4 * q] = x.x;
              v[4 * q + 1] = x.y;
              v[4 * q + 2] = x.z;
              v[4 * q + 3] = x.w;
            }
          }
          if constexpr (L::X16) {  // fp16 copy of the new rows + their LN chunk statistics
            if (row < M) __stcg(ln_stats_out + (size_t)row * ln_parts + ((n0 + c) >> 5), chunk_ln_stats(v));
            float* hb = reinterpret_cast<float*>(smem + L::LN_OFF) + (warp - 4) * 512;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 u;
              u.x = pack_half2(v[8 * q + 0], v[8 * q + 1]);
              u.y = pack_half2(v[8 * q + 2], v[8 * q + 3]);
              u.z = pack_half2(v[8 * q + 4], v[8 * q + 5]);
              u.w = pack_half2(v[8 * q + 6], v[8 * q + 7]);
              *slot16_sw64(hb, lane, q) = u;
            }
          }
          if constexpr (L::LNO) {  // the new residual row values stay in TMEM for the LN passes
            tmem_st16(taddr + c, reinterpret_cast<const uint32_t*>(v));
            tmem_st16(taddr + c + 16, reinterpret_cast<const uint32_t*>(v + 16));
#pragma unroll
            for (int k = 0; k < 32; ++k) ln_sum = __fadd_rn(ln_sum, v[k]);
          }
        } else if constexpr (EPI == EPI_F32 || EPI == EPI_F32_F16) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *slot32(buf, lane, q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 u;
            u.x = pack_half2(v[8 * q + 0], v[8 * q + 1]);
            u.y = pack_half2(v[8 * q + 2], v[8 * q + 3]);
            u.z = pack_half2(v[8 * q + 4], v[8 * q + 5]);
            u.w = pack_half2(v[8 * q + 6], v[8 * q + 7]);
            *slot16_sw64(buf, lane, q) = u;
          }
        }
        fence_proxy_async();  // generic-proxy smem writes -> visible to the TMA (async proxy) store
        __syncwarp();
        if (lane == 0) {
          if (RED) {
            tma_reduce_add_2d(&tmC, buf, n0 + c, row0);
          } else if (RESID || EPI == EPI_F32 || EPI == EPI_F32_F16) {
            tma_store_2d(&tmC, buf, n0 + c, row0);
            if constexpr (L::X16)  // same bulk group: the next chunk's wait_read0 covers both buffers
              tma_store_2d(&tmD, reinterpret_cast<float*>(smem + L::LN_OFF) + (warp - 4) * 512, n0 + c, row0);
          } else {
            tma_store_2d(&tmD, buf, n0 + c, row0);
          }
          tma_store_commit();
        }
      }
      if constexpr (L::LNO) {
        ln_rows_epilogue(taddr, quarter, half, lane, ln_sum, epi.ln_g + n0, epi.ln_b + n0,
                         reinterpret_cast<float*>(smem + L::LN_OFF + 8 * 2 * 2048),
                         reinterpret_cast<float*>(smem + L::LN_OFF) + (warp - 4) * 2 * 512, 512, &tmD, n0, row0);
        tc_fence_before();  // every TMEM read of this accumulator is done: release it
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 1) {
            mbar_arrive(&tempty[acc]);
          } else {
            mbar_arrive_leader(&tempty[acc]);
          }
        }
      }
      // dependency chain: this warp's rows of the unit are stored (CTAs wholly past M -- the second
      // CTA of a pair tile over the last, partial row block -- have no rows to announce)
      if (epi.dep_signal != nullptr && (row0 & ~127) < M) {
        if (lane == 0) {
          bulk_wait_all();
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __threadfence();
          atomicAdd(epi.dep_signal + (row0 >> 7), (bn_eff - half * 32 + 63) / 64);
        }
        __syncwarp();
      }
      if constexpr (L::X16 || EPI == EPI_F32_F16) {
        if (ln_stats_out != nullptr) {  // LN statistics: the warp completing a 32-row group finalises it
          const int nch = (bn_eff - half * 32 + 63) / 64;  // chunks this warp wrote for its 32 rows
          __threadfence();
          __syncwarp();
          int old = 0;
          if (lane == 0) old = atomicAdd(epi.ln_cnt + (row0 >> 5), nch);
          old = __shfl_sync(0xffffffffu, old, 0);
          if (old + nch == ln_parts) {
            __threadfence();
            if (row < M) __stcg(epi.ln_final + row, ln_row_stats(ln_stats_out + (size_t)row * ln_parts, ln_parts));
            if (lane == 0) epi.ln_cnt[row0 >> 5] = 0;
          }
        }
      }
      if constexpr (SPLITK) {
        if (lane == 0) *sk_flag = 0;  // both halves done with this flag: ready for the next launch
      }
      if (warp == 4 && lane == 0) GEMM_STAMP_U(it, 6);  // unit's epilogue done
    }
    if (lane == 0) bulk_wait_all();  // output writes landed before the CTA retires
    if (warp == 4 && lane == 0) GEMM_STAMP(5);
  }
  pdl_launch_dependents();  // this CTA's work is issued: the next kernel may start its prologue
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync_all();  // the peer's MMAs / arrivals are done
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_cg<L::TMEM_COLS, CG>(tmem_base);
  }
  if (threadIdx.x == 0) GEMM_STAMP(7);
}

// ---------------------------------------------------------------------------------------------
// Fused enc-dec MLP (reference _mlp_forward, model.py:505-508, inside _encdec_single :519/:527):
//   x += relu(h W1 + b1) W2 + b2      h [M, 256] fp16, hidden 1024, x [M, 256] fp32 residual
// on a CTA pair (256-row units).  The hidden activations never leave the SM: fc1 runs in eight
// 128-unit slices into two ping-pong TMEM regions, the epilogue warps turn each slice into
// relu(. + b1) fp16 packed in place (the A operand of the TS-form fc2 MMA), and fc2 accumulates
// all eight slices into a 256-column fp32 accumulator that the residual epilogue adds to x.
// TMEM per CTA: [0,128) / [128,256) fc1 slices, [256,512) fc2.  P of a slice: hidden units 64h..64h+63
// packed into columns [64h, 64h+32) of the slice (written by the warp that read those columns).
// The MMA order fc1(0) fc1(1) fc2(0) fc1(2) fc2(1) ... fc1(7) fc2(6) fc2(7) lets the conversion of
// slice e overlap fc1(e+1); an in-order tensor pipe guarantees fc2(e) has read P(e) before
// fc1(e+2) overwrites the region.
// MLP_PROBE (timing probes only, separate builds): bit 0 skips the residual epilogue, bit 1 the
// slice conversion (outputs are garbage; scripts/gpu_mlp_probe.sh)
#ifndef MLP_PROBE
#define MLP_PROBE 0
#endif
// MLP_DEFER 1: the epilogue warps copy the fc2 accumulator into registers and release it at once
// (setmaxnreg: 80 registers for the TMA / MMA warp group, 208 for the two epilogue warp groups);
// the residual add, stores and LayerNorm of unit u then run in pieces between the slice conversions
// of unit u+1, so the next unit's fc2 never waits for them.  0: the accumulator is held through
// the residual / LayerNorm epilogue (A/B builds).
#ifndef MLP_DEFER
#define MLP_DEFER 1
#endif
namespace mlpf {
constexpr int D = 256, HID = 1024, SL = 128, NSL = HID / SL;  // model dims, hidden slice, slices
constexpr int A_BYTES = BM * D * 2;                            // resident h rows of this CTA (64 KB)
constexpr int RING_BYTES = 16384;                              // one W1 (8 KB) or W2 (16 KB) k-block
constexpr int STAGES = 6;
constexpr int OFF_RING = A_BYTES;
constexpr int OFF_EPI = OFF_RING + STAGES * RING_BYTES;
constexpr int OFF_BAR = OFF_EPI + 16 * 4096;
constexpr int OFF_RED = OFF_BAR + 512;  // fused-LN row statistics exchange [4][2][32] floats
constexpr int TOTAL = OFF_RED + 1024 + 1024;
static_assert(TOTAL <= 227 * 1024, "shared memory budget");
}  // namespace mlpf

__global__ void __launch_bounds__(GEMM_THREADS, 1)
    mlp_fused_kernel(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmW1,
                     const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ CUtensorMap tmX,
                     const __grid_constant__ CUtensorMap tmLN, int M, const float* __restrict__ b1,
                     const float* __restrict__ b2, const float* __restrict__ ln_g, const float* __restrict__ ln_b) {
  // ln_g != nullptr: also LayerNorm(x) * ln_g + ln_b of the new residual rows -> tmLN (fp16), the
  // next sub-block's LN, with the same arithmetic as the GEMM's EPI_F32_RESID_LN epilogue
  using namespace mlpf;
  constexpr int CG = 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* empty = full + STAGES;
  uint64_t* a_full = empty + STAGES;
  uint64_t* a_empty = a_full + 1;
  uint64_t* s_full = a_empty + 1;   // [2] fc1 slice accumulated
  uint64_t* p_full = s_full + 2;    // [2] slice converted to P (8 epilogue warps x 2 CTAs)
  uint64_t* o_full = p_full + 2;    // fc2 accumulator complete
  uint64_t* o_empty = o_full + 1;   // fc2 accumulator drained by the residual epilogue
  uint64_t* rfull = o_empty + 1;    // [8 warps][2] residual chunk landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rfull + 16);

  const int warp = warp_id(), lane = lane_id();
  const int rank = (int)cluster_ctarank();
  const int cl = blockIdx.x / CG, ncl = gridDim.x / CG;
  const int num_units = (M + BM * CG - 1) / (BM * CG);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmH);
    tma_prefetch_desc(&tmW1);
    tma_prefetch_desc(&tmW2);
    tma_prefetch_desc(&tmX);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8 * CG);
    }
    mbar_init(o_full, 1);
    mbar_init(o_empty, 8 * CG);
    for (int i = 0; i < 16; ++i) mbar_init(&rfull[i], 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_cg<512, CG>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  // MLP_DEFER register split: every warp of a warp group executes the same setmaxnreg, at the top
  // of its role branch (warps 2 / 3 of the first group have no role after the TMEM allocation)
  auto regs_dec = [] {
    if constexpr (MLP_DEFER) asm volatile("setmaxnreg.dec.sync.aligned.u32 80;\n" ::: "memory");
  };

  // Ring sequence per unit: W1(0) W1(1) W2(0) W1(2) W2(1) ... W1(7) W2(6) W2(7); W1(e) = 4 k-blocks
  // (K = 256), W2(e) = 2 k-blocks (K = 128 hidden units of slice e).
  if (warp == 0) {
    regs_dec();
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      auto ring = [&](const CUtensorMap* map, int c0, int c1, uint32_t bytes) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * bytes);
        tma_load_2d_cg2(smem + OFF_RING + stage * RING_BYTES, map, &full[stage], c0, c1);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      };
      for (int unit = cl; unit < num_units; unit += ncl, ++it) {
        const int m0 = unit * BM * CG + rank * BM;
        mbar_wait(a_empty, (it & 1) ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(a_full, 2 * A_BYTES);
        for (int kb = 0; kb < D / BK; ++kb) tma_load_2d_cg2(smem + kb * (BM * BK * 2), &tmH, a_full, kb * BK, m0);
        auto w1 = [&](int e) {
          for (int kb = 0; kb < D / BK; ++kb) ring(&tmW1, kb * BK, e * SL + rank * (SL / 2), (SL / 2) * BK * 2);
        };
        auto w2 = [&](int e) {
          for (int kb = 0; kb < SL / BK; ++kb) ring(&tmW2, e * SL + kb * BK, rank * (D / 2), (D / 2) * BK * 2);
        };
        w1(0);
        for (int e = 1; e < NSL; ++e) {
          w1(e);
          w2(e - 1);
        }
        w2(NSL - 1);
      }
    }
  } else if (warp == 1) {
    regs_dec();
    if (rank == 0) {  // converged warp, one elected lane issues
      constexpr uint32_t idesc1 = umma_idesc_f16(BM * CG, SL);
      constexpr uint32_t idesc2 = umma_idesc_f16(BM * CG, D);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      auto next = [&]() {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        return smem_u32(smem + OFF_RING + stage * RING_BYTES);
      };
      auto release = [&]() {
        umma_commit_cg<CG>(&empty[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      };
      for (int unit = cl; unit < num_units; unit += ncl, ++it) {
        mbar_wait(a_full, it & 1);
        tc_fence_after();
        const uint32_t a0 = smem_u32(smem);
        auto fc1 = [&](int e) {  // slice e -> TMEM region e & 1
          for (int kb = 0; kb < D / BK; ++kb) {
            const uint64_t da = umma_desc_sw128(a0 + kb * (BM * BK * 2)), db = umma_desc_sw128(next());
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_f16_cg<CG>(tmem + (e & 1) * SL, da + 2 * k, db + 2 * k, idesc1, (kb | k) != 0);
            release();
          }
          umma_commit_cg<CG>(&s_full[e & 1]);
          if (e == NSL - 1) umma_commit_cg<CG>(a_empty);
        };
        auto fc2 = [&](int e) {  // A = P(e) (fp16 packed in region e & 1), accumulate into [256, 512)
          const int use = it * (NSL / 2) + (e >> 1);  // uses of region e & 1 so far
          mbar_wait(&p_full[e & 1], use & 1);
          if (e == 0) mbar_wait(o_empty, (it & 1) ^ 1);
          tc_fence_after();
          for (int kb = 0; kb < SL / BK; ++kb) {
            const uint64_t db = umma_desc_sw128(next());
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              // P of hidden units [64 kb + 16 k, +16) sits at columns 64 kb + 8 k (each epilogue warp
              // packs its 64 units into the first half of its own 64 columns)
              const uint32_t pa = tmem + (e & 1) * SL + kb * 64 + k * 8;
              if constexpr (CG == 2) {
                asm volatile(
                    "{\n\t.reg .pred p, el;\n\t"
                    "setp.ne.b32 p, %4, 0;\n\t"
                    "elect.sync _|el, 0xffffffff;\n\t"
                    "@el tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256),
                    "r"(pa), "l"(db + 2 * k), "r"(idesc2), "r"((e | kb | k) != 0 ? 1u : 0u));
              }
            }
            release();
          }
          if (e == NSL - 1) umma_commit_cg<CG>(o_full);
        };
        fc1(0);
        for (int e = 1; e < NSL; ++e) {
          fc1(e);
          fc2(e - 1);
        }
        fc2(NSL - 1);
      }
    }
  } else if (MLP_DEFER && warp >= 4) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n" ::: "memory");
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    float* bufs = reinterpret_cast<float*>(smem + OFF_EPI) + (warp - 4) * 2048;
    uint64_t* rbar = rfull + (warp - 4) * 2;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const float* const bias1 = b1;  // hoisted kernel parameters (no reloads after asm clobbers)
    const float* const bias2 = b2;
    const float* const lng = ln_g;
    const float* const lnb = ln_b;
    const bool lno = lng != nullptr;
    float* const red = reinterpret_cast<float*>(smem + OFF_RED) + quarter * 64;
    // deferred unit: its fc2 accumulator, then x + acc + b2, chunk i (columns (2 i + half) * 32 + k)
    // at st[32 i + k]; drow0: its first row for this warp
    float st[128];
    int drow0 = 0, g = 0;  // g: residual chunks loaded by this warp (buffer g & 1, phase (g >> 1) & 1)
    bool have = false;
    float ln_sum = 0.f, mu = 0.f, rstd = 0.f;
    auto resid_load = [&](int chunk, int gg) {
      mbar_arrive_expect_tx(&rbar[gg & 1], 32 * 32 * 4);
      tma_load_2d(bufs + (gg & 1) * 1024, &tmX, &rbar[gg & 1], (chunk * 2 + half) * 32, drow0);
    };
    // piece `step` of the deferred epilogue: 0..3 residual chunk `step`, 4 LN statistics, 5 / 6 LN
    // output chunks 0-1 / 2-3 (the same IEEE-pinned arithmetic as ln_rows_epilogue)
    auto defer_step = [&](auto step_c) {
      constexpr int c = decltype(step_c)::value;
      if constexpr (c < 4) {
        const int col = (c * 2 + half) * 32;
        float* buf = bufs + (g & 1) * 1024;
        if (lane == 0 && c < 3) {  // chunk c + 1 into the other buffer (chunk c - 1's store has read it)
          bulk_wait_read0();
          resid_load(c + 1, g + 1);
        }
        __syncwarp();
        const float4* bb = reinterpret_cast<const float4*>(bias2 + col);
        mbar_wait(&rbar[g & 1], (g >> 1) & 1);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 bq = __ldg(bb + q);
          float4* sp = slot32(buf, lane, q);
          float4 x = *sp;
          x.x += st[32 * c + 4 * q] + bq.x;
          x.y += st[32 * c + 4 * q + 1] + bq.y;
          x.z += st[32 * c + 4 * q + 2] + bq.z;
          x.w += st[32 * c + 4 * q + 3] + bq.w;
          *sp = x;
          st[32 * c + 4 * q] = x.x;
          st[32 * c + 4 * q + 1] = x.y;
          st[32 * c + 4 * q + 2] = x.z;
          st[32 * c + 4 * q + 3] = x.w;
        }
        if (lno) {
#pragma unroll
          for (int k = 0; k < 32; ++k) ln_sum = __fadd_rn(ln_sum, st[32 * c + k]);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmX, buf, col, drow0);
          tma_store_commit();
        }
        ++g;
      } else if constexpr (c == 4) {
        if (lno) {
          red[half * 32 + lane] = ln_sum;
          named_bar_sync(2 + quarter, 64);
          mu = __fmul_rn(__fadd_rn(red[lane], red[32 + lane]), 1.0f / 256.0f);
          named_bar_sync(2 + quarter, 64);  // both partners have read the sums before `red` is reused
          float q = 0.f;
#pragma unroll
          for (int k = 0; k < 128; ++k) {
            const float d = __fsub_rn(st[k], mu);
            q = __fmaf_rn(d, d, q);
          }
          red[half * 32 + lane] = q;
          named_bar_sync(2 + quarter, 64);
          const float var = __fmul_rn(__fadd_rn(red[lane], red[32 + lane]), 1.0f / 256.0f);
          named_bar_sync(2 + quarter, 64);
          rstd = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-6f)));
        }
      } else {
        if (lno) {
#pragma unroll
          for (int i = (c - 5) * 2; i < (c - 5) * 2 + 2; ++i) {
            const int cc = half * 32 + 64 * i;
            const float4* g4 = reinterpret_cast<const float4*>(lng + cc);
            const float4* b4 = reinterpret_cast<const float4*>(lnb + cc);
            float y[32];
#pragma unroll
            for (int qq = 0; qq < 8; ++qq) {
              const float4 gg = __ldg(g4 + qq), bb = __ldg(b4 + qq);
              y[4 * qq] = __fmaf_rn(__fmul_rn(__fsub_rn(st[32 * i + 4 * qq], mu), rstd), gg.x, bb.x);
              y[4 * qq + 1] = __fmaf_rn(__fmul_rn(__fsub_rn(st[32 * i + 4 * qq + 1], mu), rstd), gg.y, bb.y);
              y[4 * qq + 2] = __fmaf_rn(__fmul_rn(__fsub_rn(st[32 * i + 4 * qq + 2], mu), rstd), gg.z, bb.z);
              y[4 * qq + 3] = __fmaf_rn(__fmul_rn(__fsub_rn(st[32 * i + 4 * qq + 3], mu), rstd), gg.w, bb.w);
            }
            float* lb = bufs + (i & 1) * 1024;
            if (lane == 0) {  // the stores that last used this staging chunk have read it
              if (i == 0)
                bulk_wait_read0();
              else
                bulk_wait_read1();
            }
            __syncwarp();
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              uint4 u;
              u.x = pack_half2(y[8 * qq + 0], y[8 * qq + 1]);
              u.y = pack_half2(y[8 * qq + 2], y[8 * qq + 3]);
              u.z = pack_half2(y[8 * qq + 4], y[8 * qq + 5]);
              u.w = pack_half2(y[8 * qq + 6], y[8 * qq + 7]);
              *slot16_sw64(lb, lane, qq) = u;
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmLN, lb, cc, drow0);
              tma_store_commit();
            }
          }
        }
      }
    };
    // slice e of the current unit: relu(acc + b1) -> fp16 pairs over the slice's first half (own
    // columns), then piece e of the previous unit's epilogue
    auto slice = [&](auto e_c, int it) {
      constexpr int e = decltype(e_c)::value;
      const int use = it * (NSL / 2) + (e >> 1);
      mbar_wait(&s_full[e & 1], use & 1);
      tc_fence_after();
      const uint32_t rb = lane_base + (e & 1) * SL;
#pragma unroll 1
      for (int c = 0; c < ((MLP_PROBE & 2) ? 0 : 2); ++c) {
        const int col = half * 64 + c * 32;
        float v[32];
        tmem_ld32(rb + col, v);
        tmem_ld_wait();
        const float4* bb = reinterpret_cast<const float4*>(bias1 + e * SL + col);
        uint32_t pk[16];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 bq = __ldg(bb + q);
          pk[2 * q] = pack_half2(fmaxf(v[4 * q] + bq.x, 0.f), fmaxf(v[4 * q + 1] + bq.y, 0.f));
          pk[2 * q + 1] = pack_half2(fmaxf(v[4 * q + 2] + bq.z, 0.f), fmaxf(v[4 * q + 3] + bq.w, 0.f));
        }
        tmem_st16(rb + half * 64 + c * 16, pk);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&p_full[e & 1]);
      if constexpr (e < 7) {
        if (have) defer_step(e_c);
      }
    };
    int it = 0;
    for (int unit = cl; unit < num_units; unit += ncl, ++it) {
      const int row0 = unit * BM * CG + rank * BM + quarter * 32;
      slice(std::integral_constant<int, 0>{}, it);
      slice(std::integral_constant<int, 1>{}, it);
      slice(std::integral_constant<int, 2>{}, it);
      slice(std::integral_constant<int, 3>{}, it);
      slice(std::integral_constant<int, 4>{}, it);
      slice(std::integral_constant<int, 5>{}, it);
      slice(std::integral_constant<int, 6>{}, it);
      slice(std::integral_constant<int, 7>{}, it);
      // the fc2 accumulator into registers, released before any of its epilogue runs
      mbar_wait(o_full, it & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(lane_base + 256 + (c * 2 + half) * 32, st + 32 * c);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(o_empty);
      if constexpr ((MLP_PROBE & 1) != 0) continue;
      drow0 = row0;
      have = true;
      ln_sum = 0.f;
      if (lane == 0) {
        bulk_wait_read0();
        resid_load(0, g);
      }
    }
    if (have) {
      defer_step(std::integral_constant<int, 0>{});
      defer_step(std::integral_constant<int, 1>{});
      defer_step(std::integral_constant<int, 2>{});
      defer_step(std::integral_constant<int, 3>{});
      defer_step(std::integral_constant<int, 4>{});
      defer_step(std::integral_constant<int, 5>{});
      defer_step(std::integral_constant<int, 6>{});
    }
    if (lane == 0) bulk_wait_all();
  } else if (warp >= 4) {
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    float* bufs = reinterpret_cast<float*>(smem + OFF_EPI) + (warp - 4) * 2048;
    uint64_t* rbar = rfull + (warp - 4) * 2;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const float* const bias1 = b1;  // hoisted kernel parameters (no reloads after asm clobbers)
    const float* const bias2 = b2;
    int it = 0, g = 0;  // g: residual chunks processed by this warp
    for (int unit = cl; unit < num_units; unit += ncl, ++it) {
      const int row0 = unit * BM * CG + rank * BM + quarter * 32;
      // residual chunk 0 of this unit, prefetched while the slices are converted
      auto resid_load = [&](int chunk, int gg) {
        mbar_arrive_expect_tx(&rbar[gg & 1], 32 * 32 * 4);
        tma_load_2d(bufs + (gg & 1) * 1024, &tmX, &rbar[gg & 1], (chunk * 2 + half) * 32, row0);
      };
      if (lane == 0) {
        bulk_wait_read0();
        resid_load(0, g);
      }
      // slices: relu(acc + b1) -> fp16 pairs written over the slice's first half (own columns)
      for (int e = 0; e < NSL; ++e) {
        const int use = it * (NSL / 2) + (e >> 1);
        mbar_wait(&s_full[e & 1], use & 1);
        tc_fence_after();
        const uint32_t rb = lane_base + (e & 1) * SL;
#pragma unroll 1
        for (int c = 0; c < ((MLP_PROBE & 2) ? 0 : 2); ++c) {  // this warp: hidden units [64 * half, 64 * half + 64) of the slice
          const int col = half * 64 + c * 32;
          float v[32];
          tmem_ld32(rb + col, v);
          tmem_ld_wait();
          const float4* bb = reinterpret_cast<const float4*>(bias1 + e * SL + col);
          uint32_t pk[16];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 bq = __ldg(bb + q);
            pk[2 * q] = pack_half2(fmaxf(v[4 * q] + bq.x, 0.f), fmaxf(v[4 * q + 1] + bq.y, 0.f));
            pk[2 * q + 1] = pack_half2(fmaxf(v[4 * q + 2] + bq.z, 0.f), fmaxf(v[4 * q + 3] + bq.w, 0.f));
          }
          tmem_st16(rb + half * 64 + c * 16, pk);  // packed P of units [col, col+32): own columns only
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&p_full[e & 1]);
      }
      // residual epilogue: x += acc2 + b2 (this warp: 32-column chunks half, half + 2, ...)
      mbar_wait(o_full, it & 1);
      tc_fence_after();
      if constexpr ((MLP_PROBE & 1) != 0) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(o_empty);
        continue;
      }
      const bool lno = ln_g != nullptr;
      float ln_sum = 0.f;
#pragma unroll 1
      for (int c = 0; c < 4; ++c, ++g) {
        const int col = (c * 2 + half) * 32;
        float* buf = bufs + (g & 1) * 1024;
        if (lane == 0 && c < 3) {
          bulk_wait_read0();
          resid_load(c + 1, g + 1);
        }
        __syncwarp();
        float v[32];
        tmem_ld32(lane_base + 256 + col, v);
        tmem_ld_wait();
        if (c == 3 && !lno) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_leader(o_empty);
        }
        const float4* bb = reinterpret_cast<const float4*>(bias2 + col);
        mbar_wait(&rbar[g & 1], (g >> 1) & 1);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 bq = __ldg(bb + q);
          float4* sp = slot32(buf, lane, q);
          float4 x = *sp;
          x.x += v[4 * q] + bq.x;
          x.y += v[4 * q + 1] + bq.y;
          x.z += v[4 * q + 2] + bq.z;
          x.w += v[4 * q + 3] + bq.w;
          *sp = x;
          v[4 * q] = x.x;
          v[4 * q + 1] = x.y;
          v[4 * q + 2] = x.z;
          v[4 * q + 3] = x.w;
        }
        if (lno) {  // the new residual row values stay in TMEM for the LN passes
          tmem_st16(lane_base + 256 + col, reinterpret_cast<const uint32_t*>(v));
          tmem_st16(lane_base + 256 + col + 16, reinterpret_cast<const uint32_t*>(v + 16));
#pragma unroll
          for (int k = 0; k < 32; ++k) ln_sum = __fadd_rn(ln_sum, v[k]);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmX, buf, col, row0);
          tma_store_commit();
        }
      }
      if (lno) {
        ln_rows_epilogue(lane_base + 256, quarter, half, lane, ln_sum, ln_g, ln_b,
                         reinterpret_cast<float*>(smem + OFF_RED), bufs, 1024, &tmLN, 0, row0);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(o_empty);
      }
    }
    if (lane == 0) bulk_wait_all();
  } else if (warp < 4) {
    regs_dec();  // warps 2 / 3: no role
  }
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_cg<512, CG>(tmem);
  }
}

template <int BN, int STAGES, int EPI, int CG, bool PREC, bool SPLITK>
int launch_gemm(const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tB2, const CUtensorMap& tC,
                const CUtensorMap& tD, int M, int N, int K, const GemmEpi& epi, int num_sms, cudaStream_t stream) {
  using L = GemmSmem<BN, STAGES, EPI, CG>;
  auto kern = gemm_tc_kernel<BN, STAGES, EPI, CG, PREC, SPLITK>;
  static std::atomic<uint64_t> smem_set{0};
  if (const cudaError_t e = set_smem_once(smem_set, kern, L::TOTAL); e != cudaSuccess) return (int)e;
  const int tiles = ((M + BM * CG - 1) / (BM * CG)) * (N / BN) * (SPLITK ? 2 : 1);
  const int units = num_sms / CG;
  const int grid = (tiles < units ? tiles : units) * CG;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = L::TOTAL;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if constexpr (CG == 2) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled() || epi.force_pdl) pdl_attr(attr[na++]);
  cfg.attrs = attr;
  cfg.numAttrs = na;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tA, tB, tB2, tC, tD, M, N, K, epi);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaGetLastError();
}

// Deepest operand ring that fits 227 KB next to the epilogue staging (and RoPE tables).
template <int BN, int EPI, int CG>
constexpr int stages_for() {
  constexpr int stage = BM * BK * 2 + (BN / CG) * BK * 2;
  constexpr int fixed = 8 * 2 * ((EPI == EPI_F16 || EPI == EPI_F16_RELU || EPI == EPI_QKV_ROPE) ? 2048 : 4096) +
                        (EPI == EPI_QKV_ROPE ? 2 * ROPE_MAX_GRID * ROPE_PAD * 8 : 0) +
                        (EPI == EPI_F32_RESID_LN ? 8 * 2 * 2048 + 4 * 2 * 32 * 4 : 0) +
                        (EPI == EPI_F32_RESID_X16 ? 8 * 2048 : 0) + 512 + 1024;
  constexpr int n = (227 * 1024 - fixed) / stage;
  return n > 8 ? 8 : n;
}

template <int BN, int EPI, int CG>
int launch_planned(const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tB2, const CUtensorMap& tC,
                   const CUtensorMap& tD, int M, int N, int K, const GemmEpi& epi, int num_sms, cudaStream_t stream) {
  constexpr int ST = stages_for<BN, EPI, CG>();
  if (epi.acc_f16 || epi.round_f16)
    return launch_gemm<BN, ST, EPI, CG, true, false>(tA, tB, tB2, tC, tD, M, N, K, epi, num_sms, stream);
  if constexpr (EPI != EPI_F32_RESID_LN && (BN == 256 || BN == 128)) {
    if (epi.splitk > 1) return launch_gemm<BN, ST, EPI, CG, false, true>(tA, tB, tB2, tC, tD, M, N, K, epi, num_sms, stream);
  } else if (epi.splitk > 1) {
    return (int)cudaErrorInvalidValue;
  }
  return launch_gemm<BN, ST, EPI, CG, false, false>(tA, tB, tB2, tC, tD, M, N, K, epi, num_sms, stream);
}

template <int BN, int CG>
int dispatch_epi(int epi_mode, const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tB2,
                 const CUtensorMap& tC, const CUtensorMap& tD, int M, int N, int K, const GemmEpi& epi, int num_sms,
                 cudaStream_t stream) {
  switch (epi_mode) {
    case EPI_F16: return launch_planned<BN, EPI_F16, CG>(tA, tB, tB2, tC, tD, M, N, K, epi, num_sms, stream);
    case EPI_F16_RELU: return launch_planned<BN, EPI_F16_RELU, CG>(tA, tB, tB2, tC, tD, M, N, K, epi, num_sms, stream);
    case EPI_F32: return launch_planned<BN, EPI_F32, CG>(tA, tB, tB2, tC, tD, M, N, K, epi, num_sms, stream);
    case EPI_F32_RESID: return launch_planned<BN, EPI_F32_RESID, CG>(tA, tB, tB2, tC, tD, M, N, K, epi, num_sms, stream);
    case EPI_QKV_ROPE: return launch_planned<BN, EPI_QKV_ROPE, CG>(tA, tB, tB2, tC, tD, M, N, K, epi, num_sms, stream);
    case EPI_F32_F16: return launch_planned<BN, EPI_F32_F16, CG>(tA, tB, tB2, tC, tD, M, N, K, epi, num_sms, stream);
    case EPI_F32_RESID_X16:
      return launch_planned<BN, EPI_F32_RESID_X16, CG>(tA, tB, tB2, tC, tD, M, N, K, epi, num_sms, stream);
    case EPI_F32_RESID_LN:
      if constexpr (BN == 256) return launch_planned<BN, EPI_F32_RESID_LN, CG>(tA, tB, tB2, tC, tD, M, N, K, epi, num_sms, stream);
      return (int)cudaErrorInvalidValue;
  }
  return (int)cudaErrorInvalidValue;
}

GemmPlan g_forced{0, 0};  // dart_gemm_force_plan (tests / A-B measurement); bn 0 = automatic
int g_tail_halves = getenv("DART_NO_TAIL_HALVES") == nullptr;
// relative per-column efficiency of the 192 / 160-wide CTA-pair tiles (operand re-reads grow
// as the tile narrows); DART_GEMM_EFF192 / DART_GEMM_EFF160 override for A/B measurement
double env_or(const char* n, double d) {
  const char* e = getenv(n);
  return e ? atof(e) : d;
}
double g_eff192 = env_or("DART_GEMM_EFF192", 0.80), g_eff160 = env_or("DART_GEMM_EFF160", 0.70);  // measured: 192 and 160 lose to 256 on every DART shape

}  // namespace

int mlp_fused(const CUtensorMap& tH, const CUtensorMap& tW1, const CUtensorMap& tW2, const CUtensorMap& tX,
              const CUtensorMap& tLN, int M, const float* b1, const float* b2, const float* ln_g, const float* ln_b,
              int num_sms, cudaStream_t stream) {
  static std::atomic<uint64_t> smem_set{0};
  if (const cudaError_t e = set_smem_once(smem_set, mlp_fused_kernel, mlpf::TOTAL); e != cudaSuccess) return (int)e;
  const int units = (M + 255) / 256, pairs = num_sms / 2;
  const int grid = (units < pairs ? units : pairs) * 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = mlpf::TOTAL;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  int na = 1;
  if (pdl_enabled()) pdl_attr(attr[na++]);
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, mlp_fused_kernel, tH, tW1, tW2, tX, tLN, M, b1, b2, ln_g, ln_b);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaGetLastError();
}

int gemm_bn_for(int N) {
  if (N % 256 == 0) return 256;
  if (N % 128 == 0) return 128;
  if (N % 64 == 0) return 64;
  return 0;
}

// Tile plan minimising wave-quantised work.  Candidates: 1-SM 128 x BN tiles on every SM and
// 2-SM 256 x BN tiles on SM pairs.  cost = waves * BN / eff(BN): narrow tiles pay for operand
// re-reads (measured MMA efficiency relative to BN = 256 on B200: 0.66 at 128, 0.45 at 64);
// the CTA-pair form wins ties (lower operand traffic per FLOP).
GemmPlan gemm_plan(int M, int N, int epi_mode, int num_sms, int splitk) {
  if (epi_mode == EPI_F32_RESID_LN) return GemmPlan{N == 256 ? 256 : 0, 2};  // whole rows per tile
  GemmPlan best{0, 1};
  double best_cost = 0;
  for (int cg = 2; cg >= 1; --cg) {
    for (int bn : {256, 192, 160, 128, 64}) {
      if (N % bn || (cg == 1 && (bn == 192 || bn == 160))) continue;
      if (splitk > 1 && bn != 256 && bn != 128) continue;  // the split-K instantiations
      const long long tiles = (long long)((M + BM * cg - 1) / (BM * cg)) * (N / bn) * splitk;
      const long long units = num_sms / cg;
      const long long waves = (tiles + units - 1) / units;
      const double eff = bn == 256 ? 1.0 : bn == 192 ? g_eff192 : bn == 160 ? g_eff160 : bn == 128 ? 0.66 : 0.45;
      const double cost = (double)waves * bn / eff * (cg == 2 ? 0.97 : 1.0);
      if (best.bn == 0 || cost < best_cost) {
        best = GemmPlan{bn, cg};
        best_cost = cost;
      }
    }
  }
  const GemmPlan o = g_forced;
  if (o.bn > 0 && N % o.bn == 0) best = o;
  return best;
}

void gemm_force_plan(int bn, int cg) { g_forced = GemmPlan{bn, cg == 2 ? 2 : 1}; }

int gemm_set_trace(long long* device_buf) {
  return (int)cudaMemcpyToSymbol(g_gemm_trace, &device_buf, sizeof(device_buf));
}

int gemm_tc(const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap* tB2, const CUtensorMap* tC,
            const CUtensorMap* tD, int M, int N, int K, GemmPlan plan, int epi_mode, const GemmEpi& epi_in, int num_sms,
            cudaStream_t stream) {
  GemmEpi epi = epi_in;
  if (M <= 0) return 0;
  const int BN = plan.bn;
  if (K % BK != 0 || N % BN != 0) return (int)cudaErrorInvalidValue;
  if (epi.splitk != 1 && (epi.splitk != 2 || epi_mode == EPI_F32_RESID_LN || (K / BK) % 2 != 0 || !epi.tile_flags ||
                          !epi.ws || epi.acc_f16 || epi.round_f16 || (BN != 256 && BN != 128)))
    return (int)cudaErrorInvalidValue;
  if (epi_mode == EPI_QKV_ROPE && (epi.rope_grid <= 0 || epi.rope_grid > ROPE_MAX_GRID ||
                                   epi.rope_grid * epi.rope_grid != epi.rope_T || epi.rope_hd % 4 != 0 ||
                                   epi.rope_hd / 4 > ROPE_MAX_Q))
    return (int)cudaErrorInvalidValue;
  const bool f32_out = epi_mode == EPI_F32_RESID || epi_mode == EPI_F32_RESID_LN || epi_mode == EPI_F32_RESID_X16 ||
                       (epi_mode == EPI_F32 && !epi.wm_scatter);
  const bool f16_out = epi_mode == EPI_F16 || epi_mode == EPI_F16_RELU || epi_mode == EPI_QKV_ROPE ||
                       epi_mode == EPI_F32_RESID_LN || epi_mode == EPI_F32_RESID_X16;
  // LN fold: statistics per 32-column chunk, full chunks only; the fp16 copy rides on tD
  if ((epi_mode == EPI_F32_RESID_X16 || epi.ln_stats_out) &&
      (!epi.ln_stats_out || !epi.ln_cnt || !epi.ln_final || epi.ln_parts * 32 != N || epi.ln_parts % 2))
    return (int)cudaErrorInvalidValue;
  if (epi.ln_stats && (!epi.ln_colsum || (epi_mode != EPI_QKV_ROPE && epi_mode != EPI_F16_RELU)))
    return (int)cudaErrorInvalidValue;
  if (epi_mode == EPI_F32_RESID_LN && (N != BN || BN != 256 || !epi.ln_g || !epi.ln_b)) return (int)cudaErrorInvalidValue;
  if ((f32_out && !tC) || (f16_out && !tD)) return (int)cudaErrorInvalidValue;
  const CUtensorMap& c = tC ? *tC : tA;
  const CUtensorMap& d = tD ? *tD : tA;
  const CUtensorMap& b2 = tB2 ? *tB2 : tB;
  // tail halves: when the tiles leave a last wave at most half full, run it as half-width units
  epi.tail_full = 0;
  if (tB2 && g_tail_halves && epi.splitk == 1 && (BN == 256 || BN == 128) && epi_mode != EPI_F32_RESID_LN) {
    const int tiles = ((M + BM * plan.cg - 1) / (BM * plan.cg)) * (N / BN);
    const int units = num_sms / plan.cg;
    const int rem = tiles % units;
    if (tiles > units && rem > 0 && 2 * rem <= units) epi.tail_full = tiles - rem;
  }
  if (plan.cg == 2) {
    switch (BN) {
      case 256: return dispatch_epi<256, 2>(epi_mode, tA, tB, b2, c, d, M, N, K, epi, num_sms, stream);
      case 192: return dispatch_epi<192, 2>(epi_mode, tA, tB, b2, c, d, M, N, K, epi, num_sms, stream);
      case 160: return dispatch_epi<160, 2>(epi_mode, tA, tB, b2, c, d, M, N, K, epi, num_sms, stream);
      case 128: return dispatch_epi<128, 2>(epi_mode, tA, tB, b2, c, d, M, N, K, epi, num_sms, stream);
      case 64: return dispatch_epi<64, 2>(epi_mode, tA, tB, b2, c, d, M, N, K, epi, num_sms, stream);
    }
  } else {
    switch (BN) {
      case 256: return dispatch_epi<256, 1>(epi_mode, tA, tB, b2, c, d, M, N, K, epi, num_sms, stream);
      case 128: return dispatch_epi<128, 1>(epi_mode, tA, tB, b2, c, d, M, N, K, epi, num_sms, stream);
      case 64: return dispatch_epi<64, 1>(epi_mode, tA, tB, b2, c, d, M, N, K, epi, num_sms, stream);
    }
  }
  return (int)cudaErrorInvalidValue;
}

}  // namespace dart
