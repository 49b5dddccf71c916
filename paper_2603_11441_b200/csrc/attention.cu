// Flash attention, fp16 operands / fp32 online softmax, for every attention on the
// DART hot path:
//   backbone windowed + global self-attention, hd = 80 (reference model.py:390-409)
//   enc-dec self / cross / decoder attention, hd = 16   (reference model.py:491-502)
// softmax(q k^T / sqrt(hd)) v with max-subtraction (tensors.py:194-197) computed online
// in exp2 space.  Operands are read in place through strides (token / head / batch),
// so the QKV / KV GEMM outputs need no transposes; windowed blocks map in-window
// indices to tokens on the fly (reference _window_partition, model.py:375-387).
//
// This is the first correct sm_100a path: m16n8k16 mma.sync fragments, cp.async
// double-buffered K/V tiles of 64 keys, 16 query rows per warp.
#include "common.cuh"
#include "kernels.h"

namespace dart {
namespace {

constexpr int BKV = 64;

__device__ __forceinline__ long long tok_offset(int z, int i, long long batch_stride, int tok_stride,
                                                long long img_stride, int win, int grid, int nwin) {
  if (win == 0) return (long long)z * batch_stride + (long long)i * tok_stride;
  const int img = z / nwin, w = z - img * nwin;
  const int wpr = grid / win;
  const int r = (w / wpr) * win + i / win;
  const int c = (w % wpr) * win + i % win;
  return (long long)img * img_stride + (long long)(r * grid + c) * tok_stride;
}

template <int HD, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, HD == 16 ? 6 : 1) flash_attn_kernel(AttnArgs a) {
  constexpr int BQ = 16 * WARPS;
  constexpr int PITCH = HD + 8;  // halves; breaks ldmatrix bank conflicts
  constexpr int CH = HD / 8;     // 16-byte chunks per row
  constexpr int KSTEPS = HD / 16;
  constexpr int NT_O = HD / 8;   // output n-tiles
  extern __shared__ __align__(128) __half smem_attn[];
  __half* sQ = smem_attn;
  __half (*sK)[BKV * PITCH] = reinterpret_cast<__half (*)[BKV * PITCH]>(smem_attn + BQ * PITCH);
  __half (*sV)[BKV * PITCH] = reinterpret_cast<__half (*)[BKV * PITCH]>(smem_attn + BQ * PITCH + 2 * BKV * PITCH);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int z = blockIdx.z, h = blockIdx.y;
  const int q0 = blockIdx.x * BQ;

  const __half* qb = a.q + (long long)h * a.head_stride_q;
  const int zkv = a.kv_batch_mod > 0 ? z % a.kv_batch_mod : z;
  const __half* kb = a.k + (long long)h * a.head_stride_k;
  const __half* vb = a.v + (long long)h * a.head_stride_v;

  // ---- Q tile
  for (int idx = tid; idx < BQ * CH; idx += WARPS * 32) {
    const int r = idx / CH, c = idx % CH;
    const int qi = q0 + r;
    const bool ok = qi < a.Lq;
    const __half* src = qb + (ok ? tok_offset(z, qi, a.q_batch_stride, a.q_tok_stride, a.img_stride_q, a.win, a.grid, a.nwin) : 0) + c * 8;
    cp_async16(smem_u32(&sQ[r * PITCH + c * 8]), src, ok);
  }
  // K/V tile loads.  Dense items (win == 0, every enc-dec call) use per-thread source
  // pointers computed once; only the tile offset is added per tile.
  constexpr int NT = WARPS * 32;
  constexpr int NL = (BKV * CH + NT - 1) / NT;  // 16-byte chunks per thread per tile
  const __half* kp[NL];
  const __half* vp[NL];
  int krow[NL];
  uint32_t soff[NL];
#pragma unroll
  for (int i = 0; i < NL; ++i) {
    const int idx = tid + i * NT;
    const int r = idx / CH, cc = idx % CH;  // compile-time divisors
    krow[i] = idx < BKV * CH ? r : 1 << 30;
    soff[i] = (uint32_t)(r * PITCH + cc * 8);
    kp[i] = kb + (long long)zkv * a.k_batch_stride + (long long)r * a.k_tok_stride + cc * 8;
    vp[i] = vb + (long long)zkv * a.v_batch_stride + (long long)r * a.v_tok_stride + cc * 8;
  }
  const long long k_step = (long long)BKV * a.k_tok_stride, v_step = (long long)BKV * a.v_tok_stride;
  auto load_kv = [&](int buf, int kt) {
    if (a.win == 0) {
#pragma unroll
      for (int i = 0; i < NL; ++i) {
        if (krow[i] >= BKV) continue;
        const bool ok = kt * BKV + krow[i] < a.Lk;
        cp_async16(smem_u32(&sK[buf][soff[i]]), ok ? kp[i] + kt * k_step : kb, ok);
        cp_async16(smem_u32(&sV[buf][soff[i]]), ok ? vp[i] + kt * v_step : vb, ok);
      }
      return;
    }
    for (int idx = tid; idx < BKV * CH; idx += WARPS * 32) {
      const int r = idx / CH, c = idx % CH;
      const int ki = kt * BKV + r;
      const bool ok = ki < a.Lk;
      const long long ko = ok ? tok_offset(zkv, ki, a.k_batch_stride, a.k_tok_stride, a.img_stride_k, a.win, a.grid, a.nwin) : 0;
      const long long vo = ok ? tok_offset(zkv, ki, a.v_batch_stride, a.v_tok_stride, a.img_stride_v, a.win, a.grid, a.nwin) : 0;
      cp_async16(smem_u32(&sK[buf][r * PITCH + c * 8]), kb + ko + c * 8, ok);
      cp_async16(smem_u32(&sV[buf][r * PITCH + c * 8]), vb + vo + c * 8, ok);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  // V pad columns [HD, HD+8) hold ones: the extra PV n-tile then accumulates the softmax
  // row sum on the tensor core (no per-element FADD), consistent with the fp16 P used for O.
  for (int idx = tid; idx < 2 * BKV; idx += WARPS * 32) {
    const int b = idx / BKV, r = idx % BKV;
    *reinterpret_cast<uint4*>(&sV[b][r * PITCH + HD]) = make_uint4(0x3C003C00u, 0x3C003C00u, 0x3C003C00u, 0x3C003C00u);
  }

  const int nkt = (a.Lk + BKV - 1) / BKV;
  uint32_t qf[KSTEPS][4];
  float o[NT_O + 1][4];
#pragma unroll
  for (int n = 0; n <= NT_O; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY};  // running max of raw scores
  const float c = a.scale_log2;            // exp(s/sqrt(hd) - m) = exp2(s*c - m*c)
  const int t = lane & 3;

  for (int kt = 0; kt < nkt; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nkt) load_kv(buf ^ 1, kt + 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int ks = 0; ks < KSTEPS; ++ks) {
        const int row = warp * 16 + (lane & 15);
        const int col = ks * 16 + (lane >> 4) * 8;
        ldmatrix_x4(qf[ks], smem_u32(&sQ[row * PITCH + col]));
      }
    }
    // ---- S = Q K^T (16 x 64 per warp, raw scores)
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int np = 0; np < 4; ++np) {  // pairs of 8-key n-tiles
#pragma unroll
      for (int ks = 0; ks < KSTEPS; ++ks) {
        uint32_t b[4];
        const int key = np * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int dim = ks * 16 + ((lane >> 3) & 1) * 8;
        ldmatrix_x4(b, smem_u32(&sK[buf][key * PITCH + dim]));
        mma16816(s[2 * np], qf[ks], b);
        mma16816(s[2 * np + 1], qf[ks], b + 2);
      }
    }
    const int kbase = kt * BKV;
    if (kbase + BKV > a.Lk) {  // partial tile only
#pragma unroll
      for (int n = 0; n < 8; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (kbase + n * 8 + 2 * t + (e & 1) >= a.Lk) s[n][e] = -INFINITY;
    }
    // ---- online softmax
    float mx0 = fmax3f(s[0][0], s[0][1], m_r[0]);
    float mx1 = fmax3f(s[0][2], s[0][3], m_r[1]);
#pragma unroll
    for (int n = 1; n < 8; ++n) {
      mx0 = fmax3f(mx0, s[n][0], s[n][1]);
      mx1 = fmax3f(mx1, s[n][2], s[n][3]);
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, 2));
    const float corr0 = fast_exp2((m_r[0] - mx0) * c);
    const float corr1 = fast_exp2((m_r[1] - mx1) * c);
    m_r[0] = mx0;
    m_r[1] = mx1;
    const float nb0 = -mx0 * c, nb1 = -mx1 * c;
    uint32_t p[4][4];
    // hd 16 is exp-bound: the last POLY n-tiles (POLY/8 of the exps) use the FMA-pipe exp2
    constexpr int POLY = 0;  // measured: the hd-16 kernel is issue-bound, not MUFU-bound (poly made it slower)
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float p0, p1, p2, p3;
      if (n >= 8 - POLY) {
        p0 = exp2_poly(fmaf(s[n][0], c, nb0));
        p1 = exp2_poly(fmaf(s[n][1], c, nb0));
        p2 = exp2_poly(fmaf(s[n][2], c, nb1));
        p3 = exp2_poly(fmaf(s[n][3], c, nb1));
      } else {
        p0 = fast_exp2(fmaf(s[n][0], c, nb0));
        p1 = fast_exp2(fmaf(s[n][1], c, nb0));
        p2 = fast_exp2(fmaf(s[n][2], c, nb1));
        p3 = fast_exp2(fmaf(s[n][3], c, nb1));
      }
      p[n >> 1][(n & 1) * 2 + 0] = pack_half2(p0, p1);
      p[n >> 1][(n & 1) * 2 + 1] = pack_half2(p2, p3);
    }
#pragma unroll
    for (int n = 0; n <= NT_O; ++n) {
      o[n][0] *= corr0;
      o[n][1] *= corr0;
      o[n][2] *= corr1;
      o[n][3] *= corr1;
    }
    // ---- O += P [V | 1]
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t pa[4] = {p[ks][0], p[ks][1], p[ks][2], p[ks][3]};
      const int key = ks * 16 + (lane & 15);
#pragma unroll
      for (int np = 0; np < NT_O / 2; ++np) {
        uint32_t b[4];
        const int dim = np * 16 + (lane >> 4) * 8;
        ldmatrix_x4_trans(b, smem_u32(&sV[buf][key * PITCH + dim]));
        mma16816(o[2 * np], pa, b);
        mma16816(o[2 * np + 1], pa, b + 2);
      }
      uint32_t b1[2];
      ldmatrix_x2_trans(b1, smem_u32(&sV[buf][key * PITCH + HD]));
      mma16816(o[NT_O], pa, b1);
    }
    __syncthreads();
  }
  // ---- normalise by the tensor-core row sum and store
  const int g = lane >> 2;
  const float inv0 = 1.f / o[NT_O][0], inv1 = 1.f / o[NT_O][2];
  __half* ob = a.o + (long long)h * a.head_stride_o;
  const int r0 = q0 + warp * 16 + g, r1 = r0 + 8;
  if (r0 < a.Lq) {
    __half* dst = ob + tok_offset(z, r0, a.o_batch_stride, a.o_tok_stride, a.img_stride_o, a.win, a.grid, a.nwin);
#pragma unroll
    for (int n = 0; n < NT_O; ++n)
      *reinterpret_cast<uint32_t*>(dst + n * 8 + 2 * t) = pack_half2(o[n][0] * inv0, o[n][1] * inv0);
  }
  if (r1 < a.Lq) {
    __half* dst = ob + tok_offset(z, r1, a.o_batch_stride, a.o_tok_stride, a.img_stride_o, a.win, a.grid, a.nwin);
#pragma unroll
    for (int n = 0; n < NT_O; ++n)
      *reinterpret_cast<uint32_t*>(dst + n * 8 + 2 * t) = pack_half2(o[n][2] * inv1, o[n][3] * inv1);
  }
}

// Short-key attention for the encoder's text cross-attention (hd 16, <= 32 text tokens,
// reference model.py:518 via _mha :491-502): one CTA = 64 query rows of one item x ALL heads,
// so the query rows are read once as full 512-byte lines and the class's text K / V
// (32 x heads*16) are staged once per CTA instead of once per (row block, head).  Warp w: 16
// rows (w & 3) x half of the heads (w >> 2); per head S = Q_h K_h^T (4 mma.sync), exact softmax
// over the 32 keys in registers (quad shuffles), O_h = P V_h (4 mma.sync), written back over
// Q_h in shared memory, then one coalesced store of the output tile.
constexpr int XS_ROWS = 64, XS_LK = 32, XS_PITCH = 256 + 8;

__global__ void __launch_bounds__(256, 3) xattn_short_kernel(AttnArgs a) {
  extern __shared__ __align__(128) __half smem_xs[];
  __half* sQ = smem_xs;                          // [XS_ROWS][XS_PITCH]
  __half* sK = sQ + XS_ROWS * XS_PITCH;          // [XS_LK][XS_PITCH]
  __half* sV = sK + XS_LK * XS_PITCH;            // [XS_LK][XS_PITCH]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int z = blockIdx.y, q0 = blockIdx.x * XS_ROWS;
  const int E = a.heads * 16, CH = E / 8;
  const int zkv = a.kv_batch_mod > 0 ? z % a.kv_batch_mod : z;
  for (int idx = tid; idx < XS_LK * CH; idx += 256) {
    const int r = idx / CH, c = idx % CH;
    const bool ok = r < a.Lk;
    const long long kr = (long long)zkv * a.k_batch_stride + (long long)r * a.k_tok_stride + c * 8;
    const long long vr = (long long)zkv * a.v_batch_stride + (long long)r * a.v_tok_stride + c * 8;
    cp_async16(smem_u32(&sK[r * XS_PITCH + c * 8]), ok ? a.k + kr : a.k, ok);
    cp_async16(smem_u32(&sV[r * XS_PITCH + c * 8]), ok ? a.v + vr : a.v, ok);
  }
  for (int idx = tid; idx < XS_ROWS * CH; idx += 256) {
    const int r = idx / CH, c = idx % CH;
    const int qi = q0 + r;
    const bool ok = qi < a.Lq;
    const long long qo = (long long)z * a.q_batch_stride + (long long)qi * a.q_tok_stride + c * 8;
    cp_async16(smem_u32(&sQ[r * XS_PITCH + c * 8]), ok ? a.q + qo : a.q, ok);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const float c = a.scale_log2;
  const int t = lane & 3, g = lane >> 2;
  __half* rowbase = sQ + ((warp & 3) * 16) * XS_PITCH;
  const int hh = (a.heads + 1) >> 1, h_lo = (warp >> 2) * hh, h_hi = min(a.heads, h_lo + hh);
#pragma unroll 1
  for (int h = h_lo; h < h_hi; ++h) {
    uint32_t qa[4];
    ldmatrix_x4(qa, smem_u32(&rowbase[(lane & 15) * XS_PITCH + h * 16 + (lane >> 4) * 8]));
    float s[4][4];
#pragma unroll
    for (int n = 0; n < 4; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int np = 0; np < 2; ++np) {
      uint32_t b[4];
      const int key = np * 16 + (lane & 7) + ((lane >> 4) << 3);
      const int dim = h * 16 + ((lane >> 3) & 1) * 8;
      ldmatrix_x4(b, smem_u32(&sK[key * XS_PITCH + dim]));
      mma16816(s[2 * np], qa, b);
      mma16816(s[2 * np + 1], qa, b + 2);
    }
    if (a.Lk < XS_LK) {
#pragma unroll
      for (int n = 0; n < 4; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (n * 8 + 2 * t + (e & 1) >= a.Lk) s[n][e] = -INFINITY;
    }
    float mx0 = fmax3f(s[0][0], s[0][1], s[1][0]), mx1 = fmax3f(s[0][2], s[0][3], s[1][2]);
    mx0 = fmax3f(mx0, s[1][1], s[2][0]);
    mx1 = fmax3f(mx1, s[1][3], s[2][2]);
    mx0 = fmax3f(mx0, s[2][1], s[3][0]);
    mx1 = fmax3f(mx1, s[2][3], s[3][2]);
    mx0 = fmaxf(mx0, s[3][1]);
    mx1 = fmaxf(mx1, s[3][3]);
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float nb0 = -mx0 * c, nb1 = -mx1 * c;
    uint32_t pa[2][4];
    float l0 = 0.f, l1 = 0.f;
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      const __half2 h01 = __floats2half2_rn(fast_exp2(fmaf(s[n][0], c, nb0)), fast_exp2(fmaf(s[n][1], c, nb0)));
      const __half2 h23 = __floats2half2_rn(fast_exp2(fmaf(s[n][2], c, nb1)), fast_exp2(fmaf(s[n][3], c, nb1)));
      const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);  // sum what P.V multiplies
      l0 += f01.x + f01.y;
      l1 += f23.x + f23.y;
      pa[n >> 1][(n & 1) * 2 + 0] = *reinterpret_cast<const uint32_t*>(&h01);
      pa[n >> 1][(n & 1) * 2 + 1] = *reinterpret_cast<const uint32_t*>(&h23);
    }
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    float o[2][4];
#pragma unroll
    for (int n = 0; n < 2; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      uint32_t b[4];
      ldmatrix_x4_trans(b, smem_u32(&sV[(ks * 16 + (lane & 15)) * XS_PITCH + h * 16 + (lane >> 4) * 8]));
      mma16816(o[0], pa[ks], b);
      mma16816(o[1], pa[ks], b + 2);
    }
    const float inv0 = 1.f / l0, inv1 = 1.f / l1;
    __syncwarp();  // every lane has read Q_h of these rows (ldmatrix above) before it is overwritten
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      *reinterpret_cast<uint32_t*>(&rowbase[g * XS_PITCH + h * 16 + n * 8 + 2 * t]) =
          pack_half2(o[n][0] * inv0, o[n][1] * inv0);
      *reinterpret_cast<uint32_t*>(&rowbase[(g + 8) * XS_PITCH + h * 16 + n * 8 + 2 * t]) =
          pack_half2(o[n][2] * inv1, o[n][3] * inv1);
    }
  }
  __syncthreads();
  for (int idx = tid; idx < XS_ROWS * CH; idx += 256) {
    const int r = idx / CH, cc = idx % CH;
    const int qi = q0 + r;
    if (qi < a.Lq)
      *reinterpret_cast<uint4*>(a.o + (long long)z * a.o_batch_stride + (long long)qi * a.o_tok_stride + cc * 8) =
          *reinterpret_cast<const uint4*>(&sQ[r * XS_PITCH + cc * 8]);
  }
}

template <int HD>
int launch(const AttnArgs& a, cudaStream_t stream) {
  constexpr int WARPS = 4;
  constexpr int SMEM = (16 * WARPS + 4 * BKV) * (HD + 8) * 2;
  static std::atomic<uint64_t> smem_set{0};
  if (const cudaError_t e = set_smem_once(smem_set, flash_attn_kernel<HD, WARPS>, SMEM); e != cudaSuccess) return (int)e;
  dim3 grid((a.Lq + 16 * WARPS - 1) / (16 * WARPS), a.heads, a.batch);
  flash_attn_kernel<HD, WARPS><<<grid, WARPS * 32, SMEM, stream>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace

bool attention_short_supported(const AttnArgs& a, int head_dim) {
  // below ~2 waves of 64-row CTAs the per-(row block, head) kernel's finer grid wins (N=4: 19 vs 23 us)
  const long long ctas = (long long)((a.Lq + XS_ROWS - 1) / XS_ROWS) * a.batch;
  return head_dim == 16 && a.win == 0 && ctas >= 1000 && a.Lk >= 1 && a.Lk <= XS_LK && a.heads * 16 <= 256 &&
         a.head_stride_q == 16 && a.head_stride_k == 16 && a.head_stride_v == 16 && a.head_stride_o == 16 &&
         a.q_tok_stride % 8 == 0 && a.k_tok_stride % 8 == 0 && a.v_tok_stride % 8 == 0 && a.o_tok_stride % 8 == 0;
}

int attention_short(const AttnArgs& a, cudaStream_t stream) {
  constexpr int SMEM = (XS_ROWS + 2 * XS_LK) * XS_PITCH * 2;
  static std::atomic<uint64_t> smem_set{0};
  if (const cudaError_t e = set_smem_once(smem_set, xattn_short_kernel, SMEM); e != cudaSuccess) return (int)e;
  dim3 grid((a.Lq + XS_ROWS - 1) / XS_ROWS, a.batch);
  xattn_short_kernel<<<grid, 256, SMEM, stream>>>(a);
  return (int)cudaGetLastError();
}

int attention(const AttnArgs& a, int head_dim, cudaStream_t stream) {
  if (a.Lq <= 0 || a.batch <= 0) return 0;
  if (attention_short_supported(a, head_dim)) return attention_short(a, stream);
  switch (head_dim) {
    case 16: return launch<16>(a, stream);
    case 32: return launch<32>(a, stream);
    case 64: return launch<64>(a, stream);
    case 80: return launch<80>(a, stream);
  }
  return (int)cudaErrorInvalidValue;
}

}  // namespace dart
