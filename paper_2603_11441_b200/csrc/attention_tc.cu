// tcgen05 / TMEM flash attention, sm_100a: backbone windowed/global self-attention (hd 80)
// and the enc-dec encoder self-attention / decoder cross-attention (hd 16).
//
// softmax(q k^T / sqrt(hd)) v  (reference model.py:390-409 backbone, model.py:491-501 _mha).
// Every attention item is a contiguous row block of a token-major buffer (the backbone stream
// is window-major, dart_capi.cu), so all tiles are plain 2-D TMA boxes.
//
// Persistent CTAs (CTAS per SM) loop over items (q-tile of 128 rows, head, window/image/class).
//   warp 0     TMEM allocator; lane 0 is the TMA producer: Q (double-buffered, once per item)
//              and K / V tiles of BKV keys in a STAGES-deep ring with separate K and V
//              barriers (K is released as soon as S = QK^T has consumed it).  Operands are
//              16-dim column blocks with 32-byte swizzle.
//   warp 1     MMA issuer (one thread):  S_j = Q K_j^T -> TMEM (double buffered, BKV cols)
//                                        O  += P_j [V_j | 1]  (A = P read from TMEM, B = V in
//                                        smem, MN-major; the ones block makes column HD of O
//                                        the softmax row sum on the tensor core)
//   warps 2-5  softmax: one thread per query row (TMEM lane quarter = warp & 3).  The whole
//              S tile is loaded into registers once, row max by an 8-way max3 tree, P = 2^x of
//              the FFMA-scaled scores written back over S as packed fp16.  NPOLY of every 16
//              exponentials run as a degree-3 polynomial on the FMA pipe (exp2_poly) instead of
//              MUFU, balancing the two pipes (MUFU = 16/clk/SM is the hd-16 roof).  O is
//              rescaled lazily, only when the running max grows by more than 2^8 (P <= 256).
#include "common.cuh"
#include "kernels.h"

namespace dart {
namespace {

constexpr int BQ = 128;
constexpr float RESCALE_LOG2 = 8.0f;

__device__ __forceinline__ uint64_t desc_sw32(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  d |= (uint64_t)6 << 61;  // SWIZZLE_32B
  return d;
}

template <int HD, int BKV, int STAGES, int CTAS, int NS, int SPLIT>
struct FaCfg {
  static constexpr int NB = HD / 16;                 // 16-dim column blocks
  static constexpr int ON = HD + 16;                 // O columns (values + row-sum block)
  static constexpr int OCOL = NS * BKV;              // TMEM column of O
  static constexpr int TMEM_NEED = NS * BKV + ON;
  static constexpr int TMEM = TMEM_NEED <= 32 ? 32 : TMEM_NEED <= 64 ? 64 : TMEM_NEED <= 128 ? 128
                              : TMEM_NEED <= 256 ? 256 : 512;
  static_assert(TMEM_NEED <= 512 && TMEM * CTAS <= 512, "TMEM budget");
  static_assert(BKV % (8 * SPLIT) == 0 && (BKV / SPLIT) % 8 == 0, "S tile split into 8-column pieces");
  static constexpr int THREADS = 64 + 128 * SPLIT;  // TMA/alloc warp, MMA warp, 4*SPLIT softmax warps
  static constexpr int COLS = BKV / SPLIT;           // S columns per softmax warp
  static constexpr int Q_BLOCK = BQ * 32;            // bytes per Q column block
  static constexpr int KV_BLOCK = BKV * 32;          // bytes per K/V column block
  static constexpr int Q_BYTES = NB * Q_BLOCK;
  static constexpr int K_BYTES = NB * KV_BLOCK;
  static constexpr int V_BYTES = (NB + 1) * KV_BLOCK;  // + ones block
  static constexpr int OFF_K = 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + STAGES * K_BYTES;
  static constexpr int OFF_BAR = OFF_V + STAGES * V_BYTES;
  static constexpr int NBARS = 4 + 4 * STAGES + 3 * NS;
  static constexpr int OFF_RED = OFF_BAR + NBARS * 8 + 16;  // [2][SPLIT][128] partial row maxima
  static constexpr int TOTAL = OFF_RED + (SPLIT > 1 ? 2 * SPLIT * BQ * 4 : 0) + 1024;
  static_assert(TOTAL * CTAS <= 227 * 1024, "shared memory budget");
};

template <int HD, int BKV, int STAGES, int CTAS, int NS, int SPLIT, int NPOLY>
__global__ void __launch_bounds__(FaCfg<HD, BKV, STAGES, CTAS, NS, SPLIT>::THREADS, CTAS)
    fa_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV, AttnTcArgs a) {
  using L = FaCfg<HD, BKV, STAGES, CTAS, NS, SPLIT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bars;                 // 2
  uint64_t* q_empty = bars + 2;            // 2
  uint64_t* k_full = bars + 4;             // STAGES
  uint64_t* k_empty = k_full + STAGES;     // STAGES
  uint64_t* v_full = k_empty + STAGES;     // STAGES
  uint64_t* v_empty = v_full + STAGES;     // STAGES
  uint64_t* s_full = v_empty + STAGES;     // NS
  uint64_t* p_full = s_full + NS;          // NS
  uint64_t* o_done = p_full + NS;          // NS
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + NS);

  const int warp = warp_id(), lane = lane_id();
  const int q_tiles = (a.Lq + BQ - 1) / BQ;
  const int n_items = q_tiles * a.heads * a.items;
  const int nkv = a.Lkv / BKV;

  if (warp == 1 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmKV);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 4 * SPLIT);
      mbar_init(&o_done[s], 1);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    fence_barrier_init();
  }
  // ones block of every V stage (column block NB): the row-sum column of O
  for (int i = threadIdx.x; i < STAGES * BKV * 4; i += blockDim.x) {
    const int s = i / (BKV * 4), r = i % (BKV * 4);
    reinterpret_cast<uint2*>(smem + L::OFF_V + s * L::V_BYTES + L::NB * L::KV_BLOCK)[r] =
        make_uint2(0x3C003C00u, 0x3C003C00u);
  }
  fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core (async proxy)
  if (warp == 0) tmem_alloc<L::TMEM>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0, g = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        const int qt = item % q_tiles;
        const int h = (item / q_tiles) % a.heads;
        const int z = item / (q_tiles * a.heads);
        const int row0 = z * a.Lkv;
        const int qb = it & 1;
        mbar_wait_dbg(&q_empty[qb], ((it >> 1) & 1) ^ 1, 1000000 + it, a.dbg);
        mbar_arrive_expect_tx(&q_full[qb], L::Q_BYTES);
        for (int b = 0; b < L::NB; ++b)
          tma_load_2d(smem + qb * L::Q_BYTES + b * L::Q_BLOCK, &tmQ, &q_full[qb], a.q_col + h * HD + b * 16,
                      z * a.Lq + qt * BQ);
        for (int j = 0; j < nkv; ++j, ++g) {
          const int st = g % STAGES;
          const uint32_t ph = ((g / STAGES) & 1) ^ 1;
          uint8_t* sk = smem + L::OFF_K + st * L::K_BYTES;
          uint8_t* sv = smem + L::OFF_V + st * L::V_BYTES;
          mbar_wait_dbg(&k_empty[st], ph, 2000000 + g, a.dbg);
          mbar_arrive_expect_tx(&k_full[st], L::K_BYTES);
          for (int b = 0; b < L::NB; ++b)
            tma_load_2d(sk + b * L::KV_BLOCK, &tmKV, &k_full[st], a.k_col + h * HD + b * 16, row0 + j * BKV);
          mbar_wait_dbg(&v_empty[st], ph, 2500000 + g, a.dbg);
          mbar_arrive_expect_tx(&v_full[st], L::K_BYTES);
          for (int b = 0; b < L::NB; ++b)
            tma_load_2d(sv + b * L::KV_BLOCK, &tmKV, &v_full[st], a.v_col + h * HD + b * 16, row0 + j * BKV);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_f16(BQ, BKV);
      constexpr uint32_t idesc_pv = umma_idesc_f16(BQ, L::ON) | (1u << 16);  // B (V) MN-major
      int it = 0, g = 0;
      auto issue_s = [&](int gg, uint32_t sq) {
        const int st = gg % STAGES;
        mbar_wait_dbg(&k_full[st], (gg / STAGES) & 1, 3000000 + gg, a.dbg);
        tc_fence_after();
        const uint32_t sk = smem_u32(smem + L::OFF_K + st * L::K_BYTES);
#pragma unroll
        for (int b = 0; b < L::NB; ++b)
          umma_f16(tmem + (gg % NS) * BKV, desc_sw32(sq + b * L::Q_BLOCK, 16, 256),
                   desc_sw32(sk + b * L::KV_BLOCK, 16, 256), idesc_s, b > 0);
        umma_commit(&k_empty[st]);
        umma_commit(&s_full[gg % NS]);
      };
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        const int qb = it & 1;
        const uint32_t sq = smem_u32(smem + qb * L::Q_BYTES);
        mbar_wait_dbg(&q_full[qb], (it >> 1) & 1, 4000000 + it, a.dbg);
        tc_fence_after();
        for (int j = 0; j < NS && j < nkv; ++j) issue_s(g + j, sq);
        for (int j = 0; j < nkv; ++j, ++g) {
          const int sb = g % NS, st = g % STAGES;
          mbar_wait_dbg(&p_full[sb], (g / NS) & 1, 5000000 + g, a.dbg);
          mbar_wait_dbg(&v_full[st], (g / STAGES) & 1, 6000000 + g, a.dbg);
          tc_fence_after();
          const uint32_t sv = smem_u32(smem + L::OFF_V + st * L::V_BYTES);
#pragma unroll
          for (int kc = 0; kc < BKV / 16; ++kc)  // 16 keys per MMA: P columns 8*kc, V rows 16*kc
            umma_f16_ts(tmem + L::OCOL, tmem + sb * BKV + kc * 8, desc_sw32(sv + kc * 512, L::KV_BLOCK, 256),
                        idesc_pv, (j | kc) != 0);
          umma_commit(&v_empty[st]);
          umma_commit(&o_done[sb]);
          if (j + NS < nkv) issue_s(g + NS, sq);
          if (j == nkv - 1) umma_commit(&q_empty[qb]);  // every MMA reading this Q buffer issued
        }
      }
    }
  } else {
    // softmax warp: TMEM lane quarter (warp & 3), column slice `part` of every S tile
    const int quarter = warp & 3, part = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    float* red = reinterpret_cast<float*>(smem + L::OFF_RED);  // [2][SPLIT][BQ]
    const float c = a.scale_log2;
    int g = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int qt = item % q_tiles;
      const int h = (item / q_tiles) % a.heads;
      const int z = item / (q_tiles * a.heads);
      float m_ref = -INFINITY;
      for (int j = 0; j < nkv; ++j, ++g) {
        const int sb = g % NS;
        mbar_wait_dbg(&s_full[sb], (g / NS) & 1, 7000000 + g, a.dbg);
        tc_fence_after();
        const uint32_t sbase = lane_base + sb * BKV + part * L::COLS;
        float v[L::COLS];
        tmem_ld_cols<L::COLS>(sbase, v);
        tmem_ld_wait();
        float pm[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) pm[k] = v[k];
#pragma unroll
        for (int i = 8; i < L::COLS; i += 16)
#pragma unroll
          for (int k = 0; k < 8; ++k) pm[k] = i + 8 + k < L::COLS ? fmax3f(pm[k], v[i + k], v[i + 8 + k]) : fmaxf(pm[k], v[i + k]);
        float mx = fmaxf(fmax3f(pm[0], pm[1], pm[2]), fmax3f(fmax3f(pm[3], pm[4], pm[5]), pm[6], pm[7]));
        if constexpr (SPLIT > 1) {  // combine the row maxima of the SPLIT column slices
          float* rb = red + (g & 1) * SPLIT * BQ;
          rb[part * BQ + r] = mx;
          named_bar_sync(1 + quarter, 32 * SPLIT);
#pragma unroll
          for (int q = 0; q < SPLIT; ++q) mx = fmaxf(mx, rb[q * BQ + r]);
        }
        // warp-uniform decision (identical in every slice of this row quarter): tcgen05.ld/st
        // are warp-collective (.sync.aligned)
        if (__any_sync(0xffffffffu, (mx - m_ref) * c > RESCALE_LOG2)) {  // always on the first tile
          const float m_new = fmaxf(m_ref, mx);
          if (j > 0 && part == 0) {
            const int gp = g - 1;  // previous P.V must be complete before O is rescaled
            mbar_wait_dbg(&o_done[gp % NS], (gp / NS) & 1, 8000000 + gp, a.dbg);
            tc_fence_after();
            const float f = fast_exp2((m_ref - m_new) * c);
#pragma unroll 1
            for (int ch = 0; ch < L::ON / 16; ++ch) {
              float o[16];
              tmem_ld16(lane_base + L::OCOL + ch * 16, o);
              tmem_ld_wait();
              uint32_t u[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) u[i] = __float_as_uint(o[i] * f);
              tmem_st16(lane_base + L::OCOL + ch * 16, u);
            }
          }
          m_ref = m_new;
        }
        const float nb = -m_ref * c;
        const uint64_t c2 = f2_pack(c, c), nb2 = f2_pack(nb, nb);
        uint32_t p[L::COLS / 2];
#pragma unroll
        for (int i = 0; i < L::COLS / 2; ++i) {
          float x0, x1;
          f2_unpack(ffma2(f2_pack(v[2 * i], v[2 * i + 1]), c2, nb2), x0, x1);
          // NPOLY of every 16 exponentials (NPOLY / 2 of every 8 pairs) on the FMA pipe
          if ((i & 7) < NPOLY / 2) {
            exp2_poly2(x0, x1);
          } else {
            x0 = fast_exp2(x0);
            x1 = fast_exp2(x1);
          }
          p[i] = pack_half2(x0, x1);
        }
        // P (fp16 pairs) over the already-consumed S columns of this buffer: slice `part` writes
        // columns part*COLS/2 ..; every slice has loaded its S before the max exchange above
        tmem_st_cols<L::COLS / 2>(lane_base + sb * BKV + part * (L::COLS / 2), p);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
      }
      // epilogue: O / rowsum -> fp16 rows of the output; slice `part` writes 8-column chunks
      // part, part + SPLIT, ...
      const int gl = g - 1;
      mbar_wait_dbg(&o_done[gl % NS], (gl / NS) & 1, 9000000 + gl, a.dbg);
      tc_fence_after();
      float lsum[8];
      tmem_ld8(lane_base + L::OCOL + HD, lsum);
      tmem_ld_wait();
      const float inv = 1.f / lsum[0];
      const int qrow = qt * BQ + r;
      __half* dst = a.o + ((long long)z * a.Lq + qrow) * a.o_ld + h * HD;
#pragma unroll 1
      for (int ch = part; ch < HD / 8; ch += SPLIT) {
        float o[8];
        tmem_ld8(lane_base + L::OCOL + ch * 8, o);
        tmem_ld_wait();
        if (qrow < a.Lq) {
          uint4 w;
          w.x = pack_half2(o[0] * inv, o[1] * inv);
          w.y = pack_half2(o[2] * inv, o[3] * inv);
          w.z = pack_half2(o[4] * inv, o[5] * inv);
          w.w = pack_half2(o[6] * inv, o[7] * inv);
          reinterpret_cast<uint4*>(dst + ch * 8)[0] = w;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<L::TMEM>(tmem);
  }
}

// Kernel variants per head dim; variant 0 is the production choice, the others exist for A/B
// measurement (DART_FA_VARIANT, scripts/bench_attn.py).  Measured on B200 (enc self-attention
// N=80, 80x16 heads x 5184^2): variant 0 (96-key tiles, 2 CTAs/SM, 6/16 poly exps) 9.49 ms;
// 4/16 poly 9.96 ms; 8/16 poly 10.65 ms; column-split softmax (2 warps per lane quarter)
// 10.6 ms; 48-key tiles with 4 CTAs/SM 11.3 ms; 3-4 S buffers (1 CTA/SM) 12-16 ms.
template <int HD, int BKV, int STAGES, int CTAS, int NS, int SPLIT, int NPOLY>
int launch_v(const CUtensorMap& tmQ, const CUtensorMap& tmKV, const AttnTcArgs& a, int num_sms, cudaStream_t stream) {
  using Lay = FaCfg<HD, BKV, STAGES, CTAS, NS, SPLIT>;
  auto kern = fa_tc_kernel<HD, BKV, STAGES, CTAS, NS, SPLIT, NPOLY>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::TOTAL);
    if (e != cudaSuccess) return (int)e;
    configured = true;
  }
  const int items = ((a.Lq + BQ - 1) / BQ) * a.heads * a.items;
  const int grid = items < num_sms * CTAS ? items : num_sms * CTAS;
  kern<<<grid, Lay::THREADS, Lay::TOTAL, stream>>>(tmQ, tmKV, a);
  return (int)cudaGetLastError();
}

int fa_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DART_FA_VARIANT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

// (HD, variant) -> key tile; must match the launch below.
int kv_tile_of(int hd, int /*var*/) {
  if (hd == 80) return 64;
  if (hd == 16) return 96;
  return 0;
}

}  // namespace

int attention_tc_kv_tile(int head_dim) { return kv_tile_of(head_dim, fa_variant()); }

bool attention_tc_supported(int head_dim, int Lkv) {
  const int t = attention_tc_kv_tile(head_dim);
  return t > 0 && Lkv % t == 0 && Lkv >= t;
}

int attention_tc(const CUtensorMap& tmQ, const CUtensorMap& tmKV, const AttnTcArgs& a, int head_dim, int num_sms,
                 cudaStream_t stream) {
  const int var = fa_variant();
  if (head_dim == 80) {
    switch (var) {
      case 1: return launch_v<80, 64, 3, 2, 2, 2, 0>(tmQ, tmKV, a, num_sms, stream);
      case 2: return launch_v<80, 64, 3, 2, 2, 1, 2>(tmQ, tmKV, a, num_sms, stream);
      default: return launch_v<80, 64, 3, 2, 2, 1, 0>(tmQ, tmKV, a, num_sms, stream);
    }
  }
  if (head_dim == 16) {
    switch (var) {
      case 1: return launch_v<16, 96, 4, 2, 2, 1, 4>(tmQ, tmKV, a, num_sms, stream);
      case 2: return launch_v<16, 96, 4, 2, 2, 2, 6>(tmQ, tmKV, a, num_sms, stream);
      default: return launch_v<16, 96, 4, 2, 2, 1, 6>(tmQ, tmKV, a, num_sms, stream);
    }
  }
  return (int)cudaErrorInvalidValue;
}

}  // namespace dart
