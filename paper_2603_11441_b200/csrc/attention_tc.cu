// tcgen05 / TMEM flash attention for the backbone (hd = 80), sm_100a.
//
// softmax(q k^T / sqrt(hd)) v for the windowed (576-row windows) and global (5184 rows)
// self-attention of every ViT-H block (reference model.py:390-409).  The backbone stream
// is window-major (dart_capi.cu), so every attention item is a contiguous row block of the
// token-major QKV buffer [rows, 3E] and all tiles are plain 2-D TMA boxes.
//
// Persistent CTAs (one per SM) loop over items (q-tile of 128 rows, head, window/image).
//   warp 0     TMA producer: Q (once per item) and K / V tiles of 192 keys, 2 stages.
//              Operands are 16-dim column blocks with 32-byte swizzle (hd = 80 = 5 x 16).
//   warp 1     MMA issuer (one thread):  S_j = Q K_j^T  -> TMEM (double buffered, 192 cols)
//                                        O  += P_j [V_j | 1]  (A = P read from TMEM, B = V in
//                                        smem, MN-major; the ones block makes column HD of O
//                                        the softmax row sum)
//   warps 4-7  softmax: one thread per query row (TMEM lane); row max from TMEM, P = exp2 of
//              the FFMA-scaled scores written back over S as packed fp16, lazy rescaling of O
//              only when the running max grows by more than 2^8 (P stays <= 256 in fp16).
//   warp 2     TMEM allocator (512 columns: S0 | S1 | O).
#include "common.cuh"
#include "kernels.h"

namespace dart {
namespace {

constexpr int BQ = 128;
constexpr float RESCALE_LOG2 = 8.0f;

// Key-tile width per head dim: hd 80 uses 192-key tiles (TMEM 512 columns, 1 CTA/SM);
// hd 16 (enc-dec, exp-bound) uses 96-key tiles so TMEM fits 256 columns and 2 CTAs share an SM.
template <int HD>
constexpr int kv_tile() { return HD == 80 ? 192 : 96; }

__device__ __forceinline__ uint64_t desc_sw32(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  d |= (uint64_t)6 << 61;  // SWIZZLE_32B
  return d;
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

template <int HD, int BKV>
struct FaSmem {
  static constexpr int TMEM = (2 * BKV + HD + 16) <= 256 ? 256 : 512;  // S0 | S1 | O (+ row-sum block)
  static constexpr int NB = HD / 16;                 // 16-dim column blocks
  static constexpr int Q_BLOCK = BQ * 32;            // bytes per Q column block
  static constexpr int KV_BLOCK = BKV * 32;          // bytes per K/V column block
  static constexpr int Q_BYTES = NB * Q_BLOCK;
  static constexpr int K_BYTES = NB * KV_BLOCK;
  static constexpr int V_BYTES = (NB + 1) * KV_BLOCK;  // + ones block
  static constexpr int OFF_K = Q_BYTES;
  static constexpr int OFF_V = OFF_K + 2 * K_BYTES;
  static constexpr int OFF_BAR = OFF_V + 2 * V_BYTES;
  static constexpr int TOTAL = OFF_BAR + 256 + 1024;
  static constexpr int OCOL = 2 * BKV;               // TMEM column of O
  static constexpr int ON = HD + 16;                 // O columns (values + row-sum block)
};

template <int HD, int BKV>
__global__ void __launch_bounds__(256, 1)
    fa_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV, AttnTcArgs a) {
  using L = FaSmem<HD, BKV>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bars;          // 1
  uint64_t* q_empty = bars + 1;     // 1
  uint64_t* k_full = bars + 2;      // 2
  uint64_t* v_full = bars + 4;      // 2
  uint64_t* kv_empty = bars + 6;    // 2
  uint64_t* s_full = bars + 8;      // 2
  uint64_t* p_full = bars + 10;     // 2
  uint64_t* o_done = bars + 12;     // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  const int warp = warp_id(), lane = lane_id();
  const int q_tiles = (a.Lq + BQ - 1) / BQ;
  const int n_items = q_tiles * a.heads * a.items;
  const int nkv = a.Lkv / BKV;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmKV);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 4);
      mbar_init(&o_done[s], 1);
    }
    fence_barrier_init();
  }
  // ones block of every V stage (column block NB): the row-sum column of O
  for (int i = threadIdx.x; i < 2 * BKV * 4; i += blockDim.x) {
    const int s = i / (BKV * 4), r = i % (BKV * 4);
    reinterpret_cast<uint2*>(smem + L::OFF_V + s * L::V_BYTES + L::NB * L::KV_BLOCK)[r] =
        make_uint2(0x3C003C00u, 0x3C003C00u);
  }
  fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core (async proxy)
  if (warp == 2) tmem_alloc<L::TMEM>(tmem_slot);
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
        mbar_wait_dbg(q_empty, (it & 1) ^ 1, 1000000 + it, a.dbg);
        mbar_arrive_expect_tx(q_full, L::Q_BYTES);
        for (int b = 0; b < L::NB; ++b)
          tma_load_2d(smem + b * L::Q_BLOCK, &tmQ, q_full, a.q_col + h * HD + b * 16, z * a.Lq + qt * BQ);
        for (int j = 0; j < nkv; ++j, ++g) {
          const int st = g & 1;
          const uint32_t ph = (g >> 1) & 1;
          mbar_wait_dbg(&kv_empty[st], ph ^ 1, 2000000 + g, a.dbg);
          uint8_t* sk = smem + L::OFF_K + st * L::K_BYTES;
          uint8_t* sv = smem + L::OFF_V + st * L::V_BYTES;
          mbar_arrive_expect_tx(&k_full[st], L::K_BYTES);
          for (int b = 0; b < L::NB; ++b)
            tma_load_2d(sk + b * L::KV_BLOCK, &tmKV, &k_full[st], a.k_col + h * HD + b * 16, row0 + j * BKV);
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
      const uint32_t sq = smem_u32(smem);
      auto issue_s = [&](int gg) {
        const int st = gg & 1;
        mbar_wait_dbg(&k_full[st], (gg >> 1) & 1, 3000000 + gg, a.dbg);
        tc_fence_after();
        const uint32_t sk = smem_u32(smem + L::OFF_K + st * L::K_BYTES);
#pragma unroll
        for (int b = 0; b < L::NB; ++b)
          umma_f16(tmem + st * BKV, desc_sw32(sq + b * L::Q_BLOCK, 16, 256), desc_sw32(sk + b * L::KV_BLOCK, 16, 256),
                   idesc_s, b > 0);
        umma_commit(&s_full[st]);
      };
      int it = 0, g = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        mbar_wait_dbg(q_full, it & 1, 4000000 + it, a.dbg);
        tc_fence_after();
        issue_s(g);
        if (nkv > 1) issue_s(g + 1);
        for (int j = 0; j < nkv; ++j, ++g) {
          const int st = g & 1;
          const uint32_t ph = (g >> 1) & 1;
          mbar_wait_dbg(&p_full[st], ph, 5000000 + g, a.dbg);
          mbar_wait_dbg(&v_full[st], ph, 6000000 + g, a.dbg);
          tc_fence_after();
          const uint32_t sv = smem_u32(smem + L::OFF_V + st * L::V_BYTES);
#pragma unroll
          for (int kc = 0; kc < BKV / 16; ++kc)  // 16 keys per MMA: P columns 8*kc, V rows 16*kc
            umma_f16_ts(tmem + L::OCOL, tmem + st * BKV + kc * 8, desc_sw32(sv + kc * 512, L::KV_BLOCK, 256),
                        idesc_pv, (j | kc) != 0);
          umma_commit(&kv_empty[st]);
          umma_commit(&o_done[st]);
          if (j == nkv - 1) umma_commit(q_empty);  // all MMAs reading Q of this item issued
          if (j + 2 < nkv) issue_s(g + 2);
        }
      }
    }
  } else if (warp >= 4) {
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const float c = a.scale_log2;
    int g = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int qt = item % q_tiles;
      const int h = (item / q_tiles) % a.heads;
      const int z = item / (q_tiles * a.heads);
      float m_ref = -INFINITY;
      for (int j = 0; j < nkv; ++j, ++g) {
        const int st = g & 1;
        const uint32_t ph = (g >> 1) & 1;
        mbar_wait_dbg(&s_full[st], ph, 7000000 + g, a.dbg);
        tc_fence_after();
        const uint32_t sbase = lane_base + st * BKV;
        float mx = -INFINITY;
#pragma unroll 1
        for (int ch = 0; ch < BKV / 32; ++ch) {
          float v[32];
          tmem_ld32(sbase + ch * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; i += 2) mx = fmax3f(mx, v[i], v[i + 1]);
        }
        // warp-uniform decision: tcgen05.ld/st below are warp-collective (.sync.aligned)
        if (__any_sync(0xffffffffu, (mx - m_ref) * c > RESCALE_LOG2)) {  // always on the first tile
          const float m_new = fmaxf(m_ref, mx);
          if (j > 0) {
            const int gp = g - 1;  // previous P.V must be complete before O is rescaled
            mbar_wait_dbg(&o_done[gp & 1], (gp >> 1) & 1, 8000000 + gp, a.dbg);
            tc_fence_after();
            const float f = fast_exp2((m_ref - m_new) * c);
#pragma unroll 1
            for (int ch = 0; ch < L::ON / 16; ++ch) {
              float v[16];
              tmem_ld16(lane_base + L::OCOL + ch * 16, v);
              tmem_ld_wait();
              uint32_t u[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) u[i] = __float_as_uint(v[i] * f);
              tmem_st16(lane_base + L::OCOL + ch * 16, u);
            }
          }
          m_ref = m_new;
        }
        const float nb = -m_ref * c;
#pragma unroll 1
        for (int ch = 0; ch < BKV / 32; ++ch) {
          float v[32];
          tmem_ld32(sbase + ch * 32, v);
          tmem_ld_wait();
          uint32_t p[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            p[i] = pack_half2(fast_exp2(fmaf(v[2 * i], c, nb)), fast_exp2(fmaf(v[2 * i + 1], c, nb)));
          tmem_st16(sbase + ch * 16, p);  // P chunk ch overwrites already-consumed S columns
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[st]);
      }
      // epilogue: O / rowsum -> fp16 rows of the output
      const int gl = g - 1;
      mbar_wait_dbg(&o_done[gl & 1], (gl >> 1) & 1, 9000000 + gl, a.dbg);
      tc_fence_after();
      float lsum[16];
      tmem_ld16(lane_base + L::OCOL + HD, lsum);
      tmem_ld_wait();
      const float inv = 1.f / lsum[0];
      const int qrow = qt * BQ + r;
      __half* dst = a.o + ((long long)z * a.Lq + qrow) * a.o_ld + h * HD;
#pragma unroll 1
      for (int ch = 0; ch < HD / 16; ++ch) {
        float v[16];
        tmem_ld16(lane_base + L::OCOL + ch * 16, v);
        tmem_ld_wait();
        if (qrow < a.Lq) {
          uint4 w0, w1;
          w0.x = pack_half2(v[0] * inv, v[1] * inv);
          w0.y = pack_half2(v[2] * inv, v[3] * inv);
          w0.z = pack_half2(v[4] * inv, v[5] * inv);
          w0.w = pack_half2(v[6] * inv, v[7] * inv);
          w1.x = pack_half2(v[8] * inv, v[9] * inv);
          w1.y = pack_half2(v[10] * inv, v[11] * inv);
          w1.z = pack_half2(v[12] * inv, v[13] * inv);
          w1.w = pack_half2(v[14] * inv, v[15] * inv);
          reinterpret_cast<uint4*>(dst + ch * 16)[0] = w0;
          reinterpret_cast<uint4*>(dst + ch * 16)[1] = w1;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<L::TMEM>(tmem);
  }
}

template <int HD>
int launch_tc(const CUtensorMap& tmQ, const CUtensorMap& tmKV, const AttnTcArgs& a, int num_sms,
              cudaStream_t stream) {
  constexpr int BKV = kv_tile<HD>();
  using Lay = FaSmem<HD, BKV>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(fa_tc_kernel<HD, BKV>, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::TOTAL);
    if (e != cudaSuccess) return (int)e;
    configured = true;
  }
  const int ctas_per_sm = Lay::TMEM == 256 ? 2 : 1;
  const int items = ((a.Lq + BQ - 1) / BQ) * a.heads * a.items;
  const int grid = items < num_sms * ctas_per_sm ? items : num_sms * ctas_per_sm;
  fa_tc_kernel<HD, BKV><<<grid, 256, Lay::TOTAL, stream>>>(tmQ, tmKV, a);
  return (int)cudaGetLastError();
}

}  // namespace

int attention_tc_kv_tile(int head_dim) { return head_dim == 80 ? kv_tile<80>() : head_dim == 16 ? kv_tile<16>() : 0; }

bool attention_tc_supported(int head_dim, int Lkv) {
  const int t = attention_tc_kv_tile(head_dim);
  return t > 0 && Lkv % t == 0 && Lkv >= t;
}

int attention_tc(const CUtensorMap& tmQ, const CUtensorMap& tmKV, const AttnTcArgs& a, int head_dim, int num_sms,
                 cudaStream_t stream) {
  if (head_dim == 80) return launch_tc<80>(tmQ, tmKV, a, num_sms, stream);
  if (head_dim == 16) return launch_tc<16>(tmQ, tmKV, a, num_sms, stream);
  return (int)cudaErrorInvalidValue;
}

}  // namespace dart
