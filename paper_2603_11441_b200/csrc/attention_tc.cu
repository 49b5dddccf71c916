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
//   warp 1     MMA issuer (whole warp, elect.sync inside each issue so the descriptors stay
//              warp-uniform):        S_j = Q K_j^T -> TMEM (NS-buffered, BKV cols)
//                                        O  += P_j [V_j | 1]  (A = P read from TMEM, B = V in
//                                        smem, MN-major; the ones block makes column HD of O
//                                        the softmax row sum on the tensor core)
//              The second half of the grid swaps the TMA and MMA warps (warp 0 <-> 1) so
//              the two CTAs on an SM put their MMA issuers on different SM sub-partitions.
//   warps 2-5  softmax: one thread per query row (TMEM lane quarter = warp & 3).  The whole
//              S tile is loaded into registers once and P = 2^x of the FFMA-scaled scores is
//              written back over S as packed fp16.
//              Pass 0 (every item): fixed-reference softmax -- the reference max m is the row
//              max of the FIRST key tile only (8-way max3 tree), later tiles are exponentiated
//              against it with no max tracking and no O rescale.  NPOLY of every 16
//              exponentials run as a saturating degree-3 polynomial on the FMA pipe
//              (exp2_poly2_sat) instead of MUFU, balancing the two pipes (MUFU = 16/clk/SM is
//              the hd-16 roof).  A later score more than 2^16 above m overflows the fp16 P to
//              inf; the epilogue sees a non-finite row sum and flags the item in the smem
//              overflow bitmask instead of storing a wrong row.
//              Pass 1 (flagged items only, or all with force_safe): max-tracking softmax that
//              rescales O whenever the running max grows by more than 2^8 (P <= 256), MUFU
//              exponentials only.  Both passes give softmax(x) exactly up to fp16 rounding of P.
#include <type_traits>

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

// QT: query tiles per CTA (independent S -> P -> P.V chains sharing each K / V stage; chain t
// owns TMEM columns [t * CHAIN, (t + 1) * CHAIN) and softmax warps 2 + 4t .. 5 + 4t)
template <int HD, int BKV, int STAGES, int CTAS, int NS, int SPLIT, int QT = 1>
struct FaCfg {
  static constexpr int NB = HD / 16;                 // 16-dim column blocks
  static constexpr int ON = HD + 16;                 // O columns (values + row-sum block)
  static constexpr int OCOL = NS * BKV;              // TMEM column of O (within a chain)
  static constexpr int CHAIN = NS * BKV + ON;        // TMEM columns per chain
  static constexpr int TMEM_NEED = QT * CHAIN;
  static constexpr int TMEM = TMEM_NEED <= 32 ? 32 : TMEM_NEED <= 64 ? 64 : TMEM_NEED <= 128 ? 128
                              : TMEM_NEED <= 256 ? 256 : 512;
  static_assert(TMEM_NEED <= 512 && TMEM * CTAS <= 512, "TMEM budget");
  static_assert(BKV % (8 * SPLIT) == 0 && (BKV / SPLIT) % 8 == 0, "S tile split into 8-column pieces");
  static_assert(QT == 1 || SPLIT == 1, "query-tile chains use whole-row softmax warps");
  static constexpr int THREADS = 64 + 128 * SPLIT * QT;  // TMA/alloc warp, MMA warp, 4*SPLIT*QT softmax warps
  static constexpr int COLS = BKV / SPLIT;           // S columns per softmax warp
  static constexpr int Q_BLOCK = BQ * 32;            // bytes per Q column block
  static constexpr int KV_BLOCK = BKV * 32;          // bytes per K/V column block
  static constexpr int Q_TILE_BYTES = NB * Q_BLOCK;
  static constexpr int Q_BYTES = QT * Q_TILE_BYTES;  // one Q buffer (QT tiles)
  static constexpr int K_BYTES = NB * KV_BLOCK;
  static constexpr int V_BYTES = (NB + 1) * KV_BLOCK;  // + ones block
  static constexpr int OFF_K = 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + STAGES * K_BYTES;
  static constexpr int OFF_BAR = OFF_V + STAGES * V_BYTES;
  static constexpr int NBARS = 4 + 4 * STAGES + QT * (3 * NS + 1);
  static constexpr int OFF_OVF = OFF_BAR + NBARS * 8 + 16;         // overflow bitmask of local items
  static constexpr int OVF_WORDS = ATTN_TC_MAX_LOCAL_ITEMS / 32;
  static constexpr int OFF_RED = OFF_OVF + OVF_WORDS * 4;          // [2][SPLIT][128] partial row maxima
  static constexpr int TOTAL = OFF_RED + (SPLIT > 1 ? 2 * SPLIT * BQ * 4 : 0) + 1024;
  static_assert(TOTAL * CTAS <= 227 * 1024, "shared memory budget");
  static_assert(COLS % 16 == 0, "a 16-key P.V step stays inside one softmax slice");
};

// Softmax numerics.  Pass 0 (every item): the reference max m of each row is taken over the
// FIRST key tile only and kept for the whole row, so later tiles need no max, no vote and no O
// rescale: P = 2^((s - m) c) may exceed 1.  fp16 P overflows (to inf) only if a later score
// exceeds m by more than 16 / c; the fp32 row sum (ones column of O) is then not finite and
// the item is marked in a per-CTA bitmask.  Pass 1 re-runs the marked items with the classic
// per-tile running max and lazy rescale (P <= 2^8), overwriting their output rows.
// SPIN bit 0: the MMA issuer spins on its barriers; bit 1: the softmax warps spin on S-ready.
// LEAN: every tcgen05.commit occupies the tensor pipe like a ~44-clk MMA (scripts/probes/
// mma_rate.cu), so per key tile only S-ready is committed; K / V / Q stage releases become
// thread arrivals by softmax warp 2 (S(g) complete => K(g) consumed, and P.V(g-NS), issued
// before S(g), complete => V(g-NS) consumed), O-complete is committed once per item (and per
// tile only in the rare max-tracking pass, for its O rescale), and V loads get their own
// producer thread (warp 0 lane 1) so they never hold back K loads.
template <bool SPIN>
__device__ __forceinline__ void wait_sel(uint64_t* bar, uint32_t parity, int tag, int* dbg) {
  if (SPIN && dbg == nullptr)
    mbar_spin(bar, parity);
  else
    mbar_wait_dbg(bar, parity, tag, dbg);
}

// KSPL: split-KV instantiation (AttnTcArgs::kv_split, partial outputs); without it the key range is
// whole and the split bookkeeping compiles out (register pressure of the hd-16 kernel is at its cap)
template <int HD, int BKV, int STAGES, int CTAS, int NS, int SPLIT, int NPOLY, int SPIN, int LEAN, bool MASK, int QT = 1,
          bool KSPL = false>
__global__ void __launch_bounds__(FaCfg<HD, BKV, STAGES, CTAS, NS, SPLIT, QT>::THREADS, CTAS)
    fa_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV, AttnTcArgs a) {
  // SPIN bit 4 (PROD): the debug / trace / microbenchmark hooks compiled out -- every kernel
  // parameter read after an asm "memory" clobber is a constant-bank reload in the serial
  // issue and softmax loops, and each hook a branch
  constexpr bool PROD = (SPIN & 16) != 0;
  int* const dbg = PROD ? nullptr : a.dbg;
  long long* const trace = PROD ? nullptr : a.trace;
  const int sm_only = PROD ? 0 : a.softmax_only;
  using L = FaCfg<HD, BKV, STAGES, CTAS, NS, SPLIT, QT>;
  static_assert(QT == 1 || !LEAN, "query-tile chains use the commit-per-tile protocol");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bars;                 // 2
  uint64_t* q_empty = bars + 2;            // 2
  uint64_t* k_full = bars + 4;             // STAGES
  uint64_t* k_empty = k_full + STAGES;     // STAGES
  uint64_t* v_full = k_empty + STAGES;     // STAGES
  uint64_t* v_empty = v_full + STAGES;     // STAGES
  uint64_t* s_full = v_empty + STAGES;     // [QT][NS]
  uint64_t* p_full = s_full + QT * NS;     // [QT][NS]
  uint64_t* o_done = p_full + QT * NS;     // [QT][NS]
  uint64_t* item_done = o_done + QT * NS;  // [QT] (LEAN): all P.V of an item complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(item_done + QT);
  uint32_t* ovf = reinterpret_cast<uint32_t*>(smem + L::OFF_OVF);
  // TMEM column (within an S buffer) of the fp16 P pair holding key k: slice k / COLS keeps its
  // P in the first half of its own S columns
  auto p_col = [](int k) { return (k / L::COLS) * L::COLS + (k % L::COLS) / 2; };

  const int warp = warp_id(), lane = lane_id();
  const int q_tiles = (a.Lq + BQ - 1) / BQ;
  const int q_groups = (q_tiles + QT - 1) / QT;  // an item covers QT query tiles (rows past Lq: zeros)
  const int KS = KSPL ? a.kv_split : 1;
  const int n_items = q_groups * a.heads * a.items * KS;
  // MASK: Lkv not a multiple of BKV (decoder self-attention over 201 tokens, text cross-attention
  // over 32): the last key tile is partial and its keys >= Lkv are masked to P = 0
  const int nkv_all = MASK ? (a.Lkv + BKV - 1) / BKV : a.Lkv / BKV;
  // item -> (q tile, head, key split, item z) and the split's key tiles [j0, j0 + nkv)
  struct Item {
    int qt, h, s, z, j0, nkv;
  };
  auto item_of = [&](int item) {  // qt: the first query tile of the item's group
    Item it;
    it.qt = (item % q_groups) * QT;
    it.h = (item / q_groups) % a.heads;
    if constexpr (KSPL) {
      it.s = (item / (q_groups * a.heads)) % KS;
      it.z = item / (q_groups * a.heads * KS) + a.z_base;
      const int base = nkv_all / KS, rem = nkv_all % KS;
      it.j0 = it.s * base + (it.s < rem ? it.s : rem);
      it.nkv = base + (it.s < rem ? 1 : 0);
    } else {
      it.s = 0;
      it.z = item / (q_groups * a.heads) + a.z_base;
      it.j0 = 0;
      it.nkv = nkv_all;
    }
    return it;
  };
  // TMA and MMA warps (SMSPs 0 / 1).  The tcgen05.mma stream costs its SMSP issue time, which the
  // softmax warp sharing that SMSP loses; the second CTA of an SM (blocks are placed round-robin,
  // so blockIdx >= grid/2) swaps the two roles to put its MMA issue on the other SMSP.
  const bool swap_roles = (int)blockIdx.x * 2 >= (int)gridDim.x;
  const int w_load = swap_roles ? 1 : 0, w_mma = swap_roles ? 0 : 1;

  if (warp == 1 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmKV);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < QT * NS; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 4 * SPLIT);
      mbar_init(&o_done[s], 1);
    }
    for (int t = 0; t < QT; ++t) mbar_init(&item_done[t], 1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < L::OVF_WORDS; i += blockDim.x) ovf[i] = 0u;
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
  pdl_wait();  // Q / K / V of the previous kernel complete

  // pipeline state, continued across the two passes
  int p_it = 0, p_g = 0, pv_g = 0;  // producer (Q/K thread, V thread)
  int m_it = 0, m_g = 0, m_g1 = 0;  // MMA issuer (m_g1: tiles of the max-tracking pass)
  int s_g = 0, s_it = 0, s_g1 = 0;  // softmax
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      tc_fence_before();
      __syncthreads();  // every softmax warp has recorded its overflow bits
      tc_fence_after();
      if (sm_only) break;
      uint32_t any = a.force_safe;
      for (int i = 0; i < L::OVF_WORDS; ++i) any |= ovf[i];
      if (!any) break;
    }
    auto todo = [&](int local) {
      return pass == 0 || a.force_safe || ((ovf[local >> 5] >> (local & 31)) & 1u);
    };
    if (warp == w_load) {
      if (lane < (LEAN ? 2 : 1) && sm_only != 1) {
        const bool do_qk = lane == 0, do_v = !LEAN || lane == 1;
        int local = 0;
        for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
          if (!todo(local)) continue;
          const Item I = item_of(item);
          const int qt = I.qt, h = I.h, z = I.z, nkv = I.nkv;
          // kv_mod: K/V shared per class; the split's first key row
          const int row0 = (a.kv_mod > 0 ? z % a.kv_mod : z) * a.Lkv + I.j0 * BKV;
          if (do_qk) {
            const int qb = p_it & 1;
            mbar_wait_dbg(&q_empty[qb], ((p_it >> 1) & 1) ^ 1, 1000000 + p_it, dbg);
            mbar_arrive_expect_tx(&q_full[qb], L::Q_BYTES);
            for (int t = 0; t < QT; ++t)
              for (int b = 0; b < L::NB; ++b)
                tma_load_2d(smem + qb * L::Q_BYTES + t * L::Q_TILE_BYTES + b * L::Q_BLOCK, &tmQ, &q_full[qb],
                            a.q_col + h * HD + b * 16, z * a.Lq + (qt + t) * BQ);
            ++p_it;
          }
          for (int j = 0; j < nkv; ++j) {
            if (do_qk) {
              const int st = p_g % STAGES;
              mbar_wait_dbg(&k_empty[st], ((p_g / STAGES) & 1) ^ 1, 2000000 + p_g, dbg);
              mbar_arrive_expect_tx(&k_full[st], L::K_BYTES);
              uint8_t* sk = smem + L::OFF_K + st * L::K_BYTES;
              for (int b = 0; b < L::NB; ++b)
                tma_load_2d(sk + b * L::KV_BLOCK, &tmKV, &k_full[st], a.k_col + h * HD + b * 16, row0 + j * BKV);
              ++p_g;
            }
            if (do_v) {
              const int st = pv_g % STAGES;
              mbar_wait_dbg(&v_empty[st], ((pv_g / STAGES) & 1) ^ 1, 2500000 + pv_g, dbg);
              mbar_arrive_expect_tx(&v_full[st], L::K_BYTES);
              uint8_t* sv = smem + L::OFF_V + st * L::V_BYTES;
              for (int b = 0; b < L::NB; ++b)
                tma_load_2d(sv + b * L::KV_BLOCK, &tmKV, &v_full[st], a.v_col + h * HD + b * 16, row0 + j * BKV);
              ++pv_g;
            }
          }
        }
      }
      __syncwarp();
    } else if (warp == w_mma) {
      if (sm_only != 1) {  // the whole warp runs the issue loop (converged); one lane issues
        constexpr uint32_t idesc_s = umma_idesc_f16(BQ, BKV);
        constexpr uint32_t idesc_pv = umma_idesc_f16(BQ, L::ON) | (1u << 16);  // B (V) MN-major
        // the K-ready wait of S(gg) can be hoisted off the P-ready -> P.V -> S critical path
        auto wait_k = [&](int gg) {
          wait_sel<SPIN & 1>(&k_full[gg % STAGES], (gg / STAGES) & 1, 3000000 + gg, dbg);
        };
        auto issue_s = [&](int gg, uint32_t sq, bool k_waited) {
          const int st = gg % STAGES;
          if (!k_waited) wait_k(gg);
          if (trace && blockIdx.x == 0 && lane == 0 && gg >= 2 && gg - 2 < 256) trace[1536 + gg - 2] = clock64();
          tc_fence_after();
          const uint32_t sk = smem_u32(smem + L::OFF_K + st * L::K_BYTES);
#pragma unroll
          for (int b = 0; b < L::NB; ++b)
            umma_f16_w(tmem + (gg % NS) * BKV, desc_sw32(sq + b * L::Q_BLOCK, 16, 256),
                     desc_sw32(sk + b * L::KV_BLOCK, 16, 256), idesc_s, b > 0);
          if constexpr (!LEAN) umma_commit_w(&k_empty[st]);
          umma_commit_w(&s_full[gg % NS]);
        };
        int local = 0;
        if constexpr (QT == 1) {
        for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
          if (!todo(local)) continue;
          const int nkv = item_of(item).nkv;
          const int qb = m_it & 1;
          const uint32_t sq = smem_u32(smem + qb * L::Q_BYTES);
          mbar_wait_dbg(&q_full[qb], (m_it >> 1) & 1, 4000000 + m_it, dbg);
          tc_fence_after();
          for (int j = 0; j < NS && j < nkv; ++j) issue_s(m_g + j, sq, false);
          for (int j = 0; j < nkv; ++j, ++m_g) {
            const int sb = m_g % NS, st = m_g % STAGES;
            if constexpr (LEAN) {
              // V(g) and K(g+NS) have normally landed long before P(g): wait for them first,
              // so that once P(g) is ready nothing but MMA issue separates it from S(g+NS)
              wait_sel<SPIN & 1>(&v_full[st], (m_g / STAGES) & 1, 6000000 + m_g, dbg);
              if (j + NS < nkv) wait_k(m_g + NS);
              wait_sel<SPIN & 1>(&p_full[sb], (m_g / NS) & 1, 5000000 + m_g, dbg);
              if (trace && blockIdx.x == 0 && lane == 0 && m_g < 256) trace[512 + m_g] = trace[1024 + m_g] = clock64();
            } else {
              wait_sel<SPIN & 1>(&p_full[sb], (m_g / NS) & 1, 5000000 + m_g, dbg);
              if (trace && blockIdx.x == 0 && lane == 0 && m_g < 256) trace[512 + m_g] = clock64();
              wait_sel<SPIN & 1>(&v_full[st], (m_g / STAGES) & 1, 6000000 + m_g, dbg);
              if (trace && blockIdx.x == 0 && lane == 0 && m_g < 256) trace[1024 + m_g] = clock64();
            }
            tc_fence_after();
            const uint32_t sv = smem_u32(smem + L::OFF_V + st * L::V_BYTES);
            if constexpr (SPLIT == 1) {  // P of key 16*kc at column 8*kc, V rows 16*kc at +512 B
              umma_f16_ts_seq_w<BKV / 16, 8, 512 / 16>(tmem + L::OCOL, tmem + sb * BKV, desc_sw32(sv, L::KV_BLOCK, 256),
                                                       idesc_pv, j != 0);
            } else {
#pragma unroll
              for (int kc = 0; kc < BKV / 16; ++kc)  // 16 keys per MMA (V rows 16*kc); slice `part`
                umma_f16_ts_w(tmem + L::OCOL, tmem + sb * BKV + p_col(kc * 16),
                              desc_sw32(sv + kc * 512, L::KV_BLOCK, 256), idesc_pv, (j | kc) != 0);
            }
            if (trace && blockIdx.x == 0 && lane == 0 && m_g < 256) trace[1280 + m_g] = clock64();
            if constexpr (LEAN) {
              if (pass == 1) umma_commit_w(&o_done[m_g1++ % NS]);
              if (j == nkv - 1) umma_commit_w(item_done);
            } else {
              umma_commit_w(&v_empty[st]);
              umma_commit_w(&o_done[sb]);
            }
            if (j + NS < nkv) issue_s(m_g + NS, sq, LEAN);
            if (!LEAN && j == nkv - 1) umma_commit_w(&q_empty[qb]);  // every MMA reading this Q buffer issued
            if (trace && blockIdx.x == 0 && lane == 0 && m_g < 256) trace[768 + m_g] = clock64();
          }
          ++m_it;
        }
        } else {
        // commit-per-tile protocol, QT chains: per key tile, V(g) and K(g+NS) are awaited once,
        // then each chain's P.V(g) follows its own P-ready and is chased by its S(g+NS); the K / V
        // stages are released after the last chain's MMAs read them
        auto issue_s_chain = [&](int gg, uint32_t sq, int t) {
          const uint32_t sk = smem_u32(smem + L::OFF_K + (gg % STAGES) * L::K_BYTES);
#pragma unroll
          for (int b = 0; b < L::NB; ++b)
            umma_f16_w(tmem + t * L::CHAIN + (gg % NS) * BKV, desc_sw32(sq + t * L::Q_TILE_BYTES + b * L::Q_BLOCK, 16, 256),
                       desc_sw32(sk + b * L::KV_BLOCK, 16, 256), idesc_s, b > 0);
          umma_commit_w(&s_full[t * NS + gg % NS]);
        };
        for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
          if (!todo(local)) continue;
          const int nkv = item_of(item).nkv;
          const int qb = m_it & 1;
          const uint32_t sq = smem_u32(smem + qb * L::Q_BYTES);
          mbar_wait_dbg(&q_full[qb], (m_it >> 1) & 1, 4000000 + m_it, dbg);
          tc_fence_after();
          for (int j = 0; j < NS && j < nkv; ++j) {
            wait_k(m_g + j);
            tc_fence_after();
#pragma unroll
            for (int t = 0; t < QT; ++t) issue_s_chain(m_g + j, sq, t);
            umma_commit_w(&k_empty[(m_g + j) % STAGES]);
          }
          for (int j = 0; j < nkv; ++j, ++m_g) {
            const int sb = m_g % NS, st = m_g % STAGES;
            const bool more = j + NS < nkv;
            const uint32_t sv = smem_u32(smem + L::OFF_V + st * L::V_BYTES);
            // P-ready first: the K(g+NS) wait sits behind the first P.V, off the P -> P.V path
#pragma unroll
            for (int t = 0; t < QT; ++t) {
              wait_sel<SPIN & 1>(&p_full[t * NS + sb], (m_g / NS) & 1, 5000000 + m_g, dbg);
              if (t == 0) wait_sel<SPIN & 1>(&v_full[st], (m_g / STAGES) & 1, 6000000 + m_g, dbg);
              if (t == 0 && trace && blockIdx.x == 0 && lane == 0 && m_g < 256) trace[512 + m_g] = clock64();
              tc_fence_after();
              if constexpr (SPLIT == 1) {  // P of key 16*kc at column 8*kc, V rows 16*kc at +512 B
                umma_f16_ts_seq_w<BKV / 16, 8, 512 / 16>(tmem + t * L::CHAIN + L::OCOL, tmem + t * L::CHAIN + sb * BKV,
                                                         desc_sw32(sv, L::KV_BLOCK, 256), idesc_pv, j != 0);
              } else {
#pragma unroll
                for (int kc = 0; kc < BKV / 16; ++kc)  // 16 keys per MMA (V rows 16*kc); slice `part`
                  umma_f16_ts_w(tmem + L::OCOL, tmem + sb * BKV + p_col(kc * 16),
                                desc_sw32(sv + kc * 512, L::KV_BLOCK, 256), idesc_pv, (j | kc) != 0);
              }
              if (t == QT - 1) umma_commit_w(&v_empty[st]);
              umma_commit_w(&o_done[t * NS + sb]);
              if (more) {
                if (t == 0) {
                  wait_k(m_g + NS);
                  tc_fence_after();
                }
                issue_s_chain(m_g + NS, sq, t);
                if (t == QT - 1) umma_commit_w(&k_empty[(m_g + NS) % STAGES]);
              }
            }
            if (trace && blockIdx.x == 0 && lane == 0 && m_g < 256) trace[1280 + m_g] = clock64();
            if (j == nkv - 1) umma_commit_w(&q_empty[qb]);  // every MMA reading this Q buffer issued
            if (trace && blockIdx.x == 0 && lane == 0 && m_g < 256) trace[768 + m_g] = clock64();
          }
          ++m_it;
        }
        }
      }
      __syncwarp();
    } else {
      // the two softmax passes are separate instantiations: the fast pass carries none of the
      // max-tracking pass's code (register allocation, branches) and vice versa
      auto softmax_pass = [&](auto pass_c) {
        constexpr int PASS = decltype(pass_c)::value;
        // softmax warp: TMEM lane quarter (warp & 3), column slice `part` of every S tile
        // chain: the query tile of the item this warp's rows belong to (QT > 1: warps 2+4t..5+4t)
        const int quarter = warp & 3, part = QT > 1 ? 0 : (warp - 2) >> 2, chain = QT > 1 ? (warp - 2) >> 2 : 0;
        const int r = quarter * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16) + chain * L::CHAIN;
        uint64_t* const c_s_full = s_full + chain * NS;
        uint64_t* const c_p_full = p_full + chain * NS;
        uint64_t* const c_o_done = o_done + chain * NS;
        [[maybe_unused]] float* red = reinterpret_cast<float*>(smem + L::OFF_RED);  // [2][SPLIT][BQ]
        const float c = a.scale_log2;
        // row max of the loaded S slice, combined over the SPLIT slices of this row
        auto row_max = [&](const float* v, int gg) {
          float pm[8];
  #pragma unroll
          for (int k = 0; k < 8; ++k) pm[k] = v[k];
  #pragma unroll
          for (int i = 8; i < L::COLS; i += 16)
  #pragma unroll
            for (int k = 0; k < 8; ++k)
              pm[k] = i + 8 + k < L::COLS ? fmax3f(pm[k], v[i + k], v[i + 8 + k]) : fmaxf(pm[k], v[i + k]);
          float mx = fmaxf(fmax3f(pm[0], pm[1], pm[2]), fmax3f(fmax3f(pm[3], pm[4], pm[5]), pm[6], pm[7]));
          if constexpr (SPLIT > 1) {
            float* rb = red + (gg & 1) * SPLIT * BQ;
            rb[part * BQ + r] = mx;
            named_bar_sync(1 + quarter, 32 * SPLIT);
  #pragma unroll
            for (int q = 0; q < SPLIT; ++q) mx = fmaxf(mx, rb[q * BQ + r]);
          }
          return mx;
        };
        int local = 0;
        for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
          if (!todo(local)) continue;
          const Item I = item_of(item);
          const int qt = I.qt, h = I.h, z = I.z, nkv = I.nkv;
          float m_ref = -INFINITY;
          float nb = 0.f, cr = 0.f, br = 0.f;
          for (int j = 0; j < nkv; ++j, ++s_g) {
            const int sb = s_g % NS;
            if (sm_only != 1) wait_sel<(SPIN >> 1) & 1>(&c_s_full[sb], (s_g / NS) & 1, 7000000 + s_g, dbg);
            if (trace && blockIdx.x == 0 && warp == 2 && lane == 0 && s_g < 256) trace[s_g] = clock64();
            if (LEAN && warp == 2 && lane == 0 && sm_only != 1) {
              mbar_arrive(&k_empty[s_g % STAGES]);                    // S(g) has consumed K(g)
              if (s_g >= NS) mbar_arrive(&v_empty[(s_g - NS) % STAGES]);  // P.V(g-NS) precedes S(g)
              if (j == nkv - 1) mbar_arrive(&q_empty[s_it & 1]);      // last S of the item read Q
            }
            if (sm_only == 2) {  // microbenchmark: MMA/TMA pipeline alone
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&c_p_full[sb]);
              continue;
            }
            tc_fence_after();
            const uint32_t sbase = lane_base + sb * BKV + part * L::COLS;
            float v[L::COLS];
            tmem_ld_cols<L::COLS>(sbase, v);
            tmem_ld_wait();
            if constexpr (MASK) {  // keys past Lkv in a partial last tile: score -inf -> P = 0
              const int valid = a.Lkv - (I.j0 + j) * BKV - part * L::COLS;
              if (valid < L::COLS) {
  #pragma unroll
                for (int k = 0; k < L::COLS; ++k)
                  if (k >= valid) v[k] = -INFINITY;
              }
            }
            uint32_t p[L::COLS / 2];
            if (PASS == 0) {
              if (j == 0) {
                m_ref = row_max(v, s_g);
                nb = -m_ref * c;
                cr = c * (1.0f / EXP_R);
                br = (nb - EXP_XMIN) * (1.0f / EXP_R);
              }
              const uint64_t c2 = f2_pack(c, c), nb2 = f2_pack(nb, nb);
  #pragma unroll
              for (int i = 0; i < L::COLS / 2; ++i) {
                float x0, x1;
                // NPOLY of every 16 exponentials on the FMA pipe (the first NPOLY / 2 pairs of every 8);
                // NPOLY >= 256 (placement search, attention_search.inc): pair i iff bit (i & 7) of NPOLY - 256
                if (NPOLY >= 256 ? ((NPOLY - 256) >> (i & 7)) & 1 : (i & 7) < NPOLY / 2) {
                  exp2_poly2_sat(v[2 * i], v[2 * i + 1], cr, br, x0, x1);
                } else {
                  f2_unpack(ffma2(f2_pack(v[2 * i], v[2 * i + 1]), c2, nb2), x0, x1);
                  x0 = fast_exp2(x0);
                  x1 = fast_exp2(x1);
                }
                p[i] = pack_half2(x0, x1);
              }
            } else {
              const float mx = row_max(v, s_g);
              // warp-uniform decision (identical in every slice of this row quarter): tcgen05.ld/st
              // are warp-collective (.sync.aligned)
              if (__any_sync(0xffffffffu, (mx - m_ref) * c > RESCALE_LOG2)) {  // always on the first tile
                const float m_new = fmaxf(m_ref, mx);
                if (j > 0 && part == 0) {
                  const int gp = LEAN ? s_g1 - 1 : s_g - 1;  // previous P.V complete before O is rescaled
                  mbar_wait_dbg(&c_o_done[gp % NS], (gp / NS) & 1, 8000000 + gp, dbg);
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
              nb = -m_ref * c;
              const uint64_t c2 = f2_pack(c, c), nb2 = f2_pack(nb, nb);
  #pragma unroll
              for (int i = 0; i < L::COLS / 2; ++i) {
                float x0, x1;
                f2_unpack(ffma2(f2_pack(v[2 * i], v[2 * i + 1]), c2, nb2), x0, x1);
                p[i] = pack_half2(fast_exp2(x0), fast_exp2(x1));
              }
            }
            // P (fp16 pairs) over this slice's own, already loaded S columns (no cross-slice hazard)
            tmem_st_cols<L::COLS / 2>(lane_base + sb * BKV + part * L::COLS, p);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0 && sm_only != 1) mbar_arrive(&c_p_full[sb]);
            if (PASS == 1) ++s_g1;
            if (trace && blockIdx.x == 0 && lane == 0 && s_g < 256) {
              if (warp == 2) trace[256 + s_g] = clock64();
              trace[1792 + (warp - 2) * 256 + s_g] = clock64();  // P done, per softmax warp
            }
          }
          // epilogue: O / rowsum -> fp16 rows of the output; slice `part` writes 8-column chunks
          // part, part + SPLIT, ...
          [[maybe_unused]] const int gl = s_g - 1;
          if (sm_only != 1) {
            if constexpr (LEAN)
              mbar_wait_dbg(item_done, s_it & 1, 9000000 + s_it, dbg);
            else
              mbar_wait_dbg(&c_o_done[gl % NS], (gl / NS) & 1, 9000000 + gl, dbg);
          }
          ++s_it;
          tc_fence_after();
          float lsum[8];
          tmem_ld8(lane_base + L::OCOL + HD, lsum);
          tmem_ld_wait();
          const int qrow = (qt + chain) * BQ + r;
          if (PASS == 0) {
            const bool bad = qrow < a.Lq && !(fabsf(lsum[0]) < INFINITY);
            if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&ovf[local >> 5], 1u << (local & 31));
          }
          if (KSPL) {  // split-KV: unnormalised O, row sum and reference max (log2 units)
            float4* dp = reinterpret_cast<float4*>(a.part + ((((size_t)z * a.heads + h) * KS + I.s) * a.Lq + qrow) * 20);
#pragma unroll 1
            for (int ch = part; ch < HD / 8; ch += SPLIT) {
              float o[8];
              tmem_ld8(lane_base + L::OCOL + ch * 8, o);  // warp-collective: every lane loads
              tmem_ld_wait();
              if (qrow < a.Lq) {
                dp[2 * ch] = make_float4(o[0], o[1], o[2], o[3]);
                dp[2 * ch + 1] = make_float4(o[4], o[5], o[6], o[7]);
              }
            }
            if (part == 0 && qrow < a.Lq) dp[HD / 4] = make_float4(lsum[0], m_ref * c, 0.f, 0.f);
            continue;
          }
          const float inv = 1.f / lsum[0];
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
      };
      if (pass == 0)
        softmax_pass(std::integral_constant<int, 0>{});
      else
        softmax_pass(std::integral_constant<int, 1>{});
    }
  }
  pdl_launch_dependents();  // every item of this CTA is done: the next kernel may start its prologue
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<L::TMEM>(tmem);
  }
}

// Kernel variants per head dim; variant 0 is the production choice, the others exist for A/B
// measurement (DART_FA_VARIANT, scripts/bench_attn.py).
template <int HD, int BKV, int STAGES, int CTAS, int NS, int SPLIT, int NPOLY, int SPIN, int LEAN, bool MASK = false,
          int QT = 1, bool KSPL = false>
int launch_v(const CUtensorMap& tmQ, const CUtensorMap& tmKV, const AttnTcArgs& a, int num_sms, cudaStream_t stream) {
  using Lay = FaCfg<HD, BKV, STAGES, CTAS, NS, SPLIT, QT>;
  auto kern = fa_tc_kernel<HD, BKV, STAGES, CTAS, NS, SPLIT, NPOLY, SPIN, LEAN, MASK, QT, KSPL>;
  if (!KSPL && a.kv_split != 1) return (int)cudaErrorInvalidValue;
  static std::atomic<uint64_t> smem_set{0};
  if (const cudaError_t e = set_smem_once(smem_set, kern, Lay::TOTAL); e != cudaSuccess) return (int)e;
  // items of one launch: each CTA may own at most ATTN_TC_MAX_LOCAL_ITEMS (overflow bitmask)
  const long long per_z = (long long)(((a.Lq + BQ - 1) / BQ + QT - 1) / QT) * a.heads * a.kv_split;
  const long long max_grid = (long long)num_sms * CTAS;
  int zchunk = a.items;
  while (zchunk > 1 && (per_z * zchunk + max_grid - 1) / max_grid > ATTN_TC_MAX_LOCAL_ITEMS) zchunk = (zchunk + 1) / 2;
  for (int z0 = 0; z0 < a.items; z0 += zchunk) {
    AttnTcArgs b = a;
    b.items = a.items - z0 < zchunk ? a.items - z0 : zchunk;
    b.z_base = a.z_base + z0;
    const long long items = per_z * b.items;
    const int grid = (int)(items < max_grid ? items : max_grid);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(Lay::THREADS);
    cfg.dynamicSmemBytes = Lay::TOTAL;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    if (pdl_enabled()) {
      pdl_attr(attr[0]);
      cfg.attrs = attr;
      cfg.numAttrs = 1;
    }
    cudaLaunchKernelEx(&cfg, kern, tmQ, tmKV, b);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}

int g_fa_variant = -1;  // DART_FA_VARIANT, or attention_tc_set_variant (A/B microbenchmarks)
int fa_variant() {
  if (g_fa_variant < 0) {
    const char* e = getenv("DART_FA_VARIANT");
    g_fa_variant = e ? atoi(e) : 0;
  }
  return g_fa_variant;
}

// Variant tables (HD, BKV, STAGES, CTAS/SM, S buffers, column slices, poly exps per 16, SPIN,
// LEAN, query-tile chains per CTA).  Variant 0 is the default, dispatched below to its hook-free
// production twin.
#define DART_FA80_VARIANTS(X)         \
  X(0, 80, 64, 3, 2, 2, 1, 0, 0, 0, 1) \
  X(1, 80, 64, 3, 2, 2, 1, 0, 0, 1, 1) \
  X(2, 80, 64, 3, 2, 2, 1, 4, 0, 0, 1)
#define DART_FA16_VARIANTS(X)           \
  X(0, 16, 96, 4, 2, 2, 1, 6, 0, 0, 1)   \
  X(1, 16, 96, 4, 2, 2, 1, 6, 0, 1, 1)   \
  X(2, 16, 96, 4, 2, 2, 1, 8, 0, 0, 1)   \
  X(3, 16, 96, 4, 2, 2, 1, 4, 0, 0, 1)   \
  X(4, 16, 96, 4, 2, 2, 2, 6, 16, 0, 1)  \
  X(5, 16, 80, 4, 2, 2, 1, 6, 16, 0, 1)  \
  X(7, 16, 64, 4, 1, 1, 1, 6, 16, 0, 4)  \
  X(8, 16, 96, 4, 1, 1, 1, 6, 16, 0, 3)
// hd 80 with polynomial exponentials (hook-free NPOLY 2 / 4 / 6 of 16, interleaved A/B,
// profiles/r02/attn_hd80_poly_share_ab.log): global 168 -> 175 / 177 / 178 us, windowed 27.4-28.3
// -> 27.2-27.7 us (noise): the hd-80 tile is co-bound by MUFU (512 clk per 128 x 64 tile) and the
// tensor pipe (352 clk), so the FMA-pipe polynomial only lengthens the softmax instruction stream.
// Variant 0 issues MMAs from the converged warp 1 (warp-collective umma_*_w, one elected lane):
// the per-MMA issue path shrank from ~77 to ~40 clk (no per-lane R2UR waterfall), which took hd 80
// global attention 217 -> 193 us and windowed 36.5 -> 33.2 us (scripts/ab_attn.py); with it the
// commit-per-tile protocol (LEAN = 0) beats the lean one (LEAN = 1: 210 / 35.6 us; hd 16 equal).
// Measured on B200 (scripts/bench_attn.py, hd 16 enc self-attention N=80 = 80x16 heads x 5184^2;
// box-to-box spread ~8%): variant 0 8.7-9.4 ms; NPOLY 8 9.7, NPOLY 4 9.1; 2 column slices
// 9.6-10.5; 64-key tiles with 3 S buffers 11.0; 48-key tiles at 4 CTAs/SM 11.1-11.7; one CTA/SM
// with 3-4 S buffers 15.3; spin waits 9.8.  Softmax alone (no MMA) 6.76 ms, MMA/TMA pipeline
// alone 6.7-6.9 ms.  tcgen05.mma costs >= 44 clk per instruction and issuer even at N = 32, each
// commit ~44 clk and each mbarrier wait ~40 clk of the issuer's tensor stream
// (scripts/probes/mma_rate.cu), so the 6 P.V steps of a 96-key tile plus S, commits and waits
// make a ~600-clk per-tile MMA chain (scripts/trace_attn.py timelines) that S(g+2) sits behind.
// Query-tile chains (QT tiles per CTA, one CTA per SM, each chain its own S buffers / O / softmax
// warp group, K / V stages shared; profiles/r02/attn_hd16_chains.log), enc self N=20: production
// 1987 us; QT 3 x (2 x 64-key S) 2311, QT 4 x (1 x 64) 2097 (variant 7), QT 3 x (1 x 96) 2202
// (variant 8), QT 2 x (2 x 96) 2299, QT 3 x 64 NPOLY 8 2420 us -- the register file (64 K per SM)
// caps 12-16 softmax warps at 96-128 registers, below one S tile plus its P, so the extra chains
// spill; the one-chain-per-CTA code path is kept as it was for QT = 1.
// Staging P in shared memory or in separate TMEM buffers (S released at load time) was slower
// (11.4 / 14.0 ms): the extra per-tile softmax work outweighed the decoupling.  A decoupled
// variant at 96-key tiles (2 S buffers | one P buffer | O without the ones block, row sums in
// registers; git history "fa_dec_kernel") was correct but also slower: N=20 2.67-2.78 vs 2.41 ms.
#ifdef DART_FA_SEARCH
#include "attention_search.inc"
#else
#define DART_FA16_SEARCH_VARIANTS(X)
#endif

int kv_tile_of(int hd, int var) {
#define X(V, HD, BKV, ST, CT, NS, SP, NP, SN, LN, QT) \
  if (hd == HD && var == V) return BKV;
  DART_FA80_VARIANTS(X)
  DART_FA16_VARIANTS(X)
  DART_FA16_SEARCH_VARIANTS(X)
#undef X
  if (hd == 80) return 64;
  if (hd == 16) return 96;
  return 0;
}

// One thread per (item, head, query row): w_s = 2^(m_s - max m), o = sum w_s O_s / sum w_s l_s.
template <int HD>
__global__ void split_combine_kernel(const float* __restrict__ part, __half* __restrict__ o, int o_ld, int items,
                                     int heads, int Lq, int KS) {
  pdl_wait();
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)items * heads * Lq) return;
  const int row = (int)(t % Lq);
  const int h = (int)((t / Lq) % heads);
  const int z = (int)(t / ((long long)Lq * heads));
  const float4* p0 = reinterpret_cast<const float4*>(part) + (((size_t)z * heads + h) * KS * Lq + row) * 5;
  const size_t sstride = (size_t)Lq * 5;  // float4s between splits
  float mx = -INFINITY;
  for (int s = 0; s < KS; ++s) mx = fmaxf(mx, p0[s * sstride + HD / 4].y);
  float acc[HD], l = 0.f;
#pragma unroll
  for (int k = 0; k < HD; ++k) acc[k] = 0.f;
  for (int s = 0; s < KS; ++s) {
    const float4* ps = p0 + s * sstride;
    const float4 lm = ps[HD / 4];
    const float w = exp2f(lm.y - mx);
    l = fmaf(w, lm.x, l);
#pragma unroll
    for (int k = 0; k < HD / 4; ++k) {
      const float4 v = ps[k];
      acc[4 * k] = fmaf(w, v.x, acc[4 * k]);
      acc[4 * k + 1] = fmaf(w, v.y, acc[4 * k + 1]);
      acc[4 * k + 2] = fmaf(w, v.z, acc[4 * k + 2]);
      acc[4 * k + 3] = fmaf(w, v.w, acc[4 * k + 3]);
    }
  }
  const float inv = 1.f / l;
  uint4* dst = reinterpret_cast<uint4*>(o + ((long long)z * Lq + row) * o_ld + h * HD);
#pragma unroll
  for (int k = 0; k < HD / 8; ++k)
    dst[k] = make_uint4(pack_half2(acc[8 * k] * inv, acc[8 * k + 1] * inv), pack_half2(acc[8 * k + 2] * inv, acc[8 * k + 3] * inv),
                        pack_half2(acc[8 * k + 4] * inv, acc[8 * k + 5] * inv), pack_half2(acc[8 * k + 6] * inv, acc[8 * k + 7] * inv));
  pdl_launch_dependents();
}

}  // namespace

int attention_split_combine(const float* part, __half* o, int o_ld, int items, int heads, int Lq, int kv_split,
                            int hd, cudaStream_t stream) {
  if (hd != 16) return (int)cudaErrorInvalidValue;
  const long long n = (long long)items * heads * Lq;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((n + 127) / 128));
  cfg.blockDim = dim3(128);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  if (pdl_enabled()) {
    pdl_attr(attr[0]);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  cudaLaunchKernelEx(&cfg, split_combine_kernel<16>, part, o, o_ld, items, heads, Lq, kv_split);
  return (int)cudaGetLastError();
}

void attention_tc_set_variant(int v) { g_fa_variant = v < 0 ? 0 : v; }

// Short key sets at hd 16 (the encoder's text cross-attention over L_t = 32 tokens, model.py:518)
// run on 32-key tiles at 4 CTAs per SM (TMEM 2 x 32 + 32 columns per CTA).
constexpr int SHORT_KV = 32;

int attention_tc_kv_tile(int head_dim, int Lkv) {
  if (head_dim == 16 && Lkv <= SHORT_KV) return SHORT_KV;
  return kv_tile_of(head_dim, fa_variant());
}

bool attention_tc_supported(int head_dim, int Lkv) {
  const int t = attention_tc_kv_tile(head_dim, Lkv);
  return t > 0 && Lkv >= 1;  // ragged Lkv: masked instantiation
}

int attention_tc(const CUtensorMap& tmQ, const CUtensorMap& tmKV, const AttnTcArgs& a, int head_dim, int num_sms,
                 cudaStream_t stream) {
  const int var = fa_variant();
#define X(V, HD, BKV, ST, CT, NS, SP, NP, SN, LN, QT) \
  if (V != 0 && head_dim == HD && var == V && a.kv_split == 1)                               \
    return a.Lkv % BKV ? launch_v<HD, BKV, ST, CT, NS, SP, NP, SN, LN, true, QT>(tmQ, tmKV, a, num_sms, stream) \
                       : launch_v<HD, BKV, ST, CT, NS, SP, NP, SN, LN, false, QT>(tmQ, tmKV, a, num_sms, stream);
  DART_FA80_VARIANTS(X)
  DART_FA16_VARIANTS(X)
  DART_FA16_SEARCH_VARIANTS(X)
#undef X
  // the production instantiations (SPIN bit 4) carry no debug / trace / microbenchmark hooks;
  // a launch that asks for one of them runs the hooked twin (identical arithmetic)
  const bool hooks = a.dbg != nullptr || a.trace != nullptr || a.softmax_only != 0;
  if (head_dim == 80) {
    if (a.Lkv % 64 != 0) return launch_v<80, 64, 3, 2, 2, 1, 0, 16, 0, true>(tmQ, tmKV, a, num_sms, stream);
    return hooks ? launch_v<80, 64, 3, 2, 2, 1, 0, 0, 0>(tmQ, tmKV, a, num_sms, stream)
                 : launch_v<80, 64, 3, 2, 2, 1, 0, 16, 0>(tmQ, tmKV, a, num_sms, stream);
  }
  if (head_dim == 16) {
    if (a.Lkv <= SHORT_KV)  // text cross-attention: one (possibly partial) 32-key tile per item
      return a.Lkv == SHORT_KV ? launch_v<16, SHORT_KV, 2, 4, 2, 1, 0, 16, 0>(tmQ, tmKV, a, num_sms, stream)
                               : launch_v<16, SHORT_KV, 2, 4, 2, 1, 0, 16, 0, true>(tmQ, tmKV, a, num_sms, stream);
    if (a.kv_split > 1)  // split-KV (decoder cross-attention)
      return a.Lkv % 96 ? launch_v<16, 96, 4, 2, 2, 1, 6, 16, 0, true, 1, true>(tmQ, tmKV, a, num_sms, stream)
                        : launch_v<16, 96, 4, 2, 2, 1, 6, 16, 0, false, 1, true>(tmQ, tmKV, a, num_sms, stream);
    if (a.Lkv % 96 != 0)  // decoder self-attention (201 = 2 x 96 + 9 keys)
      return launch_v<16, 96, 4, 2, 2, 1, 6, 16, 0, true>(tmQ, tmKV, a, num_sms, stream);
    return hooks ? launch_v<16, 96, 4, 2, 2, 1, 6, 0, 0>(tmQ, tmKV, a, num_sms, stream)
                 : launch_v<16, 96, 4, 2, 2, 1, 6, 16, 0>(tmQ, tmKV, a, num_sms, stream);
  }
  return (int)cudaErrorInvalidValue;
}

}  // namespace dart
