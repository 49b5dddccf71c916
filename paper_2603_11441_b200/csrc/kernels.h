// Internal (C++) launcher declarations shared by the kernel files and the C ABI.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dart {

enum EpiMode {
  EPI_F16 = 0,        // out16 = acc + bias
  EPI_F16_RELU = 1,   // out16 = relu(acc + bias)
  EPI_F32 = 2,        // out32 = acc + bias
  EPI_F32_RESID = 3,  // out32 += acc + bias       (fp32 residual stream)
  EPI_QKV_ROPE = 4,   // out16 = rope(acc + bias) on columns < rope_cols
  EPI_F32_F16 = 5,    // out32 = acc + bias, out2_16 = same in fp16
  // out32 += acc + bias, then out2_16 = LayerNorm(out32) * ln_g + ln_b over each full row
  // (N == BN: the enc-dec's d = 256 rows sit in one tile; fuses the NEXT sub-block's LN)
  EPI_F32_RESID_LN = 6,
  // out32 += acc + bias, out2_16 = fp16(out32), and LayerNorm row statistics of out32 per 32-column
  // chunk into ln_stats_out (see GemmEpi): the producer half of the LN fold (backbone blocks)
  EPI_F32_RESID_X16 = 7,
};

struct GemmEpi {
  const float* bias = nullptr;
  void* out = nullptr;
  int ldo = 0;
  void* out2 = nullptr;
  int ldo2 = 0;
  const float* rope_cos = nullptr;
  const float* rope_sin = nullptr;
  int rope_T = 1;     // tokens per image (rows repeat with period rope_T)
  int rope_grid = 0;  // sqrt(rope_T): the tables are the reference's 2-D RoPE (row | column angles)
  int rope_hd = 2;
  int rope_cols = 0;
  // Window-major row order (grid x grid tokens, win x win windows): rows are stored window by
  // window.  wm_grid > 0 makes the RoPE epilogue look up the true token of a row, and
  // wm_scatter additionally writes output rows back in token-major order (FPN level 0).
  int wm_grid = 0;
  int wm_win = 0;
  int wm_scatter = 0;
  int dbg_noload = 0;  // microbenchmarks only: after the first ring fill, stages are re-used without TMA
  // Split-K (every epilogue but EPI_F32_RESID_LN): splitk = 2 runs each output tile as two K
  // halves on neighbouring CTA pairs (units 2t, 2t+1).  Per epilogue warp, the half that reaches
  // its epilogue first
  // (atomic claim on tile_flags) writes its fp32 partial accumulator to `ws`; the second adds
  // it to its own (fp32 addition commutes: the sum is the same bits whichever half finished
  // first) and runs the normal epilogue.  Nothing waits on a unit that has not claimed, so the
  // protocol cannot deadlock when the grid is only partly resident.  tile_flags:
  // splitk_flag_count(tiles, cg) ints, zero before the first launch (the combining warp resets
  // its flag); ws: splitk_ws_floats(tiles, bn, cg) floats.
  int splitk = 1;
  int* tile_flags = nullptr;
  float* ws = nullptr;
  // Tail halves: the first tail_full tiles (a whole number of waves) run as BN-wide units, the
  // remaining tiles as two BN/2-wide units each, so the last wave is half as long (0 = off).
  int tail_full = 0;
  // Precision-study disciplines (reference tensors.py:111-170):
  // acc_f16 = 1 accumulates in fp16 on the tensor core (D format f16 in TMEM, the negative
  // control); round_f16 = 1 rounds every fp32 output (and the residual stream after the add)
  // to fp16-representable values (fp16 storage).
  int acc_f16 = 0;
  int round_f16 = 0;
  // EPI_F32_RESID_LN: affine of the fused LayerNorm (population variance, eps 1e-6; out2 / ldo2
  // receive the fp16 normalised rows)
  const float* ln_g = nullptr;
  const float* ln_b = nullptr;
  // LayerNorm folded into the consuming GEMM (backbone LN1 -> QKV, LN2 -> fc1):
  //   LN(x) W + b = rstd * (x W' - mu * colsum(W')) + (b + beta W),  W' = diag(gamma) W
  // Producer (EPI_F32_RESID_X16, or EPI_F32_F16 with ln_stats_out set): writes fp16(x) as the
  // consumer's A operand and, per row and 32-column chunk, the chunk's (mean, M2) as a float2 at
  // ln_stats_out[row * ln_parts + col / 32] (two-pass within the chunk).  Each epilogue warp then
  // adds its chunk count to ln_cnt[row / 32]; the warp that completes a 32-row group (count ==
  // ln_parts) combines the rows' chunks in order (Chan et al.) into ln_final[row] = (mean, rstd)
  // and resets the counter (zero before the first launch).  Consumer (EPI_QKV_ROPE /
  // EPI_F16_RELU with ln_stats = ln_final): v = rstd * (acc - mu * ln_colsum[n]) before bias /
  // RoPE / ReLU.
  float2* ln_stats_out = nullptr;
  int* ln_cnt = nullptr;
  float2* ln_final = nullptr;
  const float2* ln_stats = nullptr;
  const float* ln_colsum = nullptr;
  int ln_parts = 0;  // 32-column chunks per row (E / 32)
  // Row-block dependency chain across kernel boundaries (backbone fc1 -> fc2 -> LN1 -> QKV): instead
  // of waiting for the whole previous grid (griddepcontrol.wait), a consumer starts on the rows
  // whose producer tiles are done, so it fills the SMs the producer's last wave leaves idle.
  //   dep_signal: after a unit's stores complete, each epilogue warp adds the number of 32-column
  //     chunks it wrote to dep_signal[row / 128] (a 128-row block is complete when its counter
  //     gains N / 8).
  //   dep_wait: before loading the A rows [m0, m0 + 128) of a unit the producer waits until
  //     dep_wait[m0 / 128] >= dep_mult * (dep_per_row ? rows of that block in [0, M) : 1).
  //   early_trigger: griddepcontrol.launch_dependents right after this kernel's own wait, so the
  //     next kernel's CTAs take the SMs this grid's CTAs free.  skip_pdl_wait: no griddepcontrol
  //     .wait (every input other than the dep_wait rows is complete before the launch);
  //     force_pdl: launched with programmatic stream serialization whatever dart_set_pdl says.
  // Counters are cumulative (dep_mult grows by one chain epoch per use), so nothing resets them.
  int* dep_signal = nullptr;
  const int* dep_wait = nullptr;
  int dep_mult = 0;
  int dep_per_row = 0;
  int early_trigger = 0;
  int skip_pdl_wait = 0;
  int force_pdl = 0;
};

// window-major row index <-> token index within one image
__host__ __device__ inline int wm_to_token(int r, int grid, int win) {
  const int w2 = win * win, nw = grid / win;
  const int w = r / w2, i = r - w * w2;
  return ((w / nw) * win + i / win) * grid + (w % nw) * win + i % win;
}
__host__ __device__ inline int token_to_wm(int t, int grid, int win) {
  const int r = t / grid, c = t - r * grid, nw = grid / win;
  return (((r / win) * nw + c / win) * win + r % win) * win + c % win;
}

int gemm_bn_for(int N);
// Tile plan: 128 x bn tiles per SM (cg 1) or 256 x bn tiles per CTA pair (cg 2).
struct GemmPlan {
  int bn, cg;
};
GemmPlan gemm_plan(int M, int N, int epi_mode, int num_sms, int splitk = 1);
// split-K workspace sizes for `tiles` output tiles of a plan (see GemmEpi::splitk)
inline long long splitk_flag_count(long long tiles, int cg) { return tiles * cg * 8; }
inline long long splitk_ws_floats(long long tiles, int bn, int cg) { return tiles * cg * 128LL * bn; }
void gemm_force_plan(int bn, int cg);
int gemm_set_trace(long long* device_buf);  // bn 0: automatic
// tA: map over A [M, K] with box {64, 128}; tB: map over W [N, K] with box {64, plan.bn / plan.cg}.
// Output maps over out [M, N] (row stride ldo), box {32, 32}: tC fp32 with 128B swizzle
// (EPI_F32 / EPI_F32_F16 without wm_scatter, and the EPI_F32_RESID residual), tD fp16 with 64B
// swizzle (EPI_F16, EPI_F16_RELU, EPI_QKV_ROPE); the unused one may be null.
// tB2: W map with box {64, plan.bn / 2 / plan.cg} for the tail-halves units (may be null: no tail halves).
int gemm_tc(const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap* tB2, const CUtensorMap* tC,
            const CUtensorMap* tD, int M, int N, int K, GemmPlan plan, int epi_mode, const GemmEpi& epi, int num_sms,
            cudaStream_t stream);

// Fused enc-dec MLP: x[M,256] += relu(h W1^T + b1) W2^T + b2 with W1 [1024, 256], W2 [256, 1024]
// fp16 K-major, hidden activations kept in TMEM.  tH: box {64, 128} over h [M, 256];
// tW1: box {64, 64} over W1; tW2: box {64, 128} over W2; tX: fp32 box {32, 32} 128B swizzle over x.
// tLN / ln_g / ln_b: with ln_g != nullptr the epilogue also writes h = LayerNorm(x) * ln_g + ln_b
// (fp16 [M, 256], box {32, 32} 64B swizzle) -- the next sub-block's LN (tLN unused otherwise).
int mlp_fused(const CUtensorMap& tH, const CUtensorMap& tW1, const CUtensorMap& tW2, const CUtensorMap& tX,
              const CUtensorMap& tLN, int M, const float* b1, const float* b2, const float* ln_g, const float* ln_b,
              int num_sms, cudaStream_t stream);

// Flash attention (fp16 operands, fp32 softmax/accumulation).
struct AttnArgs {
  const __half* q;
  const __half* k;
  const __half* v;
  __half* o;
  int q_tok_stride, k_tok_stride, v_tok_stride, o_tok_stride;  // elements between consecutive tokens
  long long q_batch_stride, k_batch_stride, v_batch_stride, o_batch_stride;  // elements between batch items
  int head_stride_q, head_stride_k, head_stride_v, head_stride_o;            // elements between heads
  int Lq, Lk;
  int heads;
  int batch;
  float scale_log2;      // log2(e) / sqrt(hd)
  // windowed token map (win > 0): batch item z covers window (z % nwin) of image (z / nwin);
  // in-window index i -> token ((wr*win + i/win) * grid + wc*win + i%win), image stride = img_stride
  int win, grid, nwin;
  int kv_batch_mod;      // > 0: K/V batch item = z % kv_batch_mod (class-shared image, per-class text)
  long long img_stride_q, img_stride_k, img_stride_v, img_stride_o;
};
// attention() dispatches short-key (text cross-attention) calls to the all-heads-per-CTA kernel.
int attention(const AttnArgs& a, int head_dim, cudaStream_t stream);
bool attention_short_supported(const AttnArgs& a, int head_dim);

// tcgen05 flash attention over contiguous row blocks of a token-major QKV buffer.
struct AttnTcArgs {
  int Lq, Lkv;                 // query / key rows per item (a partial last key tile is masked)
  int heads, items;
  int q_col, k_col, v_col;     // column offsets of q / k / v in the QKV buffer
  __half* o;                   // [items * L, o_ld]
  int o_ld;
  float scale_log2;
  int* dbg = nullptr;          // host-mapped hang report (tests only), see mbar_wait_dbg
  int force_safe = 0;          // tests: re-run every item through the max-tracking softmax pass
  int z_base = 0;              // first item of this launch (items are chunked on the host)
  int softmax_only = 0;        // microbenchmark: softmax warps run on stale S without MMA / TMA
  long long* trace = nullptr;  // microbenchmark: CTA 0 clock64 stamps [7][256] of the first 256 tiles
  int kv_mod = 0;              // > 0: item z reads K/V item z % kv_mod (text K/V shared by a class's images)
  // Split-KV (flash-decoding): kv_split > 1 runs each (q tile, head, item) as kv_split CTAs over
  // consecutive ranges of key tiles; each writes its rows' unnormalised O, row sum and reference
  // max (log2 units) to part[(((z * heads + h) * kv_split + s) * Lq + row) * 20 + {0..15, 16, 17}]
  // and attention_split_combine merges them into o.  For launches with too few items to fill
  // the GPU (decoder cross-attention at small N: 201 queries x 5184 keys per class).
  int kv_split = 1;
  float* part = nullptr;
};
// Merge of the kv_split partial results of attention_tc (hd 16): o row = sum_s w_s O_s / sum_s w_s l_s
// with w_s = 2^(m_s - max m).
int attention_split_combine(const float* part, __half* o, int o_ld, int items, int heads, int Lq, int kv_split,
                            int hd, cudaStream_t stream);
constexpr int ATTN_TC_MAX_LOCAL_ITEMS = 4096;  // items per CTA per launch (overflow bitmask in smem)
int attention_tc_kv_tile(int head_dim, int Lkv);  // key tile (64 hd 80, 96 hd 16, 32 hd 16 short), 0 = unsupported
void attention_tc_set_variant(int v);  // microbenchmarks (DART_FA_VARIANT otherwise)
bool attention_tc_supported(int head_dim, int Lkv);
// tmQ: 2-D map over the Q buffer [items*Lq, cols] fp16, box {16, 128}, 32B swizzle;
// tmKV: map over the K/V buffer [items*Lkv, cols], box {16, kv_tile}.
int attention_tc(const CUtensorMap& tmQ, const CUtensorMap& tmKV, const AttnTcArgs& a, int head_dim, int num_sms,
                 cudaStream_t stream);

// Row kernels.
// LayerNorm in a row-block dependency chain (see GemmEpi::dep_*): wait_cnt == nullptr: full wait on the
// previous grid; else row r waits until wait_cnt[r / 128] >= wait_target.  Each finished row adds 1 to
// sig_cnt[r / 128]; the kernel triggers its dependents as soon as it starts.
int layernorm_f32_to_f16_chain(const float* x, const float* gamma, const float* beta, __half* y, int rows, int dim,
                               const int* wait_cnt, int wait_target, int* sig_cnt, cudaStream_t stream);
int layernorm_f32_to_f16(const float* x, const float* gamma, const float* beta, __half* y, int rows, int dim,
                         int ld_in, int ld_out, cudaStream_t stream);
int layernorm_f32_to_f32(const float* x, const float* gamma, const float* beta, float* y, int rows, int dim,
                         cudaStream_t stream);
int cast_f32_to_f16(const float* x, __half* y, long long n, cudaStream_t stream);
int patchify(const float* images, __half* patches, int B, int S, int p, int kpad, int win, int* flags,
             cudaStream_t stream);
int pool_tokens(const float* x, __half* y, int B, int grid, int dim, int factor, int win, cudaStream_t stream);
int finite_check(const float* x, long long n, int* flags, int bit, cudaStream_t stream);
int broadcast_rows(const float* src, float* dst, long long row_elems, int reps, cudaStream_t stream);
int gather_rows_f16(const float* table, const int* rows, __half* out, int n, int dim, cudaStream_t stream);
int heads_forward(const float* qf, int rows_per_item, int nq, int items, int d, const float* w_box,
                  const float* b_box, const float* w_score, const float* b_score, const float* w_pres,
                  const float* b_pres, double* boxes, double* scores, double* presence, float* qf_out,
                  cudaStream_t stream);

// Post-processing: per-class gates, (score desc, query asc) order, greedy NMS in fp64.
int postprocess_classes(const double* boxes, const double* score_logits, const double* presence_logits, int N, int Q,
                        double presence_thr, double score_thr, double nms_thr, int* kept_count, int* kept_query,
                        double* kept_score, double* presence_prob, cudaStream_t stream);
int postprocess_cross_class(const double* boxes, const int* kept_count, const int* kept_query,
                            const double* kept_score, int N, int Q, double nms_thr, int* keep_flag, int* scratch,
                            cudaStream_t stream);

}  // namespace dart
