/*
 * dart_b200.h -- C ABI of the B200-native DART multi-class detection path.
 *
 * The reference exposes this path as a Python function API (no FFI); each entry
 * point below replaces the arithmetic of one reference function, and the Python
 * mirror in paper_2603_11441_b200/ binds them with ctypes:
 *
 *   dart_model_create   <- build_model / load_model weight hand-off
 *                          (/root/reference/pkg/src/dart/model.py:306-334, 657-681)
 *   dart_backbone       <- backbone_forward (model.py:454-459: patch_tokens :426,
 *                          _block_forward x num_blocks :412, fpn_from_tokens :446)
 *   dart_encdec         <- encdec_forward (model.py:536-570, per class _encdec_single :511-533)
 *   dart_postprocess    <- postprocess (pipeline.py:266-294)
 *
 * Conventions: plain C, no exceptions across the boundary.  Every function returns
 * an int status (DART_OK = 0); on failure dart_last_error() returns a thread-local
 * message.  All tensor pointers are caller-owned DEVICE pointers, row-major,
 * contiguous; `stream` is a cudaStream_t passed as void*.  No host synchronisation
 * happens inside any entry point except dart_model_create.  A model handle owns its
 * device weights and an activation workspace, and must be used from one stream at
 * a time (one handle per GPU / per concurrent stream).
 */
#ifndef DART_B200_H
#define DART_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DART_OK 0
#define DART_ERR_INVALID 1 /* bad argument / shape: maps to ValueError      */
#define DART_ERR_CUDA 2    /* CUDA launch or allocation failure: RuntimeError */

/* Status-flag bits written by dart_backbone into `flags` (device int32; cleared by the call). */
#define DART_FLAG_IMAGE_RANGE 1   /* some image value outside [0, 1] or NaN (model.py:432-433) */
#define DART_FLAG_NONFINITE 2     /* some FPN level non-finite (model.py:161-166)              */

#define DART_MAX_BLOCKS 256

/* Model dimensions: the fields of the reference ModelConfig (model.py:41-56) plus the
 * per-block structure of DetectorModel (block_kinds / attn_enabled / mlp_enabled,
 * model.py:140-149). */
typedef struct dart_model_desc {
  int32_t image_size, patch_size, embed_dim, num_blocks, window_size, num_heads;
  int32_t fpn_dims[3];
  int32_t text_tokens, text_dim, num_queries, num_encoder_layers, num_decoder_layers;
  int32_t block_global[DART_MAX_BLOCKS]; /* 1 = global attention, 0 = windowed */
  int32_t attn_enabled[DART_MAX_BLOCKS];
  int32_t mlp_enabled[DART_MAX_BLOCKS];
} dart_model_desc;

typedef struct dart_model dart_model;

/* Upload weights.  `weights` holds `n_weights` HOST float32 pointers in the reference's
 * parameter declaration order without the mask head (model.py:216-303, the DARTM1
 * order), each tensor row-major in the reference's [in, out] layout. */
int dart_model_create(const dart_model_desc* desc, const float* const* weights, int32_t n_weights,
                      dart_model** out);
/* A second handle on the same device weights (no copy) with its own activation workspace, so
 * two streams can run the path concurrently (inter-frame pipelining: the backbone of frame t+1
 * on one handle while the enc-dec of frame t runs on the other; the reference models this
 * schedule analytically in scheduler.py:128-187).  Weights stay alive until the last handle
 * sharing them is destroyed. */
int dart_model_fork(const dart_model* parent, dart_model** out);
void dart_model_destroy(dart_model* m);

/* Backbone arithmetic discipline of this handle (forks copy it), for the precision study
 * (reference pipeline.py:318-367, tensors.py:111-170):
 *   0  fp16 operands, fp32 tensor-core accumulation, fp32 residual stream (default, the
 *      detection path);
 *   1  fp16 storage: every backbone GEMM output and the residual stream after each add are
 *      rounded to fp16 (the reference's FP16_ACCUM_FP32 storage discipline);
 *   2  fp16 storage and fp16 accumulation on the tensor core (tcgen05 D format f16): the
 *      FP16_ACCUM_FP16 negative control.
 * Applies to the backbone's GEMMs (patch embed, QKV, out-proj, MLP, FPN); attention and the
 * enc-dec keep fp32 accumulation.  DART_ERR_INVALID for other values. */
int dart_model_set_precision(dart_model* m, int32_t precision);
int32_t dart_model_get_precision(const dart_model* m);

/* Number of parameter tensors dart_model_create expects for `desc`. */
int32_t dart_expected_weight_count(const dart_model_desc* desc);

/* images [B, S, S, 3] float32 in [0,1] -> L0 [B, T, F0], L1 [B, T/4, F1], L2 [B, T/16, F2]
 * float32.  The level-0 features are also kept (fp16) in the workspace for a following
 * dart_encdec(.., l0 = NULL, ..).  `flags` (device int32, zeroed by the caller) receives
 * DART_FLAG_* bits. */
int dart_backbone(dart_model* m, const float* images, int32_t B, float* l0, float* l1, float* l2, int32_t* flags,
                  void* stream);
/* The backbone in stages, for callers that re-run part of it (the reference's pruning search,
 * pruning.py:154-204, memoises the activations entering each block):
 * dart_backbone_embed: images -> x [B*T, E] fp32 (patch embedding; x rows in the engine's
 *   window-major order: window-major row r of image b is token wm_to_token(r));
 * dart_backbone_blocks: x <- blocks [b0, b1) applied in place, attn_on / mlp_on HOST int32
 *   arrays of num_blocks sub-block enables (NULL: the handle's own flags);
 * dart_backbone_fpn: x -> L0 / L1 / L2 (token-major) + finiteness flag bits (OR-ed in).
 * dart_backbone == embed + blocks(0, num_blocks) + fpn. */
int dart_backbone_embed(dart_model* m, const float* images, int32_t B, float* x, int32_t* flags, void* stream);
int dart_backbone_blocks(dart_model* m, float* x, int32_t B, int32_t b0, int32_t b1, const int32_t* attn_on,
                         const int32_t* mlp_on, void* stream);
int dart_backbone_fpn(dart_model* m, const float* x, int32_t B, float* l0, float* l1, float* l2, int32_t* flags,
                      void* stream);

/* Class-batched encoder-decoder for B images x N classes.
 *   l0    [B, T, F0] float32 level-0 features, or NULL to reuse the last dart_backbone output
 *   text  [N, L_t, d] float32 text embeddings (rows of text.table, model.py:470-484)
 * outputs (item = b * N + c), float64 like the reference's RawQueryOutputs (model.py:177-188):
 *   boxes [B*N, Q, 4]  sigmoid (cx, cy, w, h);  score_logits [B*N, Q];  presence_logits [B*N]
 *   query_features [B*N, Q, d] float32, or NULL. */
int dart_encdec(dart_model* m, const float* l0, int32_t B, const float* text, int32_t N, double* boxes,
                double* score_logits, double* presence_logits, float* query_features, void* stream);

/* The same enc-dec split at its class-independent prefix (model.py:513-517: input projection and
 * encoder layer-0 self-attention; text first enters at :518), for class sharding across GPUs
 * (SURVEY 8(e) config 5): dart_encdec_prefix writes e1 [B, T, d] float32 (l0 NULL: the last
 * dart_backbone output), which a caller may exchange between ranks (NCCL all-gather) before each
 * rank runs dart_encdec_from_prefix on its own class shard.  dart_encdec == prefix + from_prefix
 * (bitwise). */
int dart_encdec_prefix(dart_model* m, const float* l0, int32_t B, float* e1, void* stream);
int dart_encdec_from_prefix(dart_model* m, const float* e1, int32_t B, const float* text, int32_t N, double* boxes,
                            double* score_logits, double* presence_logits, float* query_features, void* stream);

/* The model description a handle was created with (dimensions of its workspaces). */
const dart_model_desc* dart_model_get_desc(const dart_model* m);

/* ---- NCCL helpers for class sharding across GPUs ----
 * One communicator per rank (one rank per GPU); libnccl.so.2 is opened at first use, so a host
 * without NCCL still loads the library (dart_nccl_available() == 0 then).  Every call only
 * enqueues on `stream`.  Unique-id exchange between the ranks is the caller's (any side channel:
 * torch.distributed, MPI, a file).  Replaces the torch.distributed collectives of
 * paper_2603_11441_b200/distributed.py:class_sharded_raw for hosts without torch. */
#define DART_NCCL_ID_BYTES 128
typedef struct dart_comm dart_comm;
int dart_nccl_available(void);
int dart_nccl_unique_id(uint8_t* id /* [DART_NCCL_ID_BYTES], host */);
int dart_nccl_comm_create(const uint8_t* id, int32_t nranks, int32_t rank, dart_comm** out);
void dart_nccl_comm_destroy(dart_comm* c);
/* Failure detection: 0 while the communicator is healthy, else the asynchronous NCCL error (a
 * dead peer, a broken link) as a status + dart_last_error; never blocks.  dart_nccl_comm_abort
 * aborts the communicator (ncclCommAbort) so that no rank stays blocked in a collective; later
 * calls on it fail.  The timeout policy is the caller's (Python: distributed.NcclComm.wait). */
int dart_nccl_comm_check(dart_comm* c);
int dart_nccl_comm_abort(dart_comm* c);
int32_t dart_nccl_comm_size(const dart_comm* c);
int32_t dart_nccl_comm_rank(const dart_comm* c);
/* recv [nranks * bytes_per_rank] <- send [bytes_per_rank] of every rank, in rank order */
int dart_nccl_all_gather(dart_comm* c, const void* send, void* recv, int64_t bytes_per_rank, void* stream);
int dart_nccl_all_reduce_max_i32(dart_comm* c, int32_t* buf, int64_t count, void* stream);
/* One class-sharded round (model.py:513-517 prefix, 559-564 class loop): this rank's images
 * [B, S, S, 3] -> backbone + enc-dec prefix -> all-gather of e1 (fp32) -> this rank's contiguous
 * class shard (ClassShardPlan: the first N % W ranks get ceil(N/W) classes) of text [N, L_t, d]
 * decoded for all W*B images -> all-gather of the raw outputs -> boxes [B*N, Q, 4], score_logits
 * [B*N, Q], presence_logits [B*N] float64 of THIS rank's images over all N classes (item b*N+c,
 * bitwise equal to dart_encdec on the same images), flags (zeroed by the caller) MAX-reduced
 * over the ranks.  Every rank must call it with the same B and N. */
int dart_class_sharded(dart_model* m, dart_comm* c, const float* images, int32_t B, const float* text, int32_t N,
                       double* boxes, double* score_logits, double* presence_logits, int32_t* flags, void* stream);

/* Presence gate, score gate, (score desc, query asc) ordering and greedy per-class NMS,
 * decisions in fp64 (pipeline.py:243-294).  Inputs float64 [N,Q,4] / [N,Q] / [N].  For N items of Q queries:
 *   kept_count [N] int32, kept_query [N, Q] int32, kept_score [N, Q] float64 (sigmoid),
 *   presence_prob [N] float64.
 * cross_class != 0 additionally runs cross-class NMS and writes keep_flag [N, Q] int32
 * (1 = survivor of slot k of item c); scratch must hold N*(2Q+1)+1 int32. */
int dart_postprocess(dart_model* m, const double* boxes, const double* score_logits, const double* presence_logits,
                     int32_t N, int32_t Q, double presence_threshold, double score_threshold,
                     double nms_iou_threshold, int32_t cross_class, int32_t* kept_count, int32_t* kept_query,
                     double* kept_score, double* presence_prob, int32_t* keep_flag, int32_t* scratch,
                     void* stream);

/* Mask head (the non-detection-only path, mask_head_forward, model.py:573-579).
 * dart_model_set_mask_head uploads the four mask tensors (HOST float32, reference [in, out]
 * layout: mask.query_proj.w [d, d], .b [d], mask.feat_proj.w [F0, d], .b [d]).
 * dart_mask_head: query_features [B*N, Q, d] fp32 (dart_encdec's optional output), l0 [B, T, F0]
 * fp32 -> masks [B*N, Q, T] fp32 = (qf Wq + bq) (L0[b] Wf + bf)^T per image b. */
int dart_model_set_mask_head(dart_model* m, const float* wq, const float* bq, const float* wf, const float* bf);
int dart_mask_head(dart_model* m, const float* query_features, int32_t B, int32_t N, const float* l0, float* masks,
                   void* stream);

/* Kernel-level entry points (used by the per-kernel parity tests and microbenchmarks).
 * dart_gemm: out = epilogue(A[M,K] . W[N,K]^T + bias), A/W fp16 K-major, K % 64 == 0,
 *   N % 64 == 0; epi 0 fp16 out, 1 fp16 relu, 2 fp32 out, 3 fp32 out += , 4 fp16 with RoPE on
 *   columns < rope_cols (the model's 2-D RoPE tables [rope_T, rope_hd/2] = row | column angles,
 *   rope_T a square grid <= 72^2, rope_hd / 4 <= 20), 5 fp32 out + fp16 out2.
 * dart_gemm_plan: the tile plan dart_gemm / the model forwards use for (M, N, epi) on this GPU
 *   (bn = tile width, cg = 1: 128-row tiles per SM, 2: 256-row tiles per CTA pair).
 * dart_gemm_force_plan: force (bn, cg) for every later GEMM whose N allows it (tests and A/B
 *   measurement); bn = 0 restores the automatic plan.  With DART_SPLITK=1 in the environment the
 *   model path runs residual GEMMs with K >= 4096 (backbone fc2) split-K (measured slower; A/B only).
 * dart_attention: o = softmax(q k^T / sqrt(hd)) v, fp16 in/out, tokens `*_tok_stride`
 *   elements apart, heads hd apart, batch items `*_batch_stride` apart; win > 0 selects the
 *   windowed token map over a grid x grid token image (batch = images * (grid/win)^2). */
int dart_gemm(const void* A, const void* W, const float* bias, void* out, void* out2, int32_t M, int32_t N,
              int32_t K, int32_t epi, const float* rope_cos, const float* rope_sin, int32_t rope_T, int32_t rope_hd,
              int32_t rope_cols, void* stream);
/* The enc-dec's sub-block-closing residual GEMM with the NEXT sub-block's LayerNorm fused into its
 * epilogue (d = 256, whole rows per tile): x[M, 256] += A[M, K] . W[256, K]^T + bias, then
 * h[M, 256] (fp16) = LayerNorm(x) * ln_g + ln_b (population variance, eps 1e-6; reference
 * tensors.py:215-227, model.py:516-527). */
int dart_gemm_resid_ln(const void* A, const void* W, const float* bias, float* x, void* h, const float* ln_g,
                       const float* ln_b, int32_t M, int32_t K, void* stream);
void dart_gemm_plan(int32_t M, int32_t N, int32_t epi, int32_t* bn, int32_t* cg);
void dart_gemm_force_plan(int32_t bn, int32_t cg);
/* Timeline microbenchmarks: per-CTA %globaltimer stamps (8 int64 per CTA: entry, after the PDL
 * wait, first operand stage landed, first / last accumulator committed, first accumulator seen by
 * the epilogue, epilogue done, exit) of every following GEMM launch into device_buf; NULL = off. */
int dart_gemm_trace(int64_t* device_buf);
/* Fused enc-dec MLP (reference _mlp_forward, model.py:505-508, d = 256, hidden 1024):
 * x[M, 256] += relu(h W1^T + b1) W2^T + b2, h fp16 [M, 256], W1 fp16 [1024, 256], W2 fp16 [256, 1024]
 * (both [out, in]), x fp32; the hidden activations never leave the SM (TMEM). */
int dart_mlp_fused(const void* h, const void* w1, const float* b1, const void* w2, const float* b2, float* x, int32_t M,
                   void* stream);
/* The same with the next sub-block's LayerNorm fused into the residual epilogue: also
 * h_out[M, 256] (fp16) = LayerNorm(x) * ln_g + ln_b of the new rows (h_out may alias h).
 * ln_g == NULL: plain dart_mlp_fused. */
int dart_mlp_fused_ln(const void* h, const void* w1, const float* b1, const void* w2, const float* b2, float* x,
                      void* h_out, const float* ln_g, const float* ln_b, int32_t M, void* stream);
/* y = LayerNorm(x) per row (population variance, eps 1e-6; reference tensors.py:215-227), fp32 in,
 * fp16 (out_f16 = 1) or fp32 out; dim in {32, 64, 128, 256, 512, 1024, 1280}. */
int dart_layernorm(const float* x, const float* gamma, const float* beta, void* y, int32_t rows, int32_t dim,
                   int32_t out_f16, void* stream);
/* Tests: s = 2 makes later dart_gemm residual calls (epi 3, K/64 even) run split-K (two K halves
 * per tile on different CTA pairs, deterministic adds); s = 1 restores the default. */
void dart_gemm_force_splitk(int32_t s);
/* Tests: later dart_gemm calls use precision discipline p (see dart_model_set_precision:
 * 1 fp16 storage, 2 fp16 storage + fp16 accumulation); 0 restores the default. */
void dart_gemm_force_precision(int32_t p);
int dart_attention(const void* q, const void* k, const void* v, void* o, int32_t batch, int32_t heads, int32_t Lq,
                   int32_t Lk, int32_t hd, int32_t q_tok_stride, int32_t kv_tok_stride, int32_t o_tok_stride,
                   int64_t q_batch_stride, int64_t kv_batch_stride, int64_t o_batch_stride, int32_t win,
                   int32_t grid, void* stream);

/* tcgen05/TMEM flash attention on a packed QKV buffer [items * L, 3 * heads * hd] fp16 (q | k | v
 * column blocks, head-major inside each), o [items * L, heads * hd] fp16.  hd = 80, L % 192 == 0
 * (the backbone's windowed and global attention, model.py:390-409).  debug_host: NULL, or host-mapped
 * int32[8] that receives a protocol-hang report (tests only). */
int dart_attention_qkv(const void* qkv, void* o, int32_t items, int32_t heads, int32_t L, int32_t hd,
                       int32_t* debug_host, void* stream);
/* Tests: on != 0 makes every later tcgen05 attention launch re-run all of its items through the
 * max-tracking softmax pass (the path items take when the fixed-reference pass overflows). */
void dart_attention_force_safe(int32_t on);
/* Microbenchmarks: device int64[11 * 256] receiving CTA 0's clock64 stamps of its first 256 key
 * tiles (S ready, P written, P seen by the MMA issuer, MMAs issued, V ready, P.V issued, next K
 * ready, then P done per softmax warp 2..5); NULL disables. */
void dart_attention_trace(int64_t* device_buf);
/* Microbenchmarks: select the tcgen05 attention kernel variant (0 = production). */
void dart_attention_variant(int32_t v);

/* Programmatic dependent launch for the calling host thread's later launches: 1 = on (each GEMM /
 * attention / LayerNorm kernel may start its prologue while its predecessor drains: +2% on one
 * stream), 0 = off (fully serialised kernel boundaries: measured better when several streams
 * share the GPU, as in the inter-frame pipeline), -1 = the process default (on; DART_NO_PDL=1
 * turns it off). */
void dart_set_pdl(int32_t mode);

/* Backbone LayerNorms folded into the consuming GEMMs in dart_backbone (the residual producers
 * also write fp16(x) and per-row chunk statistics).  Mask: bit 0 LN1 -> QKV, bit 1 LN2 -> fc1;
 * 0 = the standalone LayerNorm passes (the default: measured faster on the B200; DART_LN_FOLD
 * sets the process default).  Folded weights are built by handles created while the mask is
 * non-zero.  Process wide; tests and A/B measurement. */
void dart_set_ln_fold(int32_t mask);

/* Split-KV factor (1..8) of the enc-dec decoder cross-attention: each (query tile, head, class) item
 * over the T image keys runs as k CTAs over consecutive key ranges, merged by a small kernel.
 * 1 = off (the default: it helps only small N, DART_ATTN_SPLIT sets the process default).
 * Process wide; tests and A/B measurement. */
void dart_attention_kv_split(int32_t k);

/* Row-block dependency chain inside dart_backbone (fc1 -> fc2 -> next LN1 -> QKV start on the row
 * blocks their producer finished, in its last wave): 1 = on, 0 = off (the default: measured no
 * faster; DART_CHAIN sets the process default).  Results are bitwise identical either way.
 * Process wide; tests and A/B measurement. */
void dart_set_chain(int32_t on);

/* Kernel launches issued by the last dart_backbone + dart_encdec + dart_postprocess calls
 * on this handle (for the bench's gpu_launches evidence). */
int64_t dart_launch_count(const dart_model* m);
void dart_reset_launch_count(dart_model* m);

const char* dart_last_error(void);
const char* dart_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DART_B200_H */
