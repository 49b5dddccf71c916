// C ABI of the DART B200 path (include/dart_b200.h): weight upload, workspace, and
// the orchestration of the backbone / class-batched enc-dec / post-processing kernels.
//
// Data layout in HBM (per model handle):
//   weights   GEMM weights transposed to [out, in] fp16 (K-major for tcgen05), one TMA
//             descriptor each (128B swizzle, box 64 x BN); biases, LN affine, RoPE tables,
//             text table and heads in fp32.  The 6 encoder cross-attention K/V projections
//             and the 6 decoder cross-attention K/V projections are each concatenated into
//             one [6*2d, d] weight so one GEMM per pass reads its input once.
//   backbone  residual stream x [B*T, E] fp32; LN outputs / qkv / attention out / MLP hidden fp16.
//   enc-dec   class-shared prefix e1 [B*T, d] fp32; per-class residual e [B*N*T, d] fp32;
//             decoder memory K/V for all layers [B*N*T, 6*2d] fp16; decoder stream [B*N*201, d] fp32.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/dart_b200.h"
#include "common.cuh"
#include "kernels.h"

using namespace dart;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CK(expr)                                                                                   \
  do {                                                                                             \
    int _e = (int)(expr);                                                                          \
    if (_e != 0) {                                                                                 \
      char _b[256];                                                                                \
      snprintf(_b, sizeof(_b), "%s failed: %s (%s:%d)", #expr, cudaGetErrorString((cudaError_t)_e), \
               __FILE__, __LINE__);                                                                \
      return fail(DART_ERR_CUDA, _b);                                                              \
    }                                                                                              \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D fp16 tensor map over [rows, inner] with row stride `ld` elements, 128B swizzle.
bool make_tmap_ex(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t rows, uint64_t ld, uint32_t box_inner,
                  uint32_t box_rows, CUtensorMapSwizzle swz) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
bool make_tmap(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t rows, uint64_t ld, uint32_t box_rows) {
  return make_tmap_ex(m, ptr, inner, rows, ld, 64, box_rows, CU_TENSOR_MAP_SWIZZLE_128B);
}
// fp32 [rows, inner] map with 32 x 32 boxes (128 B rows, 128B swizzle): the GEMM residual tiles.
bool make_tmap_f32(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t rows, uint64_t ld) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Attention implementation switch for A/B tests: DART_ATTN_IMPL=mma forces the mma.sync kernel.
bool tc_attention_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DART_ATTN_IMPL");
    v = (e && strcmp(e, "mma") == 0) ? 0 : 1;
  }
  return v == 1;
}

// Tests: route every tcgen05 attention item through the max-tracking (overflow-safe) pass too.
int g_attn_force_safe = 0;
// Split-K (two K halves per tile, partial-accumulator combine; gemm_tc.cu) for the backbone GEMMs
// whose tile count leaves a badly filled last wave at one image (5184 rows): bit 1 QKV (315
// CTA-pair tiles = 4.26 waves on 74 pairs), bit 2 attn.out and bit 4 mlp.fc2 (105 tiles = 1.42
// waves).  Chosen per (N, K) only, so the arithmetic of a row never depends on the batch size.
// Off by default: measured slower on every shape (profiles/r02/gemm_splitk.log -- a CTA writes its
// 128 KB fp32 partial at ~26 GB/s, ~5 us, as long as the attn.out half-tile main loop).
// DART_SPLITK=<mask> enables it for A/B measurement.
int g_splitk_mask = getenv("DART_SPLITK") ? atoi(getenv("DART_SPLITK")) : 0;
// Backbone LayerNorms folded into the GEMMs that consume them (see bb_blocks).  Mask: bit 0
// LN1 -> QKV (producers: patch embed, mlp.fc2), bit 1 LN2 -> fc1 (producer: attn.out).  Off by
// default: parity-equivalent but slower on the B200 (profiles/r02/ln_fold_ab.log) -- the residual
// GEMM's epilogue, which bounds attn.out and the last fc2 wave, grows by the fp16 copy and the
// statistics more than the LayerNorm pass it replaces costs.  The folded weights exist only in
// handles created while the fold is enabled (DART_LN_FOLD=<mask> or dart_set_ln_fold).
int g_ln_fold = getenv("DART_LN_FOLD") ? atoi(getenv("DART_LN_FOLD")) : 0;
// Row-block dependency chain fc1 -> fc2 -> LN1(next block) -> QKV inside the backbone (GemmEpi::dep_*):
// each consumer starts on the 128-row blocks its producer has finished, in the SMs the producer's
// last wave leaves idle.  Correct (parity B / C, batch invariance) but not faster: serial step
// -0.5%, inter-frame pipeline -1 to -2% (the store-completion waits behind each signal and the
// chain LayerNorm's fences cost what the overlap saves; profiles/r02/chain_ab.log).  Off by default;
// DART_CHAIN=1 turns it on (A/B).
int g_chain = getenv("DART_CHAIN") ? atoi(getenv("DART_CHAIN")) : 0;
// split-KV factor of the decoder cross-attention (xattn); DART_ATTN_SPLIT=<k>, <= 1: off.  Off by
// default: 2-way saves 40 us per N=4 step (128 items for 296 CTA slots) but costs ~0.5 ms per N=80
// step (partials + merge where the items already fill the GPU), and a split that depended on N
// would break the bitwise batch invariance of a class's rows (profiles/r02/attn_hd16_chains.log).
int g_attn_split = getenv("DART_ATTN_SPLIT") ? atoi(getenv("DART_ATTN_SPLIT")) : 1;
int g_gemm_splitk = 1;  // dart_gemm_force_splitk (kernel-level tests)
int g_gemm_precision = 0;  // dart_gemm_force_precision (kernel-level tests)
int g_fused_mlp = getenv("DART_NO_FUSED_MLP") == nullptr;  // enc-dec MLP on the fused kernel
int g_fused_ln = getenv("DART_NO_FUSED_LN") == nullptr;    // enc-dec LayerNorms in the residual epilogues
long long* g_attn_trace = nullptr;

// tcgen05 attention: Q rows [items*Lq, q_ld] (q at column q_col, head h at +h*hd), K/V rows
// [items*Lkv, kv_ld] (k at k_col, v at v_col), output [items*Lq, o_ld] at column h*hd.
int attn_tc(const __half* qbuf, int q_ld, int q_col, const __half* kvbuf, int kv_ld, int k_col, int v_col, __half* o,
            int o_ld, int items, int heads, int Lq, int Lkv, int hd, int num_sms, cudaStream_t s, int* dbg = nullptr,
            int kv_mod = 0, int kv_split = 1, float* part = nullptr) {
  CUtensorMap tq, tkv;  // maps cover exactly the used column ranges
  const int q_inner = q_col + heads * hd, kv_inner = (k_col > v_col ? k_col : v_col) + heads * hd;
  const int kv_items = kv_mod > 0 ? kv_mod : items;
  if (!make_tmap_ex(&tq, qbuf, q_inner, (uint64_t)items * Lq, q_ld, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B) ||
      !make_tmap_ex(&tkv, kvbuf, kv_inner, (uint64_t)kv_items * Lkv, kv_ld, 16, attention_tc_kv_tile(hd, Lkv),
                    CU_TENSOR_MAP_SWIZZLE_32B))
    return fail(DART_ERR_CUDA, "cuTensorMapEncodeTiled failed (attention)");
  AttnTcArgs a;
  a.Lq = Lq;
  a.Lkv = Lkv;
  a.heads = heads;
  a.items = items;
  a.q_col = q_col;
  a.k_col = k_col;
  a.v_col = v_col;
  a.o = o;
  a.o_ld = o_ld;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
  a.dbg = dbg;
  a.force_safe = g_attn_force_safe;
  a.trace = g_attn_trace;
  a.kv_mod = kv_mod;
  a.kv_split = kv_split;
  a.part = part;
  {
    const char* e = getenv("DART_FA_SOFTMAX_ONLY");  // microbenchmarks: 1 softmax alone, 2 MMA alone
    a.softmax_only = e ? atoi(e) : 0;
  }
  int rc = attention_tc(tq, tkv, a, hd, num_sms, s);
  if (!rc && kv_split > 1) rc = attention_split_combine(part, o, o_ld, items, heads, Lq, kv_split, hd, s);
  if (rc) return fail(DART_ERR_CUDA, std::string("attention_tc: ") + cudaGetErrorString((cudaError_t)rc));
  return 0;
}

// Backbone self-attention on a packed QKV buffer [items * L, 3E].
int attn_tc_packed(const __half* qkv, __half* o, int items, int heads, int L, int hd, int E, int num_sms,
                   cudaStream_t s, int* dbg = nullptr) {
  return attn_tc(qkv, 3 * E, 0, qkv, 3 * E, E, 2 * E, o, E, items, heads, L, L, hd, num_sms, s, dbg);
}

struct GemmW {
  __half* w = nullptr;  // [N, K] fp16
  float* b = nullptr;   // [N]
  float* colsum = nullptr;  // LN-folded weights only: [N] column sums of the fp16 W' (GemmEpi::ln_colsum)
  int N = 0, K = 0;
  CUtensorMap tmap[6];  // box rows 256 / 128 / 64 / 32 / 96 / 80 (index = box_slot(rows)), built where N allows
};
constexpr int kBoxRows[6] = {256, 128, 64, 32, 96, 80};
inline int box_slot(int rows) {
  return rows == 256 ? 0 : rows == 128 ? 1 : rows == 64 ? 2 : rows == 32 ? 3 : rows == 96 ? 4 : 5;
}
struct LNW {
  float* g = nullptr;
  float* b = nullptr;
};
struct AttnW {
  GemmW q, kv, out;
  GemmW qkv;  // self-attention: [q | kv] rows in one [3d, d] weight (one GEMM reads LN1(x) once)
};
struct BlockW {
  LNW ln1, ln2;
  GemmW qkv, out, fc1, fc2;
  GemmW qkv_f, fc1_f;  // qkv / fc1 with LN1 / LN2 folded in (W' = diag(gamma) W, b' = b + beta W)
};
struct XLayerW {
  LNW ln1, ln2, ln3;
  AttnW self, cross;
  GemmW fc1, fc2;
};

__global__ void transpose_cast_kernel(const float* __restrict__ src, __half* __restrict__ dst, int in, int out,
                                      int kpad) {
  // src [in, out] fp32 -> dst [out, kpad] fp16 (zero for k >= in)
  __shared__ float tile[32][33];
  const int o0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = i0 + r, o = o0 + threadIdx.x;
    tile[r][threadIdx.x] = (i < in && o < out) ? src[(long long)i * out + o] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int o = o0 + r, i = i0 + threadIdx.x;
    if (o < out && i < kpad) dst[(long long)o * kpad + i] = __float2half_rn(tile[threadIdx.x][r]);
  }
}

struct Workspace {
  std::vector<void*> allocs;
  size_t bytes = 0;
  void* get(size_t n) {
    n = (n + 255) & ~size_t(255);
    void* p = nullptr;
    if (cudaMalloc(&p, n) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    bytes += n;
    return p;
  }
  void release() {
    for (void* p : allocs) cudaFree(p);
    allocs.clear();
    bytes = 0;
  }
};

// Device weight buffers, shared by a model handle and its forks (dart_model_fork).
struct OwnedBuffers {
  std::vector<void*> p;
  ~OwnedBuffers() {
    for (void* x : p) cudaFree(x);
  }
};

}  // namespace

struct dart_model {
  dart_model_desc d;
  int T = 0, G = 0, E = 0, H = 0, hd = 0, kpatch = 0, kpad = 0, D = 0, Lt = 0, Q1 = 0, F0 = 0, F1 = 0, F2 = 0;
  int num_sms = 148;
  std::shared_ptr<OwnedBuffers> owned = std::make_shared<OwnedBuffers>();
  GemmW patch;
  float* rope_cos = nullptr;
  float* rope_sin = nullptr;
  std::vector<BlockW> blocks;
  GemmW fpn[3];
  float* text_table = nullptr;
  GemmW enc_in;
  std::vector<XLayerW> enc, dec;
  LNW enc_final, dec_final;
  GemmW enc_cross_kv_all, dec_cross_kv_all;
  float* queries = nullptr;  // [Q+1, d] fp32 (queries then presence token)
  float *box_w = nullptr, *box_b = nullptr, *score_w = nullptr, *score_b = nullptr, *pres_w = nullptr,
        *pres_b = nullptr;
  // optional mask head (dart_model_set_mask_head)
  bool has_mask = false;
  GemmW mask_q, mask_f;
  // workspaces
  Workspace bb_ws, ed_ws, mask_ws;
  size_t mask_cap_rows = 0, mask_cap_tok = 0;
  __half *mk_qf = nullptr, *mk_l0 = nullptr, *mk_mq = nullptr, *mk_mf = nullptr;
  int bb_cap = 0, ed_cap_items = 0, ed_cap_n = 0, ed_cap_b = 0;
  int last_backbone_B = 0;
  struct {
    __half *patches, *h, *qkv, *ao, *hid, *pool1, *pool2, *l0h;
    float* x;
    float2* lnst;  // LN fold: per-row chunk statistics of x [rows, E / 32] (h holds fp16(x))
    float2* lnfin;  // LN fold: per-row (mean, rstd) of x [rows]
    int* lncnt;     // LN fold: chunk counters per 32-row group [rows / 32] (zeroed at allocation)
    int* chain;     // row-block dependency chain counters [3][rows / 128 + 1]: fc1, fc2, LN1 (zeroed)
  } bb{};
  struct {
    float *e1, *e, *qd, *qd0, *qf;
    __half *l0h, *h, *q, *kv, *o, *hid, *dkv, *text, *tkv, *dh, *dq, *dkvs, *do_, *dhid;
  } ed{};
  int64_t launches = 0;
  // backbone arithmetic discipline (dart_model_set_precision): 0 fp32 accumulate + fp32 residual,
  // 1 fp16 storage (outputs and residual rounded to fp16), 2 fp16 storage + fp16 accumulation
  int precision = 0;
  bool in_backbone = false;  // set while a backbone stage issues its GEMMs
  bool x16_valid = false;    // LN fold: bb.h holds fp16 of the backbone residual stream (last producer)
  // row-block dependency chain (bb_blocks): rows the counters were last used for, and the number of
  // completed signalling launches per counter array (the cumulative targets)
  int chain_rows = -1;
  int chain_epoch[3] = {0, 0, 0};
  // split-K claim flags and partial accumulators, per handle (a fork gets its own)
  int* splitk_flags = nullptr;
  long long splitk_cap = 0;  // flags
  float* splitk_ws = nullptr;
  long long splitk_ws_cap = 0;  // floats
  float* attn_part = nullptr;  // split-KV attention partials (per handle)
  size_t attn_part_cap = 0;    // floats

  ~dart_model() {
    if (attn_part) cudaFree(attn_part);
    if (splitk_flags) cudaFree(splitk_flags);
    if (splitk_ws) cudaFree(splitk_ws);
    bb_ws.release();
    ed_ws.release();
    mask_ws.release();
  }
};

namespace {

template <typename T>
T* dev_alloc(dart_model* m, size_t n) {
  void* p = nullptr;
  if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) return nullptr;
  m->owned->p.push_back(p);
  return reinterpret_cast<T*>(p);
}

float* upload_f32(dart_model* m, const float* h, size_t n) {
  float* d = dev_alloc<float>(m, n);
  if (d && cudaMemcpy(d, h, n * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  return d;
}

// Transposed fp16 weight from a host [in, out] fp32 matrix, written at row offset `row0`
// of a [total_out, kpad] destination.
bool upload_wT(dart_model* m, const float* h, int in, int out, __half* dst, int kpad, int row0, float* scratch) {
  if (cudaMemcpy(scratch, h, (size_t)in * out * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess) return false;
  dim3 grid((out + 31) / 32, (kpad + 31) / 32);
  transpose_cast_kernel<<<grid, dim3(32, 8)>>>(scratch, dst + (size_t)row0 * kpad, in, out, kpad);
  return cudaGetLastError() == cudaSuccess;
}

// LayerNorm folded into the following linear (GemmEpi::ln_stats): from the host-layout fp32
// [in, out] weight in `src`: wT[n, k] = fp16(gamma[k] W[k, n]), bias'[n] = b[n] + sum_k beta[k] W[k, n],
// colsum[n] = sum_k float(wT[n, k]) -- the column sums of exactly the fp16 values the MMA reads.
__global__ void ln_fold_kernel(const float* __restrict__ src, const float* __restrict__ g, const float* __restrict__ beta,
                               const float* __restrict__ bias, int in, int out, __half* __restrict__ wT,
                               float* __restrict__ bias_f, float* __restrict__ colsum) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= out) return;
  float bacc = bias[n], cs = 0.f;
  for (int k = 0; k < in; ++k) {
    const float wv = src[(long long)k * out + n];
    const __half h = __float2half_rn(g[k] * wv);
    wT[(long long)n * in + k] = h;
    cs += __half2float(h);
    bacc = fmaf(beta[k], wv, bacc);
  }
  bias_f[n] = bacc;
  colsum[n] = cs;
}

bool finish_gemmw(GemmW& g);
// Folded twin of `g` (whose host fp32 [in, out] weight is still in `scratch`, see upload_wT).
bool make_folded(dart_model* m, const GemmW& g, const LNW& ln, const float* scratch, GemmW& f) {
  f.N = g.N;
  f.K = g.K;
  f.w = dev_alloc<__half>(m, (size_t)f.N * f.K);
  f.b = dev_alloc<float>(m, f.N);
  f.colsum = dev_alloc<float>(m, f.N);
  if (!f.w || !f.b || !f.colsum) return false;
  ln_fold_kernel<<<(f.N + 127) / 128, 128>>>(scratch, ln.g, ln.b, g.b, g.K, g.N, f.w, f.b, f.colsum);
  return cudaGetLastError() == cudaSuccess && finish_gemmw(f);
}

bool finish_gemmw(GemmW& g) {
  bool any = false;
  for (int rows : kBoxRows) {  // W box rows = plan.bn / plan.cg
    if (g.N % rows) continue;
    if (!make_tmap(&g.tmap[box_slot(rows)], g.w, g.K, g.N, g.K, rows)) return false;
    any = true;
  }
  return any;
}

struct WeightCursor {
  const float* const* w;
  int n, i = 0;
  const float* next() { return i < n ? w[i++] : nullptr; }
};

bool make_gemm(dart_model* m, WeightCursor& c, int in, int out, float* scratch, GemmW& g, int kpad = 0) {
  const float* wh = c.next();
  const float* bh = c.next();
  if (!wh || !bh) return false;
  g.N = out;
  g.K = kpad ? kpad : in;
  g.w = dev_alloc<__half>(m, (size_t)g.N * g.K);
  if (!g.w || !upload_wT(m, wh, in, out, g.w, g.K, 0, scratch)) return false;
  g.b = upload_f32(m, bh, out);
  return g.b && finish_gemmw(g);
}

bool make_ln(dart_model* m, WeightCursor& c, int dim, LNW& l) {
  const float* gh = c.next();
  const float* bh = c.next();
  if (!gh || !bh) return false;
  l.g = upload_f32(m, gh, dim);
  l.b = upload_f32(m, bh, dim);
  return l.g && l.b;
}

// Attention projections; when `fused` is non-null the K/V projection of this layer is
// also written into the concatenated [layers*2d, d] weight at row offset `row0`.
bool make_attn(dart_model* m, WeightCursor& c, int d, float* scratch, AttnW& a, GemmW* fused, int row0) {
  if (!make_gemm(m, c, d, d, scratch, a.q)) return false;
  const float* kvw = c.next();
  const float* kvb = c.next();
  if (!kvw || !kvb) return false;
  if (fused) {
    if (!upload_wT(m, kvw, d, 2 * d, fused->w, d, row0, scratch)) return false;
    if (cudaMemcpy(fused->b + row0, kvb, 2 * d * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess) return false;
  } else {
    a.kv.N = 2 * d;
    a.kv.K = d;
    a.kv.w = dev_alloc<__half>(m, (size_t)2 * d * d);
    if (!a.kv.w || !upload_wT(m, kvw, d, 2 * d, a.kv.w, d, 0, scratch)) return false;
    a.kv.b = upload_f32(m, kvb, 2 * d);
    if (!a.kv.b || !finish_gemmw(a.kv)) return false;
    // fused self-attention projection: rows [0, d) = q, [d, 3d) = k | v
    a.qkv.N = 3 * d;
    a.qkv.K = d;
    a.qkv.w = dev_alloc<__half>(m, (size_t)3 * d * d);
    a.qkv.b = dev_alloc<float>(m, 3 * d);
    if (!a.qkv.w || !a.qkv.b) return false;
    if (cudaMemcpy(a.qkv.w, a.q.w, (size_t)d * d * 2, cudaMemcpyDeviceToDevice) != cudaSuccess ||
        cudaMemcpy(a.qkv.w + (size_t)d * d, a.kv.w, (size_t)2 * d * d * 2, cudaMemcpyDeviceToDevice) != cudaSuccess ||
        cudaMemcpy(a.qkv.b, a.q.b, d * 4, cudaMemcpyDeviceToDevice) != cudaSuccess ||
        cudaMemcpy(a.qkv.b + d, a.kv.b, 2 * d * 4, cudaMemcpyDeviceToDevice) != cudaSuccess || !finish_gemmw(a.qkv))
      return false;
  }
  return make_gemm(m, c, d, d, scratch, a.out);
}

bool make_xlayer(dart_model* m, WeightCursor& c, int d, float* scratch, XLayerW& L, GemmW* fused, int row0) {
  return make_ln(m, c, d, L.ln1) && make_attn(m, c, d, scratch, L.self, nullptr, 0) && make_ln(m, c, d, L.ln2) &&
         make_attn(m, c, d, scratch, L.cross, fused, row0) && make_ln(m, c, d, L.ln3) &&
         make_gemm(m, c, d, 4 * d, scratch, L.fc1) && make_gemm(m, c, 4 * d, d, scratch, L.fc2);
}

int check_desc(const dart_model_desc* d) {
  if (!d) return fail(DART_ERR_INVALID, "null model desc");
  if (d->patch_size <= 0 || d->image_size % d->patch_size) return fail(DART_ERR_INVALID, "image_size % patch_size");
  const int g = d->image_size / d->patch_size;
  if (d->window_size <= 0 || g % d->window_size || g % 4) return fail(DART_ERR_INVALID, "grid/window");
  if (d->num_blocks < 0 || d->num_blocks > DART_MAX_BLOCKS) return fail(DART_ERR_INVALID, "num_blocks");
  if (d->num_heads <= 0 || d->embed_dim % d->num_heads) return fail(DART_ERR_INVALID, "embed_dim % heads");
  const int hd = d->embed_dim / d->num_heads, hde = d->text_dim / d->num_heads;
  auto hd_ok = [](int h) { return h == 16 || h == 32 || h == 64 || h == 80; };
  if (!hd_ok(hd) || !hd_ok(hde)) return fail(DART_ERR_INVALID, "unsupported head_dim (16/32/64/80)");
  if (d->embed_dim % 64 || d->text_dim % 64 || d->fpn_dims[0] % 64 || d->fpn_dims[1] % 64 || d->fpn_dims[2] % 64)
    return fail(DART_ERR_INVALID, "embed/text/fpn dims must be multiples of 64");
  if (d->num_queries < 1 || d->num_queries + 1 > 1024) return fail(DART_ERR_INVALID, "num_queries");
  if (d->text_tokens < 1 || d->num_encoder_layers < 1 || d->num_decoder_layers < 1)
    return fail(DART_ERR_INVALID, "text_tokens / layer counts");
  return DART_OK;
}

// ---------------------------------------------------------------- launch helpers
// Output tensor maps of a GEMM epilogue (see gemm_tc): fp32 box 32x32 SW128, fp16 box 32x32 SW64.
bool make_out_maps(int epi, const GemmEpi& e, int M, int N, CUtensorMap* tc, CUtensorMap* td) {
  if (epi == EPI_F32_RESID_LN)  // residual stream in/out + the fp16 LayerNorm rows
    return make_tmap_f32(tc, e.out, N, M, e.ldo) &&
           make_tmap_ex(td, e.out2, N, M, e.ldo2, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  if (epi == EPI_F32_RESID_X16)  // residual stream in/out + its fp16 copy
    return make_tmap_f32(tc, e.out, N, M, e.ldo) &&
           make_tmap_ex(td, e.out2, N, M, e.ldo2, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  if (epi == EPI_F32_RESID || (epi == EPI_F32 && !e.wm_scatter))
    return make_tmap_f32(tc, e.out, N, M, e.ldo);
  if (epi == EPI_F16 || epi == EPI_F16_RELU || epi == EPI_QKV_ROPE)
    return make_tmap_ex(td, e.out, N, M, e.ldo, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  return true;
}

int gemm(dart_model* m, const __half* A, int M, int lda, const GemmW& W, int epi, GemmEpi e, cudaStream_t s) {
  if (M <= 0) return 0;
  CUtensorMap ta;
  if (!make_tmap(&ta, A, W.K, M, lda, 128)) return fail(DART_ERR_CUDA, "cuTensorMapEncodeTiled failed (A)");
  if (e.bias == nullptr) e.bias = W.b;
  if (m->in_backbone && m->precision > 0) {
    e.round_f16 = 1;
    e.acc_f16 = m->precision == 2;
  }
  m->launches++;
  CUtensorMap tc, td;
  if (!make_out_maps(epi, e, M, W.N, &tc, &td)) return fail(DART_ERR_CUDA, "cuTensorMapEncodeTiled failed (out)");
  int bit = 0;
  if (m->in_backbone && m->precision == 0 && (W.K / 64) % 2 == 0 && epi != EPI_F32_RESID_LN) {
    if (W.N == 3 * m->E && W.K == m->E) bit = 1;    // attn.qkv
    else if (W.N == m->E && W.K == m->E) bit = 2;   // attn.out
    else if (W.N == m->E && W.K > m->E) bit = 4;    // mlp.fc2
  }
  const int splitk = (g_splitk_mask & bit) ? 2 : 1;
  const GemmPlan plan = gemm_plan(M, W.N, epi, m->num_sms, splitk);
  if (splitk == 2) {
    const long long tiles = (long long)((M + 128 * plan.cg - 1) / (128 * plan.cg)) * (W.N / plan.bn);
    const long long nflags = splitk_flag_count(tiles, plan.cg), nws = splitk_ws_floats(tiles, plan.bn, plan.cg);
    if (nflags > m->splitk_cap) {  // new flags start at zero; the combining warps reset them after use
      if (m->splitk_flags) cudaFree(m->splitk_flags);
      m->splitk_flags = nullptr;
      m->splitk_cap = 0;
      if (cudaMalloc(&m->splitk_flags, nflags * sizeof(int)) != cudaSuccess ||
          cudaMemsetAsync(m->splitk_flags, 0, nflags * sizeof(int), s) != cudaSuccess) {
        m->splitk_flags = nullptr;
        return fail(DART_ERR_CUDA, "split-K flag allocation failed");
      }
      m->splitk_cap = nflags;
    }
    if (nws > m->splitk_ws_cap) {
      if (m->splitk_ws) cudaFree(m->splitk_ws);
      m->splitk_ws = nullptr;
      m->splitk_ws_cap = 0;
      if (cudaMalloc(&m->splitk_ws, nws * sizeof(float)) != cudaSuccess) {
        m->splitk_ws = nullptr;
        return fail(DART_ERR_CUDA, "split-K workspace allocation failed");
      }
      m->splitk_ws_cap = nws;
    }
    e.splitk = 2;
    e.tile_flags = m->splitk_flags;
    e.ws = m->splitk_ws;
  }
  const int half_rows = plan.bn / 2 / plan.cg;  // tail-halves B box (tiles of the last wave split in two)
  const CUtensorMap* tb2 = (half_rows == 128 || half_rows == 64 || half_rows == 32) && W.N % half_rows == 0
                               ? &W.tmap[box_slot(half_rows)]
                               : nullptr;
  int rc = gemm_tc(ta, W.tmap[box_slot(plan.bn / plan.cg)], tb2, &tc, &td, M, W.N, W.K, plan, epi, e, m->num_sms, s);
  if (rc) return fail(DART_ERR_CUDA, std::string("gemm_tc: ") + cudaGetErrorString((cudaError_t)rc));
  return 0;
}

GemmEpi epi_out(void* out, int ldo) {
  GemmEpi e;
  e.out = out;
  e.ldo = ldo;
  return e;
}

AttnArgs attn_base(int heads, int hd) {
  AttnArgs a;
  memset(&a, 0, sizeof(a));
  a.heads = heads;
  a.head_stride_q = a.head_stride_k = a.head_stride_v = a.head_stride_o = hd;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
  return a;
}

int attn(dart_model* m, const AttnArgs& a, int hd, cudaStream_t s) {
  m->launches++;
  int rc = attention(a, hd, s);
  if (rc) return fail(DART_ERR_CUDA, std::string("attention: ") + cudaGetErrorString((cudaError_t)rc));
  return 0;
}

#define LAUNCH(expr)                                                                                      \
  do {                                                                                                    \
    m->launches++;                                                                                        \
    int _rc = (int)(expr);                                                                                \
    if (_rc) return fail(DART_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString((cudaError_t)_rc)); \
  } while (0)
#define RUN(expr)          \
  do {                     \
    int _rc = (expr);      \
    if (_rc) return _rc;   \
  } while (0)

int ensure_backbone_ws(dart_model* m, int B) {
  if (B <= m->bb_cap) return 0;
  m->bb_ws.release();
  const size_t rows = (size_t)B * m->T, E = m->E;
  auto& w = m->bb_ws;
  m->bb.patches = (__half*)w.get(rows * m->kpad * 2);
  m->bb.x = (float*)w.get(rows * E * 4);
  m->bb.h = (__half*)w.get(rows * E * 2);
  m->bb.qkv = (__half*)w.get(rows * 3 * E * 2);
  m->bb.ao = (__half*)w.get(rows * E * 2);
  m->bb.hid = (__half*)w.get(rows * 4 * E * 2);
  m->bb.pool1 = (__half*)w.get(rows / 4 * E * 2);
  m->bb.pool2 = (__half*)w.get(rows / 16 * E * 2);
  m->bb.l0h = (__half*)w.get(rows * m->F0 * 2);
  m->bb.lnst = (float2*)w.get(rows * (E / 32) * sizeof(float2));
  m->bb.lnfin = (float2*)w.get(rows * sizeof(float2));
  m->bb.lncnt = (int*)w.get((rows / 32 + 1) * sizeof(int));
  m->bb.chain = (int*)w.get(3 * (rows / 128 + 1) * sizeof(int));
  m->chain_rows = -1;  // counters zeroed below; the first chained call starts the epochs
  if (!m->bb.patches || !m->bb.x || !m->bb.h || !m->bb.qkv || !m->bb.ao || !m->bb.hid || !m->bb.pool1 ||
      !m->bb.pool2 || !m->bb.l0h || !m->bb.lnst || !m->bb.lnfin || !m->bb.lncnt || !m->bb.chain ||
      cudaMemset(m->bb.lncnt, 0, (rows / 32 + 1) * sizeof(int)) != cudaSuccess ||
      cudaMemset(m->bb.chain, 0, 3 * (rows / 128 + 1) * sizeof(int)) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {  // counters zero before any stream uses them
    m->bb_ws.release();
    m->bb_cap = 0;
    return fail(DART_ERR_CUDA, "backbone workspace allocation failed");
  }
  m->bb_cap = B;
  return 0;
}

int ensure_encdec_ws(dart_model* m, int B, int N) {
  if (B * N <= m->ed_cap_items && N <= m->ed_cap_n && B <= m->ed_cap_b) return 0;
  m->ed_ws.release();
  const int items = B * N;
  const size_t T = m->T, D = m->D, rows = (size_t)items * T, drows = (size_t)items * m->Q1;
  const int ne = m->d.num_encoder_layers, nd = m->d.num_decoder_layers;
  auto& w = m->ed_ws;
  auto& e = m->ed;
  e.e1 = (float*)w.get((size_t)B * T * D * 4);
  e.l0h = (__half*)w.get((size_t)B * T * m->F0 * 2);
  e.e = (float*)w.get(rows * D * 4);
  e.h = (__half*)w.get(rows * D * 2);
  e.q = (__half*)w.get(rows * D * 2);
  e.kv = (__half*)w.get(rows * 3 * D * 2);  // self-attention [q | k | v]
  e.o = (__half*)w.get(rows * D * 2);
  e.hid = (__half*)w.get(rows * 4 * D * 2);
  e.dkv = (__half*)w.get(rows * nd * 2 * D * 2);
  e.text = (__half*)w.get((size_t)N * m->Lt * D * 2);
  e.tkv = (__half*)w.get((size_t)N * m->Lt * ne * 2 * D * 2);
  e.qd0 = (float*)w.get((size_t)m->Q1 * D * 4);
  e.qd = (float*)w.get(drows * D * 4);
  e.qf = (float*)w.get(drows * D * 4);
  e.dh = (__half*)w.get(drows * D * 2);
  e.dq = (__half*)w.get(drows * D * 2);
  e.dkvs = (__half*)w.get(drows * 3 * D * 2);
  e.do_ = (__half*)w.get(drows * D * 2);
  e.dhid = (__half*)w.get(drows * 4 * D * 2);
  void* all[] = {e.e1, e.l0h, e.e, e.h, e.q, e.kv, e.o, e.hid, e.dkv, e.text, e.tkv, e.qd0, e.qd, e.qf,
                 e.dh, e.dq, e.dkvs, e.do_, e.dhid};
  for (void* p : all)
    if (!p) {
      m->ed_ws.release();
      m->ed_cap_items = m->ed_cap_n = m->ed_cap_b = 0;
      return fail(DART_ERR_CUDA, "enc-dec workspace allocation failed");
    }
  m->ed_cap_items = items;
  m->ed_cap_n = N;
  m->ed_cap_b = B;
  return 0;
}

// One pre-LN attention sub-block + residual over `rows` rows of the fp32 stream `x`:
// x += out_proj(MHA(LN(x), kv_source)).  Self-attention when kv16 == nullptr.
struct XAttnSpec {
  int items, Lq;                 // batch items and query rows per item
  const __half* kv16 = nullptr;  // external K/V (cross-attention): [.., tok_stride] fp16
  int kv_tok_stride = 0, Lk = 0, kv_mod = 0;
  long long kv_batch_stride = 0;
};

// The residual GEMM that closes an enc-dec sub-block: x += o W + b, and with `next` also
// h = LN_next(x) in the same epilogue (d = 256: whole rows per tile), so the next sub-block's
// LayerNorm pass disappears (reference model.py:516-527: every sub-block starts with an LN).
int resid_gemm(dart_model* m, const __half* A, int rows, int lda, const GemmW& W, float* x, const LNW* next, __half* h,
               cudaStream_t s) {
  GemmEpi e = epi_out(x, m->D);
  if (next && g_fused_ln && W.N == 256) {
    e.out2 = h;
    e.ldo2 = m->D;
    e.ln_g = next->g;
    e.ln_b = next->b;
    return gemm(m, A, rows, lda, W, EPI_F32_RESID_LN, e, s);
  }
  RUN(gemm(m, A, rows, lda, W, EPI_F32_RESID, e, s));
  if (next) LAUNCH(layernorm_f32_to_f16(x, next->g, next->b, h, rows, m->D, m->D, m->D, s));
  return 0;
}

// One pre-LN sub-block.  h_ready: h already holds LN(x) (fused into the previous sub-block's
// residual epilogue); next: also leave LN_next(x) in h for the following sub-block.
int xattn(dart_model* m, float* x, const LNW& ln, const AttnW& w, const XAttnSpec& sp, __half* h, __half* q,
          __half* kv, __half* o, cudaStream_t s, bool h_ready = false, const LNW* next = nullptr) {
  const int D = m->D, H = m->H, hd = D / H;
  const int rows = sp.items * sp.Lq;
  if (!h_ready) LAUNCH(layernorm_f32_to_f16(x, ln.g, ln.b, h, rows, D, D, D, s));
  const int Lk = sp.kv16 == nullptr ? sp.Lq : sp.Lk;
  if (sp.kv16 == nullptr && w.qkv.w) {  // self-attention: one [q | k | v] GEMM into kv (3D wide)
    RUN(gemm(m, h, rows, D, w.qkv, EPI_F16, epi_out(kv, 3 * D), s));
    if (tc_attention_enabled() && attention_tc_supported(hd, Lk)) {
      m->launches++;
      RUN(attn_tc(kv, 3 * D, 0, kv, 3 * D, D, 2 * D, o, D, sp.items, H, sp.Lq, Lk, hd, m->num_sms, s));
    } else {
      AttnArgs a = attn_base(H, hd);
      a.q = kv;
      a.k = kv + D;
      a.v = kv + 2 * D;
      a.q_tok_stride = a.k_tok_stride = a.v_tok_stride = 3 * D;
      a.q_batch_stride = a.k_batch_stride = a.v_batch_stride = (long long)sp.Lq * 3 * D;
      a.o = o;
      a.o_tok_stride = D;
      a.o_batch_stride = (long long)sp.Lq * D;
      a.Lq = a.Lk = sp.Lq;
      a.batch = sp.items;
      RUN(attn(m, a, hd, s));
    }
    return resid_gemm(m, o, rows, D, w.out, x, next, h, s);
  }
  RUN(gemm(m, h, rows, D, w.q, EPI_F16, epi_out(q, D), s));
  if (tc_attention_enabled() && attention_tc_supported(hd, Lk) &&
      (sp.kv16 == nullptr || sp.kv_batch_stride == (long long)Lk * sp.kv_tok_stride)) {
    // tcgen05 path: encoder self-attention (T x T), decoder cross-attention (201 x T) and the
    // encoder's text cross-attention (T x 32, K/V of class c shared by every image: kv_mod = N)
    if (sp.kv16 == nullptr) {
      RUN(gemm(m, h, rows, D, w.kv, EPI_F16, epi_out(kv, 2 * D), s));
      m->launches++;
      RUN(attn_tc(q, D, 0, kv, 2 * D, 0, D, o, D, sp.items, H, sp.Lq, Lk, hd, m->num_sms, s));
    } else {
      // split-KV for the decoder cross-attention (201 queries over T = 5184 keys; g_attn_split,
      // off by default): at small N its (q tile, head, class) items leave most CTA slots idle
      // (4 classes: 2 x 16 x 4 = 128 items for 296 slots, each over 54 key tiles); when enabled
      // every item's key range runs on g_attn_split CTAs and is merged.  The factor does not
      // depend on N, so a class's rows stay bitwise independent of the batch
      const int ks = (hd == 16 && Lk >= 1024 && g_attn_split > 1) ? g_attn_split : 1;
      if (ks > 1) {
        const size_t need = (size_t)sp.items * H * ks * sp.Lq * 20;
        if (need > m->attn_part_cap) {
          if (m->attn_part) cudaFree(m->attn_part);
          m->attn_part = nullptr;
          m->attn_part_cap = 0;
          if (cudaMalloc(&m->attn_part, need * sizeof(float)) != cudaSuccess)
            return fail(DART_ERR_CUDA, "split-KV workspace allocation failed");
          m->attn_part_cap = need;
        }
        m->launches++;  // the merge kernel
      }
      m->launches++;
      RUN(attn_tc(q, D, 0, sp.kv16, sp.kv_tok_stride, 0, D, o, D, sp.items, H, sp.Lq, Lk, hd, m->num_sms, s, nullptr,
                  sp.kv_mod, ks, m->attn_part));
    }
    return resid_gemm(m, o, rows, D, w.out, x, next, h, s);
  }
  AttnArgs a = attn_base(H, hd);
  a.q = q;
  a.q_tok_stride = D;
  a.q_batch_stride = (long long)sp.Lq * D;
  a.o = o;
  a.o_tok_stride = D;
  a.o_batch_stride = (long long)sp.Lq * D;
  a.Lq = sp.Lq;
  a.batch = sp.items;
  if (sp.kv16 == nullptr) {
    RUN(gemm(m, h, rows, D, w.kv, EPI_F16, epi_out(kv, 2 * D), s));
    a.k = kv;
    a.v = kv + D;
    a.k_tok_stride = a.v_tok_stride = 2 * D;
    a.k_batch_stride = a.v_batch_stride = (long long)sp.Lq * 2 * D;
    a.Lk = sp.Lq;
  } else {
    a.k = sp.kv16;
    a.v = sp.kv16 + D;
    a.k_tok_stride = a.v_tok_stride = sp.kv_tok_stride;
    a.k_batch_stride = a.v_batch_stride = sp.kv_batch_stride;
    a.Lk = sp.Lk;
    a.kv_batch_mod = sp.kv_mod;
  }
  RUN(attn(m, a, hd, s));
  return resid_gemm(m, o, rows, D, w.out, x, next, h, s);
}

// x += relu(h W1 + b1) W2 + b2 on the fused kernel (hidden activations stay in TMEM)
int mlp_fused_call(dart_model* m, const __half* h, const GemmW& fc1, const GemmW& fc2, float* x, int rows,
                   cudaStream_t s, const LNW* next = nullptr, __half* h_out = nullptr) {
  CUtensorMap th, tw1, tw2, tx, tln;
  if (!make_tmap(&th, h, 256, rows, 256, 128) || !make_tmap(&tw1, fc1.w, 256, 1024, 256, 64) ||
      !make_tmap(&tw2, fc2.w, 1024, 256, 1024, 128) || !make_tmap_f32(&tx, x, 256, rows, 256) ||
      !make_tmap_ex(&tln, next ? h_out : h, 256, rows, 256, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
    return fail(DART_ERR_CUDA, "cuTensorMapEncodeTiled failed (fused MLP)");
  m->launches++;
  const int rc = mlp_fused(th, tw1, tw2, tx, tln, rows, fc1.b, fc2.b, next ? next->g : nullptr,
                           next ? next->b : nullptr, m->num_sms, s);
  if (rc) return fail(DART_ERR_CUDA, std::string("mlp_fused: ") + cudaGetErrorString((cudaError_t)rc));
  return DART_OK;
}

int xmlp(dart_model* m, float* x, const LNW& ln, const GemmW& fc1, const GemmW& fc2, int rows, __half* h,
         __half* hid, cudaStream_t s, bool h_ready = false, const LNW* next = nullptr) {
  const int D = m->D;
  if (!h_ready) LAUNCH(layernorm_f32_to_f16(x, ln.g, ln.b, h, rows, D, D, D, s));
  // fused above ~2 waves of 256-row units (N=80: 423 vs 580 us per layer; N=4 equal); both forms
  // fuse the next sub-block's LN into their residual epilogue with identical arithmetic
  if (g_fused_mlp && D == 256 && fc1.N == 1024 && fc2.K == 1024 && fc2.N == 256 && rows >= 256 * m->num_sms) {
    if (next && g_fused_ln) return mlp_fused_call(m, h, fc1, fc2, x, rows, s, next, h);
    RUN(mlp_fused_call(m, h, fc1, fc2, x, rows, s));
    if (next) LAUNCH(layernorm_f32_to_f16(x, next->g, next->b, h, rows, D, D, D, s));
    return 0;
  }
  RUN(gemm(m, h, rows, D, fc1, EPI_F16_RELU, epi_out(hid, 4 * D), s));
  return resid_gemm(m, hid, rows, 4 * D, fc2, x, next, h, s);
}

}  // namespace

// ============================================================================ C ABI

extern "C" {

const char* dart_last_error(void) { return g_last_error.c_str(); }
const dart_model_desc* dart_model_get_desc(const dart_model* m) { return m ? &m->d : nullptr; }
const char* dart_version(void) { return "dart-b200 0.2 (sm_100a, tcgen05 GEMM + tcgen05 flash attention)"; }

int32_t dart_expected_weight_count(const dart_model_desc* d) {
  if (!d) return -1;
  return 4 + 12 * d->num_blocks + 6 + 3 + 22 * d->num_encoder_layers + 2 + 2 + 22 * d->num_decoder_layers + 2 + 6;
}

int dart_model_create(const dart_model_desc* desc, const float* const* weights, int32_t n_weights,
                      dart_model** out) {
  if (!out) return fail(DART_ERR_INVALID, "null out");
  *out = nullptr;
  RUN(check_desc(desc));
  if (n_weights != dart_expected_weight_count(desc))
    return fail(DART_ERR_INVALID, "weight count does not match the model description");
  if (!encode_fn()) return fail(DART_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable (no CUDA driver?)");
  dart_model* m = new dart_model();
  m->d = *desc;
  m->G = desc->image_size / desc->patch_size;
  m->T = m->G * m->G;
  m->E = desc->embed_dim;
  m->H = desc->num_heads;
  m->hd = m->E / m->H;
  m->kpatch = 3 * desc->patch_size * desc->patch_size;
  m->kpad = (m->kpatch + 63) / 64 * 64;
  m->D = desc->text_dim;
  m->Lt = desc->text_tokens;
  m->Q1 = desc->num_queries + 1;
  m->F0 = desc->fpn_dims[0];
  m->F1 = desc->fpn_dims[1];
  m->F2 = desc->fpn_dims[2];
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (m->F0 != m->D) {
    delete m;
    return fail(DART_ERR_INVALID, "fpn_dims[0] must equal text_dim (encdec.input is [F0, d])");
  }

  // scratch for fp32 uploads (largest weight matrix)
  const int E = m->E, D = m->D;
  size_t biggest = std::max<size_t>((size_t)E * 4 * E, (size_t)1024 * D);
  biggest = std::max<size_t>(biggest, (size_t)m->kpatch * E);
  float* scratch = nullptr;
  if (cudaMalloc(&scratch, biggest * sizeof(float)) != cudaSuccess) {
    delete m;
    return fail(DART_ERR_CUDA, "weight upload scratch allocation failed");
  }
  WeightCursor c{weights, n_weights};
  bool ok = make_gemm(m, c, m->kpatch, E, scratch, m->patch, m->kpad);
  const float* rc = c.next();
  const float* rs = c.next();
  ok = ok && rc && rs;
  if (ok) {
    m->rope_cos = upload_f32(m, rc, (size_t)m->T * (m->hd / 2));
    m->rope_sin = upload_f32(m, rs, (size_t)m->T * (m->hd / 2));
    ok = m->rope_cos && m->rope_sin;
  }
  m->blocks.resize(desc->num_blocks);
  for (int b = 0; ok && b < desc->num_blocks; ++b) {
    BlockW& B = m->blocks[b];
    const bool fold = g_ln_fold != 0;  // folded twins only when the fold is enabled at creation
    ok = make_ln(m, c, E, B.ln1) && make_gemm(m, c, E, 3 * E, scratch, B.qkv) &&
         (!fold || make_folded(m, B.qkv, B.ln1, scratch, B.qkv_f)) && make_gemm(m, c, E, E, scratch, B.out) &&
         make_ln(m, c, E, B.ln2) && make_gemm(m, c, E, 4 * E, scratch, B.fc1) &&
         (!fold || make_folded(m, B.fc1, B.ln2, scratch, B.fc1_f)) && make_gemm(m, c, 4 * E, E, scratch, B.fc2);
  }
  for (int l = 0; ok && l < 3; ++l) ok = make_gemm(m, c, E, desc->fpn_dims[l], scratch, m->fpn[l]);
  if (ok) {
    const float* tt = c.next();
    ok = tt && (m->text_table = upload_f32(m, tt, (size_t)1024 * D)) != nullptr;
  }
  ok = ok && make_gemm(m, c, m->F0, D, scratch, m->enc_in);
  const int ne = desc->num_encoder_layers, nd = desc->num_decoder_layers;
  auto init_fused = [&](GemmW& g, int layers) {
    g.N = layers * 2 * D;
    g.K = D;
    g.w = dev_alloc<__half>(m, (size_t)g.N * g.K);
    g.b = dev_alloc<float>(m, g.N);
    return g.w && g.b;
  };
  ok = ok && init_fused(m->enc_cross_kv_all, ne) && init_fused(m->dec_cross_kv_all, nd);
  m->enc.resize(ne);
  for (int l = 0; ok && l < ne; ++l) ok = make_xlayer(m, c, D, scratch, m->enc[l], &m->enc_cross_kv_all, l * 2 * D);
  ok = ok && make_ln(m, c, D, m->enc_final);
  if (ok) {
    const float* qw = c.next();
    const float* pw = c.next();
    ok = qw && pw && (m->queries = dev_alloc<float>(m, (size_t)m->Q1 * D)) != nullptr;
    ok = ok && cudaMemcpy(m->queries, qw, (size_t)desc->num_queries * D * 4, cudaMemcpyHostToDevice) == cudaSuccess;
    ok = ok && cudaMemcpy(m->queries + (size_t)desc->num_queries * D, pw, (size_t)D * 4, cudaMemcpyHostToDevice) ==
                   cudaSuccess;
  }
  m->dec.resize(nd);
  for (int l = 0; ok && l < nd; ++l) ok = make_xlayer(m, c, D, scratch, m->dec[l], &m->dec_cross_kv_all, l * 2 * D);
  ok = ok && make_ln(m, c, D, m->dec_final);
  ok = ok && finish_gemmw(m->enc_cross_kv_all) && finish_gemmw(m->dec_cross_kv_all);
  if (ok) {
    const float* h[6];
    for (int i = 0; i < 6; ++i) h[i] = c.next();
    ok = h[5] != nullptr;
    if (ok) {
      m->box_w = upload_f32(m, h[0], (size_t)D * 4);
      m->box_b = upload_f32(m, h[1], 4);
      m->score_w = upload_f32(m, h[2], D);
      m->score_b = upload_f32(m, h[3], 1);
      m->pres_w = upload_f32(m, h[4], D);
      m->pres_b = upload_f32(m, h[5], 1);
      ok = m->box_w && m->box_b && m->score_w && m->score_b && m->pres_w && m->pres_b;
    }
  }
  cudaError_t se = cudaDeviceSynchronize();
  cudaFree(scratch);
  if (!ok || se != cudaSuccess || c.i != n_weights) {
    delete m;
    return fail(DART_ERR_CUDA, std::string("weight upload failed: ") + cudaGetErrorString(cudaGetLastError()));
  }
  *out = m;
  return DART_OK;
}

void dart_model_destroy(dart_model* m) { delete m; }

int dart_model_fork(const dart_model* parent, dart_model** out) {
  if (!parent || !out) return fail(DART_ERR_INVALID, "dart_model_fork: bad args");
  dart_model* f = new dart_model(*parent);  // shares the weights (shared_ptr), copies dims and maps
  f->bb_ws = Workspace();                   // own, initially empty activation workspaces
  f->ed_ws = Workspace();
  f->mask_ws = Workspace();
  f->mask_cap_rows = f->mask_cap_tok = 0;
  f->mk_qf = f->mk_l0 = f->mk_mq = f->mk_mf = nullptr;
  f->bb_cap = f->ed_cap_items = f->ed_cap_n = f->ed_cap_b = 0;
  f->last_backbone_B = 0;
  f->bb = {};
  f->ed = {};
  f->launches = 0;
  f->splitk_flags = nullptr;
  f->splitk_cap = 0;
  f->splitk_ws = nullptr;
  f->splitk_ws_cap = 0;
  f->attn_part = nullptr;
  f->attn_part_cap = 0;
  *out = f;
  return DART_OK;
}

int dart_model_set_precision(dart_model* m, int32_t precision) {
  if (!m || precision < 0 || precision > 2) return fail(DART_ERR_INVALID, "dart_model_set_precision: precision must be 0, 1 or 2");
  m->precision = precision;
  return DART_OK;
}

int32_t dart_model_get_precision(const dart_model* m) { return m ? m->precision : -1; }

int64_t dart_launch_count(const dart_model* m) { return m ? m->launches : 0; }
void dart_reset_launch_count(dart_model* m) {
  if (m) m->launches = 0;
}

}  // extern "C"

namespace {

// Marks the GEMMs a backbone stage issues (they follow the handle's precision discipline).
struct BackboneScope {
  dart_model* m;
  explicit BackboneScope(dart_model* mm) : m(mm) { m->in_backbone = true; }
  ~BackboneScope() { m->in_backbone = false; }
};

// Backbone stages on a caller-chosen residual stream x [B*T, E] fp32 in window-major row order
// (each 24x24 window a contiguous block; global attention, LN and the MLP are order-invariant,
// the patchify / RoPE / FPN kernels map rows to tokens).
// Backbone LayerNorms folded into the GEMMs that consume them (GemmEpi::ln_stats; LN1 -> QKV,
// LN2 -> fc1): the producers of the residual stream x (patch embed, attn.out, mlp.fc2) also write
// fp16(x) and per-row chunk statistics, so no LayerNorm pass runs.  Only the whole-backbone entry
// point (dart_backbone) in the detection discipline folds (g_ln_fold); the staged entry points
// (pruning) and the precision-study disciplines always run the LayerNorm kernels.
int ln_fold_on(const dart_model* m) {
  const bool ok = m->precision == 0 && m->E % 32 == 0 && !m->blocks.empty() && m->blocks[0].qkv_f.w != nullptr;
  return ok ? g_ln_fold & 3 : 0;
}

int bb_embed(dart_model* m, const float* images, int B, float* x, int32_t* flags, cudaStream_t s, int fold = 0) {
  BackboneScope scope(m);
  auto& w = m->bb;
  const int rows = B * m->T, win = m->d.window_size;
  if (cudaMemsetAsync(flags, 0, sizeof(int32_t), s) != cudaSuccess) return fail(DART_ERR_CUDA, "flags memset");
  LAUNCH(patchify(images, w.patches, B, m->d.image_size, m->d.patch_size, m->kpad, win, flags, s));
  m->x16_valid = (fold & 1) != 0;
  if (fold & 1) {  // x, fp16(x) and its LN chunk statistics (block 0's LN1 is folded)
    GemmEpi e = epi_out(x, m->E);
    e.out2 = w.h;
    e.ldo2 = m->E;
    e.ln_stats_out = w.lnst;
    e.ln_cnt = w.lncnt;
    e.ln_final = w.lnfin;
    e.ln_parts = m->E / 32;
    return gemm(m, w.patches, rows, m->kpad, m->patch, EPI_F32_F16, e, s);
  }
  return gemm(m, w.patches, rows, m->kpad, m->patch, EPI_F32, epi_out(x, m->E), s);
}

// fold (mask, see g_ln_fold): with bit 0, fp16(x) in w.h and its statistics are current on entry
// (bb_embed with the same mask)
int bb_blocks(dart_model* m, float* x, int B, int b0, int b1, const int32_t* attn_on, const int32_t* mlp_on,
              cudaStream_t s, int fold = 0) {
  BackboneScope scope(m);
  const int T = m->T, E = m->E, H = m->H, hd = m->hd, G = m->G;
  const int rows = B * T;
  auto& w = m->bb;
  const int win = m->d.window_size, nwin = (G / win) * (G / win);
  // the producer epilogue of x (fold: + fp16(x) into w.h and the LN statistics)
  // the next LN's fold bit decides what the producer writes: attn.out feeds LN2 (bit 1), fc2 LN1
  auto resid = [&](const __half* A, int K, const GemmW& W, int next_bit) {
    GemmEpi e = epi_out(x, E);
    m->x16_valid = (fold & next_bit) != 0;
    if (!(fold & next_bit)) return gemm(m, A, rows, K, W, EPI_F32_RESID, e, s);
    e.out2 = w.h;
    e.ldo2 = E;
    e.ln_stats_out = w.lnst;
    e.ln_cnt = w.lncnt;
    e.ln_final = w.lnfin;
    e.ln_parts = E / 32;
    return gemm(m, A, rows, K, W, EPI_F32_RESID_X16, e, s);
  };
  auto folded_in = [&](GemmEpi& e, const GemmW& Wf) {  // consumer of LN(x): (mean, rstd) + column sums
    e.ln_stats = w.lnfin;
    e.ln_colsum = Wf.colsum;
  };
  // row-block dependency chain (g_chain): fc1 -> fc2 -> LN1 of the next block -> its QKV, for blocks
  // that run both sub-blocks on the model's own enable flags in the detection discipline
  const bool chain = g_chain && !fold && m->precision == 0 && E == 1280 && !attn_on && !mlp_on && x == w.x;
  const int nblk = rows / 128 + 1;
  int* const c_fc1 = w.chain;
  int* const c_fc2 = w.chain + nblk;
  int* const c_ln = w.chain + 2 * nblk;
  int* const ep = m->chain_epoch;
  if (chain && m->chain_rows != rows) {  // counters are cumulative per row-block layout
    if (cudaMemsetAsync(w.chain, 0, 3 * nblk * sizeof(int), s) != cudaSuccess) return fail(DART_ERR_CUDA, "chain reset");
    m->chain_rows = rows;
    ep[0] = ep[1] = ep[2] = 0;
  }
  auto chained = [&](int blk) { return chain && m->d.attn_enabled[blk] && m->d.mlp_enabled[blk]; };
  bool fc2_signalled = false;  // the previous block's fc2 counts its row blocks into c_fc2
  for (int b = b0; b < b1; ++b) {
    const BlockW& bw = m->blocks[b];
    if (attn_on ? attn_on[b] : m->d.attn_enabled[b]) {
      GemmEpi e = epi_out(w.qkv, 3 * E);
      if (chained(b)) {  // LN1 row by row as fc2 finishes its rows; QKV block by block as LN1 does
        LAUNCH(layernorm_f32_to_f16_chain(x, bw.ln1.g, bw.ln1.b, w.h, rows, E, fc2_signalled ? c_fc2 : nullptr,
                                          ep[1] * (E / 8), c_ln, s));
        ++ep[2];
        e.dep_wait = c_ln;
        e.dep_mult = ep[2];
        e.dep_per_row = 1;
        e.skip_pdl_wait = 1;
        e.force_pdl = 1;
      } else if (!(fold & 1)) {
        LAUNCH(layernorm_f32_to_f16(x, bw.ln1.g, bw.ln1.b, w.h, rows, E, E, E, s));
      }
      fc2_signalled = false;
      if (fold & 1) folded_in(e, bw.qkv_f);
      e.rope_cos = m->rope_cos;
      e.rope_sin = m->rope_sin;
      e.rope_T = T;
      e.rope_grid = G;
      e.rope_hd = hd;
      e.rope_cols = 2 * E;  // q and k
      e.wm_grid = G;
      e.wm_win = win;
      RUN(gemm(m, w.h, rows, E, (fold & 1) ? bw.qkv_f : bw.qkv, EPI_QKV_ROPE, e, s));
      AttnArgs a = attn_base(H, hd);
      a.q = w.qkv;
      a.k = w.qkv + E;
      a.v = w.qkv + 2 * E;
      a.o = w.ao;
      a.q_tok_stride = a.k_tok_stride = a.v_tok_stride = 3 * E;
      a.o_tok_stride = E;
      if (m->d.block_global[b]) {
        a.q_batch_stride = a.k_batch_stride = a.v_batch_stride = (long long)T * 3 * E;
        a.o_batch_stride = (long long)T * E;
        a.Lq = a.Lk = T;
        a.batch = B;
      } else {  // windows are contiguous blocks of win*win rows
        a.q_batch_stride = a.k_batch_stride = a.v_batch_stride = (long long)win * win * 3 * E;
        a.o_batch_stride = (long long)win * win * E;
        a.Lq = a.Lk = win * win;
        a.batch = B * nwin;
      }
      if (tc_attention_enabled() && attention_tc_supported(hd, a.Lq)) {
        m->launches++;
        RUN(attn_tc_packed(w.qkv, w.ao, a.batch, H, a.Lq, hd, E, m->num_sms, s));
      } else {
        RUN(attn(m, a, hd, s));
      }
      RUN(resid(w.ao, E, bw.out, 2));
    }
    if (mlp_on ? mlp_on[b] : m->d.mlp_enabled[b]) {
      GemmEpi e = epi_out(w.hid, 4 * E);
      if (fold & 2)
        folded_in(e, bw.fc1_f);
      else
        LAUNCH(layernorm_f32_to_f16(x, bw.ln2.g, bw.ln2.b, w.h, rows, E, E, E, s));
      fc2_signalled = false;
      if (chained(b)) {  // fc1 counts its finished row blocks; fc2 starts on them in fc1's last wave
        e.dep_signal = c_fc1;
        e.early_trigger = 1;
        RUN(gemm(m, w.h, rows, E, bw.fc1, EPI_F16_RELU, e, s));
        ++ep[0];
        GemmEpi e2 = epi_out(x, E);
        e2.dep_wait = c_fc1;
        e2.dep_mult = ep[0] * (4 * E / 8);
        e2.skip_pdl_wait = 1;
        e2.force_pdl = 1;
        if (b + 1 < b1 && chained(b + 1)) {  // the next block's LN1 starts on fc2's finished rows
          e2.dep_signal = c_fc2;
          e2.early_trigger = 1;
        }
        RUN(gemm(m, w.hid, rows, 4 * E, bw.fc2, EPI_F32_RESID, e2, s));
        if (e2.dep_signal) {
          ++ep[1];
          fc2_signalled = true;
        }
      } else {
        RUN(gemm(m, w.h, rows, E, (fold & 2) ? bw.fc1_f : bw.fc1, EPI_F16_RELU, e, s));
        RUN(resid(w.hid, 4 * E, bw.fc2, 1));
      }
    }
  }
  return DART_OK;
}

// FPN (model.py:446-451): L0 from tokens, L1 / L2 from 2x2 / 4x4 mean-pooled tokens
// fold: w.h already holds fp16(x) (the last producer's copy), so the cast is skipped
int bb_fpn(dart_model* m, const float* x, int B, float* l0, float* l1, float* l2, int32_t* flags, cudaStream_t s,
           int fold = 0) {
  BackboneScope scope(m);
  auto& w = m->bb;
  const int rows = B * m->T, E = m->E, G = m->G, win = m->d.window_size;
  if (!fold) LAUNCH(cast_f32_to_f16(x, w.h, (long long)rows * E, s));
  GemmEpi e0 = epi_out(l0, m->F0);  // rows scattered back to token-major order
  e0.out2 = w.l0h;
  e0.ldo2 = m->F0;
  e0.wm_grid = G;
  e0.wm_win = win;
  e0.wm_scatter = 1;
  RUN(gemm(m, w.h, rows, E, m->fpn[0], EPI_F32_F16, e0, s));
  LAUNCH(pool_tokens(x, w.pool1, B, G, E, 2, win, s));
  RUN(gemm(m, w.pool1, rows / 4, E, m->fpn[1], EPI_F32, epi_out(l1, m->F1), s));
  LAUNCH(pool_tokens(x, w.pool2, B, G, E, 4, win, s));
  RUN(gemm(m, w.pool2, rows / 16, E, m->fpn[2], EPI_F32, epi_out(l2, m->F2), s));
  LAUNCH(finite_check(l0, (long long)rows * m->F0, flags, DART_FLAG_NONFINITE, s));
  LAUNCH(finite_check(l1, (long long)rows / 4 * m->F1, flags, DART_FLAG_NONFINITE, s));
  LAUNCH(finite_check(l2, (long long)rows / 16 * m->F2, flags, DART_FLAG_NONFINITE, s));
  m->last_backbone_B = B;
  return DART_OK;
}

}  // namespace

extern "C" {

int dart_backbone(dart_model* m, const float* images, int32_t B, float* l0, float* l1, float* l2, int32_t* flags,
                  void* stream) {
  if (!m || !images || B <= 0 || !l0 || !l1 || !l2 || !flags) return fail(DART_ERR_INVALID, "dart_backbone: bad args");
  cudaStream_t s = (cudaStream_t)stream;
  RUN(ensure_backbone_ws(m, B));
  const int fold = ln_fold_on(m);
  RUN(bb_embed(m, images, B, m->bb.x, flags, s, fold));
  RUN(bb_blocks(m, m->bb.x, B, 0, m->d.num_blocks, nullptr, nullptr, s, fold));
  return bb_fpn(m, m->bb.x, B, l0, l1, l2, flags, s, m->x16_valid);  // last producer left fp16(x) in bb.h
}

int dart_backbone_embed(dart_model* m, const float* images, int32_t B, float* x, int32_t* flags, void* stream) {
  if (!m || !images || B <= 0 || !x || !flags) return fail(DART_ERR_INVALID, "dart_backbone_embed: bad args");
  RUN(ensure_backbone_ws(m, B));
  return bb_embed(m, images, B, x, flags, (cudaStream_t)stream);
}

int dart_backbone_blocks(dart_model* m, float* x, int32_t B, int32_t b0, int32_t b1, const int32_t* attn_on,
                         const int32_t* mlp_on, void* stream) {
  if (!m || !x || B <= 0 || b0 < 0 || b1 > m->d.num_blocks || b0 > b1)
    return fail(DART_ERR_INVALID, "dart_backbone_blocks: bad args");
  RUN(ensure_backbone_ws(m, B));
  return bb_blocks(m, x, B, b0, b1, attn_on, mlp_on, (cudaStream_t)stream);
}

int dart_backbone_fpn(dart_model* m, const float* x, int32_t B, float* l0, float* l1, float* l2, int32_t* flags,
                      void* stream) {
  if (!m || !x || B <= 0 || !l0 || !l1 || !l2 || !flags) return fail(DART_ERR_INVALID, "dart_backbone_fpn: bad args");
  RUN(ensure_backbone_ws(m, B));
  return bb_fpn(m, x, B, l0, l1, l2, flags, (cudaStream_t)stream);
}

}  // extern "C"

namespace {

// Class-independent enc-dec prefix, once per image: input projection + encoder layer-0
// self-attention sub-block (model.py:513-517; text first enters at :518) -> e1 [B, T, d] fp32.
// The enc-dec workspace must hold B images (ensure_encdec_ws).
int ed_prefix(dart_model* m, const float* l0, int B, float* e1, cudaStream_t s) {
  const int T = m->T, D = m->D;
  auto& w = m->ed;
  const __half* l0h = m->bb.l0h;
  if (l0) {
    LAUNCH(cast_f32_to_f16(l0, w.l0h, (long long)B * T * m->F0, s));
    l0h = w.l0h;
  }
  RUN(gemm(m, l0h, B * T, m->F0, m->enc_in, EPI_F32, epi_out(e1, D), s));
  XAttnSpec sp;
  sp.items = B;
  sp.Lq = T;
  return xattn(m, e1, m->enc[0].ln1, m->enc[0].self, sp, w.h, w.q, w.kv, w.o, s);
}

// The class-batched rest of the enc-dec for B images x N classes, from the prefix output e1.
int ed_body(dart_model* m, const float* e1, int B, const float* text, int N, double* boxes, double* score_logits,
            double* presence_logits, float* query_features, cudaStream_t s) {
  const int T = m->T, D = m->D, Q1 = m->Q1, Q = m->d.num_queries, Lt = m->Lt;
  const int ne = m->d.num_encoder_layers, nd = m->d.num_decoder_layers;
  const int items = B * N;
  auto& w = m->ed;
  for (int b = 0; b < B; ++b)
    LAUNCH(broadcast_rows(e1 + (size_t)b * T * D, w.e + (size_t)b * N * T * D, (long long)T * D, N, s));
  // ---- text K/V for all 6 encoder cross-attentions in one GEMM
  LAUNCH(cast_f32_to_f16(text, w.text, (long long)N * Lt * D, s));
  RUN(gemm(m, w.text, N * Lt, D, m->enc_cross_kv_all, EPI_F16, epi_out(w.tkv, ne * 2 * D), s));
  const int rows = items * T;
  // every LayerNorm after the first is fused into the residual epilogue of the sub-block before it
  // (h then already holds it: `ready`), except after the fused MLP kernel (xmlp)
  for (int l = 0; l < ne; ++l) {
    const XLayerW& L = m->enc[l];
    if (l > 0) {
      XAttnSpec sp;
      sp.items = items;
      sp.Lq = T;
      RUN(xattn(m, w.e, L.ln1, L.self, sp, w.h, w.q, w.kv, w.o, s, true, &L.ln2));
    }
    XAttnSpec cx;
    cx.items = items;
    cx.Lq = T;
    cx.kv16 = w.tkv + (size_t)l * 2 * D;
    cx.kv_tok_stride = ne * 2 * D;
    cx.kv_batch_stride = (long long)Lt * ne * 2 * D;
    cx.Lk = Lt;
    cx.kv_mod = N;
    RUN(xattn(m, w.e, L.ln2, L.cross, cx, w.h, w.q, w.kv, w.o, s, l > 0, &L.ln3));
    RUN(xmlp(m, w.e, L.ln3, L.fc1, L.fc2, rows, w.h, w.hid, s, true, l + 1 < ne ? &m->enc[l + 1].ln1 : &m->enc_final));
  }
  // ---- encoder memory: final LN (h, from the last MLP's epilogue), then K/V of all 6 decoder
  //      cross-attentions in one GEMM
  RUN(gemm(m, w.h, rows, D, m->dec_cross_kv_all, EPI_F16, epi_out(w.dkv, nd * 2 * D), s));
  // ---- decoder: layer-0 self-attention over the learned queries is class-independent
  CK(cudaMemcpyAsync(w.qd0, m->queries, (size_t)Q1 * D * 4, cudaMemcpyDeviceToDevice, s));
  {
    XAttnSpec sp;
    sp.items = 1;
    sp.Lq = Q1;
    RUN(xattn(m, w.qd0, m->dec[0].ln1, m->dec[0].self, sp, w.dh, w.dq, w.dkvs, w.do_, s));
  }
  LAUNCH(broadcast_rows(w.qd0, w.qd, (long long)Q1 * D, items, s));
  const int drows = items * Q1;
  for (int l = 0; l < nd; ++l) {
    const XLayerW& L = m->dec[l];
    if (l > 0) {
      XAttnSpec sp;
      sp.items = items;
      sp.Lq = Q1;
      RUN(xattn(m, w.qd, L.ln1, L.self, sp, w.dh, w.dq, w.dkvs, w.do_, s, true, &L.ln2));
    }
    XAttnSpec cx;
    cx.items = items;
    cx.Lq = Q1;
    cx.kv16 = w.dkv + (size_t)l * 2 * D;
    cx.kv_tok_stride = nd * 2 * D;
    cx.kv_batch_stride = (long long)T * nd * 2 * D;
    cx.Lk = T;
    RUN(xattn(m, w.qd, L.ln2, L.cross, cx, w.dh, w.dq, w.dkvs, w.do_, s, l > 0, &L.ln3));
    RUN(xmlp(m, w.qd, L.ln3, L.fc1, L.fc2, drows, w.dh, w.dhid, s, true, l + 1 < nd ? &m->dec[l + 1].ln1 : nullptr));
  }
  LAUNCH(layernorm_f32_to_f32(w.qd, m->dec_final.g, m->dec_final.b, w.qf, drows, D, s));
  LAUNCH(heads_forward(w.qf, Q1, Q, items, D, m->box_w, m->box_b, m->score_w, m->score_b, m->pres_w, m->pres_b, boxes,
                       score_logits, presence_logits, query_features, s));
  return DART_OK;
}

}  // namespace

extern "C" {

int dart_encdec(dart_model* m, const float* l0, int32_t B, const float* text, int32_t N, double* boxes,
                double* score_logits, double* presence_logits, float* query_features, void* stream) {
  if (!m || B <= 0 || N <= 0 || !text || !boxes || !score_logits || !presence_logits)
    return fail(DART_ERR_INVALID, "dart_encdec: bad args");
  if (!l0 && (m->bb_cap == 0 || m->last_backbone_B != B))
    return fail(DART_ERR_INVALID, "dart_encdec: l0 == NULL but no matching dart_backbone output");
  cudaStream_t s = (cudaStream_t)stream;
  RUN(ensure_encdec_ws(m, B, N));
  RUN(ed_prefix(m, l0, B, m->ed.e1, s));
  return ed_body(m, m->ed.e1, B, text, N, boxes, score_logits, presence_logits, query_features, s);
}

int dart_encdec_prefix(dart_model* m, const float* l0, int32_t B, float* e1, void* stream) {
  if (!m || B <= 0 || !e1) return fail(DART_ERR_INVALID, "dart_encdec_prefix: bad args");
  if (!l0 && (m->bb_cap == 0 || m->last_backbone_B != B))
    return fail(DART_ERR_INVALID, "dart_encdec_prefix: l0 == NULL but no matching dart_backbone output");
  RUN(ensure_encdec_ws(m, B, 1));  // e1 is caller-owned: a later (B, N) workspace growth keeps it
  return ed_prefix(m, l0, B, e1, (cudaStream_t)stream);
}

int dart_encdec_from_prefix(dart_model* m, const float* e1, int32_t B, const float* text, int32_t N, double* boxes,
                            double* score_logits, double* presence_logits, float* query_features, void* stream) {
  if (!m || !e1 || B <= 0 || N <= 0 || !text || !boxes || !score_logits || !presence_logits)
    return fail(DART_ERR_INVALID, "dart_encdec_from_prefix: bad args");
  RUN(ensure_encdec_ws(m, B, N));
  return ed_body(m, e1, B, text, N, boxes, score_logits, presence_logits, query_features, (cudaStream_t)stream);
}

int dart_postprocess(dart_model* m, const double* boxes, const double* score_logits, const double* presence_logits,
                     int32_t N, int32_t Q, double presence_threshold, double score_threshold,
                     double nms_iou_threshold, int32_t cross_class, int32_t* kept_count, int32_t* kept_query,
                     double* kept_score, double* presence_prob, int32_t* keep_flag, int32_t* scratch,
                     void* stream) {
  if (!boxes || !score_logits || !presence_logits || N <= 0 || Q <= 0 || !kept_count || !kept_query ||
      !kept_score || !presence_prob)
    return fail(DART_ERR_INVALID, "dart_postprocess: bad args");
  if (cross_class && (!keep_flag || !scratch)) return fail(DART_ERR_INVALID, "cross-class NMS needs keep_flag/scratch");
  cudaStream_t s = (cudaStream_t)stream;
  if (m) m->launches++;
  int rc = postprocess_classes(boxes, score_logits, presence_logits, N, Q, presence_threshold, score_threshold,
                               nms_iou_threshold, kept_count, kept_query, kept_score, presence_prob, s);
  if (rc) return fail(DART_ERR_CUDA, std::string("postprocess: ") + cudaGetErrorString((cudaError_t)rc));
  if (cross_class) {
    if (m) m->launches++;
    rc = postprocess_cross_class(boxes, kept_count, kept_query, kept_score, N, Q, nms_iou_threshold, keep_flag,
                                 scratch, s);
    if (rc) return fail(DART_ERR_CUDA, std::string("cross-class NMS: ") + cudaGetErrorString((cudaError_t)rc));
  }
  return DART_OK;
}

int dart_gemm_resid_ln(const void* A, const void* W, const float* bias, float* x, void* h, const float* ln_g,
                       const float* ln_b, int32_t M, int32_t K, void* stream) {
  if (!A || !W || !x || !h || !ln_g || !ln_b || M <= 0 || K % 64) return fail(DART_ERR_INVALID, "dart_gemm_resid_ln: bad args");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int N = 256;
  const GemmPlan plan = gemm_plan(M, N, EPI_F32_RESID_LN, sms);
  GemmEpi e;
  e.bias = bias;
  e.out = x;
  e.ldo = N;
  e.out2 = h;
  e.ldo2 = N;
  e.ln_g = ln_g;
  e.ln_b = ln_b;
  CUtensorMap ta, tb, tc, td;
  if (!make_tmap(&ta, A, K, M, K, 128) || !make_tmap(&tb, W, K, N, K, plan.bn / plan.cg) ||
      !make_out_maps(EPI_F32_RESID_LN, e, M, N, &tc, &td))
    return fail(DART_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  const int rc = gemm_tc(ta, tb, nullptr, &tc, &td, M, N, K, plan, EPI_F32_RESID_LN, e, sms, (cudaStream_t)stream);
  if (rc) return fail(DART_ERR_CUDA, std::string("gemm_tc: ") + cudaGetErrorString((cudaError_t)rc));
  return DART_OK;
}

int dart_gemm(const void* A, const void* W, const float* bias, void* out, void* out2, int32_t M, int32_t N,
              int32_t K, int32_t epi, const float* rope_cos, const float* rope_sin, int32_t rope_T, int32_t rope_hd,
              int32_t rope_cols, void* stream) {
  if (!A || !W || !out || M <= 0 || K % 64 || gemm_bn_for(N) == 0 || epi < 0 || epi > 5)
    return fail(DART_ERR_INVALID, "dart_gemm: bad args");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const GemmPlan plan = gemm_plan(M, N, epi, sms, g_gemm_splitk == 2 && epi != EPI_F32_RESID_LN ? 2 : 1);
  CUtensorMap ta, tb, tc;
  if (!make_tmap(&ta, A, K, M, K, 128) || !make_tmap(&tb, W, K, N, K, plan.bn / plan.cg))
    return fail(DART_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  GemmEpi e;
  e.bias = bias;
  e.out = out;
  e.ldo = N;
  e.out2 = out2;
  e.ldo2 = N;
  e.rope_cos = rope_cos;
  e.rope_sin = rope_sin;
  e.rope_T = rope_T > 0 ? rope_T : 1;
  e.rope_grid = (int)lround(sqrt((double)e.rope_T));
  e.rope_hd = rope_hd > 0 ? rope_hd : 2;
  e.rope_cols = rope_cols;
  e.dbg_noload = getenv("DART_GEMM_NOLOAD") != nullptr;
  e.round_f16 = g_gemm_precision > 0;
  e.acc_f16 = g_gemm_precision == 2;
  CUtensorMap td;
  if (!make_out_maps(epi, e, M, N, &tc, &td)) return fail(DART_ERR_CUDA, "cuTensorMapEncodeTiled failed (out)");
  if (g_gemm_splitk == 2) {  // tests: the split-K path (flags and workspace per device, tests only)
    static int* flags_of[64] = {};
    static float* ws_of[64] = {};
    static long long ws_cap_of[64] = {};
    int dev_id = 0;
    cudaGetDevice(&dev_id);
    int*& flags = flags_of[dev_id & 63];
    float*& ws = ws_of[dev_id & 63];
    constexpr long long kFlags = 1 << 20;
    const long long tiles = (long long)((M + 128 * plan.cg - 1) / (128 * plan.cg)) * (N / plan.bn);
    if (splitk_flag_count(tiles, plan.cg) > kFlags) return fail(DART_ERR_INVALID, "dart_gemm: too many split-K tiles");
    if (!flags && (cudaMalloc(&flags, kFlags * sizeof(int)) != cudaSuccess ||
                   cudaMemset(flags, 0, kFlags * sizeof(int)) != cudaSuccess))
      return fail(DART_ERR_CUDA, "flags");
    const long long nws = splitk_ws_floats(tiles, plan.bn, plan.cg);
    if (nws > ws_cap_of[dev_id & 63]) {
      if (ws) cudaFree(ws);
      if (cudaMalloc(&ws, nws * sizeof(float)) != cudaSuccess) return fail(DART_ERR_CUDA, "split-K workspace");
      ws_cap_of[dev_id & 63] = nws;
    }
    e.splitk = 2;
    e.tile_flags = flags;
    e.ws = ws;
  }
  CUtensorMap tb2;
  const int half_rows = plan.bn / 2 / plan.cg;
  const bool has_b2 = half_rows >= 32 && make_tmap(&tb2, W, K, N, K, half_rows);
  int rc = gemm_tc(ta, tb, has_b2 ? &tb2 : nullptr, &tc, &td, M, N, K, plan, epi, e, sms, (cudaStream_t)stream);
  if (rc) return fail(DART_ERR_CUDA, std::string("gemm_tc: ") + cudaGetErrorString((cudaError_t)rc));
  return DART_OK;
}

void dart_gemm_plan(int32_t M, int32_t N, int32_t epi, int32_t* bn, int32_t* cg) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const GemmPlan p = gemm_plan(M, N, epi, sms);
  if (bn) *bn = p.bn;
  if (cg) *cg = p.cg;
}

void dart_gemm_force_plan(int32_t bn, int32_t cg) { gemm_force_plan(bn, cg); }
int dart_gemm_trace(int64_t* device_buf) { return gemm_set_trace((long long*)device_buf); }

int dart_layernorm(const float* x, const float* gamma, const float* beta, void* y, int32_t rows, int32_t dim,
                   int32_t out_f16, void* stream) {
  if (!x || !gamma || !beta || !y || rows <= 0) return fail(DART_ERR_INVALID, "dart_layernorm: bad args");
  const int rc = out_f16 ? layernorm_f32_to_f16(x, gamma, beta, (__half*)y, rows, dim, dim, dim, (cudaStream_t)stream)
                         : layernorm_f32_to_f32(x, gamma, beta, (float*)y, rows, dim, (cudaStream_t)stream);
  if (rc) return fail(DART_ERR_CUDA, std::string("layernorm: ") + cudaGetErrorString((cudaError_t)rc));
  return DART_OK;
}
void dart_gemm_force_splitk(int32_t s) { g_gemm_splitk = s == 2 ? 2 : 1; }
void dart_set_pdl(int32_t mode) { pdl_set_thread(mode); }
void dart_set_ln_fold(int32_t on) { g_ln_fold = on & 3; }
void dart_attention_kv_split(int32_t k) { g_attn_split = k < 1 ? 1 : k > 8 ? 8 : k; }
void dart_set_chain(int32_t on) { g_chain = on != 0; }
void dart_gemm_force_precision(int32_t p) { g_gemm_precision = p >= 0 && p <= 2 ? p : 0; }

int dart_mlp_fused_ln(const void* h, const void* w1, const float* b1, const void* w2, const float* b2, float* x,
                      void* h_out, const float* ln_g, const float* ln_b, int32_t M, void* stream) {
  if (!h || !w1 || !b1 || !w2 || !b2 || !x || M <= 0 || (ln_g && (!ln_b || !h_out)))
    return fail(DART_ERR_INVALID, "dart_mlp_fused: bad args");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  CUtensorMap th, tw1, tw2, tx, tln;
  if (!make_tmap(&th, h, 256, M, 256, 128) || !make_tmap(&tw1, w1, 256, 1024, 256, 64) ||
      !make_tmap(&tw2, w2, 1024, 256, 1024, 128) || !make_tmap_f32(&tx, x, 256, M, 256) ||
      !make_tmap_ex(&tln, ln_g ? h_out : h, 256, M, 256, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
    return fail(DART_ERR_CUDA, "cuTensorMapEncodeTiled failed (fused MLP)");
  const int rc = mlp_fused(th, tw1, tw2, tx, tln, M, b1, b2, ln_g, ln_b, sms, (cudaStream_t)stream);
  if (rc) return fail(DART_ERR_CUDA, std::string("mlp_fused: ") + cudaGetErrorString((cudaError_t)rc));
  return DART_OK;
}

int dart_mlp_fused(const void* h, const void* w1, const float* b1, const void* w2, const float* b2, float* x, int32_t M,
                   void* stream) {
  return dart_mlp_fused_ln(h, w1, b1, w2, b2, x, nullptr, nullptr, nullptr, M, stream);
}

int dart_attention(const void* q, const void* k, const void* v, void* o, int32_t batch, int32_t heads, int32_t Lq,
                   int32_t Lk, int32_t hd, int32_t q_tok_stride, int32_t kv_tok_stride, int32_t o_tok_stride,
                   int64_t q_batch_stride, int64_t kv_batch_stride, int64_t o_batch_stride, int32_t win,
                   int32_t grid, void* stream) {
  if (!q || !k || !v || !o || batch <= 0 || heads <= 0 || Lq <= 0 || Lk <= 0)
    return fail(DART_ERR_INVALID, "dart_attention: bad args");
  AttnArgs a = attn_base(heads, hd);
  a.q = (const __half*)q;
  a.k = (const __half*)k;
  a.v = (const __half*)v;
  a.o = (__half*)o;
  a.q_tok_stride = q_tok_stride;
  a.k_tok_stride = a.v_tok_stride = kv_tok_stride;
  a.o_tok_stride = o_tok_stride;
  a.q_batch_stride = q_batch_stride;
  a.k_batch_stride = a.v_batch_stride = kv_batch_stride;
  a.o_batch_stride = o_batch_stride;
  a.Lq = Lq;
  a.Lk = Lk;
  a.batch = batch;
  if (win > 0) {
    a.win = win;
    a.grid = grid;
    a.nwin = (grid / win) * (grid / win);
    a.img_stride_q = q_batch_stride;
    a.img_stride_k = a.img_stride_v = kv_batch_stride;
    a.img_stride_o = o_batch_stride;
  }
  int rc = attention(a, hd, (cudaStream_t)stream);
  if (rc) return fail(DART_ERR_CUDA, std::string("attention: ") + cudaGetErrorString((cudaError_t)rc));
  return DART_OK;
}

}  // extern "C"

extern "C" int dart_model_set_mask_head(dart_model* m, const float* wq, const float* bq, const float* wf,
                                        const float* bf) {
  if (!m || !wq || !bq || !wf || !bf) return fail(DART_ERR_INVALID, "dart_model_set_mask_head: bad args");
  const int D = m->D, F0 = m->F0;
  float* scratch = nullptr;
  if (cudaMalloc(&scratch, (size_t)std::max(D, F0) * D * sizeof(float)) != cudaSuccess)
    return fail(DART_ERR_CUDA, "mask head upload scratch");
  const float* ptrs[4] = {wq, bq, wf, bf};
  WeightCursor c{ptrs, 4};
  const bool ok = make_gemm(m, c, D, D, scratch, m->mask_q) && make_gemm(m, c, F0, D, scratch, m->mask_f);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaFree(scratch);
  if (!ok || e != cudaSuccess) return fail(DART_ERR_CUDA, "mask head weight upload failed");
  m->has_mask = true;
  return DART_OK;
}

extern "C" int dart_mask_head(dart_model* m, const float* query_features, int32_t B, int32_t N, const float* l0,
                              float* masks, void* stream) {
  if (!m || !query_features || !l0 || !masks || B <= 0 || N <= 0) return fail(DART_ERR_INVALID, "dart_mask_head: bad args");
  if (!m->has_mask) return fail(DART_ERR_INVALID, "dart_mask_head: no mask head uploaded (dart_model_set_mask_head)");
  cudaStream_t s = (cudaStream_t)stream;
  const int D = m->D, F0 = m->F0, T = m->T, Q = m->d.num_queries;
  const size_t rows = (size_t)B * N * Q, tok = (size_t)B * T;
  if (rows > m->mask_cap_rows || tok > m->mask_cap_tok) {
    m->mask_ws.release();
    m->mk_qf = (__half*)m->mask_ws.get(rows * D * 2);
    m->mk_mq = (__half*)m->mask_ws.get(rows * D * 2);
    m->mk_l0 = (__half*)m->mask_ws.get(tok * F0 * 2);
    m->mk_mf = (__half*)m->mask_ws.get(tok * D * 2);
    if (!m->mk_qf || !m->mk_mq || !m->mk_l0 || !m->mk_mf) {
      m->mask_ws.release();
      m->mask_cap_rows = m->mask_cap_tok = 0;
      return fail(DART_ERR_CUDA, "mask head workspace allocation failed");
    }
    m->mask_cap_rows = rows;
    m->mask_cap_tok = tok;
  }
  // mq = qf Wq + bq, mf = L0 Wf + bf (model.py:577-578), fp16 operands / fp32 accumulation
  LAUNCH(cast_f32_to_f16(query_features, m->mk_qf, (long long)rows * D, s));
  LAUNCH(cast_f32_to_f16(l0, m->mk_l0, (long long)tok * F0, s));
  RUN(gemm(m, m->mk_qf, (int)rows, D, m->mask_q, EPI_F16, epi_out(m->mk_mq, D), s));
  RUN(gemm(m, m->mk_l0, (int)tok, F0, m->mask_f, EPI_F16, epi_out(m->mk_mf, D), s));
  // logits[b, c] = mq[b, c] mf[b]^T (model.py:579): mf[b] is the K-major "weight" of a GEMM
  for (int b = 0; b < B; ++b) {
    GemmW g;
    g.w = m->mk_mf + (size_t)b * T * D;
    g.b = nullptr;
    g.N = T;
    g.K = D;
    if (!finish_gemmw(g)) return fail(DART_ERR_INVALID, "dart_mask_head: tokens must be a multiple of 32");
    RUN(gemm(m, m->mk_mq + (size_t)b * N * Q * D, N * Q, D, g, EPI_F32, epi_out(masks + (size_t)b * N * Q * T, T), s));
  }
  return DART_OK;
}

extern "C" void dart_attention_force_safe(int32_t on) { g_attn_force_safe = on ? 1 : 0; }
extern "C" void dart_attention_trace(int64_t* device_buf) { g_attn_trace = (long long*)device_buf; }
extern "C" void dart_attention_variant(int32_t v) { attention_tc_set_variant(v); }

extern "C" int dart_attention_qkv(const void* qkv, void* o, int32_t items, int32_t heads, int32_t L, int32_t hd,
                                  int32_t* debug_host, void* stream) {
  if (!qkv || !o || items <= 0 || heads <= 0 || L <= 0) return fail(DART_ERR_INVALID, "dart_attention_qkv: bad args");
  if (!attention_tc_supported(hd, L)) return fail(DART_ERR_INVALID, "dart_attention_qkv: unsupported hd / L");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return attn_tc_packed((const __half*)qkv, (__half*)o, items, heads, L, hd, heads * hd, sms, (cudaStream_t)stream,
                        debug_host);
}

// error channel of the other C-ABI translation units (nccl_shard.cu)
namespace dart {
int set_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace dart
