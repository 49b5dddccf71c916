// Detection-only post-processing (reference pipeline.py:243-294), one CTA per class.
//
// Decisions must be identical to the reference on identical inputs, so every decision-bearing
// value is computed in fp64 in the reference's operation order with explicit round-to-nearest
// intrinsics (no FMA contraction), the exponential correctly rounded (exp_cr below):
//   presence = sigmoid(presence_logit); class skipped if presence < thr   (pipeline.py:277-279)
//   s_q = sigmoid(score_logit_q); candidate iff s_q >= thr                (pipeline.py:280-285)
//   order by (s desc, q asc)                                              (pipeline.py:286)
//   greedy NMS: keep iff IoU(e, k) < thr for every kept k                 (pipeline.py:257-263)
//   IoU from (cx,cy,w,h) corners, 0 if iw<=0 or ih<=0                     (pipeline.py:243-254)
#include "common.cuh"
#include "kernels.h"

namespace dart {
namespace {

constexpr int PP_THREADS = 256;
constexpr int PP_MAXQ = 1024;

// ---- correctly rounded exp in double-double arithmetic.  CUDA's exp() is faithful (<= 1 ulp)
// but not correctly rounded; the reference's NumPy exp is another <= 1 ulp implementation
// (measured here: numpy 2.3 AVX-512 exp differs from the correctly rounded value on ~4.6% of
// inputs, glibc's on ~0.07%).  Rounding the exact value makes the device scores a function of
// the logit alone (platform independent), and tests/test_gpu_parity.py pins it against a
// 50-digit decimal evaluation.  Cost is irrelevant here (<= N*Q evaluations per image).
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = __dadd_rn(a, b), bb = __dsub_rn(s, a);
  return {s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  const double p = __dmul_rn(a, b);
  return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  return quick_two_sum(s.hi, __dadd_rn(s.lo, __dadd_rn(a.lo, b.lo)));
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  return quick_two_sum(p.hi, __fma_rn(a.hi, b.lo, __fma_rn(a.lo, b.hi, p.lo)));
}

__device__ double exp_cr(double x) {
  // x = k ln2 + r, |r| <= ln2/2, ln2 = L0 + L1 + L2 (L0 has 21 significant bits: k L0 is exact)
  const double L0 = 0x1.62e42p-1, L1 = 0x1.fdf473de6af28p-22, L2 = -0x1.c4c67fc0d0951p-76;
  const double k = rint(x * 0x1.71547652b82fep0);
  dd r = two_sum(x, -k * L0);
  r = dd_add(r, two_prod(-k, L1));
  r = dd_add(r, dd{__dmul_rn(-k, L2), 0.0});
  // exp(r) = exp(r / 2^10)^(2^10); Taylor to degree 10 at |r / 2^10| < 3.4e-4 (tail < 1e-41)
  r.hi = ldexp(r.hi, -10);
  r.lo = ldexp(r.lo, -10);
  const dd c[11] = {{1.0, 0.0},
                    {1.0, 0.0},
                    {0.5, 0.0},
                    {0x1.5555555555555p-3, 0x1.5555555555555p-57},
                    {0x1.5555555555555p-5, 0x1.5555555555555p-59},
                    {0x1.1111111111111p-7, 0x1.1111111111111p-63},
                    {0x1.6c16c16c16c17p-10, -0x1.f49f49f49f49fp-65},
                    {0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-73},
                    {0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-76},
                    {0x1.71de3a556c734p-19, -0x1.c154f8ddc6c00p-73},
                    {0x1.27e4fb7789f5cp-22, 0x1.cbbc05b4fa99ap-76}};
  dd e = c[10];
#pragma unroll
  for (int i = 9; i >= 0; --i) e = dd_add(dd_mul(e, r), c[i]);
#pragma unroll
  for (int i = 0; i < 10; ++i) e = dd_mul(e, e);
  // hi = fl(hi + lo): the double nearest the ~1e-29-accurate value, i.e. the correctly
  // rounded exp except within 1e-29 (relative) of a rounding midpoint; 2^k scaling is exact
  // in the used range |x| <= 60
  return ldexp(__dadd_rn(e.hi, e.lo), (int)k);
}

// sigmoid with the reference's clip and operation order (model.py:351-353)
__device__ __forceinline__ double sigmoid_d(double x) {
  x = fmin(fmax(x, -60.0), 60.0);
  return __ddiv_rn(1.0, __dadd_rn(1.0, exp_cr(-x)));
}

__device__ __forceinline__ double iou_d(const double* a, const double* b) {
  const double ax0 = __dsub_rn(a[0], a[2] / 2), ax1 = __dadd_rn(a[0], a[2] / 2);
  const double ay0 = __dsub_rn(a[1], a[3] / 2), ay1 = __dadd_rn(a[1], a[3] / 2);
  const double bx0 = __dsub_rn(b[0], b[2] / 2), bx1 = __dadd_rn(b[0], b[2] / 2);
  const double by0 = __dsub_rn(b[1], b[3] / 2), by1 = __dadd_rn(b[1], b[3] / 2);
  const double iw = __dsub_rn(fmin(ax1, bx1), fmax(ax0, bx0));
  const double ih = __dsub_rn(fmin(ay1, by1), fmax(ay0, by0));
  if (iw <= 0.0 || ih <= 0.0) return 0.0;
  const double inter = __dmul_rn(iw, ih);
  const double uni = __dsub_rn(__dadd_rn(__dmul_rn(a[2], a[3]), __dmul_rn(b[2], b[3])), inter);
  return __ddiv_rn(inter, uni);
}

// priority order: higher score first, then lower index
__device__ __forceinline__ bool before(double sa, int qa, double sb, int qb) {
  return sa > sb || (sa == sb && qa < qb);
}

// One CTA per class.  Dynamic smem: scores [P] f64 | query ids [P] | candidate boxes [Q][4] f64 |
// suppression masks [Q][W] u64 (W = ceil(Q/64)) | kept list [Q].
__global__ void __launch_bounds__(PP_THREADS) pp_class_kernel(const double* __restrict__ boxes,
                                                              const double* __restrict__ score_logits,
                                                              const double* __restrict__ presence_logits, int Q,
                                                              double pthr, double sthr, double nthr, int* kept_count,
                                                              int* kept_query, double* kept_score,
                                                              double* presence_prob) {
  extern __shared__ __align__(16) uint8_t pp_smem[];
  int P = 2;
  while (P < Q) P <<= 1;
  const int W = (Q + 63) >> 6;
  double* ss = reinterpret_cast<double*>(pp_smem);
  double* cb = ss + P;                                      // [Q][4]
  uint64_t* mask = reinterpret_cast<uint64_t*>(cb + 4 * Q);  // [Q][W]
  int* sq = reinterpret_cast<int*>(mask + (size_t)Q * W);    // [P]
  int* kept = sq + P;                                       // [Q]
  __shared__ int nkept, ncand;
  __shared__ bool skip;
  const int c = blockIdx.x, tid = threadIdx.x;
  if (tid == 0) {
    const double p = sigmoid_d(presence_logits[c]);
    presence_prob[c] = p;
    skip = p < pthr;
    nkept = 0;
    ncand = 0;
  }
  __syncthreads();
  if (skip) {
    if (tid == 0) kept_count[c] = 0;
    return;
  }
  for (int i = tid; i < P; i += PP_THREADS) {
    if (i < Q) {
      const double s = sigmoid_d(score_logits[(long long)c * Q + i]);
      const bool ok = s >= sthr;
      ss[i] = ok ? s : -1.0;  // rejected candidates sort last
      sq[i] = i;
      if (ok) atomicAdd(&ncand, 1);
    } else {
      ss[i] = -2.0;
      sq[i] = 0x7fffffff;
    }
  }
  __syncthreads();
  // bitonic sort into priority order
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < P; i += PP_THREADS) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const bool sw = up ? before(ss[l], sq[l], ss[i], sq[i]) : before(ss[i], sq[i], ss[l], sq[l]);
          if (sw) {
            const double ts = ss[i];
            ss[i] = ss[l];
            ss[l] = ts;
            const int tq = sq[i];
            sq[i] = sq[l];
            sq[l] = tq;
          }
        }
      }
      __syncthreads();
    }
  }
  // candidate boxes in priority order, then the suppression matrix in parallel:
  // bit k of row e (k < e) = !(IoU(e, k) < thr), the reference's test (pipeline.py:261)
  const int n = ncand;
  const double* bc = boxes + (long long)c * Q * 4;
  for (int i = tid; i < n * 4; i += PP_THREADS) cb[i] = bc[sq[i >> 2] * 4 + (i & 3)];
  __syncthreads();
  for (int it = tid; it < n * W; it += PP_THREADS) {
    const int e = it / W, w = it - e * W;
    uint64_t m = 0;
    const int k1 = min(e, 64 * w + 64);
    for (int k = 64 * w; k < k1; ++k)
      if (!(iou_d(cb + 4 * e, cb + 4 * k) < nthr)) m |= 1ull << (k - 64 * w);
    mask[it] = m;
  }
  __syncthreads();
  // greedy pass in priority order (one warp): e survives iff no kept k suppresses it
  if (tid < 32) {
    uint64_t km = 0;  // lane w: kept bits of word w
    int nk = 0;
    for (int e = 0; e < n; ++e) {
      const uint64_t m = tid < W ? mask[e * W + tid] : 0;
      if (!__any_sync(0xffffffffu, (m & km) != 0)) {
        if (tid == (e >> 6)) km |= 1ull << (e & 63);
        if (tid == 0) kept[nk] = e;
        ++nk;
      }
    }
    if (tid == 0) nkept = nk;
  }
  __syncthreads();
  const int nk = nkept;
  for (int k = tid; k < nk; k += PP_THREADS) {
    kept_query[(long long)c * Q + k] = sq[kept[k]];
    kept_score[(long long)c * Q + k] = ss[kept[k]];
  }
  if (tid == 0) kept_count[c] = nk;
}

// Cross-class NMS over the per-class survivors (pipeline.py:289-293): order by
// (score desc, detection index asc), greedy NMS, survivors keep their original order.
__global__ void __launch_bounds__(1024) pp_cross_kernel(const double* __restrict__ boxes, const int* kept_count,
                                                        const int* kept_query, const double* kept_score, int N, int Q,
                                                        double nthr, int* keep_flag, int* scratch) {
  __shared__ int total;
  __shared__ int nk;
  const int tid = threadIdx.x;
  int* off = scratch;              // [N+1]
  int* rank_of = scratch + N + 1;  // [total] detection index at each priority rank
  int* kept = rank_of + N * Q;     // [total]
  if (tid == 0) {
    int acc = 0;
    for (int c = 0; c < N; ++c) {
      off[c] = acc;
      acc += kept_count[c];
    }
    off[N] = acc;
    total = acc;
    nk = 0;
  }
  __syncthreads();
  const int T = total;
  auto locate = [&](int i, int& c, int& k) {
    int lo = 0, hi = N;  // off[lo] <= i < off[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (off[mid] <= i) lo = mid; else hi = mid;
    }
    c = lo;
    k = i - off[lo];
  };
  for (int i = tid; i < T; i += blockDim.x) {
    int ci, ki;
    locate(i, ci, ki);
    const double si = kept_score[(long long)ci * Q + ki];
    int r = 0;
    for (int j = 0; j < T; ++j) {
      int cj, kj;
      locate(j, cj, kj);
      const double sj = kept_score[(long long)cj * Q + kj];
      r += before(sj, j, si, i);
    }
    rank_of[r] = i;
    keep_flag[(long long)ci * Q + ki] = 0;
  }
  __syncthreads();
  for (int r = 0; r < T; ++r) {
    const int i = rank_of[r];
    int ci, ki;
    locate(i, ci, ki);
    const int qi = kept_query[(long long)ci * Q + ki];
    double be[4];
    for (int j = 0; j < 4; ++j) be[j] = boxes[((long long)ci * Q + qi) * 4 + j];
    bool sup = false;
    for (int k = tid; k < nk; k += blockDim.x) {
      int ck, kk;
      locate(kept[k], ck, kk);
      const int qk = kept_query[(long long)ck * Q + kk];
      double bk[4];
      for (int j = 0; j < 4; ++j) bk[j] = boxes[((long long)ck * Q + qk) * 4 + j];
      sup |= !(iou_d(be, bk) < nthr);
    }
    const bool any = __syncthreads_or(sup);
    if (!any && tid == 0) {
      kept[nk] = i;
      nk = nk + 1;
      keep_flag[(long long)ci * Q + ki] = 1;
    }
    __syncthreads();
  }
}

}  // namespace

int postprocess_classes(const double* boxes, const double* score_logits, const double* presence_logits, int N, int Q,
                        double presence_thr, double score_thr, double nms_thr, int* kept_count, int* kept_query,
                        double* kept_score, double* presence_prob, cudaStream_t stream) {
  if (N <= 0) return 0;
  if (Q > PP_MAXQ) return (int)cudaErrorInvalidValue;
  int P = 2;
  while (P < Q) P <<= 1;
  const size_t smem = (size_t)P * 8 + (size_t)Q * 32 + (size_t)Q * ((Q + 63) / 64) * 8 + (size_t)P * 4 + (size_t)Q * 4;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(pp_class_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  pp_class_kernel<<<N, PP_THREADS, smem, stream>>>(boxes, score_logits, presence_logits, Q, presence_thr, score_thr,
                                                nms_thr, kept_count, kept_query, kept_score, presence_prob);
  return (int)cudaGetLastError();
}

int postprocess_cross_class(const double* boxes, const int* kept_count, const int* kept_query,
                            const double* kept_score, int N, int Q, double nms_thr, int* keep_flag, int* scratch,
                            cudaStream_t stream) {
  if (N <= 0) return 0;
  pp_cross_kernel<<<1, 1024, 0, stream>>>(boxes, kept_count, kept_query, kept_score, N, Q, nms_thr, keep_flag,
                                          scratch);
  return (int)cudaGetLastError();
}

}  // namespace dart
