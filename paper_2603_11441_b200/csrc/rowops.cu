// Row-local kernels of the DART hot path (all HBM/L2-bound, one pass each):
//   LayerNorm fp32 -> fp16/fp32          reference tensors.py:215-227 (population var, eps 1e-6)
//   patchify + [0,1] range flag          reference model.py:426-436
//   2x2 / 4x4 token mean-pool            reference model.py:439-443
//   finiteness flag                      reference model.py:161-166
//   text-row gather (embedding cache)    reference model.py:462-484
//   box / score / presence heads         reference model.py:528-532, sigmoid model.py:351-353
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace dart {
namespace {

constexpr float LN_EPS = 1e-6f;

// One warp per RPW rows (RPW = 1 or 2: both rows' loads in flight before either reduction);
// VPL values per lane.  VPL % 4 == 0: float4 loads of columns 128*i + 4*lane .. +3 (fully
// coalesced 512 B per warp instruction) and 8-byte fp16 stores.  Two-pass (mean, then centred
// variance) in fp32, population variance, eps 1e-6 (reference tensors.py:215-227).
template <int VPL, typename OutT, int RPW = 1>
__global__ void layernorm_vec_kernel(const float* __restrict__ x, const float* __restrict__ gamma,
                                     const float* __restrict__ beta, OutT* __restrict__ y, int rows, int ld_in,
                                     int ld_out) {
  pdl_wait();
  constexpr int V4 = VPL / 4;
  const int row0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * RPW;
  const int lane = threadIdx.x & 31;
  if (row0 >= rows) return;
  float4 v[RPW][V4];
  float s[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    s[r] = 0.f;
    const int row = row0 + r < rows ? row0 + r : row0;
    const float4* xr = reinterpret_cast<const float4*>(x + (size_t)row * ld_in);
#pragma unroll
    for (int i = 0; i < V4; ++i) v[r][i] = xr[32 * i + lane];
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r)
#pragma unroll
    for (int i = 0; i < V4; ++i) s[r] += (v[r][i].x + v[r][i].y) + (v[r][i].z + v[r][i].w);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int r = 0; r < RPW; ++r) s[r] += __shfl_xor_sync(0xffffffff, s[r], o);
  float mu[RPW], q[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    mu[r] = s[r] * (1.0f / (32 * VPL));
    q[r] = 0.f;
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const float a = v[r][i].x - mu[r], b = v[r][i].y - mu[r], c = v[r][i].z - mu[r], d = v[r][i].w - mu[r];
      q[r] += (a * a + b * b) + (c * c + d * d);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int r = 0; r < RPW; ++r) q[r] += __shfl_xor_sync(0xffffffff, q[r], o);
  const float4* g4 = reinterpret_cast<const float4*>(gamma);
  const float4* b4 = reinterpret_cast<const float4*>(beta);
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    if (row0 + r >= rows) break;
    const float rstd = 1.0f / sqrtf(q[r] * (1.0f / (32 * VPL)) + LN_EPS);
    const size_t row = (size_t)(row0 + r);
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const float4 g = __ldg(g4 + 32 * i + lane), b = __ldg(b4 + 32 * i + lane);
      const float4 w = v[r][i];
      const float r0 = (w.x - mu[r]) * rstd * g.x + b.x, r1 = (w.y - mu[r]) * rstd * g.y + b.y;
      const float r2 = (w.z - mu[r]) * rstd * g.z + b.z, r3 = (w.w - mu[r]) * rstd * g.w + b.w;
      if constexpr (sizeof(OutT) == 2) {
        reinterpret_cast<uint2*>(y + row * ld_out)[32 * i + lane] = make_uint2(pack_half2(r0, r1), pack_half2(r2, r3));
      } else {
        reinterpret_cast<float4*>(y + row * ld_out)[32 * i + lane] = make_float4(r0, r1, r2, r3);
      }
    }
  }
}

// One warp per row of a row-block dependency chain (GemmEpi::dep_*): the row's 128-row block must
// be complete in wait_cnt before x is read; the finished row is counted in sig_cnt.
template <int VPL>
__device__ __forceinline__ void layernorm_chain_rows(const float* __restrict__ x, const float* __restrict__ gamma,
                                                     const float* __restrict__ beta, __half* __restrict__ y,
                                                     int rows, const int* wait_cnt, int wait_target) {
  if (wait_cnt == nullptr) pdl_wait();
  pdl_launch_dependents();  // the consumer (QKV) may take SMs as this grid's CTAs free them
  constexpr int V4 = VPL / 4, DIM = 32 * VPL;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (wait_cnt != nullptr) {  // one poller per CTA: its rows (a multiple of 8 apart) share a 128-row block
    if (threadIdx.x == 0) {
      const int blk = (blockIdx.x * (blockDim.x >> 5)) >> 7;
      long long spins = 0;
      while (*reinterpret_cast<const volatile int*>(wait_cnt + blk) < wait_target) {
        __nanosleep(512);
        if (++spins > (1ll << 24)) __trap();  // a broken chain fails loudly instead of hanging
      }
    }
    __syncthreads();
    __threadfence();
  }
  if (row >= rows) return;  // (no barrier follows inside: the caller's __syncthreads sees every warp)
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)row * DIM);
  float4 v[V4];
#pragma unroll
  for (int i = 0; i < V4; ++i) v[i] = __ldcg(xr + 32 * i + lane);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < V4; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  const float mu = s * (1.0f / DIM);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    const float a = v[i].x - mu, b = v[i].y - mu, c = v[i].z - mu, d = v[i].w - mu;
    q += (a * a + b * b) + (c * c + d * d);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffff, q, o);
  const float rstd = 1.0f / sqrtf(q * (1.0f / DIM) + LN_EPS);
  const float4* g4 = reinterpret_cast<const float4*>(gamma);
  const float4* b4 = reinterpret_cast<const float4*>(beta);
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    const float4 g = __ldg(g4 + 32 * i + lane), b = __ldg(b4 + 32 * i + lane);
    const float4 w = v[i];
    const float r0 = (w.x - mu) * rstd * g.x + b.x, r1 = (w.y - mu) * rstd * g.y + b.y;
    const float r2 = (w.z - mu) * rstd * g.z + b.z, r3 = (w.w - mu) * rstd * g.w + b.w;
    reinterpret_cast<uint2*>(y + (size_t)row * DIM)[32 * i + lane] = make_uint2(pack_half2(r0, r1), pack_half2(r2, r3));
  }
}

// the CTA's rows are announced together: barrier, then one device-scope fence + atomic (the
// grid-sync pattern: the barrier orders every warp's stores before thread 0's fence)
template <int VPL>
__global__ void layernorm_chain_kernel_cta(const float* __restrict__ x, const float* __restrict__ gamma,
                                           const float* __restrict__ beta, __half* __restrict__ y, int rows,
                                           const int* wait_cnt, int wait_target, int* sig_cnt) {
  layernorm_chain_rows<VPL>(x, gamma, beta, y, rows, wait_cnt, wait_target);
  __syncthreads();
  if (threadIdx.x == 0) {
    const int row0 = blockIdx.x * (blockDim.x >> 5);
    const int n = rows - row0 < (int)(blockDim.x >> 5) ? rows - row0 : (int)(blockDim.x >> 5);
    __threadfence();
    if (n > 0) atomicAdd(sig_cnt + (row0 >> 7), n);
  }
}

template <int VPL, typename OutT>
__global__ void layernorm_kernel(const float* __restrict__ x, const float* __restrict__ gamma,
                                 const float* __restrict__ beta, OutT* __restrict__ y, int rows, int ld_in,
                                 int ld_out) {
  pdl_wait();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* xr = x + (size_t)row * ld_in;
  float v[VPL];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    v[i] = xr[lane + 32 * i];
    s += v[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  const float mu = s * (1.0f / (32 * VPL));
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const float d = v[i] - mu;
    q += d * d;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffff, q, o);
  const float rstd = 1.0f / sqrtf(q * (1.0f / (32 * VPL)) + LN_EPS);
  OutT* yr = y + (size_t)row * ld_out;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = lane + 32 * i;
    const float r = (v[i] - mu) * rstd * __ldg(gamma + c) + __ldg(beta + c);
    if constexpr (sizeof(OutT) == 2)
      yr[c] = __float2half_rn(r);
    else
      yr[c] = r;
  }
}

int env_int(const char* n, int d) {
  const char* e = getenv(n);
  return e ? atoi(e) : d;
}
// LayerNorm launch shape (A/B: DART_LN_WARPS warps per block, DART_LN_RPW rows per warp)
int g_ln_warps = env_int("DART_LN_WARPS", 4), g_ln_rpw = env_int("DART_LN_RPW", 1);  // measured best (scripts/bench_ln.py)

template <typename OutT>
int ln_dispatch(const float* x, const float* g, const float* b, OutT* y, int rows, int dim, int ld_in, int ld_out,
                cudaStream_t st) {
  if (rows <= 0) return 0;
  const int warps = g_ln_warps;
  const int rpw = g_ln_rpw;
  // every LN launch may overlap its predecessor's tail (PDL; the kernel waits before reading x)
  auto go = [&](auto kern, dim3 gr) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = gr;
    cfg.blockDim = dim3(warps * 32);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    if (pdl_enabled()) {
      pdl_attr(attr[0]);
      cfg.attrs = attr;
      cfg.numAttrs = 1;
    }
    cudaLaunchKernelEx(&cfg, kern, x, g, b, y, rows, ld_in, ld_out);
  };
  dim3 grid((rows + warps - 1) / warps);
  if (rpw == 2 && (dim == 256 || dim == 1280)) {
    dim3 g2((rows + 2 * warps - 1) / (2 * warps));
    if (dim == 256) go(layernorm_vec_kernel<8, OutT, 2>, g2);
    else go(layernorm_vec_kernel<40, OutT, 2>, g2);
    return (int)cudaGetLastError();
  }
  switch (dim) {
    case 32: go(layernorm_kernel<1, OutT>, grid); break;
    case 64: go(layernorm_kernel<2, OutT>, grid); break;
    case 128: go(layernorm_kernel<4, OutT>, grid); break;
    case 256: go(layernorm_vec_kernel<8, OutT>, grid); break;
    case 512: go(layernorm_vec_kernel<16, OutT>, grid); break;
    case 1024: go(layernorm_vec_kernel<32, OutT>, grid); break;
    case 1280: go(layernorm_vec_kernel<40, OutT>, grid); break;
    default: return (int)cudaErrorInvalidValue;
  }
  return (int)cudaGetLastError();
}

__global__ void cast_kernel(const float* __restrict__ x, __half* __restrict__ y, long long n) {
  long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    float4 v = *reinterpret_cast<const float4*>(x + i);
    uint2 u = make_uint2(pack_half2(v.x, v.y), pack_half2(v.z, v.w));
    *reinterpret_cast<uint2*>(y + i) = u;
  } else {
    for (; i < n; ++i) y[i] = __float2half_rn(x[i]);
  }
}

// patches[b*T + t][k] for k < 3p^2 in (py, px, ch) order, zero for k in [3p^2, kpad).
// Output rows are window-major (win > 0) so every attention window is a contiguous block.
__global__ void patchify_kernel(const float* __restrict__ img, __half* __restrict__ out, int B, int S, int p,
                                int kpad, int win, int* flags) {
  const int g = S / p;
  const long long total = (long long)B * g * g * kpad;
  const int kdim = 3 * p * p;
  bool bad = false;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(idx % kpad);
    const long long tokb = idx / kpad;
    float val = 0.f;
    if (k < kdim) {
      const int b = (int)(tokb / (g * g));
      int t = (int)(tokb % (g * g));
      if (win > 0) t = wm_to_token(t, g, win);
      const int r = t / g, c = t % g;
      const int py = k / (3 * p), rem = k % (3 * p), px = rem / 3, ch = rem % 3;
      val = img[(((long long)b * S + r * p + py) * S + c * p + px) * 3 + ch];
      bad |= !(val >= 0.f && val <= 1.f);
    }
    out[idx] = __float2half_rn(val);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, 1);
}

__global__ void pool_kernel(const float* __restrict__ x, __half* __restrict__ y, int B, int grid, int dim,
                            int f, int win) {
  const int g2 = grid / f;
  const long long total = (long long)B * g2 * g2 * dim;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(idx % dim);
    const long long ot = idx / dim;
    const int b = (int)(ot / (g2 * g2));
    const int t = (int)(ot % (g2 * g2));
    const int r = t / g2, c = t % g2;
    float s = 0.f;
    for (int i = 0; i < f; ++i)
      for (int j = 0; j < f; ++j) {
        int t = (r * f + i) * grid + c * f + j;
        if (win > 0) t = token_to_wm(t, grid, win);
        s += x[((long long)b * grid * grid + t) * dim + e];
      }
    y[idx] = __float2half_rn(s / (float)(f * f));
  }
}

__global__ void finite_kernel(const float* __restrict__ x, long long n, int* flags, int bit) {
  bool bad = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, bit);
}

__global__ void broadcast_kernel(const float4* __restrict__ src, float4* __restrict__ dst, long long n4, int reps) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4 * reps;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i % n4];
}

__global__ void gather_kernel(const float* __restrict__ table, const int* __restrict__ rows, __half* __restrict__ out,
                              int n, int dim) {
  const long long total = (long long)n * dim;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x)
    out[i] = __float2half_rn(table[(long long)rows[i / dim] * dim + i % dim]);
}

__device__ __forceinline__ float sigmoid_ref(float x) {
  x = fminf(fmaxf(x, -60.f), 60.f);
  return 1.f / (1.f + expf(-x));
}

// One warp per decoder row: rows [0, nq) -> box (4, sigmoid) + score; row nq -> presence.
__global__ void heads_kernel(const float* __restrict__ qf, int rows_per_item, int nq, int items, int d,
                             const float* __restrict__ wb, const float* __restrict__ bb,
                             const float* __restrict__ ws, const float* __restrict__ bs,
                             const float* __restrict__ wp, const float* __restrict__ bp, double* boxes,
                             double* scores, double* presence, float* qf_out) {
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (gw >= items * (nq + 1)) return;
  const int item = gw / (nq + 1), q = gw % (nq + 1);
  const float* x = qf + ((long long)item * rows_per_item + q) * d;
  if (q < nq) {
    float acc[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
    for (int i = lane; i < d; i += 32) {
      const float xv = x[i];
      acc[0] += xv * wb[i * 4 + 0];
      acc[1] += xv * wb[i * 4 + 1];
      acc[2] += xv * wb[i * 4 + 2];
      acc[3] += xv * wb[i * 4 + 3];
      acc[4] += xv * ws[i];
      if (qf_out) qf_out[((long long)item * nq + q) * d + i] = xv;
    }
#pragma unroll
    for (int j = 0; j < 5; ++j)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffff, acc[j], o);
    if (lane == 0) {
      double* bx = boxes + ((long long)item * nq + q) * 4;
      for (int j = 0; j < 4; ++j) bx[j] = (double)sigmoid_ref(acc[j] + bb[j]);
      scores[(long long)item * nq + q] = (double)(acc[4] + bs[0]);
    }
  } else {
    float acc = 0.f;
    for (int i = lane; i < d; i += 32) acc += x[i] * wp[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffff, acc, o);
    if (lane == 0) presence[item] = (double)(acc + bp[0]);
  }
}

inline int grid_for(long long n, int threads = 256) {
  long long g = (n + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

int layernorm_f32_to_f16_chain(const float* x, const float* gamma, const float* beta, __half* y, int rows, int dim,
                               const int* wait_cnt, int wait_target, int* sig_cnt, cudaStream_t stream) {
  if (rows <= 0) return 0;
  if (dim != 1280 || sig_cnt == nullptr) return (int)cudaErrorInvalidValue;
  constexpr int warps = 8;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((rows + warps - 1) / warps);
  cfg.blockDim = dim3(warps * 32);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  pdl_attr(attr[0]);  // always: the chain relies on launching into the producer's tail
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, layernorm_chain_kernel_cta<40>, x, gamma, beta, y, rows, wait_cnt, wait_target, sig_cnt);
  return (int)cudaGetLastError();
}

int layernorm_f32_to_f16(const float* x, const float* gamma, const float* beta, __half* y, int rows, int dim,
                         int ld_in, int ld_out, cudaStream_t stream) {
  return ln_dispatch<__half>(x, gamma, beta, y, rows, dim, ld_in, ld_out, stream);
}
int layernorm_f32_to_f32(const float* x, const float* gamma, const float* beta, float* y, int rows, int dim,
                         cudaStream_t stream) {
  return ln_dispatch<float>(x, gamma, beta, y, rows, dim, dim, dim, stream);
}
int cast_f32_to_f16(const float* x, __half* y, long long n, cudaStream_t stream) {
  if (n <= 0) return 0;
  const long long threads = (n + 3) / 4;
  cast_kernel<<<(int)((threads + 255) / 256), 256, 0, stream>>>(x, y, n);
  return (int)cudaGetLastError();
}
int patchify(const float* images, __half* patches, int B, int S, int p, int kpad, int win, int* flags,
             cudaStream_t stream) {
  const long long total = (long long)B * (S / p) * (S / p) * kpad;
  patchify_kernel<<<grid_for(total), 256, 0, stream>>>(images, patches, B, S, p, kpad, win, flags);
  return (int)cudaGetLastError();
}
int pool_tokens(const float* x, __half* y, int B, int grid, int dim, int factor, int win, cudaStream_t stream) {
  const long long total = (long long)B * (grid / factor) * (grid / factor) * dim;
  pool_kernel<<<grid_for(total), 256, 0, stream>>>(x, y, B, grid, dim, factor, win);
  return (int)cudaGetLastError();
}
int finite_check(const float* x, long long n, int* flags, int bit, cudaStream_t stream) {
  finite_kernel<<<grid_for(n), 256, 0, stream>>>(x, n, flags, bit);
  return (int)cudaGetLastError();
}
int broadcast_rows(const float* src, float* dst, long long row_elems, int reps, cudaStream_t stream) {
  if (row_elems % 4 != 0) return (int)cudaErrorInvalidValue;
  const long long n4 = row_elems / 4;
  broadcast_kernel<<<grid_for(n4 * reps), 256, 0, stream>>>(reinterpret_cast<const float4*>(src),
                                                            reinterpret_cast<float4*>(dst), n4, reps);
  return (int)cudaGetLastError();
}
int gather_rows_f16(const float* table, const int* rows, __half* out, int n, int dim, cudaStream_t stream) {
  gather_kernel<<<grid_for((long long)n * dim), 256, 0, stream>>>(table, rows, out, n, dim);
  return (int)cudaGetLastError();
}
int heads_forward(const float* qf, int rows_per_item, int nq, int items, int d, const float* w_box,
                  const float* b_box, const float* w_score, const float* b_score, const float* w_pres,
                  const float* b_pres, double* boxes, double* scores, double* presence, float* qf_out,
                  cudaStream_t stream) {
  const int warps = 8;
  const int total = items * (nq + 1);
  heads_kernel<<<(total + warps - 1) / warps, warps * 32, 0, stream>>>(
      qf, rows_per_item, nq, items, d, w_box, b_box, w_score, b_score, w_pres, b_pres, boxes, scores, presence,
      qf_out);
  return (int)cudaGetLastError();
}

// -1: the process default (on unless DART_NO_PDL is set); 0 / 1: this host thread's launches
thread_local int g_pdl_thread = -1;
void pdl_set_thread(int mode) { g_pdl_thread = mode < 0 ? -1 : (mode ? 1 : 0); }
bool pdl_enabled() {
  static const bool on = getenv("DART_NO_PDL") == nullptr;
  return g_pdl_thread >= 0 ? g_pdl_thread == 1 : on;
}

}  // namespace dart
