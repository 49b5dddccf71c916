// NCCL helpers of the C ABI for the class-sharded mode.
//
// Reference: the per-class loop of encdec_forward (model.py:559-564) -- classes never interact
// after the class-independent prefix (model.py:513-517) -- so N classes can be split over W GPUs:
// every rank runs backbone + prefix for its own B images, the W prefix outputs e1 [B, T, d] fp32
// are all-gathered, every rank decodes ITS contiguous class shard for all W*B images in one
// class-batched pass, and the raw outputs are all-gathered so that each image's owner holds its
// raw outputs over all N classes (then post-processes them exactly like run_batched,
// pipeline.py:198-223, cross-class NMS included).  The same protocol as
// paper_2603_11441_b200/distributed.py:class_sharded_raw, for hosts that do not run
// torch.distributed.
//
// libnccl.so.2 is opened at first use (in a process that already loaded one -- torch's -- the
// dynamic linker hands back that copy), so the library itself has no link-time NCCL dependency.
// Every entry point only enqueues work on `stream`; there is no host synchronisation.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../../include/dart_b200.h"
#include "kernels.h"

namespace dart {
int set_error(int code, const std::string& msg);  // dart_capi.cu
}

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_async_error)(ncclComm_t, ncclResult_t*) = nullptr;  // optional
  ncclResult_t (*comm_abort)(ncclComm_t) = nullptr;                       // optional
  std::string why;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.get_async_error = reinterpret_cast<decltype(api.get_async_error)>(sym("ncclCommGetAsyncError"));
    api.comm_abort = reinterpret_cast<decltype(api.comm_abort)>(sym("ncclCommAbort"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather && api.all_reduce &&
             api.error_string;
    if (!api.ok) api.why = "libnccl.so.2 lacks an expected symbol";
  });
  return api;
}

int nccl_fail(const char* what, ncclResult_t r) {
  return dart::set_error(DART_ERR_CUDA, std::string(what) + ": " + nccl().error_string(r));
}

// raw-output row of one (image, class): boxes (4Q) | score logits (Q) | presence logit (1)
__global__ void pack_raw_kernel(const double* __restrict__ boxes, const double* __restrict__ scores,
                                const double* __restrict__ pres, double* __restrict__ packed, int images, int n,
                                int width, int Q) {
  const int row_len = 5 * Q + 1;
  const long long total = (long long)images * width * row_len;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i % row_len);
    const long long r = i / row_len;
    const int c = (int)(r % width), img = (int)(r / width);
    double v = 0.0;
    if (c < n) {
      const long long item = (long long)img * n + c;
      v = k < 4 * Q ? boxes[item * 4 * Q + k] : k < 5 * Q ? scores[item * Q + (k - 4 * Q)] : pres[item];
    }
    packed[i] = v;
  }
}

// parts [W ranks][W*B images][width][5Q+1] -> this rank's B images over all N classes
__global__ void unpack_raw_kernel(const double* __restrict__ parts, double* __restrict__ boxes,
                                  double* __restrict__ scores, double* __restrict__ pres, int world, int rank, int B,
                                  int N, int width, int Q) {
  const int row_len = 5 * Q + 1;
  const long long total = (long long)B * N * row_len;
  const int base = N / world, extra = N % world;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i % row_len);
    const long long r = i / row_len;
    const int cls = (int)(r % N), b = (int)(r / N);
    // owner rank of class `cls` under ClassShardPlan.bounds (contiguous, the first `extra` ranks one larger)
    const int big = extra * (base + 1);
    const int owner = cls < big ? cls / (base + 1) : extra + (cls - big) / (base > 0 ? base : 1);
    const int start = owner * base + (owner < extra ? owner : extra);
    const long long img = (long long)rank * B + b;
    const double v = parts[(((long long)owner * world * B + img) * width + (cls - start)) * row_len + k];
    const long long item = (long long)b * N + cls;
    if (k < 4 * Q)
      boxes[item * 4 * Q + k] = v;
    else if (k < 5 * Q)
      scores[item * Q + (k - 4 * Q)] = v;
    else
      pres[item] = v;
  }
}

template <typename T>
bool grow(T*& p, size_t& cap, size_t n) {
  if (n <= cap) return true;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) return false;
  cap = n;
  return true;
}

}  // namespace

struct dart_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  // workspace of dart_class_sharded (grown on demand)
  float *l0 = nullptr, *l1 = nullptr, *l2 = nullptr, *e1 = nullptr;
  size_t l0_cap = 0, l1_cap = 0, l2_cap = 0, e1_cap = 0;
  double *bx = nullptr, *sc = nullptr, *pr = nullptr, *packed = nullptr, *parts = nullptr;
  size_t bx_cap = 0, sc_cap = 0, pr_cap = 0, packed_cap = 0, parts_cap = 0;
  ~dart_comm() {
    for (void* p : {(void*)l0, (void*)l1, (void*)l2, (void*)e1, (void*)bx, (void*)sc, (void*)pr, (void*)packed,
                    (void*)parts})
      if (p) cudaFree(p);
    if (comm) nccl().comm_destroy(comm);
  }
};

extern "C" {

int dart_nccl_available(void) { return nccl().ok ? 1 : 0; }

int dart_nccl_unique_id(uint8_t* id) {
  if (!id) return dart::set_error(DART_ERR_INVALID, "dart_nccl_unique_id: null id");
  if (!nccl().ok) return dart::set_error(DART_ERR_CUDA, nccl().why);
  ncclUniqueId u;
  if (ncclResult_t r = nccl().get_unique_id(&u); r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
  static_assert(sizeof(u.internal) == DART_NCCL_ID_BYTES, "NCCL unique id size");
  memcpy(id, u.internal, DART_NCCL_ID_BYTES);
  return DART_OK;
}

int dart_nccl_comm_create(const uint8_t* id, int32_t nranks, int32_t rank, dart_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return dart::set_error(DART_ERR_INVALID, "dart_nccl_comm_create: bad args");
  *out = nullptr;
  if (!nccl().ok) return dart::set_error(DART_ERR_CUDA, nccl().why);
  ncclUniqueId u;
  memcpy(u.internal, id, DART_NCCL_ID_BYTES);
  dart_comm* c = new dart_comm();
  c->nranks = nranks;
  c->rank = rank;
  if (ncclResult_t r = nccl().comm_init_rank(&c->comm, nranks, u, rank); r != ncclSuccess) {
    c->comm = nullptr;
    delete c;
    return nccl_fail("ncclCommInitRank", r);
  }
  *out = c;
  return DART_OK;
}

void dart_nccl_comm_destroy(dart_comm* c) { delete c; }

// Failure detection: a peer that died or a broken link surfaces as an
// asynchronous communicator error; dart_nccl_comm_check reports it without blocking, and
// dart_nccl_comm_abort releases the communicator so that no rank stays blocked in a collective
// (the caller's timeout policy decides when: distributed.NcclComm.wait).
int dart_nccl_comm_check(dart_comm* c) {
  if (!c) return dart::set_error(DART_ERR_INVALID, "dart_nccl_comm_check: null communicator");
  if (!c->comm) return dart::set_error(DART_ERR_CUDA, "NCCL communicator was aborted");
  if (!nccl().get_async_error) return DART_OK;
  ncclResult_t async = ncclSuccess;
  if (ncclResult_t r = nccl().get_async_error(c->comm, &async); r != ncclSuccess)
    return nccl_fail("ncclCommGetAsyncError", r);
  return async == ncclSuccess || async == ncclInProgress ? DART_OK : nccl_fail("NCCL asynchronous error", async);
}

int dart_nccl_comm_abort(dart_comm* c) {
  if (!c) return dart::set_error(DART_ERR_INVALID, "dart_nccl_comm_abort: null communicator");
  if (!c->comm) return DART_OK;
  ncclResult_t r = nccl().comm_abort ? nccl().comm_abort(c->comm) : nccl().comm_destroy(c->comm);
  c->comm = nullptr;  // the destructor must not destroy it again
  return r == ncclSuccess ? DART_OK : nccl_fail("ncclCommAbort", r);
}

int32_t dart_nccl_comm_size(const dart_comm* c) { return c ? c->nranks : 0; }
int32_t dart_nccl_comm_rank(const dart_comm* c) { return c ? c->rank : -1; }

int dart_nccl_all_gather(dart_comm* c, const void* send, void* recv, int64_t bytes_per_rank, void* stream) {
  if (!c || !send || !recv || bytes_per_rank < 0) return dart::set_error(DART_ERR_INVALID, "dart_nccl_all_gather: bad args");
  if (!c->comm) return dart::set_error(DART_ERR_CUDA, "NCCL communicator was aborted");
  ncclResult_t r = nccl().all_gather(send, recv, (size_t)bytes_per_rank, ncclUint8, c->comm, (cudaStream_t)stream);
  return r == ncclSuccess ? DART_OK : nccl_fail("ncclAllGather", r);
}

int dart_nccl_all_reduce_max_i32(dart_comm* c, int32_t* buf, int64_t count, void* stream) {
  if (!c || !buf || count < 0) return dart::set_error(DART_ERR_INVALID, "dart_nccl_all_reduce_max_i32: bad args");
  if (!c->comm) return dart::set_error(DART_ERR_CUDA, "NCCL communicator was aborted");
  ncclResult_t r = nccl().all_reduce(buf, buf, (size_t)count, ncclInt32, ncclMax, c->comm, (cudaStream_t)stream);
  return r == ncclSuccess ? DART_OK : nccl_fail("ncclAllReduce", r);
}

int dart_class_sharded(dart_model* m, dart_comm* c, const float* images, int32_t B, const float* text, int32_t N,
                       double* boxes, double* score_logits, double* presence_logits, int32_t* flags, void* stream) {
  if (!m || !c || !images || B <= 0 || !text || N <= 0 || !boxes || !score_logits || !presence_logits || !flags)
    return dart::set_error(DART_ERR_INVALID, "dart_class_sharded: bad args");
  if (!c->comm) return dart::set_error(DART_ERR_CUDA, "NCCL communicator was aborted");
  const dart_model_desc* d = dart_model_get_desc(m);
  const int g = d->image_size / d->patch_size, T = g * g, D = d->text_dim, Q = d->num_queries, Lt = d->text_tokens;
  const int W = c->nranks, R = c->rank;
  const int base = N / W, extra = N % W;
  const int start = R * base + (R < extra ? R : extra), n = base + (R < extra ? 1 : 0);
  const int width = (N + W - 1) / W, row_len = 5 * Q + 1;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t e1_one = (size_t)B * T * D;
  if (!grow(c->l0, c->l0_cap, (size_t)B * T * d->fpn_dims[0]) ||
      !grow(c->l1, c->l1_cap, (size_t)B * (T / 4) * d->fpn_dims[1]) ||
      !grow(c->l2, c->l2_cap, (size_t)B * (T / 16) * d->fpn_dims[2]) || !grow(c->e1, c->e1_cap, e1_one * W) ||
      !grow(c->bx, c->bx_cap, (size_t)W * B * (n > 0 ? n : 1) * Q * 4) ||
      !grow(c->sc, c->sc_cap, (size_t)W * B * (n > 0 ? n : 1) * Q) ||
      !grow(c->pr, c->pr_cap, (size_t)W * B * (n > 0 ? n : 1)) ||
      !grow(c->packed, c->packed_cap, (size_t)W * B * width * row_len) ||
      !grow(c->parts, c->parts_cap, (size_t)W * W * B * width * row_len))
    return dart::set_error(DART_ERR_CUDA, "dart_class_sharded: workspace allocation failed");
  // 1. backbone + class-independent prefix of this rank's images, written in place into slot R
  //    of the gathered e1 buffer (NCCL in-place all-gather)
  if (int rc = dart_backbone(m, images, B, c->l0, c->l1, c->l2, flags, stream)) return rc;
  if (int rc = dart_encdec_prefix(m, nullptr, B, c->e1 + (size_t)R * e1_one, stream)) return rc;
  if (int rc = dart_nccl_all_gather(c, c->e1 + (size_t)R * e1_one, c->e1, (int64_t)(e1_one * sizeof(float)), stream))
    return rc;
  // status flags MAX-reduced: a bad image raises on every rank after the host reads them
  if (int rc = dart_nccl_all_reduce_max_i32(c, flags, 1, stream)) return rc;
  // 2. this rank's class shard for all W*B images (one class-batched pass)
  if (n > 0)
    if (int rc = dart_encdec_from_prefix(m, c->e1, W * B, text + (size_t)start * Lt * D, n, c->bx, c->sc, c->pr,
                                         nullptr, stream))
      return rc;
  // 3. raw outputs -> padded rows -> all-gather -> this rank's images over all N classes
  const long long packed_n = (long long)W * B * width * row_len;
  pack_raw_kernel<<<(int)((packed_n + 255) / 256 < 4096 ? (packed_n + 255) / 256 : 4096), 256, 0, s>>>(
      c->bx, c->sc, c->pr, c->packed, W * B, n, width, Q);
  if (cudaError_t e = cudaGetLastError(); e != cudaSuccess)
    return dart::set_error(DART_ERR_CUDA, std::string("pack_raw: ") + cudaGetErrorString(e));
  if (int rc = dart_nccl_all_gather(c, c->packed, c->parts, (int64_t)(packed_n * sizeof(double)), stream)) return rc;
  const long long out_n = (long long)B * N * row_len;
  unpack_raw_kernel<<<(int)((out_n + 255) / 256 < 4096 ? (out_n + 255) / 256 : 4096), 256, 0, s>>>(
      c->parts, boxes, score_logits, presence_logits, W, R, B, N, width, Q);
  if (cudaError_t e = cudaGetLastError(); e != cudaSuccess)
    return dart::set_error(DART_ERR_CUDA, std::string("unpack_raw: ") + cudaGetErrorString(e));
  return DART_OK;
}

}  // extern "C"
