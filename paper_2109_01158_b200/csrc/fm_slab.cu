// x1-slab exchange of the multi-GPU split issued from the C ABI:
// one pack kernel, ONE grouped NCCL launch (the interface-plane partials to /
// from both neighbours and the all-gather of every rank's J partials), one
// unpack kernel (g += received partials; J = the rank partials summed in rank
// order, so every rank holds the same bits).  The reference has no
// multi-device code; the split reproduces the single-domain sums because J, b
// and the element contributions are all sums over elements (gradients.py:
// 124-149, patches.py:80-83).
//
// NCCL is resolved at run time (dlopen: the copy a host process has already
// loaded — torch's — first, then the system's), so the library loads and runs
// single-GPU without NCCL and links against no particular NCCL build.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "fm_kernels.h"

namespace fm {
namespace {

struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char *(*errorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](const char *n) { return dlsym(h, n); };
    api.getUniqueId = (decltype(api.getUniqueId))sym("ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))sym("ncclCommInitRank");
    api.commDestroy = (decltype(api.commDestroy))sym("ncclCommDestroy");
    api.send = (decltype(api.send))sym("ncclSend");
    api.recv = (decltype(api.recv))sym("ncclRecv");
    api.allGather = (decltype(api.allGather))sym("ncclAllGather");
    api.groupStart = (decltype(api.groupStart))sym("ncclGroupStart");
    api.groupEnd = (decltype(api.groupEnd))sym("ncclGroupEnd");
    api.errorString = (decltype(api.errorString))sym("ncclGetErrorString");
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.send && api.recv &&
             api.allGather && api.groupStart && api.groupEnd && api.errorString;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

#define FM_NCCL(call)                                                                   \
  do {                                                                                  \
    ncclResult_t _r = (call);                                                           \
    if (_r != ncclSuccess) {                                                            \
      ::fm::set_error(std::string(#call) + ": " + ::fm::nccl().errorString(_r));        \
      return FM_CUDA_ERROR;                                                             \
    }                                                                                   \
  } while (0)

// send[k] = g[pos[k]] for the concatenated [left | right] plane positions
__global__ void k_slab_pack(int64_t n, const int64_t *__restrict__ pos,
                            const double *__restrict__ g, double *__restrict__ send) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    send[k] = g[pos[k]];
}

// g[pos[k]] += recv[k] (own + received: the same bits on both sides of a
// plane, as a + b == b + a); block 0 also J[0..2] = sum over ranks of the
// gathered partials, in rank order
__global__ void k_slab_unpack(int64_t n, const int64_t *__restrict__ pos,
                              const double *__restrict__ recv, double *__restrict__ g,
                              const double *__restrict__ jall, int world, double *J) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    g[pos[k]] += recv[k];
  if (J && blockIdx.x == 0 && threadIdx.x < 3) {
    double s = 0.0;
    for (int r = 0; r < world; ++r) s += jall[3 * r + threadIdx.x];
    J[threadIdx.x] = s;
  }
}

// Sub-slab stack on one GPU (a rank's slab split into several contexts):
// the partials of the n interface dofs shared by consecutive sub-slabs,
// s = g[a[k]] + g[b[k]], stored to both copies (bitwise equal, like the
// NCCL exchange's own + received); block 0 also J[0..2] = the K sub-slab
// partials summed in sub-slab order
__global__ void k_stack_reduce(int64_t n, const int64_t *__restrict__ a,
                               const int64_t *__restrict__ b, double *__restrict__ g,
                               const double *__restrict__ jk, int K, double *J) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = a[k], j = b[k];
    const double s = g[i] + g[j];
    g[i] = s;
    g[j] = s;
  }
  if (J && blockIdx.x == 0 && threadIdx.x < 3) {
    double s = 0.0;
    for (int r = 0; r < K; ++r) s += jk[3 * r + threadIdx.x];
    J[threadIdx.x] = s;
  }
}

}  // namespace
}  // namespace fm

struct fm_slab {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  int64_t n_plane = 0;           // doubles per interface plane
  int has_left = 0, has_right = 0;
  int64_t *pos = nullptr;        // [left | right] positions in g (device)
  double *send = nullptr, *recv = nullptr, *jall = nullptr;
};

using namespace fm;

extern "C" {

int fm_comm_unique_id(void *id_host) {
  FM_NVTX("fm_comm_unique_id");
  FM_ARG(id_host, "null argument");
  NcclApi &api = nccl();
  if (!api.ok) {
    set_error("NCCL unavailable: " + api.why);
    return FM_CUDA_ERROR;
  }
  ncclUniqueId id;
  FM_NCCL(api.getUniqueId(&id));
  std::memcpy(id_host, &id, sizeof(id));
  return FM_OK;
}

int fm_slab_create(const void *id_host, int rank, int world, int64_t n_plane,
                   const int64_t *left_pos, const int64_t *right_pos, fm_slab **out) {
  FM_NVTX("fm_slab_create");
  FM_ARG(id_host && out, "null argument");
  FM_ARG(world >= 1 && rank >= 0 && rank < world, "bad rank / world");
  FM_ARG(n_plane >= 0, "negative plane size");
  FM_ARG((rank > 0) == (left_pos != nullptr) && (rank < world - 1) == (right_pos != nullptr),
         "interface planes must be given exactly for the existing neighbours");
  NcclApi &api = nccl();
  if (!api.ok) {
    set_error("NCCL unavailable: " + api.why);
    return FM_CUDA_ERROR;
  }
  *out = nullptr;
  fm_slab *x = new fm_slab();
  auto fail = [&](int code) {
    fm_slab_destroy(x);
    return code;
  };
  x->rank = rank;
  x->world = world;
  x->n_plane = n_plane;
  x->has_left = left_pos != nullptr;
  x->has_right = right_pos != nullptr;
  ncclUniqueId id;
  std::memcpy(&id, id_host, sizeof(id));
  {
    const ncclResult_t r = api.commInitRank(&x->comm, world, id, rank);
    if (r != ncclSuccess) {
      set_error(std::string("ncclCommInitRank: ") + api.errorString(r));
      return fail(FM_CUDA_ERROR);
    }
  }
  const int np = x->has_left + x->has_right;
  const int64_t n = std::max<int64_t>(np * n_plane, 1);
  if (cudaMalloc(&x->pos, n * 8) != cudaSuccess || cudaMalloc(&x->send, n * 8) != cudaSuccess ||
      cudaMalloc(&x->recv, n * 8) != cudaSuccess ||
      cudaMalloc(&x->jall, (size_t)world * 3 * 8) != cudaSuccess) {
    set_error("cudaMalloc failed for the slab exchange buffers");
    return fail(FM_CUDA_ERROR);
  }
  int64_t o = 0;
  if (left_pos) {
    if (cudaMemcpy(x->pos, left_pos, n_plane * 8, cudaMemcpyDeviceToDevice) != cudaSuccess)
      return fail(FM_CUDA_ERROR);
    o += n_plane;
  }
  if (right_pos &&
      cudaMemcpy(x->pos + o, right_pos, n_plane * 8, cudaMemcpyDeviceToDevice) != cudaSuccess)
    return fail(FM_CUDA_ERROR);
  *out = x;
  return FM_OK;
}

int fm_stack_reduce(int64_t n, const int64_t *a, const int64_t *b, double *g, const double *jk,
                    int K, double *J, void *stream) {
  FM_NVTX("fm_stack_reduce");
  FM_ARG(n >= 0 && K >= 0, "negative size");
  FM_ARG(n == 0 || (a && b && g), "null plane positions or gradient");
  FM_ARG(!J || (jk && K > 0), "J needs the sub-slab partials");
  if (n == 0 && !J) return FM_OK;
  cudaStream_t s = as_stream(stream);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 1184));
  k_stack_reduce<<<grid, 256, 0, s>>>(n, a, b, g, jk, K, J);
  FM_CUDA(cudaGetLastError());
  return FM_OK;
}

int fm_slab_destroy(fm_slab *x) {
  if (!x) return FM_OK;
  if (x->comm) nccl().commDestroy(x->comm);
  for (void *p : {(void *)x->pos, (void *)x->send, (void *)x->recv, (void *)x->jall})
    if (p) cudaFree(p);
  delete x;
  return FM_OK;
}

int fm_slab_reduce(fm_slab *x, double *g, double *J, void *stream) {
  FM_NVTX("fm_slab_reduce");
  FM_ARG(x, "null exchange");
  FM_ARG(g || J, "nothing to reduce");
  NcclApi &api = nccl();
  cudaStream_t s = as_stream(stream);
  const int np = x->has_left + x->has_right;
  const int64_t n = g ? np * x->n_plane : 0;
  if (n) {
    k_slab_pack<<<grid_for(n, 256), 256, 0, s>>>(n, x->pos, g, x->send);
    FM_CHECK_LAUNCH();
  }
  // one grouped NCCL launch: both planes each way and the J all-gather (the
  // group is always closed, also when a call inside it fails)
  FM_NCCL(api.groupStart());
  ncclResult_t r = ncclSuccess;
  const char *what = "";
  int64_t o = 0;
  for (int side = 0; side < 2 && n && r == ncclSuccess; ++side) {
    const bool has = side == 0 ? x->has_left : x->has_right;
    if (!has) continue;
    const int peer = side == 0 ? x->rank - 1 : x->rank + 1;
    r = api.send(x->send + o, (size_t)x->n_plane, ncclFloat64, peer, x->comm, s);
    what = "ncclSend";
    if (r == ncclSuccess) {
      r = api.recv(x->recv + o, (size_t)x->n_plane, ncclFloat64, peer, x->comm, s);
      what = "ncclRecv";
    }
    o += x->n_plane;
  }
  if (J && r == ncclSuccess) {
    r = api.allGather(J, x->jall, 3, ncclFloat64, x->comm, s);
    what = "ncclAllGather";
  }
  const ncclResult_t r_end = api.groupEnd();
  if (r != ncclSuccess || r_end != ncclSuccess) {
    set_error(std::string(r != ncclSuccess ? what : "ncclGroupEnd") + ": " +
              api.errorString(r != ncclSuccess ? r : r_end));
    return FM_CUDA_ERROR;
  }
  k_slab_unpack<<<n ? grid_for(n, 256) : 1, 256, 0, s>>>(n, x->pos, x->recv, g, x->jall, x->world,
                                                         J);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

}  // extern "C"
