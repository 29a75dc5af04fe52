// tp.cu — collectives and the small kernels of tensor-parallel verification (see tp.cuh).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cfloat>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "faser/engine.h"
#include "tp.cuh"

namespace faser {
namespace {

constexpr int kMaxTp = 8;

struct Ptrs {
  const __nv_bfloat16* p[kMaxTp];
};

// bf16 partials, fp32 accumulation in rank order (deterministic), bf16 result
__global__ void sum_ranks_kernel(Ptrs in, int n_ranks, __nv_bfloat16* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float a = 0.f;
    for (int r = 0; r < n_ranks; ++r) a += __bfloat162float(in.p[r][i]);
    out[i] = __float2bfloat16_rn(a);
  }
}

// ------------------------------------------------------------------ in-process group (1 device)
class Barrier {
 public:
  explicit Barrier(int n) : n_(n) {}
  void wait() {
    std::unique_lock<std::mutex> lk(m_);
    const long gen = gen_;
    if (++count_ == n_) {
      count_ = 0;
      ++gen_;
      cv_.notify_all();
    } else {
      cv_.wait(lk, [&] { return gen_ != gen; });
    }
  }

 private:
  std::mutex m_;
  std::condition_variable cv_;
  int n_, count_ = 0;
  long gen_ = 0;
};

class LocalGroup : public TpGroup {
 public:
  explicit LocalGroup(int n) : bar_(n), slots_(n), ready_(n), done_(n), tmp_(n, nullptr), tmp_cap_(n, 0) {
    size = n;
    for (int r = 0; r < n; ++r) {
      cudaEventCreateWithFlags(&ready_[r], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&done_[r], cudaEventDisableTiming);
    }
  }
  ~LocalGroup() override {
    for (int r = 0; r < size; ++r) {
      cudaEventDestroy(ready_[r]);
      cudaEventDestroy(done_[r]);
      if (tmp_[r]) cudaFree(tmp_[r]);
    }
  }
  const char* backend() const override { return "local"; }

  cudaError_t allreduce_sum(int rank, __nv_bfloat16* buf, size_t n, cudaStream_t s) override {
    cudaError_t e;
    if (tmp_cap_[rank] < n) {
      if (tmp_[rank]) cudaFree(tmp_[rank]);
      if ((e = cudaMalloc(&tmp_[rank], n * sizeof(__nv_bfloat16))) != cudaSuccess) return e;
      tmp_cap_[rank] = n;
    }
    slots_[rank] = buf;
    if ((e = cudaEventRecord(ready_[rank], s)) != cudaSuccess) return e;
    bar_.wait();  // every rank's buffer is registered and its producer event recorded
    Ptrs in{};
    for (int q = 0; q < size; ++q) {
      in.p[q] = reinterpret_cast<const __nv_bfloat16*>(slots_[q]);
      if ((e = cudaStreamWaitEvent(s, ready_[q], 0)) != cudaSuccess) return e;
    }
    sum_ranks_kernel<<<296, 256, 0, s>>>(in, size, tmp_[rank], n);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = cudaEventRecord(done_[rank], s)) != cudaSuccess) return e;
    bar_.wait();  // every rank has enqueued its reads
    for (int q = 0; q < size; ++q)
      if ((e = cudaStreamWaitEvent(s, done_[q], 0)) != cudaSuccess) return e;
    e = cudaMemcpyAsync(buf, tmp_[rank], n * sizeof(__nv_bfloat16), cudaMemcpyDeviceToDevice, s);
    bar_.wait();  // slots_ may be overwritten by the next call only after everyone read them
    return e;
  }

  cudaError_t allgather_f2(int rank, const float2* in, float2* out, size_t n, cudaStream_t s) override {
    cudaError_t e;
    slots_[rank] = const_cast<float2*>(in);
    if ((e = cudaEventRecord(ready_[rank], s)) != cudaSuccess) return e;
    bar_.wait();
    for (int q = 0; q < size; ++q) {
      if ((e = cudaStreamWaitEvent(s, ready_[q], 0)) != cudaSuccess) return e;
      if ((e = cudaMemcpyAsync(out + q * n, static_cast<const float2*>(slots_[q]), n * sizeof(float2),
                               cudaMemcpyDeviceToDevice, s)) !=
          cudaSuccess)
        return e;
    }
    if ((e = cudaEventRecord(done_[rank], s)) != cudaSuccess) return e;
    bar_.wait();
    for (int q = 0; q < size; ++q)
      if ((e = cudaStreamWaitEvent(s, done_[q], 0)) != cudaSuccess) return e;
    bar_.wait();
    return cudaSuccess;
  }

 private:
  Barrier bar_;
  std::vector<void*> slots_;
  std::vector<cudaEvent_t> ready_, done_;
  std::vector<__nv_bfloat16*> tmp_;
  std::vector<size_t> tmp_cap_;
};

// ------------------------------------------------------------------ NCCL (dlopen'ed)
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string err;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("cannot load libnccl: ") + dlerror();
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.all_gather && api.comm_destroy;
    if (!api.ok) api.err = "libnccl lacks a required symbol";
  });
  return api;
}

class NcclGroup : public TpGroup {
 public:
  ncclComm_t comm = nullptr;
  ~NcclGroup() override {
    if (comm) nccl().comm_destroy(comm);
  }
  const char* backend() const override { return "nccl"; }
  cudaError_t allreduce_sum(int, __nv_bfloat16* buf, size_t n, cudaStream_t s) override {
    return nccl().all_reduce(buf, buf, n, ncclBfloat16, ncclSum, comm, s) == ncclSuccess ? cudaSuccess
                                                                                           : cudaErrorUnknown;
  }
  cudaError_t allgather_f2(int, const float2* in, float2* out, size_t n, cudaStream_t s) override {
    return nccl().all_gather(in, out, 2 * n, ncclFloat32, comm, s) == ncclSuccess ? cudaSuccess
                                                                                   : cudaErrorUnknown;
  }
};

// ------------------------------------------------------------------ kernels
__global__ void __launch_bounds__(128) resid_add_kernel(const __nv_bfloat16* __restrict__ part, float* __restrict__ x,
                                                        __nv_bfloat16* __restrict__ xb, float* __restrict__ ss,
                                                        int T, int d) {
  __shared__ float red[4];
  const int t = blockIdx.x, c = blockIdx.y * 128 + threadIdx.x;
  const size_t i = static_cast<size_t>(t) * d + c;
  const float v = x[i] + __bfloat162float(part[i]);
  x[i] = v;
  xb[i] = __float2bfloat16_rn(v);
  float q = v * v;
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x == 0) ss[static_cast<size_t>(blockIdx.y) * T + t] = (red[0] + red[1]) + (red[2] + red[3]);
}

__device__ __forceinline__ void better(float& bv, int& bi, float v, int i) {
  if (v > bv || (v == bv && i < bi)) {
    bv = v;
    bi = i;
  }
}

__global__ void local_argmax_kernel(int n_tiles, int T, const float2* __restrict__ amax, float2* __restrict__ loc) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= T) return;
  float bv = -FLT_MAX;
  int bi = 0x7fffffff;
  for (int m = lane; m < n_tiles; m += 32) {
    const float2 p = amax[static_cast<size_t>(m) * T + r];
    better(bv, bi, p.x, __float_as_int(p.y));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    better(bv, bi, ov, oi);
  }
  if (lane == 0) loc[r] = make_float2(bv, __int_as_float(bi));
}

__global__ void merge_argmax_kernel(int tp, int T, const float2* __restrict__ all, int* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  float bv = -FLT_MAX;
  int bi = 0x7fffffff;
  for (int r = 0; r < tp; ++r) {
    const float2 p = all[static_cast<size_t>(r) * T + t];
    better(bv, bi, p.x, __float_as_int(p.y));
  }
  out[t] = bi;
}

}  // namespace

TpGroup* tp_local_group_create(int size) {
  if (size < 1 || size > kMaxTp) return nullptr;
  return new LocalGroup(size);
}

bool tp_nccl_unique_id(uint8_t* out, const char** err) {
  NcclApi& a = nccl();
  if (!a.ok) {
    *err = a.err.c_str();
    return false;
  }
  ncclUniqueId id;
  if (a.get_unique_id(&id) != ncclSuccess) {
    *err = "ncclGetUniqueId failed";
    return false;
  }
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &id, sizeof(id));
  return true;
}

TpGroup* tp_nccl_group_create(const uint8_t* id, int size, int rank, int device, const char** err) {
  NcclApi& a = nccl();
  if (!a.ok) {
    *err = a.err.c_str();
    return nullptr;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    *err = "cudaSetDevice failed";
    return nullptr;
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  auto* g = new NcclGroup();
  g->size = size;
  if (a.comm_init_rank(&g->comm, size, uid, rank) != ncclSuccess) {
    *err = "ncclCommInitRank failed";
    g->comm = nullptr;
    delete g;
    return nullptr;
  }
  return g;
}

cudaError_t tp_resid_add(const __nv_bfloat16* part, float* x, __nv_bfloat16* xb, float* ss, int T, int d, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  resid_add_kernel<<<dim3(T, d / 128), 128, 0, s>>>(part, x, xb, ss, T, d);
  return cudaGetLastError();
}

cudaError_t tp_local_argmax(int n_tiles, int T, const float2* amax, float2* loc, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  local_argmax_kernel<<<(T * 32 + 255) / 256, 256, 0, s>>>(n_tiles, T, amax, loc);
  return cudaGetLastError();
}

cudaError_t tp_merge_argmax(int tp, int T, const float2* all, int* out, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  merge_argmax_kernel<<<(T + 127) / 128, 128, 0, s>>>(tp, T, all, out);
  return cudaGetLastError();
}

}  // namespace faser

// ------------------------------------------------------------------ C ABI
struct faser_tp_group {
  faser::TpGroup* g;
};

extern "C" {

faser_status faser_tp_nccl_unique_id(uint8_t* id128) {
  if (!id128) return FASER_EINVAL;
  const char* err = nullptr;
  return faser::tp_nccl_unique_id(id128, &err) ? FASER_OK : FASER_ENCCL;
}

faser_status faser_tp_nccl_group_create(const uint8_t* id128, int32_t size, int32_t rank, int32_t device,
                                        faser_tp_group** out) {
  if (!id128 || !out || size < 1 || size > 8 || rank < 0 || rank >= size) return FASER_EINVAL;
  const char* err = nullptr;
  faser::TpGroup* g = faser::tp_nccl_group_create(id128, size, rank, device, &err);
  if (!g) return FASER_ENCCL;
  *out = new faser_tp_group{g};
  return FASER_OK;
}

faser_status faser_tp_local_group_create(int32_t size, faser_tp_group** out) {
  if (!out || size < 1 || size > 8) return FASER_EINVAL;
  *out = new faser_tp_group{faser::tp_local_group_create(size)};
  return FASER_OK;
}

void faser_tp_group_destroy(faser_tp_group* g) {
  if (!g) return;
  delete g->g;
  delete g;
}

}  // extern "C"

namespace faser {
TpGroup* tp_group_of(faser_tp_group* g) { return g ? g->g : nullptr; }
}  // namespace faser
