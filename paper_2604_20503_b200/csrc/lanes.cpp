// lanes.cpp — green-context lane pool (see lanes.cuh). The driver entry points are resolved at
// run time through the runtime (cudaGetDriverEntryPoint), so the library does not link libcuda.
#include "lanes.cuh"

#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

namespace faser {

namespace {
typedef CUresult (*PFN_GetDevResource)(CUdevice, CUdevResource*, CUdevResourceType);
typedef CUresult (*PFN_SplitByCount)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int,
                                     unsigned int);
typedef CUresult (*PFN_GenerateDesc)(CUdevResourceDesc*, CUdevResource*, unsigned int);
typedef CUresult (*PFN_GreenCtxCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
typedef CUresult (*PFN_GreenCtxDestroy)(CUgreenCtx);
typedef CUresult (*PFN_GreenCtxStreamCreate)(CUstream*, CUgreenCtx, unsigned int, int);
typedef CUresult (*PFN_StreamDestroy)(CUstream);
typedef CUresult (*PFN_DeviceGet)(CUdevice*, int);

struct Driver {
  PFN_GetDevResource get_res = nullptr;
  PFN_SplitByCount split = nullptr;
  PFN_GenerateDesc gen_desc = nullptr;
  PFN_GreenCtxCreate gctx_create = nullptr;
  PFN_GreenCtxDestroy gctx_destroy = nullptr;
  PFN_GreenCtxStreamCreate gstream_create = nullptr;
  PFN_StreamDestroy stream_destroy = nullptr;
  PFN_DeviceGet device_get = nullptr;
  bool ok = false;
};

template <class F>
bool sym(const char* name, F* out) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
    return false;
  *out = reinterpret_cast<F>(p);
  return true;
}

const Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = sym("cuDeviceGetDevResource", &d.get_res) && sym("cuDevSmResourceSplitByCount", &d.split) &&
           sym("cuDevResourceGenerateDesc", &d.gen_desc) && sym("cuGreenCtxCreate", &d.gctx_create) &&
           sym("cuGreenCtxDestroy", &d.gctx_destroy) && sym("cuGreenCtxStreamCreate", &d.gstream_create) &&
           sym("cuStreamDestroy", &d.stream_destroy) && sym("cuDeviceGet", &d.device_get);
  });
  return d;
}
}  // namespace

struct SmLanes::Pair {
  LanePair lanes;
  CUgreenCtx g_draft = nullptr, g_verify = nullptr;
  ~Pair() {
    const Driver& d = driver();
    if (lanes.green) {
      if (lanes.draft) d.stream_destroy(reinterpret_cast<CUstream>(lanes.draft));
      if (lanes.verify) d.stream_destroy(reinterpret_cast<CUstream>(lanes.verify));
      if (g_draft) d.gctx_destroy(g_draft);
      if (g_verify) d.gctx_destroy(g_verify);
    } else {
      if (lanes.draft) cudaStreamDestroy(lanes.draft);
      if (lanes.verify) cudaStreamDestroy(lanes.verify);
    }
  }
};

SmLanes::SmLanes(int device, int total_sms) : device_(device), total_(total_sms > 0 ? total_sms : 148) {
  const char* e = std::getenv("FASER_GREEN");
  const bool off = e && e[0] == '0';
  green_ok_ = !off && driver().ok;
}

SmLanes::~SmLanes() {
  cudaSetDevice(device_);
  cudaDeviceSynchronize();
  pairs_.clear();
}

int SmLanes::draft_sms_for(double r) const {
  int d = static_cast<int>(std::lround(r * total_ / 8.0)) * 8;
  d = std::max(d, 8);
  d = std::min(d, (total_ - 8) / 8 * 8);
  return d;
}

bool SmLanes::get(double r, LanePair* out, std::string* err) {
  if (!(r > 0.0 && r < 1.0)) {
    *err = "draft SM share r must be in (0, 1)";
    return false;
  }
  const int want = draft_sms_for(r);
  std::lock_guard<std::mutex> lk(mu_);
  auto it = pairs_.find(want);
  if (it != pairs_.end()) {
    *out = it->second->lanes;
    return true;
  }
  auto p = std::make_unique<Pair>();
  if (!green_ok_) {  // plain concurrent streams on the whole GPU (no partition)
    if (cudaStreamCreateWithFlags(&p->lanes.draft, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p->lanes.verify, cudaStreamNonBlocking) != cudaSuccess) {
      *err = "cudaStreamCreate failed";
      return false;
    }
    p->lanes.draft_sms = p->lanes.verify_sms = total_;
    p->lanes.green = false;
  } else {
    const Driver& d = driver();
    CUdevice dev = 0;
    CUdevResource all{}, parts[1]{}, rest{};
    unsigned int ng = 1;
    CUdevResourceDesc dd = nullptr, dv = nullptr;
    CUresult rc = d.device_get(&dev, device_);
    if (rc == CUDA_SUCCESS) rc = d.get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM);
    if (rc == CUDA_SUCCESS) rc = d.split(parts, &ng, &all, &rest, 0, static_cast<unsigned>(want));
    if (rc == CUDA_SUCCESS && ng != 1) rc = CUDA_ERROR_INVALID_RESOURCE_CONFIGURATION;
    if (rc == CUDA_SUCCESS) rc = d.gen_desc(&dd, &parts[0], 1);
    if (rc == CUDA_SUCCESS) rc = d.gen_desc(&dv, &rest, 1);
    if (rc == CUDA_SUCCESS) rc = d.gctx_create(&p->g_draft, dd, dev, CU_GREEN_CTX_DEFAULT_STREAM);
    if (rc == CUDA_SUCCESS) rc = d.gctx_create(&p->g_verify, dv, dev, CU_GREEN_CTX_DEFAULT_STREAM);
    CUstream sd = nullptr, sv = nullptr;
    if (rc == CUDA_SUCCESS) rc = d.gstream_create(&sd, p->g_draft, CU_STREAM_NON_BLOCKING, 0);
    if (rc == CUDA_SUCCESS) rc = d.gstream_create(&sv, p->g_verify, CU_STREAM_NON_BLOCKING, 0);
    p->lanes.green = true;
    p->lanes.draft = reinterpret_cast<cudaStream_t>(sd);
    p->lanes.verify = reinterpret_cast<cudaStream_t>(sv);
    if (rc != CUDA_SUCCESS) {
      *err = "green context partition failed (CUresult " + std::to_string(static_cast<int>(rc)) + ")";
      return false;  // p's destructor releases what was created
    }
    p->lanes.draft_sms = static_cast<int>(parts[0].sm.smCount);
    p->lanes.verify_sms = static_cast<int>(rest.sm.smCount);
  }
  *out = p->lanes;
  pairs_[want] = std::move(p);
  return true;
}

}  // namespace faser
