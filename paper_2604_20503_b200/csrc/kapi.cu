// kapi.cu — kernel-level C ABI (include/faser/kernels.h): thin wrappers that validate
// arguments and call the same launchers the engine uses.
#include <cuda_runtime.h>

#include <string>

#include "faser/kernels.h"
#include "tc_gemm.cuh"

namespace faser {
namespace {

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (!n) n = 148;
  }
  return n;
}

}  // namespace
}  // namespace faser

using namespace faser;

extern "C" faser_status faser_k_gemm_bf16_plan(const void* w, const void* x, float* out, int32_t n_out,
                                               int32_t t, int32_t k, int32_t bn, int32_t splits,
                                               void* stream) {
  // bn may carry a pipeline-depth request in its upper bits: 1000 + bn = shallow, 2000 + bn = deep
  int depth = bn / 1000;
  bn %= 1000;
  if (bn != 0 && bn != 32 && bn != 64 && bn != 128 && bn != 256) return FASER_EINVAL;
  if (!w || !x || !out || n_out <= 0 || t < 0 || k <= 0) return FASER_EINVAL;
  if (n_out % 128 || k % 64) return FASER_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return FASER_ECUDA;
  if (t == 0) return FASER_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GemmOperand W, X;
  if (make_weight_operand(&W, w, n_out, k) != cudaSuccess) return FASER_ECUDA;
  if (make_act_operand(&X, x, t, k) != cudaSuccess) return FASER_ECUDA;
  GemmPlan plan = gemm_plan(n_out, t, k, num_sms());
  if (bn > 0) plan.bn = bn;
  if (depth == 1) plan.deep = false;
  if (depth == 2) plan.deep = true;
  if (splits > 0) {  // caller-forced split count (cluster size <= 8)
    const int kb = k / 64, s1 = splits < 8 ? splits : 8;
    const int kps = (kb + s1 - 1) / s1;
    plan.splits = (kb + kps - 1) / kps;
  }
  EpiArgs ea;
  ea.mode = kEpiStore;
  ea.t_stride = t;
  ea.out = out;
  cudaError_t e = gemm_fused(W, X, t, plan, ea, s);
  return e == cudaSuccess ? FASER_OK : FASER_ECUDA;
}

extern "C" faser_status faser_k_gemm_bf16(const void* w, const void* x, float* out, int32_t n_out,
                                          int32_t t, int32_t k, int32_t splits, void* stream) {
  return faser_k_gemm_bf16_plan(w, x, out, n_out, t, k, 0, splits, stream);
}
