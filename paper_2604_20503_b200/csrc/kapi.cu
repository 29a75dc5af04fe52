// kapi.cu — kernel-level C ABI (include/faser/kernels.h): thin wrappers that validate
// arguments and call the same launchers the engine uses.
#include <cuda_runtime.h>

#include <string>

#include "faser/kernels.h"
#include "tc_gemm.cuh"

namespace faser {
namespace {

__global__ void sum_splits_kernel(const float* __restrict__ ws, float* __restrict__ out,
                                  int splits, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float a = 0.f;
    for (int z = 0; z < splits; ++z) a += ws[z * n + i];
    out[i] = a;
  }
}

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

extern "C" faser_status faser_k_gemm_bf16(const void* w, const void* x, float* out, int32_t n_out,
                                          int32_t t, int32_t k, int32_t splits, void* stream) {
  if (!w || !x || !out || n_out <= 0 || t < 0 || k <= 0) return FASER_EINVAL;
  if (n_out % 128 || k % 64) return FASER_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return FASER_ECUDA;
  if (t == 0) return FASER_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GemmOperand W, X;
  if (make_weight_operand(&W, w, n_out, k) != cudaSuccess) return FASER_ECUDA;
  if (make_act_operand(&X, x, t, k) != cudaSuccess) return FASER_ECUDA;
  if (splits <= 0) splits = gemm_splits_for(n_out, t, k, num_sms());
  const int z = gemm_effective_splits(k, splits);
  float* ws = out;
  if (z > 1 && cudaMallocAsync(&ws, sizeof(float) * z * static_cast<size_t>(t) * n_out, s) != cudaSuccess)
    return FASER_ENOMEM;
  cudaError_t e = gemm_tn(W, X, ws, t, nullptr, t, splits, s);
  if (e == cudaSuccess && z > 1) {
    const size_t n = static_cast<size_t>(t) * n_out;
    sum_splits_kernel<<<static_cast<int>((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0, s>>>(ws, out, z, n);
    e = cudaGetLastError();
  }
  if (z > 1) cudaFreeAsync(ws, s);
  return e == cudaSuccess ? FASER_OK : FASER_ECUDA;
}
