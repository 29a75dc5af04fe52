// kapi.cu — kernel-level C ABI (include/faser/kernels.h): thin wrappers that validate
// arguments and call the same launchers the engine uses.
#include <cuda_runtime.h>

#include <string>

#include "faser/kernels.h"
#include "llama.cuh"
#include "tc_gemm.cuh"

namespace faser {
namespace {

__global__ void iota_kernel(int* a, int n, int* n_rows, int total) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
  if (i == 0) *n_rows = total;
}

int num_sms() {
  static const int n = [] {  // thread-safe one-time init (TP ranks call from several threads)
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v ? v : 148;
  }();
  return n;
}

}  // namespace
}  // namespace faser

using namespace faser;

extern "C" faser_status faser_k_gemm_bf16_trace(const void* w, const void* x, float* out, int32_t n_out,
                                                int32_t t, int32_t k, int32_t bn, int32_t splits, void* stream,
                                                unsigned long long* trace);

extern "C" faser_status faser_k_gemm_bf16_plan(const void* w, const void* x, float* out, int32_t n_out,
                                               int32_t t, int32_t k, int32_t bn, int32_t splits,
                                               void* stream) {
  return faser_k_gemm_bf16_trace(w, x, out, n_out, t, k, bn, splits, stream, nullptr);
}

extern "C" faser_status faser_k_gemm_bf16_trace(const void* w, const void* x, float* out, int32_t n_out,
                                                int32_t t, int32_t k, int32_t bn, int32_t splits, void* stream,
                                                unsigned long long* trace) {
  // bn may carry a pipeline-depth request in its upper bits: 1000 + bn = shallow, 2000 + bn = deep
  // bn may carry requests in its upper digits: 10000 * mc + 1000 * depth + bn
  const int mc = bn / 10000;
  bn %= 10000;
  int depth = bn / 1000;
  bn %= 1000;
  if (mc != 0 && mc != 1 && mc != 2 && mc != 4) return FASER_EINVAL;
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
  if (mc > 0) plan.mc = mc;
  if ((plan.bn > 128 && plan.mc > 2) || plan.mc * plan.bn > 512) plan.mc = 1;  // instantiated combinations / TMEM
  if (plan.mc > 1) plan.deep = true;
  if (depth == 1 && plan.mc == 1) plan.deep = false;
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
  ea.trace = trace;
  cudaError_t e = gemm_fused(W, X, t, plan, ea, s);
  return e == cudaSuccess ? FASER_OK : FASER_ECUDA;
}

extern "C" faser_status faser_k_gemm_plan_table(int32_t n_out, int32_t t, int32_t k, int32_t* out4, double* score) {
  if (!out4 || n_out <= 0 || n_out % 128 || t <= 0 || k <= 0 || k % 64) return FASER_EINVAL;
  const GemmPlan p = gemm_plan_table(n_out, t, k, score);
  out4[0] = p.bn;
  out4[1] = p.splits;
  out4[2] = p.mc;
  out4[3] = p.deep ? 1 : 0;
  return FASER_OK;
}

extern "C" faser_status faser_k_gemm_plan(int32_t n_out, int32_t t, int32_t k, int32_t* out4) {
  if (!out4 || n_out <= 0 || n_out % 128 || t <= 0 || k <= 0 || k % 64) return FASER_EINVAL;
  int n = 0, dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
    n = 148;
  cudaGetLastError();
  const GemmPlan p = gemm_plan(n_out, t, k, n);
  out4[0] = p.bn;
  out4[1] = p.splits;
  out4[2] = p.mc;
  out4[3] = p.deep ? 1 : 0;
  return FASER_OK;
}

extern "C" faser_status faser_k_gemm_bf16(const void* w, const void* x, float* out, int32_t n_out,
                                          int32_t t, int32_t k, int32_t splits, void* stream) {
  return faser_k_gemm_bf16_plan(w, x, out, n_out, t, k, 0, splits, stream);
}

extern "C" faser_status faser_k_attention(const void* q, const void* kv, const int32_t* ptab, int32_t max_pages,
                                          int32_t n_req, const int32_t* req_first, const int32_t* req_n,
                                          const int32_t* req_pos0, int32_t max_rows, int32_t max_ctx,
                                          int32_t n_q, int32_t n_kv, int32_t hd, void* out, void* scratch,
                                          int64_t scratch_bytes, void* stream) {
  if (!q || !kv || !ptab || !req_first || !req_n || !req_pos0 || !out || !scratch) return FASER_EINVAL;
  if (n_req <= 0 || max_rows <= 0 || n_q <= 0 || n_kv <= 0 || n_q % n_kv || (hd != 64 && hd != 128) ||
      scratch_bytes < (int64_t(2) << 20))
    return FASER_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return FASER_ECUDA;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // request i's slot (page-table row) is i; n_rows is unused by the kernel but kept valid.
  // Per host thread (thread_local): concurrent callers never share or free each other's buffer.
  thread_local int* d_slot = nullptr;
  thread_local int cap = 0;
  if (n_req + 1 > cap) {
    if (d_slot) cudaFree(d_slot);
    cap = n_req + 1 > 4096 ? n_req + 1 : 4096;
    if (cudaMalloc(&d_slot, sizeof(int) * cap) != cudaSuccess) return FASER_ENOMEM;
  }
  iota_kernel<<<(n_req + 255) / 256, 256, 0, s>>>(d_slot, n_req, d_slot + n_req, max_rows * n_req);
  LlamaShape m{};
  m.n_q = n_q;
  m.n_kv = n_kv;
  m.hd = hd;
  RowsDev rows{};
  rows.n_rows = d_slot + n_req;
  rows.req_first = const_cast<int*>(req_first);
  rows.req_n = const_cast<int*>(req_n);
  rows.req_slot = d_slot;
  rows.req_pos0 = const_cast<int*>(req_pos0);
  KvDev kvd{};
  kvd.pool = static_cast<__nv_bfloat16*>(const_cast<void*>(kv));
  kvd.ptab = ptab;
  kvd.max_pages = max_pages;
  kvd.layer_stride = 0;
  // TMA view of the pool (the engine's default page path): the pool holds at least
  // n_req * max_pages pages (request i's table row is i)
  GemmOperand kv_op;
  const int64_t kv_rows = static_cast<int64_t>(n_req) * max_pages * n_kv * 2 * 64;
  if (kv_rows < (int64_t(1) << 31) && make_operand(&kv_op, kv, static_cast<int>(kv_rows), hd, 64) == cudaSuccess)
    kvd.tma = &kv_op.map;
  cudaError_t e = lm_attention(m, rows, n_req, max_rows, max_ctx, kvd, 0, static_cast<const __nv_bfloat16*>(q),
                               static_cast<__nv_bfloat16*>(out), static_cast<float*>(scratch),
                               static_cast<size_t>(scratch_bytes), s);
  return e == cudaSuccess ? FASER_OK : FASER_ECUDA;
}
