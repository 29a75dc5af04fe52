// tc_gemm.cuh — host interface of the tcgen05 swap-AB GEMM (see tc_gemm.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace faser {

// A bf16 row-major [rows][k] matrix with its TMA descriptor (SWIZZLE_128B, box 64 x box_rows).
struct GemmOperand {
  CUtensorMap map;
  const void* base = nullptr;
  int rows = 0;
  int k = 0;
};

cudaError_t make_weight_operand(GemmOperand* op, const void* w, int n_out, int k);  // box 128 rows
cudaError_t make_act_operand(GemmOperand* op, const void* x, int rows_cap, int k);  // box 32 rows

// Tile width along tokens and the K split a launch over T rows will use.
int gemm_bn_for(int t);
int gemm_splits_for(int n_out, int t, int k, int num_sms);
int gemm_effective_splits(int k, int splits);

// ws[z][t][n] (z < effective splits, t < T, row stride n_out, split stride t_stride*n_out)
// = partial of sum_k W[n][k] X[t][k]. T = min(*t_dev, t) when t_dev != nullptr.
cudaError_t gemm_tn(const GemmOperand& w, const GemmOperand& x, float* ws, int t_stride,
                    const int* t_dev, int t, int splits, cudaStream_t s);

}  // namespace faser
