// tp.cuh — tensor-parallel verification of the largest target (config 5).
//
// Megatron split of the target across a TP group: QKV and gate/up column-parallel (each rank
// owns n_q/tp query heads, n_kv/tp KV heads and ffn/tp FFN rows), O and down row-parallel
// (each rank produces a partial [T][d] that is all-reduced before the residual add), LM head
// vocab-parallel (each rank scores V/tp tokens; greedy argmax = all-gather of every rank's
// per-row (max, lowest global id) and a lowest-id-on-ties merge, so all ranks agree bit-exactly).
// The draft model is replicated (deterministic kernels: every rank drafts the same tokens).
//
// Two collective backends behind one interface:
//   NCCL  : one process per GPU, ncclAllReduce / ncclAllGather over NVLink/NVSwitch (libnccl
//           is dlopen'ed, so the product library has no link-time NCCL dependency);
//   LOCAL : all ranks are threads of one process on ONE device (test/emulation backend):
//           host barriers + cross-stream events, and a rank-ordered device sum over the ranks'
//           buffers (same address space). Used to validate the sharded math on a 1-GPU box.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace faser {

class TpGroup {
 public:
  virtual ~TpGroup() = default;
  int size = 1;
  // in place: buf = sum over ranks of buf (bf16 partials, n elements: half the bytes of fp32 on
  // NVLink); stream-ordered
  virtual cudaError_t allreduce_sum(int rank, __nv_bfloat16* buf, size_t n, cudaStream_t s) = 0;
  // out[r * n + i] = in_r[i] for every rank r (float2 elements); stream-ordered
  virtual cudaError_t allgather_f2(int rank, const float2* in, float2* out, size_t n, cudaStream_t s) = 0;
  virtual const char* backend() const = 0;
};

TpGroup* tp_local_group_create(int size);
// id = 128-byte ncclUniqueId; returns nullptr (and sets *err) on failure
TpGroup* tp_nccl_group_create(const uint8_t* id, int size, int rank, int device, const char** err);
bool tp_nccl_unique_id(uint8_t* out, const char** err);

// x += part; xb = bf16(x); ss[c][t] = sum of squares of 128-column chunk c (row-parallel epilogue
// after the all-reduce), rows [0, T) of width d.
cudaError_t tp_resid_add(const __nv_bfloat16* part, float* x, __nv_bfloat16* xb, float* ss, int T, int d, cudaStream_t s);
// per-row local (max, lowest global id) over this rank's vocab tiles -> loc[T]
cudaError_t tp_local_argmax(int n_tiles, int T, const float2* amax, float2* loc, cudaStream_t s);
// merge the gathered [tp][T] partials: out[t] = lowest id among the maxima
cudaError_t tp_merge_argmax(int tp, int T, const float2* all, int* out, cudaStream_t s);

}  // namespace faser
struct faser_tp_group;
namespace faser {
TpGroup* tp_group_of(faser_tp_group* g);

}  // namespace faser
