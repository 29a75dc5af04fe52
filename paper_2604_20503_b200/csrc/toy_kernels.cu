// toy_kernels.cu — sm_100a kernels for the toy-model speculative-decoding path.
//
// K0: toy logits (SplitMix64 hash per vocab entry), interpolated intermediate logits, argmax
//     with lowest-id ties, and the rank-count exit test — replaces toylm.cpp:9-101 and
//     exitctl.cpp:56-68. INT64-ALU bound: no HBM traffic beyond token ids and hash states.
// K5: fused greedy acceptance + early-exit frontier scan + commit + state rollback —
//     replaces sdcore.cpp:61-197.
//
// Bit-exactness rules: all double arithmetic uses explicit _rn
// intrinsics so nvcc cannot contract w*zf + (1-w)*zn into an FMA (the x86-64 reference build
// has no FMA); u64 -> double conversion of a 53-bit value and the 2^-53 scale are exact.
#include <cstdint>

#include "toy_kernels.cuh"

namespace faser {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;

// rng.hpp:17-22
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += kGamma;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
// rng.hpp:24-26
__device__ __forceinline__ uint64_t hash_combine(uint64_t h, uint64_t v) {
  return mix64(h ^ (v + kGamma + (h << 6) + (h >> 2)));
}
// rng.hpp:35-37 (exact: 53-bit integer -> double, times a power of two)
__device__ __forceinline__ double to_unit(uint64_t h) {
  return __dmul_rn(__ull2double_rn(h >> 11), 0x1.0p-53);
}

// Argmax over (value, index) pairs held across the warp; ties -> lowest index
// (argmax_lowest, toylm.cpp:9-16: strict '>' scan keeps the first maximum).
__device__ __forceinline__ void warp_argmax(double& v, int& i) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(kFull, v, o);
    const int oi = __shfl_xor_sync(kFull, i, o);
    if (ov > v || (ov == v && oi < i)) {
      v = ov;
      i = oi;
    }
  }
}

// Context hash over the last `order` tokens of a prefix of length `plen`, where positions
// < base come from `row` and positions >= base from `tail` (toylm.cpp:29-40).
__device__ __forceinline__ uint64_t context_hash(const ToyDev& m, const int32_t* row, int base,
                                                 const int32_t* tail, int plen) {
  uint64_t h = mix64(m.table_seed);
  for (int q = m.order; q >= 1; --q) {
    const int pos = plen - q;
    const int tok = pos < 0 ? m.vocab : (pos < base ? row[pos] : tail[pos - base]);
    h = hash_combine(h, static_cast<uint64_t>(static_cast<int64_t>(tok)) + 1);
  }
  return h;
}

// Lane-strided logits: lane holds t = lane + 32*q for q < VPL.
template <int VPL>
__device__ __forceinline__ void logits(const ToyDev& m, uint64_t ch, uint64_t nh, bool want_noise,
                                       double (&zf)[VPL], double (&zn)[VPL]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < VPL; ++q) {
    const int t = lane + 32 * q;
    zf[q] = 0.0;
    zn[q] = 0.0;
    if (t < m.vocab) {
      zf[q] = __dmul_rn(to_unit(hash_combine(ch, static_cast<uint64_t>(t) + 1)), m.logit_scale);
      if (want_noise)
        zn[q] = __dmul_rn(to_unit(hash_combine(nh, static_cast<uint64_t>(t) + 1)), m.noise_scale);
    }
  }
}

template <int VPL>
__device__ __forceinline__ int argmax_of(const ToyDev& m, const double (&z)[VPL]) {
  const int lane = threadIdx.x & 31;
  double bv = -1.0;  // logits are >= 0
  int bi = 0x7fffffff;
#pragma unroll
  for (int q = 0; q < VPL; ++q) {
    const int t = lane + 32 * q;
    if (t < m.vocab && z[q] > bv) {  // increasing t: strict '>' keeps the lowest id
      bv = z[q];
      bi = t;
    }
  }
  warp_argmax(bv, bi);
  return bi;
}

// token_exit_test (exitctl.cpp:56-68) on z = w*zf + (1-w)*zn at `layer`:
// prune iff #{v : z[v] > z[d] or (z[v] == z[d] and v < d)} >= k.
// w = layer / L and 1 - w come from a per-block table (layer_weights): the same correctly
// rounded quotient target_logits forms (toylm.cpp:60), computed once instead of per row.
// z[d] is formed by every lane from the row's (zf[d], zn[d]) (broadcast once per row) with the
// same rounded operations lane d % 32 applies to its own entry, so it is bit-identical to it;
// the count is one ballot per vocab stripe.
template <int VPL>
__device__ __forceinline__ bool exit_test(const ToyDev& m, const double (&zf)[VPL], const double (&zn)[VPL],
                                          double zf_d, double zn_d, double w, double omw, int d, int k) {
  const int lane = threadIdx.x & 31;
  const double ref = __dadd_rn(__dmul_rn(w, zf_d), __dmul_rn(omw, zn_d));
  int cnt = 0;
#pragma unroll
  for (int q = 0; q < VPL; ++q) {
    const int t = lane + 32 * q;
    const double z = __dadd_rn(__dmul_rn(w, zf[q]), __dmul_rn(omw, zn[q]));
    cnt += __popc(__ballot_sync(kFull, (t < m.vocab) && (z > ref || (z == ref && t < d))));
  }
  return cnt >= k;
}
// tab[l] = (l / L, 1 - l / L) for l in [lo, hi), by the block's threads (needs a __syncthreads)
__device__ __forceinline__ void layer_weights(const ToyDev& m, int lo, int hi, double2* tab) {
  for (int l = lo + static_cast<int>(threadIdx.x); l < hi; l += blockDim.x) {
    const double w = __ddiv_rn(static_cast<double>(l), static_cast<double>(m.layers));
    tab[l] = make_double2(w, __dsub_rn(1.0, w));
  }
}

// ----------------------------------------------------------------------------- admit
// One warp per admitted request: copy its context into the slot row and fold the running
// hash states hash_tokens(noise_seed, ctx) / hash_tokens(mix_seed, ctx) (rng.hpp:28-32).
__device__ __forceinline__ void admit_one(const ToyDev& m, SlotState st, const AdmitEntry& a) {
  const int lane = threadIdx.x & 31;
  const int32_t* src = a.src;
  int32_t* row = st.tok + static_cast<int64_t>(a.slot) * st.max_seq;
  for (int i = lane; i < a.len; i += 32) row[i] = src[i];
  if (lane < 2) {
    uint64_t h = mix64(lane == 0 ? m.noise_seed : m.mix_seed);
    for (int i = 0; i < a.len; ++i)
      h = hash_combine(h, static_cast<uint64_t>(static_cast<int64_t>(src[i])) + 1);
    (lane == 0 ? st.nh : st.mh)[a.slot] = h;
  }
  if (lane == 0) {
    st.len[a.slot] = a.len;
    st.ncomm[a.slot] = a.ncomm;
    st.max_out[a.slot] = a.max_out;
    st.done[a.slot] = 0;
    st.exempt[a.slot] = a.exempt;
  }
}

__global__ void admit_kernel(ToyDev m, SlotState st, const StepIn* __restrict__ in) {
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (e >= in->n_admit) return;
  admit_one(m, st, in->admit()[e]);
}

// ----------------------------------------------------------------------------- draft
// SpeculativeEngine::draft_tokens (sdcore.cpp:45-59): one warp per live request, up to
// min(k_i, remaining) sequential draft_next steps (toylm.cpp:76-85), EOS stop. The mix-hash
// state after every drafted token is kept (mh_at) so commit can roll back in O(1).
template <int VPL>
__device__ __forceinline__ void draft_one(const ToyDev& m, SlotState st, const StepIn* __restrict__ in, int p,
                                          int32_t* dl) {
  const int lane = threadIdx.x & 31;
  const int slot = in->live_slot()[p];
  const int32_t* row = st.tok + static_cast<int64_t>(slot) * st.max_seq;
  const int base = st.len[slot];
  const int remaining = st.max_out[slot] - st.ncomm[slot];
  int budget = in->k()[p] < remaining ? in->k()[p] : remaining;
  if (budget > FASER_MAX_SPEC) budget = FASER_MAX_SPEC;
  uint64_t mh = st.mh[slot];
  uint64_t* mh_at = st.mh_at + static_cast<int64_t>(slot) * (FASER_MAX_SPEC + 1);
  int32_t* dout = st.draft + static_cast<int64_t>(slot) * FASER_MAX_SPEC;
  if (lane == 0) mh_at[0] = mh;
  int n = 0;
  for (int i = 0; i < budget; ++i) {
    const double u = to_unit(mh);
    int t = 0;
    if (!(u < m.divergence)) {
      const uint64_t ch = context_hash(m, row, base, dl, base + i);
      double zf[VPL], zn[VPL];
      logits<VPL>(m, ch, 0, false, zf, zn);
      t = argmax_of<VPL>(m, zf);
    }
    if (lane == 0) {
      dl[i] = t;
      dout[i] = t;
    }
    __syncwarp();
    mh = hash_combine(mh, static_cast<uint64_t>(t) + 1);
    if (lane == 0) mh_at[i + 1] = mh;
    ++n;
    if (t == m.eos) break;
  }
  if (lane == 0) st.draft_len[slot] = n;
}

template <int VPL>
__global__ void __launch_bounds__(128) draft_kernel(ToyDev m, SlotState st,
                                                    const StepIn* __restrict__ in) {
  __shared__ int32_t dl[4][FASER_MAX_SPEC];
  const int wib = threadIdx.x >> 5;
  const int p = blockIdx.x * 4 + wib;
  if (p >= in->n_live) return;
  draft_one<VPL>(m, st, in, p, dl[wib]);
}

// ----------------------------------------------------------------------------- verify
// Fused verify(+early exit) + accept + commit, one CTA per live request, warps over drafted
// positions (sdcore.cpp:61-197). Phase 1 (parallel): per position j the target logits, the
// target argmax and — for every gated layer — the exit-test bit. Phase 2 (thread 0): the
// reference's sequential frontier scan over those bits, acceptance, force-verify, commit.
constexpr int kVerifyWarps = 8;

struct VerifySmem {
  int32_t d[FASER_MAX_SPEC];
  int32_t truth[FASER_MAX_SPEC];
  uint32_t failpos[FASER_MAX_LAYERS + 1];
  uint64_t nh_at[FASER_MAX_SPEC + 1];
  double2 wt[FASER_MAX_LAYERS + 1];  // (l / L, 1 - l / L)
};

// request p's verify + commit by the whole block (kVerifyWarps warps); the block's draft for p,
// when fused, was written by warp 0 before the block barrier this starts with
template <int VPL>
__device__ __forceinline__ void verify_one(const ToyDev& m, SlotState st, const StepIn* __restrict__ in, int p,
                                           faser_round_result* __restrict__ results, VerifySmem& sm) {
  int32_t* d = sm.d;
  int32_t* truth = sm.truth;
  uint32_t* failpos = sm.failpos;
  uint64_t* nh_at = sm.nh_at;
  const int slot = in->live_slot()[p];
  const int count = st.draft_len[slot];
  const int base = st.len[slot];
  const int ncomm0 = st.ncomm[slot];
  const int exempt = st.exempt[slot];
  const int32_t* row = st.tok + static_cast<int64_t>(slot) * st.max_seq;
  const bool ee = in->early_exit != 0;
  const int lo = in->gate_lo, hi = in->gate_hi;
  for (int j = threadIdx.x; j < count; j += blockDim.x)
    d[j] = st.draft[static_cast<int64_t>(slot) * FASER_MAX_SPEC + j];
  for (int l = threadIdx.x; l <= FASER_MAX_LAYERS; l += blockDim.x) failpos[l] = 0u;
  if (ee) layer_weights(m, lo, hi, sm.wt);
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < count; j += kVerifyWarps) {
    uint64_t nh = st.nh[slot];
    for (int i = 0; i < j; ++i) nh = hash_combine(nh, static_cast<uint64_t>(d[i]) + 1);
    if (lane == 0) {
      nh_at[j] = nh;
      if (j == count - 1) nh_at[count] = hash_combine(nh, static_cast<uint64_t>(d[j]) + 1);
    }
    const uint64_t ch = context_hash(m, row, base, d, base + j);
    double zf[VPL], zn[VPL];
    logits<VPL>(m, ch, nh, ee, zf, zn);
    const int tj = argmax_of<VPL>(m, zf);
    if (lane == 0) truth[j] = tj;
    if (ee && ncomm0 + j != exempt) {  // one-round re-entry exemption (sdcore.cpp:118-119)
      const int dj = d[j];
      double zf_d = zf[0], zn_d = zn[0];
#pragma unroll
      for (int q = 1; q < VPL; ++q)
        if (q == (dj >> 5)) {
          zf_d = zf[q];
          zn_d = zn[q];
        }
      zf_d = __shfl_sync(kFull, zf_d, dj & 31);
      zn_d = __shfl_sync(kFull, zn_d, dj & 31);
#pragma unroll 2
      for (int l = lo; l < hi; ++l) {
        if (exit_test<VPL>(m, zf, zn, zf_d, zn_d, sm.wt[l].x, sm.wt[l].y, dj, in->k_table[l]) && lane == 0)
          atomicOr(&failpos[l], 1u << j);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;

  // ---- phase 2: reference control flow (sdcore.cpp:111-180) on the computed bits
  const int L = m.layers;
  faser_round_result* rr = results + p;
  faser_verify_outcome& o = rr->outcome;
  int prune_layer[FASER_MAX_SPEC];
  int active = count;
  for (int j = 0; j < count; ++j) prune_layer[j] = L;
  int gate_layers = 0, n_pl = 0, pr_j = -1, pr_l = -1;
  bool pruned = false;
  if (ee) {
    for (int l = lo; l < hi && active > 0; ++l) {
      ++gate_layers;
      const uint32_t live = active >= 32 ? 0xffffffffu : ((1u << active) - 1u);
      const uint32_t f = failpos[l] & live;
      if (f) {
        const int j = __ffs(f) - 1;
        for (int jj = j; jj < active; ++jj) prune_layer[jj] = l;
        active = j;
        pruned = true;
        pr_j = j;
        pr_l = l;
        o.prune_layers[n_pl++] = l;
      }
    }
  }
  int acc = 0, rec = -1;
  bool mismatch = false;
  for (int j = 0; j < active; ++j) {
    if (d[j] == truth[j]) {
      ++acc;
    } else {
      rec = truth[j];
      mismatch = true;
      break;
    }
  }
  if (ee && active == 0) {  // progress guarantee: force-verify token 0 (sdcore.cpp:150-166)
    if (d[0] == truth[0]) {
      acc = 1;
    } else {
      rec = truth[0];
      mismatch = true;
    }
    if (count > 1) {
      pr_j = 1;
      pr_l = prune_layer[1];
    } else {
      pruned = false;
      pr_j = pr_l = -1;
    }
    active = 1;
  }
  double flr = 0.0;
  if (ee) {
    for (int j = 0; j < count; ++j) flr += (j < active) ? L : prune_layer[j];
  } else {
    flr = static_cast<double>(L) * count;
  }
  int false_prune = 0;
  if (pruned && !mismatch && acc == pr_j && pr_j < count) false_prune = (d[pr_j] == truth[pr_j]);

  o.submitted = count;
  o.accepted_count = acc;
  o.has_recovery = rec >= 0;
  o.recovery_token = rec;
  o.has_pruned = pruned;
  o.pruned_index = pruned ? pr_j : -1;
  o.pruned_layer = pruned ? pr_l : -1;
  o.gate_layers = gate_layers;
  o.full_layers_run = flr;
  o.false_prune = false_prune;
  o.n_prune_layers = n_pl;
  o.base_len = base;
  rr->req_id = in->req_id()[p];
  rr->spec_length = in->k()[p];
  rr->drafted = count;

  // ---- commit (sdcore.cpp:182-197) + O(1) state rollback to the committed length
  int c = 0;
  if (in->commit) {
    int done = st.done[slot];
    int nc = ncomm0;
    const int mo = st.max_out[slot];
    int32_t* out_row = st.tok + static_cast<int64_t>(slot) * st.max_seq + base;
    for (int j = 0; j < acc && !done; ++j) {
      out_row[c] = d[j];
      rr->tokens[c++] = d[j];
      ++nc;
      if (d[j] == m.eos || nc == mo) done = 1;
    }
    bool rec_committed = false;
    if (rec >= 0 && !done) {
      out_row[c] = rec;
      rr->tokens[c++] = rec;
      ++nc;
      rec_committed = true;
      if (rec == m.eos || nc == mo) done = 1;
    }
    const uint64_t* mh_at = st.mh_at + static_cast<int64_t>(slot) * (FASER_MAX_SPEC + 1);
    const int keep = rec_committed ? acc : c;  // drafted prefix kept
    uint64_t nh = nh_at[keep], mh = mh_at[keep];
    if (rec_committed) {
      nh = hash_combine(nh, static_cast<uint64_t>(rec) + 1);
      mh = hash_combine(mh, static_cast<uint64_t>(rec) + 1);
    }
    st.nh[slot] = nh;
    st.mh[slot] = mh;
    st.len[slot] = base + c;
    st.ncomm[slot] = nc;
    st.done[slot] = done;
    int ex = exempt;
    if (in->exempt_rule) ex = pruned ? ncomm0 + pr_j : -1;
    st.exempt[slot] = ex;
    rr->done = done;
    rr->exempt_position = ex;
    rr->n_committed_total = nc;
  }
  if (!in->commit) {
    rr->done = st.done[slot];
    rr->exempt_position = exempt;
    rr->n_committed_total = ncomm0;
  }
  rr->committed = c;
}

template <int VPL>
__global__ void __launch_bounds__(kVerifyWarps * 32) verify_kernel(ToyDev m, SlotState st,
                                                                   const StepIn* __restrict__ in,
                                                                   faser_round_result* __restrict__ results) {
  __shared__ VerifySmem sm;
  const int p = blockIdx.x;
  if (p >= in->n_live) return;
  verify_one<VPL>(m, st, in, p, results, sm);
}

// One launch per round: block p admits (when new) and drafts request p on warp 0 (the other
// warps wait at the barrier) and then verifies + commits it with all warps — no grid-wide draft/verify boundary,
// so a request with a short draft starts verifying while others still draft.
template <int VPL>
__global__ void __launch_bounds__(kVerifyWarps * 32) draft_verify_kernel(ToyDev m, SlotState st,
                                                                         const StepIn* __restrict__ in,
                                                                         faser_round_result* __restrict__ results) {
  __shared__ VerifySmem sm;
  __shared__ int32_t dl[FASER_MAX_SPEC];
  const int p = blockIdx.x;
  if (p >= in->n_live) return;
  if (threadIdx.x < 32) {
    // a request admitted this round: its slot state first (admit_kernel's work, same warp)
    const int slot = in->live_slot()[p];
    for (int e = 0; e < in->n_admit; ++e)
      if (in->admit()[e].slot == slot) admit_one(m, st, in->admit()[e]);
    __syncwarp();
    draft_one<VPL>(m, st, in, p, dl);
  }
  __syncthreads();  // the draft (global st.draft / draft_len / mh_at) is visible block-wide
  verify_one<VPL>(m, st, in, p, results, sm);
}

// ----------------------------------------------------------------------------- rows
template <int VPL>
__global__ void __launch_bounds__(128) rows_kernel(ToyDev m, int op, int n,
                                                   const int32_t* __restrict__ tokens,
                                                   const int64_t* __restrict__ off,
                                                   const int32_t* __restrict__ layers, double* z0,
                                                   double* z1, int32_t* out) {
  const int r = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  const int32_t* row = tokens + off[r];
  const int len = static_cast<int>(off[r + 1] - off[r]);
  uint64_t nh = mix64(m.noise_seed), mh = mix64(m.mix_seed);
  for (int i = 0; i < len; ++i) {
    const uint64_t v = static_cast<uint64_t>(static_cast<int64_t>(row[i])) + 1;
    nh = hash_combine(nh, v);
    mh = hash_combine(mh, v);
  }
  if (op == 3 && to_unit(mh) < m.divergence) {
    if (lane == 0) out[r] = 0;
    return;
  }
  const uint64_t ch = context_hash(m, row, len, nullptr, len);
  double zf[VPL], zn[VPL];
  logits<VPL>(m, ch, nh, op <= 1, zf, zn);
  if (op >= 2) {
    const int t = argmax_of<VPL>(m, zf);
    if (lane == 0) out[r] = t;
    return;
  }
  const int64_t ob = static_cast<int64_t>(r) * m.vocab;
  const int layer = op == 1 ? layers[r] : m.layers;
  const double w = __ddiv_rn(static_cast<double>(layer), static_cast<double>(m.layers));
  const double omw = __dsub_rn(1.0, w);
#pragma unroll
  for (int q = 0; q < VPL; ++q) {
    const int t = lane + 32 * q;
    if (t >= m.vocab) continue;
    if (op == 0) {
      z0[ob + t] = zf[q];
      z1[ob + t] = zn[q];
    } else {
      z0[ob + t] = layer == m.layers ? zf[q] : __dadd_rn(__dmul_rn(w, zf[q]), __dmul_rn(omw, zn[q]));
    }
  }
}

}  // namespace

bool toy_vocab_supported(int vocab) { return vocab >= 2 && vocab <= 256; }

#define FASER_VPL_SWITCH(vocab, CALL) \
  do {                                \
    const int vpl_ = ((vocab) + 31) / 32; \
    if (vpl_ <= 1) { constexpr int VPL = 1; CALL; }      \
    else if (vpl_ <= 2) { constexpr int VPL = 2; CALL; } \
    else if (vpl_ <= 4) { constexpr int VPL = 4; CALL; } \
    else { constexpr int VPL = 8; CALL; }                \
  } while (0)

cudaError_t toy_admit(const ToyDev& m, SlotState st, const StepIn* in_dev, int n_admit,
                      cudaStream_t stream) {
  if (n_admit <= 0) return cudaSuccess;
  admit_kernel<<<(n_admit + 3) / 4, 128, 0, stream>>>(m, st, in_dev);
  return cudaGetLastError();
}

cudaError_t toy_draft(const ToyDev& m, SlotState st, const StepIn* in_dev, int n_live,
                      cudaStream_t stream) {
  if (n_live <= 0) return cudaSuccess;
  FASER_VPL_SWITCH(m.vocab, (draft_kernel<VPL><<<(n_live + 3) / 4, 128, 0, stream>>>(m, st, in_dev)));
  return cudaGetLastError();
}

cudaError_t toy_verify_commit(const ToyDev& m, SlotState st, const StepIn* in_dev, int n_live,
                              faser_round_result* results, cudaStream_t stream) {
  if (n_live <= 0) return cudaSuccess;
  FASER_VPL_SWITCH(m.vocab, (verify_kernel<VPL><<<n_live, kVerifyWarps * 32, 0, stream>>>(
                                m, st, in_dev, results)));
  return cudaGetLastError();
}

cudaError_t toy_draft_verify_commit(const ToyDev& m, SlotState st, const StepIn* in_dev, int n_live,
                                    faser_round_result* results, cudaStream_t stream) {
  if (n_live <= 0) return cudaSuccess;
  FASER_VPL_SWITCH(m.vocab, (draft_verify_kernel<VPL><<<n_live, kVerifyWarps * 32, 0, stream>>>(
                                m, st, in_dev, results)));
  return cudaGetLastError();
}

cudaError_t toy_rows(const ToyDev& m, int op, int n, const int32_t* tokens, const int64_t* off,
                     const int32_t* layers, double* z0, double* z1, int32_t* out,
                     cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  FASER_VPL_SWITCH(m.vocab, (rows_kernel<VPL><<<(n + 3) / 4, 128, 0, stream>>>(
                                m, op, n, tokens, off, layers, z0, z1, out)));
  return cudaGetLastError();
}

}  // namespace faser
