// lanes.cuh — SM-partitioned execution lanes for the overlapped (FULL) mode: a pool of CUDA
// green-context pairs, one pair per draft SM share, each pair = a draft partition of
// round8(r * SMs) SMs and a verify partition of the remaining SMs, with one stream in each.
//
// This is the real counterpart of the reference's abstract SM split: OverlapPlan.r is the
// draft-side share (overlap.hpp:11-17) and the latency models evaluate the draft stage at share r
// and the target stage at 1 - r (latmodel.cpp:32-62). The paper provisions the same pool with
// cuda-python Green Contexts. Partitions come in multiples of 8 SMs on sm_90+
// (cuda.h, cuDevSmResourceSplitByCount), so r is quantised; `LanePair` reports the SM counts the
// driver actually provisioned.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <mutex>
#include <string>

namespace faser {

struct LanePair {
  cudaStream_t draft = nullptr;   // stream in the draft partition
  cudaStream_t verify = nullptr;  // stream in the verify partition
  int draft_sms = 0, verify_sms = 0;
  bool green = false;             // false: plain streams sharing every SM (FASER_GREEN=0 / unsupported)
};

class SmLanes {
 public:
  SmLanes(int device, int total_sms);
  ~SmLanes();
  SmLanes(const SmLanes&) = delete;
  SmLanes& operator=(const SmLanes&) = delete;
  // The pair for draft share r in (0, 1). Created on first use and cached by its draft SM count.
  // Returns false (with *err) if the driver refuses the partition.
  bool get(double r, LanePair* out, std::string* err);
  // SM count the draft partition of share r gets (multiple of 8, at least 8, leaves >= 8).
  int draft_sms_for(double r) const;
  bool green_available() const { return green_ok_; }
  int total_sms() const { return total_; }

 private:
  struct Pair;
  int device_ = 0, total_ = 148;
  bool green_ok_ = false;
  std::mutex mu_;
  std::map<int, std::unique_ptr<Pair>> pairs_;
};

}  // namespace faser
