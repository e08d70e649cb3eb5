// Internal plumbing shared by the C ABI translation units (capi.cpp: model,
// cluster, planning, memory, weights, barrier; capi_exec.cpp: the executor).
// No exception crosses the ABI: every entry point runs its body in
// rr::capi::guarded(), which maps exceptions to rr_status + rr_last_error().
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "rlplan/realloc.hpp"
#include "rr_realloc.h"

namespace rr {
std::string& last_error_slot();  // thread-local message behind rr_last_error()

namespace capi {

using namespace rlplan;
struct StatusError {
  rr_status status;
  std::string message;
};

[[noreturn]] inline void raise(rr_status s, const std::string& msg) { throw StatusError{s, msg}; }

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(RR_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
inline void check_cuda(int e, const char* what) { check_cuda(static_cast<cudaError_t>(e), what); }

template <class F>
rr_status guarded(F&& f) {
  try {
    f();
    return RR_OK;
  } catch (const StatusError& e) {
    last_error_slot() = e.message;
    return e.status;
  } catch (const ValidationError& e) {
    last_error_slot() = e.what();
    return RR_EINVAL;
  } catch (const std::bad_alloc&) {
    last_error_slot() = "out of host memory";
    return RR_ENOMEM;
  } catch (const std::exception& e) {
    last_error_slot() = e.what();
    return RR_EINVAL;
  }
}

inline void need(bool ok, const char* what) {
  if (!ok) raise(RR_EINVAL, what);
}

}  // namespace capi
}  // namespace rr

// ---------------------------------------------------------------------------
// Plan object
// ---------------------------------------------------------------------------

struct rr_plan {
  rlplan::ModelSpec model;
  rlplan::Placement src, dst;
  rlplan::ClusterSpec cluster;
  rlplan::ReallocPlan plan;
  std::vector<std::vector<int32_t>> remote_dst, local_dst;  // int32 copies for rr_op
  std::vector<rlplan::LoweredOp> lowered;
  mutable std::map<std::pair<int, rlplan::DeviceId>, rlplan::ShardLayout> layouts;
  mutable std::mutex mu;  // guards lazily built layouts
  bool data = false;  // inter-call data transfer plan (plan_data_transfer)
  rlplan::Bytes data_total = 0;  // its total data bytes

  const rlplan::ShardLayout& layout(int side, rlplan::DeviceId d) const {
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_pair(side, d);
    auto it = layouts.find(key);
    if (it == layouts.end()) {
      rlplan::ShardLayout lay = data ? rlplan::data_layout(side ? dst : src, cluster, d, data_total, side == 0)
                                     : rlplan::shard_layout(model, side ? dst : src, cluster, d);
      it = layouts.emplace(key, std::move(lay)).first;
    }
    return it->second;
  }

  // Logical width of a tensor (for the weight value function's index).
  std::vector<rlplan::Count> tensor_cols() const {
    std::vector<rlplan::Count> cols;
    if (!data)
      for (const auto& t : rlplan::tensor_inventory(model)) cols.push_back(t.cols);
    return cols;
  }
  rlplan::Count cols_of(const std::vector<rlplan::Count>& cols, int tensor) const {
    return tensor == rlplan::kDataTensor ? data_total / 2 : cols.at(static_cast<size_t>(tensor));
  }
};
