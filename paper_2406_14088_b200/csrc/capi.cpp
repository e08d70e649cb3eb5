// C ABI (include/rr_realloc.h) over the rlplan C++ library and the sm_100a
// kernels. No exception crosses this boundary: ValidationError -> RR_EINVAL
// with the reference's message (reference common.hpp:22-25), CUDA failures
// -> RR_ECUDA, allocation failures -> RR_ENOMEM.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "rlplan/realloc.hpp"
#include "exec_plan.hpp"
#include "rr_internal.hpp"
#include "rr_realloc.h"

using namespace rlplan;

namespace {

thread_local std::string g_error;

struct StatusError {
  rr_status status;
  std::string message;
};

[[noreturn]] void raise(rr_status s, const std::string& msg) { throw StatusError{s, msg}; }

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(RR_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void check_cuda(int e, const char* what) { check_cuda(static_cast<cudaError_t>(e), what); }

template <class F>
rr_status guarded(F&& f) {
  try {
    f();
    return RR_OK;
  } catch (const StatusError& e) {
    g_error = e.message;
    return e.status;
  } catch (const ValidationError& e) {
    g_error = e.what();
    return RR_EINVAL;
  } catch (const std::bad_alloc&) {
    g_error = "out of host memory";
    return RR_ENOMEM;
  } catch (const std::exception& e) {
    g_error = e.what();
    return RR_EINVAL;
  }
}

void need(bool ok, const char* what) {
  if (!ok) raise(RR_EINVAL, what);
}

ModelSpec to_model(const rr_model* m) {
  need(m != nullptr, "null model");
  ModelSpec s;
  s.name = m->name ? m->name : "";
  s.hidden_size = m->hidden_size;
  s.intermediate_size = m->intermediate_size;
  s.num_layers = m->num_layers;
  s.num_attention_heads = m->num_attention_heads;
  s.num_kv_heads = m->num_kv_heads;
  s.vocab_size = m->vocab_size;
  s.max_position_embeddings = m->max_position_embeddings;
  s.param_bytes = m->param_bytes;
  s.grad_bytes = m->grad_bytes;
  s.optimizer_bytes_per_param = m->optimizer_bytes_per_param;
  s.has_output_head = m->has_output_head != 0;
  return s;
}

ClusterSpec to_cluster(const rr_cluster* c) {
  need(c != nullptr, "null cluster");
  ClusterSpec s;
  s.n_nodes = c->n_nodes;
  s.gpus_per_node = c->gpus_per_node;
  s.mem_per_device = c->mem_per_device;
  s.intra_node_bw = c->intra_node_bw;
  s.inter_node_bw = c->inter_node_bw;
  s.host_to_device_bw = c->host_to_device_bw;
  return s;
}

DeviceMesh to_mesh(const rr_mesh* m) {
  need(m != nullptr, "null mesh");
  return DeviceMesh{m->node_offset, m->node_count, m->gpu_offset, m->gpu_count};
}

rr_mesh from_mesh(const DeviceMesh& m) {
  return rr_mesh{m.node_offset, m.node_count, m.gpu_offset, m.gpu_count};
}

Placement to_placement(const rr_placement* p) {
  need(p != nullptr, "null placement");
  Placement out;
  out.mesh = to_mesh(&p->mesh);
  out.strategy = ParallelStrategy{p->dp, p->tp, p->pp, p->n_microbatches};
  need(p->qkv_layout >= 0 && p->qkv_layout <= 2, "qkv_layout must be 0, 1 or 2");
  need(p->gate_up_layout >= 0 && p->gate_up_layout <= 1, "gate_up_layout must be 0 or 1");
  out.qkv = static_cast<QkvLayout>(p->qkv_layout);
  out.gate_up = static_cast<GateUpLayout>(p->gate_up_layout);
  return out;
}

rr_shard to_shard(const ShardDescriptor& d) {
  return rr_shard{d.layer_start, d.layer_end, d.tp_rank, d.tp_degree, d.replicated ? 1 : 0};
}

}  // namespace

// ---------------------------------------------------------------------------
// Plan object
// ---------------------------------------------------------------------------

struct rr_plan {
  ModelSpec model;
  Placement src, dst;
  ClusterSpec cluster;
  ReallocPlan plan;
  std::vector<std::vector<int32_t>> remote_dst, local_dst;  // int32 copies for rr_op
  std::vector<LoweredOp> lowered;
  std::map<std::pair<int, DeviceId>, ShardLayout> layouts;
  std::mutex mu;  // guards lazily built layouts
  bool data = false;     // inter-call data transfer plan (plan_data_transfer)
  Bytes data_total = 0;  // its total data bytes

  const ShardLayout& layout(int side, DeviceId d) {
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_pair(side, d);
    auto it = layouts.find(key);
    if (it == layouts.end()) {
      ShardLayout lay = data ? data_layout(side ? dst : src, cluster, d, data_total, side == 0)
                             : shard_layout(model, side ? dst : src, cluster, d);
      it = layouts.emplace(key, std::move(lay)).first;
    }
    return it->second;
  }

  // Logical width of a tensor (for the weight value function's index).
  std::vector<Count> tensor_cols() const {
    std::vector<Count> cols;
    if (!data)
      for (const auto& t : tensor_inventory(model)) cols.push_back(t.cols);
    return cols;
  }
  Count cols_of(const std::vector<Count>& cols, int tensor) const {
    return tensor == kDataTensor ? data_total / 2 : cols.at(static_cast<size_t>(tensor));
  }
};

// ---------------------------------------------------------------------------
// Executor object
// ---------------------------------------------------------------------------

struct rr_exec {
  struct Phase {
    rr::CopyItem* d = nullptr;  // 16-byte (vec) items first, then 2-byte items
    int n = 0, n_vec = 0;
    int64_t read = 0, written = 0;
  };
  int cuda_device = 0;
  Phase phase[2];  // [0] direct copies, [1] in-host fan-out from leader replicas
  int fence_sys = 0;
  int default_ctas = 0;
  // 0 = LDG/STG rr_copy_kernel, 1..kBulkVariants = TMA bulk ring. Default:
  // variant 1 (4 x 16 KiB stages, 3 CTAs/SM), the fastest in the r01 sweep.
  int kernel = 1;
  int bulk_ctas = 0;
  unsigned int* d_sched = nullptr;  // dynamic work counter (see retire_cta)
  int64_t wire_in = 0, wire_out = 0;  // bytes crossing into / out of this host
  uint32_t epoch = 0;                 // relay flag epoch, advanced by every phase-0 launch

  // Onload pipelining (rr_exec_enable_onload): phase-0 items regrouped into
  // segments by the last host->device chunk they read; segment s may start
  // once chunk s has landed.
  rr::ItemSet phase0_host;             // items + provenance as built
  std::vector<void*> src_bases;        // source buffer per plan device
  struct Segment {
    int offset = 0, n = 0, n_vec = 0;
  };
  std::vector<Segment> segments;       // [0] = no dependency, [1 + c] waits for chunk c
  rr::CopyItem* d_onload = nullptr;
  struct Chunk {
    int32_t device;
    int64_t offset, bytes;
  };
  std::vector<Chunk> chunks;
  std::vector<cudaEvent_t> events;
};

struct rr_barrier {
  int cuda_device = 0;
  int rank = 0, world = 0;
  uint32_t epoch = 0;
  uint32_t** d_flags = nullptr;
  int* d_timed_out = nullptr;
};

namespace rr {
void set_last_error(const std::string& msg) { g_error = msg; }
}  // namespace rr

// Definitions take C linkage from the declarations in rr_realloc.h.

const char* rr_last_error(void) { return g_error.c_str(); }
int rr_abi_version(void) { return RR_ABI_VERSION; }

// ---- model-arith ----------------------------------------------------------

rr_status rr_model_validate(const rr_model* m) {
  return guarded([&] { to_model(m).validate(); });
}
rr_status rr_param_count(const rr_model* m, int include, int64_t* out) {
  return guarded([&] { *out = param_count(to_model(m), include != 0); });
}
rr_status rr_natural_param_count(const rr_model* m, int64_t* out) {
  return guarded([&] { *out = natural_param_count(to_model(m)); });
}
rr_status rr_flops(const rr_model* m, int backward, int64_t tokens, int64_t ctx, double* out) {
  return guarded([&] { *out = flops(to_model(m), backward ? Phase::Backward : Phase::Forward, tokens, ctx); });
}
rr_status rr_layer_flops_fwd(const rr_model* m, int64_t tokens, int64_t ctx, double* out) {
  return guarded([&] { *out = layer_flops_fwd(to_model(m), tokens, ctx); });
}
rr_status rr_kv_cache_bytes(const rr_model* m, int64_t batch, int64_t seq, int64_t* out) {
  return guarded([&] { *out = kv_cache_bytes(to_model(m), batch, seq); });
}
rr_status rr_logits_bytes(int64_t vocab, int64_t batch, int64_t ctx, int64_t elem, int64_t* out) {
  return guarded([&] { *out = logits_bytes(vocab, batch, ctx, elem); });
}
rr_status rr_static_param_bytes(const rr_model* m, int64_t* params, int64_t* grads, int64_t* opt) {
  return guarded([&] {
    const auto s = static_param_bytes(to_model(m));
    *params = s.params;
    *grads = s.grads;
    *opt = s.optimizer;
  });
}

// ---- cluster-topo -----------------------------------------------------------

rr_status rr_cluster_validate(const rr_cluster* c) {
  return guarded([&] { to_cluster(c).validate(); });
}
rr_status rr_validate_mesh(const rr_mesh* m, const rr_cluster* c) {
  return guarded([&] { validate_mesh(to_mesh(m), to_cluster(c)); });
}
rr_status rr_mesh_devices(const rr_mesh* m, const rr_cluster* c, int32_t* out, int cap, int* n) {
  return guarded([&] {
    const auto d = to_mesh(m).devices(to_cluster(c));
    *n = static_cast<int>(d.size());
    if (static_cast<int>(d.size()) > cap) raise(RR_ERANGE, "rr_mesh_devices: buffer too small");
    std::copy(d.begin(), d.end(), out);
  });
}
rr_status rr_mesh_contains(const rr_mesh* m, const rr_cluster* c, int32_t device, int* out) {
  return guarded([&] { *out = to_mesh(m).contains(to_cluster(c), device) ? 1 : 0; });
}
rr_status rr_enumerate_meshes(const rr_cluster* c, rr_mesh* out, int cap, int* n) {
  return guarded([&] {
    const auto all = enumerate_meshes(to_cluster(c));
    *n = static_cast<int>(all.size());
    if (static_cast<int>(all.size()) > cap) raise(RR_ERANGE, "rr_enumerate_meshes: buffer too small");
    for (size_t i = 0; i < all.size(); ++i) out[i] = from_mesh(all[i]);
  });
}
rr_status rr_overlap(const rr_mesh* a, const rr_mesh* b, const rr_cluster* c, int* out) {
  return guarded([&] { *out = overlap(to_mesh(a), to_mesh(b), to_cluster(c)) ? 1 : 0; });
}
rr_status rr_link_bandwidth(const rr_cluster* c, int32_t a, int32_t b, double* out) {
  return guarded([&] { *out = link_bandwidth(to_cluster(c), a, b); });
}
rr_status rr_mesh_to_string(const rr_mesh* m, const rr_cluster* c, char* buf, size_t cap, size_t* needed) {
  return guarded([&] {
    const std::string s = mesh_to_string(to_mesh(m), to_cluster(c));
    *needed = s.size() + 1;
    if (cap < s.size() + 1) raise(RR_ERANGE, "rr_mesh_to_string: buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}
rr_status rr_mesh_from_string(const char* text, const rr_cluster* c, rr_mesh* out) {
  return guarded([&] {
    need(text != nullptr, "null mesh string");
    *out = from_mesh(mesh_from_string(text, to_cluster(c)));
  });
}

// ---- realloc planning -------------------------------------------------------

rr_status rr_stage_layer_map(int64_t num_layers, int pp, int64_t* starts, int64_t* ends) {
  return guarded([&] {
    const auto st = stage_layer_map(num_layers, pp);
    for (size_t i = 0; i < st.size(); ++i) {
      starts[i] = st[i].first;
      ends[i] = st[i].second;
    }
  });
}

rr_status rr_validate_placement(const rr_model* m, const rr_placement* p, const rr_cluster* c) {
  return guarded([&] { validate_placement(to_model(m), to_placement(p), to_cluster(c)); });
}

rr_status rr_plan_create(const rr_model* m, const rr_placement* src, const rr_placement* dst,
                         const rr_cluster* c, int policy, rr_plan** out) {
  return guarded([&] {
    need(out != nullptr, "null output");
    need(policy == 0 || policy == 1, "policy must be 0 (spec) or 1 (balanced)");
    auto p = std::make_unique<rr_plan>();
    p->model = to_model(m);
    p->src = to_placement(src);
    p->dst = to_placement(dst);
    p->cluster = to_cluster(c);
    p->plan = plan_param_realloc(p->model, p->src, p->dst, p->cluster, static_cast<SourcePolicy>(policy));
    for (const auto& op : p->plan.ops) p->remote_dst.emplace_back(op.dst.begin(), op.dst.end());
    for (const auto& op : p->plan.local_ops) p->local_dst.emplace_back(op.dst.begin(), op.dst.end());
    p->lowered = lower_plan(p->model, p->src, p->dst, p->cluster, p->plan);
    *out = p.release();
  });
}

rr_status rr_plan_create_data(const rr_placement* producer, const rr_placement* consumer, const rr_cluster* c,
                              int64_t data_bytes_per_dp_shard, int policy, rr_plan** out) {
  return guarded([&] {
    need(out != nullptr, "null output");
    need(policy == 0 || policy == 1, "policy must be 0 (spec) or 1 (balanced)");
    auto p = std::make_unique<rr_plan>();
    p->model.name = "data";
    p->src = to_placement(producer);
    p->dst = to_placement(consumer);
    p->cluster = to_cluster(c);
    p->data = true;
    p->plan = plan_data_transfer(p->src, p->dst, data_bytes_per_dp_shard, p->cluster,
                                 static_cast<SourcePolicy>(policy));
    p->data_total = data_bytes_per_dp_shard * p->src.strategy.dp;
    for (const auto& op : p->plan.ops) p->remote_dst.emplace_back(op.dst.begin(), op.dst.end());
    for (const auto& op : p->plan.local_ops) p->local_dst.emplace_back(op.dst.begin(), op.dst.end());
    p->lowered = lower_data_plan(p->src, p->dst, p->cluster, p->data_total, p->plan);
    *out = p.release();
  });
}

void rr_plan_destroy(rr_plan* plan) { delete plan; }

rr_status rr_plan_totals(const rr_plan* plan, int64_t* total_bytes, double* est_time) {
  return guarded([&] {
    need(plan != nullptr, "null plan");
    *total_bytes = plan->plan.total_bytes;
    *est_time = plan->plan.est_time;
  });
}

rr_status rr_plan_num_ops(const rr_plan* plan, int local, int* n) {
  return guarded([&] {
    need(plan != nullptr, "null plan");
    *n = static_cast<int>(local ? plan->plan.local_ops.size() : plan->plan.ops.size());
  });
}

rr_status rr_plan_get_op(const rr_plan* plan, int local, int index, rr_op* out) {
  return guarded([&] {
    need(plan != nullptr, "null plan");
    const auto& list = local ? plan->plan.local_ops : plan->plan.ops;
    const auto& dsts = local ? plan->local_dst : plan->remote_dst;
    need(index >= 0 && index < static_cast<int>(list.size()), "op index out of range");
    const auto& op = list[static_cast<size_t>(index)];
    out->src = op.src;
    out->n_dst = static_cast<int32_t>(op.dst.size());
    out->dst = dsts[static_cast<size_t>(index)].data();
    out->payload = to_shard(op.payload);
    out->bytes = op.bytes;
  });
}

rr_status rr_plan_to_json(const rr_plan* plan, char* buf, size_t cap, size_t* needed) {
  return guarded([&] {
    need(plan != nullptr, "null plan");
    const std::string s = plan_to_json(plan->plan, plan->model, plan->src, plan->dst, plan->cluster);
    *needed = s.size() + 1;
    if (cap < s.size() + 1) raise(RR_ERANGE, "rr_plan_to_json: buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

rr_status rr_plan_shard_bytes(const rr_plan* plan, int side, int32_t device, int64_t* bytes) {
  return guarded([&] {
    need(plan != nullptr, "null plan");
    *bytes = const_cast<rr_plan*>(plan)->layout(side, device).bytes;
  });
}

rr_status rr_plan_device_traffic(const rr_plan* plan, int32_t device, int64_t* wire_in,
                                 int64_t* wire_out, int64_t* local) {
  return guarded([&] {
    need(plan != nullptr, "null plan");
    int64_t in = 0, out = 0, loc = 0;
    for (const auto& op : plan->lowered) {
      int64_t bytes = 0;
      for (const auto& r : op.rects) bytes += r.row_bytes * r.rows;
      for (DeviceId d : op.dst) {
        if (d == op.src) {
          if (d == device) loc += bytes;
        } else {
          if (d == device) in += bytes;
          if (op.src == device) out += bytes;
        }
      }
    }
    *wire_in = in;
    *wire_out = out;
    *local = loc;
  });
}

rr_status rr_plan_num_rects(const rr_plan* plan, int64_t* n) {
  return guarded([&] {
    need(plan != nullptr, "null plan");
    int64_t k = 0;
    for (const auto& op : plan->lowered) k += static_cast<int64_t>(op.rects.size());
    *n = k;
  });
}

rr_status rr_plan_layout(const rr_plan* plan, int side, int32_t device, int64_t* out,
                         int64_t cap_blocks, int64_t* n_blocks) {
  return guarded([&] {
    need(plan != nullptr, "null plan");
    const auto& lay = const_cast<rr_plan*>(plan)->layout(side, device);
    *n_blocks = static_cast<int64_t>(lay.blocks.size());
    if (cap_blocks < *n_blocks) raise(RR_ERANGE, "rr_plan_layout: buffer too small");
    for (size_t i = 0; i < lay.blocks.size(); ++i) {
      const auto& b = lay.blocks[i];
      int64_t* o = out + 6 * i;
      o[0] = b.tensor;
      o[1] = b.r0;
      o[2] = b.r1;
      o[3] = b.c0;
      o[4] = b.c1;
      o[5] = b.offset;
    }
  });
}

rr_status rr_plan_num_lowered(const rr_plan* plan, int* n) {
  return guarded([&] {
    need(plan != nullptr, "null plan");
    *n = static_cast<int>(plan->lowered.size());
  });
}

rr_status rr_plan_get_lowered(const rr_plan* plan, int index, int32_t* src, int32_t* dst, int* n_dst,
                              int64_t* rects, int64_t cap_rects, int64_t* n_rects) {
  return guarded([&] {
    need(plan != nullptr, "null plan");
    need(index >= 0 && index < static_cast<int>(plan->lowered.size()), "lowered op index out of range");
    const auto& op = plan->lowered[static_cast<size_t>(index)];
    need(op.dst.size() <= 64, "more than 64 destinations");
    *src = op.src;
    *n_dst = static_cast<int>(op.dst.size());
    std::copy(op.dst.begin(), op.dst.end(), dst);
    *n_rects = static_cast<int64_t>(op.rects.size());
    if (!rects) return;
    if (cap_rects < *n_rects) raise(RR_ERANGE, "rr_plan_get_lowered: rect buffer too small");
    for (size_t i = 0; i < op.rects.size(); ++i) {
      const auto& r = op.rects[i];
      int64_t* o = rects + 6 * i;
      o[0] = r.src_off;
      o[1] = r.dst_off;
      o[2] = r.row_bytes;
      o[3] = r.src_pitch;
      o[4] = r.dst_pitch;
      o[5] = r.rows;
    }
  });
}

// ---- device memory and peer mapping ----------------------------------------

rr_status rr_device_count(int* n) {
  return guarded([&] {
    int k = 0;
    const cudaError_t e = cudaGetDeviceCount(&k);
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
      cudaGetLastError();
      k = 0;
    } else {
      check_cuda(e, "cudaGetDeviceCount");
    }
    *n = k;
  });
}

rr_status rr_device_alloc(int cuda_device, size_t bytes, void** out) {
  return guarded([&] {
    check_cuda(cudaSetDevice(cuda_device), "cudaSetDevice");
    const cudaError_t e = cudaMalloc(out, bytes ? bytes : 256);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      raise(RR_ENOMEM, "cudaMalloc: out of device memory");
    }
    check_cuda(e, "cudaMalloc");
  });
}

rr_status rr_device_free(void* ptr) {
  return guarded([&] { check_cuda(cudaFree(ptr), "cudaFree"); });
}

rr_status rr_host_alloc(size_t bytes, void** out) {
  return guarded([&] {
    const cudaError_t e = cudaMallocHost(out, bytes ? bytes : 256);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      raise(RR_ENOMEM, "cudaMallocHost: out of pinned memory");
    }
    check_cuda(e, "cudaMallocHost");
  });
}

rr_status rr_host_free(void* ptr) {
  return guarded([&] { check_cuda(cudaFreeHost(ptr), "cudaFreeHost"); });
}

rr_status rr_memcpy(void* dst, const void* src, size_t bytes, int kind, void* stream, int synchronous) {
  return guarded([&] {
    static const cudaMemcpyKind kinds[] = {cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost,
                                           cudaMemcpyDeviceToDevice};
    need(kind >= 0 && kind <= 2, "memcpy kind must be 0, 1 or 2");
    auto s = static_cast<cudaStream_t>(stream);
    check_cuda(cudaMemcpyAsync(dst, src, bytes, kinds[kind], s), "cudaMemcpyAsync");
    if (synchronous) check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  });
}

rr_status rr_memset(void* dst, int value, size_t bytes, void* stream) {
  return guarded([&] {
    check_cuda(cudaMemsetAsync(dst, value, bytes, static_cast<cudaStream_t>(stream)), "cudaMemsetAsync");
  });
}

rr_status rr_stream_sync(void* stream) {
  return guarded([&] {
    check_cuda(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "cudaStreamSynchronize");
  });
}

rr_status rr_ipc_handle(void* device_ptr, void* handle64) {
  return guarded([&] {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    check_cuda(cudaIpcGetMemHandle(&h, device_ptr), "cudaIpcGetMemHandle");
    std::memcpy(handle64, &h, sizeof(h));
  });
}

rr_status rr_ipc_open(int cuda_device, const void* handle64, void** out) {
  return guarded([&] {
    check_cuda(cudaSetDevice(cuda_device), "cudaSetDevice");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    check_cuda(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  });
}

rr_status rr_ipc_close(void* ptr) {
  return guarded([&] { check_cuda(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle"); });
}

rr_status rr_enable_peer(int cuda_device, int peer_device) {
  return guarded([&] {
    int ok = 0;
    check_cuda(cudaDeviceCanAccessPeer(&ok, cuda_device, peer_device), "cudaDeviceCanAccessPeer");
    if (!ok) raise(RR_EUNSUPPORTED, "peer access not supported between these devices");
    check_cuda(cudaSetDevice(cuda_device), "cudaSetDevice");
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
      cudaGetLastError();
      return;
    }
    check_cuda(e, "cudaDeviceEnablePeerAccess");
  });
}

// ---- execution ----------------------------------------------------------------

namespace {

// Host map for an executor: `local` plan devices form this host; without an
// explicit table every other device is its own host.
rr::HostMap host_map(const rr_plan* plan, int n_local, const int32_t* local, const int32_t* host_of) {
  const int n = plan->cluster.device_count();
  rr::HostMap hm;
  hm.host.resize(static_cast<size_t>(n));
  if (host_of) {
    for (int d = 0; d < n; ++d) hm.host[static_cast<size_t>(d)] = host_of[d];
    need(n_local > 0, "host_of needs at least one local device");
    need(local[0] >= 0 && local[0] < n, "local device out of range");
    hm.me = host_of[local[0]];
    for (int i = 0; i < n_local; ++i) {
      need(local[i] >= 0 && local[i] < n, "local device out of range");
      need(host_of[local[i]] == hm.me, "local devices must share one host");
    }
    return hm;
  }
  hm.hierarchical = false;
  for (int d = 0; d < n; ++d) hm.host[static_cast<size_t>(d)] = n + d;  // distinct remote hosts
  hm.me = -1;
  for (int i = 0; i < n_local; ++i) {
    need(local[i] >= 0 && local[i] < n, "local device out of range");
    hm.host[static_cast<size_t>(local[i])] = hm.me;
  }
  return hm;
}

void upload(const rr::ItemSet& set, rr_exec::Phase& ph) {
  ph.n = static_cast<int>(set.items.size());
  ph.n_vec = set.n_vec;
  ph.read = set.read;
  ph.written = set.written;
  if (set.items.empty()) return;
  const size_t bytes = set.items.size() * sizeof(rr::CopyItem);
  check_cuda(cudaMalloc(&ph.d, bytes), "cudaMalloc(items)");
  check_cuda(cudaMemcpy(ph.d, set.items.data(), bytes, cudaMemcpyHostToDevice), "upload items");
}

void launch_phase(rr_exec* ex, const rr_exec::Phase& ph, void* stream, int ctas) {
  check_cuda(cudaSetDevice(ex->cuda_device), "cudaSetDevice");
  if (ph.n == 0) return;
  if (ex->kernel == 0) {
    check_cuda(rr::launch_copy(ph.d, ph.n, ctas > 0 ? ctas : ex->default_ctas, ex->fence_sys, stream, ex->d_sched,
                               ex->epoch),
               "rr_copy_kernel launch");
    return;
  }
  // Relay, multicast and 2-byte items take the LDG/STG kernel, launched
  // first so relay chains start immediately; then the TMA bulk kernel.
  if (ph.n > ph.n_vec)
    check_cuda(rr::launch_copy(ph.d + ph.n_vec, ph.n - ph.n_vec, ctas > 0 ? ctas : ex->default_ctas, ex->fence_sys,
                               stream, ex->d_sched, ex->epoch),
               "rr_copy_kernel launch (relay / multicast / 2-byte items)");
  if (ph.n_vec > 0)
    check_cuda(rr::launch_bulk(ex->kernel, ph.d, ph.n_vec, ctas > 0 ? ctas : ex->bulk_ctas, ex->fence_sys, stream,
                               nullptr, ex->d_sched),
               "rr_bulk_kernel launch");
}

}  // namespace

rr_status rr_plan_work(const rr_plan* plan, int n_local, const int32_t* local, const int32_t* host_of, int mode,
                       int64_t* out6) {
  return guarded([&] {
    need(plan != nullptr && out6 != nullptr, "null plan/output");
    need(mode == 0 || mode == 1, "mode must be 0 (push) or 1 (pull)");
    const rr::HostMap hm = host_map(plan, n_local, local, host_of);
    const auto jobs = rr::build_jobs(plan->lowered, hm, mode);
    const auto a = rr::build_items(jobs, 0, hm, nullptr, nullptr, int64_t{1} << 30);
    const auto b = rr::build_items(jobs, 1, hm, nullptr, nullptr, int64_t{1} << 30);
    out6[0] = a.read;
    out6[1] = a.written;
    out6[2] = b.read;
    out6[3] = b.written;
    rr::host_wire_bytes(plan->lowered, hm, &out6[4], &out6[5]);
  });
}

rr_status rr_exec_create(const rr_plan* plan, int cuda_device, int n_devices, void* const* src_bufs,
                         void* const* dst_bufs, int n_local, const int32_t* local, const int32_t* host_of,
                         int mode, int64_t chunk_bytes, rr_exec** out) {
  rr_exec_options opt;
  opt.mode = mode;
  opt.chunk_bytes = chunk_bytes;
  opt.host_of = host_of;
  opt.mc_bufs = nullptr;
  opt.relay_flags = nullptr;
  opt.relay_chain = 0;
  opt.overlap_fanout = 0;
  return rr_exec_create_ex(plan, cuda_device, n_devices, src_bufs, dst_bufs, n_local, local, &opt, out);
}

rr_status rr_exec_create_ex(const rr_plan* plan, int cuda_device, int n_devices, void* const* src_bufs,
                            void* const* dst_bufs, int n_local, const int32_t* local,
                            const rr_exec_options* options, rr_exec** out) {
  return guarded([&] {
    need(plan != nullptr && out != nullptr && options != nullptr, "null plan/options/output");
    const int mode = options->mode;
    int64_t chunk_bytes = options->chunk_bytes;
    need(mode == 0 || mode == 1, "mode must be 0 (push) or 1 (pull)");
    need(n_devices >= plan->cluster.device_count(), "buffer tables must cover every cluster device");
    if (chunk_bytes <= 0) chunk_bytes = 256 << 10;
    need(chunk_bytes >= 16, "chunk_bytes too small");
    rr::HostMap hm = host_map(plan, n_local, local, options->host_of);
    if (options->mc_bufs) {
      need(options->host_of != nullptr, "multicast needs a host_of table");
      need(mode == 0, "multicast is a push-mode path");
      hm.mc.resize(hm.host.size());
      for (size_t d = 0; d < hm.mc.size(); ++d) hm.mc[d] = reinterpret_cast<uint64_t>(options->mc_bufs[d]);
    }
    hm.relay_chunk = chunk_bytes;
    if (options->relay_flags) {
      need(options->host_of != nullptr && mode == 0, "relay needs a host_of table and push mode");
      hm.relay_flags.resize(hm.host.size());
      for (size_t d = 0; d < hm.relay_flags.size(); ++d)
        hm.relay_flags[d] = reinterpret_cast<uint64_t>(options->relay_flags[d]);
      hm.relay_chain = options->relay_chain != 0;
      hm.relay_star = options->overlap_fanout != 0;
    }
    const auto jobs = rr::build_jobs(plan->lowered, hm, mode);
    const auto a = rr::build_items(jobs, 0, hm, src_bufs, dst_bufs, chunk_bytes);
    const auto b = rr::build_items(jobs, 1, hm, src_bufs, dst_bufs, chunk_bytes);

    auto ex = std::make_unique<rr_exec>();
    ex->cuda_device = cuda_device;
    // Remote accesses (peer stores, or peer loads in pull mode) must be
    // visible system-wide before the following barrier releases them.
    int64_t win = 0, wout = 0;
    rr::host_wire_bytes(plan->lowered, hm, &win, &wout);
    ex->fence_sys = (a.remote_stores || win || wout) ? 1 : 0;
    ex->wire_in = win;
    ex->wire_out = wout;
    check_cuda(cudaSetDevice(cuda_device), "cudaSetDevice");
    int per_sm = 0, sms = 0;
    check_cuda(rr::copy_max_ctas(&per_sm, &sms), "occupancy query");
    ex->default_ctas = std::max(1, per_sm) * sms;
    upload(a, ex->phase[0]);
    upload(b, ex->phase[1]);
    ex->phase0_host = a;
    ex->src_bases.assign(static_cast<size_t>(n_devices), nullptr);
    for (int d = 0; d < n_devices; ++d) ex->src_bases[static_cast<size_t>(d)] = src_bufs ? src_bufs[d] : nullptr;
    check_cuda(cudaMalloc(&ex->d_sched, 4 * sizeof(unsigned int)), "cudaMalloc(sched)");
    check_cuda(cudaMemset(ex->d_sched, 0, 4 * sizeof(unsigned int)), "cudaMemset(sched)");
    check_cuda(rr::launch_bulk(ex->kernel, nullptr, 0, 0, 0, nullptr, &ex->bulk_ctas, nullptr), "bulk occupancy");
    *out = ex.release();
  });
}

rr_status rr_exec_launch(rr_exec* ex, void* stream, int ctas) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    ++ex->epoch;  // every rank launches phase 0 the same number of times
    launch_phase(ex, ex->phase[0], stream, ctas);
  });
}

rr_status rr_exec_kernel_count(const rr_exec* ex, int* phase0, int* phase1) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    auto count = [&](const rr_exec::Phase& ph) {
      if (ph.n == 0) return 0;
      if (ex->kernel == 0) return 1;
      return (ph.n > ph.n_vec ? 1 : 0) + (ph.n_vec > 0 ? 1 : 0);
    };
    *phase0 = count(ex->phase[0]);
    *phase1 = count(ex->phase[1]);
  });
}

rr_status rr_exec_relay_timeouts(rr_exec* ex, int64_t* timeouts) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    check_cuda(cudaSetDevice(ex->cuda_device), "cudaSetDevice");
    unsigned int h[4];
    check_cuda(cudaMemcpy(h, ex->d_sched, sizeof(h), cudaMemcpyDeviceToHost), "read relay status");
    *timeouts = h[2];
  });
}

rr_status rr_plan_relay_slots(const rr_plan* plan, const int32_t* host_of, int64_t chunk_bytes, int relay_chain,
                              int overlap_fanout, int64_t* slots) {
  return guarded([&] {
    need(plan != nullptr && host_of != nullptr, "null plan/host table");
    rr::HostMap hm;
    for (int d = 0; d < plan->cluster.device_count(); ++d) hm.host.push_back(host_of[d]);
    hm.relay_chunk = chunk_bytes > 0 ? chunk_bytes : (256 << 10);
    hm.relay_chain = relay_chain != 0;
    hm.relay_star = overlap_fanout != 0;
    *slots = rr::relay_slots(plan->lowered, hm);
  });
}

rr_status rr_exec_launch_fanout(rr_exec* ex, void* stream, int ctas) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    launch_phase(ex, ex->phase[1], stream, ctas);
  });
}

rr_status rr_exec_set_kernel(rr_exec* ex, int kernel) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    need(kernel >= 0 && kernel <= rr::kBulkVariants, "unknown copy kernel");
    ex->kernel = kernel;
    if (kernel > 0) {
      check_cuda(cudaSetDevice(ex->cuda_device), "cudaSetDevice");
      check_cuda(rr::launch_bulk(kernel, nullptr, 0, 0, 0, nullptr, &ex->bulk_ctas, nullptr), "bulk occupancy");
    }
  });
}

rr_status rr_exec_stats(const rr_exec* ex, int phase, int64_t* items, int64_t* written, int64_t* read) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    need(phase == 0 || phase == 1, "phase must be 0 or 1");
    const auto& ph = ex->phase[phase];
    *items = ph.n;
    *written = ph.written;
    *read = ph.read;
  });
}

rr_status rr_exec_wire(const rr_exec* ex, int64_t* wire_in, int64_t* wire_out) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    *wire_in = ex->wire_in;
    *wire_out = ex->wire_out;
  });
}

rr_status rr_exec_enable_onload(rr_exec* ex, int n_src, const int32_t* src_devices, const int64_t* src_bytes,
                                 int64_t chunk_bytes) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    need(n_src >= 0 && chunk_bytes >= 4096, "bad onload arguments");
    check_cuda(cudaSetDevice(ex->cuda_device), "cudaSetDevice");
    for (auto e : ex->events) cudaEventDestroy(e);
    ex->events.clear();
    ex->chunks.clear();
    std::map<DeviceId, int> first_chunk;
    for (int i = 0; i < n_src; ++i) {
      need(src_devices[i] >= 0 && src_devices[i] < static_cast<int>(ex->src_bases.size()), "onload device range");
      need(ex->src_bases[static_cast<size_t>(src_devices[i])] != nullptr, "onload device has no source buffer");
      first_chunk[src_devices[i]] = static_cast<int>(ex->chunks.size());
      for (int64_t off = 0; off < src_bytes[i]; off += chunk_bytes)
        ex->chunks.push_back({src_devices[i], off, std::min(chunk_bytes, src_bytes[i] - off)});
    }
    // Segment of each item: 0 = independent of the onload, 1 + c = needs chunk c.
    const rr::ItemSet& a = ex->phase0_host;
    const size_t n = a.items.size(), C = ex->chunks.size();
    std::vector<std::vector<int>> seg_vec(C + 1), seg_other(C + 1);
    for (size_t i = 0; i < n; ++i) {
      int seg = 0;
      const auto it = first_chunk.find(a.src_dev[i]);
      if (a.items[i].wait_flag) {
        // Relay / overlapped fan-out items wait on other GPUs' pushes, which
        // may depend on this GPU's own pushes: launch them after every chunk
        // (and so every push of this GPU) so no launch waits on a later one.
        seg = static_cast<int>(C);
      } else if (it != first_chunk.end() && !a.src_is_dst[i]) {
        const DeviceId d = a.src_dev[i];
        int64_t total = 0;
        for (int k = 0; k < n_src; ++k)
          if (src_devices[k] == d) total = src_bytes[k];
        need(a.src_end[i] <= total, "an item reads beyond the onloaded bytes of its source");
        seg = 1 + it->second + static_cast<int>((a.src_end[i] - 1) / chunk_bytes);
      }
      (static_cast<int>(i) < a.n_vec ? seg_vec : seg_other)[static_cast<size_t>(seg)].push_back(static_cast<int>(i));
    }
    std::vector<rr::CopyItem> ordered;
    ordered.reserve(n);
    ex->segments.assign(C + 1, {});
    for (size_t s = 0; s <= C; ++s) {
      auto& sg = ex->segments[s];
      sg.offset = static_cast<int>(ordered.size());
      for (int i : seg_vec[s]) ordered.push_back(a.items[static_cast<size_t>(i)]);
      sg.n_vec = static_cast<int>(seg_vec[s].size());
      for (int i : seg_other[s]) ordered.push_back(a.items[static_cast<size_t>(i)]);
      sg.n = static_cast<int>(ordered.size()) - sg.offset;
    }
    if (ex->d_onload) cudaFree(ex->d_onload);
    ex->d_onload = nullptr;
    if (!ordered.empty()) {
      check_cuda(cudaMalloc(&ex->d_onload, ordered.size() * sizeof(rr::CopyItem)), "cudaMalloc(onload items)");
      check_cuda(cudaMemcpy(ex->d_onload, ordered.data(), ordered.size() * sizeof(rr::CopyItem),
                            cudaMemcpyHostToDevice),
                 "upload onload items");
    }
    ex->events.resize(C);
    for (auto& e : ex->events) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  });
}

rr_status rr_exec_launch_onload(rr_exec* ex, void* const* host_bufs, void* copy_stream, void* stream, int ctas) {
  return guarded([&] {
    need(ex != nullptr && host_bufs != nullptr, "null executor/host buffers");
    need(!ex->segments.empty(), "rr_exec_enable_onload has not been called");
    check_cuda(cudaSetDevice(ex->cuda_device), "cudaSetDevice");
    ++ex->epoch;  // a phase-0 launch like rr_exec_launch
    auto cs = static_cast<cudaStream_t>(copy_stream);
    auto ks = static_cast<cudaStream_t>(stream);
    // The copy stream must not overwrite sources still read by an earlier
    // launch on the compute stream.
    cudaEvent_t ready;
    check_cuda(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "cudaEventCreate");
    check_cuda(cudaEventRecord(ready, ks), "cudaEventRecord");
    check_cuda(cudaStreamWaitEvent(cs, ready, 0), "cudaStreamWaitEvent");
    cudaEventDestroy(ready);
    for (size_t c = 0; c < ex->chunks.size(); ++c) {
      const auto& ch = ex->chunks[c];
      const void* h = host_bufs[ch.device];
      need(h != nullptr, "missing host buffer for an onloaded device");
      char* dst = static_cast<char*>(ex->src_bases[static_cast<size_t>(ch.device)]) + ch.offset;
      check_cuda(cudaMemcpyAsync(dst, static_cast<const char*>(h) + ch.offset, static_cast<size_t>(ch.bytes),
                                 cudaMemcpyHostToDevice, cs),
                 "onload cudaMemcpyAsync");
      check_cuda(cudaEventRecord(ex->events[c], cs), "cudaEventRecord");
    }
    for (size_t s = 0; s < ex->segments.size(); ++s) {
      if (s > 0) check_cuda(cudaStreamWaitEvent(ks, ex->events[s - 1], 0), "cudaStreamWaitEvent");
      const auto& sg = ex->segments[s];
      if (sg.n == 0) continue;
      rr_exec::Phase ph;
      ph.d = ex->d_onload + sg.offset;
      ph.n = sg.n;
      ph.n_vec = sg.n_vec;
      launch_phase(ex, ph, stream, ctas);
    }
  });
}

void rr_exec_destroy(rr_exec* ex) {
  if (!ex) return;
  cudaSetDevice(ex->cuda_device);
  for (auto& ph : ex->phase)
    if (ph.d) cudaFree(ph.d);
  if (ex->d_sched) cudaFree(ex->d_sched);
  if (ex->d_onload) cudaFree(ex->d_onload);
  for (auto e : ex->events) cudaEventDestroy(e);
  delete ex;
}

// ---- deterministic weights ----------------------------------------------------

namespace {

std::vector<rr::FillItem> fill_items(const ShardLayout& lay, const rr_plan& plan, uint64_t base) {
  const auto cols = plan.tensor_cols();
  constexpr uint32_t kChunk = 1u << 16;
  std::vector<rr::FillItem> items;
  for (const auto& b : lay.blocks) {
    const uint64_t n = static_cast<uint64_t>((b.r1 - b.r0) * (b.c1 - b.c0));
    if (n >= (uint64_t{1} << 32)) raise(RR_EINVAL, "layout block larger than 2^32 elements");
    for (uint64_t e = 0; e < n; e += kChunk) {
      rr::FillItem it;
      it.base = base + static_cast<uint64_t>(b.offset);
      it.r0 = static_cast<uint64_t>(b.r0);
      it.c0 = static_cast<uint64_t>(b.c0);
      it.full_cols = static_cast<uint64_t>(plan.cols_of(cols, b.tensor));
      it.cols = static_cast<uint32_t>(b.c1 - b.c0);
      it.tensor = static_cast<uint32_t>(b.tensor);
      it.elem0 = static_cast<uint32_t>(e);
      it.n = static_cast<uint32_t>(std::min<uint64_t>(kChunk, n - e));
      items.push_back(it);
    }
  }
  return items;
}

template <class T>
struct DeviceArray {
  T* ptr = nullptr;
  explicit DeviceArray(const std::vector<T>& host) {
    if (host.empty()) return;
    check_cuda(cudaMalloc(&ptr, host.size() * sizeof(T)), "cudaMalloc(items)");
    check_cuda(cudaMemcpy(ptr, host.data(), host.size() * sizeof(T), cudaMemcpyHostToDevice), "upload items");
  }
  ~DeviceArray() {
    if (ptr) cudaFree(ptr);
  }
};

}  // namespace

rr_status rr_fill_shard(const rr_plan* plan, int side, int32_t device, void* buf, uint64_t seed, void* stream) {
  return guarded([&] {
    need(plan != nullptr && buf != nullptr, "null plan/buffer");
    const auto& lay = const_cast<rr_plan*>(plan)->layout(side, device);
    const auto items = fill_items(lay, *plan, reinterpret_cast<uint64_t>(buf));
    DeviceArray<rr::FillItem> d(items);
    auto s = static_cast<cudaStream_t>(stream);
    check_cuda(rr::launch_fill(d.ptr, static_cast<int>(items.size()), seed, s), "rr_fill_kernel launch");
    check_cuda(cudaStreamSynchronize(s), "fill sync");
  });
}

rr_status rr_verify_shard(const rr_plan* plan, int side, int32_t device, const void* buf, uint64_t seed,
                          void* stream, int64_t* mismatches, int64_t* first) {
  return guarded([&] {
    need(plan != nullptr && buf != nullptr, "null plan/buffer");
    const auto& lay = const_cast<rr_plan*>(plan)->layout(side, device);
    const uint64_t base = reinterpret_cast<uint64_t>(buf);
    const auto items = fill_items(lay, *plan, base);
    DeviceArray<rr::FillItem> d(items);
    const std::vector<unsigned long long> init = {0ull, ~0ull};
    DeviceArray<unsigned long long> counters(init);
    auto s = static_cast<cudaStream_t>(stream);
    check_cuda(rr::launch_verify(d.ptr, static_cast<int>(items.size()), seed, counters.ptr, base, s),
               "rr_verify_kernel launch");
    unsigned long long host[2];
    check_cuda(cudaMemcpyAsync(host, counters.ptr, sizeof(host), cudaMemcpyDeviceToHost, s), "verify readback");
    check_cuda(cudaStreamSynchronize(s), "verify sync");
    *mismatches = static_cast<int64_t>(host[0]);
    *first = host[0] ? static_cast<int64_t>(host[1]) : -1;
  });
}

uint16_t rr_weight_value(uint64_t seed, int64_t tensor_id, int64_t logical_index) {
  return rr::weight_value(seed, static_cast<uint64_t>(tensor_id), static_cast<uint64_t>(logical_index));
}

// ---- barrier -------------------------------------------------------------------

rr_status rr_barrier_create(int cuda_device, int rank, int world, void* const* flags, rr_barrier** out) {
  return guarded([&] {
    need(world >= 1 && world <= 32 && rank >= 0 && rank < world, "bad rank/world");
    auto b = std::make_unique<rr_barrier>();
    b->cuda_device = cuda_device;
    b->rank = rank;
    b->world = world;
    check_cuda(cudaSetDevice(cuda_device), "cudaSetDevice");
    std::vector<uint32_t*> host(static_cast<size_t>(world));
    for (int p = 0; p < world; ++p) {
      need(flags[p] != nullptr, "missing flag buffer");
      host[static_cast<size_t>(p)] = static_cast<uint32_t*>(flags[p]);
    }
    check_cuda(cudaMalloc(&b->d_flags, host.size() * sizeof(uint32_t*)), "cudaMalloc(flags)");
    check_cuda(cudaMemcpy(b->d_flags, host.data(), host.size() * sizeof(uint32_t*), cudaMemcpyHostToDevice),
               "upload flags");
    check_cuda(cudaMalloc(&b->d_timed_out, sizeof(int)), "cudaMalloc(timeout)");
    check_cuda(cudaMemset(b->d_timed_out, 0, sizeof(int)), "cudaMemset(timeout)");
    *out = b.release();
  });
}

rr_status rr_barrier_launch(rr_barrier* b, void* stream) {
  return guarded([&] {
    need(b != nullptr, "null barrier");
    check_cuda(cudaSetDevice(b->cuda_device), "cudaSetDevice");
    ++b->epoch;
    check_cuda(rr::launch_barrier(b->d_flags, b->rank, b->world, b->epoch, b->d_timed_out, stream),
               "rr_barrier_kernel launch");
  });
}

rr_status rr_barrier_status(rr_barrier* b, int* timed_out) {
  return guarded([&] {
    need(b != nullptr, "null barrier");
    check_cuda(cudaSetDevice(b->cuda_device), "cudaSetDevice");
    check_cuda(cudaMemcpy(timed_out, b->d_timed_out, sizeof(int), cudaMemcpyDeviceToHost), "barrier status");
  });
}

void rr_barrier_destroy(rr_barrier* b) {
  if (!b) return;
  cudaSetDevice(b->cuda_device);
  cudaFree(b->d_flags);
  cudaFree(b->d_timed_out);
  delete b;
}
