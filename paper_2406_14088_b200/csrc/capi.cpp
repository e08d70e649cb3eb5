// C ABI (include/rr_realloc.h) over the rlplan C++ library and the sm_100a
// kernels. No exception crosses this boundary: ValidationError -> RR_EINVAL
// with the reference's message (reference common.hpp:22-25), CUDA failures
// -> RR_ECUDA, allocation failures -> RR_ENOMEM. The executor entry points
// live in capi_exec.cpp.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "capi_internal.hpp"
#include "rr_internal.hpp"

using namespace rlplan;
using rr::capi::check_cuda;
using rr::capi::guarded;
using rr::capi::need;
using rr::capi::raise;

namespace {

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
  need(p->kv_layout >= 0 && p->kv_layout <= 1, "kv_layout must be 0 or 1");
  out.qkv = static_cast<QkvLayout>(p->qkv_layout);
  out.gate_up = static_cast<GateUpLayout>(p->gate_up_layout);
  out.kv = static_cast<KvLayout>(p->kv_layout);
  return out;
}

rr_shard to_shard(const ShardDescriptor& d) {
  return rr_shard{d.layer_start, d.layer_end, d.tp_rank, d.tp_degree, d.replicated ? 1 : 0, d.part};
}

}  // namespace

struct rr_barrier {
  int cuda_device = 0;
  int rank = 0, world = 0;
  uint32_t epoch = 0;
  uint32_t** d_flags = nullptr;
  int* d_timed_out = nullptr;

  rr_barrier() = default;
  rr_barrier(const rr_barrier&) = delete;
  rr_barrier& operator=(const rr_barrier&) = delete;
  ~rr_barrier() {  // also on a failed rr_barrier_create
    cudaSetDevice(cuda_device);
    if (d_flags) cudaFree(d_flags);
    if (d_timed_out) cudaFree(d_timed_out);
  }
};

namespace rr {
std::string& last_error_slot() {
  thread_local std::string message;
  return message;
}
void set_last_error(const std::string& msg) { last_error_slot() = msg; }
}  // namespace rr

// Definitions take C linkage from the declarations in rr_realloc.h.

const char* rr_last_error(void) { return rr::last_error_slot().c_str(); }
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
    *bytes = plan->layout(side, device).bytes;
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
    const auto& lay = plan->layout(side, device);
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
    // Whole 2 MiB pages: an allocation whose size is not a 2 MiB multiple
    // reached peers' copy engines at 551 instead of 777 GB/s over CUDA IPC
    // (profiles/r01_ce_alloc_probe_n2.txt)
    const size_t kPage = size_t{2} << 20;
    const size_t padded = bytes ? (bytes + kPage - 1) / kPage * kPage : kPage;
    const cudaError_t e = cudaMalloc(out, padded);
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
    const auto& lay = plan->layout(side, device);
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
    const auto& lay = plan->layout(side, device);
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

void rr_barrier_destroy(rr_barrier* b) { delete b; }
