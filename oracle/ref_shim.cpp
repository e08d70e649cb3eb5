// TEST INFRASTRUCTURE — extern "C" shim over the reference's own C++
// (/root/reference/proj/src/model_arith.cpp and cluster.cpp, compiled from
// where they lie by oracle/Makefile into oracle/_ref/librlplan_ref.so).
// Lets the tests pin the oracle and the product against the reference's
// real outputs for the model-arith and cluster-topo functions on the path.
#include <cstring>
#include <string>

#include "rlplan/cluster.hpp"
#include "rlplan/model_arith.hpp"

using namespace rlplan;

namespace {
ModelSpec make(const char* name, const long long* d, int has_head) {
  ModelSpec s;
  s.name = name;
  s.hidden_size = d[0];
  s.intermediate_size = d[1];
  s.num_layers = d[2];
  s.num_attention_heads = d[3];
  s.num_kv_heads = d[4];
  s.vocab_size = d[5];
  s.max_position_embeddings = d[6];
  s.param_bytes = d[7];
  s.grad_bytes = d[8];
  s.optimizer_bytes_per_param = d[9];
  s.has_output_head = has_head != 0;
  return s;
}
ClusterSpec cluster(int nodes, int gpus) {
  ClusterSpec c;
  c.n_nodes = nodes;
  c.gpus_per_node = gpus;
  c.mem_per_device = 1;
  c.intra_node_bw = 900e9;
  c.inter_node_bw = 50e9;
  c.host_to_device_bw = 55e9;
  return c;
}
thread_local std::string err;
}  // namespace

extern "C" {

const char* ref_last_error() { return err.c_str(); }

// dims: hidden, ffn, layers, heads, kv, vocab, maxpos, param_b, grad_b, opt_b
int ref_param_count(const long long* dims, int has_head, int include, long long* out) {
  try {
    *out = param_count(make("ref", dims, has_head), include != 0);
    return 0;
  } catch (const ValidationError& e) {
    err = e.what();
    return 1;
  }
}

int ref_static_param_bytes(const long long* dims, int has_head, long long* out3) {
  try {
    const auto s = static_param_bytes(make("ref", dims, has_head));
    out3[0] = s.params;
    out3[1] = s.grads;
    out3[2] = s.optimizer;
    return 0;
  } catch (const ValidationError& e) {
    err = e.what();
    return 1;
  }
}

int ref_flops(const long long* dims, int has_head, int backward, long long tokens, long long ctx, double* out) {
  try {
    *out = flops(make("ref", dims, has_head), backward ? Phase::Backward : Phase::Forward, tokens, ctx);
    return 0;
  } catch (const ValidationError& e) {
    err = e.what();
    return 1;
  }
}

long long ref_kv_cache_bytes(const long long* dims, int has_head, long long batch, long long seq) {
  return kv_cache_bytes(make("ref", dims, has_head), batch, seq);
}

long long ref_logits_bytes(long long v, long long b, long long c, long long e) { return logits_bytes(v, b, c, e); }

// meshes as 4 ints each
int ref_enumerate_meshes(int nodes, int gpus, int* out, int cap) {
  const auto all = enumerate_meshes(cluster(nodes, gpus));
  if ((int)all.size() > cap) return -(int)all.size();
  for (size_t i = 0; i < all.size(); ++i) {
    out[4 * i] = all[i].node_offset;
    out[4 * i + 1] = all[i].node_count;
    out[4 * i + 2] = all[i].gpu_offset;
    out[4 * i + 3] = all[i].gpu_count;
  }
  return (int)all.size();
}

int ref_validate_mesh(int nodes, int gpus, const int* m) {
  try {
    validate_mesh(DeviceMesh{m[0], m[1], m[2], m[3]}, cluster(nodes, gpus));
    return 0;
  } catch (const ValidationError& e) {
    err = e.what();
    return 1;
  }
}

int ref_mesh_devices(int nodes, int gpus, const int* m, int* out) {
  const auto d = DeviceMesh{m[0], m[1], m[2], m[3]}.devices(cluster(nodes, gpus));
  for (size_t i = 0; i < d.size(); ++i) out[i] = d[i];
  return (int)d.size();
}

int ref_overlap(int nodes, int gpus, const int* a, const int* b) {
  return overlap(DeviceMesh{a[0], a[1], a[2], a[3]}, DeviceMesh{b[0], b[1], b[2], b[3]}, cluster(nodes, gpus)) ? 1 : 0;
}

int ref_link_bandwidth(int nodes, int gpus, int a, int b, double* out) {
  try {
    *out = link_bandwidth(cluster(nodes, gpus), a, b);
    return 0;
  } catch (const ValidationError& e) {
    err = e.what();
    return 1;
  }
}

int ref_mesh_to_string(int nodes, int gpus, const int* m, char* buf, int cap) {
  const std::string s = mesh_to_string(DeviceMesh{m[0], m[1], m[2], m[3]}, cluster(nodes, gpus));
  std::strncpy(buf, s.c_str(), cap);
  return (int)s.size();
}

int ref_mesh_from_string(int nodes, int gpus, const char* text, int* out) {
  try {
    const auto m = mesh_from_string(text, cluster(nodes, gpus));
    out[0] = m.node_offset;
    out[1] = m.node_count;
    out[2] = m.gpu_offset;
    out[3] = m.gpu_count;
    return 0;
  } catch (const ValidationError& e) {
    err = e.what();
    return 1;
  }
}

}  // extern "C"
