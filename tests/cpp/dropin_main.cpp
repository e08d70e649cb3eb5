// A reference-style caller of the rlplan API:
// compiled against include/rlplan/*.hpp and linked with librrealloc.so.
// With -DREF_HEADERS_ONLY it uses only the declarations that exist in the
// reference's own proj/include headers, so it can be compiled against them.
#include <cstdio>
#include <iostream>

#ifdef REF_HEADERS_ONLY
#include "rlplan/cluster.hpp"
#include "rlplan/model_arith.hpp"
#else
#include "rlplan/realloc.hpp"
#endif

using namespace rlplan;

int main() {
  ClusterSpec box;
  box.n_nodes = 1;
  box.gpus_per_node = 8;
  box.mem_per_device = 180000000000LL;
  box.intra_node_bw = 900e9;
  box.inter_node_bw = 50e9;
  box.host_to_device_bw = 55e9;
  ModelSpec m;
  m.name = "llama7b";
  m.hidden_size = 4096;
  m.intermediate_size = 14336;
  m.num_layers = 32;
  m.num_attention_heads = 32;
  m.num_kv_heads = 8;
  m.vocab_size = 128256;
  m.max_position_embeddings = 8192;
  std::printf("param_count %lld %lld\n", (long long)param_count(m, true), (long long)param_count(m, false));
  std::printf("meshes %zu\n", enumerate_meshes(box).size());
  const DeviceMesh q = mesh_from_string("trainer01:gpu[4-7]", box);
  std::printf("mesh %s first %d\n", mesh_to_string(q, box).c_str(), q.first_device(box));
  try {
    mesh_from_string("trainer01:gpu[1-2]", box);
  } catch (const ValidationError& e) {
    std::printf("error %s\n", e.what());
  }
#ifndef REF_HEADERS_ONLY
  Placement train{mesh_from_string("trainer01", box), {1, 8, 1, 1}};
  Placement gen{mesh_from_string("trainer01", box), {8, 1, 1, 1}};
  const ReallocPlan plan = plan_param_realloc(m, train, gen, box);
  std::printf("plan ops %zu local %zu total %lld\n", plan.ops.size(), plan.local_ops.size(),
              (long long)plan.total_bytes);
  const auto stages = stage_layer_map(5, 2);
  std::printf("stages [%lld,%lld) [%lld,%lld)\n", (long long)stages[0].first, (long long)stages[0].second,
              (long long)stages[1].first, (long long)stages[1].second);
#endif
  return 0;
}
