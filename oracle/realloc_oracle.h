/*
 * TEST INFRASTRUCTURE — CPU oracle of the parameter-reallocation path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this. The product (librrealloc.so) never
 * links or calls it.
 *
 * Plain-C restatement of the reference algorithm:
 *   - parameter inventory: reference proj/src/model_arith.cpp:28-46
 *   - device order of a mesh: reference proj/src/cluster.cpp:23-30
 *   - link classes: reference proj/src/cluster.cpp:95-101
 *   - stage_layer_map: SPEC.md:560-568
 *   - plan_param_realloc: SPEC.md:569-577
 *   - CPU reallocation: executes the plan's ops with memcpy on host buffers
 *     (the "reference CPU reallocation" of BASELINE.json north_star; the
 *     reference itself moves no bytes)
 * plus the layout contract of DESIGN.md §3 (the reference leaves the byte
 * layout open), written independently of the product's block-intersection
 * lowering: here every element is addressed through a per-tensor address
 * function.
 *
 * Parity pinning: the arithmetic/topology parts are checked against the
 * reference's own C++ compiled from /root/reference (oracle/_ref); the plan is
 * checked against every SPEC example (tests/golden/spec_examples.json) and the
 * SPEC replay criterion. Byte-level layout decisions have no
 * reference fixture (the reference never materialises weights);
 * they are pinned against third-party code instead: vLLM's tensor-parallel
 * weight loaders (tests/golden/vllm_tp_shards.json) and HF transformers'
 * LLaMA parameter inventory (tests/golden/hf_llama_inventory.json).
 */
#ifndef REALLOC_ORACLE_H_
#define REALLOC_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_DST 64

typedef struct {
  int64_t hidden, ffn, layers, heads, kv_heads, vocab;
  int64_t param_bytes;
  int32_t has_output_head;
} orc_model;

typedef struct {
  int32_t n_nodes, gpus_per_node;
  double intra_bw, inter_bw;
} orc_cluster;

typedef struct {
  int32_t node_offset, node_count, gpu_offset, gpu_count;
  int32_t dp, tp, pp;
  int32_t qkv_layout;     /* 0 separate, 1 concat, 2 grouped */
  int32_t gate_up_layout; /* 0 separate, 1 concat */
  int32_t kv_layout;      /* 0 k/v rows split over tp, 1 whole KV heads replicated when tp > kv */
} orc_placement;

typedef struct {
  int32_t src;
  int32_t n_dst;
  int32_t dst[ORC_MAX_DST];
  int64_t layer_start, layer_end;
  int32_t slice, slices, replicated;
  int64_t bytes;
  int32_t part; /* 0 every split tensor, 1 all but k/v, 2 k/v only */
} orc_op;

int64_t orc_param_count(const orc_model* m, int include_output_embedding);
int orc_stage_layer_map(int64_t layers, int pp, int64_t* starts, int64_t* ends);
/* 0 ok, -1 invalid. */
int orc_plan(const orc_model* m, const orc_placement* src, const orc_placement* dst,
             const orc_cluster* c, int policy, orc_op* ops, int cap, int* n_ops, orc_op* local,
             int cap_local, int* n_local, int64_t* total_bytes, double* est_time);
int64_t orc_shard_bytes(const orc_model* m, const orc_placement* p, const orc_cluster* c, int dev);
/* bf16 bits of logical element `index` of `tensor`. Seed bit 62 selects the
 * special-value mode (signed zeros, infinities, quiet/signalling NaNs with
 * payloads, subnormals, extreme normals, arbitrary 16-bit words). */
#define ORC_SEED_SPECIAL (1ull << 62)
uint16_t orc_value(uint64_t seed, int64_t tensor, int64_t index);
/* Fill a device's shard (all held elements; padding untouched). */
int orc_fill(const orc_model* m, const orc_placement* p, const orc_cluster* c, int dev,
             uint64_t seed, uint16_t* buf);
/* Bytes [offset, offset + len) of a device's expected shard (padding zero),
 * element by element like orc_fill, with `threads` threads; offset and len
 * even and inside the shard. 0 ok, -1 invalid. */
int orc_fill_range(const orc_model* m, const orc_placement* p, const orc_cluster* c, int dev, uint64_t seed,
                   int64_t offset, int64_t len, uint16_t* buf, int threads);
/* Compare `got` (len bytes) with that window: *mismatches = differing bf16
 * elements (padding included), *first = first differing element index
 * within the window or -1. */
int orc_check_range(const orc_model* m, const orc_placement* p, const orc_cluster* c, int dev, uint64_t seed,
                    int64_t offset, int64_t len, const uint16_t* got, int threads, int64_t* mismatches,
                    int64_t* first);
/* CPU reallocation: run ops and local ops on host buffers indexed by device. */
int orc_execute(const orc_model* m, const orc_placement* src, const orc_placement* dst,
                const orc_cluster* c, const orc_op* ops, int n_ops, void* const* src_bufs,
                void* const* dst_bufs, int threads);

/* ---- inter-call data transfer: SPEC.md:578-586, PAPER.md:522 ----
 * DP indexes disjoint data slices (finest common slicing lcm(dp)), TP and PP
 * index replicas: every device of a DP group holds (producer) or needs
 * (consumer) that group's slices, so identical placements move nothing
 * (SPEC.md:584). Data elements are bf16 words of tensor id ORC_DATA_TENSOR. */
#define ORC_DATA_TENSOR 0x7fff0000
int orc_plan_data(const orc_placement* producer, const orc_placement* consumer, const orc_cluster* c,
                  int policy, int64_t data_bytes_per_dp_shard, orc_op* ops, int cap, int* n_ops,
                  orc_op* local, int cap_local, int* n_local, int64_t* total_bytes, double* est_time);
/* Bytes of a device's data buffer (0 if it holds/needs none). */
int64_t orc_data_shard_bytes(const orc_placement* p, const orc_cluster* c, int dev, int producer,
                             int64_t total_bytes);
int orc_data_fill(const orc_placement* p, const orc_cluster* c, int dev, int producer, int64_t total_bytes,
                  uint64_t seed, uint16_t* buf);
int orc_data_execute(const orc_placement* producer, const orc_placement* consumer, const orc_cluster* c,
                     int64_t total_bytes, const orc_op* ops, int n_ops, void* const* src_bufs,
                     void* const* dst_bufs);
/* The same with `threads` worker threads (1 MiB memcpy tasks). */
int orc_data_execute_mt(const orc_placement* producer, const orc_placement* consumer, const orc_cluster* c,
                        int64_t total_bytes, const orc_op* ops, int n_ops, void* const* src_bufs,
                        void* const* dst_bufs, int threads);

#ifdef __cplusplus
}
#endif

#endif
