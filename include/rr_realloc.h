/*
 * rr_realloc.h — C ABI of the B200 parameter-reallocation library
 * (paper_2406_14088_b200/librrealloc.so).
 *
 * The reference (arXiv 2406.14088, ReaL) exposes this path only as the C++
 * `rlplan` namespace (proj/include/rlplan/{common,model_arith,cluster}.hpp) plus the SPEC-declared
 * realloc module; its runtime executes plans with NCCL
 * broadcasts. This header is the flat, exception-free
 * boundary a foreign caller (Python ctypes, cgo, JNI, the upstream runtime's
 * C++ model worker) binds instead. Every entry point names the reference
 * interface it replaces. Plain pointers and sizes only; no torch or CUDA
 * types appear in the signatures (streams are passed as `void*` holding a
 * cudaStream_t, NULL = legacy default stream).
 *
 * Errors: every function returns rr_status; on failure rr_last_error()
 * returns a thread-local message. RR_EINVAL carries the text of the
 * reference's ValidationError (common.hpp:22-25).
 *
 * Threading: planning functions are pure and reentrant.
 * A plan is immutable once created and may be read concurrently. An
 * executor is bound to one CUDA device and one set of buffers; launches are
 * asynchronous and ordered on the caller's stream.
 */
#ifndef RR_REALLOC_H_
#define RR_REALLOC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RR_ABI_VERSION 5 /* 2: rr_placement.kv_layout, rr_shard.part; 3: rr_exec_options.ce_min_run_bytes; 4: staged gather;
                            5: rr_exec_options.ce_transport / ce_flags, rr_plan_ce_*, multicast member export */

typedef enum {
  RR_OK = 0,
  RR_EINVAL = 1,       /* ValidationError or bad argument */
  RR_ECUDA = 2,        /* CUDA runtime/driver error */
  RR_ENOMEM = 3,       /* allocation failed */
  RR_EUNSUPPORTED = 4, /* feature absent on this device (e.g. multicast) */
  RR_ETIMEOUT = 5,     /* cross-GPU barrier did not complete */
  RR_ERANGE = 6        /* caller buffer too small; *needed says how large */
} rr_status;

/* ---- vocabulary (reference model_arith.hpp:13-35, cluster.hpp:14-41) ---- */

typedef struct {
  const char* name; /* may be NULL */
  int64_t hidden_size;
  int64_t intermediate_size;
  int64_t num_layers;
  int64_t num_attention_heads;
  int64_t num_kv_heads;
  int64_t vocab_size;
  int64_t max_position_embeddings;
  int64_t param_bytes;
  int64_t grad_bytes;
  int64_t optimizer_bytes_per_param;
  int32_t has_output_head;
} rr_model;

typedef struct {
  int32_t n_nodes;
  int32_t gpus_per_node;
  int64_t mem_per_device;
  double intra_node_bw;
  double inter_node_bw;
  double host_to_device_bw;
} rr_cluster;

typedef struct {
  int32_t node_offset;
  int32_t node_count;
  int32_t gpu_offset;
  int32_t gpu_count;
} rr_mesh;

/* qkv_layout: 0 separate, 1 concat [Q;K;V], 2 Megatron grouped.
 * gate_up_layout: 0 separate, 1 concat [G;U]. (DESIGN.md §3 G4)
 * kv_layout: 0 k/v rows split over tp, 1 whole KV heads replicated when
 * tp > kv heads (Megatron / vLLM). (DESIGN.md §3 G6) */
typedef struct {
  rr_mesh mesh;
  int32_t dp, tp, pp, n_microbatches;
  int32_t qkv_layout;
  int32_t gate_up_layout;
  int32_t kv_layout;
} rr_placement;

typedef struct { /* SPEC.md:547-549; layers -1 and L are embed / final+head */
  int64_t layer_start;
  int64_t layer_end;
  int32_t tp_rank;
  int32_t tp_degree;
  int32_t replicated;
  int32_t part; /* 0 every TP-split tensor, 1 all but k/v, 2 k/v only (G6) */
} rr_shard;

typedef struct {
  int32_t src;
  int32_t n_dst;
  const int32_t* dst; /* valid for the plan's lifetime */
  rr_shard payload;
  int64_t bytes;
} rr_op;

typedef struct rr_plan rr_plan;
typedef struct rr_exec rr_exec;
typedef struct rr_barrier rr_barrier;

const char* rr_last_error(void);
int rr_abi_version(void);

/* ---- model-arith (reference model_arith.hpp:37-72) ---- */
rr_status rr_model_validate(const rr_model* m);                                 /* ModelSpec::validate, model_arith.hpp:31 */
rr_status rr_param_count(const rr_model* m, int include_output_embedding, int64_t* out); /* model_arith.hpp:42 */
rr_status rr_natural_param_count(const rr_model* m, int64_t* out);              /* model_arith.hpp:46 */
rr_status rr_flops(const rr_model* m, int backward, int64_t tokens, int64_t context_len, double* out); /* model_arith.hpp:54 */
rr_status rr_layer_flops_fwd(const rr_model* m, int64_t tokens, int64_t context_len, double* out);     /* model_arith.hpp:57 */
rr_status rr_kv_cache_bytes(const rr_model* m, int64_t batch, int64_t seq_len, int64_t* out);          /* model_arith.hpp:60 */
rr_status rr_logits_bytes(int64_t vocab, int64_t batch, int64_t ctx_len, int64_t elem_bytes, int64_t* out); /* model_arith.hpp:63 */
rr_status rr_static_param_bytes(const rr_model* m, int64_t* params, int64_t* grads, int64_t* optimizer); /* model_arith.hpp:72 */

/* ---- cluster-topo (reference cluster.hpp:14-63) ---- */
rr_status rr_cluster_validate(const rr_cluster* c);                             /* ClusterSpec::validate, cluster.hpp:23 */
rr_status rr_validate_mesh(const rr_mesh* m, const rr_cluster* c);               /* cluster.hpp:45 */
rr_status rr_mesh_devices(const rr_mesh* m, const rr_cluster* c, int32_t* out, int cap, int* n); /* DeviceMesh::devices, cluster.hpp:38 */
rr_status rr_mesh_contains(const rr_mesh* m, const rr_cluster* c, int32_t device, int* out);      /* DeviceMesh::contains, cluster.hpp:40 */
rr_status rr_enumerate_meshes(const rr_cluster* c, rr_mesh* out, int cap, int* n);             /* cluster.hpp:49 */
rr_status rr_overlap(const rr_mesh* a, const rr_mesh* b, const rr_cluster* c, int* out);        /* cluster.hpp:51 */
rr_status rr_link_bandwidth(const rr_cluster* c, int32_t a, int32_t b, double* out);            /* cluster.hpp:55 */
rr_status rr_mesh_to_string(const rr_mesh* m, const rr_cluster* c, char* buf, size_t cap, size_t* needed); /* cluster.hpp:62 */
rr_status rr_mesh_from_string(const char* text, const rr_cluster* c, rr_mesh* out);            /* cluster.hpp:63 */

/* ---- realloc planning ---- */
rr_status rr_stage_layer_map(int64_t num_layers, int pp, int64_t* starts, int64_t* ends);
rr_status rr_validate_placement(const rr_model* m, const rr_placement* p, const rr_cluster* c);
/* policy: 0 = SPEC tie-break (lowest id), 1 = balanced egress. */
rr_status rr_plan_create(const rr_model* m, const rr_placement* src, const rr_placement* dst,
                         const rr_cluster* c, int policy, rr_plan** out);                     /* plan_param_realloc */
/* plan_data_transfer: inter-call data, DP-partitioned on
 * the producer's last stage, re-sliced at lcm(dp) for every consumer device.
 * The resulting plan executes like a parameter plan (rr_exec_*); its shard
 * layout is one 1-D bf16 block per device (tensor id 0x7fff0000). */
rr_status rr_plan_create_data(const rr_placement* producer, const rr_placement* consumer,
                              const rr_cluster* c, int64_t data_bytes_per_dp_shard, int policy,
                              rr_plan** out);
void rr_plan_destroy(rr_plan* plan);
rr_status rr_plan_totals(const rr_plan* plan, int64_t* total_bytes, double* est_time);
rr_status rr_plan_num_ops(const rr_plan* plan, int local, int* n);
rr_status rr_plan_get_op(const rr_plan* plan, int local, int index, rr_op* out);
rr_status rr_plan_to_json(const rr_plan* plan, char* buf, size_t cap, size_t* needed);        /* realloc-plan */
/* side 0 = source placement, 1 = destination placement. 0 bytes if the
 * device is not part of that placement. */
rr_status rr_plan_shard_bytes(const rr_plan* plan, int side, int32_t device, int64_t* bytes);
/* Per-device traffic of the lowered plan (bytes): over links in/out, and
 * copied locally (src and dst on the same device). */
rr_status rr_plan_device_traffic(const rr_plan* plan, int32_t device, int64_t* wire_in,
                                 int64_t* wire_out, int64_t* local);
rr_status rr_plan_num_rects(const rr_plan* plan, int64_t* n);
/* Shard layout block table for (side, device): 6 int64 per block
 * {tensor, r0, r1, c0, c1, offset}. */
rr_status rr_plan_layout(const rr_plan* plan, int side, int32_t device, int64_t* out, int64_t cap_blocks,
                         int64_t* n_blocks);

/* Lowered plan inspection (host only): op i of the merged (remote + local)
 * list has source *src, destinations dst[0..*n_dst) (cap 64) and *n_rects
 * copy rectangles, 6 int64 each {src_off, dst_off, row_bytes, src_pitch,
 * dst_pitch, rows}; pass rects = NULL to query *n_rects. */
rr_status rr_plan_num_lowered(const rr_plan* plan, int* n);
rr_status rr_plan_get_lowered(const rr_plan* plan, int index, int32_t* src, int32_t* dst, int* n_dst,
                              int64_t* rects, int64_t cap_rects, int64_t* n_rects);
/* Work an executor driving `local` (with `host_of`, see rr_exec_create)
 * would do, host only, no CUDA. out6 = {phase-0 bytes read, phase-0 bytes
 * written, phase-1 bytes read, phase-1 bytes written, bytes entering this
 * host over links, bytes leaving it}. */
rr_status rr_plan_work(const rr_plan* plan, int n_local, const int32_t* local, const int32_t* host_of,
                       int mode, int64_t* out6);

/* ---- device memory and peer mapping (plumbing) ---- */
rr_status rr_device_count(int* n);
rr_status rr_device_alloc(int cuda_device, size_t bytes, void** out);
rr_status rr_device_free(void* ptr);
rr_status rr_host_alloc(size_t bytes, void** out); /* pinned */
rr_status rr_host_free(void* ptr);
/* kind: 0 host->device, 1 device->host, 2 device->device. */
rr_status rr_memcpy(void* dst, const void* src, size_t bytes, int kind, void* stream, int synchronous);
rr_status rr_memset(void* dst, int value, size_t bytes, void* stream);
rr_status rr_stream_sync(void* stream);
rr_status rr_ipc_handle(void* device_ptr, void* handle64);            /* 64-byte cudaIpcMemHandle */
rr_status rr_ipc_open(int cuda_device, const void* handle64, void** out);
rr_status rr_ipc_close(void* ptr);
rr_status rr_enable_peer(int cuda_device, int peer_device);

/* ---- execution: the B200 replacement of the upstream NCCL-broadcast
 *      executor ----
 *
 * src_bufs / dst_bufs are indexed by global DeviceId (n_devices entries,
 * NULL where unused) and must be addressable from `cuda_device` (local
 * allocations, or IPC-opened / peer-enabled pointers). `local` lists the
 * plan devices whose SMs this executor drives (the plan devices hosted on
 * cuda_device). host_of[d] (NULL = every non-local device is its own host)
 * names the GPU hosting plan device d: a payload bound for several devices
 * of one remote host crosses NVLink once, into the lowest-id one (phase 0),
 * and that host replicates it locally (phase 1, rr_exec_launch_fanout,
 * after a cross-GPU barrier).
 * mode 0 = PUSH: a local source reads its shard once and stores every
 *          destination copy (local relayout + NVLink peer stores, K1/K2).
 * mode 1 = PULL: a local destination loads from the (possibly remote)
 *          source and stores locally.
 * chunk_bytes: work-item granularity. 0 = library default: 256 KiB, except
 * that a plain phase too small for that is cut into ~16 items per resident
 * bulk CTA (>= 32 KiB), or ~1 item per CTA below 64 MiB stored (>= 4 KiB). */
rr_status rr_exec_create(const rr_plan* plan, int cuda_device, int n_devices,
                         void* const* src_bufs, void* const* dst_bufs, int n_local,
                         const int32_t* local, const int32_t* host_of, int mode, int64_t chunk_bytes,
                         rr_exec** out);
/* Phase 0 (all direct copies). ctas = 0 picks the resident-CTA capacity. */
rr_status rr_exec_launch(rr_exec* ex, void* stream, int ctas);
/* Phase 1 (in-host fan-out from leader replicas); no-op when empty. */
rr_status rr_exec_launch_fanout(rr_exec* ex, void* stream, int ctas);
/* Copy kernel: 0 = vectorised LDG/STG kernel; 1 or 5 = TMA bulk-copy ring
 * (cp.async.bulk through shared-memory stages; 1 = 4 x 16 KiB stages, the
 * default; 5 = 3 x 16 KiB stages). Other values: RR_EINVAL.
 * 2-byte-aligned and multicast items always take the LDG/STG kernel.
 * Without this call, a plain phase storing fewer than the small-phase bytes
 * (default 64 MiB, rr_exec_set_small_phase_bytes; 0 = never) takes the
 * LDG/STG kernel: few items, latency-bound. */
rr_status rr_exec_set_kernel(rr_exec* ex, int kernel);
rr_status rr_exec_set_small_phase_bytes(rr_exec* ex, int64_t bytes);
/* The same for flag-synchronised phases (relay chains, overlapped fan-out),
 * which run as one kernel: the bulk variant when every item is TMA-eligible,
 * else the LDG/STG kernel. Default 5. */
rr_status rr_exec_set_flag_kernel(rr_exec* ex, int kernel);
/* Per phase: items, bytes stored (sum over destinations), bytes read. */
rr_status rr_exec_stats(const rr_exec* ex, int phase, int64_t* items, int64_t* bytes_written,
                        int64_t* bytes_read);
/* Onload of parked parameters pipelined with the reallocation (PAPER.md:514:
 * host<->device copies on an additional stream). enable: the local source
 * shards src_devices[i] are onloaded (their first src_bytes[i] bytes) in
 * chunk_bytes pieces, in this order; phase-0 copies are regrouped by the
 * last chunk they read. launch: H2D copies on copy_stream from
 * host_bufs[device] (pinned) into the executor's source buffers, each
 * phase-0 segment launched on `stream` as soon as its chunk has landed. */
rr_status rr_exec_enable_onload(rr_exec* ex, int n_src, const int32_t* src_devices, const int64_t* src_bytes,
                                int64_t chunk_bytes);
rr_status rr_exec_launch_onload(rr_exec* ex, void* const* host_bufs, void* copy_stream, void* stream, int ctas);
/* Offload of parameters being parked ("host-device (e.g.,
 * offload)"; SPEC.md:423 offload nodes): the local source shards
 * src_devices[i] (their first src_bytes[i] bytes) are copied device->host
 * into host_bufs[device] (pinned) on copy_stream, starting once the work
 * already on `stream` is done. A reallocation launched on `stream` after
 * this call overlaps the copies: both only read the sources. The caller
 * must order any later write to those source buffers after copy_stream. */
rr_status rr_exec_launch_offload(rr_exec* ex, int n_src, const int32_t* src_devices, const int64_t* src_bytes,
                                 void* const* host_bufs, void* copy_stream, void* stream);
/* Kernels one rr_exec_launch / rr_exec_launch_fanout issues (0..2 each). */
rr_status rr_exec_kernel_count(const rr_exec* ex, int* phase0, int* phase1);
/* Which kernels a phase launches: *ldst = 1 if the LDG/STG kernel runs,
 * *bulk = the TMA bulk variant that runs (0 = none). */
rr_status rr_exec_phase_kernels(const rr_exec* ex, int phase, int* ldst, int* bulk);
/* Bytes entering / leaving this executor's host over links per launch. */
rr_status rr_exec_wire(const rr_exec* ex, int64_t* wire_in, int64_t* wire_out);
void rr_exec_destroy(rr_exec* ex);

/* Executor options (superset of rr_exec_create's arguments).
 * mc_bufs[d] (NULL table = no multicast): the NVLS multicast address whose
 * member buffers are the destination shards of one plan device per host
 * (rr_mcast_bind). A payload whose destination hosts are exactly that
 * group is stored once through multimem.st and replicated by the NVSwitch
 * (push mode, K3) instead of one peer store per host. */
typedef struct {
  int32_t mode;               /* 0 push, 1 pull */
  int64_t chunk_bytes;        /* 0 = 256 KiB */
  const int32_t* host_of;     /* NULL = flat delivery */
  void* const* mc_bufs;       /* NULL = no multicast */
  /* Pipelined relay (push, hierarchical): relay_flags[d] = the uint32 flag
   * array (rr_plan_relay_slots entries, mapped here) of plan device d's host.
   * Each array belongs to exactly one executor per host and must be zero when
   * that executor is created (epochs restart at 1 in every executor, so stale
   * values would release waits early): rr_exec_create_ex reads this host's
   * array and fails with RR_EINVAL if it is not zero. A payload reaching >= 2 other hosts then travels
   * source -> host 1 -> host 2 ... chunk by chunk, each host forwarding and
   * fanning out locally as chunks land. NULL = no relay. */
  void* const* relay_flags;
  int32_t relay_chain;    /* with relay_flags: chain relay for >= 2 remote hosts */
  int32_t overlap_fanout; /* with relay_flags: per-chunk in-host fan-out inside phase 0 */
  /* Copy-engine runs (push mode): where a local source shard and a remote
   * destination shard hold the same blocks at the same relative offsets over
   * >= this many bytes, and the plan moves (>= 98% of) that range between
   * them, phase 0 moves it with one copy-engine copy (cudaMemcpyAsync on a
   * side stream, forked from and joined back into the launch stream) instead
   * of SM peer stores. 0 = default (256 MiB), < 0 = never. */
  int64_t ce_min_run_bytes;
  /* Staged gather (ABI v4; pull mode with host_of, host ids 0..n_hosts-1):
   * every remote source shard this host reads is pushed whole by its host's
   * copy engine into a staging buffer here, in stage_chunk_bytes pieces,
   * in rounds that pair each host with one sender at a time
   * (rr_plan_stage_slots); each piece is flagged in the receiver's stage
   * flag array and the unpack items here wait per piece. src_bufs[d] of a
   * remote source d is this host's staging buffer for d.
   * stage_remote[d * n_hosts + h]: host h's staging buffer for local source
   * d, mapped here (NULL where h does not read d). stage_flags[h]: host h's
   * stage flag array (rr_plan_stage_slots uint32), mapped here; same
   * ownership rule as relay_flags (zero at create, one executor per array).
   * Each piece's flag is written by the sender's copy stream
   * (cuStreamWriteValue32 after the copy), never by a kernel, so spinning
   * unpack CTAs cannot starve it. stage_chunk_bytes = 0: off. */
  int64_t stage_chunk_bytes;
  int32_t n_hosts;
  void* const* stage_remote;
  void* const* stage_flags;
  /* Copy-engine transport (ABI v5; push mode): every remote destination of
   * the plain phase-0 work moves by copy engine straight into the
   * destination shard — the per-layer pieces of one tensor kind merged into
   * one cudaMemcpy2DAsync (contiguous pieces, rows = layers) or one
   * cudaMemcpy3DAsync (row-parallel pieces) per (source, destination) —
   * issued on a side stream in rotation rounds (round r to the host r places
   * after this one), beside the SM kernel that does the local copies. No
   * staging, no unpack pass. Copy engines carry more payload per NVLink byte
   * than SM stores (~780 vs ~710 GB/s). Excludes relay / overlapped fan-out
   * jobs (they stay on SM stores); copy-engine runs are not used with it.
   * 0 = off; 1 = on; 2 = hybrid: row-parallel pieces whose layers do not
   * merge into one 3D copy (per-layer 2D copies) stay on SM peer stores
   * beside the copy engines; 3 = on, and payloads reaching >= 2 other hosts
   * travel host to host by copy engines in <= 256 MiB pieces (copy-engine
   * relay; needs ce_flags). */
  int32_t ce_transport;
  /* Copy flags (with ce_transport; host ids 0..n_hosts-1): ce_flags[h] =
   * host h's copy flag array (rr_plan_ce_slots uint32, mapped here; zero at
   * create, one executor per array). With them the transport copies follow
   * a global schedule (no receiver takes two senders at once): a transfer
   * waits on this host's array (cuStreamWaitValue32) for the previous
   * transfer into its receiver, whose sender raises it after its last copy
   * (cuStreamWriteValue32). With overlap_fanout also set (copy-engine star),
   * every copy raises a slot on the receiving host and that host's in-host
   * fan-out runs inside phase 0, each item waiting for the copy that filled
   * the leader bytes it reads. NULL = rotation order only, fan-out in
   * phase 1. */
  void* const* ce_flags;
} rr_exec_options;
/* Length of the relay flag array for this host map, chunk size and scheme
 * switches (identical on every rank). */
rr_status rr_plan_relay_slots(const rr_plan* plan, const int32_t* host_of, int64_t chunk_bytes, int relay_chain,
                              int overlap_fanout, int64_t* slots);
/* Staged gather: length of the stage flag array every host allocates (the
 * maximum over hosts of its pieces, then one round token per host: round r's
 * push into a receiver waits, on the copy stream, for the round r-1 sender
 * into that receiver to finish) for this host map and piece size. */
rr_status rr_plan_stage_slots(const rr_plan* plan, const int32_t* host_of, int64_t chunk_bytes, int64_t* slots);
/* Copy-engine runs a push executor driving `local` (with `host_of`) would
 * issue, host only: 5 int64 per run {src device, dst device, src byte
 * offset, dst byte offset, bytes}; pass out5 = NULL to query *n. */
rr_status rr_plan_ce_runs(const rr_plan* plan, int n_local, const int32_t* local, const int32_t* host_of,
                          int64_t min_run_bytes, int64_t* out5, int cap, int* n);
/* Copy-engine transport copies a push executor driving `local` (with
 * `host_of`) would issue, host only, in issue order: 11 int64 per copy {src
 * device, dst device, src offset, dst offset, width, height, depth, src
 * pitch, dst pitch, src slice stride, dst slice stride}; out11 = NULL
 * queries *n. */
rr_status rr_plan_ce_copies(const rr_plan* plan, int n_local, const int32_t* local, const int32_t* host_of,
                            int64_t* out11, int cap, int* n);
/* Copy flags: length of the copy flag array every host allocates (maximum
 * over hosts of its incoming copy slots plus its schedule waits). */
rr_status rr_plan_ce_slots(const rr_plan* plan, const int32_t* host_of, int64_t* slots);
/* The copy-engine schedule of every host (host only): 6 doubles per
 * transfer {sender host, receiver host, simulated start s, end s, waits for
 * another sender (0/1), bytes}, each sender's transfers in issue order;
 * out6 = NULL queries *n. */
rr_status rr_plan_ce_schedule(const rr_plan* plan, const int32_t* host_of, double* out6, int cap, int* n);
/* Staged-gather pieces this executor pushes per launch, and their bytes. */
rr_status rr_exec_stage_pushes(const rr_exec* ex, int* n_pushes, int64_t* bytes);
/* Copy-engine submissions phase 0 issues (copy-engine runs, see
 * rr_exec_options.ce_min_run_bytes, or copy-engine transport copies). */
rr_status rr_exec_ce_runs(const rr_exec* ex, int* n_runs, int64_t* bytes);
/* Relay waits that timed out (bounded spins) since the executor was created. */
rr_status rr_exec_relay_timeouts(rr_exec* ex, int64_t* timeouts);
rr_status rr_exec_create_ex(const rr_plan* plan, int cuda_device, int n_devices, void* const* src_bufs,
                            void* const* dst_bufs, int n_local, const int32_t* local,
                            const rr_exec_options* options, rr_exec** out);

/* ---- NVLS multicast objects (K3), one process per GPU ----
 * root: rr_mcast_create -> POSIX fd + padded size (share the fd with the
 * other ranks, e.g. SCM_RIGHTS); others: rr_mcast_import(fd); then, after
 * every rank has created/imported (a barrier), each rank rr_mcast_bind:
 * local physical memory bound into the object, mapped twice — a unicast
 * address (ordinary loads/stores on this GPU) and the multicast address
 * (multimem stores reach every member). */
typedef struct rr_mcast rr_mcast;
rr_status rr_mcast_supported(int cuda_device, int* supported);
rr_status rr_mcast_create(int cuda_device, size_t bytes, int n_devices, int* fd_out, size_t* size_out,
                          rr_mcast** out);
rr_status rr_mcast_import(int cuda_device, int fd, size_t size, int n_devices, rr_mcast** out);
rr_status rr_mcast_bind(rr_mcast* m, void** unicast_ptr, void** multicast_ptr);
rr_status rr_mcast_size(const rr_mcast* m, size_t* size);
void rr_mcast_destroy(rr_mcast* m);
/* A bound member reached by the other GPUs through ordinary peer stores
 * (schemes that do not use the multicast address): export its physical
 * memory as a POSIX fd; a peer imports and maps it (read/write from
 * cuda_device) and closes the mapping with rr_peer_mem_close. */
typedef struct rr_peer_mem rr_peer_mem;
rr_status rr_mcast_export_member(rr_mcast* m, int* fd_out);
rr_status rr_peer_mem_import(int cuda_device, int fd, size_t size, void** ptr, rr_peer_mem** out);
void rr_peer_mem_close(rr_peer_mem* p);

/* ---- deterministic weights (test/bench infrastructure) ----
 * Fill or check a device's shard under one side of a plan with
 * bf16 value = hash(seed, tensor_id, logical_index). Seeds with
 * RR_SEED_SPECIAL set draw special bf16 words instead (signed zeros,
 * infinities, quiet and signalling NaNs with payloads, subnormals, extreme
 * normals, arbitrary 16-bit patterns). */
#define RR_SEED_SPECIAL (1ull << 62)
rr_status rr_fill_shard(const rr_plan* plan, int side, int32_t device, void* buf, uint64_t seed,
                        void* stream);
/* Synchronous; *mismatches = number of differing elements, *first = buffer
 * element index of the first difference (or -1). */
rr_status rr_verify_shard(const rr_plan* plan, int side, int32_t device, const void* buf,
                          uint64_t seed, void* stream, int64_t* mismatches, int64_t* first);
/* Host-side reference of the value function (for KATs). */
uint16_t rr_weight_value(uint64_t seed, int64_t tensor_id, int64_t logical_index);

/* ---- cross-GPU barrier for one-process-per-GPU execution ----
 * flags[p] = rank p's flag array (world uint32), mapped into this process. */
rr_status rr_barrier_create(int cuda_device, int rank, int world, void* const* flags,
                            rr_barrier** out);
rr_status rr_barrier_launch(rr_barrier* b, void* stream);
/* Nonzero *timed_out if any launch gave up waiting (bounded spin). */
rr_status rr_barrier_status(rr_barrier* b, int* timed_out);
void rr_barrier_destroy(rr_barrier* b);

#ifdef __cplusplus
}
#endif

#endif /* RR_REALLOC_H_ */
