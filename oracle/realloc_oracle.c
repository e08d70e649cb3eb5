/*
 * TEST INFRASTRUCTURE — CPU oracle of the parameter-reallocation path.
 * See realloc_oracle.h for what is restated from where and who may use it.
 */
#include "realloc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- tensor inventory: reference proj/src/model_arith.cpp:28-46 ---------- */

enum { SPLIT_ROWS = 0, SPLIT_COLS = 1, REPLICATED = 2 };
enum { K_LN1, K_Q, K_K, K_V, K_O, K_LN2, K_GATE, K_UP, K_DOWN };

typedef struct {
  int64_t rows, cols, layer; /* layer: -1 embed, L final */
  int split;
} tensor_shape;

static int64_t n_tensors(const orc_model* m) { return 3 + 9 * m->layers; }

static tensor_shape shape_of(const orc_model* m, int64_t id) {
  const int64_t h = m->hidden, hd = m->hidden / m->heads;
  tensor_shape s = {1, h, 0, REPLICATED};
  if (id == 0) {
    s.rows = m->vocab; s.layer = -1; s.split = SPLIT_ROWS;
    return s;
  }
  if (id == 1 + 9 * m->layers) { s.layer = m->layers; return s; } /* final norm [1,h] */
  if (id == 2 + 9 * m->layers) {
    s.layer = m->layers;
    if (m->has_output_head) { s.rows = m->vocab; s.split = SPLIT_ROWS; }
    return s; /* vocab head [V,h] or scalar head [1,h] */
  }
  s.layer = (id - 1) / 9;
  switch ((id - 1) % 9) {
    case K_LN1: case K_LN2: break;
    case K_Q: s.rows = m->heads * hd; s.split = SPLIT_ROWS; break;
    case K_K: case K_V: s.rows = m->kv_heads * hd; s.split = SPLIT_ROWS; break;
    case K_O: s.rows = h; s.cols = m->heads * hd; s.split = SPLIT_COLS; break;
    case K_GATE: case K_UP: s.rows = m->ffn; s.split = SPLIT_ROWS; break;
    case K_DOWN: s.rows = h; s.cols = m->ffn; s.split = SPLIT_COLS; break;
  }
  return s;
}

int64_t orc_param_count(const orc_model* m, int include_output_embedding) {
  /* Sum of every tensor (the shape-summation oracle of SPEC.md:47). */
  int64_t total = 0;
  for (int64_t id = 0; id < n_tensors(m); ++id) {
    const tensor_shape s = shape_of(m, id);
    if (id == 2 + 9 * m->layers && m->has_output_head && !include_output_embedding) continue;
    total += s.rows * s.cols;
  }
  if (include_output_embedding && !m->has_output_head) total += m->vocab * m->hidden;
  return total;
}

/* ---- stage map: SPEC.md:560-568 ------------------------------------------- */

int orc_stage_layer_map(int64_t layers, int pp, int64_t* starts, int64_t* ends) {
  if (pp < 1 || pp > layers) return -1;
  int64_t at = 0;
  for (int s = 0; s < pp; ++s) {
    const int64_t n = layers / pp + (s < layers % pp ? 1 : 0);
    starts[s] = at;
    ends[s] = at + n;
    at += n;
  }
  return 0;
}

/* Extended layer range [lo, hi) of stage s (embedding on the first stage,
 * final norm + head on the last). */
static void stage_range(const orc_model* m, int pp, int s, int64_t* lo, int64_t* hi) {
  int64_t st[256], en[256];
  orc_stage_layer_map(m->layers, pp, st, en);
  *lo = s == 0 ? -1 : st[s];
  *hi = s == pp - 1 ? m->layers + 1 : en[s];
}

/* ---- placements: rank order over reference cluster.cpp:23-30 ------------ */

static int mesh_size(const orc_placement* p) { return p->node_count * p->gpu_count; }

static int mesh_device(const orc_placement* p, const orc_cluster* c, int idx) {
  const int node = idx / p->gpu_count, gpu = idx % p->gpu_count;
  return (p->node_offset + node) * c->gpus_per_node + p->gpu_offset + gpu;
}

static int device_at(const orc_placement* p, const orc_cluster* c, int pp, int dp, int tp) {
  return mesh_device(p, c, (pp * p->dp + dp) * p->tp + tp);
}

/* -1 if d is not in the placement. */
static int rank_of(const orc_placement* p, const orc_cluster* c, int d, int* pp, int* dp, int* tp) {
  for (int i = 0; i < mesh_size(p); ++i) {
    if (mesh_device(p, c, i) != d) continue;
    *tp = i % p->tp;
    *dp = (i / p->tp) % p->dp;
    *pp = i / (p->tp * p->dp);
    return 0;
  }
  return -1;
}

/* Mesh shape rules of reference cluster.cpp:43-61, placement rules of
 * SPEC.md:261/268 and the layout codes of DESIGN.md §3. */
static int mesh_ok(const orc_placement* p, const orc_cluster* c) {
  const int M = c->gpus_per_node;
  if (p->node_count < 1 || p->gpu_count < 1 || p->node_offset < 0 || p->gpu_offset < 0) return 0;
  if (p->node_offset + p->node_count > c->n_nodes || p->gpu_offset + p->gpu_count > M) return 0;
  if (p->gpu_count == M ? p->gpu_offset != 0
                        : (p->node_count != 1 || M % p->gpu_count || p->gpu_offset % p->gpu_count))
    return 0;
  if (p->dp < 1 || p->tp < 1 || p->pp < 1) return 0;
  return p->dp * p->tp * p->pp == mesh_size(p);
}

static int placement_ok(const orc_model* m, const orc_placement* p, const orc_cluster* c) {
  if (!mesh_ok(p, c)) return 0;
  if (p->qkv_layout < 0 || p->qkv_layout > 2 || p->gate_up_layout < 0 || p->gate_up_layout > 1) return 0;
  if (p->pp > m->layers || (p->tp & (p->tp - 1)) || m->heads % p->tp) return 0;
  if (p->qkv_layout == 2 && m->kv_heads % p->tp) return 0;
  if (p->kv_layout < 0 || p->kv_layout > 1) return 0;
  if (p->kv_layout == 1 && p->tp > m->kv_heads && p->tp % m->kv_heads) return 0;
  return 1;
}

/* Distinct K/V slices over the TP ranks (DESIGN.md §3 G6): whole KV heads
 * when they are replicated and tp exceeds them, else one slice per rank. */
static int kv_slices(const orc_model* m, const orc_placement* p) {
  return p->kv_layout == 1 && p->tp > m->kv_heads ? (int)m->kv_heads : p->tp;
}

static int is_kv(const orc_model* m, int64_t id) {
  if (id < 1 || id > 9 * m->layers) return 0;
  const int kind = (int)((id - 1) % 9);
  return kind == K_K || kind == K_V;
}

/* reference cluster.cpp:95-101 */
static double bandwidth(const orc_cluster* c, int a, int b) {
  if (a == b) return INFINITY;
  return a / c->gpus_per_node == b / c->gpus_per_node ? c->intra_bw : c->inter_bw;
}

/* ---- plan: SPEC.md:569-577 ------------------------------------------------ */

/* Whether tensor id travels in a payload of this kind (part: 0 every split
 * tensor, 1 all but k/v, 2 k/v only). */
static int in_part(const orc_model* m, int64_t id, int replicated, int part) {
  const tensor_shape s = shape_of(m, id);
  if ((s.split == REPLICATED) != replicated) return 0;
  if (replicated || part == 0) return 1;
  return (part == 2) == is_kv(m, id);
}

static int64_t range_bytes(const orc_model* m, int64_t lo, int64_t hi, int replicated, int64_t slices, int part) {
  int64_t n = 0;
  for (int64_t id = 0; id < n_tensors(m); ++id) {
    const tensor_shape s = shape_of(m, id);
    if (s.layer < lo || s.layer >= hi) continue;
    if (!in_part(m, id, replicated, part)) continue;
    n += s.rows * s.cols / (replicated ? 1 : slices);
  }
  return n * m->param_bytes;
}

static int64_t gcd64(int64_t a, int64_t b) {
  while (b) { const int64_t t = a % b; a = b; b = t; }
  return a;
}

typedef struct {
  orc_op* list;
  int cap, n;
} op_list;

static int add_need(op_list* L, int src, int dst, int64_t lo, int64_t hi, int k, int G, int rep, int part,
                    int64_t bytes) {
  for (int i = 0; i < L->n; ++i) {
    orc_op* op = &L->list[i];
    if (op->src == src && op->layer_start == lo && op->layer_end == hi && op->slice == k &&
        op->slices == G && op->replicated == rep && op->part == part) {
      if (op->n_dst >= ORC_MAX_DST) return -1;
      op->dst[op->n_dst++] = dst;
      return 0;
    }
  }
  if (L->n >= L->cap) return -1;
  orc_op* op = &L->list[L->n++];
  memset(op, 0, sizeof(*op));
  op->src = src; op->n_dst = 1; op->dst[0] = dst;
  op->layer_start = lo; op->layer_end = hi;
  op->slice = k; op->slices = G; op->replicated = rep; op->part = part; op->bytes = bytes;
  return 0;
}

/* Cheapest holder: self, else the best link class; ties by
 * lowest id (policy 0) or least egress so far then lowest id (policy 1). */
static int pick_source(const orc_cluster* c, const int* holders, int nh, int d, int policy,
                       int64_t* egress, int64_t bytes) {
  double best = -1;
  for (int i = 0; i < nh; ++i) if (holders[i] == d) return d;
  for (int i = 0; i < nh; ++i) {
    const double bw = bandwidth(c, holders[i], d);
    if (bw > best) best = bw;
  }
  int pick = -1;
  for (int i = 0; i < nh; ++i) {
    if (bandwidth(c, holders[i], d) != best) continue;
    if (pick < 0 || (policy == 1 && egress[holders[i]] < egress[pick])) pick = holders[i];
    if (policy == 0) break;
  }
  egress[pick] += bytes;
  return pick;
}

static int cmp_int(const void* a, const void* b) { return *(const int*)a - *(const int*)b; }

int orc_plan(const orc_model* m, const orc_placement* src, const orc_placement* dst,
             const orc_cluster* c, int policy, orc_op* ops, int cap, int* n_ops, orc_op* local,
             int cap_local, int* n_local, int64_t* total_bytes, double* est_time) {
  if (!placement_ok(m, src, c) || !placement_ok(m, dst, c)) return -1;
  const int G = (int)(src->tp / gcd64(src->tp, dst->tp) * dst->tp);
  /* K/V travel separately when either side replicates KV heads (G6). */
  const int e1 = kv_slices(m, src), e2 = kv_slices(m, dst);
  const int kv_sep = e1 != src->tp || e2 != dst->tp;
  const int Gkv = (int)(e1 / gcd64(e1, e2) * e2);
  const int split_part = kv_sep ? 1 : 0;
  for (int64_t id = 0; id < n_tensors(m); ++id) {
    const tensor_shape s = shape_of(m, id);
    if (kv_sep && is_kv(m, id)) {
      if (s.rows % Gkv) return -1;
      continue;
    }
    if (s.split == SPLIT_ROWS && s.rows % G) return -1;
    if (s.split == SPLIT_COLS && s.cols % G) return -1;
  }
  const int n_dev = c->n_nodes * c->gpus_per_node;
  int64_t* egress = calloc((size_t)n_dev, sizeof(int64_t));
  int* holders = malloc(sizeof(int) * (size_t)n_dev);
  op_list R = {ops, cap, 0}, Lc = {local, cap_local, 0};
  int rc = 0;
  for (int i = 0; i < src->pp && !rc; ++i) {
    int64_t ilo, ihi;
    stage_range(m, src->pp, i, &ilo, &ihi);
    for (int j = 0; j < dst->pp && !rc; ++j) {
      int64_t jlo, jhi;
      stage_range(m, dst->pp, j, &jlo, &jhi);
      const int64_t lo = ilo > jlo ? ilo : jlo, hi = ihi < jhi ? ihi : jhi;
      if (lo >= hi) continue;
      const int64_t split_b = range_bytes(m, lo, hi, 0, G, split_part), rep_b = range_bytes(m, lo, hi, 1, 1, 0);
      const int64_t kv_b = kv_sep ? range_bytes(m, lo, hi, 0, Gkv, 2) : 0;
      for (int dp = 0; dp < dst->dp && !rc; ++dp) {
        for (int tr = 0; tr < dst->tp && !rc; ++tr) {
          const int d = device_at(dst, c, j, dp, tr);
          if (split_b > 0) {
            const int per_dst = G / dst->tp, per_src = G / src->tp;
            for (int k = tr * per_dst; k < (tr + 1) * per_dst && !rc; ++k) {
              int nh = 0;
              for (int sdp = 0; sdp < src->dp; ++sdp) holders[nh++] = device_at(src, c, i, sdp, k / per_src);
              qsort(holders, (size_t)nh, sizeof(int), cmp_int);
              const int s = pick_source(c, holders, nh, d, policy, egress, split_b);
              rc = add_need(s == d ? &Lc : &R, s, d, lo, hi, k, G, 0, split_part, split_b);
            }
          }
          if (kv_b > 0) {
            /* the K/V slice this rank holds, at the finest common slicing;
             * holders are every source rank whose own K/V slice covers it */
            const int mine = tr * e2 / dst->tp, per_dst = Gkv / e2, per_src = Gkv / e1;
            for (int k = mine * per_dst; k < (mine + 1) * per_dst && !rc; ++k) {
              int nh = 0;
              for (int sdp = 0; sdp < src->dp; ++sdp)
                for (int st = 0; st < src->tp; ++st)
                  if (st * e1 / src->tp == k / per_src) holders[nh++] = device_at(src, c, i, sdp, st);
              qsort(holders, (size_t)nh, sizeof(int), cmp_int);
              const int s = pick_source(c, holders, nh, d, policy, egress, kv_b);
              rc = add_need(s == d ? &Lc : &R, s, d, lo, hi, k, Gkv, 0, 2, kv_b);
            }
          }
          if (rep_b > 0 && !rc) {
            int nh = 0;
            for (int sdp = 0; sdp < src->dp; ++sdp)
              for (int st = 0; st < src->tp; ++st) holders[nh++] = device_at(src, c, i, sdp, st);
            qsort(holders, (size_t)nh, sizeof(int), cmp_int);
            const int s = pick_source(c, holders, nh, d, policy, egress, rep_b);
            rc = add_need(s == d ? &Lc : &R, s, d, lo, hi, 0, 1, 1, 0, rep_b);
          }
        }
      }
    }
  }
  free(holders);
  if (rc) { free(egress); return -1; }
  /* est_time: sources in parallel, one source's ops in sequence. */
  double* busy = calloc((size_t)n_dev, sizeof(double));
  int64_t total = 0;
  for (int i = 0; i < R.n; ++i) {
    double bw = INFINITY;
    for (int k = 0; k < R.list[i].n_dst; ++k) {
      const double b = bandwidth(c, R.list[i].src, R.list[i].dst[k]);
      if (b < bw) bw = b;
    }
    busy[R.list[i].src] += (double)R.list[i].bytes / bw;
    total += R.list[i].bytes * R.list[i].n_dst;
  }
  double est = 0;
  for (int d = 0; d < n_dev; ++d) if (busy[d] > est) est = busy[d];
  free(busy);
  free(egress);
  *n_ops = R.n;
  *n_local = Lc.n;
  *total_bytes = total;
  *est_time = est;
  return 0;
}

/* ---- layout contract: per-tensor address functions --------- */

enum { MODE_NONE = 0, MODE_ROWS, MODE_COLS, MODE_FULL, MODE_GROUPED };

typedef struct {
  int mode;
  int64_t base;      /* byte offset of the tensor (or of its fused entry) */
  int64_t lo, hi;    /* held rows (MODE_ROWS/GROUPED) or cols (MODE_COLS) */
  int64_t g_lo;      /* first local KV group (MODE_GROUPED) */
  int role;          /* 0 q, 1 k, 2 v (MODE_GROUPED) */
} tensor_loc;

typedef struct {
  tensor_loc* loc; /* n_tensors entries */
  int64_t bytes;
  int tp_rank, tp;
  int kv_slice, kv_slices; /* K/V rows held: slice kv_slice of kv_slices (G6) */
} dev_layout;

static int64_t align256(int64_t v) { return (v + 255) / 256 * 256; }

static void place_split(const orc_model* m, dev_layout* L, int64_t id, int64_t* at) {
  const tensor_shape s = shape_of(m, id);
  tensor_loc* t = &L->loc[id];
  t->base = *at;
  if (s.split == SPLIT_ROWS && is_kv(m, id)) {
    t->mode = MODE_ROWS;
    t->lo = L->kv_slice * s.rows / L->kv_slices;
    t->hi = (L->kv_slice + 1) * s.rows / L->kv_slices;
    *at += (t->hi - t->lo) * s.cols * m->param_bytes;
  } else if (s.split == SPLIT_ROWS) {
    t->mode = MODE_ROWS;
    t->lo = L->tp_rank * s.rows / L->tp;
    t->hi = (L->tp_rank + 1) * s.rows / L->tp;
    *at += (t->hi - t->lo) * s.cols * m->param_bytes;
  } else if (s.split == SPLIT_COLS) {
    t->mode = MODE_COLS;
    t->lo = L->tp_rank * s.cols / L->tp;
    t->hi = (L->tp_rank + 1) * s.cols / L->tp;
    *at += (t->hi - t->lo) * s.rows * m->param_bytes;
  } else {
    t->mode = MODE_FULL;
    t->lo = 0;
    t->hi = s.rows;
    *at += s.rows * s.cols * m->param_bytes;
  }
}

/* 0 if the device holds nothing under this placement. */
static int build_layout(const orc_model* m, const orc_placement* p, const orc_cluster* c, int dev,
                        dev_layout* L) {
  int pr, dr, tr;
  L->loc = calloc((size_t)n_tensors(m), sizeof(tensor_loc));
  L->bytes = 0;
  if (rank_of(p, c, dev, &pr, &dr, &tr)) return 0;
  L->tp_rank = tr;
  L->tp = p->tp;
  L->kv_slices = kv_slices(m, p);
  L->kv_slice = tr * L->kv_slices / p->tp;
  int64_t lo, hi, at = 0;
  stage_range(m, p->pp, pr, &lo, &hi);
  for (int64_t e = lo; e < hi; ++e) {
    if (e == -1) {
      at = align256(at);
      place_split(m, L, 0, &at);
      continue;
    }
    if (e == m->layers) {
      at = align256(at);
      place_split(m, L, 1 + 9 * m->layers, &at);
      at = align256(at);
      place_split(m, L, 2 + 9 * m->layers, &at);
      continue;
    }
    const int64_t b = 1 + 9 * e;
    at = align256(at);
    place_split(m, L, b + K_LN1, &at);
    if (p->qkv_layout == 0) {
      for (int k = K_Q; k <= K_V; ++k) { at = align256(at); place_split(m, L, b + k, &at); }
    } else if (p->qkv_layout == 1) {
      at = align256(at);
      for (int k = K_Q; k <= K_V; ++k) place_split(m, L, b + k, &at);
    } else {
      /* Megatron grouping: per local KV group [q heads of g; k_g; v_g]. */
      at = align256(at);
      const int64_t hd = m->hidden / m->heads, groups_per_rank = m->kv_heads / p->tp;
      const int64_t q_rows_per_group = m->heads / m->kv_heads * hd;
      for (int k = K_Q; k <= K_V; ++k) {
        tensor_loc* t = &L->loc[b + k];
        t->mode = MODE_GROUPED;
        t->base = at;
        t->g_lo = tr * groups_per_rank;
        t->role = k - K_Q;
        const int64_t per = k == K_Q ? q_rows_per_group : hd;
        t->lo = t->g_lo * per;
        t->hi = (t->g_lo + groups_per_rank) * per;
      }
      at += groups_per_rank * (q_rows_per_group + 2 * hd) * m->hidden * m->param_bytes;
    }
    at = align256(at);
    place_split(m, L, b + K_O, &at);
    at = align256(at);
    place_split(m, L, b + K_LN2, &at);
    if (p->gate_up_layout == 1) {
      at = align256(at);
      place_split(m, L, b + K_GATE, &at);
      place_split(m, L, b + K_UP, &at);
    } else {
      at = align256(at);
      place_split(m, L, b + K_GATE, &at);
      at = align256(at);
      place_split(m, L, b + K_UP, &at);
    }
    at = align256(at);
    place_split(m, L, b + K_DOWN, &at);
  }
  L->bytes = align256(at);
  return 1;
}

/* Byte offset of logical element (r, c) of tensor id; -1 if not held. */
static int64_t addr_of(const orc_model* m, const dev_layout* L, int64_t id, int64_t r, int64_t c) {
  const tensor_loc* t = &L->loc[id];
  const tensor_shape s = shape_of(m, id);
  const int64_t pb = m->param_bytes;
  switch (t->mode) {
    case MODE_ROWS:
      if (r < t->lo || r >= t->hi) return -1;
      return t->base + ((r - t->lo) * s.cols + c) * pb;
    case MODE_COLS:
      if (c < t->lo || c >= t->hi) return -1;
      return t->base + (r * (t->hi - t->lo) + (c - t->lo)) * pb;
    case MODE_FULL:
      return t->base + (r * s.cols + c) * pb;
    case MODE_GROUPED: {
      if (r < t->lo || r >= t->hi) return -1;
      const int64_t hd = m->hidden / m->heads, qg = m->heads / m->kv_heads * hd;
      const int64_t stride = qg + 2 * hd;
      int64_t g, within;
      if (t->role == 0) { g = r / qg; within = r - g * qg; }
      else { g = r / hd; within = qg + (t->role - 1) * hd + (r - g * hd); }
      return t->base + ((g - t->g_lo) * stride + within) * m->hidden * pb + c * pb;
    }
    default:
      return -1;
  }
}

int64_t orc_shard_bytes(const orc_model* m, const orc_placement* p, const orc_cluster* c, int dev) {
  dev_layout L;
  build_layout(m, p, c, dev, &L);
  free(L.loc);
  return L.bytes;
}

/* ---- weights: DESIGN.md §4 value function (splitmix64) ------------------- */

/* Special-value mode (seed bit 62): class c = bits 24..27 of the hash picks
 * one of seven bf16 special classes (c < 7) or the raw low 16 bits; bit 16 is
 * the sign, bits 17..23 a 7-bit field m for payloads / denormal mantissas.
 * Written branch-free (selects), so the checker's row loop vectorises. */
static inline uint64_t hash_of(uint64_t seed, uint64_t tensor, uint64_t index) {
  uint64_t z = (seed ^ (tensor << 40) ^ index) + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint16_t normal_of(uint64_t z) {
  const uint32_t sign = (uint32_t)(z >> 63), expo = 117u + (uint32_t)((z >> 8) & 7u);
  return (uint16_t)((sign << 15) | (expo << 7) | (uint32_t)(z & 0x7fu));
}

static inline uint16_t special_of(uint64_t z) {
  const uint32_t cls = (uint32_t)((z >> 24) & 15u);
  const uint32_t s = (uint32_t)((z >> 16) & 1u) << 15;
  const uint32_t m = (uint32_t)((z >> 17) & 0x7fu);
  const uint32_t m63 = m - 63u * (uint32_t)(m >= 63u) - 63u * (uint32_t)(m >= 126u); /* m % 63 */
#define ORC_PICK(k, val) v = (v & ~(0u - (uint32_t)(cls == (k)))) | ((val) & (0u - (uint32_t)(cls == (k))))
  uint32_t v = (uint32_t)(z & 0xffffu);      /* any 16-bit pattern (classes 7..15) */
  ORC_PICK(0u, s);                           /* signed zero */
  ORC_PICK(1u, s + 0x7f80u);                 /* infinity */
  ORC_PICK(2u, s + 0x7fc0u + (m & 63u));     /* quiet NaN + payload */
  ORC_PICK(3u, s + 0x7f81u + m63);           /* signalling NaN */
  ORC_PICK(4u, s + (m | 1u));                /* subnormal */
  ORC_PICK(5u, s + 0x7f7fu);                 /* largest finite */
  ORC_PICK(6u, s + 0x80u);                   /* smallest normal */
#undef ORC_PICK
  return (uint16_t)v;
}

uint16_t orc_value(uint64_t seed, int64_t tensor, int64_t index) {
  const uint64_t z = hash_of(seed, (uint64_t)tensor, (uint64_t)index);
  return (seed >> 62) & 1u ? special_of(z) : normal_of(z);
}

int orc_fill(const orc_model* m, const orc_placement* p, const orc_cluster* c, int dev,
             uint64_t seed, uint16_t* buf) {
  dev_layout L;
  if (!build_layout(m, p, c, dev, &L)) { free(L.loc); return -1; }
  for (int64_t id = 0; id < n_tensors(m); ++id) {
    const tensor_loc* t = &L.loc[id];
    if (t->mode == MODE_NONE) continue;
    const tensor_shape s = shape_of(m, id);
    const int64_t r0 = t->mode == MODE_COLS ? 0 : t->lo, r1 = t->mode == MODE_COLS ? s.rows : t->hi;
    const int64_t c0 = t->mode == MODE_COLS ? t->lo : 0, c1 = t->mode == MODE_COLS ? t->hi : s.cols;
    for (int64_t r = r0; r < r1; ++r) {
      uint16_t* row = buf + addr_of(m, &L, id, r, c0) / 2;
      for (int64_t col = c0; col < c1; ++col) row[col - c0] = orc_value(seed, id, r * s.cols + col);
    }
  }
  free(L.loc);
  return 0;
}

/* ---- streamed windows of a shard ------------------------------------------ *
 * Expected bytes [off, off + len) of a device's shard, computed per element
 * through the same address function as orc_fill, without materialising the
 * shard: the full-size parity tests compare every destination byte of
 * multi-GB shards window by window, and the CPU baseline fills its sources
 * with several threads. */

/* Local rows of a tensor as laid out: count, column range, and whether row i
 * is logical row first + i at base + i * row_bytes (all modes but grouped). */
static int64_t local_rows(const orc_model* m, const tensor_loc* t, int64_t id, int64_t* c0, int64_t* c1,
                          int64_t* first) {
  const tensor_shape s = shape_of(m, id);
  *c0 = t->mode == MODE_COLS ? t->lo : 0;
  *c1 = t->mode == MODE_COLS ? t->hi : s.cols;
  *first = t->mode == MODE_COLS || t->mode == MODE_FULL ? 0 : t->lo;
  return t->mode == MODE_COLS || t->mode == MODE_FULL ? s.rows : t->hi - t->lo;
}

/* The checker computes every element of multi-GB shards: the row loop is
 * compiled twice, for AVX-512 (x86-64-v4: eight 64-bit hash lanes per
 * instruction) and baseline x86-64, and picked at load time. */
__attribute__((target_clones("arch=x86-64-v4", "default")))
static void fill_window(const orc_model* m, const dev_layout* L, uint64_t seed, int64_t off, int64_t len,
                        uint16_t* buf) {
  const int64_t pb = m->param_bytes, end = off + len;
  memset(buf, 0, (size_t)len);
  for (int64_t id = 0; id < n_tensors(m); ++id) {
    const tensor_loc* t = &L->loc[id];
    if (t->mode == MODE_NONE) continue;
    const tensor_shape s = shape_of(m, id);
    int64_t c0, c1, first;
    const int64_t n = local_rows(m, t, id, &c0, &c1, &first);
    const int64_t row_bytes = (c1 - c0) * pb;
    int64_t i0 = 0, i1 = n;
    if (t->mode != MODE_GROUPED) { /* rows are consecutive: clip to the window */
      if (t->base >= end || t->base + n * row_bytes <= off) continue;
      if (off > t->base) i0 = (off - t->base) / row_bytes;
      if (end < t->base + n * row_bytes) i1 = (end - t->base + row_bytes - 1) / row_bytes;
    }
    for (int64_t i = i0; i < i1; ++i) {
      const int64_t r = first + i;
      const int64_t a = addr_of(m, L, id, r, c0);
      if (a >= end || a + row_bytes <= off) continue;
      int64_t ca = c0, cb = c1;
      if (a < off) ca = c0 + (off - a) / pb;
      if (a + row_bytes > end) cb = c0 + (end - a) / pb;
      const int64_t at = (a - off) / pb - c0; /* window element of column 0 of this row */
      const uint64_t row0 = (uint64_t)(r * s.cols);
      if ((seed >> 62) & 1u)
        for (int64_t col = ca; col < cb; ++col)
          buf[at + col] = special_of(hash_of(seed, (uint64_t)id, row0 + (uint64_t)col));
      else
        for (int64_t col = ca; col < cb; ++col)
          buf[at + col] = normal_of(hash_of(seed, (uint64_t)id, row0 + (uint64_t)col));
    }
  }
}

typedef struct {
  const orc_model* m;
  const dev_layout* L;
  uint64_t seed;
  int64_t off, len, piece;
  uint16_t* out;         /* fill target (NULL when checking) */
  const uint16_t* got;   /* bytes to check (NULL when filling) */
  int64_t next;          /* next piece (atomic) */
  int64_t bad, first;    /* mismatching elements, first mismatching element index of the window */
  pthread_mutex_t mu;
} window_job;

static void* window_worker(void* arg) {
  window_job* j = (window_job*)arg;
  uint16_t* scratch = j->got ? malloc((size_t)j->piece) : NULL;
  int64_t bad = 0, first = -1;
  for (;;) {
    const int64_t k = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
    const int64_t a = k * j->piece;
    if (a >= j->len) break;
    const int64_t n = a + j->piece < j->len ? j->piece : j->len - a;
    if (j->out) {
      fill_window(j->m, j->L, j->seed, j->off + a, n, j->out + a / 2);
      continue;
    }
    fill_window(j->m, j->L, j->seed, j->off + a, n, scratch);
    const uint16_t* g = j->got + a / 2;
    if (memcmp(scratch, g, (size_t)n) == 0) continue;
    for (int64_t e = 0; e < n / 2; ++e)
      if (scratch[e] != g[e]) {
        if (first < 0 || a / 2 + e < first) first = a / 2 + e;
        ++bad;
      }
  }
  free(scratch);
  pthread_mutex_lock(&j->mu);
  j->bad += bad;
  if (first >= 0 && (j->first < 0 || first < j->first)) j->first = first;
  pthread_mutex_unlock(&j->mu);
  return NULL;
}

static int run_window(const orc_model* m, const orc_placement* p, const orc_cluster* c, int dev, uint64_t seed,
                      int64_t off, int64_t len, uint16_t* out, const uint16_t* got, int threads, int64_t* bad,
                      int64_t* first) {
  dev_layout L;
  if (!build_layout(m, p, c, dev, &L) || off < 0 || len < 0 || off + len > L.bytes || (off | len) & 1) {
    free(L.loc);
    return -1;
  }
  window_job j;
  memset(&j, 0, sizeof(j));
  j.m = m;
  j.L = &L;
  j.seed = seed;
  j.off = off;
  j.len = len;
  j.piece = 4 << 20;
  j.out = out;
  j.got = got;
  j.first = -1;
  pthread_mutex_init(&j.mu, NULL);
  if (threads < 1) threads = 1;
  if ((int64_t)threads > len / j.piece + 1) threads = (int)(len / j.piece + 1);
  pthread_t* th = malloc(sizeof(pthread_t) * (size_t)threads);
  for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, window_worker, &j);
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  free(th);
  pthread_mutex_destroy(&j.mu);
  free(L.loc);
  if (bad) *bad = j.bad;
  if (first) *first = j.first;
  return 0;
}

int orc_fill_range(const orc_model* m, const orc_placement* p, const orc_cluster* c, int dev, uint64_t seed,
                   int64_t offset, int64_t len, uint16_t* buf, int threads) {
  return run_window(m, p, c, dev, seed, offset, len, buf, NULL, threads, NULL, NULL);
}

int orc_check_range(const orc_model* m, const orc_placement* p, const orc_cluster* c, int dev, uint64_t seed,
                    int64_t offset, int64_t len, const uint16_t* got, int threads, int64_t* mismatches,
                    int64_t* first) {
  return run_window(m, p, c, dev, seed, offset, len, NULL, got, threads, mismatches, first);
}

/* ---- CPU reallocation ------------------------------------------------------ */

typedef struct {
  int op, dst, id;
  int64_t r0, r1, c0, c1;
} task;

typedef struct {
  const orc_model* m;
  const orc_op* ops;
  dev_layout* s_lay; /* by device */
  dev_layout* d_lay;
  void* const* src_bufs;
  void* const* dst_bufs;
  task* tasks;
  int64_t n_tasks;
  int64_t next;
} exec_ctx;

static void* worker(void* arg) {
  exec_ctx* x = (exec_ctx*)arg;
  const int64_t pb = x->m->param_bytes;
  for (;;) {
    const int64_t i = __atomic_fetch_add(&x->next, 1, __ATOMIC_RELAXED);
    if (i >= x->n_tasks) break;
    const task* t = &x->tasks[i];
    const orc_op* op = &x->ops[t->op];
    const dev_layout* S = &x->s_lay[op->src];
    const dev_layout* D = &x->d_lay[t->dst];
    const char* sb = (const char*)x->src_bufs[op->src];
    char* db = (char*)x->dst_bufs[t->dst];
    const size_t w = (size_t)((t->c1 - t->c0) * pb);
    for (int64_t r = t->r0; r < t->r1; ++r)
      memcpy(db + addr_of(x->m, D, t->id, r, t->c0), sb + addr_of(x->m, S, t->id, r, t->c0), w);
  }
  return NULL;
}

int orc_execute(const orc_model* m, const orc_placement* src, const orc_placement* dst,
                const orc_cluster* c, const orc_op* ops, int n_ops, void* const* src_bufs,
                void* const* dst_bufs, int threads) {
  const int n_dev = c->n_nodes * c->gpus_per_node;
  exec_ctx x;
  memset(&x, 0, sizeof(x));
  x.m = m;
  x.ops = ops;
  x.src_bufs = src_bufs;
  x.dst_bufs = dst_bufs;
  x.s_lay = calloc((size_t)n_dev, sizeof(dev_layout));
  x.d_lay = calloc((size_t)n_dev, sizeof(dev_layout));
  for (int d = 0; d < n_dev; ++d) {
    build_layout(m, src, c, d, &x.s_lay[d]);
    build_layout(m, dst, c, d, &x.d_lay[d]);
  }
  int64_t cap = 1024;
  x.tasks = malloc(sizeof(task) * (size_t)cap);
  for (int o = 0; o < n_ops; ++o) {
    const orc_op* op = &ops[o];
    for (int k = 0; k < op->n_dst; ++k) {
      for (int64_t id = 0; id < n_tensors(m); ++id) {
        const tensor_shape s = shape_of(m, id);
        if (s.layer < op->layer_start || s.layer >= op->layer_end) continue;
        if (!in_part(m, id, op->replicated, op->part)) continue;
        int64_t r0 = 0, r1 = s.rows, c0 = 0, c1 = s.cols;
        if (s.split == SPLIT_ROWS) {
          r0 = op->slice * s.rows / op->slices;
          r1 = (op->slice + 1) * s.rows / op->slices;
        } else if (s.split == SPLIT_COLS) {
          c0 = op->slice * s.cols / op->slices;
          c1 = (op->slice + 1) * s.cols / op->slices;
        }
        for (int64_t r = r0; r < r1; r += 512) {
          if (x.n_tasks == cap) {
            cap *= 2;
            x.tasks = realloc(x.tasks, sizeof(task) * (size_t)cap);
          }
          task t = {o, op->dst[k], (int)id, r, r + 512 < r1 ? r + 512 : r1, c0, c1};
          x.tasks[x.n_tasks++] = t;
        }
      }
    }
  }
  if (threads < 1) threads = 1;
  pthread_t* th = malloc(sizeof(pthread_t) * (size_t)threads);
  for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, worker, &x);
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  free(th);
  free(x.tasks);
  for (int d = 0; d < n_dev; ++d) {
    free(x.s_lay[d].loc);
    free(x.d_lay[d].loc);
  }
  free(x.s_lay);
  free(x.d_lay);
  return 0;
}

/* ---- inter-call data transfer: SPEC.md:578-586, PAPER.md:522 ------------- */

/* Data placements need only a valid mesh and dp*tp*pp == mesh size. */
static int strategy_ok(const orc_placement* p, const orc_cluster* c) { return mesh_ok(p, c); }

int orc_plan_data(const orc_placement* prod, const orc_placement* cons, const orc_cluster* c, int policy,
                  int64_t per_shard, orc_op* ops, int cap, int* n_ops, orc_op* local, int cap_local,
                  int* n_local, int64_t* total_bytes, double* est_time) {
  if (!strategy_ok(prod, c) || !strategy_ok(cons, c) || per_shard <= 0) return -1;
  const int G = (int)(prod->dp / gcd64(prod->dp, cons->dp) * cons->dp);
  const int64_t total = per_shard * prod->dp;
  if (total % (2 * G)) return -1;
  const int64_t slice = total / G;
  const int n_dev = c->n_nodes * c->gpus_per_node;
  int64_t* egress = calloc((size_t)n_dev, sizeof(int64_t));
  int holders[64];
  op_list R = {ops, cap, 0}, Lc = {local, cap_local, 0};
  int rc = 0;
  /* consumers in ascending device order == (pp, dp, tp) rank order */
  for (int i = 0; i < mesh_size(cons) && !rc; ++i) {
    const int d = mesh_device(cons, c, i);
    const int dp_r = (i / cons->tp) % cons->dp;
    for (int k = dp_r * (G / cons->dp); k < (dp_r + 1) * (G / cons->dp) && !rc; ++k) {
      int nh = 0; /* PP and TP are both replica axes of a DP group's data */
      for (int s = 0; s < prod->pp; ++s)
        for (int t = 0; t < prod->tp; ++t) holders[nh++] = device_at(prod, c, s, k / (G / prod->dp), t);
      qsort(holders, (size_t)nh, sizeof(int), cmp_int);
      const int s = pick_source(c, holders, nh, d, policy, egress, slice);
      rc = add_need(s == d ? &Lc : &R, s, d, 0, 0, k, G, 0, 0, slice);
    }
  }
  if (rc) { free(egress); return -1; }
  double* busy = calloc((size_t)n_dev, sizeof(double));
  int64_t tb = 0;
  for (int i = 0; i < R.n; ++i) {
    double bw = INFINITY;
    for (int k = 0; k < R.list[i].n_dst; ++k) {
      const double b = bandwidth(c, R.list[i].src, R.list[i].dst[k]);
      if (b < bw) bw = b;
    }
    busy[R.list[i].src] += (double)R.list[i].bytes / bw;
    tb += R.list[i].bytes * R.list[i].n_dst;
  }
  double est = 0;
  for (int d = 0; d < n_dev; ++d) if (busy[d] > est) est = busy[d];
  free(busy);
  free(egress);
  *n_ops = R.n;
  *n_local = Lc.n;
  *total_bytes = tb;
  *est_time = est;
  return 0;
}

/* First element and element count of a device's data, or -1. */
static int64_t data_range(const orc_placement* p, const orc_cluster* c, int dev, int producer, int64_t total,
                          int64_t* first) {
  int pr, dr, tr;
  if (rank_of(p, c, dev, &pr, &dr, &tr)) return -1;
  (void)producer; /* producers and consumers hold their DP group's data */
  const int64_t per = total / 2 / p->dp;
  *first = dr * per;
  return per;
}

int64_t orc_data_shard_bytes(const orc_placement* p, const orc_cluster* c, int dev, int producer, int64_t total) {
  int64_t first;
  const int64_t n = data_range(p, c, dev, producer, total, &first);
  return n < 0 ? 0 : align256(n * 2);
}

int orc_data_fill(const orc_placement* p, const orc_cluster* c, int dev, int producer, int64_t total,
                  uint64_t seed, uint16_t* buf) {
  int64_t first;
  const int64_t n = data_range(p, c, dev, producer, total, &first);
  if (n < 0) return -1;
  for (int64_t e = 0; e < n; ++e) buf[e] = orc_value(seed, ORC_DATA_TENSOR, first + e);
  return 0;
}

typedef struct {
  uint16_t* dst;
  const uint16_t* src;
  size_t bytes;
} data_piece;

typedef struct {
  data_piece* pieces;
  int64_t n, next;
} data_ctx;

static void* data_worker(void* arg) {
  data_ctx* x = (data_ctx*)arg;
  for (;;) {
    const int64_t i = __atomic_fetch_add(&x->next, 1, __ATOMIC_RELAXED);
    if (i >= x->n) break;
    memcpy(x->pieces[i].dst, x->pieces[i].src, x->pieces[i].bytes);
  }
  return NULL;
}

int orc_data_execute_mt(const orc_placement* prod, const orc_placement* cons, const orc_cluster* c, int64_t total,
                        const orc_op* ops, int n_ops, void* const* src_bufs, void* const* dst_bufs, int threads) {
  const int64_t elems = total / 2, piece = 1 << 19; /* 1 MiB of bf16 words per task */
  data_ctx x = {NULL, 0, 0};
  int64_t cap = 256;
  x.pieces = malloc(sizeof(data_piece) * (size_t)cap);
  for (int o = 0; o < n_ops; ++o) {
    const orc_op* op = &ops[o];
    const int64_t s0 = op->slice * elems / op->slices, s1 = (op->slice + 1) * elems / op->slices;
    int64_t sf, df;
    if (data_range(prod, c, op->src, 1, total, &sf) < 0) {
      free(x.pieces);
      return -1;
    }
    for (int k = 0; k < op->n_dst; ++k) {
      if (data_range(cons, c, op->dst[k], 0, total, &df) < 0) {
        free(x.pieces);
        return -1;
      }
      for (int64_t e = s0; e < s1; e += piece) {
        if (x.n == cap) {
          cap *= 2;
          x.pieces = realloc(x.pieces, sizeof(data_piece) * (size_t)cap);
        }
        const int64_t n = e + piece < s1 ? piece : s1 - e;
        data_piece p = {(uint16_t*)dst_bufs[op->dst[k]] + (e - df), (const uint16_t*)src_bufs[op->src] + (e - sf),
                        (size_t)n * 2};
        x.pieces[x.n++] = p;
      }
    }
  }
  if (threads < 1) threads = 1;
  pthread_t* th = malloc(sizeof(pthread_t) * (size_t)threads);
  for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, data_worker, &x);
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  free(th);
  free(x.pieces);
  return 0;
}

int orc_data_execute(const orc_placement* prod, const orc_placement* cons, const orc_cluster* c, int64_t total,
                     const orc_op* ops, int n_ops, void* const* src_bufs, void* const* dst_bufs) {
  return orc_data_execute_mt(prod, cons, c, total, ops, n_ops, src_bufs, dst_bufs, 1);
}
