// Internal device-side structures shared by capi.cpp and kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace rr {

// Thread-local message returned by rr_last_error() (defined in capi.cpp).
void set_last_error(const std::string& msg);

// Maximum destinations one work item stores to (fan-out of a broadcast op
// that is executed by one source read). Larger fan-outs are split.
constexpr int kMaxFan = 8;

// Hard cap on units per work item so that the float row/col split in the
// copy kernel stays exact (see rr_copy_kernel).
constexpr uint32_t kMaxItemUnits = 1u << 20;

// CopyItem::vec flags.
constexpr uint16_t kItemVec = 1;         // 16-byte units (else 2-byte units)
constexpr uint16_t kItemMulticast0 = 2;  // dst[0] is an NVLS multicast address

// One chunk of a 2D copy: `nrows` rows of `row_units` units; unit = 16 bytes
// when vec has kItemVec, else 2 bytes (one bf16). Source read once, stored to
// every dst[0..ndst).
struct alignas(16) CopyItem {
  uint64_t src;
  uint64_t dst[kMaxFan];
  uint32_t row_units;
  uint32_t nrows;
  uint32_t src_pitch;  // units
  uint32_t dst_pitch;  // units
  float inv_row;       // 1.0f / row_units
  uint16_t ndst;
  uint16_t vec;
  // Pipelined relay (exec_plan.cpp): wait until *wait_flag >= epoch before
  // reading the source (it is being written by the previous GPU of the
  // chain), and after the copy store epoch into *signal_flag on the next
  // GPU (release, system scope). 0 = none.
  uint64_t wait_flag;
  uint64_t signal_flag;
};
static_assert(sizeof(CopyItem) % 16 == 0, "CopyItem must be a multiple of 16 bytes");

// A run of elements of one layout block for hash fill / verify.
struct alignas(16) FillItem {
  uint64_t base;       // address of the block's first element
  uint64_t r0;         // logical row of the block's first row
  uint64_t c0;         // logical column of the block's first column
  uint64_t full_cols;  // logical tensor width
  uint32_t cols;       // block width (elements)
  uint32_t tensor;
  uint32_t elem0;      // first element (within the block) of this item
  uint32_t n;          // elements in this item
};

// splitmix64 finaliser: the weight value function of DESIGN.md §4.
__host__ __device__ inline uint64_t mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Seed flag of the special-value fill (DESIGN.md §3 "Weights"): bf16 words
// that a value-preserving copy must not disturb — ±0, ±Inf, quiet NaNs with
// payloads, signalling NaNs, denormals, ±max / ±min normals — interleaved
// with arbitrary 16-bit patterns. Shards are opaque bytes; this
// mode proves every copy path moves them as such.
constexpr uint64_t kSeedSpecial = uint64_t{1} << 62;

__host__ __device__ inline uint16_t special_value(uint64_t h) {
  const uint32_t r = static_cast<uint32_t>(h >> 16);
  const uint32_t sign = (r & 1u) << 15;
  const uint32_t m7 = (r >> 1) & 0x7fu;
  switch ((r >> 8) & 15u) {
    case 0: return static_cast<uint16_t>(sign);                            // +-0
    case 1: return static_cast<uint16_t>(sign | 0x7f80u);                  // +-Inf
    case 2: return static_cast<uint16_t>(sign | 0x7fc0u | (m7 & 0x3fu));   // quiet NaN, payload
    case 3: return static_cast<uint16_t>(sign | 0x7f80u | (1u + m7 % 63u));  // signalling NaN
    case 4: return static_cast<uint16_t>(sign | m7 | 1u);                  // denormal
    case 5: return static_cast<uint16_t>(sign | 0x7f7fu);                  // +-max normal
    case 6: return static_cast<uint16_t>(sign | 0x0080u);                  // +-min normal
    default: return static_cast<uint16_t>(h);                              // any 16-bit pattern
  }
}

// bf16 bits: random sign, exponent in [2^-10, 2^-3], random 7-bit mantissa
// (never NaN/Inf/denormal); with kSeedSpecial in the seed, special_value.
__host__ __device__ inline uint16_t weight_value(uint64_t seed, uint64_t tensor, uint64_t idx) {
  const uint64_t h = mix64(seed ^ (tensor << 40) ^ idx);
  if (seed & kSeedSpecial) return special_value(h);
  const uint32_t sign = static_cast<uint32_t>(h >> 63);
  const uint32_t expo = 117u + static_cast<uint32_t>((h >> 8) & 7u);
  const uint32_t mant = static_cast<uint32_t>(h & 0x7fu);
  return static_cast<uint16_t>((sign << 15) | (expo << 7) | mant);
}

// Host-callable launchers (kernels.cu). All return a cudaError_t as int.
// sched: 4 device uints (next item, retired CTAs, relay timeouts, unused);
// epoch: value relay flags are compared against / set to.
int launch_copy(const CopyItem* items, int n_items, int ctas, int fence_sys, void* stream, unsigned int* sched,
                uint32_t epoch = 0);
int copy_max_ctas(int* ctas_per_sm, int* sms);
// TMA bulk variant (kBulkVariantA / kBulkVariantB = stage ring shapes); items must all be vec items
// without multicast (relay wait / signal flags are supported). With max_ctas != NULL only reports
// the resident-CTA capacity.
int launch_bulk(int variant, const CopyItem* items, int n_items, int ctas, int fence_sys, void* stream,
                int* max_ctas, unsigned int* sched, uint32_t epoch = 0);
constexpr int kBulkVariantA = 1;  // 4 x 16 KiB stages (plain phases)
constexpr int kBulkVariantB = 5;  // 3 x 16 KiB stages (flag-synchronised phases)
inline bool valid_kernel(int k) { return k == 0 || k == kBulkVariantA || k == kBulkVariantB; }
int launch_fill(const FillItem* items, int n_items, uint64_t seed, void* stream);
int launch_verify(const FillItem* items, int n_items, uint64_t seed, unsigned long long* counters,
                  uint64_t buf_base, void* stream);
int launch_barrier(uint32_t* const* flags, int rank, int world, uint32_t epoch, int* timed_out,
                   void* stream);

}  // namespace rr
