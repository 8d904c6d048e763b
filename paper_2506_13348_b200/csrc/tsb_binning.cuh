// tsb_binning.cuh — kernels and argument blocks of the hand-written binning
// (tsb_binning.cu), launched by tsb_render_binning (tsb_forward.cu).
#pragma once

#include <cstdint>

#include "tsb_internal.cuh"

namespace tsb {

constexpr int kRadixBits = 8;
constexpr uint32_t kRadixBins = 1u << kRadixBits;
constexpr int kOsThreads = 256;   // one-sweep CTA: 8 warps, one digit per thread
constexpr int kOsWarps = kOsThreads / 32;
constexpr int kOsItems = 8;       // items per thread (tile-y pass)
constexpr int kOsTile = kOsThreads * kOsItems;
constexpr int kOsItemsDepth = 8;  // depth passes: P is small, more CTAs in flight
constexpr int kOsTileDepth = kOsThreads * kOsItemsDepth;
constexpr int kDupCache = 3072;  // entries of a k_dup_tx CTA kept in shared memory
constexpr int kDepthPasses = 4;   // 32-bit depth key, 8-bit digits
constexpr uint32_t kDepthCulled32 = 0xFFFFFFFFu;
constexpr int kShortRun = 32;     // runs of equal 32-bit keys up to 33 long: one thread
constexpr int kMaxTileAxis = 256; // tile_x, tile_y < 256: (ty << 8 | tx) entry keys

// Device-side binning state (workspace `bin` region, zeroed per frame).
struct BinCounters {
  int32_t tickets[8];          // one-sweep CTA tickets: 4 depth passes, dup, tile-y
  int32_t kept;                // splats with centre in front and a non-empty rect
  int32_t n_long;              // long runs of equal depth keys
  int32_t pad[6];
  int32_t hist_depth[kDepthPasses][kRadixBins];  // digit counts of the depth key
  int32_t hist_tx[kRadixBins + 1];               // difference arrays of the entries'
  int32_t hist_ty[kRadixBins + 1];               // tile columns / rows
};

constexpr int32_t kOsPlain = 0;  // (tile-y pass)
constexpr int32_t kOsFirst = 1;  // depth pass 1: culled items (key 0xFFFFFFFF) to the tail
constexpr int32_t kOsLater = 2;  // depth passes 2-4: rank [0, K), the tail passes through

struct OnesweepArgs {
  const uint32_t* kin;
  const uint32_t* vin;
  uint32_t* kout;
  uint32_t* vout;
  int32_t n;
  const int64_t* n_dev;  // if set: n = *n_dev (0 when it exceeds cap)
  int64_t cap;
  int32_t shift;
  const int32_t* hist;
  int32_t hist_is_diff;
  int32_t tiles_x;       // > 0: output key (ty << 8 | tx) -> tile index ty * tiles_x + tx
  uint32_t* status;      // pass_status_words(nb) words
  int32_t nb;            // CTAs of the pass (grid size)
  int32_t mode;          // kOsPlain / kOsFirst / kOsLater
  const int32_t* kept;   // depth passes: the kept count K (device)
  int32_t* ticket;
};

// k_preprocess's per-splat binning record (by id): .x = record slot, .y =
// tile box tx0 | ty0 << 8 | (ntx - 1) << 16 | (nty - 1) << 24, or
// kBinNoTiles (no entries; unambiguous: tx0 + ntx <= 256).
constexpr uint32_t kBinNoTiles = 0xFFFFFFFFu;

struct DupArgs {
  const int32_t* sorted_ids;
  const uint2* bin_rec;
  const int32_t* kept;
  const int64_t* total;
  int64_t cap;
  const int32_t* hist_tx;
  uint32_t* kout;
  uint32_t* vout;
  uint32_t* status;
  int32_t nb;
  int32_t* ticket;
};

struct FixRunsArgs {
  int32_t P;
  const uint32_t* k32;
  const uint64_t* k64;
  int32_t* ids;
  int32_t* rank;
  int32_t* n_long;
  int32_t* long_runs;
};

struct LongRunArgs {
  const int32_t* n_long;
  const int32_t* long_runs;
  const uint64_t* k64;
  int32_t* ids;
  int32_t* scratch;
  int32_t* rank;
};

constexpr int kGroupCtas = 32;  // cta_prefix group size
// look-back words of one pass of nb CTAs: per-CTA counts, group sums, group done counters
constexpr size_t pass_status_words(int nb) {
  return (size_t)nb * kRadixBins + (size_t)((nb + kGroupCtas - 1) / kGroupCtas) * (kRadixBins + 1);
}

template <int ITEMS>
__global__ void k_onesweep(OnesweepArgs a);
__global__ void k_dup_tx(DupArgs a);
__global__ void k_fix_runs(FixRunsArgs a);
__global__ void k_sort_long_runs(LongRunArgs a);
__global__ void k_ranges(int64_t cap, const uint32_t* __restrict__ keys,
                         const int64_t* __restrict__ counters, int32_t* __restrict__ ranges,
                         int64_t* __restrict__ max_needed);

}  // namespace tsb
