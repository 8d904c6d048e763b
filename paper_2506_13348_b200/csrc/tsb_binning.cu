// tsb_binning.cu — hand-written sm_100a binning: the draw order and the tile
// lists of one frame, replacing `np.lexsort((ids, z))` (rasterize.py:178-182)
// and `_tile_lists` (rasterize.py:246-258). No library kernels.
//
//   S1  depth order   stable LSD radix sort of a 32-bit monotone depth key
//                     (the high word of the fp64 centre depth's bit pattern,
//                     minus near's) over ids in id order: four one-sweep
//                     passes of 8 bits (k_onesweep). Ties of the 32-bit key
//                     are re-ordered by the full fp64 key in k_fix_runs
//                     (runs of <= kShortRun + 1: one thread; longer runs: one
//                     warp per run, an O(run) stable warp radix sort on the
//                     low word;
//                     a run whose full keys are already ordered — e.g. a
//                     frontal plane at one depth — costs a parallel check).
//                     Result == np.lexsort((ids, z)) on the kept splats.
//   S2  tile lists    entry key = (tile_y << 8) | tile_x. Pass 1 is FUSED with
//                     the duplication (k_dup_tx): each CTA takes 256 splats in
//                     draw order, enumerates their tiles and scatters the
//                     entries stably by tile_x; pass 2 (k_onesweep) stably by
//                     tile_y, writing the tile index. Per-tile lists keep draw
//                     order == keys (tile << 32) | rank.
//
// One-sweep pass (single kernel per pass, in the spirit of Merrill & Garland's
// one-sweep radix sort): a CTA takes a tile of items in order (CTA ids from
// an atomic ticket, so a CTA only waits on CTAs that started earlier), ranks
// them stably per digit with warp-private running counters
// (__match_any_sync groups equal digits within a 32-item round), publishes
// its per-digit counts, and gets its global offset from a two-level prefix
// over its predecessors (cta_prefix: group sums + in-group counts, all
// loads independent).
// Digit histograms come from k_preprocess (depth digits; tile-column and
// tile-row difference arrays), so no pass re-reads the keys to count.

#include "tsb_internal.cuh"
#include "tsb_binning.cuh"

namespace tsb {

namespace {

constexpr uint32_t kStAgg = 1u << 30, kStMask = (1u << 30) - 1u;

__device__ __forceinline__ uint32_t ld_status(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_status(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Exclusive prefix, over the CTAs before `bid`, of digit d's count (all 256
// threads call this, thread d for digit d). Two levels, so that every load
// of the walk is independent (no chain of dependent round trips even when
// all CTAs are resident at once): CTAs form groups of kGroup; a CTA adds
// its counts into its group's sums and bumps the group's done counter, and
// publishes its own counts (flag | count). The prefix = the sums of all
// earlier (complete) groups + the counts of the earlier CTAs of its own
// group. Layout of `status` per pass: [nb][256] words, then [ng][256] group
// sums, then [ng] done counters (all zeroed per frame).
constexpr int kGroup = kGroupCtas;
__device__ __forceinline__ uint32_t cta_prefix(uint32_t* status, int nb, int bid, int d,
                                               uint32_t cnt) {
  const int ng = (nb + kGroup - 1) / kGroup;
  uint32_t* gsum = status + (size_t)nb * kRadixBins;
  uint32_t* gdone = gsum + (size_t)ng * kRadixBins;
  const int g = bid / kGroup;
  st_status(status + (size_t)bid * kRadixBins + d, kStAgg | cnt);
  if (cnt) atomicAdd(gsum + (size_t)g * kRadixBins + d, cnt);
  __syncthreads();  // (CTA-scope: the group adds above happen before the release below)
  if (threadIdx.x == 0)  // release: cumulative over the CTA's adds ordered by the barrier
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gdone + g) : "memory");
  // earlier groups: wait until complete (thread t < g polls group t, acquire)
  for (int t = threadIdx.x; t < g; t += blockDim.x) {
    uint32_t v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gdone + t) : "memory");
    } while (v < (uint32_t)kGroup);
  }
  __syncthreads();
  uint32_t excl = 0;
  for (int t = 0; t < g; ++t) excl += ld_status(gsum + (size_t)t * kRadixBins + d);
  for (int q = g * kGroup; q < bid;) {  // in-group predecessors, 8 loads per round trip
    uint32_t w[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      w[j] = q + j < bid ? ld_status(status + (size_t)(q + j) * kRadixBins + d) : kStAgg;
    int used = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (used < j || (w[j] >> 30) == 0) continue;  // stop at the first unpublished word
      excl += w[j] & kStMask;
      ++used;
    }
    q += used;
  }
  return excl;
}

// Block-wide exclusive scan of one value per thread (blockDim == 256).
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp,
                                                         uint32_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < 8 ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < 8) s_warp[lane] = t;  // inclusive warp totals
  }
  __syncthreads();
  const uint32_t before = w ? s_warp[w - 1] : 0u;
  if (total) *total = s_warp[7];
  __syncthreads();
  return before + x - v;
}

// Global exclusive digit offsets of a pass from its histogram (counts or a
// difference array of 257 entries whose prefix sums are the counts).
__device__ __forceinline__ void digit_offsets(const int32_t* hist, bool is_diff, uint32_t* s_goff,
                                              uint32_t* s_warp) {
  const int d = threadIdx.x;
  uint32_t c = (uint32_t)hist[d];
  if (is_diff) c = block_exclusive_scan(c, s_warp, nullptr) + c;  // inclusive: the count
  s_goff[d] = block_exclusive_scan(c, s_warp, nullptr);
}

// Stable rank of this lane's item among the warp's items with the same digit
// (digits 0..kRadixBins; kRadixBins + 1 = no item): running counter per
// (warp, digit) — wrun has kRadixBins + 1 entries — advanced
// by the group leader. Returns the counter value for this item.
__device__ __forceinline__ uint32_t warp_rank(uint32_t* wrun, uint32_t d, int lane) {
  const uint32_t peers = __match_any_sync(0xffffffffu, d);
  const int leader = __ffs(peers) - 1;
  uint32_t old = 0;
  if (lane == leader && d <= kRadixBins) old = atomicAdd(&wrun[d], (uint32_t)__popc(peers));
  old = __shfl_sync(0xffffffffu, old, leader);
  return old + (uint32_t)__popc(peers & ((1u << lane) - 1u));
}

}  // namespace

// ---------------------------------------------------------------------------
// Generic one-sweep pass over (key, value) pairs.
// ---------------------------------------------------------------------------
template <int ITEMS>
__global__ void __launch_bounds__(kOsThreads) k_onesweep(OnesweepArgs a) {
  pdl_wait();
  constexpr int TILE = kOsThreads * ITEMS;
  constexpr uint32_t kCulledBin = kRadixBins;  // depth pass 1: culled items' own counter
  __shared__ uint32_t whist[kOsWarps][kRadixBins + 1];
  __shared__ uint32_t s_goff[kRadixBins];
  __shared__ uint32_t s_warp[8];
  __shared__ uint32_t s_culled_before;
  __shared__ int s_bid;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int n = a.n;
  if (a.n_dev) {
    const int64_t e = *a.n_dev;
    n = e > a.cap ? 0 : (int)e;  // overflowed frame: nothing to sort
  }
  // depth passes: items [0, K) are the kept splats (after pass 1), the culled
  // tail [K, n) stays in id order; ranked items are those below `nr`
  const int K = a.kept ? *a.kept : n;
  const int nr = a.mode == kOsLater ? K : n;
  if (tid == 0) s_bid = atomicAdd(a.ticket, 1);
  __syncthreads();
  const int bid = s_bid;
  if (bid * TILE >= n) return;  // (CTAs beyond the items: before any scan)
  for (int i = tid; i < kOsWarps * (int)(kRadixBins + 1); i += kOsThreads) (&whist[0][0])[i] = 0u;
  digit_offsets(a.hist, a.hist_is_diff, s_goff, s_warp);  // (syncs the block)
  // a later depth pass whose digit is the same for every kept item is the identity
  const bool trivial =
      a.mode == kOsLater && __syncthreads_or(a.hist[tid] == K && K > 0);
  uint32_t key[ITEMS], val[ITEMS];
  const int base = bid * TILE + w * (TILE / kOsWarps);
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const int i = base + r * 32 + lane;
    key[r] = i < n ? a.kin[i] : 0u;
    val[r] = i < n ? a.vin[i] : 0u;
  }
  if (trivial) {
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
      const int i = base + r * 32 + lane;
      if (i < n) {
        a.kout[i] = key[r];
        a.vout[i] = val[r];
      }
    }
    return;
  }
  // ranks within the warp (stable: rounds in order, lanes in order)
  uint32_t rank[ITEMS];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const int i = base + r * 32 + lane;
    uint32_t d = (key[r] >> a.shift) & (kRadixBins - 1);
    if (a.mode == kOsFirst && key[r] == kDepthCulled32) d = kCulledBin;
    if (i >= nr) d = kRadixBins + 1;  // no item / pass-through tail
    rank[r] = warp_rank(whist[w], d, lane);
  }
  __syncthreads();
  {  // warp exclusive prefixes per digit, then the CTA's global offsets
    const int d = tid;
    uint32_t c = 0;
#pragma unroll
    for (int v = 0; v < kOsWarps; ++v) {
      const uint32_t t = whist[v][d];
      whist[v][d] = c;
      c += t;
    }
    const uint32_t excl = cta_prefix(a.status, a.nb, bid, d, c);
    s_goff[d] += excl;
    if (a.mode == kOsFirst) {
      // culled items before this CTA = items before it - kept items before it
      uint32_t kb = excl;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) kb += __shfl_xor_sync(0xffffffffu, kb, o);
      if (lane == 0) s_warp[w] = kb;
      __syncthreads();
      if (tid == 0) {
        uint32_t t = 0;
        for (int v = 0; v < kOsWarps; ++v) t += s_warp[v];
        s_culled_before = (uint32_t)(bid * TILE) - t;
        uint32_t cw = 0;  // warp prefixes of the culled counter
        for (int v = 0; v < kOsWarps; ++v) {
          const uint32_t x = whist[v][kCulledBin];
          whist[v][kCulledBin] = cw;
          cw += x;
        }
      }
    }
  }
  __syncthreads();
  // stable scatter: CTA offset + warp prefix + rank within the warp
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const int i = base + r * 32 + lane;
    if (i >= n) continue;
    uint32_t pos;
    if (i >= nr) {
      pos = (uint32_t)i;  // the culled tail passes through
    } else if (a.mode == kOsFirst && key[r] == kDepthCulled32) {
      pos = (uint32_t)K + s_culled_before + whist[w][kCulledBin] + rank[r];
    } else {
      const uint32_t d = (key[r] >> a.shift) & (kRadixBins - 1);
      pos = s_goff[d] + whist[w][d] + rank[r];
    }
    uint32_t k = key[r];
    if (a.tiles_x > 0) k = (k >> 8) * (uint32_t)a.tiles_x + (k & 255u);  // -> tile index
    a.kout[pos] = k;
    a.vout[pos] = val[r];
  }
}

// ---------------------------------------------------------------------------
// Pass 1 of the tile sort fused with the duplication: CTA b takes the splats
// of draw-order ranks [256 b, 256 b + 256), enumerates each one's tiles (the
// test box's tile rectangle, row by row — the order of _tile_lists) and
// scatters (tile_y << 8 | tile_x, record slot) stably by tile_x.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kOsThreads) k_dup_tx(DupArgs a) {
  pdl_wait();
  __shared__ uint32_t whist[kOsWarps][kRadixBins + 1];
  __shared__ uint32_t s_goff[kRadixBins];
  __shared__ uint32_t s_base[kOsThreads + 33];
  __shared__ uint32_t s_box[kOsThreads];  // tx0 | ty0 << 8 | ntx << 16
  __shared__ int32_t s_slot[kOsThreads];
  __shared__ uint32_t s_mag[kOsThreads];
  __shared__ uint2 s_cache[kDupCache];
  __shared__ uint32_t s_warp[8];
  __shared__ int s_bid;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t E = *a.total;
  if (tid == 0) s_bid = atomicAdd(a.ticket, 1);
  __syncthreads();
  const int bid = s_bid;
  const int K = *a.kept;
  if (E > a.cap || bid * kOsThreads >= K) return;  // (before any scan)
  for (int i = tid; i < kOsWarps * (int)(kRadixBins + 1); i += kOsThreads) (&whist[0][0])[i] = 0u;
  digit_offsets(a.hist_tx, true, s_goff, s_warp);
  const int r = bid * kOsThreads + tid;
  uint32_t cnt = 0, box = 0;
  int32_t sl = 0;
  if (r < K) {
    const uint2 br = a.bin_rec[a.sorted_ids[r]];
    if (br.y != kBinNoTiles) {
      sl = (int32_t)br.x;
      const uint32_t ntx = ((br.y >> 16) & 255u) + 1u, nty = (br.y >> 24) + 1u;
      cnt = ntx * nty;
      box = (br.y & 0xFFFFu) | (ntx << 16);
    }
  }
  // the CTA's splats with entries, compacted (draw order kept): entry starts
  // s_base[] strictly increase, so each round can find its entries' owners
  // from one 32-bit mask of start positions
  uint32_t C, M;
  const uint32_t base = block_exclusive_scan(cnt, s_warp, &C);
  const uint32_t ci = block_exclusive_scan(cnt ? 1u : 0u, s_warp, &M);
  if (cnt) {
    s_base[ci] = base;
    s_box[ci] = box;
    s_slot[ci] = sl;
    const uint32_t ntx = box >> 16;
    s_mag[ci] = ntx > 1u ? (uint32_t)(0xFFFFFFFFull / ntx + 1ull) : 0u;
  }
  for (int i = (int)M + tid; i < kOsThreads + 33; i += kOsThreads) s_base[i] = 0xFFFFFFFFu;
  __syncthreads();
  // warp w owns entries [lo, hi) of the CTA's C entries (contiguous: stable)
  const uint32_t lo = (uint32_t)(((uint64_t)C * w) / kOsWarps);
  const uint32_t hi = (uint32_t)(((uint64_t)C * (w + 1)) / kOsWarps);
  int o_lo = 0;  // owner of entry lo: last j with s_base[j] <= lo
  {
    int l = 0, h = (int)M;
    while (h - l > 1) {
      const int m = (l + h) >> 1;
      if (s_base[m] <= lo) l = m; else h = m;
    }
    o_lo = l;
  }
  // entries e0 + lane of a round: owner, then (tile_y << 8 | tile_x) and slot;
  // advances `o0` to the owner of e0 + 32
  auto round = [&](uint32_t e0, int& o0, uint32_t& key16, int32_t& slot) {
    const uint32_t p = s_base[o0 + 1 + lane] - e0;  // start positions of the next 32 splats
    const uint32_t pm = __reduce_or_sync(0xffffffffu, p < 32u ? 1u << p : 0u);
    const int owner = o0 + __popc(pm & ((2u << lane) - 1u));
    o0 += __popc(pm) + (__any_sync(0xffffffffu, p == 32u) ? 1 : 0);
    const uint32_t bx = s_box[owner];
    const uint32_t ntx = bx >> 16, j = e0 + lane - s_base[owner];
    // j / ntx: multiply-high by ceil(2^32 / ntx), exact for j, ntx < 2^16
    const uint32_t row = ntx == 1u ? j : __umulhi(j, s_mag[owner]);
    key16 = (((bx >> 8) & 255u) + row) << 8 | ((bx & 255u) + (j - row * ntx));
    slot = s_slot[owner];
  };
  // rank the entries; the CTA's entries (<= kDupCache) keep (key16 | rank << 16,
  // slot) in shared memory for the scatter, larger CTAs recompute them
  const bool cached = C <= (uint32_t)kDupCache;
  int o0 = o_lo;
  for (uint32_t e0 = lo; e0 < hi; e0 += 32) {
    uint32_t k16;
    int32_t es;
    round(e0, o0, k16, es);
    const uint32_t rk = warp_rank(whist[w], e0 + lane < hi ? (k16 & 255u) : kRadixBins + 1, lane);
    if (cached && e0 + lane < hi) s_cache[e0 + lane] = make_uint2(k16 | (rk << 16), (uint32_t)es);
  }
  __syncthreads();
  {
    const int d = tid;
    uint32_t c = 0;
#pragma unroll
    for (int v = 0; v < kOsWarps; ++v) {
      const uint32_t t = whist[v][d];
      whist[v][d] = c;
      c += t;
    }
    s_goff[d] += cta_prefix(a.status, a.nb, bid, d, c);
  }
  __syncthreads();
  if (cached) {
    for (uint32_t e = tid; e < C; e += kOsThreads) {
      const uint2 c = s_cache[e];
      const uint32_t k16 = c.x & 0xFFFFu, d = k16 & 255u;
      // the warp that ranked entry e: the last w with floor(C w / 8) <= e
      const int we = (int)(((uint64_t)(e + 1) * kOsWarps - 1) / C);
      const uint32_t pos = s_goff[d] + whist[we][d] + (c.x >> 16);
      a.kout[pos] = k16;
      a.vout[pos] = c.y;
    }
    return;
  }
  o0 = o_lo;
  for (uint32_t e0 = lo; e0 < hi; e0 += 32) {  // (uncached) sweep 2: stable scatter
    const uint32_t e = e0 + lane;
    uint32_t k16;
    int32_t es;
    round(e0, o0, k16, es);
    const uint32_t d = e < hi ? (k16 & 255u) : kRadixBins + 1;
    const uint32_t pos = warp_rank(whist[w], d, lane) + (e < hi ? s_goff[d] : 0u);
    if (e < hi) {
      a.kout[pos] = k16;
      a.vout[pos] = (uint32_t)es;
    }
  }
}

// ---------------------------------------------------------------------------
// Runs of equal 32-bit depth keys: re-order by (full fp64 key, id). The input
// order inside a run is id order (stable passes over id-ordered input).
// ---------------------------------------------------------------------------
__global__ void k_fix_runs(FixRunsArgs a) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.P) return;
  const uint32_t k = a.k32[i];
  if (k == kDepthCulled32) return;                 // the culled tail keeps id order
  if (i > 0 && a.k32[i - 1] == k) return;          // inside a run: its start handles it
  int end = i;
  while (end + 1 < a.P && end - i <= kShortRun && a.k32[end + 1] == k) ++end;
  if (end - i > kShortRun) {
    // long run: its end by binary search (the keys are sorted), then
    // k_sort_long_runs (one warp per run) orders it and writes its ranks
    int lo = end, hi = a.P;  // k32[lo] == k, answer in (lo, hi]
    while (hi - lo > 1) {
      const int m = (lo + hi) >> 1;
      if (a.k32[m] == k) lo = m; else hi = m;
    }
    const int slot = atomicAdd(a.n_long, 1);
    a.long_runs[2 * slot] = i;
    a.long_runs[2 * slot + 1] = hi - i;
    return;
  }
  int32_t* ids = a.ids;
  for (int q = i + 1; q <= end; ++q) {  // insertion sort by (full key, id)
    const int id = ids[q];
    const uint64_t key = a.k64[id];
    int b = q - 1;
    while (b >= i) {
      const int ob = ids[b];
      const uint64_t kb = a.k64[ob];
      if (kb < key || (kb == key && ob < id)) break;
      ids[b + 1] = ob;
      --b;
    }
    ids[b + 1] = id;
  }
  for (int q = i; q <= end; ++q) a.rank[ids[q]] = q;
}

// One warp per long run: if the run's full keys are not already in order, a
// stable LSD radix sort (4 x 8 bits) of the run on the low word of the fp64
// key (the high word is the run's common key), ids ping-ponging through
// `scratch`. O(run) per pass; then the ranks.
__global__ void __launch_bounds__(128) k_sort_long_runs(LongRunArgs a) {
  pdl_wait();
  __shared__ uint32_t run_ctr[4][kRadixBins + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gw = blockIdx.x * 4 + w, nw = gridDim.x * 4;
  const int nl = *a.n_long;
  for (int li = gw; li < nl; li += nw) {
    const int s = a.long_runs[2 * li], len = a.long_runs[2 * li + 1];
    int32_t* ids = a.ids + s;
    bool sorted = true;
    for (int q = lane; q + 1 < len; q += 32) {
      const uint64_t k0 = a.k64[ids[q]], k1 = a.k64[ids[q + 1]];
      sorted = sorted && k0 <= k1;  // equal keys: ids ascend already
    }
    if (!__all_sync(0xffffffffu, sorted)) {
      int32_t* src = ids;
      int32_t* dst = a.scratch + s;
      for (int pass = 0; pass < 4; ++pass) {
        uint32_t* ctr = run_ctr[w];
        for (int d = lane; d < kRadixBins; d += 32) ctr[d] = 0u;
        __syncwarp();
        for (int q0 = 0; q0 < len; q0 += 32) {  // histogram
          const int q = q0 + lane;
          const uint32_t d = q < len ? ((uint32_t)a.k64[src[q]] >> (8 * pass)) & 255u : kRadixBins + 1;
          warp_rank(ctr, d, lane);
        }
        __syncwarp();
        uint32_t run = 0;  // exclusive scan of the 256 counters, 8 per lane
        uint32_t c8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) c8[j] = ctr[lane * 8 + j];
        uint32_t t = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) t += c8[j];
        uint32_t incl = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        run = incl - t;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          ctr[lane * 8 + j] = run;
          run += c8[j];
        }
        __syncwarp();
        for (int q0 = 0; q0 < len; q0 += 32) {  // stable scatter
          const int q = q0 + lane;
          const int id = q < len ? src[q] : 0;
          const uint32_t d = q < len ? ((uint32_t)a.k64[id] >> (8 * pass)) & 255u : kRadixBins + 1;
          const uint32_t pos = warp_rank(ctr, d, lane);
          if (q < len) dst[pos] = id;
        }
        __syncwarp();
        int32_t* tmp = src; src = dst; dst = tmp;
      }
      // four passes: the result is back in `ids`
    }
    __syncwarp();
    for (int q = lane; q < len; q += 32) a.rank[ids[q]] = s + q;
  }
}

template __global__ void k_onesweep<kOsItems>(OnesweepArgs a);
static_assert(kOsItemsDepth == kOsItems, "one instantiation serves both pass kinds");

// K4: tile ranges from the tile-sorted entry keys.
__global__ void k_ranges(int64_t cap, const uint32_t* __restrict__ keys,
                         const int64_t* __restrict__ counters, int32_t* __restrict__ ranges,
                         int64_t* __restrict__ max_needed) {
  pdl_wait();
  int64_t total = counters[0];
  if (blockIdx.x == 0 && threadIdx.x == 0)  // running max (tsb_frame_workspace_max_needed_offset)
    atomicMax(reinterpret_cast<unsigned long long*>(max_needed), (unsigned long long)total);
  if (total > cap) total = 0;  // overflowed frame: leave every tile empty
  // grid-stride over the frame's entries (a fixed grid: the capacity does not
  // cost launch work)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = keys[i];
    if (i == 0 || keys[i - 1] != t) ranges[2 * t] = (int32_t)i;
    if (i == total - 1 || keys[i + 1] != t) ranges[2 * t + 1] = (int32_t)(i + 1);
  }
}

}  // namespace tsb
