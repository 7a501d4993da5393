// Insert stage: move every point into its leaf, input order kept within a leaf
// (reference partition.py:244-271; the stable argsort at partition.py:262 is what makes
// within-leaf order = input order, hazard H3).
//
// GPU form: stable LSD counting sort of the point records keyed by leaf id, reduce-then-
// scan per pass (<= 11-bit digits, at most 2 passes for <= 2^22 leaves).  The input is cut
// into CHUNKS of 4096-point sub-tiles (one CTA each):
//   K_hist    per chunk: leaf id of every point (first pass: through the target table from
//             the finest main-grid key K_count stored per point, pkey -- no record read,
//             extension descent only inside extension grids; the ids are stored for the
//             scatter), digit histogram in shared memory -> counts[chunk][B]
//   K_scan    per digit: exclusive prefix over chunks + the digit's global base (known
//             from the leaf counts of the pyramid) -> first slot of every (chunk, digit)
//   K_scatter per tile: stable in-tile ranks (warp-major, item-major, lane = input order);
//             f32 records are then permuted in shared memory into destination order and
//             stored by consecutive threads (k_dist_scatter_staged: each leaf's run leaves
//             as full sectors), f64 / leaf-id-array passes store directly (k_dist_scatter).
// Scatter CTAs take the chunks in REVERSE order: the last chunks K_hist read may still be
// in L2.  Concurrent CTAs hold adjacent chunks, so every leaf has ONE contiguous write
// front and L2 merges the 16-B records into full sectors before they reach HBM (per-
// segment fronts spread over the leaf left half-written lines and doubled DRAM traffic).
// The same happens when more records are in flight at once: 8192-point tiles, or 3 CTAs
// per SM instead of 2, raised DRAM writes from 1.0x to 2.0-2.4x of the 16 B/pt (each half-
// written sector evicted early costs a read-modify-write), so the tile stays at 4096 x 2.
// No inter-CTA waiting (no look-back chain); the counts matrix is chunks x B x 4 B
// (= 2 n bytes at 11-bit digits).  HBM traffic per point, single pass: 4 B read + 4 B
// written (hist), 4 B + 16 B read and 16 B written (scatter).
#include <algorithm>

#include "kernels.h"

namespace lod {

namespace {

constexpr int kW = kRadixThreads / 32;
constexpr int K = kRadixItems;


// Leaf ids of one warp's K x 32 items starting at `base`.  FIRST: through the target table
// from the point's finest main-grid key (no record read, no fp64 projection); points inside
// extension grids (target <= -2) take the id K_ext_leaf resolved from the extension list
// (ext_leaf, indexed by point); else the ids of the previous pass.
template <int FMT, bool FIRST, bool TAGIN>
__device__ __forceinline__ void load_items(const SplitView& v, const void* in_rec, const uint32_t* in_leaf,
                                           const uint32_t* ext_leaf, uint64_t base, int lane, uint32_t (&leaf)[K],
                                           bool& unresolved) {
  const uint64_t last = v.n - 1;
  if (FIRST) {
    uint32_t key[K];
    const uint64_t keep = policy_evict_last(), stream = policy_evict_first();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t i = base + (uint64_t)k * 32 + lane;
      key[k] = ld_hint(v.pkey + (i < last ? i : last), stream);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) leaf[k] = (uint32_t)ld_hint(v.t8 + key[k], keep);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t i = base + (uint64_t)k * 32 + lane;
      int32_t t = (int32_t)leaf[k];
      if (t <= -2) t = (int32_t)__ldcg(ext_leaf + (i < last ? i : last));
      if (t < 0) {
        unresolved |= i < v.n;
        t = 0;
      }
      leaf[k] = (uint32_t)t;
    }
  } else if (TAGIN) {  // 2nd pass: the digit from the byte stream pass 1 wrote (f32), else the record's pad
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t i = base + (uint64_t)k * 32 + lane;
      leaf[k] = in_leaf ? (uint32_t)__ldcs(reinterpret_cast<const uint8_t*>(in_leaf) + (i < last ? i : last))
                        : Rec<FMT>::tag(Rec<FMT>::load(in_rec, i < last ? i : last));  // re-read at the store
    }
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t i = base + (uint64_t)k * 32 + lane;
      leaf[k] = __ldg(in_leaf + (i < last ? i : last));
    }
  }
}


// ---------------------------------------------------------------------------
// K_hist: per-chunk digit counts
// ---------------------------------------------------------------------------
template <int FMT, bool FIRST, bool TAGIN>
__global__ void __launch_bounds__(kRadixThreads, 3)
    k_dist_hist(SplitView v, const void* in_rec, const uint32_t* in_leaf, uint32_t* leaf_out, int shift, int bits,
                uint32_t seg_tiles, uint32_t tiles, uint32_t* counts) {
  pdl_wait();
  extern __shared__ __align__(16) uint32_t hist[];
  const int B = 1 << bits;
  for (int d = threadIdx.x; d < B; d += kRadixThreads) hist[d] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bool unresolved = false;
  const uint32_t t0 = blockIdx.x * seg_tiles, t1 = min(t0 + seg_tiles, tiles);
  for (uint32_t tile = t0; tile < t1; ++tile) {
    const uint64_t base = (uint64_t)tile * kRadixTile + (uint64_t)warp * 32 * K;
    uint32_t leaf[K];
    load_items<FMT, FIRST, TAGIN>(v, in_rec, in_leaf, leaf_out, base, lane, leaf, unresolved);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool valid = base + (uint64_t)k * 32 + lane < v.n;
      if (FIRST && valid) leaf_out[base + (uint64_t)k * 32 + lane] = leaf[k];  // the scatter reuses it
      const uint32_t d = (leaf[k] >> shift) & (B - 1);
      if (TAGIN) {  // 2nd pass: the records are sorted by the 1st digit, the 2nd is scattered
        if (valid) atomicAdd(hist + d, 1u);
        continue;
      }
      // warp-uniform digit (coherent scans): one add; otherwise plain shared atomics
      // (MATCH.ANY would saturate the MIO pipe: it was the top stall here)
      const uint32_t d0 = __shfl_sync(0xFFFFFFFFu, d, 0);
      const unsigned act = __ballot_sync(0xFFFFFFFFu, valid);
      if (__all_sync(0xFFFFFFFFu, !valid || d == d0)) {
        if (lane == 0 && act) atomicAdd(hist + d0, (uint32_t)__popc(act));
      } else if (valid) {
        atomicAdd(hist + d, 1u);
      }
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < B; d += kRadixThreads) counts[(uint64_t)blockIdx.x * B + d] = hist[d];
  if (FIRST) {
    if (__any_sync(0xFFFFFFFFu, unresolved) && lane == 0) raise_err(v.st, ERR_UNRESOLVED);
  }
}

// ---------------------------------------------------------------------------
// K_scan: counts[g][d] -> digit_base[d] + sum_{g' < g} counts[g'][d]  (first slots), as
// three parallel steps over (32-digit column, segment of rows) blocks:
//   part  per segment and digit: the segment's column sums        -> part[seg][d]
//   scan  per digit: exclusive prefix over the segments + base     (one small block)
//   apply per segment: exclusive prefix of its rows from part[seg][d], in place
// (one block per 32 digits walking every row serially took 2.7 ms at 500M points).
// Inside a block the segment's rows are split over the 32 warps; lanes are digits.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void rows_of(uint32_t rows, uint32_t seg_rows, uint32_t seg, int warp, uint32_t& g0,
                                        uint32_t& g1) {
  const uint32_t r0 = min(rows, seg * seg_rows), r1 = min(rows, r0 + seg_rows);
  const uint32_t per = (r1 - r0 + 31) / 32;
  g0 = min(r1, r0 + warp * per);
  g1 = min(r1, g0 + per);
}

__global__ void __launch_bounds__(1024) k_dist_scan_part(const uint32_t* counts, uint32_t rows, uint32_t seg_rows,
                                                         int B, uint32_t* part) {
  pdl_wait();
  __shared__ uint32_t sm[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = blockIdx.x * 32 + lane;
  uint32_t g0, g1;
  rows_of(rows, seg_rows, blockIdx.y, warp, g0, g1);
  uint32_t sum = 0;
  if (d < B) {
#pragma unroll 8
    for (uint32_t g = g0; g < g1; ++g) sum += __ldcg(counts + (uint64_t)g * B + d);
  }
  sm[warp][lane] = sum;
  __syncthreads();
  if (warp == 0 && d < B) {
    uint32_t t = 0;
    for (int w = 0; w < 32; ++w) t += sm[w][lane];
    part[(uint64_t)blockIdx.y * B + d] = t;
  }
}

// exclusive prefix of rows [0, rows) of a[g][d], plus base[d] (if any), in place
__global__ void __launch_bounds__(1024) k_dist_scan_apply(uint32_t* a, uint32_t rows, uint32_t seg_rows, int B,
                                                          const uint32_t* seg_base, const uint64_t* base) {
  pdl_wait();
  __shared__ uint32_t part[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = blockIdx.x * 32 + lane;
  uint32_t g0, g1;
  rows_of(rows, seg_rows, blockIdx.y, warp, g0, g1);
  uint32_t sum = 0;
  if (d < B) {
#pragma unroll 8
    for (uint32_t g = g0; g < g1; ++g) sum += a[(uint64_t)g * B + d];
  }
  part[warp][lane] = sum;
  __syncthreads();
  if (warp == 0) {
    uint32_t run = d >= B ? 0 : seg_base ? seg_base[(uint64_t)blockIdx.y * B + d] : (uint32_t)base[d];
    for (int w = 0; w < 32; ++w) {
      const uint32_t c = part[w][lane];
      part[w][lane] = run;
      run += c;
    }
  }
  __syncthreads();
  if (d < B) {  // the loads run ahead of the dependent stores
    uint32_t run = part[warp][lane];
    uint32_t g = g0;
    for (; g + 8 <= g1; g += 8) {
      uint32_t c[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) c[q] = a[(uint64_t)(g + q) * B + d];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        a[(uint64_t)(g + q) * B + d] = run;
        run += c[q];
      }
    }
    for (; g < g1; ++g) {
      const uint32_t c = a[(uint64_t)g * B + d];
      a[(uint64_t)g * B + d] = run;
      run += c;
    }
  }
}

// first slots of every (tile, digit); part: >= 2 * kScanSegs * B words of scratch
constexpr uint32_t kScanSegs = 512;
int launch_dist_scan(uint32_t* counts, uint32_t rows, int B, const uint64_t* digit_base, uint32_t* part,
                     cudaStream_t s) {
  const uint32_t dcols = ceil_div_u32(B, 32);
  const uint32_t seg_rows = std::max<uint32_t>(768, ceil_div_u32(rows, kScanSegs));  // ~24 rows per warp
  const uint32_t segs = ceil_div_u32(rows, seg_rows);
  if (segs <= 1) {
    launch_pdl(k_dist_scan_apply, dim3(dcols, 1), 1024, 0, s, counts, rows, rows, B, nullptr, digit_base);
    return 1;
  }
  launch_pdl(k_dist_scan_part, dim3(dcols, segs), 1024, 0, s, counts, rows, seg_rows, B, part);
  launch_pdl(k_dist_scan_apply, dim3(dcols, 1), 1024, 0, s, part, segs, segs, B, nullptr, digit_base);
  launch_pdl(k_dist_scan_apply, dim3(dcols, segs), 1024, 0, s, counts, rows, seg_rows, B, part, nullptr);
  return 3;
}

// ---------------------------------------------------------------------------
// K_scatter: stable scatter; chunks in reverse launch order, sub-tiles in order
// ---------------------------------------------------------------------------
// OUT: what travels to the next pass with each record
enum { OUT_FINAL = 0, OUT_LEAF = 1, OUT_TAG = 2 };

template <int FMT, bool TAGIN, int OUT>
__global__ void __launch_bounds__(kRadixThreads, 2)
    k_dist_scatter(SplitView v, const void* in_rec, const uint32_t* in_leaf, void* out_rec, uint32_t* out_leaf,
                   int shift, int bits, int tag_shift, uint32_t seg_tiles, uint32_t tiles, const uint32_t* firsts) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t smem[];
  const int B = 1 << bits;
  uint32_t* run = reinterpret_cast<uint32_t*>(smem);               // [B] first slot of the sub-tile
  uint32_t* tot = run + B;                                          // [B] sub-tile digit totals
  uint16_t* wh = reinterpret_cast<uint16_t*>(smem + (size_t)B * 8);  // [kW][B] warp counts -> prefixes
  const uint32_t chunk = gridDim.x - 1 - blockIdx.x;
  for (int d = threadIdx.x; d < B; d += kRadixThreads) run[d] = firsts[(uint64_t)chunk * B + d];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt_mask = (1u << lane) - 1;
  bool unresolved = false;
  const uint32_t t0 = chunk * seg_tiles, t1 = min(t0 + seg_tiles, tiles);
  for (uint32_t tile = t0; tile < t1; ++tile) {
    for (int i = threadIdx.x; i < kW * B / 2; i += kRadixThreads) reinterpret_cast<uint32_t*>(wh)[i] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)tile * kRadixTile + (uint64_t)warp * 32 * K;
    uint32_t leaf[K];
    uint16_t rk[K];
    load_items<FMT, false, TAGIN>(v, in_rec, in_leaf, nullptr, base, lane, leaf, unresolved);
    // stable in-warp ranks (item-major, lane order)
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool valid = base + (uint64_t)k * 32 + lane < v.n;
      const uint32_t d = (leaf[k] >> shift) & (B - 1);
      // lanes with the same digit: multi-split by ballots over the digit bits (a handful
      // of VOTEs instead of one MATCH.ANY, which bottlenecked on the MIO pipe)
      unsigned peers = __ballot_sync(0xFFFFFFFFu, valid);
      const unsigned act = peers;
      for (int b = 0; b < bits; ++b) {
        const bool on = (d >> b) & 1;
        const unsigned m = __ballot_sync(0xFFFFFFFFu, on);
        peers &= on ? m : ~m;
      }
      uint32_t rank = 0;
      if (valid) {
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (lane == leader) {
          old = wh[warp * B + d];
          wh[warp * B + d] = (uint16_t)(old + __popc(peers));
        }
        old = __shfl_sync(act, old, leader);
        rank = old + __popc(peers & lt_mask);
      }
      rk[k] = (uint16_t)rank;
      __syncwarp();
    }
    __syncthreads();
    // cross-warp exclusive prefix per digit (the sub-tile's block for digit d starts at run[d])
    for (int d = threadIdx.x; d < B; d += kRadixThreads) {
      uint32_t r = 0;
#pragma unroll 4
      for (int w = 0; w < kW; ++w) {
        const uint32_t c = wh[w * B + d];
        wh[w * B + d] = (uint16_t)r;
        r += c;
      }
      tot[d] = r;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t i = base + (uint64_t)k * 32 + lane;
      if (i < v.n) {
        const uint32_t d = (leaf[k] >> shift) & (B - 1);
        const uint64_t dest = (uint64_t)run[d] + wh[warp * B + d] + rk[k];
        auto rec = Rec<FMT>::load(in_rec, i);
        if (OUT == OUT_TAG) Rec<FMT>::set_tag(rec, leaf[k] >> tag_shift);  // the next pass's digit
        if (OUT == OUT_FINAL && TAGIN) Rec<FMT>::set_tag(rec, 0);
        Rec<FMT>::store(out_rec, dest, rec);
        if (OUT == OUT_LEAF) out_leaf[dest] = leaf[k];
      }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < B; d += kRadixThreads) run[d] += tot[d];
  }
}

// ---------------------------------------------------------------------------
// K_scatter, staged form (f32 records, digit from the leaf ids): the same stable ranks, but
// the tile is permuted in shared memory into destination order (digit, then rank) before it
// is stored, so consecutive threads store consecutive slots of a leaf's run -- full sectors
// and a few lines per warp instead of 32 scattered 16-B writes (313 -> ~200 us of stores at
// terrain20M).  The per-(digit, warp) count rows and the record stage share one region:
// the rows are dead once every point knows its slot.
// ---------------------------------------------------------------------------
template <int NB>
__device__ __forceinline__ unsigned digit_peers(uint32_t d, unsigned peers) {
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const bool on = (d & (1u << b)) != 0;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, on);
    peers &= on ? m : ~m;
  }
  return peers;
}

// digit-major rows of kW u16 counts, padded to an odd word stride so one thread prefixes a
// row with 8 word loads and the leaders of a warp (distinct digits) spread over the banks
constexpr int kRowWords = kW / 2 + 1;
__host__ __device__ constexpr size_t staged_region(int B) {  // count rows / record stage (16-B aligned)
  return std::max<size_t>(((size_t)B * kRowWords * 4 + 15) & ~(size_t)15, (size_t)kRadixTile * 16);
}
__host__ __device__ constexpr size_t staged_smem(int B) { return staged_region(B) + (size_t)kRadixTile * 4 + (size_t)B * 8; }

// TAGOUT (1st of 2 passes): the 2nd digit travels in the record's pad AND in a byte stream in
// destination order (out_tag, 1 B/pt), so the 2nd pass reads its digits -- histogram and
// ranks -- from 1 B/pt instead of re-reading the 16-B records.  TAGIN: digits from that
// stream (in_leaf, as bytes); the pad is cleared on output.
template <bool TAGIN, bool TAGOUT, int NB>
__global__ void __launch_bounds__(kRadixThreads, 2)
    k_dist_scatter_staged(SplitView v, const void* in_rec, const uint32_t* in_leaf, void* out_rec, int bits,
                          int tag_shift, const uint32_t* firsts, uint8_t* out_tag) {
  pdl_wait();
  extern __shared__ __align__(16) uint32_t sm[];
  const int B = 1 << bits;
  uint32_t* wh = sm;                        // [B][kRowWords] counts, then
  uint4* srec = reinterpret_cast<uint4*>(wh);  // [tile] the records in destination order
  uint32_t* sdst = sm + staged_region(B) / 4;  // [tile] global slot of local slot j
  uint32_t* run = sdst + kRadixTile;        // [B] the tile's first global slot per digit
  uint32_t* tf = run + B;                   // [B] tile-local first slot per digit
  uint16_t* wh16 = reinterpret_cast<uint16_t*>(wh);
  const uint32_t tile = gridDim.x - 1 - blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    const uint32_t n4 = (uint32_t)(((size_t)B * kRowWords + 3) / 4);
    for (uint32_t i = threadIdx.x; i < n4; i += kRadixThreads) reinterpret_cast<uint4*>(wh)[i] = make_uint4(0, 0, 0, 0);
    for (int d = threadIdx.x; d < B; d += kRadixThreads) run[d] = __ldcs(firsts + (uint64_t)tile * B + d);
  }
  const uint64_t base = (uint64_t)tile * kRadixTile + (uint64_t)warp * 32 * K;
  const uint64_t last = v.n - 1;
  uint32_t leaf[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint64_t i = min(base + (uint64_t)k * 32 + lane, last);
    leaf[k] = TAGIN ? (uint32_t)__ldcs(reinterpret_cast<const uint8_t*>(in_leaf) + i) : __ldcs(in_leaf + i);
  }
  __syncthreads();
  // stable in-warp ranks (item-major, lane order)
  const uint32_t lt_mask = (1u << lane) - 1;
  uint32_t rk[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool valid = base + (uint64_t)k * 32 + lane < v.n;
    const uint32_t d = leaf[k] & (B - 1);
    const unsigned act = __ballot_sync(0xFFFFFFFFu, valid);
    const unsigned peers = digit_peers<NB>(d, act);
    uint32_t rank = 0;
    if (valid) {
      const int leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if (lane == leader) {
        uint16_t* c = wh16 + (size_t)d * (2 * kRowWords) + warp;
        old = *c;
        *c = (uint16_t)(old + __popc(peers));
      }
      old = __shfl_sync(act, old, leader);
      rank = old + __popc(peers & lt_mask);
    }
    rk[k] = rank;
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive prefix over the warps in warp order; the row total -> tf
  for (int d = threadIdx.x; d < B; d += kRadixThreads) {
    uint32_t* row = wh + (size_t)d * kRowWords;
    uint32_t r = 0;
#pragma unroll
    for (int q = 0; q < kW / 2; ++q) {
      const uint32_t c = row[q], lo = c & 0xFFFF;
      row[q] = r | ((r + lo) << 16);
      r += lo + (c >> 16);
    }
    tf[d] = r;
  }
  __syncthreads();
  {  // tile-local first slot per digit: exclusive scan of the totals (consecutive digits per thread)
    __shared__ uint32_t wsum[kW + 1];
    const int per = (B + kRadixThreads - 1) / kRadixThreads;
    const int d0 = threadIdx.x * per;
    uint32_t c = 0;
    for (int j = 0; j < per; ++j) c += d0 + j < B ? tf[d0 + j] : 0;
    uint32_t tot;
    uint32_t x = block_excl_scan<uint32_t, kRadixThreads>(c, &tot, wsum);
    for (int j = 0; j < per; ++j)
      if (d0 + j < B) {
        const uint32_t t = tf[d0 + j];
        tf[d0 + j] = x;
        x += t;
      }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (base + (uint64_t)k * 32 + lane < v.n) {
      const uint32_t d = leaf[k] & (B - 1);
      const uint32_t w = wh16[(size_t)d * (2 * kRowWords) + warp] + rk[k];
      rk[k] = tf[d] + w;          // local slot
      sdst[rk[k]] = run[d] + w;   // its global slot
    }
  }
  __syncthreads();  // the count rows are dead: the region becomes the record stage
  constexpr int G = 4;
#pragma unroll
  for (int g = 0; g < K; g += G) {
    uint4 r[G];
#pragma unroll
    for (int u = 0; u < G; ++u) r[u] = __ldcs(reinterpret_cast<const uint4*>(in_rec) + min(base + (uint64_t)(g + u) * 32 + lane, last));
#pragma unroll
    for (int u = 0; u < G; ++u) {
      if (base + (uint64_t)(g + u) * 32 + lane < v.n) {
        if (TAGOUT) r[u].w = (r[u].w & 0xFFFFFFu) | ((leaf[g + u] >> tag_shift) << 24);  // the next pass's digit
        if (TAGIN) r[u].w &= 0xFFFFFFu;
        srec[rk[g + u]] = r[u];
      }
    }
  }
  __syncthreads();
  const uint32_t tile_n = (uint32_t)min((uint64_t)kRadixTile, v.n - (uint64_t)tile * kRadixTile);
  for (uint32_t j = threadIdx.x; j < tile_n; j += kRadixThreads) {
    const uint4 r = srec[j];
    reinterpret_cast<uint4*>(out_rec)[sdst[j]] = r;
    if (TAGOUT) out_tag[sdst[j]] = (uint8_t)(r.w >> 24);
  }
}

// ---------------------------------------------------------------------------
// K_scatter, TMA form (f32 records, digits <= 9 bits: the 2-pass distributes of large clouds).
// The staged kernel loads the tile's records only after ranking it; here one thread starts a
// 1-D bulk copy (cp.async.bulk, completion on an mbarrier) of the tile's 64 KB of records into
// shared memory at kernel entry, so the load streams in under the whole ranking.  Per local
// slot one word {item in tile (12 b), digit (9 b), next pass's tag (8 b)} replaces the slot
// arrays; the store pass gathers slot j's record from the stage and writes it to
// run[d] + (j - first local slot of d).  102 KB of shared memory at B = 512: 2 CTAs per SM.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__host__ __device__ constexpr size_t tma_rows(int B) { return ((size_t)B * kRowWords * 4 + 15) & ~(size_t)15; }
__host__ __device__ constexpr size_t tma_smem(int B) {
  return (size_t)kRadixTile * 16 + tma_rows(B) + (size_t)kRadixTile * 4 + (size_t)B * 8;
}

template <bool TAGIN, bool TAGOUT, int NB>
__global__ void __launch_bounds__(kRadixThreads, 2)
    k_dist_scatter_tma(SplitView v, const void* in_rec, const uint32_t* in_leaf, void* out_rec, int bits,
                       int tag_shift, const uint32_t* firsts, uint8_t* out_tag) {
  pdl_wait();
  extern __shared__ __align__(128) uint32_t sm[];
  __shared__ __align__(8) uint64_t bar;
  const int B = 1 << bits;
  uint4* srec = reinterpret_cast<uint4*>(sm);                                        // [tile] input order
  uint32_t* wh = sm + kRadixTile * 4;                                                // [B][kRowWords]
  uint32_t* sinfo = wh + tma_rows(B) / 4;                                            // [tile] per local slot
  uint32_t* run = sinfo + kRadixTile;                                                // [B]
  uint32_t* tf = run + B;                                                            // [B]
  uint16_t* wh16 = reinterpret_cast<uint16_t*>(wh);
  const uint32_t tile = gridDim.x - 1 - blockIdx.x;
  const uint32_t tile_n = (uint32_t)min((uint64_t)kRadixTile, v.n - (uint64_t)tile * kRadixTile);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(tile_n * 16)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(srec)),
                 "l"(reinterpret_cast<const uint4*>(in_rec) + (uint64_t)tile * kRadixTile), "r"(tile_n * 16),
                 "r"(smem_u32(&bar))
                 : "memory");
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    const uint32_t n4 = (uint32_t)(((size_t)B * kRowWords + 3) / 4);
    for (uint32_t i = threadIdx.x; i < n4; i += kRadixThreads) reinterpret_cast<uint4*>(wh)[i] = make_uint4(0, 0, 0, 0);
    for (int d = threadIdx.x; d < B; d += kRadixThreads) run[d] = __ldcs(firsts + (uint64_t)tile * B + d);
  }
  const uint32_t item0 = (uint32_t)warp * 32 * K;
  const uint64_t base = (uint64_t)tile * kRadixTile + item0;
  const uint64_t last = v.n - 1;
  uint32_t leaf[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint64_t i = min(base + (uint64_t)k * 32 + lane, last);
    leaf[k] = TAGIN ? (uint32_t)__ldcs(reinterpret_cast<const uint8_t*>(in_leaf) + i) : __ldcs(in_leaf + i);
  }
  __syncthreads();
  const uint32_t lt_mask = (1u << lane) - 1;
  uint32_t rk[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool valid = base + (uint64_t)k * 32 + lane < v.n;
    const uint32_t d = leaf[k] & (B - 1);
    const unsigned act = __ballot_sync(0xFFFFFFFFu, valid);
    const unsigned peers = digit_peers<NB>(d, act);
    uint32_t rank = 0;
    if (valid) {
      const int leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if (lane == leader) {
        uint16_t* c = wh16 + (size_t)d * (2 * kRowWords) + warp;
        old = *c;
        *c = (uint16_t)(old + __popc(peers));
      }
      old = __shfl_sync(act, old, leader);
      rank = old + __popc(peers & lt_mask);
    }
    rk[k] = rank;
    __syncwarp();
  }
  __syncthreads();
  for (int d = threadIdx.x; d < B; d += kRadixThreads) {
    uint32_t* row = wh + (size_t)d * kRowWords;
    uint32_t r = 0;
#pragma unroll
    for (int q = 0; q < kW / 2; ++q) {
      const uint32_t c = row[q], lo = c & 0xFFFF;
      row[q] = r | ((r + lo) << 16);
      r += lo + (c >> 16);
    }
    tf[d] = r;
  }
  __syncthreads();
  {
    __shared__ uint32_t wsum[kW + 1];
    const int per = (B + kRadixThreads - 1) / kRadixThreads;
    const int d0 = threadIdx.x * per;
    uint32_t c = 0;
    for (int j = 0; j < per; ++j) c += d0 + j < B ? tf[d0 + j] : 0;
    uint32_t tot;
    uint32_t x = block_excl_scan<uint32_t, kRadixThreads>(c, &tot, wsum);
    for (int j = 0; j < per; ++j)
      if (d0 + j < B) {
        const uint32_t t = tf[d0 + j];
        tf[d0 + j] = x;
        x += t;
      }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (base + (uint64_t)k * 32 + lane < v.n) {
      const uint32_t d = leaf[k] & (B - 1);
      const uint32_t slot = tf[d] + wh16[(size_t)d * (2 * kRowWords) + warp] + rk[k];
      const uint32_t tag = TAGOUT ? (leaf[k] >> tag_shift) & 0xFF : 0u;
      sinfo[slot] = (item0 + (uint32_t)k * 32 + lane) | (d << 12) | (tag << 21);
    }
  }
  __syncthreads();
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(&bar))
      : "memory");
  for (uint32_t j = threadIdx.x; j < tile_n; j += kRadixThreads) {
    const uint32_t info = sinfo[j];
    const uint32_t d = (info >> 12) & 0x1FF;
    uint4 r = srec[info & 0xFFF];
    if (TAGOUT) r.w = (r.w & 0xFFFFFFu) | ((info >> 21) << 24);
    if (TAGIN) r.w &= 0xFFFFFFu;
    const uint32_t g = run[d] + (j - tf[d]);
    reinterpret_cast<uint4*>(out_rec)[g] = r;
    if (TAGOUT) out_tag[g] = (uint8_t)(info >> 21);
  }
}

// Global exclusive prefix per digit, from the leaf counts (leaf ids are the sort keys).
__global__ void k_digit_hist(const uint32_t* leaf_count, uint32_t n_leaves, int shift, int bits,
                             unsigned long long* hist) {
  pdl_wait();
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_leaves) return;
  atomicAdd(hist + ((j >> shift) & ((1u << bits) - 1)), (unsigned long long)leaf_count[j]);
}

__global__ void __launch_bounds__(1024) k_digit_scan(uint64_t* hist, int B) {
  pdl_wait();
  __shared__ uint64_t sm[1024 / 32 + 1];
  uint64_t a = (2 * threadIdx.x < (unsigned)B) ? hist[2 * threadIdx.x] : 0;
  uint64_t b = (2 * threadIdx.x + 1 < (unsigned)B) ? hist[2 * threadIdx.x + 1] : 0;
  uint64_t tot;
  uint64_t ex = block_excl_scan<uint64_t, 1024>(a + b, &tot, sm);
  if (2 * threadIdx.x < (unsigned)B) hist[2 * threadIdx.x] = ex;
  if (2 * threadIdx.x + 1 < (unsigned)B) hist[2 * threadIdx.x + 1] = ex + a;
}

// One digit pass.  FIRST: the leaf ids are resolved once by K_hist, which stores them
// (leaf_tmp) for K_scatter.  TAGIN: the digit is read from the records' pad (written by the
// previous pass with OUT_TAG); OUT_LEAF: the leaf ids travel in a separate array.
template <int FMT, bool FIRST, bool TAGIN, int OUT>
int run_pass(const SplitView& v, const void* in_rec, const uint32_t* in_leaf, uint32_t* leaf_tmp, void* out_rec,
             uint32_t* out_leaf, int shift, int bits, int tag_shift, const uint64_t* digit_base, const RadixPlan& p,
             cudaStream_t s, uint8_t* out_tag = nullptr) {
  const int B = 1 << bits;
  auto hist = k_dist_hist<FMT, FIRST, TAGIN>;
  auto scat = k_dist_scatter<FMT, TAGIN, OUT>;
  const size_t hsm = (size_t)B * 4, ssm = (size_t)B * 8 + (size_t)kW * B * 2 + 4 * kW;
  const uint32_t* leaf_in = FIRST ? leaf_tmp : in_leaf;
  launch_pdl(hist, p.segs, kRadixThreads, hsm, s, v, in_rec, in_leaf, leaf_tmp, shift, bits, p.seg_tiles, p.tiles, p.counts);
  if (FIRST && p.aux) cudaStreamWaitEvent(s, p.aux_ev[1], 0);  // the digit bases
  const int nscan = launch_dist_scan(p.counts, p.segs, B, digit_base, p.scan_part, s);
  const cudaEvent_t* ev = p.scatter_ev + (FIRST ? 0 : 2);
  if (ev[0]) cudaEventRecord(ev[0], s);
  // staged, coalesced stores whenever the digit starts at bit 0 (pass 1: leaf id; pass 2: pad)
  constexpr bool kStaged = FMT == LOD_POINTS_F32 && (FIRST || TAGIN) && OUT != OUT_LEAF;
  if (kStaged && p.seg_tiles == 1 && shift == 0) {
    // one ballot per digit bit in the in-warp multi-split: instantiate the exact width
    using K = void (*)(SplitView, const void*, const uint32_t*, void*, int, int, const uint32_t*, uint8_t*);
    constexpr bool TO = OUT == OUT_TAG;
    const K by_bits[kRadixMaxBits + 1] = {
        k_dist_scatter_staged<TAGIN, TO, 1>, k_dist_scatter_staged<TAGIN, TO, 1>, k_dist_scatter_staged<TAGIN, TO, 2>,
        k_dist_scatter_staged<TAGIN, TO, 3>, k_dist_scatter_staged<TAGIN, TO, 4>, k_dist_scatter_staged<TAGIN, TO, 5>,
        k_dist_scatter_staged<TAGIN, TO, 6>, k_dist_scatter_staged<TAGIN, TO, 7>, k_dist_scatter_staged<TAGIN, TO, 8>,
        k_dist_scatter_staged<TAGIN, TO, 9>, k_dist_scatter_staged<TAGIN, TO, 10>, k_dist_scatter_staged<TAGIN, TO, 11>};
    const K by_bits_tma[10] = {
        k_dist_scatter_tma<TAGIN, TO, 1>, k_dist_scatter_tma<TAGIN, TO, 1>, k_dist_scatter_tma<TAGIN, TO, 2>,
        k_dist_scatter_tma<TAGIN, TO, 3>, k_dist_scatter_tma<TAGIN, TO, 4>, k_dist_scatter_tma<TAGIN, TO, 5>,
        k_dist_scatter_tma<TAGIN, TO, 6>, k_dist_scatter_tma<TAGIN, TO, 7>, k_dist_scatter_tma<TAGIN, TO, 8>,
        k_dist_scatter_tma<TAGIN, TO, 9>};
    if (bits <= 9 && (reinterpret_cast<uintptr_t>(in_rec) & 15) == 0)  // records in flight under the ranking
      launch_pdl(by_bits_tma[bits], p.segs, kRadixThreads, tma_smem(B), s, v, in_rec, leaf_in, out_rec, bits, tag_shift,
                 p.counts, out_tag);
    else
      launch_pdl(by_bits[bits], p.segs, kRadixThreads, staged_smem(B), s, v, in_rec, leaf_in, out_rec, bits,
                 tag_shift, p.counts, out_tag);
  } else {
    launch_pdl(scat, p.segs, kRadixThreads, ssm, s, v, in_rec, leaf_in, out_rec, out_leaf, shift, bits, tag_shift,
               p.seg_tiles, p.tiles, p.counts);
  }
  if (ev[1]) cudaEventRecord(ev[1], s);
  return 2 + nscan;
}

template <int FMT>
int distribute_fmt(const SplitView& v, RadixPlan& p, void* leaf_out, cudaStream_t s) {
  int launches = 0;
  const int B0 = 1 << p.bits[0];
  const int B1 = p.passes > 1 ? 1 << p.bits[1] : 0;
  uint64_t* base0 = p.digit_base;
  uint64_t* base1 = p.digit_base + B0;
  // the global digit bases (from the leaf counts) on the side stream, under the first K_hist;
  // run_pass waits for them before its scan
  cudaStream_t a = p.aux ? p.aux : s;
  if (p.aux) {
    cudaEventRecord(p.aux_ev[0], s);
    cudaStreamWaitEvent(a, p.aux_ev[0], 0);
  }
  cudaMemsetAsync(p.digit_base, 0, (size_t)(B0 + B1) * 8, a);
  uint32_t lb = ceil_div_u32(v.n_leaves, 256);
  launch_pdl(k_digit_hist, lb, 256, 0, a, v.leaf_count, v.n_leaves, 0, p.bits[0],
             reinterpret_cast<unsigned long long*>(base0));
  launch_pdl(k_digit_scan, 1, 1024, 0, a, base0, B0);
  launches += 2;
  if (p.passes > 1) {
    launch_pdl(k_digit_hist, lb, 256, 0, a, v.leaf_count, v.n_leaves, p.bits[0], p.bits[1],
               reinterpret_cast<unsigned long long*>(base1));
    launch_pdl(k_digit_scan, 1, 1024, 0, a, base1, B1);
    launches += 2;
  }
  if (p.aux) cudaEventRecord(p.aux_ev[1], a);
  if (v.elist) launches += launch_ext_leaf(v, p.tmp_leaf, s);  // leaf ids of the extension points
  if (p.passes == 1)
    return launches + run_pass<FMT, true, false, OUT_FINAL>(v, v.pts, nullptr, p.tmp_leaf, leaf_out, nullptr, 0,
                                                           p.bits[0], 0, base0, p, s);
  if (p.bits[1] <= Rec<FMT>::kTagBits) {
    // the 2nd digit rides in the record pad: no scattered 4-B leaf-id stream (its partial
    // sectors cost read-modify-writes), the 2nd pass reads digits from the records
    // f32: the 2nd digit also as a byte stream in destination order (after the input-order ids)
    uint8_t* tags = FMT == LOD_POINTS_F32 ? reinterpret_cast<uint8_t*>(p.tmp_leaf + v.n) : nullptr;
    launches += run_pass<FMT, true, false, OUT_TAG>(v, v.pts, nullptr, p.tmp_leaf, p.tmp_rec, nullptr, 0,
                                                    p.bits[0], p.bits[0], base0, p, s, tags);
    launches += run_pass<FMT, false, true, OUT_FINAL>(v, p.tmp_rec, reinterpret_cast<const uint32_t*>(tags), nullptr,
                                                      leaf_out, nullptr, 0, p.bits[1], 0, base1, p, s);
    return launches;
  }
  uint32_t* sorted_leaf = p.tmp_leaf + v.n;
  launches += run_pass<FMT, true, false, OUT_LEAF>(v, v.pts, nullptr, p.tmp_leaf, p.tmp_rec, sorted_leaf, 0,
                                                   p.bits[0], 0, base0, p, s);
  launches += run_pass<FMT, false, false, OUT_FINAL>(v, p.tmp_rec, sorted_leaf, nullptr, leaf_out, nullptr,
                                                     p.bits[0], p.bits[1], 0, base1, p, s);
  return launches;
}

}  // namespace

// Chunking of n points: one sub-tile per chunk.  Larger chunks shrink the counts matrix
// but spread each leaf's write front over many half-written lines (measured: 4 sub-tiles
// per chunk -> +35% DRAM writes, +75% reads from read-modify-write of partial sectors).
__global__ void k_check_count(DevState* st, uint64_t n) {
  pdl_wait();
  if (st->count_b != n) raise_err(st, ERR_COUNT);  // partition.py:268-269
}

int launch_check_count(DevState* st, uint64_t n, cudaStream_t s) {
  launch_pdl(k_check_count, 1, 1, 0, s, st, n);
  return 1;
}

void plan_segments(RadixPlan& p, uint64_t n, int sms) {
  (void)sms;
  p.tiles = (uint32_t)((n + kRadixTile - 1) / kRadixTile);
  p.seg_tiles = 1;
  p.segs = std::max<uint32_t>(1, (p.tiles + p.seg_tiles - 1) / p.seg_tiles);
}

int launch_distribute(int fmt, const SplitView& v, RadixPlan& p, void* leaf_out, cudaStream_t s) {
  if (p.passes == 0) {  // one leaf: the whole cloud in input order
    size_t rec = fmt == LOD_POINTS_F32 ? 16 : 32;
    cudaMemcpyAsync(leaf_out, v.pts, v.n * rec, cudaMemcpyDeviceToDevice, s);
    return 0;
  }
  if (fmt == LOD_POINTS_F32) return distribute_fmt<LOD_POINTS_F32>(v, p, leaf_out, s);
  return distribute_fmt<LOD_POINTS_F64>(v, p, leaf_out, s);
}

}  // namespace lod
