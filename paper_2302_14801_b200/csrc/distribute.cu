// Insert stage: move every point into its leaf, input order kept within a leaf
// (reference partition.py:244-271; the stable argsort at partition.py:262 is what makes
// within-leaf order = input order, hazard H3).
//
// GPU form: stable LSD radix sort of the point records keyed by leaf id, one-sweep style
// (one pass per digit, <= 11-bit digits, at most 2 passes for <= 2^22 leaves):
//   - the leaf id is computed on the fly in the first pass (main finest-cell target +
//     extension descent), so no key array is ever materialised for single-pass builds;
//   - per tile (8192 points) warps rank their items with __match_any_sync and a
//     per-warp smem histogram, which keeps ranks stable (warp-major, round-major, lane);
//   - tiles find their global per-digit offsets with decoupled look-back over
//     epoch-tagged 64-bit status words (no per-pass clearing);
//   - global digit offsets come from the leaf counts already known from the pyramid,
//     so there is no histogram pass over the points.
// HBM traffic per point, single pass: 16 B read + 16 B written (+ the L2-resident
// target-table read).  Records are re-read for the scatter from L2.
#include "kernels.h"

namespace lod {

namespace {

constexpr int kW = kRadixThreads / 32;
constexpr uint64_t kFlagA = 1ull, kFlagP = 2ull;

__device__ __forceinline__ uint64_t pack_status(uint32_t epoch, uint64_t flag, uint64_t val) {
  return ((uint64_t)(epoch & 0xFFFF) << 48) | (flag << 46) | (val & ((1ull << 46) - 1));
}

__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <int FMT, bool FIRST, bool LAST>
__global__ void __launch_bounds__(kRadixThreads, 2)
    k_radix(SplitView v, const void* in_rec, const uint32_t* in_leaf, void* out_rec, uint32_t* out_leaf,
            int shift, int bits, const uint64_t* digit_base, uint64_t* status, uint32_t epoch,
            uint32_t* ticket) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int B = 1 << bits;
  uint16_t* wh = reinterpret_cast<uint16_t*>(smem);                       // [kW][B] warp histograms
  uint64_t* tbase = reinterpret_cast<uint64_t*>(smem + (size_t)kW * B * 2);  // [B] tile digit bases
  __shared__ uint32_t s_tile;

  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  for (int i = threadIdx.x; i < kW * B / 2; i += kRadixThreads) reinterpret_cast<uint32_t*>(wh)[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t base = (uint64_t)tile * kRadixTile + (uint64_t)warp * 32 * kRadixItems;
  const uint32_t lt_mask = (1u << lane) - 1;

  const double lo0 = v.st->lo[0], lo1 = v.st->lo[1], lo2 = v.st->lo[2];
  const double size = v.st->size, inv = v.st->inv_size;
  bool bad = false, unresolved = false;
  uint32_t leaf[kRadixItems];
  uint16_t rk[kRadixItems];

  // --- 1a. leaf ids.  Straight-line batches (clamped indices, no per-item branches) so
  //     the 16 record loads, then the 16 target-table loads, are all in flight together.
  if (FIRST) {
    uint32_t key[kRadixItems];
#pragma unroll
    for (int k0 = 0; k0 < kRadixItems; k0 += 8) {
      typename Rec<FMT>::Raw r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint64_t i = base + (uint64_t)(k0 + u) * 32 + lane;
        r[u] = Rec<FMT>::load(in_rec, i < v.n ? i : v.n - 1);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        Cell16 c;
        c.x = quant16(Rec<FMT>::x(r[u]), lo0, size, inv, bad);
        c.y = quant16(Rec<FMT>::y(r[u]), lo1, size, inv, bad);
        c.z = quant16(Rec<FMT>::z(r[u]), lo2, size, inv, bad);
        key[k0 + u] = (uint32_t)level_key(c, v.D);
      }
    }
#pragma unroll
    for (int k = 0; k < kRadixItems; ++k) leaf[k] = (uint32_t)__ldg(v.t8 + key[k]);
#pragma unroll
    for (int k = 0; k < kRadixItems; ++k) {
      int32_t t = (int32_t)leaf[k];
      if (t <= -2) {  // inside an extension grid (rare): recompute the cell, descend
        const uint64_t i = base + (uint64_t)k * 32 + lane;
        const auto r = Rec<FMT>::load(in_rec, i < v.n ? i : v.n - 1);
        Cell16 c;
        c.x = quant16(Rec<FMT>::x(r), lo0, size, inv, bad);
        c.y = quant16(Rec<FMT>::y(r), lo1, size, inv, bad);
        c.z = quant16(Rec<FMT>::z(r), lo2, size, inv, bad);
        t = leaf_of_point(v, c);
      }
      if (t < 0) {
        unresolved |= base + (uint64_t)k * 32 + lane < v.n;
        t = 0;
      }
      leaf[k] = (uint32_t)t;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kRadixItems; ++k) {
      const uint64_t i = base + (uint64_t)k * 32 + lane;
      leaf[k] = __ldg(in_leaf + (i < v.n ? i : v.n - 1));
    }
  }
  // --- 1b. stable in-warp ranks (warp-major, round-major, lane order) ---
#pragma unroll
  for (int k = 0; k < kRadixItems; ++k) {
    const bool valid = base + (uint64_t)k * 32 + lane < v.n;
    const uint32_t d = (leaf[k] >> shift) & (B - 1);
    const unsigned act = __ballot_sync(0xFFFFFFFFu, valid);
    uint32_t rank = 0;
    if (valid) {
      const unsigned peers = __match_any_sync(act, d);
      const int leader = 31 - __clz(peers & (0u - peers));  // lowest peer lane
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

  // --- 2. cross-warp prefix per digit, decoupled look-back across tiles ---
  for (int d = threadIdx.x; d < B; d += kRadixThreads) {
    uint32_t run = 0;
#pragma unroll 4
    for (int w = 0; w < kW; ++w) {
      uint32_t c = wh[w * B + d];
      wh[w * B + d] = (uint16_t)run;
      run += c;
    }
    uint64_t* mine = status + (uint64_t)tile * B + d;
    uint64_t excl = 0;
    if (tile == 0) {
      st_relaxed(mine, pack_status(epoch, kFlagP, run));
    } else {
      st_relaxed(mine, pack_status(epoch, kFlagA, run));
      // look back over up to 8 predecessors per trip (independent loads), summing
      // aggregates until an inclusive prefix is found
      int64_t t = (int64_t)tile - 1;
      bool done = false;
      while (!done) {
        uint64_t w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) w[q] = t - q >= 0 ? ld_relaxed(status + (uint64_t)(t - q) * B + d) : 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (done || t - q < 0) break;
          const uint64_t flag = (w[q] >> 46) & 3;
          if ((uint32_t)(w[q] >> 48) != (epoch & 0xFFFF) || flag == 0) {  // not published yet
            t -= q;
            __nanosleep(20);
            goto retry;
          }
          excl += w[q] & ((1ull << 46) - 1);
          if (flag == kFlagP) done = true;
        }
        t -= 8;
      retry:;
      }
      st_relaxed(mine, pack_status(epoch, kFlagP, excl + run));
    }
    tbase[d] = digit_base[d] + excl;
  }
  __syncthreads();

  // --- 3. scatter: records re-read from L2 (the tile was just read), batched so the loads
  //        overlap; destinations of equal-digit runs are adjacent, so L2 merges the sectors ---
#pragma unroll
  for (int k0 = 0; k0 < kRadixItems; k0 += 4) {
    typename Rec<FMT>::Raw r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t i = base + (uint64_t)(k0 + u) * 32 + lane;
      r[u] = Rec<FMT>::load(in_rec, i < v.n ? i : v.n - 1);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + u;
      const uint64_t i = base + (uint64_t)k * 32 + lane;
      if (i < v.n) {
        const uint32_t d = (leaf[k] >> shift) & (B - 1);
        const uint64_t dest = tbase[d] + wh[warp * B + d] + rk[k];
        Rec<FMT>::store(out_rec, dest, r[u]);
        if (!LAST) out_leaf[dest] = leaf[k];
      }
    }
  }
  if (FIRST) {
    if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) raise_err(v.st, ERR_OUTSIDE);
    if (__any_sync(0xFFFFFFFFu, unresolved) && lane == 0) raise_err(v.st, ERR_UNRESOLVED);
  }
}

// Global exclusive prefix per digit, from the leaf counts (leaf ids are the sort keys).
__global__ void k_digit_hist(const uint32_t* leaf_count, uint32_t n_leaves, int shift, int bits,
                             unsigned long long* hist) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_leaves) return;
  atomicAdd(hist + ((j >> shift) & ((1u << bits) - 1)), (unsigned long long)leaf_count[j]);
}

__global__ void __launch_bounds__(1024) k_digit_scan(uint64_t* hist, int B) {
  __shared__ uint64_t sm[1024 / 32 + 1];
  uint64_t a = (2 * threadIdx.x < (unsigned)B) ? hist[2 * threadIdx.x] : 0;
  uint64_t b = (2 * threadIdx.x + 1 < (unsigned)B) ? hist[2 * threadIdx.x + 1] : 0;
  uint64_t tot;
  uint64_t ex = block_excl_scan<uint64_t, 1024>(a + b, &tot, sm);
  if (2 * threadIdx.x < (unsigned)B) hist[2 * threadIdx.x] = ex;
  if (2 * threadIdx.x + 1 < (unsigned)B) hist[2 * threadIdx.x + 1] = ex + a;
}

template <int FMT, bool FIRST, bool LAST>
void run_pass(const SplitView& v, const void* in_rec, const uint32_t* in_leaf, void* out_rec, uint32_t* out_leaf,
              int shift, int bits, const uint64_t* digit_base, RadixPlan& p, uint32_t* ticket, cudaStream_t s) {
  size_t smem = (size_t)kW * (1u << bits) * 2 + (size_t)(1u << bits) * 8;
  auto kern = k_radix<FMT, FIRST, LAST>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<p.tiles, kRadixThreads, smem, s>>>(v, in_rec, in_leaf, out_rec, out_leaf, shift, bits, digit_base,
                                            p.status, p.epoch, ticket);
}

template <int FMT>
int distribute_fmt(const SplitView& v, RadixPlan& p, void* leaf_out, cudaStream_t s) {
  int launches = 0;
  const int B0 = 1 << p.bits[0];
  const int B1 = p.passes > 1 ? 1 << p.bits[1] : 0;
  uint64_t* base0 = p.digit_base;
  uint64_t* base1 = p.digit_base + B0;
  cudaMemsetAsync(p.digit_base, 0, (size_t)(B0 + B1) * 8, s);
  cudaMemsetAsync(p.tile_ticket, 0, 2 * sizeof(uint32_t), s);
  uint32_t lb = ceil_div_u32(v.n_leaves, 256);
  k_digit_hist<<<lb, 256, 0, s>>>(v.leaf_count, v.n_leaves, 0, p.bits[0],
                                  reinterpret_cast<unsigned long long*>(base0));
  k_digit_scan<<<1, 1024, 0, s>>>(base0, B0);
  launches += 2;
  if (p.passes == 1) {
    run_pass<FMT, true, true>(v, v.pts, nullptr, leaf_out, nullptr, 0, p.bits[0], base0, p, p.tile_ticket, s);
    p.epoch++;
    return launches + 1;
  }
  k_digit_hist<<<lb, 256, 0, s>>>(v.leaf_count, v.n_leaves, p.bits[0], p.bits[1],
                                  reinterpret_cast<unsigned long long*>(base1));
  k_digit_scan<<<1, 1024, 0, s>>>(base1, B1);
  run_pass<FMT, true, false>(v, v.pts, nullptr, p.tmp_rec, p.tmp_leaf, 0, p.bits[0], base0, p, p.tile_ticket, s);
  p.epoch++;
  run_pass<FMT, false, true>(v, p.tmp_rec, p.tmp_leaf, leaf_out, nullptr, p.bits[0], p.bits[1], base1, p,
                             p.tile_ticket + 1, s);
  p.epoch++;
  return launches + 4;
}

}  // namespace

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
