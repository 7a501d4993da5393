// Device-wide exclusive scan / order-preserving compaction over a functor domain.
//
// Three launches (block sums -> one-block scan of the sums -> per-block rescan + store).
// Used for the small, structural passes of the split (anchors, node enumeration, leaf
// numbering, leaf offsets); the per-point passes never go through here.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace lod {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xFFFFFFFFu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive prefix and
// writes the block total to *total (all threads).
template <typename T, int NT>
__device__ __forceinline__ T block_excl_scan(T v, T* total, T* smem /* >= NT/32 + 1 */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T incl = warp_incl_scan(v);
  if (lane == 31) smem[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    T w = (lane < NT / 32) ? smem[lane] : T(0);
    T wi = warp_incl_scan(w);
    if (lane < NT / 32) smem[lane] = wi - w;
    if (lane == NT / 32 - 1) smem[NT / 32] = wi;
  }
  __syncthreads();
  T out = smem[warp] + incl - v;
  *total = smem[NT / 32];
  __syncthreads();
  return out;
}

// Scan functors provide value(i), store(i, excl, item) and limit(n): the live length, which
// may be a device-side count below the launch length (blocks past it do no work).
template <class F>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(uint64_t n, F f, uint64_t* block_sums) {
  pdl_wait();
  __shared__ uint64_t sm[kScanThreads / 32 + 1];
  uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  n = f.limit(n);
  if (base >= n) {
    if (threadIdx.x == 0) block_sums[blockIdx.x] = 0;
    return;
  }
  uint64_t s = 0;
#pragma unroll 4
  for (int k = 0; k < kScanItems; ++k) {
    uint64_t i = base + (uint64_t)k * kScanThreads + threadIdx.x;
    if (i < n) s += f.value(i);
  }
  uint64_t tot;
  block_excl_scan<uint64_t, kScanThreads>(s, &tot, sm);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

// Exclusive scan of block sums in one block; adds *base_in (if any) and writes the grand
// total (+ base) to *total_out.
__global__ void __launch_bounds__(1024) k_scan_sums(uint64_t* sums, uint32_t nb, const uint64_t* base_in,
                                                    uint64_t* total_out);

template <class F>
__global__ void __launch_bounds__(kScanThreads) k_scan_store(uint64_t n, F f, const uint64_t* block_sums) {
  pdl_wait();
  // 16 coalesced trips of 256 consecutive items; a block-wide scan per trip keeps the order
  __shared__ uint64_t warp_tot[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t running = block_sums[blockIdx.x];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  n = f.limit(n);
  if (base >= n) return;
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t i = base + (uint64_t)k * kScanThreads + threadIdx.x;
    const uint64_t v = i < n ? f.value(i) : 0;
    const uint64_t incl = warp_incl_scan(v);
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    uint64_t off = running, trip = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) {
      uint64_t t = warp_tot[w];
      off += w < warp ? t : 0;
      trip += t;
    }
    if (i < n) f.store(i, off + incl - v, v);
    running += trip;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Order-preserving compaction of predicate hits (f.pred(i) -> bool, f.emit(i, pos)).
// Warps own contiguous 512-item runs of a 4096-item tile and rank hits with ballots, so
// every load is coalesced and there is one block barrier per tile.
// ---------------------------------------------------------------------------
template <class F>
__global__ void __launch_bounds__(kScanThreads) k_compact_count(uint64_t n, F f, uint64_t* block_sums) {
  pdl_wait();
  __shared__ uint32_t wc[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)warp * 32 * kScanItems;
  uint32_t c = 0;
#pragma unroll 4
  for (int k = 0; k < kScanItems; ++k) {
    uint64_t i = base + (uint64_t)k * 32 + lane;
    c += __popc(__ballot_sync(0xFFFFFFFFu, i < n && f.pred(i)));
  }
  if (lane == 0) wc[warp] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) t += wc[w];
    block_sums[blockIdx.x] = t;
  }
}

template <class F>
__global__ void __launch_bounds__(kScanThreads) k_compact_store(uint64_t n, F f, const uint64_t* block_sums) {
  pdl_wait();
  __shared__ uint32_t wc[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)warp * 32 * kScanItems;
  uint32_t hits[kScanItems];
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    uint64_t i = base + (uint64_t)k * 32 + lane;
    hits[k] = __ballot_sync(0xFFFFFFFFu, i < n && f.pred(i));
    c += __popc(hits[k]);
  }
  if (lane == 0) wc[warp] = c;
  __syncthreads();
  uint64_t pos = block_sums[blockIdx.x];
  for (int w = 0; w < warp; ++w) pos += wc[w];
  const uint32_t lt = (1u << lane) - 1;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (hits[k] >> lane & 1) f.emit(base + (uint64_t)k * 32 + lane, pos + __popc(hits[k] & lt));
    pos += __popc(hits[k]);
  }
}

struct ScanScratch {
  uint64_t* sums = nullptr;
  uint64_t cap = 0;
};

// Runs the scan of f over [0, n). f.value(i) -> u64 item, f.store(i, excl, item).
// base_in (device, may be null) is added to every prefix; *total_out (device) receives
// base + sum.  Returns the number of launches.
template <class F>
int device_scan(uint64_t n, F f, ScanScratch& scr, const uint64_t* base_in, uint64_t* total_out,
                cudaStream_t st) {
  uint32_t nb = (uint32_t)((n + kScanTile - 1) / kScanTile);
  if (nb == 0) nb = 1;
  if (scr.cap < nb + 1) return -1;
  launch_pdl(k_scan_reduce<F>, nb, kScanThreads, 0, st, n, f, scr.sums);
  launch_pdl(k_scan_sums, 1, 1024, 0, st, scr.sums, nb, base_in, total_out);
  launch_pdl(k_scan_store<F>, nb, kScanThreads, 0, st, n, f, scr.sums);
  return 3;
}

// Two halves of device_compact, for callers that read the count on the host in between and
// skip the store when there is nothing to store.
template <class F>
int device_compact_count(uint64_t n, F f, ScanScratch& scr, uint64_t* total_out, cudaStream_t st) {
  uint32_t nb = (uint32_t)((n + kScanTile - 1) / kScanTile);
  if (nb == 0) nb = 1;
  if (scr.cap < nb + 1) return -1;
  launch_pdl(k_compact_count<F>, nb, kScanThreads, 0, st, n, f, scr.sums);
  launch_pdl(k_scan_sums, 1, 1024, 0, st, scr.sums, nb, nullptr, total_out);
  return 2;
}
template <class F>
int device_compact_store(uint64_t n, F f, ScanScratch& scr, cudaStream_t st) {
  uint32_t nb = (uint32_t)((n + kScanTile - 1) / kScanTile);
  if (nb == 0) nb = 1;
  launch_pdl(k_compact_store<F>, nb, kScanThreads, 0, st, n, f, scr.sums);
  return 1;
}

// Compaction of f.pred hits over [0, n); writes the hit count to *total_out (device).
template <class F>
int device_compact(uint64_t n, F f, ScanScratch& scr, uint64_t* total_out, cudaStream_t st) {
  uint32_t nb = (uint32_t)((n + kScanTile - 1) / kScanTile);
  if (nb == 0) nb = 1;
  if (scr.cap < nb + 1) return -1;
  launch_pdl(k_compact_count<F>, nb, kScanThreads, 0, st, n, f, scr.sums);
  launch_pdl(k_scan_sums, 1, 1024, 0, st, scr.sums, nb, nullptr, total_out);
  launch_pdl(k_compact_store<F>, nb, kScanThreads, 0, st, n, f, scr.sums);
  return 3;
}

}  // namespace lod
