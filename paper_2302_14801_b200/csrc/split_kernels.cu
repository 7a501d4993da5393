// Split stage: hierarchical counting sort into octree leaves (reference partition.py).
//
//   K1 k_bounds / k_bounds_finalize   world cube            model.py:199-209
//   K2 k_count                        256^3 counting grid   partition.py:99-105
//   K3 k_ext_create / k_ext_count     extension pyramids    partition.py:109-151
//   K4 k_mark_anchors / k_merge       2x2x2 merge pyramid   partition.py:36-61, 155-170
//   K5 k_build_nodes / k_link / ...   node table + targets  partition.py:174-240
//
// Layout in HBM: every counting pyramid (the main one, then one per extension grid) lives
// in ONE u32 buffer; a pyramid of L levels stores level l at offset (8^l - 1) / 7, x-major
// within a level.  A node is a non-zero cell ("slot") of that buffer, so node enumeration
// is one order-preserving compaction over the buffer.
#include <cooperative_groups.h>

#include "kernels.h"

namespace lod {

constexpr int kThreads = 256;

__device__ __forceinline__ int ceil_log2_u64(uint64_t x) { return x <= 1 ? 0 : 64 - __clzll(x - 1); }

// ---------------------------------------------------------------------------
// K1: bounds
// ---------------------------------------------------------------------------
// float32 records: min / max / finiteness in fp32 (exact; widened once at the end)
__global__ void __launch_bounds__(kThreads) k_bounds_f32(const void* pts, uint64_t n, DevState* st) {
  pdl_wait();
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  uint32_t expmax = 0;  // non-finite <=> exponent field all ones
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  constexpr int U = 4;
  const uint4* p = reinterpret_cast<const uint4*>(pts);
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = __ldcs(p + min(i0 + u * stride, n - 1));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t w[3] = {r[u].x, r[u].y, r[u].z};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const float f = __uint_as_float(w[a]);
        expmax = max(expmax, w[a] & 0x7F800000u);
        lo[a] = fminf(lo[a], f);
        hi[a] = fmaxf(hi[a], f);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fminf(lo[a], __shfl_xor_sync(0xFFFFFFFFu, lo[a], o));
      hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xFFFFFFFFu, hi[a], o));
    }
  }
  __shared__ float s_lo[kThreads / 32][3], s_hi[kThreads / 32][3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int a = 0; a < 3; ++a) s_lo[warp][a] = lo[a], s_hi[warp][a] = hi[a];
  if (__syncthreads_or(expmax == 0x7F800000u) && threadIdx.x == 0) raise_err(st, ERR_NONFINITE);
  if (threadIdx.x < 3) {
    int a = threadIdx.x;
    float l = s_lo[0][a], h = s_hi[0][a];
    for (int w = 1; w < kThreads / 32; ++w) l = fminf(l, s_lo[w][a]), h = fmaxf(h, s_hi[w][a]);
    atomicMin(&st->lo_key[a], dkey((double)l));
    atomicMax(&st->hi_key[a], dkey((double)h));
  }
}

template <int FMT>
__global__ void __launch_bounds__(kThreads) k_bounds(const void* pts, uint64_t n, DevState* st) {
  pdl_wait();
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  bool bad = false;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  constexpr int U = 4;  // independent 16-B loads in flight per thread
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    typename Rec<FMT>::Raw r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = Rec<FMT>::load(pts, min(i0 + u * stride, n - 1));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double p[3] = {Rec<FMT>::x(r[u]), Rec<FMT>::y(r[u]), Rec<FMT>::z(r[u])};
#pragma unroll
      for (int a = 0; a < 3; ++a) {  // clamped duplicates of the last point are harmless
        bad |= !isfinite(p[a]);
        lo[a] = fmin(lo[a], p[a]);
        hi[a] = fmax(hi[a], p[a]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xFFFFFFFFu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xFFFFFFFFu, hi[a], o));
    }
  }
  __shared__ double s_lo[kThreads / 32][3], s_hi[kThreads / 32][3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int a = 0; a < 3; ++a) s_lo[warp][a] = lo[a], s_hi[warp][a] = hi[a];
  if (__syncthreads_or(bad) && threadIdx.x == 0) raise_err(st, ERR_NONFINITE);
  if (threadIdx.x < 3) {
    int a = threadIdx.x;
    double l = s_lo[0][a], h = s_hi[0][a];
    for (int w = 1; w < kThreads / 32; ++w) l = fmin(l, s_lo[w][a]), h = fmax(h, s_hi[w][a]);
    atomicMin(&st->lo_key[a], dkey(l));
    atomicMax(&st->hi_key[a], dkey(h));
  }
}

// size = max_axis(max - min), 1.0 when degenerate (model.py:206-209)
__global__ void k_bounds_finalize(DevState* st, int user, double ux, double uy, double uz, double us) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  if (user) {
    st->lo[0] = ux, st->lo[1] = uy, st->lo[2] = uz, st->size = us;
    st->inv_size = __drcp_rn(us);
    return;
  }
  double ext = 0.0;
  for (int a = 0; a < 3; ++a) {
    double l = dunkey(st->lo_key[a]), h = dunkey(st->hi_key[a]);
    st->lo[a] = l;
    ext = fmax(ext, __dsub_rn(h, l));
  }
  st->size = ext > 0.0 ? ext : 1.0;
  st->inv_size = __drcp_rn(st->size);
}

int launch_bounds(int fmt, const void* pts, uint64_t n, DevState* st, const double* ub, cudaStream_t s) {
  if (ub) {
    launch_pdl(k_bounds_finalize, 1, 32, 0, s, st, 1, ub[0], ub[1], ub[2], ub[3]);
    return 1;
  }
  uint32_t blocks = (uint32_t)std::min<uint64_t>((n + kThreads - 1) / kThreads, 148ull * 8);
  if (fmt == LOD_POINTS_F32)
    launch_pdl(k_bounds_f32, blocks, kThreads, 0, s, pts, n, st);
  else
    launch_pdl(k_bounds<LOD_POINTS_F64>, blocks, kThreads, 0, s, pts, n, st);
  launch_pdl(k_bounds_finalize, 1, 32, 0, s, st, 0, 0, 0, 0, 0);
  return 2;
}

// ---------------------------------------------------------------------------
// K2: count into the main finest grid, warp-aggregated atomics
// ---------------------------------------------------------------------------
constexpr int kCountUnroll = 4;
#ifndef LOD_HOT_SLOTS
#define LOD_HOT_SLOTS 1024
#endif
#ifndef LOD_HOT_RESET
#define LOD_HOT_RESET 64
#endif
constexpr int kHotSlots = LOD_HOT_SLOTS;  // per-CTA hot-counter cache (common.cuh HotCounts)
constexpr int kHotReset = LOD_HOT_RESET;  // loop trips between flushes (64 x 1024 points per CTA)

// A point's main finest-level key: certified fp32 cell first, exact fp64 otherwise (H1).
template <int FMT>
__device__ __forceinline__ uint32_t point_key(const typename Rec<FMT>::Raw& r, const Frame32& fr, float lim,
                                              const DevState& st, int D, bool& bad) {
  uint32_t cx, cy, cz;
  if (FMT == LOD_POINTS_F32 && fast_cell(Rec<FMT>::xf(r), fr.lo[0], fr.s, fr.band, lim, cx) &&
      fast_cell(Rec<FMT>::yf(r), fr.lo[1], fr.s, fr.band, lim, cy) &&
      fast_cell(Rec<FMT>::zf(r), fr.lo[2], fr.s, fr.band, lim, cz))
    return (cx << (2 * D)) | (cy << D) | cz;
  return (uint32_t)level_key(cell16<FMT>(r, st, bad), D);
}

// Candidate cells in shared memory: open addressing over 2 x kCandCap slots.
constexpr uint32_t kCandSlots = 2 * kCandCap;
constexpr int kCandBits = __builtin_ctz(kCandSlots);
static_assert((kCandSlots & (kCandSlots - 1)) == 0, "power-of-two slots");
__device__ __forceinline__ uint32_t cand_slot(uint32_t k) { return (k * 0x9E3779B1u) >> (32 - kCandBits); }
__device__ __forceinline__ bool cand_probe(const uint32_t* h, uint32_t k) {
  uint32_t s = cand_slot(k);
  while (true) {
    const uint32_t c = h[s];
    if (c == k) return true;
    if (c == 0xFFFFFFFFu) return false;
    s = (s + 1) & (kCandSlots - 1);
  }
}

// K_count.  CAND (single-GPU split): points of the candidate cells (sampled count, below) are
// also appended, with their exact depth-16 cells, to the candidate list -- each warp fills
// kCandChunk-slot chunks it reserves with one atomic, unused slots become holes -- so the
// first extension round reads 16 B per candidate instead of gathering records (cluster2B:
// 1 in 10 records, a 128-B line each, 25.6 GB).
// The list pays only when candidates are a minority of the points (clustered clouds): at most
// kCandCap candidate cells, and an estimated (sampled) candidate count <= n / 8 (measured: cluster2B,
// 10 %, gains; scene500M, 21 %, loses -- K_count's extra work outweighs the gathers it saves).
__device__ __forceinline__ bool cand_usable(const DevState& st, uint64_t n) {
  return st.cand_cells > 0 && st.cand_cells <= kCandCap && st.cand_est * (uint64_t)kCandStride <= n / 8;
}

// One warp writes 32 list slots of its chunk (chunks are kCandChunk slots, a multiple of 32):
// lane's candidate `it` {index, key} with its depth-16 cell if `have`, else a hole.
template <int FMT>
__device__ __forceinline__ void cand_emit(const SplitView& v, const DevState& st, const Frame32& f16, uint2 it,
                                          bool have, unsigned long long& wbase, uint32_t& wleft, int lane, bool& bad) {
  if (wleft == 0) {  // uniform
    unsigned long long b = 0;
    if (lane == 0) b = atomicAdd(&v.st->cand_n, (unsigned long long)kCandChunk);
    wbase = __shfl_sync(0xFFFFFFFFu, b, 0);
    wleft = kCandChunk;
  }
  uint4 e = make_uint4(~0u, 0, 0, 0);
  if (have) {
    const auto r = Rec<FMT>::load(v.pts, it.x);
    Cell16 cc;  // certified fp32 first (as K_count's main key), exact fp64 otherwise
    if (!(FMT == LOD_POINTS_F32 && fast_cell(Rec<FMT>::xf(r), f16.lo[0], f16.s, f16.band, 65536.f, cc.x) &&
          fast_cell(Rec<FMT>::yf(r), f16.lo[1], f16.s, f16.band, 65536.f, cc.y) &&
          fast_cell(Rec<FMT>::zf(r), f16.lo[2], f16.s, f16.band, 65536.f, cc.z)))
      cc = cell16<FMT>(r, st, bad);
    e = make_uint4(it.x, it.y, cc.x | (cc.y << 16), cc.z);
  }
  if (wbase + lane < v.cand_cap) v.cand[wbase + lane] = e;
  wbase += 32;
  wleft -= 32;
}

template <int FMT, bool CAND>
__global__ void __launch_bounds__(kThreads, 4) k_count(SplitView v) {
  pdl_wait();
  __shared__ HotCounts<kHotSlots> hot;
  __shared__ uint32_t chash[CAND ? kCandSlots : 1];
  __shared__ Frame32 sf16;
  // per warp: up to 63 pending candidates {index, key}; their depth-16 cells are taken 32 at a
  // time, one per lane (record re-read from L2: this warp loaded it a few trips before), so the
  // projection and the list store run at full warp width -- computing them inline for the ~3
  // candidate lanes of a clustered cloud's warp-iteration was slower (cluster2B count 21.7 ->
  // 25.4 ms)
  __shared__ uint2 cbuf[CAND ? kThreads / 32 : 1][CAND ? 64 : 1];
  hot.clear();
  const DevState st = *v.st;
  const bool cand_on = CAND && cand_usable(st, v.n);  // CTA-uniform
  if (CAND && threadIdx.x == 0) sf16 = make_frame32(st.lo[0], st.lo[1], st.lo[2], st.size, 16);
  if (CAND && cand_on) {
    for (uint32_t i = threadIdx.x; i < kCandSlots; i += blockDim.x) chash[i] = 0xFFFFFFFFu;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < (uint32_t)st.cand_cells; i += blockDim.x) {
      const uint32_t k = __ldg(v.cand_keys + i);
      uint32_t sl = cand_slot(k);
      while (atomicCAS(chash + sl, 0xFFFFFFFFu, k) != 0xFFFFFFFFu) sl = (sl + 1) & (kCandSlots - 1);
    }
  }
  __syncthreads();
  const Frame32 fr = make_frame32(st.lo[0], st.lo[1], st.lo[2], st.size, v.D);
  const float lim = (float)(1u << v.D);
  uint32_t* grid = v.pyr + level_off(v.D);
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  bool bad = false;
  uint32_t trip = 0;
  unsigned long long wbase = 0;  // warp-uniform: next free slot of the warp's chunk, slots left,
  uint32_t wleft = 0;            // finished entries waiting in the warp's buffer
  uint32_t wpend = 0;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < v.n; base += stride * kCountUnroll) {
    if (++trip % kHotReset == 0) hot.flush(grid);
    typename Rec<FMT>::Raw r[kCountUnroll];
#pragma unroll
    for (int u = 0; u < kCountUnroll; ++u) {
      uint64_t i = base + u * stride + threadIdx.x;
      if (i < v.n) r[u] = Rec<FMT>::load(v.pts, i);
    }
#pragma unroll
    for (int u = 0; u < kCountUnroll; ++u) {
      uint64_t i = base + u * stride + threadIdx.x;
      bool valid = i < v.n;
      uint32_t key = 0;
      if (valid) {
        key = point_key<FMT>(r[u], fr, lim, st, v.D, bad);
        v.pkey[i] = key;  // reused by extension counting and the distribute (no re-projection)
      }
      if (CAND && cand_on) {
        const bool c = valid && cand_probe(chash, key);
        const unsigned m = __ballot_sync(0xFFFFFFFFu, c);
        if (m) {
          uint2* wb = cbuf[threadIdx.x >> 5];
          if (c) wb[wpend + __popc(m & lt)] = make_uint2((uint32_t)i, key);
          wpend += __popc(m);
          if (wpend >= 32) {  // uniform: 32 entries to the warp's chunk
            __syncwarp();
            cand_emit<FMT>(v, st, sf16, wb[lane], true, wbase, wleft, lane, bad);
            const uint2 rest = wb[32 + lane];
            __syncwarp();
            wb[lane] = rest;
            __syncwarp();
            wpend -= 32;
          }
        }
      }
      // warp-uniform cell (coherent scans): one aggregated add; otherwise through the
      // CTA's hot-counter cache (interleaved dense clusters), else one RED per point
      // (MATCH would saturate the ADU pipe)
      const uint32_t k0 = __shfl_sync(0xFFFFFFFFu, key, 0);
      const unsigned act = __ballot_sync(0xFFFFFFFFu, valid);
      if (__all_sync(0xFFFFFFFFu, !valid || key == k0)) {
        if (lane == 0 && act) atomicAdd(grid + k0, (uint32_t)__popc(act));
      } else if (valid) {
        hot.add(grid, key, 1u);
      }
    }
  }
  if (CAND && cand_on) {
    if (wpend) {  // uniform: the last < 32 entries, holes after them
      __syncwarp();
      cand_emit<FMT>(v, st, sf16, cbuf[threadIdx.x >> 5][lane], lane < wpend, wbase, wleft, lane, bad);
    }
    for (uint32_t q = lane; q < wleft; q += 32)  // the rest of the last chunk: holes
      if (wbase + q < v.cand_cap) v.cand[wbase + q] = make_uint4(~0u, 0, 0, 0);
  }
  hot.flush(grid);
  if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) raise_err(v.st, ERR_OUTSIDE);
}

uint32_t count_blocks(uint64_t n) { return (uint32_t)std::min<uint64_t>((n + kThreads - 1) / kThreads, 148ull * 8); }

int launch_count(int fmt, const SplitView& v, cudaStream_t s) {
  const uint32_t blocks = count_blocks(v.n);
  if (v.sgrid) {
    if (fmt == LOD_POINTS_F32) launch_pdl(k_count<LOD_POINTS_F32, true>, blocks, kThreads, 0, s, v);
    else launch_pdl(k_count<LOD_POINTS_F64, true>, blocks, kThreads, 0, s, v);
  } else {
    if (fmt == LOD_POINTS_F32) launch_pdl(k_count<LOD_POINTS_F32, false>, blocks, kThreads, 0, s, v);
    else launch_pdl(k_count<LOD_POINTS_F64, false>, blocks, kThreads, 0, s, v);
  }
  return 1;
}

// Candidate cells: every kCandStride-th point counted into sgrid; a cell with >= cand_thresh
// samples (half the samples a cell of T points would get) is a candidate.  Any anchor that is
// not a candidate (adversarial input orders) turns the list off (k_cand_check) and the first
// extension round falls back to the full scan, so the sample only decides speed, never results.
template <int FMT>
__global__ void __launch_bounds__(kThreads) k_cand_sample(SplitView v) {
  pdl_wait();
  __shared__ HotCounts<kHotSlots> hot;  // dense clusters: a few cells take most samples
  hot.clear();
  __syncthreads();
  const DevState st = *v.st;
  const Frame32 fr = make_frame32(st.lo[0], st.lo[1], st.lo[2], st.size, v.D);
  const float lim = (float)(1u << v.D);
  const uint64_t ns = (v.n + kCandStride - 1) / kCandStride;
  bool bad = false;  // points outside the cube are reported by K_count
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ns; j += (uint64_t)gridDim.x * blockDim.x) {
    // one point at a hashed offset inside every block of kCandStride: periodic input orders
    // (e.g. every 10th point in one cell) cannot dodge a fixed stride
    const uint64_t i = j * kCandStride + (((uint32_t)j * 0x9E3779B1u) >> 25);
    if (i >= v.n) continue;
    const auto r = Rec<FMT>::load(v.pts, i);
    const uint32_t key = point_key<FMT>(r, fr, lim, st, v.D, bad);
    if (!bad) hot.add(v.sgrid, key, 1u);
  }
  hot.flush(v.sgrid);
}

struct CandF {
  const uint32_t* sgrid;
  uint32_t thresh;
  uint32_t* out;
  __device__ bool pred(uint64_t i) const { return __ldg(sgrid + i) >= thresh; }
  unsigned long long* est;
  __device__ void emit(uint64_t i, uint64_t pos) const {
    if (pos < kCandCap) out[pos] = (uint32_t)i;
    atomicAdd(est, (unsigned long long)__ldg(sgrid + i));
  }
};

int launch_cand_sample(int fmt, const SplitView& v, ScanScratch& scr, cudaStream_t s) {
  const uint64_t ns = (v.n + kCandStride - 1) / kCandStride;
  const uint32_t blocks = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((ns + kThreads - 1) / kThreads, 148ull * 8));
  if (fmt == LOD_POINTS_F32) launch_pdl(k_cand_sample<LOD_POINTS_F32>, blocks, kThreads, 0, s, v);
  else launch_pdl(k_cand_sample<LOD_POINTS_F64>, blocks, kThreads, 0, s, v);
  const int r = device_compact(1ull << (3 * v.D), CandF{v.sgrid, v.cand_thresh, v.cand_keys, &v.st->cand_est}, scr, &v.st->cand_cells, s);
  return r < 0 ? r : r + 1;
}

__global__ void k_cand_check(SplitView v, const uint64_t* anchors, uint32_t na) {
  pdl_wait();
  const DevState* st = v.st;
  bool miss = false;
  if (blockIdx.x == 0 && threadIdx.x == 0)
    miss = !cand_usable(*st, v.n) || st->cand_n > v.cand_cap;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < na; j += gridDim.x * blockDim.x)
    miss |= __ldg(v.sgrid + anchors[j]) < v.cand_thresh;
  if (miss) atomicOr(&v.st->cand_miss, 1u);
}

int launch_cand_check(const SplitView& v, const uint64_t* anchors, uint32_t na, cudaStream_t s) {
  launch_pdl(k_cand_check, std::max<uint32_t>(1, std::min<uint32_t>(ceil_div_u32(na, kThreads), 148)), kThreads, 0, s,
             v, anchors, na);
  return 1;
}

// ---------------------------------------------------------------------------
// K3: extension pyramids (partition.py:109-151)
// ---------------------------------------------------------------------------
struct AnchorF {  // main finest cells with count > T (partition.py:111)
  const uint32_t* grid;
  uint32_t T;
  uint64_t* out;
  __device__ bool pred(uint64_t i) const { return __ldg(grid + i) > T; }
  __device__ void emit(uint64_t i, uint64_t pos) const { out[pos] = i; }
};

int launch_find_anchors(const SplitView& v, uint64_t* list, ScanScratch& scr, cudaStream_t s, bool store) {
  AnchorF f{v.pyr + level_off(v.D), v.T, list};
  if (!store) return device_compact_count(1ull << (3 * v.D), f, scr, &v.st->count_a, s);
  return device_compact_store(1ull << (3 * v.D), f, scr, s);
}

struct SubAnchorF {  // extension finest cells with count > T (partition.py:140-143)
  const uint32_t* pyr;
  const ExtMeta* meta;
  uint32_t first;
  int ext;
  uint32_t T;
  uint64_t* out;
  __device__ bool pred(uint64_t i) const {
    uint64_t cells = 1ull << (3 * ext);
    const ExtMeta& m = meta[first + i / cells];
    return pyr[m.pyr_off + level_off(ext) + i % cells] > T;
  }
  __device__ void emit(uint64_t i, uint64_t pos) const { out[pos] = i; }
};

int launch_find_subanchors(const SplitView& v, uint32_t first_ext, uint32_t n_ext_round, int ext_levels,
                           uint64_t* list, ScanScratch& scr, cudaStream_t s) {
  SubAnchorF f{v.pyr, v.meta, first_ext, ext_levels, v.T, list};
  return device_compact((uint64_t)n_ext_round << (3 * ext_levels), f, scr, &v.st->count_a, s);
}

__global__ void k_ext_create(SplitView v, int round, uint32_t first, uint32_t count, const uint64_t* list,
                             uint32_t parent_first, uint64_t pyr_base, uint64_t tgt_base, int base_depth,
                             int ext) {
  pdl_wait();
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  uint32_t e = first + i;
  ExtMeta m;
  m.pyr_off = pyr_base + (uint64_t)i * level_off(ext + 1);
  m.tgt_off = tgt_base + ((uint64_t)i << (3 * ext));
  m.base = (uint8_t)base_depth;
  m.ext = (uint8_t)ext;
  uint64_t key = list[i];
  if (round == 0) {  // anchor = main finest cell `key`
    int D = v.D;
    uint32_t msk = (1u << D) - 1;
    m.ax = (uint16_t)(key >> (2 * D));
    m.ay = (uint16_t)((key >> D) & msk);
    m.az = (uint16_t)(key & msk);
    m.anchor_slot = level_off(D) + key;
    v.t8[key] = -(int32_t)(e + 2);
    if (v.abits) atomicOr(v.abits + (key >> 5), 1u << (key & 31));
  } else {  // anchor = finest cell r of parent extension pyramid
    const ExtMeta& p = v.meta[parent_first];
    int pe = p.ext;
    uint64_t cells = 1ull << (3 * pe);
    const ExtMeta mp = v.meta[parent_first + key / cells];
    uint32_t r = (uint32_t)(key % cells), msk = (1u << pe) - 1;
    m.ax = (uint16_t)(((uint32_t)mp.ax << pe) + (r >> (2 * pe)));
    m.ay = (uint16_t)(((uint32_t)mp.ay << pe) + ((r >> pe) & msk));
    m.az = (uint16_t)(((uint32_t)mp.az << pe) + (r & msk));
    m.anchor_slot = mp.pyr_off + level_off(pe) + r;
    v.te[mp.tgt_off + r] = -(int32_t)(e + 2);
  }
  v.meta[e] = m;
}

int launch_ext_create(const SplitView& v, int round, uint32_t first_ext, uint32_t count, const uint64_t* list,
                      uint32_t parent_first, uint64_t pyr_base, uint64_t tgt_base, int base_depth,
                      int ext_levels, cudaStream_t s) {
  if (!count) return 0;
  launch_pdl(k_ext_create, ceil_div_u32(count, kThreads), kThreads, 0, s, v, round, first_ext, count, list, parent_first,
                                                                   pyr_base, tgt_base, base_depth, ext_levels);
  return 1;
}

// Extension rounds (partition.py:109-151).  The first round scans every point's main
// finest key (pkey) against the anchor bitmap; an extension point's record is projected once
// to its depth-16 cell and appended to the extension list {index, round-1 extension id,
// x | y << 16, z} (one global atomic per CTA trip for the list cursor), so later rounds and
// the distribute's leaf resolution read only the list.  Counts go through the CTA's
// hot-counter cache: an anchor cell is by definition dense, and interleaved clusters would
// otherwise serialise millions of atomics on a few extension-grid cells.
__device__ __forceinline__ void ext_count_point(const SplitView& v, HotCounts<kHotSlots>& hot, const Cell16& c,
                                                int32_t t, uint32_t round_first) {
  uint32_t e, rr;
  uint64_t slot;
  if (ext_descend(v, c, e, rr, t, nullptr, &slot) && e >= round_first) {
    if (slot < 0xFFFFFFFFull) hot.add(v.pyr, (uint32_t)slot, 1u);
    else atomicAdd(v.pyr + slot, 1u);
  }
}

__device__ __forceinline__ bool is_anchor(const SplitView& v, uint32_t key) {
  return v.abits ? (__ldg(v.abits + (key >> 5)) >> (key & 31)) & 1 : v.t8[key] <= -2;
}

template <int FMT>
__global__ void __launch_bounds__(kThreads) k_ext_first(SplitView v) {
  pdl_wait();
  if (v.sgrid && !v.st->cand_miss) return;  // k_ext_first_list did the round from the candidate list
  constexpr int U = 8;   // 16 measured slower (registers: 3 CTAs/SM either way, +10% time)
  __shared__ HotCounts<kHotSlots> hot;
  __shared__ uint32_t wsum[kThreads / 32 + 1];
  __shared__ unsigned long long lbase;
  __shared__ uint32_t sidx[kThreads * U], skey[kThreads * U];  // this trip's extension points
  hot.clear();
  __syncthreads();
  const DevState st = *v.st;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  bool bad = false;
  uint32_t since_flush = 0;
  const uint64_t stream = policy_evict_first();
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 - threadIdx.x < v.n; i0 += U * stride) {
    // 1: which of this trip's points are extension points (anchor bitmap, no record read)
    uint32_t key[U];
#pragma unroll
    for (int u = 0; u < U; ++u) key[u] = ld_hint(v.pkey + min(i0 + u * stride, v.n - 1), stream);
    uint32_t flags = 0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < v.n && is_anchor(v, key[u])) flags |= 1u << u;
    uint32_t tot;
    uint32_t x = block_excl_scan<uint32_t, kThreads>((uint32_t)__popc(flags), &tot, wsum);
    if (tot == 0) continue;  // uniform: tot is the CTA's total
#pragma unroll
    for (int u = 0; u < U; ++u)
      if ((flags >> u) & 1) sidx[x] = (uint32_t)(i0 + u * stride), skey[x] = key[u], ++x;
    if (threadIdx.x == 0) lbase = atomicAdd(&v.st->ext_n, (unsigned long long)tot);
    __syncthreads();
    // 2: the trip's extension points, densely over the CTA: project once, list, count
    for (uint32_t j = threadIdx.x; j < tot; j += kThreads) {
      const uint32_t i = sidx[j];
      const Cell16 c = cell16<FMT>(Rec<FMT>::load(v.pts, i), st, bad);
      const int32_t t = v.t8[skey[j]];
      const uint64_t pos = lbase + j;
      if (pos < v.elist_cap) v.elist[pos] = make_uint4(i, (uint32_t)(-(t + 2)), c.x | (c.y << 16), c.z);
      ext_count_point(v, hot, c, t, 0);
    }
    since_flush += tot;
    if (since_flush >= 16384) {  // uniform
      hot.flush(v.pyr);
      since_flush = 0;
    } else {
      __syncthreads();  // sidx / skey / lbase are rewritten by the next trip
    }
  }
  hot.flush(v.pyr);
  if (__any_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) raise_err(v.st, ERR_OUTSIDE);
}

// First extension round from the candidate list (K_count): the candidates inside anchor cells
// are the extension points; their depth-16 cells come with them, so no record is read.
__global__ void __launch_bounds__(kThreads) k_ext_first_list(SplitView v) {
  pdl_wait();
  if (v.st->cand_miss) return;  // k_ext_first scans every point instead
  constexpr int U = 4;
  __shared__ HotCounts<kHotSlots> hot;
  __shared__ uint32_t wsum[kThreads / 32 + 1];
  __shared__ unsigned long long lbase;
  hot.clear();
  __syncthreads();
  const uint64_t n = min((uint64_t)v.st->cand_n, v.cand_cap);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t since_flush = 0;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 - threadIdx.x < n; i0 += U * stride) {
    uint4 q[U];
    int32_t t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) q[u] = __ldcs(v.cand + min(i0 + u * stride, n - 1));
    uint32_t flags = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      t[u] = -1;
      if (i0 + u * stride < n && q[u].x != ~0u && is_anchor(v, q[u].y)) {
        t[u] = v.t8[q[u].y];
        flags |= 1u << u;
      }
    }
    uint32_t tot;
    uint32_t x = block_excl_scan<uint32_t, kThreads>((uint32_t)__popc(flags), &tot, wsum);
    if (tot == 0) continue;  // uniform
    if (threadIdx.x == 0) lbase = atomicAdd(&v.st->ext_n, (unsigned long long)tot);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < U; ++u)
      if ((flags >> u) & 1) {
        const uint64_t pos = lbase + x++;
        if (pos < v.elist_cap) v.elist[pos] = make_uint4(q[u].x, (uint32_t)(-(t[u] + 2)), q[u].z, q[u].w);
        ext_count_point(v, hot, Cell16{q[u].z & 0xFFFF, q[u].z >> 16, q[u].w}, t[u], 0);
      }
    since_flush += tot;
    if (since_flush >= 16384) {  // uniform
      hot.flush(v.pyr);
      since_flush = 0;
    } else {
      __syncthreads();  // lbase is rewritten by the next trip
    }
  }
  hot.flush(v.pyr);
}

__global__ void __launch_bounds__(kThreads) k_ext_more(SplitView v, uint32_t round_first) {
  pdl_wait();
  __shared__ HotCounts<kHotSlots> hot;
  hot.clear();
  __syncthreads();
  const uint64_t n = min((uint64_t)v.st->ext_n, v.elist_cap);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  constexpr int U = 4;
  uint32_t trip = 0;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 - threadIdx.x < n; i0 += U * stride) {
    if (++trip % 16 == 0) hot.flush(v.pyr);
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) q[u] = __ldcs(v.elist + min(i0 + u * stride, n - 1));
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < n)
        ext_count_point(v, hot, Cell16{q[u].z & 0xFFFF, q[u].z >> 16, q[u].w}, -(int32_t)q[u].y - 2, round_first);
  }
  hot.flush(v.pyr);
}

int launch_ext_count(int fmt, const SplitView& v, uint32_t round_first, cudaStream_t s) {
  if (round_first == 0) {
    int r = 1;
    if (v.sgrid) {  // candidate list first; k_ext_first returns at once unless it was unusable
      launch_pdl(k_ext_first_list, 148 * 8, kThreads, 0, s, v);
      ++r;
    }
    uint32_t blocks = (uint32_t)std::min<uint64_t>((v.n + kThreads - 1) / kThreads, 148ull * 8);
    if (fmt == LOD_POINTS_F32) launch_pdl(k_ext_first<LOD_POINTS_F32>, blocks, kThreads, 0, s, v);
    else launch_pdl(k_ext_first<LOD_POINTS_F64>, blocks, kThreads, 0, s, v);
    return r;
  } else {
    launch_pdl(k_ext_more, 148 * 8, kThreads, 0, s, v, round_first);
  }
  return 1;
}

__global__ void k_anchor_sum(SplitView v, const uint64_t* list, uint32_t n) {
  pdl_wait();
  const uint32_t* grid = v.pyr + level_off(v.D);
  unsigned long long s = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s += grid[list[i]];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(&v.st->ext_n, s);
}

int launch_anchor_sum(const SplitView& v, const uint64_t* list, uint32_t n, cudaStream_t s) {
  launch_pdl(k_anchor_sum, std::max<uint32_t>(1, std::min<uint32_t>(ceil_div_u32(n, kThreads), 148)), kThreads, 0,
             s, v, list, n);
  return 1;
}

// leaf of every extension point, descending from its round-1 grid (partition.py:273-287)
__global__ void __launch_bounds__(kThreads) k_ext_leaf(SplitView v, uint32_t* leaf_out) {
  pdl_wait();
  const uint64_t n = min((uint64_t)v.st->ext_n, v.elist_cap);
  bool unresolved = false;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  constexpr int U = 4;  // independent descents in flight per thread (each is a chain of loads)
  for (uint64_t j0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j0 < n; j0 += U * stride) {
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) q[u] = __ldcs(v.elist + min(j0 + u * stride, n - 1));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int32_t t = -(int32_t)q[u].y - 2, nt;
      uint32_t e, rr;
      if (ext_descend(v, Cell16{q[u].z & 0xFFFF, q[u].z >> 16, q[u].w}, e, rr, t, &nt)) t = nt;
      if (t < 0) unresolved = true, t = 0;
      if (j0 + u * stride < n) leaf_out[q[u].x] = (uint32_t)t;
    }
  }
  if (__any_sync(0xFFFFFFFFu, unresolved) && (threadIdx.x & 31) == 0) raise_err(v.st, ERR_UNRESOLVED);
}

int launch_ext_leaf(const SplitView& v, uint32_t* leaf_out, cudaStream_t s) {
  launch_pdl(k_ext_leaf, 148 * 8, kThreads, 0, s, v, leaf_out);
  return 1;
}

// ---------------------------------------------------------------------------
// K4: merge (partition.py:36-61 rule; anchors pre-flagged, partition.py:157-159,165-167)
// ---------------------------------------------------------------------------
__global__ void k_mark_anchors(SplitView v) {
  pdl_wait();
  uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < v.n_ext) v.pyr[v.meta[e].anchor_slot] = UNMERGEABLE;
}

// One parent cell (pyramid p, cell c of level lp): the 2x2x2 merge rule.
__device__ __forceinline__ void merge_cell(uint32_t* pyr, uint64_t first, uint64_t stride, int lp, uint32_t T,
                                         uint64_t p, uint64_t c) {
  const uint32_t dp = 1u << lp, dc = dp << 1, msk = dp - 1;
  uint32_t px = (uint32_t)(c >> (2 * lp)), py = (uint32_t)(c >> lp) & msk, pz = (uint32_t)c & msk;
  uint32_t* base = pyr + first + p * stride;
  uint32_t* ch = base + level_off(lp + 1);
  uint64_t sum = 0;
  bool flag = false;
  uint64_t at[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    uint32_t x = 2 * px + (k & 1), y = 2 * py + ((k >> 1) & 1), z = 2 * pz + (k >> 2);
    at[k] = ((uint64_t)x * dc + y) * dc + z;
    uint32_t val = ch[at[k]];
    if (val == UNMERGEABLE)
      flag = true;
    else
      sum += val;
  }
  uint32_t parent;
  if (!flag && sum > 0 && sum < T) {
    parent = (uint32_t)sum;
#pragma unroll
    for (int k = 0; k < 8; ++k) ch[at[k]] = 0;
  } else {
    parent = (flag || sum > 0) ? UNMERGEABLE : 0u;
  }
  base[level_off(lp) + c] = parent;
}

// One parent level `lp` of `n_pyr` equally shaped pyramids starting at `first`, stride `stride`.
__global__ void __launch_bounds__(kThreads) k_merge(uint32_t* pyr, uint64_t first, uint64_t stride, uint32_t n_pyr,
                                                     int lp, uint32_t T) {
  pdl_wait();
  const uint64_t cells = 1ull << (3 * lp);
  const uint64_t total = cells * n_pyr;
  for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (uint64_t)gridDim.x * blockDim.x)
    merge_cell(pyr, first, stride, lp, T, idx / cells, idx % cells);
}

// The main pyramid's small levels top..0 in one block (barriers between levels): they are
// a few thousand cells, where separate launches cost more than the work.
__global__ void __launch_bounds__(1024) k_merge_small(uint32_t* pyr, int top, uint32_t T) {
  pdl_wait();
  for (int lp = top; lp >= 0; --lp) {
    for (uint64_t c = threadIdx.x; c < (1ull << (3 * lp)); c += blockDim.x) merge_cell(pyr, 0, 0, lp, T, 0, c);
    __syncthreads();
  }
}

// Extension roots must come out UNMERGEABLE (partition.py:169-170); the root slot then
// duplicates the anchor node and is cleared so node enumeration skips it (partition.py:216).
__global__ void k_ext_roots(SplitView v) {
  pdl_wait();
  uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= v.n_ext) return;
  uint64_t s = v.meta[e].pyr_off;
  if (v.pyr[s] != UNMERGEABLE) raise_err(v.st, ERR_EXT_ROOT, e);
  v.pyr[s] = 0;
}

static uint32_t merge_blocks(uint64_t total) {
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((total + kThreads - 1) / kThreads, 148ull * 16));
}

// merge_pyramid on a standalone pyramid (the reference's module function, partition.py:36-61):
// the finest level L at level_off(L) in, levels L-1..0 computed in place
int launch_merge_standalone(uint32_t* pyr, int L, uint32_t T, cudaStream_t s) {
  for (int lp = L - 1; lp >= 0; --lp)
    launch_pdl(k_merge, merge_blocks(1ull << (3 * lp)), kThreads, 0, s, pyr, (uint64_t)0, (uint64_t)0, 1u, lp, T);
  return L;
}

int launch_merge_all(const SplitView& v, const uint32_t* round_first, const uint32_t* round_count,
                     const int* round_ext, const uint64_t* round_pyr_base, int n_rounds, cudaStream_t s) {
  int launches = 0;
  if (v.n_ext) {
    launch_pdl(k_mark_anchors, ceil_div_u32(v.n_ext, kThreads), kThreads, 0, s, v);
    ++launches;
  }
  for (int r = n_rounds - 1; r >= 0; --r) {
    if (!round_count[r]) continue;
    int e = round_ext[r];
    for (int lp = e - 1; lp >= 0; --lp) {
      launch_pdl(k_merge, merge_blocks((uint64_t)round_count[r] << (3 * lp)), kThreads, 0, s,
          v.pyr, round_pyr_base[r], level_off(e + 1), round_count[r], lp, v.T);
      ++launches;
    }
  }
  if (v.n_ext) {
    launch_pdl(k_ext_roots, ceil_div_u32(v.n_ext, kThreads), kThreads, 0, s, v);
    ++launches;
  }
  const int small = std::min(v.D - 1, 4);
  for (int lp = v.D - 1; lp > small; --lp) {
    launch_pdl(k_merge, merge_blocks(1ull << (3 * lp)), kThreads, 0, s, v.pyr, 0, 0, 1, lp, v.T);
    ++launches;
  }
  if (small >= 0) {
    launch_pdl(k_merge_small, 1, 1024, 0, s, v.pyr, small, v.T);
    ++launches;
  }
  return launches;
}

// ---------------------------------------------------------------------------
// K5: node table (partition.py:174-240)
// ---------------------------------------------------------------------------
struct NonZeroF {
  const uint32_t* pyr;
  uint64_t* out;
  __device__ bool pred(uint64_t i) const { return __ldg(pyr + i) != 0; }
  __device__ void emit(uint64_t i, uint64_t pos) const { out[pos] = i; }
};

int launch_count_nodes(const SplitView& v, uint64_t total_slots, uint64_t* slots_out, ScanScratch& scr,
                       cudaStream_t s) {
  NonZeroF f{v.pyr, slots_out};
  return device_compact(total_slots, f, scr, &v.st->count_b, s);
}

struct SlotInfo {
  int32_t ext;      // -1 main
  int lvl;          // level inside its pyramid
  uint32_t rx, ry, rz;  // cell inside that level
};

__device__ __forceinline__ SlotInfo decode_slot(const SplitView& v, uint64_t s) {
  SlotInfo o;
  uint64_t local;
  int top;
  if (s < v.main_cells) {
    o.ext = -1;
    local = s;
    top = v.D;
  } else {  // binary search the extension owning the slot (meta sorted by pyr_off)
    uint32_t lo = 0, hi = v.n_ext;
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) >> 1;
      if (v.meta[mid].pyr_off <= s) lo = mid; else hi = mid;
    }
    o.ext = (int32_t)lo;
    local = s - v.meta[lo].pyr_off;
    top = v.meta[lo].ext;
  }
  int l = top;
  while (l > 0 && level_off(l) > local) --l;
  o.lvl = l;
  uint64_t lin = local - level_off(l);
  uint32_t msk = (1u << l) - 1;
  o.rx = (uint32_t)(lin >> (2 * l));
  o.ry = (uint32_t)(lin >> l) & msk;
  o.rz = (uint32_t)lin & msk;
  return o;
}

__global__ void __launch_bounds__(kThreads) k_build_nodes(SplitView v, const uint64_t* slots) {
  pdl_wait();
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= v.n_nodes) return;
  uint64_t s = slots[k];
  SlotInfo si = decode_slot(v, s);
  uint32_t x = si.rx, y = si.ry, z = si.rz, depth, fine_depth;
  bool finest;
  if (si.ext < 0) {
    depth = si.lvl;
    finest = si.lvl == v.D;
    fine_depth = v.D;
  } else {
    const ExtMeta& m = v.meta[si.ext];
    x += (uint32_t)m.ax << si.lvl;
    y += (uint32_t)m.ay << si.lvl;
    z += (uint32_t)m.az << si.lvl;
    depth = m.base + si.lvl;
    finest = si.lvl == m.ext;
    fine_depth = m.base + m.ext;
  }
  uint32_t val = v.pyr[s];
  uint32_t flags = 0;
  if (val != UNMERGEABLE) {
    flags |= NODE_LEAF;
    if (val > v.T) {  // oversized only at the finest level at max depth (partition.py:222-224)
      flags |= NODE_OVERSIZED;
      if (!(finest && (int)fine_depth >= v.max_depth)) raise_err(v.st, ERR_OVERSIZED, k);
    }
  }
  v.node_idx[s] = (int32_t)k;
  v.n_cell[k] = pack_cell(x, y, z, depth, flags);
  v.n_val[k] = val;
  v.n_slot[k] = s;
  v.n_extid[k] = si.ext;
  v.n_lvl[k] = (uint8_t)si.lvl;
  v.n_parent[k] = -1;
  v.n_count[k] = 0;
  v.n_first[k] = 0;
#pragma unroll
  for (int o = 0; o < 8; ++o) v.n_child[8ull * k + o] = -1;
}

__global__ void __launch_bounds__(kThreads) k_link(SplitView v) {
  pdl_wait();
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= v.n_nodes) return;
  uint64_t cell = v.n_cell[k];
  uint32_t depth = (uint32_t)(cell >> 48) & 0xFF;
  if (depth == 0) {
    if (k != 0) raise_err(v.st, ERR_NO_ROOT, k);
    return;
  }
  int lvl = v.n_lvl[k];
  int32_t e = v.n_extid[k];
  uint64_t s = v.n_slot[k];
  uint64_t ps;
  if (e < 0 || lvl >= 2) {
    uint64_t pyr0 = e < 0 ? 0 : v.meta[e].pyr_off;
    uint64_t lin = s - pyr0 - level_off(lvl);
    uint32_t d = 1u << lvl, msk = d - 1;
    uint32_t rx = (uint32_t)(lin >> (2 * lvl)) >> 1, ry = ((uint32_t)(lin >> lvl) & msk) >> 1,
             rz = ((uint32_t)lin & msk) >> 1;
    uint32_t dp = d >> 1;
    ps = pyr0 + level_off(lvl - 1) + ((uint64_t)rx * dp + ry) * dp + rz;
  } else {
    ps = v.meta[e].anchor_slot;  // extension level 1 hangs off its anchor cell
  }
  if (v.pyr[ps] != UNMERGEABLE) {
    raise_err(v.st, ERR_NO_PARENT, k);
    return;
  }
  int32_t p = v.node_idx[ps];
  uint32_t oct = ((uint32_t)cell & 1) | (((uint32_t)(cell >> 16) & 1) << 1) | (((uint32_t)(cell >> 32) & 1) << 2);
  v.n_parent[k] = p;
  v.n_child[8ull * p + oct] = (int32_t)k;
}

// bounds_at(world, path): sequential child_bounds fold (model.py:62-81, hazard H2)
__global__ void __launch_bounds__(kThreads) k_node_bounds(SplitView v) {
  pdl_wait();
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= v.n_nodes) return;
  uint64_t cell = v.n_cell[k];
  uint32_t cx = (uint32_t)cell & 0xFFFF, cy = (uint32_t)(cell >> 16) & 0xFFFF, cz = (uint32_t)(cell >> 32) & 0xFFFF;
  int depth = (int)(cell >> 48) & 0xFF;
  double x = v.st->lo[0], y = v.st->lo[1], z = v.st->lo[2], size = v.st->size;
  for (int b = depth - 1; b >= 0; --b) {
    double h = __ddiv_rn(size, 2.0);
    x = __dadd_rn(x, __dmul_rn(h, (double)((cx >> b) & 1)));
    y = __dadd_rn(y, __dmul_rn(h, (double)((cy >> b) & 1)));
    z = __dadd_rn(z, __dmul_rn(h, (double)((cz >> b) & 1)));
    size = h;
  }
  v.n_box[k] = make_double4(x, y, z, size);
}

int launch_build_nodes(const SplitView& v, const uint64_t* slots, cudaStream_t s) {
  uint32_t b = ceil_div_u32(v.n_nodes, kThreads);
  launch_pdl(k_build_nodes, b, kThreads, 0, s, v, slots);
  launch_pdl(k_link, b, kThreads, 0, s, v);
  launch_pdl(k_node_bounds, b, kThreads, 0, s, v);
  return 3;
}

struct LeafNumF {
  const uint32_t* val;
  int32_t* n_leaf;
  uint32_t* leaf_node;
  __device__ uint64_t limit(uint64_t n) const { return n; }
  __device__ uint64_t value(uint64_t k) const { return val[k] != UNMERGEABLE ? 1 : 0; }
  __device__ void store(uint64_t k, uint64_t ex, uint64_t v) const {
    n_leaf[k] = v ? (int32_t)ex : -1;
    if (v) leaf_node[ex] = (uint32_t)k;
  }
};

int launch_number_leaves(const SplitView& v, ScanScratch& scr, cudaStream_t s) {
  LeafNumF f{v.n_val, v.n_leaf, v.leaf_node};
  return device_scan(v.n_nodes, f, scr, nullptr, &v.st->count_a, s);
}

// Leaf allocation = exclusive prefix of leaf counts (partition.py:264-265 searchsorted bounds)
struct LeafOffF {
  const uint32_t* val;       // per node (pyramid counts) or null
  const uint32_t* cnt;       // per leaf counts when val is null
  const uint32_t* leaf_node;
  uint64_t* leaf_first;
  uint32_t* leaf_count;
  uint64_t* n_first;
  uint32_t* n_count;
  __device__ uint64_t limit(uint64_t n) const { return n; }
  __device__ uint64_t value(uint64_t j) const { return val ? val[leaf_node[j]] : cnt[j]; }
  __device__ void store(uint64_t j, uint64_t ex, uint64_t v) const {
    uint32_t k = leaf_node[j];
    leaf_first[j] = ex;
    leaf_count[j] = (uint32_t)v;
    n_first[k] = ex;
    n_count[k] = (uint32_t)v;
  }
};

// Per leaf, the bounds of its parent (the node whose 128^3 grid its points are sampled
// into, sampling.py:29-38) and RN(1/size) = RN(1/world_size) * 2^depth (exact scaling).
__global__ void k_leaf_parent_boxes(SplitView v) {
  pdl_wait();
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= v.n_leaves) return;
  int32_t par = v.n_parent[v.leaf_node[j]];
  if (par < 0) {
    v.leaf_pbox[j] = make_double4(0, 0, 0, -1.0);
    v.leaf_pinv[j] = 0;
    return;
  }
  int depth = (int)(v.n_cell[par] >> 48) & 0xFF;
  v.leaf_pbox[j] = v.n_box[par];
  v.leaf_pinv[j] = __dmul_rn(v.st->inv_size, (double)(1ull << depth));
}

int launch_leaf_parent_boxes(const SplitView& v, cudaStream_t s) {
  launch_pdl(k_leaf_parent_boxes, ceil_div_u32(v.n_leaves, kThreads), kThreads, 0, s, v);
  return 1;
}

int launch_leaf_offsets(const SplitView& v, ScanScratch& scr, cudaStream_t s) {
  LeafOffF f{v.n_val, nullptr, v.leaf_node, v.leaf_first, v.leaf_count, v.n_first, v.n_count};
  return device_scan(v.n_leaves, f, scr, nullptr, &v.st->count_b, s);
}

// multi-GPU: leaf offsets from this process's per-leaf counts (already in leaf_count)
int launch_leaf_offsets_local(const SplitView& v, ScanScratch& scr, cudaStream_t s) {
  LeafOffF f{nullptr, v.leaf_count, v.leaf_node, v.leaf_first, v.leaf_count, v.n_first, v.n_count};
  return device_scan(v.n_leaves, f, scr, nullptr, &v.st->count_b, s);
}

// Per cell: the leaf that owns it after merging (partition.py:250-258 "iterate upwards"),
// computed top-down one level at a time: a plain non-zero cell is its own leaf, an
// UNMERGEABLE cell owns nothing, an empty cell inherits its parent's owner.  The result is
// written in place over node_idx (level l reads level l-1's finished targets); the finest
// level goes to t8, where extension anchors keep their -(ext+2) pointer.
// ptarget: the parent cell's target when the caller already has it (k_target_level), else
// INT32_MIN and it is loaded here
__device__ __forceinline__ void target_cell(const SplitView& v, int l, uint64_t c, uint32_t val,
                                            int32_t ptarget = INT32_MIN) {
  const uint64_t s = level_off(l) + c;
  int32_t t;
  if (val == UNMERGEABLE) {
    t = -1;
  } else if (val != 0) {
    t = v.n_leaf[v.node_idx[s]];
  } else if (l == 0) {
    t = -1;
  } else if (ptarget != INT32_MIN) {
    t = ptarget;
  } else {
    const uint32_t msk = (1u << l) - 1;
    uint32_t x = (uint32_t)(c >> (2 * l)) >> 1, y = ((uint32_t)(c >> l) & msk) >> 1, z = ((uint32_t)c & msk) >> 1;
    uint32_t dp = 1u << (l - 1);
    t = v.node_idx[level_off(l - 1) + ((uint64_t)x * dp + y) * dp + z];
  }
  if (l == v.D) {
    // anchors keep -(ext+2); t8 was cleared to -1, so cells without an owning leaf
    // (most of the grid for surfaces) need no write
    if (val != UNMERGEABLE && t != -1) v.t8[c] = t;
  } else {
    v.node_idx[s] = t;
  }
}

// levels 0..top in one block (small levels, block barriers between them)
__global__ void __launch_bounds__(1024) k_target_small(SplitView v, int top) {
  pdl_wait();
  for (int l = 0; l <= top; ++l) {
    for (uint64_t c = threadIdx.x; c < (1ull << (3 * l)); c += blockDim.x) target_cell(v, l, c, v.pyr[level_off(l) + c]);
    __syncthreads();
  }
}

// four consecutive cells per thread per trip (l >= 2: same x, y; z0 % 4 == 0): their pyramid
// values and the targets of their two parent cells are loaded together, so an empty /
// merged cell's target costs no dependent load (one cell per thread left this pass
// latency-bound)
__global__ void __launch_bounds__(kThreads) k_target_level(SplitView v, int l) {
  pdl_wait();
  const uint64_t cells = 1ull << (3 * l);
  const uint32_t msk = (1u << l) - 1, dp = 1u << (l - 1);
  for (uint64_t c0 = 4 * ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x); c0 < cells;
       c0 += 4ull * gridDim.x * blockDim.x) {
    uint32_t val[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) val[u] = v.pyr[level_off(l) + c0 + u];
    const uint32_t x = (uint32_t)(c0 >> (2 * l)) >> 1, y = ((uint32_t)(c0 >> l) & msk) >> 1, z = ((uint32_t)c0 & msk) >> 1;
    const uint64_t ps = level_off(l - 1) + ((uint64_t)x * dp + y) * dp + z;
    const int32_t par[2] = {v.node_idx[ps], v.node_idx[ps + 1]};
#pragma unroll
    for (int u = 0; u < 4; ++u) target_cell(v, l, c0 + u, val[u], par[u >> 1]);
  }
}

__global__ void __launch_bounds__(kThreads) k_target_ext(SplitView v, uint32_t first, uint32_t count, int ext) {
  pdl_wait();
  const uint64_t cells = 1ull << (3 * ext);
  const uint64_t total = cells * count;
  const uint32_t msk = (1u << ext) - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const ExtMeta& m = v.meta[first + i / cells];
    uint64_t r = i % cells;
    int32_t* tp = v.te + m.tgt_off + r;
    if (*tp <= -2) continue;
    uint32_t x = (uint32_t)(r >> (2 * ext)), y = (uint32_t)(r >> ext) & msk, z = (uint32_t)r & msk;
    int32_t t = -1;
    for (int l = ext; l >= 1; --l) {
      int sh = ext - l;
      uint64_t s = m.pyr_off + level_off(l) +
                   (((uint64_t)(x >> sh) << (2 * l)) | ((uint64_t)(y >> sh) << l) | (z >> sh));
      uint32_t val = v.pyr[s];
      if (val == 0) continue;
      if (val != UNMERGEABLE) t = v.n_leaf[v.node_idx[s]];
      break;
    }
    *tp = t;
  }
}

int launch_targets(const SplitView& v, cudaStream_t s) {
  const int small = std::min(v.D, 3);  // one block for levels 0..3 (a block for 0..5 took 46 us)
  launch_pdl(k_target_small, 1, 1024, 0, s, v, small);
  int launches = 1;
  for (int l = small + 1; l <= v.D; ++l, ++launches)
    launch_pdl(k_target_level, merge_blocks(1ull << (3 * l - 2)), kThreads, 0, s, v, l);
  return launches;
}

int launch_targets_ext(const SplitView& v, uint32_t first, uint32_t count, int ext, cudaStream_t s) {
  if (!count) return 0;
  launch_pdl(k_target_ext, merge_blocks((uint64_t)count << (3 * ext)), kThreads, 0, s, v, first, count, ext);
  return 1;
}

__global__ void k_depth_hist(SplitView v, uint32_t* depth_count) {
  pdl_wait();
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= v.n_nodes) return;
  uint64_t cell = v.n_cell[k];
  uint32_t depth = (uint32_t)(cell >> 48) & 0xFF;
  if (v.n_val[k] == UNMERGEABLE) atomicAdd(depth_count + depth, 1u);
  atomicMax(depth_count + kMaxDepth + 1, depth);
}

int launch_depth_lists(const SplitView& v, uint32_t* depth_count, cudaStream_t s) {
  launch_pdl(k_depth_hist, ceil_div_u32(v.n_nodes, kThreads), kThreads, 0, s, v, depth_count);
  return 1;
}

__global__ void k_depth_scatter(SplitView v, const uint32_t* depth_off, uint32_t* cursor, uint32_t* lists) {
  pdl_wait();
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= v.n_nodes || v.n_val[k] != UNMERGEABLE) return;
  uint32_t depth = (uint32_t)(v.n_cell[k] >> 48) & 0xFF;
  lists[depth_off[depth] + atomicAdd(cursor + depth, 1u)] = k;
}

int launch_depth_scatter(const SplitView& v, const uint32_t* depth_off, uint32_t* depth_cursor, uint32_t* lists,
                         cudaStream_t s) {
  launch_pdl(k_depth_scatter, ceil_div_u32(v.n_nodes, kThreads), kThreads, 0, s, v, depth_off, depth_cursor, lists);
  return 1;
}

__global__ void k_export_nodes(SplitView v, lod_node* out) {
  pdl_wait();
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= v.n_nodes) return;
  lod_node o;
  double4 b = v.n_box[k];
  o.min[0] = b.x, o.min[1] = b.y, o.min[2] = b.z, o.size = b.w;
  o.first = v.n_first[k];
  o.count = v.n_count[k];
  o.parent = v.n_parent[k];
  uint64_t c = v.n_cell[k];
  o.cell[0] = (uint16_t)c, o.cell[1] = (uint16_t)(c >> 16), o.cell[2] = (uint16_t)(c >> 32);
  o.depth = (uint8_t)(c >> 48);
  o.flags = (uint8_t)(c >> 56);
  for (int i = 0; i < 8; ++i) o.child[i] = v.n_child[8ull * k + i];
  out[k] = o;
}

int launch_export_nodes(const SplitView& v, lod_node* out, cudaStream_t s) {
  launch_pdl(k_export_nodes, ceil_div_u32(v.n_nodes, kThreads), kThreads, 0, s, v, out);
  return 1;
}

}  // namespace lod
