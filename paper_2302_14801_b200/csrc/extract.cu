// The reference's per-node sampling helpers on arbitrary sample arrays
// (sampling.py:21-133: project_child_samples, extract_first_come / _random / _average /
// _weighted), for callers that drive the stages themselves (the reference's own tests do,
// test_sampling.py).  The build path samples whole levels in voxelize.cu; this is the same
// arithmetic for ONE node's sample list:
//   K_keys    floor(gpos) -> x-major key (sampling.py:50-52), occupancy bitmap (2^21 bits)
//   K_prefix  one CTA: exclusive popcount prefix over the 65536 bitmap words -> voxel ranks
//   K_acc     per sample into its voxel: exact u64 sums (average), max (rand12 | ordinal20)
//             (random), min ordinal (first-come); weighted: 2^-24 fixed-point u64 sums over the
//             occupied cells of the 2x2x2 neighbourhood
//   K_out     per voxel (key by binary search over the word prefixes): coordinates + colour, in
//             ascending key order; first-come: winners ranked by ordinal through an S-bit bitmap
#include "kernels.h"

namespace lod {

namespace {

constexpr uint32_t kXWords = 1u << 16;
constexpr int kXT = 256;

__device__ __forceinline__ uint64_t xmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct XState {
  uint32_t m;       // occupied cells
  uint32_t bad;     // a sample outside the 128^3 grid
  uint32_t zero_w;  // weighted: an occupied cell with no weight
};

__global__ void k_x_keys(const double* __restrict__ g, uint64_t S, uint32_t* __restrict__ keys,
                         uint32_t* __restrict__ bits, XState* st) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S; i += (uint64_t)gridDim.x * blockDim.x) {
    const double x = floor(g[3 * i]), y = floor(g[3 * i + 1]), z = floor(g[3 * i + 2]);
    if (!(x >= 0.0 && x < 128.0 && y >= 0.0 && y < 128.0 && z >= 0.0 && z < 128.0)) {
      st->bad = 1;
      keys[i] = 0;
      continue;
    }
    const uint32_t key = ((uint32_t)x << 14) | ((uint32_t)y << 7) | (uint32_t)z;
    keys[i] = key;
    atomicOr(bits + (key >> 5), 1u << (key & 31));
  }
}

__global__ void __launch_bounds__(1024) k_x_prefix(const uint32_t* __restrict__ bits, uint32_t* __restrict__ pre,
                                                   XState* st) {
  __shared__ uint32_t wsum[1024 / 32 + 1];
  constexpr uint32_t per = kXWords / 1024;
  uint32_t c = 0;
  for (uint32_t q = 0; q < per; ++q) c += __popc(bits[threadIdx.x * per + q]);
  uint32_t tot;
  uint32_t r = block_excl_scan<uint32_t, 1024>(c, &tot, wsum);
  for (uint32_t q = 0; q < per; ++q) {
    pre[threadIdx.x * per + q] = r;
    r += __popc(bits[threadIdx.x * per + q]);
  }
  if (threadIdx.x == 0) st->m = tot;
}

__device__ __forceinline__ uint32_t x_rank(const uint32_t* bits, const uint32_t* pre, uint32_t key) {
  return pre[key >> 5] + __popc(bits[key >> 5] & ((1u << (key & 31)) - 1));
}

__device__ __forceinline__ bool x_occupied(const uint32_t* bits, uint32_t key) {
  return (bits[key >> 5] >> (key & 31)) & 1u;
}

constexpr double kXW = 16777216.0;  // 2^24 fixed point (as voxelize.cu k_scatter_w)

__global__ void k_x_acc(int mode, const double* __restrict__ g, const uint8_t* __restrict__ rgb, uint64_t S,
                        const uint32_t* __restrict__ keys, const uint32_t* __restrict__ bits,
                        const uint32_t* __restrict__ pre, uint64_t hash, unsigned long long* __restrict__ acc) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t key = keys[i];
    if (mode == LOD_MODE_WEIGHTED) {  // sampling.py:108-127
      const double gp[3] = {g[3 * i], g[3 * i + 1], g[3 * i + 2]};
      uint32_t base[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) base[a] = (uint32_t)fmin(fmax(floor(__dsub_rn(gp[a], 0.5)), 0.0), 126.0);
      const double col[3] = {(double)rgb[3 * i], (double)rgb[3 * i + 1], (double)rgb[3 * i + 2]};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t c[3] = {base[0] + (q >> 2), base[1] + ((q >> 1) & 1), base[2] + (q & 1)};
        const uint32_t k = (c[0] << 14) | (c[1] << 7) | c[2];
        if (!x_occupied(bits, k)) continue;
        double s2 = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double d = __dsub_rn(gp[a], __dadd_rn((double)c[a], 0.5));
          s2 = __dadd_rn(s2, __dmul_rn(d, d));
        }
        if (s2 >= 1.0) continue;
        const double w = __dsub_rn(1.0, __dsqrt_rn(s2));
        if (!(w > 0.0)) continue;
        unsigned long long* a = acc + 4ull * x_rank(bits, pre, k);
        atomicAdd(a, (unsigned long long)__double2ll_rn(__dmul_rn(w, kXW)));
#pragma unroll
        for (int ch = 0; ch < 3; ++ch)
          if (col[ch] != 0.0) atomicAdd(a + 1 + ch, (unsigned long long)__double2ll_rn(__dmul_rn(__dmul_rn(w, col[ch]), kXW)));
      }
      continue;
    }
    const uint32_t r = x_rank(bits, pre, key);
    if (mode == LOD_MODE_AVERAGE) {
      unsigned long long* a = acc + 4ull * r;
      atomicAdd(a, (unsigned long long)rgb[3 * i]);
      atomicAdd(a + 1, (unsigned long long)rgb[3 * i + 1]);
      atomicAdd(a + 2, (unsigned long long)rgb[3 * i + 2]);
      atomicAdd(a + 3, 1ull);
    } else if (mode == LOD_MODE_RANDOM) {  // sampling.py:77-80
      const uint32_t enc = ((uint32_t)(xmix64(hash ^ i) >> 32) & 0xFFF00000u) | ((uint32_t)i & 0xFFFFFu);
      atomicMax(reinterpret_cast<unsigned int*>(acc) + r, enc);
    } else {  // first-come: the smallest ordinal (sampling.py:61-66)
      atomicMin(reinterpret_cast<unsigned int*>(acc) + r, (unsigned int)i);
    }
  }
}

// key of voxel rank r: the last word whose prefix <= r, then select-in-word
__device__ __forceinline__ uint32_t x_key_of_rank(const uint32_t* bits, const uint32_t* pre, uint32_t r) {
  uint32_t lo = 0, hi = kXWords - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= r) lo = mid;
    else hi = mid - 1;
  }
  return (lo << 5) + __fns(bits[lo], 0, (int)(r - pre[lo]) + 1);
}

__global__ void k_x_out(int mode, const uint8_t* __restrict__ rgb, const uint32_t* __restrict__ bits,
                        const uint32_t* __restrict__ pre, const unsigned long long* __restrict__ acc, XState* st,
                        uint32_t* __restrict__ win_bits, uint8_t* __restrict__ coords, uint8_t* __restrict__ colors) {
  const uint32_t m = st->m;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
    const uint32_t key = x_key_of_rank(bits, pre, r);
    uint8_t c[3];
    if (mode == LOD_MODE_AVERAGE) {  // (2 sum + n) // (2 n), sampling.py:94-96
      const unsigned long long* a = acc + 4ull * r;
      const unsigned long long n = a[3];
      for (int ch = 0; ch < 3; ++ch) c[ch] = (uint8_t)((2 * a[ch] + n) / (2 * n));
    } else if (mode == LOD_MODE_WEIGHTED) {  // floor(sum(w c) / sum(w) + 0.5), sampling.py:129-133
      const unsigned long long* a = acc + 4ull * r;
      const double W = (double)a[0];
      if (!(W > 0.0)) st->zero_w = 1;
      for (int ch = 0; ch < 3; ++ch)
        c[ch] = (uint8_t)fmin(fmax(floor(__dadd_rn(__ddiv_rn((double)a[1 + ch], W), 0.5)), 0.0), 255.0);
    } else {
      const uint32_t e = reinterpret_cast<const unsigned int*>(acc)[r];
      const uint32_t ord = mode == LOD_MODE_RANDOM ? (e & 0xFFFFFu) : e;
      for (int ch = 0; ch < 3; ++ch) c[ch] = rgb[3ull * ord + ch];
      if (mode == LOD_MODE_FIRST_COME) {  // placed by winner ordinal in k_x_fc
        atomicOr(win_bits + (ord >> 5), 1u << (ord & 31));
        continue;
      }
    }
    coords[3ull * r] = (uint8_t)(key >> 14);
    coords[3ull * r + 1] = (uint8_t)((key >> 7) & 127);
    coords[3ull * r + 2] = (uint8_t)(key & 127);
    for (int ch = 0; ch < 3; ++ch) colors[3ull * r + ch] = c[ch];
  }
}

// first-come: stored order = ascending winner ordinal; position = rank among the winners
__global__ void k_x_fc(const double* __restrict__ g, const uint8_t* __restrict__ rgb, uint64_t S,
                       const uint32_t* __restrict__ win_bits, const uint32_t* __restrict__ win_pre,
                       uint8_t* __restrict__ coords, uint8_t* __restrict__ colors) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t w = win_bits[i >> 5];
    if (!((w >> (i & 31)) & 1)) continue;
    const uint64_t p = win_pre[i >> 5] + __popc(w & ((1u << (i & 31)) - 1));
    for (int a = 0; a < 3; ++a) coords[3 * p + a] = (uint8_t)floor(g[3 * i + a]);
    for (int ch = 0; ch < 3; ++ch) colors[3 * p + ch] = rgb[3 * i + ch];
  }
}

__global__ void k_x_word_prefix(const uint32_t* __restrict__ w, uint64_t nw, uint32_t* __restrict__ pre) {
  // single CTA, sequential chunks (winner bitmaps are S/32 words: small)
  __shared__ uint32_t wsum[1024 / 32 + 1];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t b = 0; b < nw; b += 1024) {
    const uint64_t i = b + threadIdx.x;
    const uint32_t c = i < nw ? __popc(w[i]) : 0u;
    uint32_t tot;
    const uint32_t x = block_excl_scan<uint32_t, 1024>(c, &tot, wsum);
    if (i < nw) pre[i] = carry + x;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

// projection of one child's samples into its parent's 128^3 grid (sampling.py:29-44)
__global__ void k_x_project(int kind, const void* __restrict__ in, uint64_t n, double lx, double ly, double lz,
                            double size, int octant, double* __restrict__ out) {
  const double upper = 0x1.fffffffffffffp+6;  // nextafter(128, 0)
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (kind == 0) {  // leaf points (f64 xyz): clip((p - min) / size * 128, 0, nextafter(128, 0))
      const double* p = static_cast<const double*>(in) + 3 * i;
      const double lo[3] = {lx, ly, lz};
      for (int a = 0; a < 3; ++a)
        out[3 * i + a] = fmin(fmax(__dmul_rn(__ddiv_rn(__dsub_rn(p[a], lo[a]), size), 128.0), 0.0), upper);
    } else {  // child voxels (u8 coords): off + (c + 0.5) / 2
      const uint8_t* c = static_cast<const uint8_t*>(in) + 3 * i;
      for (int a = 0; a < 3; ++a)
        out[3 * i + a] = 64.0 * ((octant >> a) & 1) + ((double)c[a] + 0.5) / 2.0;
    }
  }
}

}  // namespace

int fail(int code, const char* fmt, ...);

}  // namespace lod

using namespace lod;

extern "C" {

int lod_extract(int mode, const double* d_gpos, const uint8_t* d_rgb, uint64_t S, uint64_t seed, uint64_t node_hash,
                uint8_t* d_coords, uint8_t* d_colors, uint64_t* m_out, void* stream) {
  if (mode < LOD_MODE_RANDOM || mode > LOD_MODE_WEIGHTED) return fail(LOD_EVALUE, "unknown sampling strategy: %d", mode);
  if (!m_out || (S && (!d_gpos || !d_rgb || !d_coords || !d_colors))) return fail(LOD_EVALUE, "null argument");
  if (mode == LOD_MODE_RANDOM && S >= (1ull << 20))  // sampling.py:73-75
    return fail(LOD_ECONSISTENCY, "%llu samples exceed the 20-bit index limit of random sampling",
                (unsigned long long)S);
  *m_out = 0;
  if (!S) return LOD_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t acc_words = mode == LOD_MODE_AVERAGE || mode == LOD_MODE_WEIGHTED ? 4 : 1;
  const uint64_t nwin = (S + 31) / 32;
  // workspace: state, bitmap, prefix, keys, accumulators (<= S voxels), winner bitmap + prefix
  const size_t off_bits = 256, off_pre = off_bits + kXWords * 4, off_keys = off_pre + kXWords * 4;
  const size_t off_acc = (off_keys + S * 4 + 255) & ~(size_t)255;
  const size_t off_win = (off_acc + S * acc_words * 8 + 255) & ~(size_t)255;
  const size_t off_wpre = off_win + nwin * 4;
  const size_t bytes = off_wpre + nwin * 4;
  char* w = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&w), bytes, s);
  if (e != cudaSuccess) return fail(LOD_ECUDA, "extract workspace: %s", cudaGetErrorString(e));
  XState* st = reinterpret_cast<XState*>(w);
  uint32_t* bits = reinterpret_cast<uint32_t*>(w + off_bits);
  uint32_t* pre = reinterpret_cast<uint32_t*>(w + off_pre);
  uint32_t* keys = reinterpret_cast<uint32_t*>(w + off_keys);
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(w + off_acc);
  uint32_t* win = reinterpret_cast<uint32_t*>(w + off_win);
  uint32_t* wpre = reinterpret_cast<uint32_t*>(w + off_wpre);
  cudaMemsetAsync(w, 0, off_keys, s);
  cudaMemsetAsync(acc, mode == LOD_MODE_FIRST_COME ? 0xFF : 0, S * acc_words * 8, s);
  cudaMemsetAsync(win, 0, nwin * 4, s);
  const uint32_t grid = (uint32_t)std::min<uint64_t>((S + kXT - 1) / kXT, 148ull * 8);
  k_x_keys<<<grid, kXT, 0, s>>>(d_gpos, S, keys, bits, st);
  k_x_prefix<<<1, 1024, 0, s>>>(bits, pre, st);
  k_x_acc<<<grid, kXT, 0, s>>>(mode, d_gpos, d_rgb, S, keys, bits, pre, seed ^ node_hash, acc);
  k_x_out<<<grid, kXT, 0, s>>>(mode, d_rgb, bits, pre, acc, st, win, d_coords, d_colors);
  if (mode == LOD_MODE_FIRST_COME) {
    k_x_word_prefix<<<1, 1024, 0, s>>>(win, nwin, wpre);
    k_x_fc<<<grid, kXT, 0, s>>>(d_gpos, d_rgb, S, win, wpre, d_coords, d_colors);
  }
  XState h{};
  cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(w, s);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(LOD_ECUDA, "extract: %s", cudaGetErrorString(e));
  if (h.bad) return fail(LOD_EVALUE, "sample positions outside the 128^3 sampling grid");
  if (h.zero_w) return fail(LOD_ECONSISTENCY, "occupied cell accumulated zero weight");  // sampling.py:129-130
  *m_out = h.m;
  return LOD_OK;
}

int lod_project_samples(int kind, const void* d_in, uint64_t n, const double* node_min3, double node_size, int octant,
                        double* d_gpos, void* stream) {
  if ((kind != 0 && kind != 1) || !node_min3 || octant < 0 || octant > 7) return fail(LOD_EVALUE, "bad projection arguments");
  if (!n) return LOD_OK;
  const uint32_t grid = (uint32_t)std::min<uint64_t>((n + kXT - 1) / kXT, 148ull * 8);
  k_x_project<<<grid, kXT, 0, (cudaStream_t)stream>>>(kind, d_in, n, node_min3[0], node_min3[1], node_min3[2],
                                                       node_size, octant, d_gpos);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LOD_ECUDA, "project: %s", cudaGetErrorString(e));
  return LOD_OK;
}

}  // extern "C"
