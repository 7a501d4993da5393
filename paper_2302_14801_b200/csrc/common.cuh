// Shared device helpers for the LOD-construction path (sm_100a).
//
// Point records (device layout, one per input point):
//   LOD_POINTS_F32: 16 B {f32 x, y, z; u8 r, g, b, pad}   -- the north-star record,
//                   one 128-bit load per point
//   LOD_POINTS_F64: 32 B {f64 x, y, z; u8 r, g, b, pad[5]} -- exact path for clouds whose
//                   coordinates are not float32-representable (reference PointCloud is f64)
//
// Geometry is the reference's fp64 projection (model.py:84-98, partition.py:130-135):
//   q = RN(RN(p - lo) / size);  cell_L = min(floor(q * 2^L), 2^L - 1)
// Because q * 2^L is exact, every level's cell is a right shift of the depth-16 cell
// c16 = min(floor(q * 65536), 65535), so each point is projected once per pass.
#pragma once
#include <cstdint>
#include <map>
#include <mutex>
#include <utility>
#include <cuda_runtime.h>

#include "../../include/lodb200.h"

namespace lod {

constexpr uint32_t UNMERGEABLE = 0xFFFFFFFFu;  // partition.py:20
constexpr int kGrid = 128;                      // model.py:18
constexpr int kMaxDepth = 16;                   // model.py:19
constexpr int kRandomLimit = 1 << 20;           // sampling.py:18

// device error bits (first error wins the detail fields)
enum : uint32_t {
  ERR_NONFINITE = 1u << 0,     // model.py:204-205 -> ValueError
  ERR_OUTSIDE = 1u << 1,       // model.py:94-95 -> ConsistencyError
  ERR_EXT_ROOT = 1u << 2,      // partition.py:169-170
  ERR_OVERSIZED = 1u << 3,     // partition.py:223-224
  ERR_NO_PARENT = 1u << 4,     // partition.py:238-239
  ERR_UNRESOLVED = 1u << 5,    // partition.py:259-260, 285-286
  ERR_RANDOM_LIMIT = 1u << 6,  // sampling.py:73-75
  ERR_ARENA = 1u << 7,         // internal: voxel arena too small, host grows and re-runs
  ERR_EMPTY_CHILD = 1u << 8,   // sampling.py:34-35
  ERR_COUNT = 1u << 9,         // partition.py:268-269
  ERR_NO_ROOT = 1u << 10,      // partition.py:189-191
  ERR_ZERO_WEIGHT = 1u << 11,  // sampling.py:129-130
  ERR_F32_SUMS = 1u << 12,     // internal: an f32 colour sum reached 2^24, re-run with u64 sums
};
// bits only the split raises (lod_build reports them after the voxelizer, api.cu)
constexpr uint32_t kSplitErrors = ERR_NONFINITE | ERR_OUTSIDE | ERR_EXT_ROOT | ERR_OVERSIZED | ERR_NO_PARENT |
                                  ERR_UNRESOLVED | ERR_COUNT | ERR_NO_ROOT;

// Device-resident scalars of one build; read back with a single small D2H copy.
struct DevState {
  unsigned long long lo_key[3];   // order-preserving encodings of per-axis min / max
  unsigned long long hi_key[3];
  double lo[3];                   // world cube (model.py:199-209 or caller bounds)
  double size;
  double inv_size;                // RN(1 / size), fast-path projection
  unsigned long long ext_n;       // entries of the extension-point list (first extension round)
  uint32_t err;
  uint32_t err_detail;            // node id for voxelize errors
  unsigned long long err_value;   // e.g. the sample count of the 2^20 violation
  uint64_t count_a;               // compaction outputs
  uint64_t count_b;
  unsigned long long vox_cursor;  // voxel arena bump pointer
  uint32_t work[kMaxDepth + 1];   // per-depth node tickets for the voxelizer
  uint32_t cand_miss;             // candidate list unusable (too many candidate cells / an anchor missed)
  uint64_t cand_cells;            // candidate cells of the sampled count
  unsigned long long cand_est;    // their sampled points (x kCandStride ~ candidate points)
  unsigned long long cand_n;      // candidate-list slots handed out (K_count, per-warp chunks)
};

__device__ __forceinline__ void raise_err(DevState* st, uint32_t bit, uint32_t detail = 0,
                                          unsigned long long value = 0) {
  uint32_t old = atomicOr(&st->err, bit);
  if (old == 0) {
    st->err_detail = detail;
    st->err_value = value;
  }
}

// Per-CTA cache of hot counters in shared memory.  Counting passes whose points pile into a
// few cells (dense clusters interleaved with other points, so warps see distinct hot keys
// and warp aggregation cannot help) would serialise millions of L2 atomics on a handful of
// addresses.  Each key may live in one of two slots; a slot is claimed once (CAS from EMPTY)
// and counts in shared memory until the periodic flush; keys that find both slots taken go
// to global memory directly.  Resetting every few ten thousand points gives hot keys that
// lost their slots to cold ones another chance.
template <int SLOTS>
struct HotCounts {
  static constexpr uint32_t kEmpty = 0xFFFFFFFFu;
  uint32_t key[SLOTS];
  uint32_t cnt[SLOTS];
  __device__ __forceinline__ void clear() {
    for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) key[i] = kEmpty, cnt[i] = 0;
  }
  __device__ __forceinline__ void add(uint32_t* global, uint32_t k, uint32_t inc) {
    static_assert((SLOTS & (SLOTS - 1)) == 0, "power of two");
    constexpr int B = __builtin_ctz(SLOTS);
    const uint32_t s1 = (k * 0x9E3779B1u) >> (32 - B);
    const uint32_t s2 = (s1 + 1 + ((k * 0x85EBCA77u) >> (33 - B))) & (SLOTS - 1);
    uint32_t s = s1, cur = key[s1];
    if (cur != k) {
      if (cur == kEmpty) {
        cur = atomicCAS(key + s1, kEmpty, k);
        if (cur == kEmpty) cur = k;
      }
      if (cur != k) {
        s = s2;
        cur = key[s2];
        if (cur == kEmpty) {
          cur = atomicCAS(key + s2, kEmpty, k);
          if (cur == kEmpty) cur = k;
        }
      }
    }
    if (cur == k) atomicAdd(cnt + s, inc);
    else atomicAdd(global + k, inc);
  }
  // every thread of the CTA: all adds done -> counts to global, slots emptied
  __device__ __forceinline__ void flush(uint32_t* global) {
    __syncthreads();
    for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) {
      const uint32_t k = key[i], c = cnt[i];
      if (k != kEmpty && c) atomicAdd(global + k, c);
      key[i] = kEmpty;
      cnt[i] = 0;
    }
    __syncthreads();
  }
};

// order-preserving u64 key of a double (for atomicMin / atomicMax)
__device__ __forceinline__ unsigned long long dkey(double d) {
  unsigned long long u = (unsigned long long)__double_as_longlong(d);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dunkey(unsigned long long k) {
  unsigned long long u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)u);
}

// ---------------------------------------------------------------------------
// point records
// ---------------------------------------------------------------------------
template <int FMT>
struct Rec;

template <>
struct Rec<LOD_POINTS_F32> {
  static constexpr int kVec = 1;  // 16-byte words per record
  struct Raw { uint4 a; };
  __device__ __forceinline__ static Raw load(const void* base, uint64_t i) {
    return Raw{__ldg(reinterpret_cast<const uint4*>(base) + i)};
  }
  __device__ __forceinline__ static Raw load_cg(const void* base, uint64_t i) {
    return Raw{__ldcg(reinterpret_cast<const uint4*>(base) + i)};
  }
  // streaming (evict-first): for the last read of a record stream, so the L2 keeps the
  // lookup tables / counting grids / partially written output lines instead
  __device__ __forceinline__ static Raw load_cs(const void* base, uint64_t i) {
    return Raw{__ldcs(reinterpret_cast<const uint4*>(base) + i)};
  }
  __device__ __forceinline__ static void store(void* base, uint64_t i, const Raw& r) {
    reinterpret_cast<uint4*>(base)[i] = r.a;
  }
  __device__ __forceinline__ static float xf(const Raw& r) { return __uint_as_float(r.a.x); }
  __device__ __forceinline__ static float yf(const Raw& r) { return __uint_as_float(r.a.y); }
  __device__ __forceinline__ static float zf(const Raw& r) { return __uint_as_float(r.a.z); }
  __device__ __forceinline__ static double x(const Raw& r) { return (double)__uint_as_float(r.a.x); }
  __device__ __forceinline__ static double y(const Raw& r) { return (double)__uint_as_float(r.a.y); }
  __device__ __forceinline__ static double z(const Raw& r) { return (double)__uint_as_float(r.a.z); }
  __device__ __forceinline__ static uint32_t rgb(const Raw& r) { return r.a.w & 0xFFFFFFu; }
  // the pad byte carries the 2nd-pass distribute digit between the two passes
  static constexpr int kTagBits = 8;
  __device__ __forceinline__ static uint32_t tag(const Raw& r) { return r.a.w >> 24; }
  __device__ __forceinline__ static void set_tag(Raw& r, uint32_t t) { r.a.w = (r.a.w & 0xFFFFFFu) | (t << 24); }
};

template <>
struct Rec<LOD_POINTS_F64> {
  static constexpr int kVec = 2;
  struct Raw { uint4 a, b; };
  __device__ __forceinline__ static Raw load(const void* base, uint64_t i) {
    const uint4* p = reinterpret_cast<const uint4*>(base) + 2 * i;
    return Raw{__ldg(p), __ldg(p + 1)};
  }
  __device__ __forceinline__ static Raw load_cg(const void* base, uint64_t i) {
    const uint4* p = reinterpret_cast<const uint4*>(base) + 2 * i;
    return Raw{__ldcg(p), __ldcg(p + 1)};
  }
  __device__ __forceinline__ static Raw load_cs(const void* base, uint64_t i) {
    const uint4* p = reinterpret_cast<const uint4*>(base) + 2 * i;
    return Raw{__ldcs(p), __ldcs(p + 1)};
  }
  __device__ __forceinline__ static void store(void* base, uint64_t i, const Raw& r) {
    uint4* p = reinterpret_cast<uint4*>(base) + 2 * i;
    p[0] = r.a;
    p[1] = r.b;
  }
  __device__ __forceinline__ static float xf(const Raw& r) { return (float)x(r); }
  __device__ __forceinline__ static float yf(const Raw& r) { return (float)y(r); }
  __device__ __forceinline__ static float zf(const Raw& r) { return (float)z(r); }
  __device__ __forceinline__ static double x(const Raw& r) {
    return __hiloint2double((int)r.a.y, (int)r.a.x);
  }
  __device__ __forceinline__ static double y(const Raw& r) {
    return __hiloint2double((int)r.a.w, (int)r.a.z);
  }
  __device__ __forceinline__ static double z(const Raw& r) {
    return __hiloint2double((int)r.b.y, (int)r.b.x);
  }
  __device__ __forceinline__ static uint32_t rgb(const Raw& r) { return r.b.z & 0xFFFFFFu; }
  static constexpr int kTagBits = 32;
  __device__ __forceinline__ static uint32_t tag(const Raw& r) { return r.b.w; }
  __device__ __forceinline__ static void set_tag(Raw& r, uint32_t t) { r.b.w = t; }
};

// ---------------------------------------------------------------------------
// projection (reference model.py:84-98; hazard H1: correctly rounded fp64)
// ---------------------------------------------------------------------------

// floor(RN(rel / size) * 2^k) exactly.  Fast path multiplies by inv = RN(1/size): the
// product is within 2 ulp of RN(rel/size), i.e. within 2^(k-51) of the exact scaled value,
// so the floor can only differ when the scaled value lies within 2^-30 of an integer; those
// (about 1e-9 of the points) take the correctly rounded division (hazard H1).
template <int K>
__device__ __forceinline__ double exact_scaled_floor(double rel, double size, double inv) {
  constexpr double scale = (double)(1u << K);
  double f = __dmul_rn(__dmul_rn(rel, inv), scale);
  double c = floor(f);
  double fr = __dsub_rn(f, c);
  if (fr < 0x1p-30 || fr > 1.0 - 0x1p-30) c = floor(__dmul_rn(__ddiv_rn(rel, size), scale));
  return c;
}

// One axis of the depth-16 cell; sets *bad if p lies outside [lo, lo + size].
__device__ __forceinline__ uint32_t quant16(double p, double lo, double size, double inv, bool& bad) {
  double rel = __dsub_rn(p, lo);
  bad |= !(rel >= 0.0) || (rel > size);
  double f = exact_scaled_floor<16>(rel, size, inv);
  f = fmin(fmax(f, 0.0), 65535.0);
  return (uint32_t)f;
}

struct Cell16 {
  uint32_t x, y, z;
};

template <int FMT>
__device__ __forceinline__ Cell16 cell16(const typename Rec<FMT>::Raw& r, const DevState& st, bool& bad) {
  Cell16 c;
  c.x = quant16(Rec<FMT>::x(r), st.lo[0], st.size, st.inv_size, bad);
  c.y = quant16(Rec<FMT>::y(r), st.lo[1], st.size, st.inv_size, bad);
  c.z = quant16(Rec<FMT>::z(r), st.lo[2], st.size, st.inv_size, bad);
  return c;
}

// Leaf point -> cell of its parent's 128^3 sampling grid (sampling.py:29-38):
// clip((p - min) / size * 128, 0, nextafter(128, 0)) floored == clamp(floor(.), 0, 127).
// `inv` = RN(1/size) of the parent = RN(1/world_size) * 2^depth exactly.
__device__ __forceinline__ uint32_t grid_cell128(double p, double lo, double size, double inv) {
  double f = exact_scaled_floor<7>(__dsub_rn(p, lo), size, inv);
  return (uint32_t)fmin(fmax(f, 0.0), 127.0);
}

// ---------------------------------------------------------------------------
// fp32 fast path for float32 coordinates (exactness kept by a certificate):
//   v = fl32(fl32(p - lo32) * s32),  lo32 = fl32(lo), s32 = fl32(2^K / size)
// differs from the reference's RN64(RN64(p - lo) / size) * 2^K by at most
//   band = 2^-24 2^K (|lo| / size + 3) (1 + 1e-3) + 1e-12
// (one rounding of lo, p - lo, s and the product; the fp64 roundings are ~2^-52).  When v
// is farther than `band` from every integer and inside (0, 2^K), floor(v) IS the exact cell
// and the point is inside the bounds; otherwise the caller takes the exact fp64 path.  At
// K = 7..8 the band is ~1e-4 cells, so about 1e-4 of the axes fall back.
// ---------------------------------------------------------------------------
struct Frame32 {
  float lo[3];
  float s;       // fl32(2^K / size)
  float band;
};

__host__ __device__ __forceinline__ Frame32 make_frame32(double lx, double ly, double lz, double size, int K) {
  Frame32 f;
  f.lo[0] = (float)lx, f.lo[1] = (float)ly, f.lo[2] = (float)lz;
  const double scale = (double)(1u << K) / size;
  f.s = (float)scale;
  const double m = fmax(fabs(lx), fmax(fabs(ly), fabs(lz)));
  const double band = 0x1p-24 * (double)(1u << K) * (m / size + 3.0) * 1.001 + 1e-12;
  f.band = band < 0.25 && isfinite(scale) && scale < 1e30 ? (float)band : 1.0f;  // 1.0: never certain
  return f;
}

__device__ __forceinline__ bool fast_cell(float p, float lo32, float s32, float band, float lim, uint32_t& cell) {
  const float v = __fmul_rn(__fsub_rn(p, lo32), s32);
  const float f = floorf(v);
  const float fr = v - f;  // exact (Sterbenz)
  if (fr > band && fr < 1.0f - band && f >= 0.0f && f < lim) {
    cell = (uint32_t)f;
    return true;
  }
  return false;
}

// linear x-major key of the cell at `depth` (partition.py:23-24)
__device__ __forceinline__ uint64_t level_key(const Cell16& c, int depth) {
  int s = kMaxDepth - depth;
  return ((uint64_t)(c.x >> s) << (2 * depth)) | ((uint64_t)(c.y >> s) << depth) | (uint64_t)(c.z >> s);
}

// first cell index of pyramid level l inside a pyramid buffer: (8^l - 1) / 7
__host__ __device__ __forceinline__ uint64_t level_off(int l) { return ((1ull << (3 * l)) - 1) / 7; }

// ---------------------------------------------------------------------------
// extension pyramids (partition.py:64-76)
// ---------------------------------------------------------------------------
struct ExtMeta {
  uint64_t pyr_off;      // first slot of this pyramid in the unified pyramid buffer
  uint64_t tgt_off;      // first entry of its finest-level target table
  uint64_t anchor_slot;  // slot of the anchor cell (main finest level or parent ext finest level)
  uint16_t ax, ay, az;   // anchor cell, absolute coordinates at depth `base`
  uint8_t base;          // depth of the anchor cell
  uint8_t ext;           // levels below the anchor (finest grid 2^ext per axis)
};

// Packed node cell: x | y << 16 | z << 32 | depth << 48 | flags << 56
enum : uint32_t { NODE_LEAF = 1u, NODE_OVERSIZED = 2u };
__device__ __forceinline__ uint64_t pack_cell(uint32_t x, uint32_t y, uint32_t z, uint32_t depth,
                                              uint32_t flags) {
  return (uint64_t)x | ((uint64_t)y << 16) | ((uint64_t)z << 32) | ((uint64_t)depth << 48) |
         ((uint64_t)flags << 56);
}

__host__ __device__ __forceinline__ uint32_t ceil_div_u32(uint64_t a, uint64_t b) {
  return (uint32_t)((a + b - 1) / b);
}

// ---------------------------------------------------------------------------
// L2 residency hints for lookup tables read at random while a large array streams past:
// the table (targets, pyramid) is loaded evict-last, the stream (per-point keys)
// evict-first, so the stream does not push the table out of L2.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int32_t ld_hint(const int32_t* a, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_hint(const uint32_t* a, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}

// ---------------------------------------------------------------------------
// Programmatic dependent launch: every kernel is launched with programmatic stream
// serialization and begins with griddepcontrol.wait, so the next grid's launch and block
// scheduling overlap the previous grid's tail while memory ordering stays exactly that of
// plain stream order (the wait returns once the preceding grid has completed and flushed).
// A build is ~75 dependent launches, many of them short.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// More than 48 KB of dynamic shared memory is an opt-in per kernel AND per device: remembered
// per (device, kernel) so a process driving several GPUs sets it on each.
inline void allow_dynamic_smem(const void* kernel, size_t bytes) {
  if (bytes <= 48u * 1024) return;
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  size_t& cur = done[{dev, kernel}];
  if (cur >= bytes) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  cur = bytes;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  allow_dynamic_smem(reinterpret_cast<const void*>(kernel), smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

#define LOD_CUDA_CHECK(expr)                                  \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return ::lod::fail_cuda(_e, #expr); \
  } while (0)

int fail_cuda(cudaError_t e, const char* what);
int fail(int code, const char* fmt, ...);

}  // namespace lod
