// Ingest decoders (reference ingest.py:59-198) and structural checks (checks.py:18-92)
// on the device.
//
// Ingest: the raw record bytes of an LAS / binary-PLY file are streamed to HBM as-is (the
// host only parses the header); one thread per record decodes them into point records:
//   LAS  x = RN(RN(X * scale) + offset) per axis (ingest.py:104-105, no FMA), rgb = the
//        16-bit channel >> 8, or grey 128 without colour (ingest.py:106-111)
//   PLY  any scalar property widened to f64 (exact), colours cast to u8 (ingest.py:190-197)
// Checks: one CTA per node (grid-strided); per-node failure bits, reduced on the host into
// the reference's CheckResult list.
#include "kernels.h"

namespace lod {

namespace {

template <class T>
__device__ __forceinline__ T ld_unaligned(const uint8_t* p) {
  T v;
  memcpy(&v, p, sizeof(T));
  return v;
}

__global__ void k_ingest_las(const uint8_t* raw, uint64_t n, uint32_t reclen, int32_t rgb_off, double sx, double sy,
                             double sz, double ox, double oy, double oz, uint4* out) {
  pdl_wait();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t* r = raw + i * reclen;
    const double x = __dadd_rn(__dmul_rn((double)ld_unaligned<int32_t>(r), sx), ox);
    const double y = __dadd_rn(__dmul_rn((double)ld_unaligned<int32_t>(r + 4), sy), oy);
    const double z = __dadd_rn(__dmul_rn((double)ld_unaligned<int32_t>(r + 8), sz), oz);
    uint32_t rgb = 0x808080u;
    if (rgb_off >= 0) {
      const uint8_t* c = r + rgb_off;
      rgb = (uint32_t)(ld_unaligned<uint16_t>(c) >> 8) | ((uint32_t)(ld_unaligned<uint16_t>(c + 2) >> 8) << 8) |
            ((uint32_t)(ld_unaligned<uint16_t>(c + 4) >> 8) << 16);
    }
    const unsigned long long bx = __double_as_longlong(x), by = __double_as_longlong(y),
                             bz = __double_as_longlong(z);
    out[2 * i] = make_uint4((uint32_t)bx, (uint32_t)(bx >> 32), (uint32_t)by, (uint32_t)(by >> 32));
    out[2 * i + 1] = make_uint4((uint32_t)bz, (uint32_t)(bz >> 32), rgb, 0);
  }
}

// PLY scalar types (include/lodb200.h lod_ply_type)
__device__ __forceinline__ double ply_value(const uint8_t* p, int t) {
  switch (t) {
    case LOD_PLY_I8: return (double)(int8_t)p[0];
    case LOD_PLY_U8: return (double)p[0];
    case LOD_PLY_I16: return (double)ld_unaligned<int16_t>(p);
    case LOD_PLY_U16: return (double)ld_unaligned<uint16_t>(p);
    case LOD_PLY_I32: return (double)ld_unaligned<int32_t>(p);
    case LOD_PLY_U32: return (double)ld_unaligned<uint32_t>(p);
    case LOD_PLY_F32: return (double)ld_unaligned<float>(p);
    default: return ld_unaligned<double>(p);
  }
}

// numpy astype(uint8): integers wrap modulo 256, floats truncate toward zero first
__device__ __forceinline__ uint32_t ply_u8(const uint8_t* p, int t) {
  switch (t) {
    case LOD_PLY_F32: return (uint32_t)(long long)truncf(ld_unaligned<float>(p)) & 0xFF;
    case LOD_PLY_F64: return (uint32_t)(long long)trunc(ld_unaligned<double>(p)) & 0xFF;
    case LOD_PLY_U32: case LOD_PLY_I32: return ld_unaligned<uint32_t>(p) & 0xFF;
    case LOD_PLY_U16: case LOD_PLY_I16: return ld_unaligned<uint16_t>(p) & 0xFF;
    default: return p[0];
  }
}

struct PlyLayout {
  int32_t type[6];
  uint32_t off[6];
};

__global__ void k_ingest_ply(const uint8_t* raw, uint64_t n, uint32_t stride, PlyLayout L, int has_rgb, int fmt,
                             uint4* out) {
  pdl_wait();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t* r = raw + i * stride;
    uint32_t rgb = 0x808080u;
    if (has_rgb) rgb = ply_u8(r + L.off[3], L.type[3]) | (ply_u8(r + L.off[4], L.type[4]) << 8) |
                       (ply_u8(r + L.off[5], L.type[5]) << 16);
    const double x = ply_value(r + L.off[0], L.type[0]), y = ply_value(r + L.off[1], L.type[1]),
                 z = ply_value(r + L.off[2], L.type[2]);
    if (fmt == LOD_POINTS_F32) {
      out[i] = make_uint4(__float_as_uint((float)x), __float_as_uint((float)y), __float_as_uint((float)z), rgb);
    } else {
      const unsigned long long bx = __double_as_longlong(x), by = __double_as_longlong(y),
                               bz = __double_as_longlong(z);
      out[2 * i] = make_uint4((uint32_t)bx, (uint32_t)(bx >> 32), (uint32_t)by, (uint32_t)(by >> 32));
      out[2 * i + 1] = make_uint4((uint32_t)bz, (uint32_t)(bz >> 32), rgb, 0);
    }
  }
}

// ---------------------------------------------------------------------------
// checks.py:18-92, one CTA per node
// ---------------------------------------------------------------------------
template <int FMT>
__global__ void __launch_bounds__(256) k_checks(SplitView v, const void* leaf_pts, const uint2* vox, int voxels,
                                                uint32_t T, int max_depth, uint8_t* flags) {
  pdl_wait();
  __shared__ int s_bad;
  for (uint32_t k = blockIdx.x; k < v.n_nodes; k += gridDim.x) {
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    const uint64_t cell = v.n_cell[k];
    const int depth = (int)(cell >> 48) & 0xFF;
    const bool leaf = v.n_leaf[k] >= 0;
    const uint64_t first = v.n_first[k];
    const uint32_t count = v.n_count[k];
    uint32_t f = 0;
    if (leaf) {
      const bool over = (cell >> 56) & NODE_OVERSIZED;
      if (!over && count > T) f |= LOD_CHECK_CAPACITY;
      if (over && depth != max_depth) f |= LOD_CHECK_OVERSIZED;
      if (count == 0) f |= LOD_CHECK_CONTAINMENT;
      const double4 b = v.n_box[k];
      const double tol = __dmul_rn(b.w, 1e-6);  // checks.py:61
      bool bad = false;
      for (uint32_t j = threadIdx.x; j < count; j += blockDim.x) {
        const auto r = Rec<FMT>::load(leaf_pts, first + j);
        const double rel[3] = {__dsub_rn(Rec<FMT>::x(r), b.x), __dsub_rn(Rec<FMT>::y(r), b.y),
                               __dsub_rn(Rec<FMT>::z(r), b.z)};
#pragma unroll
        for (int a = 0; a < 3; ++a) bad |= rel[a] < -tol || rel[a] > __dadd_rn(b.w, tol);
      }
      if (bad) s_bad = 1;
    } else {
      uint32_t leaf_kids = 0, kids = 0;
      uint64_t kid_points = 0;
      for (int o = 0; o < 8; ++o) {
        const int32_t c = v.n_child[8ull * k + o];
        if (c < 0) continue;
        ++kids;
        if (v.n_leaf[c] >= 0) ++leaf_kids, kid_points += v.n_count[c];
      }
      if (!kids) f |= LOD_CHECK_NO_CHILDREN;
      if (kids && leaf_kids == kids && kid_points < T) f |= LOD_CHECK_MAXIMALITY;
      if (!voxels || count == 0) f |= LOD_CHECK_EMPTY_INNER;
      if (voxels) {
        bool dup = false, range = false;  // the key-ordered arena: unique <=> strictly ascending
        for (uint32_t j = threadIdx.x; j < count; j += blockDim.x) {
          const uint32_t key = vox[first + j].x;
          range |= key >= (1u << 21);
          if (j) dup |= vox[first + j - 1].x >= key;
        }
        if (dup) atomicOr(&s_bad, 2);
        if (range) atomicOr(&s_bad, 4);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (leaf && s_bad) f |= LOD_CHECK_CONTAINMENT;
      if (!leaf && (s_bad & 2)) f |= LOD_CHECK_UNIQUENESS;
      if (!leaf && (s_bad & 4)) f |= LOD_CHECK_VOXEL_BOUNDS;
      flags[k] = (uint8_t)f;
    }
    __syncthreads();
  }
}

}  // namespace

int launch_ingest_las(const void* raw, uint64_t n, uint32_t reclen, int32_t rgb_off, const double* sc,
                      const double* of, void* out, cudaStream_t s) {
  if (!n) return 0;
  const uint32_t grid = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
  launch_pdl(k_ingest_las, grid, 256, 0, s, reinterpret_cast<const uint8_t*>(raw), n, reclen, rgb_off, sc[0], sc[1], sc[2],
                                    of[0], of[1], of[2], reinterpret_cast<uint4*>(out));
  return 1;
}

int launch_ingest_ply(const void* raw, uint64_t n, uint32_t stride, const int32_t* types, const uint32_t* offs,
                      int has_rgb, int fmt, void* out, cudaStream_t s) {
  if (!n) return 0;
  PlyLayout L;
  for (int i = 0; i < 6; ++i) L.type[i] = types[i], L.off[i] = offs[i];
  const uint32_t grid = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
  launch_pdl(k_ingest_ply, grid, 256, 0, s, reinterpret_cast<const uint8_t*>(raw), n, stride, L, has_rgb, fmt,
                                    reinterpret_cast<uint4*>(out));
  return 1;
}

int launch_checks(int fmt, const SplitView& v, const void* leaf_pts, const uint2* vox, int voxels, uint32_t T,
                  int max_depth, uint8_t* flags, cudaStream_t s) {
  const uint32_t grid = std::min<uint32_t>(v.n_nodes, 148u * 16);
  if (fmt == LOD_POINTS_F32)
    launch_pdl(k_checks<LOD_POINTS_F32>, grid, 256, 0, s, v, leaf_pts, vox, voxels, T, max_depth, flags);
  else
    launch_pdl(k_checks<LOD_POINTS_F64>, grid, 256, 0, s, v, leaf_pts, vox, voxels, T, max_depth, flags);
  return 1;
}

}  // namespace lod
