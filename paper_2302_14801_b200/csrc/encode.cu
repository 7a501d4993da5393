// VLPC payload on the device (reference codec.py:28-47, 49-83).
//
//   leaf  nodes: 16-B records {f32 off[3] = clip(f32(p - node_min), 0, f32(size)); u8 r, g, b; 0}
//                (codec.py:34-39; fp64 subtraction, one rounding to f32, clip in f32)
//   inner nodes:  6-B records {u8 cx, cy, cz, r, g, b} in the node's stored voxel order
//                (codec.py:42-46)
// The caller supplies the node order (sorted by path, codec.py:51) and each node's byte
// offset in the payload; header and node table are host-side bytes (a few per node).
// One CTA per node, grid-strided, so the records of a node are written coalesced.
#include "kernels.h"

namespace lod {

namespace {

template <int FMT>
__global__ void __launch_bounds__(256) k_encode(SplitView v, const void* leaf_pts, const uint2* vox,
                                                const int32_t* order, const uint64_t* offs, uint32_t n,
                                                uint8_t* out) {
  pdl_wait();
  for (uint32_t q = blockIdx.x; q < n; q += gridDim.x) {
    const int32_t node = order[q];
    const uint64_t off = offs[q];
    const uint64_t first = v.n_first[node];
    const uint32_t count = v.n_count[node];
    if (v.n_leaf[node] >= 0) {
      const double4 b = v.n_box[node];
      const float fs = __double2float_rn(b.w);
      uint4* dst = reinterpret_cast<uint4*>(out + off);
      for (uint32_t j = threadIdx.x; j < count; j += blockDim.x) {
        const auto r = Rec<FMT>::load(leaf_pts, first + j);
        const float ox = fminf(fmaxf(__double2float_rn(__dsub_rn(Rec<FMT>::x(r), b.x)), 0.f), fs);
        const float oy = fminf(fmaxf(__double2float_rn(__dsub_rn(Rec<FMT>::y(r), b.y)), 0.f), fs);
        const float oz = fminf(fmaxf(__double2float_rn(__dsub_rn(Rec<FMT>::z(r), b.z)), 0.f), fs);
        const uint4 rec = make_uint4(__float_as_uint(ox), __float_as_uint(oy), __float_as_uint(oz), Rec<FMT>::rgb(r));
        // widest store the node's offset allows (6-B voxel runs before it keep it only even)
        const uint32_t w[4] = {rec.x, rec.y, rec.z, rec.w};
        if ((off & 15) == 0) {
          dst[j] = rec;
        } else if ((off & 3) == 0) {
          uint32_t* d = reinterpret_cast<uint32_t*>(out + off + 16ull * j);
#pragma unroll
          for (int k = 0; k < 4; ++k) d[k] = w[k];
        } else {
          uint16_t* d = reinterpret_cast<uint16_t*>(out + off + 16ull * j);
#pragma unroll
          for (int k = 0; k < 4; ++k) d[2 * k] = (uint16_t)w[k], d[2 * k + 1] = (uint16_t)(w[k] >> 16);
        }
      }
    } else {
      uint16_t* dst = reinterpret_cast<uint16_t*>(out + off);  // offsets are even (16 a + 6 b)
      for (uint32_t j = threadIdx.x; j < count; j += blockDim.x) {
        const uint2 e = vox[first + j];
        const uint32_t x = e.x >> 14, y = (e.x >> 7) & 127, z = e.x & 127;
        dst[3 * j] = (uint16_t)(x | (y << 8));
        dst[3 * j + 1] = (uint16_t)(z | ((e.y & 0xFF) << 8));
        dst[3 * j + 2] = (uint16_t)((e.y >> 8) & 0xFFFF);
      }
    }
  }
}

}  // namespace

int launch_encode(int fmt, const SplitView& v, const void* leaf_pts, const uint2* vox, const int32_t* order,
                  const uint64_t* offs, uint32_t n, uint8_t* out, cudaStream_t s) {
  if (!n) return 0;
  const uint32_t grid = std::min<uint32_t>(n, 148u * 16);
  if (fmt == LOD_POINTS_F32)
    launch_pdl(k_encode<LOD_POINTS_F32>, grid, 256, 0, s, v, leaf_pts, vox, order, offs, n, out);
  else
    launch_pdl(k_encode<LOD_POINTS_F64>, grid, 256, 0, s, v, leaf_pts, vox, order, offs, n, out);
  return 1;
}

}  // namespace lod
