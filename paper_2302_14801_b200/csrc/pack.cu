// Device packing of caller arrays into point records (the drop-in's upload path).
//
// The reference's PointCloud holds float64 (n,3) positions + uint8 (n,3) colours
// (ingest.py:21-35).  The Python drop-in uploads those arrays as they are (24 + 3 B/pt, or
// 12 + 3 B/pt for float32 input to the fused entry) and packs them here, instead of building
// records with numpy on one host core (~20 M pts/s):
//   k_f32_exact  -- do all float64 coordinates survive a float32 round trip?  (then the 16-B
//                   record is exact; NaN is never exact, so non-finite input keeps the f64
//                   record and the split reports it, model.py:204-205)
//   k_pack_f32   -- {f32 x, y, z, rgb} 16-B records from f32 or (exact) f64 coordinates
//   k_pack_f64   -- {f64 x, y, z, rgb, pad} 32-B records
// All three are grid-stride streams bound by HBM bandwidth (one read of the inputs, one write
// of the records).
#include "kernels.h"

namespace lod {

namespace {

__global__ void k_f32_exact(const double* __restrict__ xyz, uint64_t m, uint32_t* __restrict__ flag) {
  pdl_wait();
  bool ok = true;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const double v = __ldcs(xyz + i);
    ok &= (double)__double2float_rn(v) == v;
  }
  if (!__all_sync(0xFFFFFFFFu, ok) && (threadIdx.x & 31) == 0) atomicExch(flag, 0u);
}

template <bool F64_IN>
__global__ void k_pack_f32(const void* __restrict__ xyz, const uint8_t* __restrict__ rgb, uint64_t n,
                           uint4* __restrict__ out) {
  pdl_wait();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    float x, y, z;
    if (F64_IN) {
      const double* p = static_cast<const double*>(xyz) + 3 * i;
      x = __double2float_rn(__ldcs(p)), y = __double2float_rn(__ldcs(p + 1)), z = __double2float_rn(__ldcs(p + 2));
    } else {
      const float* p = static_cast<const float*>(xyz) + 3 * i;
      x = __ldcs(p), y = __ldcs(p + 1), z = __ldcs(p + 2);
    }
    const uint8_t* c = rgb + 3 * i;
    const uint32_t col = (uint32_t)__ldcs(c) | ((uint32_t)__ldcs(c + 1) << 8) | ((uint32_t)__ldcs(c + 2) << 16);
    out[i] = make_uint4(__float_as_uint(x), __float_as_uint(y), __float_as_uint(z), col);
  }
}

template <bool F64_IN>
__global__ void k_pack_f64(const void* __restrict__ xyz, const uint8_t* __restrict__ rgb, uint64_t n,
                           uint4* __restrict__ out) {
  pdl_wait();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    double x, y, z;
    if (F64_IN) {
      const double* p = static_cast<const double*>(xyz) + 3 * i;
      x = __ldcs(p), y = __ldcs(p + 1), z = __ldcs(p + 2);
    } else {
      const float* p = static_cast<const float*>(xyz) + 3 * i;
      x = __ldcs(p), y = __ldcs(p + 1), z = __ldcs(p + 2);
    }
    const uint8_t* c = rgb + 3 * i;
    const uint32_t col = (uint32_t)__ldcs(c) | ((uint32_t)__ldcs(c + 1) << 8) | ((uint32_t)__ldcs(c + 2) << 16);
    const unsigned long long bx = __double_as_longlong(x), by = __double_as_longlong(y), bz = __double_as_longlong(z);
    out[2 * i] = make_uint4((uint32_t)bx, (uint32_t)(bx >> 32), (uint32_t)by, (uint32_t)(by >> 32));
    out[2 * i + 1] = make_uint4((uint32_t)bz, (uint32_t)(bz >> 32), col, 0u);
  }
}

uint32_t stream_blocks(uint64_t n) { return (uint32_t)std::min<uint64_t>((n + 255) / 256, 148ull * 8); }

}  // namespace

int launch_f32_exact(const double* xyz, uint64_t n, uint32_t* flag, cudaStream_t s) {
  if (!n) return 0;
  launch_pdl(k_f32_exact, stream_blocks(3 * n), 256, 0, s, xyz, 3 * n, flag);
  return 1;
}

int launch_pack(const void* xyz, bool f64_in, const uint8_t* rgb, uint64_t n, int out_format, void* out,
                cudaStream_t s) {
  if (!n) return 0;
  uint4* o = static_cast<uint4*>(out);
  const uint32_t b = stream_blocks(n);
  if (out_format == LOD_POINTS_F32) {
    if (f64_in) launch_pdl(k_pack_f32<true>, b, 256, 0, s, xyz, rgb, n, o);
    else launch_pdl(k_pack_f32<false>, b, 256, 0, s, xyz, rgb, n, o);
  } else {
    if (f64_in) launch_pdl(k_pack_f64<true>, b, 256, 0, s, xyz, rgb, n, o);
    else launch_pdl(k_pack_f64<false>, b, 256, 0, s, xyz, rgb, n, o);
  }
  return 1;
}

}  // namespace lod
