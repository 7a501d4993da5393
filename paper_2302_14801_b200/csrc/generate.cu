// Device generators for the BASELINE synthetic clouds, bit-identical to the numpy
// generators in paper_2302_14801_b200/generators.py (same splitmix64 streams, same fp64
// operation order with explicit round-to-nearest intrinsics, no FMA contraction).
// Used to produce the 500M-4B point configs directly in HBM.
#include "kernels.h"

namespace lod {

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  uint64_t z = x + kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// rng.stream(seed, .)[k] -> to_unit
__device__ __forceinline__ double unit(uint64_t seed, uint64_t k) {
  return (double)(mix64(seed + k * kGolden) >> 11) * 0x1p-53;
}

struct Dir { double x, y, z; };

__device__ __forceinline__ Dir sphere_dir(double u0, double u1, double u2) {
  double vx = __dsub_rn(__dmul_rn(2.0, u0), 1.0);
  double vy = __dsub_rn(__dmul_rn(2.0, u1), 1.0);
  double vz = __dsub_rn(__dmul_rn(2.0, u2), 1.0);
  double r = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz)));
  if (r == 0.0) {
    vx = 1.0;
    r = 1.0;
  }
  return Dir{__ddiv_rn(vx, r), __ddiv_rn(vy, r), __ddiv_rn(vz, r)};
}

__device__ __forceinline__ uint32_t pack_rgb(double r, double g, double b) {
  return (uint32_t)r | ((uint32_t)g << 8) | ((uint32_t)b << 16);
}

__device__ __forceinline__ void put(uint4* out, uint64_t i, double x, double y, double z, uint32_t rgb) {
  out[i] = make_uint4(__float_as_uint(__double2float_rn(x)), __float_as_uint(__double2float_rn(y)),
                      __float_as_uint(__double2float_rn(z)), rgb);
}

__device__ __forceinline__ void sphere_row(double u0, double u1, double u2, double& x, double& y, double& z,
                                           uint32_t& rgb) {
  Dir w = sphere_dir(u0, u1, u2);
  x = __dadd_rn(0.5, __dmul_rn(0.5, w.x));
  y = __dadd_rn(0.5, __dmul_rn(0.5, w.y));
  z = __dadd_rn(0.5, __dmul_rn(0.5, w.z));
  rgb = pack_rgb(floor(__dmul_rn(255.0, x)), floor(__dmul_rn(255.0, y)), floor(__dmul_rn(255.0, z)));
}

__device__ __forceinline__ double lattice(uint64_t seed, int oct, int64_t ix, int64_t iy) {
  uint64_t key = ((uint64_t)((seed * 8 + oct) & 0xFFFFFF) << 40) ^ ((uint64_t)ix << 20) ^ (uint64_t)iy;
  double t = (double)(mix64(key) >> 11) * 0x1p-53;
  return __dsub_rn(__dmul_rn(t, 2.0), 1.0);
}

__device__ __forceinline__ void terrain_row(uint64_t seed, double x, double y, double jit, double& z,
                                            uint32_t& rgb) {
  double h = 0.0, amp = 1.0;
  for (int k = 0; k < 4; ++k) {
    double cells = (double)(4 << k);
    double gx = __dmul_rn(x, cells), gy = __dmul_rn(y, cells);
    double ix = floor(gx), iy = floor(gy);
    double fx = __dsub_rn(gx, ix), fy = __dsub_rn(gy, iy);
    int64_t ixi = (int64_t)ix, iyi = (int64_t)iy;
    double a = lattice(seed, k, ixi, iyi), b = lattice(seed, k, ixi + 1, iyi);
    double c = lattice(seed, k, ixi, iyi + 1), d = lattice(seed, k, ixi + 1, iyi + 1);
    double top = __dadd_rn(a, __dmul_rn(__dsub_rn(b, a), fx));
    double bot = __dadd_rn(c, __dmul_rn(__dsub_rn(d, c), fx));
    h = __dadd_rn(h, __dmul_rn(amp, __dadd_rn(top, __dmul_rn(__dsub_rn(bot, top), fy))));
    amp = __dmul_rn(amp, 0.5);
  }
  z = __dadd_rn(__dadd_rn(0.5, __dmul_rn(0.08, h)), __dmul_rn(0.001, __dsub_rn(jit, 0.5)));
  double t = __ddiv_rn(__dsub_rn(z, 0.35), 0.3);
  t = fmin(fmax(t, 0.0), 1.0);
  bool checker = fmod(__dadd_rn(floor(__dmul_rn(x, 8.0)), floor(__dmul_rn(y, 8.0))), 2.0) == 0.0;
  rgb = pack_rgb(floor(__dmul_rn(255.0, t)), floor(__dmul_rn(255.0, __dsub_rn(1.0, t))), checker ? 200.0 : 60.0);
}

// kind: 0 sphere, 1 terrain, 2 scene, 3 cluster, 4 surface
__global__ void k_generate(int kind, uint64_t seed, uint64_t start, uint64_t n, uint4* out, const double* table) {
  pdl_wait();
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = start + t;
    double x, y, z;
    uint32_t rgb;
    if (kind == 0 || kind == 3) {
      double u0 = unit(seed, 3 * i), u1 = unit(seed, 3 * i + 1), u2 = unit(seed, 3 * i + 2);
      sphere_row(u0, u1, u2, x, y, z, rgb);
      if (kind == 3) {
        if (i % 10 == 0) {  // dense cube of side 2^-12 at one of 16 corners
          uint64_t cid = (i / 10) % 16;
          double cs[3];
          for (int a = 0; a < 3; ++a)
            cs[a] = __dadd_rn(0.1, __dmul_rn(0.8, unit(seed ^ 0x5EEDull, 3 * cid + a)));
          x = __dadd_rn(cs[0], __dmul_rn(1.0 / 4096.0, u0));
          y = __dadd_rn(cs[1], __dmul_rn(1.0 / 4096.0, u1));
          z = __dadd_rn(cs[2], __dmul_rn(1.0 / 4096.0, u2));
        } else if (i % 10 == 5 && i / 10 < 50001) {  // exact duplicates -> oversized leaf
          x = 0.25, y = 0.5, z = 0.75;
        }
      }
    } else if (kind == 1 || kind == 4) {
      double u0 = unit(seed, 4 * i), u1 = unit(seed, 4 * i + 1), u2 = unit(seed, 4 * i + 2);
      if (kind == 4 && (i % 2) == 0) {
        sphere_row(u0, u1, u2, x, y, z, rgb);
      } else {
        x = u0;
        y = u1;
        terrain_row(seed, u0, u1, u2, z, rgb);
      }
    } else {  // scene: table = 65 rows {kind, p0..p6, cdf}
      double u[6];
      for (int a = 0; a < 6; ++a) u[a] = unit(seed, 6 * i + a);
      int lo = 0, hi = 65;  // searchsorted(cdf, u0, side="right")
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (table[9 * mid + 8] <= u[0]) lo = mid + 1; else hi = mid;
      }
      int obj = lo < 64 ? lo : 64;
      const double* p = table + 9 * obj + 1;
      int k = (int)table[9 * obj];
      if (k == 0) {
        x = __dmul_rn(1000.0, u[1]);
        y = __dmul_rn(1000.0, u[2]);
        z = 0.0;
      } else if (k == 1) {
        Dir w = sphere_dir(u[1], u[2], u[3]);
        x = __dadd_rn(p[0], __dmul_rn(p[3], w.x));
        y = __dadd_rn(p[1], __dmul_rn(p[3], w.y));
        z = __dadd_rn(p[2], __dmul_rn(p[3], w.z));
      } else {
        int face = (int)floor(__dmul_rn(6.0, u[1]));
        double a2 = __dsub_rn(__dmul_rn(2.0, u[2]), 1.0), a3 = __dsub_rn(__dmul_rn(2.0, u[3]), 1.0);
        double sign = (face % 2 == 0) ? -1.0 : 1.0;
        int axis = face / 2;
        double l0 = axis == 0 ? sign : a2;
        double l1 = axis == 1 ? sign : (axis == 0 ? a2 : a3);
        double l2 = axis == 2 ? sign : a3;
        x = __dadd_rn(p[0], __dmul_rn(p[3], l0));
        y = __dadd_rn(p[1], __dmul_rn(p[4], l1));
        z = __dadd_rn(p[2], __dmul_rn(p[5], l2));
      }
      uint64_t base = mix64((uint64_t)obj + seed * 131ull);
      uint32_t jit = (uint32_t)floor(__dmul_rn(40.0, u[4]));
      rgb = (((uint32_t)(base >> 8) & 0xBF) + jit) | ((((uint32_t)(base >> 24) & 0xBF) + jit) << 8) |
            ((((uint32_t)(base >> 40) & 0xBF) + jit) << 16);
    }
    put(out, t, x, y, z, rgb);
  }
}

}  // namespace

int launch_generate(int kind, uint64_t seed, uint64_t start, uint64_t n, void* out, const double* table,
                    cudaStream_t s) {
  uint32_t blocks = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
  if (blocks == 0) return 0;
  launch_pdl(k_generate, blocks, 256, 0, s, kind, seed, start, n, reinterpret_cast<uint4*>(out), table);
  return 1;
}

}  // namespace lod
