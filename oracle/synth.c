/* Host restatement of the BASELINE synthetic clouds (TEST INFRASTRUCTURE, not product code).
 *
 * Bit-identical to `paper_2302_14801_b200/generators.py::synthetic_rows` (numpy) and to
 * `csrc/generate.cu` (device): the same splitmix64 counter streams (reference rng.py:16-45)
 * and the same fp64 operation order, compiled with -ffp-contract=off so no FMA is formed.
 * numpy is ~1 M points/s for these generators; this file exists so that
 * `tests/golden/make_subsets.py` can scan the 500M-4B point configs on the build container's
 * cores, pick inner octree nodes, and hand the points inside them (in input order) to the real
 * reference for subtree-subset goldens.
 *
 * kinds: 0 sphere, 1 terrain, 2 scene (table = 65 rows {kind, p0..p6, cdf}), 3 cluster, 4 surface
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ull

static inline uint64_t mix64(uint64_t x) { /* rng.py:16-21 */
  uint64_t z = x + GOLDEN;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline double unit(uint64_t seed, uint64_t k) { /* rng.stream + to_unit, rng.py:36-45 */
  return (double)(mix64(seed + k * GOLDEN) >> 11) * 0x1p-53;
}

static inline void sphere_dir(double u0, double u1, double u2, double* wx, double* wy, double* wz) {
  double vx = 2.0 * u0 - 1.0, vy = 2.0 * u1 - 1.0, vz = 2.0 * u2 - 1.0;
  double r = sqrt((vx * vx + vy * vy) + vz * vz);
  if (r == 0.0) {
    vx = 1.0;
    r = 1.0;
  }
  *wx = vx / r;
  *wy = vy / r;
  *wz = vz / r;
}

static inline uint32_t pack_rgb(double r, double g, double b) {
  return (uint32_t)r | ((uint32_t)g << 8) | ((uint32_t)b << 16);
}

static inline void sphere_row(double u0, double u1, double u2, double* x, double* y, double* z, uint32_t* rgb) {
  double wx, wy, wz;
  sphere_dir(u0, u1, u2, &wx, &wy, &wz);
  *x = 0.5 + 0.5 * wx;
  *y = 0.5 + 0.5 * wy;
  *z = 0.5 + 0.5 * wz;
  *rgb = pack_rgb(floor(255.0 * *x), floor(255.0 * *y), floor(255.0 * *z));
}

static inline double lattice(uint64_t seed, int oct, int64_t ix, int64_t iy) {
  uint64_t key = ((uint64_t)((seed * 8 + oct) & 0xFFFFFF) << 40) ^ ((uint64_t)ix << 20) ^ (uint64_t)iy;
  double t = (double)(mix64(key) >> 11) * 0x1p-53;
  return t * 2.0 - 1.0;
}

static inline void terrain_row(uint64_t seed, double x, double y, double jit, double* z, uint32_t* rgb) {
  double h = 0.0, amp = 1.0;
  for (int k = 0; k < 4; ++k) {
    double cells = (double)(4 << k);
    double gx = x * cells, gy = y * cells;
    double ix = floor(gx), iy = floor(gy);
    double fx = gx - ix, fy = gy - iy;
    int64_t ixi = (int64_t)ix, iyi = (int64_t)iy;
    double a = lattice(seed, k, ixi, iyi), b = lattice(seed, k, ixi + 1, iyi);
    double c = lattice(seed, k, ixi, iyi + 1), d = lattice(seed, k, ixi + 1, iyi + 1);
    double top = a + (b - a) * fx;
    double bot = c + (d - c) * fx;
    h = h + amp * (top + (bot - top) * fy);
    amp = amp * 0.5;
  }
  *z = (0.5 + 0.08 * h) + 0.001 * (jit - 0.5);
  double t = (*z - 0.35) / 0.3;
  t = fmin(fmax(t, 0.0), 1.0);
  int checker = fmod(floor(x * 8.0) + floor(y * 8.0), 2.0) == 0.0;
  *rgb = pack_rgb(floor(255.0 * t), floor(255.0 * (1.0 - t)), checker ? 200.0 : 60.0);
}

/* One row i of cloud `kind`: float32 xyz (as the device record stores them) + packed rgb. */
static inline void row(int kind, uint64_t seed, uint64_t i, const double* table, float* p, uint32_t* rgb) {
  double x, y, z;
  if (kind == 0 || kind == 3) {
    double u0 = unit(seed, 3 * i), u1 = unit(seed, 3 * i + 1), u2 = unit(seed, 3 * i + 2);
    sphere_row(u0, u1, u2, &x, &y, &z, rgb);
    if (kind == 3) {
      if (i % 10 == 0) {
        uint64_t cid = (i / 10) % 16;
        double cs[3];
        for (int a = 0; a < 3; ++a) cs[a] = 0.1 + 0.8 * unit(seed ^ 0x5EEDull, 3 * cid + a);
        x = cs[0] + (1.0 / 4096.0) * u0;
        y = cs[1] + (1.0 / 4096.0) * u1;
        z = cs[2] + (1.0 / 4096.0) * u2;
      } else if (i % 10 == 5 && i / 10 < 50001) {
        x = 0.25, y = 0.5, z = 0.75;
      }
    }
  } else if (kind == 1 || kind == 4) {
    double u0 = unit(seed, 4 * i), u1 = unit(seed, 4 * i + 1), u2 = unit(seed, 4 * i + 2);
    if (kind == 4 && (i % 2) == 0) {
      sphere_row(u0, u1, u2, &x, &y, &z, rgb);
    } else {
      x = u0;
      y = u1;
      terrain_row(seed, u0, u1, u2, &z, rgb);
    }
  } else {
    double u[6];
    for (int a = 0; a < 6; ++a) u[a] = unit(seed, 6 * i + a);
    int lo = 0, hi = 65;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (table[9 * mid + 8] <= u[0]) lo = mid + 1; else hi = mid;
    }
    int obj = lo < 64 ? lo : 64;
    const double* q = table + 9 * obj + 1;
    int k = (int)table[9 * obj];
    if (k == 0) {
      x = 1000.0 * u[1];
      y = 1000.0 * u[2];
      z = 0.0;
    } else if (k == 1) {
      double wx, wy, wz;
      sphere_dir(u[1], u[2], u[3], &wx, &wy, &wz);
      x = q[0] + q[3] * wx;
      y = q[1] + q[3] * wy;
      z = q[2] + q[3] * wz;
    } else {
      int face = (int)floor(6.0 * u[1]);
      double a2 = 2.0 * u[2] - 1.0, a3 = 2.0 * u[3] - 1.0;
      double sign = (face % 2 == 0) ? -1.0 : 1.0;
      int axis = face / 2;
      double l0 = axis == 0 ? sign : a2;
      double l1 = axis == 1 ? sign : (axis == 0 ? a2 : a3);
      double l2 = axis == 2 ? sign : a3;
      x = q[0] + q[3] * l0;
      y = q[1] + q[4] * l1;
      z = q[2] + q[5] * l2;
    }
    uint64_t base = mix64((uint64_t)obj + seed * 131ull);
    uint32_t jit = (uint32_t)floor(40.0 * u[4]);
    *rgb = (((uint32_t)(base >> 8) & 0xBF) + jit) | ((((uint32_t)(base >> 24) & 0xBF) + jit) << 8) |
           ((((uint32_t)(base >> 40) & 0xBF) + jit) << 16);
  }
  p[0] = (float)x;
  p[1] = (float)y;
  p[2] = (float)z;
}

/* reference cells_of (model.py:84-98) at dim = 2^depth: clip(floor((p - min) / size * dim)) */
static inline uint32_t cell_key(const float* p, const double* wb, int depth) {
  const double dim = (double)(1u << depth);
  uint32_t key = 0;
  for (int a = 0; a < 3; ++a) {
    double c = floor(((double)p[a] - wb[a]) / wb[3] * dim);
    if (c < 0) c = 0;
    if (c > dim - 1) c = dim - 1;
    key = key * (1u << depth) + (uint32_t)c; /* x-major (partition.py:23-24) */
  }
  return key;
}

/* rows start..start+n-1 -> pos (n,3) f32, col (n,3) u8 */
void synth_rows(int kind, uint64_t seed, uint64_t start, uint64_t n, const double* table, float* pos,
                uint8_t* col) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < (int64_t)n; ++t) {
    uint32_t rgb;
    row(kind, seed, start + (uint64_t)t, table, pos + 3 * t, &rgb);
    col[3 * t] = rgb & 255;
    col[3 * t + 1] = (rgb >> 8) & 255;
    col[3 * t + 2] = (rgb >> 16) & 255;
  }
}

/* arbitrary row indices idx[0..m) -> pos, col */
void synth_rows_idx(int kind, uint64_t seed, const uint64_t* idx, uint64_t m, const double* table, float* pos,
                    uint8_t* col) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < (int64_t)m; ++t) {
    uint32_t rgb;
    row(kind, seed, idx[t], table, pos + 3 * t, &rgb);
    col[3 * t] = rgb & 255;
    col[3 * t + 1] = (rgb >> 8) & 255;
    col[3 * t + 2] = (rgb >> 16) & 255;
  }
}

/* per-axis min / max (as f64 of the f32 coordinates) of rows start..start+n-1; returns the
 * number of non-finite coordinates */
uint64_t synth_bounds(int kind, uint64_t seed, uint64_t start, uint64_t n, const double* table, double* out6) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  uint64_t bad = 0;
#pragma omp parallel
  {
    double lmn[3] = {INFINITY, INFINITY, INFINITY}, lmx[3] = {-INFINITY, -INFINITY, -INFINITY};
    uint64_t lbad = 0;
#pragma omp for schedule(static)
    for (int64_t t = 0; t < (int64_t)n; ++t) {
      float p[3];
      uint32_t rgb;
      row(kind, seed, start + (uint64_t)t, table, p, &rgb);
      for (int a = 0; a < 3; ++a) {
        if (!isfinite(p[a])) { ++lbad; continue; }
        if (p[a] < lmn[a]) lmn[a] = p[a];
        if (p[a] > lmx[a]) lmx[a] = p[a];
      }
    }
#pragma omp critical
    {
      for (int a = 0; a < 3; ++a) {
        if (lmn[a] < mn[a]) mn[a] = lmn[a];
        if (lmx[a] > mx[a]) mx[a] = lmx[a];
      }
      bad += lbad;
    }
  }
  for (int a = 0; a < 3; ++a) {
    out6[a] = mn[a];
    out6[3 + a] = mx[a];
  }
  return bad;
}

/* hist[key at `depth`] += 1 over rows start..start+n-1 (u64 counters, atomic) */
void synth_hist(int kind, uint64_t seed, uint64_t start, uint64_t n, const double* table, const double* wb,
                int depth, uint64_t* hist) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < (int64_t)n; ++t) {
    float p[3];
    uint32_t rgb;
    row(kind, seed, start + (uint64_t)t, table, p, &rgb);
    __atomic_fetch_add(hist + cell_key(p, wb, depth), 1, __ATOMIC_RELAXED);
  }
}

/* sel[t] = lut[key at `depth`] for rows start..start+n-1 (lut: int16 per cell, -1 = none) */
void synth_select(int kind, uint64_t seed, uint64_t start, uint64_t n, const double* table, const double* wb,
                  int depth, const int16_t* lut, int16_t* sel) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < (int64_t)n; ++t) {
    float p[3];
    uint32_t rgb;
    row(kind, seed, start + (uint64_t)t, table, p, &rgb);
    sel[t] = lut[cell_key(p, wb, depth)];
  }
}
