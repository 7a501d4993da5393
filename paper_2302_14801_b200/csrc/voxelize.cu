// Voxel sampling of inner nodes, one launch per octree depth, deepest first
// (reference sampling.py:165-176 build_lod; per node sampling.py:21-97).
//
// One 2-CTA cluster per node (persistent clusters pull node tickets).  The node's 128^3
// sampling grid is an occupancy BITMAP split by the x-high bit across the pair's shared
// memory (2 x 128 KB, DSMEM for the rare cross-half sample).  Because keys are x-major,
// every key of half 0 precedes every key of half 1, so
//     voxel index of key = rank(key) = #occupied keys < key
// is a local prefix-popcount lookup (+ half 0's total for half 1).  Voxels therefore come
// out in ascending key order (sampling.py:83-85, 97) with no sort, and the per-voxel
// accumulators are compact (m entries, L2-resident) instead of a 128^3 dense grid.
//
//   pass A  samples -> atomicOr occupancy bits
//   rank    per-word prefix popcounts (u16 within 64-word superblocks + u32 superblock base)
//   emit    voxel keys in rank order, accumulators zeroed
//   pass B  average: exact integer channel sums + counts (sampling.py:88-97)
//           random : atomicMax of (rand12 | ordinal20) (sampling.py:69-85, PAPER Listing 1)
//   final   average: (2*sum + n) / (2*n) per channel; random: winner's colour (pass C)
//
// CTA h of the pair processes the children whose octant has x-bit h: voxel children map
// into half h exactly, leaf children except at the boundary, so DSMEM traffic is rare.
#include <cooperative_groups.h>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace lod {

namespace {

constexpr int kVT = 1024;
constexpr int kHalfWords = 1 << 15;  // 2^20 cells per half / 32
constexpr int kSuperShift = 6;       // 64 words per superblock
constexpr int kNumSuper = kHalfWords >> kSuperShift;
constexpr uint32_t kWideS = 1u << 24;  // below this, 32-bit channel sums cannot overflow

struct __align__(16) VoxSmem {
  uint32_t bits[kHalfWords];
  uint16_t rel[kHalfWords];
  uint32_t super[kNumSuper];
  uint64_t cfirst[8];
  uint32_t ccount[8];
  uint32_t cbase[8];   // ordinal of the child's first sample (octant order over ALL children)
  int32_t ckind[8];    // 1 leaf, 0 inner, -1 absent
  uint32_t mine[4];    // octants processed by this CTA
  uint32_t mine_pre[5];
  double lo[3];
  double size;
  unsigned long long hash;
  unsigned long long vbase;
  uint32_t node, S, total, peer_total, ticket, n_mine;
  int skip;
  uint32_t scan[kVT / 32 + 1];
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// child voxel key c in octant o -> parent key floor(off + (c + 0.5) / 2) = off + c / 2
// (sampling.py:41-44)
__device__ __forceinline__ uint32_t voxel_to_parent(int o, uint32_t k) {
  uint32_t x = ((uint32_t)(o & 1) << 6) | (k >> 15);
  uint32_t y = ((uint32_t)((o >> 1) & 1) << 6) | ((k >> 8) & 63);
  uint32_t z = ((uint32_t)(o >> 2) << 6) | ((k & 127) >> 1);
  return (x << 14) | (y << 7) | z;
}

// floor((2 s + n) / (2 n)) -- round half up (sampling.py:96) -- without a 64-bit divide:
// a float quotient is within one of the result, an integer check fixes it.
__device__ __forceinline__ uint32_t mean_round(uint64_t s, uint64_t n) {
  uint64_t a = 2 * s + n, b = 2 * n;
  uint32_t q = (uint32_t)__fdividef((float)a, (float)b);
  if ((uint64_t)q * b > a) --q;
  else if ((uint64_t)(q + 1) * b <= a) ++q;
  return q;
}

__device__ __forceinline__ uint32_t rank_in(const VoxSmem* s, uint32_t k20) {
  uint32_t w = k20 >> 5, b = k20 & 31;
  return s->super[w >> kSuperShift] + s->rel[w] + __popc(s->bits[w] & ((1u << b) - 1));
}

// Visit this CTA's samples: fn(ordinal, key in this node's grid, rgb).  Leaf children
// come from the distribute stash (key already in this grid), inner children from the
// voxel arena.  Four independent loads per thread per trip keep enough bytes in flight.
template <class Fn>
__device__ __forceinline__ void for_my_samples(const VoxView& v, const VoxSmem& s, Fn fn) {
  constexpr int U = 4;
  for (uint32_t c = 0; c < s.n_mine; ++c) {
    const int o = (int)s.mine[c];
    const uint32_t cnt = s.ccount[o];
    const bool leaf = s.ckind[o] == 1;
    const uint2* src = (leaf ? v.stash : v.vox) + s.cfirst[o];
    const uint32_t ob = s.cbase[o];
    for (uint32_t j0 = threadIdx.x; j0 < cnt; j0 += U * kVT) {
      uint2 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint32_t j = j0 + u * kVT;
        if (j < cnt) r[u] = __ldg(src + j);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint32_t j = j0 + u * kVT;
        if (j < cnt) fn(ob + j, leaf ? r[u].x : voxel_to_parent(o, r[u].x), r[u].y);
      }
    }
  }
}

template <int FMT, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kVT, 1) k_voxelize(VoxView v) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  VoxSmem& s = *reinterpret_cast<VoxSmem*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t h = cluster.block_rank();
  VoxSmem* peer = cluster.map_shared_rank(&s, (int)(h ^ 1));
  const int tid = threadIdx.x;
  uint64_t* acc = v.scratch + (uint64_t)(blockIdx.x >> 1) * v.scratch_per_slot;
  uint32_t* acc32 = reinterpret_cast<uint32_t*>(acc);

  while (true) {
    if (h == 0 && tid == 0) {
      uint32_t t = atomicAdd(&v.st->work[v.depth], 1u);
      s.ticket = t;
      peer->ticket = t;
    }
    cluster.sync();
    if (s.ticket >= v.list_n) break;

    // ---- node setup (both CTAs read the same global state) ----
    if (tid == 0) {
      uint32_t node = v.list[s.ticket];
      s.node = node;
      double4 b = v.n_box[node];
      s.lo[0] = b.x, s.lo[1] = b.y, s.lo[2] = b.z, s.size = b.w;
      uint32_t ord = 0, nm = 0;
      int empty = 0;
      s.mine_pre[0] = 0;
      for (int o = 0; o < 8; ++o) {
        int32_t c = v.n_child[8ull * node + o];
        s.cbase[o] = ord;
        if (c < 0) {
          s.ckind[o] = -1;
          s.ccount[o] = 0;
          continue;
        }
        s.ckind[o] = v.n_leaf[c] >= 0 ? 1 : 0;
        s.ccount[o] = v.n_count[c];
        s.cfirst[o] = v.n_first[c];
        empty |= v.n_count[c] == 0;
        ord += v.n_count[c];
        if ((uint32_t)(o & 1) == h) {
          s.mine[nm] = o;
          s.mine_pre[nm + 1] = s.mine_pre[nm] + v.n_count[c];
          ++nm;
        }
      }
      s.n_mine = nm;
      s.S = ord;
      // path_hash(seed, path): key = mix64(8 key + octant + 1) per digit (rng.py:48-53)
      uint64_t cell = v.n_cell[node];
      uint32_t cx = (uint32_t)cell & 0xFFFF, cy = (uint32_t)(cell >> 16) & 0xFFFF, cz = (uint32_t)(cell >> 32) & 0xFFFF;
      int depth = (int)(cell >> 48) & 0xFF;
      uint64_t key = v.seed;
      for (int b2 = depth - 1; b2 >= 0; --b2) {
        uint32_t oc = ((cx >> b2) & 1) | (((cy >> b2) & 1) << 1) | (((cz >> b2) & 1) << 2);
        key = mix64(key * 8 + oc + 1);
      }
      s.hash = v.seed ^ key;
      int skip = 0;
      if (empty) {
        skip = 1;
        if (h == 0) raise_err(v.st, ERR_EMPTY_CHILD, node);
      } else if (MODE == LOD_MODE_RANDOM && ord >= (uint32_t)kRandomLimit) {
        skip = 1;
        if (h == 0) raise_err(v.st, ERR_RANDOM_LIMIT, node, ord);
      }
      s.skip = skip;
    }
    for (int w = tid; w < kHalfWords; w += kVT) s.bits[w] = 0;
    cluster.sync();  // both halves cleared before any cross-half OR
    if (s.skip) {
      if (h == 0 && tid == 0) {
        v.n_count[s.node] = 0;
        v.n_first[s.node] = 0;
      }
      continue;  // the loop-top cluster.sync keeps the pair in step
    }

    // ---- pass A: occupancy ----
    for_my_samples(v, s, [&](uint32_t, uint32_t key, uint32_t) {
      uint32_t w = (key & 0xFFFFF) >> 5, bit = 1u << (key & 31);
      uint32_t* dst = ((key >> 20) == h) ? s.bits : peer->bits;
      if (!(dst[w] & bit)) atomicOr(dst + w, bit);  // most samples land in an occupied cell
    });
    cluster.sync();

    // ---- rank structure over this half ----
    {
      const int warp = tid >> 5, lane = tid & 31;
      for (int sb = warp; sb < kNumSuper; sb += kVT / 32) {
        int w0 = (sb << kSuperShift) + 2 * lane;
        uint32_t c0 = __popc(s.bits[w0]), c1 = __popc(s.bits[w0 + 1]);
        uint32_t incl = warp_incl_scan(c0 + c1);
        s.rel[w0] = (uint16_t)(incl - c0 - c1);
        s.rel[w0 + 1] = (uint16_t)(incl - c1);
        if (lane == 31) s.super[sb] = incl;
      }
      __syncthreads();
      uint32_t val = tid < kNumSuper ? s.super[tid] : 0;
      uint32_t tot;
      uint32_t ex = block_excl_scan<uint32_t, kVT>(val, &tot, s.scan);
      if (tid < kNumSuper) s.super[tid] = ex;
      if (tid == 0) {
        s.total = tot;
        peer->peer_total = tot;
      }
    }
    cluster.sync();
    const uint32_t total0 = h == 0 ? s.total : s.peer_total;
    const uint32_t m = s.total + s.peer_total;
    if (h == 0 && tid == 0) {
      unsigned long long b = atomicAdd(&v.st->vox_cursor, (unsigned long long)m);
      int over = b + m > v.vox_cap;
      if (over) raise_err(v.st, ERR_ARENA, s.node, b + m);
      s.vbase = b;
      peer->vbase = b;
      s.skip = over;
      peer->skip = over;
      v.n_first[s.node] = b;
      v.n_count[s.node] = over ? 0 : m;
    }
    cluster.sync();
    if (s.skip) continue;
    const uint64_t vbase = s.vbase;
    const uint32_t rank_off = h == 0 ? 0 : total0;
    const bool wide = MODE == LOD_MODE_AVERAGE && s.S >= kWideS;

    // ---- emit keys in rank order, clear accumulators ----
    for (int w = tid; w < kHalfWords; w += kVT) {
      uint32_t bw = s.bits[w];
      if (!bw) continue;
      uint32_t r = rank_off + s.super[w >> kSuperShift] + s.rel[w];
      while (bw) {
        uint32_t b = __ffs(bw) - 1;
        bw &= bw - 1;
        v.vox[vbase + r].x = (h << 20) | ((uint32_t)w << 5) | b;
        if (MODE == LOD_MODE_AVERAGE) {
          acc[2ull * r] = 0;
          acc[2ull * r + 1] = 0;
          if (wide) v.vox[vbase + r].y = 0;
        } else {
          acc32[r] = 0;
        }
        ++r;
      }
    }
    __threadfence();
    cluster.sync();

    auto global_rank = [&](uint32_t key) -> uint32_t {
      uint32_t kh = key >> 20;
      const VoxSmem* own = (kh == h) ? &s : peer;
      return (kh ? total0 : 0) + rank_in(own, key & 0xFFFFF);
    };

    if (MODE == LOD_MODE_RANDOM) {
      // ---- pass B: max (rand12 | ordinal20) per voxel ----
      const uint64_t hs = s.hash;
      for_my_samples(v, s, [&](uint32_t ord, uint32_t key, uint32_t) {
        uint32_t enc = ((uint32_t)(mix64(hs ^ (uint64_t)ord) >> 32) & 0xFFF00000u) | (ord & 0xFFFFFu);
        atomicMax(acc32 + global_rank(key), enc);
      });
      __threadfence();
      cluster.sync();
      // ---- pass C: the winning sample writes its colour ----
      for_my_samples(v, s, [&](uint32_t ord, uint32_t key, uint32_t rgb) {
        uint32_t enc = ((uint32_t)(mix64(hs ^ (uint64_t)ord) >> 32) & 0xFFF00000u) | (ord & 0xFFFFFu);
        uint32_t r = global_rank(key);
        if (__ldcg(acc32 + r) == enc) v.vox[vbase + r].y = rgb;
      });
    } else {
      const int passes = wide ? 3 : 1;
      for (int p = 0; p < passes; ++p) {
        // ---- pass B: exact integer sums + counts ----
        for_my_samples(v, s, [&](uint32_t, uint32_t key, uint32_t rgb) {
          uint32_t r = global_rank(key);
          if (!wide) {
            atomicAdd((unsigned long long*)(acc + 2ull * r),
                      (unsigned long long)(rgb & 0xFF) | ((unsigned long long)((rgb >> 8) & 0xFF) << 32));
            atomicAdd((unsigned long long*)(acc + 2ull * r + 1),
                      (unsigned long long)((rgb >> 16) & 0xFF) | (1ull << 32));
          } else {
            atomicAdd((unsigned long long*)(acc + 2ull * r), (unsigned long long)((rgb >> (8 * p)) & 0xFF));
            atomicAdd((unsigned long long*)(acc + 2ull * r + 1), 1ull);
          }
        });
        __threadfence();
        cluster.sync();
        // ---- finalize own ranks: (2*sum + n) // (2*n), round half up (sampling.py:96) ----
        const uint32_t own = s.total;
        for (uint32_t i = tid; i < own; i += kVT) {
          uint32_t r = rank_off + i;
          uint64_t a = __ldcg(acc + 2ull * r), b = __ldcg(acc + 2ull * r + 1);
          if (!wide) {
            uint64_t n = b >> 32;
            v.vox[vbase + r].y = mean_round(a & 0xFFFFFFFFull, n) | (mean_round(a >> 32, n) << 8) |
                                 (mean_round(b & 0xFFFFFFFFull, n) << 16);
          } else {
            v.vox[vbase + r].y |= mean_round(a, b) << (8 * p);
            acc[2ull * r] = 0;
            acc[2ull * r + 1] = 0;
          }
        }
        if (wide && p + 1 < passes) {
          __threadfence();
          cluster.sync();
        }
      }
    }
  }
}

template <int FMT, int MODE>
void launch_one(const VoxView& v, int n_clusters, cudaStream_t st) {
  auto kern = k_voxelize<FMT, MODE>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(VoxSmem));
    configured = true;
  }
  kern<<<2 * n_clusters, kVT, sizeof(VoxSmem), st>>>(v);
}

}  // namespace

int voxelize_smem_bytes() { return (int)sizeof(VoxSmem); }

int launch_voxelize_level(const VoxView& v, int n_clusters, cudaStream_t s) {
  if (v.fmt == LOD_POINTS_F32) {
    if (v.mode == LOD_MODE_RANDOM)
      launch_one<LOD_POINTS_F32, LOD_MODE_RANDOM>(v, n_clusters, s);
    else
      launch_one<LOD_POINTS_F32, LOD_MODE_AVERAGE>(v, n_clusters, s);
  } else {
    if (v.mode == LOD_MODE_RANDOM)
      launch_one<LOD_POINTS_F64, LOD_MODE_RANDOM>(v, n_clusters, s);
    else
      launch_one<LOD_POINTS_F64, LOD_MODE_AVERAGE>(v, n_clusters, s);
  }
  return 1;
}

}  // namespace lod
