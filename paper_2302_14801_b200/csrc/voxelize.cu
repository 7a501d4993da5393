// Voxel sampling of inner nodes, one level at a time, deepest first
// (reference sampling.py:165-176 build_lod; per node sampling.py:21-97).
//
// Level-wide data parallel design (every SM works on every level, however few nodes it has):
//
//   per inner node at this depth, an occupancy BITMAP of its 128^3 grid (2^21 bits, 256 KB)
//   plus a per-word exclusive popcount PREFIX (256 KB) live in HBM/L2.  Because keys are
//   x-major, the voxel index of a key is its rank among occupied keys:
//       rank(key) = prefix[key >> 5] + popc(bits[key >> 5] & ((1 << (key & 31)) - 1))
//   so voxels come out in ascending key order (sampling.py:83-85, 97) with no sort.
//
//   K0 setup     one thread per node: children, ordinals, sample chunks (sampling.py:21-47)
//   K1 occupy    all samples, test-and-set their bit (L2 atomics only on first touch)
//   K2 words     per 4096-word block: popcount sums; node offsets; word prefixes, voxel
//                keys, the block's accumulators zeroed (one coalesced sweep of its ranks)
//   K3 scatter   every sample of the level -- leaf points (projected once by K1, stashed)
//                and child voxels (key c in octant o -> off + c/2, sampling.py:41-44) --
//                into its voxel's accumulator: integer channel sums + count as one f32x4
//                reduction (average, sampling.py:88-97), atomicMax of (rand12 | ordinal20)
//                (random, sampling.py:69-85 / PAPER Listing 1), atomicMax of ~ordinal
//                (first-come).  The octant region's bits + prefixes sit in shared memory.
//   K4 finalize  per voxel, from its accumulator alone (no gather from the child level:
//                pushing child voxels was ~2x cheaper than pulling each parent voxel's
//                2x2x2 block through the child's rank structure).
//   Average: (2*sum + n) // (2*n) per channel over the children's ROUNDED colours (H5).
//   Random : max (rand12 | ordinal20); the winning ordinal names the sample directly.
//   First-come (sampling.py:61-66): min ordinal per cell, where a child voxel's ordinal is
//            octant base + its STORED position in the child (vpos).  The node's voxels are
//            then listed by winning ordinal: K4 marks the winners in an ordinal bitmap (S
//            bits per node), one popcount scan over the level's live words gives every winner its stored
//            position p (vpos, used by the parent) and the voxel is written to
//            vout[vbase + p].  The arena itself stays in key order.
//   Weighted (sampling.py:100-133): every sample (leaf points AND child voxels) adds
//            w = clamp(1 - |g - centre|, 0, 1) to the occupied cells of its 2x2x2
//            neighbourhood, as exact 2^-24 fixed-point u64 sums (order-independent, so
//            repeated builds are bit-identical); colour = floor(sum(w c) / sum(w) + 0.5),
//            within +-1 of the reference's sequential fp64 sums.
//
// Bitmaps/prefixes of a level are kept while the next (coarser) level runs (the
// multi-GPU import path rebuilds them for imported subtree roots): two buffers alternate by
// depth parity.
#include "kernels.h"

namespace lod {

namespace {

constexpr uint32_t kWords = 1u << 16;        // 2^21 cells / 32
constexpr uint32_t kBlkWords = 4096;         // words per K2 block
constexpr uint32_t kBlksPerNode = kWords / kBlkWords;
constexpr uint32_t kVoxChunk = 2048;         // voxels per K4 chunk
constexpr int kT = 256;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// child voxel key c in octant o -> parent key off + c / 2 (floor(off + (c + 0.5) / 2))
__device__ __forceinline__ uint32_t voxel_to_parent(int o, uint32_t k) {
  uint32_t x = ((uint32_t)(o & 1) << 6) | (k >> 15);
  uint32_t y = ((uint32_t)((o >> 1) & 1) << 6) | ((k >> 8) & 63);
  uint32_t z = ((uint32_t)(o >> 2) << 6) | ((k & 127) >> 1);
  return (x << 14) | (y << 7) | z;
}

// floor((2 s + n) / (2 n)): round half up (sampling.py:96) without a 64-bit divide
__device__ __forceinline__ uint32_t mean_round(uint64_t s, uint64_t n) {
  uint64_t a = 2 * s + n, b = 2 * n;
  uint32_t q = (uint32_t)__fdividef((float)a, (float)b);
  if ((uint64_t)q * b > a) --q;
  else if ((uint64_t)(q + 1) * b <= a) ++q;
  return q;
}

__device__ __forceinline__ uint32_t rand_enc(uint64_t hash, uint32_t ord) {
  return ((uint32_t)(mix64(hash ^ (uint64_t)ord) >> 32) & 0xFFF00000u) | (ord & 0xFFFFFu);
}

__device__ __forceinline__ uint32_t* bits_of(const VoxLevel& L, int parity, uint32_t slot) {
  return L.bits + ((uint64_t)parity * L.slots + slot) * kWords;
}
__device__ __forceinline__ uint32_t* pre_of(const VoxLevel& L, int parity, uint32_t slot) {
  return L.pre + ((uint64_t)parity * L.slots + slot) * kWords;
}

// ---------------------------------------------------------------------------
// K0: per-node setup; eight lanes per node, one per child octant
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kT) k_setup(VoxLevel L) {
  pdl_wait();
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t s = g >> 3;
  const int o = (int)(g & 7);
  const bool live = s < L.list_n && !(L.st->err & ERR_ARENA);
  const uint32_t node = live ? L.list[s] : 0;
  const int32_t c = live ? L.n_child[8ull * node + o] : -1;
  uint32_t cnt = 0;
  uint64_t first = 0;
  int32_t cslot = -2;  // absent
  if (c >= 0) {
    const bool leaf = L.n_leaf[c] >= 0;
    cnt = L.n_count[c];
    first = L.n_first[c];
    cslot = leaf ? -1 : (int32_t)L.node_slot[c];
  }
  // inclusive scan of the counts over the node's 8 lanes -> ordinal bases (sampling.py:5-6)
  uint32_t incl = cnt;
#pragma unroll
  for (int d = 1; d < 8; d <<= 1) {
    uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d, 8);
    if (o >= d) incl += t;
  }
  const uint32_t S = __shfl_sync(0xFFFFFFFFu, incl, 7, 8);
  const uint32_t emask = (__ballot_sync(0xFFFFFFFFu, c >= 0 && cnt == 0) >> (threadIdx.x & 24)) & 0xFF;
  const bool empty = emask != 0;
  // the reference raises on the first empty child in octant order (sampling.py:33-35)
  const int32_t empty_child = __shfl_sync(0xFFFFFFFFu, c, (threadIdx.x & 24) + (empty ? __ffs(emask) - 1 : 0));
  if (!live) return;
  VoxNode& info = L.info[s];
  info.cbase[o] = incl - cnt;
  info.ccount[o] = cnt;
  info.cfirst[o] = first;
  info.cslot[o] = cslot;
  bool skip = false;
  if (empty) skip = true;
  else if (L.mode == LOD_MODE_RANDOM && S >= (uint32_t)kRandomLimit) skip = true;
  if (o == 0) {
    info.S = S;
    info.node = node;
    // path_hash(seed, path): key = mix64(8 key + octant + 1) per digit (rng.py:48-53)
    uint64_t cell = L.n_cell[node];
    uint32_t cx = (uint32_t)cell & 0xFFFF, cy = (uint32_t)(cell >> 16) & 0xFFFF, cz = (uint32_t)(cell >> 32) & 0xFFFF;
    int depth = (int)(cell >> 48) & 0xFF;
    uint64_t key = L.seed;
    for (int b = depth - 1; b >= 0; --b) {
      uint32_t oc = ((cx >> b) & 1) | (((cy >> b) & 1) << 1) | (((cz >> b) & 1) << 2);
      key = mix64(key * 8 + oc + 1);
    }
    info.hash = L.seed ^ key;
    info.box = L.n_box[node];
    info.inv = __dmul_rn(L.inv_world, (double)(1ull << depth));
    info.vbase = 0;
    info.m = 0;
    info.skip = skip;
    L.node_slot[node] = s;
    if (empty) raise_err(L.st, ERR_EMPTY_CHILD, (uint32_t)empty_child);
    else if (skip) raise_err(L.st, ERR_RANDOM_LIMIT, node, S);
  }
  if (skip || cnt == 0) return;
  const uint32_t chunk = L.chunk;
  const uint32_t nch = (cnt + chunk - 1) / chunk;
  uint32_t at = atomicAdd(L.counters + 0, nch);
  for (uint32_t j = 0; j < cnt; j += chunk) {
    uint4 ch = make_uint4(s, (uint32_t)o, j, min(cnt, j + chunk));
    L.chunks[at++] = ch;
  }
}

// ---------------------------------------------------------------------------
// K1: occupancy.  A chunk holds samples of ONE child octant o, and those land in the node
// grid's octant-o region (64^3 cells = 8192 words) -- always for voxel children, and for
// leaf points except the rare boundary spill.  The region bitmap is built in shared memory
// and OR-ed into the node bitmap once; spills go straight to the global bitmap.
// Leaf points are projected here, once, into the node's grid (sampling.py:29-38) and
// stashed as {key, rgb} for K3/K4.
// ---------------------------------------------------------------------------
constexpr int kRT = 512;                       // threads of the region kernels
constexpr uint32_t kRegionWords = 8192;        // 64 x 64 rows x 2 words

__device__ __forceinline__ bool region_word(uint32_t key, int o, uint32_t& lw) {
  const uint32_t x = key >> 14, y = (key >> 7) & 127, z = key & 127;
  if ((x >> 6) != (uint32_t)(o & 1) || (y >> 6) != (uint32_t)((o >> 1) & 1) || (z >> 6) != (uint32_t)(o >> 2))
    return false;
  lw = (((x & 63) << 6) | (y & 63)) << 1 | ((z >> 5) & 1);
  return true;
}
__device__ __forceinline__ uint32_t region_to_global(uint32_t lw, int o) {
  const uint32_t lx = lw >> 7, ly = (lw >> 1) & 63, lz = lw & 1;
  return ((((uint32_t)(o & 1) << 6 | lx) << 7) | ((uint32_t)((o >> 1) & 1) << 6 | ly)) << 2 |
         ((uint32_t)(o >> 2) << 1 | lz);
}

template <int FMT>
__global__ void __launch_bounds__(kRT, 2) k_occupy(VoxLevel L) {
  pdl_wait();
  if (L.st->err & ERR_ARENA) return;
  __shared__ uint32_t rb[kRegionWords];
  const uint32_t nch = L.counters[0];
  constexpr int U = FMT == LOD_POINTS_F32 ? 8 : 4;  // records in flight per thread
  for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const uint4 ch = L.chunks[c];
    const VoxNode& nd = L.info[ch.x];
    uint32_t* bits = bits_of(L, L.parity, ch.x);
    const int o = (int)ch.y;
    const uint64_t first = nd.cfirst[o];
    for (uint32_t i = threadIdx.x; i < kRegionWords; i += kRT) rb[i] = 0;
    __syncthreads();
    auto mark = [&](uint32_t key) {
      const uint32_t bit = 1u << (key & 31);
      uint32_t lw;
      if (region_word(key, o, lw)) {
        if (!(rb[lw] & bit)) atomicOr(rb + lw, bit);
      } else {  // boundary spill of a leaf point into a neighbouring octant
        atomicOr(bits + (key >> 5), bit);
      }
    };
    if (nd.cslot[o] == -1) {
      const double4 b = nd.box;
      const double inv = nd.inv;
      const Frame32 fr = make_frame32(b.x, b.y, b.z, b.w, 7);  // certified fp32 first (common.cuh)
      for (uint32_t j0 = ch.z + threadIdx.x; j0 < ch.w; j0 += U * kRT) {
        typename Rec<FMT>::Raw r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = Rec<FMT>::load_cs(L.leaf_pts, first + min(j0 + u * kRT, ch.w - 1));
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t j = j0 + u * kRT;
          if (j >= ch.w) continue;
          uint32_t cx, cy, cz, key;
          if (FMT == LOD_POINTS_F32 && fast_cell(Rec<FMT>::xf(r[u]), fr.lo[0], fr.s, fr.band, 128.f, cx) &&
              fast_cell(Rec<FMT>::yf(r[u]), fr.lo[1], fr.s, fr.band, 128.f, cy) &&
              fast_cell(Rec<FMT>::zf(r[u]), fr.lo[2], fr.s, fr.band, 128.f, cz))
            key = (cx << 14) | (cy << 7) | cz;
          else
            key = (grid_cell128(Rec<FMT>::x(r[u]), b.x, b.w, inv) << 14) |
                  (grid_cell128(Rec<FMT>::y(r[u]), b.y, b.w, inv) << 7) | grid_cell128(Rec<FMT>::z(r[u]), b.z, b.w, inv);
          L.stash[first + j] = make_uint2(key, Rec<FMT>::rgb(r[u]));
          mark(key);
        }
      }
    } else {
      const uint2* src = L.vox + first;
      for (uint32_t j0 = ch.z + threadIdx.x; j0 < ch.w; j0 += U * kRT) {
        uint32_t k[U];
#pragma unroll
        for (int u = 0; u < U; ++u) k[u] = __ldg(&src[min(j0 + u * kRT, ch.w - 1)].x);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (j0 + u * kRT < ch.w) mark(voxel_to_parent(o, k[u]));
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < kRegionWords; i += kRT) {
      const uint32_t v = rb[i];
      if (v) atomicOr(bits + region_to_global(i, o), v);
    }
    __syncthreads();
  }
}

template <int NT>
__device__ void alloc_level(const VoxLevel& L) {
  if (L.st->err & ERR_ARENA) return;
  __shared__ uint64_t sm[NT / 32 + 1];
  __shared__ uint64_t carry, ocarry;
  if (threadIdx.x == 0) {
    ocarry = 0;
    carry = L.st->vox_cursor;
    L.level_start[0] = carry;
  }
  __syncthreads();
  for (uint32_t s0 = 0; s0 < L.list_n; s0 += NT) {
    const uint32_t s = s0 + threadIdx.x;
    uint32_t m = 0;
    if (s < L.list_n) {  // the node's 16 block sums as 4 vector loads, all in flight
      uint4* bs = reinterpret_cast<uint4*>(L.blk_sum + s * kBlksPerNode);
      uint4 q[kBlksPerNode / 4];
#pragma unroll
      for (uint32_t b = 0; b < kBlksPerNode / 4; ++b) q[b] = __ldcg(bs + b);
      uint32_t run = 0;
#pragma unroll
      for (uint32_t b = 0; b < kBlksPerNode / 4; ++b) {  // -> the blocks' exclusive prefixes
        const uint4 v = q[b];
        q[b] = make_uint4(run, run + v.x, run + v.x + v.y, run + v.x + v.y + v.z);
        run += v.x + v.y + v.z + v.w;
      }
#pragma unroll
      for (uint32_t b = 0; b < kBlksPerNode / 4; ++b) bs[b] = q[b];
      m = run;
    }
    uint64_t tot;
    uint64_t ex = block_excl_scan<uint64_t, NT>(m, &tot, sm);
    uint64_t ow = 0;  // first-come: words of the node's ordinal bitmap
    if (s < L.list_n && L.mode == LOD_MODE_FIRST_COME && !L.info[s].skip) ow = (L.info[s].S + 31) / 32;
    uint64_t otot;
    uint64_t oex = block_excl_scan<uint64_t, NT>(ow, &otot, sm);
    if (s < L.list_n) {
      VoxNode& nd = L.info[s];
      nd.obase = ocarry + oex;
      uint64_t vb = carry + ex;
      nd.vbase = vb;
      nd.m = m;
      L.n_first[nd.node] = vb;
      L.n_count[nd.node] = m;
      uint32_t nv = (m + L.vchunk - 1) / L.vchunk;
      uint32_t at = atomicAdd(L.counters + 2, nv);
      for (uint32_t q = 0; q < nv; ++q) L.vchunks[at + q] = make_uint2(s, q * L.vchunk);
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += tot, ocarry += otot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (carry > L.vox_cap || carry - L.level_start[0] > L.acc_cap || ocarry > L.ocap)
      raise_err(L.st, ERR_ARENA, 0, carry);
    L.counters[4] = (uint32_t)min(ocarry, (uint64_t)L.ocap);  // first-come: ordinal words in use
    L.st->vox_cursor = carry;
  }
}

// ---------------------------------------------------------------------------
// K2: popcount sums per 4096-word block, node offsets, word prefixes
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kT) k_block_sums(VoxLevel L) {
  pdl_wait();
  const uint32_t s = blockIdx.x / kBlksPerNode, blk = blockIdx.x % kBlksPerNode;
  __shared__ uint32_t red[kT / 32];
  uint32_t c = 0;
  if (!L.info[s].skip && !(L.st->err & ERR_ARENA)) {
    const uint4* b = reinterpret_cast<const uint4*>(bits_of(L, L.parity, s) + blk * kBlkWords);
    for (uint32_t i = threadIdx.x; i < kBlkWords / 4; i += kT) {
      uint4 q = __ldcg(b + i);
      c += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kT / 32; ++w) t += red[w];
    L.blk_sum[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(L.counters + 6, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    alloc_level<kT>(L);
  }
}

// one block: per-node voxel counts -> arena offsets (bump pointer), K4 voxel chunks.  Run by
// the last K2 block to finish (no launch of its own).
// Stage one 4096-word block of a node's bitmap in shared memory and compute every word's
// exclusive popcount prefix (= voxel rank of its first set bit) into spre; returns the
// block's voxel count.
__device__ __forceinline__ uint32_t stage_block(const VoxLevel& L, uint32_t s, uint32_t blk, uint32_t* sbits,
                                                uint32_t* spre, uint32_t* sm) {
  const uint32_t* bits = bits_of(L, L.parity, s) + blk * kBlkWords;
  for (uint32_t i = threadIdx.x; i < kBlkWords / 4; i += kT)
    reinterpret_cast<uint4*>(sbits)[i] = __ldcg(reinterpret_cast<const uint4*>(bits) + i);
  __syncthreads();
  constexpr uint32_t per = kBlkWords / kT;  // 16 consecutive words per thread
  uint32_t c = 0;
#pragma unroll
  for (uint32_t q = 0; q < per; ++q) c += __popc(sbits[threadIdx.x * per + ((q + threadIdx.x) & (per - 1))]);
  uint32_t tot;
  uint32_t r = block_excl_scan<uint32_t, kT>(c, &tot, sm) + L.blk_sum[s * kBlksPerNode + blk];
#pragma unroll
  for (uint32_t q = 0; q < per; ++q) {
    spre[threadIdx.x * per + q] = r;
    r += __popc(sbits[threadIdx.x * per + q]);
  }
  __syncthreads();
  return tot;
}

// K2b: word prefixes to HBM (for rank lookups by K3 and the parent level's gathers), the
// voxel keys, and the block's accumulators zeroed -- its voxels are the contiguous rank
// range [blk_sum, blk_sum + tot), so the zeroing is one coalesced sweep.
__global__ void __launch_bounds__(kT) k_prefix(VoxLevel L) {
  pdl_wait();
  const uint32_t s = blockIdx.x / kBlksPerNode, blk = blockIdx.x % kBlksPerNode;
  const VoxNode& nd = L.info[s];
  if (nd.skip || L.st->err & ERR_ARENA) return;
  __shared__ uint32_t sm[kT / 32 + 1];
  __shared__ __align__(16) uint32_t sbits[kBlkWords];
  __shared__ __align__(16) uint32_t spre[kBlkWords];
  const uint32_t tot = stage_block(L, s, blk, sbits, spre, sm);
  uint32_t* pre = pre_of(L, L.parity, s) + blk * kBlkWords;
  // a prefix is only ever read for a word with a set bit (rank of an occupied key), so the
  // prefixes of empty 4-word groups are not written: sparse (surface) nodes skip most of it
  for (uint32_t i = threadIdx.x; i < kBlkWords / 4; i += kT) {
    const uint4 b4 = reinterpret_cast<const uint4*>(sbits)[i];
    if (b4.x | b4.y | b4.z | b4.w) reinterpret_cast<uint4*>(pre)[i] = reinterpret_cast<const uint4*>(spre)[i];
  }
  // voxel keys in rank order (K4 reads them back voxel-parallel), one thread per voxel so the
  // records are written coalesced: the voxel's word by binary search over the word prefixes
  // (the last word whose prefix <= rank holds it), its bit by select-in-word
  const uint32_t r0 = spre[0];
  for (uint32_t i = threadIdx.x; i < tot; i += kT) {
    const uint32_t r = r0 + i;
    uint32_t lo = 0, hi = kBlkWords - 1;
#pragma unroll
    for (int step = 0; step < 12; ++step) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (spre[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const uint32_t bit = __fns(sbits[lo], 0, (int)(r - spre[lo]) + 1);
    L.vox[nd.vbase + r] = make_uint2(((blk * kBlkWords + lo) << 5) + bit, 0u);
  }
  const uint64_t a0 = nd.vbase - L.level_start[0] + L.blk_sum[blockIdx.x];
  for (uint32_t i = threadIdx.x; i < tot; i += kT) {
    if (L.mode == LOD_MODE_AVERAGE && !L.exact_sums) {
      reinterpret_cast<uint4*>(L.acc)[a0 + i] = make_uint4(0, 0, 0, 0);
    } else if (L.mode == LOD_MODE_WEIGHTED || L.mode == LOD_MODE_AVERAGE) {
      reinterpret_cast<uint4*>(L.acc)[2 * (a0 + i)] = make_uint4(0, 0, 0, 0);
      reinterpret_cast<uint4*>(L.acc)[2 * (a0 + i) + 1] = make_uint4(0, 0, 0, 0);
    } else {
      reinterpret_cast<uint32_t*>(L.acc)[a0 + i] = 0;
    }
  }
}

__device__ __forceinline__ uint32_t rank_of(const uint32_t* bits, const uint32_t* pre, uint32_t key) {
  const uint32_t w = key >> 5;
  return __ldcg(pre + w) + __popc(__ldcg(bits + w) & ((1u << (key & 31)) - 1));
}

// ---------------------------------------------------------------------------
// K3: leaf-point samples (average: and child voxels) -> accumulators.  The octant region's
// bits + prefixes are staged in shared memory, so a sample's rank costs two shared loads;
// only the accumulator atomics reach L2.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kRT, 2) k_scatter(VoxLevel L) {
  pdl_wait();
  if (L.st->err & ERR_ARENA) return;
  extern __shared__ __align__(16) uint32_t rsm[];
  uint32_t* rbits = rsm;
  uint32_t* rpre = rsm + kRegionWords;
  // child VOXELS are pushed here too (one reduction / atomicMax each into the level's
  // accumulators, L2-resident) -- cheaper than K4 gathering every parent voxel's 2x2x2 block
  // through the child's rank structure (~7 scattered sectors per voxel); random and
  // first-come keep the winner's ordinal, which names the sample for K4
  const uint32_t nch = L.counters[0];
  for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const uint4 ch = L.chunks[c];
    const VoxNode& nd = L.info[ch.x];
    const uint32_t* bits = bits_of(L, L.parity, ch.x);
    const uint32_t* pre = pre_of(L, L.parity, ch.x);
    const uint64_t acc0 = nd.vbase - L.level_start[0];
    const int o = (int)ch.y;
    for (uint32_t i = threadIdx.x; i < kRegionWords; i += kRT) {
      const uint32_t gw = region_to_global(i, o);
      const uint32_t w = __ldcg(bits + gw);
      rbits[i] = w;
      if (w) rpre[i] = __ldcg(pre + gw);  // empty words' prefixes are never read (nor written)
    }
    __syncthreads();
    const bool leafc = nd.cslot[o] == -1;
    const uint2* src = (leafc ? L.stash : L.vox) + nd.cfirst[o];
    const uint32_t ob = nd.cbase[o];
    constexpr int U = 4;
    for (uint32_t j0 = ch.z + threadIdx.x; j0 < ch.w; j0 += U * kRT) {
      uint2 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) r[u] = __ldg(src + min(j0 + u * kRT, ch.w - 1));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t j = j0 + u * kRT;
        if (j >= ch.w) continue;
        const uint32_t key = leafc ? r[u].x : voxel_to_parent(o, r[u].x);
        const uint32_t mask = (1u << (key & 31)) - 1;
        uint32_t lw, rank;
        if (region_word(key, o, lw))
          rank = rpre[lw] + __popc(rbits[lw] & mask);
        else
          rank = __ldg(pre + (key >> 5)) + __popc(__ldg(bits + (key >> 5)) & mask);
        const uint64_t a = acc0 + rank;
        const uint32_t rgb = r[u].y;
        if (L.mode == LOD_MODE_AVERAGE && !L.exact_sums) {
          // one vector reduction per sample: {r, g, b, 1} as f32, exact while every sum
          // stays below 2^24 (checked in K4; otherwise the build re-runs with u64 sums)
          float* p = reinterpret_cast<float*>(L.acc) + 4 * a;
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"((float)(rgb & 0xFF)),
                       "f"((float)((rgb >> 8) & 0xFF)), "f"((float)((rgb >> 16) & 0xFF)), "f"(1.0f)
                       : "memory");
        } else if (L.mode == LOD_MODE_AVERAGE) {
          // exact fallback: four u64 sums {r, g, b, count} per voxel (32 B), exact for any
          // sample count (the reference sums in int64, sampling.py:92-96)
          unsigned long long* p = reinterpret_cast<unsigned long long*>(L.acc) + 4 * a;
          atomicAdd(p, (unsigned long long)(rgb & 0xFF));
          atomicAdd(p + 1, (unsigned long long)((rgb >> 8) & 0xFF));
          atomicAdd(p + 2, (unsigned long long)((rgb >> 16) & 0xFF));
          atomicAdd(p + 3, 1ull);
        } else if (L.mode == LOD_MODE_RANDOM) {  // a child voxel's ordinal is its index in the child
          atomicMax(reinterpret_cast<uint32_t*>(L.acc) + a, rand_enc(nd.hash, ob + j));
        } else {  // first-come: the smallest ordinal is the largest complement; a child voxel's
                  // ordinal is its STORED position in the child (sampling.py:5-6, 64-66)
          const uint32_t ord = ob + (leafc ? j : __ldg(L.vpos + nd.cfirst[o] + j));
          atomicMax(reinterpret_cast<uint32_t*>(L.acc) + a, ~ord);
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K3w: weighted -- every sample of the level (leaf points and child voxels) adds its
// 2x2x2 neighbourhood weights to the occupied cells (sampling.py:108-127).  The octant
// region's bits + prefixes are staged in shared memory; neighbours across the region
// border go to the global rank structure.
// ---------------------------------------------------------------------------
constexpr double kWScale = 16777216.0;  // 2^24 fixed point: sum(w) < 2^56 for < 2^32 samples

__device__ __forceinline__ double wdist_axis(double g, uint32_t c) {
  const double d = __dsub_rn(g, __dadd_rn((double)c, 0.5));
  return __dmul_rn(d, d);
}

__global__ void __launch_bounds__(kRT, 2) k_scatter_w(VoxLevel L) {
  pdl_wait();
  if (L.st->err & ERR_ARENA) return;
  extern __shared__ __align__(16) uint32_t rsm[];
  uint32_t* rbits = rsm;
  uint32_t* rpre = rsm + kRegionWords;
  const uint32_t nch = L.counters[0];
  for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const uint4 ch = L.chunks[c];
    const VoxNode& nd = L.info[ch.x];
    const uint32_t* bits = bits_of(L, L.parity, ch.x);
    const uint32_t* pre = pre_of(L, L.parity, ch.x);
    const uint64_t acc0 = nd.vbase - L.level_start[0];
    const int o = (int)ch.y;
    for (uint32_t i = threadIdx.x; i < kRegionWords; i += kRT) {
      const uint32_t gw = region_to_global(i, o);
      const uint32_t w = __ldcg(bits + gw);
      rbits[i] = w;
      if (w) rpre[i] = __ldcg(pre + gw);  // empty words' prefixes are never read (nor written)
    }
    __syncthreads();
    const bool leaf = nd.cslot[o] == -1;
    const uint64_t first = nd.cfirst[o];
    const double4 b = nd.box;
    const double upper = 0x1.fffffffffffffp+6;  // nextafter(128, 0), sampling.py:30
    for (uint32_t j = ch.z + threadIdx.x; j < ch.w; j += kRT) {
      double g[3];
      uint32_t rgb;
      if (leaf) {  // (p - min) / size * 128, clipped (sampling.py:37-38)
        double p[3];
        if (L.fmt == LOD_POINTS_F32) {
          const auto r = Rec<LOD_POINTS_F32>::load(L.leaf_pts, first + j);
          p[0] = Rec<LOD_POINTS_F32>::x(r), p[1] = Rec<LOD_POINTS_F32>::y(r), p[2] = Rec<LOD_POINTS_F32>::z(r);
          rgb = Rec<LOD_POINTS_F32>::rgb(r);
        } else {
          const auto r = Rec<LOD_POINTS_F64>::load(L.leaf_pts, first + j);
          p[0] = Rec<LOD_POINTS_F64>::x(r), p[1] = Rec<LOD_POINTS_F64>::y(r), p[2] = Rec<LOD_POINTS_F64>::z(r);
          rgb = Rec<LOD_POINTS_F64>::rgb(r);
        }
        const double lo[3] = {b.x, b.y, b.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double q = __dmul_rn(__ddiv_rn(__dsub_rn(p[a], lo[a]), b.w), 128.0);
          g[a] = fmin(fmax(q, 0.0), upper);
        }
      } else {     // child voxel c in octant o: off + (c + 0.5) / 2, exact (sampling.py:41-44)
        const uint2 v = __ldg(L.vox + first + j);
        const uint32_t cc[3] = {v.x >> 14, (v.x >> 7) & 127, v.x & 127};
#pragma unroll
        for (int a = 0; a < 3; ++a) g[a] = 64.0 * ((o >> a) & 1) + ((double)cc[a] + 0.5) * 0.5;
        rgb = v.y;
      }
      uint32_t base[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) base[a] = (uint32_t)fmin(fmax(floor(__dsub_rn(g[a], 0.5)), 0.0), 126.0);
      const double col[3] = {(double)(rgb & 0xFF), (double)((rgb >> 8) & 0xFF), (double)((rgb >> 16) & 0xFF)};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t cx = base[0] + (q >> 2), cy = base[1] + ((q >> 1) & 1), cz = base[2] + (q & 1);
        // the cheap tests first, each exact: occupancy (sampling.py:125-128), then the squared
        // distance (sqrt(s) >= 1 for s >= 1, so w = 1 - RN(sqrt(s)) <= 0 there), then w itself
        const uint32_t key = (cx << 14) | (cy << 7) | cz;
        const uint32_t bit = 1u << (key & 31);
        uint32_t lw, word, rank;
        const bool local = region_word(key, o, lw);
        word = local ? rbits[lw] : __ldcg(bits + (key >> 5));
        if (!(word & bit)) continue;
        const double s2 = __dadd_rn(__dadd_rn(wdist_axis(g[0], cx), wdist_axis(g[1], cy)), wdist_axis(g[2], cz));
        if (s2 >= 1.0) continue;
        const double w = __dsub_rn(1.0, __dsqrt_rn(s2));
        if (!(w > 0.0)) continue;
        rank = (local ? rpre[lw] : __ldcg(pre + (key >> 5))) + __popc(word & (bit - 1));
        unsigned long long* acc = reinterpret_cast<unsigned long long*>(L.acc) + 4 * (acc0 + rank);
        atomicAdd(acc, (unsigned long long)__double2ll_rn(__dmul_rn(w, kWScale)));
#pragma unroll
        for (int k = 0; k < 3; ++k)
          if (col[k] != 0.0) atomicAdd(acc + 1 + k, (unsigned long long)__double2ll_rn(__dmul_rn(__dmul_rn(w, col[k]), kWScale)));
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K4: finalize every voxel of the level
// ---------------------------------------------------------------------------
// Colour of the sample with node ordinal `ord`: octant o = the child holding it, index =
// ord - cbase[o] in the child's stored order (leaf: stash; inner: arena, or the stored-order
// copy for first-come).
__device__ __forceinline__ uint32_t winner_rgb(const VoxLevel& L, const VoxNode& nd, uint32_t ord) {
  int oo = 7;
  while (oo > 0 && (nd.ccount[oo] == 0 || nd.cbase[oo] > ord)) --oo;
  const uint64_t at = nd.cfirst[oo] + (ord - nd.cbase[oo]);
  if (nd.cslot[oo] == -1) return __ldg(&L.stash[at].y);
  return __ldg(L.mode == LOD_MODE_FIRST_COME ? &L.vout[at].y : &L.vox[at].y);
}

// Colour of voxel `r` of node `nd` from its accumulator (every sample was pushed by K3):
// writes the record's colour (and, first-come, the winning ordinal).
__device__ __forceinline__ void finalize_voxel(const VoxLevel& L, const VoxNode& nd, uint64_t acc0, uint32_t key,
                                               uint32_t r) {
  if (L.mode == LOD_MODE_WEIGHTED) {
    const unsigned long long* a = reinterpret_cast<const unsigned long long*>(L.acc) + 4 * (acc0 + r);
    const double W = (double)__ldcg(a);
    uint32_t rgb = 0;
    if (!(W > 0.0)) raise_err(L.st, ERR_ZERO_WEIGHT, nd.node);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double m = floor(__dadd_rn(__ddiv_rn((double)__ldcg(a + 1 + k), W), 0.5));
      rgb |= (uint32_t)fmin(fmax(m, 0.0), 255.0) << (8 * k);
    }
    L.vox[nd.vbase + r] = make_uint2(key, rgb);
    return;
  }
  uint64_t sr = 0, sg = 0, sb = 0, n = 0;
  uint32_t rgb;
  if (L.mode == LOD_MODE_AVERAGE) {
    if (L.exact_sums) {
      const ulonglong2* a = reinterpret_cast<const ulonglong2*>(L.acc) + 2 * (acc0 + r);
      const ulonglong2 a0 = __ldcg(a), a1 = __ldcg(a + 1);
      sr += a0.x, sg += a0.y, sb += a1.x, n += a1.y;
    } else {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(L.acc) + acc0 + r);
      if (fmaxf(fmaxf(a.x, a.y), fmaxf(a.z, a.w)) >= 16777216.0f) raise_err(L.st, ERR_F32_SUMS, nd.node);
      sr += (uint64_t)a.x, sg += (uint64_t)a.y, sb += (uint64_t)a.z, n += (uint64_t)a.w;
    }
    rgb = mean_round(sr, n) | (mean_round(sg, n) << 8) | (mean_round(sb, n) << 16);
  } else if (L.mode == LOD_MODE_RANDOM) {
    const uint32_t e = __ldcg(reinterpret_cast<const uint32_t*>(L.acc) + acc0 + r);
    rgb = winner_rgb(L, nd, e & 0xFFFFFu);  // the winning ordinal names the sample
  } else {
    uint32_t* a = reinterpret_cast<uint32_t*>(L.acc) + acc0 + r;
    const uint32_t ord = ~__ldcg(a);
    rgb = winner_rgb(L, nd, ord);
    *a = ord;  // winning ordinal, ranked by K5 through the node's ordinal bitmap
    atomicOr(L.obits + 2 * (nd.obase + (ord >> 5)), 1u << (ord & 31));
  }
  L.vox[nd.vbase + r] = make_uint2(key, rgb);  // the whole record: no half-written sectors
}

// K4: finalize every voxel of the level, one thread per voxel (rank chunks): a word-walk
// per block serialised each thread's gathers and ran 5x slower (measured).
__global__ void __launch_bounds__(kT) k_finalize(VoxLevel L) {
  pdl_wait();
  if (L.st->err & ERR_ARENA) return;
  const uint32_t nch = L.counters[2];
  for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const uint2 ch = L.vchunks[c];
    const VoxNode& nd = L.info[ch.x];
    const uint32_t r1 = min(nd.m, ch.y + L.vchunk);
    const uint64_t acc0 = nd.vbase - L.level_start[0];
    for (uint32_t r = ch.y + threadIdx.x; r < r1; r += kT) finalize_voxel(L, nd, acc0, __ldcg(&L.vox[nd.vbase + r].x), r);
  }
}

// ---------------------------------------------------------------------------
// K5 (first-come): stored order = ascending winning ordinal (sampling.py:64-66)
// ---------------------------------------------------------------------------
struct OrdScanF {  // exclusive popcount prefix over the level's ordinal bitmaps (packed pairs)
  uint32_t* bp;
  const uint32_t* live;  // words in use this level (K2's allocation)
  __device__ uint64_t limit(uint64_t n) const { return min(n, (uint64_t)__ldcg(live)); }
  __device__ uint64_t value(uint64_t i) const { return __popc(__ldcg(bp + 2 * i)); }
  __device__ void store(uint64_t i, uint64_t excl, uint64_t) const { bp[2 * i + 1] = (uint32_t)excl; }
};

__global__ void __launch_bounds__(kT) k_fc_pos(VoxLevel L) {
  pdl_wait();
  if (L.st->err & ERR_ARENA) return;
  const uint32_t nch = L.counters[2];
  for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const uint2 ch = L.vchunks[c];
    const VoxNode& nd = L.info[ch.x];
    const uint32_t r1 = min(nd.m, ch.y + L.vchunk);
    const uint64_t acc0 = nd.vbase - L.level_start[0];
    const uint32_t p0 = __ldcg(L.obits + 2 * nd.obase + 1);
    for (uint32_t r = ch.y + threadIdx.x; r < r1; r += kT) {
      const uint32_t ord = __ldcg(reinterpret_cast<const uint32_t*>(L.acc) + acc0 + r);
      const uint2 e = __ldcg(reinterpret_cast<const uint2*>(L.obits) + nd.obase + (ord >> 5));  // {bits, prefix}
      const uint32_t p = e.y - p0 + __popc(e.x & ((1u << (ord & 31)) - 1));
      L.vpos[nd.vbase + r] = p;
      L.vout[nd.vbase + p] = L.vox[nd.vbase + r];
    }
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// Import path (multi-GPU, rank 0): inner nodes whose voxels were computed on another GPU.
// Their rank structures (bitmap + prefix) are rebuilt from the voxel keys in slots
// [slot_base, slot_base + list_n) of the level's parity buffer, so the next level up can
// gather from them exactly like from locally voxelized children.
// ---------------------------------------------------------------------------
__global__ void k_import_setup(VoxLevel L, uint32_t slot_base) {
  pdl_wait();
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.list_n) return;
  const uint32_t node = L.list[i], s = slot_base + i;
  VoxNode info{};
  info.node = node;
  info.vbase = L.n_first[node];
  info.m = L.n_count[node];
  L.info[s] = info;
  L.node_slot[node] = s;
}

__global__ void __launch_bounds__(kT) k_import_bits(VoxLevel L, uint32_t slot_base) {
  pdl_wait();
  const uint32_t i = blockIdx.x / kBlksPerNode, part = blockIdx.x % kBlksPerNode;
  const VoxNode& nd = L.info[slot_base + i];
  uint32_t* bits = bits_of(L, L.parity, slot_base + i);
  const uint32_t per = (nd.m + kBlksPerNode - 1) / kBlksPerNode;
  const uint32_t r0 = part * per, r1 = min(nd.m, r0 + per);
  for (uint32_t r = r0 + threadIdx.x; r < r1; r += kT) {
    const uint32_t key = __ldg(&L.vox[nd.vbase + r].x);
    atomicOr(bits + (key >> 5), 1u << (key & 31));
  }
}

__global__ void __launch_bounds__(kT) k_import_block_sums(VoxLevel L, uint32_t slot_base) {
  pdl_wait();
  const uint32_t s = slot_base + blockIdx.x / kBlksPerNode, blk = blockIdx.x % kBlksPerNode;
  __shared__ uint32_t red[kT / 32];
  const uint4* b = reinterpret_cast<const uint4*>(bits_of(L, L.parity, s) + blk * kBlkWords);
  uint32_t c = 0;
  for (uint32_t i = threadIdx.x; i < kBlkWords / 4; i += kT) {
    uint4 q = __ldcg(b + i);
    c += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kT / 32; ++w) t += red[w];
    L.blk_sum[blockIdx.x] = t;
  }
}

__global__ void k_import_block_prefix(VoxLevel L) {
  pdl_wait();
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.list_n) return;
  uint32_t run = 0;
  for (uint32_t b = 0; b < kBlksPerNode; ++b) {
    uint32_t v = L.blk_sum[i * kBlksPerNode + b];
    L.blk_sum[i * kBlksPerNode + b] = run;
    run += v;
  }
}

__global__ void __launch_bounds__(kT) k_import_prefix(VoxLevel L, uint32_t slot_base) {
  pdl_wait();
  const uint32_t s = slot_base + blockIdx.x / kBlksPerNode, blk = blockIdx.x % kBlksPerNode;
  __shared__ uint32_t sm[kT / 32 + 1];
  const uint32_t* bits = bits_of(L, L.parity, s) + blk * kBlkWords;
  uint32_t* pre = pre_of(L, L.parity, s) + blk * kBlkWords;
  constexpr uint32_t per = kBlkWords / kT;
  uint32_t w[per], c = 0;
#pragma unroll
  for (uint32_t q = 0; q < per; ++q) c += __popc(w[q] = __ldcg(bits + threadIdx.x * per + q));
  uint32_t tot;
  uint32_t r = block_excl_scan<uint32_t, kT>(c, &tot, sm) + L.blk_sum[blockIdx.x];
#pragma unroll
  for (uint32_t q = 0; q < per; ++q) {
    pre[threadIdx.x * per + q] = r;
    r += __popc(w[q]);
  }
}

// first-come imports arrive in stored order (in vout): put the arena in key order and
// record each voxel's stored position for the parent's gather
__global__ void __launch_bounds__(kT) k_import_fc(VoxLevel L, uint32_t slot_base) {
  pdl_wait();
  const uint32_t i = blockIdx.x / kBlksPerNode, part = blockIdx.x % kBlksPerNode;
  const VoxNode& nd = L.info[slot_base + i];
  const uint32_t* bits = bits_of(L, L.parity, slot_base + i);
  const uint32_t* pre = pre_of(L, L.parity, slot_base + i);
  const uint32_t per = (nd.m + kBlksPerNode - 1) / kBlksPerNode;
  const uint32_t p0 = part * per, p1 = min(nd.m, p0 + per);
  for (uint32_t p = p0 + threadIdx.x; p < p1; p += kT) {
    const uint2 v = __ldg(L.vout + nd.vbase + p);
    const uint32_t r = rank_of(bits, pre, v.x);
    L.vox[nd.vbase + r] = v;
    L.vpos[nd.vbase + r] = p;
  }
}

int launch_voxelize_import(const VoxLevel& L, uint32_t slot_base, cudaStream_t s) {
  if (!L.list_n) return 0;
  launch_pdl(k_import_setup, ceil_div_u32(L.list_n, kT), kT, 0, s, L, slot_base);
  launch_pdl(k_import_bits, L.list_n * kBlksPerNode, kT, 0, s, L, slot_base);
  launch_pdl(k_import_block_sums, L.list_n * kBlksPerNode, kT, 0, s, L, slot_base);
  launch_pdl(k_import_block_prefix, ceil_div_u32(L.list_n, kT), kT, 0, s, L);
  launch_pdl(k_import_prefix, L.list_n * kBlksPerNode, kT, 0, s, L, slot_base);
  if (L.mode != LOD_MODE_FIRST_COME) return 5;
  launch_pdl(k_import_fc, L.list_n * kBlksPerNode, kT, 0, s, L, slot_base);
  return 6;
}

// One depth level in two halves.  front (stream s): setup, occupancy, allocation, rank
// structures, accumulation -- counters[0..6] must be zero on entry and the level's bitmaps
// cleared, and the child level's colours must be final before K3 (the caller orders it).
// back (its own stream): K4 finalize (+ first-come K5).  The back half of level L overlaps the
// front half of level L+1 up to its K3: the accumulators and K4 chunk lists alternate by depth
// parity, every other buffer they share is written by one and not read by the other.
int launch_voxelize_front(const VoxLevel& L, int sms, cudaStream_t s) {
  launch_pdl(k_setup, ceil_div_u32(8ull * L.list_n, kT), kT, 0, s, L);
  if (L.fmt == LOD_POINTS_F32)
    launch_pdl(k_occupy<LOD_POINTS_F32>, sms * 2, kRT, 0, s, L);
  else
    launch_pdl(k_occupy<LOD_POINTS_F64>, sms * 2, kRT, 0, s, L);
  launch_pdl(k_block_sums, L.list_n * kBlksPerNode, kT, 0, s, L);  // + the arena allocation (last block)
  launch_pdl(k_prefix, L.list_n * kBlksPerNode, kT, 0, s, L);
  return 4;
}

int launch_voxelize_accumulate(const VoxLevel& L, int sms, cudaStream_t s) {
  if (L.mode == LOD_MODE_WEIGHTED)
    launch_pdl(k_scatter_w, sms * 2, kRT, 2 * kRegionWords * 4, s, L);
  else
    launch_pdl(k_scatter, sms * 2, kRT, 2 * kRegionWords * 4, s, L);
  return 1;
}

int launch_voxelize_back(const VoxLevel& L, int sms, ScanScratch& scr, cudaStream_t s) {
  const int grid = sms * 8;
  int launches = 1;
  if (L.mode == LOD_MODE_FIRST_COME) cudaMemsetAsync(L.obits, 0, L.ocap * 8, s);  // K4 marks winners
  launch_pdl(k_finalize, grid, kT, 0, s, L);
  if (L.mode == LOD_MODE_FIRST_COME) {
    const int r = device_scan(L.ocap, OrdScanF{L.obits, L.counters + 4}, scr, nullptr, nullptr, s);
    if (r < 0) return r;
    launch_pdl(k_fc_pos, grid, kT, 0, s, L);
    launches += 1 + r;
  }
  return launches;
}

uint32_t voxelize_acc_bytes(int mode, bool exact_sums) {
  return mode == LOD_MODE_AVERAGE ? (exact_sums ? 32 : 16) : mode == LOD_MODE_WEIGHTED ? 32 : 4;
}

// chunk sizes: small levels get small chunks so every SM has work
uint32_t voxelize_chunk(uint32_t nodes) { return nodes <= 8 ? 4096 : 16384; }
uint32_t voxelize_vchunk(uint32_t nodes) { return nodes <= 8 ? 128 : nodes <= 64 ? 512 : kVoxChunk; }
uint64_t voxelize_chunk_capacity(uint64_t samples, uint32_t nodes) { return samples / 4096 + 8ull * nodes + 16; }
uint64_t voxelize_vchunk_capacity(uint64_t voxels, uint32_t nodes) { return voxels / 128 + nodes + 16; }

}  // namespace lod
