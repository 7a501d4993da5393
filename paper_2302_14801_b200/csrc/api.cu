// C ABI + host orchestration of one LOD build (include/lodb200.h).
//
// The host side only sequences launches and reads a handful of scalars back; all
// per-point and per-cell work is on the device.  Synchronisation points per build:
//   1. after counting (+1 per extension round)   -> extension grids to create
//   2. after node enumeration                    -> node-table size
//   3. after leaf numbering                      -> leaf count, per-depth inner lists
//   4. end of distribute / end of voxelize       -> error flags
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.h"

namespace lod {

static thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int fail_cuda(cudaError_t e, const char* what) {
  return fail(LOD_ECUDA, "CUDA error %s (%s) at %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
}

// Device memory: cudaMalloc, or the caller's allocator (lod_set_allocator) so that e.g.
// torch's caching allocator accounts for the trees' buffers.  A buffer remembers which
// allocator made it.
static lod_alloc_fn g_alloc = nullptr;
static lod_free_fn g_free = nullptr;
static void* g_alloc_ctx = nullptr;

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  bool ext = false;  // from the caller's allocator
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

static void release(DevBuf& b) {
  if (!b.p) return;
  if (b.ext) {
    int d = 0;
    cudaGetDevice(&d);
    cudaDeviceSynchronize();  // the library's streams may still use it; the caller's pool reuses at once
    g_free(b.p, b.cap, d, g_alloc_ctx);
  } else {
    cudaFree(b.p);
  }
  b.p = nullptr;
  b.cap = 0;
  b.ext = false;
}

static size_t round_up(size_t b) { return (b + (2u << 20) - 1) & ~(size_t)((2u << 20) - 1); }

// grow-only; keep_bytes of the old contents are preserved when growing
static cudaError_t ensure(DevBuf& b, size_t bytes, size_t keep_bytes = 0, cudaStream_t s = 0) {
  if (bytes <= b.cap) return cudaSuccess;
  void* np = nullptr;
  size_t cap = round_up(bytes);
  const bool ext = g_alloc != nullptr;
  if (ext) {
    int d = 0;
    cudaGetDevice(&d);
    np = g_alloc(cap, d, g_alloc_ctx);
    if (!np) return cudaErrorMemoryAllocation;
  } else {
    cudaError_t e = cudaMalloc(&np, cap);
    if (e != cudaSuccess) return e;
  }
  if (b.p) {
    if (keep_bytes) {
      cudaError_t e = cudaMemcpyAsync(np, b.p, keep_bytes, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return e;
      cudaStreamSynchronize(s);
    }
    release(b);
  }
  b.p = np;
  b.cap = cap;
  b.ext = ext;
  return cudaSuccess;
}

struct Round {
  uint32_t first, count;
  int ext, base;
  uint64_t pyr_base, tgt_base;
};

}  // namespace lod

using namespace lod;

struct lod_tree {
  int device = 0;
  int fmt = LOD_POINTS_F32;
  uint64_t n = 0;
  lod_config cfg{};
  bool split_done = false;
  int voxel_mode = -1;
  uint64_t n_voxels = 0;
  uint64_t launches = 0;
  bool timing = false;
  cudaEvent_t ev[6] = {};
  cudaEvent_t kev[4] = {};  // the distribute's K_scatter, per pass (the dominant single kernel)
  // voxelize runs each level on three streams: front (K0-K2b) on vfront, K3 on the caller's
  // stream, back (K4/K5) on vback -- so level L+1's front overlaps level L's K3 and K4
  cudaStream_t vfront = nullptr, vback = nullptr;
  cudaEvent_t vev[6] = {};  // fork/join, front done, K3 done, back done (x2: depth parity), spare
  cudaStream_t cstream = nullptr;  // second copy engine for large host copies (copy_split)
  cudaEvent_t cev[2] = {};
  float stage_ms[5] = {};

  DevBuf state, pyr, node_idx, t8, te, meta, list, scan, slots;
  DevBuf n_cell, n_val, n_parent, n_child, n_slot, n_extid, n_lvl, n_leaf, n_box, n_first, n_count;
  DevBuf leaf_node, leaf_first, leaf_count, leaf_pbox, leaf_pinv, depth_count, depth_off, depth_cursor, depth_lists;
  DevBuf leaf_pts, status, digit_base, tmp_rec, tmp_leaf, pkey, elist, abits;
  DevBuf sgrid, cand_keys;  // candidate path of the single-GPU split (k_cand_sample)
  bool cand = false;
  uint64_t elist_cap = 0;
  cudaEvent_t out_wait = nullptr;  // lod_tree_set_output_wait (next split only)
  bool use_abits = false;
  DevBuf vox, export_buf, stash;
  DevBuf vbits, vpre, vinfo, vblk, vcount, vlevel_start, node_slot, vacc, vchunks, vvchunks;
  DevBuf vpos, vout, obits;  // first-come: stored positions, stored-order voxels, ordinal bitmaps
  // pinned, device-mapped mirror of the device state (+ the per-depth counts): the build's
  // small device<->host exchanges are done by kernels over mapped memory, never by the copy
  // engines, so they do not queue behind bulk uploads / downloads of other streams (a
  // pipelined caller's 400-MB tree download held every build back by its full length)
  DevState* host_state = nullptr;
  DevState* host_state_dev = nullptr;
  uint32_t* host_depth = nullptr;  // [kMaxDepth + 2]: inner nodes per depth, deepest used
  uint32_t* host_depth_dev = nullptr;

  uint32_t n_nodes = 0, n_leaves = 0, n_ext = 0, max_depth_used = 0;
  uint32_t inner_per_depth[kMaxDepth + 1] = {};
  uint32_t inner_off[kMaxDepth + 1] = {};
  std::vector<Round> rounds;
  uint64_t total_slots = 0;
  double world[4] = {};
  double inv_world = 0;
  RadixPlan plan{};
  // split phase state
  const void* pts = nullptr;
  uint64_t n_global = 0;
  uint64_t ext_pyr_used = 0, ext_tgt_used = 0;
  uint32_t round_cur = 0, round_first = 0, round_parent_first = 0;
  int round_base = 0;
  bool dist = false;
  DevBuf local_main, local_ext;   // multi-GPU: this process's counts before the all-reduce
  DevBuf plan_lists, seg;
  int dist_stage = 0;
};

namespace {

// word copies by one CTA: device -> mapped host memory (and small device-side sets)
__global__ void k_copy_words(uint32_t* dst, const uint32_t* src, uint32_t n) {
  pdl_wait();
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldcg(src + i);
}
__global__ void k_state_set(DevState* dst, DevState v) {
  pdl_wait();
  if (threadIdx.x == 0) *dst = v;
}
struct DepthWords {
  uint32_t v[kMaxDepth + 1];
};
__global__ void k_depth_set(uint32_t* dst, DepthWords w) {
  pdl_wait();
  if (threadIdx.x <= kMaxDepth) dst[threadIdx.x] = w.v[threadIdx.x];
}
__global__ void k_set_u64(uint64_t* dst, uint64_t v) {
  pdl_wait();
  *dst = v;
}

int read_state(lod_tree* t, cudaStream_t s) {
  static_assert(sizeof(DevState) % 4 == 0, "DevState is copied as words");
  launch_pdl(k_copy_words, 1, 64, 0, s, reinterpret_cast<uint32_t*>(t->host_state_dev),
             reinterpret_cast<const uint32_t*>(t->state.p), (uint32_t)(sizeof(DevState) / 4));
  LOD_CUDA_CHECK(cudaGetLastError());
  LOD_CUDA_CHECK(cudaStreamSynchronize(s));
  return LOD_OK;
}

// Every entry point runs on the tree's device and gives the caller's current device back
// (the ABI must not change torch's current device for the calling thread).
struct DeviceGuard {
  int prev = -1;
  cudaError_t status;
  explicit DeviceGuard(int d) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    status = cudaSetDevice(d);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

std::string path_of(uint64_t cell) {
  uint32_t cx = (uint32_t)cell & 0xFFFF, cy = (uint32_t)(cell >> 16) & 0xFFFF, cz = (uint32_t)(cell >> 32) & 0xFFFF;
  int depth = (int)(cell >> 48) & 0xFF;
  std::string p = "(";
  for (int b = depth - 1; b >= 0; --b) {
    int o = ((cx >> b) & 1) | (((cy >> b) & 1) << 1) | (((cz >> b) & 1) << 2);
    p += std::to_string(o);
    if (b > 0 || depth == 1) p += depth == 1 ? "," : ", ";
  }
  return p + ")";
}

// Map device error bits to the reference's exceptions (messages as in the reference).
int check_errors(lod_tree* t, cudaStream_t s) {
  const DevState& h = *t->host_state;
  uint32_t e = h.err;
  if (!e) return LOD_OK;
  auto node_path = [&](uint32_t k) -> std::string {
    uint64_t cell = 0;
    if (t->n_cell.p && k < t->n_nodes)
      cudaMemcpy(&cell, t->n_cell.as<uint64_t>() + k, 8, cudaMemcpyDeviceToHost);
    return path_of(cell);
  };
  (void)s;
  if (e & ERR_NONFINITE) return fail(LOD_EVALUE, "point coordinates must be finite");
  if (e & ERR_OUTSIDE) return fail(LOD_ECONSISTENCY, "point outside bounds during grid projection");
  if (e & ERR_EXT_ROOT) return fail(LOD_ECONSISTENCY, "extended pyramid root must be unmergeable");
  if (e & ERR_OVERSIZED) return fail(LOD_ECONSISTENCY, "oversized leaf away from max depth");
  if (e & ERR_NO_ROOT) return fail(LOD_ECONSISTENCY, "partition produced no root node");
  if (e & ERR_NO_PARENT)
    return fail(LOD_ECONSISTENCY, "node %s has no inner parent", node_path(h.err_detail).c_str());
  if (e & ERR_UNRESOLVED) return fail(LOD_ECONSISTENCY, "point did not resolve to a leaf node");
  if (e & ERR_COUNT) return fail(LOD_ECONSISTENCY, "leaf received a different count than allocated");
  if (e & ERR_RANDOM_LIMIT) {
    // The reference raises at the first offending node in (depth desc, DFS preorder) order
    // (sampling.py:171-173); levels run deepest first, so the first raise fixed the depth.
    // Pick the DFS-first offender at that depth from the node table.
    std::vector<uint64_t> cell(t->n_nodes);
    std::vector<uint32_t> val(t->n_nodes), cnt(t->n_nodes);
    std::vector<int32_t> child(8ull * t->n_nodes);
    cudaMemcpy(cell.data(), t->n_cell.p, 8ull * t->n_nodes, cudaMemcpyDeviceToHost);
    cudaMemcpy(val.data(), t->n_val.p, 4ull * t->n_nodes, cudaMemcpyDeviceToHost);
    cudaMemcpy(cnt.data(), t->n_count.p, 4ull * t->n_nodes, cudaMemcpyDeviceToHost);
    cudaMemcpy(child.data(), t->n_child.p, 32ull * t->n_nodes, cudaMemcpyDeviceToHost);
    int d0 = (int)(cell[h.err_detail] >> 48) & 0xFF;
    uint64_t best_code = ~0ull, best_s = h.err_value;
    for (uint32_t k = 0; k < t->n_nodes; ++k) {
      if (val[k] != UNMERGEABLE || (int)((cell[k] >> 48) & 0xFF) != d0) continue;
      uint64_t S = 0;
      for (int o = 0; o < 8; ++o)
        if (child[8ull * k + o] >= 0) S += cnt[child[8ull * k + o]];
      if (S < (uint64_t)kRandomLimit) continue;
      uint32_t cx = (uint32_t)cell[k] & 0xFFFF, cy = (uint32_t)(cell[k] >> 16) & 0xFFFF,
               cz = (uint32_t)(cell[k] >> 32) & 0xFFFF;
      uint64_t code = 0;
      for (int b = d0 - 1; b >= 0; --b)
        code = code * 8 + (((cx >> b) & 1) | (((cy >> b) & 1) << 1) | (((cz >> b) & 1) << 2));
      if (code < best_code) best_code = code, best_s = S;
    }
    return fail(LOD_ECONSISTENCY, "%llu samples exceed the 20-bit index limit of random sampling",
                (unsigned long long)best_s);
  }
  if (e & ERR_EMPTY_CHILD)  // f"child {child.path} has no samples" (sampling.py:35)
    return fail(LOD_ECONSISTENCY, "child %s has no samples", node_path(h.err_detail).c_str());
  if (e & ERR_ZERO_WEIGHT) return fail(LOD_ECONSISTENCY, "occupied cell accumulated zero weight");
  return fail(LOD_ECONSISTENCY, "device error 0x%x", e);
}

SplitView make_view(lod_tree* t, const void* pts) {
  SplitView v{};
  v.st = t->state.as<DevState>();
  v.pts = pts;
  v.n = t->n;
  v.D = t->cfg.initial_depth;
  v.max_depth = t->cfg.max_depth;
  v.T = t->cfg.T;
  v.pyr = t->pyr.as<uint32_t>();
  v.main_cells = level_off(v.D + 1);
  v.node_idx = t->node_idx.as<int32_t>();
  v.t8 = t->t8.as<int32_t>();
  v.pkey = t->pkey.as<uint32_t>();
  v.elist = t->elist_cap ? t->elist.as<uint4>() : nullptr;
  v.elist_cap = t->elist_cap;
  v.abits = t->use_abits ? t->abits.as<uint32_t>() : nullptr;
  v.te = t->te.as<int32_t>();
  if (t->cand) {
    v.sgrid = t->sgrid.as<uint32_t>();
    v.cand_keys = t->cand_keys.as<uint32_t>();
    v.cand = t->tmp_rec.as<uint4>();
    v.cand_cap = t->tmp_rec.cap / 16;
    // 0.85 of the samples a cell of T points gets (~3 sigma below it at T = 50k): fewer
    // false candidates; an anchor below it is caught by k_cand_check (full-scan fallback)
    v.cand_thresh = std::max<uint32_t>(1, (uint32_t)(0.85 * (double)t->cfg.T / kCandStride));
  }
  v.meta = t->meta.as<ExtMeta>();
  v.n_ext = t->n_ext;
  v.n_cell = t->n_cell.as<uint64_t>();
  v.n_val = t->n_val.as<uint32_t>();
  v.n_parent = t->n_parent.as<int32_t>();
  v.n_child = t->n_child.as<int32_t>();
  v.n_slot = t->n_slot.as<uint64_t>();
  v.n_extid = t->n_extid.as<int32_t>();
  v.n_lvl = t->n_lvl.as<uint8_t>();
  v.n_leaf = t->n_leaf.as<int32_t>();
  v.n_box = t->n_box.as<double4>();
  v.n_first = t->n_first.as<uint64_t>();
  v.n_count = t->n_count.as<uint32_t>();
  v.n_nodes = t->n_nodes;
  v.leaf_node = t->leaf_node.as<uint32_t>();
  v.leaf_first = t->leaf_first.as<uint64_t>();
  v.leaf_count = t->leaf_count.as<uint32_t>();
  v.leaf_pbox = t->leaf_pbox.as<double4>();
  v.leaf_pinv = t->leaf_pinv.as<double>();
  v.n_leaves = t->n_leaves;
  return v;
}

int ceil_log2(uint64_t x) {
  int b = 0;
  while ((1ull << b) < x) ++b;
  return b;
}

#define CK(expr) LOD_CUDA_CHECK(expr)
#define RUN(expr)            \
  do {                       \
    int _r = (expr);         \
    if (_r < 0) return fail(LOD_ECUDA, "internal scratch too small: %s", #expr); \
    t->launches += _r;       \
  } while (0)

#define RUN_NOTREE(expr)     \
  do {                       \
    if ((expr) < 0) return fail(LOD_ECUDA, "internal scratch too small: %s", #expr); \
  } while (0)

constexpr uint32_t kThreads_count() { return 256; }  // K_count's block (split_kernels.cu kThreads)
// LODB200_NO_CAND=1 turns the candidate list off (A/B and a fallback switch)
// below 2^27 points the sample + candidate compaction (~50 us) outweighs what it saves;
// LODB200_CAND_MIN_N overrides (tests run the golden cases through both extension paths)
uint64_t cand_min_points() {
  const char* e = getenv("LODB200_CAND_MIN_N");
  return e ? strtoull(e, nullptr, 10) : (1ull << 27);
}
bool cand_enabled() {
  static const bool on = [] {
    const char* e = getenv("LODB200_NO_CAND");
    return !(e && e[0] == '1');
  }();
  return on;
}

void mark(lod_tree* t, int i, cudaStream_t s) {
  if (t->timing) cudaEventRecord(t->ev[i], s);
}

// ---------------------------------------------------------------------------
// split phases.  Single GPU: init, bounds, count, [anchors, {round, subanchors}*],
// skeleton, distribute.  Multi-GPU (dist.py) calls the same phases with collectives in
// between (world bounds, counting grids and extension grids are all-reduced).
// ---------------------------------------------------------------------------
int phase_init(lod_tree* t, const void* pts, uint64_t n, int fmt, const double* ub, const lod_config* cfg,
               cudaStream_t s) {
  if (!t) return fail(LOD_EVALUE, "null tree");
  if (!cfg) return fail(LOD_EVALUE, "null config");
  if (n == 0 && !t->dist) return fail(LOD_EVALUE, "cannot partition an empty point cloud");
  if (cfg->T < 1) return fail(LOD_EVALUE, "T must be >= 1");
  if (cfg->max_depth < cfg->initial_depth) return fail(LOD_EVALUE, "max_depth must be >= initial_depth");
  if (cfg->max_depth > kMaxDepth) return fail(LOD_EVALUE, "max_depth must be <= %d", kMaxDepth);
  if (cfg->initial_depth < 0 || cfg->initial_depth > 10)
    return fail(LOD_EUNSUPPORTED, "initial_depth must be in [0, 10] on the GPU path");
  if (cfg->extension_depth < 1 || cfg->extension_depth > 5)
    return fail(LOD_EUNSUPPORTED, "extension_depth must be in [1, 5] on the GPU path");
  if (fmt != LOD_POINTS_F32 && fmt != LOD_POINTS_F64) return fail(LOD_EVALUE, "unknown point format %d", fmt);
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  // a build that ended early (error path) may have left work on the tree's side streams
  CK(cudaEventRecord(t->vev[4], t->vfront));
  CK(cudaStreamWaitEvent(s, t->vev[4], 0));
  CK(cudaEventRecord(t->vev[5], t->vback));
  CK(cudaStreamWaitEvent(s, t->vev[5], 0));
  if (n >= 0xFFFFFFFFull) return fail(LOD_EUNSUPPORTED, "at most 2^32 - 2 points per GPU build");
  if (ub && !(ub[3] > 0)) return fail(LOD_EVALUE, "AABB size must be positive");
  t->split_done = false;
  t->voxel_mode = -1;
  t->n_voxels = 0;
  t->launches = 0;
  t->n = n;
  t->pts = pts;
  t->fmt = fmt;
  t->cfg = *cfg;
  t->n_ext = 0;
  t->n_nodes = t->n_leaves = 0;
  t->rounds.clear();
  t->elist_cap = 0;
  t->use_abits = false;
  t->cand = false;
  t->ext_pyr_used = t->ext_tgt_used = 0;
  t->round_cur = 0;
  const int D = cfg->initial_depth;
  const uint64_t main_cells = level_off(D + 1);
  const uint64_t fine_cells = 1ull << (3 * D);
  mark(t, 0, s);
  DevState init{};
  for (int a = 0; a < 3; ++a) init.lo_key[a] = ~0ull, init.hi_key[a] = 0;
  *t->host_state = init;
  CK(ensure(t->state, sizeof(DevState)));
  launch_pdl(k_state_set, 1, 32, 0, s, t->state.as<DevState>(), init);
  CK(ensure(t->pyr, main_cells * 4));
  CK(cudaMemsetAsync(t->pyr.p, 0, main_cells * 4, s));
  CK(ensure(t->t8, fine_cells * 4));
  CK(cudaMemsetAsync(t->t8.p, 0xFF, fine_cells * 4, s));
  CK(ensure(t->pkey, std::max<uint64_t>(n, 1) * 4));
  uint64_t scan_blocks = (std::max<uint64_t>(main_cells, n) + kScanTile - 1) / kScanTile + 2;
  CK(ensure(t->scan, scan_blocks * 8));
  return LOD_OK;
}

int phase_bounds(lod_tree* t, const double* ub, cudaStream_t s) {
  SplitView v = make_view(t, t->pts);
  if (t->n == 0 && !ub) return LOD_OK;  // empty shard: identity min/max keys
  RUN(launch_bounds(t->fmt, t->pts, t->n, v.st, ub, s));
  return LOD_OK;
}

int phase_count(lod_tree* t, cudaStream_t s) {
  if (t->cand) {  // sampled count -> candidate cells; K_count lists their points (tmp_rec)
    const uint64_t fine_cells = 1ull << (3 * t->cfg.initial_depth);
    CK(ensure(t->sgrid, fine_cells * 4));
    CK(cudaMemsetAsync(t->sgrid.p, 0, fine_cells * 4, s));
    CK(ensure(t->cand_keys, kCandCap * 4));
    const uint64_t slack = (uint64_t)count_blocks(t->n) * (kThreads_count() / 32) * kCandChunk + kCandChunk;
    CK(ensure(t->tmp_rec, (t->n + slack) * 16));
    SplitView v = make_view(t, t->pts);
    ScanScratch scr{t->scan.as<uint64_t>(), t->scan.cap / 8};
    RUN(launch_cand_sample(t->fmt, v, scr, s));
  }
  SplitView v = make_view(t, t->pts);
  if (t->n) RUN(launch_count(t->fmt, v, s));
  mark(t, 1, s);
  return LOD_OK;
}

// Anchors of the first extension round from the (global) main finest counts.
int phase_anchors(lod_tree* t, uint32_t* cur, cudaStream_t s) {
  *cur = 0;
  const int D = t->cfg.initial_depth;
  if (t->cfg.max_depth <= D) return LOD_OK;
  const uint64_t fine_cells = 1ull << (3 * D);
  uint64_t max_anchor = std::min<uint64_t>(fine_cells, t->n_global / ((uint64_t)t->cfg.T + 1) + 1);
  CK(ensure(t->list, max_anchor * 8 + 8));
  ScanScratch scr{t->scan.as<uint64_t>(), t->scan.cap / 8};
  SplitView v = make_view(t, t->pts);
  RUN(launch_find_anchors(v, t->list.as<uint64_t>(), scr, s, false));
  int r = read_state(t, s);
  if (r) return r;
  if ((r = check_errors(t, s))) return r;
  *cur = (uint32_t)t->host_state->count_a;
  if (*cur) RUN(launch_find_anchors(v, t->list.as<uint64_t>(), scr, s, true));  // none: no store pass
  if (*cur && t->cand) RUN(launch_cand_check(v, t->list.as<uint64_t>(), *cur, s));
  // anchor bitmap for the first extension round's membership test (2 MB at depth 8)
  t->use_abits = *cur && 3 * D <= 27;
  if (t->use_abits) {
    CK(ensure(t->abits, (fine_cells + 7) / 8));
    CK(cudaMemsetAsync(t->abits.p, 0, (fine_cells + 7) / 8, s));
  }
  t->round_base = D;
  t->round_first = 0;
  t->round_parent_first = 0;
  t->round_cur = *cur;
  return LOD_OK;
}

// Create the next extension round from t->list and count the local points into it.
int phase_round(lod_tree* t, cudaStream_t s) {
  const uint32_t cur = t->round_cur;
  const int base = t->round_base;
  const int ext = std::min(t->cfg.extension_depth, t->cfg.max_depth - base);
  const uint64_t main_cells = level_off(t->cfg.initial_depth + 1);
  const uint64_t psz = level_off(ext + 1), tsz = 1ull << (3 * ext);
  const uint64_t pyr_base = main_cells + t->ext_pyr_used, tgt_base = t->ext_tgt_used;
  const uint64_t new_pyr = (uint64_t)cur * psz, new_tgt = (uint64_t)cur * tsz;
  const uint32_t first = t->round_first;
  CK(ensure(t->pyr, (pyr_base + new_pyr) * 4, pyr_base * 4, s));
  CK(ensure(t->te, (tgt_base + new_tgt) * 4, tgt_base * 4, s));
  CK(ensure(t->meta, (size_t)(first + cur) * sizeof(ExtMeta), (size_t)first * sizeof(ExtMeta), s));
  CK(cudaMemsetAsync(t->pyr.as<uint32_t>() + pyr_base, 0, new_pyr * 4, s));
  CK(cudaMemsetAsync(t->te.as<int32_t>() + tgt_base, 0xFF, new_tgt * 4, s));
  SplitView v = make_view(t, t->pts);
  if (t->rounds.empty()) {
    // extension-list capacity: the points under the anchors (all-reduced counts in the
    // multi-GPU path: an upper bound of the local ones)
    DevState* st = t->state.as<DevState>();
    CK(cudaMemsetAsync(&st->ext_n, 0, sizeof(st->ext_n), s));
    RUN(launch_anchor_sum(v, t->list.as<uint64_t>(), cur, s));
    int r = read_state(t, s);
    if (r) return r;
    t->elist_cap = std::min<uint64_t>(t->n, t->host_state->ext_n);
    CK(ensure(t->elist, std::max<uint64_t>(t->elist_cap, 1) * 16));
    CK(cudaMemsetAsync(&st->ext_n, 0, sizeof(st->ext_n), s));
  }
  RUN(launch_ext_create(v, (int)t->rounds.size(), first, cur, t->list.as<uint64_t>(), t->round_parent_first,
                        pyr_base, tgt_base, base, ext, s));
  t->n_ext = first + cur;
  v = make_view(t, t->pts);
  if (t->n) RUN(launch_ext_count(t->fmt, v, first, s));
  t->rounds.push_back(Round{first, cur, ext, base, pyr_base, tgt_base});
  t->ext_pyr_used += new_pyr;
  t->ext_tgt_used += new_tgt;
  return LOD_OK;
}

// After the last round's counts are final (all-reduced): the next round's anchors.
int phase_subanchors(lod_tree* t, uint32_t* next, cudaStream_t s) {
  *next = 0;
  const Round& rd = t->rounds.back();
  if (rd.base + rd.ext < t->cfg.max_depth) {
    const uint64_t tsz = 1ull << (3 * rd.ext);
    uint64_t cap_needed = std::min<uint64_t>((uint64_t)rd.count * tsz, t->n_global / ((uint64_t)t->cfg.T + 1) + 1);
    CK(ensure(t->list, cap_needed * 8 + 8));
    uint64_t sb = ((uint64_t)rd.count * tsz + kScanTile - 1) / kScanTile + 2;
    CK(ensure(t->scan, sb * 8));
    ScanScratch scr{t->scan.as<uint64_t>(), t->scan.cap / 8};
    SplitView v = make_view(t, t->pts);
    RUN(launch_find_subanchors(v, rd.first, rd.count, rd.ext, t->list.as<uint64_t>(), scr, s));
    int r = read_state(t, s);
    if (r) return r;
    *next = (uint32_t)t->host_state->count_a;
  }
  t->round_parent_first = rd.first;
  t->round_first = rd.first + rd.count;
  t->round_base = rd.base + rd.ext;
  t->round_cur = *next;
  return LOD_OK;
}

// merge + node table + targets + per-depth inner lists (partition.py:155-240)
int phase_skeleton(lod_tree* t, cudaStream_t s) {
  mark(t, 2, s);
  const int D = t->cfg.initial_depth;
  const uint64_t main_cells = level_off(D + 1);
  {
    std::vector<uint32_t> rf, rc;
    std::vector<int> re;
    std::vector<uint64_t> rb;
    for (auto& rd : t->rounds)
      rf.push_back(rd.first), rc.push_back(rd.count), re.push_back(rd.ext), rb.push_back(rd.pyr_base);
    SplitView v = make_view(t, t->pts);
    RUN(launch_merge_all(v, rf.data(), rc.data(), re.data(), rb.data(), (int)t->rounds.size(), s));
  }
  t->total_slots = main_cells + t->ext_pyr_used;
  uint64_t slot_cap = std::min<uint64_t>(t->total_slots, t->n_global * (uint64_t)(t->cfg.max_depth + 1) + 1);
  CK(ensure(t->slots, slot_cap * 8));
  CK(ensure(t->node_idx, t->total_slots * 4));
  uint64_t sb = (t->total_slots + kScanTile - 1) / kScanTile + 2;
  CK(ensure(t->scan, sb * 8));
  ScanScratch scr{t->scan.as<uint64_t>(), t->scan.cap / 8};
  SplitView v = make_view(t, t->pts);
  RUN(launch_count_nodes(v, t->total_slots, t->slots.as<uint64_t>(), scr, s));
  int r = read_state(t, s);
  if (r) return r;
  if ((r = check_errors(t, s))) return r;
  t->n_nodes = (uint32_t)t->host_state->count_b;
  if (t->n_nodes == 0) return fail(LOD_ECONSISTENCY, "partition produced no root node");
  const uint64_t nn = t->n_nodes;
  CK(ensure(t->n_cell, nn * 8));
  CK(ensure(t->n_val, nn * 4));
  CK(ensure(t->n_parent, nn * 4));
  CK(ensure(t->n_child, nn * 32));
  CK(ensure(t->n_slot, nn * 8));
  CK(ensure(t->n_extid, nn * 4));
  CK(ensure(t->n_lvl, nn));
  CK(ensure(t->n_leaf, nn * 4));
  CK(ensure(t->n_box, nn * 32));
  CK(ensure(t->n_first, nn * 8));
  CK(ensure(t->n_count, nn * 4));
  CK(ensure(t->leaf_node, nn * 4));
  CK(ensure(t->leaf_first, nn * 8));
  CK(ensure(t->leaf_count, nn * 4));
  CK(ensure(t->leaf_pbox, nn * 32));
  CK(ensure(t->leaf_pinv, nn * 8));
  CK(ensure(t->depth_count, 64 * 4));
  CK(cudaMemsetAsync(t->depth_count.p, 0, 64 * 4, s));
  v = make_view(t, t->pts);
  RUN(launch_build_nodes(v, t->slots.as<uint64_t>(), s));
  RUN(launch_number_leaves(v, scr, s));
  RUN(launch_depth_lists(v, t->depth_count.as<uint32_t>(), s));
  launch_pdl(k_copy_words, 1, 64, 0, s, t->host_depth_dev, t->depth_count.as<uint32_t>(), (uint32_t)(kMaxDepth + 2));
  // the targets (node_idx / t8 / te: a chain of per-level passes) only need the node table
  // and the leaf numbering: on the front stream, under this host round trip and the leaf
  // offsets / parent boxes / depth lists below, which touch none of those arrays
  CK(cudaEventRecord(t->vev[0], s));
  CK(cudaStreamWaitEvent(t->vfront, t->vev[0], 0));
  RUN(launch_targets(v, t->vfront));
  for (auto& rd : t->rounds) RUN(launch_targets_ext(v, rd.first, rd.count, rd.ext, t->vfront));
  CK(cudaEventRecord(t->vev[1], t->vfront));
  if ((r = read_state(t, s)) || (r = check_errors(t, s))) {
    cudaStreamWaitEvent(s, t->vev[1], 0);  // nothing of this build may outlive the call
    return r;
  }
  for (int d = 0; d <= kMaxDepth; ++d) t->inner_per_depth[d] = t->host_depth[d];
  t->max_depth_used = t->host_depth[kMaxDepth + 1];
  t->n_leaves = (uint32_t)t->host_state->count_a;
  v = make_view(t, t->pts);
  RUN(launch_leaf_offsets(v, scr, s));
  RUN(launch_leaf_parent_boxes(v, s));
  uint32_t off = 0;
  for (int d = 0; d <= kMaxDepth; ++d) t->inner_off[d] = off, off += t->inner_per_depth[d];
  CK(ensure(t->depth_lists, (size_t)std::max<uint32_t>(off, 1) * 4));
  CK(ensure(t->depth_off, 64 * 4));
  CK(ensure(t->depth_cursor, 64 * 4));
  {
    DepthWords w;
    for (int d = 0; d <= kMaxDepth; ++d) w.v[d] = t->inner_off[d];
    launch_pdl(k_depth_set, 1, 64, 0, s, t->depth_off.as<uint32_t>(), w);
  }
  CK(cudaMemsetAsync(t->depth_cursor.p, 0, 64 * 4, s));
  RUN(launch_depth_scatter(v, t->depth_off.as<uint32_t>(), t->depth_cursor.as<uint32_t>(),
                           t->depth_lists.as<uint32_t>(), s));
  CK(cudaStreamWaitEvent(s, t->vev[1], 0));  // join the targets
  for (int a = 0; a < 3; ++a) t->world[a] = t->host_state->lo[a];
  t->world[3] = t->host_state->size;
  t->inv_world = t->host_state->inv_size;
  mark(t, 3, s);
  return LOD_OK;
}

// Stable distribute of the local points into their leaves (partition.py:244-271).  Uses
// t->leaf_count (per leaf, this process's points) for the digit bases and offsets.
int phase_distribute(lod_tree* t, cudaStream_t s, bool sync = true) {
  const uint64_t n = t->n;
  const size_t rec = t->fmt == LOD_POINTS_F32 ? 16 : 32;
  CK(ensure(t->leaf_pts, std::max<uint64_t>(n, 1) * rec));
  RadixPlan& p = t->plan;
  int bits = ceil_log2(t->n_leaves);
  if (bits > 2 * kRadixMaxBits)
    return fail(LOD_EUNSUPPORTED, "%u leaves exceed the 2-pass distribute limit", t->n_leaves);
  p.passes = (t->n_nodes == 1 || n == 0) ? 0 : (bits <= kRadixMaxBits ? 1 : 2);
  p.bits[0] = bits;
  p.bits[1] = 0;
  if (p.passes == 2) {  // prefer a 2nd digit that fits the record pad (distribute.cu OUT_TAG)
    const int tagb = t->fmt == LOD_POINTS_F32 ? 8 : kRadixMaxBits;
    p.bits[1] = std::min(tagb, bits - bits / 2);
    p.bits[0] = bits - p.bits[1];
    if (p.bits[0] > kRadixMaxBits) p.bits[0] = bits / 2, p.bits[1] = bits - bits / 2;
  }
  if (p.passes) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, t->device);
    plan_segments(p, n, sms);
    const int maxb = std::max(p.bits[0], p.bits[1]);
    CK(ensure(t->status, (((size_t)p.segs + 1024) << maxb) * 4));
    CK(ensure(t->digit_base, (size_t)(2 << kRadixMaxBits) * 8 * 2));
    if (p.passes == 2) CK(ensure(t->tmp_rec, n * rec));
    CK(ensure(t->tmp_leaf, n * 4 * p.passes));  // leaf ids in input order (+ sorted by the 1st digit)
    for (int i = 0; i < 4; ++i) p.scatter_ev[i] = t->timing ? t->kev[i] : nullptr;
    p.aux = t->vfront;
    p.aux_ev[0] = t->vev[4];
    p.aux_ev[1] = t->vev[5];
    p.counts = t->status.as<uint32_t>();
    p.scan_part = p.counts + ((size_t)p.segs << maxb);
    p.digit_base = t->digit_base.as<uint64_t>();
    p.tmp_rec = t->tmp_rec.p;
    p.tmp_leaf = t->tmp_leaf.as<uint32_t>();
  }
  SplitView v = make_view(t, t->pts);
  RUN(launch_distribute(t->fmt, v, p, t->leaf_pts.p, s));
  mark(t, 4, s);
  if (!sync) {  // lod_build: the leaf-count invariant is checked on the device, reported after voxelize
    RUN(launch_check_count(v.st, n, s));
    CK(cudaGetLastError());
    return LOD_OK;
  }
  int r = read_state(t, s);
  if (r) return r;
  if ((r = check_errors(t, s))) return r;
  if (t->host_state->count_b != n) return fail(LOD_ECONSISTENCY, "leaf received a different count than allocated");
  CK(cudaGetLastError());
  return LOD_OK;
}

// lod_tree_set_output_wait: the node table and the leaf buffer are rewritten from the skeleton on
int wait_outputs(lod_tree* t, cudaStream_t s) {
  if (t->out_wait) {
    CK(cudaStreamWaitEvent(s, t->out_wait, 0));
    t->out_wait = nullptr;  // one split only
  }
  return LOD_OK;
}

int do_split(lod_tree* t, const void* pts, uint64_t n, int fmt, const double* ub, const lod_config* cfg,
             cudaStream_t s, bool final_sync = true) {
  if (t) t->dist = false;
  int r = phase_init(t, pts, n, fmt, ub, cfg, s);
  if (r) return r;
  t->n_global = n;
  // candidate list for the first extension round: clouds large enough for the sampled count
  // to see a cell of T points (and a main grid whose candidate bitmap is small)
  t->cand = cand_enabled() && cfg->max_depth > cfg->initial_depth && cfg->initial_depth <= 9 &&
            n >= cand_min_points() && n / ((uint64_t)cfg->T + 1) >= 1;
  if ((r = phase_bounds(t, ub, s)) || (r = phase_count(t, s))) return r;
  uint32_t cur = 0;
  if ((r = phase_anchors(t, &cur, s))) return r;
  while (cur > 0) {
    if ((r = phase_round(t, s)) || (r = phase_subanchors(t, &cur, s))) return r;
  }
  if ((r = wait_outputs(t, s)) || (r = phase_skeleton(t, s)) || (r = phase_distribute(t, s, final_sync))) return r;
  t->split_done = true;
  return LOD_OK;
}

// Optional restriction of a voxelize call (multi-GPU): which inner nodes to sample here,
// whether to keep the arena's current contents, and voxel runs imported from other GPUs.
struct VoxPlan {
  const uint8_t* mask = nullptr;      // per node: 1 = sample here (host)
  bool append = false;                // keep the arena and earlier results
  const int32_t* imp_nodes = nullptr; // imported inner nodes (host)
  const uint32_t* imp_counts = nullptr;
  uint32_t n_imp = 0;
  uint32_t imp_slot_base = 0;         // first parity slot free for imports at their depth
  const void* d_imp_vox = nullptr;    // their voxels, concatenated (device)
};

int do_voxelize(lod_tree* t, int mode, uint64_t seed, cudaStream_t s, const VoxPlan* plan = nullptr,
                bool split_errors_pending = false) {
  if (!t || !t->split_done) return fail(LOD_EVALUE, "lod_voxelize before a successful lod_split");
  if (mode < LOD_MODE_RANDOM || mode > LOD_MODE_WEIGHTED) return fail(LOD_EVALUE, "unknown sampling strategy: %d", mode);
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  CK(cudaEventRecord(t->vev[4], t->vfront));  // side-stream work of an earlier call that ended early
  CK(cudaStreamWaitEvent(s, t->vev[4], 0));
  CK(cudaEventRecord(t->vev[5], t->vback));
  CK(cudaStreamWaitEvent(s, t->vev[5], 0));
  t->voxel_mode = -1;
  if (!(plan && plan->append)) t->n_voxels = 0;
  uint32_t widest = 0;
  for (int d = 0; d <= kMaxDepth; ++d) widest = std::max(widest, t->inner_per_depth[d]);
  // per-depth work lists: all inner nodes, or the plan's subset (+ imports)
  uint32_t lst_n[kMaxDepth + 1] = {}, lst_off[kMaxDepth + 1] = {}, imp_n[kMaxDepth + 1] = {},
           imp_off[kMaxDepth + 1] = {};
  const uint32_t* d_lists = t->depth_lists.as<uint32_t>();
  const uint32_t* d_imp = nullptr;
  if (plan) {
    std::vector<uint64_t> cell(t->n_nodes);
    std::vector<uint32_t> val(t->n_nodes);
    CK(cudaMemcpy(cell.data(), t->n_cell.p, 8ull * t->n_nodes, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(val.data(), t->n_val.p, 4ull * t->n_nodes, cudaMemcpyDeviceToHost));
    std::vector<std::vector<uint32_t>> by(kMaxDepth + 1), ib(kMaxDepth + 1);
    for (uint32_t k = 0; k < t->n_nodes; ++k)
      if (val[k] == UNMERGEABLE && plan->mask && plan->mask[k]) by[(cell[k] >> 48) & 0xFF].push_back(k);
    for (uint32_t i = 0; i < plan->n_imp; ++i) ib[(cell[plan->imp_nodes[i]] >> 48) & 0xFF].push_back(plan->imp_nodes[i]);
    std::vector<uint32_t> flat;
    for (int d = 0; d <= kMaxDepth; ++d) lst_off[d] = flat.size(), lst_n[d] = by[d].size(), flat.insert(flat.end(), by[d].begin(), by[d].end());
    for (int d = 0; d <= kMaxDepth; ++d) imp_off[d] = flat.size(), imp_n[d] = ib[d].size(), flat.insert(flat.end(), ib[d].begin(), ib[d].end());
    for (int d = 0; d <= kMaxDepth; ++d) widest = std::max(widest, plan->imp_slot_base + imp_n[d]);
    CK(ensure(t->plan_lists, std::max<size_t>(flat.size(), 1) * 4));
    if (!flat.empty()) CK(cudaMemcpyAsync(t->plan_lists.p, flat.data(), flat.size() * 4, cudaMemcpyHostToDevice, s));
    d_lists = t->plan_lists.as<uint32_t>();
    d_imp = d_lists;
  } else {
    for (int d = 0; d <= kMaxDepth; ++d) lst_n[d] = t->inner_per_depth[d], lst_off[d] = t->inner_off[d];
  }
  uint32_t total = 0;
  for (int d = 0; d <= kMaxDepth; ++d) total += lst_n[d] + imp_n[d];
  mark(t, 4, s);
  if (total == 0 && !(plan && plan->n_imp)) {  // single-leaf root: nothing to voxelize (test_sampling.py:163-166)
    if (split_errors_pending) {  // lod_build: the split's deferred device checks
      int r = read_state(t, s);
      if (r || (r = check_errors(t, s))) return r;
    }
    t->voxel_mode = mode;
    mark(t, 5, s);
    return LOD_OK;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, t->device);
  const uint64_t kWordsPerNode = 1ull << 16;
  const size_t keep = plan && plan->append;
  CK(ensure(t->vbits, 2ull * widest * kWordsPerNode * 4, keep ? t->vbits.cap : 0, s));
  CK(ensure(t->vpre, 2ull * widest * kWordsPerNode * 4, keep ? t->vpre.cap : 0, s));
  CK(ensure(t->vinfo, 2ull * widest * sizeof(VoxNode), keep ? t->vinfo.cap : 0, s));
  CK(ensure(t->vblk, (size_t)widest * 16 * 4));
  CK(ensure(t->vcount, 64 * 4 * (kMaxDepth + 1)));
  CK(ensure(t->vlevel_start, 8 * (kMaxDepth + 1)));
  CK(ensure(t->node_slot, (size_t)t->n_nodes * 4, keep ? t->node_slot.cap : 0, s));
  uint64_t imp_total = 0;
  for (uint32_t i = 0; plan && i < plan->n_imp; ++i) imp_total += plan->imp_counts[i];
  const uint64_t base_cursor = keep ? t->n_voxels : 0;
  // first guess at the arena (grown and re-run on ERR_ARENA): surfaces give V/N ~ 0.3-1.0,
  // volumes up to ~1.8; very large clouds start lean to leave HBM for the rest
  const uint64_t guess = t->n <= (1ull << 27) ? t->n + t->n / 2 : t->n - t->n / 4;
  // LODB200_TINY_ARENA=1 (tests only): start from a tiny arena so the grow-and-retry path runs
  static const bool tiny_arena = getenv("LODB200_TINY_ARENA") && getenv("LODB200_TINY_ARENA")[0] == '1';
  uint64_t cap = (tiny_arena ? 4096 : std::max<uint64_t>(guess, 1ull << 21)) + base_cursor + imp_total;
  if (t->vox.cap / 8 > cap && !tiny_arena) cap = t->vox.cap / 8;
  uint32_t acc_stride = voxelize_acc_bytes(mode, false);
  const bool fc = mode == LOD_MODE_FIRST_COME;
  uint64_t acc_cap = tiny_arena ? 1024 : std::max<uint64_t>(t->n <= (1ull << 27) ? t->n / 2 : t->n / 4, 1ull << 21);
  if (t->vacc.cap / (2 * acc_stride) > acc_cap && !tiny_arena) acc_cap = t->vacc.cap / (2 * acc_stride);
  bool exact_sums = false;
  for (int attempt = 0; attempt < 8; ++attempt) {
    acc_stride = voxelize_acc_bytes(mode, exact_sums);  // the u64 fallback needs 32 B per voxel
    CK(ensure(t->vox, cap * 8, base_cursor * 8, s));
    cap = t->vox.cap / 8;
    CK(ensure(t->vacc, 2 * acc_cap * acc_stride));  // two depth parities (launch_voxelize_back)
    acc_cap = t->vacc.cap / (2 * acc_stride) & ~3ull;  // each parity half 16-B aligned
    // first-come: a level samples at most every leaf point once plus every child voxel
    const uint64_t ocap = fc ? (t->n + cap) / 32 + 2ull * widest + 64 : 0;
    if (fc) {
      CK(ensure(t->vpos, cap * 4, base_cursor * 4, s));
      CK(ensure(t->vout, cap * 8, base_cursor * 8, s));
      CK(ensure(t->obits, ocap * 8));
      CK(ensure(t->scan, (ocap / kScanTile + 2) * 8));
    }
    const uint64_t chunk_cap = voxelize_chunk_capacity(t->n + cap, widest);
    const uint64_t vchunk_cap = voxelize_vchunk_capacity(cap, widest);
    CK(ensure(t->vchunks, 2 * chunk_cap * 16));  // two depth parities
    CK(ensure(t->vvchunks, 2 * vchunk_cap * 8));
    if (!(split_errors_pending && attempt == 0))  // else the split's device checks report with ours
      CK(cudaMemsetAsync((char*)t->state.p + offsetof(DevState, err), 0,
                         sizeof(DevState) - offsetof(DevState, err), s));
    else
      CK(cudaMemsetAsync((char*)t->state.p + offsetof(DevState, vox_cursor), 0,
                         sizeof(DevState) - offsetof(DevState, vox_cursor), s));
    // arena: [earlier results][imports][this call's voxels]
    uint64_t cursor = base_cursor;
    if (plan && plan->n_imp) {
      CK(cudaMemcpyAsync(t->vox.as<uint2>() + cursor, plan->d_imp_vox, imp_total * 8, cudaMemcpyDeviceToDevice, s));
      if (fc)  // stored order; launch_voxelize_import puts the arena copy in key order
        CK(cudaMemcpyAsync(t->vout.as<uint2>() + cursor, plan->d_imp_vox, imp_total * 8, cudaMemcpyDeviceToDevice, s));
      for (uint32_t i = 0; i < plan->n_imp; ++i) {
        uint64_t f = cursor;
        uint32_t c = plan->imp_counts[i];
        CK(cudaMemcpyAsync(t->n_first.as<uint64_t>() + plan->imp_nodes[i], &f, 8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(t->n_count.as<uint32_t>() + plan->imp_nodes[i], &c, 4, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));  // host sources are stack values
        cursor += c;
      }
    }
    if (cursor) {
      launch_pdl(k_set_u64, 1, 1, 0, s, reinterpret_cast<uint64_t*>((char*)t->state.p + offsetof(DevState, vox_cursor)),
                 (uint64_t)cursor);
    } else {
      CK(cudaMemsetAsync((char*)t->state.p + offsetof(DevState, vox_cursor), 0, 8, s));
    }
    CK(cudaMemsetAsync(t->vcount.p, 0, 64 * 4 * (kMaxDepth + 1), s));
    VoxLevel L{};
    L.st = t->state.as<DevState>();
    // the stash lives only during voxelize: reuse the 2-pass distribute's record scratch
    // (dead after the split, 16-32 B/pt) instead of another 8 B/pt
    if (t->tmp_rec.cap >= std::max<uint64_t>(t->n, 1) * 8) {
      L.stash = t->tmp_rec.as<uint2>();
    } else {
      CK(ensure(t->stash, std::max<uint64_t>(t->n, 1) * 8));
      L.stash = t->stash.as<uint2>();
    }
    L.fmt = t->fmt;
    L.leaf_pts = t->leaf_pts.p;
    L.n_box = t->n_box.as<double4>();
    L.inv_world = t->inv_world;
    L.n_cell = t->n_cell.as<uint64_t>();
    L.n_child = t->n_child.as<int32_t>();
    L.n_leaf = t->n_leaf.as<int32_t>();
    L.n_first = t->n_first.as<uint64_t>();
    L.n_count = t->n_count.as<uint32_t>();
    L.node_slot = t->node_slot.as<uint32_t>();
    L.slots = widest;
    L.bits = t->vbits.as<uint32_t>();
    L.pre = t->vpre.as<uint32_t>();
    L.blk_sum = t->vblk.as<uint32_t>();
    L.vox = t->vox.as<uint2>();
    L.vox_cap = cap;
    L.acc_cap = acc_cap;
    L.mode = mode;
    L.exact_sums = exact_sums ? 1 : 0;
    L.seed = seed;
    L.vpos = t->vpos.as<uint32_t>();
    L.vout = t->vout.as<uint2>();
    L.obits = t->obits.as<uint32_t>();
    L.ocap = ocap;
    ScanScratch vscr{t->scan.as<uint64_t>(), t->scan.cap / 8};
    const uint64_t vchunk_half = t->vvchunks.cap / 16, chunk_half = t->vchunks.cap / 32;
    // Per level L: front(L) on vfront, K3(L) on s, back(L) on vback.  front(L) reuses the
    // depth-parity buffers of the last level of its parity, so it waits for that level's back
    // half; K3(L) waits for front(L) and for the children's colours (the last back half of the
    // other parity).  front(L+1) thus runs under K3(L) and back(L).
    cudaEvent_t& e_fork = t->vev[0];
    cudaEvent_t& e_front = t->vev[1];
    cudaEvent_t& e_k3 = t->vev[2];
    cudaEvent_t* e_back = t->vev + 3;  // [parity]
    cudaEvent_t& e_misc = t->vev[5];
    CK(cudaEventRecord(e_fork, s));
    CK(cudaStreamWaitEvent(t->vfront, e_fork, 0));
    CK(cudaStreamWaitEvent(t->vback, e_fork, 0));
    bool has_back[2] = {false, false};
    for (int d = kMaxDepth; d >= 0; --d) {  // deepest first (sampling.py:171)
      if (!lst_n[d] && !imp_n[d]) continue;
      L.parity = d & 1;
      L.info = t->vinfo.as<VoxNode>() + (size_t)L.parity * widest;
      L.counters = t->vcount.as<uint32_t>() + 64 * d;
      L.level_start = t->vlevel_start.as<uint64_t>() + d;
      L.acc = reinterpret_cast<uint64_t*>(t->vacc.as<char>() + (size_t)L.parity * acc_cap * acc_stride);
      L.vchunks = t->vvchunks.as<uint2>() + (size_t)L.parity * vchunk_half;
      L.chunks = t->vchunks.as<uint4>() + (size_t)L.parity * chunk_half;
      if (lst_n[d]) {
        L.list = d_lists + lst_off[d];
        L.list_n = lst_n[d];
        L.chunk = voxelize_chunk(L.list_n);
        L.vchunk = voxelize_vchunk(L.list_n);
        if (has_back[L.parity]) CK(cudaStreamWaitEvent(t->vfront, e_back[L.parity], 0));
        CK(cudaMemsetAsync(L.bits + (size_t)L.parity * widest * kWordsPerNode, 0,
                           (size_t)L.list_n * kWordsPerNode * 4, t->vfront));
        RUN(launch_voxelize_front(L, sms, t->vfront));
        CK(cudaEventRecord(e_front, t->vfront));
        CK(cudaStreamWaitEvent(s, e_front, 0));
        if (has_back[1 - L.parity]) CK(cudaStreamWaitEvent(s, e_back[1 - L.parity], 0));  // children's colours
        RUN(launch_voxelize_accumulate(L, sms, s));
        CK(cudaEventRecord(e_k3, s));
        CK(cudaStreamWaitEvent(t->vback, e_k3, 0));
        RUN(launch_voxelize_back(L, sms, vscr, t->vback));
        CK(cudaEventRecord(e_back[L.parity], t->vback));
        has_back[L.parity] = true;
      }
      if (imp_n[d]) {  // imports (multi-GPU rank 0): everything before them done, everything after waits
        for (int q = 0; q < 2; ++q)
          if (has_back[q]) CK(cudaStreamWaitEvent(s, e_back[q], 0));
        CK(cudaEventRecord(e_misc, t->vfront));
        CK(cudaStreamWaitEvent(s, e_misc, 0));
        L.list = d_imp + imp_off[d];
        L.list_n = imp_n[d];
        CK(cudaMemsetAsync(L.bits + ((size_t)L.parity * widest + plan->imp_slot_base) * kWordsPerNode, 0,
                           (size_t)L.list_n * kWordsPerNode * 4, s));
        RUN(launch_voxelize_import(L, plan->imp_slot_base, s));
        CK(cudaEventRecord(e_misc, s));
        CK(cudaStreamWaitEvent(t->vfront, e_misc, 0));
        CK(cudaStreamWaitEvent(t->vback, e_misc, 0));
      }
    }
    for (int q = 0; q < 2; ++q)  // join
      if (has_back[q]) CK(cudaStreamWaitEvent(s, e_back[q], 0));
    CK(cudaEventRecord(e_misc, t->vfront));
    CK(cudaStreamWaitEvent(s, e_misc, 0));
    int r = read_state(t, s);
    if (r) return r;
    CK(cudaGetLastError());
    // lod_build defers the split's device checks to here: report them before any retry
    // (a retry clears the error word, and the arena size in err_value would be the split's)
    if (split_errors_pending && (t->host_state->err & kSplitErrors)) return check_errors(t, s);
    if ((t->host_state->err & ERR_ARENA) && !(t->host_state->err & ERR_RANDOM_LIMIT)) {
      uint64_t need = t->host_state->err_value;
      cap = std::max<uint64_t>(cap * 2, need + (need >> 2));
      acc_cap = std::max<uint64_t>(acc_cap * 2, need / 2);
      continue;
    }
    if (t->host_state->err == ERR_F32_SUMS && !exact_sums) {  // >= 65794 samples in one voxel
      exact_sums = true;
      continue;
    }
    if ((r = check_errors(t, s))) return r;
    t->n_voxels = t->host_state->vox_cursor;
    t->voxel_mode = mode;
    mark(t, 5, s);
    return LOD_OK;
  }
  return fail(LOD_ECUDA, "voxel arena could not be sized");
}

// ---------------------------------------------------------------------------
// multi-GPU stages (driven by paper_2302_14801_b200/dist.py)
// ---------------------------------------------------------------------------
int dist_begin(lod_tree* t, const void* pts, uint64_t n, int fmt, const lod_config* cfg, double* out6,
               cudaStream_t s) {
  if (t) t->dist = true;
  int r = phase_init(t, pts, n, fmt, nullptr, cfg, s);
  if (r) return r;
  t->dist_stage = 1;
  for (int a = 0; a < 3; ++a) out6[a] = INFINITY, out6[3 + a] = -INFINITY;
  if (n == 0) return LOD_OK;
  if ((r = phase_bounds(t, nullptr, s)) || (r = read_state(t, s))) return r;
  if ((r = check_errors(t, s))) return r;
  for (int a = 0; a < 3; ++a) {  // decode the order-preserving keys on the host
    uint64_t lk = t->host_state->lo_key[a], hk = t->host_state->hi_key[a];
    uint64_t lu = (lk >> 63) ? (lk & 0x7FFFFFFFFFFFFFFFull) : ~lk, hu = (hk >> 63) ? (hk & 0x7FFFFFFFFFFFFFFFull) : ~hk;
    memcpy(&out6[a], &lu, 8);
    memcpy(&out6[3 + a], &hu, 8);
  }
  return LOD_OK;
}

int dist_count(lod_tree* t, uint64_t n_global, const double* world, lod_span* out, cudaStream_t s) {
  if (!t || t->dist_stage != 1) return fail(LOD_EVALUE, "lod_dist_count out of order");
  t->n_global = n_global;
  SplitView v = make_view(t, t->pts);
  RUN(launch_bounds(t->fmt, t->pts, t->n, v.st, world, s));  // forced (global) cube
  int r = phase_count(t, s);
  if (r) return r;
  if ((r = read_state(t, s)) || (r = check_errors(t, s))) return r;  // points outside the cube
  const uint64_t fine = 1ull << (3 * t->cfg.initial_depth);
  CK(ensure(t->local_main, fine * 4));
  CK(cudaMemcpyAsync(t->local_main.p, t->pyr.as<uint32_t>() + level_off(t->cfg.initial_depth), fine * 4,
                     cudaMemcpyDeviceToDevice, s));
  out->ptr = t->pyr.as<uint32_t>() + level_off(t->cfg.initial_depth);
  out->n = fine;
  t->dist_stage = 2;
  return LOD_OK;
}

int dist_extend(lod_tree* t, lod_span* out, cudaStream_t s) {
  if (!t || (t->dist_stage != 2 && t->dist_stage != 3)) return fail(LOD_EVALUE, "lod_dist_extend out of order");
  out->ptr = nullptr;
  out->n = 0;
  uint32_t cur = 0;
  int r = t->dist_stage == 2 ? phase_anchors(t, &cur, s) : phase_subanchors(t, &cur, s);
  if (r) return r;
  if (cur == 0) {
    t->dist_stage = 4;
    return LOD_OK;
  }
  const uint64_t before = t->ext_pyr_used;
  if ((r = phase_round(t, s))) return r;
  const uint64_t main_cells = level_off(t->cfg.initial_depth + 1);
  const uint64_t n_new = t->ext_pyr_used - before;
  CK(ensure(t->local_ext, t->ext_pyr_used * 4, before * 4, s));
  CK(cudaMemcpyAsync(t->local_ext.as<uint32_t>() + before, t->pyr.as<uint32_t>() + main_cells + before, n_new * 4,
                     cudaMemcpyDeviceToDevice, s));
  out->ptr = t->pyr.as<uint32_t>() + main_cells + before;
  out->n = n_new;
  t->dist_stage = 3;
  return LOD_OK;
}

int dist_skeleton(lod_tree* t, uint32_t* h_counts, cudaStream_t s) {
  if (!t || t->dist_stage != 4) return fail(LOD_EVALUE, "lod_dist_skeleton out of order");
  int r = wait_outputs(t, s);
  if (r || (r = phase_skeleton(t, s))) return r;
  std::vector<uint32_t> rf, rc;
  std::vector<int> re;
  std::vector<uint64_t> rb;
  for (auto& rd : t->rounds) rf.push_back(rd.first), rc.push_back(rd.count), re.push_back(rd.ext), rb.push_back(rd.pyr_base);
  SplitView v = make_view(t, t->pts);
  RUN(launch_local_leaf_counts(v, t->local_main.as<uint32_t>(), t->local_ext.as<uint32_t>(), rf.data(), rc.data(),
                               re.data(), rb.data(), (int)t->rounds.size(), s));
  ScanScratch scr{t->scan.as<uint64_t>(), t->scan.cap / 8};
  RUN(launch_leaf_offsets_local(v, scr, s));
  if ((r = phase_distribute(t, s))) return r;
  if (t->host_state->count_b != t->n)
    return fail(LOD_ECONSISTENCY, "leaf received a different count than allocated");
  if (h_counts) CK(cudaMemcpy(h_counts, t->leaf_count.p, 4ull * t->n_leaves, cudaMemcpyDeviceToHost));
  t->split_done = true;
  t->dist_stage = 5;
  return LOD_OK;
}

int dist_copy_segments(lod_tree* t, const void* src, void* dst, const uint64_t* hs, const uint64_t* hd,
                       const uint32_t* hc, uint64_t nseg, cudaStream_t s) {
  if (!t) return fail(LOD_EVALUE, "null tree");
  if (!nseg) return LOD_OK;
  CK(ensure(t->seg, nseg * 20));
  uint64_t* ds = t->seg.as<uint64_t>();
  CK(cudaMemcpyAsync(ds, hs, nseg * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(ds + nseg, hd, nseg * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(ds + 2 * nseg, hc, nseg * 4, cudaMemcpyHostToDevice, s));
  RUN(launch_copy_segments(src ? src : t->leaf_pts.p, dst ? dst : t->leaf_pts.p, ds, ds + nseg,
                           reinterpret_cast<uint32_t*>(ds + 2 * nseg), nseg, t->fmt == LOD_POINTS_F32 ? 16 : 32, s));
  CK(cudaStreamSynchronize(s));
  return LOD_OK;
}

int dist_adopt(lod_tree* t, const void* recs, uint64_t n, const uint32_t* h_counts, cudaStream_t s) {
  if (!t || t->dist_stage != 5) return fail(LOD_EVALUE, "lod_dist_adopt out of order");
  const size_t rec = t->fmt == LOD_POINTS_F32 ? 16 : 32;
  if (recs != t->leaf_pts.p) {  // else: already received in place (lod_dist_leaf_buffer)
    CK(ensure(t->leaf_pts, std::max<uint64_t>(n, 1) * rec));
    if (n) CK(cudaMemcpyAsync(t->leaf_pts.p, recs, n * rec, cudaMemcpyDeviceToDevice, s));
  } else if (t->leaf_pts.cap < n * rec) {
    return fail(LOD_EVALUE, "leaf buffer smaller than the adopted records");
  }
  CK(cudaMemcpyAsync(t->leaf_count.p, h_counts, 4ull * t->n_leaves, cudaMemcpyHostToDevice, s));
  ScanScratch scr{t->scan.as<uint64_t>(), t->scan.cap / 8};
  SplitView v = make_view(t, t->pts);
  RUN(launch_leaf_offsets_local(v, scr, s));
  int r = read_state(t, s);
  if (r) return r;
  if (t->host_state->count_b != n) return fail(LOD_EVALUE, "adopted records do not match the leaf counts");
  t->n = n;
  return LOD_OK;
}

}  // namespace

extern "C" {

lod_tree* lod_tree_create(int device) {
  lod_tree* t = new lod_tree();
  t->device = device;
  void* hm = nullptr;
  void* hm_dev = nullptr;
  const size_t depth_at = (sizeof(DevState) + 15) & ~(size_t)15;
  DeviceGuard dg_(device);
  if (dg_.status != cudaSuccess ||
      cudaHostAlloc(&hm, depth_at + 4 * (kMaxDepth + 2), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(&hm_dev, hm, 0) != cudaSuccess) {
    if (hm) cudaFreeHost(hm);
    fail(LOD_ECUDA, "cannot initialise CUDA device %d", device);
    delete t;
    return nullptr;
  }
  t->host_state = static_cast<DevState*>(hm);
  t->host_state_dev = static_cast<DevState*>(hm_dev);
  t->host_depth = reinterpret_cast<uint32_t*>(static_cast<char*>(hm) + depth_at);
  t->host_depth_dev = reinterpret_cast<uint32_t*>(static_cast<char*>(hm_dev) + depth_at);
  for (auto& e : t->ev) cudaEventCreate(&e);
  for (auto& e : t->kev) cudaEventCreate(&e);
  for (auto& e : t->vev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  cudaStreamCreateWithFlags(&t->vback, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&t->vfront, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&t->cstream, cudaStreamNonBlocking);
  for (auto& e : t->cev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  return t;
}

void lod_tree_destroy(lod_tree* t) {
  if (!t) return;
  DeviceGuard dg_(t->device);
  DevBuf* all[] = {&t->state, &t->pyr, &t->node_idx, &t->t8, &t->te, &t->meta, &t->list, &t->scan, &t->slots,
                   &t->n_cell, &t->n_val, &t->n_parent, &t->n_child, &t->n_slot, &t->n_extid, &t->n_lvl,
                   &t->n_leaf, &t->n_box, &t->n_first, &t->n_count, &t->leaf_node, &t->leaf_first, &t->leaf_count,
                   &t->leaf_pbox, &t->leaf_pinv, &t->depth_count, &t->depth_off, &t->depth_cursor, &t->depth_lists, &t->leaf_pts, &t->status,
                   &t->digit_base, &t->tmp_rec, &t->tmp_leaf, &t->vox, &t->export_buf,
                   &t->stash, &t->vbits, &t->vpre, &t->vinfo, &t->vblk, &t->vcount, &t->vlevel_start,
                   &t->node_slot, &t->vacc, &t->vchunks, &t->vvchunks, &t->local_main, &t->local_ext, &t->plan_lists, &t->seg,
                   &t->vpos, &t->vout, &t->obits, &t->pkey, &t->elist, &t->abits};
  for (DevBuf* b : all) release(*b);
  for (auto& e : t->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : t->kev)
    if (e) cudaEventDestroy(e);
  for (auto& e : t->vev)
    if (e) cudaEventDestroy(e);
  if (t->vback) cudaStreamDestroy(t->vback);
  if (t->vfront) cudaStreamDestroy(t->vfront);
  if (t->cstream) cudaStreamDestroy(t->cstream);
  for (auto& e : t->cev)
    if (e) cudaEventDestroy(e);
  if (t->host_state) cudaFreeHost(t->host_state);
  delete t;
}

int lod_split(lod_tree* t, const void* d_points, uint64_t n, int format, const double* bounds_or_null,
              const lod_config* config, void* stream) {
  return do_split(t, d_points, n, format, bounds_or_null, config, (cudaStream_t)stream);
}

int lod_voxelize(lod_tree* t, int mode, uint64_t seed, void* stream) {
  return do_voxelize(t, mode, seed, (cudaStream_t)stream);
}

int lod_build(lod_tree* t, const void* d_points, uint64_t n, int format, const lod_config* config, int mode,
              uint64_t seed, void* stream) {
  if (mode < LOD_MODE_RANDOM || mode > LOD_MODE_WEIGHTED) return fail(LOD_EVALUE, "unknown sampling strategy: %d", mode);
  // one host round trip fewer: the split's last invariants are checked on the device and
  // reported together with the voxelizer's
  int r = do_split(t, d_points, n, format, nullptr, config, (cudaStream_t)stream, false);
  if (r) return r;
  return do_voxelize(t, mode, seed, (cudaStream_t)stream, nullptr, true);
}

int lod_tree_get_info(const lod_tree* t, lod_tree_info* o) {
  if (!t || !o) return fail(LOD_EVALUE, "null argument");
  memset(o, 0, sizeof(*o));
  o->n_points = t->n;
  o->n_voxels = t->n_voxels;
  o->n_nodes = t->n_nodes;
  o->n_leaves = t->n_leaves;
  o->n_inner = t->n_nodes - t->n_leaves;
  o->depth = t->max_depth_used;
  o->point_format = t->fmt;
  o->voxel_mode = t->voxel_mode;
  for (int a = 0; a < 3; ++a) o->world_min[a] = t->world[a];
  o->world_size = t->world[3];
  o->n_ext_grids = t->n_ext;
  o->radix_passes = (uint32_t)t->plan.passes;
  return LOD_OK;
}

static const void* stored_voxels(const lod_tree* t);

int lod_tree_copy_nodes(const lod_tree* tc, lod_node* host, void* stream) {
  lod_tree* t = const_cast<lod_tree*>(tc);
  if (!t || !t->split_done) return fail(LOD_EVALUE, "no tree built");
  cudaStream_t s = (cudaStream_t)stream;
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  CK(ensure(t->export_buf, (size_t)t->n_nodes * sizeof(lod_node)));
  SplitView v = make_view(t, nullptr);
  launch_export_nodes(v, t->export_buf.as<lod_node>(), s);
  CK(cudaMemcpyAsync(host, t->export_buf.p, (size_t)t->n_nodes * sizeof(lod_node), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return LOD_OK;
}

int lod_tree_set_output_wait(lod_tree* t, void* event) {
  if (!t) return fail(LOD_EVALUE, "null tree");
  t->out_wait = (cudaEvent_t)event;
  return LOD_OK;
}

// Large device<->host copies go out as 256-MB pieces alternating between the caller's stream and
// the tree's copy stream, so two copy engines serve the direction: with the other direction busy
// (the pipelined e2e: next upload || this download) one engine reached 45.8 GB/s per direction,
// two 49.2 (scripts/micro/pcie_big.py, 8-GB pinned buffers).  Ordered on `s` like one copy.
static int copy_split(lod_tree* t, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
  constexpr size_t kPiece = 256ull << 20;
  if (bytes < 2 * kPiece) {
    CK(cudaMemcpyAsync(dst, src, bytes, kind, s));
    return LOD_OK;
  }
  CK(cudaEventRecord(t->cev[0], s));
  CK(cudaStreamWaitEvent(t->cstream, t->cev[0], 0));
  size_t k = 0;
  for (size_t o = 0; o < bytes; o += kPiece, ++k)
    CK(cudaMemcpyAsync(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, std::min(kPiece, bytes - o), kind,
                       (k & 1) ? t->cstream : s));
  CK(cudaEventRecord(t->cev[1], t->cstream));
  CK(cudaStreamWaitEvent(s, t->cev[1], 0));
  return LOD_OK;
}

int lod_tree_copy_async(const lod_tree* tc, void* h_leaf, void* h_vox, lod_node* h_nodes, void* stream) {
  lod_tree* t = const_cast<lod_tree*>(tc);
  if (!t || !t->split_done) return fail(LOD_EVALUE, "no tree built");
  if (h_vox && t->voxel_mode < 0) return fail(LOD_EVALUE, "no voxels built");
  cudaStream_t s = (cudaStream_t)stream;
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  if (h_nodes) {
    CK(ensure(t->export_buf, (size_t)t->n_nodes * sizeof(lod_node)));
    SplitView v = make_view(t, nullptr);
    launch_export_nodes(v, t->export_buf.as<lod_node>(), s);
    CK(cudaMemcpyAsync(h_nodes, t->export_buf.p, (size_t)t->n_nodes * sizeof(lod_node), cudaMemcpyDeviceToHost, s));
  }
  const size_t rec = t->fmt == LOD_POINTS_F32 ? 16 : 32;
  int r;
  if (h_leaf && t->n && (r = copy_split(t, h_leaf, t->leaf_pts.p, t->n * rec, cudaMemcpyDeviceToHost, s))) return r;
  if (h_vox && t->n_voxels &&
      (r = copy_split(t, h_vox, stored_voxels(t), t->n_voxels * 8, cudaMemcpyDeviceToHost, s)))
    return r;
  return LOD_OK;
}

int lod_tree_leaf_points(const lod_tree* t, const void** p) {
  if (!t || !t->split_done) return fail(LOD_EVALUE, "no tree built");
  *p = t->leaf_pts.p;
  return LOD_OK;
}

// the stored-order voxel array: first-come lists voxels by winning ordinal
static const void* stored_voxels(const lod_tree* t) {
  return t->voxel_mode == LOD_MODE_FIRST_COME ? t->vout.p : t->vox.p;
}

int lod_tree_voxels(const lod_tree* t, const void** p) {
  if (!t || t->voxel_mode < 0) return fail(LOD_EVALUE, "no voxels built");
  *p = stored_voxels(t);
  return LOD_OK;
}

int lod_tree_copy_leaf_points(const lod_tree* t, void* host, void* stream) {
  if (!t || !t->split_done) return fail(LOD_EVALUE, "no tree built");
  size_t rec = t->fmt == LOD_POINTS_F32 ? 16 : 32;
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  CK(cudaMemcpyAsync(host, t->leaf_pts.p, t->n * rec, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return LOD_OK;
}

int lod_tree_copy_voxels(const lod_tree* t, void* host, void* stream) {
  if (!t || t->voxel_mode < 0) return fail(LOD_EVALUE, "no voxels built");
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  if (t->n_voxels)
    CK(cudaMemcpyAsync(host, stored_voxels(t), t->n_voxels * 8, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return LOD_OK;
}

int lod_tree_copy_range(const lod_tree* t, int what, uint64_t first, uint64_t count, void* host, void* stream) {
  if (!t || !t->split_done) return fail(LOD_EVALUE, "no tree built");
  if (what != 0 && what != 1) return fail(LOD_EVALUE, "unknown output %d", what);
  if (what == 1 && t->voxel_mode < 0) return fail(LOD_EVALUE, "no voxels built");
  const uint64_t total = what == 0 ? t->n : t->n_voxels;
  if (first > total || count > total - first)
    return fail(LOD_EVALUE, "range [%llu, +%llu) outside the %llu %s", (unsigned long long)first,
                (unsigned long long)count, (unsigned long long)total, what == 0 ? "points" : "voxels");
  const size_t rec = what == 1 ? 8 : t->fmt == LOD_POINTS_F32 ? 16 : 32;
  const char* src = static_cast<const char*>(what == 0 ? t->leaf_pts.p : stored_voxels(t));
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  if (count) CK(cudaMemcpyAsync(host, src + first * rec, count * rec, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return LOD_OK;
}

int lod_tree_encode_payload(const lod_tree* tc, const int32_t* h_order, const uint64_t* h_offsets, uint32_t n,
                            void* d_payload, void* stream) {
  lod_tree* t = const_cast<lod_tree*>(tc);
  if (!t || !t->split_done) return fail(LOD_EVALUE, "no tree built");
  if (t->voxel_mode < 0 && t->n_nodes > t->n_leaves)
    return fail(LOD_EVALUE, "encode needs voxels: run lod_voxelize first");
  if (n > t->n_nodes) return fail(LOD_EVALUE, "node order longer than the node table");
  cudaStream_t s = (cudaStream_t)stream;
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  CK(ensure(t->export_buf, (size_t)n * 12 + 16));
  int32_t* d_order = t->export_buf.as<int32_t>();
  uint64_t* d_offs = reinterpret_cast<uint64_t*>(t->export_buf.as<uint8_t>() + (((size_t)n * 4 + 15) & ~(size_t)15));
  CK(cudaMemcpyAsync(d_order, h_order, (size_t)n * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_offs, h_offsets, (size_t)n * 8, cudaMemcpyHostToDevice, s));
  SplitView v = make_view(t, nullptr);
  launch_encode(t->fmt, v, t->leaf_pts.p, reinterpret_cast<const uint2*>(stored_voxels(t)), d_order, d_offs, n,
                reinterpret_cast<uint8_t*>(d_payload), s);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  return LOD_OK;
}

int lod_ingest_las(const void* d_raw, uint64_t n, uint32_t record_length, int32_t rgb_offset, const double* scale3,
                   const double* offset3, void* d_records, void* stream) {
  if (!scale3 || !offset3) return fail(LOD_EVALUE, "null scale / offset");
  if (record_length < 12) return fail(LOD_EVALUE, "record length %u too short", record_length);
  if (rgb_offset >= 0 && (uint32_t)rgb_offset + 6 > record_length)
    return fail(LOD_EVALUE, "rgb offset %d outside the %u-byte record", rgb_offset, record_length);
  launch_ingest_las(d_raw, n, record_length, rgb_offset, scale3, offset3, d_records, (cudaStream_t)stream);
  CK(cudaGetLastError());
  return LOD_OK;
}

int lod_ingest_ply(const void* d_raw, uint64_t n, uint32_t stride, const int32_t* types6, const uint32_t* offsets6,
                   int has_rgb, int out_format, void* d_records, void* stream) {
  if (!types6 || !offsets6) return fail(LOD_EVALUE, "null property layout");
  for (int i = 0; i < (has_rgb ? 6 : 3); ++i) {
    if (types6[i] < LOD_PLY_I8 || types6[i] > LOD_PLY_F64) return fail(LOD_EVALUE, "bad PLY type %d", types6[i]);
    const uint32_t w = types6[i] <= LOD_PLY_U8 ? 1 : types6[i] <= LOD_PLY_U16 ? 2 : types6[i] == LOD_PLY_F64 ? 8 : 4;
    if (offsets6[i] + w > stride) return fail(LOD_EVALUE, "PLY property outside the %u-byte record", stride);
  }
  if (out_format != LOD_POINTS_F32 && out_format != LOD_POINTS_F64)
    return fail(LOD_EVALUE, "unknown point format %d", out_format);
  launch_ingest_ply(d_raw, n, stride, types6, offsets6, has_rgb, out_format, d_records, (cudaStream_t)stream);
  CK(cudaGetLastError());
  return LOD_OK;
}

int lod_tree_checks(const lod_tree* tc, uint32_t T, int32_t max_depth, uint8_t* h_flags, void* stream) {
  lod_tree* t = const_cast<lod_tree*>(tc);
  if (!t || !t->split_done) return fail(LOD_EVALUE, "no tree built");
  cudaStream_t s = (cudaStream_t)stream;
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  CK(ensure(t->export_buf, (size_t)t->n_nodes + 16));
  SplitView v = make_view(t, nullptr);
  // uniqueness is checked on the key-ordered arena (first-come's stored order is a permutation)
  launch_checks(t->fmt, v, t->leaf_pts.p, t->vox.as<uint2>(), t->voxel_mode >= 0 ? 1 : 0, T, max_depth,
                t->export_buf.as<uint8_t>(), s);
  CK(cudaMemcpyAsync(h_flags, t->export_buf.p, t->n_nodes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return LOD_OK;
}

uint64_t lod_tree_device_bytes(const lod_tree* t) {
  if (!t) return 0;
  const DevBuf* all[] = {&t->state, &t->pyr, &t->node_idx, &t->t8, &t->te, &t->meta, &t->list, &t->scan,
                         &t->slots, &t->n_cell, &t->n_val, &t->n_parent, &t->n_child, &t->n_slot, &t->n_extid,
                         &t->n_lvl, &t->n_leaf, &t->n_box, &t->n_first, &t->n_count, &t->leaf_node,
                         &t->leaf_first, &t->leaf_count, &t->leaf_pbox, &t->leaf_pinv, &t->depth_count, &t->depth_off, &t->depth_cursor, &t->depth_lists,
                         &t->leaf_pts, &t->status, &t->digit_base, &t->tmp_rec, &t->tmp_leaf,
                         &t->vox, &t->export_buf, &t->stash, &t->vbits, &t->vpre, &t->vinfo,
                         &t->vblk, &t->vcount, &t->vlevel_start, &t->node_slot, &t->vacc, &t->vchunks,
                         &t->vvchunks, &t->local_main, &t->local_ext, &t->plan_lists, &t->seg,
                   &t->vpos, &t->vout, &t->obits, &t->pkey, &t->elist, &t->abits};
  uint64_t b = 0;
  for (const DevBuf* x : all) b += x->cap;
  return b;
}

int lod_set_timing(lod_tree* t, int enabled) {
  if (!t) return fail(LOD_EVALUE, "null tree");
  t->timing = enabled != 0;
  return LOD_OK;
}

int lod_tree_stage_ms(const lod_tree* tc, float* out) {
  lod_tree* t = const_cast<lod_tree*>(tc);
  if (!t || !t->timing) return fail(LOD_EVALUE, "timing not enabled");
  for (int i = 0; i < 5; ++i) {  // a stage the last build did not bracket (multi-GPU calls) -> NaN
    out[i] = 0;
    if (cudaEventElapsedTime(&out[i], t->ev[i], t->ev[i + 1]) != cudaSuccess || out[i] < 0) out[i] = NAN;
  }
  cudaGetLastError();
  return LOD_OK;
}

int lod_tree_kernel_ms(const lod_tree* tc, float* out) {
  lod_tree* t = const_cast<lod_tree*>(tc);
  if (!t || !t->timing) return fail(LOD_EVALUE, "timing not enabled");
  out[0] = 0;
  for (int p = 0; p < t->plan.passes; ++p) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, t->kev[2 * p], t->kev[2 * p + 1]) == cudaSuccess) out[0] += ms;
  }
  cudaGetLastError();
  return LOD_OK;
}

uint64_t lod_tree_launches(const lod_tree* t) { return t ? t->launches : 0; }

int lod_set_allocator(lod_alloc_fn alloc, lod_free_fn free_fn, void* ctx) {
  if ((alloc == nullptr) != (free_fn == nullptr)) return fail(LOD_EVALUE, "allocator needs both functions");
  g_alloc = alloc;
  g_free = free_fn;
  g_alloc_ctx = ctx;
  return LOD_OK;
}

int lod_workspace_bytes(uint64_t n, int format, const lod_config* cfg, int mode, uint64_t* bytes) {
  if (!cfg || !bytes) return fail(LOD_EVALUE, "null argument");
  if (format != LOD_POINTS_F32 && format != LOD_POINTS_F64) return fail(LOD_EVALUE, "unknown point format %d", format);
  const uint64_t rec = format == LOD_POINTS_F32 ? 16 : 32;
  const int D = cfg->initial_depth;
  const uint64_t fine = 1ull << (3 * D), main_cells = level_off(D + 1);
  const uint64_t leaves_max = std::max<uint64_t>(1, n / std::max<uint32_t>(cfg->T, 1) * 8 + 1);
  uint64_t b = 0;
  b += main_cells * 4 + fine * 4 + fine / 8;            // pyramid, targets t8, anchor bitmap
  b += main_cells * 8 * 2;                              // node slots, scan scratch
  b += n * 4;                                           // pkey
  b += n * rec;                                         // leaf buffer
  // 2-pass distribute record copy; the first extension round's candidate list shares it
  const bool cand = cand_enabled() && cfg->max_depth > D && D <= 9 && n >= cand_min_points();
  b += std::max<uint64_t>(leaves_max >= (1u << kRadixMaxBits) ? n * rec : 0, cand ? n * 16 + (40ull << 20) : 0);
  b += cand ? fine * 4 : 0;                             // sampled counts
  b += n * 8;                                           // leaf ids (input + sorted order)
  b += n / 2;                                           // tile digit counts (11-bit digits)
  b += n / 10 * 16;                                     // extension-point list (10% in extension grids)
  const uint64_t vox = n + n / 2;                       // voxel arena (V/N <= 1.5 for surfaces)
  b += vox * 8;                                         // arena
  b += n * 8;                                           // leaf stash {key, rgb}
  b += 2 * std::max<uint64_t>(n / 4, 1ull << 21) * (mode == LOD_MODE_WEIGHTED ? 32 : mode == LOD_MODE_AVERAGE ? 16 : 4);
  if (mode == LOD_MODE_FIRST_COME) b += vox * 12 + (n + vox) / 4;  // vpos, vout, ordinal bitmaps
  b += leaves_max * 160;                                // node table
  b += 2ull * std::min<uint64_t>(leaves_max, 4096) * (1u << 19);  // rank structures of the widest level
  *bytes = b;
  return LOD_OK;
}

int lod_pack_points(const void* d_xyz, int xyz_is_f64, const uint8_t* d_rgb, uint64_t n, int out_format,
                    void* d_records, int* chosen_format, void* stream) {
  if (n && (!d_xyz || !d_rgb || !d_records)) return fail(LOD_EVALUE, "null buffer");
  if (out_format != -1 && out_format != LOD_POINTS_F32 && out_format != LOD_POINTS_F64)
    return fail(LOD_EVALUE, "unknown point format %d", out_format);
  cudaStream_t s = (cudaStream_t)stream;
  int fmt = out_format;
  if (fmt == -1) {
    fmt = LOD_POINTS_F32;
    if (xyz_is_f64 && n) {
      uint32_t* flag = nullptr;
      uint32_t h = 1;
      CK(cudaMallocAsync(reinterpret_cast<void**>(&flag), 4, s));
      CK(cudaMemcpyAsync(flag, &h, 4, cudaMemcpyHostToDevice, s));
      launch_f32_exact(static_cast<const double*>(d_xyz), n, flag, s);
      CK(cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, s));
      CK(cudaFreeAsync(flag, s));
      CK(cudaStreamSynchronize(s));
      if (!h) fmt = LOD_POINTS_F64;
    }
  }
  if (chosen_format) *chosen_format = fmt;
  launch_pack(d_xyz, xyz_is_f64 != 0, d_rgb, n, fmt, d_records, s);
  CK(cudaGetLastError());
  return LOD_OK;
}

int lod_generate(const char* kind, uint64_t seed, uint64_t start, uint64_t n, void* d_out, const double* table,
                 void* stream) {
  static const char* kinds[] = {"sphere", "terrain", "scene", "cluster", "surface"};
  int k = -1;
  for (int i = 0; i < 5; ++i)
    if (kind && strcmp(kind, kinds[i]) == 0) k = i;
  if (k < 0) return fail(LOD_EVALUE, "unknown synthetic kind: %s", kind ? kind : "(null)");
  if (k == 2 && !table) return fail(LOD_EVALUE, "scene generator needs the object table");
  launch_generate(k, seed, start, n, d_out, table, (cudaStream_t)stream);
  CK(cudaGetLastError());
  return LOD_OK;
}

int lod_dist_begin(lod_tree* t, const void* d_points, uint64_t n_local, int format, const lod_config* config,
                   double* out_min_max, void* stream) {
  return dist_begin(t, d_points, n_local, format, config, out_min_max, (cudaStream_t)stream);
}
int lod_dist_count(lod_tree* t, uint64_t n_global, const double* world, lod_span* out, void* stream) {
  return dist_count(t, n_global, world, out, (cudaStream_t)stream);
}
int lod_dist_extend(lod_tree* t, lod_span* out, void* stream) { return dist_extend(t, out, (cudaStream_t)stream); }
int lod_dist_skeleton(lod_tree* t, uint32_t* h_local_leaf_counts, void* stream) {
  return dist_skeleton(t, h_local_leaf_counts, (cudaStream_t)stream);
}
int lod_dist_leaf_counts(const lod_tree* tc, uint32_t* h) {
  lod_tree* t = const_cast<lod_tree*>(tc);
  if (!t || t->dist_stage < 5) return fail(LOD_EVALUE, "no distributed split");
  CK(cudaMemcpy(h, t->leaf_count.p, 4ull * t->n_leaves, cudaMemcpyDeviceToHost));
  return LOD_OK;
}
int lod_dist_copy_segments(lod_tree* t, const void* d_src, void* d_dst, const uint64_t* h_src, const uint64_t* h_dst,
                           const uint32_t* h_cnt, uint64_t nseg, void* stream) {
  return dist_copy_segments(t, d_src, d_dst, h_src, h_dst, h_cnt, nseg, (cudaStream_t)stream);
}
int lod_dist_leaf_buffer(lod_tree* t, uint64_t n, void** d_out) {
  if (!t || t->dist_stage != 5 || !d_out) return fail(LOD_EVALUE, "lod_dist_leaf_buffer out of order");
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  CK(ensure(t->leaf_pts, std::max<uint64_t>(n, 1) * (t->fmt == LOD_POINTS_F32 ? 16 : 32)));
  *d_out = t->leaf_pts.p;
  return LOD_OK;
}
int lod_dist_adopt(lod_tree* t, const void* d_records, uint64_t n, const uint32_t* h_leaf_counts, void* stream) {
  return dist_adopt(t, d_records, n, h_leaf_counts, (cudaStream_t)stream);
}
int lod_merge_pyramid(uint32_t* d_pyr, int L, uint32_t T, void* stream) {
  if (!d_pyr || L < 0 || L > 10) return fail(LOD_EVALUE, "bad pyramid (levels 0..10)");
  if (T < 1) return fail(LOD_EVALUE, "T must be >= 1");
  RUN_NOTREE(launch_merge_standalone(d_pyr, L, T, (cudaStream_t)stream));
  CK(cudaGetLastError());
  return LOD_OK;
}

// the stage exports are readable from the count stage on (lod_dist_count / lod_split)
static bool counted(const lod_tree* t) { return t && (t->split_done || t->dist_stage >= 2); }

int lod_tree_copy_point_keys(const lod_tree* t, uint32_t* h, void* stream) {
  if (!counted(t)) return fail(LOD_EVALUE, "no counted tree");
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  if (t->n) CK(cudaMemcpyAsync(h, t->pkey.p, t->n * 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return LOD_OK;
}

int lod_tree_copy_pyramids(const lod_tree* t, uint32_t* h, uint64_t* n_out, void* stream) {
  if (!counted(t) || !n_out) return fail(LOD_EVALUE, "no counted tree");
  const uint64_t n = level_off(t->cfg.initial_depth + 1) + t->ext_pyr_used;
  *n_out = n;
  if (!h) return LOD_OK;
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  CK(cudaMemcpyAsync(h, t->pyr.p, n * 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return LOD_OK;
}

int lod_tree_ext_grids(const lod_tree* t, lod_ext_grid* h, uint32_t* n_out, void* stream) {
  if (!counted(t) || !n_out) return fail(LOD_EVALUE, "no counted tree");
  *n_out = t->n_ext;
  if (!h || !t->n_ext) return LOD_OK;
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  std::vector<ExtMeta> m(t->n_ext);
  CK(cudaMemcpyAsync(m.data(), t->meta.p, t->n_ext * sizeof(ExtMeta), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  for (uint32_t e = 0; e < t->n_ext; ++e)
    h[e] = lod_ext_grid{m[e].pyr_off, m[e].ax, m[e].ay, m[e].az, m[e].base, m[e].ext};
  return LOD_OK;
}

int lod_tree_ext_points(const lod_tree* t, uint32_t* h_index, uint64_t* h_cell16, uint64_t* n_out, void* stream) {
  if (!counted(t) || !n_out) return fail(LOD_EVALUE, "no counted tree");
  const uint64_t n = t->elist_cap ? std::min<uint64_t>(t->host_state->ext_n, t->elist_cap) : 0;
  *n_out = n;
  if (!h_index || !h_cell16 || !n) return LOD_OK;
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  std::vector<uint4> q(n);
  CK(cudaMemcpyAsync(q.data(), t->elist.p, n * 16, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  for (uint64_t j = 0; j < n; ++j) {
    h_index[j] = q[j].x;
    h_cell16[j] = (uint64_t)q[j].z | ((uint64_t)q[j].w << 32);  // x | y << 16, z
  }
  return LOD_OK;
}

int lod_dist_export_roots(lod_tree* t, const int32_t* h_nodes, uint32_t n, void* d_out, uint32_t* h_counts,
                          void* stream) {
  if (!t || t->voxel_mode < 0) return fail(LOD_EVALUE, "no voxels built");
  if (n && (!h_nodes || !d_out || !h_counts)) return fail(LOD_EVALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  DeviceGuard dg_(t->device);
  CK(dg_.status);
  if (!n) return LOD_OK;
  // counts and destination offsets from the node table (one small copy each way)
  std::vector<uint32_t> cnt(t->n_nodes);
  CK(cudaMemcpyAsync(cnt.data(), t->n_count.p, 4ull * t->n_nodes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<uint64_t> off(n);
  uint64_t total = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (h_nodes[i] < 0 || (uint32_t)h_nodes[i] >= t->n_nodes) return fail(LOD_EVALUE, "node %d out of range", h_nodes[i]);
    h_counts[i] = cnt[h_nodes[i]];
    off[i] = total;
    total += cnt[h_nodes[i]];
  }
  CK(ensure(t->seg, (size_t)n * 12 + 16));
  int32_t* d_nodes = t->seg.as<int32_t>();
  uint64_t* d_off = reinterpret_cast<uint64_t*>(t->seg.as<char>() + (((size_t)n * 4 + 15) & ~(size_t)15));
  CK(cudaMemcpyAsync(d_nodes, h_nodes, (size_t)n * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_off, off.data(), (size_t)n * 8, cudaMemcpyHostToDevice, s));
  RUN(launch_export_runs(stored_voxels(t), t->n_first.as<uint64_t>(), t->n_count.as<uint32_t>(), d_nodes, d_off, n,
                         d_out, s));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));  // the host arrays above are locals
  return LOD_OK;
}

int lod_dist_voxelize(lod_tree* t, int mode, uint64_t seed, const uint8_t* h_mask, int append,
                      const int32_t* h_imp_nodes, const uint32_t* h_imp_counts, uint32_t n_imp, uint32_t imp_slot_base,
                      const void* d_imp_vox, void* stream) {
  VoxPlan p;
  p.mask = h_mask;
  p.append = append != 0;
  p.imp_nodes = h_imp_nodes;
  p.imp_counts = h_imp_counts;
  p.n_imp = n_imp;
  p.imp_slot_base = imp_slot_base;
  p.d_imp_vox = d_imp_vox;
  return do_voxelize(t, mode, seed, (cudaStream_t)stream, &p);
}

const char* lod_last_error(void) { return g_err.c_str(); }

const char* lod_version(void) { return "lodb200 0.1.0 sm_100a"; }

}  // extern "C"
