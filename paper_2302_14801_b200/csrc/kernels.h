// Host-callable launch wrappers of the split / distribute / voxelize kernels.
// Every wrapper enqueues on `st` and returns the number of kernels it launched.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "scan.cuh"

namespace lod {

// Unified device view of a tree's split state, passed by value to kernels.
struct SplitView {
  DevState* st;
  const void* pts;        // input records
  uint64_t n;
  int D;                  // initial_depth
  int max_depth;
  uint32_t T;
  uint32_t* pyr;          // unified pyramid buffer: main pyramid at 0, ext pyramids after
  uint64_t main_cells;    // cells of the main pyramid = level_off(D + 1)
  int32_t* node_idx;      // slot -> node id (valid at non-zero slots)
  int32_t* t8;            // main finest level: leaf id, -(ext+2), or -1
  uint32_t* pkey;         // per point: its main finest-level key (written by K_count)
  uint4* elist;           // extension points {index, round-1 extension id, x | y << 16, z}
                          // (depth-16 cell), appended by the first extension round
  uint64_t elist_cap;
  uint32_t* abits;        // anchor bitmap over the main finest grid (null: test t8)
  int32_t* te;            // ext finest levels: same encoding
  // candidate list (single-GPU split, LOD_CAND): points of the cells a sampled count marks as
  // possibly over T, with their exact depth-16 cells, so the first extension round reads no records
  uint32_t* sgrid;        // sampled counts over the main finest grid (null: candidate path off)
  uint32_t* cand_keys;    // candidate cells (ascending), <= kCandCap
  uint4* cand;            // {index, main finest key, x | y << 16, z}; index ~0u = hole
  uint64_t cand_cap;
  uint32_t cand_thresh;   // a cell is a candidate at >= cand_thresh samples
  ExtMeta* meta;
  uint32_t n_ext;
  // node table
  uint64_t* n_cell;
  uint32_t* n_val;
  int32_t* n_parent;
  int32_t* n_child;       // 8 per node
  uint64_t* n_slot;
  int32_t* n_extid;      // owning extension or -1
  uint8_t* n_lvl;
  int32_t* n_leaf;        // leaf index or -1
  double4* n_box;         // min xyz, size
  uint64_t* n_first;      // leaf: first point; inner: first voxel
  uint32_t* n_count;      // leaf: points; inner: voxels
  uint32_t n_nodes;
  uint32_t* leaf_node;
  uint64_t* leaf_first;
  uint32_t* leaf_count;   // per leaf: points of THIS process (global count on one GPU)
  double4* leaf_pbox;     // per leaf: parent bounds (w < 0 for a root leaf)
  double* leaf_pinv;      // per leaf: RN(1 / parent size)
  uint32_t n_leaves;
};

// Descend the extension chain of a point; returns the finest-cell index inside extension
// `e_out` (the deepest one containing the point), or false if the point is in none.
// `tgt_out` (optional) receives that cell's target, `pyr_out` its counting slot.
__device__ __forceinline__ bool ext_descend(const SplitView& v, const Cell16& c, uint32_t& e_out, uint32_t& r_out,
                                            int32_t t, int32_t* tgt_out = nullptr, uint64_t* pyr_out = nullptr) {
  if (t > -2) return false;
  uint32_t e = (uint32_t)(-(t + 2));
  while (true) {
    const ExtMeta m = v.meta[e];
    int s = kMaxDepth - (m.base + m.ext);
    uint32_t rx = (c.x >> s) - ((uint32_t)m.ax << m.ext);
    uint32_t ry = (c.y >> s) - ((uint32_t)m.ay << m.ext);
    uint32_t rz = (c.z >> s) - ((uint32_t)m.az << m.ext);
    uint32_t r = (rx << (2 * m.ext)) | (ry << m.ext) | rz;
    int32_t nt = v.te[m.tgt_off + r];
    if (nt > -2) {
      e_out = e;
      r_out = r;
      if (tgt_out) *tgt_out = nt;
      if (pyr_out) *pyr_out = m.pyr_off + level_off(m.ext) + r;
      return true;
    }
    e = (uint32_t)(-(nt + 2));
  }
}


// Leaf id of a point: main finest-cell target, then down the extension chain
// (partition.py:244-287 insert / _resolve_extended).  -1 if unresolved.
__device__ __forceinline__ int32_t leaf_of_point(const SplitView& v, const Cell16& c) {
  int32_t t = v.t8[level_key(c, v.D)];
  uint32_t e, r;
  int32_t nt;
  if (ext_descend(v, c, e, r, t, &nt)) t = nt;
  return t;
}

// --- split (split_kernels.cu) ---
int launch_bounds(int fmt, const void* pts, uint64_t n, DevState* st, const double* user_bounds,
                  cudaStream_t s);
int launch_count(int fmt, const SplitView& v, cudaStream_t s);
#ifndef LOD_CAND_CAP
#define LOD_CAND_CAP 2048
#endif
constexpr uint32_t kCandCap = LOD_CAND_CAP;  // candidate cells the count kernel holds in shared memory
constexpr uint32_t kCandStride = 128; // every kCandStride-th point is sampled
constexpr uint32_t kCandChunk = 256;  // list slots a warp reserves at a time (a multiple of 32)
uint32_t count_blocks(uint64_t n);  // K_count's grid
int launch_cand_sample(int fmt, const SplitView& v, ScanScratch& scr, cudaStream_t s);
int launch_cand_check(const SplitView& v, const uint64_t* anchors, uint32_t n_anchors, cudaStream_t s);
// count pass (store = false; hit count -> st->count_a), then, if any, the store pass
int launch_find_anchors(const SplitView& v, uint64_t* list, ScanScratch& scr, cudaStream_t s, bool store);
int launch_find_subanchors(const SplitView& v, uint32_t first_ext, uint32_t n_ext_round, int ext_levels,
                           uint64_t* list, ScanScratch& scr, cudaStream_t s);
int launch_ext_create(const SplitView& v, int round, uint32_t first_ext, uint32_t count,
                      const uint64_t* list, uint32_t parent_first, uint64_t pyr_base, uint64_t tgt_base,
                      int base_depth, int ext_levels, cudaStream_t s);
int launch_ext_count(int fmt, const SplitView& v, uint32_t round_first_ext, cudaStream_t s);
// sum of the anchors' main-grid counts (t->list[0..n)) -> st->ext_n (extension-list capacity)
int launch_anchor_sum(const SplitView& v, const uint64_t* list, uint32_t n, cudaStream_t s);
// leaf ids of the extension-list points -> leaf_out[index] (before the distribute's K_hist)
int launch_ext_leaf(const SplitView& v, uint32_t* leaf_out, cudaStream_t s);

__device__ __forceinline__ Cell16 unpack_c16(uint64_t p) {
  return Cell16{(uint32_t)p & 0xFFFF, (uint32_t)(p >> 16) & 0xFFFF, (uint32_t)(p >> 32) & 0xFFFF};
}
int launch_merge_all(const SplitView& v, const uint32_t* round_first, const uint32_t* round_count,
                     const int* round_ext, const uint64_t* round_pyr_base, int n_rounds, cudaStream_t s);
int launch_merge_standalone(uint32_t* pyr, int L, uint32_t T, cudaStream_t s);
int launch_count_nodes(const SplitView& v, uint64_t total_slots, uint64_t* slots_out, ScanScratch& scr,
                       cudaStream_t s);
int launch_build_nodes(const SplitView& v, const uint64_t* slots, cudaStream_t s);
int launch_number_leaves(const SplitView& v, ScanScratch& scr, cudaStream_t s);
int launch_leaf_offsets(const SplitView& v, ScanScratch& scr, cudaStream_t s);
int launch_leaf_offsets_local(const SplitView& v, ScanScratch& scr, cudaStream_t s);
int launch_leaf_parent_boxes(const SplitView& v, cudaStream_t s);
int launch_targets(const SplitView& v, cudaStream_t s);
int launch_targets_ext(const SplitView& v, uint32_t first, uint32_t count, int ext, cudaStream_t s);
int launch_depth_lists(const SplitView& v, uint32_t* depth_count, cudaStream_t s);
int launch_depth_scatter(const SplitView& v, const uint32_t* depth_off, uint32_t* depth_cursor,
                         uint32_t* lists, cudaStream_t s);
int launch_export_nodes(const SplitView& v, lod_node* out, cudaStream_t s);

// --- distribute (distribute.cu) ---
struct RadixPlan {
  int passes;             // 0 = single leaf (plain copy)
  int bits[2];            // digit widths
  uint32_t tiles;         // kRadixTile-point sub-tiles
  uint32_t segs;          // chunks (one CTA each)
  uint32_t seg_tiles;     // sub-tiles per chunk
  uint32_t* counts;       // [segs][2^bits] digit counts -> first slots (reused per pass)
  uint32_t* scan_part;    // 2 x 512 x 2^bits words: per-segment column sums of the counts
  uint64_t* digit_base;   // per pass: 2^bits global exclusive prefix
  cudaEvent_t scatter_ev[4];  // timing: start/end of each pass's K_scatter (null = off)
  cudaStream_t aux;           // side stream for the digit bases (null: the build's stream)
  cudaEvent_t aux_ev[2];      // fork, digit bases done
  void* tmp_rec;          // pass-0 output records (2 passes)
  uint32_t* tmp_leaf;     // leaf ids: input order (K_hist, pass 0) [+ sorted by digit 0]
};
constexpr int kRadixThreads = 512;
constexpr int kRadixItems = 8;
constexpr int kRadixTile = kRadixThreads * kRadixItems;
constexpr int kRadixMaxBits = 11;
void plan_segments(RadixPlan& plan, uint64_t n, int sms);
int launch_check_count(DevState* st, uint64_t n, cudaStream_t s);
int launch_distribute(int fmt, const SplitView& v, RadixPlan& plan, void* leaf_out, cudaStream_t s);

// --- voxelize (voxelize.cu) ---
struct VoxNode {           // per inner node of the level being sampled (by list slot)
  uint32_t node, S, m, skip;
  uint64_t vbase, hash;    // first voxel in the arena; seed ^ path_hash(seed, path)
  double4 box;             // node bounds (min xyz, size) for projecting leaf points
  double inv;              // RN(1 / size)
  uint64_t cfirst[8];      // child's first point (leaf) / first voxel (inner)
  uint32_t cbase[8];       // ordinal of the child's first sample (octant order)
  uint32_t ccount[8];
  int32_t cslot[8];        // -2 absent, -1 leaf child, >= 0 slot of an inner child
  uint64_t obase;          // first-come: first word of the node's ordinal bitmap
};

struct VoxLevel {
  DevState* st;
  int fmt;
  const void* leaf_pts;    // leaf buffer (input record format)
  uint2* stash;            // per leaf point {key in the leaf-parent grid, rgb}, written by K1
  const uint64_t* n_cell;
  const int32_t* n_child;
  const int32_t* n_leaf;
  const double4* n_box;
  double inv_world;        // RN(1 / world size)
  uint64_t* n_first;
  uint32_t* n_count;
  uint32_t* node_slot;     // node id -> slot in its level's list
  const uint32_t* list;    // inner nodes of this depth
  uint32_t list_n;
  int parity;              // depth & 1: which bitmap/prefix/info buffers this level owns
  uint32_t slots;          // slots per parity
  uint32_t* bits;          // [2][slots][2^16] occupancy words
  uint32_t* pre;           // [2][slots][2^16] exclusive popcount prefix per word
  VoxNode* info;           // this level's infos (parity slice)
  uint32_t* blk_sum;       // [list_n * 16]
  uint32_t* counters;      // [0] sample chunks, [2] voxel chunks, [4] first-come ordinal words,
                           // [6] K2 blocks done
  uint4* chunks;
  uint2* vchunks;
  uint64_t* level_start;   // arena cursor at the start of this level
  uint2* vox;              // arena: {key, rgb}
  uint64_t vox_cap;
  uint64_t* acc;           // per voxel of this level: 2 u64 (average), 4 u64 (weighted) or
                           // u32 (random, first-come)
  uint64_t acc_cap;        // voxels
  uint32_t* vpos;          // first-come: per voxel (arena index), stored position in its node
  uint2* vout;             // first-come: voxels in stored order (winning ordinal)
  uint32_t* obits;         // first-come: per-level ordinal bitmaps (node runs at obase), packed
                           // with their exclusive popcount prefix: [2 w] bits, [2 w + 1] prefix
  uint64_t ocap;           // bitmap words of obits
  uint32_t chunk;          // samples per K1/K3 chunk
  uint32_t vchunk;         // voxels per K4 chunk
  int mode;
  int exact_sums;          // average: u64 sums (fallback) instead of f32 vector reductions
  uint64_t seed;
};
int launch_voxelize_front(const VoxLevel& L, int sms, cudaStream_t s);
int launch_voxelize_accumulate(const VoxLevel& L, int sms, cudaStream_t s);
int launch_voxelize_back(const VoxLevel& L, int sms, ScanScratch& scr, cudaStream_t s);
uint32_t voxelize_acc_bytes(int mode, bool exact_sums);
int launch_voxelize_import(const VoxLevel& L, uint32_t slot_base, cudaStream_t s);
uint32_t voxelize_chunk(uint32_t nodes);
uint32_t voxelize_vchunk(uint32_t nodes);
uint64_t voxelize_chunk_capacity(uint64_t samples, uint32_t nodes);
uint64_t voxelize_vchunk_capacity(uint64_t voxels, uint32_t nodes);

// --- multi-GPU helpers (dist_kernels.cu) ---
// per-leaf counts of this process's points from its saved (pre all-reduce) counting grids
int launch_local_leaf_counts(const SplitView& v, const uint32_t* local_main, const uint32_t* local_ext,
                             const uint32_t* round_first, const uint32_t* round_count, const int* round_ext,
                             const uint64_t* round_pyr_base, int n_rounds, cudaStream_t s);
// copy nseg record segments (src, dst, count in records; rec_bytes 16 or 32)
int launch_copy_segments(const void* src, void* dst, const uint64_t* seg_src, const uint64_t* seg_dst,
                         const uint32_t* seg_cnt, uint64_t nseg, int rec_bytes, cudaStream_t s);

// --- VLPC payload (encode.cu) ---
int launch_encode(int fmt, const SplitView& v, const void* leaf_pts, const uint2* vox, const int32_t* order,
                  const uint64_t* offs, uint32_t n, uint8_t* out, cudaStream_t s);

// --- ingest + structural checks (ingest_checks.cu) ---
int launch_ingest_las(const void* raw, uint64_t n, uint32_t reclen, int32_t rgb_off, const double* scale,
                      const double* offset, void* out, cudaStream_t s);
int launch_ingest_ply(const void* raw, uint64_t n, uint32_t stride, const int32_t* types, const uint32_t* offs,
                      int has_rgb, int fmt, void* out, cudaStream_t s);
int launch_checks(int fmt, const SplitView& v, const void* leaf_pts, const uint2* vox, int voxels, uint32_t T,
                  int max_depth, uint8_t* flags, cudaStream_t s);

// --- generators (generate.cu) ---
int launch_f32_exact(const double* xyz, uint64_t n, uint32_t* flag, cudaStream_t s);
int launch_pack(const void* xyz, bool f64_in, const uint8_t* rgb, uint64_t n, int out_format, void* out,
                cudaStream_t s);
int launch_export_runs(const void* vox, const uint64_t* n_first, const uint32_t* n_count, const int32_t* d_nodes,
                       const uint64_t* d_off, uint32_t n, void* out, cudaStream_t s);
int launch_generate(int kind, uint64_t seed, uint64_t start, uint64_t n, void* out, const double* table,
                    cudaStream_t s);

}  // namespace lod
