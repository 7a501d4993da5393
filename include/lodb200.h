/*
 * lodb200 -- C ABI of the B200-native LOD-construction path.
 *
 * Drop-in boundary for the reference's two-stage Python API
 *   partition(cloud, config) -> Octree        pkg/src/lodforge/partition.py:300-302
 *     (+ forced world bounds: Partitioner(cloud, config, bounds), partition.py:82,87)
 *   build_lod(tree, strategy, seed) -> Octree  pkg/src/lodforge/sampling.py:165-176
 * and of the north-star fused form build_lod(points, colors, T, grid, mode).
 *
 * Conventions
 *  - Plain pointers and sizes only.  Point buffers are DEVICE pointers to packed records
 *    (see lod_point_format); the library never frees caller memory.
 *  - Calls are synchronous with respect to the given CUDA stream (passed as void*,
 *    NULL = legacy default stream) and return a status code; lod_last_error() gives the
 *    message of the last failure on the calling thread.
 *  - A lod_tree owns its device buffers (leaf points, voxels, node table, scratch) and
 *    reuses them across builds (grow-only), so repeated builds do not allocate.
 *  - Not reentrant per lod_tree; distinct trees may be used from distinct threads.
 *
 * Status codes map to the reference's exceptions at the Python boundary:
 *   LOD_EVALUE        -> ValueError        (empty cloud, non-finite bounds, bad config,
 *                                            unknown strategy; model.py:118-124,202-205,
 *                                            partition.py:83-84, sampling.py:169-170)
 *   LOD_ECONSISTENCY  -> ConsistencyError  (2^20 random limit sampling.py:73-75, internal
 *                                            invariants partition.py:170,191,224,239,260,269,286)
 *   LOD_ECUDA         -> RuntimeError      (CUDA / NCCL failure)
 *   LOD_EUNSUPPORTED  -> NotImplementedError (configs outside the supported envelope)
 */
#ifndef LODB200_H
#define LODB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOD_OK 0
#define LOD_EVALUE 1
#define LOD_ECONSISTENCY 2
#define LOD_ECUDA 3
#define LOD_EUNSUPPORTED 4

/* Point record layouts (device). */
enum lod_point_format {
  LOD_POINTS_F32 = 0, /* 16 B: float x, y, z; uint8 r, g, b, pad */
  LOD_POINTS_F64 = 1  /* 32 B: double x, y, z; uint8 r, g, b, pad[5] */
};

/* Voxel sampling strategies (model.py:127 STRATEGIES). */
enum lod_mode {
  LOD_MODE_RANDOM = 0,     /* sampling.py:69-85 */
  LOD_MODE_AVERAGE = 1,    /* sampling.py:88-97 ("color_filter") */
  LOD_MODE_FIRST_COME = 2, /* sampling.py:61-66, the reference default (model.py:115); voxels
                              listed by winning sample ordinal, not by key */
  LOD_MODE_WEIGHTED = 3    /* sampling.py:100-133; colours within +-1 per channel of the
                              reference's sequential fp64 sums */
};

/* BuildConfig (model.py:108-124). grid_size is not a field: the reference never reads it. */
typedef struct lod_config {
  uint32_t T;              /* max points per non-oversized leaf, >= 1 */
  int32_t initial_depth;   /* main counting grid depth (8 -> 256^3), 0..10 */
  int32_t extension_depth; /* levels per extension round, 1..5 */
  int32_t max_depth;       /* initial_depth..16 */
} lod_config;

/* Summary of a built tree. */
typedef struct lod_tree_info {
  uint64_t n_points;
  uint64_t n_voxels;       /* sum of inner-node voxels after lod_voxelize, else 0 */
  uint32_t n_nodes;
  uint32_t n_leaves;
  uint32_t n_inner;
  uint32_t depth;          /* deepest node depth */
  int32_t point_format;
  int32_t voxel_mode;      /* -1 until lod_voxelize succeeded */
  double world_min[3];
  double world_size;
  uint32_t n_ext_grids;    /* extension pyramids created (partition.py:109-151) */
  uint32_t radix_passes;   /* stable-distribute passes used */
} lod_tree_info;

/* One node of the exported node table (DFS-independent order: main pyramid levels
 * coarse->fine, then extension pyramids).  Node 0 is the root. */
typedef struct lod_node {
  double min[3];           /* bounds_at(world, path) min, sequential fp64 adds (model.py:62-81) */
  double size;
  uint64_t first;          /* leaf: first point in the leaf buffer; inner: first voxel */
  uint32_t count;          /* leaf: points; inner: voxels (0 before lod_voxelize) */
  int32_t parent;          /* -1 for the root */
  uint16_t cell[3];        /* absolute cell coordinates at `depth`; path digits are its bits */
  uint8_t depth;
  uint8_t flags;           /* bit0 leaf, bit1 oversized (partition.py:222) */
  int32_t child[8];        /* node ids by octant, -1 if absent */
} lod_node;

typedef struct lod_tree lod_tree;

/* Handle lifecycle.  `device` is the CUDA ordinal the tree's buffers live on.  Calls on one
 * tree must not overlap; different trees may build concurrently on different streams (a tree
 * owns a private stream for its voxelize overlap and a small pinned, device-mapped status
 * block, so its host reads never wait behind other streams' bulk copies). */
lod_tree* lod_tree_create(int device);
void lod_tree_destroy(lod_tree* tree);

/* partition(): split n points (device records of `format`) into leaves of <= T points.
 * bounds_or_null: NULL -> cubic world bounds of the points (model.py:199-209); else
 * {min_x, min_y, min_z, size} forced bounds (points outside -> LOD_ECONSISTENCY). */
int lod_split(lod_tree* tree, const void* d_points, uint64_t n, int format,
              const double* bounds_or_null, const lod_config* config, void* stream);

/* build_lod(tree, strategy, seed): fill every inner node with voxels, deepest first. */
int lod_voxelize(lod_tree* tree, int mode, uint64_t seed, void* stream);

/* north-star fused build: lod_split (world bounds) + lod_voxelize. */
int lod_build(lod_tree* tree, const void* d_points, uint64_t n, int format,
              const lod_config* config, int mode, uint64_t seed, void* stream);

int lod_tree_get_info(const lod_tree* tree, lod_tree_info* out);

/* Copy the node table to host memory (n_nodes entries). */
int lod_tree_copy_nodes(const lod_tree* tree, lod_node* host_nodes, void* stream);

/* Device pointers of the outputs (valid until the next build on this tree):
 * leaf points: n_points records of the input format, grouped by leaf, input order within
 *              a leaf (partition.py:262 stable order);
 * voxels: n_voxels x {uint32 key = (x*128 + y)*128 + z, uint32 rgb = r | g<<8 | b<<16},
 *         per inner node in the reference's stored order: ascending key (random, average,
 *         weighted: sampling.py:83-85, 97, 131-133) or ascending winning ordinal
 *         (first-come: sampling.py:64-66). */
int lod_tree_leaf_points(const lod_tree* tree, const void** d_ptr);
int lod_tree_voxels(const lod_tree* tree, const void** d_ptr);

/* Enqueue the whole tree's device->host copies on `stream` without waiting: leaf points,
 * voxels (stored order) and node table, each skipped when its pointer is NULL.  Host
 * buffers should be pinned; synchronize the stream before reading them.  Lets a caller
 * overlap the copies of build k with the upload / build of build k+1 (PCIe is duplex).
 * Copies of >= 512 MB go out as 256-MB pieces alternating between `stream` and the tree's
 * own copy stream (two copy engines), joined back into `stream`: ordered like one copy. */
int lod_tree_copy_async(const lod_tree* tree, void* h_leaf_points, void* h_voxels, lod_node* h_nodes,
                        void* stream);
/* The NEXT lod_split (or lod_dist_skeleton) on this tree makes its stream wait on `event` (a
 * cudaEvent_t) right before it rewrites the node table and the leaf buffer -- i.e. after its
 * bounds, count and extension rounds -- so a caller still downloading the previous build's
 * outputs (lod_tree_copy_async on another stream) overlaps that download with the next
 * build's first stages.  Voxels are rewritten by lod_voxelize, which the caller orders itself.
 * NULL clears it. */
int lod_tree_set_output_wait(lod_tree* tree, void* event);

/* Host copies of the outputs (sizes from lod_tree_get_info). */
int lod_tree_copy_leaf_points(const lod_tree* tree, void* host, void* stream);
int lod_tree_copy_voxels(const lod_tree* tree, void* host, void* stream);

/* Copy a range of one output to host memory and wait: what = 0 leaf points (records
 * [first, first+count) of the leaf buffer), what = 1 voxels (stored order).  With a node's
 * lod_node.first / count this fetches one node's points or voxels without the whole tree
 * (reference OctreeNode.point_positions / voxel_coords of a single node, model.py:130-168). */
int lod_tree_copy_range(const lod_tree* tree, int what, uint64_t first, uint64_t count, void* host,
                        void* stream);

/* VLPC payload (reference codec.py:28-47): for the n nodes h_order[i] (node ids, in the
 * file's path order, codec.py:51) write each node's records at byte h_offsets[i] of the
 * device buffer d_payload -- leaves 16-B {f32 offset from node min, rgb, pad}, inner nodes
 * 6-B {cx, cy, cz, r, g, b} in stored order.  Header and node table are host bytes
 * (paper_2302_14801_b200/codec.py). */
int lod_tree_encode_payload(const lod_tree* tree, const int32_t* h_order, const uint64_t* h_offsets,
                            uint32_t n, void* d_payload, void* stream);

/* Ingest (reference ingest.py:59-198): decode raw file records already in device memory.
 * LAS point formats 0-3 / 6-8: d_raw = n records of record_length bytes; x = X*scale+offset
 * per axis in fp64 (no FMA), colour = 16-bit channel >> 8 at rgb_offset (-1: grey 128);
 * output n LOD_POINTS_F64 records. */
int lod_ingest_las(const void* d_raw, uint64_t n, uint32_t record_length, int32_t rgb_offset,
                   const double* scale3, const double* offset3, void* d_records, void* stream);

/* PLY scalar property types (ingest.py:122-131). */
enum lod_ply_type { LOD_PLY_I8 = 0, LOD_PLY_U8 = 1, LOD_PLY_I16 = 2, LOD_PLY_U16 = 3, LOD_PLY_I32 = 4,
                    LOD_PLY_U32 = 5, LOD_PLY_F32 = 6, LOD_PLY_F64 = 7 };

/* binary_little_endian PLY vertex records (stride bytes each): types6/offsets6 give x, y, z,
 * red, green, blue; has_rgb = 0 -> grey 128.  out_format LOD_POINTS_F32 only when x, y, z
 * are float properties (exact), else LOD_POINTS_F64. */
int lod_ingest_ply(const void* d_raw, uint64_t n, uint32_t stride, const int32_t* types6,
                   const uint32_t* offsets6, int has_rgb, int out_format, void* d_records, void* stream);

/* Structural checks (reference checks.py:18-92) on the built tree against the config's T
 * and max_depth: per node (node-table order) a byte of LOD_CHECK_* failure bits in h_flags
 * (n_nodes entries). */
enum lod_check_bit {
  LOD_CHECK_CAPACITY = 1,      /* non-oversized leaf with > T points */
  LOD_CHECK_OVERSIZED = 2,     /* oversized leaf away from max_depth */
  LOD_CHECK_MAXIMALITY = 4,    /* inner node whose children are all leaves with < T points */
  LOD_CHECK_CONTAINMENT = 8,   /* empty leaf, or a point outside its node (+-size*1e-6) */
  LOD_CHECK_VOXEL_BOUNDS = 16, /* voxel coordinate outside the 128^3 grid */
  LOD_CHECK_UNIQUENESS = 32,   /* duplicate voxel cell */
  LOD_CHECK_EMPTY_INNER = 64,  /* inner node without voxels (after lod_voxelize) */
  LOD_CHECK_NO_CHILDREN = 128  /* inner node without children */
};
int lod_tree_checks(const lod_tree* tree, uint32_t T, int32_t max_depth, uint8_t* h_flags, void* stream);

/* Device memory.  By default trees allocate with cudaMalloc (grow-only buffers, freed by
 * lod_tree_destroy).  lod_set_allocator routes every later allocation through the caller's
 * pool instead (e.g. torch.cuda.caching_allocator_alloc, so the framework's allocator sees the
 * HBM the trees hold); both functions or neither; buffers are returned to the allocator that
 * made them, after a device synchronize.  Process-wide; set it before creating trees. */
typedef void* (*lod_alloc_fn)(uint64_t bytes, int device, void* ctx);
typedef void (*lod_free_fn)(void* ptr, uint64_t bytes, int device, void* ctx);
int lod_set_allocator(lod_alloc_fn alloc, lod_free_fn free_fn, void* ctx);

/* Planning estimate of the device bytes one build of n points needs (tree buffers, not the
 * input): an upper bound for surface-like clouds (voxels <= 1.5 n, <= 10% of the points in
 * extension grids); denser volumes grow the voxel arena on demand. */
int lod_workspace_bytes(uint64_t n, int format, const lod_config* config, int mode, uint64_t* bytes);

/* Device memory currently held by the tree, bytes. */
uint64_t lod_tree_device_bytes(const lod_tree* tree);

/* Per-stage device times of the last build in milliseconds (CUDA events), for profiling:
 * out[0] bounds+count, [1] extension, [2] merge+nodes+targets, [3] distribute, [4] voxelize;
 * NaN for a stage the last build did not bracket (the multi-GPU stage calls).
 * Timing is recorded only when enabled (small overhead from event records). */
int lod_set_timing(lod_tree* tree, int enabled);
int lod_tree_stage_ms(const lod_tree* tree, float* out5);

/* Device time of the dominant single kernel of the last build (timing enabled):
 * out[0] = the distribute's K_scatter, summed over its passes, milliseconds. */
int lod_tree_kernel_ms(const lod_tree* tree, float* out1);

/* Number of kernel launches issued by the last lod_split + lod_voxelize. */
uint64_t lod_tree_launches(const lod_tree* tree);

/* Pack caller arrays into point records on the device (the drop-in's upload path; the
 * reference's PointCloud is float64 (n,3) + uint8 (n,3), ingest.py:21-35).
 * d_xyz: n x 3 coordinates, float64 (xyz_is_f64 = 1) or float32; d_rgb: n x 3 uint8.
 * out_format: LOD_POINTS_F32, LOD_POINTS_F64, or -1 = F32 when every float64 coordinate
 * survives a float32 round trip (exact), else F64 (float32 input is always F32).
 * d_records must hold n records of the chosen format (32 B/pt covers both); *chosen_format
 * receives it.  Waits for the exactness test (one 4-byte read); the packing is enqueued. */
int lod_pack_points(const void* d_xyz, int xyz_is_f64, const uint8_t* d_rgb, uint64_t n, int out_format,
                    void* d_records, int* chosen_format, void* stream);

/* ---------------------------------------------------------------------------------
 * Stage-level access (the reference's Partitioner stages and module functions,
 * partition.py:36-287), for callers that drive count / extend / merge / targets / insert
 * one at a time: the single-GPU build runs through the lod_dist_* stages with one rank.
 * ------------------------------------------------------------------------------- */
/* merge_pyramid(finest, T) (partition.py:36-61): d_pyr holds the levels of one pyramid, level l
 * at (8^l - 1) / 7 u32 cells, x-major; the finest level L is the input (counts or 0xFFFFFFFF =
 * UNMERGEABLE); levels L-1..0 are computed in place and merged children zeroed. */
int lod_merge_pyramid(uint32_t* d_pyr, int L, uint32_t T, void* stream);
/* the main finest-grid key of every point (pkey: (cx * dim + cy) * dim + cz), n entries */
int lod_tree_copy_point_keys(const lod_tree* tree, uint32_t* h_keys, void* stream);
/* every counting pyramid of the last split (main pyramid at 0, extension pyramids at their
 * pyr_off), u32 per cell after the merge; h_cells NULL: *n_out = the number of cells */
int lod_tree_copy_pyramids(const lod_tree* tree, uint32_t* h_cells, uint64_t* n_out, void* stream);
typedef struct lod_ext_grid {
  uint64_t pyr_off;        /* its pyramid in the pyramid buffer (levels 0..ext) */
  uint16_t ax, ay, az;     /* anchor cell, absolute coordinates at depth base */
  uint8_t base, ext;       /* anchor depth, levels below it */
} lod_ext_grid;
/* the extension grids (partition.py:64-76 ExtendedPyramid), h NULL: *n_out = their number */
int lod_tree_ext_grids(const lod_tree* tree, lod_ext_grid* h, uint32_t* n_out, void* stream);
/* the extension points: input index and depth-16 cell (x | y << 16 | z << 32); h NULL: count */
int lod_tree_ext_points(const lod_tree* tree, uint32_t* h_index, uint64_t* h_cell16, uint64_t* n_out,
                        void* stream);

/* The reference's per-node sampling helpers on ONE node's sample list (sampling.py:21-133), for
 * callers driving the stages themselves:
 * lod_project_samples: one child's samples into the parent's 128^3 grid -- kind 0: n leaf points
 *   (f64 xyz) -> clip((p - min) / size * 128, 0, nextafter(128, 0)); kind 1: n child voxels
 *   (u8 xyz) in octant `octant` -> off + (c + 0.5) / 2; d_gpos: n x 3 f64 (sampling.py:29-44).
 * lod_extract: extract_first_come / _random / _average / _weighted (mode = lod_mode) on S grid
 *   positions (f64 x 3) + colours (u8 x 3); writes the m voxels' u8 coordinates and colours
 *   (buffers of S x 3 bytes) in the reference's stored order and *m_out.  random: seed and the
 *   node's path_hash (rng.py:48-53); raises the reference's 2^20 ConsistencyError. */
int lod_project_samples(int kind, const void* d_in, uint64_t n, const double* node_min3, double node_size,
                        int octant, double* d_gpos, void* stream);
int lod_extract(int mode, const double* d_gpos, const uint8_t* d_rgb, uint64_t S, uint64_t seed,
                uint64_t node_hash, uint8_t* d_coords, uint8_t* d_colors, uint64_t* m_out, void* stream);

/* Deterministic synthetic generators on the device, rows
 * [start, start+n) of cloud `kind` ("sphere", "terrain", "scene", "cluster", "surface")
 * written as LOD_POINTS_F32 records.  `table`: scene object table from the host
 * generator (65 x {kind, 7 params, cdf}) or NULL for the other kinds. */
int lod_generate(const char* kind, uint64_t seed, uint64_t start, uint64_t n, void* d_out,
                 const double* table_or_null, void* stream);

/* ---------------------------------------------------------------------------------
 * Multi-GPU stages (one process per GPU; the collectives run through lod_comm_* below --
 * NCCL on the build's stream -- or any equivalent the caller drives; see
 * paper_2302_14801_b200/dist.py).  Subtree sharding per
 * world bounds and counting grids are all-reduced, every rank derives the
 * identical node table, leaves are assigned to ranks by top-level subtree, points are
 * exchanged all-to-all (source-rank order keeps the global input order), each rank samples
 * its subtrees and rank 0 merges the coarsest levels from the imported subtree roots.
 * ------------------------------------------------------------------------------- */
typedef struct lod_span { void* ptr; uint64_t n; } lod_span; /* device array of uint32 */

/* init + local min xyz / max xyz of this rank's points (host out[6]; +inf/-inf if none) */
int lod_dist_begin(lod_tree* tree, const void* d_points, uint64_t n_local, int format,
                   const lod_config* config, double* out_min_max, void* stream);
/* count the local points in the GLOBAL cube world = {min xyz, size}; *out = the main
 * counting grid, to be all-reduced (SUM) in place before the next call */
int lod_dist_count(lod_tree* tree, uint64_t n_global, const double* world, lod_span* out, void* stream);
/* next extension round from the reduced counts; *out = its grids to all-reduce (SUM) in
 * place, out->n == 0 when no further round is needed (partition.py:109-151) */
int lod_dist_extend(lod_tree* tree, lod_span* out, void* stream);
/* merge + node table + targets on the reduced pyramids, then the stable local distribute;
 * h_local_leaf_counts (n_leaves) receives this rank's points per leaf */
int lod_dist_skeleton(lod_tree* tree, uint32_t* h_local_leaf_counts, void* stream);
/* this rank's points per leaf after lod_dist_skeleton / lod_dist_adopt (n_leaves entries) */
int lod_dist_leaf_counts(const lod_tree* tree, uint32_t* h_counts);
/* copy record segments (in records) from d_src to d_dst; NULL = the tree's leaf buffer */
int lod_dist_copy_segments(lod_tree* tree, const void* d_src, void* d_dst, const uint64_t* h_src,
                           const uint64_t* h_dst, const uint32_t* h_cnt, uint64_t nseg, void* stream);
/* the tree's leaf buffer grown to n records (contents undefined): receive the exchanged
 * records straight into it, then lod_dist_adopt(tree, that pointer, ...) adopts them in place
 * (call after the send buffer was packed from the old leaf buffer) */
int lod_dist_leaf_buffer(lod_tree* tree, uint64_t n, void** d_out);
/* make d_records (leaf-major, per-leaf counts h_leaf_counts) this rank's leaf buffer (copied,
 * or adopted in place when d_records is the pointer lod_dist_leaf_buffer returned) */
int lod_dist_adopt(lod_tree* tree, const void* d_records, uint64_t n, const uint32_t* h_leaf_counts,
                   void* stream);
/* voxelize the inner nodes with h_mask[node] = 1; append = keep earlier results; the
 * n_imp imported inner nodes (voxels concatenated in d_imp_vox, counts h_imp_counts) are
 * placed in the arena and made gatherable from parity slot imp_slot_base on */
int lod_dist_voxelize(lod_tree* tree, int mode, uint64_t seed, const uint8_t* h_mask, int append,
                      const int32_t* h_imp_nodes, const uint32_t* h_imp_counts, uint32_t n_imp,
                      uint32_t imp_slot_base, const void* d_imp_vox, void* stream);

/* the voxel runs of n inner nodes h_nodes[i], concatenated into d_out (8-B voxels, stored
 * order) in ONE launch; h_counts[i] receives each node's voxel count (the subtree roots a
 * rank sends to rank 0) */
int lod_dist_export_roots(lod_tree* tree, const int32_t* h_nodes, uint32_t n, void* d_out, uint32_t* h_counts,
                          void* stream);

/* ---------------------------------------------------------------------------------
 * NCCL communicator of the multi-GPU build (NVLink / NVSwitch), issued on the build's stream.
 * NCCL is loaded on first use (libnccl.so.2).  Bootstrap: rank 0 calls lod_comm_unique_id,
 * the caller broadcasts the 128 bytes (any host channel), every rank calls lod_comm_init.
 * dtype: 0 u32, 1 u64, 2 f64, 3 i64; op: 0 sum, 1 min, 2 max.
 * ------------------------------------------------------------------------------- */
typedef struct lod_comm lod_comm;
int lod_comm_unique_id(uint8_t* out128);
int lod_comm_init(const uint8_t* id128, int nranks, int rank, int device, lod_comm** out);
int lod_comm_destroy(lod_comm* comm);
int lod_comm_allreduce(lod_comm* comm, void* d_buf, uint64_t count, int dtype, int op, void* stream);
int lod_comm_allgather(lod_comm* comm, const void* d_send, void* d_recv, uint64_t bytes, void* stream);
/* grouped ncclSend / ncclRecv: send_bytes[q] consecutive bytes to rank q, recv_bytes[q] from
 * rank q, received in source-rank order (keeps each leaf's points in global input order) */
int lod_comm_alltoallv(lod_comm* comm, const void* d_send, const uint64_t* send_bytes, void* d_recv,
                       const uint64_t* recv_bytes, void* stream);
/* every rank sends `bytes`; `root` receives recv_bytes[q] from each q, in rank order */
int lod_comm_gatherv(lod_comm* comm, const void* d_send, uint64_t bytes, void* d_recv, const uint64_t* recv_bytes,
                     int root, void* stream);

/* Message of the last failure on the calling thread. */
const char* lod_last_error(void);

/* Library version string. */
const char* lod_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LODB200_H */
