// Multi-GPU helpers: local per-leaf counts, record segment copies (pack / unpack of the
// subtree exchange) and the export of subtree-root voxel runs.  The collectives themselves
// are comm.cu (NCCL).
#include "kernels.h"

namespace lod {

namespace {

constexpr int kT = 256;

__global__ void k_local_main(SplitView v, const uint32_t* local_main) {
  pdl_wait();
  const uint64_t cells = 1ull << (3 * v.D);
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t n = local_main[c];
    if (!n) continue;
    const int32_t t = v.t8[c];
    if (t >= 0) atomicAdd(v.leaf_count + t, n);  // anchors (t <= -2) are counted in their grids
  }
}

__global__ void k_local_ext(SplitView v, const uint32_t* local_ext, uint32_t first, uint32_t count, int ext,
                            uint64_t pyr_base, uint64_t main_cells) {
  pdl_wait();
  const uint64_t cells = 1ull << (3 * ext);
  const uint64_t total = cells * count;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = i / cells, r = i % cells;
    const ExtMeta& m = v.meta[first + e];
    // local_ext mirrors the extension part of the pyramid buffer (offset main_cells)
    const uint32_t n = local_ext[m.pyr_off - main_cells + level_off(ext) + r];
    if (!n) continue;
    const int32_t t = v.te[m.tgt_off + r];
    if (t >= 0) atomicAdd(v.leaf_count + t, n);
  }
  (void)pyr_base;
}

__global__ void k_copy_segments(const uint4* src, uint4* dst, const uint64_t* seg_src, const uint64_t* seg_dst,
                                const uint32_t* seg_cnt, uint64_t nseg, int vec) {
  pdl_wait();
  for (uint64_t g = blockIdx.x; g < nseg; g += gridDim.x) {
    const uint64_t a = seg_src[g] * vec, b = seg_dst[g] * vec, n = (uint64_t)seg_cnt[g] * vec;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) dst[b + i] = __ldg(src + a + i);
  }
}

// voxel runs (8-B units) of the listed nodes, concatenated: one CTA per run
__global__ void k_export_runs(const uint2* vox, const uint64_t* n_first, const uint32_t* n_count, const int32_t* nodes,
                              const uint64_t* dst_off, uint32_t n, uint2* out) {
  pdl_wait();
  for (uint32_t g = blockIdx.x; g < n; g += gridDim.x) {
    const int32_t k = nodes[g];
    const uint64_t a = n_first[k], b = dst_off[g];
    const uint32_t c = n_count[k];
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) out[b + i] = __ldg(vox + a + i);
  }
}

}  // namespace

int launch_export_runs(const void* vox, const uint64_t* n_first, const uint32_t* n_count, const int32_t* d_nodes,
                       const uint64_t* d_off, uint32_t n, void* out, cudaStream_t s) {
  if (!n) return 0;
  launch_pdl(k_export_runs, std::min<uint32_t>(n, 148 * 16), kT, 0, s, reinterpret_cast<const uint2*>(vox), n_first,
             n_count, d_nodes, d_off, n, reinterpret_cast<uint2*>(out));
  return 1;
}

int launch_local_leaf_counts(const SplitView& v, const uint32_t* local_main, const uint32_t* local_ext,
                             const uint32_t* round_first, const uint32_t* round_count, const int* round_ext,
                             const uint64_t* round_pyr_base, int n_rounds, cudaStream_t s) {
  cudaMemsetAsync(v.leaf_count, 0, (size_t)v.n_leaves * 4, s);
  const uint64_t cells = 1ull << (3 * v.D);
  launch_pdl(k_local_main, (uint32_t)std::min<uint64_t>((cells + kT - 1) / kT, 148ull * 16), kT, 0, s, v, local_main);
  int launches = 1;
  const uint64_t main_cells = level_off(v.D + 1);
  for (int r = 0; r < n_rounds; ++r) {
    if (!round_count[r]) continue;
    const uint64_t total = (uint64_t)round_count[r] << (3 * round_ext[r]);
    launch_pdl(k_local_ext, (uint32_t)std::min<uint64_t>((total + kT - 1) / kT, 148ull * 16), kT, 0, s, 
        v, local_ext, round_first[r], round_count[r], round_ext[r], round_pyr_base[r], main_cells);
    ++launches;
  }
  return launches;
}

int launch_copy_segments(const void* src, void* dst, const uint64_t* seg_src, const uint64_t* seg_dst,
                         const uint32_t* seg_cnt, uint64_t nseg, int rec_bytes, cudaStream_t s) {
  if (!nseg) return 0;
  const uint32_t blocks = (uint32_t)std::min<uint64_t>(nseg, 148ull * 16);
  launch_pdl(k_copy_segments, blocks, kT, 0, s, reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), seg_src,
                                        seg_dst, seg_cnt, nseg, rec_bytes / 16);
  return 1;
}

}  // namespace lod
