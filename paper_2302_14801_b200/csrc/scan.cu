#include "scan.cuh"

namespace lod {

__global__ void __launch_bounds__(1024) k_scan_sums(uint64_t* sums, uint32_t nb, const uint64_t* base_in,
                                                    uint64_t* total_out) {
  pdl_wait();
  __shared__ uint64_t sm[1024 / 32 + 1];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = base_in ? *base_in : 0;
  __syncthreads();
  for (uint32_t b0 = 0; b0 < nb; b0 += 1024) {
    uint32_t i = b0 + threadIdx.x;
    uint64_t v = (i < nb) ? sums[i] : 0;
    uint64_t tot;
    uint64_t ex = block_excl_scan<uint64_t, 1024>(v, &tot, sm);
    if (i < nb) sums[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total_out) *total_out = carry;
}

}  // namespace lod
