// Read-bandwidth probe: how fast can one kernel stream N x 16-B records on this B200?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void rd(const uint4* p, uint64_t n, unsigned* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned acc = 0;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = __ldg(p + min(i0 + u * stride, n - 1));
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= r[u].x ^ r[u].y ^ r[u].z ^ r[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int U>
__global__ void rd_blk(const uint4* p, uint64_t n, unsigned* out) {  // contiguous block-tile per CTA
  const uint64_t tile = (uint64_t)blockDim.x * U;
  unsigned acc = 0;
  for (uint64_t b = (uint64_t)blockIdx.x * tile; b < n; b += (uint64_t)gridDim.x * tile) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = __ldg(p + min(b + u * blockDim.x + threadIdx.x, n - 1));
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= r[u].x ^ r[u].y ^ r[u].z ^ r[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void cp(const uint4* a, uint4* b, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) b[i] = a[i];
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (uint64_t mb : {320ull, 2048ull}) {
    uint64_t n = mb * 1000000ull / 16;
    uint4 *a, *b;
    unsigned* o;
    cudaMalloc(&a, n * 16);
    cudaMalloc(&b, n * 16);
    cudaMalloc(&o, 4);
    cudaMemset(a, 1, n * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch, double bytes) {
      for (int w = 0; w < 3; ++w) launch();
      cudaEventRecord(e0);
      for (int i = 0; i < 10; ++i) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%5llu MB %-28s %8.1f us  %7.0f GB/s\n", (unsigned long long)mb, name, ms * 100, bytes / (ms / 10) / 1e6);
    };
    for (int bpsm : {4, 8, 16, 32}) {
      char nm[64];
      snprintf(nm, 64, "rd<1> 256t x %d/SM", bpsm);
      run(nm, [&] { rd<1><<<sms * bpsm, 256>>>(a, n, o); }, n * 16.0);
      snprintf(nm, 64, "rd<4> 256t x %d/SM", bpsm);
      run(nm, [&] { rd<4><<<sms * bpsm, 256>>>(a, n, o); }, n * 16.0);
      snprintf(nm, 64, "rd_blk<8> 256t x %d/SM", bpsm);
      run(nm, [&] { rd_blk<8><<<sms * bpsm, 256>>>(a, n, o); }, n * 16.0);
    }
    run("rd_blk<8> 512t grid=n/4096", [&] { rd_blk<8><<<(n + 4095) / 4096, 512>>>(a, n, o); }, n * 16.0);
    run("copy 256t x 8/SM", [&] { cp<<<sms * 8, 256>>>(a, b, n); }, n * 32.0);
    cudaFree(a);
    cudaFree(b);
  }
  return 0;
}
