// L2 atomic throughput probe: 20M random-address accumulations into 9M 16-B slots.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
__global__ void u64x2(unsigned long long* a, uint32_t n, uint32_t m) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t s = hsh(i) % m;
    atomicAdd(a + 2 * s, 0x100000001ull);
    atomicAdd(a + 2 * s + 1, 0x100000001ull);
  }
}
__global__ void u64x1(unsigned long long* a, uint32_t n, uint32_t m) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t s = hsh(i) % m;
    atomicAdd(a + 2 * s, 0x100000001ull);
  }
}
__global__ void f32x4(float* a, uint32_t n, uint32_t m) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t s = hsh(i) % m;
    float* p = a + 4 * s;
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(2.f), "f"(3.f), "f"(1.f) : "memory");
  }
}
__global__ void u32x4(unsigned* a, uint32_t n, uint32_t m) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t s = hsh(i) % m;
    atomicAdd(a + 4 * s, 1u); atomicAdd(a + 4 * s + 1, 2u); atomicAdd(a + 4 * s + 2, 3u); atomicAdd(a + 4 * s + 3, 1u);
  }
}
__global__ void st16(uint4* a, uint32_t n, uint32_t m) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t s = hsh(i) % m;
    a[s] = make_uint4(i, 1, 2, 3);
  }
}
// 16-B reductions where consecutive samples mostly hit nearby slots (spatially sorted input)
__global__ void f32x4_local(float* a, uint32_t n, uint32_t m) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t s = (uint32_t)(((uint64_t)i * m) / n) + (hsh(i) & 63);
    if (s >= m) s = m - 1;
    float* p = a + 4 * s;
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(2.f), "f"(3.f), "f"(1.f) : "memory");
  }
}
// count-grid pattern (k_count on cluster2B): 4-B REDs to `m` random cells spread over a 64 MB grid
__global__ void u32x1_grid(unsigned* a, uint32_t n, uint32_t m) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t s = (uint32_t)(((uint64_t)(hsh(i) % m) * 2654435761u) & ((1u << 24) - 1));
    atomicAdd(a + s, 1u);
  }
}
static void grid_reds() {
  const uint32_t n = 400000000;
  void* a; cudaMalloc(&a, (size_t)4 << 24); cudaMemset(a, 0, (size_t)4 << 24);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (uint32_t m : {200000u, 2000000u, 16000000u}) {
    for (int w = 0; w < 2; ++w) u32x1_grid<<<148 * 8, 256>>>((unsigned*)a, n, m);
    cudaEventRecord(e0); u32x1_grid<<<148 * 8, 256>>>((unsigned*)a, n, m); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("u32 REDs, %8u random cells of a 64 MB grid: %.2f ms for %u = %.1f G/s\n", m, ms, n, n / ms / 1e6);
  }
  cudaFree(a);
}
int main(int argc, char**) {
  if (argc > 1) { grid_reds(); return 0; }
  const uint32_t n = 20000000;
  for (uint32_t m : {5000000u, 1000000u, 100000u}) {
    void* a; cudaMalloc(&a, (size_t)m * 16); cudaMemset(a, 0, (size_t)m * 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* nm, auto f) {
      for (int w = 0; w < 2; ++w) f();
      cudaEventRecord(e0); for (int i = 0; i < 5; ++i) f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); printf("slots %8u %-10s %8.1f us\n", m, nm, ms * 200);
    };
    run("u64x2", [&] { u64x2<<<148 * 8, 256>>>((unsigned long long*)a, n, m); });
    run("u64x1", [&] { u64x1<<<148 * 8, 256>>>((unsigned long long*)a, n, m); });
    run("f32x4", [&] { f32x4<<<148 * 8, 256>>>((float*)a, n, m); });
    run("u32x4", [&] { u32x4<<<148 * 8, 256>>>((unsigned*)a, n, m); });
    run("st16", [&] { st16<<<148 * 8, 256>>>((uint4*)a, n, m); });
    run("f32x4loc", [&] { f32x4_local<<<148 * 8, 256>>>((float*)a, n, m); });
    cudaFree(a);
  }
}
