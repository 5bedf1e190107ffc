// Microbenchmark: throughput of per-sample cell-count atomics on B200 (keys kernel design).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

__global__ void k_ret(const uint32_t* key, int n, uint32_t* cnt, uint32_t* rank) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    rank[i] = atomicAdd(cnt + key[i], 1u);
}
__global__ void k_red(const uint32_t* key, int n, uint32_t* cnt, uint32_t* rank) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    atomicAdd(cnt + key[i], 1u); rank[i] = 0;
  }
}
template <int U>
__global__ void k_retU(const uint32_t* key, int n, uint32_t* cnt, uint32_t* rank) {
  int t = blockIdx.x * blockDim.x + threadIdx.x, T = gridDim.x * blockDim.x;
  for (int i0 = t; i0 < n; i0 += T * U) {
    uint32_t k[U], r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) k[u] = (i0 + u * T < n) ? key[i0 + u * T] : 0xFFFFFFFFu;
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = k[u] != 0xFFFFFFFFu ? atomicAdd(cnt + k[u], 1u) : 0;
#pragma unroll
    for (int u = 0; u < U; ++u) if (i0 + u * T < n) rank[i0 + u * T] = r[u];
  }
}
__global__ void k_copy(const uint32_t* key, int n, uint32_t* cnt, uint32_t* rank) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) rank[i] = key[i];
}

int main(int argc, char** argv) {
  int n = 2073600, cells = 120000;
  std::vector<uint32_t> h;
  if (argc > 2) {
    n = atoi(argv[2]); cells = atoi(argv[3]);
    h.resize(n);
    FILE* f = fopen(argv[1], "rb"); fread(h.data(), 4, n, f); fclose(f);
    printf("real keys n=%d cells=%d\n", n, cells);
  } else {
    h.resize(n);
    std::mt19937 g(1);
    for (int i = 0; i < n; ++i) h[i] = g() % cells;
  }
  uint32_t *key, *cnt, *rank;
  cudaMalloc(&key, n * 4); cudaMalloc(&cnt, cells * 4); cudaMalloc(&rank, n * 4);
  cudaMemcpy(key, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, void (*k)(const uint32_t*, int, uint32_t*, uint32_t*), int grid, int block) {
    for (int w = 0; w < 3; ++w) { cudaMemset(cnt, 0, cells * 4); k<<<grid, block>>>(key, n, cnt, rank); }
    cudaMemset(cnt, 0, cells * 4);
    cudaEventRecord(a); k<<<grid, block>>>(key, n, cnt, rank); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-12s grid %6d: %8.1f us  (%.2f G atom/s)\n", name, grid, ms * 1e3, n / (ms * 1e-3) / 1e9);
  };
  for (int grid : {148 * 8, 148 * 32, (n + 255) / 256}) {
    run("copy", k_copy, grid, 256);
    run("red", k_red, grid, 256);
    run("ret", k_ret, grid, 256);
    run("ret_u4", k_retU<4>, grid, 256);
    run("ret_u8", k_retU<8>, grid, 256);
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
