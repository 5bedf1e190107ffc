// Microbenchmark: global float-vector reduction throughput (RED.E.ADD.F32x4) on B200,
// random addresses inside a small (L2-resident) gradient buffer, as in k_fwdbwd's pass 2.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void red4(float* a, float x, float y, float z, float w) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}
__device__ __forceinline__ uint32_t hash(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
template <int V>
__global__ void k(float* buf, uint32_t nvec, int n, int rep) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t h = hash(i);
    for (int r = 0; r < rep; ++r) {
      float* a = buf + 12 * ((h + r * 7919u) % nvec);
      if (V == 3) { red4(a, 1, 1, 1, 1); red4(a + 4, 1, 1, 1, 1); red4(a + 8, 1, 1, 1, 1); }
      else atomicAdd(a, 1.f);
    }
  }
}
int main() {
  const uint32_t nvec = 87040;            // cfg2 Gaussians
  float* buf; cudaMalloc(&buf, nvec * 48); cudaMemset(buf, 0, nvec * 48);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int n = 3500000;
  for (int v : {3, 1}) {
    for (int w = 0; w < 2; ++w) { if (v == 3) k<3><<<148 * 8, 256>>>(buf, nvec, n, 1); else k<1><<<148 * 8, 256>>>(buf, nvec, n, 1); }
    cudaEventRecord(a);
    if (v == 3) k<3><<<148 * 8, 256>>>(buf, nvec, n, 1); else k<1><<<148 * 8, 256>>>(buf, nvec, n, 1);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%s: %d groups in %.1f us -> %.1f G ops/s\n", v == 3 ? "3x RED.v4 (48B)" : "1x RED f32", n, ms * 1e3,
           n * (v == 3 ? 3.0 : 1.0) / (ms * 1e-3) / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
