// alg1.cu -- batch runner of the device-callable Algorithm 1 helper (include/gscache_device.cuh;
// next row f3, Alg. 1, sec.3.4): one thread per path.
#include "../../include/gscache_device.cuh"
#include "common.cuh"

namespace gsc {

__global__ void k_alg1(const float* __restrict__ sigma, const int32_t* __restrict__ n, int nmax, float C,
                       const float* __restrict__ beta, const float* __restrict__ q, float eps, int64_t P,
                       int32_t* terminate, float* tr_out, float* beta_next) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const int ni = min(max(n[i], 0), nmax);
    const gc_alg1_result r = gc_alg1(sigma + 3 * (size_t)nmax * i, ni, C, beta ? beta[i] : 1.f, q[i], eps);
    terminate[i] = r.terminate;
    tr_out[3 * i] = r.tr_out[0]; tr_out[3 * i + 1] = r.tr_out[1]; tr_out[3 * i + 2] = r.tr_out[2];
    beta_next[i] = r.beta_next;
  }
}

}  // namespace gsc

extern "C" gc_status gc_alg1_terminate(const float* sigma, const int32_t* n, int nmax, float C, const float* beta,
                                       const float* q, float eps, int64_t P, int32_t* terminate, float* tr_out,
                                       float* beta_next, gc_stream stream) {
  if (P < 0 || nmax < 0 || (P > 0 && (!sigma || !n || !q || !terminate || !tr_out || !beta_next)))
    return GC_ERR_ARG;
  if (P == 0) return GC_OK;
  const int blocks = (int)std::min<int64_t>((P + 255) / 256, 148 * 8);
  gsc::k_alg1<<<blocks, 256, 0, (cudaStream_t)stream>>>(sigma, n, nmax, C, beta, q, eps, P, terminate, tr_out,
                                                        beta_next);
  return cudaGetLastError() == cudaSuccess ? GC_OK : GC_ERR_CUDA;
}
