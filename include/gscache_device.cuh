/*
 * gscache_device.cuh -- device-callable renderer-side helpers of the GSCache path tracer
 * (next row f3 of SURVEY 8(f)); header-only, for the renderer's own CUDA kernels, and run in
 * batch by gc_alg1_terminate (include/gscache.h).
 *
 * gc_alg1: the early path-termination heuristic of Algorithm 1 (sec.3.3.2) with the
 * throughput importance sampling and the cascaded cache-radiance probability beta of
 * sec.3.4.1-3.4.2:
 *
 *   Tr_out <- prod_{k=1..n} sigma_k                       (RGB path attenuation)
 *   Tr     <- clamp(C * luminance(Tr_out), 0, 1)
 *   if Tr < 0.9:                                          ("throughput values less than 0.9")
 *     q ~ U(0,1)                                          (drawn by the caller, passed in)
 *     p <- 1 - Tr
 *     if q < p: return TERMINATE                          (read the cache at this level)
 *     Tr_out <- Tr_out / (Tr + eps)
 *     beta_{n+1} <- beta_n * Tr
 *   return CONTINUE
 *
 * Readings (A22): luminance = Rec. 709 / sRGB weights (0.2126, 0.7152, 0.0722)
 * (the paper names "luminance" only); eps is an argument (the paper leaves it unnamed;
 * default 1e-6 in gc_alg1_terminate's documentation); on the Tr >= 0.9 path and on
 * termination beta_{n+1} = beta_n and Tr_out = the plain product (Alg. 1 assigns neither
 * there).  On a cache hit at depth n the renderer weights the cached radiance by
 * prod sigma / beta_{n-1} (Eq. 3) -- gc_query_radiance's epilogue.
 *
 * Arithmetic: fp32, every product / sum rounded on its own in the written order
 * (__fmul_rn / __fadd_rn, no FMA contraction), so the termination decision q < 1 - Tr is
 * reproducible bit for bit by an fp32 reference taking the same steps.
 */
#ifndef GSCACHE_DEVICE_CUH_
#define GSCACHE_DEVICE_CUH_

#include <cuda_runtime.h>

struct gc_alg1_result {
  int terminate;        /* 1: terminate the path into the cache at this vertex */
  float tr_out[3];      /* effective path throughput weight (RGB) */
  float beta_next;      /* beta_{n+1} */
};

/* sigma: n RGB albedos sigma_1..sigma_n (sigma[3k + c]); C: termination coefficient; beta_n;
 * q: the uniform random number in [0, 1); eps: the importance-sampling guard. */
__device__ inline gc_alg1_result gc_alg1(const float* sigma, int n, float C, float beta_n, float q, float eps) {
  gc_alg1_result r;
  float t0 = 1.f, t1 = 1.f, t2 = 1.f;
  for (int k = 0; k < n; ++k) {
    t0 = __fmul_rn(t0, sigma[3 * k]); t1 = __fmul_rn(t1, sigma[3 * k + 1]); t2 = __fmul_rn(t2, sigma[3 * k + 2]);
  }
  const float lum = __fadd_rn(__fadd_rn(__fmul_rn(0.2126f, t0), __fmul_rn(0.7152f, t1)), __fmul_rn(0.0722f, t2));
  float tr = __fmul_rn(C, lum);
  tr = tr < 0.f ? 0.f : (tr > 1.f ? 1.f : tr);      /* clamp(., 0, 1) */
  r.terminate = 0;
  r.tr_out[0] = t0; r.tr_out[1] = t1; r.tr_out[2] = t2;
  r.beta_next = beta_n;
  if (tr < 0.9f) {
    const float p = 1.f - tr;
    if (q < p) { r.terminate = 1; return r; }
    const float d = __fadd_rn(tr, eps);
    r.tr_out[0] = __fdiv_rn(t0, d); r.tr_out[1] = __fdiv_rn(t1, d); r.tr_out[2] = __fdiv_rn(t2, d);
    r.beta_next = __fmul_rn(beta_n, tr);
  }
  return r;
}

#endif /* GSCACHE_DEVICE_CUH_ */
