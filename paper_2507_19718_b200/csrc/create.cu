// create.cu -- gc_create's device work (C7): gather of the nested level subsets, Eq. 2
// initial scales from a brute-force fp64 3-NN search, and the pack/unpack of the
// paper-order parameter layout used by gc_params / gc_set_params.
#include "common.cuh"
#include "kernels.h"

namespace gsc {

__global__ void k_gather_init(int64_t N0, const float* __restrict__ pos, const float* __restrict__ rgb,
                              const float* __restrict__ log_scale, const int64_t* __restrict__ src,
                              int64_t G, float* P, float logit) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < G; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = src[j];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      P[(P_MU + a) * G + j] = pos[3 * i + a];
      P[(P_C + a) * G + j] = rgb[3 * i + a];
      P[(P_S + a) * G + j] = log_scale ? log_scale[3 * i + a] : 0.f;
    }
    P[P_Q * G + j] = 1.f; P[(P_Q + 1) * G + j] = 0.f; P[(P_Q + 2) * G + j] = 0.f; P[(P_Q + 3) * G + j] = 0.f;
    P[P_O * G + j] = logit;
  }
}

// dbar_i = mean distance to the 3 nearest other points of the level (fp64, no contraction,
// comparisons in the oracle's order so the distances and their mean are bit-identical).
__global__ void __launch_bounds__(256) k_knn3(const float* __restrict__ P, int64_t G, int64_t base,
                                              int64_t n, double* dbar) {
  __shared__ double sx[256], sy[256], sz[256];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double xi = 0, yi = 0, zi = 0;
  if (i < n) { xi = P[P_MU * G + base + i]; yi = P[(P_MU + 1) * G + base + i]; zi = P[(P_MU + 2) * G + base + i]; }
  double b0 = INFINITY, b1 = INFINITY, b2 = INFINITY;
  for (int64_t t0 = 0; t0 < n; t0 += 256) {
    __syncthreads();
    const int64_t jl = t0 + threadIdx.x;
    if (jl < n) {
      sx[threadIdx.x] = P[P_MU * G + base + jl]; sy[threadIdx.x] = P[(P_MU + 1) * G + base + jl];
      sz[threadIdx.x] = P[(P_MU + 2) * G + base + jl];
    }
    __syncthreads();
    const int m = (int)((n - t0) < 256 ? (n - t0) : 256);
    if (i < n) {
      for (int k = 0; k < m; ++k) {
        if (t0 + k == i) continue;
        const double dx = __dsub_rn(sx[k], xi), dy = __dsub_rn(sy[k], yi), dz = __dsub_rn(sz[k], zi);
        // squared distances are ranked (the correctly rounded sqrt is monotone, so the three
        // smallest distances are the square roots of the three smallest squares: exact)
        const double d = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
        if (d < b2) {
          if (d < b1) { b2 = b1; if (d < b0) { b1 = b0; b0 = d; } else { b1 = d; } }
          else b2 = d;
        }
      }
    }
  }
  if (i < n) {
    const int k = (int)((n - 1) < 3 ? (n - 1) : 3);
    double s = 0.0;
    if (k >= 1) s = __dadd_rn(s, __dsqrt_rn(b0));
    if (k >= 2) s = __dadd_rn(s, __dsqrt_rn(b1));
    if (k >= 3) s = __dadd_rn(s, __dsqrt_rn(b2));
    dbar[i] = k > 0 ? __ddiv_rn(s, (double)k) : 0.0;
  }
}

// One thread, sequential in index order (same rounding sequence as the oracle): mean and
// population std of dbar, the level's AABB diagonal, then cap = mu + zcap * sigma.
__global__ void k_eq2_stats(const float* __restrict__ P, int64_t G, int64_t base, int64_t n,
                            const double* __restrict__ dbar, double zcap, double* out /*cap, floor*/) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double mu = 0.0;
  for (int64_t i = 0; i < n; ++i) mu = __dadd_rn(mu, dbar[i]);
  mu = __ddiv_rn(mu, (double)n);
  double var = 0.0;
  for (int64_t i = 0; i < n; ++i) { const double d = __dsub_rn(dbar[i], mu); var = __dadd_rn(var, __dmul_rn(d, d)); }
  var = __ddiv_rn(var, (double)n);
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      const double v = P[(P_MU + a) * G + base + i];
      if (v < lo[a]) lo[a] = v;
      if (v > hi[a]) hi[a] = v;
    }
  const double dx = __dsub_rn(hi[0], lo[0]), dy = __dsub_rn(hi[1], lo[1]), dz = __dsub_rn(hi[2], lo[2]);
  const double diag = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
  out[0] = __dadd_rn(mu, __dmul_rn(zcap, __dsqrt_rn(var)));
  out[1] = __dmul_rn(1e-6, diag);
}

__global__ void k_eq2_apply(int64_t n, const double* __restrict__ dbar, const double* __restrict__ capfl,
                            double factor, float* P, int64_t G, int64_t base) {
  const double cap = capfl[0], fl = capfl[1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double r = dbar[i] > fl ? dbar[i] : fl;
    const double s = __dmul_rn(cap < r ? cap : r, factor);
    const float ls = (float)log(s);
    P[P_S * G + base + i] = ls; P[(P_S + 1) * G + base + i] = ls; P[(P_S + 2) * G + base + i] = ls;
  }
}

// paper layout segments of one level: pos [n][3] | rot [n][4] | color [n][3] | log_scale [n][3] | opacity [n]
__global__ void k_pack(const float* __restrict__ P, int64_t G, int64_t base, int64_t n, float* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int a = 0; a < 3; ++a) out[3 * i + a] = P[(P_MU + a) * G + base + i];
    for (int a = 0; a < 4; ++a) out[3 * n + 4 * i + a] = P[(P_Q + a) * G + base + i];
    for (int a = 0; a < 3; ++a) out[7 * n + 3 * i + a] = P[(P_C + a) * G + base + i];
    for (int a = 0; a < 3; ++a) out[10 * n + 3 * i + a] = P[(P_S + a) * G + base + i];
    out[13 * n + i] = P[P_O * G + base + i];
  }
}

__global__ void k_unpack(const float* __restrict__ in, int64_t G, int64_t base, int64_t n, float* P) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int a = 0; a < 3; ++a) P[(P_MU + a) * G + base + i] = in[3 * i + a];
    for (int a = 0; a < 4; ++a) P[(P_Q + a) * G + base + i] = in[3 * n + 4 * i + a];
    for (int a = 0; a < 3; ++a) P[(P_C + a) * G + base + i] = in[7 * n + 3 * i + a];
    for (int a = 0; a < 3; ++a) P[(P_S + a) * G + base + i] = in[10 * n + 3 * i + a];
    P[P_O * G + base + i] = in[13 * n + i];
  }
}

static int blocks_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

void launch_gather_init(int64_t N0, const float* pos, const float* rgb, const float* log_scale,
                        const int64_t* src, int64_t G, float* P, float opacity_logit, cudaStream_t s) {
  k_gather_init<<<blocks_for(G), 256, 0, s>>>(N0, pos, rgb, log_scale, src, G, P, opacity_logit);
}

void launch_eq2_level(const float* P, int64_t G, int64_t base, int64_t n, double* dbar, double* capfl,
                      double zcap, double factor, float* Pw, cudaStream_t s) {
  k_knn3<<<(int)((n + 255) / 256), 256, 0, s>>>(P, G, base, n, dbar);
  k_eq2_stats<<<1, 32, 0, s>>>(P, G, base, n, dbar, zcap, capfl);
  k_eq2_apply<<<blocks_for(n), 256, 0, s>>>(n, dbar, capfl, factor, Pw, G, base);
}

void launch_pack(const float* P, int64_t G, int64_t base, int64_t n, float* out, cudaStream_t s) {
  k_pack<<<blocks_for(n), 256, 0, s>>>(P, G, base, n, out);
}

void launch_unpack(const float* in, int64_t G, int64_t base, int64_t n, float* P, cudaStream_t s) {
  k_unpack<<<blocks_for(n), 256, 0, s>>>(in, G, base, n, P);
}

}  // namespace gsc
