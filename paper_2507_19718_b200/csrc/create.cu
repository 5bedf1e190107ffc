// create.cu -- gc_create's device work (C7): gather of the nested level subsets, Eq. 2
// initial scales from an exact fp64 3-NN search over a uniform grid, and the
// pack/unpack of the paper-order parameter layout used by gc_params / gc_set_params.
#include <algorithm>
#include <cmath>
#include <vector>

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

// dbar_i = mean distance to the 3 nearest other points of the level (Eq. 2).
// Exact k-NN over a uniform grid (sub-quadratic, next row f2): the level's points are binned
// into ~n/2 cells, then each point visits cells in Chebyshev shells r = 0, 1, 2, ... around
// its own and stops once its third-smallest squared distance lies strictly below the squared
// distance to the unvisited region (minus a slack far above the rounding of the cell bounds),
// so the three smallest squared distances are those of the brute-force search.  They are
// computed in fp64 with the oracle's operation sequence (no contraction) and ranked by value:
// the multiset of the three smallest values, hence their square roots and mean summed in
// ascending order, are bit-identical to the oracle whatever the visiting order.

__global__ void __launch_bounds__(1024) k_knn_bbox(const float* __restrict__ P, int64_t G, int64_t base,
                                                   int64_t n, float* box /*lo[3], hi[3]*/) {
  __shared__ float slo[3][32], shi[3][32];
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float v = P[(P_MU + a) * G + base + i];
      lo[a] = fminf(lo[a], v); hi[a] = fmaxf(hi[a], v);
    }
#pragma unroll
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (ln == 0)
    for (int a = 0; a < 3; ++a) { slo[a][w] = lo[a]; shi[a][w] = hi[a]; }
  __syncthreads();
  if (threadIdx.x < 3) {
    float l = INFINITY, h = -INFINITY;
    for (int k = 0; k < nw; ++k) { l = fminf(l, slo[threadIdx.x][k]); h = fmaxf(h, shi[threadIdx.x][k]); }
    box[threadIdx.x] = l; box[3 + threadIdx.x] = h;
  }
}

struct KnnGrid {
  double lo[3], inv[3], edge[3];
  int dims[3];
};

__device__ __forceinline__ int knn_cell_axis(double x, const KnnGrid& g, int a) {
  const int c = (int)__dmul_rn(__dsub_rn(x, g.lo[a]), g.inv[a]);
  return c < 0 ? 0 : (c >= g.dims[a] ? g.dims[a] - 1 : c);
}

__global__ void k_knn_count(const float* __restrict__ P, int64_t G, int64_t base, int64_t n, KnnGrid g,
                            int32_t* __restrict__ cell_of, uint32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int cx = knn_cell_axis(P[P_MU * G + base + i], g, 0);
    const int cy = knn_cell_axis(P[(P_MU + 1) * G + base + i], g, 1);
    const int cz = knn_cell_axis(P[(P_MU + 2) * G + base + i], g, 2);
    const int q = (cz * g.dims[1] + cy) * g.dims[0] + cx;
    cell_of[i] = q;
    atomicAdd(&cnt[q], 1u);
  }
}

// exclusive scan of the cell counts into start[0..cells] (one block: create-time only)
__global__ void __launch_bounds__(1024) k_knn_scan(const uint32_t* __restrict__ cnt, int64_t cells,
                                                   uint32_t* __restrict__ start) {
  __shared__ uint32_t part[1024];
  const int64_t per = (cells + blockDim.x - 1) / blockDim.x;
  const int64_t b = threadIdx.x * per, e = b + per < cells ? b + per : cells;
  uint32_t t = 0;
  for (int64_t k = b; k < e; ++k) t += cnt[k];
  part[threadIdx.x] = t;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {
    const uint32_t v = threadIdx.x >= (unsigned)o ? part[threadIdx.x - o] : 0u;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t run = part[threadIdx.x] - t;
  for (int64_t k = b; k < e; ++k) { start[k] = run; run += cnt[k]; }
  if (threadIdx.x == blockDim.x - 1) start[cells] = part[threadIdx.x];
}

__global__ void k_knn_scatter(const float* __restrict__ P, int64_t G, int64_t base, int64_t n,
                              const int32_t* __restrict__ cell_of, const uint32_t* __restrict__ start,
                              uint32_t* __restrict__ fill, float4* __restrict__ sorted) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int q = cell_of[i];
    const uint32_t k = start[q] + atomicAdd(&fill[q], 1u);
    sorted[k] = make_float4(P[P_MU * G + base + i], P[(P_MU + 1) * G + base + i], P[(P_MU + 2) * G + base + i],
                            __int_as_float((int)i));
  }
}

// one thread per sorted slot (neighbouring threads share cells), dbar written at the point's index
__global__ void __launch_bounds__(256) k_knn3_grid(const float4* __restrict__ sorted, int64_t n,
                                                   const uint32_t* __restrict__ start, KnnGrid g,
                                                   double slack, double* __restrict__ dbar) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const float4 me = sorted[t];
  const int i = __float_as_int(me.w);
  const double xi = me.x, yi = me.y, zi = me.z;
  const int c[3] = {knn_cell_axis(xi, g, 0), knn_cell_axis(yi, g, 1), knn_cell_axis(zi, g, 2)};
  const double pt[3] = {xi, yi, zi};
  double b0 = INFINITY, b1 = INFINITY, b2 = INFINITY;
  const int rmax = max(g.dims[0], max(g.dims[1], g.dims[2]));
  for (int r = 0; r <= rmax; ++r) {
    const int z0 = max(0, c[2] - r), z1 = min(g.dims[2] - 1, c[2] + r);
    const int y0 = max(0, c[1] - r), y1 = min(g.dims[1] - 1, c[1] + r);
    for (int z = z0; z <= z1; ++z)
      for (int y = y0; y <= y1; ++y) {
        // a face row of the shell visits every x of the cube; an inner row only its two ends
        const bool face = abs(z - c[2]) == r || abs(y - c[1]) == r;
        const int xa = c[0] - r, xb = c[0] + r;
        const int x0 = face ? max(0, xa) : xa, x1 = face ? min(g.dims[0] - 1, xb) : xb;
        const int step = face ? 1 : 2 * r;
        for (int x = x0; x <= x1; x += step) {
          if (x < 0 || x >= g.dims[0]) continue;
          const int q = (z * g.dims[1] + y) * g.dims[0] + x;
          for (uint32_t k = start[q], ke = start[q + 1]; k < ke; ++k) {
            const float4 o = sorted[k];
            if (__float_as_int(o.w) == i) continue;
            const double dx = __dsub_rn((double)o.x, xi), dy = __dsub_rn((double)o.y, yi), dz = __dsub_rn((double)o.z, zi);
            const double d = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            if (d < b2) {
              if (d < b1) { b2 = b1; if (d < b0) { b1 = b0; b0 = d; } else { b1 = d; } }
              else b2 = d;
            }
          }
        }
      }
    // distance from the point to the region outside the visited (2r+1)^3 cube
    double bound = INFINITY;
    for (int a = 0; a < 3; ++a) {
      if (c[a] - r > 0) bound = fmin(bound, pt[a] - (g.lo[a] + (c[a] - r) * g.edge[a]));
      if (c[a] + r < g.dims[a] - 1) bound = fmin(bound, (g.lo[a] + (c[a] + r + 1) * g.edge[a]) - pt[a]);
    }
    if (bound == INFINITY) break;                   // the whole grid has been visited
    bound -= slack;
    if (bound > 0.0 && b2 < bound * bound) break;   // nothing unvisited can enter the top 3
  }
  const int k = (int)((n - 1) < 3 ? (n - 1) : 3);
  double s = 0.0;
  if (k >= 1) s = __dadd_rn(s, __dsqrt_rn(b0));
  if (k >= 2) s = __dadd_rn(s, __dsqrt_rn(b1));
  if (k >= 3) s = __dadd_rn(s, __dsqrt_rn(b2));
  dbar[i] = k > 0 ? __ddiv_rn(s, (double)k) : 0.0;
}

static cudaError_t knn3_level(const float* P, int64_t G, int64_t base, int64_t n, double* dbar, cudaStream_t s) {
  float* box = nullptr;
  cudaError_t e = cudaMalloc(&box, 6 * sizeof(float));
  if (e != cudaSuccess) return e;
  k_knn_bbox<<<1, 1024, 0, s>>>(P, G, base, n, box);
  float hb[6];
  e = cudaMemcpyAsync(hb, box, sizeof(hb), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(box);
  if (e != cudaSuccess) return e;
  KnnGrid g;
  double ext[3], diag2 = 0.0;
  for (int a = 0; a < 3; ++a) { g.lo[a] = hb[a]; ext[a] = (double)hb[3 + a] - (double)hb[a]; diag2 += ext[a] * ext[a]; }
  const double diag = std::sqrt(diag2);
  // cell edge: ~2 points per cell of the (floored) bounding volume, total cells <= 2n + 8
  const int64_t cap = 2 * n + 8;
  double vol = 1.0;
  for (int a = 0; a < 3; ++a) vol *= std::max(ext[a], 1e-3 * diag);
  double edge = diag > 0.0 ? std::cbrt(vol / (0.5 * (double)n)) : 1.0;
  for (int it = 0; it < 400; ++it) {
    int64_t prod = 1;
    for (int a = 0; a < 3; ++a) {
      g.dims[a] = ext[a] > 0.0 ? (int)std::max(1.0, std::min(1024.0, std::ceil(ext[a] / edge))) : 1;
      prod *= g.dims[a];
    }
    if (prod <= cap) break;
    edge *= 1.25;
  }
  for (int a = 0; a < 3; ++a) {
    g.inv[a] = ext[a] > 0.0 ? (double)g.dims[a] / ext[a] : 0.0;
    g.edge[a] = ext[a] > 0.0 ? ext[a] / (double)g.dims[a] : 0.0;
  }
  const int64_t cells = (int64_t)g.dims[0] * g.dims[1] * g.dims[2];
  int32_t* cell_of = nullptr;
  uint32_t *cnt = nullptr, *start = nullptr;
  float4* sorted = nullptr;
  if ((e = cudaMalloc(&cell_of, sizeof(int32_t) * n)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&cnt, sizeof(uint32_t) * cells)) == cudaSuccess &&
      (e = cudaMalloc(&start, sizeof(uint32_t) * (cells + 1))) == cudaSuccess &&
      (e = cudaMalloc(&sorted, sizeof(float4) * n)) == cudaSuccess &&
      (e = cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * cells, s)) == cudaSuccess) {
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
    k_knn_count<<<nb, 256, 0, s>>>(P, G, base, n, g, cell_of, cnt);
    k_knn_scan<<<1, 1024, 0, s>>>(cnt, cells, start);
    cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * cells, s);
    k_knn_scatter<<<nb, 256, 0, s>>>(P, G, base, n, cell_of, start, cnt, sorted);
    // slack: 1e-9 of the diagonal, orders of magnitude above the rounding of lo + c * edge
    k_knn3_grid<<<(int)((n + 255) / 256), 256, 0, s>>>(sorted, n, start, g, 1e-9 * diag, dbar);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  cudaFree(cell_of); cudaFree(cnt); cudaFree(start); cudaFree(sorted);
  return e;
}

// One CTA: mean and population std of dbar, the level's AABB diagonal, then
// cap = mu + zcap * sigma.  Each thread sums the indices congruent to it mod the block size in
// index order, then a fixed-shape tree combines the partials: deterministic, and within a
// few fp64 ulp of the oracle's sequential sums (DESIGN A19); min / max are order-free.
__device__ __forceinline__ double eq2_block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x >> 1; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024) k_eq2_stats(const float* __restrict__ P, int64_t G, int64_t base,
                                                    int64_t n, const double* __restrict__ dbar, double zcap,
                                                    double* out /*cap, floor*/) {
  __shared__ double sh[1024];
  __shared__ float sb[6][1024];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc = __dadd_rn(acc, dbar[i]);
  const double mu = __ddiv_rn(eq2_block_sum(acc, sh), (double)n);
  acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = __dsub_rn(dbar[i], mu);
    acc = __dadd_rn(acc, __dmul_rn(d, d));
  }
  const double var = __ddiv_rn(eq2_block_sum(acc, sh), (double)n);
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    for (int a = 0; a < 3; ++a) {
      const float v = P[(P_MU + a) * G + base + i];
      lo[a] = fminf(lo[a], v); hi[a] = fmaxf(hi[a], v);
    }
  for (int a = 0; a < 3; ++a) { sb[a][threadIdx.x] = lo[a]; sb[3 + a][threadIdx.x] = hi[a]; }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double l[3], h[3];
  for (int a = 0; a < 3; ++a) {
    float fl = INFINITY, fh = -INFINITY;
    for (int k = 0; k < (int)blockDim.x; ++k) { fl = fminf(fl, sb[a][k]); fh = fmaxf(fh, sb[3 + a][k]); }
    l[a] = fl; h[a] = fh;
  }
  const double dx = __dsub_rn(h[0], l[0]), dy = __dsub_rn(h[1], l[1]), dz = __dsub_rn(h[2], l[2]);
  const double diag = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
  out[0] = __dadd_rn(mu, __dmul_rn(zcap, __dsqrt_rn(var)));
  out[1] = diag > 0.0 ? __dmul_rn(1e-6, diag) : 1e-6;   // reading A20: degenerate level (one point /
}                                                         // coincident points) -> absolute floor

__global__ void k_eq2_apply(int64_t n, const double* __restrict__ dbar, const double* __restrict__ capfl,
                            double factor, float* P, int64_t G, int64_t base) {
  const double cap = capfl[0], fl = capfl[1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    // Eq. 2 with the floor applied after the cap (reading A20): s = max(min(cap, dbar), fl)
    const double r = cap < dbar[i] ? cap : dbar[i];
    const double s = __dmul_rn(r > fl ? r : fl, factor);
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

// ------------------------------------------------------------- permutation pi on the device
// pi = stable argsort of splitmix64(seed + i), i < N0 (C7 / reading A9).  splitmix64 is a
// bijection of its 64-bit input, so the N0 keys are distinct and any correct sort is the
// stable one; a bitonic network over the next power of two (padding keys (2^64-1, 2^63-1)
// sort last) sorts (key, index) pairs: global passes for strides >= 1024, then one
// shared-memory kernel per 2048-element tile for every smaller stride of a merge level.
__device__ __forceinline__ uint64_t splitmix64_d(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ bool kv_less(uint64_t ka, int64_t ia, uint64_t kb, int64_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

__global__ void k_perm_keys(int64_t N0, int64_t Np, uint64_t seed, uint64_t* key, int64_t* idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < Np; i += (int64_t)gridDim.x * blockDim.x) {
    key[i] = i < N0 ? splitmix64_d(seed + (uint64_t)i) : ~0ull;
    idx[i] = i < N0 ? i : (int64_t)0x7FFFFFFFFFFFFFFFll;
  }
}

__global__ void k_bitonic_global(uint64_t* key, int64_t* idx, int64_t Np, int64_t k, int64_t j) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < Np; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i ^ j;
    if (p <= i) continue;
    const bool up = (i & k) == 0;
    const uint64_t ka = key[i], kb = key[p];
    const int64_t ia = idx[i], ib = idx[p];
    if (kv_less(kb, ib, ka, ia) == up) { key[i] = kb; key[p] = ka; idx[i] = ib; idx[p] = ia; }
  }
}

constexpr int kBitTile = 2048;
__global__ void __launch_bounds__(1024) k_bitonic_shared(uint64_t* key, int64_t* idx, int64_t k, int64_t j0) {
  __shared__ uint64_t sk[kBitTile];
  __shared__ int64_t si[kBitTile];
  const int64_t base = (int64_t)blockIdx.x * kBitTile;
  for (int t = threadIdx.x; t < kBitTile; t += blockDim.x) { sk[t] = key[base + t]; si[t] = idx[base + t]; }
  __syncthreads();
  for (int64_t j = j0; j > 0; j >>= 1) {
    for (int t = threadIdx.x; t < kBitTile; t += blockDim.x) {
      const int p = t ^ (int)j;
      if (p > t) {
        const bool up = ((base + t) & k) == 0;
        if (kv_less(sk[p], si[p], sk[t], si[t]) == up) {
          const uint64_t a = sk[t]; sk[t] = sk[p]; sk[p] = a;
          const int64_t b = si[t]; si[t] = si[p]; si[p] = b;
        }
      }
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < kBitTile; t += blockDim.x) { key[base + t] = sk[t]; idx[base + t] = si[t]; }
}

// src[goff[l] + i] = i on level 0 (caller order), pi[i] on level l >= 1 (nested prefixes)
__global__ void k_level_src(const int64_t* __restrict__ pi, LevelGeom g, int64_t* src) {
  const int64_t G = g.goff[g.L];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < G; j += (int64_t)gridDim.x * blockDim.x) {
    const int l = level_of_gaussian(g, j);
    const int64_t i = j - g.goff[l];
    src[j] = l == 0 ? i : pi[i];
  }
}

int64_t sort_kv_size(int64_t n) {
  int64_t Np = kBitTile;
  while (Np < n) Np <<= 1;
  return Np;
}

void launch_sort_kv(uint64_t* key, int64_t* idx, int64_t Np, cudaStream_t s) {
  for (int64_t k = 2; k <= Np; k <<= 1) {
    int64_t j = k >> 1;
    for (; j >= kBitTile; j >>= 1) k_bitonic_global<<<blocks_for(Np), 256, 0, s>>>(key, idx, Np, k, j);
    k_bitonic_shared<<<(unsigned)(Np / kBitTile), 1024, 0, s>>>(key, idx, k, j);
  }
}

cudaError_t launch_level_sources(int64_t N0, uint64_t seed, const LevelGeom& g, int64_t* src, cudaStream_t s) {
  const int64_t Np = sort_kv_size(N0);
  uint64_t* key = nullptr;
  int64_t* idx = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&key, sizeof(uint64_t) * Np, s);
  if (e != cudaSuccess) return e;
  e = cudaMallocAsync((void**)&idx, sizeof(int64_t) * Np, s);
  if (e != cudaSuccess) return e;
  k_perm_keys<<<blocks_for(Np), 256, 0, s>>>(N0, Np, seed, key, idx);
  launch_sort_kv(key, idx, Np, s);
  k_level_src<<<blocks_for(g.goff[g.L]), 256, 0, s>>>(idx, g, src);
  cudaFreeAsync(key, s);
  cudaFreeAsync(idx, s);
  return cudaGetLastError();
}

// ------------------------------------------------------- culling-grid statistics per level
// One CTA per level: the AABB of the means (fp32 values, exact min/max) and the mean over the
// level of (e^{s0} + e^{s1} + e^{s2}) / 3 in fp64, summed in a fixed tree order -- the inputs of
// the R1 grid rule, which the host finishes (a handful of flops per level).  out[l] = (lo[3],
// hi[3], mean e^s).
__global__ void __launch_bounds__(1024) k_grid_stats(const float* __restrict__ P, int64_t G, LevelGeom g,
                                                     double* out) {
  __shared__ double sh[1024];
  __shared__ float sb[6][32];
  const int l = blockIdx.x;
  const int64_t base = g.goff[l], n = g.goff[l + 1] - base;
  double acc = 0.0;
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t j = base + i;
    const double e = __dadd_rn(__dadd_rn(exp((double)P[P_S * G + j]), exp((double)P[(P_S + 1) * G + j])),
                               exp((double)P[(P_S + 2) * G + j]));
    acc = __dadd_rn(acc, __ddiv_rn(e, 3.0));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float v = P[(P_MU + a) * G + j];
      lo[a] = fminf(lo[a], v); hi[a] = fmaxf(hi[a], v);
    }
  }
  const double tot = eq2_block_sum(acc, sh);
#pragma unroll
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int a = 0; a < 3; ++a) { sb[a][w] = lo[a]; sb[3 + a][w] = hi[a]; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int a = 0; a < 3; ++a) {
      float fl = INFINITY, fh = -INFINITY;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { fl = fminf(fl, sb[a][k]); fh = fmaxf(fh, sb[3 + a][k]); }
      out[7 * l + a] = fl; out[7 * l + 3 + a] = fh;
    }
    out[7 * l + 6] = __ddiv_rn(tot, (double)(n > 0 ? n : 1));
  }
}

cudaError_t launch_grid_stats(const float* P, int64_t G, const LevelGeom& g, double* out, cudaStream_t s) {
  k_grid_stats<<<g.L, 1024, 0, s>>>(P, G, g, out);
  return cudaGetLastError();
}

void launch_gather_init(int64_t N0, const float* pos, const float* rgb, const float* log_scale,
                        const int64_t* src, int64_t G, float* P, float opacity_logit, cudaStream_t s) {
  k_gather_init<<<blocks_for(G), 256, 0, s>>>(N0, pos, rgb, log_scale, src, G, P, opacity_logit);
}

cudaError_t launch_eq2_level(const float* P, int64_t G, int64_t base, int64_t n, double* dbar, double* capfl,
                             double zcap, double factor, float* Pw, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const cudaError_t e = knn3_level(P, G, base, n, dbar, s);
  if (e != cudaSuccess) return e;
  k_eq2_stats<<<1, 1024, 0, s>>>(P, G, base, n, dbar, zcap, capfl);
  k_eq2_apply<<<blocks_for(n), 256, 0, s>>>(n, dbar, capfl, factor, Pw, G, base);
  return cudaGetLastError();
}

void launch_pack(const float* P, int64_t G, int64_t base, int64_t n, float* out, cudaStream_t s) {
  k_pack<<<blocks_for(n), 256, 0, s>>>(P, G, base, n, out);
}

void launch_unpack(const float* in, int64_t G, int64_t base, int64_t n, float* P, cudaStream_t s) {
  k_unpack<<<blocks_for(n), 256, 0, s>>>(in, G, base, n, P);
}

}  // namespace gsc
