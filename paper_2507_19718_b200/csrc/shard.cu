// shard.cu -- level-sharded multi-GPU mode (gc_set_comm mode 1, north star "the
// level-sharded alternative"): the level plan (host), the routing of fit samples and lookups
// to the ranks owning their level, and the return of lookup results to caller order.
//
// A level is owned by one group of consecutive ranks; inside a group its samples are split
// round-robin (data parallel over the group, gradients summed over the group's communicator),
// so level 0 -- most Gaussians and samples -- can be DP over a sub-group while the small levels
// share one rank (the "hybrid" of SURVEY 8(e)).  No parameter replication is needed for the
// math: a rank steps only the levels it owns (DevState::owned).
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "record.cuh"

namespace gsc {

// ----------------------------------------------------------------------------- plan (host)
// Level sharding uses as many groups as it can: K = min(L, W).
//  W >= L: one group per level; the W - L extra ranks go, one at a time, to the level with the
//    largest weight per rank (greedy, exact for min max w_l / n_l); level 0 -- most samples and
//    Gaussians -- becomes data parallel over its group (the hybrid of SURVEY 8(e)).
//  W < L: one rank per group; the levels are cut into W contiguous ranges minimising the
//    largest range weight (exact dynamic programme, O(L^2 W)).
// Ties resolve to the lowest level / earliest cut, so every rank computes the identical plan.
int level_plan(int L, const double* w_in, int W, int* group_of_level, int* first_rank, int* group_size) {
  if (L < 1 || W < 1 || L > kMaxL) return 0;
  double w[kMaxL];
  for (int l = 0; l < L; ++l) w[l] = w_in[l] > 0.0 ? w_in[l] : 0.0;
  if (W >= L) {
    int n[kMaxL];
    for (int l = 0; l < L; ++l) n[l] = 1;
    for (int extra = W - L; extra > 0; --extra) {
      int best = 0;
      for (int l = 1; l < L; ++l)
        if (w[l] / n[l] > w[best] / n[best] * (1.0 + 1e-12)) best = l;
      n[best] += 1;
    }
    int r = 0;
    for (int l = 0; l < L; ++l) { group_of_level[l] = l; first_rank[l] = r; group_size[l] = n[l]; r += n[l]; }
    return L;
  }
  const double inf = 1e300;
  std::vector<double> pre(L + 1, 0.0);
  for (int l = 0; l < L; ++l) pre[l + 1] = pre[l] + w[l];
  // best[k][i]: levels [0, i) cut into k groups; cut[k][i]: start of the last group
  std::vector<double> best((size_t)(W + 1) * (L + 1), inf);
  std::vector<int> cut((size_t)(W + 1) * (L + 1), -1);
  auto at = [&](int k, int i) { return (size_t)k * (L + 1) + i; };
  best[at(0, 0)] = 0.0;
  for (int k = 1; k <= W; ++k)
    for (int i = k; i <= L; ++i)
      for (int j = k - 1; j < i; ++j) {
        if (best[at(k - 1, j)] >= inf) continue;
        const double c = std::max(best[at(k - 1, j)], pre[i] - pre[j]);
        if (c < best[at(k, i)] * (1.0 - 1e-12)) { best[at(k, i)] = c; cut[at(k, i)] = j; }
      }
  int i = L;
  for (int k = W; k >= 1; --k) {
    const int j = cut[at(k, i)];
    if (j < 0) return 0;
    for (int l = j; l < i; ++l) group_of_level[l] = k - 1;
    first_rank[k - 1] = k - 1; group_size[k - 1] = 1;
    i = j;
  }
  return W;
}

// ----------------------------------------------------------------------------- routing
constexpr int kRouteThreads = 256, kRouteK = 8;            // 2048 samples per tile
constexpr int kMaxWorld = 1024;

// Destination rank of sample i, or -1 when it is dropped (same validity rule and level as
// k_keys, C2): level l = min(n, L) - 1; the owning group's member (i + rank) mod size.
__device__ __forceinline__ int route_dest(const RoutePlan& p, const float* pos, const int32_t* len,
                                          const float* rgb, int level_fixed, int64_t i, int* lvl) {
  const float x = pos[3 * i], y = pos[3 * i + 1], z = pos[3 * i + 2];
  bool ok = isfinite(x) && isfinite(y) && isfinite(z);
  int l = level_fixed;
  if (level_fixed < 0) {
    const int n = len[i];
    ok = ok && n >= 1;
    l = min(n, p.L) - 1;
  }
  if (rgb) ok = ok && isfinite(rgb[3 * i]) && isfinite(rgb[3 * i + 1]) && isfinite(rgb[3 * i + 2]);
  *lvl = l;
  if (!ok) return -1;
  if (p.colrank) {                    // owner-computes: the owner of the sample's cell column (C8 cell)
    const int32_t cx = clampcell(floor(__dmul_rn(__dsub_rn((double)x, p.geom.origin[l][0]), p.geom.inv_cell[l][0])),
                                 p.geom.dims[l][0]);
    return p.colrank[l * kMaxCols + cx];
  }
  const int n = p.size[l];
  return p.first[l] + (int)((i + p.rank) % n);
}

// pass 0: per-destination counts (tile histogram in shared memory, one global atomic per
// (tile, destination)).  pass 1: packs every routed sample into the destination's segment of
// the send buffer (segment base `base[d]`, a tile's range reserved with one atomic on
// cursor[d]); fit records are 8 words (x y z n r g b 0), lookups 4 (x y z n) plus perm[slot]
// = caller index; dropped lookups get out_zero = 0.
__global__ void __launch_bounds__(kRouteThreads) k_route(const float* __restrict__ pos, const int32_t* __restrict__ len,
                                                         const float* __restrict__ rgb, int level_fixed, int64_t S,
                                                         RoutePlan p, int pass, uint32_t* count,
                                                         const uint32_t* __restrict__ base, uint32_t* cursor,
                                                         float4* sendbuf, uint32_t* perm, float* out_zero) {
  __shared__ uint32_t hist[kMaxWorld], tbase[kMaxWorld];
  const int W = p.world;
  for (int64_t t0 = (int64_t)blockIdx.x * kRouteThreads * kRouteK; t0 < S;
       t0 += (int64_t)gridDim.x * kRouteThreads * kRouteK) {
    for (int d = threadIdx.x; d < W; d += kRouteThreads) hist[d] = 0u;
    __syncthreads();
    int dest[kRouteK], lv[kRouteK];
    uint32_t lrank[kRouteK];
#pragma unroll
    for (int u = 0; u < kRouteK; ++u) {
      const int64_t i = t0 + u * kRouteThreads + threadIdx.x;
      dest[u] = -1; lv[u] = 0; lrank[u] = 0u;
      if (i < S) {
        dest[u] = route_dest(p, pos, len, rgb, level_fixed, i, &lv[u]);
        if (dest[u] >= 0) lrank[u] = atomicAdd(&hist[dest[u]], 1u);
        else if (pass == 1 && out_zero) { out_zero[3 * i] = 0.f; out_zero[3 * i + 1] = 0.f; out_zero[3 * i + 2] = 0.f; }
      }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < W; d += kRouteThreads) {
      const uint32_t h = hist[d];
      if (pass == 0) { if (h) atomicAdd(count + d, h); }
      else tbase[d] = h ? base[d] + atomicAdd(cursor + d, h) : 0u;
    }
    __syncthreads();
    if (pass == 1) {
#pragma unroll
      for (int u = 0; u < kRouteK; ++u) {
        if (dest[u] < 0) continue;
        const int64_t i = t0 + u * kRouteThreads + threadIdx.x;
        const uint32_t slot = tbase[dest[u]] + lrank[u];
        const int n = level_fixed < 0 ? len[i] : level_fixed + 1;
        const float4 a = make_float4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], __int_as_float(n));
        if (rgb) {
          sendbuf[2 * (size_t)slot] = a;
          sendbuf[2 * (size_t)slot + 1] = make_float4(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2], 0.f);
        } else {
          sendbuf[slot] = a;
          perm[slot] = (uint32_t)i;
        }
      }
    }
    __syncthreads();
  }
}

// received records -> the SoA inputs of the fit / lookup pipeline
__global__ void k_unpack_routed(const float4* __restrict__ recv, int64_t R, int fit, float* pos, int32_t* len,
                                float* rgb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = fit ? recv[2 * i] : recv[i];
    pos[3 * i] = a.x; pos[3 * i + 1] = a.y; pos[3 * i + 2] = a.z;
    len[i] = __float_as_int(a.w);
    if (fit) {
      const float4 b = recv[2 * i + 1];
      rgb[3 * i] = b.x; rgb[3 * i + 1] = b.y; rgb[3 * i + 2] = b.z;
    }
  }
}

// returned lookup results (slot order of the send buffer) -> caller order
__global__ void k_unroute(const float* __restrict__ res, const uint32_t* __restrict__ perm, int64_t n, float* out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t i = perm[k];
    out[3 * (size_t)i] = res[3 * k]; out[3 * (size_t)i + 1] = res[3 * k + 1]; out[3 * (size_t)i + 2] = res[3 * k + 2];
  }
}

// ------------------------------------------------------------------ owner-computes (mode 2)
// owner[j] = the rank of the column of the cell holding Gaussian j's mean (fixed at set_comm)
__global__ void k_owner(const float* __restrict__ P, int64_t G, LevelGeom g, const int32_t* __restrict__ colrank,
                        uint8_t* owner) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < G; j += (int64_t)gridDim.x * blockDim.x) {
    const int l = level_of_gaussian(g, j);
    const int32_t cx = clampcell(floor(__dmul_rn(__dsub_rn((double)P[P_MU * G + j], g.origin[l][0]), g.inv_cell[l][0])),
                                 g.dims[l][0]);
    owner[j] = (uint8_t)colrank[l * kMaxCols + cx];
  }
}

// need[j] (owned j): bit r for every rank r owning a column of j's C8 cell range (its own bit
// included); 0 for Gaussians owned elsewhere (the all-reduce then yields every owner's mask)
__global__ void k_need(const float* __restrict__ P, int64_t G, double tau, LevelGeom g,
                       const int32_t* __restrict__ colrank, const uint8_t* __restrict__ owner, int me, uint32_t* need) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < G; j += (int64_t)gridDim.x * blockDim.x) {
    uint32_t m = 0u;
    if (owner[j] == me) {
      float p[kNP];
#pragma unroll
      for (int k = 0; k < kNP; ++k) p[k] = P[k * G + j];
      const int l = level_of_gaussian(g, j);
      int32_t lo[3], hi[3];
      double r2;
      cull_range(p, tau, g, l, lo, hi, r2);
      m = 1u << me;
      for (int32_t cx = lo[0]; cx <= hi[0]; ++cx) m |= 1u << colrank[l * kMaxCols + cx];
    }
    need[j] = m;
  }
}

__global__ void k_bflag(const uint32_t* __restrict__ need, int64_t G, uint32_t* flag) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < G; j += (int64_t)gridDim.x * blockDim.x)
    flag[j] = __popc(need[j]) > 1 ? 1u : 0u;
}

__global__ void k_bcompact(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos, int64_t G, int32_t* idx) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < G; j += (int64_t)gridDim.x * blockDim.x)
    if (flag[j]) idx[pos[j]] = (int32_t)j;
}

__global__ void k_rows_grad(float* grad, float* buf, const int32_t* __restrict__ idx, int64_t n, int scatter) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 12 * n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / 12, k = t % 12;
    float* g = grad + 12 * (int64_t)idx[r] + k;
    if (scatter) *g = buf[t]; else buf[t] = *g;
  }
}

__global__ void k_rows_param(float* P, int64_t G, float* buf, const int32_t* __restrict__ idx, int64_t n,
                             const uint8_t* __restrict__ owner, int me, int scatter) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < kNP * n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / kNP, k = t % kNP, j = idx[r];
    if (scatter) P[k * G + j] = buf[t];
    else buf[t] = owner[j] == me ? P[k * G + j] : 0.f;
  }
}

static int route_grid(int64_t S) {
  const int64_t t = (S + kRouteThreads * kRouteK - 1) / (kRouteThreads * kRouteK);
  return (int)std::max<int64_t>(1, std::min<int64_t>(t, 148 * 8));
}

void launch_route(const float* pos, const int32_t* len, const float* rgb, int level_fixed, int64_t S,
                  const RoutePlan& p, int pass, uint32_t* count, const uint32_t* base, uint32_t* cursor,
                  float4* sendbuf, uint32_t* perm, float* out_zero, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, pass == 0 ? "route_count" : "route_pack", s);
  if (S > 0)
    k_route<<<route_grid(S), kRouteThreads, 0, s>>>(pos, len, rgb, level_fixed, S, p, pass, count, base, cursor,
                                                    sendbuf, perm, out_zero);
}

void launch_unpack_routed(const float4* recv, int64_t R, bool fit, float* pos, int32_t* len, float* rgb,
                          cudaStream_t s) {
  if (R > 0) k_unpack_routed<<<route_grid(R), 256, 0, s>>>(recv, R, fit ? 1 : 0, pos, len, rgb);
}

void launch_unroute(const float* res, const uint32_t* perm, int64_t n, float* out, cudaStream_t s) {
  if (n > 0) k_unroute<<<route_grid(n), 256, 0, s>>>(res, perm, n, out);
}

// gc_params under owner-computes: zero the rows of the packed level copy this rank does not own
__global__ void k_zero_nonowned(float* t, int64_t n, int64_t base, const uint8_t* __restrict__ owner, int me) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (owner[base + i] == me) continue;
    for (int a = 0; a < 3; ++a) { t[3 * i + a] = 0.f; t[7 * n + 3 * i + a] = 0.f; t[10 * n + 3 * i + a] = 0.f; }
    for (int a = 0; a < 4; ++a) t[3 * n + 4 * i + a] = 0.f;
    t[13 * n + i] = 0.f;
  }
}
void launch_zero_nonowned(float* t, int64_t n, int64_t base, const uint8_t* owner, int me, cudaStream_t s) {
  k_zero_nonowned<<<route_grid(n), 256, 0, s>>>(t, n, base, owner, me);
}

__global__ void k_pack_slice(const float* __restrict__ P, int64_t G, int64_t g0, int64_t n, int64_t np, float* buf) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < kNP * np; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t / np, i = t % np;
    buf[t] = i < n ? P[k * G + g0 + i] : 0.f;
  }
}
__global__ void k_unpack_slices(const float* __restrict__ buf, int W, int64_t np, float* P, int64_t G) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)W * kNP * np;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / (kNP * np), rem = t % (kNP * np), k = rem / np, i = rem % np;
    const int64_t j = r * np + i;
    if (j < G) P[k * G + j] = buf[t];
  }
}
void launch_pack_slice(const float* P, int64_t G, int64_t g0, int64_t n, int64_t np, float* buf, cudaStream_t s) {
  k_pack_slice<<<route_grid(kNP * np), 256, 0, s>>>(P, G, g0, n, np, buf);
}
void launch_unpack_slices(const float* buf, int W, int64_t np, float* P, int64_t G, cudaStream_t s) {
  k_unpack_slices<<<route_grid((int64_t)W * kNP * np), 256, 0, s>>>(buf, W, np, P, G);
}

void launch_owner(const float* P, int64_t G, const LevelGeom& g, const int32_t* colrank, uint8_t* owner, cudaStream_t s) {
  k_owner<<<route_grid(G), 256, 0, s>>>(P, G, g, colrank, owner);
}
void launch_need(const float* P, int64_t G, double tau, const LevelGeom& g, const int32_t* colrank,
                 const uint8_t* owner, int rank, uint32_t* need, cudaStream_t s) {
  k_need<<<route_grid(G), 256, 0, s>>>(P, G, tau, g, colrank, owner, rank, need);
}
void launch_boundary(const uint32_t* need, int64_t G, uint32_t* flag, uint32_t* bsums, uint32_t* total,
                     int32_t* idx, cudaStream_t s) {
  k_bflag<<<route_grid(G), 256, 0, s>>>(need, G, flag);
  uint32_t* pos = flag + G;                        // flag buffer holds [G] flags + [G] positions
  launch_scan_u32(flag, G, bsums, total, pos, s);
  k_bcompact<<<route_grid(G), 256, 0, s>>>(flag, pos, G, idx);
}
void launch_rows_grad(float* grad, float* buf, const int32_t* idx, int64_t n, int scatter, cudaStream_t s) {
  if (n > 0) k_rows_grad<<<route_grid(12 * n), 256, 0, s>>>(grad, buf, idx, n, scatter);
}
void launch_rows_param(float* P, int64_t G, float* buf, const int32_t* idx, int64_t n, const uint8_t* owner, int rank,
                       int scatter, cudaStream_t s) {
  if (n > 0) k_rows_param<<<route_grid(kNP * n), 256, 0, s>>>(P, G, buf, idx, n, owner, rank, scatter);
}

// Column slabs (host): per level, the grid columns (x cell index) are cut into W contiguous
// ranges holding about G_l / W Gaussian means each (greedy on the prefix counts: rank r takes
// the columns whose cumulative count lies in [r G_l / W, (r + 1) G_l / W)).  Deterministic.
void slab_plan(int L, const int64_t* goff, const float* means, const LevelGeom& g, int W, int32_t* colrank) {
  // means: the x coordinates of the Gaussian means [G]
  const int64_t G = goff[L];
  for (int l = 0; l < L; ++l) {
    const int dx = g.dims[l][0];
    std::vector<int64_t> cnt(dx, 0);
    for (int64_t j = goff[l]; j < goff[l + 1]; ++j) {
      const double f = std::floor(((double)means[j] - g.origin[l][0]) * g.inv_cell[l][0]);
      int32_t cx = !(f >= 0.0) ? 0 : (f > (double)(dx - 1) ? dx - 1 : (int32_t)f);
      cnt[cx] += 1;
    }
    const int64_t n = goff[l + 1] - goff[l];
    int64_t acc = 0;
    for (int c = 0; c < kMaxCols; ++c) {
      int r = 0;
      if (c < dx) {
        r = n > 0 ? (int)std::min<int64_t>(W - 1, (acc * W) / n) : 0;   // owner of the column's first mean
        acc += cnt[c];
      } else {
        r = W - 1;
      }
      colrank[l * kMaxCols + c] = r;
    }
  }
  (void)G;
}

}  // namespace gsc

extern "C" gc_status gc_level_plan(int levels, const double* weights, int world, int32_t* group_of_level,
                                   int32_t* group_first_rank, int32_t* group_size, int* n_groups) {
  if (levels < 1 || levels > GC_MAX_LEVELS || world < 1 || world > gsc::kMaxWorld || !weights ||
      !group_of_level || !group_first_rank || !group_size || !n_groups)
    return GC_ERR_ARG;
  int gl[GC_MAX_LEVELS], fr[GC_MAX_LEVELS], gs[GC_MAX_LEVELS];
  const int ng = gsc::level_plan(levels, weights, world, gl, fr, gs);
  if (ng <= 0) return GC_ERR_ARG;
  for (int l = 0; l < levels; ++l) group_of_level[l] = gl[l];
  for (int g = 0; g < ng; ++g) { group_first_rank[g] = fr[g]; group_size[g] = gs[g]; }
  *n_groups = ng;
  return GC_OK;
}

extern "C" gc_status gc_slab_plan(int levels, const int64_t* counts, const float* means_x, const double* origin,
                                  const double* inv_cell, const int32_t* dims, int world, int32_t* col_rank) {
  if (levels < 1 || levels > GC_MAX_LEVELS || world < 1 || world > 32 || !counts || !means_x || !origin ||
      !inv_cell || !dims || !col_rank)
    return GC_ERR_ARG;
  gsc::LevelGeom g{};
  g.L = levels;
  g.goff[0] = 0;
  for (int l = 0; l < levels; ++l) {
    g.goff[l + 1] = g.goff[l] + counts[l];
    for (int a = 0; a < 3; ++a) {
      g.origin[l][a] = origin[3 * l + a]; g.inv_cell[l][a] = inv_cell[3 * l + a]; g.dims[l][a] = dims[3 * l + a];
    }
    if (dims[3 * l] < 1 || dims[3 * l] > gsc::kMaxCols) return GC_ERR_ARG;
  }
  std::vector<int32_t> cr((size_t)gsc::kMaxL * gsc::kMaxCols);
  gsc::slab_plan(levels, g.goff, means_x, g, world, cr.data());
  for (int l = 0; l < levels; ++l)
    for (int c = 0; c < gsc::kMaxCols; ++c) col_rank[l * gsc::kMaxCols + c] = cr[(size_t)l * gsc::kMaxCols + c];
  return GC_OK;
}
