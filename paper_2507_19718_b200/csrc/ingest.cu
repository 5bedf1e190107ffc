// ingest.cu -- SoA sample ingest binned by (level, cell): validation and level assignment
// (C2; sec.3.5 per-level path buffers), fp64 cell keys (C8), a counting sort
// whose histogram ranks come from warp-aggregated atomics, and the scatter into planar bins.
#include "common.cuh"
#include "kernels.h"

namespace gsc {

__global__ void __launch_bounds__(256) k_keys(const float* __restrict__ pos, const int32_t* __restrict__ len,
                                              const float* __restrict__ rgb, int level_fixed, int64_t S,
                                              LevelGeom g, IngestBufs b, float* out_zero) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // warp-uniform trip count so that __match_any_sync sees full warps
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < S; i0 += stride) {
    int64_t i = i0 + lane;
    bool ok = i < S;
    uint32_t key = kInvalidKey;
    if (ok) {
      float x = pos[3 * i], y = pos[3 * i + 1], z = pos[3 * i + 2];
      ok = isfinite(x) && isfinite(y) && isfinite(z);
      int l = level_fixed;
      if (level_fixed < 0) {
        int n = len[i];
        ok = ok && n >= 1;
        l = min(n, g.L) - 1;
      }
      if (rgb) ok = ok && isfinite(rgb[3 * i]) && isfinite(rgb[3 * i + 1]) && isfinite(rgb[3 * i + 2]);
      if (ok) key = (uint32_t)sample_cell(g, l, x, y, z);
      else if (out_zero) { out_zero[3 * i] = 0.f; out_zero[3 * i + 1] = 0.f; out_zero[3 * i + 2] = 0.f; }
    }
    unsigned peers = __match_any_sync(0xffffffffu, key);
    uint32_t rank = 0;
    if (key != kInvalidKey) {
      int leader = __ffs(peers) - 1;
      uint32_t base = 0;
      if (lane == leader) base = atomicAdd(b.cell_count + key, (uint32_t)__popc(peers));
      base = __shfl_sync(peers, base, leader);
      rank = base + __popc(peers & ((1u << lane) - 1u));
    }
    if (i < S) { b.key[i] = key; b.rank[i] = rank; }
  }
}

__global__ void __launch_bounds__(256) k_scatter(const float* __restrict__ pos, const float* __restrict__ rgb,
                                                 int64_t S, const uint32_t* __restrict__ cell_start, IngestBufs b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t key = b.key[i];
    if (key == kInvalidKey) continue;
    uint32_t d = cell_start[key] + b.rank[i];
    b.bx[d] = pos[3 * i]; b.by[d] = pos[3 * i + 1]; b.bz[d] = pos[3 * i + 2];
    if (rgb) { b.br[d] = rgb[3 * i]; b.bg[d] = rgb[3 * i + 1]; b.bb[d] = rgb[3 * i + 2]; }
    if (b.bidx) b.bidx[d] = (uint32_t)i;
  }
}

__global__ void k_levels_of(const uint32_t* key, int64_t S, LevelGeom g, int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t k = key[i];
    out[i] = (k == kInvalidKey) ? -1 : level_of_cell(g, k);
  }
}

static int grid_for(int64_t n, int per_sm = 8) {
  int64_t b = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * per_sm));
}

void launch_keys(const float* pos, const int32_t* len, const float* rgb, int level_fixed,
                 int64_t S, const LevelGeom& g, IngestBufs b, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, "ingest_keys", s);
  k_keys<<<grid_for(S), 256, 0, s>>>(pos, len, rgb, level_fixed, S, g, b, nullptr);
}

void launch_keys_query(const float* pos, const int32_t* len, int level_fixed, int64_t S,
                       const LevelGeom& g, IngestBufs b, float* out, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, "query_keys", s);
  k_keys<<<grid_for(S), 256, 0, s>>>(pos, len, nullptr, level_fixed, S, g, b, out);
}

void launch_scatter(const float* pos, const float* rgb, int64_t S, const uint32_t* cell_start,
                    IngestBufs b, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, rgb ? "ingest_scatter" : "query_scatter", s);
  k_scatter<<<grid_for(S), 256, 0, s>>>(pos, rgb, S, cell_start, b);
}

void launch_levels_of(const uint32_t* key, int64_t S, const LevelGeom& g, int32_t* out, cudaStream_t s) {
  k_levels_of<<<grid_for(S), 256, 0, s>>>(key, S, g, out);
}

}  // namespace gsc
