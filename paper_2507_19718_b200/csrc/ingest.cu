// ingest.cu -- SoA sample ingest binned by (level, cell): validation and level assignment
// (C2; sec.3.5 per-level path buffers), fp64 cell keys (C8), a counting sort
// whose ranks come from warp-aggregated atomics, and the scatter into cell-major bins of
// full 32-byte sectors.  Each thread handles kU samples with all loads issued up front
// (memory-level parallelism: the kernels are latency-bound otherwise).
#include "common.cuh"
#include "kernels.h"

namespace gsc {

constexpr int kU = 4;   // samples per thread per iteration
#ifndef GSC_INGEST_MINB
#define GSC_INGEST_MINB 4   // resident CTAs per SM the register budget is sized for
#endif

__global__ void __launch_bounds__(256, GSC_INGEST_MINB) k_keys(const float* __restrict__ pos, const int32_t* __restrict__ len,
                                                 const float* __restrict__ rgb, int level_fixed, int64_t S,
                                                 LevelGeom g, IngestBufs b, float* out_zero) {
  pdl_enter();
  // per-level grid in shared memory: indexed by a runtime level, the kernel-parameter copy
  // would go through dynamically indexed constant loads
  __shared__ double s_org[kMaxL][3], s_inv[kMaxL][3];
  __shared__ int32_t s_dim[kMaxL][3];
  __shared__ int64_t s_coff[kMaxL];
  if (threadIdx.x < kMaxL * 3) {
    const int l = threadIdx.x / 3, a = threadIdx.x % 3;
    s_org[l][a] = g.origin[l][a]; s_inv[l][a] = g.inv_cell[l][a]; s_dim[l][a] = g.dims[l][a];
    if (a == 0) s_coff[l] = g.coff[l];
  }
  __syncthreads();
  GSC_CHECK(S <= b.cap, "keys: samples past the scratch capacity");
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i0 = warp * 32 * kU; i0 < S; i0 += nwarps * 32 * kU) {
    float x[kU], y[kU], z[kU], c[kU][3];
    int n[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + u * 32 + lane;
      if (i < S) {
        x[u] = __ldcs(pos + 3 * i); y[u] = __ldcs(pos + 3 * i + 1); z[u] = __ldcs(pos + 3 * i + 2);
        n[u] = level_fixed < 0 ? __ldcs(len + i) : 1;
        if (rgb) { c[u][0] = __ldcs(rgb + 3 * i); c[u][1] = __ldcs(rgb + 3 * i + 1); c[u][2] = __ldcs(rgb + 3 * i + 2); }
      } else {
        x[u] = y[u] = z[u] = 0.f; n[u] = 0;
      }
    }
    uint32_t key[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + u * 32 + lane;
      bool ok = i < S && isfinite(x[u]) && isfinite(y[u]) && isfinite(z[u]);
      int l = level_fixed;
      if (level_fixed < 0) { ok = ok && n[u] >= 1; l = min(n[u], g.L) - 1; }
      if (rgb) ok = ok && isfinite(c[u][0]) && isfinite(c[u][1]) && isfinite(c[u][2]);
      if (ok) {
        const int32_t c0 = clampcell(floor(__dmul_rn(__dsub_rn((double)x[u], s_org[l][0]), s_inv[l][0])), s_dim[l][0]);
        const int32_t c1 = clampcell(floor(__dmul_rn(__dsub_rn((double)y[u], s_org[l][1]), s_inv[l][1])), s_dim[l][1]);
        const int32_t c2 = clampcell(floor(__dmul_rn(__dsub_rn((double)z[u], s_org[l][2]), s_inv[l][2])), s_dim[l][2]);
        key[u] = (uint32_t)(s_coff[l] + ((int64_t)c2 * s_dim[l][1] + c1) * s_dim[l][0] + c0);
      } else {
        key[u] = kInvalidKey;
      }
      if (!ok && out_zero && i < S) { out_zero[3 * i] = 0.f; out_zero[3 * i + 1] = 0.f; out_zero[3 * i + 2] = 0.f; }
    }
    // Returning atomics, all kU in flight before any result is consumed.  Random renderer
    // order leaves nothing to aggregate within a warp: one atomic per sample.  A screen-coherent
    // order (neighbouring lanes in one cell, detected warp-uniformly) aggregates per distinct
    // key instead, so a warp's samples of one cell do not serialise on one address.  Counter
    // replica r = (i >> 5) % kRep spreads a hot cell's arrivals over kRep addresses (the
    // same-address L2 atomic rate, ~55 M/s, otherwise serialises a 4k-sample cell for 70 us).
    uint32_t rank[kU];
    unsigned peers[kU];
    bool agg[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t prev = __shfl_up_sync(0xffffffffu, key[u], 1);
      agg[u] = __any_sync(0xffffffffu, lane > 0 && key[u] != kInvalidKey && prev == key[u]);
      peers[u] = agg[u] ? __match_any_sync(0xffffffffu, key[u]) : (1u << lane);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      rank[u] = 0u;
      const uint32_t r = (uint32_t)(((i0 + u * 32) >> 5) & (kRep - 1));
      if (key[u] != kInvalidKey && lane == __ffs(peers[u]) - 1)
#ifdef GSC_EXP_KEYS_NOATOMIC   // timing experiment only: ranks are wrong
        rank[u] = r;
#else
        rank[u] = atomicAdd(b.cell_count + (size_t)r * b.nc + key[u], (uint32_t)__popc(peers[u]));
#endif
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (agg[u]) {                              // warp-uniform
        const uint32_t bb = __shfl_sync(0xffffffffu, rank[u], __ffs(peers[u]) - 1);
        rank[u] = key[u] != kInvalidKey ? bb + __popc(peers[u] & ((1u << lane) - 1u)) : 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + u * 32 + lane;
      if (i < S) b.kr[i] = make_uint2(key[u], rank[u]);
    }
  }
}

// ---- keys pass with the inputs staged by the TMA engine (cp.async.bulk): one CTA per tile of
// kBT consecutive samples; thread 0 issues one bulk copy per input array into shared memory
// (completion on an mbarrier), so no thread holds loads in registers and every thread keeps
// kBU samples' rank atomics in flight at once.  Same arithmetic, keys, replicas and warp
// aggregation as k_keys (the partial last tile goes to k_keys).  Built with -DGSC_KEYS_BULK only:
// measured (same-box A/B, cfg2 frame) 0.373 ms with k_keys vs 0.393 / 0.388 / 0.385 / 0.379 ms
// for 2048 / 1024 / 1024 (8 CTAs/SM) / 512-sample tiles -- the pass is bound by its rank
// atomics and dependent chain, not by load issue, and the staging shared memory crowds the
// kernels that run beside it; parity tests pass with it (53 world-space GPU tests).
#ifndef GSC_KB_GRID
#define GSC_KB_GRID 4
#endif
#ifndef GSC_KBT
#define GSC_KBT 2048
#endif
constexpr int kBT = GSC_KBT, kBThreads = 256, kBU = kBT / kBThreads;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}

__global__ void __launch_bounds__(kBThreads) k_keys_bulk(const float* __restrict__ pos, const int32_t* __restrict__ len,
                                                        const float* __restrict__ rgb, int level_fixed,
                                                        int64_t ntiles, LevelGeom g, IngestBufs b, float* out_zero) {
  pdl_enter();
  extern __shared__ float4 s_dyn[];
  float* s_pos = reinterpret_cast<float*>(s_dyn);
  int32_t* s_len = reinterpret_cast<int32_t*>(s_pos + 3 * kBT);
  float* s_rgb = reinterpret_cast<float*>(s_len + kBT);
  __shared__ __align__(8) unsigned long long s_bar;
  __shared__ double s_org[kMaxL][3], s_inv[kMaxL][3];
  __shared__ int32_t s_dim[kMaxL][3];
  __shared__ int64_t s_coff[kMaxL];
  if (threadIdx.x < kMaxL * 3) {
    const int l = threadIdx.x / 3, a = threadIdx.x % 3;
    s_org[l][a] = g.origin[l][a]; s_inv[l][a] = g.inv_cell[l][a]; s_dim[l][a] = g.dims[l][a];
    if (a == 0) s_coff[l] = g.coff[l];
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s_bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t phase = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t i0 = t * kBT;
    if (threadIdx.x == 0) {
      const uint32_t bytes = 12u * kBT + (level_fixed < 0 ? 4u * kBT : 0u) + (rgb ? 12u * kBT : 0u);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&s_bar)), "r"(bytes)
                   : "memory");
      bulk_g2s(s_pos, pos + 3 * i0, 12u * kBT, &s_bar);
      if (level_fixed < 0) bulk_g2s(s_len, len + i0, 4u * kBT, &s_bar);
      if (rgb) bulk_g2s(s_rgb, rgb + 3 * i0, 12u * kBT, &s_bar);
    }
    asm volatile("{\n\t.reg .pred P1;\n\tKBWAIT:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@!P1 bra KBWAIT;\n\t}\n" ::"r"(smem_addr(&s_bar)), "r"(phase) : "memory");
    phase ^= 1u;
    uint32_t key[kBU], rank[kBU];
    unsigned peers[kBU];
    bool agg[kBU];
#pragma unroll
    for (int u = 0; u < kBU; ++u) {
      const int j = u * kBThreads + threadIdx.x;
      const float x = s_pos[3 * j], y = s_pos[3 * j + 1], z = s_pos[3 * j + 2];
      const int n = level_fixed < 0 ? s_len[j] : 1;
      bool ok = isfinite(x) && isfinite(y) && isfinite(z);
      int l = level_fixed;
      if (level_fixed < 0) { ok = ok && n >= 1; l = min(n, g.L) - 1; }
      if (rgb) ok = ok && isfinite(s_rgb[3 * j]) && isfinite(s_rgb[3 * j + 1]) && isfinite(s_rgb[3 * j + 2]);
      if (ok) {
        const int32_t c0 = clampcell(floor(__dmul_rn(__dsub_rn((double)x, s_org[l][0]), s_inv[l][0])), s_dim[l][0]);
        const int32_t c1 = clampcell(floor(__dmul_rn(__dsub_rn((double)y, s_org[l][1]), s_inv[l][1])), s_dim[l][1]);
        const int32_t c2 = clampcell(floor(__dmul_rn(__dsub_rn((double)z, s_org[l][2]), s_inv[l][2])), s_dim[l][2]);
        key[u] = (uint32_t)(s_coff[l] + ((int64_t)c2 * s_dim[l][1] + c1) * s_dim[l][0] + c0);
      } else {
        key[u] = kInvalidKey;
        if (out_zero) { const int64_t i = i0 + j; out_zero[3 * i] = 0.f; out_zero[3 * i + 1] = 0.f; out_zero[3 * i + 2] = 0.f; }
      }
    }
#pragma unroll
    for (int u = 0; u < kBU; ++u) {
      const uint32_t prev = __shfl_up_sync(0xffffffffu, key[u], 1);
      agg[u] = __any_sync(0xffffffffu, lane > 0 && key[u] != kInvalidKey && prev == key[u]);
      peers[u] = agg[u] ? __match_any_sync(0xffffffffu, key[u]) : (1u << lane);
    }
#pragma unroll
    for (int u = 0; u < kBU; ++u) {
      rank[u] = 0u;
      const int64_t i = i0 + u * kBThreads + threadIdx.x;
      const uint32_t r = (uint32_t)((i >> 5) & (kRep - 1));
      if (key[u] != kInvalidKey && lane == __ffs(peers[u]) - 1)
        rank[u] = atomicAdd(b.cell_count + (size_t)r * b.nc + key[u], (uint32_t)__popc(peers[u]));
    }
#pragma unroll
    for (int u = 0; u < kBU; ++u) {
      if (agg[u]) {
        const uint32_t bb = __shfl_sync(0xffffffffu, rank[u], __ffs(peers[u]) - 1);
        rank[u] = key[u] != kInvalidKey ? bb + __popc(peers[u] & ((1u << lane) - 1u)) : 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < kBU; ++u) b.kr[i0 + u * kBThreads + threadIdx.x] = make_uint2(key[u], rank[u]);
    __syncthreads();                             // the tile's shared copy is read: next copy may land
  }
}

__global__ void __launch_bounds__(256, GSC_INGEST_MINB) k_scatter(const float* __restrict__ pos, const float* __restrict__ rgb,
                                                 int64_t S, const uint32_t* __restrict__ cell_start, IngestBufs b) {
  pdl_enter();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (t >> 5) * 32 * kU + (t & 31); i0 < S; i0 += T * kU) {
    uint32_t key[kU], rank[kU], d[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + u * 32;
      const uint2 kr = i < S ? __ldcs(b.kr + i) : make_uint2(kInvalidKey, 0u);
      key[u] = kr.x; rank[u] = kr.y;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      d[u] = key[u] != kInvalidKey
                 ? __ldg(cell_start + (size_t)(((i0 + u * 32) >> 5) & (kRep - 1)) * b.nc + key[u]) + rank[u]
                 : 0u;
    float v[kU][6];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + u * 32;
      if (key[u] != kInvalidKey) {
        v[u][0] = __ldcs(pos + 3 * i); v[u][1] = __ldcs(pos + 3 * i + 1); v[u][2] = __ldcs(pos + 3 * i + 2);
        if (rgb) { v[u][3] = __ldcs(rgb + 3 * i); v[u][4] = __ldcs(rgb + 3 * i + 1); v[u][5] = __ldcs(rgb + 3 * i + 2); }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (key[u] == kInvalidKey) continue;
      const int64_t i = i0 + u * 32;
      GSC_CHECK(d[u] < b.cap, "scatter: bin slot past the capacity");
      if (rgb) {
        st_v8(b.bin + 2 * (int64_t)d[u], make_float4(v[u][0], v[u][1], v[u][2], v[u][3]),
              make_float4(v[u][4], v[u][5], 0.f, 0.f));
      } else {   // full 32-B sectors here too: a half-sector write costs a read-modify-write in DRAM
        st_v8(b.bin + 2 * (int64_t)d[u], make_float4(v[u][0], v[u][1], v[u][2], __uint_as_float((uint32_t)i)),
              make_float4(0.f, 0.f, 0.f, 0.f));
      }
    }
  }
}

__global__ void k_levels_of(const uint2* kr, int64_t S, LevelGeom g, int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t k = kr[i].x;
    out[i] = (k == kInvalidKey) ? -1 : level_of_cell(g, k);
  }
}

#ifndef GSC_INGEST_GRID
#define GSC_INGEST_GRID 12   // CTAs per SM of the keys / scatter grids (A/B knob)
#endif
static int grid_for(int64_t n, int per_sm = GSC_INGEST_GRID) {
  int64_t b = (n + 256 * kU - 1) / (256 * kU);
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * per_sm));
}

// Whole kBT-sample tiles through k_keys_bulk when every input array is 16-byte aligned (the
// bulk copies' rule), the rest (and misaligned inputs) through k_keys.
static void keys_any(const float* pos, const int32_t* len, const float* rgb, int level_fixed, int64_t S,
                     const LevelGeom& g, IngestBufs b, float* out, cudaStream_t s) {
  const bool aligned = ((reinterpret_cast<uintptr_t>(pos) | reinterpret_cast<uintptr_t>(rgb) |
                         (level_fixed < 0 ? reinterpret_cast<uintptr_t>(len) : 0)) & 15) == 0;
  int64_t nt = 0;
#ifdef GSC_KEYS_BULK
  nt = aligned ? S / kBT : 0;
#else
  (void)aligned;
#endif
  if (nt > 0) {
    const size_t smem = (size_t)kBT * (12 + 4 + 12);
    cudaFuncSetAttribute(k_keys_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = (int)std::min<int64_t>(nt, 148 * GSC_KB_GRID);
    launch_pdl(k_keys_bulk, dim3(grid), dim3(kBThreads), smem, s, pos, len, rgb, level_fixed, nt, g, b, out);
  }
  const int64_t off = nt * kBT;
  if (S - off > 0) {
    IngestBufs bt = b;
    bt.kr = b.kr + off;
    bt.cap = b.cap - off;
    launch_pdl(k_keys, dim3(grid_for(S - off)), dim3(256), 0, s, pos + 3 * off, len ? len + off : len,
               rgb ? rgb + 3 * off : rgb, level_fixed, S - off, g, bt, out ? out + 3 * off : out);
  }
}

void launch_keys(const float* pos, const int32_t* len, const float* rgb, int level_fixed,
                 int64_t S, const LevelGeom& g, IngestBufs b, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, "ingest_keys", s);
  keys_any(pos, len, rgb, level_fixed, S, g, b, nullptr, s);
}

void launch_keys_query(const float* pos, const int32_t* len, int level_fixed, int64_t S,
                       const LevelGeom& g, IngestBufs b, float* out, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, "query_keys", s);
  keys_any(pos, len, nullptr, level_fixed, S, g, b, out, s);
}

void launch_scatter(const float* pos, const float* rgb, int64_t S, const uint32_t* cell_start,
                    IngestBufs b, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, rgb ? "ingest_scatter" : "query_scatter", s);
  launch_pdl(k_scatter, dim3(grid_for(S)), dim3(256), 0, s, pos, rgb, S, cell_start, b);
}

void launch_levels_of(const uint2* kr, int64_t S, const LevelGeom& g, int32_t* out, cudaStream_t s) {
  k_levels_of<<<grid_for(S), 256, 0, s>>>(kr, S, g, out);
}

}  // namespace gsc
