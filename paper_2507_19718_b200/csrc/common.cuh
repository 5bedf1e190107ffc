// common.cuh -- internal types and device helpers of libgscache (sm_100a only).
// Not part of the ABI; see include/gscache.h and DESIGN.md.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gscache.h"

// Checked build (-DGSC_CHECKED, tools/build_variant.py): device-side bounds checks on the
// index arithmetic of the hot kernels (bins, work items, list entries, gradient rows, outputs,
// screen-space key / range / image buffers).  A failed check prints the site and traps, so
// the call fails with a sticky CUDA error.  The GPU pool refuses compute-sanitizer; the
// whole `-m gpu` suite runs against this build instead.  Compiled out of
// the product build.
#include <cstdio>
#ifdef GSC_CHECKED
#define GSC_CHECK(cond, what)                                                                  \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("GSC_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,   \
             (int)blockIdx.x, (int)threadIdx.x);                                               \
      __trap();                                                                                \
    }                                                                                          \
  } while (0)
#else
#define GSC_CHECK(cond, what) do { } while (0)
#endif

namespace gsc {

constexpr int kMaxL = GC_MAX_LEVELS;
constexpr int kNP = 14;              // raw floats per Gaussian
constexpr int kCH = 64;              // samples per work item: one warp, two samples per lane
#ifndef GSC_SCAN_THREADS
#define GSC_SCAN_THREADS 1024
#endif
#ifndef GSC_SCAN_MINB
#define GSC_SCAN_MINB 1
#endif
constexpr int kScanThreads = GSC_SCAN_THREADS;   // one scan tile per CTA: kScanThreads threads x 8 items
constexpr int kScanTile = 8 * kScanThreads;
#ifndef GSC_KREP
#define GSC_KREP 4
#endif
constexpr int kRep = GSC_KREP;        // replicated per-cell sample counters (hot-cell atomics / kRep;
                                      // measured cfg2 frame: 4 -> 0.382 ms, 8 -> 0.385, 2 -> 0.430, 1 -> 0.459)
constexpr uint32_t kInvalidKey = 0xFFFFFFFFu;

// Plane index of raw parameter column k in the SoA parameter store (paper order).
enum { P_MU = 0, P_Q = 3, P_C = 7, P_S = 10, P_O = 13 };

// Per-level geometry, passed by value to kernels (fixed at create).
struct LevelGeom {
  int L;
  int64_t goff[kMaxL + 1];           // Gaussian offsets of each level in the global arrays
  int64_t coff[kMaxL + 1];           // cell offsets of each level's grid in the global cell ids
  double origin[kMaxL][3];
  double inv_cell[kMaxL][3];
  double edge[kMaxL][3];             // 1.0 / inv_cell (IEEE division on the host, as the oracle)
  int32_t dims[kMaxL][3];
};

// Device-resident optimizer / schedule state (persistent across calls; graph friendly).
struct DevState {
  long long t;                       // Eq. 5 counter: stepping fits since create / reset
  long long adam_step[kMaxL];        // per-level AdamW bias-correction counters (A12)
  double b1pow[kMaxL], b2pow[kMaxL]; // beta^adam_step, kept as running products
  float eta[GC_NGROUPS];             // eta_g(t) of the current step
  float bc1[kMaxL], bc2[kMaxL];      // 1 - beta^step per level (current step)
  float inv3k[kMaxL];                // 1 / (3 k_l) (0 when the level is skipped)
  int active[kMaxL];                 // level takes a step this call
  int stepped;                       // this call stepped (>= 1 valid sample)
  unsigned long long nonfinite;      // non-finite gradient elements skipped by a deferred step
  unsigned int csr_overflow;         // a rebuild dropped entries past the list capacity (the
                                     // host guard detects it from the entry count, csr_guard)
  unsigned int ovf_next;             // bump allocator of the wide-range rank slots (per rebuild)
  unsigned int owned;                // bit l: this rank steps level l (all ones unless level-sharded)
  // the culling lists (entries [lcap][4] float4) and the wide-range rank slots [lovf_cap]: read
  // by the kernels from here rather than from launch arguments, so that CUDA graphs captured
  // before a capacity growth use the grown buffers
  float4* lrec;
  uint32_t* lovf;
  uint32_t lcap, lovf_cap;
};

// Per-call level statistics; summed over ranks under data parallelism (all doubles so a
// single NCCL all-reduce covers them).
struct LvlStats {
  double count[kMaxL];
  double loss_sum[kMaxL];            // sum over samples of sum_ch (x-y)^2/(y+eps)^2
  double n_pairs, n_cand, n_valid, n_in;
};

// Work item of the binned sample stream: samples [start, start+count) of cell `cell`.
struct WorkItem { int cell, start, count, level; };

__device__ __forceinline__ int level_of_cell(const LevelGeom& g, int64_t cell) {
  int l = 0;
#pragma unroll 1
  for (int k = 1; k < g.L; ++k) l += (cell >= g.coff[k]);
  return l;
}

__device__ __forceinline__ int level_of_gaussian(const LevelGeom& g, int64_t j) {
  int l = 0;
#pragma unroll 1
  for (int k = 1; k < g.L; ++k) l += (j >= g.goff[k]);
  return l;
}

// C8 clamp of a floored cell coordinate (NaN / -inf -> 0, large -> dims-1).
__device__ __forceinline__ int32_t clampcell(double f, int32_t dim) {
  if (!(f >= 0.0)) return 0;
  if (f > (double)(dim - 1)) return dim - 1;
  return (int32_t)f;
}

// Sample cell (C8), fp64 without contraction: floor((x - origin) * inv_cell).
__device__ __forceinline__ int64_t sample_cell(const LevelGeom& g, int l, float x, float y, float z) {
  int32_t c0 = clampcell(floor(__dmul_rn(__dsub_rn((double)x, g.origin[l][0]), g.inv_cell[l][0])), g.dims[l][0]);
  int32_t c1 = clampcell(floor(__dmul_rn(__dsub_rn((double)y, g.origin[l][1]), g.inv_cell[l][1])), g.dims[l][1]);
  int32_t c2 = clampcell(floor(__dmul_rn(__dsub_rn((double)z, g.origin[l][2]), g.inv_cell[l][2])), g.dims[l][2]);
  return g.coff[l] + ((int64_t)c2 * g.dims[l][1] + c1) * g.dims[l][0] + c0;
}

// Programmatic dependent launch: every hot-path kernel waits for its predecessor's memory at
// its top and immediately allows its own successor to be scheduled (the successor's CTAs then
// sit in griddepcontrol.wait while this grid drains, hiding the launch gap).
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 32-byte global accesses (sm_100: LDG/STG.E.ENL2.256): one instruction and one sector per
// fit sample bin.
__device__ __forceinline__ void st_v8(float4* p, const float4& a, const float4& b) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(a.x), "f"(a.y), "f"(a.z), "f"(a.w),
               "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w) : "memory");
}
__device__ __forceinline__ void ld_v8_nc(const float4* p, float4& a, float4& b) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
               : "l"(p));
}

// Vector reduction into global memory (sm_90+): REDG.E.ADD.F32x4.
__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}

// Evaluation record (48 B, 3 x float4): the upper-triangular Cholesky factor U of
// A = Sigma^-1 = U^T U (Q = |U (x - mu)|^2), the mean mu and the amplitude v = w max(0, c):
//   r0 = (U00, U01, U02, U11)  r1 = (U12, U22, mu_x, mu_y)  r2 = (mu_z, v0, v1, v2)

}  // namespace gsc
