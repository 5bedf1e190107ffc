// stats.cuh -- per-call level statistics and the step scalars (Eq. 5 schedule, per-level
// AdamW skip and bias corrections).  Device functions shared by the standalone kernels (data
// parallel: an all-reduce runs between them) and the last CTA of k_fwdbwd (single GPU).
#pragma once
#include "common.cuh"

namespace gsc {

// per-CTA partial of k_fwdbwd: loss sums [kMaxL], fitted-sample counts [kMaxL], pairs, candidates
constexpr int kPart = 2 * kMaxL + 2;

struct StepHP {
  float lr[GC_NGROUPS]; float beta1, beta2; int schedule; int L;
};

// Sums the per-CTA partials, stored column-major ([kPart][nblocks]: a column is contiguous),
// one warp per column with columns strided over nwarps warps: loss sums, k_l (valid fitted
// samples per level) and the pair / candidate counters.  Fixed summation order.
__device__ __forceinline__ void stats_reduce(const double* partial, int nblocks, const uint32_t* /*unused*/,
                                             const LevelGeom& g, int64_t S, LvlStats* lvl, int warp,
                                             int nwarps, int lane) {
  for (int col = warp; col < kPart; col += nwarps) {
    const double* p = partial + (int64_t)col * nblocks;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    int b = lane;
    for (; b + 96 < nblocks; b += 128) {       // four independent loads in flight per lane
#pragma unroll
      for (int q = 0; q < 4; ++q) a[q] += __ldcg(p + b + 32 * q);
    }
    for (; b < nblocks; b += 32) a[0] += __ldcg(p + b);
    double acc = (a[0] + a[1]) + (a[2] + a[3]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      if (col < kMaxL) lvl->loss_sum[col] = acc;
      else if (col < 2 * kMaxL) lvl->count[col - kMaxL] = col - kMaxL < g.L ? acc : 0.0;
      else if (col == 2 * kMaxL) lvl->n_pairs = acc;
      else lvl->n_cand = acc;
    }
  }
}

__device__ __forceinline__ void stats_totals(const LvlStats* lvl, const LevelGeom& g, int64_t S, LvlStats* out) {
  double tot = 0.0;
  for (int l = 0; l < g.L; ++l) tot += lvl->count[l];
  out->n_valid = tot;
  out->n_in = (double)S;
}

// One warp: Eq. 5 schedule, per-level skip (A12), bias corrections, stats.  Lane l
// owns level l; beta^step is a running product (no pow on the critical path).
__device__ __forceinline__ void step_scalars_warp(const LvlStats* lvl, DevState* st, const StepHP& hp,
                                                  gc_fit_stats* out, int lane) {
  double tot = 0.0;
  for (int l = 0; l < hp.L; ++l) tot += lvl->count[l];
  const int stepped = tot > 0.0;
  const long long t = st->t + stepped;
  __syncwarp();
  if (lane < GC_NGROUPS)
    st->eta[lane] = hp.schedule ? (float)((double)hp.lr[lane] / (1.0 + log((double)t))) : hp.lr[lane];
  if (lane < kMaxL) {
    const int l = lane;
    const double k = l < hp.L ? lvl->count[l] : 0.0;
    const int act = stepped && k > 0.0;
    st->active[l] = act;
    double p1 = st->b1pow[l], p2 = st->b2pow[l];
    if (act) {
      st->adam_step[l] += 1;
      p1 *= (double)hp.beta1; p2 *= (double)hp.beta2;
      st->b1pow[l] = p1; st->b2pow[l] = p2;
    }
    st->bc1[l] = (float)(1.0 - p1);
    st->bc2[l] = (float)(1.0 - p2);
    st->inv3k[l] = act ? (float)(1.0 / (3.0 * k)) : 0.f;
    out->count[l] = (int64_t)k;
    out->loss[l] = k > 0.0 ? lvl->loss_sum[l] / (3.0 * k) : 0.0;
  }
  if (lane == 0) {
    st->stepped = stepped;
    st->nonfinite = 0ull;
    st->t = t;
    out->n_in = (int64_t)lvl->n_in;
    out->n_valid = (int64_t)lvl->n_valid;
    out->n_dropped = (int64_t)(lvl->n_in - lvl->n_valid);
    out->step = stepped ? t : 0;
    out->nonfinite_grads = 0;
    out->n_pairs = (int64_t)lvl->n_pairs;
    out->n_candidates = (int64_t)lvl->n_cand;
  }
}

}  // namespace gsc
