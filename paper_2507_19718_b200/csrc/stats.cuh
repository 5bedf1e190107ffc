// stats.cuh -- per-call level statistics and the step scalars (Eq. 5 schedule, per-level
// AdamW skip and bias corrections).  Device functions of k_stats (single GPU: both in one
// launch) and k_step_scalars (data parallel: the all-reduce runs between them).
#pragma once
#include "common.cuh"

namespace gsc {

// partials of k_fwdbwd: loss sums [kMaxL], fitted-sample counts [kMaxL], pairs, candidates;
// accumulated into kSlots slots [kSlots][kPart] (zero between calls)
constexpr int kPart = 2 * kMaxL + 2;
constexpr int kSlots = 16;

struct StepHP {
  float lr[GC_NGROUPS]; float beta1, beta2; int schedule; int L;
};

// Sums the kSlots slotted partials per column in a fixed order and re-zeroes the slots (one
// CTA of >= kSlots * kPart threads): loss sums, k_l (valid fitted samples per level) and the
// pair / candidate counters.
__device__ __forceinline__ void stats_reduce(double* partial, const LevelGeom& g, LvlStats* lvl) {
  __shared__ double s_v[kSlots][kPart];
  const int t = threadIdx.x;
  if (t < kSlots * kPart) {
    s_v[t / kPart][t % kPart] = __ldcg(partial + t);
    partial[t] = 0.0;
  }
  __syncthreads();
  if (t < kPart) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < kSlots; ++q) acc += s_v[q][t];
    if (t < kMaxL) lvl->loss_sum[t] = acc;
    else if (t < 2 * kMaxL) lvl->count[t - kMaxL] = t - kMaxL < g.L ? acc : 0.0;
    else if (t == 2 * kMaxL) lvl->n_pairs = acc;
    else lvl->n_cand = acc;
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
  // lists that overflowed at their last rebuild were incomplete for this call's fwd/bwd:
  // skip the step (reported in gc_fit_stats.flags; the host grows the lists on its next call)
  const unsigned int ovf = *(volatile unsigned int*)&st->csr_overflow;
  const int stepped = tot > 0.0 && ovf == 0u;
  const long long t = st->t + stepped;
  __syncwarp();
  if (lane < GC_NGROUPS)
    st->eta[lane] = hp.schedule ? (float)((double)hp.lr[lane] / (1.0 + log((double)t))) : hp.lr[lane];
  if (lane < kMaxL) {
    const int l = lane;
    const double k = l < hp.L ? lvl->count[l] : 0.0;
    const int act = stepped && k > 0.0 && ((st->owned >> l) & 1u);   // level-sharded: own levels only
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
    st->t = t;
    out->n_in = (int64_t)lvl->n_in;
    out->n_valid = (int64_t)lvl->n_valid;
    out->n_dropped = (int64_t)(lvl->n_in - lvl->n_valid);
    out->step = stepped ? t : 0;
    out->nonfinite_grads = (int64_t)st->nonfinite;   // a deferred previous step's count, else 0
    st->nonfinite = 0ull;
    out->n_pairs = (int64_t)lvl->n_pairs;
    out->n_candidates = (int64_t)lvl->n_cand;
    out->flags = ovf ? (int64_t)GC_FLAG_LISTS_OVERFLOWED : 0;
  }
}

}  // namespace gsc
