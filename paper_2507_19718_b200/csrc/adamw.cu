// adamw.cu -- per-call level statistics, the Eq. 5 schedule scalars, and the fused
// normalise + chain rule + AdamW + next-step record/cull-count kernel (A6).
#include "common.cuh"
#include "kernels.h"
#include "record.cuh"
#include "stats.cuh"

namespace gsc {


constexpr int kStatsThreads = ((kSlots * kPart + 31) / 32) * 32;

// Level statistics of the call; with do_step (single GPU: no all-reduce in between) warp 0
// then takes the step scalars in the same launch.
__global__ void __launch_bounds__(kStatsThreads) k_stats(double* __restrict__ partial, LevelGeom g, int64_t S,
                                                         LvlStats* lvl, int do_step, DevState* st, StepHP hp,
                                                         gc_fit_stats* out) {
  pdl_enter();
  stats_reduce(partial, g, lvl);
  __syncthreads();
  if (threadIdx.x == 0) stats_totals(lvl, g, S, lvl);
  if (!do_step) return;
  __syncthreads();
  if (threadIdx.x < 32) step_scalars_warp(lvl, st, hp, out, threadIdx.x);
}

__global__ void k_step_scalars(const LvlStats* __restrict__ lvl, DevState* st, StepHP hp,
                               gc_fit_stats* out) {
  pdl_enter();
  step_scalars_warp(lvl, st, hp, out, threadIdx.x);
}

constexpr int kAdamThreads = 128, kAdamBlocksPerSM = 4;
#ifndef GSC_ADAM_GRID
#define GSC_ADAM_GRID kAdamBlocksPerSM   // CTAs per SM of the grid (A/B: fewer leave the ingest room)
#endif

struct AdamHP {
  float wd[GC_NGROUPS]; float beta1, beta2, eps; double tau;
  int frozen;               // bit g: reading A16, lr 0 -> group g excluded from the optimizer
  const uint8_t* owner;     // owner-computes (mode 2): step only Gaussians with owner[j] == me
  int me;
  int64_t gb, ge;           // ZeRO data parallel (mode 3): step only Gaussians in [gb, ge)
};

__device__ __forceinline__ int group_of(int k) { return k < 3 ? 0 : (k < 7 ? 1 : (k < 10 ? 2 : (k < 13 ? 3 : 4))); }

// Chain rule (C5) from the 12 coefficient gradients (dmu, packed dA, dv) to 14 raw grads.
__device__ void chain_rule(const float p[kNP], const float cg[12], float out[kNP]) {
  out[0] = cg[0]; out[1] = cg[1]; out[2] = cg[2];
  const float wo = 1.f / (1.f + expf(-p[P_O]));
  const float c0 = fmaxf(p[P_C], 0.f), c1 = fmaxf(p[P_C + 1], 0.f), c2 = fmaxf(p[P_C + 2], 0.f);
  const float dwo = cg[9] * c0 + cg[10] * c1 + cg[11] * c2;
  out[P_O] = dwo * wo * (1.f - wo);
  out[P_C] = p[P_C] > 0.f ? wo * cg[9] : 0.f;
  out[P_C + 1] = p[P_C + 1] > 0.f ? wo * cg[10] : 0.f;
  out[P_C + 2] = p[P_C + 2] > 0.f ? wo * cg[11] : 0.f;
  if (cg[3] == 0.f && cg[4] == 0.f && cg[5] == 0.f && cg[6] == 0.f && cg[7] == 0.f && cg[8] == 0.f) {
    // dL/dA = 0 (the lite backward of an isotropic chunk with the scale group frozen):
    // ds = -2 D (R^T 0 R) = 0 and dR = 2 * 0 * R D = 0 exactly -- skip the rotation algebra
    out[3] = out[4] = out[5] = out[6] = 0.f;
    out[P_S] = out[P_S + 1] = out[P_S + 2] = 0.f;
    return;
  }
  const float qw0 = p[P_Q], qx0 = p[P_Q + 1], qy0 = p[P_Q + 2], qz0 = p[P_Q + 3];
  const float n2 = qw0 * qw0 + qx0 * qx0 + qy0 * qy0 + qz0 * qz0;
  const bool deg = n2 < 1e-24f;
  float qn = sqrtf(n2), w = 1.f, x = 0.f, y = 0.f, z = 0.f;
  if (!deg) { w = qw0 / qn; x = qx0 / qn; y = qy0 / qn; z = qz0 / qn; }
  float R[3][3];
  R[0][0] = 1.f - 2.f * (y * y + z * z); R[0][1] = 2.f * (x * y - w * z); R[0][2] = 2.f * (x * z + w * y);
  R[1][0] = 2.f * (x * y + w * z); R[1][1] = 1.f - 2.f * (x * x + z * z); R[1][2] = 2.f * (y * z - w * x);
  R[2][0] = 2.f * (x * z - w * y); R[2][1] = 2.f * (y * z + w * x); R[2][2] = 1.f - 2.f * (x * x + y * y);
  const float D[3] = {expf(-2.f * p[P_S]), expf(-2.f * p[P_S + 1]), expf(-2.f * p[P_S + 2])};
  const float G[3][3] = {{cg[3], cg[6], cg[7]}, {cg[6], cg[4], cg[8]}, {cg[7], cg[8], cg[5]}};
  // GR = G R ; M_kk = (R^T G R)_kk ; dR = 2 G R D
  float GR[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) GR[a][b] = G[a][0] * R[0][b] + G[a][1] * R[1][b] + G[a][2] * R[2][b];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float Mkk = R[0][k] * GR[0][k] + R[1][k] * GR[1][k] + R[2][k] * GR[2][k];
    out[P_S + k] = -2.f * D[k] * Mkk;
  }
  if (deg) {
    out[3] = out[4] = out[5] = out[6] = 0.f;
  } else {
    float dR[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) dR[a][b] = 2.f * GR[a][b] * D[b];
    // dR/dq_hat (C5) contracted with dR
    const float dw = 2.f * (-z * dR[0][1] + y * dR[0][2] + z * dR[1][0] - x * dR[1][2] - y * dR[2][0] + x * dR[2][1]);
    const float dx = 2.f * (y * dR[0][1] + z * dR[0][2] + y * dR[1][0] - 2.f * x * dR[1][1] - w * dR[1][2] +
                            z * dR[2][0] + w * dR[2][1] - 2.f * x * dR[2][2]);
    const float dy = 2.f * (-2.f * y * dR[0][0] + x * dR[0][1] + w * dR[0][2] + x * dR[1][0] + z * dR[1][2] -
                            w * dR[2][0] + z * dR[2][1] - 2.f * y * dR[2][2]);
    const float dz = 2.f * (-2.f * z * dR[0][0] - w * dR[0][1] + x * dR[0][2] + w * dR[1][0] - 2.f * z * dR[1][1] +
                            y * dR[1][2] + x * dR[2][0] + y * dR[2][1]);
    const float dot = w * dw + x * dx + y * dy + z * dz;
    out[3] = (dw - w * dot) / qn; out[4] = (dx - x * dot) / qn;
    out[5] = (dy - y * dot) / qn; out[6] = (dz - z * dot) / qn;
  }
}

// Fused normalise + chain rule + AdamW of one Gaussian per thread (A6); zeroes the gradient
// slots it consumes.  The next step's evaluation record and culling counts are emitted by
// k_record_cull right after (split so both kernels stay spill-free and latency-hidden).
#ifndef GSC_ADAM_MINB
#define GSC_ADAM_MINB kAdamBlocksPerSM
#endif
__global__ void __launch_bounds__(kAdamThreads, GSC_ADAM_MINB) k_adamw(
    int64_t G, float* __restrict__ P, float* __restrict__ M, float* __restrict__ V, float* __restrict__ grad,
    float* __restrict__ dbg, DevState* st, AdamHP hp, LevelGeom g, unsigned long long* nonfinite,
    const float* __restrict__ rawg) {
  pdl_enter();
  // the culling rebuild that follows this kernel (k_record_cull -> scan -> k_cull_emit) sets the
  // overflow flag afresh; the previous rebuild's flag has been read by this call's k_stats
  if (blockIdx.x == 0 && threadIdx.x == 0) st->csr_overflow = 0u;
  unsigned long long bad = 0;
  float eta[GC_NGROUPS], dec[GC_NGROUPS];
#pragma unroll
  for (int k = 0; k < GC_NGROUPS; ++k) { eta[k] = st->eta[k]; dec[k] = 1.f - eta[k] * hp.wd[k]; }
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < G; j += (int64_t)gridDim.x * blockDim.x) {
    // every load of the Gaussian is issued before any is consumed (one memory latency, not three)
    float4* gp = reinterpret_cast<float4*>(grad + 12 * j);
    const float4 c0 = gp[0], c1 = gp[1], c2 = gp[2];
    float p[kNP], m[kNP], v[kNP];
#pragma unroll
    for (int k = 0; k < kNP; ++k) { p[k] = P[k * G + j]; m[k] = M[k * G + j]; v[k] = V[k * G + j]; }
    const int l = level_of_gaussian(g, j);
    const bool act = st->active[l] != 0 && (!hp.owner || hp.owner[j] == hp.me) && j >= hp.gb && j < hp.ge;
    const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
    gp[0] = zero; gp[1] = zero; gp[2] = zero;
    if (!act && !dbg) continue;
    const float s = st->inv3k[l];
    const float cg[12] = {c0.x * s, c0.y * s, c0.z * s, c0.w * s, c1.x * s, c1.y * s,
                          c1.z * s, c1.w * s, c2.x * s, c2.y * s, c2.z * s, c2.w * s};
    float raw[kNP];
    if (rawg) {                      // screen-space path: raw gradients given (normalised here)
#pragma unroll
      for (int k = 0; k < kNP; ++k) raw[k] = rawg[k * G + j] * s;
    } else {
      chain_rule(p, cg, raw);
    }
    if (dbg) {
#pragma unroll
      for (int k = 0; k < kNP; ++k) dbg[k * G + j] = raw[k];
    }
    if (!act) continue;
    const float ibc1 = 1.f / st->bc1[l], ibc2 = 1.f / st->bc2[l];
#pragma unroll
    for (int k = 0; k < kNP; ++k) {
      const int grp = k < 3 ? 0 : (k < 7 ? 1 : (k < 10 ? 2 : (k < 13 ? 3 : 4)));   // constant after unroll
      if ((hp.frozen >> grp) & 1) continue;    // parameters and moments unchanged (A16)
      const float gk = raw[k];
      const bool ok = isfinite(gk);
      bad += !ok;
      const float mk = hp.beta1 * m[k] + (1.f - hp.beta1) * gk;
      const float vk = hp.beta2 * v[k] + (1.f - hp.beta2) * gk * gk;
      const float pk = p[k] * dec[grp] - eta[grp] * (mk * ibc1) / (sqrtf(vk * ibc2) + hp.eps);
      if (ok) { M[k * G + j] = mk; V[k * G + j] = vk; P[k * G + j] = pk; }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(nonfinite, bad);
}

static StepHP step_hp(const gc_hparams& hp, int L) {
  StepHP h;
  for (int k = 0; k < GC_NGROUPS; ++k) h.lr[k] = hp.lr[k];
  h.beta1 = hp.beta1; h.beta2 = hp.beta2; h.schedule = hp.lr_schedule; h.L = L;
  return h;
}

void launch_stats(double* partial, const LevelGeom& g, int64_t S, LvlStats* lvl, bool with_step, DevState* st,
                  const gc_hparams& hp, int L, gc_fit_stats* dev_stats, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, "stats", s);
  launch_pdl(k_stats, dim3(1), dim3(kStatsThreads), 0, s, partial, g, S, lvl, with_step ? 1 : 0, st,
             step_hp(hp, L), dev_stats);
}

void launch_step_scalars(const LvlStats* lvl, DevState* st, const gc_hparams& hp, int L,
                         gc_fit_stats* dev_stats, cudaStream_t s) {
  launch_pdl(k_step_scalars, dim3(1), dim3(32), 0, s, lvl, st, step_hp(hp, L), dev_stats);
}

void launch_adamw(int64_t G, float* P, float* M, float* V, float* grad, CullBufs cb, float* dbg_grad,
                  DevState* st, const gc_hparams& hp,
                  const LevelGeom& g, unsigned long long* nonfinite, cudaStream_t s, Profiler* prof,
                  const float* raw_grad, const uint8_t* owner, int me, bool with_record, int64_t g_begin,
                  int64_t g_end) {
  AdamHP h;
  for (int k = 0; k < GC_NGROUPS; ++k) h.wd[k] = hp.weight_decay[k];
  h.beta1 = hp.beta1; h.beta2 = hp.beta2; h.eps = hp.adam_eps; h.tau = (double)hp.cutoff_sigma;
  h.frozen = 0;
  h.owner = owner; h.me = me;
  h.gb = g_begin; h.ge = g_end < 0 ? G : g_end;
  for (int k = 0; k < GC_NGROUPS; ++k) h.frozen |= (hp.lr[k] == 0.f ? 1 : 0) << k;
  {
    ProfScope ps(prof, "adamw", s);
    int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((G + kAdamThreads - 1) / kAdamThreads, 148 * GSC_ADAM_GRID));
    launch_pdl(k_adamw, dim3(blocks), dim3(kAdamThreads), 0, s, G, P, M, V, grad, dbg_grad, st, h, g, nonfinite,
               raw_grad);
  }
  if (with_record) {
    ProfScope ps(prof, "record_cull", s);
    launch_record_cull(G, P, h.tau, g, cb, st, s);
  }
}

}  // namespace gsc
