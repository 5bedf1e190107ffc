// fwdbwd.cu -- the fused forward + HDR loss + backward kernel of gc_fit (A4) and the
// forward-only lookup kernel of gc_query (A7).  Warp-centric: no block barriers.
//
// A work item is <= 64 binned samples of one (level, cell) bin; one warp owns it, every lane
// two samples (s = lane, lane + 32; one when the item has <= 32) so that each staged
// candidate feeds two evaluations, run as packed fp32x2 (FADD2/FMUL2/FFMA2) issues.  The
// cell's culling list (C8: 64-B entries, record + Gaussian index) is staged into the warp's
// shared memory 32 candidates at a time, recentred on the centre of the item's cell.
//   pass 1 (lane = sample pair): yhat = sum v_j e^{-Q/2} over the candidates with
//          Q <= tau^2 (C3); lane k keeps candidate k's inside ballots (which samples it
//          covers); the Eq. 4 loss and g = dL/dyhat (C4, unnormalised -- the 1/(3 k_l)
//          factor is applied by the optimizer once k_l is known globally, C9).
//   pass 2 (lane = slice of contributing pairs): per chunk, the pairs in candidate-major
//          order are cut into 32 contiguous slices; a lane walks its slice through the
//          ballots, recomputes e with pass 1's arithmetic, accumulates the C5 coefficient
//          gradients of the current Gaussian in registers and issues red.global.add.v4.f32
//          at each change of Gaussian.  Work is proportional to the contributing pairs;
//          never shared-memory float atomics (a CAS loop on sm_100a).  Cells with more than
//          384 candidates re-derive their pairs in batches (dense fallback).
#include <type_traits>
#include "common.cuh"
#include "kernels.h"
#include "stats.cuh"

namespace gsc {

constexpr int kWarps = 8;                                 // warps per CTA
constexpr int kPairCap = 512;                             // pair batch of the dense fallback path
constexpr int kMaskChunks = 12;                           // chunks whose inside masks are kept (C <= 384)
constexpr uint32_t kClaimFit = 1, kClaimQuery = 2;        // work items per claim (measured: the
                                                          // lookups' lighter items gain from 2, fwd/bwd's tail loses)
constexpr float kNegHalfLog2e = -0.72134752044448170f;    // -0.5 * log2(e)
static_assert(kCH == 64, "two samples per lane");

// Staged candidate (64 B in shared memory), relative to the work item's reference point
// x_ref (the centre of its cell, CellRef): c = U (mu - x_ref), so that for x' = x - x_ref
//   w = U x' - c = U (x - mu),  Q = |w|^2   (9 FMA per pair; recentring keeps fp32 exact enough)
struct ChunkSmem {
  float4 r0[32];                   // U00 U01 U02 U11
  float4 r1[32];                   // U12 U22 -c0 -c1
  float4 r2[32];                   // -c2 v0 v1 v2
  float4 r3[32];                   // mu - x_ref, gid (as bits)
};

struct WarpSmem : ChunkSmem {
  float4 sxg[64];                  // sample x', y', z', g0
  float2 sg[64];                   // sample g1, g2
  union {
    uint2 mask[kMaskChunks][32];   // pass 1 -> 2: which samples (a | b<<32) lie inside candidate k of chunk c
    struct {                       // dense fallback: a batch of pairs, candidate-major
      uint16_t pkey[kPairCap];     // (candidate-in-chunk << 6) | sample
      float pe[kPairCap];          // e = exp(-Q/2) of the pair
    } list;
  } u;
  int offs[32];                    // pass 2: first pair of candidate k in the chunk's pair order
};

struct Cand { float u00, u01, u02, u11, u12, u22, nc0, nc1, nc2, v0, v1, v2; };

__device__ __forceinline__ Cand cand_from(const ChunkSmem& w, int k) {
  const float4 p = w.r0[k], q = w.r1[k], r = w.r2[k];
  return Cand{p.x, p.y, p.z, p.w, q.x, q.y, q.z, q.w, r.x, r.y, r.z, r.w};
}

// w = U x' - c and Q = |w|^2, with the operation order fixed (identical in every pass).
__device__ __forceinline__ float cand_q(const Cand& g, float x, float y, float z, float& w0, float& w1, float& w2) {
  w0 = __fmaf_rn(g.u02, z, __fmaf_rn(g.u01, y, __fmaf_rn(g.u00, x, g.nc0)));
  w1 = __fmaf_rn(g.u12, z, __fmaf_rn(g.u11, y, g.nc1));
  w2 = __fmaf_rn(g.u22, z, g.nc2);
  return __fmaf_rn(w2, w2, __fmaf_rn(w1, w1, __fmul_rn(w0, w0)));
}

// Stages one chunk and returns (warp-uniformly) whether every candidate is isotropic
// (U = u I, exact for equal log-scales; the paper's setting).  Isotropic chunks use the
// layout r0 = (mu - x_ref, tau^2/u^2), r1 = (-0.5 log2e u^2, v), r2.x = u^2, r3 as usual;
// general chunks r0..r2 as documented on ChunkSmem.  (The expanded form g|x'|^2 + g|m|^2 -
// 2g x'.m saves 2 ops per test but its cancellation costs ~1e-5 relative: measured, rejected.)
__device__ __forceinline__ bool stage_chunk(ChunkSmem& w, const float4* __restrict__ lrec, int base, int kc, int lane,
                                            float xr, float yr, float zr, float tau2, int64_t G) {
  __syncwarp();
  float4 p = make_float4(0.f, 0.f, 0.f, 0.f), q = p, r = p;
  int gid = 0;
  if (lane < kc) {
    float4 t;                                    // list entry: record (3 x float4) + gid
    ld_v8_nc(lrec + 4 * (int64_t)(base + lane), p, q);
    ld_v8_nc(lrec + 4 * (int64_t)(base + lane) + 2, r, t);
    gid = __float_as_int(t.x);
    GSC_CHECK(gid >= 0 && gid < G, "list entry Gaussian index");
  }
  const bool iso = __all_sync(0xffffffffu, lane >= kc || (p.y == 0.f && p.z == 0.f && q.x == 0.f &&
                                                           p.x == p.w && p.w == q.y));
  if (lane < kc) {
    const float m0 = q.z - xr, m1 = q.w - yr, m2 = r.x - zr;
    if (iso) {
      const float u2 = p.x * p.x;
      w.r0[lane] = make_float4(m0, m1, m2, tau2 / u2);
      w.r1[lane] = make_float4(kNegHalfLog2e * u2, r.y, r.z, r.w);
      w.r2[lane] = make_float4(u2, 0.f, 0.f, 0.f);
    } else {
      const float c0 = fmaf(p.z, m2, fmaf(p.y, m1, p.x * m0));
      const float c1 = fmaf(q.x, m2, p.w * m1);
      const float c2 = q.y * m2;
      w.r0[lane] = p;
      w.r1[lane] = make_float4(q.x, q.y, -c0, -c1);
      w.r2[lane] = make_float4(-c2, r.y, r.z, r.w);
    }
    w.r3[lane] = make_float4(m0, m1, m2, __int_as_float(gid));
  }
  __syncwarp();
  return iso;
}

// Isotropic test value s = |x' - m|^2 (operation order fixed: every pass agrees).
__device__ __forceinline__ float iso_s(const float (&x)[3], const float4& c) {
  const float dx = __fsub_rn(x[0], c.x), dy = __fsub_rn(x[1], c.y), dz = __fsub_rn(x[2], c.z);
  return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

// Isotropic chunk: s = |x' - m|^2 <= tau^2/u^2, e = 2^{-0.5 log2e u^2 s} (7 ops per test).
// Branch-free: e is computed for every lane and zeroed outside (MUFU has the slack; a
// divergent inside block costs more issue slots than it saves).  kMask (pass 1 of a fit):
// lane k also keeps candidate k's ballots (which samples it covers) in cm -- three
// instructions per candidate instead of appending a pair list.  kTwo = false: the item has
// <= 32 samples, sample b is skipped.
template <bool kMask, bool kTwo>
__device__ __forceinline__ void eval_chunk_iso(const ChunkSmem& w, int kc, const float (&xa)[3], const float (&xb)[3],
                                               float (&ya)[3], float (&yb)[3], uint2& cm, int lane) {
  if constexpr (kTwo) {
    // Both samples at once in packed fp32x2 arithmetic (FADD2 / FMUL2 / FFMA2, the candidate's
    // values as broadcast operands): each half rounds exactly like the scalar form below, so
    // the results are bit-identical to iso_s and pass 2's recomputation, at ~40% fewer issues.
    const float2 X = make_float2(xa[0], xb[0]), Y = make_float2(xa[1], xb[1]), Z = make_float2(xa[2], xb[2]);
    float2 A0 = make_float2(ya[0], yb[0]), A1 = make_float2(ya[1], yb[1]), A2 = make_float2(ya[2], yb[2]);
#pragma unroll 2
    for (int k = 0; k < kc; ++k) {
      const float4 c = w.r0[k], f = w.r1[k];
      const float2 dx = __fadd2_rn(X, make_float2(-c.x, -c.x)), dy = __fadd2_rn(Y, make_float2(-c.y, -c.y)),
                   dz = __fadd2_rn(Z, make_float2(-c.z, -c.z));
      const float2 s = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
      const bool ina = s.x <= c.w, inb = s.y <= c.w;
      const float2 t = __fmul2_rn(s, make_float2(f.x, f.x));
      const float ea_ = ex2_approx(t.x), eb_ = ex2_approx(t.y);
      const float2 e = make_float2(ina ? ea_ : 0.f, inb ? eb_ : 0.f);
      A0 = __ffma2_rn(e, make_float2(f.y, f.y), A0);
      A1 = __ffma2_rn(e, make_float2(f.z, f.z), A1);
      A2 = __ffma2_rn(e, make_float2(f.w, f.w), A2);
      if constexpr (kMask) {
        const uint32_t ma = __ballot_sync(0xffffffffu, ina), mb = __ballot_sync(0xffffffffu, inb);
        if (lane == k) cm = make_uint2(ma, mb);
      }
    }
    ya[0] = A0.x; ya[1] = A1.x; ya[2] = A2.x;
    yb[0] = A0.y; yb[1] = A1.y; yb[2] = A2.y;
    __syncwarp();
    return;
  }
#pragma unroll 2
  for (int k = 0; k < kc; ++k) {
    const float4 c = w.r0[k], f = w.r1[k];
    const float sa = iso_s(xa, c), sb = kTwo ? iso_s(xb, c) : 0.f;
    const bool ina = sa <= c.w, inb = kTwo && sb <= c.w;
    const float xa_ = ex2_approx(f.x * sa);
    const float ea = ina ? xa_ : 0.f;
    ya[0] = fmaf(f.y, ea, ya[0]); ya[1] = fmaf(f.z, ea, ya[1]); ya[2] = fmaf(f.w, ea, ya[2]);
    if constexpr (kTwo) {
      const float xb_ = ex2_approx(f.x * sb);
      const float eb = inb ? xb_ : 0.f;
      yb[0] = fmaf(f.y, eb, yb[0]); yb[1] = fmaf(f.z, eb, yb[1]); yb[2] = fmaf(f.w, eb, yb[2]);
    }
    if constexpr (kMask) {
      const uint32_t ma = __ballot_sync(0xffffffffu, ina), mb = kTwo ? __ballot_sync(0xffffffffu, inb) : 0u;
      if (lane == k) cm = make_uint2(ma, mb);
    }
  }
  __syncwarp();
}

// Two samples per lane (a = lane, b = lane + 32; inactive samples carry x' = NaN, never
// inside).  Accumulates yhat and, if kMask, candidate k's ballots into lane k's cm.
template <bool kMask, bool kTwo>
__device__ __forceinline__ void eval_chunk(const ChunkSmem& w, int kc, const float (&xa)[3], const float (&xb)[3],
                                           float tau2, float (&ya)[3], float (&yb)[3], uint2& cm, int lane) {
  if constexpr (kTwo) {            // packed fp32x2, bit-identical to cand_q per half (see eval_chunk_iso)
    const float2 X = make_float2(xa[0], xb[0]), Y = make_float2(xa[1], xb[1]), Z = make_float2(xa[2], xb[2]);
    float2 A0 = make_float2(ya[0], yb[0]), A1 = make_float2(ya[1], yb[1]), A2 = make_float2(ya[2], yb[2]);
#pragma unroll 2
    for (int k = 0; k < kc; ++k) {
      const Cand g = cand_from(w, k);
      const float2 w0 = __ffma2_rn(Z, make_float2(g.u02, g.u02), __ffma2_rn(Y, make_float2(g.u01, g.u01),
                                   __ffma2_rn(X, make_float2(g.u00, g.u00), make_float2(g.nc0, g.nc0))));
      const float2 w1 = __ffma2_rn(Z, make_float2(g.u12, g.u12), __ffma2_rn(Y, make_float2(g.u11, g.u11),
                                   make_float2(g.nc1, g.nc1)));
      const float2 w2 = __ffma2_rn(Z, make_float2(g.u22, g.u22), make_float2(g.nc2, g.nc2));
      const float2 Q = __ffma2_rn(w2, w2, __ffma2_rn(w1, w1, __fmul2_rn(w0, w0)));
      const bool ina = Q.x <= tau2, inb = Q.y <= tau2;
      const float2 t = __fmul2_rn(Q, make_float2(kNegHalfLog2e, kNegHalfLog2e));
      const float ea_ = ex2_approx(t.x), eb_ = ex2_approx(t.y);
      const float2 e = make_float2(ina ? ea_ : 0.f, inb ? eb_ : 0.f);
      A0 = __ffma2_rn(e, make_float2(g.v0, g.v0), A0);
      A1 = __ffma2_rn(e, make_float2(g.v1, g.v1), A1);
      A2 = __ffma2_rn(e, make_float2(g.v2, g.v2), A2);
      if constexpr (kMask) {
        const uint32_t ma = __ballot_sync(0xffffffffu, ina), mb = __ballot_sync(0xffffffffu, inb);
        if (lane == k) cm = make_uint2(ma, mb);
      }
    }
    ya[0] = A0.x; ya[1] = A1.x; ya[2] = A2.x;
    yb[0] = A0.y; yb[1] = A1.y; yb[2] = A2.y;
    __syncwarp();
    return;
  }
#pragma unroll 2
  for (int k = 0; k < kc; ++k) {
    const Cand g = cand_from(w, k);
    float w0, w1, w2;
    const float Qa = cand_q(g, xa[0], xa[1], xa[2], w0, w1, w2);
    const float Qb = kTwo ? cand_q(g, xb[0], xb[1], xb[2], w0, w1, w2) : 0.f;
    const bool ina = Qa <= tau2, inb = kTwo && Qb <= tau2;
    const float xa_ = ex2_approx(Qa * kNegHalfLog2e);
    const float ea = ina ? xa_ : 0.f;
    ya[0] = fmaf(g.v0, ea, ya[0]); ya[1] = fmaf(g.v1, ea, ya[1]); ya[2] = fmaf(g.v2, ea, ya[2]);
    if constexpr (kTwo) {
      const float xb_ = ex2_approx(Qb * kNegHalfLog2e);
      const float eb = inb ? xb_ : 0.f;
      yb[0] = fmaf(g.v0, eb, yb[0]); yb[1] = fmaf(g.v1, eb, yb[1]); yb[2] = fmaf(g.v2, eb, yb[2]);
    }
    if constexpr (kMask) {
      const uint32_t ma = __ballot_sync(0xffffffffu, ina), mb = kTwo ? __ballot_sync(0xffffffffu, inb) : 0u;
      if (lane == k) cm = make_uint2(ma, mb);
    }
  }
  __syncwarp();
}

// One chunk of pass 1 (kMask) or of a lookup: the isotropic or general evaluator, with
// both samples per lane only when the item has more than 32.
template <bool kMask>
__device__ __forceinline__ void eval_any(const ChunkSmem& w, bool iso, bool two, int kc, const float (&xa)[3],
                                         const float (&xb)[3], float tau2, float (&ya)[3], float (&yb)[3],
                                         uint2& cm, int lane) {
  if (iso) {
    if (two) eval_chunk_iso<kMask, true>(w, kc, xa, xb, ya, yb, cm, lane);
    else eval_chunk_iso<kMask, false>(w, kc, xa, xb, ya, yb, cm, lane);
  } else {
    if (two) eval_chunk<kMask, true>(w, kc, xa, xb, tau2, ya, yb, cm, lane);
    else eval_chunk<kMask, false>(w, kc, xa, xb, tau2, ya, yb, cm, lane);
  }
}

// Gradient terms of pairs [p0, p1) of the staged chunk: 12 coefficient gradients (C5).  The
// candidate-major pair list is cut into 32 contiguous slices, one per lane; a lane walks its
// slice accumulating the current Gaussian's terms in registers and issues
// red.global.add.v4.f32 whenever the Gaussian changes and at the end -- so every run of a
// Gaussian's pairs costs one reduction per lane piece, with no shuffles at all.
// kLite (isotropic chunk, scale group frozen with lr 0, no gradient export): the 6 dA terms
// only feed dL/ds, whose update is frozen, and dL/dq, which is exactly 0 for isotropic
// Gaussians -- so only d mu and d v are accumulated (dead work skipped, not approximated).
template <bool kLite>
__device__ __forceinline__ void flush_grad(float* __restrict__ grad, int gid, const float (&acc)[kLite ? 6 : 12]) {
  float* gp = grad + 12 * (int64_t)gid;
  if constexpr (kLite) {
    red_add_v4(gp, acc[0], acc[1], acc[2], 0.f);
    red_add_v4(gp + 8, 0.f, acc[3], acc[4], acc[5]);
  } else {
    red_add_v4(gp, acc[0], acc[1], acc[2], acc[3]);
    red_add_v4(gp + 4, acc[4], acc[5], acc[6], acc[7]);
    red_add_v4(gp + 8, acc[8], acc[9], acc[10], acc[11]);
  }
}

template <bool kLite>
__device__ __forceinline__ void chunk_pairs_bwd_impl(const WarpSmem& w, int p0, int p1, float* __restrict__ grad,
                                                     int lane, bool iso) {
  constexpr int NV = kLite ? 6 : 12;
  const int n = p1 - p0;
  const int pa = p0 + ((n * lane) >> 5), pe_ = p0 + ((n * (lane + 1)) >> 5);
  float acc[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.f;
  int kcur = -1, gid = 0;
  float4 mu = make_float4(0.f, 0.f, 0.f, 0.f);
  float u2 = 0.f, v0 = 0.f, v1 = 0.f, v2 = 0.f;
  Cand g{};
  for (int p = pa; p < pe_; ++p) {
    const uint32_t key = w.u.list.pkey[p];
    const float e = w.u.list.pe[p];
    const int k = key >> 6, s = key & 63;
    if (k != kcur) {
      if (kcur >= 0) {
        flush_grad<kLite>(grad, gid, acc);
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] = 0.f;
      }
      kcur = k;
      mu = w.r3[k];
      gid = __float_as_int(mu.w);
      if (iso) {
        const float4 f = w.r1[k];
        u2 = w.r2[k].x; v0 = f.y; v1 = f.z; v2 = f.w;
      } else {
        g = cand_from(w, k);
        v0 = g.v0; v1 = g.v1; v2 = g.v2;
      }
    }
    const float4 sx = w.sxg[s];
    const float2 sg = w.sg[s];
    const float dx = sx.x - mu.x, dy = sx.y - mu.y, dz = sx.z - mu.z;
    float tx, ty, tz;
    if (iso) {                                                     // t = A d = u^2 d
      tx = u2 * dx; ty = u2 * dy; tz = u2 * dz;
    } else {                                                       // t = A d = U^T w
      float w0, w1, w2;
      cand_q(g, sx.x, sx.y, sx.z, w0, w1, w2);
      tx = g.u00 * w0;
      ty = fmaf(g.u11, w1, g.u01 * w0);
      tz = fmaf(g.u22, w2, fmaf(g.u12, w1, g.u02 * w0));
    }
    const float he = (sx.w * v0 + sg.x * v1 + sg.y * v2) * e;
    acc[0] = fmaf(he, tx, acc[0]); acc[1] = fmaf(he, ty, acc[1]); acc[2] = fmaf(he, tz, acc[2]);   // d mu
    if constexpr (kLite) {
      acc[3] = fmaf(sx.w, e, acc[3]); acc[4] = fmaf(sg.x, e, acc[4]); acc[5] = fmaf(sg.y, e, acc[5]);   // d v
    } else {
      const float kk = -0.5f * he;
      const float kx = kk * dx, ky = kk * dy, kz = kk * dz;
      acc[3] = fmaf(kx, dx, acc[3]); acc[4] = fmaf(ky, dy, acc[4]); acc[5] = fmaf(kz, dz, acc[5]);   // dA00 dA11 dA22
      acc[6] = fmaf(kx, dy, acc[6]); acc[7] = fmaf(kx, dz, acc[7]); acc[8] = fmaf(ky, dz, acc[8]);   // dA01 dA02 dA12
      acc[9] = fmaf(sx.w, e, acc[9]); acc[10] = fmaf(sg.x, e, acc[10]); acc[11] = fmaf(sg.y, e, acc[11]);   // d v
    }
  }
  if (kcur >= 0) flush_grad<kLite>(grad, gid, acc);
  __syncwarp();
}

__device__ __forceinline__ void chunk_pairs_bwd(const WarpSmem& w, int p0, int p1, float* __restrict__ grad,
                                                int lane, bool iso, bool lite_ok) {
  if (iso && lite_ok) chunk_pairs_bwd_impl<true>(w, p0, p1, grad, lane, true);
  else chunk_pairs_bwd_impl<false>(w, p0, p1, grad, lane, iso);
}

// Position of the set bit of rank r (0-based) in x (binary search on popcounts).
__device__ __forceinline__ int select_bit(uint32_t x, int r) {
  int pos = 0;
#pragma unroll
  for (int wd = 16; wd; wd >>= 1) {
    const int c = __popc(x & ((1u << wd) - 1u));
    if (c <= r) { r -= c; x >>= wd; pos += wd; }
  }
  return pos;
}

// End of a Gaussian's run in pass 2: acc[0..2] holds sum h e d (isotropic) or sum h e w
// (general); d mu = u^2 * that, or U^T * that (t = A d = U^T U d = U^T w).
template <int NV>
__device__ __forceinline__ void run_to_dmu(bool iso, float u2, const Cand& g, float (&acc)[NV]) {
  if (iso) {
    acc[0] *= u2; acc[1] *= u2; acc[2] *= u2;
  } else {
    const float a0 = acc[0], a1 = acc[1], a2 = acc[2];
    acc[0] = g.u00 * a0;
    acc[1] = fmaf(g.u11, a1, g.u01 * a0);
    acc[2] = fmaf(g.u22, a2, fmaf(g.u12, a1, g.u02 * a0));
  }
}

// Backward of one staged chunk from pass 1's inside masks: the chunk's pairs in candidate-major
// order (candidate k's samples a then b, ascending) are cut into 32 contiguous slices, one per
// lane; a lane finds its first pair by a binary search over the candidates' pair offsets and a
// select on the mask, then walks on bit by bit, recomputing e = exp(-Q/2) exactly as pass 1
// did, accumulating the current Gaussian's coefficient gradients in registers and issuing
// red.global.add.v4.f32 whenever the Gaussian changes and at the end.
template <bool kLite, bool kWide>
__device__ __forceinline__ void chunk_bwd_masks_impl(const WarpSmem& w, const uint2* __restrict__ mask, int P,
                                                     uint32_t nz, float tau2, float* __restrict__ grad, int lane,
                                                     bool iso) {
  constexpr int NV = kLite ? 6 : 12;
  const int pa = (P * lane) >> 5, pend = (P * (lane + 1)) >> 5;
  if (pa >= pend) return;
  int k = 0;
#pragma unroll
  for (int st = 16; st; st >>= 1)
    if (w.offs[k + st] <= pa) k += st;
  // items of <= 32 samples (kWide false) have empty high mask words: 32-bit bit walk
  using M = typename std::conditional<kWide, uint64_t, uint32_t>::type;
  uint2 mk = mask[k];
  M m = kWide ? (M)(((uint64_t)mk.y << 32) | mk.x) : (M)mk.x;
  {                                            // drop the candidate's first (pa - offs[k]) pairs
    const int r = pa - w.offs[k], pl = __popc(mk.x);
    if (!kWide || r < pl) m &= ~(M)((1u << select_bit(mk.x, r)) - 1u);
    else m = (M)((uint64_t)(mk.y & ~((1u << select_bit(mk.y, r - pl)) - 1u)) << 32);
  }
  float acc[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.f;
  int kcur = -1, gid = 0;
  float4 mu = make_float4(0.f, 0.f, 0.f, 0.f);
  float u2 = 0.f, gx = 0.f, v0 = 0.f, v1 = 0.f, v2 = 0.f;
  Cand g{};
  for (int p = pa; p < pend; ++p) {
    if (m == 0) {                              // next candidate with pairs (nz: non-empty masks)
      k = __ffs(nz & (0xFFFFFFFEu << k)) - 1;
      if constexpr (kWide) { mk = mask[k]; m = ((uint64_t)mk.y << 32) | mk.x; }
      else m = mask[k].x;
    }
    const int s = kWide ? __ffsll((long long)m) - 1 : __ffs((int)m) - 1;
    m &= m - 1;
    if (k != kcur) {
      if (kcur >= 0) {
        run_to_dmu(iso, u2, g, acc);
        flush_grad<kLite>(grad, gid, acc);
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] = 0.f;
      }
      kcur = k;
      mu = w.r3[k];
      gid = __float_as_int(mu.w);
      if (iso) {
        const float4 f = w.r1[k];
        u2 = w.r2[k].x; gx = f.x; v0 = f.y; v1 = f.z; v2 = f.w;
      } else {
        g = cand_from(w, k);
        v0 = g.v0; v1 = g.v1; v2 = g.v2;
      }
    }
    const float4 sx = w.sxg[s];
    const float2 sg = w.sg[s];
    // d = x' - mu (r3 and r0 hold the same recentred mu, so this is also iso_s's difference)
    const float dx = __fsub_rn(sx.x, mu.x), dy = __fsub_rn(sx.y, mu.y), dz = __fsub_rn(sx.z, mu.z);
    // d mu = sum_p h_p e_p A d_p = A sum_p h_p e_p d_p over the run (A fixed per Gaussian):
    // the run accumulates h e d (isotropic, A = u^2 I) or h e w (general, A d = U^T w) and
    // run_to_dmu applies u^2 or U^T once per run instead of per pair
    float tx, ty, tz, e;
    if (iso) {                                                     // same arithmetic as pass 1
      e = ex2_approx(gx * __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx))));
      tx = dx; ty = dy; tz = dz;
    } else {
      e = ex2_approx(cand_q(g, sx.x, sx.y, sx.z, tx, ty, tz) * kNegHalfLog2e);
    }
    const float he = (sx.w * v0 + sg.x * v1 + sg.y * v2) * e;
    acc[0] = fmaf(he, tx, acc[0]); acc[1] = fmaf(he, ty, acc[1]); acc[2] = fmaf(he, tz, acc[2]);   // d mu
    if constexpr (kLite) {
      acc[3] = fmaf(sx.w, e, acc[3]); acc[4] = fmaf(sg.x, e, acc[4]); acc[5] = fmaf(sg.y, e, acc[5]);   // d v
    } else {
      const float kk = -0.5f * he;
      const float kx = kk * dx, ky = kk * dy, kz = kk * dz;
      acc[3] = fmaf(kx, dx, acc[3]); acc[4] = fmaf(ky, dy, acc[4]); acc[5] = fmaf(kz, dz, acc[5]);   // dA00 dA11 dA22
      acc[6] = fmaf(kx, dy, acc[6]); acc[7] = fmaf(kx, dz, acc[7]); acc[8] = fmaf(ky, dz, acc[8]);   // dA01 dA02 dA12
      acc[9] = fmaf(sx.w, e, acc[9]); acc[10] = fmaf(sg.x, e, acc[10]); acc[11] = fmaf(sg.y, e, acc[11]);   // d v
    }
  }
  run_to_dmu(iso, u2, g, acc);
  flush_grad<kLite>(grad, gid, acc);
}

__device__ __forceinline__ void load_pos(const float4* __restrict__ bin, int stride, int start, int count, int s,
                                         float (&x)[3], float4& p) {
  if (s < count) {
    p = __ldcs(bin + stride * (int64_t)(start + s));
    x[0] = p.x; x[1] = p.y; x[2] = p.z;
  } else {
    x[0] = x[1] = x[2] = __int_as_float(0x7fffffff);     // NaN: never inside
    p = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// n / d for n >= 0, d >= 1 (n < 2^22): a float quotient estimate (off by at most one) corrected
// exactly -- a few instructions instead of the integer division routine.
__device__ __forceinline__ int div_small(int n, int d, float inv_d) {
  if (n >= (1 << 22)) return n / d;              // (estimate error could exceed one)
  int q = __float2int_rz(__int2float_rn(n) * inv_d);
  const int r = n - q * d;
  q += (r >= d) - (r < 0);
  return q;
}

// Centre of a work item's cell (fp32; any point of the cell would do as long as every pass
// of the item uses the same one).
__device__ __forceinline__ void cell_centre(const CellRef& r, int cell, int l, float& x, float& y, float& z) {
  const int loc = cell - r.coff[l], dx = r.dx[l], dy = r.dy[l];
  const int t = div_small(loc, dx, r.idx[l]), cz = div_small(t, dy, r.idy[l]);
  const int cx = loc - t * dx, cy = t - cz * dy;
  x = fmaf((float)cx + 0.5f, r.edge[l][0], r.org[l][0]);
  y = fmaf((float)cy + 0.5f, r.edge[l][1], r.org[l][1]);
  z = fmaf((float)cz + 0.5f, r.edge[l][2], r.org[l][2]);
}

__device__ __forceinline__ void hdr_grad(int mode, float eps, const float (&y)[3], const float (&t)[3],
                                         float (&g)[3], float& ls) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    // d >= eps > 0: the MUFU reciprocal (~1 ulp) instead of an IEEE division (its slow path
    // and branches); the loss and g stay within ~1e-7 relative of the exact quotient
    const float d = y[c] + eps, r = t[c] - y[c], i = __fdividef(1.f, d * d);
    ls += r * r * i;
    g[c] = mode == 0 ? -2.f * r * i : __fdividef(-2.f * r * (t[c] + eps) * i, d);
  }
}

// Output of one query in caller order, with the optional renderer epilogue (f3): natural
// termination keeps a non-zero unbiased radiance; otherwise Eq. 3,
// yhat * attenuation / beta.
__device__ __forceinline__ void query_out(float* out, const float* att, const float* beta, const float* unb,
                                          int64_t i, const float (&y)[3]) {
  float o0 = y[0], o1 = y[1], o2 = y[2];
  if (att) { o0 *= att[3 * i]; o1 *= att[3 * i + 1]; o2 *= att[3 * i + 2]; }
  if (beta) { const float ib = 1.f / beta[i]; o0 *= ib; o1 *= ib; o2 *= ib; }
  if (unb) {
    const float u0 = unb[3 * i], u1 = unb[3 * i + 1], u2 = unb[3 * i + 2];
    if (u0 != 0.f || u1 != 0.f || u2 != 0.f) { o0 = u0; o1 = u1; o2 = u2; }
  }
  __stcs(out + 3 * i, o0); __stcs(out + 3 * i + 1, o1); __stcs(out + 3 * i + 2, o2);
}

__global__ void __launch_bounds__(256, 4) k_fwdbwd(FitArgs a) {
  pdl_enter();
  // the culling lists are reached through DevState, so a CUDA graph captured before a capacity
  // growth (csr_guard) reads the current lists
  const float4* __restrict__ lrec = a.st->lrec;
  const uint32_t lcap = a.st->lcap;
  extern __shared__ __align__(16) unsigned char dsm[];
  WarpSmem* sm = reinterpret_cast<WarpSmem*>(dsm);
  __shared__ double s_loss[kWarps][kMaxL];
  __shared__ unsigned long long s_cnt[kWarps][2];
  __shared__ uint32_t s_nfit[kWarps][kMaxL];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSmem& w = sm[wid];
  if (lane < kMaxL) { s_loss[wid][lane] = 0.0; s_nfit[wid][lane] = 0u; }
  unsigned long long pairs_acc = 0, cand_acc = 0;
  const uint32_t n_work = a.n_work[0];
  uint32_t* next = const_cast<uint32_t*>(a.n_work) + 1;   // dynamic work counter (zeroed by the scan)
  const float tau2 = a.tau2, eps = a.hdr_eps;

  uint32_t claim = 0, left = 0;          // items are claimed kClaimFit at a time (fewer contended atomics)
  for (;;) {
    if (left == 0) {
      uint32_t c0 = 0;
      if (lane == 0) c0 = atomicAdd(next, kClaimFit);
      claim = __shfl_sync(0xffffffffu, c0, 0);
      left = kClaimFit;
    }
    const uint32_t it = claim++;
    --left;
    if (it >= n_work) break;
    const WorkItem wi = a.work[it];
    GSC_CHECK(wi.start >= 0 && wi.count >= 1 && wi.count <= kCH && (int64_t)wi.start + wi.count <= a.bin_cap &&
              wi.level >= 0 && wi.level < a.L && wi.cell >= 0, "fit work item");
    // clamped to the list capacity: after an overflowing rebuild the offsets run past it (the
    // entries there were dropped; the call reports GC_FLAG_LISTS_OVERFLOWED and skips its step)
    const int lo = (int)min(__ldg(a.csr_off + wi.cell), lcap);
    const int C = (int)min(__ldg(a.csr_off + wi.cell + 1), lcap) - lo;
    float xa[3], xb[3], ta[3] = {0.f, 0.f, 0.f}, tb[3] = {0.f, 0.f, 0.f};
    {                                            // one 32-byte load per sample: x y z r | g b - -
      const float kNaN = __int_as_float(0x7fffffff);   // inactive samples: never inside
      xa[0] = xa[1] = xa[2] = xb[0] = xb[1] = xb[2] = kNaN;
      float4 p, q;
      if (lane < wi.count) {
        ld_v8_nc(a.bin + 2 * (int64_t)(wi.start + lane), p, q);
        xa[0] = p.x; xa[1] = p.y; xa[2] = p.z; ta[0] = p.w; ta[1] = q.x; ta[2] = q.y;
      }
      if (lane + 32 < wi.count) {
        ld_v8_nc(a.bin + 2 * (int64_t)(wi.start + lane + 32), p, q);
        xb[0] = p.x; xb[1] = p.y; xb[2] = p.z; tb[0] = p.w; tb[1] = q.x; tb[2] = q.y;
      }
    }
    float xref, yref, zref;                                 // the cell's centre (CellRef)
    cell_centre(a.ref, wi.cell, wi.level, xref, yref, zref);
    xa[0] -= xref; xa[1] -= yref; xa[2] -= zref;            // NaN stays NaN
    xb[0] -= xref; xb[1] -= yref; xb[2] -= zref;
    // ---------------- pass 1 (keeps each candidate's inside masks while they fit)
    float ya[3] = {0.f, 0.f, 0.f}, yb[3] = {0.f, 0.f, 0.f};
    int np = 0;
    bool iso = false;
    const bool masked = C <= 32 * kMaskChunks;
    for (int cb = 0, c = 0; cb < C; cb += 32, ++c) {
      const int kc = min(32, C - cb);
      iso = stage_chunk(w, lrec, lo + cb, kc, lane, xref, yref, zref, tau2, a.G);
      uint2 cm = make_uint2(0u, 0u);
      eval_any<true>(w, iso, wi.count > 32, kc, xa, xb, tau2, ya, yb, cm, lane);
      if (masked) w.u.mask[c][lane] = cm;
      np += (int)__reduce_add_sync(0xffffffffu, (unsigned)(__popc(cm.x) + __popc(cm.y)));
    }
    // ---------------- Eq. 4 loss and dL/dyhat (unnormalised)
    float ga[3] = {0.f, 0.f, 0.f}, gb[3] = {0.f, 0.f, 0.f}, ls = 0.f;
    if (lane < wi.count) hdr_grad(a.mode, eps, ya, ta, ga, ls);
    if (lane + 32 < wi.count) hdr_grad(a.mode, eps, yb, tb, gb, ls);
    w.sxg[lane] = make_float4(xa[0], xa[1], xa[2], ga[0]);
    w.sg[lane] = make_float2(ga[1], ga[2]);
    w.sxg[lane + 32] = make_float4(xb[0], xb[1], xb[2], gb[0]);
    w.sg[lane + 32] = make_float2(gb[1], gb[2]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
    if (lane == 0) { s_loss[wid][wi.level] += (double)ls; s_nfit[wid][wi.level] += (uint32_t)wi.count; }
    pairs_acc += (unsigned)np;
    cand_acc += (unsigned long long)wi.count * (unsigned long long)C;
    __syncwarp();
    if (np == 0) continue;
    // ---------------- pass 2
    if (masked) {
      // last chunk first: pass 1 left it staged, so only the earlier chunks are re-staged
      const int nch = (C + 31) >> 5;
      for (int c = nch - 1; c >= 0; --c) {
        const int cb = 32 * c;
        const uint2 mk = w.u.mask[c][lane];
        const int nk = __popc(mk.x) + __popc(mk.y);
        const uint32_t nz = __ballot_sync(0xffffffffu, nk > 0);
        int incl = nk;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const int P = __shfl_sync(0xffffffffu, incl, 31);
        if (P == 0) continue;
        if (c != nch - 1) iso = stage_chunk(w, lrec, lo + cb, 32, lane, xref, yref, zref, tau2, a.G);
        w.offs[lane] = incl - nk;
        __syncwarp();
        if (wi.count > 32) {
          if (iso && a.lite) chunk_bwd_masks_impl<true, true>(w, w.u.mask[c], P, nz, tau2, a.grad, lane, true);
          else chunk_bwd_masks_impl<false, true>(w, w.u.mask[c], P, nz, tau2, a.grad, lane, iso);
        } else {
          if (iso && a.lite) chunk_bwd_masks_impl<true, false>(w, w.u.mask[c], P, nz, tau2, a.grad, lane, true);
          else chunk_bwd_masks_impl<false, false>(w, w.u.mask[c], P, nz, tau2, a.grad, lane, iso);
        }
        __syncwarp();
      }
    } else {
      // rare dense case: re-derive each chunk's pairs exactly as pass 1 did, in batches
      const uint32_t lt = (1u << lane) - 1u;
      for (int cb = 0; cb < C; cb += 32) {
        const int kc = min(32, C - cb);
        const bool ci = stage_chunk(w, lrec, lo + cb, kc, lane, xref, yref, zref, tau2, a.G);
        int pb = 0;
        for (int k = 0; k < kc; ++k) {
          float Qa, Qb, ea, eb;                    // same arithmetic as eval_chunk[_iso]
          bool ina, inb;
          if (ci) {
            const float4 cc = w.r0[k], f = w.r1[k];
            Qa = iso_s(xa, cc); Qb = iso_s(xb, cc);
            ina = Qa <= cc.w; inb = Qb <= cc.w;
            ea = ex2_approx(f.x * Qa); eb = ex2_approx(f.x * Qb);
          } else {
            const Cand g = cand_from(w, k);
            float w0, w1, w2;
            Qa = cand_q(g, xa[0], xa[1], xa[2], w0, w1, w2);
            Qb = cand_q(g, xb[0], xb[1], xb[2], w0, w1, w2);
            ina = Qa <= tau2; inb = Qb <= tau2;
            ea = ex2_approx(Qa * kNegHalfLog2e); eb = ex2_approx(Qb * kNegHalfLog2e);
          }
          const uint32_t ma = __ballot_sync(0xffffffffu, ina), mb = __ballot_sync(0xffffffffu, inb);
          if (!(ma | mb)) continue;
          if (pb + 64 > kPairCap) { chunk_pairs_bwd(w, 0, pb, a.grad, lane, ci, a.lite); pb = 0; }
          if (ina) {
            const int pos = pb + __popc(ma & lt);
            w.u.list.pkey[pos] = (uint16_t)((k << 6) | lane);
            w.u.list.pe[pos] = ea;
          }
          if (inb) {
            const int pos = pb + __popc(ma) + __popc(mb & lt);
            w.u.list.pkey[pos] = (uint16_t)((k << 6) | (lane + 32));
            w.u.list.pe[pos] = eb;
          }
          pb += __popc(ma) + __popc(mb);
          __syncwarp();
        }
        chunk_pairs_bwd(w, 0, pb, a.grad, lane, ci, a.lite);
      }
    }
  }
  if (lane == 0) { s_cnt[wid][0] = pairs_acc; s_cnt[wid][1] = cand_acc; }
  __syncthreads();
  // per-CTA partials go into kSlots slotted fp64 accumulators (slot = CTA mod kSlots: a few
  // dozen same-address reductions each), read and re-zeroed by k_stats
  double* part = a.partial + (int64_t)(blockIdx.x % kSlots) * kPart;
  if (threadIdx.x < kMaxL) {
    double s = 0.0;
    unsigned long long n = 0;
    for (int q = 0; q < kWarps; ++q) { s += s_loss[q][threadIdx.x]; n += s_nfit[q][threadIdx.x]; }
    if (s != 0.0) atomicAdd(part + threadIdx.x, s);
    if (n) atomicAdd(part + kMaxL + threadIdx.x, (double)n);
  }
  if (threadIdx.x == 0) {
    unsigned long long p = 0, c = 0;
    for (int q = 0; q < kWarps; ++q) { p += s_cnt[q][0]; c += s_cnt[q][1]; }
    if (p) atomicAdd(part + 2 * kMaxL, (double)p);
    if (c) atomicAdd(part + 2 * kMaxL + 1, (double)c);
  }
}

__global__ void __launch_bounds__(256, 4) k_query(QueryArgs a) {
  pdl_enter();
  const float4* __restrict__ lrec = a.st->lrec;
  const uint32_t lcap = a.st->lcap;
  __shared__ ChunkSmem sm[kWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  ChunkSmem& w = sm[wid];
  const uint32_t n_work = a.n_work[0];
  uint32_t* next = const_cast<uint32_t*>(a.n_work) + 1;   // dynamic work counter (zeroed by the scan)
  const float tau2 = a.tau2;
  uint32_t claim = 0, left = 0;          // items are claimed kClaimQuery at a time (fewer contended atomics)
  for (;;) {
    if (left == 0) {
      uint32_t c0 = 0;
      if (lane == 0) c0 = atomicAdd(next, kClaimQuery);
      claim = __shfl_sync(0xffffffffu, c0, 0);
      left = kClaimQuery;
    }
    const uint32_t it = claim++;
    --left;
    if (it >= n_work) break;
    const WorkItem wi = a.work[it];
    GSC_CHECK(wi.start >= 0 && wi.count >= 1 && wi.count <= kCH && (int64_t)wi.start + wi.count <= a.bin_cap &&
              wi.cell >= 0, "lookup work item");
    // clamped to the list capacity: after an overflowing rebuild the offsets run past it (the
    // entries there were dropped; the call reports GC_FLAG_LISTS_OVERFLOWED and skips its step)
    const int lo = (int)min(__ldg(a.csr_off + wi.cell), lcap);
    const int C = (int)min(__ldg(a.csr_off + wi.cell + 1), lcap) - lo;
    float xa[3], xb[3];
    float4 pa, pb4;
    load_pos(a.bin, 2, wi.start, wi.count, lane, xa, pa);
    load_pos(a.bin, 2, wi.start, wi.count, lane + 32, xb, pb4);
    float xref, yref, zref;
    cell_centre(a.ref, wi.cell, wi.level, xref, yref, zref);
    xa[0] -= xref; xa[1] -= yref; xa[2] -= zref;
    xb[0] -= xref; xb[1] -= yref; xb[2] -= zref;
    float ya[3] = {0.f, 0.f, 0.f}, yb[3] = {0.f, 0.f, 0.f};
    for (int cb = 0; cb < C; cb += 32) {
      const int kc = min(32, C - cb);
      const bool iso = stage_chunk(w, lrec, lo + cb, kc, lane, xref, yref, zref, tau2, a.G);
      uint2 cm;
      eval_any<false>(w, iso, wi.count > 32, kc, xa, xb, tau2, ya, yb, cm, lane);
    }
    GSC_CHECK(lane >= wi.count || __float_as_uint(pa.w) < (uint64_t)a.S, "lookup output index");
    GSC_CHECK(lane + 32 >= wi.count || __float_as_uint(pb4.w) < (uint64_t)a.S, "lookup output index");
    if (lane < wi.count) query_out(a.out, a.att, a.beta, a.unb, __float_as_uint(pa.w), ya);
    if (lane + 32 < wi.count) query_out(a.out, a.att, a.beta, a.unb, __float_as_uint(pb4.w), yb);
  }
}

CellRef cell_ref(const LevelGeom& g) {
  CellRef r{};
  for (int l = 0; l < g.L; ++l) {
    for (int a = 0; a < 3; ++a) { r.org[l][a] = (float)g.origin[l][a]; r.edge[l][a] = (float)g.edge[l][a]; }
    r.dx[l] = g.dims[l][0]; r.dy[l] = g.dims[l][1]; r.coff[l] = (int)g.coff[l];
    r.idx[l] = 1.f / (float)r.dx[l]; r.idy[l] = 1.f / (float)r.dy[l];
  }
  return r;
}

constexpr size_t kFwdBwdSmem = sizeof(WarpSmem) * kWarps;

static int persistent_grid(const void* fn, size_t smem) {
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 256, smem);
  return sms * std::max(per, 1);
}

// Both are per device: called by gc_create after cudaSetDevice (the dynamic shared-memory
// attribute is a property of the current device's context; a handle on another device sets
// its own).  Returns 0 on failure.
int fwdbwd_grid() {
  if (cudaFuncSetAttribute(k_fwdbwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFwdBwdSmem) != cudaSuccess)
    return 0;
  return persistent_grid((const void*)k_fwdbwd, kFwdBwdSmem);
}
int query_grid() { return persistent_grid((const void*)k_query, 0); }

void launch_fwdbwd(const FitArgs& a, int grid, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, "fwdbwd", s);
  launch_pdl(k_fwdbwd, dim3(grid), dim3(256), kFwdBwdSmem, s, a);
}

void launch_query(const QueryArgs& a, int grid, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, "query_fwd", s);
  launch_pdl(k_query, dim3(grid), dim3(256), 0, s, a);
}

}  // namespace gsc
