// record.cuh -- evaluation record (A2) and exact conservative cell range (C8) of one
// Gaussian; shared by the create/set_params path and the fused optimizer epilogue.
#pragma once
#include "common.cuh"

namespace gsc {

// Upper bounds of 2^(r/32): the smallest doubles >= 2^(r/32) (C8; hex literals of the spec).
static __device__ const double kT32[32] = {
    0x1.0000000000000p+0, 0x1.059b0d3158575p+0, 0x1.0b5586cf98910p+0, 0x1.11301d0125b51p+0,
    0x1.172b83c7d517bp+0, 0x1.1d4873168b9abp+0, 0x1.2387a6e756239p+0, 0x1.29e9df51fdee2p+0,
    0x1.306fe0a31b716p+0, 0x1.371a7373aa9cbp+0, 0x1.3dea64c123423p+0, 0x1.44e086061892ep+0,
    0x1.4bfdad5362a28p+0, 0x1.5342b569d4f82p+0, 0x1.5ab07dd48542ap+0, 0x1.6247eb03a5585p+0,
    0x1.6a09e667f3bcdp+0, 0x1.71f75e8ec5f74p+0, 0x1.7a11473eb0187p+0, 0x1.82589994cce13p+0,
    0x1.8ace5422aa0dcp+0, 0x1.93737b0cdc5e5p+0, 0x1.9c49182a3f091p+0, 0x1.a5503b23e255dp+0,
    0x1.ae89f995ad3aep+0, 0x1.b7f76f2fb5e47p+0, 0x1.c199bdd85529dp+0, 0x1.cb720dcef906ap+0,
    0x1.d5818dcfba488p+0, 0x1.dfc97337b9b5fp+0, 0x1.ea4afa2a490dap+0, 0x1.f50765b6e4541p+0};
constexpr double kK32 = 0x1.71547652b82fep+5;   // 32 log2(e)

// Record of one Gaussian from its raw parameters (C1): A = R diag(e^-2s) R^T is formed and
// Cholesky-factored in fp64 (A = U^T U), stored in fp32 with mu and v = w max(0, c).
__device__ __forceinline__ void make_record(const float p[kNP], float4 out[3]) {
  const float wo = 1.f / (1.f + expf(-p[P_O]));
  out[2] = make_float4(p[P_MU + 2], wo * fmaxf(p[P_C], 0.f), wo * fmaxf(p[P_C + 1], 0.f), wo * fmaxf(p[P_C + 2], 0.f));
  if (p[P_S] == p[P_S + 1] && p[P_S + 1] == p[P_S + 2]) {
    // isotropic: A = e^{-2s} R R^T = e^{-2s} I exactly, U = e^{-s} I (the rotation drops out);
    // with the paper's scale LR of 0 and isotropic Eq. 2 init every Gaussian stays here
    const float u = expf(-p[P_S]);
    out[0] = make_float4(u, 0.f, 0.f, u);
    out[1] = make_float4(0.f, u, p[P_MU], p[P_MU + 1]);
    return;
  }
  double w = p[P_Q], x = p[P_Q + 1], y = p[P_Q + 2], z = p[P_Q + 3];
  const double n2 = w * w + x * x + y * y + z * z;
  if (n2 < 1e-24) { w = 1.0; x = y = z = 0.0; }
  else { const double n = sqrt(n2); w /= n; x /= n; y /= n; z /= n; }
  double R[3][3];
  R[0][0] = 1.0 - 2.0 * (y * y + z * z); R[0][1] = 2.0 * (x * y - w * z); R[0][2] = 2.0 * (x * z + w * y);
  R[1][0] = 2.0 * (x * y + w * z); R[1][1] = 1.0 - 2.0 * (x * x + z * z); R[1][2] = 2.0 * (y * z - w * x);
  R[2][0] = 2.0 * (x * z - w * y); R[2][1] = 2.0 * (y * z + w * x); R[2][2] = 1.0 - 2.0 * (x * x + y * y);
  const double D0 = expf(-2.f * p[P_S]), D1 = expf(-2.f * p[P_S + 1]), D2 = expf(-2.f * p[P_S + 2]);
  double A[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b) A[a][b] = R[a][0] * R[b][0] * D0 + R[a][1] * R[b][1] * D1 + R[a][2] * R[b][2] * D2;
  const double U00 = sqrt(A[0][0]);
  const double U01 = A[0][1] / U00, U02 = A[0][2] / U00;
  const double U11 = sqrt(fmax(A[1][1] - U01 * U01, 1e-300));
  const double U12 = (A[1][2] - U01 * U02) / U11;
  const double U22 = sqrt(fmax(A[2][2] - U02 * U02 - U12 * U12, 1e-300));
  out[0] = make_float4((float)U00, (float)U01, (float)U02, (float)U11);
  out[1] = make_float4((float)U12, (float)U22, p[P_MU], p[P_MU + 1]);
}

// C8 cell range of one Gaussian (AABB of its tau-ellipsoid, bounded with U_b >= e^{s_b}) and
// r2 = tau^2 max_b U_b^2; fp64 with explicitly rounded + - * / sqrt only (no FMA, no exp), in
// the order the oracle writes them, so both produce the same integers.
__device__ __forceinline__ void cull_range(const float p[kNP], double tau, const LevelGeom& g, int l,
                                           int32_t lo[3], int32_t hi[3], double& r2) {
  double U1[3], U2[3];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    double sk = __dmul_rn((double)p[P_S + b], kK32);
    if (!(sk >= -32000.0)) sk = (sk != sk) ? 32000.0 : -32000.0;
    if (sk > 32000.0) sk = 32000.0;
    int32_t k = (int32_t)ceil(sk) + 1;
    int32_t Qe = (k >= 0) ? k / 32 : -((-k + 31) / 32);
    U1[b] = ldexp(kT32[k - 32 * Qe], Qe);
    U2[b] = __dmul_rn(U1[b], U1[b]);
  }
  double h[3];
  if (p[P_S] == p[P_S + 1] && p[P_S + 1] == p[P_S + 2]) {
    // isotropic: a ball of radius tau e^s <= tau U (R R^T = I), no rotation needed
    h[0] = h[1] = h[2] = __dmul_rn(tau, U1[0]);
  } else {
    double w = p[P_Q], x = p[P_Q + 1], y = p[P_Q + 2], z = p[P_Q + 3];
    double n2 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(w, w), __dmul_rn(x, x)), __dmul_rn(y, y)), __dmul_rn(z, z));
    if (n2 < 1e-24) { w = 1.0; x = 0.0; y = 0.0; z = 0.0; }
    else {
      double n = __dsqrt_rn(n2);
      w = __ddiv_rn(w, n); x = __ddiv_rn(x, n); y = __ddiv_rn(y, n); z = __ddiv_rn(z, n);
    }
    double R[3][3];
    R[0][0] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(y, y), __dmul_rn(z, z))));
    R[0][1] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(x, y), __dmul_rn(w, z)));
    R[0][2] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, z), __dmul_rn(w, y)));
    R[1][0] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, y), __dmul_rn(w, z)));
    R[1][1] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, x), __dmul_rn(z, z))));
    R[1][2] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(y, z), __dmul_rn(w, x)));
    R[2][0] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(x, z), __dmul_rn(w, y)));
    R[2][1] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(y, z), __dmul_rn(w, x)));
    R[2][2] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y))));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double s0 = __dmul_rn(__dmul_rn(R[a][0], R[a][0]), U2[0]);
      double s1 = __dmul_rn(__dmul_rn(R[a][1], R[a][1]), U2[1]);
      double s2 = __dmul_rn(__dmul_rn(R[a][2], R[a][2]), U2[2]);
      h[a] = __dmul_rn(tau, __dsqrt_rn(__dadd_rn(__dadd_rn(s0, s1), s2)));
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double mu = (double)p[P_MU + a];
    lo[a] = clampcell(floor(__dmul_rn(__dsub_rn(__dsub_rn(mu, h[a]), g.origin[l][a]), g.inv_cell[l][a])), g.dims[l][a]);
    hi[a] = clampcell(floor(__dmul_rn(__dsub_rn(__dadd_rn(mu, h[a]), g.origin[l][a]), g.inv_cell[l][a])), g.dims[l][a]);
  }
  double um = U2[0];
  if (U2[1] > um) um = U2[1];
  if (U2[2] > um) um = U2[2];
  r2 = __dmul_rn(__dmul_rn(tau, tau), um);
}

// Cell membership (C8): squared distance from mu to the cell's box <= r2; border cells reach
// to infinity outwards (A17).  The oracle's orc_cell_hit computes, per axis,
// d_a = dist(mu_a, [o_a + c_a e_a, o_a + (c_a+1) e_a]), e_a = 1/inv_a, D2 = (d_x^2 + d_y^2) + d_z^2;
// the same per-axis terms are tabulated here once per Gaussian (bit-identical doubles).
__device__ __forceinline__ double axis_d2(double mu, int32_t c, const LevelGeom& g, int l, int a) {
  const double e = g.edge[l][a];                          // 1.0 / inv_cell (same rounding as the oracle)
  const double lo = c == 0 ? -INFINITY : __dadd_rn(g.origin[l][a], __dmul_rn((double)c, e));
  const double hi = c == g.dims[l][a] - 1 ? INFINITY : __dadd_rn(g.origin[l][a], __dmul_rn((double)(c + 1), e));
  const double d = mu < lo ? __dsub_rn(lo, mu) : (mu > hi ? __dsub_rn(mu, hi) : 0.0);
  return __dmul_rn(d, d);
}

constexpr int kAxisTab = 8;

// Visit every listed cell of one Gaussian: f(cell_linear_index).
template <class F>
__device__ __forceinline__ void for_each_cell(const int32_t lo[3], const int32_t hi[3], double m0, double m1,
                                              double m2, double r2, const LevelGeom& g, int l, F&& f) {
  const int64_t dx = g.dims[l][0], dy = g.dims[l][1];
  const bool tab = hi[0] - lo[0] < kAxisTab && hi[1] - lo[1] < kAxisTab && hi[2] - lo[2] < kAxisTab;
  double tx[kAxisTab], ty[kAxisTab];
  if (tab) {
    for (int32_t c = lo[0]; c <= hi[0]; ++c) tx[c - lo[0]] = axis_d2(m0, c, g, l, 0);
    for (int32_t c = lo[1]; c <= hi[1]; ++c) ty[c - lo[1]] = axis_d2(m1, c, g, l, 1);
  }
  for (int32_t cz = lo[2]; cz <= hi[2]; ++cz) {
    const double dz2 = axis_d2(m2, cz, g, l, 2);
    for (int32_t cy = lo[1]; cy <= hi[1]; ++cy) {
      const double dy2 = tab ? ty[cy - lo[1]] : axis_d2(m1, cy, g, l, 1);
      for (int32_t cx = lo[0]; cx <= hi[0]; ++cx) {
        const double dx2 = tab ? tx[cx - lo[0]] : axis_d2(m0, cx, g, l, 0);
        if (__dadd_rn(__dadd_rn(dx2, dy2), dz2) <= r2) f(g.coff[l] + ((int64_t)cz * dy + cy) * dx + cx);
      }
    }
  }
}

// Record, C8 range and membership counts of Gaussian j; the counting atomics return each
// entry's rank inside its cell (see CullBufs).
__device__ __forceinline__ void record_and_count(int64_t j, const float p[kNP], double tau, const LevelGeom& g,
                                                 const CullBufs& cb, DevState* st) {
  float4 r[3];
  make_record(p, r);
  cb.rec[3 * j] = r[0]; cb.rec[3 * j + 1] = r[1]; cb.rec[3 * j + 2] = r[2];
  const int l = level_of_gaussian(g, j);
  int32_t lo[3], hi[3];
  double r2;
  cull_range(p, tau, g, l, lo, hi, r2);
  cb.rad2[j] = r2;
  const double m0 = p[P_MU], m1 = p[P_MU + 1], m2 = p[P_MU + 2];
  const int32_t nx = hi[0] - lo[0] + 1, ny = hi[1] - lo[1] + 1, nz = hi[2] - lo[2] + 1;
  uint32_t w;
  if (cb.need && !((cb.need[j] >> cb.me) & 1u)) {
    w = 0u;                                       // owner-computes: not needed here, not listed
  } else if (nx <= 3 && ny <= 3 && nz <= 3) {
    // common case: all counting atomics of the Gaussian in flight before any rank is stored
    const int64_t dx = g.dims[l][0], dy = g.dims[l][1];
    double tx[3], ty[3], tz[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      tx[c] = c < nx ? axis_d2(m0, lo[0] + c, g, l, 0) : 0.0;
      ty[c] = c < ny ? axis_d2(m1, lo[1] + c, g, l, 1) : 0.0;
      tz[c] = c < nz ? axis_d2(m2, lo[2] + c, g, l, 2) : 0.0;
    }
    uint32_t mask = 0, rk[27];
#pragma unroll
    for (int q = 0; q < 27; ++q) {
      const int qx = q % 3, qy = (q / 3) % 3, qz = q / 9;
      if (qx < nx && qy < ny && qz < nz && __dadd_rn(__dadd_rn(tx[qx], ty[qy]), tz[qz]) <= r2) {
        mask |= 1u << q;
        rk[q] = atomicAdd(cb.count + g.coff[l] + ((int64_t)(lo[2] + qz) * dy + (lo[1] + qy)) * dx + (lo[0] + qx), 1u);
      }
    }
#pragma unroll
    for (int q = 0; q < 27; ++q)
      if ((mask >> q) & 1u) cb.rank[27 * j + q] = rk[q];
    w = mask;
  } else {
    int n = 0;
    for_each_cell(lo, hi, m0, m1, m2, r2, g, l, [&](int64_t) { ++n; });
    const uint32_t base = atomicAdd(&st->ovf_next, (uint32_t)n);
    int i = 0;
    for_each_cell(lo, hi, m0, m1, m2, r2, g, l, [&](int64_t cell) {
      const uint32_t rk = atomicAdd(cb.count + cell, 1u);
      if (base + i < cb.ovf_cap) cb.ovf[base + i] = rk;
      else atomicOr(&st->csr_overflow, 1u);
      ++i;
    });
    w = 0x80000000u | (base & 0x7FFFFFFFu);
  }
  cb.range[j] = make_uint4((uint32_t)lo[0] | ((uint32_t)hi[0] << 16), (uint32_t)lo[1] | ((uint32_t)hi[1] << 16),
                           (uint32_t)lo[2] | ((uint32_t)hi[2] << 16), w);
}

}  // namespace gsc
