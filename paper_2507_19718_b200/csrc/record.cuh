// record.cuh -- evaluation record (A2) and exact conservative cell range (C8) of one
// Gaussian; shared by the create/set_params path and the fused optimizer epilogue.
#pragma once
#include "common.cuh"

namespace gsc {

// Upper bounds of 2^(r/8): the smallest doubles >= 2^(r/8) (C8; hex literals of the spec).
static __device__ const double kT8[8] = {
    0x1.0000000000000p+0, 0x1.172b83c7d517bp+0, 0x1.306fe0a31b716p+0, 0x1.4bfdad5362a28p+0,
    0x1.6a09e667f3bcdp+0, 0x1.8ace5422aa0dcp+0, 0x1.ae89f995ad3aep+0, 0x1.d5818dcfba488p+0};
constexpr double kK8 = 0x1.71547652b82fep+3;   // 8 log2(e)

// Record of one Gaussian from its raw parameters (C1): A = R diag(e^-2s) R^T is formed and
// Cholesky-factored in fp64 (A = U^T U), stored in fp32 with mu and v = w max(0, c).
__device__ __forceinline__ void make_record(const float p[kNP], float4 out[3]) {
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
  const float wo = 1.f / (1.f + expf(-p[P_O]));
  out[0] = make_float4((float)U00, (float)U01, (float)U02, (float)U11);
  out[1] = make_float4((float)U12, (float)U22, p[P_MU], p[P_MU + 1]);
  out[2] = make_float4(p[P_MU + 2], wo * fmaxf(p[P_C], 0.f), wo * fmaxf(p[P_C + 1], 0.f), wo * fmaxf(p[P_C + 2], 0.f));
}

// C8 cell range of one Gaussian, fp64 with explicitly rounded + - * / sqrt only.
__device__ __forceinline__ void cull_range(const float p[kNP], double tau, const LevelGeom& g, int l,
                           int32_t lo[3], int32_t hi[3]) {
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
  double U2[3];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    double sk = __dmul_rn((double)p[P_S + b], kK8);
    if (!(sk >= -8000.0)) sk = (sk != sk) ? 8000.0 : -8000.0;
    if (sk > 8000.0) sk = 8000.0;
    int32_t k = (int32_t)ceil(sk) + 1;
    int32_t Qe = (k >= 0) ? k / 8 : -((-k + 7) / 8);
    double U = ldexp(kT8[k - 8 * Qe], Qe);
    U2[b] = __dmul_rn(U, U);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double s0 = __dmul_rn(__dmul_rn(R[a][0], R[a][0]), U2[0]);
    double s1 = __dmul_rn(__dmul_rn(R[a][1], R[a][1]), U2[1]);
    double s2 = __dmul_rn(__dmul_rn(R[a][2], R[a][2]), U2[2]);
    double h = __dmul_rn(tau, __dsqrt_rn(__dadd_rn(__dadd_rn(s0, s1), s2)));
    double mu = (double)p[P_MU + a];
    lo[a] = clampcell(floor(__dmul_rn(__dsub_rn(__dsub_rn(mu, h), g.origin[l][a]), g.inv_cell[l][a])), g.dims[l][a]);
    hi[a] = clampcell(floor(__dmul_rn(__dsub_rn(__dadd_rn(mu, h), g.origin[l][a]), g.inv_cell[l][a])), g.dims[l][a]);
  }
}

__device__ __forceinline__ void record_and_count(int64_t j, const float p[kNP], double tau, const LevelGeom& g,
                                 float4* rec, uint4* range, uint32_t* csr_count) {
  float4 r[3];
  make_record(p, r);
  rec[3 * j] = r[0]; rec[3 * j + 1] = r[1]; rec[3 * j + 2] = r[2];
  int l = level_of_gaussian(g, j);
  int32_t lo[3], hi[3];
  cull_range(p, tau, g, l, lo, hi);
  uint32_t cnt = (uint32_t)(hi[0] - lo[0] + 1) * (uint32_t)(hi[1] - lo[1] + 1) * (uint32_t)(hi[2] - lo[2] + 1);
  range[j] = make_uint4((uint32_t)lo[0] | ((uint32_t)hi[0] << 16), (uint32_t)lo[1] | ((uint32_t)hi[1] << 16),
                        (uint32_t)lo[2] | ((uint32_t)hi[2] << 16), cnt);
  const int64_t dx = g.dims[l][0], dy = g.dims[l][1];
  for (int32_t cz = lo[2]; cz <= hi[2]; ++cz)
    for (int32_t cy = lo[1]; cy <= hi[1]; ++cy)
      for (int32_t cx = lo[0]; cx <= hi[0]; ++cx)
        atomicAdd(csr_count + g.coff[l] + ((int64_t)cz * dy + cy) * dx + cx, 1u);
}

}  // namespace gsc
