/*
 * oracle/gscache_oracle.c -- plain, slow, fp64 CPU oracle of the GSCache hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2507_19718_b200/) never links, imports or executes anything under oracle/,
 * and shares no code, header, table or constant generator with it.
 *
 * What it computes (PAPER.md = "P:", SPEC.md = "S:", SURVEY.md section 8(c) readings C1-C8):
 *   - create: nested MIP-style level subsets (sec.3.2, P:9) + Eq. 2 isotropic
 *     initial scales (Eq. 2) + 3DGS-like init        -> orc_create
 *   - activation of the 14 raw parameters (App. B)     -> orc_activate
 *   - evaluator: additive world-space mixture with Mahalanobis cut-off tau
 *     (reading A1/A2/A3 of DESIGN.md; low-opacity limit of P:68)           -> orc_eval_*
 *   - HDR loss Eq. 4 averaged per level over 3k valid samples   -> orc_loss_grad
 *   - analytic gradients into all 5 parameter groups ("inverse splatting")
 *   - AdamW (sec.3.6) with per-group LRs and Eq. 5 schedule
 *   - exact conservative culling rule C8 (transcendental-free, fp64)        -> orc_cull_*
 *
 * Everything is fp64, single-threaded, evaluated in the written order; compile with
 * -ffp-contract=off.  Brute force is the definition; the culled evaluator is an
 * independently written second path cross-checked to give the identical pair set.
 *
 * Parameter row layout (paper order): [0..2] position, [3..6] rotation
 * quaternion (w,x,y,z), [7..9] colour (raw), [10..12] log-scale, [13] opacity logit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NP 14

/* ------------------------------------------------------------------ create (C7) */

/* splitmix64 (standard constants) applied to state x; "fixed random permutation". */
uint64_t orc_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

typedef struct { uint64_t key; int64_t i; } orc_kv;
static int orc_kv_cmp(const void* a, const void* b) {
  const orc_kv* x = (const orc_kv*)a; const orc_kv* y = (const orc_kv*)b;
  if (x->key < y->key) return -1;
  if (x->key > y->key) return 1;
  return (x->i < y->i) ? -1 : (x->i > y->i);
}

/* perm = stable argsort of splitmix64(seed + i), i in [0, n). */
int orc_permutation(int64_t n, uint64_t seed, int64_t* perm) {
  orc_kv* kv = (orc_kv*)malloc(sizeof(orc_kv) * (size_t)(n > 0 ? n : 1));
  if (!kv) return -1;
  for (int64_t i = 0; i < n; ++i) { kv[i].key = orc_splitmix64(seed + (uint64_t)i); kv[i].i = i; }
  qsort(kv, (size_t)n, sizeof(orc_kv), orc_kv_cmp);
  for (int64_t i = 0; i < n; ++i) perm[i] = kv[i].i;
  free(kv);
  return 0;
}

/* Eq. 2 inner term: dbar_i = (1/3) sum_{j<3} d_ij, the mean distance to the 3 nearest
 * OTHER points, brute force over all pairs.  With fewer than 4 points the
 * available neighbours are averaged; a single point gets 0 (then floored). */
void orc_knn3_mean(int64_t n, const double* pts, double* dbar) {
  for (int64_t i = 0; i < n; ++i) {
    double best[3] = {INFINITY, INFINITY, INFINITY};
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      double dx = pts[3 * j + 0] - pts[3 * i + 0];
      double dy = pts[3 * j + 1] - pts[3 * i + 1];
      double dz = pts[3 * j + 2] - pts[3 * i + 2];
      double d = sqrt((dx * dx + dy * dy) + dz * dz);
      if (d < best[2]) {
        if (d < best[1]) {
          best[2] = best[1];
          if (d < best[0]) { best[1] = best[0]; best[0] = d; } else { best[1] = d; }
        } else {
          best[2] = d;
        }
      }
    }
    int k = (int)(n - 1 < 3 ? n - 1 : 3);
    if (k <= 0) { dbar[i] = 0.0; continue; }
    double sum = 0.0;
    for (int a = 0; a < k; ++a) sum = sum + best[a];
    dbar[i] = sum / (double)k;
  }
}

/* Eq. 2: s_i = max(min(mu_N + zcap*sigma_N, dbar_i), fl) * factor
 * ("\land" read as min; sigma population, ddof 0; floor for duplicate points).
 * fl = 1e-6*diag, or 1e-6 (world units) when diag = 0 -- a level of one point or of
 * coincident points (reading A20): the floor is applied after the cap so that no level can
 * produce s = 0 (ln s = -inf). */
void orc_eq2_from_dbar(int64_t n, const double* dbar, double diag, double zcap, double factor,
                       double* s) {
  double mu = 0.0;
  for (int64_t i = 0; i < n; ++i) mu = mu + dbar[i];
  mu = mu / (double)n;
  double var = 0.0;
  for (int64_t i = 0; i < n; ++i) { double d = dbar[i] - mu; var = var + d * d; }
  var = var / (double)n;
  double cap = mu + zcap * sqrt(var);
  double fl = diag > 0.0 ? 1e-6 * diag : 1e-6;
  for (int64_t i = 0; i < n; ++i) {
    double r = cap < dbar[i] ? cap : dbar[i];
    s[i] = (r > fl ? r : fl) * factor;
  }
}

/* AABB diagonal of a point set (floor reference for Eq. 2). */
double orc_diag(int64_t n, const double* pts) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      if (pts[3 * i + a] < lo[a]) lo[a] = pts[3 * i + a];
      if (pts[3 * i + a] > hi[a]) hi[a] = pts[3 * i + a];
    }
  if (n <= 0) return 0.0;
  double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
  return sqrt((dx * dx + dy * dy) + dz * dz);
}

/* Full create (C7).  counts non-increasing, counts[0] = N0.  P out: [sum counts][14]. */
int orc_create(int L, const int64_t* counts, const double* init_pos, const double* init_rgb,
               const double* init_log_scale, uint64_t seed, double init_opacity, double zcap,
               double factor, double* P) {
  int64_t N0 = counts[0];
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N0 > 0 ? N0 : 1));
  if (!perm) return -1;
  orc_permutation(N0, seed, perm);
  double logit = log(init_opacity / (1.0 - init_opacity));
  int64_t base = 0;
  for (int l = 0; l < L; ++l) {
    int64_t n = counts[l];
    double* pts = (double*)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
    double* dbar = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* s = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
      int64_t src = (l == 0) ? i : perm[i];
      double* row = P + (base + i) * NP;
      for (int a = 0; a < 3; ++a) { row[a] = init_pos[3 * src + a]; pts[3 * i + a] = row[a]; }
      row[3] = 1.0; row[4] = 0.0; row[5] = 0.0; row[6] = 0.0;
      for (int a = 0; a < 3; ++a) row[7 + a] = init_rgb[3 * src + a];
      row[13] = logit;
      if (init_log_scale)
        for (int a = 0; a < 3; ++a) row[10 + a] = init_log_scale[3 * src + a];
    }
    if (!init_log_scale && n > 0) {
      orc_knn3_mean(n, pts, dbar);
      orc_eq2_from_dbar(n, dbar, orc_diag(n, pts), zcap, factor, s);
      for (int64_t i = 0; i < n; ++i) {
        double ls = log(s[i]);
        double* row = P + (base + i) * NP;
        row[10] = ls; row[11] = ls; row[12] = ls;
      }
    }
    free(pts); free(dbar); free(s);
    base += n;
  }
  free(perm);
  return 0;
}

/* ------------------------------------------------------------- activation (C1) */

#include "gscache_oracle.h"

/* R(q) for a unit quaternion (w,x,y,z), standard 3DGS formula, written order. */
static void orc_rot(const double q[4], double R[3][3]) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0][0] = 1.0 - 2.0 * (y * y + z * z); R[0][1] = 2.0 * (x * y - w * z); R[0][2] = 2.0 * (x * z + w * y);
  R[1][0] = 2.0 * (x * y + w * z); R[1][1] = 1.0 - 2.0 * (x * x + z * z); R[1][2] = 2.0 * (y * z - w * x);
  R[2][0] = 2.0 * (x * z - w * y); R[2][1] = 2.0 * (y * z + w * x); R[2][2] = 1.0 - 2.0 * (x * x + y * y);
}

/* q_hat = q/||q||; ||q||^2 < 1e-24 -> identity rotation, zero rotation gradient (C1/A6). */
static void orc_qnorm(const double* q, double qhat[4], double* qn, int* degenerate) {
  double n2 = ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3];
  if (n2 < 1e-24) {
    qhat[0] = 1.0; qhat[1] = 0.0; qhat[2] = 0.0; qhat[3] = 0.0; *qn = 0.0; *degenerate = 1;
    return;
  }
  double n = sqrt(n2);
  for (int a = 0; a < 4; ++a) qhat[a] = q[a] / n;
  *qn = n; *degenerate = 0;
}

void orc_activate_row(const double* p, orc_gauss* g) {
  for (int a = 0; a < 3; ++a) g->mu[a] = p[a];
  orc_qnorm(p + 3, g->qhat, &g->qnorm, &g->degenerate);
  orc_rot(g->qhat, g->R);
  for (int k = 0; k < 3; ++k) g->D[k] = exp(-2.0 * p[10 + k]);       /* Sigma^-1 = R diag(e^-2s) R^T */
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += g->R[a][k] * g->D[k] * g->R[b][k];
      g->A[a][b] = acc;
    }
  g->w = 1.0 / (1.0 + exp(-p[13]));                                  /* sigmoid opacity (A5) */
  for (int c = 0; c < 3; ++c) {
    g->chat[c] = p[7 + c] > 0.0 ? p[7 + c] : 0.0;                     /* max(0, c) (A4)      */
    g->v[c] = g->w * g->chat[c];
  }
}

/* Exported for tests: A (row-major 3x3) and v of one parameter row. */
void orc_activate(const double* p, double* A9, double* v3, double* w) {
  orc_gauss g;
  orc_activate_row(p, &g);
  for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) A9[3 * a + b] = g.A[a][b];
  for (int c = 0; c < 3; ++c) v3[c] = g.v[c];
  *w = g.w;
}

static double orc_Q(const orc_gauss* g, const double* x, double d[3], double t[3]) {
  for (int a = 0; a < 3; ++a) d[a] = x[a] - g->mu[a];
  for (int a = 0; a < 3; ++a) t[a] = g->A[a][0] * d[0] + g->A[a][1] * d[1] + g->A[a][2] * d[2];
  return d[0] * t[0] + d[1] * t[1] + d[2] * t[2];
}

/* ------------------------------------------------------------- evaluator (C3) */

static orc_gauss* orc_activate_all(int64_t G, const double* P) {
  orc_gauss* g = (orc_gauss*)malloc(sizeof(orc_gauss) * (size_t)(G > 0 ? G : 1));
  if (!g) return NULL;
  for (int64_t j = 0; j < G; ++j) orc_activate_row(P + j * NP, &g[j]);
  return g;
}

/* yhat(x) = sum_j v_j exp(-Q_j(x)/2) [Q_j(x) <= tau^2] -- brute force over one level's
 * G Gaussians.  amb (nullable, [S][3]) receives the A3 allowance sum of v_j e^{-tau^2/2}
 * over pairs with |Q - tau^2| <= amb_rel*tau^2; amb_n (nullable, [S]) counts them. */
void orc_eval_brute(int64_t G, const double* P, double tau, int64_t S, const double* x,
                    double* y, int64_t* npairs, double amb_rel, double* amb, int32_t* amb_n) {
  orc_gauss* g = orc_activate_all(G, P);
  double t2 = tau * tau;
  int64_t np = 0;
  for (int64_t i = 0; i < S; ++i) {
    double acc[3] = {0.0, 0.0, 0.0}, al[3] = {0.0, 0.0, 0.0};
    int32_t na = 0;
    for (int64_t j = 0; j < G; ++j) {
      double d[3], t[3];
      double Q = orc_Q(&g[j], x + 3 * i, d, t);
      if (amb && fabs(Q - t2) <= amb_rel * t2) {
        for (int c = 0; c < 3; ++c) al[c] += g[j].v[c] * exp(-0.5 * t2);
        ++na;
      }
      if (Q <= t2) {
        double e = exp(-0.5 * Q);
        for (int c = 0; c < 3; ++c) acc[c] += g[j].v[c] * e;
        ++np;
      }
    }
    for (int c = 0; c < 3; ++c) y[3 * i + c] = acc[c];
    if (amb) for (int c = 0; c < 3; ++c) amb[3 * i + c] = al[c];
    if (amb_n) amb_n[i] = na;
  }
  if (npairs) *npairs = np;
  free(g);
}

/* Dense Q matrix [S][G] (tiny cases only; containment / ambiguity tests). */
void orc_q_matrix(int64_t G, const double* P, int64_t S, const double* x, double* Qout) {
  orc_gauss* g = orc_activate_all(G, P);
  for (int64_t i = 0; i < S; ++i)
    for (int64_t j = 0; j < G; ++j) {
      double d[3], t[3];
      Qout[i * G + j] = orc_Q(&g[j], x + 3 * i, d, t);
    }
  free(g);
}

/* ------------------------------------------------ exact conservative culling (C8) */

/* Upper bounds of 2^(r/32), r = 0..31: the smallest doubles >= 2^(r/32) (C8). */
static const double orc_T32[32] = {
  0x1.0000000000000p+0, 0x1.059b0d3158575p+0, 0x1.0b5586cf98910p+0, 0x1.11301d0125b51p+0,
  0x1.172b83c7d517bp+0, 0x1.1d4873168b9abp+0, 0x1.2387a6e756239p+0, 0x1.29e9df51fdee2p+0,
  0x1.306fe0a31b716p+0, 0x1.371a7373aa9cbp+0, 0x1.3dea64c123423p+0, 0x1.44e086061892ep+0,
  0x1.4bfdad5362a28p+0, 0x1.5342b569d4f82p+0, 0x1.5ab07dd48542ap+0, 0x1.6247eb03a5585p+0,
  0x1.6a09e667f3bcdp+0, 0x1.71f75e8ec5f74p+0, 0x1.7a11473eb0187p+0, 0x1.82589994cce13p+0,
  0x1.8ace5422aa0dcp+0, 0x1.93737b0cdc5e5p+0, 0x1.9c49182a3f091p+0, 0x1.a5503b23e255dp+0,
  0x1.ae89f995ad3aep+0, 0x1.b7f76f2fb5e47p+0, 0x1.c199bdd85529dp+0, 0x1.cb720dcef906ap+0,
  0x1.d5818dcfba488p+0, 0x1.dfc97337b9b5fp+0, 0x1.ea4afa2a490dap+0, 0x1.f50765b6e4541p+0};
static const double orc_K32 = 0x1.71547652b82fep+5; /* 32*log2(e) */

static int32_t orc_clampcell(double f, int32_t dim) {
  if (!(f >= 0.0)) return 0;                 /* also catches -inf */
  if (f > (double)(dim - 1)) return dim - 1;
  return (int32_t)f;
}

/* Sample cell c_a = clamp(floor((x_a - origin_a)*inv_cell_a), 0, dims_a-1). */
void orc_sample_cell(const double* x, const double* origin, const double* inv_cell,
                     const int32_t* dims, int32_t* c3) {
  for (int a = 0; a < 3; ++a) c3[a] = orc_clampcell(floor((x[a] - origin[a]) * inv_cell[a]), dims[a]);
}

/* C8 per Gaussian: inclusive cell range [lo, hi] per axis (the AABB of the tau-ellipsoid
 * bounded with U_b >= e^{s_b}) and r2 = tau^2 max_b U_b^2, the squared radius of a sphere
 * containing the ellipsoid.  Only + - * / sqrt floor ceil ldexp; written order, no FMA.
 * U_b = ldexp(T32[r], Q) with k_b = ceil(s_b * 32 log2 e) + 1, Q = floor(k_b/32), r = k_b - 32Q,
 * so U_b / e^{s_b} lies in (2^{1/32}, 2^{2/32}]. */
void orc_cull_ranges(int64_t G, const double* P, double tau, const double* origin,
                     const double* inv_cell, const int32_t* dims, int32_t* rng /*[G][6]*/,
                     double* r2 /*[G] or NULL*/) {
  for (int64_t j = 0; j < G; ++j) {
    const double* p = P + j * NP;
    double qh[4], qn, R[3][3], U1[3], U2[3];
    int deg;
    orc_qnorm(p + 3, qh, &qn, &deg);
    orc_rot(qh, R);
    for (int b = 0; b < 3; ++b) {
      double sk = p[10 + b] * orc_K32;          /* clamp keeps the int conversion defined   */
      if (!(sk >= -32000.0)) sk = (sk != sk) ? 32000.0 : -32000.0;   /* NaN -> huge extent */
      if (sk > 32000.0) sk = 32000.0;
      int32_t k = (int32_t)ceil(sk) + 1;
      int32_t Qe = (k >= 0) ? k / 32 : -((-k + 31) / 32);   /* floor(k/32) */
      int32_t r = k - 32 * Qe;
      double U = ldexp(orc_T32[r], Qe);
      U1[b] = U;
      U2[b] = U * U;
    }
    /* isotropic (s_0 = s_1 = s_2): the ellipsoid is a ball of radius tau e^s <= tau U, so
     * h_a = tau U exactly (R R^T = I; C8) */
    const int iso = p[10] == p[11] && p[11] == p[12];
    for (int a = 0; a < 3; ++a) {
      double s0 = R[a][0] * R[a][0] * U2[0];
      double s1 = R[a][1] * R[a][1] * U2[1];
      double s2 = R[a][2] * R[a][2] * U2[2];
      double h = iso ? tau * U1[0] : tau * sqrt((s0 + s1) + s2);
      double flo = floor(((p[a] - h) - origin[a]) * inv_cell[a]);
      double fhi = floor(((p[a] + h) - origin[a]) * inv_cell[a]);
      rng[6 * j + a] = orc_clampcell(flo, dims[a]);
      rng[6 * j + 3 + a] = orc_clampcell(fhi, dims[a]);
    }
    if (r2) {
      double um = U2[0];
      if (U2[1] > um) um = U2[1];
      if (U2[2] > um) um = U2[2];
      r2[j] = (tau * tau) * um;
    }
  }
}

/* Is cell c (per-axis indices) within the sphere |x - mu|^2 <= r2 of a Gaussian?  Squared
 * distance from mu to the cell's box [o + c*e, o + (c+1)*e] with e = 1/inv_cell; border
 * cells extend to infinity outwards (samples outside the grid clamp into them, A17). */
int orc_cell_hit(const double* mu, double r2, const int32_t* c, const double* origin,
                 const double* inv_cell, const int32_t* dims) {
  double D2 = 0.0;
  for (int a = 0; a < 3; ++a) {
    double e = 1.0 / inv_cell[a];
    double lo = c[a] == 0 ? -INFINITY : origin[a] + (double)c[a] * e;
    double hi = c[a] == dims[a] - 1 ? INFINITY : origin[a] + (double)(c[a] + 1) * e;
    double d = mu[a] < lo ? lo - mu[a] : (mu[a] > hi ? mu[a] - hi : 0.0);
    D2 = D2 + d * d;
  }
  return D2 <= r2;
}

/* CSR cell -> ascending Gaussian indices (local to the level): Gaussian j is listed in every
 * cell of its range that passes orc_cell_hit.  offsets: [cells+1].  If idx == NULL only the
 * offsets are produced (returns total entries). */
int64_t orc_build_csr(int64_t G, const double* P, const int32_t* rng, const double* r2,
                      const double* origin, const double* inv_cell, const int32_t* dims,
                      int64_t* offsets, int32_t* idx) {
  int64_t cells = (int64_t)dims[0] * dims[1] * dims[2];
  for (int64_t c = 0; c <= cells; ++c) offsets[c] = 0;
  for (int pass = 0; pass < 2; ++pass) {
    int64_t* cur = NULL;
    if (pass == 1) {
      if (!idx) break;
      for (int64_t c = 0; c < cells; ++c) offsets[c + 1] += offsets[c];
      cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cells > 0 ? cells : 1));
      for (int64_t c = 0; c < cells; ++c) cur[c] = offsets[c];
    }
    for (int64_t j = 0; j < G; ++j) {
      const int32_t* r = rng + 6 * j;
      const double* mu = P + j * NP;
      int32_t c3[3];
      for (c3[2] = r[2]; c3[2] <= r[5]; ++c3[2])
        for (c3[1] = r[1]; c3[1] <= r[4]; ++c3[1])
          for (c3[0] = r[0]; c3[0] <= r[3]; ++c3[0]) {
            if (!orc_cell_hit(mu, r2[j], c3, origin, inv_cell, dims)) continue;
            int64_t cell = ((int64_t)c3[2] * dims[1] + c3[1]) * dims[0] + c3[0];
            if (pass == 0) offsets[cell + 1] += 1;
            else idx[cur[cell]++] = (int32_t)j;
          }
    }
    if (cur) free(cur);
  }
  if (!idx) for (int64_t c = 0; c < cells; ++c) offsets[c + 1] += offsets[c];
  return offsets[cells];
}

/* ------------------------------------------ loss (C4), gradients (C5), fit (C6) */

typedef struct {
  const double* origin; const double* inv_cell; const int32_t* dims; /* per level, [L][3] */
} orc_grids;

typedef struct { int64_t cells; int64_t* off; int32_t* idx; int32_t* rng; } orc_csr;

static int orc_csr_make(int64_t G, const double* P, double tau, const double* origin,
                        const double* inv_cell, const int32_t* dims, orc_csr* c) {
  c->cells = (int64_t)dims[0] * dims[1] * dims[2];
  c->rng = (int32_t*)malloc(sizeof(int32_t) * 6 * (size_t)(G > 0 ? G : 1));
  double* r2 = (double*)malloc(sizeof(double) * (size_t)(G > 0 ? G : 1));
  c->off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(c->cells + 1));
  orc_cull_ranges(G, P, tau, origin, inv_cell, dims, c->rng, r2);
  int64_t n = orc_build_csr(G, P, c->rng, r2, origin, inv_cell, dims, c->off, NULL);
  c->idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  orc_build_csr(G, P, c->rng, r2, origin, inv_cell, dims, c->off, c->idx);
  free(r2);
  return 0;
}
static void orc_csr_free(orc_csr* c) { free(c->rng); free(c->off); free(c->idx); }

/* C2: level = min(n, L) - 1 for n >= 1; n <= 0 or non-finite pos/rgb -> dropped (-1). */
int32_t orc_level_of(int32_t n, int L, const double* x, const double* rgb) {
  if (n <= 0) return -1;
  for (int a = 0; a < 3; ++a) if (!isfinite(x[a])) return -1;
  if (rgb) for (int a = 0; a < 3; ++a) if (!isfinite(rgb[a])) return -1;
  return (n < L ? n : L) - 1;
}

/* Evaluate the level mixture at each sample (query semantics; level per sample or fixed).
 * level_fixed >= 0 overrides len.  Invalid samples get y = 0 and level -1.
 * grids == NULL -> brute force, else the independent culled evaluator. */
int orc_query(int L, const int64_t* goff, const double* P, double tau, int64_t S,
              const double* x, const int32_t* len, int level_fixed,
              const double* g_origin, const double* g_inv, const int32_t* g_dims,
              int32_t* level_of, double* y, int64_t* npairs) {
  int64_t np = 0;
  orc_gauss* gs = orc_activate_all(goff[L], P);
  orc_csr* csr = NULL;
  if (g_origin) {
    csr = (orc_csr*)malloc(sizeof(orc_csr) * (size_t)L);
    for (int l = 0; l < L; ++l)
      orc_csr_make(goff[l + 1] - goff[l], P + goff[l] * NP, tau, g_origin + 3 * l, g_inv + 3 * l,
                   g_dims + 3 * l, &csr[l]);
  }
  double t2 = tau * tau;
  for (int64_t i = 0; i < S; ++i) {
    const double* xi = x + 3 * i;
    int32_t l = level_fixed >= 0 ? level_fixed : orc_level_of(len[i], L, xi, NULL);
    if (level_fixed >= 0) for (int a = 0; a < 3; ++a) if (!isfinite(xi[a])) l = -1;
    level_of[i] = l;
    double acc[3] = {0.0, 0.0, 0.0};
    if (l >= 0) {
      if (!csr) {
        for (int64_t j = goff[l]; j < goff[l + 1]; ++j) {
          double d[3], t[3];
          double Q = orc_Q(&gs[j], xi, d, t);
          if (Q <= t2) { double e = exp(-0.5 * Q); for (int c = 0; c < 3; ++c) acc[c] += gs[j].v[c] * e; ++np; }
        }
      } else {
        int32_t c3[3];
        orc_sample_cell(xi, g_origin + 3 * l, g_inv + 3 * l, g_dims + 3 * l, c3);
        const int32_t* dm = g_dims + 3 * l;
        int64_t cell = ((int64_t)c3[2] * dm[1] + c3[1]) * dm[0] + c3[0];
        for (int64_t k = csr[l].off[cell]; k < csr[l].off[cell + 1]; ++k) {
          int64_t j = goff[l] + csr[l].idx[k];
          double d[3], t[3];
          double Q = orc_Q(&gs[j], xi, d, t);
          if (Q <= t2) { double e = exp(-0.5 * Q); for (int c = 0; c < 3; ++c) acc[c] += gs[j].v[c] * e; ++np; }
        }
      }
    }
    for (int c = 0; c < 3; ++c) y[3 * i + c] = acc[c];
  }
  if (csr) { for (int l = 0; l < L; ++l) orc_csr_free(&csr[l]); free(csr); }
  free(gs);
  if (npairs) *npairs = np;
  return 0;
}

/* dR/dq_hat_c for c = w,x,y,z (C5), as 2*[...] matrices. */
static void orc_dRdq(const double q[4], double dR[4][3][3]) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  double Mw[3][3] = {{0, -z, y}, {z, 0, -x}, {-y, x, 0}};
  double Mx[3][3] = {{0, y, z}, {y, -2 * x, -w}, {z, w, -2 * x}};
  double My[3][3] = {{-2 * y, x, w}, {x, 0, z}, {-w, z, -2 * y}};
  double Mz[3][3] = {{-2 * z, -w, x}, {w, -2 * z, y}, {x, y, 0}};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      dR[0][a][b] = 2 * Mw[a][b]; dR[1][a][b] = 2 * Mx[a][b];
      dR[2][a][b] = 2 * My[a][b]; dR[3][a][b] = 2 * Mz[a][b];
    }
}

/* Chain rule from the coefficient gradients (dmu, full symmetric dA, dv) of one Gaussian
 * to its 14 raw-parameter gradients (C5). */
static void orc_chain(const orc_gauss* g, const double* p, const double dmu[3],
                      double dA[3][3], const double dv[3], double* out) {
  for (int a = 0; a < 3; ++a) out[a] = dmu[a];
  /* M = R^T dA R ; ds_k = -2 D_k M_kk */
  double M[3][3];
  for (int k = 0; k < 3; ++k)
    for (int l = 0; l < 3; ++l) {
      double acc = 0.0;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) acc += g->R[a][k] * dA[a][b] * g->R[b][l];
      M[k][l] = acc;
    }
  for (int k = 0; k < 3; ++k) out[10 + k] = -2.0 * g->D[k] * M[k][k];
  /* dR = 2 dA R D (dA symmetric) */
  double dR[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int c = 0; c < 3; ++c) acc += dA[a][c] * g->R[c][b];
      dR[a][b] = 2.0 * acc * g->D[b];
    }
  if (g->degenerate) {
    for (int c = 0; c < 4; ++c) out[3 + c] = 0.0;
  } else {
    double J[4][3][3], dqh[4];
    orc_dRdq(g->qhat, J);
    for (int c = 0; c < 4; ++c) {
      double acc = 0.0;
      for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) acc += dR[a][b] * J[c][a][b];
      dqh[c] = acc;
    }
    double dot = 0.0;
    for (int c = 0; c < 4; ++c) dot += g->qhat[c] * dqh[c];
    for (int c = 0; c < 4; ++c) out[3 + c] = (dqh[c] - g->qhat[c] * dot) / g->qnorm;
  }
  /* v = w * max(0,c): dw = sum dv*chat ; do = dw w (1-w) ; dc = w dv [c>0] */
  double dw = 0.0;
  for (int c = 0; c < 3; ++c) dw += dv[c] * g->chat[c];
  out[13] = dw * g->w * (1.0 - g->w);
  for (int c = 0; c < 3; ++c) out[7 + c] = p[7 + c] > 0.0 ? g->w * dv[c] : 0.0;
}

/* One forward + HDR loss + backward over a batch (C2-C5).
 *   P [G][14], goff [L+1]; samples x [S][3], len [S], rgb [S][3].
 *   mode 0: stop-gradient denominator (reading A10), 1: full quotient.
 * Outputs: level_of [S], yhat [S][3] (nullable), count [L], loss [L] (L_l of C4),
 * grad [G][14] raw gradients of L = sum_l L_l, npairs (nullable).
 * g_origin == NULL -> brute force, else the culled evaluator (identical pair set). */
int orc_loss_grad(int L, const int64_t* goff, const double* P, double tau, double hdr_eps,
                  int mode, int64_t S, const double* x, const int32_t* len, const double* rgb,
                  const double* g_origin, const double* g_inv, const int32_t* g_dims,
                  int32_t* level_of, double* yhat, int64_t* count, double* loss, double* grad,
                  int64_t* npairs, double* cgrad) {
  int64_t G = goff[L];
  orc_gauss* gs = orc_activate_all(G, P);
  double* cg = (double*)calloc((size_t)(G > 0 ? G : 1) * 15, sizeof(double)); /* dmu3 dA9 dv3 */
  double* yy = (double*)malloc(sizeof(double) * 3 * (size_t)(S > 0 ? S : 1));
  orc_csr* csr = NULL;
  if (g_origin) {
    csr = (orc_csr*)malloc(sizeof(orc_csr) * (size_t)L);
    for (int l = 0; l < L; ++l)
      orc_csr_make(goff[l + 1] - goff[l], P + goff[l] * NP, tau, g_origin + 3 * l, g_inv + 3 * l,
                   g_dims + 3 * l, &csr[l]);
  }
  double t2 = tau * tau;
  int64_t np = 0;
  for (int l = 0; l < L; ++l) { count[l] = 0; loss[l] = 0.0; }
  for (int64_t i = 0; i < S; ++i) {
    level_of[i] = orc_level_of(len[i], L, x + 3 * i, rgb + 3 * i);
    if (level_of[i] >= 0) count[level_of[i]] += 1;
  }
  /* pass 1: yhat and per-sample loss */
  for (int64_t i = 0; i < S; ++i) {
    int32_t l = level_of[i];
    double acc[3] = {0.0, 0.0, 0.0};
    if (l >= 0) {
      const double* xi = x + 3 * i;
      int64_t kbeg, kend; int64_t cell = 0;
      if (csr) {
        int32_t c3[3]; const int32_t* dm = g_dims + 3 * l;
        orc_sample_cell(xi, g_origin + 3 * l, g_inv + 3 * l, dm, c3);
        cell = ((int64_t)c3[2] * dm[1] + c3[1]) * dm[0] + c3[0];
        kbeg = csr[l].off[cell]; kend = csr[l].off[cell + 1];
      } else { kbeg = goff[l]; kend = goff[l + 1]; }
      for (int64_t k = kbeg; k < kend; ++k) {
        int64_t j = csr ? goff[l] + csr[l].idx[k] : k;
        double d[3], t[3];
        double Q = orc_Q(&gs[j], xi, d, t);
        if (Q <= t2) { double e = exp(-0.5 * Q); for (int c = 0; c < 3; ++c) acc[c] += gs[j].v[c] * e; ++np; }
      }
    }
    for (int c = 0; c < 3; ++c) yy[3 * i + c] = acc[c];
  }
  /* loss (Eq. 4 per level, averaged over 3 k_l) and dL/dyhat */
  for (int64_t i = 0; i < S; ++i) {
    int32_t l = level_of[i];
    if (l < 0) continue;
    double k3 = 3.0 * (double)count[l];
    double gch[3];
    for (int c = 0; c < 3; ++c) {
      double xh = rgb[3 * i + c], yh = yy[3 * i + c];
      double den = yh + hdr_eps;
      loss[l] += (xh - yh) * (xh - yh) / (den * den);
      if (mode == 0) gch[c] = (-2.0 * (xh - yh) / (den * den)) / k3;
      else gch[c] = (-2.0 * (xh - yh) * (xh + hdr_eps) / (den * den * den)) / k3;
    }
    /* pass 2: per pair contributions */
    const double* xi = x + 3 * i;
    int64_t kbeg, kend;
    if (csr) {
      int32_t c3[3]; const int32_t* dm = g_dims + 3 * l;
      orc_sample_cell(xi, g_origin + 3 * l, g_inv + 3 * l, dm, c3);
      int64_t cell = ((int64_t)c3[2] * dm[1] + c3[1]) * dm[0] + c3[0];
      kbeg = csr[l].off[cell]; kend = csr[l].off[cell + 1];
    } else { kbeg = goff[l]; kend = goff[l + 1]; }
    for (int64_t k = kbeg; k < kend; ++k) {
      int64_t j = csr ? goff[l] + csr[l].idx[k] : k;
      double d[3], t[3];
      double Q = orc_Q(&gs[j], xi, d, t);
      if (!(Q <= t2)) continue;
      double e = exp(-0.5 * Q);
      double h = gch[0] * gs[j].v[0] + gch[1] * gs[j].v[1] + gch[2] * gs[j].v[2];
      double* cj = cg + 15 * j;
      for (int a = 0; a < 3; ++a) cj[a] += h * e * t[a];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) cj[3 + 3 * a + b] += -0.5 * h * e * d[a] * d[b];
      for (int c = 0; c < 3; ++c) cj[12 + c] += gch[c] * e;
    }
  }
  for (int l = 0; l < L; ++l) if (count[l] > 0) loss[l] = loss[l] / (3.0 * (double)count[l]);
  for (int64_t j = 0; j < G; ++j) {
    double dA[3][3];
    const double* cj = cg + 15 * j;
    for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) dA[a][b] = cj[3 + 3 * a + b];
    orc_chain(&gs[j], P + j * NP, cj, dA, cj + 12, grad + j * NP);
  }
  if (yhat) memcpy(yhat, yy, sizeof(double) * 3 * (size_t)S);
  /* cgrad (nullable, [G][15]): the coefficient gradients of C5 before the chain rule --
   * dL/dmu (3), dL/dA as the full symmetric 3x3 (9, row-major), dL/dv (3) */
  if (cgrad) memcpy(cgrad, cg, sizeof(double) * 15 * (size_t)G);
  if (npairs) *npairs = np;
  if (csr) { for (int l = 0; l < L; ++l) orc_csr_free(&csr[l]); free(csr); }
  free(yy); free(cg); free(gs);
  return 0;
}

/* AdamW on n scalars (C6, PyTorch order).  Non-finite gradient elements are skipped
 * (element and moments unchanged) and counted.  step = Adam counter after increment. */
int64_t orc_adamw(int64_t n, double* p, double* m, double* v, const double* g, double lr,
                  double wd, double b1, double b2, double eps, int64_t step) {
  int64_t bad = 0;
  double bc1 = 1.0 - pow(b1, (double)step), bc2 = 1.0 - pow(b2, (double)step);
  for (int64_t i = 0; i < n; ++i) {
    if (!isfinite(g[i])) { ++bad; continue; }
    p[i] = p[i] * (1.0 - lr * wd);
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];
    v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
    p[i] = p[i] - lr * (m[i] / bc1) / (sqrt(v[i] / bc2) + eps);
  }
  return bad;
}

/* Eq. 5: eta_t = eta_0 / (1 + ln t), natural log (reading A14). */
double orc_lr_schedule(double eta0, int64_t t) { return eta0 / (1.0 + log((double)t)); }

/* group of raw parameter column k: 0 pos, 1 rot, 2 colour, 3 scale, 4 opacity */
static int orc_group(int k) { return k < 3 ? 0 : (k < 7 ? 1 : (k < 10 ? 2 : (k < 13 ? 3 : 4))); }

int orc_opt_step(int L, const int64_t* goff, double* P, double* M, double* V, int64_t* adam_step,
                 int64_t* t_sched, const double* hp, const int64_t* count, const double* grad,
                 int64_t* nonfinite);

/* hp layout: lr[5], wd[5], beta1, beta2, adam_eps, hdr_eps, tau, mode, schedule (17 doubles)
 * One gc_fit step (C6): returns 0 = stepped, 1 = no valid sample (no-op, t not advanced). */
int orc_fit_step(int L, const int64_t* goff, double* P, double* M, double* V, int64_t* adam_step,
                 int64_t* t_sched, const double* hp, int64_t S, const double* x,
                 const int32_t* len, const double* rgb, const double* g_origin,
                 const double* g_inv, const int32_t* g_dims, int64_t* count, double* loss,
                 double* grad, int64_t* nonfinite, int64_t* npairs) {
  int64_t G = goff[L];
  int32_t* lv = (int32_t*)malloc(sizeof(int32_t) * (size_t)(S > 0 ? S : 1));
  orc_loss_grad(L, goff, P, hp[14], hp[13], (int)hp[15], S, x, len, rgb, g_origin, g_inv, g_dims,
                lv, NULL, count, loss, grad, npairs, NULL);
  free(lv);
  return orc_opt_step(L, goff, P, M, V, adam_step, t_sched, hp, count, grad, nonfinite);
}

/* The optimizer half of a step (C6) on a given normalised raw gradient grad [G][14] with the
 * per-level sample counts `count` (a level with count 0 skips, A12; none at all: no-op).
 * Shared by orc_fit_step and the screen-space fit of the tests (next row f1). */
int orc_opt_step(int L, const int64_t* goff, double* P, double* M, double* V, int64_t* adam_step,
                 int64_t* t_sched, const double* hp, const int64_t* count, const double* grad,
                 int64_t* nonfinite) {
  int64_t G = goff[L];
  int64_t tot = 0;
  for (int l = 0; l < L; ++l) tot += count[l];
  *nonfinite = 0;
  if (tot == 0) return 1;
  *t_sched += 1;
  double eta[5];
  for (int gI = 0; gI < 5; ++gI) eta[gI] = hp[16] != 0.0 ? orc_lr_schedule(hp[gI], *t_sched) : hp[gI];
  for (int l = 0; l < L; ++l) {
    if (count[l] == 0) continue;                                     /* A12: skip level */
    adam_step[l] += 1;
    for (int64_t j = goff[l]; j < goff[l + 1]; ++j)
      for (int k = 0; k < NP; ++k) {
        int gI = orc_group(k);
        /* reading A16: a group whose learning rate is 0 is excluded from the optimizer
         * (App. A.2: covariance optimization "by default we disabled"): its parameters
         * and AdamW moments stay unchanged and its gradients are not counted */
        if (hp[gI] == 0.0) continue;
        *nonfinite += orc_adamw(1, P + j * NP + k, M + j * NP + k, V + j * NP + k,
                                grad + j * NP + k, eta[gI], hp[5 + gI], hp[10], hp[11], hp[12],
                                adam_step[l]);
      }
  }
  (void)G;
  return 0;
}

/* ------------------------------------- A3 boundary allowance of the gradients (tests) */

/* Reading A3 lets a pair with |Q - tau^2| <= amb_rel tau^2 fall on either side of the cut-off
 * in fp32.  A flip changes the flipped pair's own contribution to its Gaussian's gradient and,
 * through yhat_i, the loss gradient g_i of its sample and hence every pair of that sample.
 * This bounds both to first order, per Gaussian, as absolute values:
 *   a_i,ch  = sum_{ambiguous j} v_j,ch e^{-Q_ij/2}       (|d yhat_i|)
 *   gam_i,ch = |dg/dyhat|_i,ch a_i,ch                   (|d g_i|)
 *   inside pair, not ambiguous:  |d(dmu)| <= Gam e |t|, |d(dA)| <= Gam e |d d^T| / 2,
 *     |d(dv_ch)| <= gam_ch e, with Gam = sum_ch gam_ch v_j,ch;
 *   ambiguous pair: its whole contribution with |g| + gam in place of g.
 * allow_coef [G][15] (dmu 3, dA 9 full, dv 3) and allow_raw [G][14] (the bound carried through
 * the chain rule of C5 with absolute values).  Samples with an ambiguous pair are counted in
 * *n_amb.  Culled evaluation when g_origin != NULL (same pair sets as orc_loss_grad). */
/* cond != 0 computes instead the CONDITION magnitudes of the same gradients: every pair inside
 * the cut-off contributes with absolute values (|g| in place of g, |h e t|, |h e d d^T| / 2,
 * |g e|) and the chain rule is applied with absolute values, so kappa_i >= |grad_i|; a
 * relative perturbation delta of every summed term (fp32 rounding, atomic summation order)
 * changes grad_i by at most delta kappa_i to first order. */
int orc_grad_allowance(int L, const int64_t* goff, const double* P, double tau, double hdr_eps,
                       int mode, int64_t S, const double* x, const int32_t* len, const double* rgb,
                       const double* g_origin, const double* g_inv, const int32_t* g_dims,
                       double amb_rel, int cond, double* allow_coef, double* allow_raw, int64_t* n_amb) {
  int64_t G = goff[L];
  orc_gauss* gs = orc_activate_all(G, P);
  orc_csr* csr = NULL;
  if (g_origin) {
    csr = (orc_csr*)malloc(sizeof(orc_csr) * (size_t)L);
    for (int l = 0; l < L; ++l)
      orc_csr_make(goff[l + 1] - goff[l], P + goff[l] * NP, tau, g_origin + 3 * l, g_inv + 3 * l,
                   g_dims + 3 * l, &csr[l]);
  }
  int64_t* count = (int64_t*)calloc((size_t)L, sizeof(int64_t));
  int32_t* lv = (int32_t*)malloc(sizeof(int32_t) * (size_t)(S > 0 ? S : 1));
  for (int64_t i = 0; i < S; ++i) {
    lv[i] = orc_level_of(len[i], L, x + 3 * i, rgb + 3 * i);
    if (lv[i] >= 0) count[lv[i]] += 1;
  }
  for (int64_t k = 0; k < 15 * G; ++k) allow_coef[k] = 0.0;
  double t2 = tau * tau;
  int64_t na = 0;
  for (int64_t i = 0; i < S; ++i) {
    int32_t l = lv[i];
    if (l < 0) continue;
    const double* xi = x + 3 * i;
    int64_t kbeg, kend;
    if (csr) {
      int32_t c3[3]; const int32_t* dm = g_dims + 3 * l;
      orc_sample_cell(xi, g_origin + 3 * l, g_inv + 3 * l, dm, c3);
      int64_t cell = ((int64_t)c3[2] * dm[1] + c3[1]) * dm[0] + c3[0];
      kbeg = csr[l].off[cell]; kend = csr[l].off[cell + 1];
    } else { kbeg = goff[l]; kend = goff[l + 1]; }
    double y[3] = {0.0, 0.0, 0.0}, a[3] = {0.0, 0.0, 0.0};
    int amb = 0;
    for (int64_t k = kbeg; k < kend; ++k) {
      int64_t j = csr ? goff[l] + csr[l].idx[k] : k;
      double d[3], t[3];
      double Q = orc_Q(&gs[j], xi, d, t);
      double e = exp(-0.5 * Q);
      if (Q <= t2) for (int c = 0; c < 3; ++c) y[c] += gs[j].v[c] * e;
      if (isfinite(t2) && fabs(Q - t2) <= amb_rel * t2) { amb = 1; for (int c = 0; c < 3; ++c) a[c] += gs[j].v[c] * e; }
    }
    if (!amb && !cond) continue;
    na += amb;
    double k3 = 3.0 * (double)count[l], g[3], gam[3];
    for (int c = 0; c < 3; ++c) {
      double xh = rgb[3 * i + c], r = xh - y[c], dd = y[c] + hdr_eps;
      double dgdy;
      if (mode == 0) { g[c] = (-2.0 * r / (dd * dd)) / k3; dgdy = (2.0 / (dd * dd) + 4.0 * r / (dd * dd * dd)) / k3; }
      else {
        g[c] = (-2.0 * r * (xh + hdr_eps) / (dd * dd * dd)) / k3;
        dgdy = (2.0 * (xh + hdr_eps) / (dd * dd * dd) + 6.0 * r * (xh + hdr_eps) / (dd * dd * dd * dd)) / k3;
      }
      gam[c] = fabs(dgdy) * a[c];
    }
    for (int64_t k = kbeg; k < kend; ++k) {
      int64_t j = csr ? goff[l] + csr[l].idx[k] : k;
      double d[3], t[3];
      double Q = orc_Q(&gs[j], xi, d, t);
      int isamb = isfinite(t2) && fabs(Q - t2) <= amb_rel * t2;   /* tau = inf: no boundary */
      if (cond) { if (!(Q <= t2)) continue; }
      else if (!(Q <= t2) && !isamb) continue;
      double e = exp(-0.5 * Q), H = 0.0, gg[3];
      for (int c = 0; c < 3; ++c) {
        gg[c] = cond ? fabs(g[c]) : (isamb ? fabs(g[c]) + gam[c] : gam[c]);
        H += gg[c] * gs[j].v[c];
      }
      double* aj = allow_coef + 15 * j;
      for (int u = 0; u < 3; ++u) aj[u] += H * e * fabs(t[u]);
      for (int u = 0; u < 3; ++u)
        for (int w = 0; w < 3; ++w) aj[3 + 3 * u + w] += 0.5 * H * e * fabs(d[u] * d[w]);
      for (int c = 0; c < 3; ++c) aj[12 + c] += gg[c] * e;
    }
  }
  /* the chain rule of C5 with absolute values */
  for (int64_t j = 0; j < G; ++j) {
    const orc_gauss* gj = &gs[j];
    const double* aj = allow_coef + 15 * j;
    const double* p = P + j * NP;
    double* out = allow_raw + NP * j;
    for (int u = 0; u < 3; ++u) out[u] = aj[u];
    for (int k = 0; k < 3; ++k) {
      double acc = 0.0;
      for (int u = 0; u < 3; ++u)
        for (int w = 0; w < 3; ++w) acc += fabs(gj->R[u][k]) * aj[3 + 3 * u + w] * fabs(gj->R[w][k]);
      out[10 + k] = 2.0 * gj->D[k] * acc;
    }
    if (gj->degenerate) {
      for (int c = 0; c < 4; ++c) out[3 + c] = 0.0;
    } else {
      double dR[3][3], J[4][3][3], dqh[4], s = 0.0;
      for (int u = 0; u < 3; ++u)
        for (int b = 0; b < 3; ++b) {
          double acc = 0.0;
          for (int c = 0; c < 3; ++c) acc += aj[3 + 3 * u + c] * fabs(gj->R[c][b]);
          dR[u][b] = 2.0 * acc * gj->D[b];
        }
      orc_dRdq(gj->qhat, J);
      for (int c = 0; c < 4; ++c) {
        double acc = 0.0;
        for (int u = 0; u < 3; ++u) for (int b = 0; b < 3; ++b) acc += dR[u][b] * fabs(J[c][u][b]);
        dqh[c] = acc;
        s += fabs(gj->qhat[c]) * acc;
      }
      for (int c = 0; c < 4; ++c) out[3 + c] = (dqh[c] + fabs(gj->qhat[c]) * s) / gj->qnorm;
    }
    double dw = 0.0;
    for (int c = 0; c < 3; ++c) dw += aj[12 + c] * gj->chat[c];
    out[13] = dw * gj->w * (1.0 - gj->w);
    for (int c = 0; c < 3; ++c) out[7 + c] = p[7 + c] > 0.0 ? gj->w * aj[12 + c] : 0.0;
  }
  *n_amb = na;
  if (csr) { for (int l = 0; l < L; ++l) orc_csr_free(&csr[l]); free(csr); }
  free(count); free(lv); free(gs);
  return 0;
}
