/*
 * oracle/screen_oracle.c -- plain fp64 CPU oracle of the paper's SCREEN-SPACE cache read path
 * (next row f1 of SURVEY 8(f)): each cache level is "rasterized into images using the ...
 * Gaussian splatting rasterization technique" (sec.3.1, after Kerbl et al.), one image
 * per level, read by the path tracer at the pixel where a path of that length is terminated,
 * and fitted to the noisy per-level path radiance images with Eq. 4 (sec.3.5).
 *
 * TEST INFRASTRUCTURE ONLY (see gscache_oracle.c): loaded by tests/ only; shares no code with
 * paper_2507_19718_b200/.  Gradients of this path are defined as the derivative of this
 * forward: the tests take them by fp64 central finite differences of orc_image_loss.
 *
 * The rasterizer, step by step in the 3DGS order (readings A23 of DESIGN.md where the paper,
 * which defers to Kerbl et al., fixes nothing):
 *   activation (C1): Sigma = R diag(e^{2s}) R^T, w = sigmoid(o), chat = max(0, c)
 *   camera: t = Rv mu + tv (view = [Rv | tv], row-major 3x4, camera looks down +z); culled if
 *     t_z <= znear or the projected centre lies outside [-0.15 W, 1.15 W] x [-0.15 H, 1.15 H]
 *   centre: u = fx t_x / t_z + cx, v = fy t_y / t_z + cy (pixel (px, py) is sampled at
 *     (px + 0.5, py + 0.5))
 *   EWA: J = [[fx/t_z, 0, -fx t_x/t_z^2], [0, fy/t_z, -fy t_y/t_z^2]], T = J Rv,
 *     Sigma2 = T Sigma T^T + 0.3 I (low-pass), conic = Sigma2^{-1}; culled if det <= 0
 *   radius r = ceil(3 sqrt(lambda_max)), lambda_max = mid + sqrt(max(0.1, mid^2 - det))
 *   tiles 16 x 16: x0 = clamp(floor((u - r)/16), 0, TX), x1 = clamp(floor((u + r + 15)/16), 0, TX)
 *     (same for y); culled if the rectangle is empty.  A Gaussian reaches only the pixels of
 *     the tiles of its rectangle.
 *   per pixel, the Gaussians reaching it in (depth t_z, index) order, front to back:
 *     power = -(conic_a dx^2 + conic_c dy^2)/2 - conic_b dx dy, d = (u, v) - pixel;
 *     skip if power > 0; alpha = min(0.99, w e^{power}); skip if alpha < 1/255;
 *     T' = T (1 - alpha); stop if T' < 1e-4; C += chat alpha T; T = T'.
 *   background 0; the image holds C, and T is the final transmittance.
 * amb[pixel] = 1 when a discrete decision of that pixel is within a relative 1e-4 of its
 * threshold (alpha vs 1/255, T' vs 1e-4, a rectangle bound of a Gaussian reaching the pixel's
 * tile neighbourhood): there fp32 may take the other branch (reading A23, like A3).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NP 14

#include "gscache_oracle.h"

typedef struct {
  int W, H;
  double fx, fy, cx, cy;
  double view[12];
  double znear;
} orc_cam;

typedef struct {
  int ok;
  double u, v, depth, conic[3], w, chat[3];
  int x0, x1, y0, y1, rect_amb;
} orc_proj;

static int orc_clampi(double f, int hi) {
  if (!(f >= 0.0)) return 0;
  if (f > (double)hi) return hi;
  return (int)f;
}

/* the clamped tile range [lo, hi) of centre c and radius r3 (before the ceil) */
static void orc_rect(double c, double r3, int n, int* lo, int* hi) {
  const double r = ceil(r3);
  *lo = orc_clampi(floor((c - r) / 16.0), n);
  *hi = orc_clampi(floor((c + r + 15.0) / 16.0), n);
}

/* 1 if moving the centre or the radius by a relative 1e-4 changes the clamped range */
static int orc_rect_amb(double c, double r3, int n) {
  int lo, hi;
  orc_rect(c, r3, n, &lo, &hi);
  const double dc = 1e-4 * (fabs(c) > 1.0 ? fabs(c) : 1.0), dr = 1e-4 * r3;
  for (int a = -1; a <= 1; a += 2)
    for (int b = -1; b <= 1; b += 2) {
      int l2, h2;
      orc_rect(c + a * dc, r3 + b * dr, n, &l2, &h2);
      if (l2 != lo || h2 != hi) return 1;
    }
  return 0;
}

void orc_project(const double* p, const orc_cam* cam, double* out /* 16 doubles */) {
  orc_gauss g;
  orc_proj pr;
  memset(&pr, 0, sizeof pr);
  orc_activate_row(p, &g);
  const double* V = cam->view;
  double t[3];
  for (int a = 0; a < 3; ++a) t[a] = ((V[4 * a] * g.mu[0] + V[4 * a + 1] * g.mu[1]) + V[4 * a + 2] * g.mu[2]) + V[4 * a + 3];
  pr.ok = 0;
  if (t[2] > cam->znear) {
    const double u = cam->fx * t[0] / t[2] + cam->cx, v = cam->fy * t[1] / t[2] + cam->cy;
    if (u >= -0.15 * cam->W && u <= 1.15 * cam->W && v >= -0.15 * cam->H && v <= 1.15 * cam->H) {
      /* Sigma = R diag(e^{2s}) R^T */
      double S[3][3];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          double acc = 0.0;
          for (int k = 0; k < 3; ++k) acc += g.R[a][k] * exp(2.0 * p[10 + k]) * g.R[b][k];
          S[a][b] = acc;
        }
      const double J[2][3] = {{cam->fx / t[2], 0.0, -cam->fx * t[0] / (t[2] * t[2])},
                              {0.0, cam->fy / t[2], -cam->fy * t[1] / (t[2] * t[2])}};
      double T[2][3];
      for (int i = 0; i < 2; ++i)
        for (int b = 0; b < 3; ++b) T[i][b] = (J[i][0] * V[b] + J[i][1] * V[4 + b]) + J[i][2] * V[8 + b];
      double C2[2][2];
      for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 2; ++k) {
          double acc = 0.0;
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) acc += T[i][a] * S[a][b] * T[k][b];
          C2[i][k] = acc;
        }
      const double a_ = C2[0][0] + 0.3, b_ = C2[0][1], c_ = C2[1][1] + 0.3;
      const double det = a_ * c_ - b_ * b_;
      if (det > 0.0) {
        const double mid = 0.5 * (a_ + c_);
        const double disc = mid * mid - det;
        const double lam = mid + sqrt(disc > 0.1 ? disc : 0.1);
        const double r3 = 3.0 * sqrt(lam);
        const int TX = (cam->W + 15) / 16, TY = (cam->H + 15) / 16;
        orc_rect(u, r3, TX, &pr.x0, &pr.x1);
        orc_rect(v, r3, TY, &pr.y0, &pr.y1);
        pr.rect_amb = orc_rect_amb(u, r3, TX) || orc_rect_amb(v, r3, TY);
        if (pr.x0 < pr.x1 && pr.y0 < pr.y1) {
          pr.ok = 1;
          pr.u = u; pr.v = v; pr.depth = t[2];
          pr.conic[0] = c_ / det; pr.conic[1] = -b_ / det; pr.conic[2] = a_ / det;
          pr.w = g.w;
          for (int c = 0; c < 3; ++c) pr.chat[c] = g.chat[c];
        }
      }
    }
  }
  out[0] = pr.ok; out[1] = pr.u; out[2] = pr.v; out[3] = pr.depth;
  out[4] = pr.conic[0]; out[5] = pr.conic[1]; out[6] = pr.conic[2]; out[7] = pr.w;
  out[8] = pr.chat[0]; out[9] = pr.chat[1]; out[10] = pr.chat[2];
  out[11] = pr.x0; out[12] = pr.x1; out[13] = pr.y0; out[14] = pr.y1; out[15] = pr.rect_amb;
}

typedef struct { double depth; int64_t j; } orc_dk;
static int orc_dk_cmp(const void* a, const void* b) {
  const orc_dk* x = (const orc_dk*)a; const orc_dk* y = (const orc_dk*)b;
  if (x->depth < y->depth) return -1;
  if (x->depth > y->depth) return 1;
  return (x->j > y->j) - (x->j < y->j);
}

/* Render one level's n Gaussians (rows P[n][14]) into rgb [H][W][3] and T [H][W]; amb [H][W]
 * (nullable).  Only the pixels listed in `pix` ([npix] linear indices py*W+px) when pix !=
 * NULL (sampled checks at full size); the others are left untouched. */
int orc_render(int64_t n, const double* P, const orc_cam* cam, int64_t npix, const int64_t* pix,
               double* rgb, double* Tout, int32_t* amb) {
  double* pj = (double*)malloc(sizeof(double) * 16 * (size_t)(n > 0 ? n : 1));
  orc_dk* order = (orc_dk*)malloc(sizeof(orc_dk) * (size_t)(n > 0 ? n : 1));
  int64_t m = 0;
  for (int64_t j = 0; j < n; ++j) {
    orc_project(P + NP * j, cam, pj + 16 * j);
    if (pj[16 * j] != 0.0) { order[m].depth = pj[16 * j + 3]; order[m].j = j; ++m; }
  }
  qsort(order, (size_t)m, sizeof(orc_dk), orc_dk_cmp);
  const int64_t total = npix >= 0 && pix ? npix : (int64_t)cam->W * cam->H;
  for (int64_t k = 0; k < total; ++k) {
    const int64_t lin = pix ? pix[k] : k;
    const int px = (int)(lin % cam->W), py = (int)(lin / cam->W);
    const int tx = px / 16, ty = py / 16;
    const double fx = px + 0.5, fy = py + 0.5;
    double T = 1.0, C[3] = {0.0, 0.0, 0.0};
    int am = 0;
    for (int64_t q = 0; q < m; ++q) {
      const double* g = pj + 16 * order[q].j;
      const int x0 = (int)g[11], x1 = (int)g[12], y0 = (int)g[13], y1 = (int)g[14];
      if (g[15] != 0.0 && tx >= x0 - 1 && tx <= x1 && ty >= y0 - 1 && ty <= y1) am = 1;
      if (tx < x0 || tx >= x1 || ty < y0 || ty >= y1) continue;
      const double dx = g[1] - fx, dy = g[2] - fy;
      const double power = -0.5 * (g[4] * dx * dx + g[6] * dy * dy) - g[5] * dx * dy;
      if (power > 0.0) continue;
      const double a0 = g[7] * exp(power);
      const double alpha = a0 < 0.99 ? a0 : 0.99;
      if (fabs(alpha - 1.0 / 255.0) <= 1e-4 / 255.0) am = 1;
      if (alpha < 1.0 / 255.0) continue;
      const double Tn = T * (1.0 - alpha);
      if (fabs(Tn - 1e-4) <= 1e-8) am = 1;
      if (Tn < 1e-4) break;
      for (int c = 0; c < 3; ++c) C[c] += g[8 + c] * alpha * T;
      T = Tn;
    }
    for (int c = 0; c < 3; ++c) rgb[3 * lin + c] = C[c];
    if (Tout) Tout[lin] = T;
    if (amb) amb[lin] = am;
  }
  free(pj); free(order);
  return 0;
}

/* Eq. 4 on the per-level images: L = sum_l (1/(3 k_l)) sum_{valid px} sum_ch
 * (x - y)^2 / (d + eps)^2 with d = y (full quotient) or d = denom (a frozen image: the
 * stop-gradient reading A10, whose finite differences give the mode-0 gradient); k_l = valid
 * pixels of level l.  target, denom: [L][H][W][3]; valid: [L][H][W] bytes or NULL (all).
 * per_level [L] (nullable) receives each level's term. */
double orc_image_loss(int L, const int64_t* goff, const double* P, const orc_cam* cam, const double* target,
                      const uint8_t* valid, const double* denom, double hdr_eps, double* per_level) {
  const int64_t npx = (int64_t)cam->W * cam->H;
  double* img = (double*)malloc(sizeof(double) * 3 * (size_t)npx);
  double total = 0.0;
  for (int l = 0; l < L; ++l) {
    orc_render(goff[l + 1] - goff[l], P + NP * goff[l], cam, -1, NULL, img, NULL, NULL);
    double s = 0.0;
    int64_t k = 0;
    for (int64_t i = 0; i < npx; ++i) {
      if (valid && !valid[l * npx + i]) continue;
      ++k;
      for (int c = 0; c < 3; ++c) {
        const double y = img[3 * i + c], x = target[3 * (l * npx + i) + c];
        const double d = (denom ? denom[3 * (l * npx + i) + c] : y) + hdr_eps;
        s += (x - y) * (x - y) / (d * d);
      }
    }
    const double Ll = k > 0 ? s / (3.0 * (double)k) : 0.0;
    if (per_level) per_level[l] = Ll;
    total += Ll;
  }
  free(img);
  return total;
}
