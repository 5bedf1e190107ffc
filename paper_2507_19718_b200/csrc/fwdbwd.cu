// fwdbwd.cu -- the fused forward + HDR loss + backward kernel of gc_fit (A4) and the
// forward-only lookup kernel of gc_query (A7).
//
// One persistent CTA of 256 threads walks the work list; a work item is <= 256 samples of
// one (level, cell) bin.  The cell's culling list (C8) is gathered into shared memory as
// 48-byte evaluation records, 256 Gaussians per tile.
//   pass 1 (thread = sample): yhat = sum v_j e^{-Q/2} over the staged Gaussians with
//          Q <= tau^2 (C3), the Eq. 4 loss and g = dL/dyhat (C4, unnormalised; the 1/(3k_l)
//          factor is applied by the optimizer once k_l is known globally, C9);
//   pass 2 (thread = Gaussian x sample-split): the 12 coefficient-gradient terms of C5
//          accumulated in registers over the shared-memory samples, merged across the K
//          sample splits with __shfl_xor_sync, then 3 x red.global.add.v4.f32 per
//          (Gaussian, work item) that touched any sample -- never shared-memory float atomics.
#include "common.cuh"
#include "kernels.h"

namespace gsc {

constexpr int kPart = kMaxL + 2;
constexpr float kNegHalfLog2e = -0.72134752044448170f;   // -0.5 * log2(e)

__global__ void __launch_bounds__(256, 4) k_fwdbwd(FitArgs a) {
  __shared__ float4 s_r0[kTG], s_r1[kTG], s_r2[kTG];
  __shared__ int s_gid[kTG];
  __shared__ float s_x[kCH], s_y[kCH], s_z[kCH], s_g0[kCH], s_g1[kCH], s_g2[kCH];
  __shared__ float s_wl[8];
  __shared__ int s_wp[8];
  __shared__ double s_loss[kMaxL];
  __shared__ unsigned long long s_pairs, s_cand;

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t < kMaxL) s_loss[t] = 0.0;
  if (t == 0) { s_pairs = 0ull; s_cand = 0ull; }
  const uint32_t n_work = *a.n_work;
  const float tau2 = a.tau2, eps = a.hdr_eps;

  for (uint32_t w = blockIdx.x; w < n_work; w += gridDim.x) {
    const WorkItem wi = a.work[w];
    const int lo = (int)a.csr_off[wi.cell];
    const int C = (int)a.csr_off[wi.cell + 1] - lo;
    const int n = wi.count;
    const bool act = t < n;
    float x = 0.f, y = 0.f, z = 0.f, xr = 0.f, xg = 0.f, xb = 0.f;
    if (act) {
      const int si = wi.start + t;
      x = a.bx[si]; y = a.by[si]; z = a.bz[si];
      xr = a.br[si]; xg = a.bg[si]; xb = a.bb[si];
    }
    // ---------------- pass 1: thread = sample
    float y0 = 0.f, y1 = 0.f, y2 = 0.f;
    int np = 0;
    for (int tb = 0; tb < C; tb += kTG) {
      const int Ct = min(kTG, C - tb);
      __syncthreads();
      if (t < Ct) {
        const int gid = a.csr_idx[lo + tb + t];
        s_gid[t] = gid;
        s_r0[t] = __ldg(a.rec + 3 * gid); s_r1[t] = __ldg(a.rec + 3 * gid + 1); s_r2[t] = __ldg(a.rec + 3 * gid + 2);
      }
      __syncthreads();
      if (act) {
#pragma unroll 4
        for (int k = 0; k < Ct; ++k) {
          const float4 p = s_r0[k], q = s_r1[k], r = s_r2[k];
          const Rec g{p.x, p.y, p.z, p.w, q.x, q.y, q.z, q.w, r.x, r.y, r.z, r.w};
          float dx, dy, dz, tx, ty, tz;
          const float Q = quad_form(g, x, y, z, dx, dy, dz, tx, ty, tz);
          if (Q <= tau2) {
            const float e = ex2_approx(Q * kNegHalfLog2e);
            y0 = fmaf(g.v0, e, y0); y1 = fmaf(g.v1, e, y1); y2 = fmaf(g.v2, e, y2);
            ++np;
          }
        }
      }
    }
    // ---------------- Eq. 4 loss and dL/dyhat (unnormalised)
    float g0 = 0.f, g1 = 0.f, g2 = 0.f, ls = 0.f;
    if (act) {
      const float d0 = y0 + eps, d1 = y1 + eps, d2 = y2 + eps;
      const float r0 = xr - y0, r1 = xg - y1, r2 = xb - y2;
      const float i0 = 1.f / (d0 * d0), i1 = 1.f / (d1 * d1), i2 = 1.f / (d2 * d2);
      ls = r0 * r0 * i0 + r1 * r1 * i1 + r2 * r2 * i2;
      if (a.mode == 0) { g0 = -2.f * r0 * i0; g1 = -2.f * r1 * i1; g2 = -2.f * r2 * i2; }
      else {
        g0 = -2.f * r0 * (xr + eps) * i0 / d0; g1 = -2.f * r1 * (xg + eps) * i1 / d1;
        g2 = -2.f * r2 * (xb + eps) * i2 / d2;
      }
    }
    __syncthreads();
    s_x[t] = x; s_y[t] = y; s_z[t] = z; s_g0[t] = g0; s_g1[t] = g1; s_g2[t] = g2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ls += __shfl_xor_sync(0xffffffffu, ls, o);
      np += __shfl_xor_sync(0xffffffffu, np, o);
    }
    if (lane == 0) { s_wl[warp] = ls; s_wp[warp] = np; }
    __syncthreads();
    if (t == 0) {
      float bl = 0.f; int bp = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) { bl += s_wl[k]; bp += s_wp[k]; }
      s_loss[wi.level] += (double)bl;
      s_pairs += (unsigned long long)bp;
      s_cand += (unsigned long long)n * (unsigned long long)C;
    }
    // ---------------- pass 2: thread = (Gaussian jj, sample split sp)
    for (int tb = 0; tb < C; tb += kTG) {
      const int Ct = min(kTG, C - tb);
      if (C > kTG) {
        __syncthreads();
        if (t < Ct) {
          const int gid = a.csr_idx[lo + tb + t];
          s_gid[t] = gid;
          s_r0[t] = __ldg(a.rec + 3 * gid); s_r1[t] = __ldg(a.rec + 3 * gid + 1); s_r2[t] = __ldg(a.rec + 3 * gid + 2);
        }
        __syncthreads();
      }
      // K = number of sample splits per Gaussian: largest power of two with K * Ct <= 256, K <= 32
      int logK = 0;
      while (logK < 5 && (Ct << (logK + 1)) <= kCH) ++logK;
      const int K = 1 << logK;
      const int jj = t >> logK, sp = t & (K - 1);
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, a4 = 0.f, a5 = 0.f, a6 = 0.f, a7 = 0.f,
            a8 = 0.f, a9 = 0.f, a10 = 0.f, a11 = 0.f;
      bool touched = false;
      if (jj < Ct) {
        const float4 p = s_r0[jj], q = s_r1[jj], r = s_r2[jj];
        const Rec g{p.x, p.y, p.z, p.w, q.x, q.y, q.z, q.w, r.x, r.y, r.z, r.w};
        for (int s = sp; s < n; s += K) {
          float dx, dy, dz, tx, ty, tz;
          const float Q = quad_form(g, s_x[s], s_y[s], s_z[s], dx, dy, dz, tx, ty, tz);
          if (Q <= tau2) {
            const float e = ex2_approx(Q * kNegHalfLog2e);
            const float c0 = s_g0[s], c1 = s_g1[s], c2 = s_g2[s];
            const float he = (c0 * g.v0 + c1 * g.v1 + c2 * g.v2) * e;
            a0 = fmaf(he, tx, a0); a1 = fmaf(he, ty, a1); a2 = fmaf(he, tz, a2);   // d mu
            const float k = -0.5f * he;
            const float kx = k * dx, ky = k * dy, kz = k * dz;
            a3 = fmaf(kx, dx, a3); a4 = fmaf(ky, dy, a4); a5 = fmaf(kz, dz, a5);   // dA00 dA11 dA22
            a6 = fmaf(kx, dy, a6); a7 = fmaf(kx, dz, a7); a8 = fmaf(ky, dz, a8);   // dA01 dA02 dA12
            a9 = fmaf(c0, e, a9); a10 = fmaf(c1, e, a10); a11 = fmaf(c2, e, a11);  // d v
            touched = true;
          }
        }
      }
      for (int o = K >> 1; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o); a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o); a3 += __shfl_xor_sync(0xffffffffu, a3, o);
        a4 += __shfl_xor_sync(0xffffffffu, a4, o); a5 += __shfl_xor_sync(0xffffffffu, a5, o);
        a6 += __shfl_xor_sync(0xffffffffu, a6, o); a7 += __shfl_xor_sync(0xffffffffu, a7, o);
        a8 += __shfl_xor_sync(0xffffffffu, a8, o); a9 += __shfl_xor_sync(0xffffffffu, a9, o);
        a10 += __shfl_xor_sync(0xffffffffu, a10, o); a11 += __shfl_xor_sync(0xffffffffu, a11, o);
        touched = touched | (bool)__shfl_xor_sync(0xffffffffu, (int)touched, o);
      }
      if (sp == 0 && jj < Ct && touched) {
        float* gp = a.grad + 12 * (int64_t)s_gid[jj];
        red_add_v4(gp, a0, a1, a2, a3);
        red_add_v4(gp + 4, a4, a5, a6, a7);
        red_add_v4(gp + 8, a8, a9, a10, a11);
      }
    }
  }
  __syncthreads();
  double* part = a.partial + (int64_t)blockIdx.x * kPart;
  if (t < kMaxL) part[t] = s_loss[t];
  if (t == 0) { part[kMaxL] = (double)s_pairs; part[kMaxL + 1] = (double)s_cand; }
}

__global__ void __launch_bounds__(256, 4) k_query(QueryArgs a) {
  __shared__ float4 s_r0[kTG], s_r1[kTG], s_r2[kTG];
  const int t = threadIdx.x;
  const uint32_t n_work = *a.n_work;
  const float tau2 = a.tau2;
  for (uint32_t w = blockIdx.x; w < n_work; w += gridDim.x) {
    const WorkItem wi = a.work[w];
    const int lo = (int)a.csr_off[wi.cell];
    const int C = (int)a.csr_off[wi.cell + 1] - lo;
    const bool act = t < wi.count;
    float x = 0.f, y = 0.f, z = 0.f;
    if (act) { const int si = wi.start + t; x = a.bx[si]; y = a.by[si]; z = a.bz[si]; }
    float y0 = 0.f, y1 = 0.f, y2 = 0.f;
    for (int tb = 0; tb < C; tb += kTG) {
      const int Ct = min(kTG, C - tb);
      __syncthreads();
      if (t < Ct) {
        const int gid = a.csr_idx[lo + tb + t];
        s_r0[t] = __ldg(a.rec + 3 * gid); s_r1[t] = __ldg(a.rec + 3 * gid + 1); s_r2[t] = __ldg(a.rec + 3 * gid + 2);
      }
      __syncthreads();
      if (act) {
#pragma unroll 4
        for (int k = 0; k < Ct; ++k) {
          const float4 p = s_r0[k], q = s_r1[k], r = s_r2[k];
          const Rec g{p.x, p.y, p.z, p.w, q.x, q.y, q.z, q.w, r.x, r.y, r.z, r.w};
          float dx, dy, dz, tx, ty, tz;
          const float Q = quad_form(g, x, y, z, dx, dy, dz, tx, ty, tz);
          if (Q <= tau2) {
            const float e = ex2_approx(Q * kNegHalfLog2e);
            y0 = fmaf(g.v0, e, y0); y1 = fmaf(g.v1, e, y1); y2 = fmaf(g.v2, e, y2);
          }
        }
      }
    }
    if (act) {
      const uint32_t i = a.bidx[wi.start + t];
      a.out[3 * (int64_t)i] = y0; a.out[3 * (int64_t)i + 1] = y1; a.out[3 * (int64_t)i + 2] = y2;
    }
  }
}

static int persistent_grid(const void* fn) {
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 256, 0);
  return sms * std::max(per, 1);
}

int fwdbwd_grid() { static int g = persistent_grid((const void*)k_fwdbwd); return g; }
int query_grid() { static int g = persistent_grid((const void*)k_query); return g; }

void launch_fwdbwd(const FitArgs& a, int grid, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, "fwdbwd", s);
  k_fwdbwd<<<grid, 256, 0, s>>>(a);
}

void launch_query(const QueryArgs& a, int grid, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, "query_fwd", s);
  k_query<<<grid, 256, 0, s>>>(a);
}

}  // namespace gsc
