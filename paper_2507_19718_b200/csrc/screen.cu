// screen.cu -- the paper's screen-space cache read / train path (next row f1 of SURVEY 8(f)):
// every cache level is rasterized into an image with the 3D Gaussian splatting rasterizer
// (sec.3.1, after Kerbl et al.) and fitted to the per-level noisy path-radiance images
// with Eq. 4 (sec.3.5), sharing the parameter store (A2) and the optimizer (A6)
// with the world-space path.  All levels are rasterized in ONE pass over a joint
// (level, tile)-keyed list -- the "joint rasterization and optimization pipeline" the paper
// names as future work (sec.5).  Readings A23; the oracle is
// oracle/screen_oracle.c.
//
// Pipeline of gc_render / gc_fit_image:
//   k_sproject   per Gaussian: EWA projection, conic, radius, tile rectangle, tiles touched
//   scan         exclusive offsets of the tiles touched (3 small kernels)
//   k_skeys      (level * tiles + tile) << 32 | depth bits  ->  Gaussian index
//   sort         bitonic (key, index): per tile, depth order, ties by index
//   k_sranges    [start, end) of every (level, tile)
//   k_sraster    one CTA per (tile, level), 16 x 16 threads, batches of 256 Gaussians staged in
//                shared memory, front-to-back compositing; C, final T, last contributor
//   gc_fit_image adds k_sloss (Eq. 4 terms + dL/dC, level statistics), k_sraster_bwd (back to
//                front, per-Gaussian transposing warp reductions, then float reds) and
//                k_sproject_bwd (EWA / projection chain rule to the 14 raw parameters), then
//                the shared AdamW (raw-gradient mode) and the culling rebuild.
#include "common.cuh"
#include "kernels.h"
#include "stats.cuh"

namespace gsc {

constexpr int kTile = 16;
constexpr int kTileThreads = kTile * kTile;

SCam make_scam(const gc_camera& c) {
  SCam s;
  s.W = c.width; s.H = c.height; s.TX = (c.width + kTile - 1) / kTile; s.TY = (c.height + kTile - 1) / kTile;
  s.fx = c.fx; s.fy = c.fy; s.cx = c.cx; s.cy = c.cy; s.znear = c.znear;
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) s.R[3 * a + b] = c.view[4 * a + b];
    s.t[a] = c.view[4 * a + 3];
  }
  return s;
}

__device__ __forceinline__ void quat_rot(float w, float x, float y, float z, float R[3][3]) {
  R[0][0] = 1.f - 2.f * (y * y + z * z); R[0][1] = 2.f * (x * y - w * z); R[0][2] = 2.f * (x * z + w * y);
  R[1][0] = 2.f * (x * y + w * z); R[1][1] = 1.f - 2.f * (x * x + z * z); R[1][2] = 2.f * (y * z - w * x);
  R[2][0] = 2.f * (x * z - w * y); R[2][1] = 2.f * (y * z + w * x); R[2][2] = 1.f - 2.f * (x * x + y * y);
}

__device__ __forceinline__ int clamp_tile(float f, int n) {
  if (!(f >= 0.f)) return 0;
  if (f > (float)n) return n;
  return (int)f;
}

// --------------------------------------------------------------------------- projection
// pa = (u, v, depth, w), pb = (conic a, b, c, -), pc = (chat, ok), rect = (x0, x1, y0, y1)
__global__ void k_sproject(const float* __restrict__ P, int64_t G, int64_t g0, int64_t g1, SCam cam,
                           float4* pa, float4* pb, float4* pc, int4* rect, uint32_t* touched) {
  for (int64_t j = g0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < g1; j += (int64_t)gridDim.x * blockDim.x) {
    uint32_t n = 0;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a, c = a;
    int4 r = make_int4(0, 0, 0, 0);
    const float mx = P[P_MU * G + j], my = P[(P_MU + 1) * G + j], mz = P[(P_MU + 2) * G + j];
    const float tx = cam.R[0] * mx + cam.R[1] * my + cam.R[2] * mz + cam.t[0];
    const float ty = cam.R[3] * mx + cam.R[4] * my + cam.R[5] * mz + cam.t[1];
    const float tz = cam.R[6] * mx + cam.R[7] * my + cam.R[8] * mz + cam.t[2];
    if (tz > cam.znear) {
      const float u = cam.fx * tx / tz + cam.cx, v = cam.fy * ty / tz + cam.cy;
      if (u >= -0.15f * cam.W && u <= 1.15f * cam.W && v >= -0.15f * cam.H && v <= 1.15f * cam.H) {
        float qw = P[P_Q * G + j], qx = P[(P_Q + 1) * G + j], qy = P[(P_Q + 2) * G + j], qz = P[(P_Q + 3) * G + j];
        const float n2 = qw * qw + qx * qx + qy * qy + qz * qz;
        if (n2 < 1e-24f) { qw = 1.f; qx = qy = qz = 0.f; }
        else { const float in = rsqrtf(n2); qw *= in; qx *= in; qy *= in; qz *= in; }
        float R[3][3];
        quat_rot(qw, qx, qy, qz, R);
        const float e2[3] = {expf(2.f * P[P_S * G + j]), expf(2.f * P[(P_S + 1) * G + j]), expf(2.f * P[(P_S + 2) * G + j])};
        // T = J Rv (2 x 3), then T R (2 x 3), Sigma2 = (T R) diag(e^{2s}) (T R)^T + 0.3 I
        const float j00 = cam.fx / tz, j02 = -cam.fx * tx / (tz * tz), j11 = cam.fy / tz, j12 = -cam.fy * ty / (tz * tz);
        float T[2][3];
        for (int bcol = 0; bcol < 3; ++bcol) {
          T[0][bcol] = j00 * cam.R[bcol] + j02 * cam.R[6 + bcol];
          T[1][bcol] = j11 * cam.R[3 + bcol] + j12 * cam.R[6 + bcol];
        }
        float TR[2][3];
        for (int i = 0; i < 2; ++i)
          for (int k = 0; k < 3; ++k) TR[i][k] = T[i][0] * R[0][k] + T[i][1] * R[1][k] + T[i][2] * R[2][k];
        const float A = TR[0][0] * TR[0][0] * e2[0] + TR[0][1] * TR[0][1] * e2[1] + TR[0][2] * TR[0][2] * e2[2] + 0.3f;
        const float B = TR[0][0] * TR[1][0] * e2[0] + TR[0][1] * TR[1][1] * e2[1] + TR[0][2] * TR[1][2] * e2[2];
        const float Cc = TR[1][0] * TR[1][0] * e2[0] + TR[1][1] * TR[1][1] * e2[1] + TR[1][2] * TR[1][2] * e2[2] + 0.3f;
        const float det = A * Cc - B * B;
        if (det > 0.f) {
          const float mid = 0.5f * (A + Cc);
          const float lam = mid + sqrtf(fmaxf(0.1f, mid * mid - det));
          const float rad = ceilf(3.f * sqrtf(lam));
          r.x = clamp_tile(floorf((u - rad) / kTile), cam.TX); r.y = clamp_tile(floorf((u + rad + 15.f) / kTile), cam.TX);
          r.z = clamp_tile(floorf((v - rad) / kTile), cam.TY); r.w = clamp_tile(floorf((v + rad + 15.f) / kTile), cam.TY);
          if (r.x < r.y && r.z < r.w) {
            n = (uint32_t)((r.y - r.x) * (r.w - r.z));
            const float id = 1.f / det;
            const float w = 1.f / (1.f + expf(-P[P_O * G + j]));
            a = make_float4(u, v, tz, w);
            b = make_float4(Cc * id, -B * id, A * id, 0.f);
            c = make_float4(fmaxf(P[P_C * G + j], 0.f), fmaxf(P[(P_C + 1) * G + j], 0.f), fmaxf(P[(P_C + 2) * G + j], 0.f), 1.f);
          }
        }
      }
    }
    pa[j] = a; pb[j] = b; pc[j] = c; rect[j] = r;
    touched[j - g0] = n;
  }
}

// --------------------------------------------------------------------------- scan (uint32)
constexpr int kScanB = 1024, kScanPer = 4, kScanChunk = kScanB * kScanPer;

__device__ __forceinline__ uint32_t block_scan_excl(uint32_t v, uint32_t* total) {
  __shared__ uint32_t ws[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = v;
  for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += y; }
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    uint32_t x = ws[lane];
    for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
    ws[lane] = x;
  }
  __syncthreads();
  const uint32_t before = (w > 0 ? ws[w - 1] : 0u) + inc - v;
  *total = ws[31];
  __syncthreads();
  return before;
}

__global__ void __launch_bounds__(kScanB) k_sscan_blocks(const uint32_t* __restrict__ in, int64_t n, uint32_t* sums) {
  const int64_t base = (int64_t)blockIdx.x * kScanChunk + threadIdx.x * kScanPer;
  uint32_t s = 0;
  for (int k = 0; k < kScanPer; ++k) s += base + k < n ? in[base + k] : 0u;
  uint32_t tot;
  block_scan_excl(s, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanB) k_sscan_top(uint32_t* sums, int nb, uint32_t* total) {
  uint32_t carry = 0;
  for (int b0 = 0; b0 < nb; b0 += kScanB) {
    const int i = b0 + threadIdx.x;
    const uint32_t v = i < nb ? sums[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_scan_excl(v, &tot);
    if (i < nb) sums[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kScanB) k_sscan_apply(const uint32_t* __restrict__ in, int64_t n,
                                                        const uint32_t* __restrict__ sums, uint32_t* out) {
  const int64_t base = (int64_t)blockIdx.x * kScanChunk + threadIdx.x * kScanPer;
  uint32_t v[kScanPer], s = 0;
  for (int k = 0; k < kScanPer; ++k) { v[k] = base + k < n ? in[base + k] : 0u; s += v[k]; }
  uint32_t tot;
  uint32_t off = sums[blockIdx.x] + block_scan_excl(s, &tot);
  for (int k = 0; k < kScanPer; ++k) if (base + k < n) { out[base + k] = off; off += v[k]; }
}

// exclusive scan of n u32 (bsums: >= n / 4096 + 2 words, total: 1 word), deterministic
void launch_scan_u32(const uint32_t* in, int64_t n, uint32_t* bsums, uint32_t* total, uint32_t* out, cudaStream_t s) {
  const int nb = (int)((n + kScanChunk - 1) / kScanChunk);
  k_sscan_blocks<<<std::max(nb, 1), kScanB, 0, s>>>(in, n, bsums);
  k_sscan_top<<<1, kScanB, 0, s>>>(bsums, nb, total);
  k_sscan_apply<<<std::max(nb, 1), kScanB, 0, s>>>(in, n, bsums, out);
}

// --------------------------------------------------------------------------- keys / ranges
__global__ void k_skeys(int64_t g0, int64_t g1, LevelGeom g, int lev0, int ntiles_img, int TX,
                        const float4* __restrict__ pa, const int4* __restrict__ rect,
                        const uint32_t* __restrict__ off, uint64_t* key, int64_t* val) {
  for (int64_t j = g0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < g1; j += (int64_t)gridDim.x * blockDim.x) {
    const int4 r = rect[j];
    if (!(r.x < r.y && r.z < r.w)) continue;
    const int l = level_of_gaussian(g, j) - lev0;
    const uint32_t dbits = __float_as_uint(pa[j].z);     // depth > znear > 0: bits order like values
    uint32_t o = off[j - g0];
    for (int ty = r.z; ty < r.w; ++ty)
      for (int tx = r.x; tx < r.y; ++tx) {
        const uint64_t tile = (uint64_t)l * ntiles_img + (uint64_t)ty * TX + tx;
        key[o] = (tile << 32) | dbits;
        val[o] = j;
        ++o;
      }
  }
}

__global__ void k_sranges(const uint64_t* __restrict__ key, int64_t n, uint2* ranges) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(key[i] >> 32);
    if (i == 0 || (uint32_t)(key[i - 1] >> 32) != t) ranges[t].x = (uint32_t)i;
    if (i == n - 1 || (uint32_t)(key[i + 1] >> 32) != t) ranges[t].y = (uint32_t)(i + 1);
  }
}

// --------------------------------------------------------------------------- raster forward
struct SRasterArgs {
  const uint2* ranges; const int64_t* val;
  const float4 *pa, *pb, *pc;
  float* out;           // [Lr][H][W][3]
  float* outT;          // [Lr][H][W] (nullable)
  uint32_t* last;       // [Lr][H][W] last contributor count (nullable)
  SCam cam;
};

__global__ void __launch_bounds__(kTileThreads) k_sraster(SRasterArgs a) {
  __shared__ float2 s_uv[kTileThreads];
  __shared__ float4 s_co[kTileThreads];     // conic a, b, c, w
  __shared__ float4 s_c[kTileThreads];
  const int tile = blockIdx.x, l = blockIdx.y;
  const int ntiles = a.cam.TX * a.cam.TY;
  const int tx = tile % a.cam.TX, ty = tile / a.cam.TX;
  const int px = tx * kTile + (threadIdx.x % kTile), py = ty * kTile + (threadIdx.x / kTile);
  const bool inside = px < a.cam.W && py < a.cam.H;
  const float fx = px + 0.5f, fy = py + 0.5f;
  const uint2 rg = a.ranges[(size_t)l * ntiles + tile];
  const int n = rg.y > rg.x ? (int)(rg.y - rg.x) : 0;
  bool done = !inside;
  float T = 1.f, C0 = 0.f, C1 = 0.f, C2 = 0.f;
  uint32_t contributor = 0, last = 0;
  for (int b0 = 0; b0 < n; b0 += kTileThreads) {
    if (__syncthreads_count(done) == kTileThreads) break;
    const int q = b0 + threadIdx.x;
    if (q < n) {
      const int64_t j = a.val[rg.x + q];
      const float4 p = a.pa[j];
      s_uv[threadIdx.x] = make_float2(p.x, p.y);
      const float4 b = a.pb[j];
      s_co[threadIdx.x] = make_float4(b.x, b.y, b.z, p.w);
      s_c[threadIdx.x] = a.pc[j];
    }
    __syncthreads();
    const int m = min(kTileThreads, n - b0);
    for (int k = 0; !done && k < m; ++k) {
      ++contributor;
      const float2 uv = s_uv[k];
      const float4 co = s_co[k];
      const float dx = uv.x - fx, dy = uv.y - fy;
      const float power = -0.5f * (co.x * dx * dx + co.z * dy * dy) - co.y * dx * dy;
      if (power > 0.f) continue;
      const float alpha = fminf(0.99f, co.w * __expf(power));
      if (alpha < 1.f / 255.f) continue;
      const float Tn = T * (1.f - alpha);
      if (Tn < 1e-4f) { done = true; break; }
      const float4 c = s_c[k];
      const float wgt = alpha * T;
      C0 += c.x * wgt; C1 += c.y * wgt; C2 += c.z * wgt;
      T = Tn;
      last = contributor;
    }
  }
  if (inside) {
    const size_t pix = ((size_t)l * a.cam.H + py) * a.cam.W + px;
    a.out[3 * pix] = C0; a.out[3 * pix + 1] = C1; a.out[3 * pix + 2] = C2;
    if (a.outT) a.outT[pix] = T;
    if (a.last) a.last[pix] = last;
  }
}

// --------------------------------------------------------------------------- Eq. 4 on images
// dLdC = d/dy of sum_ch (x - y)^2 / (y + eps)^2 with the denominator frozen (mode 0, reading
// A10) or the full quotient (mode 1); the 1/(3 k_l) normalisation is applied by AdamW (inv3k).
// Per-level loss sums and valid-pixel counts go to the kSlots fp64 partials (k_stats layout).
__global__ void k_sloss(const float* __restrict__ img, const float* __restrict__ target,
                        const uint8_t* __restrict__ valid, int Lr, int64_t npx, float eps, int mode,
                        float* dLdC, double* partial) {
  const int l = blockIdx.y;
  double ls = 0.0, cnt = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npx; i += (int64_t)gridDim.x * blockDim.x) {
    const size_t p = (size_t)l * npx + i;
    const bool ok = !valid || valid[p];
    float g[3] = {0.f, 0.f, 0.f};
    if (ok) {
      cnt += 1.0;
      for (int c = 0; c < 3; ++c) {
        const float y = img[3 * p + c], x = target[3 * p + c];
        const float r = x - y, d = y + eps;
        ls += (double)(r * r / (d * d));
        g[c] = mode == 0 ? -2.f * r / (d * d) : -2.f * r * (x + eps) / (d * d * d);
      }
    }
    dLdC[3 * p] = g[0]; dLdC[3 * p + 1] = g[1]; dLdC[3 * p + 2] = g[2];
  }
  for (int o = 16; o > 0; o >>= 1) { ls += __shfl_xor_sync(0xffffffffu, ls, o); cnt += __shfl_xor_sync(0xffffffffu, cnt, o); }
  if ((threadIdx.x & 31) == 0) {
    double* slot = partial + (size_t)(blockIdx.x % kSlots) * kPart;
    atomicAdd(slot + l, ls);
    atomicAdd(slot + kMaxL + l, cnt);
  }
}

// --------------------------------------------------------------------------- raster backward
// Back to front over each pixel's accepted Gaussians (T recovered by division, alpha <= 0.99):
//   dC/dchat = alpha T, dC/dalpha = T (chat - behind), alpha = min(0.99, w G), G = e^power,
//   power = -(a dx^2 + c dy^2)/2 - b dx dy, dx = u - px, dy = v - py.
// Per Gaussian and warp the 9 partials (du, dv, da, db, dc, dw, dchat) are summed with
// shuffles, then one red.global.add.v4.f32 x 3 per warp into g2d[j] (12 floats).
struct SBwdArgs {
  const uint2* ranges; const int64_t* val;
  const float4 *pa, *pb, *pc;
  const float* outT; const uint32_t* last; const float* dLdC;
  float* g2d;           // [G][12]: du dv da db | dc dw dc0 dc1 | dc2 - - -
  SCam cam;
};

__global__ void __launch_bounds__(kTileThreads) k_sraster_bwd(SBwdArgs a) {
  __shared__ float2 s_uv[kTileThreads];
  __shared__ float4 s_co[kTileThreads];
  __shared__ float4 s_c[kTileThreads];
  __shared__ int64_t s_j[kTileThreads];
  const int tile = blockIdx.x, l = blockIdx.y;
  const int ntiles = a.cam.TX * a.cam.TY;
  const int tx = tile % a.cam.TX, ty = tile / a.cam.TX;
  const int px = tx * kTile + (threadIdx.x % kTile), py = ty * kTile + (threadIdx.x / kTile);
  const bool inside = px < a.cam.W && py < a.cam.H;
  const float fx = px + 0.5f, fy = py + 0.5f;
  const uint2 rg = a.ranges[(size_t)l * ntiles + tile];
  const int n = rg.y > rg.x ? (int)(rg.y - rg.x) : 0;
  const size_t pix = ((size_t)l * a.cam.H + min(py, a.cam.H - 1)) * a.cam.W + min(px, a.cam.W - 1);
  float T = inside ? a.outT[pix] : 1.f;
  const uint32_t lastc = inside ? a.last[pix] : 0u;
  const float g0 = inside ? a.dLdC[3 * pix] : 0.f, g1 = inside ? a.dLdC[3 * pix + 1] : 0.f,
              g2 = inside ? a.dLdC[3 * pix + 2] : 0.f;
  float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f;        // colour behind (normalised)
  float la = 0.f, lc0 = 0.f, lc1 = 0.f, lc2 = 0.f; // last processed (behind) Gaussian
  uint32_t contributor = (uint32_t)n;
  const int lane = threadIdx.x & 31;
  for (int b1 = n; b1 > 0; b1 -= kTileThreads) {
    const int b0 = max(0, b1 - kTileThreads);
    __syncthreads();
    const int q = b0 + threadIdx.x;
    if (q < b1) {
      const int64_t j = a.val[rg.x + q];
      const float4 p = a.pa[j];
      s_uv[threadIdx.x] = make_float2(p.x, p.y);
      const float4 b = a.pb[j];
      s_co[threadIdx.x] = make_float4(b.x, b.y, b.z, p.w);
      s_c[threadIdx.x] = a.pc[j];
      s_j[threadIdx.x] = j;
    }
    __syncthreads();
    for (int k = b1 - b0 - 1; k >= 0; --k) {
      float d[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      bool use = false;
      if (inside && contributor-- <= lastc) {
        const float2 uv = s_uv[k];
        const float4 co = s_co[k];
        const float dx = uv.x - fx, dy = uv.y - fy;
        const float power = -0.5f * (co.x * dx * dx + co.z * dy * dy) - co.y * dx * dy;
        if (power <= 0.f) {
          const float G = __expf(power);
          const float a0 = co.w * G;
          const float alpha = fminf(0.99f, a0);
          if (alpha >= 1.f / 255.f) {
            use = true;
            T = T / (1.f - alpha);
            const float4 c = s_c[k];
            const float wgt = alpha * T;
            d[6] = wgt * g0; d[7] = wgt * g1; d[8] = wgt * g2;                  // dL/dchat
            acc0 = la * lc0 + (1.f - la) * acc0;
            acc1 = la * lc1 + (1.f - la) * acc1;
            acc2 = la * lc2 + (1.f - la) * acc2;
            la = alpha; lc0 = c.x; lc1 = c.y; lc2 = c.z;
            const float dLda = T * ((c.x - acc0) * g0 + (c.y - acc1) * g1 + (c.z - acc2) * g2);
            if (a0 < 0.99f) {
              d[5] = dLda * G;                                                  // dL/dw
              const float dLdp = dLda * co.w * G;                               // dL/dpower
              d[0] = -dLdp * (co.x * dx + co.y * dy);                           // dL/du
              d[1] = -dLdp * (co.z * dy + co.y * dx);                           // dL/dv
              d[2] = -0.5f * dLdp * dx * dx;                                    // dL/dconic_a
              d[3] = -dLdp * dx * dy;                                           // dL/dconic_b
              d[4] = -0.5f * dLdp * dy * dy;                                    // dL/dconic_c
            }
          }
        }
      }
      // per-warp reduction, then one vector red per warp (skipped when no lane contributed)
      if (__any_sync(0xffffffffu, use)) {
        // transposing reduction of d[0..7] (each level keeps half of the values and sends the
        // other half: 4 + 2 + 1 shuffles, then 2 plain levels) -- lane L ends with the sum of
        // value 4 bit4(L) + 2 bit3(L) + bit2(L) when L % 4 == 0; d[8] by a plain tree.
        // (A/B: fit_image 1470 -> 1342 us at 1080p against 9 plain 5-level trees.)
        const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
        float t4[4], t2[2], t1;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float keep = h16 ? d[4 + i] : d[i], send = h16 ? d[i] : d[4 + i];
          t4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const float keep = h8 ? t4[2 + i] : t4[i], send = h8 ? t4[i] : t4[2 + i];
          t2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
        {
          const float keep = h4 ? t2[1] : t2[0], send = h4 ? t2[0] : t2[1];
          t1 = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        t1 += __shfl_xor_sync(0xffffffffu, t1, 2);
        t1 += __shfl_xor_sync(0xffffffffu, t1, 1);
        float d8 = d[8];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d8 += __shfl_xor_sync(0xffffffffu, d8, o);
        float* gj = a.g2d + 12 * s_j[k];
        if ((lane & 3) == 0) atomicAdd(gj + (h16 ? 4 : 0) + (h8 ? 2 : 0) + (h4 ? 1 : 0), t1);
        if (lane == 0) atomicAdd(gj + 8, d8);
      }
    }
  }
}

// --------------------------------------------------------------------------- projection bwd
// From g2d (du, dv, dconic, dw, dchat) to the raw 14-parameter gradient (unnormalised sums):
// conic = Sigma2^{-1} -> dSigma2 = -K dK K; Sigma2 = T Sigma T^T + 0.3 I with T = J Rv ->
// dSigma = T^T dSigma2 T, dT = 2 dSigma2 T Sigma, dJ = dT Rv^T -> dt (camera-space mean, with
// the centre's own du/dt, dv/dt) -> dmu = Rv^T dt; Sigma = M M^T, M = R diag(e^s) -> ds, dR ->
// dq through dR/dq_hat (C5) and the normalisation; dw -> do = dw w (1-w); dchat -> dc [c > 0].
// Zeroes the g2d slots it consumes.
__global__ void k_sproject_bwd(const float* __restrict__ P, int64_t G, int64_t g0, int64_t g1, SCam cam,
                               const float4* __restrict__ pc, float* g2d, float* raw) {
  for (int64_t j = g0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < g1; j += (int64_t)gridDim.x * blockDim.x) {
    float4* gp = reinterpret_cast<float4*>(g2d + 12 * j);
    const float4 q0 = gp[0], q1 = gp[1], q2 = gp[2];
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    gp[0] = z; gp[1] = z; gp[2] = z;
    float out[kNP];
    for (int k = 0; k < kNP; ++k) out[k] = 0.f;
    if (pc[j].w != 0.f) {
      const float du = q0.x, dv = q0.y, dca = q0.z, dcb = q0.w, dcc = q1.x, dw = q1.y;
      const float dch[3] = {q1.z, q1.w, q2.x};
      const float mx = P[P_MU * G + j], my = P[(P_MU + 1) * G + j], mz = P[(P_MU + 2) * G + j];
      const float tx = cam.R[0] * mx + cam.R[1] * my + cam.R[2] * mz + cam.t[0];
      const float ty = cam.R[3] * mx + cam.R[4] * my + cam.R[5] * mz + cam.t[1];
      const float tz = cam.R[6] * mx + cam.R[7] * my + cam.R[8] * mz + cam.t[2];
      const float qw0 = P[P_Q * G + j], qx0 = P[(P_Q + 1) * G + j], qy0 = P[(P_Q + 2) * G + j], qz0 = P[(P_Q + 3) * G + j];
      const float n2 = qw0 * qw0 + qx0 * qx0 + qy0 * qy0 + qz0 * qz0;
      const bool deg = n2 < 1e-24f;
      const float qn = sqrtf(n2);
      float w = 1.f, x = 0.f, y = 0.f, zq = 0.f;
      if (!deg) { w = qw0 / qn; x = qx0 / qn; y = qy0 / qn; zq = qz0 / qn; }
      float R[3][3];
      quat_rot(w, x, y, zq, R);
      const float es[3] = {expf(P[P_S * G + j]), expf(P[(P_S + 1) * G + j]), expf(P[(P_S + 2) * G + j])};
      float M[3][3], Sg[3][3];
      for (int a_ = 0; a_ < 3; ++a_)
        for (int k = 0; k < 3; ++k) M[a_][k] = R[a_][k] * es[k];
      for (int a_ = 0; a_ < 3; ++a_)
        for (int b_ = 0; b_ < 3; ++b_) Sg[a_][b_] = M[a_][0] * M[b_][0] + M[a_][1] * M[b_][1] + M[a_][2] * M[b_][2];
      const float j00 = cam.fx / tz, j02 = -cam.fx * tx / (tz * tz), j11 = cam.fy / tz, j12 = -cam.fy * ty / (tz * tz);
      float T[2][3];
      for (int b_ = 0; b_ < 3; ++b_) {
        T[0][b_] = j00 * cam.R[b_] + j02 * cam.R[6 + b_];
        T[1][b_] = j11 * cam.R[3 + b_] + j12 * cam.R[6 + b_];
      }
      // Sigma2 and K = Sigma2^-1
      float TS[2][3];
      for (int i = 0; i < 2; ++i)
        for (int b_ = 0; b_ < 3; ++b_) TS[i][b_] = T[i][0] * Sg[0][b_] + T[i][1] * Sg[1][b_] + T[i][2] * Sg[2][b_];
      const float A = TS[0][0] * T[0][0] + TS[0][1] * T[0][1] + TS[0][2] * T[0][2] + 0.3f;
      const float B = TS[0][0] * T[1][0] + TS[0][1] * T[1][1] + TS[0][2] * T[1][2];
      const float Cc = TS[1][0] * T[1][0] + TS[1][1] * T[1][1] + TS[1][2] * T[1][2] + 0.3f;
      const float id = 1.f / (A * Cc - B * B);
      const float K[2][2] = {{Cc * id, -B * id}, {-B * id, A * id}};
      const float dK[2][2] = {{dca, 0.5f * dcb}, {0.5f * dcb, dcc}};
      // dS2 = -K dK K (symmetric)
      float KdK[2][2], dS2[2][2];
      for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 2; ++k) KdK[i][k] = K[i][0] * dK[0][k] + K[i][1] * dK[1][k];
      for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 2; ++k) dS2[i][k] = -(KdK[i][0] * K[0][k] + KdK[i][1] * K[1][k]);
      // dSigma = T^T dS2 T ; dT = 2 dS2 T Sigma
      float dSg[3][3];
      for (int a_ = 0; a_ < 3; ++a_)
        for (int b_ = 0; b_ < 3; ++b_) {
          float acc = 0.f;
          for (int i = 0; i < 2; ++i)
            for (int k = 0; k < 2; ++k) acc += T[i][a_] * dS2[i][k] * T[k][b_];
          dSg[a_][b_] = acc;
        }
      float dT[2][3];
      for (int i = 0; i < 2; ++i)
        for (int b_ = 0; b_ < 3; ++b_) dT[i][b_] = 2.f * (dS2[i][0] * TS[0][b_] + dS2[i][1] * TS[1][b_]);
      // dJ = dT Rv^T (only the nonzero entries of J matter)
      const float dJ00 = dT[0][0] * cam.R[0] + dT[0][1] * cam.R[1] + dT[0][2] * cam.R[2];
      const float dJ02 = dT[0][0] * cam.R[6] + dT[0][1] * cam.R[7] + dT[0][2] * cam.R[8];
      const float dJ11 = dT[1][0] * cam.R[3] + dT[1][1] * cam.R[4] + dT[1][2] * cam.R[5];
      const float dJ12 = dT[1][0] * cam.R[6] + dT[1][1] * cam.R[7] + dT[1][2] * cam.R[8];
      const float iz = 1.f / tz, iz2 = iz * iz, iz3 = iz2 * iz;
      float dtx = du * cam.fx * iz + dJ02 * (-cam.fx * iz2);
      float dty = dv * cam.fy * iz + dJ12 * (-cam.fy * iz2);
      float dtz = -du * cam.fx * tx * iz2 - dv * cam.fy * ty * iz2 + dJ00 * (-cam.fx * iz2) +
                  dJ02 * (2.f * cam.fx * tx * iz3) + dJ11 * (-cam.fy * iz2) + dJ12 * (2.f * cam.fy * ty * iz3);
      for (int a_ = 0; a_ < 3; ++a_) out[P_MU + a_] = cam.R[a_] * dtx + cam.R[3 + a_] * dty + cam.R[6 + a_] * dtz;
      // Sigma = M M^T: dM = 2 dSigma M ; ds_k = sum_i dM_ik M_ik ; dR_ik = dM_ik e^{s_k}
      float dR[3][3];
      for (int a_ = 0; a_ < 3; ++a_)
        for (int k = 0; k < 3; ++k) {
          const float dM = 2.f * (dSg[a_][0] * M[0][k] + dSg[a_][1] * M[1][k] + dSg[a_][2] * M[2][k]);
          out[P_S + k] += dM * M[a_][k];
          dR[a_][k] = dM * es[k];
        }
      if (!deg) {
        const float dqw = 2.f * (-zq * dR[0][1] + y * dR[0][2] + zq * dR[1][0] - x * dR[1][2] - y * dR[2][0] + x * dR[2][1]);
        const float dqx = 2.f * (y * dR[0][1] + zq * dR[0][2] + y * dR[1][0] - 2.f * x * dR[1][1] - w * dR[1][2] +
                                 zq * dR[2][0] + w * dR[2][1] - 2.f * x * dR[2][2]);
        const float dqy = 2.f * (-2.f * y * dR[0][0] + x * dR[0][1] + w * dR[0][2] + x * dR[1][0] + zq * dR[1][2] -
                                 w * dR[2][0] + zq * dR[2][1] - 2.f * y * dR[2][2]);
        const float dqz = 2.f * (-2.f * zq * dR[0][0] - w * dR[0][1] + x * dR[0][2] + w * dR[1][0] - 2.f * zq * dR[1][1] +
                                 y * dR[1][2] + x * dR[2][0] + y * dR[2][1]);
        const float dot = w * dqw + x * dqx + y * dqy + zq * dqz;
        out[P_Q] = (dqw - w * dot) / qn; out[P_Q + 1] = (dqx - x * dot) / qn;
        out[P_Q + 2] = (dqy - y * dot) / qn; out[P_Q + 3] = (dqz - zq * dot) / qn;
      }
      const float wo = 1.f / (1.f + expf(-P[P_O * G + j]));
      out[P_O] = dw * wo * (1.f - wo);
      for (int c = 0; c < 3; ++c) out[P_C + c] = P[(P_C + c) * G + j] > 0.f ? dch[c] : 0.f;
    }
    for (int k = 0; k < kNP; ++k) raw[k * G + j] = out[k];
  }
}

// --------------------------------------------------------------------------- launchers
static int sblocks(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

cudaError_t launch_sproject(const float* P, int64_t G, int64_t g0, int64_t g1, const SCam& cam, ScreenBufs& b,
                            cudaStream_t s) {
  k_sproject<<<sblocks(g1 - g0), 256, 0, s>>>(P, G, g0, g1, cam, b.pa, b.pb, b.pc, b.rect, b.touched);
  const int64_t n = g1 - g0;
  const int nb = (int)((n + kScanChunk - 1) / kScanChunk);
  k_sscan_blocks<<<std::max(nb, 1), kScanB, 0, s>>>(b.touched, n, b.bsums);
  k_sscan_top<<<1, kScanB, 0, s>>>(b.bsums, nb, b.total);
  k_sscan_apply<<<std::max(nb, 1), kScanB, 0, s>>>(b.touched, n, b.bsums, b.off);
  return cudaGetLastError();
}

cudaError_t launch_skeys_sort(int64_t g0, int64_t g1, const LevelGeom& g, int lev0, int Lr, const SCam& cam,
                              ScreenBufs& b, int64_t npairs, int64_t Np, cudaStream_t s) {
  const int ntiles = cam.TX * cam.TY;
  cudaMemsetAsync(b.key + npairs, 0xFF, sizeof(uint64_t) * (Np - npairs), s);
  cudaMemsetAsync(b.val + npairs, 0x7F, sizeof(int64_t) * (Np - npairs), s);
  k_skeys<<<sblocks(g1 - g0), 256, 0, s>>>(g0, g1, g, lev0, ntiles, cam.TX, b.pa, b.rect, b.off, b.key, b.val);
  if (Np > 1) launch_sort_kv(b.key, b.val, Np, s);
  cudaMemsetAsync(b.ranges, 0, sizeof(uint2) * (size_t)Lr * ntiles, s);
  if (npairs > 0) k_sranges<<<sblocks(npairs), 256, 0, s>>>(b.key, npairs, b.ranges);
  return cudaGetLastError();
}

// ---------------------------------------------- two-level sort: counting sort by tile, then
// a per-tile sort of (depth bits << 32 | index) in shared memory.  The 64-bit key orders a
// tile's Gaussians by depth with ties by index (the global sort's order, reading A23).
__global__ void k_tile_count(int64_t g0, int64_t g1, LevelGeom g, int lev0, int ntiles_img, int TX,
                             const int4* __restrict__ rect, uint32_t* count) {
  for (int64_t j = g0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < g1; j += (int64_t)gridDim.x * blockDim.x) {
    const int4 r = rect[j];
    if (!(r.x < r.y && r.z < r.w)) continue;
    const int l = level_of_gaussian(g, j) - lev0;
    for (int ty = r.z; ty < r.w; ++ty)
      for (int tx = r.x; tx < r.y; ++tx) atomicAdd(count + (size_t)l * ntiles_img + ty * TX + tx, 1u);
  }
}

__global__ void k_tile_scatter(int64_t g0, int64_t g1, LevelGeom g, int lev0, int ntiles_img, int TX,
                               const float4* __restrict__ pa, const int4* __restrict__ rect,
                               const uint32_t* __restrict__ start, uint32_t* cursor, uint64_t* key) {
  for (int64_t j = g0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < g1; j += (int64_t)gridDim.x * blockDim.x) {
    const int4 r = rect[j];
    if (!(r.x < r.y && r.z < r.w)) continue;
    const int l = level_of_gaussian(g, j) - lev0;
    const uint64_t k = ((uint64_t)__float_as_uint(pa[j].z) << 32) | (uint64_t)(uint32_t)j;
    for (int ty = r.z; ty < r.w; ++ty)
      for (int tx = r.x; tx < r.y; ++tx) {
        const size_t t = (size_t)l * ntiles_img + ty * TX + tx;
        key[start[t] + atomicAdd(cursor + t, 1u)] = k;
      }
  }
}

constexpr int kTileSortMax = 8192;           // items per tile sorted in shared memory (64 KB)

// one CTA per (level, tile): bitonic sort of its segment in shared memory; segments over the
// capacity flag `big` (the host then falls back to the global sort)
__global__ void __launch_bounds__(1024) k_tile_sort(const uint32_t* __restrict__ start, const uint32_t* __restrict__ total,
                                                    int nt, uint64_t* key, int64_t* val, uint2* ranges, uint32_t* big) {
  extern __shared__ uint64_t sk[];
  const int t = blockIdx.x;
  const uint32_t b0 = start[t], b1 = t + 1 < nt ? start[t + 1] : *total;
  const int n = (int)(b1 - b0);
  if (threadIdx.x == 0) ranges[t] = make_uint2(b0, b1);
  if (n <= 0) return;
  if (n > kTileSortMax) { if (threadIdx.x == 0) atomicExch(big, 1u); return; }
  int np = 1;
  while (np < n) np <<= 1;
  for (int i = threadIdx.x; i < np; i += blockDim.x) sk[i] = i < n ? key[b0 + i] : ~0ull;
  __syncthreads();
  for (int k = 2; k <= np; k <<= 1)
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int i = threadIdx.x; i < np; i += blockDim.x) {
        const int p = i ^ jj;
        if (p > i) {
          const bool up = (i & k) == 0;
          const uint64_t a = sk[i], c = sk[p];
          if ((c < a) == up) { sk[i] = c; sk[p] = a; }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < n; i += blockDim.x) val[b0 + i] = (int64_t)(uint32_t)(sk[i] & 0xFFFFFFFFull);
}

// Returns in *big_host whether some tile exceeded kTileSortMax (then the caller uses the
// global sort, launch_skeys_sort).  tile buffers: count/cursor/start [Lr * ntiles + 1].
cudaError_t launch_tile_sort(int64_t g0, int64_t g1, const LevelGeom& g, int lev0, int Lr, const SCam& cam,
                             ScreenBufs& b, uint32_t* tcount, uint32_t* tcursor, uint32_t* tstart, uint32_t* tbsums,
                             uint32_t* ttotal, uint32_t* big, cudaStream_t s) {
  const int ntiles = cam.TX * cam.TY;
  const int nt = Lr * ntiles;
  // (per call: the attribute belongs to the current device)
  cudaFuncSetAttribute(k_tile_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kTileSortMax * sizeof(uint64_t)));
  cudaMemsetAsync(tcount, 0, sizeof(uint32_t) * nt, s);
  cudaMemsetAsync(tcursor, 0, sizeof(uint32_t) * nt, s);
  cudaMemsetAsync(big, 0, sizeof(uint32_t), s);
  k_tile_count<<<sblocks(g1 - g0), 256, 0, s>>>(g0, g1, g, lev0, ntiles, cam.TX, b.rect, tcount);
  launch_scan_u32(tcount, nt, tbsums, ttotal, tstart, s);
  k_tile_scatter<<<sblocks(g1 - g0), 256, 0, s>>>(g0, g1, g, lev0, ntiles, cam.TX, b.pa, b.rect, tstart, tcursor, b.key);
  k_tile_sort<<<nt, 1024, kTileSortMax * sizeof(uint64_t), s>>>(tstart, ttotal, nt, b.key, b.val, b.ranges, big);
  return cudaGetLastError();
}

cudaError_t launch_sraster(const SCam& cam, int Lr, ScreenBufs& b, float* out, float* outT, uint32_t* last,
                           cudaStream_t s) {
  SRasterArgs a{b.ranges, b.val, b.pa, b.pb, b.pc, out, outT, last, cam};
  k_sraster<<<dim3(cam.TX * cam.TY, Lr), kTileThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sloss(const float* img, const float* target, const uint8_t* valid, int Lr, int64_t npx, float eps,
                         int mode, float* dLdC, double* partial, cudaStream_t s) {
  const int bx = (int)std::min<int64_t>((npx + 255) / 256, 256);
  k_sloss<<<dim3(std::max(bx, 1), Lr), 256, 0, s>>>(img, target, valid, Lr, npx, eps, mode, dLdC, partial);
  return cudaGetLastError();
}

cudaError_t launch_sraster_bwd(const SCam& cam, int Lr, ScreenBufs& b, const float* outT, const uint32_t* last,
                               const float* dLdC, float* g2d, cudaStream_t s) {
  SBwdArgs a{b.ranges, b.val, b.pa, b.pb, b.pc, outT, last, dLdC, g2d, cam};
  k_sraster_bwd<<<dim3(cam.TX * cam.TY, Lr), kTileThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sproject_bwd(const float* P, int64_t G, int64_t g0, int64_t g1, const SCam& cam,
                                const ScreenBufs& b, float* g2d, float* raw, cudaStream_t s) {
  k_sproject_bwd<<<sblocks(g1 - g0), 256, 0, s>>>(P, G, g0, g1, cam, b.pc, g2d, raw);
  return cudaGetLastError();
}

}  // namespace gsc
