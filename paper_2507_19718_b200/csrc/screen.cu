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
//   k_sproject   per Gaussian: EWA projection, conic, radius, tile rectangle, tiles touched,
//                per-(level, tile) key counts, their total
//   two-level sort: per-(level, tile) key counts (k_sproject) -> scan -> k_tile_scatter (keys
//                depth bits << 32 | index into their tile's segment; a warp's (Gaussian, tile)
//                pairs spread evenly over its lanes) -> k_tile_sort_warp (segment ranges; bitonic sort
//                in registers, one warp per tile of <= 256 keys) -> k_tile_sort (shared
//                memory, <= 8192); the global path (k_skeys, bitonic
//                sort of (tile, depth) keys, k_sranges) only when a tile holds more
//   k_sraster    one CTA per (tile, level), 128 threads x 2 pixels, batches of 128 Gaussians staged in
//                shared memory, front-to-back compositing; C, final T, last contributor; for
//                gc_fit_image Eq. 4 is fused in: dL/dC and the per-level loss statistics
//                instead of C
//   gc_fit_image then: k_sraster_bwd (back to front, per-Gaussian transposing warp
//                reductions, then float reds) and k_sproject_bwd (EWA / projection chain rule
//                to the 14 raw parameters), the shared AdamW (raw-gradient mode) and the
//                culling rebuild.
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
// true when some pixel centre of tile (tx, ty) lies within distance R of (u, v) (NaN: true)
__device__ __forceinline__ bool tile_hit(float u, float v, float R, int tx, int ty) {
  const float x0 = tx * kTile + 0.5f, y0 = ty * kTile + 0.5f;
  const float dx = fmaxf(fmaxf(x0 - u, u - (x0 + (kTile - 1))), 0.f);
  const float dy = fmaxf(fmaxf(y0 - v, v - (y0 + (kTile - 1))), 0.f);
  return !(dx * dx + dy * dy > R * R);
}

// pa = (u, v, depth, w), pb = (conic a, b, c, R), pc = (chat, ok), rect = (x0, x1, y0, y1);
// R bounds the pixels where alpha >= 1/255 can hold: only tiles of the rectangle with a pixel
// centre within R of (u, v) get a key
// It also counts the keys of every (level, tile) (count, fire-and-forget reductions over the
// rectangle) and their total (npairs, one warp-aggregated atomic).
__global__ void k_sproject(const float* __restrict__ P, int64_t G, int64_t g0, int64_t g1, SCam cam,
                           float4* pa, float4* pb, float4* pc, int4* rect, uint32_t* touched, LevelGeom lg,
                           int lev0, uint32_t* count, uint32_t* npairs) {
  const int ntiles_img = cam.TX * cam.TY;
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
          const float w = 1.f / (1.f + expf(-P[P_O * G + j]));
          // opacity-aware tightening: alpha >= 1/255 needs d^T Sigma2^-1 d <= 2 ln(255 w), whose
          // bounding box has half-extents sqrt(2 ln(255 w) Sigma2_xx), ..._yy (widened by 0.1 % +
          // 0.01 px for fp32); tiles of the 3-sigma rectangle outside it hold no pixel the
          // raster could accept, so dropping them changes no image (A23)
          const float r2 = 2.f * logf(255.f * w);
          float Ra = INFINITY;                           // radius of a circle around that ellipse
          if (r2 < 0.f) {
            r.y = r.x;                                   // w < 1/255: no pixel reaches the floor
          } else {
            const float hx = fmaf(sqrtf(r2 * A), 1.001f, 0.01f), hy = fmaf(sqrtf(r2 * Cc), 1.001f, 0.01f);
            if (isfinite(hx) && isfinite(hy)) {
              Ra = fmaf(sqrtf(r2 * lam), 1.001f, 0.01f);
              r.x = max(r.x, clamp_tile(floorf((u - hx - 0.5f) / kTile), cam.TX));
              r.y = min(r.y, clamp_tile(floorf((u + hx - 0.5f) / kTile) + 1.f, cam.TX));
              r.z = max(r.z, clamp_tile(floorf((v - hy - 0.5f) / kTile), cam.TY));
              r.w = min(r.w, clamp_tile(floorf((v + hy - 0.5f) / kTile) + 1.f, cam.TY));
            }
          }
          if (r.x < r.y && r.z < r.w) {
            n = 1;
            const float id = 1.f / det;
            a = make_float4(u, v, tz, w);
            b = make_float4(Cc * id, -B * id, A * id, Ra);
            c = make_float4(fmaxf(P[P_C * G + j], 0.f), fmaxf(P[(P_C + 1) * G + j], 0.f), fmaxf(P[(P_C + 2) * G + j], 0.f), 1.f);
          }
        }
      }
    }
    if (n) {
      // keys only for the tiles within the circle (the same test in the scatter and k_skeys)
      n = 0;
      const size_t lbase = (size_t)(level_of_gaussian(lg, j) - lev0) * ntiles_img;
      for (int ty = r.z; ty < r.w; ++ty)
        for (int tx = r.x; tx < r.y; ++tx)
          if (tile_hit(a.x, a.y, b.w, tx, ty)) { atomicAdd(count + lbase + ty * cam.TX + tx, 1u); ++n; }
    }
    pa[j] = a; pb[j] = b; pc[j] = c; rect[j] = r;
    touched[j - g0] = n;
    const uint32_t m = __activemask();
    const uint32_t tot = __reduce_add_sync(m, n);
    if ((threadIdx.x & 31) == __ffs(m) - 1 && tot) atomicAdd(npairs, tot);
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

// Up to kScanSingleMax entries: one CTA scans them all (one launch instead of three, which
// at these sizes -- 32 k tile counters at 1080p -- are a chain of fixed latencies).  Thread t
// owns 32 consecutive entries, loaded as 8 x uint4 all in flight before any is summed.
constexpr int kScanSinglePer = 32, kScanSingleMax = kScanB * kScanSinglePer;
__global__ void __launch_bounds__(kScanB) k_sscan_single(const uint32_t* __restrict__ in, int n, uint32_t* total,
                                                        uint32_t* out) {
  const int b = threadIdx.x * kScanSinglePer;
  uint4 v[kScanSinglePer / 4];
#pragma unroll
  for (int k = 0; k < kScanSinglePer / 4; ++k) {
    const int i = b + 4 * k;
    if (i + 4 <= n) v[k] = *reinterpret_cast<const uint4*>(in + i);
    else v[k] = make_uint4(i < n ? in[i] : 0u, i + 1 < n ? in[i + 1] : 0u, i + 2 < n ? in[i + 2] : 0u, 0u);
  }
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanSinglePer / 4; ++k) s += v[k].x + v[k].y + v[k].z + v[k].w;
  uint32_t tot;
  uint32_t off = block_scan_excl(s, &tot);
#pragma unroll
  for (int k = 0; k < kScanSinglePer / 4; ++k) {
    const int i = b + 4 * k;
    uint4 o;
    o.x = off; off += v[k].x; o.y = off; off += v[k].y; o.z = off; off += v[k].z; o.w = off; off += v[k].w;
    if (i + 4 <= n) *reinterpret_cast<uint4*>(out + i) = o;
    else {
      if (i < n) out[i] = o.x;
      if (i + 1 < n) out[i + 1] = o.y;
      if (i + 2 < n) out[i + 2] = o.z;
    }
  }
  if (threadIdx.x == 0) *total = tot;
}

// exclusive scan of n u32 (bsums: >= n / 4096 + 2 words, total: 1 word), deterministic
void launch_scan_u32(const uint32_t* in, int64_t n, uint32_t* bsums, uint32_t* total, uint32_t* out, cudaStream_t s) {
  if (n <= kScanSingleMax && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
    k_sscan_single<<<1, kScanB, 0, s>>>(in, (int)n, total, out);
    return;
  }
  const int nb = (int)((n + kScanChunk - 1) / kScanChunk);
  k_sscan_blocks<<<std::max(nb, 1), kScanB, 0, s>>>(in, n, bsums);
  k_sscan_top<<<1, kScanB, 0, s>>>(bsums, nb, total);
  k_sscan_apply<<<std::max(nb, 1), kScanB, 0, s>>>(in, n, bsums, out);
}

// --------------------------------------------------------------------------- keys / ranges
__global__ void k_skeys(int64_t g0, int64_t g1, LevelGeom g, int lev0, int ntiles_img, int TX,
                        const float4* __restrict__ pa, const float4* __restrict__ pb, const int4* __restrict__ rect,
                        const uint32_t* __restrict__ off, uint64_t* key, int64_t* val) {
  for (int64_t j = g0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < g1; j += (int64_t)gridDim.x * blockDim.x) {
    const int4 r = rect[j];
    if (!(r.x < r.y && r.z < r.w)) continue;
    const int l = level_of_gaussian(g, j) - lev0;
    const uint32_t dbits = __float_as_uint(pa[j].z);     // depth > znear > 0: bits order like values
    uint32_t o = off[j - g0];
    for (int ty = r.z; ty < r.w; ++ty)
      for (int tx = r.x; tx < r.y; ++tx) {
        if (!tile_hit(pa[j].x, pa[j].y, pb[j].w, tx, ty)) continue;
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
  // fused Eq. 4 (gc_fit_image): with dLdC set, each pixel's loss gradient is written instead
  // of its colour (out may be null) and the per-level loss sums / valid counts go to partial
  const float* target; const uint8_t* valid; float eps; int mode;
  float* dLdC; double* partial;
  int64_t kv_cap = 0;   // GSC_CHECKED bounds of the sorted (tile, depth) -> Gaussian list
};

// Eq. 4 at one pixel (reading A10: denominator frozen, mode 0, or the full quotient, mode 1):
// (one approximate reciprocal per channel; the pixel's 3 terms summed in fp32, the tile's in fp64)
__device__ __forceinline__ void pixel_loss(const float* y, const float* x, float eps, int mode, float& ls, float* g) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float r = x[c] - y[c], d = y[c] + eps;
    const float id2 = __fdividef(1.f, d * d);
    ls += r * r * id2;
    g[c] = mode == 0 ? -2.f * r * id2 : __fdividef(-2.f * r * (x[c] + eps) * id2, d);
  }
}

// Two horizontally adjacent pixels per thread (128 threads per 16 x 16 tile): the staged
// Gaussian is read from shared memory once per pixel pair and the pair's opacity chain runs in
// packed fp32x2 (pix_alpha).  The forward and the backward evaluate a pixel's opacity through
// this one function, so the backward's acceptance tests reproduce the forward's bit for bit.
constexpr float kL2E = 1.4426950408889634f;

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// The staged conic is pre-scaled into log2 units, cs = (-a/2, -b, -c/2) log2(e), so that
// t = power log2(e) = cs.x dx^2 + cs.z dy^2 + cs.y dx dy at the pixel centres (nfx = -(px + 1/2)
// of the two pixels, fy = py + 1/2); G = 2^t = e^power, a0 = w G.  A pixel accepts the Gaussian
// iff t <= 0 and a0 >= 1/255 (alpha = min(0.99, a0) >= 1/255 exactly then; reading A23).
__device__ __forceinline__ float4 scaled_conic(float a, float b, float c, float w) {
  return make_float4(a * (-0.5f * kL2E), b * -kL2E, c * (-0.5f * kL2E), w);
}
__device__ __forceinline__ void pix_alpha(float2 uv, float4 cs, float2 nfx, float fy, float2& dx, float& dy,
                                          float2& t, float2& G, float2& a0) {
  dx = __fadd2_rn(make_float2(uv.x, uv.x), nfx);
  dy = __fadd_rn(uv.y, -fy);
  const float cdd = __fmul_rn(__fmul_rn(cs.z, dy), dy);
  const float bdy = __fmul_rn(cs.y, dy);
  const float2 adx = __fmul2_rn(make_float2(cs.x, cs.x), dx);
  t = __ffma2_rn(adx, dx, make_float2(cdd, cdd));
  t = __ffma2_rn(make_float2(bdy, bdy), dx, t);
  G = make_float2(ex2_ftz(t.x), ex2_ftz(t.y));
  a0 = __fmul2_rn(make_float2(cs.w, cs.w), G);
}

constexpr int kRasterThreads = kTileThreads / 2;
#ifndef GSC_BWD_DIRECT
#define GSC_BWD_DIRECT 24
#endif

#ifdef GSC_SFWD_MINB
__global__ void __launch_bounds__(kRasterThreads, GSC_SFWD_MINB) k_sraster(SRasterArgs a) {
#else
__global__ void __launch_bounds__(kRasterThreads) k_sraster(SRasterArgs a) {
#endif
  __shared__ float2 s_uv[kRasterThreads];
  __shared__ float4 s_co[kRasterThreads];     // scaled conic (scaled_conic), w
  __shared__ float4 s_c[kRasterThreads];
  const int tile = blockIdx.x, l = blockIdx.y;
  const int ntiles = a.cam.TX * a.cam.TY;
  const int tx = tile % a.cam.TX, ty = tile / a.cam.TX;
  const int px = tx * kTile + 2 * (threadIdx.x & 7), py = ty * kTile + (threadIdx.x >> 3);
  const bool in0 = px < a.cam.W && py < a.cam.H, in1 = px + 1 < a.cam.W && py < a.cam.H;
  const float2 nfx = make_float2(-(px + 0.5f), -(px + 1.5f));
  const float fy = py + 0.5f;
  const uint2 rg = a.ranges[(size_t)l * ntiles + tile];
  const int n = rg.y > rg.x ? (int)(rg.y - rg.x) : 0;
  bool done0 = !in0, done1 = !in1;
  float2 T = make_float2(1.f, 1.f), C0 = make_float2(0.f, 0.f), C1 = C0, C2 = C0;
  uint32_t last0 = 0, last1 = 0;
  for (int b0 = 0; b0 < n; b0 += kRasterThreads) {
    if (__syncthreads_count(done0 && done1) == kRasterThreads) break;
    const int q = b0 + threadIdx.x;
    if (q < n) {
      const int64_t j = a.val[rg.x + q];
      GSC_CHECK(rg.y <= (uint64_t)a.kv_cap && j >= 0, "raster: tile range / Gaussian index");
      const float4 p = a.pa[j];
      s_uv[threadIdx.x] = make_float2(p.x, p.y);
      const float4 b = a.pb[j];
      s_co[threadIdx.x] = scaled_conic(b.x, b.y, b.z, p.w);
      s_c[threadIdx.x] = a.pc[j];
    }
    __syncthreads();
    const int m = min(kRasterThreads, n - b0);
    for (int k = 0; k < m && !(done0 && done1); ++k) {
      float2 dx, tp, G, a0;
      float dy;
      pix_alpha(s_uv[k], s_co[k], nfx, fy, dx, dy, tp, G, a0);
      const bool acc0 = !done0 && !(tp.x > 0.f) && a0.x >= 1.f / 255.f;
      const bool acc1 = !done1 && !(tp.y > 0.f) && a0.y >= 1.f / 255.f;
      if (!(acc0 || acc1)) continue;
      const float2 alpha = make_float2(fminf(0.99f, a0.x), fminf(0.99f, a0.y));
      const float2 Tn = __fmul2_rn(T, make_float2(1.f - alpha.x, 1.f - alpha.y));
      const uint32_t cnt = (uint32_t)(b0 + k + 1);        // contributor count of this Gaussian
      const bool ap0 = acc0 && !(Tn.x < 1e-4f), ap1 = acc1 && !(Tn.y < 1e-4f);
      done0 |= acc0 && !ap0;
      done1 |= acc1 && !ap1;
      const float2 wgt = make_float2(ap0 ? alpha.x * T.x : 0.f, ap1 ? alpha.y * T.y : 0.f);
      const float4 c = s_c[k];
      C0 = __ffma2_rn(wgt, make_float2(c.x, c.x), C0);
      C1 = __ffma2_rn(wgt, make_float2(c.y, c.y), C1);
      C2 = __ffma2_rn(wgt, make_float2(c.z, c.z), C2);
      if (ap0) { T.x = Tn.x; last0 = cnt; }
      if (ap1) { T.y = Tn.y; last1 = cnt; }
    }
  }
  const size_t pix = ((size_t)l * a.cam.H + min(py, a.cam.H - 1)) * a.cam.W + px;
  const float Cp[2][3] = {{C0.x, C1.x, C2.x}, {C0.y, C1.y, C2.y}};
  const float Tp[2] = {T.x, T.y};
  const uint32_t Lp[2] = {last0, last1};
  double ls = 0.0, cnt = 0.0;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    if (!(i ? in1 : in0)) continue;
    const size_t pi = pix + i;
    if (a.out) { a.out[3 * pi] = Cp[i][0]; a.out[3 * pi + 1] = Cp[i][1]; a.out[3 * pi + 2] = Cp[i][2]; }
    if (a.outT) a.outT[pi] = Tp[i];
    if (a.last) a.last[pi] = Lp[i];
    if (a.dLdC) {
      float g[3] = {0.f, 0.f, 0.f};
      if (!a.valid || a.valid[pi]) {
        cnt += 1.0;
        const float x[3] = {a.target[3 * pi], a.target[3 * pi + 1], a.target[3 * pi + 2]};
        float lp = 0.f;
        pixel_loss(Cp[i], x, a.eps, a.mode, lp, g);
        ls += (double)lp;
      }
      a.dLdC[3 * pi] = g[0]; a.dLdC[3 * pi + 1] = g[1]; a.dLdC[3 * pi + 2] = g[2];
    }
  }
  if (a.dLdC) {
    __shared__ double s_red[2][kRasterThreads / 32];
    for (int o = 16; o > 0; o >>= 1) { ls += __shfl_xor_sync(0xffffffffu, ls, o); cnt += __shfl_xor_sync(0xffffffffu, cnt, o); }
    const int wid = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { s_red[0][wid] = ls; s_red[1][wid] = cnt; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double L = 0.0, N = 0.0;
      for (int w = 0; w < kRasterThreads / 32; ++w) { L += s_red[0][w]; N += s_red[1][w]; }
      if (N > 0.0) {
        double* slot = a.partial + (size_t)(tile % kSlots) * kPart;
        atomicAdd(slot + l, L);
        atomicAdd(slot + kMaxL + l, N);
      }
    }
  }
}

// --------------------------------------------------------------------------- raster backward
// Back to front over each pixel's accepted Gaussians (T recovered by division, alpha <= 0.99):
//   dC/dchat = alpha T, dC/dalpha = T (chat - behind), alpha = min(0.99, w G), G = e^power,
//   power = -(a dx^2 + c dy^2)/2 - b dx dy, dx = u - px, dy = v - py.
// Per Gaussian and warp the 9 partials (du, dv, da, db, dc, dw, dchat) go into g2d[j] (12
// floats): with at most 24 contributing lanes each adds its own (3 vector reductions), else
// the warp sums them with a transposing shuffle reduction first (9 reductions per warp).
struct SBwdArgs {
  const uint2* ranges; const int64_t* val;
  const float4 *pa, *pb, *pc;
  const float* outT; const uint32_t* last; const float* dLdC;
  float* g2d;           // [G][12]: du dv da db | dc dw dc0 dc1 | dc2 - - -
  SCam cam;
  int64_t kv_cap = 0;   // GSC_CHECKED bounds
};

// The pixel pair's share of the backward at one Gaussian (back to front), in packed fp32x2:
// for each pixel i with u_i (accepted by the forward), recover T before the Gaussian
// (T / (1 - alpha), reciprocal refined by one Newton step), update the colour behind it and
// set d[v] to the 9 partials summed over the pair; pixels without u_i keep their state and add 0.
struct PixBwd2 {
  float2 T, g0, g1, g2, acc0, acc1, acc2, la, lc0, lc1, lc2;
};
__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }
__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 sel2(bool u0, bool u1, float2 a, float2 b) {
  return make_float2(u0 ? a.x : b.x, u1 ? a.y : b.y);
}
__device__ __forceinline__ void pix_bwd2(PixBwd2& p, bool u0, bool u1, float4 co, float4 c, float2 dx, float dy,
                                         float2 G, float2 a0, float2 alpha, float (&d)[9]) {
  const float2 oma = __fadd2_rn(f2(1.f), make_float2(-alpha.x, -alpha.y));          // 1 - alpha
  float2 r = make_float2(rcp_ftz(oma.x), rcp_ftz(oma.y));
  r = __ffma2_rn(r, __ffma2_rn(make_float2(-oma.x, -oma.y), r, f2(1.f)), r);          // Newton step
  const float2 Tq = __fmul2_rn(p.T, r);
  p.T = sel2(u0, u1, Tq, p.T);
  const float2 wgt = sel2(u0, u1, __fmul2_rn(alpha, p.T), f2(0.f));
  const float2 d6 = __fmul2_rn(wgt, p.g0), d7 = __fmul2_rn(wgt, p.g1), d8 = __fmul2_rn(wgt, p.g2);   // dL/dchat
  const float2 oml = __fadd2_rn(f2(1.f), make_float2(-p.la.x, -p.la.y));
  p.acc0 = sel2(u0, u1, __ffma2_rn(p.la, p.lc0, __fmul2_rn(oml, p.acc0)), p.acc0);
  p.acc1 = sel2(u0, u1, __ffma2_rn(p.la, p.lc1, __fmul2_rn(oml, p.acc1)), p.acc1);
  p.acc2 = sel2(u0, u1, __ffma2_rn(p.la, p.lc2, __fmul2_rn(oml, p.acc2)), p.acc2);
  p.la = sel2(u0, u1, alpha, p.la);
  p.lc0 = sel2(u0, u1, f2(c.x), p.lc0); p.lc1 = sel2(u0, u1, f2(c.y), p.lc1); p.lc2 = sel2(u0, u1, f2(c.z), p.lc2);
  float2 s3 = __fmul2_rn(__fadd2_rn(f2(c.x), make_float2(-p.acc0.x, -p.acc0.y)), p.g0);
  s3 = __ffma2_rn(__fadd2_rn(f2(c.y), make_float2(-p.acc1.x, -p.acc1.y)), p.g1, s3);
  s3 = __ffma2_rn(__fadd2_rn(f2(c.z), make_float2(-p.acc2.x, -p.acc2.y)), p.g2, s3);
  // the clamped alpha (a0 >= 0.99) has no gradient with respect to w and the power
  const float2 dLda = sel2(u0 && a0.x < 0.99f, u1 && a0.y < 0.99f, __fmul2_rn(p.T, s3), f2(0.f));
  const float2 d5 = __fmul2_rn(dLda, G);                                              // dL/dw
  const float2 ndp = __fmul2_rn(__fmul2_rn(dLda, f2(-co.w)), G);                     // -dL/dpower
  const float2 d0 = __fmul2_rn(ndp, __ffma2_rn(f2(co.x), dx, f2(co.y * dy)));          // dL/du
  const float2 d1 = __fmul2_rn(ndp, __ffma2_rn(f2(co.y), dx, f2(co.z * dy)));          // dL/dv
  const float2 d2 = __fmul2_rn(__fmul2_rn(f2(0.5f), ndp), __fmul2_rn(dx, dx));         // dL/dconic_a
  const float2 d3 = __fmul2_rn(__fmul2_rn(ndp, dx), f2(dy));                           // dL/dconic_b
  const float2 d4 = __fmul2_rn(f2(0.5f * dy * dy), ndp);                               // dL/dconic_c
  d[0] = d0.x + d0.y; d[1] = d1.x + d1.y; d[2] = d2.x + d2.y; d[3] = d3.x + d3.y; d[4] = d4.x + d4.y;
  d[5] = d5.x + d5.y; d[6] = d6.x + d6.y; d[7] = d7.x + d7.y; d[8] = d8.x + d8.y;
}

#ifdef GSC_SBWD_MINB
__global__ void __launch_bounds__(kRasterThreads, GSC_SBWD_MINB) k_sraster_bwd(SBwdArgs a) {
#else
__global__ void __launch_bounds__(kRasterThreads) k_sraster_bwd(SBwdArgs a) {
#endif
  __shared__ float2 s_uv[kRasterThreads];
  __shared__ float4 s_co[kRasterThreads];
  __shared__ float4 s_c[kRasterThreads];
  __shared__ int64_t s_j[kRasterThreads];
  const int tile = blockIdx.x, l = blockIdx.y;
  const int ntiles = a.cam.TX * a.cam.TY;
  const int tx = tile % a.cam.TX, ty = tile / a.cam.TX;
  const int px = tx * kTile + 2 * (threadIdx.x & 7), py = ty * kTile + (threadIdx.x >> 3);
  const bool in0 = px < a.cam.W && py < a.cam.H, in1 = px + 1 < a.cam.W && py < a.cam.H;
  const float2 nfx = make_float2(-(px + 0.5f), -(px + 1.5f));
  const float fy = py + 0.5f;
  const uint2 rg = a.ranges[(size_t)l * ntiles + tile];
  const int n = rg.y > rg.x ? (int)(rg.y - rg.x) : 0;
  if (n == 0) return;                                      // (uniform: an empty tile has no gradient)
  const size_t pix = ((size_t)l * a.cam.H + min(py, a.cam.H - 1)) * a.cam.W + px;
  PixBwd2 pp{};
  int last0 = 0, last1 = 0;
  if (in0) {
    pp.T.x = a.outT[pix]; last0 = (int)a.last[pix];
    pp.g0.x = a.dLdC[3 * pix]; pp.g1.x = a.dLdC[3 * pix + 1]; pp.g2.x = a.dLdC[3 * pix + 2];
  }
  if (in1) {
    pp.T.y = a.outT[pix + 1]; last1 = (int)a.last[pix + 1];
    pp.g0.y = a.dLdC[3 * pix + 3]; pp.g1.y = a.dLdC[3 * pix + 4]; pp.g2.y = a.dLdC[3 * pix + 5];
  }
  const int lastmax = max(last0, last1);                  // Gaussians at positions >= last were not accepted
  const int lane = threadIdx.x & 31;
  // the warp skips Gaussians behind all of its pixels' last contributors, the block starts at
  // the last contributor of its tile (the forward stopped there: T fell below 1e-4)
  const int warpmax = __reduce_max_sync(0xffffffffu, lastmax);
  __shared__ int s_wmax[kRasterThreads / 32];
  if (lane == 0) s_wmax[threadIdx.x >> 5] = warpmax;
  __syncthreads();
  int nb = 0;
#pragma unroll
  for (int w = 0; w < kRasterThreads / 32; ++w) nb = max(nb, s_wmax[w]);
  for (int b1 = min(n, nb); b1 > 0; b1 -= kRasterThreads) {
    const int b0 = max(0, b1 - kRasterThreads);
    __syncthreads();
    const int q = b0 + threadIdx.x;
    if (q < b1) {
      const int64_t j = a.val[rg.x + q];
      GSC_CHECK(rg.y <= (uint64_t)a.kv_cap && j >= 0, "raster: tile range / Gaussian index");
      const float4 p = a.pa[j];
      s_uv[threadIdx.x] = make_float2(p.x, p.y);
      const float4 b = a.pb[j];
      s_co[threadIdx.x] = scaled_conic(b.x, b.y, b.z, p.w);
      s_c[threadIdx.x] = a.pc[j];
      s_j[threadIdx.x] = j;
    }
    __syncthreads();
    for (int k = min(b1, warpmax) - b0 - 1; k >= 0; --k) {
      const int gpos = b0 + k;
      float d[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      bool use = false;
      if (gpos < lastmax) {
        const float4 cs = s_co[k];
        float2 dx, tp, G, a0;
        float dy;
        pix_alpha(s_uv[k], cs, nfx, fy, dx, dy, tp, G, a0);
        const bool u0 = gpos < last0 && !(tp.x > 0.f) && a0.x >= 1.f / 255.f;
        const bool u1 = gpos < last1 && !(tp.y > 0.f) && a0.y >= 1.f / 255.f;
        if (u0 || u1) {
          const float2 alpha = make_float2(fminf(0.99f, a0.x), fminf(0.99f, a0.y));
          // the conic in pixel units for the gradient formulas
          const float4 co = make_float4(cs.x * (-2.f / kL2E), cs.y * (-1.f / kL2E), cs.z * (-2.f / kL2E), cs.w);
          pix_bwd2(pp, u0, u1, co, s_c[k], dx, dy, G, a0, alpha, d);
          use = true;
        }
      }
      // per-warp reduction, then one vector red per warp (skipped when no lane contributed)
      const uint32_t users = __ballot_sync(0xffffffffu, use);
#if GSC_BWD_DIRECT
      // up to 24 contributing lanes: each adds its own 9 partials with 3 vector reductions
      // (fewer instructions than the tree; the L2 takes one vector add per lane).  A/B of the
      // threshold at 1080p: tree only 744 us per fit, 8: 739, 16: 726, 24: 722, 32 (never the
      // tree): 1080 -- full warps of same-address vector adds serialise in the L2.
      if (users && __popc(users) <= GSC_BWD_DIRECT) {
        if (use) {
          float* gj = a.g2d + 12 * s_j[k];
          red_add_v4(gj, d[0], d[1], d[2], d[3]);
          red_add_v4(gj + 4, d[4], d[5], d[6], d[7]);
          atomicAdd(gj + 8, d[8]);
        }
      } else
#endif
      if (users) {
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
                            const LevelGeom& g, int lev0, int Lr, cudaStream_t s) {
  cudaMemsetAsync(b.tcount, 0, sizeof(uint32_t) * (size_t)Lr * cam.TX * cam.TY, s);
  cudaMemsetAsync(b.total, 0, sizeof(uint32_t), s);
  k_sproject<<<sblocks(g1 - g0), 256, 0, s>>>(P, G, g0, g1, cam, b.pa, b.pb, b.pc, b.rect, b.touched, g, lev0,
                                              b.tcount, b.total);
  return cudaGetLastError();
}

cudaError_t launch_skeys_sort(int64_t g0, int64_t g1, const LevelGeom& g, int lev0, int Lr, const SCam& cam,
                              ScreenBufs& b, int64_t npairs, int64_t Np, cudaStream_t s) {
  const int ntiles = cam.TX * cam.TY;
  // per-Gaussian key offsets: exclusive scan of the tiles touched
  const int64_t n = g1 - g0;
  const int nb = (int)((n + kScanChunk - 1) / kScanChunk);
  k_sscan_blocks<<<std::max(nb, 1), kScanB, 0, s>>>(b.touched, n, b.bsums);
  k_sscan_top<<<1, kScanB, 0, s>>>(b.bsums, nb, b.total);
  k_sscan_apply<<<std::max(nb, 1), kScanB, 0, s>>>(b.touched, n, b.bsums, b.off);
  cudaMemsetAsync(b.key + npairs, 0xFF, sizeof(uint64_t) * (Np - npairs), s);
  cudaMemsetAsync(b.val + npairs, 0x7F, sizeof(int64_t) * (Np - npairs), s);
  k_skeys<<<sblocks(g1 - g0), 256, 0, s>>>(g0, g1, g, lev0, ntiles, cam.TX, b.pa, b.pb, b.rect, b.off, b.key, b.val);
  if (Np > 1) launch_sort_kv(b.key, b.val, Np, s);
  cudaMemsetAsync(b.ranges, 0, sizeof(uint2) * (size_t)Lr * ntiles, s);
  if (npairs > 0) k_sranges<<<sblocks(npairs), 256, 0, s>>>(b.key, npairs, b.ranges);
  return cudaGetLastError();
}

// ---------------------------------------------- two-level sort: counting sort by tile (counts
// from k_sproject), then a per-tile sort of (depth bits << 32 | index).  The 64-bit key orders
// a tile's Gaussians by depth with ties by index (the global sort's order, reading A23).
//
// The scatter spreads the (Gaussian, tile) pairs of a warp's Gaussians evenly over its lanes:
// a lane issues ceil(pairs / 32) returning atomics in sequence instead of its own rectangle's
// area (up to ~200 tiles for the top level at 1080p).
// Tile scatter: each warp owns kScatterGW Gaussians (lanes 0 .. kScatterGW-1 load their
// projection record, level and rectangle once), the warp's (Gaussian, tile) pairs are spread
// over all 32 lanes (prefix over the rectangles' areas, a binary search for a pair's owner),
// and a pair's record fields arrive by shuffles instead of per-pair dependent loads.  Few
// Gaussians per warp keep many warps in flight: the pass is a chain of dependent round trips
// (rectangle -> cursor atomic -> key store), not bandwidth.
constexpr int kScatterGW = 8;

__global__ void k_tile_scatter(int64_t g0, int64_t g1, LevelGeom g, int lev0, int ntiles_img, int TX,
                               const float4* __restrict__ pa, const float4* __restrict__ pb,
                               const int4* __restrict__ rect,
                               const uint32_t* __restrict__ start, uint32_t* cursor, uint64_t* key, uint32_t cap) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = g0 + warp * kScatterGW; base < g1; base += nwarps * kScatterGW) {
    const int64_t j = base + lane;
    int4 r = make_int4(0, 0, 0, 0);
    float u = 0.f, v = 0.f, R = 0.f;
    uint32_t dbits = 0u;
    int l = 0;
    if (lane < kScatterGW && j < g1) {
      r = rect[j];
      const float4 p = pa[j];
      u = p.x; v = p.y; dbits = __float_as_uint(p.z); R = pb[j].w;
      l = level_of_gaussian(g, j) - lev0;
    }
    const int w = max(r.y - r.x, 0), area = w * max(r.w - r.z, 0);
    int inc = area;
#pragma unroll
    for (int o = 1; o < kScatterGW; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const int exc = inc - area, tot = __shfl_sync(0xffffffffu, inc, kScatterGW - 1);
    for (int p0 = 0; p0 < tot; p0 += 32) {
      const int q = p0 + lane;
      int src = 0;                                  // the last owner lane with exc <= q (its area > 0)
#pragma unroll
      for (int step = kScatterGW / 2; step > 0; step >>= 1) {
        const int e = __shfl_sync(0xffffffffu, exc, src + step);
        if (e <= q) src += step;
      }
      const int rx = __shfl_sync(0xffffffffu, r.x, src), rz = __shfl_sync(0xffffffffu, r.z, src);
      const int ws = __shfl_sync(0xffffffffu, w, src), es = __shfl_sync(0xffffffffu, exc, src);
      const float us = __shfl_sync(0xffffffffu, u, src), vs = __shfl_sync(0xffffffffu, v, src);
      const float Rs = __shfl_sync(0xffffffffu, R, src);
      const uint32_t ds = __shfl_sync(0xffffffffu, dbits, src);
      const int ls = __shfl_sync(0xffffffffu, l, src);
      if (q < tot) {
        const int i = q - es, ty = rz + i / ws, tx = rx + (i - (i / ws) * ws);
        if (tile_hit(us, vs, Rs, tx, ty)) {
          const uint64_t k = ((uint64_t)ds << 32) | (uint64_t)(uint32_t)(base + src);
          const size_t t = (size_t)ls * ntiles_img + ty * TX + tx;
          const uint32_t pos = start[t] + atomicAdd(cursor + t, 1u);
          if (pos < cap) key[pos] = k;              // (over capacity: the caller grows and re-runs)
        }
      }
    }
  }
}

// Bitonic sort of one tile's n <= 32 E keys by one warp, E keys per lane in registers (lane
// holds elements lane E .. lane E + E - 1): exchanges across lanes by shuffles, within a lane
// by register compare-swaps.
template <int E>
__device__ __forceinline__ void warp_sort_tile(uint64_t* __restrict__ key, int64_t* __restrict__ val, uint32_t b0,
                                               int n, int lane) {
  uint64_t x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = lane * E + e;
    x[e] = i < n ? key[b0 + i] : ~0ull;
  }
  constexpr int NP = 32 * E;
#pragma unroll
  for (int k = 2; k <= NP; k <<= 1) {
#pragma unroll
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      if (jj >= E) {
        const int lm = jj / E;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const bool up = ((lane * E + e) & k) == 0;
          const uint64_t y = __shfl_xor_sync(0xffffffffu, x[e], lm);
          x[e] = (lower == up) ? (y < x[e] ? y : x[e]) : (y > x[e] ? y : x[e]);
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if ((e & jj) == 0) {
            const bool up = ((lane * E + e) & k) == 0;
            const uint64_t a = x[e], c = x[e | jj];
            const bool sw = (c < a) == up;
            x[e] = sw ? c : a;
            x[e | jj] = sw ? a : c;
          }
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = lane * E + e;
    if (i < n) val[b0 + i] = (int64_t)(uint32_t)(x[e] & 0xFFFFFFFFull);
  }
}

constexpr int kWarpSortMax = 256;            // tiles up to this many keys: one warp, registers
constexpr int kTileSortMax = 8192;           // items per tile sorted in shared memory (64 KB)

// one warp per (level, tile): ranges, then the register sort; larger tiles are appended to
// `list` (list_n = big[1]) for the shared-memory kernel
#ifndef GSC_TSW_MINB
#define GSC_TSW_MINB 6   // 40 registers (a little spill in the rare 256-key sort): 3 -> 6 CTAs per SM; render 277 -> 273 us, fit_image 626 -> 621 us
#endif
__global__ void __launch_bounds__(256, GSC_TSW_MINB) k_tile_sort_warp(const uint32_t* __restrict__ start, const uint32_t* __restrict__ total, int nt,
                                 uint64_t* key, int64_t* val, uint2* ranges, uint32_t* list, uint32_t* big,
                                 uint32_t cap) {
  if (*total > cap) return;                               // keys over capacity: re-run after growing
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < nt; t += nw) {
    const uint32_t b0 = start[t], b1 = t + 1 < nt ? start[t + 1] : *total;
    const int n = (int)(b1 - b0);
    if (lane == 0) ranges[t] = make_uint2(b0, b1);
    if (n <= 1) {
      if (n == 1 && lane == 0) val[b0] = (int64_t)(uint32_t)(key[b0] & 0xFFFFFFFFull);
      continue;
    }
    if (n > kWarpSortMax) {
      if (lane == 0) list[atomicAdd(big + 1, 1u)] = (uint32_t)t;
      continue;
    }
    if (n <= 32) warp_sort_tile<1>(key, val, b0, n, lane);
    else if (n <= 64) warp_sort_tile<2>(key, val, b0, n, lane);
    else if (n <= 128) warp_sort_tile<4>(key, val, b0, n, lane);
    else warp_sort_tile<8>(key, val, b0, n, lane);
  }
}

// one CTA per listed (level, tile) of more than kWarpSortMax keys: bitonic sort of its segment
// in shared memory; segments over kTileSortMax flag big[0] (the host then falls back to the
// global sort)
__global__ void __launch_bounds__(1024) k_tile_sort(const uint32_t* __restrict__ start, const uint32_t* __restrict__ total,
                                                    int nt, const uint32_t* __restrict__ list, uint64_t* key,
                                                    int64_t* val, uint32_t* big, uint32_t cap) {
  extern __shared__ uint64_t sk[];
  if (*total > cap) return;
  const uint32_t nlist = big[1];
  for (uint32_t li = blockIdx.x; li < nlist; li += gridDim.x) {
    const int t = (int)list[li];
    const uint32_t b0 = start[t], b1 = t + 1 < nt ? start[t + 1] : *total;
    const int n = (int)(b1 - b0);
    if (n > kTileSortMax) { if (threadIdx.x == 0) atomicExch(big, 1u); continue; }
    int np = 1;
    while (np < n) np <<= 1;
    __syncthreads();
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
  cudaMemsetAsync(tcursor, 0, sizeof(uint32_t) * nt, s);
  cudaMemsetAsync(big, 0, 3 * sizeof(uint32_t), s);
  // tcount was filled by k_sproject
  launch_scan_u32(tcount, nt, tbsums, ttotal, tstart, s);
  const uint32_t cap = (uint32_t)std::min<int64_t>(b.kv_cap, 0xFFFFFFFFll);
  const int scatter_blocks = (int)std::max<int64_t>(1, std::min<int64_t>((g1 - g0 + 8 * kScatterGW - 1) / (8 * kScatterGW), 148 * 16));
  k_tile_scatter<<<scatter_blocks, 256, 0, s>>>(g0, g1, g, lev0, ntiles, cam.TX, b.pa, b.pb, b.rect, tstart, tcursor,
                                                  b.key, cap);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // tcount is free after the scan: it holds the list of tiles for the shared-memory sort
  k_tile_sort_warp<<<(int)std::max<int64_t>((nt + 7) / 8, 1), 256, 0, s>>>(tstart, ttotal, nt, b.key, b.val, b.ranges,
                                                                          tcount, big, cap);
  k_tile_sort<<<sms * 2, 1024, kTileSortMax * sizeof(uint64_t), s>>>(tstart, ttotal, nt, tcount, b.key, b.val, big, cap);
  return cudaGetLastError();
}

cudaError_t launch_sraster(const SCam& cam, int Lr, ScreenBufs& b, float* out, float* outT, uint32_t* last,
                           const SLossArgs* loss, cudaStream_t s) {
  SRasterArgs a{b.ranges, b.val, b.pa, b.pb, b.pc, out, outT, last, cam,
                loss ? loss->target : nullptr, loss ? loss->valid : nullptr, loss ? loss->eps : 0.f,
                loss ? loss->mode : 0, loss ? loss->dLdC : nullptr, loss ? loss->partial : nullptr};
  a.kv_cap = b.kv_cap;
  k_sraster<<<dim3(cam.TX * cam.TY, Lr), kRasterThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sraster_bwd(const SCam& cam, int Lr, ScreenBufs& b, const float* outT, const uint32_t* last,
                               const float* dLdC, float* g2d, cudaStream_t s) {
  SBwdArgs a{b.ranges, b.val, b.pa, b.pb, b.pc, outT, last, dLdC, g2d, cam};
  a.kv_cap = b.kv_cap;
  k_sraster_bwd<<<dim3(cam.TX * cam.TY, Lr), kRasterThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sproject_bwd(const float* P, int64_t G, int64_t g0, int64_t g1, const SCam& cam,
                                const ScreenBufs& b, float* g2d, float* raw, cudaStream_t s) {
  k_sproject_bwd<<<sblocks(g1 - g0), 256, 0, s>>>(P, G, g0, g1, cam, b.pc, g2d, raw);
  return cudaGetLastError();
}

}  // namespace gsc
