// dense_tc.cu -- row A8 (optional): the tensor-core variant of the evaluator for the dense
// all-pairs case (north star: "the quadratic form expands to a GEMM (samples x 10-term monomial
// features against Gaussians x 10 coefficients, then exp, then a second contraction against
// colours)", allowed "only if it stays inside the stated tolerance").
//
// Per work item (<= 128 samples of one cell of the dense tile grid) and chunk of 128 Gaussians
// of the item's level, everything recentred on the cell centre c (x' = x - c, mu' = mu - c):
//   phi(x')   = [x'^2, y'^2, z'^2, x'y', x'z', y'z', x', y', z', 1, 0 x 6]          (A, M x 16)
//   kappa_j   = [A00, A11, A22, 2A01, 2A02, 2A12, -2(A mu')_x, -2(A mu')_y, -2(A mu')_z,
//                mu'^T A mu', 0 x 6]                                               (B, N x 16)
//   Q = phi . kappa_j = (x - mu)^T A (x - mu)  on tcgen05.mma kind::tf32, 128 x 128 x 16 in TMEM,
// with the 3xTF32 split (a = a_hi + a_lo, tf32 each; A_hi B_hi + A_hi B_lo + A_lo B_hi) so the
// products keep ~fp32 precision; recentring bounds the cancellation.  The epilogue (4 warps,
// thread = sample row) reads Q with tcgen05.ld 32x32b.x32 and does the rest on CUDA cores in
// packed fp32x2: e = 2^{-Q log2(e)/2} [Q <= tau^2], yhat += v_j e over column pairs -- the
// "second contraction against colours" (N = 3) is 3 FFMA2 per column pair, cheaper than a
// padded second MMA.  MUFU (one ex2 per pair) is the binding unit.
#include "common.cuh"
#include "kernels.h"
#include "stats.cuh"

namespace gsc {

constexpr int kTcThreads = 128;
constexpr float kTcNegHalfLog2e = -0.72134752044448170f;

struct DenseSmem {
  float a[4][128 * 8];                                       // [kstep * 2 + (hi, lo)]
  float b[4][128 * 8];
  float v[128 * 4];                 // pair-interleaved (r_j r_j+1 g_j g_j+1 b_j b_j+1 - -)
  uint64_t bar;
  uint32_t tbase;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// byte offset of (row r, k in [0, 8)) in a K-major no-swizzle tile: 8 x 16-B core matrices
__device__ __forceinline__ int kmaj(int r, int k) { return (r >> 3) * 256 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4; }
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);
}
// tf32 rounding (to nearest, ties away from zero, as cvt.rna.tf32.f32) on the integer pipe --
// the conversion instruction would compete with the epilogue's MUFU.EX2 for the XU pipe
__device__ __forceinline__ float tf32_int(float x) {
  return __int_as_float((__float_as_int(x) + 0x1000) & (int)0xFFFFE000);
}
__device__ __forceinline__ void put_split(float* tile_hi, float* tile_lo, int r, int k, float x) {
  const float h = tf32_int(x), l = tf32_int(x - h);
  *(float*)((char*)tile_hi + kmaj(r, k)) = h;
  *(float*)((char*)tile_lo + kmaj(r, k)) = l;
}

// the Gaussian amplitudes are stored pair-interleaved so that the packed epilogue reads each
// operand pair of its FFMA2s with one shared load and no register moves
__device__ __forceinline__ void put_v(float* v, int j, float4 c) {
  float* p = v + 8 * (j >> 1) + (j & 1);
  p[0] = c.x; p[2] = c.y; p[4] = c.z;
}

// one 32-column slice of the accumulator row: e = 2^(-Q/2 log2 e) (0 beyond the cut-off when
// CUT), Y += e * colour; v points at the slice's first Gaussian
template <bool CUT>
__device__ __forceinline__ void epi32(const uint32_t (&qv)[32], const float* v, float tau2, float2& Y0, float2& Y1,
                                      float2& Y2) {
#pragma unroll
  for (int k = 0; k < 32; k += 2) {
    const float2 Q = make_float2(__uint_as_float(qv[k]), __uint_as_float(qv[k + 1]));
    const float2 tt = __fmul2_rn(Q, make_float2(kTcNegHalfLog2e, kTcNegHalfLog2e));
    float e0 = ex2_approx(tt.x), e1 = ex2_approx(tt.y);
    if (CUT) {
      e0 = Q.x <= tau2 ? e0 : 0.f;
      e1 = Q.y <= tau2 ? e1 : 0.f;
    }
    const float4 P = *reinterpret_cast<const float4*>(v + 4 * k);
    const float2 B = *reinterpret_cast<const float2*>(v + 4 * k + 4);
    const float2 e = make_float2(e0, e1);
    Y0 = __ffma2_rn(e, make_float2(P.x, P.y), Y0);
    Y1 = __ffma2_rn(e, make_float2(P.z, P.w), Y1);
    Y2 = __ffma2_rn(e, B, Y2);
  }
}

__global__ void __launch_bounds__(kTcThreads, 4) k_dense_tc(DenseArgs a) {
  extern __shared__ __align__(1024) unsigned char dsm_raw[];
  DenseSmem& sm = *reinterpret_cast<DenseSmem*>(dsm_raw);
  const int t = threadIdx.x, warp = t >> 5;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&sm.bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_addr(&sm.tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = sm.tbase;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  uint32_t phase = 0;
  const uint32_t n_work = a.n_work[0];
  // tasks = (item, part of its level's Gaussian chunks): enough tasks for two per CTA even when
  // the items are few (the dense case puts a level's samples in few cells); the parts' partial
  // sums meet in red.global.add (output zeroed by the keys pass / the launcher)
  const uint32_t nsplit = n_work ? max(1u, min(16u, (2u * gridDim.x + n_work - 1) / n_work)) : 1u;
  for (uint32_t task = blockIdx.x; task < n_work * nsplit; task += gridDim.x) {
    const uint32_t it = task / nsplit, part = task % nsplit;
    const WorkItem wi = a.work[it];
    const int l = wi.level;
    // cell centre of the item (dense tile grid)
    const int loc = wi.cell - a.ref.coff[l], dx = a.ref.dx[l], dy = a.ref.dy[l];
    const int cx = loc % dx, tq = loc / dx, cy = tq % dy, cz = tq / dy;
    const float xr = fmaf((float)cx + 0.5f, a.ref.edge[l][0], a.ref.org[l][0]);
    const float yr = fmaf((float)cy + 0.5f, a.ref.edge[l][1], a.ref.org[l][1]);
    const float zr = fmaf((float)cz + 0.5f, a.ref.edge[l][2], a.ref.org[l][2]);
    float x = 0.f, y = 0.f, z = 0.f;
    uint32_t idx = 0;
    const bool valid = t < wi.count;
    if (valid) {
      const float4 p = __ldcs(a.bin + 2 * (int64_t)(wi.start + t));
      x = p.x - xr; y = p.y - yr; z = p.z - zr; idx = __float_as_uint(p.w);
    }
    __syncthreads();                               // the previous item's last chunk is done with A
    {
      const float phi[10] = {x * x, y * y, z * z, x * y, x * z, y * z, x, y, z, 1.f};
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int s = k >> 3;
        put_split(sm.a[2 * s], sm.a[2 * s + 1], t, k & 7, k < 10 ? phi[k] : 0.f);
      }
    }
    float2 Y0 = make_float2(0.f, 0.f), Y1 = Y0, Y2 = Y0;
    const int64_t nch = (a.goff[l + 1] - a.goff[l] + 127) / 128;
    const int64_t g0 = a.goff[l] + 128 * ((nch * part) / nsplit);
    const int64_t g1 = min(a.goff[l + 1], a.goff[l] + 128 * ((nch * (part + 1)) / nsplit));
    for (int64_t cb = g0; cb < g1; cb += 128) {
      const int nj = (int)(g1 - cb < 128 ? g1 - cb : 128);
      {
        float kap[10];
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (t < nj) {
          const float4 r0 = __ldg(a.rec + 3 * (cb + t)), r1 = __ldg(a.rec + 3 * (cb + t) + 1),
                       r2 = __ldg(a.rec + 3 * (cb + t) + 2);
          // A = U^T U from the Cholesky record (U00 U01 U02 U11 | U12 U22 mu_x mu_y | mu_z v)
          const float u00 = r0.x, u01 = r0.y, u02 = r0.z, u11 = r0.w, u12 = r1.x, u22 = r1.y;
          const float A00 = u00 * u00, A01 = u00 * u01, A02 = u00 * u02;
          const float A11 = fmaf(u11, u11, u01 * u01), A12 = fmaf(u11, u12, u01 * u02);
          const float A22 = fmaf(u22, u22, fmaf(u12, u12, u02 * u02));
          const float m0 = r1.z - xr, m1 = r1.w - yr, m2 = r2.x - zr;
          const float t0 = fmaf(A02, m2, fmaf(A01, m1, A00 * m0));
          const float t1 = fmaf(A12, m2, fmaf(A11, m1, A01 * m0));
          const float t2 = fmaf(A22, m2, fmaf(A12, m1, A02 * m0));
          kap[0] = A00; kap[1] = A11; kap[2] = A22; kap[3] = 2.f * A01; kap[4] = 2.f * A02; kap[5] = 2.f * A12;
          kap[6] = -2.f * t0; kap[7] = -2.f * t1; kap[8] = -2.f * t2;
          kap[9] = fmaf(m2, t2, fmaf(m1, t1, m0 * t0));
          v = make_float4(r2.y, r2.z, r2.w, 0.f);
        } else {
#pragma unroll
          for (int k = 0; k < 10; ++k) kap[k] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int s = k >> 3;
          put_split(sm.b[2 * s], sm.b[2 * s + 1], t, k & 7, k < 10 ? kap[k] : 0.f);
        }
        put_v(sm.v, t, v);
      }
      asm volatile("fence.proxy.async.shared::cta;");   // generic-proxy smem writes -> tensor core
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (t == 0) {
        // D = sum over the two K = 8 steps of A_hi B_hi + A_hi B_lo + A_lo B_hi
        int n = 0;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const int pa[3] = {0, 0, 1}, pb[3] = {0, 1, 0};
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const uint64_t da = smem_desc(smem_addr(sm.a[2 * s + pa[q]]));
            const uint64_t db = smem_desc(smem_addr(sm.b[2 * s + pb[q]]));
            const uint32_t acc = n++ > 0;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                         ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(smem_addr(&sm.bar)) : "memory");
      }
      asm volatile("{\n\t.reg .pred P1;\n\tDWAIT:\n\t"
                   "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                   "@!P1 bra DWAIT;\n\t}\n" ::"r"(smem_addr(&sm.bar)), "r"(phase));
      phase ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int nc_ep = (32 * warp < wi.count) ? nj : 0;     // warps without a valid row skip it
      for (int c0 = 0; c0 < nc_ep; c0 += 32) {
        uint32_t q[32];
        const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
                       "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]),
                       "=r"(q[15]), "=r"(q[16]), "=r"(q[17]), "=r"(q[18]), "=r"(q[19]), "=r"(q[20]), "=r"(q[21]),
                       "=r"(q[22]), "=r"(q[23]), "=r"(q[24]), "=r"(q[25]), "=r"(q[26]), "=r"(q[27]), "=r"(q[28]),
                       "=r"(q[29]), "=r"(q[30]), "=r"(q[31])
                     : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (a.tau2 < INFINITY) epi32<true>(q, sm.v + 4 * c0, a.tau2, Y0, Y1, Y2);    // zero beyond nj
        else epi32<false>(q, sm.v + 4 * c0, a.tau2, Y0, Y1, Y2);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();                             // TMEM and B are reused by the next chunk
    }
    if (valid && g0 < g1) {
      float* o = a.out + 3 * (size_t)idx;
      if (nsplit == 1) { o[0] = Y0.x + Y0.y; o[1] = Y1.x + Y1.y; o[2] = Y2.x + Y2.y; }
      else { atomicAdd(o, Y0.x + Y0.y); atomicAdd(o + 1, Y1.x + Y1.y); atomicAdd(o + 2, Y2.x + Y2.y); }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// --------------------------------------------------------------------------------------------
// Dense fit (row A8 backward, gc_fit_dense): the gradient of Eq. 4 through the all-pairs
// evaluator as two chained tensor-core products per (work item, 128-Gaussian chunk).
//
//   MMA 1   Q^T (128 Gaussians x 128 samples) = kappa (A, smem) . phi^T (B, smem)   [3xTF32]
//   epi 1   thread j (a Gaussian, its TMEM lane): e_ji = 2^(-Q/2 log2 e) [Q <= tau^2], split
//           into TF32 hi / lo and written back to tensor memory (tcgen05.st): E^T in TMEM
//   MMA 2   D2 (128 Gaussians x 48) = E^T (A, TMEM) . W (B, smem)                    [3xTF32]
//           with W[i][10 c + f] = g_ic phi_if and W[i][30 + c] = g_ic per sample i (built once
//           per item; g = dL/dy_hat from the forward pass): the sums over the item's samples
//           D2[j][10 c + f] = sum_i e_ji g_ic phi_if and D2[j][30 + c] = sum_i e_ji g_ic = dL/dv_jc
//   epi 2   thread j: dL/dkappa_jf = -1/2 sum_c v_jc D2[j][10 c + f], then the chain to the 12
//           coefficient gradients of the world-space fit (dmu, dA as a symmetric matrix, dv) with
//           mu' = mu - (cell centre), one red.global.add.v4 x 3 per (Gaussian, item part).
// No per-Gaussian reduction across threads: the sum over samples is the second product's K.
// Tensor memory: Q^T, E_hi, E_lo of one sample half (64 columns each) and D2 (48) -> 256 columns, 2 CTAs/SM.
struct DenseBwdSmem {
  float a[4][128 * 8];                                       // kappa tiles  [kstep * 2 + (hi, lo)]
  float b[4][128 * 8];                                       // phi tiles
  float w[32][48 * 8];                                       // W tiles [kstep * 2 + (hi, lo)], 16 ksteps
  uint64_t bar, bar2;                                        // MMA 1 / MMA 2 commits
  uint32_t tbase;
};
constexpr int kBwdN = 48;

// A = U^T U, mu' = mu - centre, v, and kappa of one Gaussian from its evaluation record
__device__ __forceinline__ void rec_kappa(const float4 (&rv)[3], float xr, float yr, float zr,
                                          float (&kap)[10], float (&A)[6], float (&m)[3], float (&v)[3]) {
  const float4 r0 = rv[0], r1 = rv[1], r2 = rv[2];
  const float u00 = r0.x, u01 = r0.y, u02 = r0.z, u11 = r0.w, u12 = r1.x, u22 = r1.y;
  A[0] = u00 * u00; A[3] = u00 * u01; A[4] = u00 * u02;                 // A00 A11 A22 A01 A02 A12
  A[1] = fmaf(u11, u11, u01 * u01); A[5] = fmaf(u11, u12, u01 * u02);
  A[2] = fmaf(u22, u22, fmaf(u12, u12, u02 * u02));
  m[0] = r1.z - xr; m[1] = r1.w - yr; m[2] = r2.x - zr;
  const float t0 = fmaf(A[4], m[2], fmaf(A[3], m[1], A[0] * m[0]));
  const float t1 = fmaf(A[5], m[2], fmaf(A[1], m[1], A[3] * m[0]));
  const float t2 = fmaf(A[2], m[2], fmaf(A[5], m[1], A[4] * m[0]));
  kap[0] = A[0]; kap[1] = A[1]; kap[2] = A[2]; kap[3] = 2.f * A[3]; kap[4] = 2.f * A[4]; kap[5] = 2.f * A[5];
  kap[6] = -2.f * t0; kap[7] = -2.f * t1; kap[8] = -2.f * t2;
  kap[9] = fmaf(m[2], t2, fmaf(m[1], t1, m[0] * t0));
  v[0] = r2.y; v[1] = r2.z; v[2] = r2.w;
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t phase) {
  asm volatile("{\n\t.reg .pred P1;\n\tBWAIT:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@!P1 bra BWAIT;\n\t}\n" ::"r"(smem_addr(bar)), "r"(phase));
}

#define GSC_TMEM_X32_REGS(q) "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), \
  "=r"(q[7]), "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15]),   \
  "=r"(q[16]), "=r"(q[17]), "=r"(q[18]), "=r"(q[19]), "=r"(q[20]), "=r"(q[21]), "=r"(q[22]), "=r"(q[23]),            \
  "=r"(q[24]), "=r"(q[25]), "=r"(q[26]), "=r"(q[27]), "=r"(q[28]), "=r"(q[29]), "=r"(q[30]), "=r"(q[31])
#define GSC_TMEM_X32_IN(q) "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]), "r"(q[4]), "r"(q[5]), "r"(q[6]), "r"(q[7]), \
  "r"(q[8]), "r"(q[9]), "r"(q[10]), "r"(q[11]), "r"(q[12]), "r"(q[13]), "r"(q[14]), "r"(q[15]), "r"(q[16]),          \
  "r"(q[17]), "r"(q[18]), "r"(q[19]), "r"(q[20]), "r"(q[21]), "r"(q[22]), "r"(q[23]), "r"(q[24]), "r"(q[25]),        \
  "r"(q[26]), "r"(q[27]), "r"(q[28]), "r"(q[29]), "r"(q[30]), "r"(q[31])
#define GSC_X32_LIST "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}"
#define GSC_X32_LIST1 "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32}"

__device__ __forceinline__ void tmem_ld32(uint32_t ta, uint32_t (&q)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " GSC_X32_LIST ", [%32];" : GSC_TMEM_X32_REGS(q) : "r"(ta));
}
__device__ __forceinline__ void tmem_st32(uint32_t ta, const uint32_t (&q)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], " GSC_X32_LIST1 ";" ::"r"(ta), GSC_TMEM_X32_IN(q));
}

// 8 warps: two per TMEM lane quarter; thread (t, half) handles row t (sample / Gaussian) and
// half of each row-parallel job (K steps of the phi / kappa tiles, columns of W, columns of E^T)
constexpr int kBwdThreads = 256;
// Each chunk is processed in two halves of the item's samples (64 each): MMA 1 with N = 64,
// epilogue 1 on 64 columns, MMA 2 over K = 64 samples accumulating into D2.  Tensor memory
// per CTA: Q^T [0, 64), E_hi [64, 128), E_lo [128, 192), D2 [192, 240) -> 256 columns, so two
// CTAs share an SM and overlap each other's product waits.
constexpr uint32_t kColQ = 0, kColEh = 64, kColEl = 128, kColD2 = 192, kBwdCols = 256;

// Per (item, chunk k) the threads run a software pipeline on two mbarriers: build kappa(k)
// and issue MMA 1(k, 0) while MMA 2(k-1, 1) still runs, then the chain of chunk k-1 (wait
// MMA 2), then per sample half h: epilogue 1(k, h) (wait MMA 1) and MMA 2(k, h) (+ MMA 1(k, 1)).
__device__ __forceinline__ void bwd_mma1(uint32_t tmem, const DenseBwdSmem& sm, uint32_t id1, int h) {
  int n = 0;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int pa[3] = {0, 0, 1}, pb[3] = {0, 1, 0};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const uint64_t da = smem_desc(smem_addr(sm.a[2 * s + pa[q]]));
      // samples 64 h .. 64 h + 63: eight 8-row core-matrix groups (256 B each) into the tile
      const uint64_t db = smem_desc(smem_addr(sm.b[2 * s + pb[q]]) + 2048u * (uint32_t)h);
      const uint32_t acc = n++ > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(id1), "r"(acc));
    }
  }
}

__device__ __forceinline__ void bwd_mma2(uint32_t tmem, const DenseBwdSmem& sm, uint32_t id2, int h) {
  const uint32_t d2 = tmem + kColD2;
#pragma unroll 1
  for (int sl = 0; sl < 8; ++sl) {
    const int s = 8 * h + sl;                                // K step of the item's samples
    const uint64_t bh = smem_desc(smem_addr(sm.w[2 * s])), bl = smem_desc(smem_addr(sm.w[2 * s + 1]));
    const uint32_t ah = tmem + kColEh + 8u * sl, al = tmem + kColEl + 8u * sl;
    const uint32_t acc0 = s > 0;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                 ::"r"(d2), "r"(ah), "l"(bh), "r"(id2), "r"(acc0));
    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(d2), "r"(ah), "l"(bl), "r"(id2));
    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(d2), "r"(al), "l"(bh), "r"(id2));
  }
}

__device__ __forceinline__ void mma_commit_to(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
               : "memory");
}

// the chain of one Gaussian: D2 row (33 values) -> 12 coefficient gradients, added into grad
__device__ __forceinline__ void bwd_chain(uint32_t lane_base, float* gp, const float (&Am)[6], const float (&mu)[3],
                                          const float (&v)[3], bool live) {
  uint32_t q[32], r[16];
  tmem_ld32(lane_base + kColD2, q);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(lane_base + kColD2 + 32u));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  if (!live) return;
  float D[33];
#pragma unroll
  for (int k = 0; k < 32; ++k) D[k] = __uint_as_float(q[k]);
  D[32] = __uint_as_float(r[0]);
  float Gk[10];
#pragma unroll
  for (int f = 0; f < 10; ++f) Gk[f] = -0.5f * (v[0] * D[f] + v[1] * D[10 + f] + v[2] * D[20 + f]);
  // A (symmetric, per element) and mu through kappa's dependence on A and mu' = mu - c
  const float G00 = Gk[0] - 2.f * Gk[6] * mu[0] + Gk[9] * mu[0] * mu[0];
  const float G11 = Gk[1] - 2.f * Gk[7] * mu[1] + Gk[9] * mu[1] * mu[1];
  const float G22 = Gk[2] - 2.f * Gk[8] * mu[2] + Gk[9] * mu[2] * mu[2];
  const float G01 = Gk[3] - (Gk[6] * mu[1] + Gk[7] * mu[0]) + Gk[9] * mu[0] * mu[1];
  const float G02 = Gk[4] - (Gk[6] * mu[2] + Gk[8] * mu[0]) + Gk[9] * mu[0] * mu[2];
  const float G12 = Gk[5] - (Gk[7] * mu[2] + Gk[8] * mu[1]) + Gk[9] * mu[1] * mu[2];
  const float t0 = Am[0] * mu[0] + Am[3] * mu[1] + Am[4] * mu[2];
  const float t1 = Am[3] * mu[0] + Am[1] * mu[1] + Am[5] * mu[2];
  const float t2 = Am[4] * mu[0] + Am[5] * mu[1] + Am[2] * mu[2];
  const float dm0 = -2.f * (Am[0] * Gk[6] + Am[3] * Gk[7] + Am[4] * Gk[8]) + 2.f * Gk[9] * t0;
  const float dm1 = -2.f * (Am[3] * Gk[6] + Am[1] * Gk[7] + Am[5] * Gk[8]) + 2.f * Gk[9] * t1;
  const float dm2 = -2.f * (Am[4] * Gk[6] + Am[5] * Gk[7] + Am[2] * Gk[8]) + 2.f * Gk[9] * t2;
  red_add_v4(gp, dm0, dm1, dm2, G00);
  red_add_v4(gp + 4, G11, G22, G01, G02);
  red_add_v4(gp + 8, G12, D[30], D[31], D[32]);
}

__global__ void __launch_bounds__(kBwdThreads, 2) k_dense_bwd(DenseBwdArgs a) {
  extern __shared__ __align__(1024) unsigned char dsm_raw[];
  DenseBwdSmem& sm = *reinterpret_cast<DenseBwdSmem*>(dsm_raw);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int t = tid & 127, half = tid >> 7;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&sm.bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&sm.bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&sm.tbase)),
                 "n"(kBwdCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = sm.tbase;
  const uint32_t lane_base = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
  const uint32_t id1 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t id2 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kBwdN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  uint32_t ph1 = 0, ph2 = 0;
  const uint32_t n_work = a.n_work[0];
  const uint32_t nsplit = n_work ? max(1u, min(16u, (2u * gridDim.x + n_work - 1) / n_work)) : 1u;
  for (uint32_t task = blockIdx.x; task < n_work * nsplit; task += gridDim.x) {
    const uint32_t it = task / nsplit, part = task % nsplit;
    const WorkItem wi = a.work[it];
    const int l = wi.level;
    const int loc = wi.cell - a.ref.coff[l], dx = a.ref.dx[l], dy = a.ref.dy[l];
    const int cx = loc % dx, tq = loc / dx, cy = tq % dy, cz = tq / dy;
    const float xr = fmaf((float)cx + 0.5f, a.ref.edge[l][0], a.ref.org[l][0]);
    const float yr = fmaf((float)cy + 0.5f, a.ref.edge[l][1], a.ref.org[l][1]);
    const float zr = fmaf((float)cz + 0.5f, a.ref.edge[l][2], a.ref.org[l][2]);
    const int64_t nch = (a.goff[l + 1] - a.goff[l] + 127) / 128;
    const int64_t g0 = a.goff[l] + 128 * ((nch * part) / nsplit);
    const int64_t g1 = min(a.goff[l + 1], a.goff[l] + 128 * ((nch * (part + 1)) / nsplit));
    if (g0 >= g1) continue;
    float4 rv[3];
    if (g0 + t < g1)
      for (int w = 0; w < 3; ++w) rv[w] = __ldg(a.rec + 3 * (g0 + t) + w);
    // ---- per item: phi^T (B of MMA 1) and W (B of MMA 2), sample t of the item (the previous
    // item's products have completed: every thread waited on their last commits)
    {
      float phi[10] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      float g[3] = {0.f, 0.f, 0.f};
      if (t < wi.count) {
        const float4 p = __ldcs(a.bin + 2 * (int64_t)(wi.start + t));
        const float x = p.x - xr, y = p.y - yr, z = p.z - zr;
        const uint32_t idx = __float_as_uint(p.w);
        phi[0] = x * x; phi[1] = y * y; phi[2] = z * z; phi[3] = x * y; phi[4] = x * z; phi[5] = y * z;
        phi[6] = x; phi[7] = y; phi[8] = z; phi[9] = 1.f;
        g[0] = a.g[3 * (size_t)idx]; g[1] = a.g[3 * (size_t)idx + 1]; g[2] = a.g[3 * (size_t)idx + 2];
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int s = k >> 3;
        if (s != half) continue;
        put_split(sm.b[2 * s], sm.b[2 * s + 1], t, k & 7, k < 10 ? phi[k] : 0.f);
      }
      const int ks = t >> 3, kk = t & 7;                     // W column k = t: K step t / 8
      float* wh = sm.w[2 * ks];
      float* wl = sm.w[2 * ks + 1];
#pragma unroll
      for (int n = 0; n < kBwdN; ++n) {
        if ((n >= kBwdN / 2) != (half == 1)) continue;
        const float val = n < 30 ? g[n / 10] * phi[n % 10] : (n < 33 ? g[n - 30] : 0.f);
        put_split(wh, wl, n, kk, val);
      }
    }
    float pAm[6], pmu[3], pv[3];                             // the previous chunk's Gaussian t
    bool plive = false;
    float* pgp = nullptr;
    for (int64_t cb = g0; cb < g1 + 128; cb += 128) {
      const bool have = cb < g1;                             // (the last round only drains)
      const int nj = have ? (int)(g1 - cb < 128 ? g1 - cb : 128) : 0;
      float Am[6], mu[3], v[3];
      if (have) {
        // ---- kappa(k) (A of MMA 1); MMA 1(k) runs beside MMA 2(k-1)
        float kap[10];
        if (t < nj) {
          rec_kappa(rv, xr, yr, zr, kap, Am, mu, v);
        } else {
#pragma unroll
          for (int k = 0; k < 10; ++k) kap[k] = 0.f;
#pragma unroll
          for (int k = 0; k < 6; ++k) Am[k] = 0.f;
          mu[0] = mu[1] = mu[2] = 0.f; v[0] = v[1] = v[2] = 0.f;
        }
        if (cb + 128 + t < g1)
          for (int w = 0; w < 3; ++w) rv[w] = __ldg(a.rec + 3 * (cb + 128 + t) + w);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int s = k >> 3;
          if (s != half) continue;
          put_split(sm.a[2 * s], sm.a[2 * s + 1], t, k & 7, k < 10 ? kap[k] : 0.f);
        }
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (tid == 0) { bwd_mma1(tmem + kColQ, sm, id1, 0); mma_commit_to(&sm.bar); }
      }
      if (cb > g0) {
        // ---- chain of chunk k-1 (its MMA 2 done)
        mbar_wait_parity(&sm.bar2, ph2);
        ph2 ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (half == 0) bwd_chain(lane_base, pgp, pAm, pmu, pv, plive);
      }
      if (!have) break;
      // ---- the two sample halves: epilogue 1(k, h) -> E^T (64 columns) -> MMA 2(k, h)
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        mbar_wait_parity(&sm.bar, ph1);                      // MMA 1(k, h)
        ph1 ^= 1u;
        if (h == 1) {                                        // MMA 2(k, 0) has read E
          mbar_wait_parity(&sm.bar2, ph2);
          ph2 ^= 1u;
        }
        asm volatile("tcgen05.fence::after_thread_sync;");
        {
          const uint32_t c0 = 32u * (uint32_t)half;          // this warp's 32 of the 64 columns
#pragma unroll
          for (int c1 = 0; c1 < 32; c1 += 16) {
            uint32_t q[16], lo[16];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
                           "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]),
                           "=r"(q[15])
                         : "r"(lane_base + kColQ + c0 + c1));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const float Q = __uint_as_float(q[k]);
              const float e = Q <= a.tau2 ? ex2_approx(Q * kTcNegHalfLog2e) : 0.f;
              const float hi = tf32_int(e);
              q[k] = __float_as_uint(hi);
              lo[k] = __float_as_uint(tf32_int(e - hi));
            }
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                         ::"r"(lane_base + kColEh + c0 + c1), "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]), "r"(q[4]),
                           "r"(q[5]), "r"(q[6]), "r"(q[7]), "r"(q[8]), "r"(q[9]), "r"(q[10]), "r"(q[11]), "r"(q[12]),
                           "r"(q[13]), "r"(q[14]), "r"(q[15]));
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                         ::"r"(lane_base + kColEl + c0 + c1), "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]),
                           "r"(lo[5]), "r"(lo[6]), "r"(lo[7]), "r"(lo[8]), "r"(lo[9]), "r"(lo[10]), "r"(lo[11]),
                           "r"(lo[12]), "r"(lo[13]), "r"(lo[14]), "r"(lo[15]));
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();                                     // (h = 0: all chains of k-1 read D2)
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (tid == 0) {
          bwd_mma2(tmem, sm, id2, h);
          mma_commit_to(&sm.bar2);
          if (h == 0) { bwd_mma1(tmem + kColQ, sm, id1, 1); mma_commit_to(&sm.bar); }
        }
      }
#pragma unroll
      for (int k = 0; k < 6; ++k) pAm[k] = Am[k];
#pragma unroll
      for (int k = 0; k < 3; ++k) { pmu[k] = mu[k]; pv[k] = v[k]; }
      plive = t < nj;
      pgp = a.grad + 12 * (cb + t);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kBwdCols));
}

// Eq. 4 per sample of the dense fit (caller order): y_hat from the forward pass, the target,
// the level of the sample (dropped: non-finite position or colour, n < 1 without a fixed
// level) -> g = dL/dy_hat (reading A10: mode 0 frozen denominator, mode 1 full quotient) and the
// per-level loss sums / counts into the k_stats partial slots
__global__ void k_dense_loss(const float* __restrict__ pos, const int32_t* __restrict__ len, int fixed_level, int L,
                             const float* __restrict__ rgb, const float* __restrict__ yhat, int64_t S, float eps,
                             int mode, float* g, double* partial) {
  __shared__ double s_l[kMaxL], s_n[kMaxL];
  if (threadIdx.x < kMaxL) { s_l[threadIdx.x] = 0.0; s_n[threadIdx.x] = 0.0; }
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S; i += (int64_t)gridDim.x * blockDim.x) {
    float gi[3] = {0.f, 0.f, 0.f};
    const float px = pos[3 * i], py = pos[3 * i + 1], pz = pos[3 * i + 2];
    const float x0 = rgb[3 * i], x1 = rgb[3 * i + 1], x2 = rgb[3 * i + 2];
    int l = fixed_level;
    if (len) { const int n = len[i]; l = n >= 1 ? min(n, L) - 1 : -1; }
    const bool ok = l >= 0 && isfinite(px) && isfinite(py) && isfinite(pz) && isfinite(x0) && isfinite(x1) &&
                    isfinite(x2);
    if (ok) {
      double ls = 0.0;
      const float xs[3] = {x0, x1, x2};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float y = yhat[3 * i + c], r = xs[c] - y, d = y + eps;
        ls += (double)(r * r / (d * d));
        gi[c] = mode == 0 ? -2.f * r / (d * d) : -2.f * r * (xs[c] + eps) / (d * d * d);
      }
      atomicAdd(&s_l[l], ls);
      atomicAdd(&s_n[l], 1.0);
    }
    g[3 * i] = gi[0]; g[3 * i + 1] = gi[1]; g[3 * i + 2] = gi[2];
  }
  __syncthreads();
  if (threadIdx.x < kMaxL && s_n[threadIdx.x] > 0.0) {
    double* slot = partial + (size_t)(blockIdx.x % kSlots) * kPart;
    atomicAdd(slot + threadIdx.x, s_l[threadIdx.x]);
    atomicAdd(slot + kMaxL + threadIdx.x, s_n[threadIdx.x]);
  }
}

constexpr size_t kBwdSmem = sizeof(DenseBwdSmem) + 1024;     // ~82 KB: two CTAs per SM

void launch_dense_bwd(const DenseBwdArgs& a, cudaStream_t s, Profiler* prof) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(k_dense_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBwdSmem);
  ProfScope ps(prof, "dense_bwd", s);
  k_dense_bwd<<<2 * sms, kBwdThreads, kBwdSmem, s>>>(a);       // 2 x 256 TMEM columns per SM
}

void launch_dense_loss(const float* pos, const int32_t* len, int fixed_level, int L, const float* rgb,
                       const float* yhat, int64_t S, float eps, int mode, float* g, double* partial, cudaStream_t s,
                       Profiler* prof) {
  ProfScope ps(prof, "dense_loss", s);
  const int blocks = (int)std::min<int64_t>((S + 255) / 256, 148 * 8);
  k_dense_loss<<<std::max(blocks, 1), 256, 0, s>>>(pos, len, fixed_level, L, rgb, yhat, S, eps, mode, g, partial);
}

// 4 CTAs per SM exactly: each holds 128 TMEM columns (512 per SM), so the dynamic shared
// memory request is sized to admit no fifth CTA (whose tcgen05.alloc would wait for a whole
// persistent CTA to finish).
constexpr size_t kDenseSmem = 52 * 1024;
static_assert(sizeof(DenseSmem) <= kDenseSmem, "dense tile smem");


int dense_tc_grid() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(k_dense_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDenseSmem);
  return sms * 4;
}

void launch_dense_tc(const DenseArgs& a, int grid, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, "dense_tc", s);
  k_dense_tc<<<grid, kTcThreads, kDenseSmem, s>>>(a);
}

}  // namespace gsc
