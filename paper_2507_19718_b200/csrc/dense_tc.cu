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

namespace gsc {

constexpr int kTcThreads = 128;
constexpr int kTcTile = 128 * 8 * 4;                         // bytes of one 128-row x 8 tf32 K-major tile
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
