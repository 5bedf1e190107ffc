// fwdbwd.cu -- the fused forward + HDR loss + backward kernel of gc_fit (A4) and the
// forward-only lookup kernel of gc_query (A7).  Warp-centric: no block barriers.
//
// A work item is <= 32 binned samples of one (level, cell) bin; one warp owns it.  The
// cell's culling list (C8) is staged into the warp's shared memory 32 evaluation records
// (48 B each) at a time.
//   pass 1 (lane = sample): yhat = sum v_j e^{-Q/2} over the candidates with Q <= tau^2 (C3),
//          with the warp ballot of every candidate kept as a 32-bit sample mask; the Eq. 4
//          loss and g = dL/dyhat (C4, unnormalised -- the 1/(3 k_l) factor is applied by the
//          optimizer once k_l is known globally, C9).
//   pass 2 (lane = contributing pair): the masks are expanded into a candidate-major pair list;
//          each lane evaluates the 12 coefficient-gradient terms of C5 for one pair, a
//          segmented warp-shuffle scan merges the pairs of each Gaussian, and the segment's last
//          lane issues 3 x red.global.add.v4.f32.  Work is proportional to contributing pairs,
//          every lane busy; never shared-memory float atomics (a CAS loop on sm_100a).
#include "common.cuh"
#include "kernels.h"

namespace gsc {

constexpr int kPart = kMaxL + 2;
constexpr int kWarps = 8;                                 // warps per CTA
constexpr int kPairCap = 512;                             // recorded (sample, Gaussian) pairs per warp
constexpr int kMaxChunks = 64;                            // recorded chunks per work item (C <= 2048)
constexpr float kNegHalfLog2e = -0.72134752044448170f;    // -0.5 * log2(e)

struct ChunkSmem {
  float4 r0[32], r1[32], r2[32];   // staged records of one 32-candidate chunk
  int gid[32];
};

struct WarpSmem : ChunkSmem {
  float4 sxg[32];                  // sample x, y, z, g0
  float2 sg[32];                   // sample g1, g2
  uint16_t pkey[kPairCap];         // (candidate-in-chunk << 5) | sample, chunk- then candidate-major
  float pe[kPairCap];              // e = exp(-Q/2) of the pair, as pass 1 computed it
  uint16_t cend[kMaxChunks];       // end offset of every chunk's pairs
};

__device__ __forceinline__ Rec rec_from(const ChunkSmem& w, int k) {
  const float4 p = w.r0[k], q = w.r1[k], r = w.r2[k];
  return Rec{p.x, p.y, p.z, p.w, q.x, q.y, q.z, q.w, r.x, r.y, r.z, r.w};
}

__device__ __forceinline__ void stage_chunk(ChunkSmem& w, const int32_t* __restrict__ csr_idx,
                                            const float4* __restrict__ rec, int base, int kc, int lane) {
  __syncwarp();
  if (lane < kc) {
    const int gid = __ldg(csr_idx + base + lane);
    w.gid[lane] = gid;
    w.r0[lane] = __ldg(rec + 3 * gid); w.r1[lane] = __ldg(rec + 3 * gid + 1); w.r2[lane] = __ldg(rec + 3 * gid + 2);
  }
  __syncwarp();
}

// Sample-parallel evaluation of one staged chunk (lane = sample).  Accumulates yhat and, if
// `rec` is given, appends every inside pair (k, lane, e) at pbase + rank among the ballot
// (candidate-major), up to `cap` entries; pbase advances by the ballot's popcount.
template <bool kRecord>
__device__ __forceinline__ void eval_chunk(const ChunkSmem& w, int kc, bool act, float x, float y, float z,
                                           float tau2, float& y0, float& y1, float& y2, int& np,
                                           uint16_t* pkey, float* pe, int& pbase, int cap, int lane) {
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll 2
  for (int k = 0; k < kc; ++k) {
    const Rec g = rec_from(w, k);
    float dx, dy, dz, tx, ty, tz;
    const float Q = quad_form(g, x, y, z, dx, dy, dz, tx, ty, tz);
    const bool in = act && Q <= tau2;
    const uint32_t m = __ballot_sync(0xffffffffu, in);
    if (m) {
      if (in) {
        const float e = ex2_approx(Q * kNegHalfLog2e);
        y0 = fmaf(g.v0, e, y0); y1 = fmaf(g.v1, e, y1); y2 = fmaf(g.v2, e, y2);
        ++np;
        if (kRecord) {
          const int pos = pbase + __popc(m & lt);
          if (pos < cap) { pkey[pos] = (uint16_t)((k << 5) | lane); pe[pos] = e; }
        }
      }
      if (kRecord) pbase += __popc(m);
    }
  }
  __syncwarp();
}

// Gradient terms of pairs [p0, p1) of the staged chunk (lane = pair): 12 coefficient
// gradients (C5), a <= 2-level segmented shuffle scan over each Gaussian's run of pairs,
// then red.global.add.v4.f32 from every 4th lane of a run counted from its end.
__device__ __forceinline__ void chunk_pairs_bwd(const WarpSmem& w, int p0, int p1, float* __restrict__ grad,
                                                int lane) {
  for (int pb = p0; pb < p1; pb += 32) {
    const int p = pb + lane;
    const bool valid = p < p1;
    int k = 32 + lane;                 // idle lanes form their own segments
    float v[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) v[q] = 0.f;
    if (valid) {
      const uint32_t key = w.pkey[p];
      const float e = w.pe[p];
      k = key >> 5;
      const int s = key & 31;
      const Rec g = rec_from(w, k);
      const float4 sx = w.sxg[s];
      const float2 sg = w.sg[s];
      float dx, dy, dz, tx, ty, tz;
      quad_form(g, sx.x, sx.y, sx.z, dx, dy, dz, tx, ty, tz);
      const float he = (sx.w * g.v0 + sg.x * g.v1 + sg.y * g.v2) * e;
      v[0] = he * tx; v[1] = he * ty; v[2] = he * tz;                 // d mu
      const float kk = -0.5f * he;
      const float kx = kk * dx, ky = kk * dy, kz = kk * dz;
      v[3] = kx * dx; v[4] = ky * dy; v[5] = kz * dz;                 // dA00 dA11 dA22
      v[6] = kx * dy; v[7] = kx * dz; v[8] = ky * dz;                 // dA01 dA02 dA12
      v[9] = sx.w * e; v[10] = sg.x * e; v[11] = sg.y * e;            // d v
    }
    const unsigned peers = __match_any_sync(0xffffffffu, k);
    const int head = __ffs(peers) - 1, tail = 31 - __clz(peers);
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const bool need = lane - o >= head;
      if (!__any_sync(0xffffffffu, need)) break;
#pragma unroll
      for (int q = 0; q < 12; ++q) {
        const float t = __shfl_up_sync(0xffffffffu, v[q], o);
        if (need) v[q] += t;
      }
    }
    if (valid && ((tail - lane) & 3) == 0) {
      float* gp = grad + 12 * (int64_t)w.gid[k];
      red_add_v4(gp, v[0], v[1], v[2], v[3]);
      red_add_v4(gp + 4, v[4], v[5], v[6], v[7]);
      red_add_v4(gp + 8, v[8], v[9], v[10], v[11]);
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(256, 3) k_fwdbwd(FitArgs a) {
  __shared__ WarpSmem sm[kWarps];
  __shared__ double s_loss[kWarps][kMaxL];
  __shared__ unsigned long long s_cnt[kWarps][2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSmem& w = sm[wid];
  if (lane < kMaxL) s_loss[wid][lane] = 0.0;
  unsigned long long pairs_acc = 0, cand_acc = 0;
  const uint32_t n_work = *a.n_work;
  const float tau2 = a.tau2, eps = a.hdr_eps;
  const uint32_t gw = blockIdx.x * kWarps + wid, nw = gridDim.x * kWarps;

  for (uint32_t it = gw; it < n_work; it += nw) {
    const WorkItem wi = a.work[it];
    const int lo = (int)__ldg(a.csr_off + wi.cell);
    const int C = (int)__ldg(a.csr_off + wi.cell + 1) - lo;
    const bool act = lane < wi.count;
    float x = 0.f, y = 0.f, z = 0.f, xr = 0.f, xg = 0.f, xb = 0.f;
    if (act) {
      const float4 p = __ldcs(a.bin + 2 * (int64_t)(wi.start + lane));
      const float4 q = __ldcs(a.bin + 2 * (int64_t)(wi.start + lane) + 1);
      x = p.x; y = p.y; z = p.z; xr = p.w; xg = q.x; xb = q.y;
    }
    // ---------------- pass 1 (records the inside pairs while they fit)
    float y0 = 0.f, y1 = 0.f, y2 = 0.f;
    int np = 0, pbase = 0;
    const bool chunks_fit = C <= 32 * kMaxChunks;
    for (int cb = 0, c = 0; cb < C; cb += 32, ++c) {
      const int kc = min(32, C - cb);
      stage_chunk(w, a.csr_idx, a.rec, lo + cb, kc, lane);
      eval_chunk<true>(w, kc, act, x, y, z, tau2, y0, y1, y2, np, w.pkey, w.pe, pbase, kPairCap, lane);
      if (lane == 0 && c < kMaxChunks) w.cend[c] = (uint16_t)min(pbase, 0xFFFF);
    }
    const bool recorded = chunks_fit && pbase <= kPairCap;
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
    w.sxg[lane] = make_float4(x, y, z, g0);
    w.sg[lane] = make_float2(g1, g2);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ls += __shfl_xor_sync(0xffffffffu, ls, o);
      np += __shfl_xor_sync(0xffffffffu, np, o);
    }
    if (lane == 0) s_loss[wid][wi.level] += (double)ls;
    pairs_acc += (unsigned)np;
    cand_acc += (unsigned long long)wi.count * (unsigned long long)C;
    __syncwarp();
    if (np == 0) continue;
    // ---------------- pass 2
    if (recorded) {
      int pstart = 0;
      for (int cb = 0, c = 0; cb < C; cb += 32, ++c) {
        const int pend = w.cend[c];
        if (pend == pstart) continue;
        if (C > 32) stage_chunk(w, a.csr_idx, a.rec, lo + cb, min(32, C - cb), lane);
        chunk_pairs_bwd(w, pstart, pend, a.grad, lane);
        pstart = pend;
      }
    } else {
      // rare dense case: re-derive each chunk's pairs exactly as pass 1 did, in batches
      for (int cb = 0; cb < C; cb += 32) {
        const int kc = min(32, C - cb);
        stage_chunk(w, a.csr_idx, a.rec, lo + cb, kc, lane);
        const uint32_t lt = (1u << lane) - 1u;
        int pb = 0;
        for (int k = 0; k < kc; ++k) {
          const Rec g = rec_from(w, k);
          float dx, dy, dz, tx, ty, tz;
          const float Q = quad_form(g, x, y, z, dx, dy, dz, tx, ty, tz);
          const bool in = act && Q <= tau2;
          const uint32_t m = __ballot_sync(0xffffffffu, in);
          if (!m) continue;
          if (pb + 32 > kPairCap) { chunk_pairs_bwd(w, 0, pb, a.grad, lane); pb = 0; }
          if (in) {
            const int pos = pb + __popc(m & lt);
            w.pkey[pos] = (uint16_t)((k << 5) | lane);
            w.pe[pos] = ex2_approx(Q * kNegHalfLog2e);
          }
          pb += __popc(m);
          __syncwarp();
        }
        chunk_pairs_bwd(w, 0, pb, a.grad, lane);
      }
    }
  }
  if (lane == 0) { s_cnt[wid][0] = pairs_acc; s_cnt[wid][1] = cand_acc; }
  __syncthreads();
  double* part = a.partial + (int64_t)blockIdx.x * kPart;
  if (threadIdx.x < kMaxL) {
    double s = 0.0;
    for (int q = 0; q < kWarps; ++q) s += s_loss[q][threadIdx.x];
    part[threadIdx.x] = s;
  }
  if (threadIdx.x == 0) {
    unsigned long long p = 0, c = 0;
    for (int q = 0; q < kWarps; ++q) { p += s_cnt[q][0]; c += s_cnt[q][1]; }
    part[kMaxL] = (double)p;
    part[kMaxL + 1] = (double)c;
  }
}

__global__ void __launch_bounds__(256, 4) k_query(QueryArgs a) {
  __shared__ ChunkSmem sm[kWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  ChunkSmem& w = sm[wid];
  const uint32_t n_work = *a.n_work;
  const float tau2 = a.tau2;
  const uint32_t gw = blockIdx.x * kWarps + wid, nw = gridDim.x * kWarps;
  for (uint32_t it = gw; it < n_work; it += nw) {
    const WorkItem wi = a.work[it];
    const int lo = (int)__ldg(a.csr_off + wi.cell);
    const int C = (int)__ldg(a.csr_off + wi.cell + 1) - lo;
    const bool act = lane < wi.count;
    float x = 0.f, y = 0.f, z = 0.f;
    uint32_t idx = 0;
    if (act) {
      const float4 p = __ldcs(a.bin + wi.start + lane);
      x = p.x; y = p.y; z = p.z; idx = __float_as_uint(p.w);
    }
    float y0 = 0.f, y1 = 0.f, y2 = 0.f;
    int np = 0, pb = 0;
    for (int cb = 0; cb < C; cb += 32) {
      const int kc = min(32, C - cb);
      stage_chunk(w, a.csr_idx, a.rec, lo + cb, kc, lane);
      eval_chunk<false>(w, kc, act, x, y, z, tau2, y0, y1, y2, np, nullptr, nullptr, pb, 0, lane);
    }
    if (act) {
      __stcs(a.out + 3 * (int64_t)idx, y0); __stcs(a.out + 3 * (int64_t)idx + 1, y1);
      __stcs(a.out + 3 * (int64_t)idx + 2, y2);
    }
  }
}

static int persistent_grid(const void* fn, size_t smem) {
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 256, smem);
  return sms * std::max(per, 1);
}

int fwdbwd_grid() { static int g = persistent_grid((const void*)k_fwdbwd, 0); return g; }
int query_grid() { static int g = persistent_grid((const void*)k_query, 0); return g; }

void launch_fwdbwd(const FitArgs& a, int grid, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, "fwdbwd", s);
  k_fwdbwd<<<grid, 256, 0, s>>>(a);
}

void launch_query(const QueryArgs& a, int grid, cudaStream_t s, Profiler* prof) {
  ProfScope ps(prof, "query_fwd", s);
  k_query<<<grid, 256, 0, s>>>(a);
}

}  // namespace gsc
