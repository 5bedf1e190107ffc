// cull_scan.cu -- evaluation records (A2), exact conservative culling (C8) and the
// three-phase tiled exclusive scan used for both the sample bins and the culling CSR.
#include "common.cuh"
#include "kernels.h"
#include "record.cuh"

namespace gsc {

#ifndef GSC_REC_MINB
#define GSC_REC_MINB 1
#endif
__global__ void __launch_bounds__(128, GSC_REC_MINB) k_record_cull(int64_t G, const float* __restrict__ P, double tau, LevelGeom g, CullBufs cb,
                              DevState* st) {
  pdl_enter();
  if (cb.ovf) { cb.ovf = st->lovf; cb.ovf_cap = st->lovf_cap; }   // current buffers (DevState)
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < G; j += (int64_t)gridDim.x * blockDim.x) {
    float p[kNP];
#pragma unroll
    for (int k = 0; k < kNP; ++k) p[k] = P[k * G + j];
    record_and_count(j, p, tau, g, cb, st);
  }
}

// Fill the culling lists: entry of Gaussian j in cell c = off[c] + its rank from the counting
// pass.  The order inside a cell is atomic order (unspecified); gc_debug_cull sorts on export.
__global__ void k_cull_emit(int64_t G, CullBufs cb, const float* __restrict__ P, LevelGeom g,
                            const uint32_t* __restrict__ off, uint32_t cap, DevState* st,
                            const uint32_t* total, uint32_t* host_total) {
  pdl_enter();
  cb.lrec = st->lrec; cb.ovf = st->lovf; cb.ovf_cap = st->lovf_cap; cap = st->lcap;   // current buffers
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->ovf_next = 0u;                           // the counting pass is done
    if (host_total) *host_total = *total;        // entry count for the host's capacity guard
  }
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < G; j += (int64_t)gridDim.x * blockDim.x) {
    const uint4 r = cb.range[j];
    const int l = level_of_gaussian(g, j);
    const int32_t lo[3] = {(int32_t)(r.x & 0xFFFF), (int32_t)(r.y & 0xFFFF), (int32_t)(r.z & 0xFFFF)};
    const int32_t hi[3] = {(int32_t)(r.x >> 16), (int32_t)(r.y >> 16), (int32_t)(r.z >> 16)};
    // the record travels with the index: an evaluator's staging is then one load level
    // (list entry) instead of two (index, then record)
    const float4 ra = __ldg(cb.rec + 3 * j), rb = __ldg(cb.rec + 3 * j + 1), rc = __ldg(cb.rec + 3 * j + 2);
    const float4 rd = make_float4(__int_as_float((int32_t)j), 0.f, 0.f, 0.f);
    if (!(r.w >> 31)) {
      const int64_t dx = g.dims[l][0], dy = g.dims[l][1];
      const uint32_t mask = r.w;
      uint32_t pos[27];
#pragma unroll
      for (int q = 0; q < 27; ++q) {               // all gathers in flight before the stores
        pos[q] = 0xFFFFFFFFu;
        if ((mask >> q) & 1u) {
          const int qx = q % 3, qy = (q / 3) % 3, qz = q / 9;
          pos[q] = __ldg(off + g.coff[l] + ((int64_t)(lo[2] + qz) * dy + (lo[1] + qy)) * dx + (lo[0] + qx)) +
                   __ldg(cb.rank + 27 * j + q);
        }
      }
#pragma unroll
      for (int q = 0; q < 27; ++q) {
        if (pos[q] == 0xFFFFFFFFu) continue;
        if (pos[q] < cap) {
          st_v8(cb.lrec + 4 * (size_t)pos[q], ra, rb); st_v8(cb.lrec + 4 * (size_t)pos[q] + 2, rc, rd);
        } else {
          atomicOr(&st->csr_overflow, 1u);
        }
      }
      continue;
    }
    const uint32_t base = r.w & 0x7FFFFFFFu;
    const double m0 = P[P_MU * G + j], m1 = P[(P_MU + 1) * G + j], m2 = P[(P_MU + 2) * G + j];
    uint32_t i = 0;
    for_each_cell(lo, hi, m0, m1, m2, cb.rad2[j], g, l, [&](int64_t cell) {
      if (base + i < cb.ovf_cap) {
        const uint32_t pos = off[cell] + cb.ovf[base + i];
        if (pos < cap) {
          st_v8(cb.lrec + 4 * (size_t)pos, ra, rb); st_v8(cb.lrec + 4 * (size_t)pos + 2, rc, rd);
        } else {
          atomicOr(&st->csr_overflow, 1u);
        }
      }
      ++i;
    });
  }
}

// Grid of the record / emit passes of the culling rebuild.  They run beside the next call's
// sample ingest (deferred optimizer step), one latency-bound Gaussian per thread; a grid that
// fills every SM's register file (the old 4-5 CTAs per SM at cfg2) starves the ingest on the
// frame's critical path, so the grid is capped at GSC_CULL_GRID CTAs per SM unless that would
// give a thread more than GSC_CULL_PER_THREAD Gaussians (large caches keep their parallelism).
// Measured at cfg2 (same-box A/B, frame): 32 (no cap) 0.380 ms, 4: 0.378, 3: 0.374, 2: 0.372,
// 1: 0.414.  The emit pass is capped only while the scale group is frozen (lr 0, the paper's
// setting): with scales training (rotated anisotropic caches, the bench's general leg) the
// rebuild chain is longer and a capped emit delays the evaluators (general frame: both capped
// 0.455 ms, record only 0.445, neither 0.447).
#ifndef GSC_CULL_GRID
#define GSC_CULL_GRID 2
#endif
#ifndef GSC_CULL_PER_THREAD
#define GSC_CULL_PER_THREAD 2     // cfg4 (1.4 M Gaussians): 4.288 -> 4.285 ms, i.e. unchanged
#endif
static int cull_blocks(int64_t G, bool capped = true) {
  const int64_t need = (G + 127) / 128;
  if (!capped) return (int)std::max<int64_t>(1, std::min<int64_t>(need, 148 * 32));
  const int64_t floor_ = (G + 128 * GSC_CULL_PER_THREAD - 1) / (128 * GSC_CULL_PER_THREAD);
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, std::max<int64_t>(148 * GSC_CULL_GRID, floor_)));
}

// ---------------------------------------------------------------------------- scan
// Block-wide exclusive scan of (a, b) pairs, kScanThreads threads.
__device__ __forceinline__ uint2 block_excl_scan(uint2 v, uint2& total) {
  constexpr int kW = kScanThreads / 32;
  __shared__ uint2 wsum[kW];
  __shared__ uint2 tot_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint2 inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t a = __shfl_up_sync(0xffffffffu, inc.x, o), b = __shfl_up_sync(0xffffffffu, inc.y, o);
    if (lane >= o) { inc.x += a; inc.y += b; }
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint2 w = lane < kW ? wsum[lane] : make_uint2(0, 0);
    uint2 wi = w;
#pragma unroll
    for (int o = 1; o < kW; o <<= 1) {
      uint32_t a = __shfl_up_sync(0xffffffffu, wi.x, o), b = __shfl_up_sync(0xffffffffu, wi.y, o);
      if (lane >= o) { wi.x += a; wi.y += b; }
    }
    if (lane < kW) wsum[lane] = make_uint2(wi.x - w.x, wi.y - w.y);
    if (lane == kW - 1) tot_s = wi;
  }
  __syncthreads();
  uint2 base = wsum[warp];
  total = tot_s;
  __syncthreads();
  return make_uint2(base.x + inc.x - v.x, base.y + inc.y - v.y);
}

__device__ __forceinline__ void load8(const uint32_t* cnt, int64_t n, int64_t base, uint32_t c[8]) {
  if (base + 8 <= n && ((base & 3) == 0)) {
    uint4 a = *reinterpret_cast<const uint4*>(cnt + base), b = *reinterpret_cast<const uint4*>(cnt + base + 4);
    c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w; c[4] = b.x; c[5] = b.y; c[6] = b.z; c[7] = b.w;
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = (base + k < n) ? cnt[base + k] : 0u;
  }
}

static_assert(kRep >= 1 && kRep <= 8 && (8 % kRep) == 0, "a scan thread owns 8 / kRep whole cells");
constexpr int kCPT = 8 / kRep;        // cells per scan thread (sample bins)
// ch > 0: sample bins, whose counts come as kRep replicas per cell (one thread's 8 items =
// 8 / kRep whole cells, so that work items of <= ch samples are cut per cell); ch == 0:
// plain counts.  .x = samples, .y = work items.
__device__ __forceinline__ uint2 sum8(const uint32_t c[8], int ch) {
  uint2 s = make_uint2(0, 0);
#pragma unroll
  for (int k = 0; k < 8; ++k) s.x += c[k];
  if (ch) {
#pragma unroll
    for (int q = 0; q < kCPT; ++q) {
      uint32_t t = 0;
#pragma unroll
      for (int r = 0; r < kRep; ++r) t += c[q * kRep + r];
      s.y += (t + ch - 1) / ch;
    }
  }
  return s;
}

// Sample-bin counters are replica-major ([kRep][NC]: the replicas of a cell live in different
// L2 lines, so a hot cell's atomics spread over slices); a scan thread owns the kRep
// replicas of each of its 8 / kRep cells, visiting cells in order (item k = replica
// k % kRep of cell base / kRep + k / kRep).  Plain counters: 8 consecutive entries.
__device__ __forceinline__ int64_t entry(int ch, int64_t n, int64_t base, int k) {
  if (!ch) return base + k;
  const int64_t nc = n / kRep;
  return (int64_t)(k % kRep) * nc + base / kRep + k / kRep;
}

__device__ __forceinline__ void load_counts(const uint32_t* cnt, int64_t n, int ch, int64_t base, uint32_t c[8]) {
  if (!ch) { load8(cnt, n, base, c); return; }
  const int64_t nc = n / kRep;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int64_t cell = base / kRep + k / kRep;
    c[k] = cell < nc ? cnt[(int64_t)(k % kRep) * nc + cell] : 0u;
  }
}


// Single-pass scan with decoupled look-back.  Tiles are taken in ticket order (so every
// predecessor is already running); a tile publishes its aggregate, warp 0 walks back over
// its predecessors 256 at a time until it meets an inclusive prefix, publishes its own
// inclusive prefix, and the block then writes the exclusive offsets (and an optional copy
// used as atomic cursors) and, with ch > 0, one WorkItem per chunk of <= ch samples of every
// non-empty cell.  The counts are zeroed after reading (ready for the next call) and the last
// tile publishes the grand totals.  Tile status words (flag:2 | chunks:31 | count:31) are
// ping-ponged between two arrays by a launch parity, each tile clearing its slot in the
// array the next launch will use.
__device__ __forceinline__ unsigned long long st_pack(uint32_t f, uint2 v) {
  return ((unsigned long long)f << 62) | ((unsigned long long)(v.y & 0x7FFFFFFFu) << 31) | (v.x & 0x7FFFFFFFu);
}
__device__ __forceinline__ uint32_t st_flag(unsigned long long w) { return (uint32_t)(w >> 62); }
__device__ __forceinline__ uint2 st_val(unsigned long long w) {
  return make_uint2((uint32_t)(w & 0x7FFFFFFFu), (uint32_t)((w >> 31) & 0x7FFFFFFFu));
}

__global__ void __launch_bounds__(kScanThreads, GSC_SCAN_MINB) k_scan(uint32_t* __restrict__ cnt, int64_t n, int ch,
                                              unsigned long long* state, uint32_t* ctl, int ntiles,
                                              uint32_t* totals, uint32_t* excl, uint32_t* excl_copy,
                                              WorkItem* work, LevelGeom g) {
  pdl_enter();
  __shared__ int s_tile;
  __shared__ uint32_t s_par;
  __shared__ uint2 s_prefix;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    s_par = *(volatile uint32_t*)(ctl + 1);
    __threadfence();
    s_tile = (int)atomicAdd(ctl, 1u);
  }
  __syncthreads();
  const int tile = s_tile;
  const uint32_t par = s_par;
  unsigned long long* cur = state + (size_t)par * ntiles;
  unsigned long long* nxt = state + (size_t)(par ^ 1u) * ntiles;
  int64_t base = (int64_t)tile * kScanTile + threadIdx.x * 8;
  uint32_t c[8];
  load_counts(cnt, n, ch, base, c);
  if (!ch && base + 8 <= n && ((base & 3) == 0)) {
    *reinterpret_cast<uint4*>(cnt + base) = make_uint4(0, 0, 0, 0);
    *reinterpret_cast<uint4*>(cnt + base + 4) = make_uint4(0, 0, 0, 0);
  } else if (base < n) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { const int64_t e = entry(ch, n, base, k); if (e < n && base + k < n) cnt[e] = 0u; }
  }
  const uint2 s = sum8(c, ch);
  uint2 total;
  const uint2 ex = block_excl_scan(s, total);
  if (warp == 0) {
    uint2 prefix = make_uint2(0, 0);
    if (tile == 0) {
      if (lane == 0) atomicExch(cur, st_pack(2u, total));
    } else {
      if (lane == 0) atomicExch(cur + tile, st_pack(1u, total));
      // each round covers 256 predecessors (8 per lane, lane L owns j-8L .. j-8L-7, all
      // loads in flight together): a tile walks back over a few rounds at most, even when
      // every predecessor has only published its aggregate
      int j = tile - 1;
      for (;;) {
        unsigned long long w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int idx = j - 8 * lane - q;
          w[q] = idx >= 0 ? *(volatile unsigned long long*)(cur + idx) : st_pack(2u, make_uint2(0, 0));
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int idx = j - 8 * lane - q;
          while (st_flag(w[q]) == 0u) w[q] = *(volatile unsigned long long*)(cur + idx);
        }
        int qs = 8;                              // first inclusive prefix of this lane
#pragma unroll
        for (int q = 7; q >= 0; --q) if (st_flag(w[q]) == 2u) qs = q;
        const uint32_t inc = __ballot_sync(0xffffffffu, qs < 8);
        const int stop = inc ? __ffs(inc) - 1 : 32;
        uint2 v = make_uint2(0, 0);
        if (lane <= stop) {
          const int qe = lane < stop ? 7 : qs;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q <= qe) { const uint2 t = st_val(w[q]); v.x += t.x; v.y += t.y; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
          v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
        }
        prefix.x += v.x; prefix.y += v.y;
        if (inc) break;
        j -= 256;
      }
      if (lane == 0) atomicExch(cur + tile, st_pack(2u, make_uint2(prefix.x + total.x, prefix.y + total.y)));
    }
    if (lane == 0) { s_prefix = prefix; nxt[tile] = 0ull; }
  }
  __syncthreads();
  const uint2 tp = s_prefix;
  uint32_t off = tp.x + ex.x, woff = tp.y + ex.y;
  if (ch && s.x) {                       // the thread's 8 / kRep cells (kRep replicas each)
    uint32_t o = off;
#pragma unroll
    for (int cq = 0; cq < kCPT; ++cq) {
      uint32_t t = 0;
#pragma unroll
      for (int r = 0; r < kRep; ++r) t += c[cq * kRep + r];
      if (t) {
        const int64_t cell = base / kRep + cq;
        const int lvl = level_of_cell(g, cell);
        for (uint32_t q = 0; q * ch < t; ++q)
          work[woff++] = WorkItem{(int)cell, (int)(o + q * ch), (int)min((uint32_t)ch, t - q * ch), lvl};
      }
      o += t;
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int64_t i = base + k;
    if (i < n) {
      const int64_t e = entry(ch, n, base, k);
      excl[e] = off;
      if (excl_copy) excl_copy[e] = off;
      off += c[k];
    }
    if (i == n - 1) excl[n] = off;
  }
  if (tile == ntiles - 1 && threadIdx.x == 0) {
    totals[0] = tp.x + total.x; totals[1] = tp.y + total.y;
    totals[2] = 0u;                    // dynamic work counter of the consumer kernel
    ctl[0] = 0u;                       // tickets of the next launch
    ctl[1] = par ^ 1u;                 // every block of this launch has read the parity
  }
}

int scan_state_words(int64_t n) { return (int)(2 * ((n + kScanTile - 1) / kScanTile) + 2); }

void launch_scan(uint32_t* cnt, int64_t n, int ch, uint2* state, uint32_t* totals,
                 uint32_t* excl, uint32_t* excl_copy, WorkItem* work, const LevelGeom& g,
                 cudaStream_t s, Profiler* prof) {
  const int ntiles = (int)((n + kScanTile - 1) / kScanTile);
  unsigned long long* st = reinterpret_cast<unsigned long long*>(state);
  uint32_t* ctl = reinterpret_cast<uint32_t*>(st + 2 * ntiles);
  ProfScope ps(prof, "scan", s);
  launch_pdl(k_scan, dim3(ntiles), dim3(kScanThreads), 0, s, cnt, n, ch, st, ctl, ntiles, totals, excl, excl_copy, work, g);
}

void launch_record_cull(int64_t G, const float* P, double tau, const LevelGeom& g, CullBufs cb, DevState* st,
                        cudaStream_t s) {
  const int blocks = cull_blocks(G);
  launch_pdl(k_record_cull, dim3(blocks), dim3(128), 0, s, G, P, tau, g, cb, st);
}

void launch_cull_emit(int64_t G, CullBufs cb, const float* P, const LevelGeom& g, const uint32_t* off,
                      uint32_t cap, DevState* st, const uint32_t* total, uint32_t* host_total,
                      cudaStream_t s, Profiler* prof, bool capped) {
  ProfScope ps(prof, "cull_emit", s);
  const int blocks = cull_blocks(G, capped);
  launch_pdl(k_cull_emit, dim3(blocks), dim3(128), 0, s, G, cb, P, g, off, cap, st, total, host_total);
}

}  // namespace gsc
