// kernels.h -- host-side launchers of libgscache's kernels and the per-kernel profiler.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <utility>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "stats.cuh"

namespace gsc {

// CUDA-event timing of named kernels on their launch stream (bench.py roofline).
struct Profiler {
  bool enabled = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  std::map<std::string, std::pair<double, long long>> acc;   // name -> (ms, launches)

  cudaEvent_t get() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void flush() {  // caller synchronised
    for (auto& p : pending) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, p.second.first, p.second.second) == cudaSuccess) {
        auto& a = acc[p.first];
        a.first += ms;
        a.second += 1;
      }
      pool.push_back(p.second.first);
      pool.push_back(p.second.second);
    }
    pending.clear();
  }
  ~Profiler() {
    for (auto& p : pending) { cudaEventDestroy(p.second.first); cudaEventDestroy(p.second.second); }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

struct ProfScope {
  Profiler* p; const char* name; cudaStream_t s; cudaEvent_t a = nullptr, b = nullptr;
  ProfScope(Profiler* p_, const char* n, cudaStream_t s_) : p(p_), name(n), s(s_) {
    if (p && p->enabled) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(s, &cs);
      if (cs == cudaStreamCaptureStatusNone) { a = p->get(); b = p->get(); cudaEventRecord(a, s); }
    }
  }
  ~ProfScope() {
    if (a) { cudaEventRecord(b, s); p->pending.push_back({name, {a, b}}); }
  }
};

// Launch with the programmatic-stream-serialization attribute (PDL); kernels call pdl_enter().
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// cull_scan.cu
int scan_state_words(int64_t n);   // uint2 words of look-back state for an n-entry scan (zeroed)
void launch_scan(uint32_t* cnt, int64_t n, int ch, uint2* state, uint32_t* totals,
                 uint32_t* excl, uint32_t* excl_copy, WorkItem* work, const LevelGeom& g,
                 cudaStream_t s, Profiler* prof);
// Per-Gaussian culling state.  range[j] = (lo|hi<<16 per axis, w): w < 2^31 is the 27-bit
// membership mask of the <= 3x3x3 range box, the rank of Gaussian j in cell q of that box in
// rank[27 j + q]; w >= 2^31 marks a wider range whose ranks sit in ovf[w & 0x7fffffff ...] in
// visiting order.  Ranks come from the counting atomics, so the emit pass needs neither
// atomics nor the fp64 membership tests of the common case.
struct CullBufs {
  float4* rec; uint4* range; double* rad2; uint32_t* count; uint32_t* rank; uint32_t* ovf; uint32_t ovf_cap;
  float4* lrec;         // [cap][4] the culling lists: per entry the record (3 x float4) + (gid, 0, 0, 0)
  const uint32_t* need = nullptr;   // owner-computes: list Gaussian j only if bit `me` of need[j] is set
  int me = 0;
};
void launch_record_cull(int64_t G, const float* P, double tau, const LevelGeom& g, CullBufs cb, DevState* st,
                        cudaStream_t s);
// host_total (page-locked, nullable): receives the rebuild's entry count (written by the kernel)
void launch_cull_emit(int64_t G, CullBufs cb, const float* P, const LevelGeom& g, const uint32_t* off,
                      uint32_t cap, DevState* st, const uint32_t* total, uint32_t* host_total,
                      cudaStream_t s, Profiler* prof, bool capped = true);

// ingest.cu
struct IngestBufs {
  uint2* kr;            // [S] (global cell id or kInvalidKey, arrival rank inside the cell)
  uint32_t* cell_count; // [NC]
  float4* bin;          // binned samples, cell-major, one 32-B sector each: fit (x,y,z,r | g,b,-,-),
                        // query (x,y,z, original index as bits | -)
  int64_t nc;           // cells (counters are replica-major [kRep][nc])
  int64_t cap;          // samples the bins hold (GSC_CHECKED bounds)
};
void launch_keys(const float* pos, const int32_t* len, const float* rgb, int level_fixed,
                 int64_t S, const LevelGeom& g, IngestBufs b, cudaStream_t s, Profiler* prof);
void launch_keys_query(const float* pos, const int32_t* len, int level_fixed, int64_t S,
                       const LevelGeom& g, IngestBufs b, float* out, cudaStream_t s, Profiler* prof);
// 32-B bins: fit samples (x y z r | g b - -) if rgb != NULL, else lookups (x y z idx | - - - -).
void launch_scatter(const float* pos, const float* rgb, int64_t S, const uint32_t* cell_start,
                    IngestBufs b, cudaStream_t s, Profiler* prof);
void launch_levels_of(const uint2* kr, int64_t S, const LevelGeom& g, int32_t* out,
                      cudaStream_t s);

// fwdbwd.cu
// Per-level cell geometry in fp32 for the evaluators' reference point: a work item's samples
// and staged candidates are recentred on the centre of its cell (inside the grid even when
// samples lie far outside it, reading A17), so |x - x_ref| stays at the cell scale.
struct CellRef {
  float org[kMaxL][3], edge[kMaxL][3];
  int dx[kMaxL], dy[kMaxL], coff[kMaxL];
  float idx[kMaxL], idy[kMaxL];   // 1 / dx, 1 / dy (quotient estimates, corrected exactly)
};
CellRef cell_ref(const LevelGeom& g);
struct FitArgs {
  const WorkItem* work; const uint32_t* n_work;
  const uint32_t* csr_off; const DevState* st;   // st->lrec / st->lcap: the culling lists
  const float4* bin;
  float* grad;          // [G][12]
  double* partial;      // [grid][kMaxL + 2]: per-block loss sums, pairs, candidates
  float tau2, hdr_eps; int mode; int L;
  int lite;             // scale group frozen (lr 0) and no gradient export: skip dA on isotropic chunks
  CellRef ref;
  int64_t bin_cap, G;   // GSC_CHECKED bounds: binned samples, gradient rows

};
int fwdbwd_grid();
void launch_fwdbwd(const FitArgs& a, int grid, cudaStream_t s, Profiler* prof);
struct QueryArgs {
  const WorkItem* work; const uint32_t* n_work;
  const uint32_t* csr_off; const DevState* st;
  const float4* bin;
  float* out; float tau2;
  const float* att; const float* beta; const float* unb;   // optional f3 epilogue (caller order)
  CellRef ref;
  int64_t bin_cap, G, S;   // GSC_CHECKED bounds: binned lookups, Gaussians, outputs
};
int query_grid();
void launch_query(const QueryArgs& a, int grid, cudaStream_t s, Profiler* prof);

// adamw.cu
void launch_stats(double* partial, const LevelGeom& g, int64_t S, LvlStats* lvl, bool with_step, DevState* st,
                  const gc_hparams& hp, int L, gc_fit_stats* dev_stats, cudaStream_t s, Profiler* prof);
void launch_step_scalars(const LvlStats* lvl, DevState* st, const gc_hparams& hp, int L,
                         gc_fit_stats* dev_stats, cudaStream_t s);
// nonfinite: where the count of skipped non-finite gradient elements is added (the call's
// gc_fit_stats, or DevState::nonfinite when the step is deferred into the next call)
// raw_grad (nullable): [14][G] unnormalised raw-parameter gradients (the screen-space path, f1)
// used instead of the chain rule from the 12 coefficient gradients
void launch_adamw(int64_t G, float* P, float* M, float* V, float* grad, CullBufs cb, float* dbg_grad,
                  DevState* st, const gc_hparams& hp, const LevelGeom& g, unsigned long long* nonfinite,
                  cudaStream_t s, Profiler* prof, const float* raw_grad = nullptr,
                  const uint8_t* owner = nullptr, int me = 0, bool with_record = true, int64_t g_begin = 0,
                  int64_t g_end = -1);

// dense_tc.cu -- dense all-pairs evaluator on the tensor cores (row A8)
struct DenseArgs {
  const WorkItem* work; const uint32_t* n_work;   // items of <= 128 samples of one tile-grid cell
  const float4* bin;                               // binned lookups (x, y, z, caller index), stride 2
  const float4* rec;                               // [G][3] evaluation records
  int64_t goff[kMaxL + 1];
  CellRef ref;                                     // the tile grid's cell geometry (recentring)
  float* out; float tau2;
};
int dense_tc_grid();
void launch_dense_tc(const DenseArgs& a, int grid, cudaStream_t s, Profiler* prof);
struct DenseBwdArgs {                              // gc_fit_dense's backward (k_dense_bwd)
  const WorkItem* work; const uint32_t* n_work;
  const float4* bin; const float4* rec;
  int64_t goff[kMaxL + 1];
  CellRef ref;
  const float* g;        // [S][3] dL/dy_hat per sample (caller order), 0 for dropped samples
  float* grad;           // [G][12] coefficient gradients (dmu, dA00 dA11 dA22 dA01 dA02 dA12, dv)
  float tau2;
};
void launch_dense_bwd(const DenseBwdArgs& a, cudaStream_t s, Profiler* prof);
void launch_dense_loss(const float* pos, const int32_t* len, int fixed_level, int L, const float* rgb,
                       const float* yhat, int64_t S, float eps, int mode, float* g, double* partial, cudaStream_t s,
                       Profiler* prof);

// shard.cu -- level-sharded mode (gc_set_comm mode 1)
struct RoutePlan {
  int world, rank, L;
  int first[kMaxL];     // first rank of the group that owns level l
  int size[kMaxL];      // ranks in that group (level l's samples split round-robin over them)
  const int32_t* colrank;   // owner-computes (mode 2): rank of each grid column [kMaxL][512], else NULL
  LevelGeom geom;           // mode 2: the culling grids (a sample goes to the owner of its cell's column)
};
constexpr int kMaxCols = 512;
int level_plan(int L, const double* w, int W, int* group_of_level, int* first_rank, int* group_size);
// pass 0: count[d] += samples routed to rank d; pass 1: pack them into sendbuf at base[d] +
// (tile range reserved on cursor[d]); fit records 2 x float4 (x y z n | r g b 0) when rgb != NULL,
// lookups 1 x float4 (x y z n) + perm[slot] = caller index, dropped lookups -> out_zero 0.
void launch_route(const float* pos, const int32_t* len, const float* rgb, int level_fixed, int64_t S,
                  const RoutePlan& p, int pass, uint32_t* count, const uint32_t* base, uint32_t* cursor,
                  float4* sendbuf, uint32_t* perm, float* out_zero, cudaStream_t s, Profiler* prof);
void launch_unpack_routed(const float4* recv, int64_t R, bool fit, float* pos, int32_t* len, float* rgb,
                          cudaStream_t s);
void launch_unroute(const float* res, const uint32_t* perm, int64_t n, float* out, cudaStream_t s);
// owner-computes (mode 2): column slabs per level (host), owner of every Gaussian (by the column of
// its mean), the ranks that need each owned Gaussian (its C8 cell range's columns), the boundary
// list B = {j : needed by more than its owner} (deterministic scan), and row exchanges over B
void slab_plan(int L, const int64_t* goff, const float* means, const LevelGeom& g, int W, int32_t* colrank);
void launch_owner(const float* P, int64_t G, const LevelGeom& g, const int32_t* colrank, uint8_t* owner, cudaStream_t s);
void launch_need(const float* P, int64_t G, double tau, const LevelGeom& g, const int32_t* colrank,
                 const uint8_t* owner, int rank, uint32_t* need, cudaStream_t s);
void launch_boundary(const uint32_t* need, int64_t G, uint32_t* flag, uint32_t* bsums, uint32_t* total,
                     int32_t* idx, cudaStream_t s);
// mode 0: gather rows of AoS grads [G][12] into buf[n][12]; mode 1: scatter back.  params: planes
// [14][G]; gather zeroes rows this rank does not own (the all-reduce then yields the owner's row)
void launch_rows_grad(float* grad, float* buf, const int32_t* idx, int64_t n, int scatter, cudaStream_t s);
void launch_rows_param(float* P, int64_t G, float* buf, const int32_t* idx, int64_t n, const uint8_t* owner, int rank,
                       int scatter, cudaStream_t s);
// ZeRO data parallel (mode 3): this rank's slice [g0, g0 + n) of the 14 parameter planes into
// buf [14][np] (np >= n, zero padded), and all ranks' gathered slices [W][14][np] back into P
void launch_pack_slice(const float* P, int64_t G, int64_t g0, int64_t n, int64_t np, float* buf, cudaStream_t s);
void launch_unpack_slices(const float* buf, int W, int64_t np, float* P, int64_t G, cudaStream_t s);
void launch_zero_nonowned(float* t, int64_t n, int64_t base, const uint8_t* owner, int me, cudaStream_t s);
void launch_scan_u32(const uint32_t* in, int64_t n, uint32_t* bsums, uint32_t* total, uint32_t* out, cudaStream_t s);

// screen.cu -- screen-space evaluator (next row f1)
struct SCam {
  int W, H, TX, TY;
  float fx, fy, cx, cy, znear;
  float R[9], t[3];
};
SCam make_scam(const gc_camera& c);
struct ScreenBufs {
  float4 *pa = nullptr, *pb = nullptr, *pc = nullptr;   // [G] projection records
  int4* rect = nullptr;                                  // [G] tile rectangles
  uint32_t *touched = nullptr, *off = nullptr, *bsums = nullptr, *total = nullptr, *htotal = nullptr;
  uint64_t* key = nullptr; int64_t* val = nullptr; int64_t kv_cap = 0;   // (tile, depth) -> Gaussian
  uint2* ranges = nullptr; int64_t range_cap = 0;
  float *T = nullptr, *dLdC = nullptr; uint32_t* last = nullptr; int64_t img_cap = 0;
  float *g2d = nullptr, *raw = nullptr;                  // [G][12] partials, [14][G] raw gradients
  uint32_t *tcount = nullptr, *tcursor = nullptr, *tstart = nullptr, *tbsums = nullptr, *ttotal = nullptr,
           *tbig = nullptr, *htbig = nullptr;           // two-level tile sort
  int64_t tile_cap = 0;
};
cudaError_t launch_sproject(const float* P, int64_t G, int64_t g0, int64_t g1, const SCam& cam, ScreenBufs& b,
                            const LevelGeom& g, int lev0, int Lr, cudaStream_t s);
cudaError_t launch_skeys_sort(int64_t g0, int64_t g1, const LevelGeom& g, int lev0, int Lr, const SCam& cam,
                              ScreenBufs& b, int64_t npairs, int64_t Np, cudaStream_t s);
cudaError_t launch_tile_sort(int64_t g0, int64_t g1, const LevelGeom& g, int lev0, int Lr, const SCam& cam,
                             ScreenBufs& b, uint32_t* tcount, uint32_t* tcursor, uint32_t* tstart, uint32_t* tbsums,
                             uint32_t* ttotal, uint32_t* big, cudaStream_t s);
struct SLossArgs {             // Eq. 4 fused into the forward raster (gc_fit_image)
  const float* target; const uint8_t* valid; float eps; int mode; float* dLdC; double* partial;
};
cudaError_t launch_sraster(const SCam& cam, int Lr, ScreenBufs& b, float* out, float* outT, uint32_t* last,
                           const SLossArgs* loss, cudaStream_t s);
cudaError_t launch_sraster_bwd(const SCam& cam, int Lr, ScreenBufs& b, const float* outT, const uint32_t* last,
                               const float* dLdC, float* g2d, cudaStream_t s);
cudaError_t launch_sproject_bwd(const float* P, int64_t G, int64_t g0, int64_t g1, const SCam& cam,
                                const ScreenBufs& b, float* g2d, float* raw, cudaStream_t s);

// create.cu
void launch_gather_init(int64_t N0, const float* pos, const float* rgb, const float* log_scale,
                        const int64_t* src, int64_t G, float* P, float opacity_logit, cudaStream_t s);
cudaError_t launch_eq2_level(const float* P, int64_t G, int64_t base, int64_t n, double* dbar, double* capfl,
                             double zcap, double factor, float* Pw, cudaStream_t s);
void launch_pack(const float* P, int64_t G, int64_t base, int64_t n, float* out14, cudaStream_t s);
// src[j] of every Gaussian j: level 0 -> j (caller order), level l >= 1 -> pi[j - goff[l]], with
// pi = argsort splitmix64(seed + i) computed on the device (C7)
cudaError_t launch_level_sources(int64_t N0, uint64_t seed, const LevelGeom& g, int64_t* src, cudaStream_t s);
// ascending sort of (key, idx) pairs, Np = sort_kv_size(n) entries (pad with (~0, INT64_MAX))
int64_t sort_kv_size(int64_t n);
void launch_sort_kv(uint64_t* key, int64_t* idx, int64_t Np, cudaStream_t s);
// per level: lo[3], hi[3] of the means and mean (e^s0 + e^s1 + e^s2)/3 (fp64, fixed order)
cudaError_t launch_grid_stats(const float* P, int64_t G, const LevelGeom& g, double* out7L, cudaStream_t s);
void launch_unpack(const float* in14, int64_t G, int64_t base, int64_t n, float* P, cudaStream_t s);

}  // namespace gsc
