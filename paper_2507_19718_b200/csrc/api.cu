// api.cu -- the C ABI of include/gscache.h: handle, validation, memory, stream-ordered
// orchestration of the kernels, statistics, debug exports and NCCL data parallelism.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "kernels.h"
#include "stats.cuh"

using namespace gsc;

// NVTX range around every public entry point (header-only NVTX3: visible in Nsight Systems /
// ncu --nvtx, free when no tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static thread_local std::string g_err;

static gc_status fail(gc_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(e_ == cudaErrorMemoryAllocation ? GC_ERR_OOM : GC_ERR_CUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                          \
  } while (0)

#define NK(call)                                                                              \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess) return fail(GC_ERR_NCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
  } while (0)

template <class T>
static cudaError_t dalloc(T** p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc((void**)p, n * sizeof(T));
  return e;
}

struct Scratch {
  int64_t cap = 0;
  uint2* kr = nullptr;
  float4* bin = nullptr;
  uint32_t *cell_count = nullptr, *cell_start = nullptr, *totals = nullptr;
  uint2* tiles = nullptr;
  WorkItem* work = nullptr;
  // host-input staging, two sets: a call's upload may start while the previous call still
  // reads the other set (see stage_inputs)
  float *in_pos[2] = {nullptr, nullptr}, *in_rgb[2] = {nullptr, nullptr}, *out = nullptr;
  float *y = nullptr, *g = nullptr;       // gc_fit_dense: per-sample y_hat and dL/dy_hat [cap][3]
  int32_t* in_len[2] = {nullptr, nullptr};
  int set = 0;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  bool free_rec[2] = {false, false};
  void release() {
    void* ps[] = {kr, bin, cell_count, cell_start, totals, tiles, work, out, y, g,
                  in_pos[0], in_pos[1], in_rgb[0], in_rgb[1], in_len[0], in_len[1]};
    for (void* p : ps) if (p) cudaFree(p);
    for (cudaEvent_t e : {ev_copied[0], ev_copied[1], ev_free[0], ev_free[1]}) if (e) cudaEventDestroy(e);
    *this = Scratch();
  }
};

// Pageable caller stats: the device statistics are copied into the payload's own page-locked
// slot, then a stream host callback copies the slot into the caller's struct.  Every payload
// has its own slot and a completion event, so payloads in flight never share a buffer; a
// payload is reused only once its event (recorded after the callback) has completed.
struct StatsPayload {
  gc_fit_stats* dst = nullptr;
  gc_fit_stats* src = nullptr;        // page-locked slot
  cudaEvent_t done = nullptr;
  bool used = false;
};

struct gc_cache_s {
  int device = 0, sms = 148;
  LevelGeom geom{};
  int L = 0;
  int64_t G = 0, NC = 0;
  int64_t counts[kMaxL] = {0};
  gc_hparams hp{};
  float *P = nullptr, *M = nullptr, *V = nullptr, *grad = nullptr, *dbg = nullptr;
  float4* rec = nullptr;
  uint4* range = nullptr;
  double* rad2 = nullptr;
  uint32_t *csr_count = nullptr, *csr_off = nullptr, *csr_totals = nullptr;
  uint32_t *csr_rank = nullptr, *csr_ovf = nullptr;   // entry ranks from the counting pass (CullBufs)
  float4* csr_rec = nullptr;              // [csr_cap][4] list-ordered record copies (evaluator staging)
  uint2* csr_tiles = nullptr;
  uint32_t csr_cap = 0;
  DevState* st = nullptr;
  LvlStats* lvl = nullptr;
  gc_fit_stats* dstats = nullptr;
  uint32_t* hcsr = nullptr;         // pinned: entries of the latest culling-list rebuild (capacity guard)
  double* partial = nullptr;
  int fb_grid = 0, q_grid = 0;
  bool dbg_on = false;
  Scratch fit, qry;
  int64_t last_fit_S = -1;
  std::vector<StatsPayload*> payloads;    // all payloads (freed at destroy)
  std::vector<StatsPayload*> ring;        // the reusable ones of eager calls
  size_t payload_next = 0, captured_payloads = 0;
  uint64_t list_generation = 0;           // bumped by every reallocation of the culling lists
  // gc_fit_image leaves the evaluation records and culling lists of the world-space calls
  // stale (the screen path reads the parameters directly); the next call that reads them
  // rebuilds first (refresh_stale), so consecutive image steps skip the rebuild
  bool lists_stale = false;
  CellRef cref{};                         // fp32 cell geometry of the evaluators (CellRef)
  int dbg_mode = 0;                       // gc_debug_enable_grads: bit 0 raw grads, bit 1 coef grads
  float* dbg_coef = nullptr;              // [G][12] coefficient-gradient snapshot (bit 1)
  Profiler prof;
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  // level-sharded mode (gc_set_comm mode 1): plan, the group communicator of this rank's
  // levels, and the routing buffers (shard.cu)
  int mode = 0;
  RoutePlan plan{};
  ncclComm_t gcomm = nullptr;
  int glo = 0, ghi = 0, gsize = 1;        // this rank's group: levels [glo, ghi), gsize ranks
  double lvl_w[kMaxL] = {0};
  bool has_w = false;
  uint32_t *r_count = nullptr, *r_all = nullptr, *r_base = nullptr, *r_cursor = nullptr;
  uint32_t *h_all = nullptr, *h_base = nullptr;          // pinned
  float4 *r_send = nullptr, *r_recv = nullptr;
  int64_t r_send_cap = 0, r_recv_cap = 0;
  float *r_pos = nullptr, *r_rgb = nullptr, *r_res = nullptr, *r_back = nullptr;
  int32_t* r_len = nullptr;
  uint32_t* r_perm = nullptr;
  int64_t r_in_cap = 0, r_perm_cap = 0, r_send_cap_back = 0;
  std::vector<int64_t> rt_send, rt_recv, rt_soff, rt_roff;   // last routing's per-peer counts/offsets
  // owner-computes (gc_set_comm mode 2): column slabs, Gaussian owners, need masks, boundary list B
  int32_t* d_colrank = nullptr;
  uint8_t* d_owner = nullptr;
  uint32_t *d_need = nullptr, *d_flag = nullptr, *d_bsums = nullptr, *d_btotal = nullptr, *h_btotal = nullptr;
  int32_t* d_idxB = nullptr;
  float* xbuf = nullptr;
  int64_t nB = 0;
  // ZeRO data parallel (mode 3): slice of np Gaussians per rank, gather buffers
  int64_t zp = 0;
  float *zsend = nullptr, *zrecv = nullptr;
  ScreenBufs scr;                         // screen-space evaluator buffers (gc_render / gc_fit_image)
  LevelGeom dgeom{};                      // dense tensor-core evaluator (A8): tile grid, its
  CellRef dref{};                         // fp32 cell geometry and sample scratch
  int64_t dNC = 0;
  Scratch dns;
  int dense_grid = 0;
  float* pack_tmp = nullptr;
  int64_t pack_cap = 0;
  cudaStream_t side = nullptr;            // gc_fit_query: lookups run beside the fit samples' ingest
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // deferred optimizer step (gc_set_deferred_step): the AdamW step + culling rebuild of the
  // last fit, launched by the next call on `side2`, overlapping that call's ingest
  bool defer = false, pending = false;
  cudaStream_t side2 = nullptr;
  cudaEvent_t ev_fork2 = nullptr, ev_tail = nullptr;
  cudaStream_t cp = nullptr;          // uploads of host inputs (stage_inputs)
  cudaEvent_t ev_cpfork = nullptr;
};

// ------------------------------------------------------------------------- helpers
static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  return cs != cudaStreamCaptureStatusNone;
}

static gc_status check_sticky(gc_cache c) {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(GC_ERR_CUDA, "asynchronous CUDA error: %s", cudaGetErrorString(e));
  }
  return GC_OK;
}

static gc_status ensure_scratch(gc_cache c, Scratch& sc, int64_t S, bool fit, cudaStream_t s, int64_t nc = -1) {
  if (sc.cap >= S && sc.cell_count) return GC_OK;
  if (capturing(s)) return fail(GC_ERR_STATE, "scratch too small during graph capture; call gc_reserve first");
  CK(cudaDeviceSynchronize());
  sc.release();
  if (nc < 0) nc = c->NC;
  int64_t cap = std::max<int64_t>(S, 1024);
  const int64_t nbins = nc * kRep;                    // replicated per-cell counters
  int64_t work_cap = cap / kCH + std::min<int64_t>(cap, nc) + 2;
  CK(dalloc(&sc.kr, cap));
  CK(dalloc(&sc.bin, 2 * cap));                       // 32-B bins (full sectors) for both
  CK(dalloc(&sc.cell_count, nbins)); CK(dalloc(&sc.cell_start, nbins + 1));
  CK(cudaMemset(sc.cell_count, 0, sizeof(uint32_t) * nbins));   // kept zero by the scan
  CK(dalloc(&sc.tiles, scan_state_words(nbins)));
  CK(cudaMemset(sc.tiles, 0, sizeof(uint2) * scan_state_words(nbins)));
  CK(dalloc(&sc.totals, 4));
  CK(dalloc(&sc.work, work_cap));
  sc.cap = cap;
  return GC_OK;
}

static gc_status ensure_staging(Scratch& sc, bool need_pos, bool need_len, bool need_rgb, bool need_out) {
  for (int k = 0; k < 2; ++k) {
    if (need_pos && !sc.in_pos[k]) CK(dalloc(&sc.in_pos[k], 3 * sc.cap));
    if (need_len && !sc.in_len[k]) CK(dalloc(&sc.in_len[k], sc.cap));
    if (need_rgb && !sc.in_rgb[k]) CK(dalloc(&sc.in_rgb[k], 3 * sc.cap));
    if ((need_pos || need_len || need_rgb) && !sc.ev_copied[k]) {
      CK(cudaEventCreateWithFlags(&sc.ev_copied[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&sc.ev_free[k], cudaEventDisableTiming));
    }
  }
  if (need_out && !sc.out) CK(dalloc(&sc.out, 3 * sc.cap));
  return GC_OK;
}

// Host inputs of a call are uploaded on the handle's copy stream as soon as the call is made
// -- the host data is final at call time -- into one of two staging sets, so a frame's upload
// overlaps the previous frame's work (and the previous frame's downloads, the other PCIe
// direction); the call's stream waits for the copies before its first kernel, and releases the
// set after its last reader (mark_staging_free).  Under graph capture the copy stream is
// forked from the call's stream instead (no early start).
static gc_status stage_inputs(gc_cache c, Scratch& sc, cudaStream_t s, int64_t S, const float*& pos,
                              const int32_t*& len, const float*& rgb, int& set) {
  set = -1;
  const bool hpos = pos && !is_device_ptr(pos), hlen = len && !is_device_ptr(len), hrgb = rgb && !is_device_ptr(rgb);
  if (!(hpos || hlen || hrgb) || S == 0) return GC_OK;
  const bool cap_ = capturing(s);
  if (cap_ && ((hpos && !sc.in_pos[0]) || (hlen && !sc.in_len[0]) || (hrgb && !sc.in_rgb[0])))
    return fail(GC_ERR_STATE, "staging not reserved before capture");
  if (gc_status e = ensure_staging(sc, hpos, hlen, hrgb, false)) return e;
  set = sc.set ^= 1;
  if (cap_) {
    CK(cudaEventRecord(c->ev_cpfork, s));
    CK(cudaStreamWaitEvent(c->cp, c->ev_cpfork, 0));
  }
  if (sc.free_rec[set]) CK(cudaStreamWaitEvent(c->cp, sc.ev_free[set], 0));
  if (hpos) { CK(cudaMemcpyAsync(sc.in_pos[set], pos, sizeof(float) * 3 * S, cudaMemcpyHostToDevice, c->cp)); pos = sc.in_pos[set]; }
  if (hlen) { CK(cudaMemcpyAsync(sc.in_len[set], len, sizeof(int32_t) * S, cudaMemcpyHostToDevice, c->cp)); len = sc.in_len[set]; }
  if (hrgb) { CK(cudaMemcpyAsync(sc.in_rgb[set], rgb, sizeof(float) * 3 * S, cudaMemcpyHostToDevice, c->cp)); rgb = sc.in_rgb[set]; }
  CK(cudaEventRecord(sc.ev_copied[set], c->cp));
  CK(cudaStreamWaitEvent(s, sc.ev_copied[set], 0));
  return GC_OK;
}

static gc_status mark_staging_free(Scratch& sc, cudaStream_t s, int set) {
  if (set < 0) return GC_OK;
  CK(cudaEventRecord(sc.ev_free[set], s));
  sc.free_rec[set] = true;
  return GC_OK;
}

static CullBufs cull_bufs(gc_cache c) {
  CullBufs b{c->rec, c->range, c->rad2, c->csr_count, c->csr_rank, c->csr_ovf, c->csr_cap, c->csr_rec};
  if (c->mode == 2) { b.need = c->d_need; b.me = c->rank; }   // owner-computes: owned + halo only
  return b;
}

static gc_status rebuild_csr(gc_cache c, cudaStream_t s, bool recompute_records) {
  if (recompute_records) c->lists_stale = false;
  if (recompute_records) CK(cudaMemsetAsync(&c->st->csr_overflow, 0, sizeof(unsigned int), s));
  if (recompute_records)
    launch_record_cull(c->G, c->P, (double)c->hp.cutoff_sigma, c->geom, cull_bufs(c), c->st, s);
  launch_scan(c->csr_count, c->NC, 0, c->csr_tiles, c->csr_totals, c->csr_off, nullptr, nullptr, c->geom, s,
              &c->prof);
  // (the rebuild's entry count goes to pinned memory for the capacity guard of later calls)
  launch_cull_emit(c->G, cull_bufs(c), c->P, c->geom, c->csr_off, c->csr_cap, c->st, c->csr_totals, c->hcsr,
                   s, &c->prof, c->hp.lr[GC_SCALE] == 0.f);
  CK(cudaGetLastError());
  return GC_OK;
}

// Capacity guard of the culling lists, checked on the host at the start of each call from the
// entry count of the latest completed rebuild (pinned, no synchronisation).  Lists past half
// of their capacity (Gaussians growing, scale LR > 0) are reallocated to 4x their size; lists
// that overflowed (entries past the capacity were dropped, so the lookups / fit that used them
// were incomplete) are reallocated AND rebuilt, and the call reports GC_ERR_STATE once.
// The culling-list buffers as the kernels see them (DevState::lrec / lovf / lcap / lovf_cap).
static gc_status publish_lists(gc_cache c) {
  CK(cudaMemcpy(&c->st->lrec, &c->csr_rec, sizeof(float4*), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(&c->st->lovf, &c->csr_ovf, sizeof(uint32_t*), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(&c->st->lcap, &c->csr_cap, sizeof(uint32_t), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(&c->st->lovf_cap, &c->csr_cap, sizeof(uint32_t), cudaMemcpyHostToDevice));
  return GC_OK;
}

static gc_status refresh_stale(gc_cache c, cudaStream_t s) {
  if (!c->lists_stale) return GC_OK;
  CK(cudaMemsetAsync(c->csr_count, 0, sizeof(uint32_t) * c->NC, s));
  return rebuild_csr(c, s, true);
}

static gc_status csr_guard(gc_cache c, cudaStream_t s) {
  if (gc_status e = refresh_stale(c, s)) return e;
  const uint32_t total = *(volatile uint32_t*)c->hcsr;
  if (total <= c->csr_cap / 2 || capturing(s)) return GC_OK;
  const bool overflowed = total > c->csr_cap;
  CK(cudaDeviceSynchronize());
  const uint64_t cap = std::min<uint64_t>(4ull * total, 0x7FFFFFFFull);
  uint32_t* ovf = nullptr;
  float4* lrec = nullptr;
  CK(dalloc(&ovf, cap)); CK(dalloc(&lrec, 4 * cap));
  const uint64_t keep = std::min<uint64_t>(total, c->csr_cap);
  CK(cudaMemcpy(lrec, c->csr_rec, sizeof(float4) * 4 * keep, cudaMemcpyDeviceToDevice));
  cudaFree(c->csr_ovf); cudaFree(c->csr_rec);     // (kernels reach the lists through DevState,
  c->csr_ovf = ovf; c->csr_rec = lrec; c->csr_cap = (uint32_t)cap;   // captured graphs included)
  if (gc_status e = publish_lists(c)) return e;
  c->list_generation += 1;
  if (!overflowed) return GC_OK;
  CK(cudaMemset(&c->st->csr_overflow, 0, sizeof(unsigned int)));
  if (!c->pending) {                 // a pending deferred step rebuilds with the new capacity anyway
    CK(cudaMemset(c->csr_count, 0, sizeof(uint32_t) * c->NC));
    if (gc_status e = rebuild_csr(c, s, true)) return e;
  }
  return fail(GC_ERR_STATE, "culling lists overflowed (%u entries > capacity); capacity grown to %u and lists "
              "rebuilt -- the previous call's lookups / fit used incomplete lists", total, c->csr_cap);
}

static void CUDART_CB stats_cb(void* arg) {
  StatsPayload* p = (StatsPayload*)arg;
  memcpy(p->dst, p->src, sizeof(gc_fit_stats));
}

static gc_status new_payload(StatsPayload** out) {
  StatsPayload* p = new StatsPayload();
  if (cudaHostAlloc((void**)&p->src, sizeof(gc_fit_stats), cudaHostAllocDefault) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming) != cudaSuccess) {
    if (p->src) cudaFreeHost(p->src);
    delete p;
    return fail(GC_ERR_OOM, "stats payload allocation failed");
  }
  *out = p;
  return GC_OK;
}

static bool is_pinned_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeHost;
}

// Owner-computes (mode 2) halo refresh after the owners' step: every owner marks which ranks
// need each of its Gaussians (C8 range columns), the masks are summed over ranks (disjoint
// owners: the sum is each owner's mask), the boundary list B = {needed by more than the owner}
// is compacted in index order (identical on every rank), the owners' fresh parameter rows of B
// are summed into every rank (non-owners contribute 0), and the culling lists are rebuilt from
// the owned + halo Gaussians only.  One host synchronisation (|B| sizes the NCCL calls).
static gc_status refresh_halo(gc_cache c, cudaStream_t s) {
  const int64_t G = c->G;
  launch_need(c->P, G, (double)c->hp.cutoff_sigma, c->geom, c->d_colrank, c->d_owner, c->rank, c->d_need, s);
  NK(ncclAllReduce(c->d_need, c->d_need, (size_t)G, ncclUint32, ncclSum, c->comm, s));
  launch_boundary(c->d_need, G, c->d_flag, c->d_bsums, c->d_btotal, c->d_idxB, s);
  CK(cudaMemcpyAsync(c->h_btotal, c->d_btotal, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  c->nB = *c->h_btotal;
  if (c->nB > 0) {
    launch_rows_param(c->P, G, c->xbuf, c->d_idxB, c->nB, c->d_owner, c->rank, 0, s);
    NK(ncclAllReduce(c->xbuf, c->xbuf, (size_t)kNP * c->nB, ncclFloat32, ncclSum, c->comm, s));
    launch_rows_param(c->P, G, c->xbuf, c->d_idxB, c->nB, c->d_owner, c->rank, 1, s);
  }
  CK(cudaMemsetAsync(c->csr_count, 0, sizeof(uint32_t) * c->NC, s));
  return rebuild_csr(c, s, true);
}

// ZeRO data-parallel set-up (gc_set_comm mode 3, and gc_reinit under it): the gradient buffer
// padded to `world` equal slices (ncclReduceScatter counts), the all-gather buffers.
static gc_status setup_zero(gc_cache c) {
  const int world = c->world;
  const int64_t zp = (c->G + world - 1) / world;
  float* g = nullptr;
  CK(cudaDeviceSynchronize());
  CK(dalloc(&g, (size_t)12 * zp * world));
  CK(cudaMemset(g, 0, sizeof(float) * 12 * zp * world));
  if (c->grad) cudaFree(c->grad);
  c->grad = g;
  if (c->zsend) cudaFree(c->zsend);
  if (c->zrecv) cudaFree(c->zrecv);
  CK(dalloc(&c->zsend, (size_t)kNP * zp)); CK(dalloc(&c->zrecv, (size_t)kNP * zp * world));
  c->zp = zp;
  c->mode = 3;
  return GC_OK;
}

// Owner-computes set-up (gc_set_comm mode 2, and gc_reinit under it): column slabs from the
// current means (identical on every rank: same create arguments), owners, first halo refresh.
static gc_status setup_owner_computes(gc_cache c) {
  const int64_t G = c->G;
  std::vector<float> mx((size_t)G);
  CK(cudaMemcpy(mx.data(), c->P + (size_t)P_MU * G, sizeof(float) * G, cudaMemcpyDeviceToHost));
  std::vector<int32_t> cr((size_t)kMaxL * kMaxCols, 0);
  slab_plan(c->L, c->geom.goff, mx.data(), c->geom, c->world, cr.data());
  if (!c->d_colrank) {
    CK(dalloc(&c->d_colrank, (size_t)kMaxL * kMaxCols)); CK(dalloc(&c->d_owner, G)); CK(dalloc(&c->d_need, G));
    CK(dalloc(&c->d_flag, 2 * G)); CK(dalloc(&c->d_idxB, G)); CK(dalloc(&c->d_bsums, G / 4096 + 2));
    CK(dalloc(&c->d_btotal, 1)); CK(dalloc(&c->xbuf, (size_t)kNP * G));
    CK(cudaHostAlloc((void**)&c->h_btotal, sizeof(uint32_t), cudaHostAllocDefault));
  }
  CK(cudaMemcpy(c->d_colrank, cr.data(), sizeof(int32_t) * cr.size(), cudaMemcpyHostToDevice));
  launch_owner(c->P, G, c->geom, c->d_colrank, c->d_owner, 0);
  c->plan.colrank = c->d_colrank; c->plan.geom = c->geom;
  c->glo = 0; c->ghi = c->L; c->gsize = c->world;
  c->mode = 2;
  if (gc_status e = refresh_halo(c, 0)) return e;
  CK(cudaDeviceSynchronize());
  return GC_OK;
}

// The optimizer half of a fit: AdamW (+ next-step records and culling counts) and the
// culling-list rebuild.  `nonfinite` receives the skipped-gradient count.  Owner-computes: the
// owners step their Gaussians, then the halo refresh rebuilds the lists.
static gc_status launch_tail(gc_cache c, cudaStream_t s, unsigned long long* nonfinite) {
  if (c->mode == 3 && c->comm) {     // ZeRO: step this rank's slice, all-gather every slice's rows
    const int64_t g0 = std::min<int64_t>(c->G, (int64_t)c->rank * c->zp);
    const int64_t g1 = std::min<int64_t>(c->G, g0 + c->zp);
    launch_adamw(c->G, c->P, c->M, c->V, c->grad, cull_bufs(c), c->dbg_on ? c->dbg : nullptr, c->st, c->hp, c->geom,
                 nonfinite, s, &c->prof, nullptr, nullptr, 0, false, g0, g1);
    launch_pack_slice(c->P, c->G, g0, g1 - g0, c->zp, c->zsend, s);
    NK(ncclAllGather(c->zsend, c->zrecv, (size_t)kNP * c->zp, ncclFloat32, c->comm, s));
    launch_unpack_slices(c->zrecv, c->world, c->zp, c->P, c->G, s);
    launch_record_cull(c->G, c->P, (double)c->hp.cutoff_sigma, c->geom, cull_bufs(c), c->st, s);
    return rebuild_csr(c, s, false);
  }
  if (c->mode == 2 && c->comm) {
    launch_adamw(c->G, c->P, c->M, c->V, c->grad, cull_bufs(c), c->dbg_on ? c->dbg : nullptr, c->st, c->hp, c->geom,
                 nonfinite, s, &c->prof, nullptr, c->d_owner, c->rank, false);
    return refresh_halo(c, s);
  }
  launch_adamw(c->G, c->P, c->M, c->V, c->grad, cull_bufs(c), c->dbg_on ? c->dbg : nullptr, c->st, c->hp, c->geom,
               nonfinite, s, &c->prof);
  return rebuild_csr(c, s, false);
}

// A deferred step still pending is launched on side2, forked from `s`; the returned event
// (nullptr if nothing was pending) must be waited on before anything reads the parameters,
// records or culling lists.  Work on `s` that does not (sample ingest) overlaps it.
static gc_status fork_pending(gc_cache c, cudaStream_t s, cudaEvent_t* done) {
  *done = nullptr;
  if (!c->pending) return GC_OK;
  c->pending = false;
  CK(cudaEventRecord(c->ev_fork2, s));
  CK(cudaStreamWaitEvent(c->side2, c->ev_fork2, 0));
  if (gc_status e = launch_tail(c, c->side2, &c->st->nonfinite)) return e;
  CK(cudaEventRecord(c->ev_tail, c->side2));
  *done = c->ev_tail;
  return GC_OK;
}

// Completes a pending step on `s` (every call that reads or writes the cache state first).
static gc_status flush_pending(gc_cache c, cudaStream_t s) {
  cudaEvent_t ev = nullptr;
  if (gc_status e = fork_pending(c, s, &ev)) return e;
  if (ev) CK(cudaStreamWaitEvent(s, ev, 0));
  return GC_OK;
}

static gc_status emit_stats(gc_cache c, gc_fit_stats* user, cudaStream_t s) {
  if (!user) return GC_OK;
  if (is_pinned_host(user)) {          // page-locked: one async copy, no host callback
    CK(cudaMemcpyAsync(user, c->dstats, sizeof(gc_fit_stats), cudaMemcpyDeviceToHost, s));
    return GC_OK;
  }
  StatsPayload* p = nullptr;
  const size_t ring = 64;
  if (capturing(s)) {                  // a graph owns its payload for the handle's lifetime
    if (gc_status e = new_payload(&p)) return e;
    c->payloads.push_back(p);
    c->captured_payloads += 1;
  } else {
    const size_t live = c->payloads.size() - c->captured_payloads;
    if (live < ring) {
      if (gc_status e = new_payload(&p)) return e;
      c->payloads.push_back(p);
      c->ring.push_back(p);
    } else {
      p = c->ring[c->payload_next++ % ring];
      if (p->used) CK(cudaEventSynchronize(p->done));   // its previous callback has run
    }
  }
  p->dst = user; p->used = true;
  CK(cudaMemcpyAsync(p->src, c->dstats, sizeof(gc_fit_stats), cudaMemcpyDeviceToHost, s));
  CK(cudaLaunchHostFunc(s, stats_cb, p));
  CK(cudaEventRecord(p->done, s));
  return GC_OK;
}

// ------------------------------------------------------------ level-sharded routing (mode 1)
static bool routed(gc_cache c) { return (c->mode == 1 || c->mode == 2) && c->comm != nullptr; }

template <class T>
static gc_status grow(T** p, int64_t* cap, int64_t n) {
  if (*cap >= n && *p) return GC_OK;
  if (*p) { CK(cudaDeviceSynchronize()); cudaFree(*p); *p = nullptr; }
  const int64_t m = std::max<int64_t>(n + n / 4, 1024);
  CK(dalloc(p, m));
  *cap = m;
  return GC_OK;
}

// Sends every valid sample (fit: rgb != NULL) or lookup of this rank to the rank owning its
// level (RoutePlan) and receives the ones this rank owns: per-destination counts, one
// all-gather of the W x W count matrix, a host synchronisation (NCCL point-to-point sizes are
// host arguments: mode 1 is not graph-capturable), the pack pass, and one grouped
// ncclSend/ncclRecv.  The received records are unpacked into c->r_pos / r_len / r_rgb (*R).
static gc_status route_exchange(gc_cache c, cudaStream_t s, const float* pos, const int32_t* len, const float* rgb,
                                int level_fixed, int64_t S, float* out_zero, int64_t* R) {
  const int W = c->world, me = c->rank;
  const bool fit = rgb != nullptr;
  const int words = fit ? 2 : 1;                         // float4 per record
  CK(cudaMemsetAsync(c->r_count, 0, sizeof(uint32_t) * W, s));
  CK(cudaMemsetAsync(c->r_cursor, 0, sizeof(uint32_t) * W, s));
  launch_route(pos, len, rgb, level_fixed, S, c->plan, 0, c->r_count, nullptr, nullptr, nullptr, nullptr, nullptr, s,
               &c->prof);
  NK(ncclAllGather(c->r_count, c->r_all, (size_t)W, ncclUint32, c->comm, s));
  CK(cudaMemcpyAsync(c->h_all, c->r_all, sizeof(uint32_t) * W * W, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  c->rt_send.assign(W, 0); c->rt_recv.assign(W, 0); c->rt_soff.assign(W + 1, 0); c->rt_roff.assign(W + 1, 0);
  for (int p = 0; p < W; ++p) {
    c->rt_send[p] = c->h_all[(size_t)me * W + p];
    c->rt_recv[p] = c->h_all[(size_t)p * W + me];
    c->rt_soff[p + 1] = c->rt_soff[p] + c->rt_send[p];
    c->rt_roff[p + 1] = c->rt_roff[p] + c->rt_recv[p];
  }
  const int64_t n_send = c->rt_soff[W], n_recv = c->rt_roff[W];
  if (gc_status e = grow(&c->r_send, &c->r_send_cap, words * std::max<int64_t>(n_send, 1))) return e;
  if (gc_status e = grow(&c->r_recv, &c->r_recv_cap, words * std::max<int64_t>(n_recv, 1))) return e;
  if (!fit) { if (gc_status e = grow(&c->r_perm, &c->r_perm_cap, std::max<int64_t>(n_send, 1))) return e; }
  if (c->r_in_cap < n_recv || !c->r_pos) {
    CK(cudaDeviceSynchronize());
    for (void* p : {(void*)c->r_pos, (void*)c->r_rgb, (void*)c->r_len, (void*)c->r_res}) if (p) cudaFree(p);
    const int64_t m = std::max<int64_t>(n_recv + n_recv / 4, 1024);
    CK(dalloc(&c->r_pos, 3 * m)); CK(dalloc(&c->r_rgb, 3 * m)); CK(dalloc(&c->r_len, m)); CK(dalloc(&c->r_res, 3 * m));
    c->r_in_cap = m;
  }
  for (int p = 0; p < W; ++p) c->h_base[p] = (uint32_t)c->rt_soff[p];
  CK(cudaMemcpyAsync(c->r_base, c->h_base, sizeof(uint32_t) * W, cudaMemcpyHostToDevice, s));
  launch_route(pos, len, rgb, level_fixed, S, c->plan, 1, nullptr, c->r_base, c->r_cursor, c->r_send, c->r_perm,
               out_zero, s, &c->prof);
  const size_t rb = sizeof(float4) * words;
  NK(ncclGroupStart());
  for (int p = 0; p < W; ++p) {
    if (c->rt_send[p]) NK(ncclSend(c->r_send + words * c->rt_soff[p], rb * c->rt_send[p], ncclUint8, p, c->comm, s));
    if (c->rt_recv[p]) NK(ncclRecv(c->r_recv + words * c->rt_roff[p], rb * c->rt_recv[p], ncclUint8, p, c->comm, s));
  }
  NK(ncclGroupEnd());
  launch_unpack_routed(c->r_recv, n_recv, fit, c->r_pos, c->r_len, c->r_rgb, s);
  CK(cudaGetLastError());
  *R = n_recv;
  return GC_OK;
}

// Lookup results of the routed points (c->r_res, receive order) back to their source ranks,
// then into caller order.
static gc_status route_return(gc_cache c, cudaStream_t s, float* out) {
  const int W = c->world;
  const int64_t n_send = c->rt_soff[W];
  if (gc_status e = grow(&c->r_back, &c->r_send_cap_back, 3 * std::max<int64_t>(n_send, 1))) return e;
  NK(ncclGroupStart());
  for (int p = 0; p < W; ++p) {
    if (c->rt_recv[p]) NK(ncclSend(c->r_res + 3 * c->rt_roff[p], 3 * c->rt_recv[p], ncclFloat32, p, c->comm, s));
    if (c->rt_send[p]) NK(ncclRecv(c->r_back + 3 * c->rt_soff[p], 3 * c->rt_send[p], ncclFloat32, p, c->comm, s));
  }
  NK(ncclGroupEnd());
  launch_unroute(c->r_back, c->r_perm, n_send, out, s);
  CK(cudaGetLastError());
  return GC_OK;
}


// ---------------------------------------------------------------------------- ABI
extern "C" {

const char* gc_last_error(void) { return g_err.c_str(); }

const char* gc_status_string(gc_status s) {
  switch (s) {
    case GC_OK: return "GC_OK";
    case GC_ERR_ARG: return "GC_ERR_ARG";
    case GC_ERR_STATE: return "GC_ERR_STATE";
    case GC_ERR_CUDA: return "GC_ERR_CUDA";
    case GC_ERR_OOM: return "GC_ERR_OOM";
    case GC_ERR_NCCL: return "GC_ERR_NCCL";
    case GC_ERR_UNSUPPORTED: return "GC_ERR_UNSUPPORTED";
  }
  return "?";
}

void gc_default_hparams(gc_hparams* hp) {
  if (!hp) return;
  memset(hp, 0, sizeof *hp);
  const float lr[GC_NGROUPS] = {1.16e-3f, 1e-3f, 1.25e-2f, 0.f, 1.5e-1f};
  const float wd[GC_NGROUPS] = {0.f, 1e-2f, 1e-2f, 1e-2f, 1e-2f};
  for (int k = 0; k < GC_NGROUPS; ++k) { hp->lr[k] = lr[k]; hp->weight_decay[k] = wd[k]; }
  hp->beta1 = 0.9f; hp->beta2 = 0.999f; hp->adam_eps = 1e-8f; hp->hdr_eps = 0.01f;
  hp->loss_grad_mode = 0; hp->lr_schedule = 1; hp->cutoff_sigma = 3.f; hp->init_opacity = 0.1f;
  hp->init_scale_factor = 0.5f; hp->init_zcap = 2.f; hp->cell_edge_scale = 1.f;
}


// The R1 grid rule (host fp64) from the per-level statistics of k_grid_stats (lo[3], hi[3],
// mean e^s): level AABB + 5 % of its diagonal; cell edge = scale * 2 tau mean(e^s); dims =
// clamp(ceil(extent / edge), 1, 512), total cells <= 2^22 per level.
static void build_grid(LevelGeom& g, const std::vector<double>& hstat, int L, double tau, const gc_hparams& hp) {
  g.coff[0] = 0;
  for (int l = 0; l < L; ++l) {
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) { lo[a] = hstat[7 * l + a]; hi[a] = hstat[7 * l + 3 + a]; }
    const double ms = hstat[7 * l + 6];
    double diag = std::sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) + (hi[2] - lo[2]) * (hi[2] - lo[2]));
    double ext[3];
    for (int a = 0; a < 3; ++a) {
      double pad = 0.05 * diag + 1e-6;
      lo[a] -= pad; hi[a] += pad;
      ext[a] = hi[a] - lo[a];
    }
    int32_t dims[3];
    const int fixed = hp.cells_per_axis[l];
    if (fixed > 0) {
      for (int a = 0; a < 3; ++a) dims[a] = std::min(fixed, 4096);
    } else {
      const double esc = hp.cell_edge_scale > 0.f ? (double)hp.cell_edge_scale : 1.0;
      double edge = std::isfinite(tau) ? esc * 2.0 * tau * ms : INFINITY;
      if (!(edge > 0.0)) edge = INFINITY;
      for (int it = 0; it < 200; ++it) {
        int64_t prod = 1;
        for (int a = 0; a < 3; ++a) {
          double d = std::isfinite(edge) ? std::ceil(ext[a] / edge) : 1.0;
          dims[a] = (int32_t)std::max(1.0, std::min(512.0, d));
          prod *= dims[a];
        }
        if (prod <= (int64_t)1 << 22) break;
        edge *= 1.25;
      }
    }
    for (int a = 0; a < 3; ++a) {
      g.origin[l][a] = lo[a];
      g.dims[l][a] = dims[a];
      g.inv_cell[l][a] = (double)dims[a] / ext[a];
      g.edge[l][a] = 1.0 / g.inv_cell[l][a];
    }
    g.coff[l + 1] = g.coff[l] + (int64_t)dims[0] * dims[1] * dims[2];
  }
  for (int l = L; l < kMaxL; ++l) g.coff[l + 1] = g.coff[L];
}

static gc_status create_impl(gc_cache c, const int64_t* counts, const float* init_pos,
                             const float* init_rgb, const float* init_log_scale, uint64_t seed) {
  CK(cudaSetDevice(c->device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, c->device));
  if (prop.major < 10) return fail(GC_ERR_UNSUPPORTED, "device %d is sm_%d%d; libgscache is built for sm_100a only", c->device, prop.major, prop.minor);
  c->sms = prop.multiProcessorCount;
  const int L = c->L;
  const int64_t N0 = counts[0];
  c->geom.L = L;
  c->geom.goff[0] = 0;
  for (int l = 0; l < L; ++l) { c->counts[l] = counts[l]; c->geom.goff[l + 1] = c->geom.goff[l] + counts[l]; }
  for (int l = L; l < kMaxL; ++l) c->geom.goff[l + 1] = c->geom.goff[L];
  const int64_t G = c->G = c->geom.goff[L];

  cudaStream_t s = 0;
  CK(dalloc(&c->P, kNP * G)); CK(dalloc(&c->M, kNP * G)); CK(dalloc(&c->V, kNP * G));
  CK(cudaMemset(c->M, 0, sizeof(float) * kNP * G)); CK(cudaMemset(c->V, 0, sizeof(float) * kNP * G));
  CK(dalloc(&c->rec, 3 * G)); CK(dalloc(&c->grad, 12 * G)); CK(dalloc(&c->range, G)); CK(dalloc(&c->rad2, G));
  CK(cudaMemset(c->grad, 0, sizeof(float) * 12 * G));
  CK(dalloc(&c->st, 1)); CK(cudaMemset(c->st, 0, sizeof(DevState)));
  {
    DevState h0;
    memset(&h0, 0, sizeof h0);
    for (int l = 0; l < kMaxL; ++l) { h0.b1pow[l] = 1.0; h0.b2pow[l] = 1.0; }
    h0.owned = 0xFFFFFFFFu;
    CK(cudaMemcpy(c->st, &h0, sizeof h0, cudaMemcpyHostToDevice));
  }
  CK(dalloc(&c->lvl, 1)); CK(dalloc(&c->dstats, 1)); CK(cudaMemset(c->dstats, 0, sizeof(gc_fit_stats)));
  CK(cudaHostAlloc((void**)&c->hcsr, sizeof(uint32_t), cudaHostAllocDefault));
  *c->hcsr = 0u;

  // inputs (host or device)
  float *dpos = nullptr, *drgb = nullptr, *dls = nullptr;
  int64_t* dsrc = nullptr;
  CK(dalloc(&dpos, 3 * N0)); CK(dalloc(&drgb, 3 * N0)); CK(dalloc(&dsrc, G));
  CK(cudaMemcpy(dpos, init_pos, sizeof(float) * 3 * N0, cudaMemcpyDefault));
  CK(cudaMemcpy(drgb, init_rgb, sizeof(float) * 3 * N0, cudaMemcpyDefault));
  if (init_log_scale) { CK(dalloc(&dls, 3 * N0)); CK(cudaMemcpy(dls, init_log_scale, sizeof(float) * 3 * N0, cudaMemcpyDefault)); }
  // permutation pi = stable argsort(splitmix64(seed + i)) (C7) and the source point of every
  // Gaussian, on the device (next row f2)
  CK(launch_level_sources(N0, seed, c->geom, dsrc, s));
  const double p0 = (double)c->hp.init_opacity;
  const float logit = (float)std::log(p0 / (1.0 - p0));
  launch_gather_init(N0, dpos, drgb, dls, dsrc, G, c->P, logit, s);
  CK(cudaGetLastError());
  if (!init_log_scale) {   // Eq. 2 per level
    double *dbar = nullptr, *capfl = nullptr;
    CK(dalloc(&dbar, N0)); CK(dalloc(&capfl, 2));
    for (int l = 0; l < L; ++l)
      CK(launch_eq2_level(c->P, G, c->geom.goff[l], counts[l], dbar, capfl, (double)c->hp.init_zcap,
                          (double)c->hp.init_scale_factor, c->P, s));
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaFree(dbar); cudaFree(capfl);
  }
  CK(cudaDeviceSynchronize());
  cudaFree(dpos); cudaFree(drgb); cudaFree(dsrc); if (dls) cudaFree(dls);

  // culling grids (R1 auto rule): level AABB + 5% of its diagonal; cell edge = 2 tau mean(e^s);
  // dims = clamp(ceil(extent/edge), 1, 512), total cells <= 2^22 per level.  The per-level
  // AABB and mean e^s are reduced on the device (k_grid_stats, fixed order), 7 doubles per
  // level come back; the rule's few flops run here in fp64.
  double* dstat = nullptr;
  CK(dalloc(&dstat, 7 * L));
  CK(launch_grid_stats(c->P, G, c->geom, dstat, s));
  std::vector<double> hstat(7 * (size_t)L);
  CK(cudaMemcpy(hstat.data(), dstat, sizeof(double) * 7 * L, cudaMemcpyDeviceToHost));
  cudaFree(dstat);
  const double tau = (double)c->hp.cutoff_sigma;
  build_grid(c->geom, hstat, L, tau, c->hp);
  c->NC = c->geom.coff[L];
  // the dense tensor-core evaluator's tile grid (row A8): the same rule at tau = 3 whatever the
  // cut-off, so that its tiles stay spatially compact (recentring) even for tau = infinity
  c->dgeom = c->geom;
  if (!std::isfinite(tau)) build_grid(c->dgeom, hstat, L, 3.0, c->hp);
  c->dNC = c->dgeom.coff[L];
  c->dref = cell_ref(c->dgeom);
  if (c->NC >= (int64_t)1 << 31) return fail(GC_ERR_ARG, "culling grid too large (%lld cells)", (long long)c->NC);

  // records + culling lists; exact size of the first CSR sets the list capacity
  CK(dalloc(&c->csr_count, c->NC)); CK(dalloc(&c->csr_off, c->NC + 1));
  CK(dalloc(&c->csr_tiles, scan_state_words(c->NC)));
  CK(cudaMemset(c->csr_tiles, 0, sizeof(uint2) * scan_state_words(c->NC)));
  CK(dalloc(&c->csr_totals, 4));
  CK(cudaMemset(c->csr_count, 0, sizeof(uint32_t) * c->NC));
  CK(dalloc(&c->csr_rank, 27 * G));
  // sizing pass (counts only; no wide-range rank slots yet): the first CSR's exact size sets
  // the list capacity, then the real counting pass runs with full slot capacity
  launch_record_cull(G, c->P, tau, c->geom, CullBufs{c->rec, c->range, c->rad2, c->csr_count, c->csr_rank, nullptr, 0u, nullptr},
                     c->st, s);
  launch_scan(c->csr_count, c->NC, 0, c->csr_tiles, c->csr_totals, c->csr_off, nullptr, nullptr, c->geom, s, nullptr);
  CK(cudaGetLastError());
  uint32_t total = 0;
  CK(cudaMemcpy(&total, c->csr_totals, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  uint64_t cap = std::max<uint64_t>(4ull * total, (uint64_t)total + (1u << 20));
  cap = std::min<uint64_t>(cap, 0x7FFFFFFFull);
  c->csr_cap = (uint32_t)cap;
  CK(dalloc(&c->csr_ovf, c->csr_cap));
  CK(dalloc(&c->csr_rec, 4 * (size_t)c->csr_cap));
  if (gc_status e = publish_lists(c)) return e;
  CK(cudaMemset(&c->st->csr_overflow, 0, sizeof(unsigned int)));
  CK(cudaMemset(&c->st->ovf_next, 0, sizeof(unsigned int)));
  launch_record_cull(G, c->P, tau, c->geom, cull_bufs(c), c->st, s);
  launch_scan(c->csr_count, c->NC, 0, c->csr_tiles, c->csr_totals, c->csr_off, nullptr, nullptr, c->geom, s, nullptr);
  launch_cull_emit(G, cull_bufs(c), c->P, c->geom, c->csr_off, c->csr_cap, c->st, c->csr_totals, c->hcsr, s,
                   nullptr);
  CK(cudaGetLastError());

  // per device (the dynamic shared-memory attribute and the occupancy-based persistent grid
  // sizes are properties of this device, set after cudaSetDevice above)
  c->fb_grid = fwdbwd_grid();
  c->q_grid = query_grid();
  if (c->fb_grid <= 0 || c->q_grid <= 0) return fail(GC_ERR_CUDA, "evaluator configuration failed");
  c->cref = cell_ref(c->geom);
  // a deferred optimizer step (side2) gates the next fwd/bwd and lookups: its CTAs go first
  // while it shares the GPU with the sample ingest (measured -7 us/frame; favouring either
  // half of the frame instead was slower)
  int prio_lo = 0, prio_hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithPriority(&c->side2, cudaStreamNonBlocking, prio_hi));
  CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_fork2, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_tail, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_cpfork, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&c->cp, cudaStreamNonBlocking));
  CK(dalloc(&c->partial, (size_t)kSlots * kPart));
  CK(cudaMemset(c->partial, 0, sizeof(double) * kSlots * kPart));
  CK(cudaDeviceSynchronize());
  return GC_OK;
}

static void free_screen(ScreenBufs& b) {
  for (void* p : {(void*)b.pa, (void*)b.pb, (void*)b.pc, (void*)b.rect, (void*)b.touched, (void*)b.off,
                  (void*)b.bsums, (void*)b.total, (void*)b.key, (void*)b.val, (void*)b.ranges,
                  (void*)b.T, (void*)b.dLdC, (void*)b.last, (void*)b.g2d, (void*)b.raw, (void*)b.tcount,
                  (void*)b.tcursor, (void*)b.tstart, (void*)b.tbsums, (void*)b.ttotal, (void*)b.tbig})
    if (p) cudaFree(p);
  if (b.htotal) cudaFreeHost(b.htotal);
  if (b.htbig) cudaFreeHost(b.htbig);
  b = ScreenBufs();
}

static void destroy_impl(gc_cache c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  void* ps[] = {c->P, c->M, c->V, c->grad, c->dbg, c->rec, c->range, c->rad2, c->csr_count, c->csr_off, c->csr_rank,
                c->csr_ovf,
                c->csr_totals, c->csr_rec, c->csr_tiles, c->st, c->lvl, c->dstats, c->partial, c->pack_tmp};
  for (void* p : ps) if (p) cudaFree(p);
  if (c->hcsr) cudaFreeHost(c->hcsr);
  c->fit.release();
  c->qry.release();
  c->dns.release();
  for (auto* p : c->payloads) {
    if (p->src) cudaFreeHost(p->src);
    if (p->done) cudaEventDestroy(p->done);
    delete p;
  }
  if (c->dbg_coef) cudaFree(c->dbg_coef);
  free_screen(c->scr);
  if (c->gcomm) ncclCommDestroy(c->gcomm);
  if (c->comm) ncclCommDestroy(c->comm);
  for (void* p : {(void*)c->r_count, (void*)c->r_all, (void*)c->r_base, (void*)c->r_cursor, (void*)c->r_send,
                  (void*)c->r_recv, (void*)c->r_pos, (void*)c->r_rgb, (void*)c->r_res, (void*)c->r_back,
                  (void*)c->r_len, (void*)c->r_perm})
    if (p) cudaFree(p);
  if (c->h_all) cudaFreeHost(c->h_all);
  if (c->h_base) cudaFreeHost(c->h_base);
  for (void* p : {(void*)c->d_colrank, (void*)c->d_owner, (void*)c->d_need, (void*)c->d_flag, (void*)c->d_idxB,
                  (void*)c->d_bsums, (void*)c->d_btotal, (void*)c->xbuf})
    if (p) cudaFree(p);
  if (c->h_btotal) cudaFreeHost(c->h_btotal);
  if (c->zsend) cudaFree(c->zsend);
  if (c->zrecv) cudaFree(c->zrecv);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->side2) cudaStreamDestroy(c->side2);
  for (cudaEvent_t e : {c->ev_fork, c->ev_join, c->ev_fork2, c->ev_tail, c->ev_cpfork}) if (e) cudaEventDestroy(e);
  if (c->cp) cudaStreamDestroy(c->cp);
  delete c;
}

gc_status gc_create(int levels, const int64_t* counts, const float* init_pos, const float* init_rgb,
                    const float* init_log_scale, uint64_t seed, const gc_hparams* hp, int device,
                    gc_cache* out) {
  NvtxRange nvtx_("gc_create");
  if (!out) return fail(GC_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (levels < 1 || levels > GC_MAX_LEVELS) return fail(GC_ERR_ARG, "levels must be in [1, %d]", GC_MAX_LEVELS);
  if (!counts || !init_pos || !init_rgb) return fail(GC_ERR_ARG, "counts/init_pos/init_rgb must not be NULL");
  for (int l = 0; l < levels; ++l) {
    if (counts[l] < 1) return fail(GC_ERR_ARG, "counts[%d] < 1", l);
    if (l > 0 && counts[l] > counts[l - 1]) return fail(GC_ERR_ARG, "counts must be non-increasing");
  }
  int64_t G = 0;
  for (int l = 0; l < levels; ++l) G += counts[l];
  if (G >= (int64_t)1 << 31) return fail(GC_ERR_ARG, "too many Gaussians");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return fail(GC_ERR_UNSUPPORTED, "no CUDA device %d (libgscache has no CPU fallback)", device);
  }
  gc_cache c = new gc_cache_s();
  c->device = device;
  c->L = levels;
  if (hp) c->hp = *hp; else gc_default_hparams(&c->hp);
  if (!(c->hp.cutoff_sigma > 0.f)) { delete c; return fail(GC_ERR_ARG, "cutoff_sigma must be > 0"); }
  gc_status st = create_impl(c, counts, init_pos, init_rgb, init_log_scale, seed);
  if (st != GC_OK) { std::string e = g_err; destroy_impl(c); g_err = e; return st; }
  *out = c;
  return GC_OK;
}

// Re-initialisation on a morphology change (sec.5, next row f2): a new point cloud
// for the same level counts, as gc_create would build it, on the existing handle -- its
// communicator, mode, deferral, level weights and statistics ring are kept, everything the
// point cloud determines (parameters, AdamW state, schedule, grids, culling lists, scratch)
// is rebuilt.  Implemented as a fresh internal create whose state replaces the old one.
gc_status gc_reinit(gc_cache c, const float* init_pos, const float* init_rgb, const float* init_log_scale,
                    uint64_t seed) {
  NvtxRange nvtx_("gc_reinit");
  if (!c || !init_pos || !init_rgb) return fail(GC_ERR_ARG, "NULL handle or init points");
  CK(cudaSetDevice(c->device));
  if (gc_status e = flush_pending(c, 0)) return e;
  CK(cudaDeviceSynchronize());
  gc_cache n = new gc_cache_s();
  n->device = c->device; n->L = c->L; n->hp = c->hp;
  if (gc_status e = create_impl(n, c->counts, init_pos, init_rgb, init_log_scale, seed)) {
    std::string msg = g_err; destroy_impl(n); g_err = msg; return e;
  }
  // release the old point-cloud state
  for (void* p : {(void*)c->P, (void*)c->M, (void*)c->V, (void*)c->grad, (void*)c->dbg, (void*)c->dbg_coef,
                  (void*)c->rec, (void*)c->range, (void*)c->rad2, (void*)c->csr_count, (void*)c->csr_off,
                  (void*)c->csr_rank, (void*)c->csr_ovf, (void*)c->csr_totals, (void*)c->csr_rec, (void*)c->csr_tiles,
                  (void*)c->st, (void*)c->lvl, (void*)c->dstats, (void*)c->partial})
    if (p) cudaFree(p);
  if (c->hcsr) cudaFreeHost(c->hcsr);
  c->fit.release();
  c->qry.release();
  c->dns.release();
  free_screen(c->scr);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->side2) cudaStreamDestroy(c->side2);
  if (c->cp) cudaStreamDestroy(c->cp);
  for (cudaEvent_t e : {c->ev_fork, c->ev_join, c->ev_fork2, c->ev_tail, c->ev_cpfork}) if (e) cudaEventDestroy(e);
  // take the new one
#define GSC_TAKE(f) do { c->f = n->f; n->f = decltype(n->f){}; } while (0)
  GSC_TAKE(geom); GSC_TAKE(G); GSC_TAKE(NC); GSC_TAKE(sms); GSC_TAKE(dgeom); GSC_TAKE(dref); GSC_TAKE(dNC);
  GSC_TAKE(P); GSC_TAKE(M); GSC_TAKE(V); GSC_TAKE(grad); GSC_TAKE(rec); GSC_TAKE(range); GSC_TAKE(rad2);
  GSC_TAKE(csr_count); GSC_TAKE(csr_off); GSC_TAKE(csr_totals); GSC_TAKE(csr_rank); GSC_TAKE(csr_ovf);
  GSC_TAKE(csr_rec); GSC_TAKE(csr_tiles); GSC_TAKE(csr_cap); GSC_TAKE(st); GSC_TAKE(lvl); GSC_TAKE(dstats);
  GSC_TAKE(hcsr); GSC_TAKE(partial); GSC_TAKE(fb_grid); GSC_TAKE(q_grid); GSC_TAKE(cref);
  GSC_TAKE(side); GSC_TAKE(side2); GSC_TAKE(ev_fork); GSC_TAKE(ev_join); GSC_TAKE(ev_fork2); GSC_TAKE(ev_tail);
  GSC_TAKE(cp); GSC_TAKE(ev_cpfork);
#undef GSC_TAKE
  delete n;
  c->dbg = nullptr; c->dbg_coef = nullptr;
  c->pending = false;
  c->last_fit_S = -1;
  c->list_generation += 1;
  if (c->mode == 1) {                 // this rank's levels under the level-sharded plan
    unsigned int owned = 0u;
    for (int l = c->glo; l < c->ghi; ++l) owned |= 1u << l;
    CK(cudaMemcpy(&c->st->owned, &owned, sizeof owned, cudaMemcpyHostToDevice));
  }
  if (c->dbg_mode) { const int m = c->dbg_mode; c->dbg_mode = 0; if (gc_status e = gc_debug_enable_grads(c, m)) return e; }
  if (c->mode == 3) { if (gc_status e = setup_zero(c)) return e; }   // the new gradient buffer, padded
  if (c->mode == 2) {                 // owner-computes: slabs and owners of the new cloud (collective)
    if (c->d_colrank) {
      for (void* p : {(void*)c->d_colrank, (void*)c->d_owner, (void*)c->d_need, (void*)c->d_flag, (void*)c->d_idxB,
                      (void*)c->d_bsums, (void*)c->d_btotal, (void*)c->xbuf})
        if (p) cudaFree(p);
      if (c->h_btotal) cudaFreeHost(c->h_btotal);
      c->d_colrank = nullptr; c->d_owner = nullptr; c->d_need = nullptr; c->d_flag = nullptr; c->d_idxB = nullptr;
      c->d_bsums = nullptr; c->d_btotal = nullptr; c->xbuf = nullptr; c->h_btotal = nullptr;
    }
    if (gc_status e = setup_owner_computes(c)) return e;
  }
  return GC_OK;
}

gc_status gc_destroy(gc_cache c) {
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  destroy_impl(c);
  return GC_OK;
}

gc_status gc_reserve(gc_cache c, int64_t S_fit, int64_t S_query) {
  if (!c || S_fit < 0 || S_query < 0) return fail(GC_ERR_ARG, "bad arguments");
  CK(cudaSetDevice(c->device));
  if (S_fit > 0) { gc_status s = ensure_scratch(c, c->fit, S_fit, true, 0); if (s) return s; }
  if (S_query > 0) { gc_status s = ensure_scratch(c, c->qry, S_query, false, 0); if (s) return s; }
  if (S_fit > 0) { gc_status s = ensure_staging(c->fit, true, true, true, false); if (s) return s; }
  if (S_query > 0) { gc_status s = ensure_staging(c->qry, true, true, false, true); if (s) return s; }
  return GC_OK;
}

// Epilogue inputs of a query: device pointers are used in place, host ones staged into
// temporary device buffers (freed by release_epilogue after the stream drains).
struct Epilogue {
  const float* src[3] = {nullptr, nullptr, nullptr};
  float* dev[3] = {nullptr, nullptr, nullptr};
  gc_status stage(const float* att, const float* beta, const float* unb, int64_t S, cudaStream_t s) {
    const float* ep[3] = {att, beta, unb};
    const int64_t n[3] = {3 * S, S, 3 * S};
    for (int k = 0; k < 3; ++k) {
      src[k] = ep[k];
      if (!ep[k]) continue;
      if (is_device_ptr(ep[k])) { dev[k] = const_cast<float*>(ep[k]); continue; }
      if (capturing(s)) return fail(GC_ERR_STATE, "host epilogue buffers cannot be captured");
      CK(dalloc(&dev[k], n[k]));
      CK(cudaMemcpyAsync(dev[k], ep[k], sizeof(float) * n[k], cudaMemcpyHostToDevice, s));
    }
    return GC_OK;
  }
  gc_status release(cudaStream_t s) {
    for (int k = 0; k < 3; ++k)
      if (dev[k] && dev[k] != src[k]) { CK(cudaStreamSynchronize(s)); cudaFree(dev[k]); dev[k] = nullptr; }
    return GC_OK;
  }
};


// One optimisation step (gc_fit, and the fit half of gc_fit_query: `join`, if set, is waited
// on before the optimizer step so that the lookups forked off beside it read pre-step
// parameters).  `tail_ev`: a pending deferred step already forked by the caller (else this
// call forks it itself); its ingest overlaps that step.  With deferral on, this call's own
// optimizer step is left pending.
static gc_status fit_impl(gc_cache c, const float* pos, const int32_t* path_len, const float* rgb, int64_t S,
                          gc_stream stream, gc_fit_stats* stats, cudaEvent_t join = nullptr,
                          bool forked = false, cudaEvent_t tail_ev = nullptr) {
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  if (S < 0 || S >= ((int64_t)1 << 31)) return fail(GC_ERR_ARG, "S out of range");
  if (S > 0 && (!pos || !path_len || !rgb)) return fail(GC_ERR_ARG, "NULL sample pointer");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  if (gc_status e = check_sticky(c)) return e;
  if (gc_status e = ensure_scratch(c, c->fit, std::max<int64_t>(S, 1), true, s)) return e;
  if (!forked) {
    if (gc_status e = csr_guard(c, s)) return e;
    if (gc_status e = fork_pending(c, s, &tail_ev)) return e;
  }
  const int64_t S_in = S;             // this rank's input (n_in of the statistics)
  if (routed(c)) {                    // level-sharded: fit the samples of this rank's levels
    if (capturing(s)) return fail(GC_ERR_STATE, "level-sharded mode (gc_set_comm mode 1) is not graph-capturable");
    int set0 = -1;
    if (gc_status e = stage_inputs(c, c->fit, s, S, pos, path_len, rgb, set0)) return e;
    int64_t R = 0;
    if (gc_status e = route_exchange(c, s, pos, path_len, rgb, -1, S, nullptr, &R)) return e;
    if (gc_status e = mark_staging_free(c->fit, s, set0)) return e;
    pos = c->r_pos; path_len = c->r_len; rgb = c->r_rgb; S = R;
    if (gc_status e = ensure_scratch(c, c->fit, std::max<int64_t>(S, 1), true, s)) return e;
  }
  Scratch& F = c->fit;
  int set = -1;
  if (gc_status e = stage_inputs(c, F, s, S, pos, path_len, rgb, set)) return e;
  IngestBufs b{F.kr, F.cell_count, F.bin, c->NC, F.cap};
  if (S > 0) launch_keys(pos, path_len, rgb, -1, S, c->geom, b, s, &c->prof);
  launch_scan(F.cell_count, c->NC * kRep, kCH, F.tiles, F.totals, F.cell_start, nullptr, F.work, c->geom, s, &c->prof);
  if (S > 0) launch_scatter(pos, rgb, S, F.cell_start, b, s, &c->prof);
  if (gc_status e = mark_staging_free(F, s, set)) return e;
  if (tail_ev) CK(cudaStreamWaitEvent(s, tail_ev, 0));     // the previous step is complete
  FitArgs fa;
  fa.work = F.work; fa.n_work = F.totals + 1; fa.csr_off = c->csr_off; fa.st = c->st;
  fa.bin = F.bin;
  fa.grad = c->grad; fa.partial = c->partial;
  const float tau = c->hp.cutoff_sigma;
  fa.tau2 = tau * tau; fa.hdr_eps = c->hp.hdr_eps; fa.mode = c->hp.loss_grad_mode; fa.L = c->L;
  fa.lite = (c->hp.lr[GC_SCALE] == 0.f && !c->dbg_on) ? 1 : 0;
  fa.ref = c->cref;
  fa.bin_cap = F.cap; fa.G = c->G;
  const bool dp = c->comm != nullptr;
  // with the step deferred nothing after the statistics launch touches the call's stats, so a
  // page-locked caller struct is written by the kernel itself (mapped through UVA): no copy
  const bool stats_in_place = c->defer && stats && is_pinned_host(stats);
  gc_fit_stats* out_stats = stats_in_place ? stats : c->dstats;
  launch_fwdbwd(fa, c->fb_grid, s, &c->prof);
  // single GPU: the step scalars ride in the statistics launch
  launch_stats(c->partial, c->geom, S_in, c->lvl, !dp, c->st, c->hp, c->L, out_stats, s, &c->prof);
  if (dp && c->mode == 0) {         // data parallel: one sum over ranks of grads + level stats
    NK(ncclGroupStart());
    NK(ncclAllReduce(c->grad, c->grad, (size_t)12 * c->G, ncclFloat32, ncclSum, c->comm, s));
    NK(ncclAllReduce(c->lvl, c->lvl, sizeof(LvlStats) / sizeof(double), ncclFloat64, ncclSum, c->comm, s));
    NK(ncclGroupEnd());
    launch_step_scalars(c->lvl, c->st, c->hp, c->L, out_stats, s);
  } else if (dp && c->mode == 3) {  // ZeRO data parallel: reduce-scatter, each rank sums its slice
    NK(ncclGroupStart());
    NK(ncclReduceScatter(c->grad, c->grad + (size_t)12 * c->rank * c->zp, (size_t)12 * c->zp, ncclFloat32, ncclSum,
                         c->comm, s));
    NK(ncclAllReduce(c->lvl, c->lvl, sizeof(LvlStats) / sizeof(double), ncclFloat64, ncclSum, c->comm, s));
    NK(ncclGroupEnd());
    launch_step_scalars(c->lvl, c->st, c->hp, c->L, out_stats, s);
  } else if (dp && c->mode == 2) {  // owner-computes: only the boundary Gaussians' gradients meet
    // (an interior Gaussian is touched by its owner's samples alone); level statistics over all ranks
    if (c->nB > 0) {
      launch_rows_grad(c->grad, c->xbuf, c->d_idxB, c->nB, 0, s);
      NK(ncclAllReduce(c->xbuf, c->xbuf, (size_t)12 * c->nB, ncclFloat32, ncclSum, c->comm, s));
      launch_rows_grad(c->grad, c->xbuf, c->d_idxB, c->nB, 1, s);
    }
    NK(ncclAllReduce(c->lvl, c->lvl, sizeof(LvlStats) / sizeof(double), ncclFloat64, ncclSum, c->comm, s));
    launch_step_scalars(c->lvl, c->st, c->hp, c->L, out_stats, s);
  } else if (dp) {                  // level-sharded: gradients of the group's levels summed over
    // the group (its members split those levels' samples); level statistics summed over all
    // ranks, so every rank sees the global k_l and the same schedule step t
    const int64_t g0 = c->geom.goff[c->glo], g1 = c->geom.goff[c->ghi];
    if (c->gcomm && c->gsize > 1)
      NK(ncclAllReduce(c->grad + 12 * g0, c->grad + 12 * g0, (size_t)12 * (g1 - g0), ncclFloat32, ncclSum, c->gcomm, s));
    NK(ncclAllReduce(c->lvl, c->lvl, sizeof(LvlStats) / sizeof(double), ncclFloat64, ncclSum, c->comm, s));
    launch_step_scalars(c->lvl, c->st, c->hp, c->L, out_stats, s);
  }
  if (c->dbg_mode & 2)   // debug snapshot of the coefficient gradients the optimizer will read
    CK(cudaMemcpyAsync(c->dbg_coef, c->grad, sizeof(float) * 12 * c->G, cudaMemcpyDeviceToDevice, s));
  if (join) CK(cudaStreamWaitEvent(s, join, 0));
  if (c->defer && c->mode != 2 && c->mode != 3) {   // (modes 2, 3: the tail holds collectives, never deferred)
    c->pending = true;                // AdamW + culling rebuild run at the start of the next call
  } else {
    if (gc_status e = launch_tail(c, s, reinterpret_cast<unsigned long long*>(&c->dstats->nonfinite_grads))) return e;
  }
  if (!stats_in_place) { if (gc_status e = emit_stats(c, stats, s)) return e; }
  CK(cudaGetLastError());
  c->last_fit_S = routed(c) ? -1 : S;   // (gc_debug_levels: caller order only without routing)
  return GC_OK;
}

gc_status gc_fit(gc_cache c, const float* pos, const int32_t* path_len, const float* rgb, int64_t S,
                 gc_stream stream, gc_fit_stats* stats) {
  NvtxRange nvtx_("gc_fit");
  return fit_impl(c, pos, path_len, rgb, S, stream, stats);
}

static gc_status query_impl(gc_cache c, const float* pos, const int32_t* path_len, int level, int64_t S,
                            const float* att, const float* beta, const float* unb, float* out_rgb,
                            gc_stream stream, bool forked = false, cudaEvent_t tail_ev = nullptr);

// The frame's lookups run on the handle's side stream, forked from `stream` and joined back
// before the optimizer step, so their ingest and evaluation overlap the fit samples' ingest
// and fwd/bwd (independent work; both read the pre-step parameters and culling lists).
gc_status gc_fit_query(gc_cache c, const float* pos, const int32_t* path_len, const float* rgb, int64_t S,
                       const float* qpos, const int32_t* qlen, int qlevel, int64_t S_q, const float* attenuation,
                       const float* beta, const float* unbiased_rgb, float* out_rgb, gc_stream stream,
                       gc_fit_stats* stats) {
  NvtxRange nvtx_("gc_fit_query");
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  if (S_q < 0 || S_q >= ((int64_t)1 << 31)) return fail(GC_ERR_ARG, "S_q out of range");
  if (S_q > 0 && (!qpos || !out_rgb)) return fail(GC_ERR_ARG, "NULL query pointer");
  if (S_q > 0 && !qlen && (qlevel < 0 || qlevel >= c->L)) return fail(GC_ERR_ARG, "qlevel %d not in [0, %d)", qlevel, c->L);
  if (S_q == 0) return fit_impl(c, pos, path_len, rgb, S, stream, stats);
  if (routed(c)) {                    // level-sharded: lookups (routed), then the fit (routed)
    if (gc_status e = query_impl(c, qpos, qlen, qlevel, S_q, attenuation, beta, unbiased_rgb, out_rgb, stream))
      return e;
    return fit_impl(c, pos, path_len, rgb, S, stream, stats);
  }
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  cudaEvent_t tail_ev = nullptr;      // a deferred previous step overlaps both halves' ingest
  if (gc_status e = csr_guard(c, s)) return e;
  if (gc_status e = fork_pending(c, s, &tail_ev)) return e;
  CK(cudaEventRecord(c->ev_fork, s));
  CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
  const gc_status qs = query_impl(c, qpos, qlen, qlevel, S_q, attenuation, beta, unbiased_rgb, out_rgb,
                                  (gc_stream)c->side, true, tail_ev);
  CK(cudaEventRecord(c->ev_join, c->side));     // always joined (keeps a capture well-formed)
  if (qs != GC_OK) {
    CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    if (tail_ev) CK(cudaStreamWaitEvent(s, tail_ev, 0));
    return qs;
  }
  return fit_impl(c, pos, path_len, rgb, S, stream, stats, c->ev_join, true, tail_ev);
}

gc_status gc_query(gc_cache c, const float* pos, const int32_t* path_len, int level, int64_t S,
                   float* out_rgb, gc_stream stream) {
  NvtxRange nvtx_("gc_query");
  return query_impl(c, pos, path_len, level, S, nullptr, nullptr, nullptr, out_rgb, stream);
}

gc_status gc_query_radiance(gc_cache c, const float* pos, const int32_t* path_len, int level,
                            int64_t S, const float* attenuation, const float* beta,
                            const float* unbiased_rgb, float* out_rgb, gc_stream stream) {
  NvtxRange nvtx_("gc_query_radiance");
  return query_impl(c, pos, path_len, level, S, attenuation, beta, unbiased_rgb, out_rgb, stream);
}

static gc_status query_impl(gc_cache c, const float* pos, const int32_t* path_len, int level, int64_t S,
                            const float* att, const float* beta, const float* unb, float* out_rgb,
                            gc_stream stream, bool forked, cudaEvent_t tail_ev) {
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  if (S < 0 || S >= ((int64_t)1 << 31)) return fail(GC_ERR_ARG, "S out of range");
  if (S > 0 && (!pos || !out_rgb)) return fail(GC_ERR_ARG, "NULL pointer");
  if (S == 0 && !routed(c)) return GC_OK;      // (level-sharded calls are collective)
  if (!path_len && (level < 0 || level >= c->L)) return fail(GC_ERR_ARG, "level %d not in [0, %d)", level, c->L);
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  if (gc_status e = check_sticky(c)) return e;
  if (gc_status e = ensure_scratch(c, c->qry, std::max<int64_t>(S, 1), false, s)) return e;
  if (!forked) {
    if (gc_status e = csr_guard(c, s)) return e;
    if (gc_status e = fork_pending(c, s, &tail_ev)) return e;
  }
  const int64_t S_caller = S;
  Scratch& Q = c->qry;
  const bool hout = !is_device_ptr(out_rgb);
  if (hout) {
    if (capturing(s) && !Q.out) return fail(GC_ERR_STATE, "staging not reserved before capture");
    if (gc_status e = ensure_staging(Q, false, false, false, true)) return e;
  }
  int set = -1;
  const float* no_rgb = nullptr;
  if (gc_status e = stage_inputs(c, Q, s, S, pos, path_len, no_rgb, set)) return e;
  float* dout = hout ? Q.out : out_rgb;
  float* caller_out = nullptr;       // level-sharded: results come back into caller order here
  if (routed(c)) {
    if (capturing(s)) return fail(GC_ERR_STATE, "level-sharded mode (gc_set_comm mode 1) is not graph-capturable");
    if (att || beta || unb) return fail(GC_ERR_UNSUPPORTED, "the gc_query_radiance epilogue is not available in level-sharded mode");
    int64_t R = 0;
    if (gc_status e = route_exchange(c, s, pos, path_len, nullptr, path_len ? -1 : level, S, dout, &R)) return e;
    if (gc_status e = mark_staging_free(Q, s, set)) return e;
    set = -1;
    caller_out = dout;
    pos = c->r_pos; path_len = c->r_len; level = -1; S = R;
    dout = c->r_res;
    if (gc_status e = ensure_scratch(c, c->qry, std::max<int64_t>(S, 1), false, s)) return e;
  }
  IngestBufs b{Q.kr, Q.cell_count, Q.bin, c->NC, Q.cap};
  launch_keys_query(pos, path_len, path_len ? -1 : level, S, c->geom, b, dout, s, &c->prof);
  launch_scan(Q.cell_count, c->NC * kRep, kCH, Q.tiles, Q.totals, Q.cell_start, nullptr, Q.work, c->geom, s, &c->prof);
  launch_scatter(pos, nullptr, S, Q.cell_start, b, s, &c->prof);
  if (gc_status e = mark_staging_free(Q, s, set)) return e;
  QueryArgs qa;
  qa.work = Q.work; qa.n_work = Q.totals + 1; qa.csr_off = c->csr_off; qa.st = c->st;
  qa.bin = Q.bin; qa.out = dout;
  Epilogue ep;
  if (gc_status e = ep.stage(att, beta, unb, S, s)) return e;
  qa.att = ep.dev[0]; qa.beta = ep.dev[1]; qa.unb = ep.dev[2];
  const float tau = c->hp.cutoff_sigma;
  qa.tau2 = tau * tau;
  qa.ref = c->cref;
  qa.bin_cap = Q.cap; qa.G = c->G; qa.S = S;
  if (tail_ev) CK(cudaStreamWaitEvent(s, tail_ev, 0));     // a deferred step is complete
  launch_query(qa, c->q_grid, s, &c->prof);
  if (caller_out) {
    if (gc_status e = route_return(c, s, caller_out)) return e;
    dout = caller_out; S = S_caller;
  }
  if (hout) CK(cudaMemcpyAsync(out_rgb, dout, sizeof(float) * 3 * S, cudaMemcpyDeviceToHost, s));
  if (gc_status e = ep.release(s)) return e;
  CK(cudaGetLastError());
  return GC_OK;
}

static gc_status level_io(gc_cache c, int level, gc_level_params* p, bool out, const float* planes,
                          cudaStream_t s) {
  if (!c || !p || level < 0 || level >= c->L) return fail(GC_ERR_ARG, "bad level or NULL");
  const int64_t n = c->counts[level];
  if (p->count != n) return fail(GC_ERR_ARG, "count %lld != level size %lld", (long long)p->count, (long long)n);
  if (!p->position || !p->rotation || !p->color || !p->log_scale || !p->opacity_logit) return fail(GC_ERR_ARG, "NULL field");
  CK(cudaSetDevice(c->device));
  if (c->pack_cap < kNP * n) {
    CK(cudaDeviceSynchronize());
    if (c->pack_tmp) cudaFree(c->pack_tmp);
    CK(dalloc(&c->pack_tmp, kNP * n));
    c->pack_cap = kNP * n;
  }
  float* t = c->pack_tmp;
  float* f[5] = {p->position, p->rotation, p->color, p->log_scale, p->opacity_logit};
  const int64_t off[5] = {0, 3 * n, 7 * n, 10 * n, 13 * n}, w[5] = {3, 4, 3, 3, 1};
  if (out) {
    launch_pack(planes, c->G, c->geom.goff[level], n, t, s);
    if (routed(c) && c->mode == 1 && planes == c->P && c->world > 1)   // level-sharded: the owner's copy (collective)
      NK(ncclBroadcast(t, t, (size_t)kNP * n, ncclFloat32, c->plan.first[level], c->comm, s));
    if (routed(c) && c->mode == 2 && planes == c->P && c->world > 1) {  // owner-computes: every row from its owner
      launch_zero_nonowned(t, n, c->geom.goff[level], c->d_owner, c->rank, s);
      NK(ncclAllReduce(t, t, (size_t)kNP * n, ncclFloat32, ncclSum, c->comm, s));
    }
    for (int k = 0; k < 5; ++k) CK(cudaMemcpyAsync(f[k], t + off[k], sizeof(float) * w[k] * n, cudaMemcpyDefault, s));
  } else {
    for (int k = 0; k < 5; ++k) CK(cudaMemcpyAsync(t + off[k], f[k], sizeof(float) * w[k] * n, cudaMemcpyDefault, s));
    launch_unpack(t, c->G, c->geom.goff[level], n, planes ? const_cast<float*>(planes) : c->P, s);
  }
  CK(cudaGetLastError());
  return GC_OK;
}

gc_status gc_params(gc_cache c, int level, gc_level_params* dst, gc_stream stream) {
  NvtxRange nvtx_("gc_params");
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  CK(cudaSetDevice(c->device));
  if (gc_status e = flush_pending(c, (cudaStream_t)stream)) return e;
  return level_io(c, level, dst, true, c->P, (cudaStream_t)stream);
}

gc_status gc_set_deferred_step(gc_cache c, int enable) {
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  c->defer = enable != 0;
  return GC_OK;
}

gc_status gc_flush(gc_cache c, gc_stream stream) {
  NvtxRange nvtx_("gc_flush");
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  CK(cudaSetDevice(c->device));
  return flush_pending(c, (cudaStream_t)stream);
}

gc_status gc_set_params(gc_cache c, int level, const gc_level_params* src, int reset_adam, gc_stream stream) {
  NvtxRange nvtx_("gc_set_params");
  if (!c || !src) return fail(GC_ERR_ARG, "NULL handle or src");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  if (gc_status e = flush_pending(c, s)) return e;
  gc_level_params tmp = *src;
  if (gc_status e = level_io(c, level, &tmp, false, nullptr, s)) return e;
  if (reset_adam) {
    const int64_t n = c->counts[level], b = c->geom.goff[level];
    for (int k = 0; k < kNP; ++k) {
      CK(cudaMemsetAsync(c->M + k * c->G + b, 0, sizeof(float) * n, s));
      CK(cudaMemsetAsync(c->V + k * c->G + b, 0, sizeof(float) * n, s));
    }
    CK(cudaMemsetAsync(&c->st->adam_step[level], 0, sizeof(long long), s));
    static const double one = 1.0;   // beta^0 (pageable source: the copy completes before return)
    CK(cudaMemcpyAsync(&c->st->b1pow[level], &one, sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(&c->st->b2pow[level], &one, sizeof(double), cudaMemcpyHostToDevice, s));
  }
  return rebuild_csr(c, s, true);
}

gc_status gc_reset_schedule(gc_cache c) {
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  CK(cudaSetDevice(c->device));
  if (gc_status e = flush_pending(c, 0)) return e;
  CK(cudaMemsetAsync(&c->st->t, 0, sizeof(long long), 0));
  CK(cudaDeviceSynchronize());
  return GC_OK;
}

gc_status gc_grid(gc_cache c, int level, double origin[3], double inv_cell[3], int32_t dims[3]) {
  if (!c || level < 0 || level >= c->L || !origin || !inv_cell || !dims) return fail(GC_ERR_ARG, "bad arguments");
  for (int a = 0; a < 3; ++a) {
    origin[a] = c->geom.origin[level][a]; inv_cell[a] = c->geom.inv_cell[level][a]; dims[a] = c->geom.dims[level][a];
  }
  return GC_OK;
}

gc_status gc_info(gc_cache c, int* levels, int64_t* counts) {
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  if (levels) *levels = c->L;
  if (counts) for (int l = 0; l < GC_MAX_LEVELS; ++l) counts[l] = l < c->L ? c->counts[l] : 0;
  return GC_OK;
}

gc_status gc_nccl_unique_id(void* uid128) {
  if (!uid128) return fail(GC_ERR_ARG, "NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  NK(ncclGetUniqueId((ncclUniqueId*)uid128));
  return GC_OK;
}

gc_status gc_set_level_weights(gc_cache c, const double* weights) {
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  if (!weights) { c->has_w = false; return GC_OK; }
  for (int l = 0; l < c->L; ++l)
    if (!(weights[l] >= 0.0) || !std::isfinite(weights[l])) return fail(GC_ERR_ARG, "weights[%d] not finite and >= 0", l);
  for (int l = 0; l < c->L; ++l) c->lvl_w[l] = weights[l];
  c->has_w = true;
  return GC_OK;
}

gc_status gc_set_comm(gc_cache c, const void* nccl_uid, int rank, int world, int mode) {
  NvtxRange nvtx_("gc_set_comm");
  if (!c || world < 1 || rank < 0 || rank >= world) return fail(GC_ERR_ARG, "bad rank/world");
  if (mode < 0 || mode > 3)
    return fail(GC_ERR_ARG, "mode must be 0 (data parallel), 1 (level-sharded), 2 (owner-computes) or 3 (ZeRO data parallel)");
  if (mode == 1 && world > 1024) return fail(GC_ERR_ARG, "level-sharded mode supports at most 1024 ranks");
  if (mode == 2 && world > 32) return fail(GC_ERR_ARG, "owner-computes mode supports at most 32 ranks");
  CK(cudaSetDevice(c->device));
  if (gc_status e = refresh_stale(c, 0)) return e;
  CK(cudaDeviceSynchronize());
  if (gc_status e = flush_pending(c, 0)) return e;
  CK(cudaDeviceSynchronize());
  if (c->gcomm) { ncclCommDestroy(c->gcomm); c->gcomm = nullptr; }
  if (c->comm) { ncclCommDestroy(c->comm); c->comm = nullptr; }
  const int prev_mode = c->mode;
  c->rank = rank; c->world = world; c->mode = 0;
  if (prev_mode == 2) {               // the lists were filtered to owned + halo: rebuild them all
    CK(cudaMemset(c->csr_count, 0, sizeof(uint32_t) * c->NC));
    if (gc_status e = rebuild_csr(c, 0, true)) return e;
    CK(cudaDeviceSynchronize());
  }
  const unsigned int all = 0xFFFFFFFFu;
  CK(cudaMemcpy(&c->st->owned, &all, sizeof all, cudaMemcpyHostToDevice));
  if (!nccl_uid) {
    if (world == 1) return GC_OK;     // detach
    return fail(GC_ERR_ARG, "NULL nccl_uid");
  }
  ncclUniqueId id;
  memcpy(&id, nccl_uid, sizeof id);
  NK(ncclCommInitRank(&c->comm, world, id, rank));
  if (mode == 0) return GC_OK;
  if (mode == 3) return setup_zero(c);
  if (!c->r_count) {
    CK(dalloc(&c->r_count, 1024)); CK(dalloc(&c->r_base, 1024)); CK(dalloc(&c->r_cursor, 1024));
    CK(cudaHostAlloc((void**)&c->h_base, sizeof(uint32_t) * 1024, cudaHostAllocDefault));
  }
  if (c->r_all) cudaFree(c->r_all);
  if (c->h_all) cudaFreeHost(c->h_all);
  CK(dalloc(&c->r_all, (size_t)world * world));
  CK(cudaHostAlloc((void**)&c->h_all, sizeof(uint32_t) * world * world, cudaHostAllocDefault));
  if (mode == 2) {
    c->plan = RoutePlan{};
    c->plan.world = world; c->plan.rank = rank; c->plan.L = c->L;
    if (gc_status e = setup_owner_computes(c)) { c->mode = 0; return e; }
    return GC_OK;
  }
  // level-sharded: the plan (identical on every rank: a function of L, the weights and W)
  double w[kMaxL];
  double G = 0.0;
  for (int l = 0; l < c->L; ++l) G += (double)c->counts[l];
  for (int l = 0; l < c->L; ++l) w[l] = c->has_w ? c->lvl_w[l] : (double)c->counts[l] / G;
  int gl[kMaxL], fr[kMaxL], gs[kMaxL];
  const int ng = level_plan(c->L, w, world, gl, fr, gs);
  if (ng <= 0) return fail(GC_ERR_ARG, "level plan failed");
  c->plan = RoutePlan{};
  c->plan.world = world; c->plan.rank = rank; c->plan.L = c->L;
  int mine = -1;
  for (int g = 0; g < ng; ++g) if (rank >= fr[g] && rank < fr[g] + gs[g]) mine = g;
  unsigned int owned = 0u;
  c->glo = c->L; c->ghi = 0;
  for (int l = 0; l < c->L; ++l) {
    c->plan.first[l] = fr[gl[l]]; c->plan.size[l] = gs[gl[l]];
    if (gl[l] == mine) { owned |= 1u << l; c->glo = std::min(c->glo, l); c->ghi = std::max(c->ghi, l + 1); }
  }
  c->gsize = gs[mine];
  NK(ncclCommSplit(c->comm, mine, rank, &c->gcomm, nullptr));
  CK(cudaMemcpy(&c->st->owned, &owned, sizeof owned, cudaMemcpyHostToDevice));
  c->mode = 1;
  return GC_OK;
}

gc_status gc_comm_info(gc_cache c, int* mode, int* rank, int* world, int* owned_levels_mask, int* group_size) {
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  unsigned int owned = 0u;
  if (c->mode >= 1) { for (int l = c->glo; l < c->ghi; ++l) owned |= 1u << l; }
  else owned = (c->L >= 32) ? 0xFFFFFFFFu : ((1u << c->L) - 1u);
  if (mode) *mode = c->comm ? c->mode : -1;
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  if (owned_levels_mask) *owned_levels_mask = (int)owned;
  if (group_size) *group_size = c->mode >= 1 ? c->gsize : c->world;
  return GC_OK;
}

gc_status gc_debug_enable_grads(gc_cache c, int enable) {
  if (!c || enable < 0 || enable > 3) return fail(GC_ERR_ARG, "NULL handle or enable not in 0..3");
  CK(cudaSetDevice(c->device));
  if ((enable & 1) && !c->dbg) { CK(dalloc(&c->dbg, kNP * c->G)); CK(cudaMemset(c->dbg, 0, sizeof(float) * kNP * c->G)); }
  if ((enable & 2) && !c->dbg_coef) {
    CK(dalloc(&c->dbg_coef, 12 * c->G));
    CK(cudaMemset(c->dbg_coef, 0, sizeof(float) * 12 * c->G));
  }
  c->dbg_on = (enable & 1) != 0;
  c->dbg_mode = enable;
  return GC_OK;
}

gc_status gc_debug_coef_grads(gc_cache c, int level, float* dst, gc_stream stream) {
  if (!c || !dst || level < 0 || level >= c->L) return fail(GC_ERR_ARG, "bad arguments");
  if (!c->dbg_coef) return fail(GC_ERR_STATE, "coefficient-gradient recording not enabled (gc_debug_enable_grads bit 1)");
  CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(dst, c->dbg_coef + 12 * c->geom.goff[level], sizeof(float) * 12 * c->counts[level],
                     cudaMemcpyDefault, s));
  CK(cudaStreamSynchronize(s));
  return GC_OK;
}

gc_status gc_list_generation(gc_cache c, uint64_t* gen) {
  if (!c || !gen) return fail(GC_ERR_ARG, "bad arguments");
  *gen = c->list_generation;
  return GC_OK;
}

gc_status gc_debug_grads(gc_cache c, int level, gc_level_params* dst, gc_stream stream) {
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  if (!c->dbg) return fail(GC_ERR_STATE, "gradient recording not enabled (gc_debug_enable_grads)");
  CK(cudaSetDevice(c->device));
  if (gc_status e = flush_pending(c, (cudaStream_t)stream)) return e;
  return level_io(c, level, dst, true, c->dbg, (cudaStream_t)stream);
}

// ------------------------------------------------------------ screen-space evaluator (f1)
// Projection of levels [lev0, lev1), the (tile, depth) sort and the joint raster into the
// caller's out (gc_render) or, with `loss` (gc_fit_image), into the handle's Eq. 4 gradient image
// c->scr.dLdC; T and the last-contributor counts into c->scr.T / last (or outT when given).
static gc_status screen_render(gc_cache c, const gc_camera* cam, int lev0, int lev1, float* out, float* outT,
                               cudaStream_t s, const SLossArgs* loss = nullptr) {
  if (!cam || cam->width < 1 || cam->height < 1 || cam->width > 16384 || cam->height > 16384 || !(cam->znear > 0.f))
    return fail(GC_ERR_ARG, "bad camera");
  ScreenBufs& b = c->scr;
  const int64_t G = c->G;
  if (!b.pa) {
    CK(dalloc(&b.pa, G)); CK(dalloc(&b.pb, G)); CK(dalloc(&b.pc, G)); CK(dalloc(&b.rect, G));
    CK(dalloc(&b.touched, G)); CK(dalloc(&b.off, G)); CK(dalloc(&b.bsums, G / 4096 + 2)); CK(dalloc(&b.total, 1));
    CK(cudaHostAlloc((void**)&b.htotal, sizeof(uint32_t), cudaHostAllocDefault));
    CK(dalloc(&b.g2d, 12 * G)); CK(cudaMemset(b.g2d, 0, sizeof(float) * 12 * G));
    CK(dalloc(&b.raw, kNP * G));
  }
  const SCam sc = make_scam(*cam);
  const int Lr = lev1 - lev0;
  const int64_t npx = (int64_t)cam->width * cam->height;
  const int64_t ntiles = (int64_t)sc.TX * sc.TY;
  if (b.img_cap < Lr * npx) {
    CK(cudaDeviceSynchronize());
    for (void* p : {(void*)b.T, (void*)b.dLdC, (void*)b.last}) if (p) cudaFree(p);
    CK(dalloc(&b.T, Lr * npx)); CK(dalloc(&b.dLdC, 3 * Lr * npx));
    CK(dalloc(&b.last, Lr * npx));
    b.img_cap = Lr * npx;
  }
  if (b.range_cap < Lr * ntiles) {
    CK(cudaDeviceSynchronize());
    if (b.ranges) cudaFree(b.ranges);
    CK(dalloc(&b.ranges, Lr * ntiles));
    b.range_cap = Lr * ntiles;
  }
  if ((int64_t)Lr * ntiles >= ((int64_t)1 << 31)) return fail(GC_ERR_ARG, "image too large for the tile keys");
  const int64_t g0 = c->geom.goff[lev0], g1 = c->geom.goff[lev1];
  const int64_t nt = (int64_t)Lr * ntiles;
  if (b.tile_cap < nt + 1) {
    for (void* p : {(void*)b.tcount, (void*)b.tcursor, (void*)b.tstart, (void*)b.tbsums, (void*)b.ttotal, (void*)b.tbig})
      if (p) cudaFree(p);
    CK(dalloc(&b.tcount, nt + 1)); CK(dalloc(&b.tcursor, nt + 1)); CK(dalloc(&b.tstart, nt + 1));
    CK(dalloc(&b.tbsums, nt / 4096 + 2)); CK(dalloc(&b.ttotal, 1)); CK(dalloc(&b.tbig, 3));
    if (!b.htbig) CK(cudaHostAlloc((void**)&b.htbig, sizeof(uint32_t), cudaHostAllocDefault));
    b.tile_cap = nt + 1;
  }
  // One host round trip per call: the keys are scattered into the capacity of the previous
  // calls; the number of keys and the over-8192-keys-per-tile flag come back together after
  // the sorts.  Over capacity (the first call, a camera that sees more): grow, run again.
  int64_t npairs = 0;
  for (int attempt = 0;; ++attempt) {
    CK(launch_sproject(c->P, G, g0, g1, sc, b, c->geom, lev0, Lr, s));
    // counting sort by tile + per-tile register / shared-memory sorts; the global bitonic sort
    // only when a tile holds more than 8192 Gaussians
    CK(launch_tile_sort(g0, g1, c->geom, lev0, Lr, sc, b, b.tcount, b.tcursor, b.tstart, b.tbsums, b.ttotal, b.tbig, s));
    CK(cudaMemcpyAsync(b.htbig, b.tbig, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(b.htotal, b.total, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    npairs = *b.htotal;
    if (npairs <= b.kv_cap) break;
    if (attempt > 0) return fail(GC_ERR_STATE, "screen keys over capacity after growing");
    const int64_t Np = sort_kv_size(npairs + npairs / 4 + 1024);
    if (b.key) cudaFree(b.key);
    if (b.val) cudaFree(b.val);
    CK(dalloc(&b.key, Np)); CK(dalloc(&b.val, Np));
    b.kv_cap = Np;
  }
  if (*b.htbig) CK(launch_skeys_sort(g0, g1, c->geom, lev0, Lr, sc, b, npairs, b.kv_cap, s));
  SLossArgs la{};
  if (loss) { la = *loss; la.dLdC = b.dLdC; }
  CK(launch_sraster(sc, Lr, b, out, outT ? outT : b.T, b.last, loss ? &la : nullptr, s));
  return GC_OK;
}

gc_status gc_render(gc_cache c, const gc_camera* cam, int level, float* out_rgb, float* out_T, gc_stream stream) {
  NvtxRange nvtx_("gc_render");
  if (!c || !cam || !out_rgb) return fail(GC_ERR_ARG, "NULL handle, camera or output");
  if (level < -1 || level >= c->L) return fail(GC_ERR_ARG, "level %d not in [-1, %d)", level, c->L);
  if (!is_device_ptr(out_rgb) || (out_T && !is_device_ptr(out_T))) return fail(GC_ERR_ARG, "gc_render outputs must be device memory");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  if (gc_status e = check_sticky(c)) return e;
  if (capturing(s)) return fail(GC_ERR_STATE, "gc_render is not graph-capturable");
  if (gc_status e = flush_pending(c, s)) return e;
  const int lev0 = level < 0 ? 0 : level, lev1 = level < 0 ? c->L : level + 1;
  if (gc_status e = screen_render(c, cam, lev0, lev1, out_rgb, out_T, s)) return e;
  CK(cudaGetLastError());
  return GC_OK;
}

gc_status gc_fit_image(gc_cache c, const gc_camera* cam, const float* target, const uint8_t* valid, gc_stream stream,
                       gc_fit_stats* stats) {
  NvtxRange nvtx_("gc_fit_image");
  if (!c || !cam || !target) return fail(GC_ERR_ARG, "NULL handle, camera or target");
  if (!is_device_ptr(target) || (valid && !is_device_ptr(valid))) return fail(GC_ERR_ARG, "gc_fit_image inputs must be device memory");
  if (c->comm) return fail(GC_ERR_UNSUPPORTED, "gc_fit_image is single-GPU");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  if (gc_status e = check_sticky(c)) return e;
  if (capturing(s)) return fail(GC_ERR_STATE, "gc_fit_image is not graph-capturable");
  if (gc_status e = flush_pending(c, s)) return e;
  const int L = c->L;
  ScreenBufs& b = c->scr;
  // the raster writes each pixel's Eq. 4 gradient (and the loss partials) instead of its colour
  // (b.dLdC is sized by screen_render before the raster runs)
  SLossArgs loss{target, valid, c->hp.hdr_eps, c->hp.loss_grad_mode, nullptr, c->partial};
  if (gc_status e = screen_render(c, cam, 0, L, nullptr, nullptr, s, &loss)) return e;
  const SCam sc = make_scam(*cam);
  const int64_t npx = (int64_t)cam->width * cam->height;
  launch_stats(c->partial, c->geom, (int64_t)L * npx, c->lvl, true, c->st, c->hp, L, c->dstats, s, &c->prof);
  CK(launch_sraster_bwd(sc, L, b, b.T, b.last, b.dLdC, b.g2d, s));
  CK(launch_sproject_bwd(c->P, c->G, 0, c->G, sc, b, b.g2d, b.raw, s));
  launch_adamw(c->G, c->P, c->M, c->V, c->grad, cull_bufs(c), c->dbg_on ? c->dbg : nullptr, c->st, c->hp, c->geom,
               reinterpret_cast<unsigned long long*>(&c->dstats->nonfinite_grads), s, &c->prof, b.raw, nullptr, 0,
               /*with_record=*/false);
  c->lists_stale = true;             // records + culling lists rebuilt by the next world-space call
  if (gc_status e = emit_stats(c, stats, s)) return e;
  CK(cudaGetLastError());
  return GC_OK;
}

// ------------------------------------------------------------ dense tensor-core lookups (A8)
gc_status gc_query_dense(gc_cache c, const float* pos, const int32_t* path_len, int level, int64_t S, float* out_rgb,
                         gc_stream stream) {
  NvtxRange nvtx_("gc_query_dense");
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  if (S < 0 || S >= ((int64_t)1 << 31)) return fail(GC_ERR_ARG, "S out of range");
  if (S > 0 && (!pos || !out_rgb)) return fail(GC_ERR_ARG, "NULL pointer");
  if (S == 0) return GC_OK;
  if (!path_len && (level < 0 || level >= c->L)) return fail(GC_ERR_ARG, "level %d not in [0, %d)", level, c->L);
  if (!is_device_ptr(pos) || !is_device_ptr(out_rgb) || (path_len && !is_device_ptr(path_len)))
    return fail(GC_ERR_ARG, "gc_query_dense takes device buffers");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  if (gc_status e = check_sticky(c)) return e;
  if (gc_status e = ensure_scratch(c, c->dns, S, false, s, c->dNC)) return e;
  if (gc_status e = csr_guard(c, s)) return e;
  if (gc_status e = flush_pending(c, s)) return e;
  if (!c->dense_grid) c->dense_grid = dense_tc_grid();
  Scratch& D = c->dns;
  IngestBufs b{D.kr, D.cell_count, D.bin, c->dNC, D.cap};
  CK(cudaMemsetAsync(out_rgb, 0, sizeof(float) * 3 * S, s));   // parts of a lookup add up (k_dense_tc)
  launch_keys_query(pos, path_len, path_len ? -1 : level, S, c->dgeom, b, out_rgb, s, &c->prof);
  launch_scan(D.cell_count, c->dNC * kRep, 128, D.tiles, D.totals, D.cell_start, nullptr, D.work, c->dgeom, s, &c->prof);
  launch_scatter(pos, nullptr, S, D.cell_start, b, s, &c->prof);
  DenseArgs da;
  da.work = D.work; da.n_work = D.totals + 1; da.bin = D.bin; da.rec = c->rec;
  for (int l = 0; l <= kMaxL; ++l) da.goff[l] = c->geom.goff[l];
  da.ref = c->dref; da.out = out_rgb;
  const float tau = c->hp.cutoff_sigma;
  da.tau2 = tau * tau;
  launch_dense_tc(da, c->dense_grid, s, &c->prof);
  CK(cudaGetLastError());
  return GC_OK;
}

// ------------------------------------------------------------ dense fit on the tensor cores (A8)
gc_status gc_fit_dense(gc_cache c, const float* pos, const int32_t* path_len, int level, const float* rgb, int64_t S,
                       gc_stream stream, gc_fit_stats* stats) {
  NvtxRange nvtx_("gc_fit_dense");
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  if (S < 0 || S >= ((int64_t)1 << 31)) return fail(GC_ERR_ARG, "S out of range");
  if (S > 0 && (!pos || !rgb)) return fail(GC_ERR_ARG, "NULL pointer");
  if (S > 0 && !path_len && (level < 0 || level >= c->L))
    return fail(GC_ERR_ARG, "level %d not in [0, %d)", level, c->L);
  if (c->comm) return fail(GC_ERR_UNSUPPORTED, "gc_fit_dense is single-GPU");
  if (S > 0 && (!is_device_ptr(pos) || !is_device_ptr(rgb) || (path_len && !is_device_ptr(path_len))))
    return fail(GC_ERR_ARG, "gc_fit_dense takes device buffers");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  if (gc_status e = check_sticky(c)) return e;
  if (capturing(s)) return fail(GC_ERR_STATE, "gc_fit_dense is not graph-capturable");
  if (gc_status e = flush_pending(c, s)) return e;
  if (gc_status e = ensure_scratch(c, c->dns, std::max<int64_t>(S, 1), false, s, c->dNC)) return e;
  if (gc_status e = csr_guard(c, s)) return e;
  Scratch& D = c->dns;
  if (!D.y) { CK(dalloc(&D.y, 3 * D.cap)); CK(dalloc(&D.g, 3 * D.cap)); }
  if (!c->dense_grid) c->dense_grid = dense_tc_grid();
  const int fixed = path_len ? -1 : level;
  if (S > 0) {
    // forward: y_hat of every sample (gc_query_dense's product), caller order
    IngestBufs b{D.kr, D.cell_count, D.bin, c->dNC, D.cap};
    CK(cudaMemsetAsync(D.y, 0, sizeof(float) * 3 * S, s));
    launch_keys_query(pos, path_len, fixed, S, c->dgeom, b, D.y, s, &c->prof);
    launch_scan(D.cell_count, c->dNC * kRep, 128, D.tiles, D.totals, D.cell_start, nullptr, D.work, c->dgeom, s, &c->prof);
    launch_scatter(pos, nullptr, S, D.cell_start, b, s, &c->prof);
    DenseArgs da;
    da.work = D.work; da.n_work = D.totals + 1; da.bin = D.bin; da.rec = c->rec;
    for (int l = 0; l <= kMaxL; ++l) da.goff[l] = c->geom.goff[l];
    da.ref = c->dref; da.out = D.y;
    const float tau = c->hp.cutoff_sigma;
    da.tau2 = tau * tau;
    launch_dense_tc(da, c->dense_grid, s, &c->prof);
    // Eq. 4 per sample: dL/dy_hat and the per-level loss sums / counts
    launch_dense_loss(pos, path_len, fixed, c->L, rgb, D.y, S, c->hp.hdr_eps, c->hp.loss_grad_mode, D.g, c->partial,
                      s, &c->prof);
  }
  launch_stats(c->partial, c->geom, S, c->lvl, true, c->st, c->hp, c->L, c->dstats, s, &c->prof);
  if (S > 0) {
    DenseBwdArgs ba;
    ba.work = D.work; ba.n_work = D.totals + 1; ba.bin = D.bin; ba.rec = c->rec;
    for (int l = 0; l <= kMaxL; ++l) ba.goff[l] = c->geom.goff[l];
    ba.ref = c->dref; ba.g = D.g; ba.grad = c->grad;
    const float tau = c->hp.cutoff_sigma;
    ba.tau2 = tau * tau;
    launch_dense_bwd(ba, s, &c->prof);
  }
  launch_adamw(c->G, c->P, c->M, c->V, c->grad, cull_bufs(c), c->dbg_on ? c->dbg : nullptr, c->st, c->hp, c->geom,
               reinterpret_cast<unsigned long long*>(&c->dstats->nonfinite_grads), s, &c->prof);
  if (gc_status e = rebuild_csr(c, s, false)) return e;
  if (gc_status e = emit_stats(c, stats, s)) return e;
  CK(cudaGetLastError());
  return GC_OK;
}

// AdamW state of one level (checkpoint / resume): moments in the gc_level_params
// layout, plus the schedule counter and the per-level bias-correction state.
gc_status gc_adam_state(gc_cache c, int level, gc_level_params* m, gc_level_params* v, gc_opt_counters* ctr,
                        gc_stream stream) {
  NvtxRange nvtx_("gc_adam_state");
  if (!c || !m || !v) return fail(GC_ERR_ARG, "NULL handle or moments");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  if (gc_status e = flush_pending(c, s)) return e;
  if (gc_status e = level_io(c, level, m, true, c->M, s)) return e;
  if (gc_status e = level_io(c, level, v, true, c->V, s)) return e;
  if (ctr) {
    DevState h;
    CK(cudaMemcpyAsync(&h, c->st, sizeof h, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    ctr->t = h.t;
    for (int l = 0; l < GC_MAX_LEVELS; ++l) {
      ctr->adam_step[l] = h.adam_step[l]; ctr->beta1_pow[l] = h.b1pow[l]; ctr->beta2_pow[l] = h.b2pow[l];
    }
  }
  return GC_OK;
}

gc_status gc_set_adam_state(gc_cache c, int level, const gc_level_params* m, const gc_level_params* v,
                            const gc_opt_counters* ctr, gc_stream stream) {
  NvtxRange nvtx_("gc_set_adam_state");
  if (!c || !m || !v) return fail(GC_ERR_ARG, "NULL handle or moments");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  if (gc_status e = flush_pending(c, s)) return e;
  gc_level_params tm = *m, tv = *v;
  if (gc_status e = level_io(c, level, &tm, false, c->M, s)) return e;
  if (gc_status e = level_io(c, level, &tv, false, c->V, s)) return e;
  if (ctr) {
    CK(cudaStreamSynchronize(s));
    DevState h;
    CK(cudaMemcpy(&h, c->st, sizeof h, cudaMemcpyDeviceToHost));
    h.t = ctr->t;
    for (int l = 0; l < GC_MAX_LEVELS; ++l) {
      h.adam_step[l] = ctr->adam_step[l]; h.b1pow[l] = ctr->beta1_pow[l]; h.b2pow[l] = ctr->beta2_pow[l];
    }
    CK(cudaMemcpy(c->st, &h, sizeof h, cudaMemcpyHostToDevice));
  }
  return GC_OK;
}

gc_status gc_debug_cull(gc_cache c, int level, int32_t* offsets, int32_t* idx, int64_t cap, int64_t* n,
                        gc_stream stream) {
  if (!c || level < 0 || level >= c->L || !offsets || !n) return fail(GC_ERR_ARG, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  if (gc_status e = flush_pending(c, s)) return e;
  if (gc_status e = refresh_stale(c, s)) return e;
  const int64_t c0 = c->geom.coff[level], nc = c->geom.coff[level + 1] - c0;
  std::vector<uint32_t> off((size_t)nc + 1);
  CK(cudaMemcpyAsync(off.data(), c->csr_off + c0, sizeof(uint32_t) * (nc + 1), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int64_t total = (int64_t)off[nc] - off[0];
  *n = total;
  for (int64_t k = 0; k <= nc; ++k) offsets[k] = (int32_t)(off[k] - off[0]);
  if (!idx || cap < total) return fail(GC_ERR_ARG, "idx capacity %lld < %lld", (long long)cap, (long long)total);
  std::vector<int32_t> h((size_t)std::max<int64_t>(total, 1));
  if (total > 0)                     // the Gaussian index of each list entry (its 13th word)
    CK(cudaMemcpy2DAsync(h.data(), sizeof(int32_t), reinterpret_cast<const char*>(c->csr_rec + 4 * (size_t)off[0]) + 48,
                         4 * sizeof(float4), sizeof(int32_t), (size_t)total, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int64_t g0 = c->geom.goff[level];
  for (int64_t k = 0; k < nc; ++k) {
    std::sort(h.begin() + offsets[k], h.begin() + offsets[k + 1]);
    for (int64_t e = offsets[k]; e < offsets[k + 1]; ++e) idx[e] = (int32_t)(h[e] - g0);
  }
  return GC_OK;
}

gc_status gc_debug_levels(gc_cache c, int32_t* level_of, gc_stream stream) {
  if (!c || !level_of) return fail(GC_ERR_ARG, "bad arguments");
  if (c->last_fit_S < 0) return fail(GC_ERR_STATE, "no gc_fit yet");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(c->device));
  const int64_t S = c->last_fit_S;
  if (S == 0) return GC_OK;
  if (is_device_ptr(level_of)) { launch_levels_of(c->fit.kr, S, c->geom, level_of, s); }
  else {
    int32_t* d = nullptr;
    CK(dalloc(&d, S));
    launch_levels_of(c->fit.kr, S, c->geom, d, s);
    CK(cudaMemcpyAsync(level_of, d, sizeof(int32_t) * S, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(d);
  }
  CK(cudaGetLastError());
  return GC_OK;
}

gc_status gc_profile_enable(gc_cache c, int enable) {
  if (!c) return fail(GC_ERR_ARG, "NULL handle");
  c->prof.enabled = enable != 0;
  return GC_OK;
}

gc_status gc_profile_read(gc_cache c, char* names, int64_t cap, double* ms, int64_t* launches,
                          int max_kernels, int* n_kernels, int reset) {
  if (!c || !names || !ms || !launches || !n_kernels) return fail(GC_ERR_ARG, "bad arguments");
  CK(cudaSetDevice(c->device));
  CK(cudaDeviceSynchronize());
  c->prof.flush();
  std::string all;
  int k = 0;
  for (auto& kv : c->prof.acc) {
    if (k >= max_kernels) break;
    if (k) all += ";";
    all += kv.first;
    ms[k] = kv.second.first;
    launches[k] = kv.second.second;
    ++k;
  }
  *n_kernels = k;
  if ((int64_t)all.size() + 1 > cap) return fail(GC_ERR_ARG, "names buffer too small");
  memcpy(names, all.c_str(), all.size() + 1);
  if (reset) c->prof.acc.clear();
  return GC_OK;
}

}  // extern "C"
