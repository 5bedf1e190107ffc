/*
 * gscache.h -- C ABI of the B200-native GSCache hot path: real-time fitting and querying of
 * the multi-level 3D-Gaussian path-space radiance cache of arXiv 2507.19718.
 *
 * PAPER.md lines are cited as P:<line>; SURVEY.md 8(c) readings as C1..C8 / A1..A19 and
 * restated in DESIGN.md.  The paper exposes its cache "via a C-style API" (sec.3.7);
 * these are the calls of its problem statement: the renderer supplies attenuated radiance
 * samples with their path length (P:9, sec.3.5) and reads the cache back.
 *
 * Conventions
 *  - Pointers marked "host or device" may point to either; the library detects the kind with
 *    cudaPointerGetAttributes and stages host data through its own device buffers.  Host
 *    inputs of gc_fit / gc_query / gc_fit_query are read when the call is made (uploaded on
 *    an internal copy stream, two staging sets, so a frame's upload overlaps the previous
 *    frame's work; the call's stream waits for it); host outputs are written when `stream`
 *    reaches the end of the call.
 *  - Ownership: all buffers passed in stay owned by the caller and must stay valid until
 *    the work enqueued on `stream` completes.  The library owns parameters, AdamW state,
 *    evaluation records, grids, culling lists and scratch (cudaMalloc at create/reserve).
 *  - Errors: argument errors return GC_ERR_ARG with no side effect.  Data problems are not
 *    errors: non-finite samples, path_len <= 0 and non-finite gradients are dropped and
 *    counted in gc_fit_stats.  Asynchronous CUDA/NCCL failures are sticky and
 *    returned by the next call.  No C++ exception crosses the ABI.  gc_last_error()
 *    returns a thread-local message for the last non-OK status.
 *  - Streams: every call enqueues work on `stream` (NULL = legacy default stream) and
 *    returns; calls on one handle are stream-ordered and not thread-safe.  gc_fit, gc_query
 *    and gc_fit_query are CUDA-graph capturable once gc_reserve has sized the scratch.
 *  - There is no CPU fallback: without a usable sm_100 device gc_create fails.
 */
#ifndef GSCACHE_H_
#define GSCACHE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gc_cache_s* gc_cache;      /* opaque, library-owned */
typedef void* gc_stream;                  /* a cudaStream_t */

typedef enum {
  GC_OK = 0, GC_ERR_ARG = 1, GC_ERR_STATE = 2, GC_ERR_CUDA = 3, GC_ERR_OOM = 4,
  GC_ERR_NCCL = 5, GC_ERR_UNSUPPORTED = 6
} gc_status;

/* parameter groups, paper order (App. B) */
enum { GC_POS = 0, GC_ROT = 1, GC_COLOR = 2, GC_SCALE = 3, GC_OPACITY = 4, GC_NGROUPS = 5,
       GC_MAX_LEVELS = 16 };

typedef struct {
  float lr[GC_NGROUPS];            /* 1.16e-3, 1e-3, 1.25e-2, 0, 1.5e-1         (sec.4.1)   */
  float weight_decay[GC_NGROUPS];  /* 0, 1e-2, 1e-2, 1e-2, 1e-2  AdamW lambda  (A13)      */
  float beta1, beta2, adam_eps;    /* 0.9, 0.999, 1e-8                          (A13)             */
  float hdr_eps;                   /* 0.01                                      (Eq. 4)     */
  int loss_grad_mode;              /* 0 = stop-gradient denominator (A10), 1 = full quotient      */
  int lr_schedule;                 /* 1 = Eq. 5 eta_t = eta_0/(1+ln t), 0 = constant      */
  float cutoff_sigma;              /* tau = 3 Mahalanobis cut-off (A3); INFINITY = dense          */
  float init_opacity;              /* 0.1 ("similar to Kerbl"; A5)                           */
  float init_scale_factor;         /* 0.5 ("scales ... to 50%")                              */
  float init_zcap;                 /* 2.0 ("z-score greater than 2")                         */
  int cells_per_axis[GC_MAX_LEVELS]; /* culling grid resolution; 0 = auto rule (C8)             */
  float cell_edge_scale;           /* auto rule: cell edge = scale * 2 tau mean(e^s); default 1     */
} gc_hparams;

/* Per-call statistics.  Written asynchronously: valid once the stream has synchronised. */
typedef struct {
  int64_t n_in;                    /* samples passed in                                          */
  int64_t n_valid;                 /* samples with path_len >= 1 and finite pos/rgb (C2)         */
  int64_t n_dropped;               /* n_in - n_valid                                             */
  int64_t step;                    /* schedule counter t used by this call (0 = no-op call)      */
  int64_t nonfinite_grads;         /* raw gradient elements skipped by AdamW (C6)                */
  int64_t n_pairs;                 /* contributing (sample, Gaussian) pairs, Q <= tau^2          */
  int64_t n_candidates;            /* (sample, Gaussian) pairs tested via the culling lists      */
  int64_t flags;                   /* GC_FLAG_* bits, below                                      */
  int64_t count[GC_MAX_LEVELS];    /* k_l: valid samples per level (global under DP)             */
  double loss[GC_MAX_LEVELS];      /* L_l of Eq. 4 / C4, before this call's update               */
} gc_fit_stats;

/* gc_fit_stats.flags.  GC_FLAG_LISTS_OVERFLOWED: the culling lists read by this call were
 * incomplete (their last rebuild had more entries than their capacity), so this call's
 * optimizer step was skipped (step = 0, no level stepped) and its lookups may miss
 * contributions.  Detected on the device, so it is reported under CUDA-graph replay too; the
 * next call made outside a capture grows the lists and rebuilds them (and returns
 * GC_ERR_STATE once). */
enum { GC_FLAG_LISTS_OVERFLOWED = 1 };

/* Raw parameters of one level in the paper's layout, row-major per Gaussian. */
typedef struct {
  int64_t count;
  float* position;                 /* [N][3]                                                     */
  float* rotation;                 /* [N][4] quaternion (w,x,y,z), stored unnormalised (A6)      */
  float* color;                    /* [N][3] raw colour; activation max(0,c) (A4)                */
  float* log_scale;                /* [N][3]                                                     */
  float* opacity_logit;            /* [N][1]; activation sigmoid (A5)                            */
} gc_level_params;

/* Fills the paper defaults listed above. */
void gc_default_hparams(gc_hparams* hp);

/* Create a cache of `levels` levels (1..16) on CUDA device `device`.
 *  counts [levels] (host): Gaussians per level, non-increasing, counts[0] = N0 (sec.3.2:
 *    "replicated and logarithmically sub-sampled for each level"; explicit counts, A9).
 *  init_pos, init_rgb [N0][3] (host or device): initial point cloud (positions and albedo,
 *    P:72).  Level 0 takes the points in caller order; level l >= 1 takes the first counts[l]
 *    points of the permutation pi = stable argsort(splitmix64(seed + i)) (nested subsets, C7).
 *  init_log_scale [N0][3] (host or device) or NULL: NULL computes Eq. 2 per level:
 *    s_i = max(min(mu_N + zcap sigma_N, mean 3-NN distance), fl) * factor, isotropic, with
 *    fl = 1e-6 diag (the level's AABB diagonal), or 1e-6 when diag = 0 (one point or all
 *    points coincident: reading A20), so every log-scale is finite.
 *  Rotation (1,0,0,0), opacity logit ln(p/(1-p)), colour = albedo, AdamW moments 0, t = 0.
 *  hp: NULL = defaults.  On success *out receives the handle.  Synchronises the device. */
gc_status gc_create(int levels, const int64_t* counts, const float* init_pos,
                    const float* init_rgb, const float* init_log_scale, uint64_t seed,
                    const gc_hparams* hp, int device, gc_cache* out);

gc_status gc_destroy(gc_cache c);

/* Re-initialisation for a change of the volume's morphology (sec.5: the design "requires
 * re-initialization for cases that alter the overall morphology of the visible volume"; next
 * row f2): rebuilds the cache in place from a new point cloud exactly as gc_create would with
 * the same level counts and hyper-parameters -- parameters (Eq. 2 scales when init_log_scale is
 * NULL), AdamW moments and counters, schedule t, culling grids and lists -- keeping the
 * handle's communicator, multi-GPU mode, deferral setting, debug flags and level weights.
 * init_pos / init_rgb / init_log_scale: [counts[0]][3], host or device.  Scratch is re-sized
 * on the next call (call gc_reserve again before a CUDA-graph capture); graphs captured
 * earlier must be re-captured.  Synchronises the device. */
gc_status gc_reinit(gc_cache c, const float* init_pos, const float* init_rgb, const float* init_log_scale,
                    uint64_t seed);

/* Pre-size scratch for batches of up to S_fit fit samples and S_query query points, so that
 * later gc_fit / gc_query / gc_fit_query(S_fit, S_query) calls never allocate (required
 * before CUDA-graph capture). */
gc_status gc_reserve(gc_cache c, int64_t S_fit, int64_t S_query);

/* One optimisation step on a batch of S renderer samples (sec.3.5, sec.3.6):
 *  pos [S][3] f32, path_len [S] i32, rgb [S][3] f32 (host or device).  Level of a sample
 *  l = min(n, L) - 1 (C2).  Evaluates each sample's level mixture (C3), the HDR loss Eq. 4
 *  averaged per level over 3 k_l (C4), back-propagates into all 14 raw parameters (C5) and
 *  takes one AdamW step with eta_g(t) (C6).  A level with k_l = 0 skips its step; a batch
 *  with no valid sample is a no-op (t not advanced).  stats (host, nullable) is filled when
 *  the stream reaches the end of this call's work: page-locked memory receives one
 *  cudaMemcpyAsync, pageable memory a copy made by a stream host callback. */
gc_status gc_fit(gc_cache c, const float* pos, const int32_t* path_len, const float* rgb,
                 int64_t S, gc_stream stream, gc_fit_stats* stats);

/* One frame of the real-time loop in one call (sec.3.7): the S_q cache
 * lookups of the frame are answered from the parameters as they are BEFORE this call's
 * optimisation step (the frame's renderer reads the cache fitted through the previous
 * frame), then the S fit samples take the step exactly as gc_fit.  Results equal gc_query
 * followed by gc_fit (up to fp32 summation order).  The lookups run on the handle's own
 * stream, forked from `stream` at the call and joined back before the optimizer step, so
 * their binning and evaluation overlap the fit samples' binning and fwd/bwd; to the caller
 * the call is ordered on `stream` like any other (and CUDA-graph capturable).
 *  pos/path_len/rgb/S: as gc_fit.  qpos [S_q][3] f32, qlen [S_q] i32 or NULL (then `qlevel`
 *  for every lookup), attenuation/beta/unbiased_rgb: the gc_query_radiance epilogue (each
 *  NULL = none), out_rgb [S_q][3]: caller order; all host or device.  Lookups with
 *  qlen <= 0 or non-finite position get 0.  stats as gc_fit (fit samples only). */
gc_status gc_fit_query(gc_cache c, const float* pos, const int32_t* path_len, const float* rgb,
                       int64_t S, const float* qpos, const int32_t* qlen, int qlevel, int64_t S_q,
                       const float* attenuation, const float* beta, const float* unbiased_rgb,
                       float* out_rgb, gc_stream stream, gc_fit_stats* stats);

/* Cache lookup (sec.3.1, sec.3.4): out_rgb[i] = yhat_l(x_i) (C3) for S points.
 *  pos [S][3] f32 (host or device); path_len [S] i32 (host or device) or NULL, in which case
 *  `level` in [0, L) is used for every point.  Points with path_len <= 0 or non-finite
 *  position get 0.  out_rgb [S][3] f32 (host or device), caller order.  Never mutates. */
gc_status gc_query(gc_cache c, const float* pos, const int32_t* path_len, int level, int64_t S,
                   float* out_rgb, gc_stream stream);

/* Cache lookup with the renderer-side epilogue (next-row f3): for every valid point i
 *   out_rgb[i] = unbiased_rgb[i]                        if unbiased_rgb[i] != 0 (any channel):
 *                natural termination keeps a path's own non-zero radiance (sec.3.3.1);
 *              = yhat_l(x_i) * attenuation[i] / beta[i]  otherwise: Eq. 3, the cached
 *                radiance times the path throughput prod sigma_k divided by the cascaded
 *                cache-miss probability beta_{n-1} (sec.3.4.2).
 *  attenuation [S][3] (NULL = 1), beta [S] (NULL = 1), unbiased_rgb [S][3] (NULL = none): host
 *  or device.  Points with path_len <= 0 or non-finite position get 0.  Same evaluator and
 *  binning as gc_query. */
gc_status gc_query_radiance(gc_cache c, const float* pos, const int32_t* path_len, int level,
                            int64_t S, const float* attenuation, const float* beta,
                            const float* unbiased_rgb, float* out_rgb, gc_stream stream);

/* Early path termination, Algorithm 1 (sec.3.3.2; next-row f3), for P paths at once;
 * each thread runs the device-callable gc_alg1 of include/gscache_device.cuh (the same helper
 * a renderer kernel calls inline).  All arrays device memory:
 *  sigma [P][nmax][3] f32: the RGB albedos sigma_1..sigma_n of each path's vertices so far;
 *  n [P] i32: vertices of each path (clamped to [0, nmax]); C: termination coefficient;
 *  beta [P] f32 or NULL (= 1): beta_n, the product of the earlier cache-miss probabilities
 *  (sec.3.4.2); q [P] f32: one U(0,1) draw per path (the caller's random numbers);
 *  eps: the guard of Tr_out / (Tr + eps) (unnamed in the paper; reading A22, e.g. 1e-6).
 *  Outputs: terminate [P] i32 (1 = read the cache now), tr_out [P][3] f32 (throughput weight
 *  of a continued path), beta_next [P] f32 (beta_{n+1}).  Returns GC_ERR_ARG on NULL arrays
 *  or negative sizes, GC_ERR_CUDA if the launch fails; enqueued on `stream`. */
gc_status gc_alg1_terminate(const float* sigma, const int32_t* n, int nmax, float C, const float* beta,
                            const float* q, float eps, int64_t P, int32_t* terminate, float* tr_out,
                            float* beta_next, gc_stream stream);

/* ---- screen-space cache images (next row f1: the paper's own read / train path) ----------
 * Each level is rasterized into an image with the 3D Gaussian splatting rasterizer (P:68
 * sec.3.1, after Kerbl et al.): EWA projection with a 0.3 px^2 low-pass, 16 x 16 tiles,
 * depth-ordered front-to-back alpha compositing (alpha = min(0.99, w G), skipped below 1/255,
 * stop below T = 1e-4), background 0.  All requested levels are rasterized in one pass over a
 * joint (level, tile) list -- the paper's future-work joint multi-level rasterization.
 * Readings A23; the oracle is oracle/screen_oracle.c.  Pixel (px, py) is sampled
 * at (px + 0.5, py + 0.5); a Gaussian is culled when its camera depth is <= znear, its
 * projected centre lies outside [-0.15 W, 1.15 W] x [-0.15 H, 1.15 H], or its 2D covariance
 * is not positive definite. */
typedef struct {
  int width, height;               /* image size in pixels                                        */
  float fx, fy, cx, cy;            /* pinhole intrinsics in pixels: u = fx x/z + cx, v = fy y/z + cy */
  float view[12];                  /* world -> camera [R | t], row-major 3 x 4; camera looks down +z */
  float znear;                     /* near plane (0.2 in 3DGS)                                     */
} gc_camera;

/* Cache images of level `level` (or of all L levels, jointly, when level == -1): out_rgb
 * [Lr][H][W][3] f32 and out_T [Lr][H][W] f32 (final transmittance, nullable), device memory,
 * Lr = 1 or L.  Synchronises the stream once (the number of (tile, Gaussian) pairs sizes the
 * sort); not graph-capturable. */
gc_status gc_render(gc_cache c, const gc_camera* cam, int level, float* out_rgb, float* out_T,
                    gc_stream stream);

/* One optimisation step of every level on screen-space samples (sec.3.5 "inverse
 * splatting", Eq. 4): target [L][H][W][3] f32, the noisy per-level radiance images of
 * the frame's paths; valid [L][H][W] u8 or NULL (all): pixels without a path of that length
 * carry no sample.  Renders all levels, takes Eq. 4 per level over 3 k_l (k_l = valid pixels;
 * loss_grad_mode as gc_fit), back-propagates through the compositing and the EWA projection
 * into all 14 raw parameters, and takes the shared AdamW step (schedule, level skip, frozen
 * groups as gc_fit).  The world-space calls see the new parameters: their evaluation records
 * and culling lists are rebuilt by the next call that reads them (consecutive gc_fit_image /
 * gc_render calls skip that rebuild).  stats as gc_fit (n_in = L H W pixel samples).
 * Device buffers; single GPU (GC_ERR_UNSUPPORTED with a communicator); synchronises once. */
gc_status gc_fit_image(gc_cache c, const gc_camera* cam, const float* target, const uint8_t* valid,
                       gc_stream stream, gc_fit_stats* stats);

/* Dense all-pairs lookups on the tensor cores (row A8, optional in the north star): the same
 * values as gc_query -- yhat_l(x) = sum over EVERY Gaussian of the level of v e^{-Q/2}
 * [Q <= tau^2] (C3), no culling lists -- with Q evaluated as a GEMM of 10 monomial features
 * of the sample against 10 coefficients per Gaussian (tcgen05.mma kind::tf32, 3xTF32 split,
 * TMEM accumulators), both recentred on the centre of the sample's cell of a tile grid (the
 * culling grid, or the same rule at tau = 3 when tau is infinite), and the exp / colour
 * contraction on CUDA cores.  Meant for the dense case (tau = INFINITY) and small levels; cost
 * grows with S x G.  pos [S][3], path_len [S] or NULL (then `level`), out_rgb [S][3]: DEVICE
 * buffers, caller order; invalid lookups get 0. */
gc_status gc_query_dense(gc_cache c, const float* pos, const int32_t* path_len, int level, int64_t S,
                         float* out_rgb, gc_stream stream);

/* Dense fit step on the tensor cores (row A8's backward): one gc_fit step -- Eq. 4 over the
 * frame's samples (loss_grad_mode as gc_fit), the gradient of every parameter, the
 * shared AdamW step with the Eq. 5 schedule, the records / culling lists rebuilt -- with the
 * level mixture evaluated densely over EVERY Gaussian of the sample's level (as
 * gc_query_dense; the same values as gc_fit with tau = INFINITY, or with the mask Q <= tau^2).
 * Forward: gc_query_dense's product.  Backward, per (tile-grid cell item, 128-Gaussian chunk):
 * Q^T as a product in the transposed orientation (tcgen05.mma kind::tf32, 3xTF32), e = e^{-Q/2}
 * written back to tensor memory, then E^T times [g_i phi_i, g_i] (the per-sample loss gradient
 * times the monomial features) as a second product with the A operand in TMEM: the sums over
 * the item's samples of dL/dkappa and dL/dv for each Gaussian, chained to the 12 coefficient
 * gradients (dmu, dA, dv) of gc_fit.  pos [S][3], path_len [S] or NULL (then `level`),
 * rgb [S][3]: DEVICE buffers; samples with non-finite position or colour, or n < 1, are dropped
 * (counted out of k_l).  Single GPU (GC_ERR_UNSUPPORTED with a communicator); not graph-
 * capturable; completes a pending deferred step first.  stats as gc_fit. */
gc_status gc_fit_dense(gc_cache c, const float* pos, const int32_t* path_len, int level, const float* rgb, int64_t S,
                       gc_stream stream, gc_fit_stats* stats);

/* Deferred optimizer step (enable != 0; off by default).  gc_fit / gc_fit_query then leave
 * their optimizer half -- the AdamW step with the next step's evaluation records, and the
 * culling-list rebuild -- pending, and the next call on the handle launches it on an internal
 * stream forked from its own, overlapping that call's sample ingest; the pending step always
 * completes before anything reads the cache (lookups, fwd/bwd, gc_params, gc_set_params,
 * gc_debug_*, gc_reset_schedule), so every result is the same as without deferral.
 * gc_fit_stats of a deferred call report nonfinite_grads of the PREVIOUS step (its own is not
 * known yet).  gc_flush completes a pending step on `stream`. */
gc_status gc_set_deferred_step(gc_cache c, int enable);
gc_status gc_flush(gc_cache c, gc_stream stream);

/* Copy out (gc_params) / in (gc_set_params) the raw parameters of one level in the paper's
 * layout.  dst/src arrays: host or device, `count` must equal the level's size.
 * gc_set_params rebuilds the level's evaluation records and culling lists; reset_adam != 0
 * zeroes its AdamW moments and per-level step counter. */
gc_status gc_params(gc_cache c, int level, gc_level_params* dst, gc_stream stream);
gc_status gc_set_params(gc_cache c, int level, const gc_level_params* src, int reset_adam,
                        gc_stream stream);

/* Optimizer state for checkpoint / resume: the AdamW moments of one level in the
 * gc_level_params layout (m: first, v: second moment; host or device arrays of the level's
 * size), and, if ctr != NULL, the Eq. 5 schedule counter t and every level's AdamW step counter
 * with its running beta powers (beta1^step, beta2^step, fp64 as kept on the device).
 * gc_params + gc_adam_state of every level, restored into a cache created with the same
 * arguments by gc_set_params(reset_adam = 0) + gc_set_adam_state, continue the run exactly
 * (up to the fp32 atomic summation order of later steps).  gc_adam_state synchronises the
 * stream when ctr != NULL; gc_set_adam_state with ctr synchronises it too. */
typedef struct {
  int64_t t;                             /* Eq. 5 counter (stepping fits since create / reset) */
  int64_t adam_step[GC_MAX_LEVELS];      /* per-level AdamW steps (A12)                        */
  double beta1_pow[GC_MAX_LEVELS], beta2_pow[GC_MAX_LEVELS];
} gc_opt_counters;
gc_status gc_adam_state(gc_cache c, int level, gc_level_params* m, gc_level_params* v,
                        gc_opt_counters* ctr, gc_stream stream);
gc_status gc_set_adam_state(gc_cache c, int level, const gc_level_params* m,
                            const gc_level_params* v, const gc_opt_counters* ctr, gc_stream stream);

/* Viewport / scene change: the next stepping gc_fit uses t = 1 again. */
gc_status gc_reset_schedule(gc_cache c);

/* Culling grid of a level (C8): cell c_a = clamp(floor((x_a - origin_a) * inv_cell_a), 0,
 * dims_a - 1); linear cell id (c_z * dims_y + c_y) * dims_x + c_x.  Fixed at create. */
gc_status gc_grid(gc_cache c, int level, double origin[3], double inv_cell[3], int32_t dims[3]);

/* Number of levels and per-level Gaussian counts (host array of GC_MAX_LEVELS). */
gc_status gc_info(gc_cache c, int* levels, int64_t* counts);

/* Multi-GPU (north star; none in the paper, which runs on one GPU).
 * nccl_uid: 128-byte ncclUniqueId produced by rank 0 (gc_nccl_unique_id) and broadcast by
 * the caller; rank in [0, world).  Every rank holds the same cache (same gc_create arguments).
 *  mode 0 = data parallel: every rank calls gc_fit / gc_fit_query with its own shard of the
 *    samples; one NCCL all-reduce (sum) of the per-level coefficient gradients and level
 *    statistics per step makes every replica take the identical AdamW step (C9: the result
 *    equals the one-rank result on the concatenated batch up to summation order).  Lookups
 *    are local (replicas).  Graph-capturable.
 *  mode 1 = level-sharded: levels are partitioned into contiguous groups owned by contiguous
 *    rank groups (gc_level_plan over the level weights, gc_set_level_weights, default the
 *    per-level Gaussian counts); every call is COLLECTIVE: each rank passes its own samples /
 *    lookups, which are routed (ncclSend/ncclRecv) to the owning group of their level and
 *    split round-robin inside it; a group sums its levels' gradients over its own
 *    communicator (ncclCommSplit), level statistics are summed over all ranks (global k_l,
 *    identical t), and each rank steps only the levels it owns.  Lookup results return to the
 *    caller's rank in caller order.  gc_params is collective too (the owner broadcasts the
 *    level).  Each call synchronises the host once (the routed sizes are NCCL host
 *    arguments), so mode 1 is not graph-capturable (GC_ERR_STATE under capture), and the
 *    gc_query_radiance epilogue is not available (GC_ERR_UNSUPPORTED).
 *  mode 2 = owner-computes (spatial; next row f4): every level's culling-grid columns (x cell
 *    index) are cut into `world` contiguous slabs of about equal Gaussian counts
 *    (gc_slab_plan); a Gaussian is owned by the rank of its mean's column (fixed at
 *    gc_set_comm); samples and lookups are routed to the owner of their cell's column; a rank
 *    evaluates against its owned Gaussians plus a HALO: the Gaussians of other ranks whose C8
 *    cell range reaches its columns.  Instead of a dense all-reduce, only the gradients of the
 *    boundary set B (Gaussians needed by more than their owner) are summed over ranks; every
 *    owner steps its own Gaussians; the owners' fresh rows of B are then exchanged and the
 *    culling lists rebuilt from owned + halo Gaussians.  Collective like mode 1 (one host
 *    synchronisation per call for the routed sizes and one for |B|; not graph-capturable; no
 *    deferred step; gc_params collective); world <= 32.
 *  mode 3 = ZeRO data parallel (SURVEY 8(e) "required upgrade" 1): as mode 0, but the per-level
 *    gradients are REDUCE-SCATTERED (rank r sums Gaussians [r n, (r+1) n), n = ceil(G / world)),
 *    every rank takes the AdamW step of its slice only (optimizer work and moment traffic / world),
 *    and the updated parameter rows are ALL-GATHERED so every replica holds the full cache
 *    before the (replicated) record / culling rebuild.  Same results as mode 0 up to summation
 *    order; no deferred step (the tail holds a collective); gc_adam_state returns this rank's
 *    slice of the moments (the other rows are not maintained here).  Graph-capturable.
 * nccl_uid == NULL with world == 1 detaches; a uid with world == 1 builds a one-rank
 * communicator (modes 0 and 3: the collectives run as identities; modes 1 and 2: every sample is
 * routed to this rank through ncclSend/ncclRecv to itself -- used to test the paths on one GPU). */
gc_status gc_nccl_unique_id(void* uid128);
gc_status gc_set_comm(gc_cache c, const void* nccl_uid, int rank, int world, int mode);

/* Level weights of the mode-1 plan (weights [levels], finite, >= 0; NULL = the default, each
 * level's share of the Gaussians).  Takes effect at the next gc_set_comm. */
gc_status gc_set_level_weights(gc_cache c, const double* weights);

/* The mode-1 plan as a pure host function (no device, no handle).  Levels 0..levels-1 with
 * weights [levels] (>= 0) go to n_groups = min(levels, world) groups of contiguous levels
 * owned by contiguous rank ranges (group g: ranks group_first_rank[g] .. + group_size[g]):
 *  world >= levels: one level per group; the surplus ranks join, one at a time, the level
 *    with the largest weight per rank (data parallel inside that level's group -- level 0,
 *    with most samples and Gaussians, is the hybrid case of SURVEY 8(e));
 *  world < levels: one rank per group; the levels are cut into world contiguous ranges
 *    minimising the largest range weight (exact dynamic programme).
 * Ties resolve by a fixed order, so every rank computes the same plan.  group_of_level
 * [levels], group_first_rank / group_size [>= levels] (host).  world <= 1024. */
gc_status gc_level_plan(int levels, const double* weights, int world, int32_t* group_of_level,
                        int32_t* group_first_rank, int32_t* group_size, int* n_groups);

/* The mode-2 slab plan as a pure host function: for each level l, the grid columns c in
 * [0, 512) get col_rank[l * 512 + c] in [0, world): the columns of the culling grid (origin,
 * inv_cell, dims [levels][3], as gc_grid) are cut into `world` contiguous ranges holding about
 * counts[l] / world of the level's means each (means_x [G]: x coordinates of every Gaussian,
 * level-major); columns past dims_x map to world - 1.  world <= 32, dims_x <= 512. */
gc_status gc_slab_plan(int levels, const int64_t* counts, const float* means_x, const double* origin,
                       const double* inv_cell, const int32_t* dims, int world, int32_t* col_rank);

/* Communicator state: mode (-1 none, 0, 1, 2), rank, world, the bit mask of levels this rank
 * steps, and the size of its level group (mode 0: world).  Each pointer nullable. */
gc_status gc_comm_info(gc_cache c, int* mode, int* rank, int* world, int* owned_levels_mask,
                       int* group_size);

/* ---- debug / parity exports (not on the hot path) ---------------------------------- */

/* Gradient recording of each gc_fit: enable bit 0 = the raw 14-parameter gradients (this
 * also switches the hot path's reduced "lite" backward off, because the frozen-scale ∂A terms
 * it skips are needed for them); bit 1 = a snapshot of the 12 coefficient gradients exactly as
 * the optimizer reads them (taken after the fused fwd/bwd and any all-reduce, the backward
 * itself unchanged: this is what exposes the timed lite path).  0 disables both. */
gc_status gc_debug_enable_grads(gc_cache c, int enable);
/* Coefficient gradients of the last gc_fit (bit 1 of gc_debug_enable_grads), level `level`:
 * dst [n][12] f32 (host or device), per Gaussian (dmu_x, dmu_y, dmu_z, dA00, dA11, dA22, dA01,
 * dA02, dA12, dv_r, dv_g, dv_b) with A = Sigma^-1 (full symmetric element, not doubled) and
 * v = w max(0,c) (C5), summed over the call's samples and NOT yet divided by 3 k_l (the
 * optimizer's normalisation, C4).  Synchronises the stream. */
gc_status gc_debug_coef_grads(gc_cache c, int level, float* dst, gc_stream stream);
/* Generation of the culling-list buffers: incremented whenever a capacity growth reallocated
 * them.  The kernels reach the lists through the handle's device state, not through launch
 * arguments, so CUDA graphs captured at an earlier generation stay valid and use the grown
 * lists (no re-capture needed); the counter is informational. */
gc_status gc_list_generation(gc_cache c, uint64_t* gen);
/* Raw gradients d(sum_l L_l)/d(theta) of the last gc_fit (C5), in gc_level_params layout. */
gc_status gc_debug_grads(gc_cache c, int level, gc_level_params* dst, gc_stream stream);
/* Culling lists of one level (C8): offsets [cells+1] (level-local, host), idx (host, cap
 * entries, level-local Gaussian indices, each cell's list ascending).  *n = total entries.
 * Returns GC_ERR_ARG (with *n set) if cap is too small.  Synchronises the stream. */
gc_status gc_debug_cull(gc_cache c, int level, int32_t* offsets, int32_t* idx, int64_t cap,
                        int64_t* n, gc_stream stream);
/* Level assignment of the last gc_fit's samples (C2), caller order, -1 = dropped.  level_of
 * [S] (host or device), S = that call's S. */
gc_status gc_debug_levels(gc_cache c, int32_t* level_of, gc_stream stream);

/* Per-kernel device timing (CUDA events on the call's stream), for bench.py's roofline.
 * enable != 0 records events around every kernel of gc_fit / gc_query. */
gc_status gc_profile_enable(gc_cache c, int enable);
/* Accumulated milliseconds and launch counts per named kernel since the last reset; names
 * are written as a ';'-separated list into `names` (cap bytes).  Synchronises the device. */
gc_status gc_profile_read(gc_cache c, char* names, int64_t cap, double* ms, int64_t* launches,
                          int max_kernels, int* n_kernels, int reset);

const char* gc_last_error(void);
const char* gc_status_string(gc_status s);

#ifdef __cplusplus
}
#endif
#endif /* GSCACHE_H_ */
