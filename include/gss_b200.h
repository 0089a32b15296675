/* gss_b200.h — C ABI of the B200-native GS-Scale hot path (libgss_b200.so).
 *
 * This is the drop-in boundary for the per-iteration training path of the reference
 * (/root/reference/proj/include/gss/*.hpp, header-template C++ API). Each entry point names the
 * reference function it replaces (file:line). Conventions:
 *   - fp32 data, plain pointers and sizes; no C++ or torch types cross this boundary;
 *   - device buffers are caller-allocated; every call is enqueued on the given CUDA stream and
 *     returns immediately (stream-ordered), except where a host-visible result is documented;
 *   - status codes: GSS_OK 0, GSS_ERR_CUDA 1, GSS_ERR_INVALID 2 (reference: ConfigError /
 *     std::invalid_argument), GSS_ERR_INVARIANT 3 (reference: InvariantViolation), GSS_ERR_PARSE 4
 *     (reference: ParseError, PLY ingestion only); the message of
 *     the last failure on the calling thread is returned by gss_last_error();
 *   - there is no CPU fallback: without a CUDA device every compute entry point fails with
 *     GSS_ERR_CUDA.
 */
#ifndef GSS_B200_H
#define GSS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* gss_stream_t; /* a cudaStream_t */

enum { GSS_OK = 0, GSS_ERR_CUDA = 1, GSS_ERR_INVALID = 2, GSS_ERR_INVARIANT = 3, GSS_ERR_PARSE = 4 };

/* Camera<float> (scene.hpp:77-96): world->camera p_c = rot * p + trans, row-major rot. 80 bytes,
 * layout-identical to the reference struct. */
typedef struct {
  float rot[9];
  float trans[3];
  float fx, fy, cx, cy;
  int32_t width, height;
  float near_plane, far_plane;
} gss_camera;

/* Viewport<float> (render.hpp:46-49): closed pixel rectangle; pixel (x, y) has centre (x+.5, y+.5). */
typedef struct {
  float x0, x1, y0, y1;
} gss_viewport;

/* GroupSpec + Hyperparams (adam.hpp:14-34): contiguous columns [col0, col0+dim) with their own lr. */
typedef struct {
  int32_t col0, dim;
  double lr, beta1, beta2, eps;
} gss_group;

/* Arena<float> (adam.hpp:119-159): row-major w/m/v [n][dim] + uint8 counter[n], all device
 * pointers (or pinned host pointers where documented). `step` = applied update passes; the
 * update entry points advance it on the host at enqueue time. row_stride (floats between
 * consecutive rows of w, m and v; 0 = dim) lets w/m/v share one row-interleaved buffer
 * (w = base, m = base + dim, v = base + 2*dim, row_stride >= 3*dim): a touched row is then one
 * contiguous span instead of three scattered ones (the reference layout is row_stride = dim). */
typedef struct {
  float* w;
  float* m;
  float* v;
  uint8_t* counter;
  int64_t n;
  int32_t dim;
  int32_t defer_max;
  int64_t step;
  int32_t ngroups;
  gss_group groups[8];
  int64_t row_stride;
} gss_arena;

/* SparseGrads<float> (adam.hpp:163-169): sorted ids; row(k) = rows + k*stride + col0.
 * count_dev (optional device int64) overrides count so a device-produced length (gss_cull) can
 * feed the optimizer without a host round trip. */
typedef struct {
  const int32_t* ids;
  int64_t count;
  const int64_t* count_dev;
  const float* rows;
  int64_t stride;
  int32_t col0;
} gss_sparse_grads;

/* ---- library ------------------------------------------------------------------------------ */
const char* gss_last_error(void);
int32_t gss_abi_version(void);
/* Number of CUDA devices visible (0 = no GPU; compute calls then fail with GSS_ERR_CUDA). */
int32_t gss_device_count(void);
/* Kernels launched by this library since load (process-wide; bench `gpu_launches`). */
int64_t gss_launch_count(void);

/* glibc-exact expf on the device, for n inputs (parity probe of render.hpp:105). */
int gss_expf_device(const float* x, float* y, int64_t n, gss_stream_t stream);

/* ---- frustum cull (render.hpp:243-260 cull_keep / frustum_cull) ---------------------------- */
/* Workspace for n Gaussians (per-tile look-back states). It must be zero-filled once
 * before its first use; every call leaves it ready for the next one (no per-call memset). One
 * workspace must not be used by two calls in flight at the same time. */
size_t gss_cull_workspace_bytes(int64_t n);
/* Forgets the host-side epoch of a workspace about to be freed (its look-back states are then
 * never compared again); call after its last gss_cull has been enqueued. */
void gss_cull_workspace_release(const void* workspace);
/* ids_out: capacity n, receives the kept ids ascending (bit-exact with frustum_cull);
 * mask_opt: optional bit mask, ceil(n/32) words, bit i of word i/32 = kept(i);
 * count_dev: device int64 receiving the kept count. geo rows are read with `stride` floats per
 * row (10 for the geometric tier, 59 for a dense arena). */
int gss_cull(const float* geo, int64_t n, int64_t stride, const gss_camera* cam, const gss_viewport* vp,
             float low_pass, uint32_t* mask_opt, int32_t* ids_out, int64_t* count_dev, void* workspace,
             size_t workspace_bytes, gss_stream_t stream);

/* ---- optimizer (adam.hpp:67-313) -------------------------------------------------------- */
/* Arenas whose w/m/v live in pinned host memory (the offload tier, store.hpp:149-192; row-
 * interleaved, counters on the device) are updated / restored through HBM staging: listed rows
 * are gathered over the host link, processed on the device, and written rows scattered back, in
 * chunks of this many bytes (ForwardStage chunks, store.hpp:204-213; default 32 MB). */
int gss_set_host_chunk_bytes(int64_t bytes);
/* build_group_luts (adam.hpp:67-97), fp64 on the host, cast to float. Arrays have max_delay+1
 * entries; scalars[5] = one_minus_b1, one_minus_b2, bias_correction, step_size, eps. */
int gss_build_group_luts(double lr, double beta1, double beta2, double eps, int64_t t, int32_t max_delay,
                         float* param, float* mom, float* var, float* pow_b1, float* pow_b2, float* scalars);
/* adam_step_dense (adam.hpp:198-207): every row at delay 0; grads n*dim (device) or NULL. */
int gss_adam_step_dense(gss_arena* arena, const float* grads, gss_stream_t stream);
/* deferred_update (adam.hpp:211-238): touched = has grad or counter == defer_max; touched rows are
 * restored at their delay and stepped, counters reset, others advance. Optional outputs:
 * touched_ids (device, capacity n, ascending) and touched_count_dev. Unsorted / out-of-range ids
 * are detected on the device and reported by gss_arena_check (GSS_ERR_INVARIANT). */
int gss_deferred_update(gss_arena* arena, const gss_sparse_grads* grads, int32_t* touched_ids,
                        int64_t* touched_count_dev, gss_stream_t stream);
/* restore_view (adam.hpp:252-289): out[k] = row ids[k] restored (+ the pending pass when
 * pending != NULL). ids must be ascending (the reference's merge walk assumes it).
 * ids_count_dev optionally supplies the id count from the device. Arena state untouched. */
int gss_restore_view(const gss_arena* arena, const int32_t* ids, int64_t count, const int64_t* ids_count_dev,
                     const gss_sparse_grads* pending, float* out_rows, gss_stream_t stream);
/* flush_deferred (adam.hpp:293-313). */
int gss_flush_deferred(gss_arena* arena, gss_stream_t stream);
/* Device-side invariant flag of the last deferred_update on this arena's counters:
 * returns GSS_ERR_INVARIANT if grad ids were unsorted/out of range (adam.hpp:231) or a
 * counter exceeded defer_max (adam.hpp:154-158). Synchronises the stream. */
int gss_arena_check(const gss_arena* arena, gss_stream_t stream);
/* Releases the library's per-arena scratch and sticky error flag (both keyed by arena->counter);
 * call before freeing an arena's buffers. Lifetime: the scratch and the flag are created by the
 * first gss_deferred_update / gss_restore_view / gss_arena_check on the arena and live until this
 * call (synchronises the device). */
int gss_arena_release(const gss_arena* arena);
/* AccessReport (adam.hpp:36-50) of the arena since its first use (keyed like the scratch):
 * out6 = update_passes, touched_rows, param_bytes (7*dim*4 per touched row), counter_bytes (n per
 * deferred pass), restore_rows, restore_read_bytes (4*dim*4 per restored row). Synchronises. */
int gss_arena_access(const gss_arena* arena, uint64_t* out6);

/* ---- rasterizer (render.hpp:361-640) ---------------------------------------------------- */
/* A render context is the device-side RenderResult (render.hpp:284-289): it owns the splat
 * records, the tile-binned sorted contribution lists and the per-pixel aux of the last forward,
 * which rasterize_backward consumes. Memory grows on demand from a stream-ordered pool. */
typedef struct gss_render_ctx gss_render_ctx;
gss_render_ctx* gss_render_ctx_create(void);
void gss_render_ctx_destroy(gss_render_ctx* ctx);

/* RenderScene (render.hpp:70-77). nongeo rows: compact (slot-indexed, row k = nongeo + k*stride)
 * or by global id; slot_map (optional device) remaps compact slots as NonGeoView does. */
typedef struct {
  const int32_t* ids; /* device, ascending */
  int64_t count;      /* host-known count (see count_dev) */
  const int64_t* count_dev; /* optional: read the count from the device (one sync) */
  const float* geo;
  int64_t geo_stride;
  const float* nongeo;
  int64_t nongeo_stride;
  int32_t nongeo_compact;
  const int32_t* slot_map;
  int32_t sh_degree;
  float background[3];
  float low_pass;
} gss_render_scene;

/* rasterize_forward (render.hpp:384-464) fused with compute_loss_l1 (render.hpp:497-511) when
 * gt != NULL: image (ph*pw*3 device, pixel window of vp) is bit-identical to the reference;
 * gt is the FULL camera image (height*width*3); d_img (window-sized) and loss_dev (device float)
 * receive the L1 gradient and loss normalised by `normalizer` (0 = window element count).
 * final_T_opt / n_contrib_opt: optional per-pixel transmittance and used-contribution counts.
 * meta_host (optional, host int64[6]): px0, py0, pw, ph, visible count, tile instances
 * (filling it synchronises the stream). */
int gss_rasterize_forward(gss_render_ctx* ctx, const gss_render_scene* scene, const gss_camera* cam,
                          const gss_viewport* vp, float* image, const float* gt, int64_t normalizer, float* d_img,
                          float* loss_dev, float* final_T_opt, int32_t* n_contrib_opt, int64_t* meta_host,
                          gss_stream_t stream);
/* compute_loss_l1 (render.hpp:497-511) on window-sized images; loss in fp64 then cast. */
int gss_loss_l1(const float* image, const float* gt, int64_t elems, int64_t normalizer, float* d_img,
                float* loss_dev, gss_stream_t stream);
/* rasterize_backward (render.hpp:526-640) for the ctx's last forward: d_img (window-sized).
 * Outputs per visible slot k (zero-filled by this call): grad_geo[k*geo_stride + 0..9],
 * grad_nongeo[k*ng_stride + 0..48] (use grad_geo = rows, grad_nongeo = rows + 10 and both strides
 * 59 for the reference GradBuffer layout), mean2d_opt[k*2 + 0..1]. Deterministic (no float
 * atomics): per-tile fixed-order reductions, then per-Gaussian fixed-order sums. */
int gss_rasterize_backward(gss_render_ctx* ctx, const float* d_img, float* grad_geo, int64_t geo_stride,
                           float* grad_nongeo, int64_t ng_stride, float* mean2d_opt, gss_stream_t stream);

/* Rasterizer work accounting (device counters, synchronises the device): out8[0..7] = forward
 * (warp, record) pairs walked, forward lane-pixel slots offered, forward (pixel, record) pairs in
 * box, forward contributions composited, forward eval slots issued, backward (warp, record) pairs
 * walked, backward lane-pixel slots, backward useful contributions. Counted only by a library built
 * with -DGSS_RASTER_STATS=1 (gss_raster_stats_enabled() == 1); zeros otherwise. */
int gss_raster_stats(uint64_t* out8, int32_t reset);
int32_t gss_raster_stats_enabled(void);

/* image_mse numerator (trainer.hpp:113-122) for psnr / psnr_over_views (trainer.hpp:124-145):
 * sum_dev (device double) = sum over elems of (double(a) - double(b))^2, fixed-order reduction. */
int gss_image_sq_err(const float* a, const float* b, int64_t elems, double* sum_dev, gss_stream_t stream);

/* ---- split-phase rasterizer: image-parallel rendering over N GPUs --------- */
/* The reference renders a view on one process (render.hpp:384-640) and splits it only into two
 * viewports (engine.hpp:266-273, splitter.hpp:31-123). Across GPUs the view is cut into column
 * strips: each GPU projects ITS Gaussians (a contiguous id shard) into splat records, ships every
 * record to the owner of each strip its pixel box touches, the strip owner composites the records
 * it received from all GPUs in (shard, slot) order = ascending global id, and the 9-float
 * screen-space gradient sums (the SlotAcc cut, render.hpp:538) travel back to the record owner,
 * which sums them in strip order and runs the chain (render.hpp:600-638) locally. Per-pixel
 * contribution lists equal the single-GPU ones, so strip images are bit-identical to the
 * unsplit image. */
#define GSS_SPLAT_RECORD_BYTES 64
/* project_all (render.hpp:361-380) of the scene's visible slots: records[k] (64 B each, device)
 * for slot k, pixel box clipped to vp. Host-known count only. */
int gss_project(const gss_render_scene* scene, const gss_camera* cam, const gss_viewport* vp, void* records,
                gss_stream_t stream);
/* Strip routing: strip k = pixel columns [strip_x[k], strip_x[k+1]) (strip_x: host, nstrips+1
 * ascending). dest_slots (device, nstrips*count) row k receives the ascending slots whose box
 * touches strip k; dest_counts (device int64[nstrips]) their numbers. */
int gss_route_strips(const void* records, int64_t count, const int32_t* strip_x, int32_t nstrips,
                     int32_t* dest_slots, int64_t* dest_counts, gss_stream_t stream);
/* out[i] = records[slots[i]] (packing a send buffer). */
int gss_gather_records(const void* records, const int32_t* slots, int64_t n, void* out, gss_stream_t stream);
/* dst[slots[j]*width + c] += src[j*width + c]; each slot at most once per call (call in strip
 * order for a fixed-order sum). */
int gss_scatter_add_rows(const float* src, const int32_t* slots, int64_t n, int32_t width, float* dst,
                         gss_stream_t stream);
/* Composite received records (ties in depth broken by record order) on window vp, as
 * gss_rasterize_forward does after projection; background[3] (host). loss_sum_dev (optional
 * device double) receives the fp64 sum of |image - gt| of the window, so strip losses add up to the
 * unsplit fp64 sum before the single float cast (render.hpp:510). */
int gss_rasterize_records_forward(gss_render_ctx* ctx, const void* records, int64_t count, const gss_camera* cam,
                                  const gss_viewport* vp, const float* background, float* image, const float* gt,
                                  int64_t normalizer, float* d_img, float* loss_dev, double* loss_sum_dev,
                                  float* final_T_opt, int32_t* n_contrib_opt, int64_t* meta_host,
                                  gss_stream_t stream);
/* Per-record 9-float screen-space gradient sums (rgb3, mean2d2, cov3, alpha_base; device
 * count*9) of the ctx's last records forward. */
int gss_rasterize_records_backward(gss_render_ctx* ctx, const float* d_img, float* sums, gss_stream_t stream);
/* The per-Gaussian chain (render.hpp:600-638): sums (device V*9, per slot of scene, summed over
 * strips) + the records gss_project produced -> gradient rows as gss_rasterize_backward. */
int gss_chain_backward(const gss_render_scene* scene, const gss_camera* cam, const void* records, const float* sums,
                       float* grad_geo, int64_t geo_stride, float* grad_nongeo, int64_t ng_stride, float* mean2d_opt,
                       gss_stream_t stream);

/* ---- offload engine (engine.hpp:55-522) ------------------------------------------------- */
/* OptimConfig (store.hpp:110-145) + EngineConfig (engine.hpp:30-49). */
typedef struct {
  double lr_mean, lr_scale, lr_quat, lr_opacity, lr_sh, sh_rest_divisor;
  double beta1, beta2, eps, scene_extent;
  int32_t defer_max, geo_defer_max;
  int32_t pipelined;      /* 0 = run_serial order on one stream, 1 = two-stream DAG (run_pipelined) */
  int32_t sh_degree, sh_warmup_step;
  float background[3];
  float low_pass;
  int32_t nongeo_on_host; /* 0: non-geometric tier in HBM; 1: pinned host tier (offload) */
  int64_t chunk_bytes;    /* forwarding chunk (store.hpp:204-213), default 32 MB */
} gss_engine_config;

typedef struct gss_engine gss_engine;
void gss_engine_config_default(gss_engine_config* cfg);
/* init_rows: host n x 59 (scene.hpp:13-31 row layout). cams: host; gts: host ncams*H*W*3 or NULL
 * (then gss_engine_step must supply the ground truth per step). */
gss_engine* gss_engine_create(int64_t n, const float* init_rows, int32_t ncams, const gss_camera* cams,
                              const float* gts, const gss_engine_config* cfg);
void gss_engine_destroy(gss_engine* e);
/* OffloadEngine::run (engine.hpp:73-88): n iterations over the stored cameras, drained.
 * losses / valid_counts (host, n entries) receive IterResult. */
int gss_engine_run(gss_engine* e, int32_t iters, float* losses, int32_t* valid_counts);
/* One iteration with a host-supplied camera and ground truth (pinned or pageable host memory;
 * copied H2D inside the call) returning the loss to the host — the end-to-end entry point. */
int gss_engine_step(gss_engine* e, const gss_camera* cam, const float* gt_host, float* loss_host,
                    int32_t* valid_count_host);
/* gss_engine_step without the final wait: enqueues the iteration and returns; *loss_host (pinned
 * host memory, required) receives the loss when the iteration's render completes, and gt_host must
 * stay unchanged until then (gss_engine_drain waits for both). *valid_count_host is set on return.
 * Consecutive async steps overlap step g+1's ground-truth copy and host work with step g's kernels;
 * the trajectory is bit-identical to gss_engine_step / gss_engine_run. */
int gss_engine_step_async(gss_engine* e, const gss_camera* cam, const float* gt_host, float* loss_host,
                          int32_t* valid_count_host);
/* Applies the lazy update still owed by an open step() segment (run() always drains itself). */
int gss_engine_drain(gss_engine* e);
/* SplitTable (splitter.hpp:12-23) as the OffloadEngine constructor takes it (engine.hpp:62-68):
 * per stored camera (ncams = the engine's camera count, or 0 to clear) a split flag and the
 * column s in (0, W). run() then culls a split camera's left [0, s] and right [s, W] viewports,
 * renders the two sub-passes over their std::set_union and aggregates the gradients
 * (engine.hpp:266-273, 355-371; splitter.hpp:85-123). Not inside an open step() segment. */
int gss_engine_set_splits(gss_engine* e, int32_t ncams, const int32_t* split, const int32_t* column);
/* snapshot (engine.hpp:91-111): restored parameters, host n x 59. */
int gss_engine_snapshot(gss_engine* e, float* rows_out);
/* Raw tier state (stored, not restored) for parity checks; any pointer may be NULL. */
int gss_engine_state(gss_engine* e, float* geo_w, float* ng_w, float* ng_m, float* ng_v, uint8_t* ng_counter,
                     int64_t* steps2);
/* accum_grad_norm / accum_grad_count (engine.hpp:187-188). */
int gss_engine_accum(gss_engine* e, double* norm, int32_t* cnt);
int64_t gss_engine_count(gss_engine* e);
/* Per-stage device time of the last run in ms (CUDA events): cull, forward_params, render,
 * geo_update, handoff, lazy_update. */
int gss_engine_stage_ms(gss_engine* e, double* out6);
/* Kernel launches issued by the last run/step (for bench accounting). */
int64_t gss_engine_launches(gss_engine* e);
/* Live per-kernel timing (bench roofline of the dominant kernels): when on, every forward_kernel
 * (composite) and backward_kernel (sweep) launch of the engine is bracketed by CUDA events on its
 * stream and the composited contributions are counted. gss_engine_kernel_times drains, then
 * returns ms2[0..1] = total ms of the composite / sweep launches since the last call, n2[0..1] =
 * their launch counts, *contribs = contributions composited (= useful backward contributions). */
int gss_engine_kernel_timing(gss_engine* e, int32_t on);
/* TimelineRow (engine.hpp:22-28): one row per stage of every iteration since the timeline was
 * enabled; stage 0..5 = cull, forward_params, render, geo_update, handoff, lazy_update; worker 0 =
 * the device stream, 1 = the host-tier stream; t0/t1 = CUDA-event times in ns from the epoch
 * recorded by gss_engine_timeline_enable; bytes = the stage's algorithmic bytes (lazy update: the
 * reference tally 7*49*4 per touched row + n counter bytes, from the device touched count). */
typedef struct {
  int32_t iteration, stage, worker, pad;
  int64_t t0_ns, t1_ns;
  uint64_t bytes;
} gss_timeline_row;
int gss_engine_timeline_enable(gss_engine* e, int32_t on);
/* Drains, copies min(count, cap) rows, returns the row count (negative status on error). */
int64_t gss_engine_timeline(gss_engine* e, gss_timeline_row* rows, int64_t cap);
/* Test instrumentation (the reference's EngineConfig::stage_hook, engine.hpp:42-43): a device-side
 * sleep of ns[k % n] nanoseconds at the start of the k-th stage on that stage's stream, to shake the
 * two-stream schedule; n = 0 disables. Results must not change (every edge is an event). */
int gss_engine_stage_delays(gss_engine* e, const uint32_t* ns, int32_t n);
int gss_engine_kernel_times(gss_engine* e, double* ms2, int64_t* n2, uint64_t* contribs);
/* The same with every timed render phase: ms6 / n6 = composite, sweep, geometry (projection,
 * depth sort, binning, tile sort and ranges, including the instance-count round trip), colour,
 * per-slot sums, chain. */
int gss_engine_render_times(gss_engine* e, double* ms6, int64_t* n6, uint64_t* contribs);

/* ---- densification (trainer.hpp:166-213, engine.hpp:116-163) ------------- */
/* DensifyConfig (trainer.hpp:32-47): the thresholds of plan_densify. */
typedef struct {
  double grad_threshold;      /* densify when mean |d L / d mean2d| > this */
  double percent_dense;       /* clone below percent_dense * extent, split above */
  double opacity_prune;       /* prune sigmoid(opacity) < this */
  double split_scale_divisor; /* split children's scale shrinks by this */
} gss_densify_config;
/* plan_densify on a restored snapshot in device memory (rows n x 59) with device statistics
 * accum_norm (double[n]) / accum_cnt (int32[n]): survivors (device int32, capacity n) receive the
 * ascending kept ids, children (device, capacity 2n x 59) the appended rows in the reference's order;
 * counts_host[0..4] = survivors, children, clones, splits, pruned. Decisions and child rows are
 * bit-identical to the reference (the split children's Rng / libm part runs on the host). */
int gss_plan_densify(const float* rows, int64_t n, const double* accum_norm, const int32_t* accum_cnt,
                     const gss_densify_config* cfg, double extent, uint64_t seed, int32_t* survivors,
                     float* children, int64_t* counts_host, gss_stream_t stream);
/* A densification event of the engine (drains first): snapshot, plan, apply — survivors keep
 * their stored parameters, optimizer state and counters, children get zero state; statistics reset.
 * counts_host[0..5] = survivors, children, clones, splits, pruned, new Gaussian count. */
int gss_engine_densify(gss_engine* e, const gss_densify_config* cfg, double extent, uint64_t seed,
                       int64_t* counts_host);

/* ---- scene inputs (not on the hot path) ---------------------------------------------------- */
/* synth_scene parameter + camera generation (synth.hpp:100-154), bit-identical to the reference
 * generator; cfg[14] = box, radius_min, radius_max, fov_deg, fov_ramp, target_jitter, near, far,
 * scale_min, scale_max, scale_aniso, opacity_min, opacity_max, sh_rest_noise.
 * rows_out: host n x 59; cams_out: host cams. Ground truth is rendered with gss_rasterize_forward. */
int gss_synth_scene(uint64_t seed, int64_t n, int32_t cams, int32_t width, int32_t height, int32_t sh_degree,
                    const double* cfg, float* rows_out, gss_camera* cams_out);
/* init_gaussians (scene.hpp:146-195): one Gaussian per point (host positions m x 3, colors m x 3
 * or NULL) with the exact O(M^2) kNN log-scale (fp64 on the device), identity rotation, opacity
 * logit(init_opacity), DC colour; rows_out host m x 59, bit-identical to the reference. */
int gss_init_gaussians(const float* positions, const float* colors, int32_t m, int32_t knn, double min_knn_dist,
                       double init_opacity, float* rows_out);
/* load_ply (ply.hpp:10-14, ply.cpp:53-199) in two calls: gss_ply_open parses the header and
 * returns the vertex count and whether red/green/blue (or r/g/b) properties exist; gss_ply_read
 * decodes the vertex body into positions (m x 3) and colors (m x 3 or NULL), host or device
 * pointers. Binary little-endian bodies are streamed through pinned 32 MB chunks into HBM and
 * decoded by a kernel; ASCII bodies are tokenised on the host (strtod). Values, colour
 * normalisation and every ParseError message (status GSS_ERR_PARSE) follow the reference. */
typedef struct gss_ply gss_ply;
int gss_ply_open(const char* path, gss_ply** out, int64_t* vertex_count, int32_t* has_color);
int gss_ply_read(gss_ply* ply, float* positions, float* colors, gss_stream_t stream);
void gss_ply_close(gss_ply* ply);
/* save_ply (ply.hpp:16-17, ply.cpp:201-225): host positions m x 3, colors m x 3 or NULL (0.5 grey). */
int gss_save_ply(const char* path, const float* positions, const float* colors, int64_t m, int32_t binary);
/* look_at_camera (scene.hpp:99-126). */
int gss_look_at_camera(const float* eye, const float* target, float fx, float fy, int32_t w, int32_t h,
                       float near_p, float far_p, gss_camera* out);

#ifdef __cplusplus
}
#endif
#endif /* GSS_B200_H */
