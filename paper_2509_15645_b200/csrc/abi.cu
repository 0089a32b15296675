// extern "C" entry points of libgss_b200.so (declared in include/gss_b200.h). Each one validates
// its arguments, maps library exceptions to status codes and records the message for
// gss_last_error(). No entry point has a CPU fallback.
#include <atomic>
#include <cstring>
#include <string>

#include "common.cuh"

namespace gssd {
// cull.cu
size_t cull_workspace_bytes(int64_t n);
void cull(const float* geo, int64_t n, int64_t stride, const gss_camera* cam, const gss_viewport* vp, float lp,
          uint32_t* mask, int32_t* ids, int64_t* count, void* ws, size_t ws_bytes, cudaStream_t st);
void expf_device(const float* x, float* y, int64_t n, cudaStream_t st);
// adam.cu
void build_group_luts(double lr, double b1, double b2, double eps, int64_t t, int max_delay, float* param,
                      float* mom, float* var, float* pow_b1, float* pow_b2, float* scalars);
void adam_update(gss_arena* ap, const gss_sparse_grads* grads, int32_t* touched_ids, int64_t* touched_count,
                 cudaStream_t st, const uint32_t* split_mask = nullptr, cudaEvent_t split_before_set = nullptr);
void adam_dense(gss_arena* ap, const float* grads, cudaStream_t st);
void adam_flush(gss_arena* ap, cudaStream_t st);
void adam_restore(const gss_arena* ap, const int32_t* ids, int64_t count, const int64_t* count_dev,
                  const gss_sparse_grads* pending, float* out, cudaStream_t st, cudaEvent_t after_resolve = nullptr);
int arena_check(const gss_arena* ap, cudaStream_t st);
void arena_release(const gss_arena* ap);
void arena_access(const gss_arena* ap, uint64_t* out6);
void cull_workspace_release(const void* ws);
// raster.cu
gss_render_ctx* render_ctx_create();
void render_ctx_destroy(gss_render_ctx* ctx);
void rasterize_forward(gss_render_ctx* ctx, const gss_render_scene* scene, const gss_camera* cam,
                       const gss_viewport* vp, float* image, const float* gt, int64_t normalizer, float* d_img,
                       float* loss_dev, float* final_T_opt, int32_t* ncontrib_opt, int64_t* meta, cudaStream_t st);
void loss_l1(const float* image, const float* gt, int64_t elems, int64_t normalizer, float* d_img, float* loss_dev,
             cudaStream_t st);
void rasterize_backward(gss_render_ctx* ctx, const float* d_img, float* gg, int64_t gstride, float* gn,
                        int64_t nstride, float* mean2d, cudaStream_t st);
void image_sq_err(const float* a, const float* b, int64_t elems, double* sum_dev, cudaStream_t st);
void project(const gss_render_scene* scene, const gss_camera* cam, const gss_viewport* vp, void* records,
             cudaStream_t st);
void route_strips(const void* records, int64_t count, const int32_t* strip_x, int nstrips, int32_t* dest_slots,
                  int64_t* dest_counts, cudaStream_t st);
void gather_records(const void* records, const int32_t* slots, int64_t n, void* out, cudaStream_t st);
void scatter_add_rows(const float* src, const int32_t* slots, int64_t n, int width, float* dst, cudaStream_t st);
void rasterize_records_forward(gss_render_ctx* ctx, const void* records, int64_t count, const gss_camera* cam,
                               const gss_viewport* vp, const float* background, float* image, const float* gt,
                               int64_t normalizer, float* d_img, float* loss_dev, double* loss_sum_dev,
                               float* final_T_opt, int32_t* ncontrib_opt, int64_t* meta, cudaStream_t st);
void rasterize_records_backward(gss_render_ctx* ctx, const float* d_img, float* sums, cudaStream_t st);
void chain_backward(const gss_render_scene* scene, const gss_camera* cam, const void* records, const float* sums,
                    float* gg, int64_t gstride, float* gn, int64_t nstride, float* mean2d, cudaStream_t st);
void raster_stats(uint64_t* out8, bool reset);
int raster_stats_enabled();
// ply.cu
gss_ply* ply_open(const char* path, int64_t* count, int32_t* has_color);
void ply_read(gss_ply* p, float* pos, float* col, cudaStream_t st);
void ply_close(gss_ply* p);
void save_ply(const char* path, const float* pos, const float* col, int64_t m, bool binary);
// engine.cu
void engine_config_default(gss_engine_config* c);
void init_gaussians(const float* positions, const float* colors, int m, int knn, double min_knn_dist,
                    double init_opacity, float* rows_out);
void engine_densify(gss_engine* e, const gss_densify_config* dc, double extent, uint64_t seed, int64_t* counts);
void plan_densify(const float* rows, int64_t n, const double* norm, const int32_t* cnt,
                  const gss_densify_config* dc, double extent, uint64_t seed, int32_t* survivors, float* children,
                  int64_t* counts, cudaStream_t st);
gss_engine* engine_create(int64_t n, const float* rows, int32_t ncams, const gss_camera* cams, const float* gts,
                          const gss_engine_config* cfg);
void engine_destroy(gss_engine* e);
void engine_run(gss_engine* e, int iters, float* losses, int32_t* valid);
void engine_step(gss_engine* e, const gss_camera* cam, const float* gt_host, float* loss_host, int32_t* valid_host,
                 bool wait);
void engine_drain(gss_engine* e);
void engine_set_splits(gss_engine* e, int32_t ncams, const int32_t* split, const int32_t* column);
void set_host_chunk_bytes(int64_t bytes);
void engine_snapshot(gss_engine* e, float* rows_out);
void engine_state(gss_engine* e, float* geo_w, float* ng_w, float* ng_m, float* ng_v, uint8_t* ng_counter,
                  int64_t* steps2);
void engine_accum(gss_engine* e, double* norm, int32_t* cnt);
void engine_stage_ms(gss_engine* e, double* out6);
int64_t engine_launches(gss_engine* e);
void engine_kernel_timing(gss_engine* e, bool on);
void engine_timeline_enable(gss_engine* e, bool on);
int64_t engine_timeline(gss_engine* e, gss_timeline_row* rows, int64_t cap);
void engine_stage_delays(gss_engine* e, const uint32_t* ns, int n);
void engine_kernel_times(gss_engine* e, double* ms2, int64_t* n2, uint64_t* contribs, int nk);
int64_t engine_count(gss_engine* e);

namespace {
thread_local std::string t_err;
std::atomic<int64_t> g_launches{0};

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw Error(GSS_ERR_CUDA, "no CUDA device: libgss_b200 has no CPU fallback");
  }
  // The kernels' scratch comes from the stream-ordered pool; keep freed blocks cached in the pool
  // (the default release threshold 0 returns them to the driver at every sync, turning each
  // scratch allocation into a full device allocation).
  static thread_local int pooled_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess && dev != pooled_dev) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    pooled_dev = dev;
  }
}
}  // namespace

constexpr int kMaxDevices = 64;
std::atomic<int> g_sms[kMaxDevices];

int sm_count() {
  int dev = 0;
  GSS_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) {
    int sms = 0;
    GSS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return sms;
  }
  int sms = g_sms[dev].load(std::memory_order_relaxed);
  if (sms == 0) {
    GSS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    g_sms[dev].store(sms, std::memory_order_relaxed);
  }
  return sms;
}

void set_max_dynamic_smem(const void* fn, int bytes) {
  cudaFuncAttributes fa{};
  GSS_CUDA(cudaFuncGetAttributes(&fa, fn));
  if (fa.maxDynamicSharedSizeBytes < bytes)
    GSS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

void set_error(const std::string& msg) { t_err = msg; }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launches() { return g_launches.load(std::memory_order_relaxed); }

}  // namespace gssd

using namespace gssd;

#define GSS_API extern "C" __attribute__((visibility("default")))

GSS_API const char* gss_last_error(void) { return t_err.c_str(); }
GSS_API int32_t gss_abi_version(void) { return 2; }
GSS_API int32_t gss_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}
GSS_API int64_t gss_launch_count(void) { return launches(); }

GSS_API int gss_expf_device(const float* x, float* y, int64_t n, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    require(n >= 0 && (n == 0 || (x && y)), "expf: bad arguments");
    expf_device(x, y, n, as_stream(stream));
  });
}

GSS_API size_t gss_cull_workspace_bytes(int64_t n) { return cull_workspace_bytes(n); }

GSS_API int gss_cull(const float* geo, int64_t n, int64_t stride, const gss_camera* cam, const gss_viewport* vp,
                     float low_pass, uint32_t* mask_opt, int32_t* ids_out, int64_t* count_dev, void* workspace,
                     size_t workspace_bytes, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    cull(geo, n, stride, cam, vp, low_pass, mask_opt, ids_out, count_dev, workspace, workspace_bytes,
         as_stream(stream));
  });
}

GSS_API int gss_build_group_luts(double lr, double beta1, double beta2, double eps, int64_t t, int32_t max_delay,
                                 float* param, float* mom, float* var, float* pow_b1, float* pow_b2, float* scalars) {
  return guarded([&] {
    require(t >= 1, "build_group_luts: t must be >= 1");
    require(max_delay >= 0 && max_delay <= 254, "build_group_luts: max_delay must be in [0, 254]");
    require(param && scalars, "build_group_luts: null output");
    build_group_luts(lr, beta1, beta2, eps, t, max_delay, param, mom, var, pow_b1, pow_b2, scalars);
  });
}

GSS_API int gss_adam_step_dense(gss_arena* arena, const float* grads, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    adam_dense(arena, grads, as_stream(stream));
  });
}

GSS_API int gss_deferred_update(gss_arena* arena, const gss_sparse_grads* grads, int32_t* touched_ids,
                                int64_t* touched_count_dev, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    adam_update(arena, grads, touched_ids, touched_count_dev, as_stream(stream));
  });
}

GSS_API int gss_restore_view(const gss_arena* arena, const int32_t* ids, int64_t count, const int64_t* ids_count_dev,
                             const gss_sparse_grads* pending, float* out_rows, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    adam_restore(arena, ids, count, ids_count_dev, pending, out_rows, as_stream(stream));
  });
}

GSS_API int gss_flush_deferred(gss_arena* arena, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    adam_flush(arena, as_stream(stream));
  });
}

GSS_API int gss_arena_check(const gss_arena* arena, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    arena_check(arena, as_stream(stream));
  });
}

GSS_API int gss_arena_release(const gss_arena* arena) {
  return guarded([&] { arena_release(arena); });
}

GSS_API void gss_cull_workspace_release(const void* workspace) { cull_workspace_release(workspace); }

GSS_API gss_render_ctx* gss_render_ctx_create(void) {
  gss_render_ctx* c = nullptr;
  const int st = guarded([&] { c = render_ctx_create(); });
  return st == GSS_OK ? c : nullptr;
}
GSS_API void gss_render_ctx_destroy(gss_render_ctx* ctx) { render_ctx_destroy(ctx); }

GSS_API int gss_rasterize_forward(gss_render_ctx* ctx, const gss_render_scene* scene, const gss_camera* cam,
                                  const gss_viewport* vp, float* image, const float* gt, int64_t normalizer,
                                  float* d_img, float* loss_dev, float* final_T_opt, int32_t* n_contrib_opt,
                                  int64_t* meta_host, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    rasterize_forward(ctx, scene, cam, vp, image, gt, normalizer, d_img, loss_dev, final_T_opt, n_contrib_opt,
                      meta_host, as_stream(stream));
  });
}

GSS_API int gss_loss_l1(const float* image, const float* gt, int64_t elems, int64_t normalizer, float* d_img,
                        float* loss_dev, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    loss_l1(image, gt, elems, normalizer, d_img, loss_dev, as_stream(stream));
  });
}

GSS_API int gss_rasterize_backward(gss_render_ctx* ctx, const float* d_img, float* grad_geo, int64_t geo_stride,
                                   float* grad_nongeo, int64_t ng_stride, float* mean2d_opt, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    rasterize_backward(ctx, d_img, grad_geo, geo_stride, grad_nongeo, ng_stride, mean2d_opt, as_stream(stream));
  });
}

GSS_API int gss_image_sq_err(const float* a, const float* b, int64_t elems, double* sum_dev, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    image_sq_err(a, b, elems, sum_dev, as_stream(stream));
  });
}

GSS_API int gss_project(const gss_render_scene* scene, const gss_camera* cam, const gss_viewport* vp,
                        void* records, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    project(scene, cam, vp, records, as_stream(stream));
  });
}

GSS_API int gss_route_strips(const void* records, int64_t count, const int32_t* strip_x, int32_t nstrips,
                             int32_t* dest_slots, int64_t* dest_counts, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    route_strips(records, count, strip_x, nstrips, dest_slots, dest_counts, as_stream(stream));
  });
}

GSS_API int gss_gather_records(const void* records, const int32_t* slots, int64_t n, void* out, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    gather_records(records, slots, n, out, as_stream(stream));
  });
}

GSS_API int gss_scatter_add_rows(const float* src, const int32_t* slots, int64_t n, int32_t width, float* dst,
                                 gss_stream_t stream) {
  return guarded([&] {
    require_device();
    scatter_add_rows(src, slots, n, width, dst, as_stream(stream));
  });
}

GSS_API int gss_rasterize_records_forward(gss_render_ctx* ctx, const void* records, int64_t count,
                                          const gss_camera* cam, const gss_viewport* vp, const float* background,
                                          float* image, const float* gt, int64_t normalizer, float* d_img,
                                          float* loss_dev, double* loss_sum_dev, float* final_T_opt,
                                          int32_t* n_contrib_opt, int64_t* meta_host, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    rasterize_records_forward(ctx, records, count, cam, vp, background, image, gt, normalizer, d_img, loss_dev,
                              loss_sum_dev, final_T_opt, n_contrib_opt, meta_host, as_stream(stream));
  });
}

GSS_API int gss_rasterize_records_backward(gss_render_ctx* ctx, const float* d_img, float* sums,
                                           gss_stream_t stream) {
  return guarded([&] {
    require_device();
    rasterize_records_backward(ctx, d_img, sums, as_stream(stream));
  });
}

GSS_API int gss_chain_backward(const gss_render_scene* scene, const gss_camera* cam, const void* records,
                               const float* sums, float* grad_geo, int64_t geo_stride, float* grad_nongeo,
                               int64_t ng_stride, float* mean2d_opt, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    chain_backward(scene, cam, records, sums, grad_geo, geo_stride, grad_nongeo, ng_stride, mean2d_opt,
                   as_stream(stream));
  });
}

GSS_API int gss_plan_densify(const float* rows, int64_t n, const double* accum_norm, const int32_t* accum_cnt,
                             const gss_densify_config* cfg, double extent, uint64_t seed, int32_t* survivors,
                             float* children, int64_t* counts_host, gss_stream_t stream) {
  return guarded([&] {
    require_device();
    plan_densify(rows, n, accum_norm, accum_cnt, cfg, extent, seed, survivors, children, counts_host,
                 as_stream(stream));
  });
}

GSS_API int gss_engine_densify(gss_engine* e, const gss_densify_config* cfg, double extent, uint64_t seed,
                               int64_t* counts_host) {
  return guarded([&] {
    require_device();
    engine_densify(e, cfg, extent, seed, counts_host);
  });
}

GSS_API int gss_init_gaussians(const float* positions, const float* colors, int32_t m, int32_t knn,
                               double min_knn_dist, double init_opacity, float* rows_out) {
  return guarded([&] {
    require_device();
    init_gaussians(positions, colors, m, knn, min_knn_dist, init_opacity, rows_out);
  });
}

GSS_API int gss_arena_access(const gss_arena* arena, uint64_t* out6) {
  return guarded([&] {
    require_device();
    arena_access(arena, out6);
  });
}
GSS_API int gss_raster_stats(uint64_t* out8, int32_t reset) {
  return guarded([&] {
    require_device();
    require(out8 != nullptr, "raster_stats: null output");
    GSS_CUDA(cudaDeviceSynchronize());
    raster_stats(out8, reset != 0);
  });
}
GSS_API int32_t gss_raster_stats_enabled(void) { return raster_stats_enabled(); }

GSS_API int gss_ply_open(const char* path, gss_ply** out, int64_t* vertex_count, int32_t* has_color) {
  return guarded([&] {
    require(out != nullptr, "ply: null output handle");
    *out = nullptr;
    *out = ply_open(path, vertex_count, has_color);
  });
}
GSS_API int gss_ply_read(gss_ply* ply, float* positions, float* colors, gss_stream_t stream) {
  return guarded([&] { ply_read(ply, positions, colors, as_stream(stream)); });
}
GSS_API void gss_ply_close(gss_ply* ply) { ply_close(ply); }
GSS_API int gss_save_ply(const char* path, const float* positions, const float* colors, int64_t m, int32_t binary) {
  return guarded([&] { save_ply(path, positions, colors, m, binary != 0); });
}

GSS_API void gss_engine_config_default(gss_engine_config* cfg) {
  if (cfg) engine_config_default(cfg);
}

GSS_API gss_engine* gss_engine_create(int64_t n, const float* init_rows, int32_t ncams, const gss_camera* cams,
                                      const float* gts, const gss_engine_config* cfg) {
  gss_engine* e = nullptr;
  const int st = guarded([&] {
    require_device();
    e = engine_create(n, init_rows, ncams, cams, gts, cfg);
  });
  return st == GSS_OK ? e : nullptr;
}
GSS_API void gss_engine_destroy(gss_engine* e) { engine_destroy(e); }
GSS_API int gss_engine_run(gss_engine* e, int32_t iters, float* losses, int32_t* valid_counts) {
  return guarded([&] { engine_run(e, iters, losses, valid_counts); });
}
GSS_API int gss_engine_step(gss_engine* e, const gss_camera* cam, const float* gt_host, float* loss_host,
                            int32_t* valid_count_host) {
  return guarded([&] { engine_step(e, cam, gt_host, loss_host, valid_count_host, true); });
}

GSS_API int gss_engine_step_async(gss_engine* e, const gss_camera* cam, const float* gt_host, float* loss_host,
                                  int32_t* valid_count_host) {
  return guarded([&] {
    require_device();
    engine_step(e, cam, gt_host, loss_host, valid_count_host, false);
  });
}
GSS_API int gss_set_host_chunk_bytes(int64_t bytes) {
  return guarded([&] {
    require(bytes > 0, "chunk bytes must be > 0");
    set_host_chunk_bytes(bytes);
  });
}
GSS_API int gss_engine_set_splits(gss_engine* e, int32_t ncams, const int32_t* split, const int32_t* column) {
  return guarded([&] { engine_set_splits(e, ncams, split, column); });
}
GSS_API int gss_engine_drain(gss_engine* e) {
  return guarded([&] { engine_drain(e); });
}
GSS_API int gss_engine_snapshot(gss_engine* e, float* rows_out) {
  return guarded([&] { engine_snapshot(e, rows_out); });
}
GSS_API int gss_engine_state(gss_engine* e, float* geo_w, float* ng_w, float* ng_m, float* ng_v, uint8_t* ng_counter,
                             int64_t* steps2) {
  return guarded([&] { engine_state(e, geo_w, ng_w, ng_m, ng_v, ng_counter, steps2); });
}
GSS_API int gss_engine_accum(gss_engine* e, double* norm, int32_t* cnt) {
  return guarded([&] { engine_accum(e, norm, cnt); });
}
GSS_API int64_t gss_engine_count(gss_engine* e) { return engine_count(e); }
GSS_API int gss_engine_stage_ms(gss_engine* e, double* out6) {
  return guarded([&] { engine_stage_ms(e, out6); });
}
GSS_API int64_t gss_engine_launches(gss_engine* e) { return engine_launches(e); }
GSS_API int gss_engine_kernel_timing(gss_engine* e, int32_t on) {
  return guarded([&] { engine_kernel_timing(e, on != 0); });
}
GSS_API int gss_engine_timeline_enable(gss_engine* e, int32_t on) {
  return guarded([&] { engine_timeline_enable(e, on != 0); });
}
GSS_API int64_t gss_engine_timeline(gss_engine* e, gss_timeline_row* rows, int64_t cap) {
  int64_t n = 0;
  const int st = guarded([&] { n = engine_timeline(e, rows, cap); });
  return st == GSS_OK ? n : -st;
}
GSS_API int gss_engine_stage_delays(gss_engine* e, const uint32_t* ns, int32_t n) {
  return guarded([&] { engine_stage_delays(e, ns, n); });
}
GSS_API int gss_engine_render_times(gss_engine* e, double* ms6, int64_t* n6, uint64_t* contribs) {
  return guarded([&] { engine_kernel_times(e, ms6, n6, contribs, 6); });
}
GSS_API int gss_engine_kernel_times(gss_engine* e, double* ms2, int64_t* n2, uint64_t* contribs) {
  return guarded([&] { engine_kernel_times(e, ms2, n2, contribs, 2); });
}
