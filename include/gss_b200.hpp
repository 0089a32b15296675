// gss_b200.hpp — drop-in C++ API for the reference's hot path, backed by libgss_b200.so.
//
// Needs the reference headers on the include path (gss/render.hpp, gss/adam.hpp, gss/engine.hpp
// are included here); every function keeps the
// reference signature (namespace gss -> gss_b200) and semantics, and runs on the B200 through
// the C ABI in gss_b200.h. Inputs are the reference's host containers: they are copied to the
// device, processed by the sm_100a kernels and copied back, so a caller of the reference path
// switches by changing the namespace. Hot loops that keep state resident in HBM use the C ABI
// (or gss_engine_*) directly instead.
//
//   reference (file:line)                         drop-in
//   frustum_cull        render.hpp:253-260        gss_b200::frustum_cull
//   rasterize_forward   render.hpp:384-464        gss_b200::rasterize_forward (-> gss_b200::RenderResult)
//   compute_loss_l1     render.hpp:497-511        gss_b200::compute_loss_l1
//   rasterize_backward  render.hpp:526-640        gss_b200::rasterize_backward (<- gss_b200::RenderResult)
//   OffloadEngine       engine.hpp:55-522         gss_b200::OffloadEngine (EngineConfig<float>, SplitTable)
//   adam_step_dense     adam.hpp:198-207          gss_b200::adam_step_dense
//   deferred_update     adam.hpp:211-238          gss_b200::deferred_update
//   restore_view        adam.hpp:252-289          gss_b200::restore_view
//   flush_deferred      adam.hpp:293-313          gss_b200::flush_deferred
//
// Errors map to the reference's exception types: status 2 -> gss::ConfigError (or
// std::invalid_argument where the reference throws it), 3 -> gss::InvariantViolation,
// 4 -> gss::ParseError, 1 (CUDA) -> std::runtime_error. The arena's AccessReport tally
// (adam.hpp:36-50) is maintained on the device and added to the reference arena's.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include <gss/adam.hpp>
#include <gss/engine.hpp>
#include <gss/render.hpp>

#include "gss_b200.h"

namespace gss_b200 {

inline void check(int st, bool invalid_argument = false) {
  if (st == GSS_OK) return;
  const std::string msg = gss_last_error();
  if (st == GSS_ERR_INVALID) {
    if (invalid_argument) throw std::invalid_argument(msg);
    throw gss::ConfigError(msg);
  }
  if (st == GSS_ERR_INVARIANT) throw gss::InvariantViolation(msg);
  if (st == GSS_ERR_PARSE) throw gss::ParseError(msg);
  throw std::runtime_error(msg);
}

inline void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
}

// Owning device buffer.
template <class T> class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t n) { resize(n); }
  DevBuf(const T* host, size_t n) { upload(host, n); }
  ~DevBuf() { reset(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  void reset() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  void resize(size_t n) {
    reset();
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&p_), std::max<size_t>(n, 1) * sizeof(T)));
    n_ = n;
  }
  void zero() { cuda_check(cudaMemset(p_, 0, std::max<size_t>(n_, 1) * sizeof(T))); }
  void upload(const T* host, size_t n) {
    resize(n);
    if (n) cuda_check(cudaMemcpy(p_, host, n * sizeof(T), cudaMemcpyHostToDevice));
  }
  void download(T* host, size_t n) const {
    if (n) cuda_check(cudaMemcpy(host, p_, n * sizeof(T), cudaMemcpyDeviceToHost));
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

inline const gss_camera* cam_ptr(const gss::Camera<float>& c) {
  static_assert(sizeof(gss::Camera<float>) == sizeof(gss_camera), "Camera<float> must be the 80-byte gss_camera");
  return reinterpret_cast<const gss_camera*>(&c);
}
inline gss_viewport vp_of(const gss::Viewport<float>& v) { return gss_viewport{v.x0, v.x1, v.y0, v.y1}; }

// ---- frustum_cull (render.hpp:253-260) ---------------------------------------------------
inline std::vector<int> frustum_cull(gss::RowView<float> geo, int count, const gss::Camera<float>& cam,
                                     const gss::Viewport<float>& vp, float low_pass = float(gss::kLowPass)) {
  if (count <= 0) return {};
  const size_t stride = geo.stride;
  DevBuf<float> g(geo.data, size_t(count) * stride);
  DevBuf<int32_t> ids(count);
  DevBuf<int64_t> cnt(1);
  const size_t wsb = gss_cull_workspace_bytes(count);
  DevBuf<unsigned char> ws(wsb);
  ws.zero();
  const gss_viewport v = vp_of(vp);
  check(gss_cull(g.get(), count, int64_t(stride), cam_ptr(cam), &v, low_pass, nullptr, ids.get(), cnt.get(), ws.get(),
                 wsb, nullptr));
  int64_t n = 0;
  cnt.download(&n, 1);
  std::vector<int> out(static_cast<size_t>(n));
  ids.download(out.data(), out.size());
  return out;
}

// ---- optimizer (adam.hpp:198-313) --------------------------------------------------------
// A device mirror of a reference Arena<float>: uploaded on construction, written back by sync().
class DevArena {
 public:
  explicit DevArena(const gss::Arena<float>& a)
      : w_(a.w.data(), a.w.size()), m_(a.m.data(), a.m.size()), v_(a.v.data(), a.v.size()),
        c_(a.counter.data(), a.counter.size()) {
    s_ = gss_arena{};
    s_.w = w_.get(); s_.m = m_.get(); s_.v = v_.get(); s_.counter = c_.get();
    s_.n = a.count; s_.dim = a.dim; s_.defer_max = a.defer_max; s_.step = a.step;
    if (a.groups.size() > 8) throw gss::ConfigError("arena: at most 8 groups on the device");
    s_.ngroups = int32_t(a.groups.size());
    for (size_t i = 0; i < a.groups.size(); ++i) {
      const auto& g = a.groups[i];
      s_.groups[i] = gss_group{g.col0, g.dim, g.hp.lr, g.hp.beta1, g.hp.beta2, g.hp.eps};
    }
  }
  ~DevArena() { gss_arena_release(&s_); }
  DevArena(const DevArena&) = delete;
  DevArena& operator=(const DevArena&) = delete;
  gss_arena* get() { return &s_; }
  const gss_arena* get() const { return &s_; }
  void sync(gss::Arena<float>& a) const {
    w_.download(a.w.data(), a.w.size());
    m_.download(a.m.data(), a.m.size());
    v_.download(a.v.data(), a.v.size());
    c_.download(a.counter.data(), a.counter.size());
    a.step = s_.step;
    add_access(a.access);
  }
  // The device AccessReport tally of this transient mirror, added to the reference arena's
  // (adam.hpp:36-50; restore_view mutates it through a const arena, as adam.hpp:254 does).
  void add_access(gss::AccessReport& r) const {
    uint64_t t[6] = {0, 0, 0, 0, 0, 0};
    check(gss_arena_access(&s_, t));
    r.update_passes += t[0];
    r.touched_rows += t[1];
    r.param_bytes += t[2];
    r.counter_bytes += t[3];
    r.restore_rows += t[4];
    r.restore_read_bytes += t[5];
  }

 private:
  DevBuf<float> w_, m_, v_;
  DevBuf<uint8_t> c_;
  gss_arena s_{};
};

struct DevGrads {
  DevBuf<int32_t> ids;
  DevBuf<float> rows;
  gss_sparse_grads g{};
  DevGrads(const gss::SparseGrads<float>& s, int dim) {
    const size_t k = s.ids.size();
    ids.upload(s.ids.data(), k);
    // rows are addressed as rows + i*stride + col0 .. + dim: upload the span that covers them
    const size_t span = k ? (k - 1) * s.stride + size_t(s.col0) + size_t(dim) : 0;
    rows.upload(s.rows, span);
    g = gss_sparse_grads{ids.get(), int64_t(k), nullptr, rows.get(), int64_t(s.stride), s.col0};
  }
};

inline void adam_step_dense(gss::Arena<float>& a, const float* grads) {
  DevArena d(a);
  DevBuf<float> g;
  if (grads) g.upload(grads, size_t(a.count) * a.dim);
  check(gss_adam_step_dense(d.get(), grads ? g.get() : nullptr, nullptr));
  cuda_check(cudaDeviceSynchronize());
  d.sync(a);
}

inline std::vector<int> deferred_update(gss::Arena<float>& a, const gss::SparseGrads<float>& grads) {
  DevArena d(a);
  DevGrads g(grads, a.dim);
  DevBuf<int32_t> touched(size_t(std::max(a.count, 1)));
  DevBuf<int64_t> tcount(1);
  check(gss_deferred_update(d.get(), &g.g, touched.get(), tcount.get(), nullptr));
  check(gss_arena_check(d.get(), nullptr));  // unsorted ids -> InvariantViolation (adam.hpp:231)
  d.sync(a);
  int64_t n = 0;
  tcount.download(&n, 1);
  std::vector<int> out(static_cast<size_t>(n));
  touched.download(out.data(), out.size());
  return out;
}

inline void restore_view(const gss::Arena<float>& a, std::span<const int> ids, const gss::SparseGrads<float>* pending,
                         float* out) {
  DevArena d(a);
  DevBuf<int32_t> di(ids.data(), ids.size());
  DevBuf<float> o(ids.size() * size_t(a.dim));
  if (pending) {
    DevGrads g(*pending, a.dim);
    check(gss_restore_view(d.get(), di.get(), int64_t(ids.size()), nullptr, &g.g, o.get(), nullptr));
    cuda_check(cudaDeviceSynchronize());
  } else {
    check(gss_restore_view(d.get(), di.get(), int64_t(ids.size()), nullptr, nullptr, o.get(), nullptr));
  }
  o.download(out, ids.size() * size_t(a.dim));
  d.add_access(const_cast<gss::Arena<float>&>(a).access);
}

inline void flush_deferred(gss::Arena<float>& a) {
  DevArena d(a);
  check(gss_flush_deferred(d.get(), nullptr));
  cuda_check(cudaDeviceSynchronize());
  d.sync(a);
}

// ---- compute_loss_l1 (render.hpp:497-511) -------------------------------------------------
inline float compute_loss_l1(const gss::Image<float>& img, const gss::Image<float>& gt, gss::Image<float>& d_img,
                             size_t normalizer = 0) {
  if (img.width != gt.width || img.height != gt.height)
    throw std::invalid_argument("compute_loss_l1: image and ground-truth shapes differ");
  const size_t n = img.data.size();
  DevBuf<float> di(img.data.data(), n), dg(gt.data.data(), n), dd(n), dl(1);
  check(gss_loss_l1(di.get(), dg.get(), int64_t(n), int64_t(normalizer), dd.get(), dl.get(), nullptr), true);
  d_img = gss::Image<float>(img.width, img.height);
  dd.download(d_img.data.data(), n);
  float loss = 0.0f;
  dl.download(&loss, 1);
  return loss;
}

// ---- rasterize_forward / rasterize_backward (render.hpp:384-640) ------------------------
// The device RenderResult: forward() keeps the splat records, sorted tile lists and per-pixel aux
// on the device for backward(), as RenderResult carries them between the two reference calls.
class Rasterizer {
 public:
  Rasterizer() : ctx_(gss_render_ctx_create()) {}
  ~Rasterizer() { gss_render_ctx_destroy(ctx_); }
  Rasterizer(const Rasterizer&) = delete;
  Rasterizer& operator=(const Rasterizer&) = delete;

  gss::Image<float> forward(const gss::RenderScene<float>& sc, const gss::Camera<float>& cam,
                            const gss::Viewport<float>& vp) {
    const size_t V = sc.ids.size();
    int nrows = 0;
    for (int id : sc.ids) nrows = std::max(nrows, id + 1);
    ids_.upload(sc.ids.data(), V);
    geo_.upload(sc.geo.data, size_t(nrows) * sc.geo.stride);
    const size_t ng_rows = sc.nongeo.compact ? V : size_t(nrows);
    size_t ng_rows_used = ng_rows;
    if (sc.nongeo.compact && sc.nongeo.slot_map)
      for (size_t k = 0; k < V; ++k) ng_rows_used = std::max(ng_rows_used, size_t(sc.nongeo.slot_map[k]) + 1);
    ng_.upload(sc.nongeo.data, ng_rows_used * sc.nongeo.stride);
    if (sc.nongeo.slot_map) slot_.upload(sc.nongeo.slot_map, V);
    gss_render_scene s{};
    s.ids = ids_.get();
    s.count = int64_t(V);
    s.geo = geo_.get();
    s.geo_stride = int64_t(sc.geo.stride);
    s.nongeo = ng_.get();
    s.nongeo_stride = int64_t(sc.nongeo.stride);
    s.nongeo_compact = sc.nongeo.compact ? 1 : 0;
    s.slot_map = sc.nongeo.slot_map ? slot_.get() : nullptr;
    s.sh_degree = sc.sh_degree;
    s.background[0] = sc.background.x;
    s.background[1] = sc.background.y;
    s.background[2] = sc.background.z;
    s.low_pass = sc.low_pass;
    const gss_viewport v = vp_of(vp);
    // pixel window (render.hpp:297-304) is reported back through meta
    int64_t meta[6] = {0, 0, 0, 0, 0, 0};
    const int W = std::max(cam.width, 1), H = std::max(cam.height, 1);
    img_.resize(size_t(W) * H * 3);
    check(gss_rasterize_forward(ctx_, &s, cam_ptr(cam), &v, img_.get(), nullptr, 0, nullptr, nullptr, nullptr,
                                nullptr, meta, nullptr));
    ids_host_.assign(sc.ids.begin(), sc.ids.end());
    gss::Image<float> out(static_cast<int>(meta[2]), static_cast<int>(meta[3]));
    img_.download(out.data.data(), out.data.size());
    return out;
  }

  gss::GradBuffer<float> backward(const gss::Image<float>& d_img) {
    gss::GradBuffer<float> gb;
    const size_t V = ids_host_.size();
    gb.ids = ids_host_;
    gb.rows.assign(V * gss::kParamDim, 0.0f);
    gb.mean2d.assign(V * 2, 0.0f);
    DevBuf<float> dd(d_img.data.data(), d_img.data.size());
    DevBuf<float> rows(V * gss::kParamDim), m2d(V * 2);
    check(gss_rasterize_backward(ctx_, dd.get(), rows.get(), gss::kParamDim, rows.get() + gss::kGeoDim,
                                 gss::kParamDim, m2d.get(), nullptr));
    rows.download(gb.rows.data(), gb.rows.size());
    m2d.download(gb.mean2d.data(), gb.mean2d.size());
    return gb;
  }

 private:
  gss_render_ctx* ctx_;
  DevBuf<int32_t> ids_, slot_;
  DevBuf<float> geo_, ng_, img_;
  std::vector<int> ids_host_;
};

// Reference-signature free functions (render.hpp:384, 526). gss_b200::RenderResult carries what
// the reference's RenderResult<float> carries between the two calls — the image (sized to the
// viewport's pixel window) and the window origin in `aux` — while the splat records, sorted tile
// lists and per-pixel aux stay on the device (the `dev` handle) for rasterize_backward. `workers`
// is accepted and ignored (the device schedules itself).
struct RenderAux {
  int px0 = 0, py0 = 0, pw = 0, ph = 0;
  size_t device_bytes = 0;
  size_t byte_size() const { return device_bytes; }
};
struct RenderResult {
  gss::Image<float> image;
  RenderAux aux;
  std::shared_ptr<Rasterizer> dev;
};

inline RenderResult rasterize_forward(const gss::RenderScene<float>& sc, const gss::Camera<float>& cam,
                                      const gss::Viewport<float>& vp, int workers = 1) {
  (void)workers;
  RenderResult rr;
  rr.dev = std::make_shared<Rasterizer>();
  rr.image = rr.dev->forward(sc, cam, vp);
  const gss::detail::PixWindow w = gss::detail::viewport_pixels(vp);
  rr.aux.px0 = w.px0;
  rr.aux.py0 = w.py0;
  rr.aux.pw = rr.image.width;
  rr.aux.ph = rr.image.height;
  // per-pixel final T + last index + image on the device, 64-byte splat records
  rr.aux.device_bytes = size_t(rr.aux.pw) * rr.aux.ph * 4 * 5 + sc.ids.size() * 64;
  return rr;
}

inline gss::GradBuffer<float> rasterize_backward(const gss::RenderScene<float>& sc, const gss::Camera<float>& cam,
                                                 const RenderResult& rr, const gss::Image<float>& d_img,
                                                 int workers = 1) {
  (void)cam;
  (void)workers;
  if (!rr.dev) throw gss::InvariantViolation("rasterize_backward: RenderResult has no device state");
  if (d_img.width != rr.image.width || d_img.height != rr.image.height)
    throw std::invalid_argument("rasterize_backward: d_img shape differs from the rendered window");
  gss::GradBuffer<float> gb = rr.dev->backward(d_img);
  if (gb.ids.size() != sc.ids.size()) throw gss::InvariantViolation("rasterize_backward: scene differs from forward");
  return gb;
}

// ---- OffloadEngine (engine.hpp:55-522) ----------------------------------------------------
// The reference's engine interface over gss_engine_*: the same constructor arguments
// (GaussianSet, cameras, ground truths, EngineConfig<float>, SplitTable), run(n) returning the
// per-iteration {loss, valid_count}, snapshot(), the densification statistics and the timeline.
// The engine keeps every tier on the device (or the non-geometric tier in pinned host memory when
// nongeo_on_host is set); nothing crosses back to the host per iteration except the losses.
class OffloadEngine {
 public:
  struct IterResult {
    float loss{};
    int valid_count = 0;
  };

  OffloadEngine(const gss::GaussianSet<float>& init, std::vector<gss::Camera<float>> cams,
                std::vector<gss::Image<float>> gts, gss::EngineConfig<float> cfg, gss::SplitTable splits = {},
                bool nongeo_on_host = false)
      : cams_(std::move(cams)), sh_degree_(cfg.sh_degree) {
    if (gts.size() != cams_.size()) throw gss::ConfigError("OffloadEngine: one ground truth per camera");
    const int n = init.count;
    std::vector<float> rows(size_t(n) * gss::kParamDim);
    for (int i = 0; i < n; ++i) init.full_row(i, rows.data() + size_t(i) * gss::kParamDim);
    std::vector<float> g;
    for (size_t k = 0; k < gts.size(); ++k) {
      if (gts[k].width != cams_[k].width || gts[k].height != cams_[k].height)
        throw gss::ConfigError("OffloadEngine: ground truth shape differs from its camera");
      g.insert(g.end(), gts[k].data.begin(), gts[k].data.end());
    }
    gss_engine_config c{};
    gss_engine_config_default(&c);
    const gss::OptimConfig& o = cfg.optim;
    c.lr_mean = o.lr_mean; c.lr_scale = o.lr_scale; c.lr_quat = o.lr_quat; c.lr_opacity = o.lr_opacity;
    c.lr_sh = o.lr_sh; c.sh_rest_divisor = o.sh_rest_divisor; c.beta1 = o.beta1; c.beta2 = o.beta2; c.eps = o.eps;
    c.scene_extent = o.scene_extent; c.defer_max = o.defer_max; c.geo_defer_max = o.geo_defer_max;
    c.pipelined = cfg.pipelined ? 1 : 0;
    c.sh_degree = cfg.sh_degree;
    c.sh_warmup_step = cfg.sh_warmup_step;
    c.background[0] = cfg.background.x; c.background[1] = cfg.background.y; c.background[2] = cfg.background.z;
    c.low_pass = cfg.low_pass;
    c.nongeo_on_host = nongeo_on_host ? 1 : 0;
    c.chunk_bytes = int64_t(cfg.chunk_bytes);
    std::vector<gss_camera> gc(cams_.size());
    for (size_t k = 0; k < cams_.size(); ++k) gc[k] = *cam_ptr(cams_[k]);
    e_ = gss_engine_create(n, rows.data(), int32_t(gc.size()), gc.data(), g.empty() ? nullptr : g.data(), &c);
    if (!e_) check(std::string(gss_last_error()).find("device") != std::string::npos ? GSS_ERR_CUDA : GSS_ERR_INVALID);
    if (!splits.cameras.empty()) {
      if (splits.cameras.size() != cams_.size()) throw gss::ConfigError("OffloadEngine: split table size");
      std::vector<int32_t> sp(splits.cameras.size()), col(splits.cameras.size());
      for (size_t k = 0; k < sp.size(); ++k) {
        sp[k] = splits.cameras[k].split ? 1 : 0;
        col[k] = splits.cameras[k].column;
      }
      check(gss_engine_set_splits(e_, int32_t(sp.size()), sp.data(), col.data()));
    }
  }
  ~OffloadEngine() { gss_engine_destroy(e_); }
  OffloadEngine(const OffloadEngine&) = delete;
  OffloadEngine& operator=(const OffloadEngine&) = delete;

  // engine.hpp:73-88: n iterations, drained.
  std::vector<IterResult> run(int n) {
    if (n <= 0) return {};
    std::vector<float> losses(static_cast<size_t>(n));
    std::vector<int32_t> valid(static_cast<size_t>(n));
    check(gss_engine_run(e_, n, losses.data(), valid.data()));
    std::vector<IterResult> out(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) out[i] = {losses[i], valid[i]};
    return out;
  }

  // engine.hpp:91-111: both tiers restored.
  gss::GaussianSet<float> snapshot() const {
    const int n = count();
    std::vector<float> rows(size_t(std::max(n, 1)) * gss::kParamDim);
    check(gss_engine_snapshot(e_, rows.data()));
    gss::GaussianSet<float> gs;
    gs.resize(n);
    gs.sh_degree = sh_degree_;
    for (int i = 0; i < n; ++i) gs.set_full_row(i, rows.data() + size_t(i) * gss::kParamDim);
    return gs;
  }

  int count() const { return int(gss_engine_count(e_)); }

  // engine.hpp:187-188 (densification statistics)
  std::vector<double> accum_grad_norm() const {
    std::vector<double> nrm(size_t(std::max(count(), 1)));
    std::vector<int32_t> cnt(nrm.size());
    check(gss_engine_accum(e_, nrm.data(), cnt.data()));
    nrm.resize(size_t(count()));
    return nrm;
  }
  std::vector<int> accum_grad_count() const {
    std::vector<double> nrm(size_t(std::max(count(), 1)));
    std::vector<int32_t> cnt(nrm.size());
    check(gss_engine_accum(e_, nrm.data(), cnt.data()));
    return std::vector<int>(cnt.begin(), cnt.begin() + count());
  }

  // engine.hpp:22-28: rows since the timeline was enabled (enable_timeline(true) first).
  void enable_timeline(bool on) { check(gss_engine_timeline_enable(e_, on ? 1 : 0)); }
  std::vector<gss::TimelineRow> timeline() const {
    static const char* const kStage[6] = {"cull", "forward_params", "render", "geo_update", "handoff", "lazy_update"};
    const int64_t k = gss_engine_timeline(e_, nullptr, 0);
    if (k < 0) check(int(-k));
    std::vector<gss_timeline_row> r(size_t(std::max<int64_t>(k, 1)));
    const int64_t got = gss_engine_timeline(e_, r.data(), int64_t(r.size()));
    std::vector<gss::TimelineRow> out;
    for (int64_t i = 0; i < got; ++i)
      out.push_back({r[i].iteration, kStage[r[i].stage % 6], r[i].t0_ns, r[i].t1_ns, r[i].bytes, r[i].worker});
    return out;
  }

  gss_engine* handle() const { return e_; }

 private:
  std::vector<gss::Camera<float>> cams_;
  int sh_degree_ = 3;
  gss_engine* e_ = nullptr;
};

}  // namespace gss_b200
