// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference headers (/root/reference/proj/include/gss/*.hpp),
// compiled by oracle/Makefile into oracle/_ref/libgss_ref.so. The shim owns no algorithm:
// every function forwards to the reference template instantiated for float, so the
// library *is* the reference path (render.hpp, adam.hpp, engine.hpp, trainer.hpp) and is
// used (a) to pin the C restatement in oracle/gss_oracle.c, (b) as the parity checker in
// tests/, and (c) as the `--impl reference` CPU arm of bench.py.
//
// Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs load it.

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <vector>

#include "gss/adam.hpp"
#include "gss/bench.hpp"
#include "gss/engine.hpp"
#include "gss/ply.hpp"
#include "gss/render.hpp"
#include "gss/splitter.hpp"
#include "gss/synth.hpp"
#include "gss/trainer.hpp"

using namespace gss;
using F = float;

static_assert(sizeof(Camera<F>) == 80, "Camera<float> must be the 80-byte gss_camera layout");

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {
const Camera<F>& cam_of(const void* p) { return *reinterpret_cast<const Camera<F>*>(p); }
Viewport<F> vp_of(const float* v) { return Viewport<F>{v[0], v[1], v[2], v[3]}; }

int status_of_current() {
  try {
    throw;
  } catch (const ConfigError&) {
    return 2;
  } catch (const std::invalid_argument&) {
    return 2;
  } catch (const InvariantViolation&) {
    return 3;
  } catch (...) {
    return 1;
  }
}
}  // namespace

// ---------------------------------------------------------------------------
// libm + projection + cull (render.hpp:90-148, 243-260)

REF_API float ref_expf(float x) { return std::exp(x); }

REF_API int ref_frustum_cull(const float* geo, int n, int stride, const void* cam, const float* vp, float low_pass,
                             int* out_ids) {
  const auto ids = frustum_cull<F>(RowView<F>{geo, size_t(stride)}, n, cam_of(cam), vp_of(vp), low_pass);
  if (out_ids) std::memcpy(out_ids, ids.data(), ids.size() * sizeof(int));
  return int(ids.size());
}

// out[8] = mean2d.x, mean2d.y, cov_a, cov_b, cov_c, depth, radius, valid
REF_API void ref_project_geo(const float* g, const void* cam, float low_pass, float* out) {
  const auto p = project_geo<F>(g, cam_of(cam), low_pass);
  out[0] = p.mean2d.x;
  out[1] = p.mean2d.y;
  out[2] = p.cov_a;
  out[3] = p.cov_b;
  out[4] = p.cov_c;
  out[5] = p.depth;
  out[6] = p.radius;
  out[7] = p.valid ? 1.0f : 0.0f;
}

// ---------------------------------------------------------------------------
// Rasterizer forward + L1 loss + backward (render.hpp:384-640)
//
// nongeo_compact != 0: nongeo rows are slot-indexed (forwarded slice, V x 49);
// otherwise id-indexed (dense N x 49).  d_img_in (optional) overrides the loss
// gradient (used by the gradient-parity tests).  meta[0..4] = px0, py0, pw, ph,
// total contributions (CSR length).  Returns a status code.
REF_API int ref_render(int n_ids, const int* ids, const float* geo, int geo_stride, const float* nongeo,
                       int nongeo_compact, int sh_degree, const float* bg, const void* cam, const float* vp,
                       const float* gt_full, int64_t normalizer, const float* d_img_in, int workers,
                       float* out_image, float* out_final_T, int* out_len, float* out_loss, float* out_d_img,
                       float* out_grad_rows, float* out_mean2d, float* out_proj /* n x 10 or null */,
                       int64_t* meta) {
  try {
    const Camera<F>& c = cam_of(cam);
    RenderScene<F> sc;
    sc.ids = std::span<const int>(ids, size_t(n_ids));
    sc.geo = RowView<F>{geo, size_t(geo_stride)};
    sc.nongeo = NonGeoView<F>{nongeo, size_t(kNonGeoDim), nongeo_compact != 0, nullptr};
    sc.sh_degree = sh_degree;
    sc.background = Vec3<F>{bg[0], bg[1], bg[2]};
    const RenderResult<F> rr = rasterize_forward(sc, c, vp_of(vp), workers);
    const int pw = rr.aux.pw, ph = rr.aux.ph;
    if (meta) {
      meta[0] = rr.aux.px0;
      meta[1] = rr.aux.py0;
      meta[2] = pw;
      meta[3] = ph;
      meta[4] = int64_t(rr.aux.contribs.size());
    }
    if (out_image) std::memcpy(out_image, rr.image.data.data(), rr.image.data.size() * sizeof(F));
    if (out_final_T) std::memcpy(out_final_T, rr.aux.final_trans.data(), rr.aux.final_trans.size() * sizeof(F));
    if (out_len) std::memcpy(out_len, rr.aux.len.data(), rr.aux.len.size() * sizeof(int));
    if (out_proj) {
      for (int k = 0; k < n_ids && k < int(rr.proj.size()); ++k) {
        const auto& p = rr.proj[k];
        float* o = out_proj + size_t(k) * 10;
        o[0] = p.mean2d.x; o[1] = p.mean2d.y; o[2] = p.cov_a; o[3] = p.cov_b; o[4] = p.cov_c;
        o[5] = p.depth; o[6] = p.radius; o[7] = p.rgb.x; o[8] = p.rgb.y; o[9] = p.rgb.z;
      }
    }
    Image<F> dimg;
    if (gt_full) {
      Image<F> gt_win(pw, ph);
      for (int y = 0; y < ph; ++y)
        for (int x = 0; x < pw; ++x)
          for (int ch = 0; ch < 3; ++ch)
            gt_win.at(y, x, ch) = gt_full[(size_t(y + rr.aux.py0) * c.width + (x + rr.aux.px0)) * 3 + ch];
      const F loss = compute_loss_l1(rr.image, gt_win, dimg, size_t(normalizer));
      if (out_loss) *out_loss = loss;
    }
    if (d_img_in) {
      dimg = Image<F>(pw, ph);
      std::memcpy(dimg.data.data(), d_img_in, dimg.data.size() * sizeof(F));
    }
    if (out_d_img && !dimg.data.empty()) std::memcpy(out_d_img, dimg.data.data(), dimg.data.size() * sizeof(F));
    if (out_grad_rows || out_mean2d) {
      if (dimg.data.empty()) dimg = Image<F>(pw, ph);
      const GradBuffer<F> gb = rasterize_backward(sc, c, rr, dimg, workers);
      if (out_grad_rows) std::memcpy(out_grad_rows, gb.rows.data(), gb.rows.size() * sizeof(F));
      if (out_mean2d) std::memcpy(out_mean2d, gb.mean2d.data(), gb.mean2d.size() * sizeof(F));
    }
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

REF_API int ref_loss_l1(const float* img, const float* gt, int w, int h, int64_t normalizer, float* d_img,
                        float* loss) {
  try {
    Image<F> a(w, h), b(w, h), d;
    std::memcpy(a.data.data(), img, a.data.size() * sizeof(F));
    std::memcpy(b.data.data(), gt, b.data.size() * sizeof(F));
    *loss = compute_loss_l1(a, b, d, size_t(normalizer));
    std::memcpy(d_img, d.data.data(), d.data.size() * sizeof(F));
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

// ---------------------------------------------------------------------------
// Optimizer (adam.hpp:67-313)

REF_API void ref_build_luts(double lr, double b1, double b2, double eps, int64_t t, int max_delay, float* param,
                            float* mom, float* var, float* pow_b1, float* pow_b2, float* scalars /*5*/) {
  const auto l = build_group_luts<F>(Hyperparams{lr, b1, b2, eps}, t, max_delay);
  std::memcpy(param, l.param.data(), l.param.size() * sizeof(F));
  std::memcpy(mom, l.mom.data(), l.mom.size() * sizeof(F));
  std::memcpy(var, l.var.data(), l.var.size() * sizeof(F));
  std::memcpy(pow_b1, l.pow_b1.data(), l.pow_b1.size() * sizeof(F));
  std::memcpy(pow_b2, l.pow_b2.data(), l.pow_b2.size() * sizeof(F));
  scalars[0] = l.one_minus_b1;
  scalars[1] = l.one_minus_b2;
  scalars[2] = l.bias_correction;
  scalars[3] = l.step_size;
  scalars[4] = l.eps;
}

REF_API void* ref_arena_new(int n, int dim, int ngroups, const int* col0, const int* gdim, const double* lr,
                            double b1, double b2, double eps, int defer_max, int* status) {
  try {
    auto* a = new Arena<F>();
    std::vector<GroupSpec> gs;
    for (int g = 0; g < ngroups; ++g) gs.push_back({"g" + std::to_string(g), col0[g], gdim[g], Hyperparams{lr[g], b1, b2, eps}});
    a->init(n, dim, gs, defer_max);
    *status = 0;
    return a;
  } catch (...) {
    *status = status_of_current();
    return nullptr;
  }
}
REF_API void ref_arena_free(void* h) { delete static_cast<Arena<F>*>(h); }
REF_API void ref_arena_ptrs(void* h, float** w, float** m, float** v, uint8_t** counter, int64_t** step) {
  auto* a = static_cast<Arena<F>*>(h);
  *w = a->w.data();
  *m = a->m.data();
  *v = a->v.data();
  *counter = a->counter.data();
  *step = &a->step;
}
REF_API void ref_arena_access(void* h, uint64_t* out6) {
  const auto& r = static_cast<Arena<F>*>(h)->access;
  out6[0] = r.update_passes; out6[1] = r.touched_rows; out6[2] = r.param_bytes;
  out6[3] = r.counter_bytes; out6[4] = r.restore_rows; out6[5] = r.restore_read_bytes;
}
REF_API int ref_adam_step_dense(void* h, const float* grads) {
  try {
    adam_step_dense(*static_cast<Arena<F>*>(h), grads);
    return 0;
  } catch (...) {
    return status_of_current();
  }
}
// Returns the touched count (>= 0) or -status.
REF_API int64_t ref_deferred_update(void* h, int nids, const int* ids, const float* rows, int stride, int col0,
                                    int* touched_out) {
  try {
    const SparseGrads<F> g{std::span<const int>(ids, size_t(nids)), rows, size_t(stride), col0};
    const auto t = deferred_update(*static_cast<Arena<F>*>(h), g);
    if (touched_out) std::memcpy(touched_out, t.data(), t.size() * sizeof(int));
    return int64_t(t.size());
  } catch (...) {
    return -status_of_current();
  }
}
REF_API int ref_restore_view(void* h, int nids, const int* ids, int has_pending, int npend, const int* pids,
                             const float* prows, int pstride, int pcol0, float* out) {
  try {
    const SparseGrads<F> p{std::span<const int>(pids, size_t(npend)), prows, size_t(pstride), pcol0};
    restore_view<F>(*static_cast<Arena<F>*>(h), std::span<const int>(ids, size_t(nids)), has_pending ? &p : nullptr,
                    out);
    return 0;
  } catch (...) {
    return status_of_current();
  }
}
REF_API void ref_flush_deferred(void* h) { flush_deferred(*static_cast<Arena<F>*>(h)); }
REF_API int ref_check_counters(void* h) {
  try {
    static_cast<Arena<F>*>(h)->check_counters();
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

// optim_bench (bench.hpp:41-114): out[0] = max_rel_dev, out[1] = bitwise, out[2] = touched_total,
// out[3] = deferred param bytes, out[4] = dense param bytes
REF_API void ref_optim_bench(int n, int dim, int steps, double density, int defer_max, uint64_t seed, double* out) {
  OptimBenchConfig c;
  c.n = n; c.dim = dim; c.steps = steps; c.density = density; c.defer_max = defer_max; c.seed = seed;
  const auto r = optim_bench<F>(c);
  out[0] = r.max_rel_dev;
  out[1] = r.bitwise_equal ? 1.0 : 0.0;
  out[2] = double(r.touched_total);
  out[3] = double(r.deferred_access.param_bytes);
  out[4] = double(r.dense_param_bytes);
}

// ---------------------------------------------------------------------------
// Scenes (synth.hpp:100-159). cfg_d[] = box, radius_min, radius_max, fov_deg, fov_ramp, target_jitter,
// near, far, scale_min, scale_max, scale_aniso, opacity_min, opacity_max, sh_rest_noise.
// rows_out: n x 59 truth rows; cams_out: cams x 20 floats (gss_camera); gts_out: cams x H x W x 3 or null
// (null skips nothing — synth_scene always renders; pass a buffer to keep them).
REF_API void ref_synth_scene(uint64_t seed, int n, int cams, int width, int height, int sh_degree, const double* cfg_d,
                             float* rows_out, void* cams_out, float* gts_out) {
  SynthConfig c;
  c.seed = seed; c.n = n; c.cams = cams; c.width = width; c.height = height; c.sh_degree = sh_degree;
  c.box = cfg_d[0]; c.radius_min = cfg_d[1]; c.radius_max = cfg_d[2]; c.fov_deg = cfg_d[3]; c.fov_ramp = cfg_d[4];
  c.target_jitter = cfg_d[5]; c.near_plane = cfg_d[6]; c.far_plane = cfg_d[7]; c.scale_min = cfg_d[8];
  c.scale_max = cfg_d[9]; c.scale_aniso = cfg_d[10]; c.opacity_min = cfg_d[11]; c.opacity_max = cfg_d[12];
  c.sh_rest_noise = cfg_d[13];
  const auto s = synth_scene<F>(c);
  for (int i = 0; i < n; ++i) s.truth.full_row(i, rows_out + size_t(i) * kParamDim);
  std::memcpy(cams_out, s.cameras.data(), s.cameras.size() * sizeof(Camera<F>));
  if (gts_out)
    for (int k = 0; k < cams; ++k)
      std::memcpy(gts_out + size_t(k) * width * height * 3, s.gt_images[k].data.data(),
                  s.gt_images[k].data.size() * sizeof(F));
}

namespace {
GaussianSet<F> set_from_rows(int n, const float* rows);
}  // namespace

// synth_scene (synth.hpp:100-154) without its ground-truth render (synth.hpp:156-158), for workloads
// whose CPU render of all views would take minutes (the reference arm renders only the views it
// times). Same Rng stream and operation order as synth_scene, built from the reference's own
// primitives (Rng, logit, look_at_camera); pinned equal to ref_synth_scene by tests/test_oracle.py.
REF_API void ref_synth_scene_nogt(uint64_t seed, int n, int cams, int width, int height, int sh_degree,
                                  const double* cfg_d, float* rows_out, void* cams_out) {
  SynthConfig cfg;
  cfg.seed = seed; cfg.n = n; cfg.cams = cams; cfg.width = width; cfg.height = height; cfg.sh_degree = sh_degree;
  cfg.box = cfg_d[0]; cfg.radius_min = cfg_d[1]; cfg.radius_max = cfg_d[2]; cfg.fov_deg = cfg_d[3];
  cfg.fov_ramp = cfg_d[4]; cfg.target_jitter = cfg_d[5]; cfg.near_plane = cfg_d[6]; cfg.far_plane = cfg_d[7];
  cfg.scale_min = cfg_d[8]; cfg.scale_max = cfg_d[9]; cfg.scale_aniso = cfg_d[10]; cfg.opacity_min = cfg_d[11];
  cfg.opacity_max = cfg_d[12]; cfg.sh_rest_noise = cfg_d[13];
  Rng rng(cfg.seed * 0x9E3779B97F4A7C15ull + 0xD1B54A32D192ED03ull);
  GaussianSet<F> gs;
  gs.resize(cfg.n);
  gs.sh_degree = cfg.sh_degree;
  for (int i = 0; i < cfg.n; ++i) {
    for (int a = 0; a < 3; ++a) gs.mean[i * 3 + a] = F(rng.uniform(-cfg.box, cfg.box));
    const double log_lo = std::log(cfg.scale_min * cfg.box), log_hi = std::log(cfg.scale_max * cfg.box);
    const double base = rng.uniform(log_lo, log_hi);
    for (int a = 0; a < 3; ++a) gs.scale[i * 3 + a] = F(base + rng.uniform(-cfg.scale_aniso, cfg.scale_aniso));
    double q[4];
    double qn = 0;
    for (auto& c : q) {
      c = rng.normal();
      qn += c * c;
    }
    qn = std::sqrt(qn);
    if (qn < 1e-9) { q[0] = 1; q[1] = q[2] = q[3] = 0; qn = 1; }
    for (int a = 0; a < 4; ++a) gs.quaternion[i * 4 + a] = F(q[a] / qn);
    gs.opacity[i] = F(logit(rng.uniform(cfg.opacity_min, cfg.opacity_max)));
    for (int c = 0; c < 3; ++c) gs.sh[i * kShScalars + c] = F((rng.uniform(0.08, 0.92) - 0.5) / kShC0);
    const int active = (cfg.sh_degree + 1) * (cfg.sh_degree + 1);
    for (int k = 1; k < active; ++k)
      for (int c = 0; c < 3; ++c) gs.sh[i * kShScalars + k * 3 + c] = F(rng.normal() * cfg.sh_rest_noise);
  }
  std::vector<Camera<F>> out;
  const double golden = 2.399963229728653;
  for (int i = 0; i < cfg.cams; ++i) {
    const double t = cfg.cams > 1 ? double(i) / (cfg.cams - 1) : 1.0;
    const double radius = cfg.box * (cfg.radius_min * std::pow(cfg.radius_max / cfg.radius_min, t));
    const double fov = cfg.fov_deg * (cfg.fov_ramp + (1.0 - cfg.fov_ramp) * t);
    const double fx = 0.5 * cfg.width / std::tan(0.5 * fov * M_PI / 180.0);
    const double fy = fx;
    const double az = golden * i + rng.uniform(-0.15, 0.15);
    const double el = (0.15 + 0.55 * rng.uniform()) * (i % 2 == 0 ? 1.0 : -1.0);
    Vec3<F> eye{F(radius * std::cos(el) * std::cos(az)), F(radius * std::sin(el)),
                F(radius * std::cos(el) * std::sin(az))};
    const double jig = cfg.target_jitter * (1.0 - t);
    Vec3<F> target{F(rng.uniform(-jig, jig) * cfg.box), F(rng.uniform(-jig, jig) * cfg.box),
                   F(rng.uniform(-jig, jig) * cfg.box)};
    out.push_back(look_at_camera<F>(eye, target, F(fx), F(fy), cfg.width, cfg.height, F(cfg.near_plane),
                                    F(cfg.far_plane)));
  }
  for (int i = cfg.cams - 1; i > 0; --i) {
    const int j = int(rng.next_u64() % uint64_t(i + 1));
    std::swap(out[i], out[j]);
  }
  for (int i = 0; i < n; ++i) gs.full_row(i, rows_out + size_t(i) * kParamDim);
  std::memcpy(cams_out, out.data(), out.size() * sizeof(Camera<F>));
}

// render_view (synth.hpp:81-94) of rows (n x 59) with `workers` threads: the reference's ground truth
// for one view.
REF_API void ref_render_view_rows(int n, const float* rows, const void* cam, int sh_degree, int workers,
                                  float* img_out) {
  const GaussianSet<F> gs = set_from_rows(n, rows);
  const Image<F> im = render_view(gs, cam_of(cam), sh_degree, workers);
  std::memcpy(img_out, im.data.data(), im.data.size() * sizeof(F));
}

REF_API void ref_look_at_camera(const float* eye, const float* target, float fx, float fy, int w, int h, float near_p,
                                float far_p, void* out) {
  const auto c = look_at_camera<F>(Vec3<F>{eye[0], eye[1], eye[2]}, Vec3<F>{target[0], target[1], target[2]}, fx, fy, w,
                                   h, near_p, far_p);
  std::memcpy(out, &c, sizeof(c));
}

// ---------------------------------------------------------------------------
// Offload engine + dense oracle trainer (engine.hpp:55-522, trainer.hpp:218-387)

namespace {
struct RefEngine {
  std::unique_ptr<OffloadEngine<F>> eng;
  std::unique_ptr<DenseTrainer<F>> dense;
};

GaussianSet<F> set_from_rows(int n, const float* rows) {
  GaussianSet<F> gs;
  gs.resize(n);
  gs.sh_degree = 3;
  for (int i = 0; i < n; ++i) gs.set_full_row(i, rows + size_t(i) * kParamDim);
  return gs;
}
}  // namespace

// optim_d[] = lr_mean, lr_scale, lr_quat, lr_opacity, lr_sh, sh_rest_divisor, beta1, beta2, eps, scene_extent
// flags: bit0 pipelined, bit1 dense-oracle trainer
// split / cols (optional, ncams entries): the SplitTable given to the OffloadEngine constructor
// (engine.hpp:62-68; splitter.hpp:12-23).
REF_API void* ref_engine_new_split(int n, const float* rows, int ncams, const void* cams, const float* gts,
                                   int defer_max, int geo_defer_max, int flags, int workers, int sh_degree,
                                   const float* bg, const double* optim_d, const int* split, const int* cols) {
  auto* e = new RefEngine();
  const GaussianSet<F> gs = set_from_rows(n, rows);
  std::vector<Camera<F>> cv(static_cast<const Camera<F>*>(cams), static_cast<const Camera<F>*>(cams) + ncams);
  std::vector<Image<F>> gv;
  for (int k = 0; k < ncams; ++k) {
    Image<F> im(cv[k].width, cv[k].height);
    std::memcpy(im.data.data(), gts + size_t(k) * cv[k].width * cv[k].height * 3, im.data.size() * sizeof(F));
    gv.push_back(std::move(im));
  }
  OptimConfig oc;
  oc.lr_mean = optim_d[0]; oc.lr_scale = optim_d[1]; oc.lr_quat = optim_d[2]; oc.lr_opacity = optim_d[3];
  oc.lr_sh = optim_d[4]; oc.sh_rest_divisor = optim_d[5]; oc.beta1 = optim_d[6]; oc.beta2 = optim_d[7];
  oc.eps = optim_d[8]; oc.scene_extent = optim_d[9];
  oc.defer_max = defer_max;
  oc.geo_defer_max = geo_defer_max;
  const Vec3<F> bgv{bg[0], bg[1], bg[2]};
  if (flags & 2) {
    e->dense = std::make_unique<DenseTrainer<F>>(gs, cv, gv, oc, sh_degree, bgv, workers);
  } else {
    EngineConfig<F> ec;
    ec.optim = oc;
    ec.workers = workers;
    ec.pipelined = (flags & 1) != 0;
    ec.sh_degree = sh_degree;
    ec.background = bgv;
    SplitTable st;
    if (split) {
      st.cameras.resize(ncams);
      for (int k = 0; k < ncams; ++k) {
        st.cameras[k].split = split[k] != 0;
        st.cameras[k].column = cols[k];
      }
    }
    e->eng = std::make_unique<OffloadEngine<F>>(gs, cv, gv, ec, st);
  }
  return e;
}
REF_API void* ref_engine_new(int n, const float* rows, int ncams, const void* cams, const float* gts, int defer_max,
                             int geo_defer_max, int flags, int workers, int sh_degree, const float* bg,
                             const double* optim_d) {
  return ref_engine_new_split(n, rows, ncams, cams, gts, defer_max, geo_defer_max, flags, workers, sh_degree, bg,
                              optim_d, nullptr, nullptr);
}
REF_API void ref_engine_free(void* h) { delete static_cast<RefEngine*>(h); }
REF_API int ref_engine_run(void* h, int iters, float* losses, int* valid_counts) {
  try {
    auto* e = static_cast<RefEngine*>(h);
    if (e->dense) {
      const auto r = e->dense->run(iters);
      for (int i = 0; i < iters; ++i) { losses[i] = r[i].loss; valid_counts[i] = r[i].valid_count; }
    } else {
      const auto r = e->eng->run(iters);
      for (int i = 0; i < iters; ++i) { losses[i] = r[i].loss; valid_counts[i] = r[i].valid_count; }
    }
    return 0;
  } catch (...) {
    return status_of_current();
  }
}
REF_API void ref_engine_snapshot(void* h, float* rows) {
  auto* e = static_cast<RefEngine*>(h);
  const GaussianSet<F> gs = e->dense ? e->dense->snapshot() : e->eng->snapshot();
  for (int i = 0; i < gs.count; ++i) gs.full_row(i, rows + size_t(i) * kParamDim);
}
// Raw tier state of the offload engine (stored, not restored): geo w (n x 10), nongeo w (n x 49), counters.
REF_API void ref_engine_state(void* h, float* geo_w, float* ng_w, float* ng_m, float* ng_v, uint8_t* ng_counter,
                              int64_t* steps2) {
  auto* e = static_cast<RefEngine*>(h);
  const auto& st = e->eng->store();
  if (geo_w) std::memcpy(geo_w, st.device_geo.w.data(), st.device_geo.w.size() * sizeof(F));
  if (ng_w) std::memcpy(ng_w, st.host_nongeo.w.data(), st.host_nongeo.w.size() * sizeof(F));
  if (ng_m) std::memcpy(ng_m, st.host_nongeo.m.data(), st.host_nongeo.m.size() * sizeof(F));
  if (ng_v) std::memcpy(ng_v, st.host_nongeo.v.data(), st.host_nongeo.v.size() * sizeof(F));
  if (ng_counter) std::memcpy(ng_counter, st.host_nongeo.counter.data(), st.host_nongeo.counter.size());
  if (steps2) { steps2[0] = st.device_geo.step; steps2[1] = st.host_nongeo.step; }
}
// Densification statistics (engine.hpp:187-188).
REF_API void ref_engine_accum(void* h, double* norm, int* cnt) {
  auto* e = static_cast<RefEngine*>(h);
  const auto& a = e->dense ? e->dense->accum_grad_norm() : e->eng->accum_grad_norm();
  const auto& c = e->dense ? e->dense->accum_grad_count() : e->eng->accum_grad_count();
  std::memcpy(norm, a.data(), a.size() * sizeof(double));
  std::memcpy(cnt, c.data(), c.size() * sizeof(int));
}
// Per-stage timeline totals in ns: cull, forward_params, render, geo_update, handoff, lazy_update.
REF_API void ref_engine_stage_ns(void* h, int64_t* out6) {
  auto* e = static_cast<RefEngine*>(h);
  const char* names[6] = {"cull", "forward_params", "render", "geo_update", "handoff", "lazy_update"};
  for (int k = 0; k < 6; ++k) out6[k] = 0;
  if (!e->eng) return;
  for (const auto& r : e->eng->timeline())
    for (int k = 0; k < 6; ++k)
      if (std::strcmp(r.stage, names[k]) == 0) out6[k] += r.t1_ns - r.t0_ns;
}

// Densification (trainer.hpp:166-213; engine.hpp:116-163). dcfg = grad_threshold, percent_dense,
// opacity_prune, split_scale_divisor. counts5 = survivors, children, clones, splits, pruned.
namespace {
DensifyConfig densify_cfg(const double* d) {
  DensifyConfig dc;
  dc.grad_threshold = d[0];
  dc.percent_dense = d[1];
  dc.opacity_prune = d[2];
  dc.split_scale_divisor = d[3];
  return dc;
}
}  // namespace
REF_API void ref_plan_densify(int n, const float* rows, const double* norm, const int* cnt, const double* dcfg,
                              double extent, uint64_t seed, int* survivors, float* children, int64_t* counts5) {
  const GaussianSet<F> gs = set_from_rows(n, rows);
  const std::vector<double> nv(norm, norm + n);
  const std::vector<int> cv(cnt, cnt + n);
  const DensifyPlan<F> plan = plan_densify<F>(gs, nv, cv, densify_cfg(dcfg), extent, seed);
  std::memcpy(survivors, plan.survivors.data(), plan.survivors.size() * sizeof(int));
  std::memcpy(children, plan.child_rows.data(), plan.child_rows.size() * sizeof(F));
  counts5[0] = (int64_t)plan.survivors.size();
  counts5[1] = (int64_t)(plan.child_rows.size() / kParamDim);
  counts5[2] = plan.clones;
  counts5[3] = plan.splits;
  counts5[4] = plan.pruned;
}
REF_API int ref_engine_densify(void* h, const double* dcfg, double extent, uint64_t seed, int64_t* counts5) {
  try {
    auto* e = static_cast<RefEngine*>(h);
    const GaussianSet<F> snap = e->eng->snapshot();
    const DensifyPlan<F> plan =
        plan_densify<F>(snap, e->eng->accum_grad_norm(), e->eng->accum_grad_count(), densify_cfg(dcfg), extent, seed);
    e->eng->apply_densify(plan.survivors, plan.child_rows);
    counts5[0] = (int64_t)plan.survivors.size();
    counts5[1] = (int64_t)(plan.child_rows.size() / kParamDim);
    counts5[2] = plan.clones;
    counts5[3] = plan.splits;
    counts5[4] = plan.pruned;
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

// compute_split_points (splitter.hpp:31-81) on n x 10 geo rows. out (per camera): split flag,
// column, left count, right count, search evals; ratio: used ratio.
REF_API void ref_compute_split_points(const float* geo, int n, int ncams, const void* cams, double mem_limit,
                                      int* out5, double* ratio) {
  std::vector<Camera<F>> cv(static_cast<const Camera<F>*>(cams), static_cast<const Camera<F>*>(cams) + ncams);
  const SplitTable t = compute_split_points<F>(RowView<F>{geo, kGeoDim}, n, cv, mem_limit);
  for (int i = 0; i < ncams; ++i) {
    const SplitEntry& e = t.cameras[i];
    out5[i * 5 + 0] = e.split ? 1 : 0;
    out5[i * 5 + 1] = e.column;
    out5[i * 5 + 2] = e.left_count;
    out5[i * 5 + 3] = e.right_count;
    out5[i * 5 + 4] = e.search_evals;
    ratio[i] = e.used_ratio;
  }
}

// psnr_over_views (trainer.hpp:131-145) of n x 59 rows over the given cameras / ground truths.
REF_API double ref_psnr_over_views(int n, const float* rows, int ncams, const void* cams, const float* gts,
                                   int sh_degree, int* exact) {
  const GaussianSet<F> gs = set_from_rows(n, rows);
  std::vector<Camera<F>> cv(static_cast<const Camera<F>*>(cams), static_cast<const Camera<F>*>(cams) + ncams);
  std::vector<Image<F>> gv;
  size_t off = 0;
  for (int k = 0; k < ncams; ++k) {
    Image<F> im(cv[k].width, cv[k].height);
    std::memcpy(im.data.data(), gts + off, im.data.size() * sizeof(F));
    off += im.data.size();
    gv.push_back(std::move(im));
  }
  const PsnrResult r = psnr_over_views<F>(gs, cv, gv, sh_degree, Vec3<F>{0, 0, 0}, 1);
  *exact = r.exact ? 1 : 0;
  return r.db;
}

// init_gaussians (scene.hpp:146-195) of a point cloud; rows_out m x 59.
REF_API int ref_init_gaussians(const float* positions, const float* colors, int m, int knn, double min_knn_dist,
                               double init_opacity, float* rows_out) {
  try {
    PointCloud pc;
    pc.positions.assign(positions, positions + size_t(m) * 3);
    if (colors) pc.colors.assign(colors, colors + size_t(m) * 3);
    InitConfig ic;
    ic.knn = knn;
    ic.min_knn_dist = min_knn_dist;
    ic.init_opacity = init_opacity;
    const GaussianSet<F> gs = init_gaussians<F>(pc, ic);
    for (int i = 0; i < m; ++i) gs.full_row(i, rows_out + size_t(i) * kParamDim);
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

// ---------------------------------------------------------------------------
// PLY ingestion (ply.cpp:53-225). ref_load_ply: *m / *has_color receive the cloud's size; the
// arrays are filled when cap >= *m. Returns 0, or 4 for ParseError (message in err).
REF_API int ref_load_ply(const char* path, int64_t cap, float* pos, float* col, int64_t* m, int* has_color, char* err,
                         int errlen) {
  try {
    const PointCloud pc = load_ply(path);
    *m = pc.size();
    *has_color = pc.colors.empty() ? 0 : 1;
    if (cap >= *m) {
      std::memcpy(pos, pc.positions.data(), pc.positions.size() * sizeof(float));
      if (col && !pc.colors.empty()) std::memcpy(col, pc.colors.data(), pc.colors.size() * sizeof(float));
    }
    return 0;
  } catch (const ParseError& e) {
    if (err && errlen > 0) std::snprintf(err, size_t(errlen), "%s", e.what());
    return 4;
  } catch (...) {
    return status_of_current();
  }
}
REF_API int ref_save_ply(const char* path, const float* pos, const float* col, int m, int binary) {
  try {
    PointCloud pc;
    pc.positions.assign(pos, pos + size_t(m) * 3);
    if (col) pc.colors.assign(col, col + size_t(m) * 3);
    save_ply(path, pc, binary != 0);
    return 0;
  } catch (...) {
    return status_of_current();
  }
}
