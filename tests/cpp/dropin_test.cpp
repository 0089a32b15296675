// Drop-in parity test of include/gss_b200.hpp: the reference's own C++ functions (gss::,
// compiled from the unmodified headers under /root/reference/proj/include) against the B200
// path (gss_b200::, libgss_b200.so) on identical inputs, through the reference's types.
// TEST INFRASTRUCTURE: built by oracle/Makefile (target `dropin`) into oracle/_ref/dropin_test;
// run on a GPU by tests/test_dropin_gpu.py. Exit code = number of failed checks.
//
//   bit-exact: frustum_cull ids, rasterize_forward image, compute_loss_l1 (loss + d_img),
//              adam_step_dense / deferred_update (+ touched ids) / restore_view / flush_deferred
//   tolerance: rasterize_backward rows + mean2d, rel(a,b) = |a-b|/max(1,|a|,|b|) <= 1e-4
//              (acceptance.cpp:44; the reference's own gradient tolerance)
#include <gss/adam.hpp>
#include <gss/engine.hpp>
#include <gss/render.hpp>
#include <gss/rng.hpp>
#include <gss/synth.hpp>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "gss_b200.hpp"

namespace {

int g_fail = 0;

void expect(bool ok, const char* what) {
  std::printf("%-58s %s\n", what, ok ? "ok" : "FAIL");
  if (!ok) ++g_fail;
}

template <class T> bool same_bits(const std::vector<T>& a, const std::vector<T>& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), a.size() * sizeof(T)) == 0);
}

double rel_max(const std::vector<float>& a, const std::vector<float>& b) {
  if (a.size() != b.size()) return 1e30;
  double m = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double x = a[i], y = b[i];
    m = std::max(m, std::abs(x - y) / std::max({1.0, std::abs(x), std::abs(y)}));
  }
  return m;
}

std::vector<gss::GroupSpec> nongeo_groups() {
  auto hp = [](double lr) { gss::Hyperparams h; h.lr = lr; return h; };
  return {{"opacity", 0, 1, hp(5e-2)}, {"sh_dc", 1, 3, hp(2.5e-3)}, {"sh_rest", 4, 45, hp(2.5e-3 / 20)}};
}

void test_cull() {
  gss::Rng rng(11);
  const int n = 50000;
  std::vector<float> rows(size_t(n) * 10);
  for (int i = 0; i < n; ++i) {
    float* r = rows.data() + size_t(i) * 10;
    for (int c = 0; c < 3; ++c) r[c] = float(rng.uniform(-3, 3));
    for (int c = 3; c < 6; ++c) r[c] = float(rng.uniform(-7, 1));
    double q[4], qn = 0;
    for (double& v : q) { v = rng.normal(); qn += v * v; }
    for (int c = 0; c < 4; ++c) r[6 + c] = float(q[c] / std::sqrt(qn));
  }
  const auto cam = gss::look_at_camera<float>({0.3f, 0.2f, -4.0f}, {0.f, 0.f, 0.f}, 300.f, 300.f, 320, 240, 0.5f, 8.f);
  for (auto vp : {gss::Viewport<float>::full(320, 240), gss::Viewport<float>{-5.5f, 160.25f, 10.f, 200.5f}}) {
    const auto want = gss::frustum_cull<float>({rows.data(), 10}, n, cam, vp);
    const auto got = gss_b200::frustum_cull({rows.data(), 10}, n, cam, vp);
    expect(want == got, "frustum_cull ids bit-exact (50K rows)");
  }
}

void test_adam() {
  gss::Rng rng(5);
  const int n = 3000, dim = 49;
  gss::Arena<float> ref, dev;
  ref.init(n, dim, nongeo_groups(), 15);
  for (auto& x : ref.w) x = float(rng.uniform(-1, 1));
  dev = ref;
  std::vector<float> dense(size_t(n) * dim);
  for (int pass = 0; pass < 40; ++pass) {
    std::vector<int> ids;
    for (int i = 0; i < n; ++i)
      if (rng.uniform() < 0.0828) ids.push_back(i);
    std::vector<float> g(ids.size() * dim);
    for (auto& x : g) x = float(rng.normal());
    const gss::SparseGrads<float> sg{std::span<const int>(ids), g.data(), size_t(dim), 0};
    if (pass == 20) {  // forwarding gather: restore_view with the pending pass, before the update
      std::vector<float> a(ids.size() * dim), b(ids.size() * dim);
      gss::restore_view(ref, std::span<const int>(ids), &sg, a.data());
      gss_b200::restore_view(dev, std::span<const int>(ids), &sg, b.data());
      expect(same_bits(a, b), "restore_view (+ pending pass) bit-exact");
    }
    const auto t_ref = gss::deferred_update(ref, sg);
    const auto t_dev = gss_b200::deferred_update(dev, sg);
    if (t_ref != t_dev) { expect(false, "deferred_update touched ids"); return; }
  }
  expect(same_bits(ref.w, dev.w) && same_bits(ref.m, dev.m) && same_bits(ref.v, dev.v) &&
             same_bits(ref.counter, dev.counter) && ref.step == dev.step,
         "deferred_update x40 (w, m, v, counters, step) bit-exact");
  gss::flush_deferred(ref);
  gss_b200::flush_deferred(dev);
  expect(same_bits(ref.w, dev.w) && same_bits(ref.m, dev.m) && same_bits(ref.v, dev.v) &&
             same_bits(ref.counter, dev.counter),
         "flush_deferred bit-exact");
  for (auto& x : dense) x = float(rng.normal());
  gss::adam_step_dense(ref, dense.data());
  gss_b200::adam_step_dense(dev, dense.data());
  expect(same_bits(ref.w, dev.w) && same_bits(ref.m, dev.m) && same_bits(ref.v, dev.v),
         "adam_step_dense bit-exact");
  const auto& ra = ref.access;
  const auto& da = dev.access;
  expect(ra.update_passes == da.update_passes && ra.touched_rows == da.touched_rows &&
             ra.param_bytes == da.param_bytes && ra.counter_bytes == da.counter_bytes &&
             ra.restore_rows == da.restore_rows && ra.restore_read_bytes == da.restore_read_bytes,
         "AccessReport tally (adam.hpp:36-50) equal to the reference's");
  // InvariantViolation on unsorted ids (adam.hpp:231)
  std::vector<int> bad{5, 3};
  std::vector<float> bg(2 * dim, 0.1f);
  bool threw = false;
  try {
    gss_b200::deferred_update(dev, {std::span<const int>(bad), bg.data(), size_t(dim), 0});
  } catch (const gss::InvariantViolation&) {
    threw = true;
  }
  expect(threw, "unsorted grad ids -> gss::InvariantViolation");
}

void test_raster() {
  gss::SynthConfig cfg;
  cfg.n = 400;
  cfg.cams = 4;
  cfg.width = 64;
  cfg.height = 48;
  cfg.seed = 9;
  const auto scene = gss::synth_scene<float>(cfg);
  const auto rows = gss::scene_rows(scene.truth);
  for (int ci = 0; ci < 2; ++ci) {
    const auto& cam = scene.cameras[ci];
    const auto vp = gss::Viewport<float>::full(cam.width, cam.height);
    const auto ids = gss::frustum_cull<float>(rows.geo_view(), cfg.n, cam, vp);
    gss::RenderScene<float> sc;
    sc.ids = std::span<const int>(ids);
    sc.geo = rows.geo_view();
    sc.nongeo = rows.nongeo_view();
    const auto rr = gss::rasterize_forward(sc, cam, vp);
    gss_b200::Rasterizer dev;
    const auto img = dev.forward(sc, cam, vp);
    expect(img.width == rr.image.width && img.height == rr.image.height && same_bits(img.data, rr.image.data),
           "rasterize_forward image bit-exact");
    gss::Image<float> d_ref, d_dev;
    const float l_ref = gss::compute_loss_l1(rr.image, scene.gt_images[(ci + 1) % cfg.cams], d_ref);
    const float l_dev = gss_b200::compute_loss_l1(img, scene.gt_images[(ci + 1) % cfg.cams], d_dev);
    expect(l_ref == l_dev && same_bits(d_ref.data, d_dev.data), "compute_loss_l1 loss + d_img bit-exact");
    const auto g_ref = gss::rasterize_backward(sc, cam, rr, d_ref);
    const auto g_dev = dev.backward(d_dev);
    const double dr = rel_max(g_ref.rows, g_dev.rows), dm = rel_max(g_ref.mean2d, g_dev.mean2d);
    std::printf("  backward rel dev: rows %.3e, mean2d %.3e\n", dr, dm);
    expect(g_ref.ids == g_dev.ids && dr <= 1e-4 && dm <= 1e-4, "rasterize_backward rows, mean2d within 1e-4");
  }
  {  // the reference-signature free functions: the caller's code is unchanged but for the namespace
    const auto& cam = scene.cameras[2];
    const gss::Viewport<float> vp{7.0f, 50.5f, 3.0f, 40.0f};
    const auto ids = gss::frustum_cull<float>(rows.geo_view(), cfg.n, cam, vp);
    gss::RenderScene<float> sc;
    sc.ids = std::span<const int>(ids);
    sc.geo = rows.geo_view();
    sc.nongeo = rows.nongeo_view();
    const auto rr = gss::rasterize_forward(sc, cam, vp, 2);
    const auto rd = gss_b200::rasterize_forward(sc, cam, vp, 2);
    expect(rd.aux.px0 == rr.aux.px0 && rd.aux.py0 == rr.aux.py0 && same_bits(rd.image.data, rr.image.data),
           "gss_b200::rasterize_forward (sub-viewport) image + window bit-exact");
    gss::Image<float> gt_win(rr.image.width, rr.image.height), d_ref, d_dev;
    for (int y = 0; y < gt_win.height; ++y)
      for (int x = 0; x < gt_win.width; ++x)
        for (int c = 0; c < 3; ++c) gt_win.at(y, x, c) = scene.gt_images[2].at(y + rr.aux.py0, x + rr.aux.px0, c);
    const size_t full = size_t(cam.width) * cam.height * 3;
    const float l_ref = gss::compute_loss_l1(rr.image, gt_win, d_ref, full);
    const float l_dev = gss_b200::compute_loss_l1(rd.image, gt_win, d_dev, full);
    const auto g_ref = gss::rasterize_backward(sc, cam, rr, d_ref, 2);
    const auto g_dev = gss_b200::rasterize_backward(sc, cam, rd, d_dev, 2);
    expect(l_ref == l_dev && g_ref.ids == g_dev.ids && rel_max(g_ref.rows, g_dev.rows) <= 1e-4 &&
               rel_max(g_ref.mean2d, g_dev.mean2d) <= 1e-4,
           "gss_b200::rasterize_backward (RenderResult) within 1e-4");
  }
  bool threw = false;
  gss::Image<float> a(4, 4), b(5, 4), d;
  try {
    gss_b200::compute_loss_l1(a, b, d);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  expect(threw, "shape mismatch -> std::invalid_argument");
}

// gss::OffloadEngine vs gss_b200::OffloadEngine: identical constructor arguments (EngineConfig,
// SplitTable), run() results and snapshot within the per-step tolerance, identical valid counts.
void test_engine() {
  gss::SynthConfig cfg;
  cfg.n = 600;
  cfg.cams = 5;
  cfg.width = 40;
  cfg.height = 32;
  cfg.seed = 21;
  const auto scene = gss::synth_scene<float>(cfg);
  gss::GaussianSet<float> start = scene.truth;
  for (int i = 0; i < start.count; ++i) {
    start.opacity[i] = float(std::log(0.1 / 0.9));
    for (int k = 3; k < gss::kShScalars; ++k) start.sh[i * gss::kShScalars + k] = 0.0f;
  }
  gss::EngineConfig<float> ec;
  ec.pipelined = true;
  ec.workers = 4;
  gss::SplitTable st;
  st.cameras.resize(cfg.cams);
  st.cameras[1].split = true;
  st.cameras[1].column = 17;
  st.cameras[3].split = true;
  st.cameras[3].column = 30;
  gss::OffloadEngine<float> ref(start, scene.cameras, scene.gt_images, ec, st);
  gss_b200::OffloadEngine dev(start, scene.cameras, scene.gt_images, ec, st);
  const auto r1 = ref.run(12);
  const auto r2 = dev.run(12);
  bool same_valid = r1.size() == r2.size();
  double ldev = 0.0;
  for (size_t i = 0; i < r1.size() && same_valid; ++i) {
    same_valid = r1[i].valid_count == r2[i].valid_count;
    ldev = std::max(ldev, std::abs(double(r1[i].loss) - r2[i].loss) / std::max(1.0, std::abs(double(r1[i].loss))));
  }
  std::printf("  engine loss dev %.3e\n", ldev);
  expect(same_valid && r1[0].loss == r2[0].loss && ldev <= 1e-4,
         "gss_b200::OffloadEngine (split table) run(): valid counts, first loss bit-exact, losses within 1e-4");
  const auto s1 = ref.snapshot(), s2 = dev.snapshot();
  const double sdev = std::max(rel_max(s1.mean, s2.mean), rel_max(s1.sh, s2.sh));
  expect(s1.count == s2.count && sdev <= 1e-4, "gss_b200::OffloadEngine snapshot within 1e-4");
  expect(ref.accum_grad_count() == dev.accum_grad_count(), "accum_grad_count identical");
  dev.enable_timeline(true);
  dev.run(2);
  expect(dev.timeline().size() == 12, "timeline: 6 stages x 2 iterations");
}

}  // namespace

int main() {
  if (gss_device_count() <= 0) {
    std::printf("no CUDA device\n");
    return 77;
  }
  test_cull();
  test_adam();
  test_raster();
  test_engine();
  std::printf("%d failed\n", g_fail);
  return g_fail;
}
