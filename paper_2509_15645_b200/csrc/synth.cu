// Seeded synthetic scenes (host code): restatement of synth_scene's parameter and camera
// generation (synth.hpp:100-154, rng.hpp:11-51, scene.hpp:99-126) so inputs of any size can be
// produced on the GPU box without the reference; the ground-truth images are then rendered by the
// B200 rasterizer (the CPU reference cannot render 1080p at 4M Gaussians in reasonable time).
// Bit-identical to the reference generator (tests/test_synth.py) — it only feeds the hot path.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <utility>
#include <vector>

#include "common.cuh"

namespace gssd {
namespace {

class Rng {  // rng.hpp:11-51 (splitmix64 + Box-Muller with a cached spare)
 public:
  explicit Rng(uint64_t seed) : state_(seed) {}
  uint64_t next_u64() {
    uint64_t z = (state_ += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return double(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    double u1 = uniform();
    double u2 = uniform();
    if (u1 < 1e-300) u1 = 1e-300;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586477 * u2;
    spare_ = r * std::sin(a);
    have_spare_ = true;
    return r * std::cos(a);
  }

 private:
  uint64_t state_;
  bool have_spare_ = false;
  double spare_ = 0.0;
};

struct V3 {
  float x, y, z;
};
inline float norm3(V3 v) { return std::sqrt(v.x * v.x + v.y * v.y + v.z * v.z); }
inline V3 scale3(V3 v, float s) { return {v.x * s, v.y * s, v.z * s}; }
inline V3 cross3(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }

}  // namespace

// look_at_camera (scene.hpp:99-126), float.
gss_camera look_at(const float* eye_p, const float* target_p, float fx, float fy, int w, int h, float near_p,
                   float far_p) {
  const V3 eye{eye_p[0], eye_p[1], eye_p[2]}, target{target_p[0], target_p[1], target_p[2]};
  V3 up{0.0f, 1.0f, 0.0f};
  V3 fwd{target.x - eye.x, target.y - eye.y, target.z - eye.z};
  const float fn = norm3(fwd);
  fwd = scale3(fwd, 1.0f / fn);
  V3 right = cross3(fwd, up);
  const float rn = norm3(right);
  if (rn < 1e-8f) {
    up = {1.0f, 0.0f, 0.0f};
    right = cross3(fwd, up);
  }
  right = scale3(right, 1.0f / norm3(right));
  const V3 down = cross3(fwd, right);
  gss_camera c{};
  c.rot[0] = right.x; c.rot[1] = right.y; c.rot[2] = right.z;
  c.rot[3] = down.x; c.rot[4] = down.y; c.rot[5] = down.z;
  c.rot[6] = fwd.x; c.rot[7] = fwd.y; c.rot[8] = fwd.z;
  const float rex = c.rot[0] * eye.x + c.rot[1] * eye.y + c.rot[2] * eye.z;
  const float rey = c.rot[3] * eye.x + c.rot[4] * eye.y + c.rot[5] * eye.z;
  const float rez = c.rot[6] * eye.x + c.rot[7] * eye.y + c.rot[8] * eye.z;
  c.trans[0] = -rex; c.trans[1] = -rey; c.trans[2] = -rez;
  c.fx = fx; c.fy = fy;
  c.cx = float(w) / 2.0f; c.cy = float(h) / 2.0f;
  c.width = w; c.height = h;
  c.near_plane = near_p; c.far_plane = far_p;
  return c;
}

// synth_scene parameters + cameras (synth.hpp:100-154). cfg_d as in oracle/ref_shim.cpp:
// box, radius_min, radius_max, fov_deg, fov_ramp, target_jitter, near, far, scale_min, scale_max,
// scale_aniso, opacity_min, opacity_max, sh_rest_noise. rows_out: n x 59; cams_out: cams.
void synth_scene(uint64_t seed, int64_t n, int cams, int width, int height, int sh_degree, const double* cfg,
                 float* rows_out, gss_camera* cams_out) {
  require(n >= 0 && cams >= 0 && width >= 1 && height >= 1, "synth: bad sizes");
  require(sh_degree >= 0 && sh_degree <= 3, "synth: sh_degree must be in [0,3]");
  const double box = cfg[0], radius_min = cfg[1], radius_max = cfg[2], fov_deg = cfg[3], fov_ramp = cfg[4],
               target_jitter = cfg[5], near_p = cfg[6], far_p = cfg[7], scale_min = cfg[8], scale_max = cfg[9],
               scale_aniso = cfg[10], opacity_min = cfg[11], opacity_max = cfg[12], sh_rest_noise = cfg[13];
  Rng rng(seed * 0x9E3779B97F4A7C15ull + 0xD1B54A32D192ED03ull);
  const double kShC0 = 0.28209479177387814;
  for (int64_t i = 0; i < n; ++i) {
    float* row = rows_out + i * 59;
    for (int k = 0; k < 59; ++k) row[k] = 0.0f;
    for (int a = 0; a < 3; ++a) row[a] = float(rng.uniform(-box, box));
    const double log_lo = std::log(scale_min * box), log_hi = std::log(scale_max * box);
    const double base = rng.uniform(log_lo, log_hi);
    for (int a = 0; a < 3; ++a) row[3 + a] = float(base + rng.uniform(-scale_aniso, scale_aniso));
    double q[4];
    double qn = 0;
    for (auto& c : q) {
      c = rng.normal();
      qn += c * c;
    }
    qn = std::sqrt(qn);
    if (qn < 1e-9) {
      q[0] = 1;
      q[1] = q[2] = q[3] = 0;
      qn = 1;
    }
    for (int a = 0; a < 4; ++a) row[6 + a] = float(q[a] / qn);
    const double p = rng.uniform(opacity_min, opacity_max);
    row[10] = float(std::log(p) - std::log(1.0 - p));  // logit (scene.hpp:141)
    for (int c = 0; c < 3; ++c) row[11 + c] = float((rng.uniform(0.08, 0.92) - 0.5) / kShC0);
    const int active = (sh_degree + 1) * (sh_degree + 1);
    for (int k = 1; k < active; ++k)
      for (int c = 0; c < 3; ++c) row[11 + k * 3 + c] = float(rng.normal() * sh_rest_noise);
  }
  const double golden = 2.399963229728653;
  std::vector<gss_camera> cv;
  for (int i = 0; i < cams; ++i) {
    const double t = cams > 1 ? double(i) / (cams - 1) : 1.0;
    const double radius = box * (radius_min * std::pow(radius_max / radius_min, t));
    const double fov = fov_deg * (fov_ramp + (1.0 - fov_ramp) * t);
    const double fx = 0.5 * width / std::tan(0.5 * fov * M_PI / 180.0);
    const double fy = fx;
    const double az = golden * i + rng.uniform(-0.15, 0.15);
    const double el = (0.15 + 0.55 * rng.uniform()) * (i % 2 == 0 ? 1.0 : -1.0);
    const float eye[3] = {float(radius * std::cos(el) * std::cos(az)), float(radius * std::sin(el)),
                          float(radius * std::cos(el) * std::sin(az))};
    const double jig = target_jitter * (1.0 - t);
    const float ta = float(rng.uniform(-jig, jig) * box);
    const float tb = float(rng.uniform(-jig, jig) * box);
    const float tc = float(rng.uniform(-jig, jig) * box);
    const float target[3] = {ta, tb, tc};
    cv.push_back(look_at(eye, target, float(fx), float(fy), width, height, float(near_p), float(far_p)));
  }
  for (int i = cams - 1; i > 0; --i) {
    const int j = int(rng.next_u64() % uint64_t(i + 1));
    std::swap(cv[i], cv[j]);
  }
  if (cams > 0) std::memcpy(cams_out, cv.data(), sizeof(gss_camera) * cv.size());
}

}  // namespace gssd

extern "C" __attribute__((visibility("default"))) int gss_synth_scene(uint64_t seed, int64_t n, int32_t cams,
                                                                      int32_t width, int32_t height,
                                                                      int32_t sh_degree, const double* cfg,
                                                                      float* rows_out, gss_camera* cams_out) {
  return gssd::guarded([&] { gssd::synth_scene(seed, n, cams, width, height, sh_degree, cfg, rows_out, cams_out); });
}

extern "C" __attribute__((visibility("default"))) int gss_look_at_camera(const float* eye, const float* target,
                                                                         float fx, float fy, int32_t w, int32_t h,
                                                                         float near_p, float far_p, gss_camera* out) {
  return gssd::guarded([&] { *out = gssd::look_at(eye, target, fx, fy, w, h, near_p, far_p); });
}
