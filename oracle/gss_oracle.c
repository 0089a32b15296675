/* TEST INFRASTRUCTURE ONLY — CPU restatement of the GS-Scale per-iteration hot path.
 * See gss_oracle.h. Build: oracle/Makefile (gcc -O2 -std=c11 -ffp-contract=off).
 * Parity pinned against oracle/_ref (the reference itself) and tests/golden/ by tests/test_oracle.py.
 * Every expression keeps the reference's evaluation order (left-to-right sums, no contraction).
 */
#include "gss_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* glibc 2.39 sysdeps/ieee754/flt-32/e_expf.c restated (the FMA ifunc build the reference links:
 * the compiler contracts z*x+shift, z*x-kd and the polynomial into fma). Table: 2^(i/32) rounded
 * to double, minus i<<47. Verified exhaustively against host expf over all 2^32 inputs. */
static const uint64_t kExp2Tab[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

float orc_expf(float x) {
  uint32_t ux;
  memcpy(&ux, &x, 4);
  if (ux == 0xff800000u) return 0.0f;
  if (isnan(x) || isinf(x)) return x + x;
  if (x > 0x1.62e42ep6f) return INFINITY;
  if (x < -0x1.9fe368p6f) return 0.0f;
  const double inv_ln2_n = 0x1.71547652b82fep+0 * 32, shift = 0x1.8p+52;
  const double xd = x;
  double kd = fma(inv_ln2_n, xd, shift);
  uint64_t ki;
  memcpy(&ki, &kd, 8);
  kd -= shift;
  const double r = fma(inv_ln2_n, xd, -kd);
  uint64_t t = kExp2Tab[ki % 32] + (ki << 47);
  double s;
  memcpy(&s, &t, 8);
  const double z = fma(0x1.c6af84b912394p-5 / (32.0 * 32 * 32), r, 0x1.ebfce50fac4f3p-3 / (32.0 * 32));
  const double r2 = r * r;
  double y = fma(0x1.62e42ff0c52d6p-1 / 32, r, 1.0);
  y = fma(z, r2, y);
  y = y * s;
  return (float)y;
}

static inline float fmaxz(float v) { return v < 0.0f ? 0.0f : v; } /* std::max(v, 0): NaN passes */

/* ------------------------------------------------------------------------- */
/* vecmath.hpp / scene.hpp pieces */

typedef struct { float x, y, z; } v3;

static v3 to_camera(const orc_camera* c, float x, float y, float z) { /* scene.hpp:85, vecmath.hpp:48-52 */
  const float* m = c->rot;
  v3 r;
  r.x = (m[0] * x + m[1] * y + m[2] * z) + c->trans[0];
  r.y = (m[3] * x + m[4] * y + m[5] * z) + c->trans[1];
  r.z = (m[6] * x + m[7] * y + m[8] * z) + c->trans[2];
  return r;
}

static v3 cam_position(const orc_camera* c) { /* scene.hpp:86-89 */
  const float* m = c->rot;
  const float tx = -c->trans[0], ty = -c->trans[1], tz = -c->trans[2];
  v3 r = {m[0] * tx + m[3] * ty + m[6] * tz, m[1] * tx + m[4] * ty + m[7] * tz, m[2] * tx + m[5] * ty + m[8] * tz};
  return r;
}

static void quat_to_rot(float w, float x, float y, float z, float R[9]) { /* vecmath.hpp:61-74 */
  R[0] = 1.0f - 2.0f * (y * y + z * z);
  R[1] = 2.0f * (x * y - w * z);
  R[2] = 2.0f * (x * z + w * y);
  R[3] = 2.0f * (x * y + w * z);
  R[4] = 1.0f - 2.0f * (x * x + z * z);
  R[5] = 2.0f * (y * z - w * x);
  R[6] = 2.0f * (x * z - w * y);
  R[7] = 2.0f * (y * z + w * x);
  R[8] = 1.0f - 2.0f * (x * x + y * y);
}

/* ------------------------------------------------------------------------- */
/* Projection (render.hpp:90-148) */

typedef struct {
  float mx, my, a, b, c, depth, radius;
  float rgb[3];
  float ab;
  int valid;
  /* ProjectBackward (render.hpp:82-88) */
  v3 t;
  float q_raw[4], q_unit[4], es[3];
} proj_t;

static void project(const float* g, const orc_camera* cam, float lp, proj_t* o) {
  memset(o, 0, sizeof(*o));
  const v3 t = to_camera(cam, g[0], g[1], g[2]);
  if (!(t.z > 1e-9f)) return;
  const float iz = 1.0f / t.z;
  o->depth = t.z;
  o->mx = cam->fx * t.x * iz + cam->cx;
  o->my = cam->fy * t.y * iz + cam->cy;
  const float qw = g[6], qx = g[7], qy = g[8], qz = g[9];
  const float qn = sqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
  const float qinv = qn > 1e-12f ? 1.0f / qn : 0.0f;
  const float q[4] = {qw * qinv, qx * qinv, qy * qinv, qz * qinv};
  float R[9];
  quat_to_rot(q[0], q[1], q[2], q[3], R);
  const float es[3] = {orc_expf(g[3]), orc_expf(g[4]), orc_expf(g[5])};
  float B[9], S[9];
  for (int i = 0; i < 3; ++i) {
    B[i * 3 + 0] = R[i * 3 + 0] * es[0];
    B[i * 3 + 1] = R[i * 3 + 1] * es[1];
    B[i * 3 + 2] = R[i * 3 + 2] * es[2];
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) S[i * 3 + j] = B[i * 3] * B[j * 3] + B[i * 3 + 1] * B[j * 3 + 1] + B[i * 3 + 2] * B[j * 3 + 2];
  const float j00 = cam->fx * iz, j02 = -cam->fx * t.x * iz * iz;
  const float j11 = cam->fy * iz, j12 = -cam->fy * t.y * iz * iz;
  const float* W = cam->rot;
  const float m0[3] = {j00 * W[0] + j02 * W[6], j00 * W[1] + j02 * W[7], j00 * W[2] + j02 * W[8]};
  const float m1[3] = {j11 * W[3] + j12 * W[6], j11 * W[4] + j12 * W[7], j11 * W[5] + j12 * W[8]};
  float v0[3], v1[3];
  for (int i = 0; i < 3; ++i) {
    v0[i] = S[i * 3] * m0[0] + S[i * 3 + 1] * m0[1] + S[i * 3 + 2] * m0[2];
    v1[i] = S[i * 3] * m1[0] + S[i * 3 + 1] * m1[1] + S[i * 3 + 2] * m1[2];
  }
  o->a = (m0[0] * v0[0] + m0[1] * v0[1] + m0[2] * v0[2]) + lp;
  o->b = m0[0] * v1[0] + m0[1] * v1[1] + m0[2] * v1[2];
  o->c = (m1[0] * v1[0] + m1[1] * v1[1] + m1[2] * v1[2]) + lp;
  const float mid = (o->a + o->c) / 2.0f;
  const float half = (o->a - o->c) / 2.0f;
  const float lmax = mid + sqrtf(half * half + o->b * o->b);
  o->radius = 3.0f * sqrtf(fmaxz(lmax));
  o->valid = 1;
  o->t = t;
  o->q_raw[0] = qw; o->q_raw[1] = qx; o->q_raw[2] = qy; o->q_raw[3] = qz;
  memcpy(o->q_unit, q, sizeof(q));
  memcpy(o->es, es, sizeof(es));
}

void orc_project_geo(const float* g, const orc_camera* cam, float low_pass, float* out) {
  proj_t p;
  project(g, cam, low_pass, &p);
  out[0] = p.mx; out[1] = p.my; out[2] = p.a; out[3] = p.b; out[4] = p.c;
  out[5] = p.depth; out[6] = p.radius; out[7] = p.valid ? 1.0f : 0.0f;
}

/* ------------------------------------------------------------------------- */
/* Culling (render.hpp:243-260) */

static int cull_keep(const float* g, const orc_camera* cam, const orc_viewport* vp, float lp) {
  const v3 t = to_camera(cam, g[0], g[1], g[2]);
  if (!(t.z >= cam->near_plane && t.z <= cam->far_plane)) return 0;
  proj_t p;
  project(g, cam, lp, &p);
  if (!p.valid) return 0;
  return p.mx + p.radius >= vp->x0 && p.mx - p.radius <= vp->x1 && p.my + p.radius >= vp->y0 &&
         p.my - p.radius <= vp->y1;
}

int64_t orc_frustum_cull(const float* geo, int64_t n, int64_t stride, const orc_camera* cam, const orc_viewport* vp,
                         float low_pass, int32_t* out_ids) {
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i)
    if (cull_keep(geo + i * stride, cam, vp, low_pass)) {
      if (out_ids) out_ids[k] = (int32_t)i;
      ++k;
    }
  return k;
}

/* ------------------------------------------------------------------------- */
/* Optimizer (adam.hpp:67-313) */

void orc_build_luts(double lr, double b1, double b2, double eps, int64_t t, int max_delay, float* param, float* mom,
                    float* var, float* pow_b1, float* pow_b2, float* scalars) {
  const int usable = (int)((int64_t)max_delay < t - 1 ? (int64_t)max_delay : t - 1);
  for (int i = 0; i <= max_delay; ++i) param[i] = 0.0f;
  const double scale = b1 / sqrt(b2);
  double acc = 0.0;
  for (int i = 1; i <= usable; ++i) {
    acc = scale * acc + (lr * b1) / (sqrt(b2 / (1.0 - pow(b2, (double)(t - i)))) * (1.0 - pow(b1, (double)(t - i))));
    param[i] = (float)acc;
  }
  for (int i = usable + 1; i <= max_delay; ++i) param[i] = (float)acc;
  for (int i = 0; i <= max_delay; ++i) {
    mom[i] = (float)pow(b1, (double)(i + 1));
    var[i] = (float)pow(b2, (double)(i + 1));
    pow_b1[i] = (float)pow(b1, (double)i);
    pow_b2[i] = (float)pow(b2, (double)i);
  }
  scalars[0] = (float)(1.0 - b1);
  scalars[1] = (float)(1.0 - b2);
  scalars[2] = (float)sqrt(1.0 - pow(b2, (double)t));
  scalars[3] = (float)(lr / (1.0 - pow(b1, (double)t)));
  scalars[4] = (float)eps;
}

typedef struct {
  float param[256], mom[256], var[256], pb1[256], pb2[256], sc[5];
} luts_t;

static void luts_for(const orc_arena* a, int64_t t, luts_t* l) {
  for (int g = 0; g < a->ngroups; ++g)
    orc_build_luts(a->lr[g], a->b1, a->b2, a->eps, t, a->defer_max, l[g].param, l[g].mom, l[g].var, l[g].pb1,
                   l[g].pb2, l[g].sc);
}

/* deferred_scalar (adam.hpp:102-110) */
static inline void deferred_scalar(float* w, float* m, float* v, float g, float ws, float ms, float vs,
                                   const float* sc) {
  const float m_new = ms * *m + sc[0] * g;
  const float v_new = vs * *v + sc[1] * g * g;
  *w -= (ws * *m) / (sqrtf(*v) + sc[4]);
  const float denom = sqrtf(v_new) / sc[2] + sc[4];
  *w = *w - sc[3] * m_new / denom;
  *m = m_new;
  *v = v_new;
}

static void update_row(orc_arena* a, const luts_t* l, int64_t id, int d, const float* grad) { /* adam.hpp:181-192 */
  float* wp = a->w + id * a->dim;
  float* mp = a->m + id * a->dim;
  float* vp = a->v + id * a->dim;
  for (int g = 0; g < a->ngroups; ++g) {
    const luts_t* k = &l[g];
    for (int c = a->col0[g]; c < a->col0[g] + a->gdim[g]; ++c)
      deferred_scalar(&wp[c], &mp[c], &vp[c], grad ? grad[c] : 0.0f, k->param[d], k->mom[d], k->var[d], k->sc);
  }
}

void orc_adam_step_dense(orc_arena* a, const float* grads) {
  const int64_t t = a->step + 1;
  luts_t* l = (luts_t*)malloc(sizeof(luts_t) * (size_t)a->ngroups);
  luts_for(a, t, l);
  for (int64_t id = 0; id < a->n; ++id) update_row(a, l, id, 0, grads ? grads + id * a->dim : NULL);
  a->step = t;
  free(l);
}

int64_t orc_deferred_update(orc_arena* a, int64_t nids, const int32_t* ids, const float* rows, int64_t stride,
                            int col0, int32_t* touched_out) {
  const int64_t t = a->step + 1;
  luts_t* l = (luts_t*)malloc(sizeof(luts_t) * (size_t)a->ngroups);
  luts_for(a, t, l);
  int64_t gi = 0, nt = 0;
  for (int64_t id = 0; id < a->n; ++id) {
    const int has_grad = gi < nids && ids[gi] == id;
    const int saturated = a->counter[id] == a->defer_max;
    if (has_grad || saturated) {
      update_row(a, l, id, a->counter[id], has_grad ? rows + gi * stride + col0 : NULL);
      if (touched_out) touched_out[nt] = (int32_t)id;
      ++nt;
      a->counter[id] = 0;
    } else {
      a->counter[id]++;
    }
    if (has_grad) ++gi;
  }
  free(l);
  if (gi != nids) return -3; /* InvariantViolation (adam.hpp:231) */
  a->step = t;
  return nt;
}

void orc_restore_view(const orc_arena* a, int64_t nids, const int32_t* ids, int has_pending, int64_t npend,
                      const int32_t* pids, const float* prows, int64_t pstride, int pcol0, float* out) {
  const int64_t t = a->step + 1;
  luts_t* l = (luts_t*)malloc(sizeof(luts_t) * (size_t)a->ngroups);
  luts_for(a, t, l);
  int64_t pi = 0;
  for (int64_t k = 0; k < nids; ++k) {
    const int64_t id = ids[k];
    const int d = a->counter[id];
    const float* grad = NULL;
    if (has_pending) {
      while (pi < npend && pids[pi] < id) ++pi;
      if (pi < npend && pids[pi] == id) grad = prows + pi * pstride + pcol0;
    }
    const float* wp = a->w + id * a->dim;
    const float* mp = a->m + id * a->dim;
    const float* vp = a->v + id * a->dim;
    float* o = out + k * a->dim;
    for (int g = 0; g < a->ngroups; ++g) {
      const luts_t* lt = &l[g];
      for (int c = a->col0[g]; c < a->col0[g] + a->gdim[g]; ++c) {
        if (has_pending) {
          float w = wp[c], m = mp[c], v = vp[c];
          deferred_scalar(&w, &m, &v, grad ? grad[c] : 0.0f, lt->param[d], lt->mom[d], lt->var[d], lt->sc);
          o[c] = w;
        } else {
          o[c] = wp[c] - (lt->param[d] * mp[c]) / (sqrtf(vp[c]) + lt->sc[4]); /* restore_scalar adam.hpp:112 */
        }
      }
    }
  }
  free(l);
}

void orc_flush_deferred(orc_arena* a) {
  const int64_t t = a->step + 1;
  luts_t* l = (luts_t*)malloc(sizeof(luts_t) * (size_t)a->ngroups);
  luts_for(a, t, l);
  for (int64_t id = 0; id < a->n; ++id) {
    const int d = a->counter[id];
    if (d == 0) continue;
    float* wp = a->w + id * a->dim;
    float* mp = a->m + id * a->dim;
    float* vp = a->v + id * a->dim;
    for (int g = 0; g < a->ngroups; ++g) {
      const luts_t* lt = &l[g];
      for (int c = a->col0[g]; c < a->col0[g] + a->gdim[g]; ++c) {
        wp[c] = wp[c] - (lt->param[d] * mp[c]) / (sqrtf(vp[c]) + lt->sc[4]);
        mp[c] *= lt->pb1[d];
        vp[c] *= lt->pb2[d];
      }
    }
    a->counter[id] = 0;
  }
  free(l);
}

/* ------------------------------------------------------------------------- */
/* Spherical harmonics (sh.hpp:24-125) */

#define SH_C0 0.28209479177387814
#define SH_C1 0.4886025119029199
static const double kC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                              0.5462742152960396};
static const double kC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                              -0.4570457994644658, 1.445305721320277, -0.5900435899266435};

static void sh_basis(float x, float y, float z, int deg, float* o) {
  o[0] = (float)SH_C0;
  if (deg < 1) return;
  o[1] = (float)(-SH_C1) * y;
  o[2] = (float)SH_C1 * z;
  o[3] = (float)(-SH_C1) * x;
  if (deg < 2) return;
  const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  o[4] = (float)kC2[0] * xy;
  o[5] = (float)kC2[1] * yz;
  o[6] = (float)kC2[2] * (2.0f * zz - xx - yy);
  o[7] = (float)kC2[3] * xz;
  o[8] = (float)kC2[4] * (xx - yy);
  if (deg < 3) return;
  o[9] = (float)kC3[0] * y * (3.0f * xx - yy);
  o[10] = (float)kC3[1] * xy * z;
  o[11] = (float)kC3[2] * y * (4.0f * zz - xx - yy);
  o[12] = (float)kC3[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
  o[13] = (float)kC3[4] * x * (4.0f * zz - xx - yy);
  o[14] = (float)kC3[5] * z * (xx - yy);
  o[15] = (float)kC3[6] * x * (xx - 3.0f * yy);
}

static void sh_basis_grad(float x, float y, float z, int deg, v3* o) {
  const v3 zero = {0, 0, 0};
  o[0] = zero;
  if (deg < 1) return;
  o[1] = (v3){0.0f, (float)(-SH_C1), 0.0f};
  o[2] = (v3){0.0f, 0.0f, (float)SH_C1};
  o[3] = (v3){(float)(-SH_C1), 0.0f, 0.0f};
  if (deg < 2) return;
  const float c20 = (float)kC2[0], c21 = (float)kC2[1], c22 = (float)kC2[2], c23 = (float)kC2[3], c24 = (float)kC2[4];
  o[4] = (v3){c20 * y, c20 * x, 0.0f};
  o[5] = (v3){0.0f, c21 * z, c21 * y};
  o[6] = (v3){c22 * -2.0f * x, c22 * -2.0f * y, c22 * 4.0f * z};
  o[7] = (v3){c23 * z, 0.0f, c23 * x};
  o[8] = (v3){c24 * 2.0f * x, c24 * -2.0f * y, 0.0f};
  if (deg < 3) return;
  const float c30 = (float)kC3[0], c31 = (float)kC3[1], c32 = (float)kC3[2], c33 = (float)kC3[3], c34 = (float)kC3[4],
              c35 = (float)kC3[5], c36 = (float)kC3[6];
  o[9] = (v3){c30 * 6.0f * x * y, c30 * (3.0f * x * x - 3.0f * y * y), 0.0f};
  o[10] = (v3){c31 * y * z, c31 * x * z, c31 * x * y};
  o[11] = (v3){c32 * -2.0f * x * y, c32 * (4.0f * z * z - x * x - 3.0f * y * y), c32 * 8.0f * y * z};
  o[12] = (v3){c33 * -6.0f * x * z, c33 * -6.0f * y * z, c33 * (6.0f * z * z - 3.0f * x * x - 3.0f * y * y)};
  o[13] = (v3){c34 * (4.0f * z * z - 3.0f * x * x - y * y), c34 * -2.0f * x * y, c34 * 8.0f * x * z};
  o[14] = (v3){c35 * 2.0f * x * z, c35 * -2.0f * y * z, c35 * (x * x - y * y)};
  o[15] = (v3){c36 * (3.0f * x * x - 3.0f * y * y), c36 * -6.0f * x * y, 0.0f};
}

static float clamp01(float v) { return v < 0.0f ? 0.0f : (1.0f < v ? 1.0f : v); } /* std::clamp */

/* ------------------------------------------------------------------------- */
/* Rasterizer (render.hpp:297-640) */

typedef struct {
  int px0, px1, py0, py1;
} win_t;

/* x86-64 cvttsd2si: NaN / out-of-range -> INT_MIN (the reference's int(double) on its platform). */
static int d2i(double d) {
  if (!(d >= -2147483648.0 && d < 2147483648.0)) return (int)0x80000000u;
  return (int)d;
}

static int cover_box(const proj_t* p, const win_t* w, win_t* o) { /* render.hpp:307-314 */
  const double mx = p->mx, my = p->my, r = p->radius;
  const int a0 = d2i(ceil(mx - r - 0.5)), a1 = (int)((unsigned)d2i(floor(mx + r - 0.5)) + 1u);
  const int b0 = d2i(ceil(my - r - 0.5)), b1 = (int)((unsigned)d2i(floor(my + r - 0.5)) + 1u);
  o->px0 = a0 > w->px0 ? a0 : w->px0;
  o->px1 = a1 < w->px1 ? a1 : w->px1;
  o->py0 = b0 > w->py0 ? b0 : w->py0;
  o->py1 = b1 < w->py1 ? b1 : w->py1;
  return o->px0 < o->px1 && o->py0 < o->py1;
}

typedef struct {
  float alpha, q, weight;
  int clamped, ok;
} ceval_t;

static ceval_t contrib_eval(const proj_t* p, float cx, float cy) { /* render.hpp:342-358 */
  ceval_t r = {0, 0, 0, 0, 0};
  const float det = p->a * p->c - p->b * p->b;
  if (!(det > 0.0f)) return r;
  const float dx = cx - p->mx, dy = cy - p->my;
  r.q = fmaxz((p->c * dx * dx - 2.0f * p->b * dx * dy + p->a * dy * dy) / det);
  r.weight = orc_expf(-0.5f * r.q);
  const float raw = p->ab * r.weight;
  if (raw > (float)0.999) {
    r.alpha = (float)0.999;
    r.clamped = 1;
  } else {
    r.alpha = raw;
  }
  r.ok = 1;
  return r;
}

static const proj_t* g_sort_proj;
static const int32_t* g_sort_ids;
static int cmp_order(const void* pa, const void* pb) { /* render.hpp:408-411: (depth, id) */
  const int a = *(const int*)pa, b = *(const int*)pb;
  const float da = g_sort_proj[a].depth, db = g_sort_proj[b].depth;
  if (da != db) return da < db ? -1 : 1;
  return g_sort_ids[a] < g_sort_ids[b] ? -1 : (g_sort_ids[a] > g_sort_ids[b] ? 1 : 0);
}

typedef struct {
  int32_t slot;
  float alpha, trans;
} contrib_t;

int orc_render(int64_t n_ids, const int32_t* ids, const float* geo, int64_t geo_stride, const float* nongeo,
               int nongeo_compact, int sh_degree, const float* bg, const orc_camera* cam, const orc_viewport* vp,
               const float* gt_full, int64_t normalizer, const float* d_img_in, float* out_image,
               float* out_final_T, int32_t* out_len, float* out_loss, float* out_d_img, float* out_grad_rows,
               float* out_mean2d, int64_t* meta) {
  /* viewport_pixels (render.hpp:297-304) */
  win_t win;
  win.px0 = d2i(ceil((double)vp->x0 - 0.5));
  win.px1 = d2i(ceil((double)vp->x1 - 0.5));
  win.py0 = d2i(ceil((double)vp->y0 - 0.5));
  win.py1 = d2i(ceil((double)vp->y1 - 0.5));
  if (win.px0 < 0) win.px0 = 0;
  if (win.py0 < 0) win.py0 = 0;
  const int pw = win.px1 - win.px0 > 0 ? win.px1 - win.px0 : 0;
  const int ph = win.py1 - win.py0 > 0 ? win.py1 - win.py0 : 0;
  const size_t npix = (size_t)pw * ph;
  if (meta) { meta[0] = win.px0; meta[1] = win.py0; meta[2] = pw; meta[3] = ph; meta[4] = 0; }
  const int n = (int)n_ids;
  float* img = (float*)malloc(sizeof(float) * (npix * 3 + 1));
  float* fT = (float*)malloc(sizeof(float) * (npix + 1));
  int32_t* len = (int32_t*)calloc(npix + 1, sizeof(int32_t));
  int32_t* offs = (int32_t*)calloc(npix + 1, sizeof(int32_t));
  for (size_t i = 0; i < npix; ++i) {
    for (int c = 0; c < 3; ++c) img[i * 3 + c] = bg[c];
    fT[i] = 1.0f;
  }
  proj_t* proj = (proj_t*)calloc((size_t)n + 1, sizeof(proj_t));
  contrib_t* ct = NULL;
  const v3 campos = cam_position(cam);
  if (n > 0 && npix > 0) {
    /* project_all (render.hpp:361-380) */
    for (int k = 0; k < n; ++k) {
      const int64_t id = ids[k];
      const float* g = geo + id * geo_stride;
      project(g, cam, 0.3f, &proj[k]);
      if (!proj[k].valid) continue;
      const float* ng = nongeo + (nongeo_compact ? (int64_t)k : id) * 49;
      proj[k].ab = 1.0f / (1.0f + orc_expf(-ng[0]));
      v3 dir = {g[0] - campos.x, g[1] - campos.y, g[2] - campos.z};
      const float dn = sqrtf(dir.x * dir.x + dir.y * dir.y + dir.z * dir.z);
      if (dn > 1e-12f) {
        const float inv = 1.0f / dn;
        dir.x = dir.x * inv; dir.y = dir.y * inv; dir.z = dir.z * inv;
      } else {
        dir.x = 0.0f; dir.y = 0.0f; dir.z = 1.0f;
      }
      float basis[16];
      sh_basis(dir.x, dir.y, dir.z, sh_degree, basis);
      const int nb = (sh_degree + 1) * (sh_degree + 1);
      float rgb[3] = {0.5f, 0.5f, 0.5f};
      for (int b = 0; b < nb; ++b)
        for (int c = 0; c < 3; ++c) rgb[c] += basis[b] * ng[1 + 3 * b + c];
      for (int c = 0; c < 3; ++c) proj[k].rgb[c] = clamp01(rgb[c]);
    }
    int* order = (int*)malloc(sizeof(int) * (size_t)n);
    for (int k = 0; k < n; ++k) order[k] = k;
    g_sort_proj = proj;
    g_sort_ids = ids;
    qsort(order, (size_t)n, sizeof(int), cmp_order);
    /* CSR count / prefix / fill (render.hpp:413-436) */
    win_t box;
    for (int oi = 0; oi < n; ++oi) {
      const proj_t* p = &proj[order[oi]];
      if (!p->valid || !(p->a * p->c - p->b * p->b > 0.0f)) continue;
      if (!cover_box(p, &win, &box)) continue;
      for (int y = box.py0; y < box.py1; ++y)
        for (int x = box.px0; x < box.px1; ++x) offs[(size_t)(y - win.py0) * pw + (x - win.px0) + 1]++;
    }
    for (size_t i = 1; i <= npix; ++i) offs[i] += offs[i - 1];
    if (meta) meta[4] = offs[npix];
    ct = (contrib_t*)malloc(sizeof(contrib_t) * ((size_t)offs[npix] + 1));
    int32_t* cursor = (int32_t*)malloc(sizeof(int32_t) * (npix + 1));
    memcpy(cursor, offs, sizeof(int32_t) * npix);
    for (int oi = 0; oi < n; ++oi) {
      const int slot = order[oi];
      const proj_t* p = &proj[slot];
      if (!p->valid || !(p->a * p->c - p->b * p->b > 0.0f)) continue;
      if (!cover_box(p, &win, &box)) continue;
      for (int y = box.py0; y < box.py1; ++y)
        for (int x = box.px0; x < box.px1; ++x) {
          const size_t pix = (size_t)(y - win.py0) * pw + (x - win.px0);
          ct[cursor[pix]].slot = slot;
          ct[cursor[pix]].alpha = 0.0f;
          ct[cursor[pix]].trans = 0.0f;
          cursor[pix]++;
        }
    }
    free(cursor);
    free(order);
    /* composite (render.hpp:438-462) */
    for (int y = 0; y < ph; ++y)
      for (int x = 0; x < pw; ++x) {
        const size_t pix = (size_t)y * pw + x;
        const float cx = (float)(x + win.px0) + 0.5f, cy = (float)(y + win.py0) + 0.5f;
        float T = 1.0f, col[3] = {0, 0, 0};
        int32_t used = 0;
        for (int32_t e = offs[pix]; e < offs[pix + 1]; ++e) {
          if (T < 1e-4f) break;
          const proj_t* p = &proj[ct[e].slot];
          const ceval_t ev = contrib_eval(p, cx, cy);
          ct[e].alpha = ev.alpha;
          ct[e].trans = T;
          for (int c = 0; c < 3; ++c) col[c] += p->rgb[c] * ev.alpha * T;
          T *= (1.0f - ev.alpha);
          ++used;
        }
        len[pix] = used;
        fT[pix] = T;
        for (int c = 0; c < 3; ++c) img[pix * 3 + c] = col[c] + T * bg[c];
      }
  }
  if (out_image) memcpy(out_image, img, sizeof(float) * npix * 3);
  if (out_final_T) memcpy(out_final_T, fT, sizeof(float) * npix);
  if (out_len) memcpy(out_len, len, sizeof(int32_t) * npix);

  /* compute_loss_l1 (render.hpp:497-511) */
  float* dimg = (float*)calloc(npix * 3 + 1, sizeof(float));
  if (gt_full) {
    if (normalizer == 0) normalizer = (int64_t)(npix * 3);
    const float inv = 1.0f / (float)(double)normalizer;
    double acc = 0.0;
    for (int y = 0; y < ph; ++y)
      for (int x = 0; x < pw; ++x)
        for (int c = 0; c < 3; ++c) {
          const size_t i = ((size_t)y * pw + x) * 3 + c;
          const float gtv = gt_full[((size_t)(y + win.py0) * cam->width + (x + win.px0)) * 3 + c];
          const float d = img[i] - gtv;
          acc += fabs((double)d);
          dimg[i] = d > 0.0f ? inv : (d < 0.0f ? -inv : 0.0f);
        }
    if (out_loss) *out_loss = (float)acc * inv;
  }
  if (d_img_in) memcpy(dimg, d_img_in, sizeof(float) * npix * 3);
  if (out_d_img) memcpy(out_d_img, dimg, sizeof(float) * npix * 3);

  /* rasterize_backward (render.hpp:526-640) */
  if (out_grad_rows || out_mean2d) {
    float* grows = (float*)calloc((size_t)n * 59 + 1, sizeof(float));
    float* m2d = (float*)calloc((size_t)n * 2 + 1, sizeof(float));
    if (n > 0 && npix > 0) {
      float* acc = (float*)calloc((size_t)n * 9, sizeof(float)); /* rgb3, m2d2, cov3, ab */
      for (int y = 0; y < ph; ++y)
        for (int x = 0; x < pw; ++x) {
          const size_t pix = (size_t)y * pw + x;
          const int32_t beg = offs[pix], cnt = len[pix];
          if (cnt == 0) continue;
          const float cx = (float)(x + win.px0) + 0.5f, cy = (float)(y + win.py0) + 0.5f;
          const float g0 = dimg[pix * 3], g1 = dimg[pix * 3 + 1], g2 = dimg[pix * 3 + 2];
          if (g0 == 0.0f && g1 == 0.0f && g2 == 0.0f) continue;
          float suf[3] = {fT[pix] * bg[0], fT[pix] * bg[1], fT[pix] * bg[2]};
          for (int32_t e = beg + cnt - 1; e >= beg; --e) {
            const proj_t* p = &proj[ct[e].slot];
            const float alpha = ct[e].alpha, T = ct[e].trans;
            float* sa = acc + (size_t)ct[e].slot * 9;
            const float w_rgb = alpha * T;
            sa[0] += w_rgb * g0;
            sa[1] += w_rgb * g1;
            sa[2] += w_rgb * g2;
            const float dot_c = p->rgb[0] * g0 + p->rgb[1] * g1 + p->rgb[2] * g2;
            const float dot_suf = suf[0] * g0 + suf[1] * g1 + suf[2] * g2;
            const float d_alpha = T * dot_c - dot_suf / (1.0f - alpha);
            suf[0] += p->rgb[0] * alpha * T;
            suf[1] += p->rgb[1] * alpha * T;
            suf[2] += p->rgb[2] * alpha * T;
            const ceval_t ev = contrib_eval(p, cx, cy);
            if (!ev.ok || ev.clamped) continue;
            sa[8] += ev.weight * d_alpha;
            const float d_q = -0.5f * alpha * d_alpha;
            const float det = p->a * p->c - p->b * p->b;
            const float inv_det = 1.0f / det;
            const float dx = cx - p->mx, dy = cy - p->my;
            sa[5] += d_q * (dy * dy - ev.q * p->c) * inv_det;
            sa[6] += d_q * (-2.0f * dx * dy + 2.0f * ev.q * p->b) * inv_det;
            sa[7] += d_q * (dx * dx - ev.q * p->a) * inv_det;
            const float dq_dmx = (-2.0f * p->c * dx + 2.0f * p->b * dy) * inv_det;
            const float dq_dmy = (2.0f * p->b * dx - 2.0f * p->a * dy) * inv_det;
            sa[3] += d_q * dq_dmx;
            sa[4] += d_q * dq_dmy;
          }
        }
      /* chain (render.hpp:600-638) */
      for (int k = 0; k < n; ++k) {
        const proj_t* p = &proj[k];
        if (!p->valid) continue;
        const float* sa = acc + (size_t)k * 9;
        const int64_t id = ids[k];
        const float* g = geo + id * geo_stride;
        const float* ng = nongeo + (nongeo_compact ? (int64_t)k : id) * 49;
        float* out = grows + (size_t)k * 59;
        m2d[k * 2] = sa[3];
        m2d[k * 2 + 1] = sa[4];
        const float ab = p->ab;
        out[10] += sa[8] * ab * (1.0f - ab);
        const v3 dir = {g[0] - campos.x, g[1] - campos.y, g[2] - campos.z};
        const float dn = sqrtf(dir.x * dir.x + dir.y * dir.y + dir.z * dir.z);
        v3 dmd = {0, 0, 0};
        if (dn > 1e-12f) {
          const float inv = 1.0f / dn;
          const v3 u = {dir.x * inv, dir.y * inv, dir.z * inv};
          float basis[16];
          v3 bgr[16];
          sh_basis(u.x, u.y, u.z, sh_degree, basis);
          sh_basis_grad(u.x, u.y, u.z, sh_degree, bgr);
          const int nb = (sh_degree + 1) * (sh_degree + 1);
          int clamped[3];
          for (int c = 0; c < 3; ++c) { /* eval_sh_clamp_mask (sh.hpp:114-125) */
            float v = 0.5f;
            for (int b = 0; b < nb; ++b) v += basis[b] * ng[1 + 3 * b + c];
            clamped[c] = v < 0.0f || v > 1.0f;
          }
          const float gc[3] = {clamped[0] ? 0.0f : sa[0], clamped[1] ? 0.0f : sa[1], clamped[2] ? 0.0f : sa[2]};
          v3 ddir = {0, 0, 0};
          for (int b = 0; b < nb; ++b) { /* eval_sh_backward (sh.hpp:92-110) */
            float coef_dot = 0.0f;
            for (int c = 0; c < 3; ++c) {
              out[11 + 3 * b + c] += basis[b] * gc[c];
              coef_dot += ng[1 + 3 * b + c] * gc[c];
            }
            ddir.x += bgr[b].x * coef_dot;
            ddir.y += bgr[b].y * coef_dot;
            ddir.z += bgr[b].z * coef_dot;
          }
          const float dotp = u.x * ddir.x + u.y * ddir.y + u.z * ddir.z;
          const float inv2 = 1.0f / dn;
          dmd.x = (ddir.x - u.x * dotp) * inv2;
          dmd.y = (ddir.y - u.y * dotp) * inv2;
          dmd.z = (ddir.z - u.z * dotp) * inv2;
        }
        out[0] += dmd.x;
        out[1] += dmd.y;
        out[2] += dmd.z;
        /* project_geo_backward (render.hpp:152-237) */
        const float dmx = sa[3], dmy = sa[4], da = sa[5], db = sa[6], dc = sa[7];
        const v3 t = p->t;
        const float iz = 1.0f / t.z, iz2 = iz * iz;
        float R[9];
        quat_to_rot(p->q_unit[0], p->q_unit[1], p->q_unit[2], p->q_unit[3], R);
        const float* es = p->es;
        float B[9], S[9];
        for (int i = 0; i < 3; ++i) {
          B[i * 3 + 0] = R[i * 3 + 0] * es[0];
          B[i * 3 + 1] = R[i * 3 + 1] * es[1];
          B[i * 3 + 2] = R[i * 3 + 2] * es[2];
        }
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j)
            S[i * 3 + j] = B[i * 3] * B[j * 3] + B[i * 3 + 1] * B[j * 3 + 1] + B[i * 3 + 2] * B[j * 3 + 2];
        const float fx = cam->fx, fy = cam->fy;
        const float j00 = fx * iz, j02 = -fx * t.x * iz2;
        const float j11 = fy * iz, j12 = -fy * t.y * iz2;
        const float* W = cam->rot;
        const float m0[3] = {j00 * W[0] + j02 * W[6], j00 * W[1] + j02 * W[7], j00 * W[2] + j02 * W[8]};
        const float m1[3] = {j11 * W[3] + j12 * W[6], j11 * W[4] + j12 * W[7], j11 * W[5] + j12 * W[8]};
        float v0[3], v1[3];
        for (int i = 0; i < 3; ++i) {
          v0[i] = S[i * 3] * m0[0] + S[i * 3 + 1] * m0[1] + S[i * 3 + 2] * m0[2];
          v1[i] = S[i * 3] * m1[0] + S[i * 3 + 1] * m1[1] + S[i * 3 + 2] * m1[2];
        }
        float dm0[3], dm1[3];
        for (int i = 0; i < 3; ++i) {
          dm0[i] = v0[i] * (2.0f * da) + v1[i] * db;
          dm1[i] = v1[i] * (2.0f * dc) + v0[i] * db;
        }
        float dS[9], dB[9];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) dS[i * 3 + j] = da * m0[i] * m0[j] + db * m0[i] * m1[j] + dc * m1[i] * m1[j];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            float a2 = 0.0f;
            for (int k2 = 0; k2 < 3; ++k2) a2 += (dS[i * 3 + k2] + dS[k2 * 3 + i]) * B[k2 * 3 + j];
            dB[i * 3 + j] = a2;
          }
        float G[9];
        for (int i = 0; i < 3; ++i) {
          G[i * 3 + 0] = dB[i * 3 + 0] * es[0];
          G[i * 3 + 1] = dB[i * 3 + 1] * es[1];
          G[i * 3 + 2] = dB[i * 3 + 2] * es[2];
        }
        for (int j = 0; j < 3; ++j) {
          float a2 = 0.0f;
          for (int i = 0; i < 3; ++i) a2 += dB[i * 3 + j] * R[i * 3 + j];
          out[3 + j] += a2 * (j == 0 ? es[0] : (j == 1 ? es[1] : es[2]));
        }
        /* quat_rot_backward (vecmath.hpp:78-90) */
        const float w = p->q_unit[0], x = p->q_unit[1], y = p->q_unit[2], z = p->q_unit[3];
#define GG(i, j) G[(i) * 3 + (j)]
        float dq[4];
        dq[0] = 2.0f * (-z * GG(0, 1) + y * GG(0, 2) + z * GG(1, 0) - x * GG(1, 2) - y * GG(2, 0) + x * GG(2, 1));
        dq[1] = 2.0f * (y * GG(0, 1) + z * GG(0, 2) + y * GG(1, 0) - 2.0f * x * GG(1, 1) - w * GG(1, 2) +
                        z * GG(2, 0) + w * GG(2, 1) - 2.0f * x * GG(2, 2));
        dq[2] = 2.0f * (-2.0f * y * GG(0, 0) + x * GG(0, 1) + w * GG(0, 2) + x * GG(1, 0) + z * GG(1, 2) -
                        w * GG(2, 0) + z * GG(2, 1) - 2.0f * y * GG(2, 2));
        dq[3] = 2.0f * (-2.0f * z * GG(0, 0) - w * GG(0, 1) + x * GG(0, 2) + w * GG(1, 0) - 2.0f * z * GG(1, 1) +
                        y * GG(1, 2) + x * GG(2, 0) + y * GG(2, 1));
#undef GG
        /* quat_normalize_backward (vecmath.hpp:93-100) */
        const float* qr = p->q_raw;
        const float nq = sqrtf(qr[0] * qr[0] + qr[1] * qr[1] + qr[2] * qr[2] + qr[3] * qr[3]);
        const float qi = 1.0f / nq;
        const float u4[4] = {qr[0] * qi, qr[1] * qi, qr[2] * qi, qr[3] * qi};
        const float dotq = u4[0] * dq[0] + u4[1] * dq[1] + u4[2] * dq[2] + u4[3] * dq[3];
        for (int i = 0; i < 4; ++i) out[6 + i] += (dq[i] - u4[i] * dotq) * qi;
        const float dj00 = dm0[0] * W[0] + dm0[1] * W[1] + dm0[2] * W[2];
        const float dj02 = dm0[0] * W[6] + dm0[1] * W[7] + dm0[2] * W[8];
        const float dj11 = dm1[0] * W[3] + dm1[1] * W[4] + dm1[2] * W[5];
        const float dj12 = dm1[0] * W[6] + dm1[1] * W[7] + dm1[2] * W[8];
        v3 dt;
        dt.x = dmx * fx * iz + dj02 * (-fx * iz2);
        dt.y = dmy * fy * iz + dj12 * (-fy * iz2);
        dt.z = dmx * (-fx * t.x * iz2) + dmy * (-fy * t.y * iz2) + dj00 * (-fx * iz2) + dj11 * (-fy * iz2) +
               dj02 * (2.0f * fx * t.x * iz2 * iz) + dj12 * (2.0f * fy * t.y * iz2 * iz);
        out[0] += W[0] * dt.x + W[3] * dt.y + W[6] * dt.z;
        out[1] += W[1] * dt.x + W[4] * dt.y + W[7] * dt.z;
        out[2] += W[2] * dt.x + W[5] * dt.y + W[8] * dt.z;
      }
      free(acc);
    }
    if (out_grad_rows) memcpy(out_grad_rows, grows, sizeof(float) * (size_t)n * 59);
    if (out_mean2d) memcpy(out_mean2d, m2d, sizeof(float) * (size_t)n * 2);
    free(grows);
    free(m2d);
  }
  free(dimg);
  free(ct);
  free(proj);
  free(offs);
  free(len);
  free(fT);
  free(img);
  return 0;
}
