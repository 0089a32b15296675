// Exact-arithmetic device primitives shared by the cull, rasterizer and chain kernels.
//
// Every function reproduces the float operation order of the reference headers
// (/root/reference/proj/include/gss/{vecmath,sh,render}.hpp) with IEEE round-to-nearest
// mul/add/div/sqrt and NO contraction (this translation unit family is built with -fmad=false;
// explicit __fmul_rn/__fadd_rn are used where the order must survive any flag). That is what
// makes cull ids and forward pixels bit-identical to the CPU reference.
#pragma once

#include <cstdint>

#include "gss_b200.h"

namespace gssd {

// ---------------------------------------------------------------------------
// glibc 2.39 expf, FMA ifunc variant (sysdeps/ieee754/flt-32/e_expf.c as the reference links it;
// render.hpp:105, 348, 374 call std::exp(float)). Evaluated in fp64 exactly like the host:
// kd = fma(x, 32/ln2, 2^52*1.5), r = fma(x, 32/ln2, -kd), s = 2^(k/32) from the table, cubic in r.
// Exhaustively equal to host expf over all 2^32 inputs (oracle/gss_oracle.c: orc_expf).
// Global (not __constant__) table: the index differs per lane, and indexed constant-bank loads
// serialise across distinct addresses; an L1-resident global load does not.
__device__ static const unsigned long long kExp2Tab[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

// The fp64 coefficients live in the constant bank so the DFMAs take them as c[][] operands
// (as literals they are rematerialised into register pairs on every call inside a hot loop).
static __constant__ double kExpCoef[4] = {0x1.71547652b82fep+0 * 32.0, 0x1.c6af84b912394p-5 / (32.0 * 32 * 32),
                                          0x1.ebfce50fac4f3p-3 / (32.0 * 32), 0x1.62e42ff0c52d6p-1 / 32.0};

// glibc 2.39 expf body (table-driven, FMA variant) for x in [-103.97, 88.72].
__device__ __forceinline__ float gss_expf_core(float x) {
  const double inv_ln2_n = kExpCoef[0], shift = 0x1.8p+52;
  const double xd = (double)x;
  double kd = __fma_rn(inv_ln2_n, xd, shift);
  const unsigned long long ki = (unsigned long long)__double_as_longlong(kd);
  kd = __dsub_rn(kd, shift);
  const double r = __fma_rn(inv_ln2_n, xd, -kd);
  const unsigned long long t = __ldg(&kExp2Tab[ki & 31]) + (ki << 47);
  const double s = __longlong_as_double((long long)t);
  const double z = __fma_rn(kExpCoef[1], r, kExpCoef[2]);
  const double r2 = __dmul_rn(r, r);
  double y = __fma_rn(kExpCoef[3], r, 1.0);
  y = __fma_rn(z, r2, y);
  y = __dmul_rn(y, s);
  return __double2float_rn(y);
}

// The same core with the polynomial coefficients in registers (a hot loop hoists them once).
struct ExpCoef {
  double c0, c1, c2, c3;
};
__device__ __forceinline__ ExpCoef exp_coef() { return ExpCoef{kExpCoef[0], kExpCoef[1], kExpCoef[2], kExpCoef[3]}; }
// Register-resident copy for a hot loop: the values pass through an opaque move, so the compiler
// keeps them in registers instead of reloading the constant bank before every DFMA.
__device__ __forceinline__ ExpCoef exp_coef_regs(const ExpCoef& k) {
  ExpCoef r;
  asm("mov.b64 %0, %1;" : "=d"(r.c0) : "d"(k.c0));
  asm("mov.b64 %0, %1;" : "=d"(r.c1) : "d"(k.c1));
  asm("mov.b64 %0, %1;" : "=d"(r.c2) : "d"(k.c2));
  asm("mov.b64 %0, %1;" : "=d"(r.c3) : "d"(k.c3));
  return r;
}
// Host copy, for kernels that take the coefficients as a parameter (param-space operands of DFMA).
inline ExpCoef exp_coef_host() {
  return ExpCoef{0x1.71547652b82fep+0 * 32.0, 0x1.c6af84b912394p-5 / (32.0 * 32 * 32), 0x1.ebfce50fac4f3p-3 / (32.0 * 32),
                 0x1.62e42ff0c52d6p-1 / 32.0};
}
__device__ __forceinline__ float gss_expf_core(float x, const ExpCoef& k) {
  const double shift = 0x1.8p+52;
  const double xd = (double)x;
  double kd = __fma_rn(k.c0, xd, shift);
  const unsigned long long ki = (unsigned long long)__double_as_longlong(kd);
  kd = __dsub_rn(kd, shift);
  const double r = __fma_rn(k.c0, xd, -kd);
  const unsigned long long t = __ldg(&kExp2Tab[ki & 31]) + (ki << 47);
  const double s = __longlong_as_double((long long)t);
  const double z = __fma_rn(k.c1, r, k.c2);
  const double r2 = __dmul_rn(r, r);
  double y = __fma_rn(k.c3, r, 1.0);
  y = __fma_rn(z, r2, y);
  y = __dmul_rn(y, s);
  return __double2float_rn(y);
}
// gss_expf_nonpos without a branch: the core runs for every x and the underflow guard selects 0
// (x < -103.97, including -inf); NaN flows through the core (NaN in, NaN out, as glibc's x + x).
__device__ __forceinline__ float gss_expf_nonpos_sel(float x, const ExpCoef& k) {
  const float y = gss_expf_core(x, k);
  return x < -0x1.9fe368p6f ? 0.0f : y;
}

__device__ __forceinline__ float gss_expf(float x) {
  if (!(x <= 0x1.62e42ep6f)) {                 // > 88.72 (overflow), +inf or NaN
    if (x != x) return x + x;
    return __int_as_float(0x7f800000);
  }
  if (x < -0x1.9fe368p6f) return 0.0f;         // underflow and -inf
  return gss_expf_core(x);
}

// gss_expf for x <= 0 or NaN (the compositing exponent -q/2, q >= 0): only the underflow and NaN
// guards of expf can fire; the result is identical to gss_expf on that domain.
__device__ __forceinline__ float gss_expf_nonpos(float x) {
  if (!(x >= -0x1.9fe368p6f)) return (x != x) ? x + x : 0.0f;
  return gss_expf_core(x);
}

// std::max(v, 0) as the reference evaluates it ((v < 0) ? 0 : v; NaN passes through).
__device__ __forceinline__ float max0(float v) { return v < 0.0f ? 0.0f : v; }

// int(double) with x86-64 cvttsd2si semantics (NaN / out of range -> INT_MIN), the reference's
// platform behaviour for render.hpp:299-312.
__device__ __forceinline__ int d2i_x86(double d) {
  if (!(d >= -2147483648.0 && d < 2147483648.0)) return (int)0x80000000u;
  return (int)d;
}

// ---------------------------------------------------------------------------
// Camera (scene.hpp:77-89). p_cam = rot * p + trans with left-to-right sums.
struct Cam {
  float m[9];
  float t[3];
  float fx, fy, cx, cy;
  int width, height;
  float near_plane, far_plane;
};
static_assert(sizeof(Cam) == 80, "gss_camera layout");

struct f3 {
  float x, y, z;
};

__device__ __forceinline__ f3 to_camera(const Cam& c, float x, float y, float z) {
  f3 r;
  r.x = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(c.m[0], x), __fmul_rn(c.m[1], y)), __fmul_rn(c.m[2], z)), c.t[0]);
  r.y = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(c.m[3], x), __fmul_rn(c.m[4], y)), __fmul_rn(c.m[5], z)), c.t[1]);
  r.z = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(c.m[6], x), __fmul_rn(c.m[7], y)), __fmul_rn(c.m[8], z)), c.t[2]);
  return r;
}

__device__ __forceinline__ float cam_z(const Cam& c, float x, float y, float z) {
  return __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(c.m[6], x), __fmul_rn(c.m[7], y)), __fmul_rn(c.m[8], z)), c.t[2]);
}

__device__ __forceinline__ f3 cam_position(const Cam& c) {
  const float tx = -c.t[0], ty = -c.t[1], tz = -c.t[2];
  return f3{c.m[0] * tx + c.m[3] * ty + c.m[6] * tz, c.m[1] * tx + c.m[4] * ty + c.m[7] * tz,
            c.m[2] * tx + c.m[5] * ty + c.m[8] * tz};
}

// quat_to_rot (vecmath.hpp:61-74).
__device__ __forceinline__ void quat_to_rot(float w, float x, float y, float z, float R[9]) {
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

// ---------------------------------------------------------------------------
// project_geo (render.hpp:90-148), given the camera-space mean already computed.
struct Proj {
  float mx, my, a, b, c, radius;
};

__device__ __forceinline__ void cov2d(const Cam& cam, const float* g, const f3& t, float iz, float lp, Proj& o,
                                      float* q_unit_out = nullptr, float* es_out = nullptr) {
  const float qw = g[6], qx = g[7], qy = g[8], qz = g[9];
  const float qn = sqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
  const float qinv = qn > 1e-12f ? 1.0f / qn : 0.0f;
  const float q0 = qw * qinv, q1 = qx * qinv, q2 = qy * qinv, q3 = qz * qinv;
  float R[9];
  quat_to_rot(q0, q1, q2, q3, R);
  const float es0 = gss_expf(g[3]), es1 = gss_expf(g[4]), es2 = gss_expf(g[5]);
  float B[9], S[9];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    B[i * 3 + 0] = R[i * 3 + 0] * es0;
    B[i * 3 + 1] = R[i * 3 + 1] * es1;
    B[i * 3 + 2] = R[i * 3 + 2] * es2;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      S[i * 3 + j] = B[i * 3] * B[j * 3] + B[i * 3 + 1] * B[j * 3 + 1] + B[i * 3 + 2] * B[j * 3 + 2];
  const float j00 = cam.fx * iz, j02 = -cam.fx * t.x * iz * iz;
  const float j11 = cam.fy * iz, j12 = -cam.fy * t.y * iz * iz;
  const float* W = cam.m;
  const float m00 = j00 * W[0] + j02 * W[6], m01 = j00 * W[1] + j02 * W[7], m02 = j00 * W[2] + j02 * W[8];
  const float m10 = j11 * W[3] + j12 * W[6], m11 = j11 * W[4] + j12 * W[7], m12 = j11 * W[5] + j12 * W[8];
  float v0[3], v1[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    v0[i] = S[i * 3] * m00 + S[i * 3 + 1] * m01 + S[i * 3 + 2] * m02;
    v1[i] = S[i * 3] * m10 + S[i * 3 + 1] * m11 + S[i * 3 + 2] * m12;
  }
  o.a = (m00 * v0[0] + m01 * v0[1] + m02 * v0[2]) + lp;
  o.b = m00 * v1[0] + m01 * v1[1] + m02 * v1[2];
  o.c = (m10 * v1[0] + m11 * v1[1] + m12 * v1[2]) + lp;
  const float mid = (o.a + o.c) / 2.0f;
  const float half = (o.a - o.c) / 2.0f;
  const float lmax = mid + sqrtf(half * half + o.b * o.b);
  o.radius = 3.0f * sqrtf(max0(lmax));
  if (q_unit_out) {
    q_unit_out[0] = q0; q_unit_out[1] = q1; q_unit_out[2] = q2; q_unit_out[3] = q3;
  }
  if (es_out) {
    es_out[0] = es0; es_out[1] = es1; es_out[2] = es2;
  }
}

// Full project_geo: returns false when invalid (t.z <= 1e-9 or NaN).
__device__ __forceinline__ bool project_geo(const Cam& cam, const float* g, float lp, Proj& o, f3& t) {
  t = to_camera(cam, g[0], g[1], g[2]);
  if (!(t.z > 1e-9f)) return false;
  const float iz = 1.0f / t.z;
  o.mx = cam.fx * t.x * iz + cam.cx;
  o.my = cam.fy * t.y * iz + cam.cy;
  cov2d(cam, g, t, iz, lp, o);
  return true;
}

// ---------------------------------------------------------------------------
// Spherical harmonics (sh.hpp:24-73), float with the reference's constant casts.
#define GSS_SH_C0 0.28209479177387814
#define GSS_SH_C1 0.4886025119029199

__device__ __forceinline__ void sh_basis(float x, float y, float z, int deg, float* o) {
  o[0] = (float)GSS_SH_C0;
  if (deg < 1) return;
  o[1] = (float)(-GSS_SH_C1) * y;
  o[2] = (float)GSS_SH_C1 * z;
  o[3] = (float)(-GSS_SH_C1) * x;
  if (deg < 2) return;
  const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  o[4] = (float)1.0925484305920792 * xy;
  o[5] = (float)-1.0925484305920792 * yz;
  o[6] = (float)0.31539156525252005 * (2.0f * zz - xx - yy);
  o[7] = (float)-1.0925484305920792 * xz;
  o[8] = (float)0.5462742152960396 * (xx - yy);
  if (deg < 3) return;
  o[9] = (float)-0.5900435899266435 * y * (3.0f * xx - yy);
  o[10] = (float)2.890611442640554 * xy * z;
  o[11] = (float)-0.4570457994644658 * y * (4.0f * zz - xx - yy);
  o[12] = (float)0.3731763325901154 * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
  o[13] = (float)-0.4570457994644658 * x * (4.0f * zz - xx - yy);
  o[14] = (float)1.445305721320277 * z * (xx - yy);
  o[15] = (float)-0.5900435899266435 * x * (xx - 3.0f * yy);
}

__device__ __forceinline__ void sh_basis_grad(float x, float y, float z, int deg, f3* o) {
  o[0] = f3{0.0f, 0.0f, 0.0f};
  if (deg < 1) return;
  o[1] = f3{0.0f, (float)(-GSS_SH_C1), 0.0f};
  o[2] = f3{0.0f, 0.0f, (float)GSS_SH_C1};
  o[3] = f3{(float)(-GSS_SH_C1), 0.0f, 0.0f};
  if (deg < 2) return;
  const float c20 = (float)1.0925484305920792, c21 = (float)-1.0925484305920792, c22 = (float)0.31539156525252005,
              c23 = (float)-1.0925484305920792, c24 = (float)0.5462742152960396;
  o[4] = f3{c20 * y, c20 * x, 0.0f};
  o[5] = f3{0.0f, c21 * z, c21 * y};
  o[6] = f3{c22 * -2.0f * x, c22 * -2.0f * y, c22 * 4.0f * z};
  o[7] = f3{c23 * z, 0.0f, c23 * x};
  o[8] = f3{c24 * 2.0f * x, c24 * -2.0f * y, 0.0f};
  if (deg < 3) return;
  const float c30 = (float)-0.5900435899266435, c31 = (float)2.890611442640554, c32 = (float)-0.4570457994644658,
              c33 = (float)0.3731763325901154, c34 = (float)-0.4570457994644658, c35 = (float)1.445305721320277,
              c36 = (float)-0.5900435899266435;
  o[9] = f3{c30 * 6.0f * x * y, c30 * (3.0f * x * x - 3.0f * y * y), 0.0f};
  o[10] = f3{c31 * y * z, c31 * x * z, c31 * x * y};
  o[11] = f3{c32 * -2.0f * x * y, c32 * (4.0f * z * z - x * x - 3.0f * y * y), c32 * 8.0f * y * z};
  o[12] = f3{c33 * -6.0f * x * z, c33 * -6.0f * y * z, c33 * (6.0f * z * z - 3.0f * x * x - 3.0f * y * y)};
  o[13] = f3{c34 * (4.0f * z * z - 3.0f * x * x - y * y), c34 * -2.0f * x * y, c34 * 8.0f * x * z};
  o[14] = f3{c35 * 2.0f * x * z, c35 * -2.0f * y * z, c35 * (x * x - y * y)};
  o[15] = f3{c36 * (3.0f * x * x - 3.0f * y * y), c36 * -6.0f * x * y, 0.0f};
}

__device__ __forceinline__ float clamp01(float v) { return v < 0.0f ? 0.0f : (1.0f < v ? 1.0f : v); }

}  // namespace gssd
