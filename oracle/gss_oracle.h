/* TEST INFRASTRUCTURE ONLY — the CPU restatement ("oracle") of the GS-Scale hot path.
 *
 * Plain C11, single-threaded, no FP contraction (-ffp-contract=off), every operation in the
 * reference's order so results are bit-identical to /root/reference/proj/include/gss/*.hpp
 * instantiated for float at workers=1 (pinned by tests/test_oracle.py against oracle/_ref and
 * tests/golden/). Each function cites the reference file:line it restates.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this library;
 * the product (paper_2509_15645_b200/) never links or calls it.
 */
#ifndef GSS_ORACLE_H
#define GSS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Camera<float> layout (scene.hpp:77-84): 80 bytes. */
typedef struct {
  float rot[9];
  float trans[3];
  float fx, fy, cx, cy;
  int32_t width, height;
  float near_plane, far_plane;
} orc_camera;

typedef struct {
  float x0, x1, y0, y1;
} orc_viewport;

/* glibc 2.39 expf (FMA ifunc variant) restated; equals host expf on all 2^32 inputs. */
float orc_expf(float x);

/* project_geo (render.hpp:90-148). out[8]: mx, my, a, b, c, depth, radius, valid. */
void orc_project_geo(const float* g, const orc_camera* cam, float low_pass, float* out);

/* cull_keep + frustum_cull (render.hpp:243-260). Returns count; ids ascending. */
int64_t orc_frustum_cull(const float* geo, int64_t n, int64_t stride, const orc_camera* cam,
                         const orc_viewport* vp, float low_pass, int32_t* out_ids);

/* build_group_luts (adam.hpp:67-97). scalars: one_minus_b1, one_minus_b2, bias_correction, step_size, eps. */
void orc_build_luts(double lr, double b1, double b2, double eps, int64_t t, int max_delay, float* param,
                    float* mom, float* var, float* pow_b1, float* pow_b2, float* scalars);

/* Arena (adam.hpp:119-159): row-major w/m/v [n][dim], uint8 counter[n]; groups are contiguous columns. */
typedef struct {
  int64_t n;
  int dim;
  int ngroups;
  int col0[8], gdim[8];
  double lr[8];
  double b1, b2, eps;
  int defer_max;
  int64_t step;
  float *w, *m, *v;
  uint8_t* counter;
} orc_arena;

/* adam_step_dense (adam.hpp:198-207); grads: n x dim or NULL. */
void orc_adam_step_dense(orc_arena* a, const float* grads);
/* deferred_update (adam.hpp:211-238). Returns touched count, or -3 on unsorted/out-of-range ids. */
int64_t orc_deferred_update(orc_arena* a, int64_t nids, const int32_t* ids, const float* rows, int64_t stride,
                            int col0, int32_t* touched_out);
/* restore_view (adam.hpp:252-289); pending may be absent (has_pending = 0). */
void orc_restore_view(const orc_arena* a, int64_t nids, const int32_t* ids, int has_pending, int64_t npend,
                      const int32_t* pids, const float* prows, int64_t pstride, int pcol0, float* out);
/* flush_deferred (adam.hpp:293-313). */
void orc_flush_deferred(orc_arena* a);

/* Rasterizer forward + L1 loss + backward (render.hpp:297-640), workers = 1 order.
 * nongeo: compact (slot-indexed V x 49) when nongeo_compact != 0, else id-indexed.
 * gt_full: full camera image (H x W x 3) or NULL (no loss); d_img_in overrides the loss gradient.
 * Outputs sized to the viewport pixel window (meta[0..3] = px0, py0, pw, ph; meta[4] = contributions).
 * Returns 0 or 2 (bad argument). */
int orc_render(int64_t n_ids, const int32_t* ids, const float* geo, int64_t geo_stride, const float* nongeo,
               int nongeo_compact, int sh_degree, const float* bg, const orc_camera* cam, const orc_viewport* vp,
               const float* gt_full, int64_t normalizer, const float* d_img_in, float* out_image,
               float* out_final_T, int32_t* out_len, float* out_loss, float* out_d_img, float* out_grad_rows,
               float* out_mean2d, int64_t* meta);

#ifdef __cplusplus
}
#endif
#endif
