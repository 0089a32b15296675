// Densification on the device: plan_densify (trainer.hpp:166-213) and the
// engine's apply_densify (engine.hpp:116-163) for a population resident in HBM.
//
//   plan   one thread per Gaussian classifies prune / keep / clone / split from the restored
//          snapshot row and the accumulated screen-space gradient statistics. The reference's
//          double-precision libm decisions (sigmoid(opacity) < prune, exp(max log-scale) <= clone
//          limit) are monotone in one float input, so the host turns each into an exact float
//          threshold by bisection with the reference's own formula (glibc), and the device compares
//          floats: identical decisions. Survivors and children are stream-compacted in id order.
//   split  children need the reference Rng (splitmix64 + Box-Muller with glibc log/sqrt/sin/cos):
//          split s consumes draws 6s..6s+5 of the event's stream (counter-based: jump ahead), so
//          the host computes exactly those for the (few) split parents, gathered from the device.
//   apply  new arenas = survivors' stored rows, optimizer state and counters (gathered) + children
//          with zero state; steps carry over; densification statistics reset.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "gss_math.cuh"

namespace gssd {
namespace {

constexpr int kRow = 59;

// Reference Rng (rng.hpp:11-51) with jump-ahead: draw k (0-based) of a stream seeded `seed`.
inline uint64_t splitmix_at(uint64_t seed, uint64_t k) {
  uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline double uniform_at(uint64_t seed, uint64_t k) { return double(splitmix_at(seed, k) >> 11) * 0x1.0p-53; }
// Box-Muller pair p of the stream (rng.hpp:33-46): (r cos a, r sin a) from uniforms 2p, 2p + 1.
inline void normal_pair(uint64_t seed, uint64_t p, double& n0, double& n1) {
  double u1 = uniform_at(seed, 2 * p);
  const double u2 = uniform_at(seed, 2 * p + 1);
  if (u1 < 1e-300) u1 = 1e-300;
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double a = 6.283185307179586477 * u2;
  n1 = r * std::sin(a);
  n0 = r * std::cos(a);
}

// Monotone order of non-NaN floats as integers (-0 and +0 share a key).
inline int64_t fkey(float f) {
  int32_t b;
  std::memcpy(&b, &f, 4);
  return b >= 0 ? (int64_t)b : -(int64_t)(b & 0x7fffffff);
}
inline float funkey(int64_t k) {
  const uint32_t b = k >= 0 ? (uint32_t)k : ((uint32_t)(-k) | 0x80000000u);
  float f;
  std::memcpy(&f, &b, 4);
  return f;
}
// Smallest float x (-inf..+inf) with pred(x), for pred false..false true..true; NaN if none.
template <class P> float first_true(P pred) {
  int64_t lo = fkey(-INFINITY), hi = fkey(INFINITY);
  if (pred(-INFINITY)) return -INFINITY;
  if (!pred(INFINITY)) return NAN;
  while (hi - lo > 1) {  // pred(lo) false, pred(hi) true
    const int64_t mid = lo + (hi - lo) / 2;
    if (pred(funkey(mid))) hi = mid; else lo = mid;
  }
  return funkey(hi);
}

// prune iff x < result: the smallest float x with 1/(1+exp(-x)) >= t (trainer.hpp:177-178).
float prune_threshold(double t) {
  const float x = first_true([&](float v) { return 1.0 / (1.0 + std::exp(-double(v))) >= t; });
  return std::isnan(x) ? INFINITY : x;  // no x reaches t: everything is pruned
}

// clone iff m <= result: the largest float m with exp(m) <= limit (trainer.hpp:181-190); NaN when
// there is none (never clone).
float clone_threshold(double limit) {
  const float x = first_true([&](float v) { return !(std::exp(double(v)) <= limit); });
  if (std::isnan(x)) return INFINITY;  // every m satisfies exp(m) <= limit
  if (x == -INFINITY) return NAN;
  return funkey(fkey(x) - 1);
}

// 0 prune, 1 keep, 2 clone (keep + 1 child), 3 split (2 children).
__global__ void classify_kernel(const float* rows, int64_t n, const double* norm, const int32_t* cnt, float x_prune,
                                float s_clone, double grad_thr, uint8_t* code, int32_t* n_child, int32_t* keep,
                                int32_t* split) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* r = rows + i * kRow;
  uint8_t c;
  if (r[10] < x_prune) {
    c = 0;
  } else {
    const double avg = cnt[i] > 0 ? norm[i] / cnt[i] : 0.0;
    if (!(avg > grad_thr)) {
      c = 1;
    } else {
      float m = r[3];  // std::max({s0, s1, s2}) (initializer_list: keeps the first of equals)
      if (m < r[4]) m = r[4];
      if (m < r[5]) m = r[5];
      c = (m <= s_clone) ? 2 : 3;
    }
  }
  code[i] = c;
  n_child[i] = c == 2 ? 1 : (c == 3 ? 2 : 0);
  keep[i] = (c == 1 || c == 2) ? 1 : 0;
  split[i] = c == 3 ? 1 : 0;
}

struct Flagged {
  const int32_t* f;
  __host__ __device__ bool operator()(int32_t i) const { return f[i] != 0; }
};

__global__ void clone_children_kernel(const float* rows, int64_t n, const uint8_t* code, const int32_t* child_off,
                                      float* children) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || code[i] != 2) return;
  const float* src = rows + i * kRow;
  float* dst = children + (int64_t)child_off[i] * kRow;
  for (int c = 0; c < kRow; ++c) dst[c] = src[c];
}

__global__ void gather_rows_kernel(const float* rows, const int32_t* ids, int64_t k, float* out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= k * kRow) return;
  const int64_t j = e / kRow;
  out[e] = rows[(int64_t)ids[j] * kRow + (e - j * kRow)];
}

__global__ void scatter_split_children_kernel(const float* host_children, const int32_t* split_ids, int64_t s,
                                              const int32_t* child_off, float* children) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= s * 2 * kRow) return;
  const int64_t j = e / (2 * kRow);
  const int64_t rem = e - j * 2 * kRow;
  children[(int64_t)child_off[split_ids[j]] * kRow + rem] = host_children[e];
}

}  // namespace

// The reference's split children (trainer.hpp:192-208) of split parent rows (restored, k x 59),
// split s being the s-th split in id order of the event's Rng stream `seed`.
void split_children_host(const float* parents, int64_t k, uint64_t seed, double divisor, float* out) {
  const float ldiv = float(std::log(divisor));
  for (int64_t s = 0; s < k; ++s) {
    const float* p = parents + s * kRow;
    // unit_quat (trainer.hpp:152-156) and quat_to_rot (vecmath.hpp:61-74), float arithmetic
    float qw = p[6], qx = p[7], qy = p[8], qz = p[9];
    const float qn = std::sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    if (qn < 1e-12f) {
      qw = 1.0f; qx = qy = qz = 0.0f;
    } else {
      qw = qw / qn; qx = qx / qn; qy = qy / qn; qz = qz / qn;
    }
    float R[3][3];
    R[0][0] = 1.0f - 2.0f * (qy * qy + qz * qz);
    R[0][1] = 2.0f * (qx * qy - qw * qz);
    R[0][2] = 2.0f * (qx * qz + qw * qy);
    R[1][0] = 2.0f * (qx * qy + qw * qz);
    R[1][1] = 1.0f - 2.0f * (qx * qx + qz * qz);
    R[1][2] = 2.0f * (qy * qz - qw * qx);
    R[2][0] = 2.0f * (qx * qz - qw * qy);
    R[2][1] = 2.0f * (qy * qz + qw * qx);
    R[2][2] = 1.0f - 2.0f * (qx * qx + qy * qy);
    double nv[6];
    for (int pr = 0; pr < 3; ++pr) normal_pair(seed, (uint64_t)s * 3 + pr, nv[2 * pr], nv[2 * pr + 1]);
    for (int c = 0; c < 2; ++c) {
      float* o = out + (s * 2 + c) * kRow;
      std::memcpy(o, p, kRow * sizeof(float));
      const float ex = float(nv[3 * c + 0] * std::exp(double(p[3])));
      const float ey = float(nv[3 * c + 1] * std::exp(double(p[4])));
      const float ez = float(nv[3 * c + 2] * std::exp(double(p[5])));
      const float ox = R[0][0] * ex + R[0][1] * ey + R[0][2] * ez;
      const float oy = R[1][0] * ex + R[1][1] * ey + R[1][2] * ez;
      const float oz = R[2][0] * ex + R[2][1] * ey + R[2][2] * ez;
      o[0] += ox;
      o[1] += oy;
      o[2] += oz;
      for (int a = 0; a < 3; ++a) o[3 + a] -= ldiv;
    }
  }
}

// plan_densify on device rows (restored snapshot, n x 59). survivors (cap n) and children
// (cap 2n x 59) are device buffers; counts[0..4] = survivors, children, clones, splits, pruned.
void plan_densify(const float* rows, int64_t n, const double* norm, const int32_t* cnt,
                  const gss_densify_config* dc, double extent, uint64_t seed, int32_t* survivors, float* children,
                  int64_t* counts, cudaStream_t st) {
  require(dc && counts && n >= 0 && n <= INT32_MAX, "densify: bad arguments");
  require(dc->grad_threshold > 0 && dc->opacity_prune > 0 && dc->split_scale_divisor > 0 && dc->percent_dense > 0,
          "densify: thresholds must be positive");
  for (int i = 0; i < 5; ++i) counts[i] = 0;
  if (n == 0) return;
  require(rows && norm && cnt && survivors && children, "densify: null buffer");
  const float x_prune = prune_threshold(dc->opacity_prune);
  const float s_clone = clone_threshold(dc->percent_dense * extent);
  uint8_t* code = nullptr;
  int32_t *nchild = nullptr, *keep = nullptr, *split = nullptr, *coff = nullptr, *split_ids = nullptr;
  int64_t* dcount = nullptr;
  GSS_CUDA(cudaMallocAsync((void**)&code, n, st));
  GSS_CUDA(cudaMallocAsync((void**)&nchild, (n + 1) * 4, st));
  GSS_CUDA(cudaMallocAsync((void**)&keep, n * 4, st));
  GSS_CUDA(cudaMallocAsync((void**)&split, n * 4, st));
  GSS_CUDA(cudaMallocAsync((void**)&coff, (n + 1) * 4, st));
  GSS_CUDA(cudaMallocAsync((void**)&split_ids, n * 4, st));
  GSS_CUDA(cudaMallocAsync((void**)&dcount, 2 * 8, st));
  classify_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(rows, n, norm, cnt, x_prune, s_clone,
                                                              dc->grad_threshold, code, nchild, keep, split);
  GSS_LAUNCHED();
  GSS_CUDA(cudaMemsetAsync(nchild + n, 0, 4, st));
  thrust::counting_iterator<int32_t> it(0);
  size_t b1 = 0, b2 = 0, b3 = 0;
  GSS_CUDA(cub::DeviceSelect::If(nullptr, b1, it, survivors, dcount, (int)n, Flagged{keep}, st));
  GSS_CUDA(cub::DeviceSelect::If(nullptr, b2, it, split_ids, dcount + 1, (int)n, Flagged{split}, st));
  GSS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b3, nchild, coff, (int)(n + 1), st));
  void* tmp = nullptr;
  GSS_CUDA(cudaMallocAsync(&tmp, std::max(b1, std::max(b2, b3)), st));
  GSS_CUDA(cub::DeviceSelect::If(tmp, b1, it, survivors, dcount, (int)n, Flagged{keep}, st));
  GSS_CUDA(cub::DeviceSelect::If(tmp, b2, it, split_ids, dcount + 1, (int)n, Flagged{split}, st));
  GSS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, b3, nchild, coff, (int)(n + 1), st));
  count_launch();
  int64_t hc[2];
  int32_t nch = 0;
  GSS_CUDA(cudaMemcpyAsync(hc, dcount, 16, cudaMemcpyDeviceToHost, st));
  GSS_CUDA(cudaMemcpyAsync(&nch, coff + n, 4, cudaMemcpyDeviceToHost, st));
  GSS_CUDA(cudaStreamSynchronize(st));
  const int64_t nsurv = hc[0], nsplit = hc[1];
  clone_children_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(rows, n, code, coff, children);
  GSS_LAUNCHED();
  if (nsplit > 0) {
    float* parents_dev = nullptr;
    GSS_CUDA(cudaMallocAsync((void**)&parents_dev, (size_t)nsplit * kRow * 4, st));
    gather_rows_kernel<<<(unsigned)ceil_div(nsplit * kRow, 256), 256, 0, st>>>(rows, split_ids, nsplit, parents_dev);
    GSS_LAUNCHED();
    std::vector<float> parents((size_t)nsplit * kRow), kids((size_t)nsplit * 2 * kRow);
    GSS_CUDA(cudaMemcpyAsync(parents.data(), parents_dev, parents.size() * 4, cudaMemcpyDeviceToHost, st));
    GSS_CUDA(cudaStreamSynchronize(st));
    split_children_host(parents.data(), nsplit, seed, dc->split_scale_divisor, kids.data());
    float* kids_dev = parents_dev;  // reuse: 2x the size needed
    GSS_CUDA(cudaFreeAsync(parents_dev, st));
    GSS_CUDA(cudaMallocAsync((void**)&kids_dev, kids.size() * 4, st));
    GSS_CUDA(cudaMemcpyAsync(kids_dev, kids.data(), kids.size() * 4, cudaMemcpyHostToDevice, st));
    scatter_split_children_kernel<<<(unsigned)ceil_div(nsplit * 2 * kRow, 256), 256, 0, st>>>(kids_dev, split_ids,
                                                                                              nsplit, coff, children);
    GSS_LAUNCHED();
    GSS_CUDA(cudaStreamSynchronize(st));  // kids (host vector) must outlive the copy
    GSS_CUDA(cudaFreeAsync(kids_dev, st));
  }
  counts[0] = nsurv;
  counts[1] = nch;
  counts[2] = nch - 2 * nsplit;
  counts[3] = nsplit;
  counts[4] = n - nsurv - nsplit;
  for (void* p : {(void*)code, (void*)nchild, (void*)keep, (void*)split, (void*)coff, (void*)split_ids,
                  (void*)dcount, tmp})
    GSS_CUDA(cudaFreeAsync(p, st));
}

}  // namespace gssd

// ---- init_gaussians (scene.hpp:146-195) ------------------------------------------
// Exact O(M^2) kNN on the device: thread per point, candidate points streamed through SMEM tiles,
// distances in fp64 exactly as the reference (double differences, IEEE sqrt, no contraction); the k
// smallest are kept sorted (ties keep the earlier value, as the reference's insertion sort) and
// summed ascending. mean_dist comes back to the host, whose libm takes the log (bit-identical rows).
namespace gssd {
namespace {
constexpr int kKnnMax = 16;
constexpr int kKnnTile = 256;

__global__ void knn_mean_kernel(const float* pos, int m, int k, double min_dist, double* mean_out) {
  __shared__ float tile[kKnnTile * 3];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double best[kKnnMax];
  int filled = 0;
  const double xi = i < m ? (double)pos[i * 3] : 0.0, yi = i < m ? (double)pos[i * 3 + 1] : 0.0,
               zi = i < m ? (double)pos[i * 3 + 2] : 0.0;
  for (int t0 = 0; t0 < m; t0 += kKnnTile) {
    const int nt = min(kKnnTile, m - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < nt * 3; e += blockDim.x) tile[e] = pos[t0 * 3 + e];
    __syncthreads();
    if (i >= m) continue;
    for (int jj = 0; jj < nt; ++jj) {
      const int j = t0 + jj;
      if (j == i) continue;
      const double dx = (double)tile[jj * 3] - xi;
      const double dy = (double)tile[jj * 3 + 1] - yi;
      const double dz = (double)tile[jj * 3 + 2] - zi;
      const double d = sqrt(dx * dx + dy * dy + dz * dz);
      if (filled < k) {
        int b = filled++;
        best[b] = d;
        for (; b > 0 && best[b] < best[b - 1]; --b) {
          const double tmp = best[b];
          best[b] = best[b - 1];
          best[b - 1] = tmp;
        }
      } else if (d < best[k - 1]) {
        int b = k - 1;
        best[b] = d;
        for (; b > 0 && best[b] < best[b - 1]; --b) {
          const double tmp = best[b];
          best[b] = best[b - 1];
          best[b - 1] = tmp;
        }
      }
    }
  }
  if (i >= m) return;
  double mean_dist = min_dist;
  if (m > 1) {
    double s = 0.0;
    for (int b = 0; b < filled; ++b) s += best[b];
    mean_dist = filled > 0 ? s / filled : min_dist;
    if (mean_dist < min_dist) mean_dist = min_dist;
  }
  mean_out[i] = mean_dist;
}
}  // namespace

// rows_out (host, m x 59): init_gaussians of the point cloud positions (host, m x 3) / colors
// (host m x 3 or null).
void init_gaussians(const float* positions, const float* colors, int m, int knn, double min_knn_dist,
                    double init_opacity, float* rows_out) {
  require(m >= 1, "init_gaussians: point cloud is empty");
  require(positions && rows_out, "init_gaussians: null argument");
  const int k = std::max(1, std::min(knn, m - 1));
  require(k <= kKnnMax, "init_gaussians: knn must be <= 16");
  float* pos_dev = nullptr;
  double* mean_dev = nullptr;
  GSS_CUDA(cudaMalloc(&pos_dev, (size_t)m * 12));
  GSS_CUDA(cudaMalloc(&mean_dev, (size_t)m * 8));
  GSS_CUDA(cudaMemcpy(pos_dev, positions, (size_t)m * 12, cudaMemcpyHostToDevice));
  knn_mean_kernel<<<(unsigned)ceil_div(m, 128), 128>>>(pos_dev, m, k, min_knn_dist, mean_dev);
  GSS_LAUNCHED();
  std::vector<double> mean((size_t)m);
  GSS_CUDA(cudaMemcpy(mean.data(), mean_dev, (size_t)m * 8, cudaMemcpyDeviceToHost));
  cudaFree(pos_dev);
  cudaFree(mean_dev);
  const double kShC0 = 0.28209479177387814;
  const float op = float(std::log(init_opacity) - std::log(1.0 - init_opacity));  // logit (scene.hpp:141)
  for (int i = 0; i < m; ++i) {
    float* r = rows_out + (size_t)i * kRow;
    std::memset(r, 0, kRow * sizeof(float));
    const float log_s = float(std::log(mean[i]));
    for (int a = 0; a < 3; ++a) {
      r[a] = positions[i * 3 + a];
      r[3 + a] = log_s;
    }
    r[6] = 1.0f;
    r[10] = op;
    for (int c = 0; c < 3; ++c) {
      const double col = colors ? double(colors[i * 3 + c]) : 0.5;
      r[11 + c] = float((col - 0.5) / kShC0);
    }
  }
}

}  // namespace gssd
