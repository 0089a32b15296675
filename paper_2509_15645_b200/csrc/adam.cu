// Deferred sparse Adam, dense Adam, restore/forwarding gather and flush on the device
// (reference: adam.hpp:67-313). All optimizer arithmetic is the reference's deferred_scalar /
// restore_scalar in fp32 without contraction, so post-Adam parameters are bit-identical to the
// CPU reference for identical gradients.
//
// Layout: an Arena is row-major w, m, v [n][dim] fp32 plus a uint8 defer counter per row.
// The update kernels stream the arena in 1024-row blocks: a block finds its slice of the sorted
// gradient ids by binary search, builds a row->grad-slot map in SMEM, advances/resets the
// counters (1 B/row in, 1 B/row out), compacts the touched rows and then walks the flattened
// (touched row, column) space so that every warp reads/writes contiguous 196 B row segments of
// w, m, v and the gradient. Untouched rows cost only their counter byte — the paper's deferred
// update (§4.3): traffic = 4*dim*(6 + has_grad)*touched + 2*n bytes.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <atomic>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace gssd {

constexpr int kMaxGroups = 8;
constexpr int kMaxDim = 128;

template <int K> struct LutArgs {
  int ngroups;
  int entries;  // defer_max + 1
  float param[kMaxGroups][K];
  float a1[kMaxGroups][K];  // mom (update/restore) or pow_b1 (flush)
  float a2[kMaxGroups][K];  // var (update/restore) or pow_b2 (flush)
  float sc[kMaxGroups][5];  // one_minus_b1, one_minus_b2, bias_correction, step_size, eps
  uint8_t col_group[kMaxDim];
};

// build_group_luts (adam.hpp:67-97) — fp64 host arithmetic in the reference's order.
void build_group_luts(double lr, double b1, double b2, double eps, int64_t t, int max_delay, float* param,
                      float* mom, float* var, float* pow_b1, float* pow_b2, float* scalars) {
  const int usable = (int)std::min<int64_t>(max_delay, t - 1);
  for (int i = 0; i <= max_delay; ++i) param[i] = 0.0f;
  const double scale = b1 / std::sqrt(b2);
  double acc = 0.0;
  for (int i = 1; i <= usable; ++i) {
    acc = scale * acc +
          (lr * b1) / (std::sqrt(b2 / (1.0 - std::pow(b2, double(t - i)))) * (1.0 - std::pow(b1, double(t - i))));
    param[i] = float(acc);
  }
  for (int i = usable + 1; i <= max_delay; ++i) param[i] = float(acc);
  for (int i = 0; i <= max_delay; ++i) {
    if (mom) mom[i] = float(std::pow(b1, double(i + 1)));
    if (var) var[i] = float(std::pow(b2, double(i + 1)));
    if (pow_b1) pow_b1[i] = float(std::pow(b1, double(i)));
    if (pow_b2) pow_b2[i] = float(std::pow(b2, double(i)));
  }
  scalars[0] = float(1.0 - b1);
  scalars[1] = float(1.0 - b2);
  scalars[2] = float(std::sqrt(1.0 - std::pow(b2, double(t))));
  scalars[3] = float(lr / (1.0 - std::pow(b1, double(t))));
  scalars[4] = float(eps);
}

namespace {

constexpr int kRowsPerBlock = 1024;
constexpr int kUpdThreads = 256;

template <int K> void fill_luts(const gss_arena& a, int64_t t, bool flush, LutArgs<K>& L) {
  L.ngroups = a.ngroups;
  L.entries = a.defer_max + 1;
  std::vector<float> p(K), m(K), v(K), b1(K), b2(K);
  for (int g = 0; g < a.ngroups; ++g) {
    const gss_group& G = a.groups[g];
    build_group_luts(G.lr, G.beta1, G.beta2, G.eps, t, a.defer_max, p.data(), m.data(), v.data(), b1.data(),
                     b2.data(), L.sc[g]);
    for (int i = 0; i < L.entries; ++i) {
      L.param[g][i] = p[i];
      L.a1[g][i] = flush ? b1[i] : m[i];
      L.a2[g][i] = flush ? b2[i] : v[i];
    }
    for (int c = G.col0; c < G.col0 + G.dim; ++c) L.col_group[c] = (uint8_t)g;
  }
}

struct ArenaDev {
  float* w;
  float* m;
  float* v;
  uint8_t* counter;
  int64_t n;
  int dim;
  int defer_max;
  uint32_t div_magic;  // ceil(2^32 / dim)
  int64_t stride;      // floats between rows of w, m, v (>= dim)
  int positional;      // 1: a staging copy — row of list entry k is at k * stride (host-tier passes)
};

struct GradsDev {
  const int32_t* ids;
  int64_t count;
  const int64_t* count_dev;
  const float* rows;
  int64_t stride;
  int col0;
  int vec4;  // rows 16-byte aligned with whole float4 units up to the padded dim: one 16-byte load per unit
};

// gradient unit (4 columns from c0) of grads row `sl`: zero for no row or columns past dim
__device__ __forceinline__ void grad_unit(const GradsDev& g, int64_t sl, int c0, int dim, bool ok, float out[4]) {
  const float* row = g.rows + sl * g.stride + g.col0 + c0;
  if (g.vec4) {
    const float4 v = (ok && sl >= 0) ? *reinterpret_cast<const float4*>(row) : make_float4(0.f, 0.f, 0.f, 0.f);
    out[0] = v.x;
    out[1] = c0 + 1 < dim ? v.y : 0.0f;
    out[2] = c0 + 2 < dim ? v.z : 0.0f;
    out[3] = c0 + 3 < dim ? v.w : 0.0f;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = (ok && sl >= 0 && c0 + i < dim) ? row[i] : 0.0f;
  }
}

__device__ __forceinline__ int64_t grads_count(const GradsDev& g) { return g.count_dev ? *g.count_dev : g.count; }

__device__ __forceinline__ int64_t lower_bound_ids(const int32_t* ids, int64_t n, int64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)ids[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// IEEE round-to-nearest n / d. A zero numerator (most elements of a sparse step: delay-0 rows
// have w_scale = 0, untouched rows have m = v = 0) sends CUDA's division into its slow path;
// its exact result is a signed zero (sign = sign(n) ^ sign(d)) for any nonzero, non-NaN d.
__device__ __forceinline__ float div_rn(float n, float d) {
  if (n == 0.0f && d == d && d != 0.0f) return __int_as_float((__float_as_int(n) ^ __float_as_int(d)) & 0x80000000);
  return __fdiv_rn(n, d);
}

// IEEE sqrtf with +-0 answered without CUDA's out-of-range slow path (sqrt(+-0) = +-0): rows never
// touched have v = 0 exactly, and one such lane would send its whole warp through the subroutine.
__device__ __forceinline__ float sqrt_rn(float x) {
  const float s = sqrtf(x == 0.0f ? 1.0f : x);
  return x == 0.0f ? x : s;
}

// deferred_scalar (adam.hpp:102-110)
__device__ __forceinline__ void deferred_scalar(float& w, float& m, float& v, float g, float ws, float ms, float vs,
                                                const float* sc) {
  const float m_new = ms * m + sc[0] * g;
  const float v_new = vs * v + sc[1] * g * g;
  w -= div_rn(ws * m, sqrt_rn(v) + sc[4]);
  const float denom = div_rn(sqrt_rn(v_new), sc[2]) + sc[4];
  w = w - div_rn(sc[3] * m_new, denom);
  m = m_new;
  v = v_new;
}

template <int K> struct SmemLuts {
  float param[kMaxGroups][K];
  float a1[kMaxGroups][K];
  float a2[kMaxGroups][K];
  float sc[kMaxGroups][5];
  uint8_t col_group[kMaxDim];
};

template <int K> __device__ void load_luts(SmemLuts<K>& s, const LutArgs<K>& L, int dim) {
  for (int i = threadIdx.x; i < L.ngroups * K; i += blockDim.x) {
    const int g = i / K, e = i - g * K;
    s.param[g][e] = L.param[g][e];
    s.a1[g][e] = L.a1[g][e];
    s.a2[g][e] = L.a2[g][e];
  }
  for (int i = threadIdx.x; i < L.ngroups * 5; i += blockDim.x) s.sc[i / 5][i % 5] = L.sc[i / 5][i % 5];
  for (int i = threadIdx.x; i < dim; i += blockDim.x) s.col_group[i] = L.col_group[i];
}

enum Mode : int { kDeferred = 0, kFlush = 1 };
constexpr int kDenseTally = 2, kRestoreTally = 3;  // tally_host kinds besides kDeferred

// Block index of a sorted id list: bstart[b] = lower_bound(ids, b * kRowsPerBlock) for
// b = 0 .. nblocks (so a 1024-row block finds its gradient ids with two loads instead of a
// dependent binary search), plus the reference's invariant on the list (adam.hpp:231): strictly
// ascending ids in [0, n) — a violation sets bit 0 of the arena's error flag.
__global__ void index_kernel(const int32_t* ids, int64_t count, const int64_t* count_dev, int64_t n, int nblocks,
                             int32_t* bstart, int* err_flag) {
  const int64_t V = count_dev ? *count_dev : count;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= V; k += (int64_t)gridDim.x * blockDim.x) {
    int64_t hi_b = nblocks;  // blocks b with ids[k-1] < b*R <= ids[k] start at k
    if (k < V) {
      const int32_t id = ids[k];
      if (id < 0 || (int64_t)id >= n || (k > 0 && ids[k - 1] >= id)) atomicOr(err_flag, 1);
      hi_b = id < 0 ? -1 : (int64_t)id / kRowsPerBlock;
    }
    int64_t lo_b = 0;
    if (k > 0) {
      const int32_t pid = ids[k - 1];
      lo_b = pid < 0 ? 0 : (int64_t)pid / kRowsPerBlock + 1;
    }
    if (hi_b > nblocks) hi_b = nblocks;
    for (int64_t b = lo_b; b <= hi_b; ++b) bstart[b] = (int32_t)k;
  }
}

// Pass 1 of deferred_update (adam.hpp:211-238) or flush_deferred (adam.hpp:293-313) over rows
// [blockIdx*1024, +1024): counters and the touch list that walk_kernel (pass 2) streams.
// (Arenas with defer_max 0 take dense_update_kernel instead.)
struct TouchList {  // rows a deferred pass touches (unordered; each row at most once)
  int32_t* row;
  int32_t* slot;
  uint8_t* del;
  unsigned long long* count;
  int64_t t0 = 0, t1 = INT64_MAX;  // the walk's range of list entries (a staged chunk)
  const uint32_t* filter = nullptr;  // optional row bit mask: walk only rows whose bit equals want
  int want = 0;
};

template <int K, int MODE>
__global__ void __launch_bounds__(kUpdThreads) update_kernel(ArenaDev a, GradsDev gr, const int32_t* bstart,
                                                             const __grid_constant__ LutArgs<K> L,
                                                             uint32_t* touched_mask, int64_t* touched_count,
                                                             int* err_flag, TouchList tl) {
  __shared__ int32_t slot_of[kRowsPerBlock];
  __shared__ int warp_tot[kUpdThreads / 32];
  __shared__ int ntouched;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerBlock;
  const int nrows = (int)((a.n - r0) < kRowsPerBlock ? (a.n - r0) : kRowsPerBlock);
  for (int i = tid; i < kRowsPerBlock; i += kUpdThreads) slot_of[i] = -1;
  __syncthreads();
  if (MODE == kDeferred && gr.ids) {
    // Clamped: an invalid id list (flagged by index_kernel) may leave entries unset.
    const int64_t gcount = grads_count(gr);
    const int lo = max(0, bstart[blockIdx.x]), hi = (int)min((int64_t)bstart[blockIdx.x + 1], gcount);
    for (int k = lo + tid; k < hi; k += kUpdThreads) {
      const int64_t local = (int64_t)gr.ids[k] - r0;
      if (local >= 0 && local < kRowsPerBlock) slot_of[local] = k;
    }
  }
  __syncthreads();
  // Counter pass: 4 consecutive rows per thread (one 32-bit load/store of counters).
  int my_cnt = 0;
  uint8_t del[4];
  bool tch[4];
  const bool vec_cnt = nrows == kRowsPerBlock && ((reinterpret_cast<uintptr_t>(a.counter + r0) & 3) == 0);
  uint32_t cw = 0, cw_new = 0;
  if (vec_cnt) cw = reinterpret_cast<const uint32_t*>(a.counter + r0)[tid];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int r = tid * 4 + j;
    tch[j] = false;
    del[j] = 0;
    if (r < nrows) {
      const uint8_t c = vec_cnt ? (uint8_t)(cw >> (8 * j)) : a.counter[r0 + r];
      if (c > a.defer_max) atomicOr(err_flag, 2);  // check_counters (adam.hpp:154-158)
      bool t;
      uint8_t cn;
      if (MODE == kDeferred) {
        t = slot_of[r] >= 0 || c == a.defer_max;
        cn = t ? 0 : (uint8_t)(c + 1);
      } else {
        t = c != 0;
        cn = 0;
      }
      cw_new |= (uint32_t)cn << (8 * j);
      if (!vec_cnt && cn != c) a.counter[r0 + r] = cn;
      tch[j] = t;
      del[j] = c;
      my_cnt += t;
    }
  }
  if (vec_cnt && cw_new != cw) reinterpret_cast<uint32_t*>(a.counter + r0)[tid] = cw_new;
  // Block exclusive scan of touched counts (ascending row order).
  int inc = my_cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (tid == 0) {
    int run = 0;
    for (int w = 0; w < kUpdThreads / 32; ++w) {
      const int t = warp_tot[w];
      warp_tot[w] = run;
      run += t;
    }
    ntouched = run;
  }
  __syncthreads();
  __shared__ unsigned long long gbase_s;
  if (tid == 0) {
    const int T = ntouched;
    gbase_s = T > 0 ? atomicAdd(tl.count, (unsigned long long)T) : 0ull;
    if (touched_count && T > 0) atomicAdd((unsigned long long*)touched_count, (unsigned long long)T);
  }
  __syncthreads();
  // Append this block's touched rows (ascending within the block) to the pass's touch list; the
  // walk kernel then streams the list with every warp busy (no per-block serial prologue).
  int64_t pos = (int64_t)gbase_s + warp_tot[warp] + inc - my_cnt;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (tch[j]) {
      const int r = tid * 4 + j;
      tl.row[pos] = (int32_t)(r0 + r);
      tl.del[pos] = del[j];
      tl.slot[pos] = MODE == kDeferred ? slot_of[r] : -1;
      ++pos;
    }
  if (touched_mask) {
    // word w covers rows 32w..32w+31 of this block: lanes own rows 4*lane..4*lane+3 of a
    // 128-row warp slice, so each warp emits 4 words.
    uint32_t nib = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) nib |= (tch[j] ? 1u : 0u) << j;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      // lanes 8q..8q+7 hold rows 32q..32q+31 of the warp slice
      uint32_t word = 0;
#pragma unroll
      for (int l = 0; l < 8; ++l) word |= __shfl_sync(0xffffffffu, nib, q * 8 + l) << (4 * l);
      const int64_t wrow = r0 + warp * 128 + q * 32;
      if (lane == 0 && wrow < a.n) touched_mask[wrow >> 5] = word;
    }
  }
}

// Dense immediate update of an arena with defer_max 0 (the geometric tier, store.hpp:121-124;
// engine.hpp:380-386): every row is touched at delay 0 (w_scale = 0, so the restoration term is
// w - (+-0), kept exactly) and counters stay 0. A block owns 1024 contiguous rows = one contiguous
// span of dim * 1024 floats per array, streamed as float4 (16-byte loads/stores, kU in flight per
// thread); per element the row is a magic-number division, its gradient slot comes from the
// block's SMEM row->slot map and its column constants from SMEM. Bit-identical to
// deferred_scalar at delay 0.
template <int K>
__global__ void __launch_bounds__(kUpdThreads) dense_update_kernel(ArenaDev a, GradsDev gr, const int32_t* bstart,
                                                                   const __grid_constant__ LutArgs<K> L,
                                                                   int64_t* touched_count, uint32_t* touched_mask) {
  __shared__ float4 cA[kMaxDim];  // ms, vs, one_minus_b1, one_minus_b2 per column
  __shared__ float4 cB[kMaxDim];  // bias_correction, step_size, eps, -
  __shared__ int32_t slot_of[kRowsPerBlock];
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerBlock;
  const int nrows = (int)((a.n - r0) < kRowsPerBlock ? (a.n - r0) : kRowsPerBlock);
  const int dim = a.dim;
  for (int c = tid; c < dim; c += kUpdThreads) {
    const int g = L.col_group[c];
    cA[c] = make_float4(L.a1[g][0], L.a2[g][0], L.sc[g][0], L.sc[g][1]);
    cB[c] = make_float4(L.sc[g][2], L.sc[g][3], L.sc[g][4], 0.0f);
  }
  for (int i = tid; i < kRowsPerBlock; i += kUpdThreads) slot_of[i] = -1;
  __syncthreads();
  if (gr.ids) {
    const int64_t gcount = grads_count(gr);
    const int lo = max(0, bstart[blockIdx.x]), hi = (int)min((int64_t)bstart[blockIdx.x + 1], gcount);
    for (int k = lo + tid; k < hi; k += kUpdThreads) {
      const int64_t local = (int64_t)gr.ids[k] - r0;
      if (local >= 0 && local < kRowsPerBlock) slot_of[local] = k;
    }
  }
  __syncthreads();
  const int64_t e0 = r0 * dim;
  const int ne = nrows * dim;
  float4* W = reinterpret_cast<float4*>(a.w + e0);
  float4* M = reinterpret_cast<float4*>(a.m + e0);
  float4* V = reinterpret_cast<float4*>(a.v + e0);
  const int nq = ne >> 2;
#ifndef GSS_DENSE_KU
#define GSS_DENSE_KU 1  // 0.77 vs 0.74 of HBM for 2 (tools/adam_probe.py)
#endif
  constexpr int kU = GSS_DENSE_KU;
  auto elem = [&](float& w, float& m, float& v, float gv, int col) {
    const float4 A = cA[col], B = cB[col];
    const float m_new = A.x * m + A.z * gv;
    const float v_new = A.y * v + A.w * gv * gv;
    const float num = 0.0f * m;  // w_scale(0) * m
    w = (num == 0.0f && v >= 0.0f) ? w - num : w - div_rn(num, sqrt_rn(v) + B.z);
    const float denom = div_rn(sqrt_rn(v_new), B.x) + B.z;
    w = w - div_rn(B.y * m_new, denom);
    m = m_new;
    v = v_new;
  };
  for (int q0 = tid; q0 < nq; q0 += kUpdThreads * kU) {
    float4 w[kU], m[kU], v[kU];
    float gv[kU][4];
    int col[kU][4];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int q = q0 + u * kUpdThreads;
      const bool ok = q < nq;
      w[u] = ok ? W[q] : make_float4(0.f, 0.f, 0.f, 0.f);
      m[u] = ok ? M[q] : make_float4(0.f, 0.f, 0.f, 0.f);
      v[u] = ok ? V[q] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t f = (uint32_t)(4 * q + i);
        const int row = (int)__umulhi(f, a.div_magic);
        col[u][i] = (int)f - row * dim;
        const int sl = ok ? slot_of[row] : -1;
        gv[u][i] = sl >= 0 ? gr.rows[(size_t)sl * gr.stride + gr.col0 + col[u][i]] : 0.0f;
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int q = q0 + u * kUpdThreads;
      if (q >= nq) continue;
      elem(w[u].x, m[u].x, v[u].x, gv[u][0], col[u][0]);
      elem(w[u].y, m[u].y, v[u].y, gv[u][1], col[u][1]);
      elem(w[u].z, m[u].z, v[u].z, gv[u][2], col[u][2]);
      elem(w[u].w, m[u].w, v[u].w, gv[u][3], col[u][3]);
      W[q] = w[u];
      M[q] = m[u];
      V[q] = v[u];
    }
  }
  for (int f = 4 * nq + tid; f < ne; f += kUpdThreads) {  // ragged tail of the last block
    const int row = (int)__umulhi((uint32_t)f, a.div_magic);
    const int c = f - row * dim;
    const int sl = slot_of[row];
    float w = a.w[e0 + f], m = a.m[e0 + f], v = a.v[e0 + f];
    elem(w, m, v, sl >= 0 ? gr.rows[(size_t)sl * gr.stride + gr.col0 + c] : 0.0f, c);
    a.w[e0 + f] = w;
    a.m[e0 + f] = m;
    a.v[e0 + f] = v;
  }
  if (touched_count && tid == 0 && nrows > 0)
    atomicAdd((unsigned long long*)touched_count, (unsigned long long)nrows);
  if (touched_mask) {
    for (int wi = tid; wi * 32 < nrows; wi += kUpdThreads) {
      const int rem = nrows - wi * 32;
      touched_mask[(r0 >> 5) + wi] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
    }
  }
}

// Per-(group, delay) and per-group constants of a pass, packed for 16-byte SMEM loads.
template <int K> struct PackedLuts {
  float4 gd[kMaxGroups][K];  // param (w_scale), a1, a2, -
  float4 sc[kMaxGroups];     // one_minus_b1, one_minus_b2, bias_correction, step_size
  float eps[kMaxGroups];
  uint8_t col_group[kMaxDim];
};

template <int K> __device__ void load_packed_luts(PackedLuts<K>& s, const LutArgs<K>& L, int dim) {
  for (int i = threadIdx.x; i < L.ngroups * K; i += blockDim.x) {
    const int g = i / K, e = i - g * K;
    s.gd[g][e] = make_float4(L.param[g][e], L.a1[g][e], L.a2[g][e], 0.0f);
  }
  for (int g = threadIdx.x; g < L.ngroups; g += blockDim.x) {
    s.sc[g] = make_float4(L.sc[g][0], L.sc[g][1], L.sc[g][2], L.sc[g][3]);
    s.eps[g] = L.sc[g][4];
  }
  for (int i = threadIdx.x; i < dim; i += blockDim.x) s.col_group[i] = L.col_group[i];
}

// deferred_scalar (adam.hpp:102-110) with the exact zero-numerator shortcut of the restoration
// term: (w_scale * m) / (sqrt(v) + eps) is the signed zero w_scale * m itself whenever it is zero
// and v >= 0 (the denominator is then >= eps > 0) — every delay-0 row, i.e. every row touched
// with a gradient the previous pass. Bit-identical to deferred_scalar.
__device__ __forceinline__ void deferred_scalar_fast(float& w, float& m, float& v, float g, float4 gd, float4 sc,
                                                     float eps) {
  const float m_new = gd.y * m + sc.x * g;
  const float v_new = gd.z * v + sc.y * g * g;
  const float num = gd.x * m;
  w = (num == 0.0f && v >= 0.0f) ? w - num : w - div_rn(num, sqrt_rn(v) + eps);
  const float denom = div_rn(sqrt_rn(v_new), sc.z) + eps;
  w = w - div_rn(sc.w * m_new, denom);
  m = m_new;
  v = v_new;
}

// Streams a touch list: a warp owns 32 list entries (rows) at a time and walks their flattened
// (row, column) space, 32 x dim elements = dim iterations with every lane busy (lane l takes
// elements l, l + 32, ...; consecutive lanes read consecutive columns, so each warp access is one
// or two contiguous row spans). The 32 rows' (id, delay, gradient slot) sit in the lanes'
// registers and are fetched with shuffles; kU elements per lane have all their loads in flight
// before any math.
#ifndef GSS_WALK_KU
#define GSS_WALK_KU 4
#endif
#ifndef GSS_WALK_MINB
#define GSS_WALK_MINB 4
#endif
template <int K, int MODE>
__global__ void __launch_bounds__(kUpdThreads, GSS_WALK_MINB) walk_kernel(ArenaDev a, GradsDev gr, const __grid_constant__ LutArgs<K> L,
                                                        TouchList tl) {
  __shared__ PackedLuts<K> lut;
  load_packed_luts<K>(lut, L, a.dim);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t T = (int64_t)*tl.count;
  const int dim = a.dim;
  const int dq = 32 / dim, dr = 32 - dq * dim;  // per-iteration advance of (row, col)
  constexpr int kU = GSS_WALK_KU;
  const int64_t wstride = (int64_t)gridDim.x * (kUpdThreads / 32) * 32;
  for (int64_t t0 = ((int64_t)blockIdx.x * (kUpdThreads / 32) + (threadIdx.x >> 5)) * 32; t0 < T; t0 += wstride) {
    // this lane's list entry (row t0 + lane)
    const bool mine = t0 + lane < T;
    const int32_t my_row = mine ? tl.row[t0 + lane] : -1;
    const int32_t my_del = mine ? tl.del[t0 + lane] : 0;
    const int32_t my_slot = (mine && MODE == kDeferred) ? tl.slot[t0 + lane] : -1;
    int r = lane / dim, c = lane - (lane / dim) * dim;
    for (int i0 = 0; i0 < dim; i0 += kU) {
      float w[kU], m[kU], v[kU], gv[kU];
      size_t off[kU];
      int dd[kU], cc[kU];
      bool ok[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int rr = r < 32 ? r : 31;
        const int32_t row = __shfl_sync(0xffffffffu, my_row, rr);
        const int32_t sl = __shfl_sync(0xffffffffu, my_slot, rr);
        dd[u] = __shfl_sync(0xffffffffu, my_del, rr);
        cc[u] = c;
        ok[u] = i0 + u < dim && row >= 0;
        off[u] = ok[u] ? (size_t)row * a.stride + c : 0;
        w[u] = ok[u] ? a.w[off[u]] : 0.0f;
        m[u] = ok[u] ? a.m[off[u]] : 0.0f;
        v[u] = ok[u] ? a.v[off[u]] : 0.0f;
        gv[u] = (ok[u] && sl >= 0) ? gr.rows[(size_t)sl * gr.stride + gr.col0 + c] : 0.0f;
        r += dq;
        c += dr;
        if (c >= dim) {
          c -= dim;
          ++r;
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (!ok[u]) continue;
        const int g = lut.col_group[cc[u]];
        const float4 gd = lut.gd[g][dd[u]];
        if (MODE == kDeferred) {
          deferred_scalar_fast(w[u], m[u], v[u], gv[u], gd, lut.sc[g], lut.eps[g]);
          a.w[off[u]] = w[u];
          a.m[off[u]] = m[u];
          a.v[off[u]] = v[u];
        } else {
          a.w[off[u]] = w[u] - div_rn(gd.x * m[u], sqrt_rn(v[u]) + lut.eps[g]);  // adam.hpp:112-114
          a.m[off[u]] = m[u] * gd.y;
          a.v[off[u]] = v[u] * gd.z;
        }
      }
    }
  }
}

// Vector walk for arenas whose w/m/v rows are 16-byte aligned with whole float4 row segments
// (row_stride % 4 == 0: the engine's row-interleaved non-geometric tier, w @ 0, m @ 52, v @ 104 of a
// 160-float row). A unit = 4 consecutive columns of one row: one 16-byte load/store each of w, m,
// v; a warp walks the flattened (row, unit) space of 32 list rows, so the per-element address
// arithmetic and shuffles of the scalar walk are amortised over 4 columns. Columns dim..4*nq-1 of
// the last unit are row padding (never read back as data).
#ifndef GSS_WALK4_KU
#define GSS_WALK4_KU 1  // 1 unit per lane + 4 blocks/SM: 0.64 vs 0.56 of HBM for 2 + 3 (tools/adam_probe.py)
#endif
#ifndef GSS_WALK_GRID
#define GSS_WALK_GRID 8  // walk blocks per SM (grid-stride over the touch list)
#endif
#ifndef GSS_WALK4_MINB
#define GSS_WALK4_MINB 4
#endif
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float& at(float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

template <int K, int MODE>
__global__ void __launch_bounds__(kUpdThreads, GSS_WALK4_MINB) walk4_kernel(ArenaDev a, GradsDev gr,
                                                                         const __grid_constant__ LutArgs<K> L,
                                                                         TouchList tl) {
  __shared__ PackedLuts<K> lut;
  load_packed_luts<K>(lut, L, a.dim);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t T = min((int64_t)*tl.count, tl.t1);
  const int dim = a.dim;
  const int nq = (dim + 3) >> 2;  // float4 units per row
  const int dq = 32 / nq, dr = 32 - dq * nq;
  constexpr int kU = GSS_WALK4_KU;
  const int64_t wstride = (int64_t)gridDim.x * (kUpdThreads / 32) * 32;
  for (int64_t t0 = tl.t0 + ((int64_t)blockIdx.x * (kUpdThreads / 32) + (threadIdx.x >> 5)) * 32; t0 < T;
       t0 += wstride) {
    bool mine = t0 + lane < T;
    if (mine && tl.filter) {
      const int32_t rw = tl.row[t0 + lane];
      mine = (int)((tl.filter[rw >> 5] >> (rw & 31)) & 1u) == tl.want;
    }
    const int64_t my_base =
        mine ? (a.positional ? (t0 + lane - tl.t0) : (int64_t)tl.row[t0 + lane]) * a.stride : -1;
    const int32_t my_del = mine ? tl.del[t0 + lane] : 0;
    const int32_t my_slot = (mine && MODE == kDeferred) ? tl.slot[t0 + lane] : -1;
    int r = lane / nq, q = lane - (lane / nq) * nq;
    for (int i0 = 0; i0 < nq; i0 += kU) {
      float4 w[kU], m[kU], v[kU];
      float gv[kU][4];
      int64_t base[kU];
      int dd[kU], c0[kU];
      bool ok[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int rr = r < 32 ? r : 31;
        base[u] = __shfl_sync(0xffffffffu, my_base, rr);
        const int32_t sl = __shfl_sync(0xffffffffu, my_slot, rr);
        dd[u] = __shfl_sync(0xffffffffu, my_del, rr);
        c0[u] = 4 * q;
        ok[u] = i0 + u < nq && base[u] >= 0;
        const int64_t o = ok[u] ? base[u] + c0[u] : 0;
        w[u] = ok[u] ? ld4(a.w + o) : make_float4(0.f, 0.f, 0.f, 0.f);
        m[u] = ok[u] ? ld4(a.m + o) : make_float4(0.f, 0.f, 0.f, 0.f);
        v[u] = ok[u] ? ld4(a.v + o) : make_float4(0.f, 0.f, 0.f, 0.f);
        grad_unit(gr, sl, c0[u], dim, ok[u], gv[u]);
        r += dq;
        q += dr;
        if (q >= nq) {
          q -= nq;
          ++r;
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (!ok[u]) continue;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int c = c0[u] + i < dim ? c0[u] + i : dim - 1;  // padding columns reuse a valid group
          const int g = lut.col_group[c];
          const float4 gd = lut.gd[g][dd[u]];
          if (MODE == kDeferred) {
            deferred_scalar_fast(at(w[u], i), at(m[u], i), at(v[u], i), gv[u][i], gd, lut.sc[g], lut.eps[g]);
          } else {
            at(w[u], i) = at(w[u], i) - div_rn(gd.x * at(m[u], i), sqrt_rn(at(v[u], i)) + lut.eps[g]);
            at(m[u], i) = at(m[u], i) * gd.y;
            at(v[u], i) = at(v[u], i) * gd.z;
          }
        }
        const int64_t o = base[u] + c0[u];
        st4(a.w + o, w[u]);
        st4(a.m + o, m[u]);
        st4(a.v + o, v[u]);
      }
    }
  }
}

// Can w/m/v be walked with 16-byte accesses? Row segments 16-byte aligned and non-overlapping
// when rounded up to whole float4 units.
bool vector_rows(const gss_arena& a) {
  const int64_t stride = a.row_stride > 0 ? a.row_stride : a.dim;
  if (stride % 4 != 0) return false;
  for (const float* p : {a.w, a.m, a.v})
    if (reinterpret_cast<uintptr_t>(p) % 16 != 0) return false;
  const int64_t seg = ((a.dim + 3) / 4) * 4;
  if (seg > stride) return false;
  const float* ps[3] = {a.w, a.m, a.v};
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j) {
      const int64_t d = ps[i] - ps[j];
      const int64_t ad = d < 0 ? -d : d;
      if (ad < seg && ad != 0) return false;  // same row: the padded segments must not overlap
      if (ad == 0) return false;
    }
  return true;
}

// restore_view (adam.hpp:252-289): out[k] = restored row ids[k] (+ pending pass). Grid-stride
// over 256-id chunks; per chunk each thread resolves one (id, delay, pending slot): the pending
// ids of the chunk's row span are staged in SMEM through the pending list's block index, so the
// slot is a binary search in SMEM instead of a dependent search through global memory. Then the
// flattened (id, column) walk reads the arena rows with consecutive lanes on consecutive columns.
constexpr int kRestoreChunk = kUpdThreads;
#ifndef GSS_RESTORE_MINB
#define GSS_RESTORE_MINB 4
#endif
#ifndef GSS_RESTORE_KV
#define GSS_RESTORE_KV 1  // with 4 blocks/SM: 0.57 vs 0.53 of HBM (tools/adam_probe.py)
#endif
constexpr int kSeg = 2048;
template <int K>
__global__ void __launch_bounds__(kUpdThreads, 3) restore_kernel(ArenaDev a, const int32_t* ids, int64_t count,
                                                              const int64_t* count_dev, GradsDev pend,
                                                              const int32_t* pbstart, int has_pending,
                                                              const __grid_constant__ LutArgs<K> L, float* out,
                                                              int vec) {
  __shared__ PackedLuts<K> lut;
  __shared__ int32_t cid[kRestoreChunk];
  __shared__ uint8_t cdel[kRestoreChunk];
  __shared__ int32_t cslot[kRestoreChunk];
  __shared__ int32_t seg[kSeg];
  __shared__ int seg_lo, seg_n;
  load_packed_luts<K>(lut, L, a.dim);
  const int64_t cnt = count_dev ? *count_dev : count;
  const int64_t pcnt = has_pending ? grads_count(pend) : 0;
  const int nblk = (int)((a.n + kRowsPerBlock - 1) / kRowsPerBlock);
  const int dim = a.dim;
  const int tid = threadIdx.x;
  for (int64_t k0 = (int64_t)blockIdx.x * kRestoreChunk; k0 < cnt; k0 += (int64_t)gridDim.x * kRestoreChunk) {
    const int nk = (int)((cnt - k0) < kRestoreChunk ? (cnt - k0) : kRestoreChunk);
    __syncthreads();
    int32_t id = 0;
    if (tid < nk) {
      id = ids[k0 + tid];
      cid[tid] = id;
      cdel[tid] = a.counter[id];
    }
    if (has_pending && pend.ids && tid == 0) {
      const int64_t lo_row = ids[k0], hi_row = ids[k0 + nk - 1];
      int64_t b0 = lo_row / kRowsPerBlock, b1 = hi_row / kRowsPerBlock + 1;
      b0 = b0 < 0 ? 0 : (b0 > nblk ? nblk : b0);
      b1 = b1 < 0 ? 0 : (b1 > nblk ? nblk : b1);
      int64_t p0 = pbstart[b0], p1 = pbstart[b1];
      p0 = p0 < 0 ? 0 : p0;
      p1 = p1 > pcnt ? pcnt : p1;
      seg_lo = (int)p0;
      seg_n = p1 > p0 ? (int)(p1 - p0) : 0;
    }
    __syncthreads();
    if (has_pending && pend.ids) {
      const int sn = seg_n, sl = seg_lo;
      const bool staged = sn <= kSeg;
      if (staged)
        for (int i = tid; i < sn; i += kUpdThreads) seg[i] = pend.ids[sl + i];
      __syncthreads();
      if (tid < nk) {
        int32_t s = -1;
        if (staged) {
          int lo = 0, hi = sn;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (seg[mid] < id) lo = mid + 1; else hi = mid;
          }
          if (lo < sn && seg[lo] == id) s = sl + lo;
        } else {
          const int64_t p = sl + lower_bound_ids(pend.ids + sl, sn, id);
          if (p < sl + sn && pend.ids[p] == id) s = (int32_t)p;
        }
        cslot[tid] = s;
      }
    }
    __syncthreads();
    // Flattened walk: warp w owns ids [32w, 32w + 32) of the chunk and streams their 32 x dim
    // (id, column) elements with every lane busy (see walk_kernel); all kU loads in flight first.
    const int lane = tid & 31, warp = tid >> 5;
    const int j = warp * 32 + lane;
    const int32_t my_id = j < nk ? cid[j] : -1;
    const int32_t my_del = j < nk ? cdel[j] : 0;
    const int32_t my_slot = (j < nk && has_pending && pend.ids) ? cslot[j] : -1;  // empty pending set: no slots
    if (vec && warp * 32 < nk) {
      // 16-byte units of 4 columns (see walk4_kernel): row-interleaved arenas
      const int nq = (dim + 3) >> 2;
      const int dq = 32 / nq, dr = 32 - dq * nq;
      const int64_t my_base = j < nk ? (int64_t)my_id * a.stride : -1;
      int r = lane / nq, q = lane - (lane / nq) * nq;
      constexpr int kV = GSS_RESTORE_KV;  // 16-byte units of w, m and v in flight per lane
      for (int i0 = 0; i0 < nq; i0 += kV) {
        float4 w[kV], m[kV], v[kV];
        float gv[kV][4];
        int dd[kV], c0[kV], rr4[kV];
        bool ok[kV];
#pragma unroll
        for (int u = 0; u < kV; ++u) {
          const int rr = r < 32 ? r : 31;
          const int64_t base = __shfl_sync(0xffffffffu, my_base, rr);
          const int32_t sl = __shfl_sync(0xffffffffu, my_slot, rr);
          dd[u] = __shfl_sync(0xffffffffu, my_del, rr);
          c0[u] = 4 * q;
          rr4[u] = rr;
          ok[u] = i0 + u < nq && base >= 0;
          const int64_t o = ok[u] ? base + c0[u] : 0;
          w[u] = ok[u] ? ld4(a.w + o) : make_float4(0.f, 0.f, 0.f, 0.f);
          m[u] = ok[u] ? ld4(a.m + o) : make_float4(0.f, 0.f, 0.f, 0.f);
          v[u] = ok[u] ? ld4(a.v + o) : make_float4(0.f, 0.f, 0.f, 0.f);
          grad_unit(pend, sl, c0[u], dim, ok[u], gv[u]);
          r += dq;
          q += dr;
          if (q >= nq) {
            q -= nq;
            ++r;
          }
        }
#pragma unroll
        for (int u = 0; u < kV; ++u) {
          if (!ok[u]) continue;
          float* orow = out + (size_t)(k0 + warp * 32 + rr4[u]) * dim + c0[u];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (c0[u] + i >= dim) break;
            const int g = lut.col_group[c0[u] + i];
            const float4 gd = lut.gd[g][dd[u]];
            float ww = at(w[u], i);
            if (has_pending) {
              float mm = at(m[u], i), vv = at(v[u], i);
              deferred_scalar_fast(ww, mm, vv, gv[u][i], gd, lut.sc[g], lut.eps[g]);
            } else {
              const float num = gd.x * at(m[u], i);
              ww = (num == 0.0f && at(v[u], i) >= 0.0f) ? ww - num
                                                        : ww - div_rn(num, sqrt_rn(at(v[u], i)) + lut.eps[g]);
            }
            orow[i] = ww;
          }
        }
      }
      continue;
    }
    const int dq = 32 / dim, dr = 32 - dq * dim;
    int r = lane / dim, c = lane - (lane / dim) * dim;
    constexpr int kU = GSS_WALK_KU;
    if (warp * 32 < nk) {
      for (int i0 = 0; i0 < dim; i0 += kU) {
        float w[kU], m[kU], v[kU], gv[kU];
        size_t oo[kU];
        int dd[kU], cc[kU];
        bool ok[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int rr = r < 32 ? r : 31;
          const int32_t id2 = __shfl_sync(0xffffffffu, my_id, rr);
          const int32_t sl = __shfl_sync(0xffffffffu, my_slot, rr);
          dd[u] = __shfl_sync(0xffffffffu, my_del, rr);
          cc[u] = c;
          ok[u] = i0 + u < dim && id2 >= 0;
          const size_t off = ok[u] ? (size_t)id2 * a.stride + c : 0;
          oo[u] = (size_t)(k0 + warp * 32 + rr) * dim + c;
          w[u] = ok[u] ? a.w[off] : 0.0f;
          m[u] = ok[u] ? a.m[off] : 0.0f;
          v[u] = ok[u] ? a.v[off] : 0.0f;
          gv[u] = (ok[u] && sl >= 0) ? pend.rows[(size_t)sl * pend.stride + pend.col0 + c] : 0.0f;
          r += dq;
          c += dr;
          if (c >= dim) {
            c -= dim;
            ++r;
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (!ok[u]) continue;
          const int g = lut.col_group[cc[u]];
          const float4 gd = lut.gd[g][dd[u]];
          float ww = w[u];
          if (has_pending) {
            float mm = m[u], vv = v[u];
            deferred_scalar_fast(ww, mm, vv, gv[u], gd, lut.sc[g], lut.eps[g]);
          } else {  // restore_scalar (adam.hpp:112-114), zero-numerator shortcut as deferred_scalar_fast
            const float num = gd.x * m[u];
            ww = (num == 0.0f && v[u] >= 0.0f) ? ww - num : ww - div_rn(num, sqrt_rn(v[u]) + lut.eps[g]);
          }
          out[oo[u]] = ww;
        }
      }
    }
  }
}

ArenaDev arena_dev(const gss_arena& a) {
  ArenaDev d;
  d.w = a.w; d.m = a.m; d.v = a.v; d.counter = a.counter;
  d.n = a.n; d.dim = a.dim; d.defer_max = a.defer_max;
  d.div_magic = (uint32_t)((((uint64_t)1 << 32) + (uint64_t)a.dim - 1) / (uint64_t)a.dim);
  d.stride = a.row_stride > 0 ? a.row_stride : a.dim;
  d.positional = 0;
  return d;
}

// ---- host-tier passes through HBM staging (selective offloading, store.hpp:149-222) -----------
// A pinned host arena is read and written over the host link. Kernels that read-modify-write host
// rows in place interleave read requests behind posted writes on the link (measured: 6 GB/s each
// way, profiles/r02_linkprobe.txt); pure gathers and pure scatters run at the link's rate (51 / 47
// GB/s). So a host-tier pass moves whole rows: gather the listed rows into a positional HBM
// staging copy, run the pass there at HBM speed, scatter the written rows back — in chunks of
// chunk_bytes (the reference's ForwardStage chunks, store.hpp:204-222), alternating two streams so
// one chunk's host->device gather overlaps the previous chunk's device->host scatter.
// Staging row layout: the three float4-padded segments w | m | v back to back (3 * nq float4).
__host__ __device__ inline int stage_stride(int dim) { return 3 * ((dim + 3) / 4) * 4; }

ArenaDev staged_arena(const gss_arena& a, float* stage) {
  ArenaDev d = arena_dev(a);
  const int seg = (a.dim + 3) / 4 * 4;
  d.w = stage;
  d.m = stage + seg;
  d.v = stage + 2 * seg;
  d.stride = stage_stride(a.dim);
  d.positional = 1;
  return d;
}

#ifndef GSS_MOVE_ILP
#define GSS_MOVE_ILP 8
#endif
// GATHER: stage[k] = host rows[list[t0 + k]]; else host rows[list[t0 + k]] = stage[k], for
// k < t1 - t0. Consecutive threads take consecutive 16-byte units of a row (a row's three segments
// are 39 contiguous units of the 640-byte interleaved row), GSS_MOVE_ILP loads in flight each.
template <bool GATHER>
__global__ void __launch_bounds__(256) move_rows_kernel(ArenaDev a, const int32_t* list, int64_t t0, int64_t t1,
                                                        float* stage) {
  const int nq = (a.dim + 3) >> 2;
  const uint32_t upr = 3u * (uint32_t)nq;
  // unit index math in 32 bits: callers pass at most 2^31 / upr rows per launch
  const uint32_t total = (uint32_t)((t1 - t0) * (int64_t)upr);
  const uint32_t step = gridDim.x * blockDim.x;
  const int sstride = stage_stride(a.dim);
  for (uint32_t u0 = blockIdx.x * blockDim.x + threadIdx.x; u0 < total; u0 += step * GSS_MOVE_ILP) {
    float4 val[GSS_MOVE_ILP];
    float* dst[GSS_MOVE_ILP];
#pragma unroll
    for (int i = 0; i < GSS_MOVE_ILP; ++i) {
      const uint32_t u = u0 + i * step;
      dst[i] = nullptr;
      if (u < total) {
        const uint32_t k = u / upr;
        const int j = (int)(u - k * upr);
        const int seg = j / nq, q = j - seg * nq;
        const int64_t id = list[t0 + k];
        float* hp = (seg == 0 ? a.w : (seg == 1 ? a.m : a.v)) + id * a.stride + 4 * q;
        float* sp = stage + k * sstride + seg * nq * 4 + 4 * q;
        if (GATHER) {
          val[i] = ld4(hp);
          dst[i] = sp;
        } else {
          val[i] = ld4(sp);
          dst[i] = hp;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < GSS_MOVE_ILP; ++i)
      if (dst[i]) st4(dst[i], val[i]);
  }
}
constexpr int kMoveBlocks = 64;  // 64 x 256 threads x 8 units in flight: ~2 MB outstanding per direction

// chunk size of the staged host-tier passes (the engine sets it from EngineConfig::chunk_bytes)
std::atomic<int64_t> g_host_chunk_bytes{int64_t(32) << 20};
// The staged passes are opt-in (GSS_HOST_STAGING=1): measured on the B200 (tools/host_tier_probe.py,
// 40M rows, 13% visible; profiles/r02_host_tier_ab.txt) the in-place zero-copy passes move the
// host link's bytes faster — forwarding gather 72.8 vs 81.3 ms, deferred update 124 vs 177 ms — the
// device reads and writes host rows concurrently from many SMs, while the staged chunks serialise
// gather, pass and scatter per chunk.
bool host_staging() {
  static const bool on = [] {
    const char* e = std::getenv("GSS_HOST_STAGING");
    return e && e[0] == '1';
  }();
  return on;
}

// A second stream per device for the alternating chunks, plus fork / join events.
struct AuxStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
std::mutex g_aux_mu;
std::unordered_map<int, AuxStream> g_aux;
AuxStream& aux_stream() {
  int dev = 0;
  GSS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_aux_mu);
  AuxStream& x = g_aux[dev];
  if (!x.s) {
    // highest priority: the link-bound chunks' few CTAs are scheduled ahead of a concurrent render
    int lo = 0, hi = 0;
    GSS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    GSS_CUDA(cudaStreamCreateWithPriority(&x.s, cudaStreamNonBlocking, hi));
    GSS_CUDA(cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming));
    GSS_CUDA(cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming));
  }
  return x;
}

void validate_arena(const gss_arena& a) {
  require(a.n >= 0 && a.n <= INT32_MAX, "arena: n out of range");
  require(a.dim >= 1 && a.dim <= kMaxDim, "arena: dim must be in [1, 128]");
  require(a.defer_max >= 0 && a.defer_max <= 254, "arena: defer max must be in [0, 254]");
  require(a.ngroups >= 1 && a.ngroups <= kMaxGroups, "arena: 1..8 groups");
  int covered = 0;
  for (int g = 0; g < a.ngroups; ++g) {
    const gss_group& G = a.groups[g];
    require(G.lr > 0, "hyperparams: lr must be > 0");
    require(G.beta1 >= 0 && G.beta1 < 1, "hyperparams: require 0 <= beta1 < 1");
    require(G.beta2 >= 0 && G.beta2 < 1, "hyperparams: require 0 <= beta2 < 1");
    require(G.eps > 0, "hyperparams: eps must be > 0");
    require(G.col0 == covered && G.dim >= 1, "arena: groups must tile the row contiguously");
    covered += G.dim;
  }
  require(covered == a.dim, "arena: group dims must cover the row");
  require(a.row_stride == 0 || a.row_stride >= a.dim, "arena: row_stride must be 0 or >= dim");
  require(a.n == 0 || (a.w && a.m && a.v && a.counter), "arena: null buffer");
}

GradsDev grads_dev(const gss_sparse_grads* g, int dim = 0) {
  GradsDev d{};
  if (g) {
    d.ids = g->ids; d.count = g->count; d.count_dev = g->count_dev; d.rows = g->rows;
    d.stride = g->stride; d.col0 = g->col0;
    // the engine's gradient stage: 52-float rows, col0 0, 16-byte aligned (the padding columns are
    // loaded and discarded)
#ifndef GSS_GRAD_VEC4
#define GSS_GRAD_VEC4 1
#endif
    d.vec4 = GSS_GRAD_VEC4 && dim > 0 && g->rows && reinterpret_cast<uintptr_t>(g->rows) % 16 == 0 && g->stride % 4 == 0 &&
             g->col0 % 4 == 0 && g->stride >= g->col0 + (dim + 3) / 4 * 4;
  }
  return d;
}

// Per-arena device error flag (keyed by the counter buffer), allocated lazily.
int* err_flag_for(const gss_arena& a);


// Per-arena scratch (keyed by the counter buffer, like the error flag), grown on demand from the
// stream-ordered pool and kept: a pass allocates and frees nothing. Slot 0 serves the update passes
// (block index + touch list), slot 1 the forwarding gather (pending block index), slots 2 / 3 the
// HBM staging of a host-tier update / gather (staged_walk, adam_restore); one writer per
// arena at a time (the reference engine's DAG) keeps each slot single-stream.
std::mutex g_scr_mu;
std::unordered_map<const void*, std::pair<void*, size_t>> g_scr[4];
char* arena_scratch(const gss_arena& a, int slot, size_t bytes, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_scr_mu);
  auto& e = g_scr[slot][a.counter];
  if (e.second < bytes) {
    if (e.first) GSS_CUDA(cudaFreeAsync(e.first, st));
    GSS_CUDA(cudaMallocAsync(&e.first, bytes, st));
    e.second = bytes;
  }
  return static_cast<char*>(e.first);
}

// Is the arena's w in host memory (the pinned host tier of selective offloading)? Kernels that
// walk such an arena are bound by the host link, not by SM count: they get a small grid (enough
// requests in flight to fill the link) so the render on the other stream keeps the SMs.
bool host_resident(const gss_arena& a) {
  cudaPointerAttributes at{};
  if (!a.w || cudaPointerGetAttributes(&at, a.w) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}
// (GSS_HOST_BLOCKS overrides it for A/B measurements)
int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  const int x = v ? std::atoi(v) : 0;
  return x > 0 ? x : dflt;
}
// Measured at 18M rows / 14.5% visible (profiles/r02_host_tier_grid.txt): the in-place passes move
// the host link's bytes fastest with few CTAs — the deferred walk 48 ms at 16-32 CTAs vs 57 ms at
// 256, the forwarding gather ~37 ms from 16 CTAs up.
int host_tier_blocks() {  // forwarding gather over host rows
  static const int b = env_int("GSS_HOST_BLOCKS", 32);
  return b;
}
int host_walk_blocks() {  // deferred walk over host rows (reads and writes in flight)
  static const int b = env_int("GSS_HOST_WALK_BLOCKS", 32);
  return b;
}

unsigned long long* tally_dev(const gss_arena& a);
__global__ void tally_add_kernel(unsigned long long* dst, const unsigned long long* src_u64, const int64_t* src_i64) {
  *dst += src_u64 ? *src_u64 : (unsigned long long)*src_i64;
}
// Host-known AccessReport parts: a deferred / dense pass (touched rows host-known, or 0 when the
// device adds them), or a restore of `rows` rows.
void tally_host(const gss_arena& a, int kind, int64_t rows);

// Block index of a sorted id list (nblocks + 1 entries) into `bstart`.
int32_t* build_index(const gss_arena& a, const GradsDev& g, int* err, int32_t* bstart, cudaStream_t st) {
  const int nblk = (int)ceil_div(a.n, kRowsPerBlock);
  const int64_t cap = g.count_dev ? std::max<int64_t>(g.count, a.n) : g.count;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap + 1, 256), 148 * 16));
  index_kernel<<<blocks, 256, 0, st>>>(g.ids, g.count, g.count_dev, a.n, nblk, bstart, err);
  GSS_LAUNCHED();
  return bstart;
}

// Pass 2 of a deferred / flush pass over a pinned host arena: the touch list's rows in chunks,
// each gathered into HBM staging, walked there (walk4_kernel on the positional copy) and scattered
// back; chunk c runs on stream (c & 1) so gathers and scatters of neighbouring chunks overlap on
// the link. The touched count is read back once (the host sizes the chunk loop).
int64_t* pinned_count() {
  thread_local int64_t* p = nullptr;
  if (!p) GSS_CUDA(cudaHostAlloc((void**)&p, sizeof(int64_t), cudaHostAllocDefault));
  return p;
}
char* arena_scratch(const gss_arena& a, int slot, size_t bytes, cudaStream_t st);
template <int K, int MODE>
void staged_walk(const gss_arena& a, const GradsDev& gd, const LutArgs<K>& L, const TouchList& tl, cudaStream_t st) {
  int64_t* hc = pinned_count();
  GSS_CUDA(cudaMemcpyAsync(hc, tl.count, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GSS_CUDA(cudaStreamSynchronize(st));
  const int64_t T = *hc;
  if (T <= 0) return;
  const int ss = stage_stride(a.dim);
  const int64_t C = std::max<int64_t>(1024, g_host_chunk_bytes.load() / ((int64_t)ss * 4));
  const int64_t nch = ceil_div(T, C);
  const int64_t crow = std::min<int64_t>(C, T);
  float* stage = reinterpret_cast<float*>(arena_scratch(a, 2, (size_t)(nch > 1 ? 2 : 1) * crow * ss * 4, st));
  AuxStream& ax = aux_stream();
  if (nch > 1) {
    GSS_CUDA(cudaEventRecord(ax.fork, st));
    GSS_CUDA(cudaStreamWaitEvent(ax.s, ax.fork, 0));
  }
  const int wblocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(crow, 32 * (kUpdThreads / 32)) * 4,
                                                                   (int64_t)sm_count() * GSS_WALK_GRID));
  for (int64_t c = 0; c < nch; ++c) {
    cudaStream_t sx = (c & 1) ? ax.s : st;
    float* buf = stage + (c & 1) * crow * ss;
    const int64_t t0 = c * C, t1 = std::min<int64_t>(T, t0 + C);
    move_rows_kernel<true><<<kMoveBlocks, 256, 0, sx>>>(arena_dev(a), tl.row, t0, t1, buf);
    GSS_LAUNCHED();
    TouchList tc = tl;
    tc.t0 = t0;
    tc.t1 = t1;
    walk4_kernel<K, MODE><<<wblocks, kUpdThreads, 0, sx>>>(staged_arena(a, buf), gd, L, tc);
    GSS_LAUNCHED();
    move_rows_kernel<false><<<kMoveBlocks, 256, 0, sx>>>(arena_dev(a), tl.row, t0, t1, buf);
    GSS_LAUNCHED();
  }
  if (nch > 1) {
    GSS_CUDA(cudaEventRecord(ax.join, ax.s));
    GSS_CUDA(cudaStreamWaitEvent(st, ax.join, 0));
  }
}

// A deferred pass whose walk is split by a row bit mask (the host tier's concurrent forwarding):
// rows whose bit is clear are walked first; the walk of the rows whose bit is set waits for
// `before_set` (recorded by the forwarding gather that must read them first).
struct WalkSplit {
  const uint32_t* mask = nullptr;
  cudaEvent_t before_set = nullptr;
};

template <int K, int MODE>
void launch_update(const gss_arena& a, const GradsDev& gd, int64_t t, uint32_t* tmask, int64_t* tcount,
                   cudaStream_t st, const WalkSplit* split = nullptr) {
  auto L = std::make_unique<LutArgs<K>>();
  std::memset(L.get(), 0, sizeof(LutArgs<K>));
  fill_luts<K>(a, t, MODE == kFlush, *L);
  int* err = err_flag_for(a);
  const int blocks = (int)ceil_div(a.n, kRowsPerBlock);
  const size_t n = (size_t)a.n;
  const size_t idx_bytes = ((size_t)(blocks + 1) * 4 + 255) / 256 * 256;
  char* scr = arena_scratch(a, 0, idx_bytes + 16 + n * 9, st);
  int32_t* bstart = nullptr;
  if (MODE == kDeferred && gd.ids) bstart = build_index(a, gd, err, reinterpret_cast<int32_t*>(scr), st);
  if (MODE == kDeferred && a.defer_max == 0 && (a.row_stride == 0 || a.row_stride == a.dim)) {
    dense_update_kernel<K><<<blocks, kUpdThreads, 0, st>>>(arena_dev(a), gd, bstart, *L, tcount, tmask);
    GSS_LAUNCHED();
    tally_host(a, kDeferred, a.n);  // defer_max 0: counter == MAX for every row, all touched
  } else {
    // Pass 1: counters + touch list; pass 2: stream the list.
    TouchList tl;
    char* buf = scr + idx_bytes;
    tl.count = reinterpret_cast<unsigned long long*>(buf);
    tl.row = reinterpret_cast<int32_t*>(buf + 16);
    tl.slot = tl.row + n;
    tl.del = reinterpret_cast<uint8_t*>(tl.slot + n);
    GSS_CUDA(cudaMemsetAsync(tl.count, 0, 8, st));
    update_kernel<K, MODE><<<blocks, kUpdThreads, 0, st>>>(arena_dev(a), gd, bstart, *L, tmask, tcount, err,
                                                                   tl);
    GSS_LAUNCHED();
    if (MODE == kDeferred) {  // adam.hpp:233-236; the touched count is known on the device only
      tally_host(a, kDeferred, 0);
      tally_add_kernel<<<1, 1, 0, st>>>(tally_dev(a), tl.count, nullptr);
      GSS_LAUNCHED();
    }
    int wblocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(a.n, kUpdThreads), (int64_t)sm_count() * GSS_WALK_GRID));
    if (host_resident(a) && vector_rows(a) && host_staging() && !(split && split->mask)) {
      staged_walk<K, MODE>(a, gd, *L, tl, st);
      return;
    }
    if (host_resident(a)) wblocks = std::min(wblocks, host_walk_blocks());  // reads + writes in flight
    if (split && split->mask && vector_rows(a)) {
      TouchList ta = tl, tb = tl;
      ta.filter = tb.filter = split->mask;
      ta.want = 0;
      tb.want = 1;
      walk4_kernel<K, MODE><<<wblocks, kUpdThreads, 0, st>>>(arena_dev(a), gd, *L, ta);
      GSS_LAUNCHED();
      if (split->before_set) GSS_CUDA(cudaStreamWaitEvent(st, split->before_set, 0));
      walk4_kernel<K, MODE><<<wblocks, kUpdThreads, 0, st>>>(arena_dev(a), gd, *L, tb);
      GSS_LAUNCHED();
      return;
    }
    if (vector_rows(a))
      walk4_kernel<K, MODE><<<wblocks, kUpdThreads, 0, st>>>(arena_dev(a), gd, *L, tl);
    else
      walk_kernel<K, MODE><<<wblocks, kUpdThreads, 0, st>>>(arena_dev(a), gd, *L, tl);
    GSS_LAUNCHED();
  }
}

struct IsSet {
  const uint32_t* mask;
  __device__ bool operator()(int32_t i) const { return (mask[i >> 5] >> (i & 31)) & 1u; }
};

}  // namespace

std::mutex g_flag_mu;
std::unordered_map<const void*, int*> g_flags;

namespace {
int* err_flag_for(const gss_arena& a) {
  std::lock_guard<std::mutex> lk(g_flag_mu);
  auto it = g_flags.find(a.counter);
  if (it != g_flags.end()) return it->second;
  // [0] sticky error flag; [2..3] / [4..5]: device tallies (touched rows / restored rows, u64)
  int* f = nullptr;
  GSS_CUDA(cudaMalloc(&f, 32));
  GSS_CUDA(cudaMemset(f, 0, 32));
  g_flags[a.counter] = f;
  return f;
}
unsigned long long* tally_dev(const gss_arena& a) {
  return reinterpret_cast<unsigned long long*>(err_flag_for(a) + 2);
}

// AccessReport (adam.hpp:36-50): host-known parts per arena (keyed like the flag); the device parts
// (touched rows of a deferred pass, restored rows of a device-counted view) accumulate in the meta
// block and are folded in by arena_access.
struct HostTally {
  uint64_t passes = 0, touched = 0, param_bytes = 0, counter_bytes = 0, restore_rows = 0, restore_bytes = 0;
};
std::unordered_map<const void*, HostTally> g_tally;  // guarded by g_flag_mu

}  // namespace

void adam_update(gss_arena* ap, const gss_sparse_grads* grads, int32_t* touched_ids, int64_t* touched_count,
                 cudaStream_t st, const uint32_t* split_mask, cudaEvent_t split_before_set) {
  require(ap != nullptr, "arena: null");
  gss_arena& a = *ap;
  validate_arena(a);
  const int64_t t = a.step + 1;
  const GradsDev gd = grads_dev(grads, a.dim);
  require(gd.count >= 0, "sparse grads: negative count");
  require(gd.count == 0 || gd.count_dev || (gd.ids && gd.rows), "sparse grads: null ids/rows");
  require(gd.col0 >= 0, "sparse grads: negative col0");
  if (touched_count) GSS_CUDA(cudaMemsetAsync(touched_count, 0, sizeof(int64_t), st));
  if (a.n == 0) {
    a.step = t;
    return;
  }
  uint32_t* tmask = nullptr;
  if (touched_ids) GSS_CUDA(cudaMallocAsync((void**)&tmask, (size_t)ceil_div(a.n, 32) * 4, st));
  WalkSplit ws;
  ws.mask = split_mask;
  ws.before_set = split_before_set;
  if (a.defer_max < 16)
    launch_update<16, kDeferred>(a, gd, t, tmask, touched_count, st, split_mask ? &ws : nullptr);
  else
    launch_update<256, kDeferred>(a, gd, t, tmask, touched_count, st, split_mask ? &ws : nullptr);
  if (touched_ids) {
    // Ascending touched ids from the per-row bit mask (stable device select).
    size_t tb = 0;
    void* tmp = nullptr;
    IsSet pred{tmask};
    int64_t* nsel = touched_count;
    int64_t* scratch_cnt = nullptr;
    if (!nsel) {
      GSS_CUDA(cudaMallocAsync((void**)&scratch_cnt, sizeof(int64_t), st));
      nsel = scratch_cnt;
    }
    thrust::counting_iterator<int32_t> it(0);
    GSS_CUDA(cub::DeviceSelect::If(nullptr, tb, it, touched_ids, nsel, (int)a.n, pred, st));
    GSS_CUDA(cudaMallocAsync(&tmp, tb, st));
    GSS_CUDA(cub::DeviceSelect::If(tmp, tb, it, touched_ids, nsel, (int)a.n, pred, st));
    count_launch();
    GSS_CUDA(cudaFreeAsync(tmp, st));
    GSS_CUDA(cudaFreeAsync(tmask, st));
    if (scratch_cnt) GSS_CUDA(cudaFreeAsync(scratch_cnt, st));
  }
  a.step = t;
}

namespace {
// adam_step_dense (adam.hpp:198-207): flat streaming over n*dim with d = 0 (restoration term
// w -= (0*m)/(sqrt(v)+eps) kept for bitwise parity); counters untouched.
template <int K>
__global__ void __launch_bounds__(kUpdThreads) dense_kernel(ArenaDev a, const float* grads,
                                                            const __grid_constant__ LutArgs<K> L) {
  __shared__ SmemLuts<K> lut;
  load_luts<K>(lut, L, a.dim);
  __syncthreads();
  const int64_t total = a.n * a.dim;
  for (int64_t f = blockIdx.x * (int64_t)kUpdThreads + threadIdx.x; f < total; f += (int64_t)gridDim.x * kUpdThreads) {
    const int64_t row = f / a.dim;
    const int c = (int)(f - row * a.dim);
    const int g = lut.col_group[c];
    const int64_t o = row * a.stride + c;
    float w = a.w[o], m = a.m[o], v = a.v[o];
    deferred_scalar(w, m, v, grads ? grads[f] : 0.0f, lut.param[g][0], lut.a1[g][0], lut.a2[g][0], lut.sc[g]);
    a.w[o] = w;
    a.m[o] = m;
    a.v[o] = v;
  }
}
}  // namespace

void adam_dense(gss_arena* ap, const float* grads, cudaStream_t st) {
  require(ap != nullptr, "arena: null");
  gss_arena& a = *ap;
  validate_arena(a);
  const int64_t t = a.step + 1;
  a.step = t;
  if (a.n == 0) return;
  auto L = std::make_unique<LutArgs<16>>();
  std::memset(L.get(), 0, sizeof(LutArgs<16>));
  gss_arena a0 = a;
  a0.defer_max = 0;  // only delay 0 is read
  fill_luts<16>(a0, t, false, *L);
  int dev = 0, sms = 148;
  GSS_CUDA(cudaGetDevice(&dev));
  GSS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t blocks = std::min<int64_t>(ceil_div(a.n * a.dim, kUpdThreads), (int64_t)sms * 8);
  dense_kernel<16><<<(int)blocks, kUpdThreads, 0, st>>>(arena_dev(a), grads, *L);
  GSS_LAUNCHED();
  tally_host(a, kDenseTally, a.n);
}

void adam_flush(gss_arena* ap, cudaStream_t st) {
  require(ap != nullptr, "arena: null");
  gss_arena& a = *ap;
  validate_arena(a);
  if (a.n == 0) return;
  const int64_t t = a.step + 1;
  if (a.defer_max < 16)
    launch_update<16, kFlush>(a, GradsDev{}, t, nullptr, nullptr, st);
  else
    launch_update<256, kFlush>(a, GradsDev{}, t, nullptr, nullptr, st);
}

// Split restore_view for row-interleaved arenas: a resolve pass turns each visible id into its
// (pending slot, delay) once — the counter byte and a binary search of the pending ids within the
// id's 1024-row block (index bstart) — and the walk pass then streams the rows with no barriers or
// per-chunk prologue, each warp 32 ids at a time in 16-byte units (as walk4_kernel).
#ifndef GSS_RESTORE_SPLIT
#define GSS_RESTORE_SPLIT 1
#endif
__global__ void restore_resolve_kernel(ArenaDev a, const int32_t* ids, int64_t count, const int64_t* count_dev,
                                       GradsDev pend, const int32_t* pbstart, int2* res) {
  const int64_t cnt = count_dev ? *count_dev : count;
  const int64_t pcnt = pend.ids ? grads_count(pend) : 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cnt; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t id = ids[k];
    int32_t slot = -1;
    if (pcnt > 0) {
      const int64_t b = id / kRowsPerBlock;
      int64_t lo = pbstart[b], hi = pbstart[b + 1];
      lo = lo < 0 ? 0 : lo;
      hi = hi > pcnt ? pcnt : hi;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (pend.ids[mid] < id) lo = mid + 1; else hi = mid;
      }
      if (lo < pcnt && pend.ids[lo] == id) slot = (int32_t)lo;
    }
    res[k] = make_int2(slot, (int)a.counter[id]);
  }
}

template <int K>
__global__ void __launch_bounds__(kUpdThreads, GSS_RESTORE_MINB) restore_walk_kernel(
    ArenaDev a, const int32_t* ids, int64_t count, const int64_t* count_dev, GradsDev pend, const int2* res,
    int has_pending, const __grid_constant__ LutArgs<K> L, float* out) {
  __shared__ PackedLuts<K> lut;
  load_packed_luts<K>(lut, L, a.dim);
  __syncthreads();
  const int64_t cnt = count_dev ? *count_dev : count;
  const int dim = a.dim;
  const int lane = threadIdx.x & 31;
  const int nq = (dim + 3) >> 2;
  const int dq = 32 / nq, dr = 32 - dq * nq;
  const int64_t warps = (int64_t)gridDim.x * (kUpdThreads / 32);
  for (int64_t k0 = (blockIdx.x * (int64_t)(kUpdThreads / 32) + (threadIdx.x >> 5)) * 32; k0 < cnt; k0 += warps * 32) {
    const int64_t j = k0 + lane;
    int64_t my_base = -1;
    int2 my_res = make_int2(-1, 0);
    if (j < cnt) {
      my_base = (a.positional ? j : (int64_t)ids[j]) * a.stride;
      my_res = res[j];
    }
    int r = lane / nq, q = lane - (lane / nq) * nq;
    constexpr int kV = GSS_RESTORE_KV;
    for (int i0 = 0; i0 < nq; i0 += kV) {
      float4 w[kV], m[kV], v[kV];
      float gv[kV][4];
      int dd[kV], c0[kV], rr4[kV];
      bool ok[kV];
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        const int rr = r < 32 ? r : 31;
        const int64_t base = __shfl_sync(0xffffffffu, my_base, rr);
        const int32_t sl = has_pending ? __shfl_sync(0xffffffffu, my_res.x, rr) : -1;
        dd[u] = __shfl_sync(0xffffffffu, my_res.y, rr);
        c0[u] = 4 * q;
        rr4[u] = rr;
        ok[u] = i0 + u < nq && base >= 0;
        const int64_t o = ok[u] ? base + c0[u] : 0;
        w[u] = ok[u] ? ld4(a.w + o) : make_float4(0.f, 0.f, 0.f, 0.f);
        m[u] = ok[u] ? ld4(a.m + o) : make_float4(0.f, 0.f, 0.f, 0.f);
        v[u] = ok[u] ? ld4(a.v + o) : make_float4(0.f, 0.f, 0.f, 0.f);
        grad_unit(pend, sl, c0[u], dim, ok[u], gv[u]);
        r += dq;
        q += dr;
        if (q >= nq) {
          q -= nq;
          ++r;
        }
      }
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        if (!ok[u]) continue;
        float* orow = out + (size_t)(k0 + rr4[u]) * dim + c0[u];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (c0[u] + i >= dim) break;
          const int g = lut.col_group[c0[u] + i];
          const float4 gd = lut.gd[g][dd[u]];
          float ww = at(w[u], i);
          if (has_pending) {
            float mm = at(m[u], i), vv = at(v[u], i);
            deferred_scalar_fast(ww, mm, vv, gv[u][i], gd, lut.sc[g], lut.eps[g]);
          } else {
            const float num = gd.x * at(m[u], i);
            ww = (num == 0.0f && at(v[u], i) >= 0.0f) ? ww - num
                                                      : ww - div_rn(num, sqrt_rn(at(v[u], i)) + lut.eps[g]);
          }
          orow[i] = ww;
        }
      }
    }
  }
}

void adam_restore(const gss_arena* ap, const int32_t* ids, int64_t count, const int64_t* count_dev,
                  const gss_sparse_grads* pending, float* out, cudaStream_t st, cudaEvent_t after_resolve) {
  require(ap != nullptr, "arena: null");
  const gss_arena& a = *ap;
  validate_arena(a);
  require(count >= 0, "restore_view: negative count");
  require(count == 0 || count_dev || (ids && out), "restore_view: null ids/out");
  if (count == 0 && !count_dev) return;
  const int64_t t = a.step + 1;
  GradsDev pd = grads_dev(pending, a.dim);
  if (count_dev) {  // adam.hpp:287-288 with a device-side row count
    tally_add_kernel<<<1, 1, 0, st>>>(tally_dev(a) + 1, nullptr, count_dev);
    GSS_LAUNCHED();
  } else {
    tally_host(a, kRestoreTally, count);
  }
  int dev = 0, sms = 148;
  GSS_CUDA(cudaGetDevice(&dev));
  GSS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t cap = count_dev ? std::max<int64_t>(count, a.n) : count;
  int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap, kRestoreChunk), (int64_t)sms * 64));
  if (host_resident(a)) blocks = std::min(blocks, host_tier_blocks());
  const size_t pb_bytes = ((size_t)(ceil_div(a.n, kRowsPerBlock) + 1) * 4 + 255) / 256 * 256;
  const bool host = host_resident(a);
  // Host tier with a host-known row count: gather the rows into HBM staging over the link first,
  // then restore from the staged copy (see move_rows_kernel).
  const bool staged = host && vector_rows(a) && a.defer_max < 16 && !count_dev && host_staging();
  // (after_resolve: the caller orders a counter update after the resolve pass: split path always)
  const bool split = GSS_RESTORE_SPLIT && vector_rows(a) && a.defer_max < 16 && (!host || staged || after_resolve);
  char* scr = arena_scratch(a, 1, pb_bytes + (split ? (size_t)std::max<int64_t>(cap, 1) * sizeof(int2) : 0), st);
  int32_t* pbstart = nullptr;
  if (pending && pd.ids) pbstart = build_index(a, pd, err_flag_for(a), reinterpret_cast<int32_t*>(scr), st);
  if (staged) {
    float* stage =
        reinterpret_cast<float*>(arena_scratch(a, 3, (size_t)std::max<int64_t>(count, 1) * stage_stride(a.dim) * 4, st));
    for (int64_t c0 = 0; c0 < count; c0 += int64_t(1) << 25) {  // 32-bit unit indices per launch
      const int64_t c1 = std::min<int64_t>(count, c0 + (int64_t(1) << 25));
      move_rows_kernel<true><<<kMoveBlocks, 256, 0, st>>>(arena_dev(a), ids, c0, c1,
                                                          stage + c0 * stage_stride(a.dim));
      GSS_LAUNCHED();
    }
    int2* res = reinterpret_cast<int2*>(scr + pb_bytes);
    auto L = std::make_unique<LutArgs<16>>();
    std::memset(L.get(), 0, sizeof(LutArgs<16>));
    fill_luts<16>(a, t, false, *L);
    const int rb = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap, 256), (int64_t)sms * 16));
    restore_resolve_kernel<<<rb, 256, 0, st>>>(arena_dev(a), ids, count, nullptr, pd, pbstart, res);
    GSS_LAUNCHED();
    const int wb = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap, kUpdThreads), (int64_t)sms * GSS_RESTORE_MINB));
    restore_walk_kernel<16><<<wb, kUpdThreads, 0, st>>>(staged_arena(a, stage), ids, count, nullptr, pd, res,
                                                         pending ? 1 : 0, *L, out);
  } else if (split) {
    int2* res = reinterpret_cast<int2*>(scr + pb_bytes);
    auto L = std::make_unique<LutArgs<16>>();
    std::memset(L.get(), 0, sizeof(LutArgs<16>));
    fill_luts<16>(a, t, false, *L);
    const int rb = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap, 256), (int64_t)sms * 16));
    restore_resolve_kernel<<<rb, 256, 0, st>>>(arena_dev(a), ids, count, count_dev, pd, pbstart, res);
    GSS_LAUNCHED();
    if (after_resolve) GSS_CUDA(cudaEventRecord(after_resolve, st));
    int wb = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap, kUpdThreads), (int64_t)sms * GSS_RESTORE_MINB));
    if (host) wb = std::min(wb, host_tier_blocks());
    restore_walk_kernel<16><<<wb, kUpdThreads, 0, st>>>(arena_dev(a), ids, count, count_dev, pd, res, pending ? 1 : 0,
                                                         *L, out);
  } else if (a.defer_max < 16) {
    auto L = std::make_unique<LutArgs<16>>();
    std::memset(L.get(), 0, sizeof(LutArgs<16>));
    fill_luts<16>(a, t, false, *L);
    restore_kernel<16><<<blocks, kUpdThreads, 0, st>>>(arena_dev(a), ids, count, count_dev, pd, pbstart,
                                                       pending ? 1 : 0, *L, out, vector_rows(a) ? 1 : 0);
  } else {
    auto L = std::make_unique<LutArgs<256>>();
    std::memset(L.get(), 0, sizeof(LutArgs<256>));
    fill_luts<256>(a, t, false, *L);
    restore_kernel<256><<<blocks, kUpdThreads, 0, st>>>(arena_dev(a), ids, count, count_dev, pd, pbstart,
                                                        pending ? 1 : 0, *L, out, vector_rows(a) ? 1 : 0);
  }
  GSS_LAUNCHED();
}

// Frees the per-arena scratch and error flag (keyed by the counter buffer). Called when an arena's
// buffers are released, so a later arena at a recycled address starts with a clean flag and the
// maps stay bounded by the live arenas.
void arena_release(const gss_arena* ap) {
  if (!ap || !ap->counter) return;
  GSS_CUDA(cudaDeviceSynchronize());
  {
    std::lock_guard<std::mutex> lk(g_scr_mu);
    for (auto& m : g_scr) {
      auto it = m.find(ap->counter);
      if (it != m.end()) {
        if (it->second.first) GSS_CUDA(cudaFree(it->second.first));
        m.erase(it);
      }
    }
  }
  std::lock_guard<std::mutex> lk(g_flag_mu);
  auto it = g_flags.find(ap->counter);
  if (it != g_flags.end()) {
    GSS_CUDA(cudaFree(it->second));
    g_flags.erase(it);
  }
  g_tally.erase(ap->counter);
}

namespace {
void tally_host(const gss_arena& a, int kind, int64_t rows) {
  std::lock_guard<std::mutex> lk(g_flag_mu);
  HostTally& t = g_tally[a.counter];
  const uint64_t r = (uint64_t)std::max<int64_t>(rows, 0), dim = (uint64_t)a.dim;
  if (kind == kRestoreTally) {
    t.restore_rows += r;
    t.restore_bytes += r * 4u * dim * 4u;  // adam.hpp:287-288
    return;
  }
  t.passes += 1;
  t.touched += r;
  t.param_bytes += r * 7u * dim * 4u;  // adam.hpp:204-206, 233-235
  if (kind == kDeferred) t.counter_bytes += (uint64_t)a.n;
}
}  // namespace

// AccessReport of the arena (adam.hpp:36-50): update_passes, touched_rows, param_bytes,
// counter_bytes, restore_rows, restore_read_bytes (synchronises the device).
void arena_access(const gss_arena* ap, uint64_t* out6) {
  require(ap != nullptr && out6 != nullptr, "arena_access: null argument");
  const gss_arena& a = *ap;
  unsigned long long dv[2] = {0, 0};
  unsigned long long* td = tally_dev(a);
  GSS_CUDA(cudaDeviceSynchronize());
  GSS_CUDA(cudaMemcpy(dv, td, sizeof dv, cudaMemcpyDeviceToHost));
  std::lock_guard<std::mutex> lk(g_flag_mu);
  const HostTally t = g_tally[a.counter];
  const uint64_t dim = (uint64_t)a.dim;
  out6[0] = t.passes;
  out6[1] = t.touched + dv[0];
  out6[2] = t.param_bytes + dv[0] * 7u * dim * 4u;
  out6[3] = t.counter_bytes;
  out6[4] = t.restore_rows + dv[1];
  out6[5] = t.restore_bytes + dv[1] * 4u * dim * 4u;
}

int arena_check(const gss_arena* ap, cudaStream_t st) {
  require(ap != nullptr, "arena: null");
  int* f = err_flag_for(*ap);
  int h = 0;
  GSS_CUDA(cudaMemcpyAsync(&h, f, sizeof(int), cudaMemcpyDeviceToHost, st));
  GSS_CUDA(cudaStreamSynchronize(st));
  GSS_CUDA(cudaMemsetAsync(f, 0, sizeof(int), st));
  if (h & 1) throw Error(GSS_ERR_INVARIANT, "deferred_update: gradient ids not sorted or out of range");
  if (h & 2) throw Error(GSS_ERR_INVARIANT, "arena: defer counter out of range");
  return 0;
}

void set_host_chunk_bytes(int64_t bytes) {
  if (bytes > 0) g_host_chunk_bytes.store(bytes);
}

}  // namespace gssd
