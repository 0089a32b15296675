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

#include <cmath>
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
};

struct GradsDev {
  const int32_t* ids;
  int64_t count;
  const int64_t* count_dev;
  const float* rows;
  int64_t stride;
  int col0;
};

__device__ __forceinline__ int64_t grads_count(const GradsDev& g) { return g.count_dev ? *g.count_dev : g.count; }

__device__ __forceinline__ int64_t lower_bound_ids(const int32_t* ids, int64_t n, int64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)ids[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// deferred_scalar (adam.hpp:102-110)
__device__ __forceinline__ void deferred_scalar(float& w, float& m, float& v, float g, float ws, float ms, float vs,
                                                const float* sc) {
  const float m_new = ms * m + sc[0] * g;
  const float v_new = vs * v + sc[1] * g * g;
  w -= (ws * m) / (sqrtf(v) + sc[4]);
  const float denom = sqrtf(v_new) / sc[2] + sc[4];
  w = w - sc[3] * m_new / denom;
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

// One pass of deferred_update (adam.hpp:211-238) or flush_deferred (adam.hpp:293-313) over
// rows [blockIdx*1024, +1024). Dense Adam (adam.hpp:198-207) is the deferred pass of an arena
// whose counters stay 0 with defer_max 0 (every row saturated, delay 0).
template <int K, int MODE>
__global__ void __launch_bounds__(kUpdThreads) update_kernel(ArenaDev a, GradsDev gr,
                                                             const __grid_constant__ LutArgs<K> L,
                                                             uint32_t* touched_mask, int64_t* touched_count,
                                                             int* err_flag) {
  __shared__ SmemLuts<K> lut;
  __shared__ int32_t slot_of[kRowsPerBlock];
  __shared__ uint16_t trow[kRowsPerBlock];
  __shared__ uint8_t tdel[kRowsPerBlock];
  __shared__ int32_t tslot[kRowsPerBlock];
  __shared__ int warp_tot[kUpdThreads / 32];
  __shared__ long long g_lo, g_hi;
  __shared__ int ntouched;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerBlock;
  const int nrows = (int)((a.n - r0) < kRowsPerBlock ? (a.n - r0) : kRowsPerBlock);
  load_luts<K>(lut, L, a.dim);
  for (int i = tid; i < kRowsPerBlock; i += kUpdThreads) slot_of[i] = -1;
  const int64_t gcount = MODE == kDeferred ? grads_count(gr) : 0;
  if (MODE == kDeferred && tid < 2 && gr.ids) {
    const int64_t b = lower_bound_ids(gr.ids, gcount, r0 + (tid == 0 ? 0 : kRowsPerBlock));
    if (tid == 0) g_lo = b; else g_hi = b;
  }
  __syncthreads();
  if (MODE == kDeferred && gr.ids) {
    const int64_t lo = g_lo, hi = g_hi;
    for (int64_t k = lo + tid; k < hi; k += kUpdThreads) {
      const int64_t local = (int64_t)gr.ids[k] - r0;
      if (local >= 0 && local < kRowsPerBlock) slot_of[local] = (int32_t)k;
    }
    // Sortedness / range invariant (adam.hpp:231): this block checks its share of the id list.
    const int64_t per = (gcount + gridDim.x - 1) / gridDim.x;
    const int64_t k0 = (int64_t)blockIdx.x * per, k1 = (gcount < k0 + per ? gcount : k0 + per);
    for (int64_t k = k0 + tid; k < k1; k += kUpdThreads) {
      const int32_t id = gr.ids[k];
      if (id < 0 || (int64_t)id >= a.n || (k + 1 < gcount && gr.ids[k + 1] <= id)) atomicOr(err_flag, 1);
    }
  }
  __syncthreads();
  // Counter pass: 4 consecutive rows per thread.
  int my_cnt = 0;
  uint8_t del[4];
  bool tch[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int r = tid * 4 + j;
    tch[j] = false;
    del[j] = 0;
    if (r < nrows) {
      const uint8_t c = a.counter[r0 + r];
      if (c > a.defer_max) atomicOr(err_flag, 2);  // check_counters (adam.hpp:154-158)
      bool t;
      if (MODE == kDeferred) {
        t = slot_of[r] >= 0 || c == a.defer_max;
        a.counter[r0 + r] = t ? 0 : (uint8_t)(c + 1);
      } else {
        t = c != 0;
        if (t) a.counter[r0 + r] = 0;
      }
      tch[j] = t;
      del[j] = c;
      my_cnt += t;
    }
  }
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
  int pos = warp_tot[warp] + inc - my_cnt;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (tch[j]) {
      const int r = tid * 4 + j;
      trow[pos] = (uint16_t)r;
      tdel[pos] = del[j];
      tslot[pos] = slot_of[r];
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
  __syncthreads();
  const int T = ntouched;
  if (touched_count && tid == 0 && T > 0) atomicAdd((unsigned long long*)touched_count, (unsigned long long)T);
  const int dim = a.dim;
  const int total = T * dim;
  // Flattened (touched row, column) walk: consecutive lanes take consecutive columns.
#pragma unroll 4
  for (int f = tid; f < total; f += kUpdThreads) {
    const int t = (int)__umulhi((uint32_t)f, a.div_magic);
    const int c = f - t * dim;
    const int64_t row = r0 + trow[t];
    const int d = tdel[t];
    const int g = lut.col_group[c];
    const size_t off = (size_t)row * dim + c;
    float w = a.w[off], m = a.m[off], v = a.v[off];
    if (MODE == kDeferred) {
      const int s = tslot[t];
      const float gv = s >= 0 ? gr.rows[(size_t)s * gr.stride + gr.col0 + c] : 0.0f;
      deferred_scalar(w, m, v, gv, lut.param[g][d], lut.a1[g][d], lut.a2[g][d], lut.sc[g]);
      a.w[off] = w;
      a.m[off] = m;
      a.v[off] = v;
    } else {
      a.w[off] = w - (lut.param[g][d] * m) / (sqrtf(v) + lut.sc[g][4]);  // restore_scalar (adam.hpp:112-114)
      a.m[off] = m * lut.a1[g][d];
      a.v[off] = v * lut.a2[g][d];
    }
  }
}

// restore_view (adam.hpp:252-289): out[k] = restored row ids[k] (+ pending pass). Persistent
// grid-stride over 128-id chunks; per chunk, one thread per id resolves (id, delay, pending
// slot) by binary search, then the flattened (id, column) walk reads the arena rows.
constexpr int kRestoreChunk = 128;
template <int K>
__global__ void __launch_bounds__(kUpdThreads) restore_kernel(ArenaDev a, const int32_t* ids, int64_t count,
                                                              const int64_t* count_dev, GradsDev pend,
                                                              int has_pending, const __grid_constant__ LutArgs<K> L,
                                                              float* out) {
  __shared__ SmemLuts<K> lut;
  __shared__ int32_t cid[kRestoreChunk];
  __shared__ uint8_t cdel[kRestoreChunk];
  __shared__ int32_t cslot[kRestoreChunk];
  load_luts<K>(lut, L, a.dim);
  const int64_t cnt = count_dev ? *count_dev : count;
  const int64_t pcnt = has_pending ? grads_count(pend) : 0;
  const int dim = a.dim;
  for (int64_t k0 = (int64_t)blockIdx.x * kRestoreChunk; k0 < cnt; k0 += (int64_t)gridDim.x * kRestoreChunk) {
    const int nk = (int)((cnt - k0) < kRestoreChunk ? (cnt - k0) : kRestoreChunk);
    __syncthreads();
    if (threadIdx.x < nk) {
      const int32_t id = ids[k0 + threadIdx.x];
      cid[threadIdx.x] = id;
      cdel[threadIdx.x] = a.counter[id];
      int32_t s = -1;
      if (has_pending && pend.ids) {
        const int64_t p = lower_bound_ids(pend.ids, pcnt, id);
        if (p < pcnt && pend.ids[p] == id) s = (int32_t)p;
      }
      cslot[threadIdx.x] = s;
    }
    __syncthreads();
    const int total = nk * dim;
#pragma unroll 4
    for (int f = threadIdx.x; f < total; f += kUpdThreads) {
      const int t = (int)__umulhi((uint32_t)f, a.div_magic);
      const int c = f - t * dim;
      const size_t off = (size_t)cid[t] * dim + c;
      const int d = cdel[t];
      const int g = lut.col_group[c];
      float w = a.w[off];
      const float m = a.m[off], v = a.v[off];
      if (has_pending) {
        float mm = m, vv = v;
        const int s = cslot[t];
        const float gv = s >= 0 ? pend.rows[(size_t)s * pend.stride + pend.col0 + c] : 0.0f;
        deferred_scalar(w, mm, vv, gv, lut.param[g][d], lut.a1[g][d], lut.a2[g][d], lut.sc[g]);
      } else {
        w = w - (lut.param[g][d] * m) / (sqrtf(v) + lut.sc[g][4]);
      }
      out[(size_t)(k0 + t) * dim + c] = w;
    }
  }
}

ArenaDev arena_dev(const gss_arena& a) {
  ArenaDev d;
  d.w = a.w; d.m = a.m; d.v = a.v; d.counter = a.counter;
  d.n = a.n; d.dim = a.dim; d.defer_max = a.defer_max;
  d.div_magic = (uint32_t)((((uint64_t)1 << 32) + (uint64_t)a.dim - 1) / (uint64_t)a.dim);
  return d;
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
  require(a.n == 0 || (a.w && a.m && a.v && a.counter), "arena: null buffer");
}

GradsDev grads_dev(const gss_sparse_grads* g) {
  GradsDev d{};
  if (g) {
    d.ids = g->ids; d.count = g->count; d.count_dev = g->count_dev; d.rows = g->rows;
    d.stride = g->stride; d.col0 = g->col0;
  }
  return d;
}

// Per-arena device error flag (keyed by the counter buffer), allocated lazily.
int* err_flag_for(const gss_arena& a);

template <int K, int MODE>
void launch_update(const gss_arena& a, const GradsDev& gd, int64_t t, uint32_t* tmask, int64_t* tcount,
                   cudaStream_t st) {
  auto L = std::make_unique<LutArgs<K>>();
  std::memset(L.get(), 0, sizeof(LutArgs<K>));
  fill_luts<K>(a, t, MODE == kFlush, *L);
  const int blocks = (int)ceil_div(a.n, kRowsPerBlock);
  update_kernel<K, MODE><<<blocks, kUpdThreads, 0, st>>>(arena_dev(a), gd, *L, tmask, tcount, err_flag_for(a));
  GSS_LAUNCHED();
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
  int* f = nullptr;
  GSS_CUDA(cudaMalloc(&f, sizeof(int)));
  GSS_CUDA(cudaMemset(f, 0, sizeof(int)));
  g_flags[a.counter] = f;
  return f;
}
}  // namespace

void adam_update(gss_arena* ap, const gss_sparse_grads* grads, int32_t* touched_ids, int64_t* touched_count,
                 cudaStream_t st) {
  require(ap != nullptr, "arena: null");
  gss_arena& a = *ap;
  validate_arena(a);
  const int64_t t = a.step + 1;
  const GradsDev gd = grads_dev(grads);
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
  if (a.defer_max < 16)
    launch_update<16, kDeferred>(a, gd, t, tmask, touched_count, st);
  else
    launch_update<256, kDeferred>(a, gd, t, tmask, touched_count, st);
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
    float w = a.w[f], m = a.m[f], v = a.v[f];
    deferred_scalar(w, m, v, grads ? grads[f] : 0.0f, lut.param[g][0], lut.a1[g][0], lut.a2[g][0], lut.sc[g]);
    a.w[f] = w;
    a.m[f] = m;
    a.v[f] = v;
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

void adam_restore(const gss_arena* ap, const int32_t* ids, int64_t count, const int64_t* count_dev,
                  const gss_sparse_grads* pending, float* out, cudaStream_t st) {
  require(ap != nullptr, "arena: null");
  const gss_arena& a = *ap;
  validate_arena(a);
  require(count >= 0, "restore_view: negative count");
  require(count == 0 || count_dev || (ids && out), "restore_view: null ids/out");
  if (count == 0 && !count_dev) return;
  const int64_t t = a.step + 1;
  GradsDev pd = grads_dev(pending);
  int dev = 0, sms = 148;
  GSS_CUDA(cudaGetDevice(&dev));
  GSS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t cap = count_dev ? std::max<int64_t>(count, a.n) : count;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap, kRestoreChunk), (int64_t)sms * 8));
  if (a.defer_max < 16) {
    auto L = std::make_unique<LutArgs<16>>();
    std::memset(L.get(), 0, sizeof(LutArgs<16>));
    fill_luts<16>(a, t, false, *L);
    restore_kernel<16><<<blocks, kUpdThreads, 0, st>>>(arena_dev(a), ids, count, count_dev, pd, pending ? 1 : 0, *L,
                                                       out);
  } else {
    auto L = std::make_unique<LutArgs<256>>();
    std::memset(L.get(), 0, sizeof(LutArgs<256>));
    fill_luts<256>(a, t, false, *L);
    restore_kernel<256><<<blocks, kUpdThreads, 0, st>>>(arena_dev(a), ids, count, count_dev, pd, pending ? 1 : 0,
                                                        *L, out);
  }
  GSS_LAUNCHED();
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

}  // namespace gssd
