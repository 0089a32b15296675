// Frustum cull + stream compaction: the B200 replacement of frustum_cull / cull_keep
// (render.hpp:243-260, with project_geo render.hpp:90-148 inside).
//
// Design (cull):
//  * Persistent CTAs (3 per SM), each owning a CONTIGUOUS range of 512-row tiles streamed
//    HBM->SMEM through a 3-stage ring of TMA bulk copies (cp.async.bulk + mbarrier, 20 KB each).
//    There is no block barrier per tile: the last warp done with a stage refills it.
//  * Classification per row: the camera transform, depth test, 1/z and the projected centre are
//    the reference's own arithmetic (bit-identical); the 3-sigma radius is replaced by a rigorous
//    upper bound on approximate math. A centre farther outside than the bound is culled; a centre
//    inside the closed viewport with a certified-finite covariance is kept (mx + r >= mx >= x0).
//    The rest (straddlers, uncertified rows) are queued in SMEM and resolved after the last tile
//    by the exact reference projection (IEEE div/sqrt, no contraction, glibc expf in fp64), all
//    threads in parallel. The kept set is therefore bit-identical to the CPU reference.
//  * Compaction: warp ballots give the mask words, kept in SMEM for the CTA's whole range; the CTA
//    then publishes its aggregate and sums all predecessors' aggregates in parallel (CTAs are
//    dispatched in blockIdx order and never wait on successors), and scatters its ascending ids.
//    Round-1 history (profiles/): a ticket-ordered per-tile look-back with tiles claimed four
//    ahead chained every CTA behind its predecessor's queue (6% of HBM peak); one CTA per tile
//    bounded the inclusive-prefix frontier at ~32 tiles per L2 round trip (2x slower than this).
//  * Look-back states carry a per-workspace epoch kept by the host, so the workspace is zeroed
//    once and never memset again.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "gss_math.cuh"

namespace gssd {
namespace {

constexpr int kTile = 512;
#ifndef CULL_THREADS
#define CULL_THREADS 256
#endif
constexpr int kThreads = CULL_THREADS;
#ifndef CULL_STAGES
#define CULL_STAGES 3
#endif
#ifndef CULL_CTAS_PER_SM
#define CULL_CTAS_PER_SM 3
#endif
constexpr int kStages = CULL_STAGES;
constexpr int kCtasPerSm = CULL_CTAS_PER_SM;
constexpr int kMaxTiles = 128;  // tiles per CTA (mask words kept in SMEM: 128 * 16 words)
constexpr int kDefer = 128;     // undecided rows queued per CTA
constexpr int kGeo = 10;
constexpr int kWordsPerTile = kTile / 32;
constexpr uint32_t kTileBytes = kTile * kGeo * 4;  // 20480

// Look-back state: [63:62] flag (1 = aggregate published), [61:32] epoch, [31:0] value.
constexpr unsigned long long kFlagAgg = 1ull;

struct WsHeader {  // reserved (256 B ahead of the look-back states)
  unsigned int pad[64];
};

struct CullArgs {
  Cam cam;
  float x0, x1, y0, y1, lp;
  float wn[3];   // row norms of the camera rotation (inflated)
  float wmax;    // max |W_ij|
  int all_exact; // lp outside [0, 1e30]: the fast bounds do not apply
  const float* geo;
  int64_t n, stride, ntiles;
  int tiles_per_cta;
  int64_t nwords;
  unsigned epoch;
  uint32_t* mask;
  int32_t* ids;
  int64_t* count;
  unsigned long long* state;
};

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// cull_keep (render.hpp:243-251), exact.
__device__ __forceinline__ bool keep_exact(const CullArgs& a, const float* g) {
  const f3 t = to_camera(a.cam, g[0], g[1], g[2]);
  if (!(t.z >= a.cam.near_plane && t.z <= a.cam.far_plane)) return false;
  Proj p;
  f3 t2;
  if (!project_geo(a.cam, g, a.lp, p, t2)) return false;
  return p.mx + p.radius >= a.x0 && p.mx - p.radius <= a.x1 && p.my + p.radius >= a.y0 && p.my - p.radius <= a.y1;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float max_nan(float a, float b) {  // NaN-propagating max
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// 0 = cull, 1 = keep, 2 = undecided (needs keep_exact). Decisions 0/1 are proven equal to
// keep_exact:
//  * the camera transform, depth test, 1/z (IEEE reciprocal) and projected centre are the
//    reference's own arithmetic (render.hpp:93-98, scene.hpp:85), so mx, my are bit-identical;
//  * only the radius is bounded: lmax <= cov_a + cov_c <= (|m0|^2 + |m1|^2) max(es)^2 + 2 lp with
//    |m0| <= |j00| |W0| + |j02| |W2| (row norms: valid for any W), inflated 2% for the
//    reference's float rounding and the approximate exp/sqrt. As r_ref <= r_ub and rounding is
//    monotonic, fl(mx + r_ub) < x0 implies fl(mx + r_ref) < x0. CULL needs no certificate: a NaN
//    reference radius culls as well, and r_ub <= 1e15 rules out a reference overflow to +inf.
//    KEEP needs the finite-covariance certificate (finite quaternion, log-scales <= 20,
//    |J W| <= 1e8, lp in [0, 1e30]): then r_ref is finite or +inf, and mx + r >= mx >= x0.
__device__ __forceinline__ int classify(const CullArgs& a, const float* g) {
  const Cam& c = a.cam;
  const f3 t = to_camera(c, g[0], g[1], g[2]);
  const bool dok = t.z >= c.near_plane && t.z <= c.far_plane && t.z > 1e-9f;
  const float iz = __frcp_rn(t.z);  // == S(1) / t.z
  const float px = __fmul_rn(__fmul_rn(c.fx, t.x), iz), py = __fmul_rn(__fmul_rn(c.fy, t.y), iz);
  const float mx = __fadd_rn(px, c.cx), my = __fadd_rn(py, c.cy);
  const float afx = fabsf(c.fx) * iz, afy = fabsf(c.fy) * iz;
  // |j02| = fl(fl(|fx tx| iz) iz) <= |px| iz (1 + 2^-24) (render.hpp:119-120).
  const float j02u = fabsf(px) * iz * 1.00001f, j12u = fabsf(py) * iz * 1.00001f;
  const float r0 = __fmaf_rn(j02u, a.wn[2], afx * a.wn[0]), r1 = __fmaf_rn(j12u, a.wn[2], afy * a.wn[1]);
  const float smax = max_nan(max_nan(g[3], g[4]), g[5]);
  const float e = ex2_approx(smax * 1.44269504f);
  const float msq = __fmaf_rn(r1, r1, r0 * r0) * 1.0022f;  // (1.001 ex2 error)^2 x 1.0001 x margin
  const float r_ub = __fmaf_rn(3.0303f, sqrt_approx(__fmaf_rn(msq, e * e, 2.02f * a.lp)), 1e-6f);
  const bool outside = ((mx + r_ub < a.x0) | (mx - r_ub > a.x1) | (my + r_ub < a.y0) | (my - r_ub > a.y1)) &
                       (r_ub <= 1e15f);
  const bool inside = (mx >= a.x0) & (mx <= a.x1) & (my >= a.y0) & (my <= a.y1);
  int code = (!dok || outside) ? 0 : 2;
  if (code == 2 && inside) {  // keep needs the certificate (branch taken by inside-view rows)
    const bool cert = ((afx + j02u) * a.wmax <= 0.99e8f) & ((afy + j12u) * a.wmax <= 0.99e8f) &
                      (fabsf(g[6]) <= 3.0e38f) & (fabsf(g[7]) <= 3.0e38f) & (fabsf(g[8]) <= 3.0e38f) &
                      (fabsf(g[9]) <= 3.0e38f) & (smax <= 20.0f);
    if (cert) code = 1;
  }
  return (dok && a.all_exact) ? 2 : code;
}

#ifdef CULL_TRACE
__device__ unsigned long long g_cull_trace[4096][6];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(i) do { if (threadIdx.x == 0 && blockIdx.x < 4096) g_cull_trace[blockIdx.x][i] = gtime(); } while (0)
#else
#define TRACE(i) do {} while (0)
#endif

__device__ __forceinline__ unsigned long long pack_state(unsigned long long flag, unsigned epoch,
                                                         unsigned long long v) {
  return (flag << 62) | ((unsigned long long)(epoch & 0x3fffffffu) << 32) | (v & 0xffffffffull);
}

template <bool kTma>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) cull_kernel(const __grid_constant__ CullArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* buf = reinterpret_cast<float*>(smem_raw);  // [kStages][kTile * 10]
  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ uint32_t words[kMaxTiles * kWordsPerTile];
  __shared__ int32_t tpre[kMaxTiles];
  __shared__ __align__(8) float qrow[kDefer][kGeo];  // undecided rows, resolved after the last tile
  __shared__ int32_t qidx[kDefer];
  __shared__ int qn;
  __shared__ unsigned consumed[kStages];
  __shared__ int scan_tmp[kThreads / 32];
  __shared__ unsigned long long scan_tmp2[kThreads / 32];
  __shared__ long long base_s;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TRACE(0);
  if (tid == 0) {
    qn = 0;
    for (int i = 0; i < kStages; ++i) consumed[i] = 0;
  }
  const unsigned vid = blockIdx.x;
  const long long t_begin = (long long)vid * a.tiles_per_cta;
  const long long t_end = min((long long)a.ntiles, t_begin + a.tiles_per_cta);
  const int ntl = t_end > t_begin ? (int)(t_end - t_begin) : 0;
  const long long rowc = t_begin * kTile;

  auto issue = [&](int j) {  // start the copy of local tile j into stage j % kStages
    if (!kTma || j >= ntl) return;
    const long long tile = t_begin + j;
    const int s = j % kStages;
    if ((tile + 1) * kTile <= a.n) {
      // the stage's previous contents were read through the generic proxy; order those reads
      // before the async-proxy (TMA) write that refills it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&full_bar[s], kTileBytes);
      bulk_g2s(buf + (size_t)s * kTile * kGeo, a.geo + (size_t)tile * kTile * kGeo, kTileBytes, &full_bar[s]);
    } else {
      mbar_arrive(&full_bar[s]);  // partial last tile: loaded with plain loads below
    }
  };
  if (kTma && tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full_bar[s], 1);
    fence_mbar_init();
    for (int j = 0; j < kStages; ++j) issue(j);
  }
  __syncthreads();

  for (int j = 0; j < ntl; ++j) {
    const int s = kTma ? j % kStages : 0;
    const long long row0 = (t_begin + j) * kTile;
    const long long rem = a.n - row0;
    const int rows = rem < kTile ? (int)rem : kTile;
    float* tb = buf + (size_t)s * kTile * kGeo;
    if (kTma) mbar_wait(&full_bar[s], (uint32_t)((j / kStages) & 1));
    if (!kTma || rows < kTile) {  // generic strided rows or the partial last tile
      if (kTma) __syncthreads();   // warps drift without per-tile barriers: stage s must be free
      for (int e = tid; e < rows * kGeo; e += kThreads) {
        const int r = e / kGeo, col = e - r * kGeo;
        tb[e] = a.geo[(size_t)(row0 + r) * a.stride + col];
      }
      __syncthreads();
    }
    int cls[kTile / kThreads];
#pragma unroll
    for (int h = 0; h < kTile / kThreads; ++h) {
      const int r = tid + h * kThreads;
#ifdef CULL_EXP_TRIVIAL
      cls[h] = r < rows ? (tb[r * kGeo] > 0.9f ? 1 : 0) : 0;
#else
      cls[h] = r < rows ? classify(a, tb + r * kGeo) : 0;
#endif
    }
#pragma unroll
    for (int h = 0; h < kTile / kThreads; ++h) {
      const int r = tid + h * kThreads;
      bool kp = cls[h] == 1;
      // Undecided rows go to the deferred queue (warp-aggregated append); on overflow the
      // finding thread resolves its row on the spot.
      const unsigned um = __ballot_sync(0xffffffffu, cls[h] == 2);
      if (um) {
        int qb = 0;
        if (lane == 0) qb = atomicAdd(&qn, __popc(um));
        qb = __shfl_sync(0xffffffffu, qb, 0);
        if (cls[h] == 2) {
          const int slot = qb + __popc(um & ((1u << lane) - 1u));
          const float* g = tb + r * kGeo;
          if (slot < kDefer) {
#pragma unroll
            for (int c2 = 0; c2 < kGeo; ++c2) qrow[slot][c2] = g[c2];
            qidx[slot] = (int32_t)(row0 - rowc) + r;
          } else {
            kp = keep_exact(a, g);
          }
        }
      }
      const uint32_t wbits = __ballot_sync(0xffffffffu, kp);
      if (lane == 0) words[j * kWordsPerTile + h * (kThreads / 32) + warp] = wbits;
    }
    if (kTma && rows == kTile) {
      // No block barrier per tile: the last warp to finish with stage s refills it.
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(&consumed[s], 1u) == kThreads / 32 - 1) {
          __threadfence_block();  // acquire: every warp's reads of stage s precede the refill
          consumed[s] = 0;
          issue(j + kStages);
        }
      }
    } else {
      __syncthreads();  // stage s fully consumed
      if (tid == 0) issue(j + kStages);
    }
  }
  __syncthreads();
  TRACE(1);
  // Resolve the deferred rows with the exact reference predicate, all threads in parallel.
  const int nq = min(qn, kDefer);
  for (int q = tid; q < nq; q += kThreads)
    if (keep_exact(a, qrow[q])) atomicOr(&words[qidx[q] >> 5], 1u << (qidx[q] & 31));
  __syncthreads();
  TRACE(2);
#ifdef CULL_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 4096) g_cull_trace[blockIdx.x][5] = (unsigned long long)qn;
#endif
  // Exclusive prefix of kept counts over this CTA's tiles (ascending row order).
  int tc = 0;
  if (tid < ntl) {
#pragma unroll
    for (int w = 0; w < kWordsPerTile; ++w) tc += __popc(words[tid * kWordsPerTile + w]);
  }
  static_assert(kMaxTiles <= kThreads, "one thread per tile");
  int inc = tc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) scan_tmp[warp] = inc;
  __syncthreads();
  int wbase = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    const int v = scan_tmp[w];
    if (w < warp) wbase += v;
    total += v;
  }
  if (tid < ntl) tpre[tid] = wbase + inc - tc;
  // Look-back: publish this CTA's aggregate, then sum every predecessor's with all threads in
  // parallel (all loads in flight at once; CTAs are dispatched in blockIdx order and never wait
  // on successors, so the spin terminates).
  if (tid == 0) st_release(&a.state[vid], pack_state(kFlagAgg, a.epoch, (unsigned long long)total));
  unsigned long long part = 0;
  for (unsigned q = tid; q < vid; q += kThreads) {
    unsigned long long st;
    do {
      st = ld_relaxed(&a.state[q]);  // flag and value share one word: no acquire needed
    } while ((st >> 62) == 0 || ((st >> 32) & 0x3fffffffu) != a.epoch);
    part += st & 0xffffffffull;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) scan_tmp2[warp] = part;
  __syncthreads();
  if (tid == 0) {
    unsigned long long excl = 0;
    for (int w = 0; w < kThreads / 32; ++w) excl += scan_tmp2[w];
    base_s = (long long)excl;
    if (t_end == a.ntiles && ntl > 0) *a.count = (int64_t)(excl + (unsigned long long)total);
  }
  __syncthreads();
  const long long base = base_s;
  TRACE(3);
  // Scatter ascending ids (+ optional mask words): thread per mask word (16-lane segments = one tile),
  // segmented scan of the words' popcounts for the in-tile offset, then each thread writes its word's
  // set bits (few at the sparse keep rates of a view: no per-tile serial loop).
  static_assert(kWordsPerTile == 16, "segmented scan assumes 16 words per tile");
  for (int w0 = warp * 32; w0 < ntl * kWordsPerTile; w0 += kThreads) {
    const int w = w0 + lane;
    const int jt = w / kWordsPerTile;
    const bool okw = w < ntl * kWordsPerTile;
    uint32_t wv = okw ? words[w] : 0u;
    const long long wg = (rowc >> 5) + w;
    if (a.mask && okw && wg < a.nwords) a.mask[wg] = wv;
    const int pc = __popc(wv);
    int wi = pc;
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, wi, o, 16);
      if ((lane & 15) >= o) wi += v;
    }
    if (okw) {
      long long pos = base + tpre[jt] + (wi - pc);
      const long long id0 = rowc + (long long)w * 32;
      while (wv) {
        const int bit = __ffs(wv) - 1;
        wv &= wv - 1;
        a.ids[pos++] = (int32_t)(id0 + bit);
      }
    }
  }
  TRACE(4);
}

__global__ void expf_kernel(const float* x, float* y, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = gss_expf(x[i]);
}

// Per-workspace epoch (host side): look-back states of earlier calls never match the current one.
std::mutex g_epoch_mu;
std::unordered_map<const void*, unsigned> g_epochs;

unsigned next_epoch(const void* ws) {
  std::lock_guard<std::mutex> lk(g_epoch_mu);
  unsigned& e = g_epochs[ws];
  e = (e + 1) & 0x3fffffffu;
  if (e == 0) e = 1;  // a zero-filled workspace holds epoch 0 with flag 0
  return e;
}


}  // namespace

void cull_workspace_release(const void* ws) {
  std::lock_guard<std::mutex> lk(g_epoch_mu);
  g_epochs.erase(ws);
}

size_t cull_workspace_bytes(int64_t n) {
  const int64_t ntiles = ceil_div(n > 0 ? n : 1, kTile);
  return sizeof(WsHeader) + (size_t)ntiles * 8;
}

void cull(const float* geo, int64_t n, int64_t stride, const gss_camera* cam, const gss_viewport* vp, float lp,
          uint32_t* mask, int32_t* ids, int64_t* count, void* ws, size_t ws_bytes, cudaStream_t st) {
  require(n >= 0 && n <= INT32_MAX, "cull: n out of range (ids are int32)");
  require(stride >= kGeo, "cull: stride must be >= 10");
  require(cam && vp && ids && count, "cull: null argument");
  require(n == 0 || geo, "cull: null geo");
  if (n == 0) {
    GSS_CUDA(cudaMemsetAsync(count, 0, sizeof(int64_t), st));
    return;
  }
  const size_t need = cull_workspace_bytes(n);
  require(ws && ws_bytes >= need, "cull: workspace too small (gss_cull_workspace_bytes)");
  CullArgs a;
  static_assert(sizeof(Cam) == sizeof(gss_camera), "camera layout");
  std::memcpy(&a.cam, cam, sizeof(Cam));
  a.x0 = vp->x0; a.x1 = vp->x1; a.y0 = vp->y0; a.y1 = vp->y1;
  a.lp = lp;
  {
    float wmax = 0.0f;
    for (int r = 0; r < 3; ++r) {
      const double n2 = (double)cam->rot[3 * r] * cam->rot[3 * r] + (double)cam->rot[3 * r + 1] * cam->rot[3 * r + 1] +
                        (double)cam->rot[3 * r + 2] * cam->rot[3 * r + 2];
      a.wn[r] = (float)(std::sqrt(n2) * (1.0 + 1e-6));
      for (int k = 0; k < 3; ++k) wmax = std::max(wmax, std::fabs(cam->rot[3 * r + k]));
    }
    a.wmax = wmax * 1.000001f;
    a.all_exact = !(lp >= 0.0f && lp <= 1e30f);
  }
  a.geo = geo;
  a.n = n;
  a.stride = stride;
  a.ntiles = ceil_div(n, kTile);
  // Whole waves of co-resident CTAs with equal tile counts: a grid of k full waves (k the fewest
  // waves whose CTAs hold every tile at <= kMaxTiles each) instead of ceil(ntiles / kMaxTiles)
  // CTAs, whose last wave would run partly empty (40M rows: 611 CTAs = 1.4 waves of 444, i.e. two
  // CTA durations of 128 tiles; now 888 CTAs of 88 tiles = two durations of 88).
  const int64_t wave = (int64_t)sm_count() * kCtasPerSm;
  const int64_t waves = std::max<int64_t>(1, ceil_div(a.ntiles, wave * kMaxTiles));
  const int64_t ctas = std::min<int64_t>(a.ntiles, wave * waves);
  a.tiles_per_cta = (int)ceil_div(a.ntiles, ctas);
  const int grid = (int)ceil_div(a.ntiles, a.tiles_per_cta);
  a.mask = mask;
  a.nwords = ceil_div(n, 32);
  a.ids = ids;
  a.count = count;
  a.state = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + sizeof(WsHeader));
  a.epoch = next_epoch(ws);
  const bool tma = stride == kGeo && (reinterpret_cast<uintptr_t>(geo) % 16 == 0);
  if (tma) {
    const size_t smem = (size_t)kStages * kTileBytes;
    set_max_dynamic_smem(reinterpret_cast<const void*>(cull_kernel<true>), (int)smem);
    cull_kernel<true><<<grid, kThreads, smem, st>>>(a);
  } else {
    cull_kernel<false><<<grid, kThreads, (size_t)kTileBytes, st>>>(a);
  }
  GSS_LAUNCHED();
}

void expf_device(const float* x, float* y, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  expf_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(x, y, n);
  GSS_LAUNCHED();
}

}  // namespace gssd
