// Frustum cull + stream compaction: the B200 replacement of frustum_cull / cull_keep
// (render.hpp:243-260, with project_geo render.hpp:90-148 inside).
//
// Design:
//  * Persistent CTAs (2 per SM) claim 512-Gaussian tiles from a global ticket, in increasing
//    order. Each tile's 20 KB of geometric rows (N x 10 fp32, 40 B/row) is moved HBM->SMEM by the
//    TMA bulk-copy engine (cp.async.bulk + mbarrier) through a 4-stage ring, so ~160 KB per SM are
//    in flight while the SM classifies the previous tiles.
//  * Classification is exact but cheap for most Gaussians: the depth test and the projected
//    centre need ~40 fp32 ops; a centre inside the closed viewport with a provably finite
//    covariance is kept without computing the radius (mx + r >= mx >= x0 for r >= 0), and a
//    rigorous upper bound on the 3-sigma radius culls far-outside ones. Only the undecided rest
//    (Gaussians straddling the viewport border) run the full reference projection — queued in
//    SMEM so the exact path is warp-coherent. Every float op on the exact path follows the
//    reference order without FMA, expf is the glibc algorithm in fp64, so the kept set is
//    bit-identical to the CPU reference.
//  * Compaction: warp ballots build the 32-bit mask words, a warp scan gives the tile count,
//    and a decoupled look-back over per-tile states publishes the global offset, so the id list
//    comes out ascending in one pass (no second kernel).
#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "gss_math.cuh"

namespace gssd {
namespace {

constexpr int kTile = 512;
constexpr int kThreads = 256;
constexpr int kStages = 4;
constexpr int kGeo = 10;
constexpr uint32_t kTileBytes = kTile * kGeo * 4;  // 20480

constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

struct CullArgs {
  Cam cam;
  float x0, x1, y0, y1, lp;
  const float* geo;
  int64_t n, stride, ntiles;
  uint32_t* mask;
  int32_t* ids;
  int64_t* count;
  unsigned long long* state;
  unsigned int* ticket;
};

// cull_keep (render.hpp:243-251), exact.
__device__ __forceinline__ bool keep_exact(const CullArgs& a, const float* g) {
  const f3 t = to_camera(a.cam, g[0], g[1], g[2]);
  if (!(t.z >= a.cam.near_plane && t.z <= a.cam.far_plane)) return false;
  Proj p;
  f3 t2;
  if (!project_geo(a.cam, g, a.lp, p, t2)) return false;
  return p.mx + p.radius >= a.x0 && p.mx - p.radius <= a.x1 && p.my + p.radius >= a.y0 && p.my - p.radius <= a.y1;
}

// 0 = cull, 1 = keep, 2 = undecided (needs keep_exact). Decisions 0/1 are proven equal to
// keep_exact; see DESIGN.md §cull for the bound.
__device__ __forceinline__ int classify(const CullArgs& a, const float* g) {
  const Cam& c = a.cam;
  const float tz = cam_z(c, g[0], g[1], g[2]);
  if (!(tz >= c.near_plane && tz <= c.far_plane)) return 0;
  if (!(tz > 1e-9f)) return 0;
  const f3 t = to_camera(c, g[0], g[1], g[2]);
  const float iz = 1.0f / t.z;
  const float mx = c.fx * t.x * iz + c.cx;
  const float my = c.fy * t.y * iz + c.cy;
  // Rows of J*W exactly as project_geo forms them (render.hpp:119-123).
  const float j00 = c.fx * iz, j02 = -c.fx * t.x * iz * iz;
  const float j11 = c.fy * iz, j12 = -c.fy * t.y * iz * iz;
  const float* W = c.m;
  const float m00 = j00 * W[0] + j02 * W[6], m01 = j00 * W[1] + j02 * W[7], m02 = j00 * W[2] + j02 * W[8];
  const float m10 = j11 * W[3] + j12 * W[6], m11 = j11 * W[4] + j12 * W[7], m12 = j11 * W[5] + j12 * W[8];
  // fmaxf drops NaN operands, so finiteness is tested per component (a NaN compares false).
  const bool mfin = fabsf(m00) <= 1e8f && fabsf(m01) <= 1e8f && fabsf(m02) <= 1e8f && fabsf(m10) <= 1e8f &&
                    fabsf(m11) <= 1e8f && fabsf(m12) <= 1e8f;
  const bool qfin = fabsf(g[6]) <= 3.0e38f && fabsf(g[7]) <= 3.0e38f && fabsf(g[8]) <= 3.0e38f &&
                    fabsf(g[9]) <= 3.0e38f;
  // Finite-covariance certificate: finite quaternion, log-scales <= 20, |J W| <= 1e8, lp in
  // [0, 1e30]: then |cov| < 1e35, so lmax is finite or +inf and the radius is never NaN.
  const bool certified = mfin && qfin && (g[3] <= 20.0f) && (g[4] <= 20.0f) &&
                         (g[5] <= 20.0f) && (a.lp >= 0.0f) && (a.lp <= 1e30f) && (fabsf(mx) <= 1e30f) &&
                         (fabsf(my) <= 1e30f);
  if (!certified) return 2;
  if (mx >= a.x0 && mx <= a.x1 && my >= a.y0 && my <= a.y1) return 1;
  // Upper bound: r = 3 sqrt(lmax), lmax <= cov_a + cov_c <= (|m0|^2 + |m1|^2) max(es)^2 + 2 lp,
  // inflated for float rounding of the reference computation and for __expf's error.
  const float smax = fmaxf(fmaxf(g[3], g[4]), g[5]);
  const float e_ub = __expf(smax) * 1.001f;
  const float msq = (m00 * m00 + m01 * m01 + m02 * m02) + (m10 * m10 + m11 * m11 + m12 * m12);
  const float r_ub = 3.01f * sqrtf((msq * (e_ub * e_ub) + 2.0f * a.lp) * 1.01f) + 1e-6f;
  if (mx + r_ub < a.x0 || mx - r_ub > a.x1 || my + r_ub < a.y0 || my - r_ub > a.y1) return 0;
  return 2;
}

template <bool kTma>
__global__ void __launch_bounds__(kThreads, 2) cull_kernel(const __grid_constant__ CullArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* buf = reinterpret_cast<float*>(smem_raw);  // [kStages][kTile * 10]
  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ long long stage_tile[kStages];
  __shared__ uint8_t keep[kTile];
  __shared__ int16_t queue[kTile];
  __shared__ int qcount;
  __shared__ uint32_t words[kTile / 32];
  __shared__ uint32_t word_prefix[kTile / 32];
  __shared__ long long tile_base;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  auto issue = [&](int s) {  // thread 0 only: claim a tile, start its copy into stage s
    const long long tile = (long long)atomicAdd(a.ticket, 1u);
    stage_tile[s] = tile;
    if (kTma) {
      if (tile < a.ntiles && (tile + 1) * kTile <= a.n) {
        mbar_expect_tx(&full_bar[s], kTileBytes);
        bulk_g2s(buf + (size_t)s * kTile * kGeo, a.geo + (size_t)tile * kTile * kGeo, kTileBytes, &full_bar[s]);
      } else {
        mbar_arrive(&full_bar[s]);
      }
    }
  };

  if (tid == 0) {
    if (kTma) {
      for (int s = 0; s < kStages; ++s) mbar_init(&full_bar[s], 1);
      fence_mbar_init();
    }
    for (int s = 0; s < (kTma ? kStages : 1); ++s) issue(s);
  }
  __syncthreads();

  for (int it = 0;; ++it) {
    const int s = kTma ? it % kStages : 0;
    const uint32_t phase = kTma ? (uint32_t)((it / kStages) & 1) : 0u;
    const long long tile = stage_tile[s];
    if (tile >= a.ntiles) break;
    const long long row0 = tile * kTile;
    const long long rem = a.n - row0;
    const int rows = rem < kTile ? (int)rem : kTile;
    float* tb = buf + (size_t)s * kTile * kGeo;
    if (kTma) mbar_wait(&full_bar[s], phase);
    if (!kTma || rows < kTile) {  // generic strided rows or the partial last tile
      for (int e = tid; e < rows * kGeo; e += kThreads) {
        const int r = e / kGeo, col = e - r * kGeo;
        tb[e] = a.geo[(size_t)(row0 + r) * a.stride + col];
      }
      __syncthreads();
    }
    if (tid == 0) qcount = 0;
    __syncthreads();
#pragma unroll
    for (int h = 0; h < kTile / kThreads; ++h) {
      const int r = tid + h * kThreads;
      int cls = 0;
      if (r < rows) cls = classify(a, tb + r * kGeo);
      keep[r] = (uint8_t)(cls == 1);
      if (cls == 2) queue[atomicAdd(&qcount, 1)] = (int16_t)r;
    }
    __syncthreads();
    for (int q = tid; q < qcount; q += kThreads) {
      const int r = queue[q];
      keep[r] = (uint8_t)keep_exact(a, tb + r * kGeo);
    }
    __syncthreads();
    // Ballot into mask words (word j covers rows 32j .. 32j+31 of the tile).
#pragma unroll
    for (int h = 0; h < kTile / 32 / (kThreads / 32); ++h) {
      const int j = warp + h * (kThreads / 32);
      const uint32_t wbits = __ballot_sync(0xffffffffu, keep[j * 32 + lane] != 0);
      if (lane == 0) {
        words[j] = wbits;
        if (a.mask) {
          const long long widx = (row0 >> 5) + j;
          if (widx * 32 < a.n) a.mask[widx] = wbits;
        }
      }
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t cnt = lane < kTile / 32 ? (uint32_t)__popc(words[lane]) : 0u;
      uint32_t inc = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
      }
      if (lane < kTile / 32) word_prefix[lane] = inc - cnt;
      const unsigned long long total = __shfl_sync(0xffffffffu, inc, 31);
      if (lane == 0) {
        // Decoupled look-back (tiles are claimed in increasing order, so every predecessor
        // belongs to a CTA that is running or done: forward progress is guaranteed).
        unsigned long long excl = 0;
        if (tile == 0) {
          st_release(&a.state[0], kFlagInc | total);
        } else {
          st_release(&a.state[tile], kFlagAgg | total);
          long long p = tile - 1;
          while (true) {
            unsigned long long st;
            do {
              st = ld_acquire(&a.state[p]);
            } while ((st & ~kValMask) == 0);
            excl += st & kValMask;
            if ((st & ~kValMask) == kFlagInc) break;
            --p;
          }
          st_release(&a.state[tile], kFlagInc | (excl + total));
        }
        tile_base = (long long)excl;
        if (tile == a.ntiles - 1) *a.count = (int64_t)(excl + total);
      }
    }
    __syncthreads();
    // Scatter ascending ids.
#pragma unroll
    for (int h = 0; h < kTile / 32 / (kThreads / 32); ++h) {
      const int j = warp + h * (kThreads / 32);
      const uint32_t wbits = words[j];
      if (wbits & (1u << lane)) {
        const long long pos = tile_base + word_prefix[j] + __popc(wbits & ((1u << lane) - 1u));
        a.ids[pos] = (int32_t)(row0 + j * 32 + lane);
      }
    }
    __syncthreads();  // stage s, keep[], words[] free again
    if (tid == 0) issue(s);
    if (!kTma) __syncthreads();  // single stage: stage_tile[0] is re-read at the top
  }
}

__global__ void expf_kernel(const float* x, float* y, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = gss_expf(x[i]);
}

}  // namespace

size_t cull_workspace_bytes(int64_t n) {
  const int64_t ntiles = ceil_div(n > 0 ? n : 1, kTile);
  return (size_t)ntiles * 8 + 256;
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
  a.geo = geo;
  a.n = n;
  a.stride = stride;
  a.ntiles = ceil_div(n, kTile);
  a.mask = mask;
  a.ids = ids;
  a.count = count;
  a.state = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + 256);
  a.ticket = reinterpret_cast<unsigned int*>(ws);
  GSS_CUDA(cudaMemsetAsync(ws, 0, need, st));
  int dev = 0, sms = 148;
  GSS_CUDA(cudaGetDevice(&dev));
  GSS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const bool tma = stride == kGeo && (reinterpret_cast<uintptr_t>(geo) % 16 == 0);
  const int grid = (int)std::min<int64_t>(a.ntiles, (int64_t)sms * 2);
  if (tma) {
    const size_t smem = (size_t)kStages * kTileBytes;
    static bool attr = false;
    if (!attr) {
      GSS_CUDA(cudaFuncSetAttribute(cull_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = true;
    }
    cull_kernel<true><<<grid, kThreads, smem, st>>>(a);
  } else {
    const size_t smem = (size_t)kTileBytes;
    cull_kernel<false><<<grid, kThreads, smem, st>>>(a);
  }
  GSS_LAUNCHED();
}

void expf_device(const float* x, float* y, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  expf_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(x, y, n);
  GSS_LAUNCHED();
}

}  // namespace gssd
